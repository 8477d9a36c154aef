"""Achievable HBM read bandwidth probe: reduce a 10 GB bf16 buffer (read-only traffic)."""
import torch
x = torch.empty(5 << 30, dtype=torch.bfloat16, device="cuda").normal_()
for f in (lambda: x.sum(dtype=torch.float32), lambda: x.view(-1, 1024).amax(dim=1)):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(5)]; b.record(); torch.cuda.synchronize()
    print("read GB/s", x.numel() * 2 * 5 / (a.elapsed_time(b) * 1e-3) / 1e9)
