"""Measured dense TF32 tensor-core peak of this B200, the denominator of the fp32 mode's
roofline (the fp32-mode fraction had no measured peak behind it).

Same method as the driver's MEASURED_PEAKS.json bf16 figures: cuBLAS `torch.matmul` of
8192^3 fp32 matrices with TF32 tensor cores allowed (2 * N^3 flops), best of 10 timed
individually (burst), and back to back for 4 s (sustained, the power-capped clock). The fp32
mode (K1f) issues three kind::tf32 MMAs per product (hi*hi + hi*lo + lo*hi), so its ceiling in
algorithmic fp32 flops is tf32 / 3; both are written. Prints one JSON line; run under gpurun:
    python scripts/tf32_peak.py > profiles/r02/tf32_peak.json
"""
import json
import time

import torch


def main():
    n = 8192
    dev = torch.device("cuda", 0)
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn((n, n), device=dev)
    b = torch.randn((n, n), device=dev)
    flops = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        time.sleep(0.2)  # idle gap: each launch starts at the burst clock
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = flops / (best / 1e3) / 1e12
    t_end = time.time() + 4.0
    reps, e0 = 0, torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        for _ in range(8):
            torch.matmul(a, b)
        reps += 8
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained = flops * reps / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({
        "tf32_tflops": burst, "tf32_tflops_sustained": sustained,
        "fp32_mode_ceiling_tflops": burst / 3, "fp32_mode_ceiling_tflops_sustained": sustained / 3,
        "gpu": torch.cuda.get_device_name(dev), "torch": torch.__version__,
        "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32 tensor cores): best of 10 "
               "with idle gaps (burst) and back to back for 4 s (sustained); fp32 mode = 3 tf32 "
               "MMAs per product"}))


if __name__ == "__main__":
    main()
