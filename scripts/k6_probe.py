"""K6 (fused peer all-gather + merge) latency with every rank's kernel in flight at once.

G ranks are driven from one process on one GPU (LocalPeerGroup: tsv_peer_attach, no IPC), each
on its own stream. A gate (a short device sleep on a side stream, all rank streams wait on its
event) lets every rank's launch be queued before any starts, so the time is gate -> last rank
done, without host launch skew. The exchange moves the same bytes as on an NVSwitch node;
what is missing here is NVLink's latency (~1-2 us per remote store batch) — the protocol,
the merge and the in-kernel waits are measured. K4 alone (the merge of the NCCL path's
gathered [G, B, k] lists) is timed beside it.

    python scripts/k6_probe.py  -> one line per (G, B, k)
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import merge_topk  # noqa: E402
from paper_2407_00326_b200.sharded import LocalPeerGroup  # noqa: E402


def lists(G, B, k, dev, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    s = torch.sort(torch.rand((G, B, k), generator=g, device=dev), dim=2, descending=True)[0]
    i = torch.arange(G * B * k, device=dev, dtype=torch.int32).reshape(G, B, k)
    return s.contiguous(), i


def main():
    dev = torch.device("cuda", 0)
    reps = 30
    for G in (2, 4, 8):
        for B, k in ((1024, 10), (1024, 100), (16, 10)):
            grp = LocalPeerGroup([0] * G, B, k)
            grp.set_timeout_ms(5000)
            s, i = lists(G, B, k, dev, G * 1000 + k)
            streams = [torch.cuda.Stream(dev) for _ in range(G)]
            side = torch.cuda.Stream(dev)
            outs = [grp.allgather_merge(r, s[r], i[r], k, stream=streams[r]) for r in range(G)]
            torch.cuda.synchronize()
            times = []
            for _ in range(reps):
                gate = torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(side):
                    torch.cuda._sleep(200_000)  # ~100 us: every launch below is queued first
                    gate.record(side)
                ends = []
                for r in range(G):
                    streams[r].wait_event(gate)
                    grp.allgather_merge(r, s[r], i[r], k, stream=streams[r], out=outs[r])
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(streams[r])
                    ends.append(e)
                torch.cuda.synchronize()
                times.append(max(gate.elapsed_time(e) for e in ends) * 1000)
            grp.status()
            ref_s, ref_i = merge_topk(s, i, k)
            same = all(torch.equal(outs[r][1], ref_i) for r in range(G))
            # K4 alone over the gathered lists (what the NCCL path runs after its all-gather)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                merge_topk(s, i, k)
            a.record()
            for _ in range(reps):
                merge_topk(s, i, k)
            b.record()
            torch.cuda.synchronize()
            times.sort()
            print(json.dumps({"G": G, "B": B, "k": k, "k6_us_p50": round(times[len(times) // 2], 2),
                              "k6_us_min": round(times[0], 2), "k6_us_max": round(times[-1], 2),
                              "bytes_pushed_per_rank": (G - 1) * B * k * 8,
                              "k4_merge_us": round(a.elapsed_time(b) / reps * 1000, 2),
                              "equal_to_k4": same}), flush=True)
            grp.close()


if __name__ == "__main__":
    main()
