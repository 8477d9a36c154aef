"""Summarise an ncu report: key counters + top stall sites (used to write profiles/*.md)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "gpc__cycles_elapsed.max.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res = []
    for vals in rows[2:]:
        res.append({h: (u, v) for h, u, v in zip(rows[0], rows[1], vals)})
    return res


def stalls(path, top=15):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = rows[2:]
    i_src = hdr.index("Source")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data)
    best = sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]
    return tot, [(r[i_src].strip(), float(r[i_s] or 0) / tot, r[i_e]) for r in best]


if __name__ == "__main__":
    p = sys.argv[1]
    for k in raw(p):
        for key in KEYS:
            if key in k:
                print(f"{key}: {k[key][1]} {k[key][0]}")
    tot, st = stalls(p)
    print(f"stall samples: {tot:.0f}")
    for src, frac, ex in st:
        print(f"  {frac * 100:5.1f}%  exec={ex:>10}  {src[:90]}")
