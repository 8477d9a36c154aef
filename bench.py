#!/usr/bin/env python
"""Benchmark of the retrieval hot path: vector-search queries/s on a 10M x 1024 bf16 corpus.

Workload (BASELINE.json metric, config C4 at k=10): B=1024 queries per step against a
10,000,000 x 1024 bf16 corpus (cosine = inner product over L2-normalised rows), top-10 per
query. With --gpus N the corpus is sharded N ways (strong scaling: total work fixed); each
rank runs the fused scan + top-k (K1) and the range merge (K4) on its shard, and the per-rank
top-k lists are exchanged and merged by one kernel that pushes them into the peers' buffers
over NVLink (K6; --exchange nccl: NCCL all-gather + K4 instead). One step = one batch of B
queries through that path.

value : queries/s with queries already resident in HBM (device time, max over ranks).
e2e   : the same through the public API with host buffers — every step copies the pinned
        query batch host->device and the (scores, ids) result device->host.
Warm-up: the W steps, then more untimed steps until --min-warmup-s (1 s) of load has passed, so
the timed steps run at the settled power-capped clock; the K timed steps of each region then
run in 4 blocks, alternating which region goes first, with no idle gap.
The corpus (20.5 GB) is far larger than L2, so no explicit L2 flush is needed.

--impl reference times the reference CPU path (the C oracle port, all host threads) on the
same config, each step a bounded sample of the corpus scaled to the full corpus.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--storage", choices=("bf16", "bf16_tiled", "f32"), default="bf16",
                    help="f32 = fp32 mode (3xTF32 tensor-core products, scores within 1e-5)")
    ap.add_argument("--min-warmup-s", type=float, default=1.0,
                    help="keep warming up until this much load time has passed (power-capped "
                         "clocks settle), in addition to the --warmup steps")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the bounded cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-step-s", type=float, default=4.0,
                    help="--impl reference: CPU seconds per step before the corpus is sampled "
                         "(the whole corpus is searched when it fits)")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="N>1: fused peer all-gather + merge over NVLink, or NCCL all-gather + K4")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks, agree on the shard plan and print it (no kernels); "
                         "checks the N-rank launch without a GPU")
    return ap.parse_args()


# ---------------------------------------------------------------------- N-rank launch
def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1) started without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (one GPU per rank), forwarding the
    arguments; rank 0's JSON line is this process's output. A box with fewer than N GPUs is
    refused up front (NCCL cannot put two ranks on one GPU) unless BENCH_DIST_BACKEND=gloo."""
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "nccl" and args.impl == "ours" and not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, found "
                  f"{have} (NCCL runs one rank per GPU)", file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, BENCH_SPAWNED="1", OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    print(f"bench.py: starting {args.gpus} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr,
          flush=True)
    return subprocess.run(cmd, env=env, cwd=str(ROOT)).returncode


def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def check_world(args, world: int) -> None:
    """Every line is measured on exactly --gpus ranks: a mismatch is an error, never a line."""
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} "
                         f"rank(s); refusing to report a {world}-rank measurement as "
                         f"{args.gpus}")


def run_dry(args) -> int:
    """The N-rank plan without kernels: ranks join the process group, each reports its shard,
    rank 0 prints the agreed plan (world size as the process group sees it)."""
    import torch.distributed as dist

    from paper_2407_00326_b200.sharded import shard_range

    rank, world, _ = dist_env()
    check_world(args, world)
    group_world = 1
    shards = [shard_range(args.rows, 0, 1)]
    if world > 1:
        dist.init_process_group(os.environ.get("BENCH_DIST_BACKEND", "nccl"))
        group_world = dist.get_world_size()
        got = [None] * group_world
        dist.all_gather_object(got, (rank, *shard_range(args.rows, rank, world)))
        shards = [(lo, hi) for _, lo, hi in sorted(got)]
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "world_size_from_group": group_world,
                          "spawned": os.environ.get("BENCH_SPAWNED") == "1",
                          "shards": shards, "config": _config(args)}),
              flush=True)
    return 0


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples nvidia-smi clocks / throttle reasons every 200 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index  # CUDA ordinal, or the GPU UUID (robust to CUDA_VISIBLE_DEVICES)
        self.rows: list[list[str]] = []
        self.first = 0  # rows before this index were sampled before the timed region
        self.proc = None
        self.thread = None

    def mark(self):
        """Start of the timed region: later statistics use only samples taken after this."""
        self.first = len(self.rows)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = []
        sm_max = None
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows[self.first:]:
            try:
                sm.append(float(r[0]))
                sm_max = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": sm_max, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def simulated_reference_ms(load: float):
    """The reference's modelled latency for one `vdb-search0` batch of `load` queries: its
    hand-written profile table (pkg/src/teola_sim/profiles/default.json:47-70, captured in
    tests/golden/ref_profiles.json) through engines.latency (engines.py:85-109)."""
    try:
        from paper_2407_00326_b200 import engines as E

        prof = json.loads((ROOT / "tests" / "golden" / "ref_profiles.json").read_text())
        es = E.EngineSet.from_dict(prof["default"]["profiles"])
        return E.latency(es["vdb-search0"], float(load))
    except Exception:  # informative only
        return None


# ---------------------------------------------------------------------- CPU baseline
def host_corpus(n: int, dim: int, seed: int = 0):
    """n x dim seeded N(0, 1) rows, L2-normalised, as bf16 bit patterns (uint16) on the host,
    generated in 128K-row chunks with torch's multi-threaded CPU kernels (the reference arm's
    corpus; the CPU has no access to the device-generated one)."""
    import numpy as np
    import torch

    out = np.empty((n, dim), dtype=np.uint16)
    g = torch.Generator().manual_seed(seed)
    for a in range(0, n, 1 << 17):
        b = min(n, a + (1 << 17))
        x = torch.randn((b - a, dim), generator=g)
        x = (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16)
        out[a:b] = x.view(torch.int16).numpy().view(np.uint16)
    return out


def cpu_sample(dim: int, batch: int, k: int, target_s: float, rows_dev=None,
               max_rows: int | None = None):
    """A bounded sample of the workload for the CPU reference path: `batch` queries against
    the first n_s corpus rows, n_s sized for ~target_s of CPU work per search (at most the whole
    corpus, max_rows). Returns (queries, rows, n_s, threads, oracle variant)."""
    import numpy as np

    from oracle import c_oracle
    from oracle import oracle as orc

    lib = c_oracle.load()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(1)
    q = orc.normalize_rows(rng.standard_normal((batch, dim), dtype=np.float32))
    qb = orc.bf16_bits(q)
    probe_rows = 32768
    cb = (_host_rows(rows_dev, probe_rows) if rows_dev is not None
          else host_corpus(probe_rows, dim))
    time_cpu(qb, cb, k, threads)  # first call: thread pool, AMX permission
    t = time.perf_counter()
    c_oracle.search(qb, cb, k, nthreads=threads)
    dt = max(time.perf_counter() - t, 1e-4)
    n_s = int(max(probe_rows * target_s / dt, 8192))
    if max_rows is not None:
        n_s = min(n_s, max_rows)
    if n_s != max_rows:
        n_s -= n_s % 1024
    cb = (_host_rows(rows_dev, n_s) if rows_dev is not None else host_corpus(n_s, dim))
    return qb, cb, n_s, threads, lib.variant


def _host_rows(rows_dev, n):
    import numpy as np
    import torch

    n = min(n, rows_dev.shape[0])
    return rows_dev[:n].view(torch.int16).cpu().numpy().view(np.uint16)


def torch_cpu_baseline(qb, cb, k, threads, n_total, seconds=3.0):
    """Informative second CPU path: torch on the host cores, bf16 GEMM
    (oneDNN; AMX where the CPU has it) + torch.topk, on the same bounded sample."""
    import numpy as np
    import torch

    try:
        torch.set_num_threads(threads)
        q = torch.from_numpy(qb.view(np.int16).copy()).view(torch.bfloat16)
        c = torch.from_numpy(cb.view(np.int16).copy()).view(torch.bfloat16)
        n_s = c.shape[0]
        def run():  # 128K-row chunks keep the score block at 0.5 GB
            vals, ids = [], []
            for a in range(0, n_s, 1 << 17):
                v, i = torch.topk(torch.matmul(q, c[a:a + (1 << 17)].t()).float(), k, dim=1)
                vals.append(v)
                ids.append(i + a)
            v, j = torch.topk(torch.cat(vals, 1), k, dim=1)
            return v, torch.gather(torch.cat(ids, 1), 1, j)

        reps, total = 0, 0.0
        while reps == 0 or total < seconds:
            t = time.perf_counter()
            run()
            total += time.perf_counter() - t
            reps += 1
        dt = total / reps
        return {"value": qb.shape[0] / (dt * n_total / n_s), "unit": "queries/s",
                "cores": threads,
                "sample": f"torch {torch.__version__} bf16 matmul + topk (128K-row chunks) on "
                          f"the same {n_s} rows, {reps} repetitions"}
    except Exception as exc:  # informative only
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def time_cpu(qb, cb, k, threads):
    from oracle import c_oracle

    t = time.perf_counter()
    c_oracle.search(qb, cb, k, nthreads=threads)
    return time.perf_counter() - t


# ---------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference CPU path (the C oracle port: AMX-BF16 tiles where the host has them, else
    AVX-512 / AVX2; all host threads) on the same metric and config. Each step searches the
    batch over the whole corpus when that fits ~--ref-step-s of CPU time, else over the first
    rows_timed rows, with the step time scaled to the full corpus (`extrapolated`)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    qb, cb, n_s, threads, variant = cpu_sample(args.dim, args.batch, args.k,
                                               target_s=args.ref_step_s, max_rows=args.rows)
    for _ in range(args.warmup):
        time_cpu(qb, cb, args.k, threads)
    total = 0.0
    for _ in range(args.steps):
        total += time_cpu(qb, cb, args.k, threads)
    scale = args.rows / n_s
    ms_per_step = total / args.steps * scale * 1000.0
    value = args.batch / (ms_per_step / 1000.0)
    sample = (f"{args.batch} queries x {'all' if n_s == args.rows else 'first'} {n_s} of the "
              f"{args.rows}-row corpus per step"
              + (f" (time scaled x{scale:.2f})" if n_s != args.rows else "")
              + f"; C oracle {variant}, fp32 accumulate, OpenMP")
    line = {
        "impl": "reference",
        "metric": "vector-search queries/s (10Mx1024 corpus, k=10)",
        "value": value, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) rows, L2-normalised)",
        "config": _config(args),
        "rows_timed": n_s, "extrapolated": n_s != args.rows,
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "port",
                         "variant": variant, "cpu_model": cpu_model(), "sample": sample,
                         "rows_timed": n_s, "extrapolated": n_s != args.rows},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(args, shard_rows=None):
    """The workload, from the arguments alone: both arms (ours and --impl reference) print the
    identical dict for the same command line."""
    if shard_rows is None:  # rank 0's shard (paper_2407_00326_b200.sharded.shard_range)
        shard_rows = args.rows // args.gpus
    return {
        "workload": f"C4/metric: flat inner-product (cosine) search, {args.rows}x{args.dim} "
                    f"{getattr(args, 'storage', 'bf16')} corpus, batch {args.batch}, k={args.k}",
        "storage": getattr(args, "storage", "bf16"),
        "rows": args.rows, "dim": args.dim, "batch": args.batch, "k": args.k,
        "shard_rows": shard_rows, "parallelism": f"corpus-shard x{args.gpus}",
        "exchange": args.exchange if args.gpus > 1 else None,
        "l2": "inputs larger than L2 (corpus streamed from HBM every step)",
    }


# ---------------------------------------------------------------------- our arm
def build_shard(idx_cls, rows, dim, lo, hi, device, storage="bf16"):
    """Corpus rows [lo, hi) of the global seeded corpus; chunk c of 2^20 rows is drawn from a
    generator seeded with c, so the corpus is identical for every sharding."""
    import torch

    chunk = 1 << 20
    idx = idx_cls(dim, hi - lo, metric="cosine", device=device.index, storage=storage)
    c0 = lo // chunk
    while c0 * chunk < hi:
        a, b = c0 * chunk, min(rows, (c0 + 1) * chunk)
        g = torch.Generator(device=device).manual_seed(1000 + c0)
        block = torch.randn((b - a, dim), generator=g, device=device)
        s, e = max(a, lo), min(b, hi)
        idx.append(block[s - a:e - a].contiguous())
        del block
        c0 += 1
    torch.cuda.synchronize(device)
    return idx


def make_queries(N, D, B, dev, normalize_rows):
    """SURVEY.md §8(d) query mix: the first B/2 queries are corpus rows + N(0, 0.05^2) noise
    (planted neighbours; the row is regenerated from its chunk's seed), the rest fresh N(0, 1);
    all L2-normalised. Returns (queries [B, D] bf16, planted global ids [B/2])."""
    import torch

    g = torch.Generator(device=dev).manual_seed(1)
    q = torch.randn((B, D), generator=g, device=dev)
    n_pl = B // 2
    gid = torch.randint(0, N, (n_pl,), generator=g, device=dev)
    noise = torch.randn((n_pl, D), generator=g, device=dev) * 0.05
    chunk = 1 << 20
    ids = gid.tolist()
    for c in sorted({i // chunk for i in ids}):
        a, b = c * chunk, min(N, (c + 1) * chunk)
        block = torch.randn((b - a, D), generator=torch.Generator(device=dev).manual_seed(1000 + c),
                            device=dev)
        sel = [j for j, i in enumerate(ids) if i // chunk == c]
        q[sel] = block[torch.tensor([ids[j] - a for j in sel], device=dev)] + noise[sel]
        del block
    return normalize_rows(q), gid


def p2p_self_check(sharded, q, k, dev, backend) -> None:
    """First sharded step through the fused peer exchange (K6), checked against the NCCL
    all-gather + K4 merge of the same per-rank lists: the ranks agree (all-reduce) to keep p2p
    only if every rank's exchange completed and matched bit for bit; otherwise every rank
    switches to NCCL and the JSON line says why. Peer waits are bounded (10 s here) so a peer
    mapping that does not deliver surfaces as an error instead of a hang."""
    import torch
    import torch.distributed as dist

    from paper_2407_00326_b200.errors import TeolaError

    ok, why = 1, ""
    try:
        s_p, i_p = sharded.search(q, k)  # creates the peer group (collective) on first use
        if sharded.exchange == "p2p" and sharded._peer is not None:
            sharded._peer.set_timeout_ms(10_000)
            s_p, i_p = sharded.search(q, k)
            torch.cuda.synchronize(dev)
            sharded._peer.status()
            sharded._peer.set_timeout_ms(60_000)
        s_p, i_p = s_p.clone(), i_p.clone()
    except (TeolaError, RuntimeError) as exc:
        ok, why = 0, f"{type(exc).__name__}: {exc}"
        s_p = i_p = None
    saved = sharded.exchange
    sharded.exchange = "nccl"
    s_n, i_n = sharded.search(q, k)
    torch.cuda.synchronize(dev)
    if ok and saved == "p2p" and not (torch.equal(s_p, s_n) and torch.equal(i_p, i_n)):
        ok, why = 0, "fused exchange result differs from NCCL all-gather + merge"
    flag = torch.tensor([ok], dtype=torch.int32, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 1 and saved == "p2p":
        sharded.exchange = "p2p"
        sharded.p2p_checked = "first step bit-identical to NCCL all-gather + merge on every rank"
    elif saved == "p2p":
        sharded.p2p_error = why or "another rank's p2p self-check failed"


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows
    from paper_2407_00326_b200.sharded import ShardedSearch, shard_range

    rank, world, local = dist_env()
    check_world(args, world)
    # NCCL's own log stays on (to a file per rank, so stdout keeps exactly one JSON line)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/bench_nccl.{os.getpid()}.log")
    # BENCH_DIST_BACKEND=gloo (test only): run the N>1 code path with every rank on the GPUs
    # present (ranks share a GPU when there are fewer GPUs than ranks; NCCL refuses that)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl" or local >= torch.cuda.device_count():
        # gloo test runs share a GPU; a launcher that gives every rank its own
        # CUDA_VISIBLE_DEVICES shows each process one device
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _native.load()
    group_world = dist.get_world_size() if world > 1 else 1
    check_world(args, group_world)
    # every rank's device (distinct physical GPUs under NCCL), gathered for the JSON line
    me = f"{torch.cuda.get_device_name(dev)} {torch.cuda.get_device_properties(dev).uuid}"
    device_names = [me]
    if world > 1:
        device_names = [None] * world
        dist.all_gather_object(device_names, me)

    B, D, k, N = args.batch, args.dim, args.k, args.rows
    lo, hi = shard_range(N, rank, world)
    idx = build_shard(DeviceIndex, N, D, lo, hi, dev, storage=args.storage)

    q_dev, planted = make_queries(N, D, B, dev, normalize_rows)
    q_host = torch.empty((B, D), dtype=torch.bfloat16, pin_memory=True)
    q_host.copy_(q_dev)
    s_host = torch.empty((B, k), dtype=torch.float32, pin_memory=True)
    i_host = torch.empty((B, k), dtype=torch.int32, pin_memory=True)
    sharded = ShardedSearch(idx, N, rank=rank, world=world, exchange=args.exchange)
    if world > 1 and sharded.exchange == "p2p":
        p2p_self_check(sharded, q_dev, k, dev, backend)

    def step(q):
        return sharded.search(q, k)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # The clock sampler starts before the warm-up, so the timed blocks follow the warm-up with
    # no idle gap (an idle pause would hand the first block burst clocks); only samples taken
    # inside the timed region are reported.
    try:  # nvidia-smi numbers GPUs physically; the UUID names this process's device exactly
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:  # noqa: BLE001
        smi_id = local
    clocks = ClockSampler(smi_id)
    clocks.start()
    for _ in range(args.warmup):
        step(q_dev)
    # Keep warming up (more untimed steps) until --min-warmup-s of load has passed and every
    # rank's sampler has produced a sample (at most 3 s more): under the 1 kW cap the SM clock
    # settles during the first ~0.5-1 s of load, and both timed regions should see the settled
    # clock rather than whatever is left of the burst. The decision is collective because a
    # sharded step is.
    t_w = time.time()
    warm_extra = 0
    torch.cuda.synchronize(dev)
    while max_over_ranks(float(time.time() - t_w < 3.0 + args.min_warmup_s and (
            time.time() - t_w < args.min_warmup_s
            or (clocks.proc is not None and not clocks.rows)))) > 0:
        for _ in range(4):  # synchronise every few steps only: no idle gaps in the warm-up
            step(q_dev)
        torch.cuda.synchronize(dev)
        warm_extra += 4
    barrier()

    def device_region(steps):
        """Queries resident in HBM; returns (ms, launches, scan ms, scan launches)."""
        idx.set_timing(True)
        idx.scan_time()
        n0 = _native.launch_count()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(steps):
            step(q_dev)
        ev1.record()
        barrier()
        launches = _native.launch_count() - n0
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        scan_ms, scan_launches = idx.scan_time()
        idx.set_timing(False)
        return ms, launches, scan_ms, scan_launches

    # End-to-end region (host buffers, copies inside). Every step copies its query batch
    # host->device and its (scores, ids) device->host; the copies run on a copy stream with
    # double-buffered device/host buffers, so batch i+1's upload and batch i-1's download
    # overlap batch i's search (the way a serving loop feeds the index).
    copy = torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)
    q_bufs = [torch.empty_like(q_dev), torch.empty_like(q_dev)]
    h_s = [s_host, torch.empty_like(s_host).pin_memory()]
    h_i = [i_host, torch.empty_like(i_host).pin_memory()]

    # double-buffered results (world == 1 writes them in place; world > 1 returns new tensors)
    r_s = [torch.empty((B, k), dtype=torch.float32, device=dev) for _ in range(2)]
    r_i = [torch.empty((B, k), dtype=torch.int32, device=dev) for _ in range(2)]

    def e2e_region(steps):
        up = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        fetched = [torch.cuda.Event(), torch.cuda.Event()]
        barrier()
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(comp)
        copy.wait_stream(comp)
        with torch.cuda.stream(copy):
            q_bufs[0].copy_(q_host, non_blocking=True)
            up[0].record(copy)
        for step_i in range(steps):
            b = step_i & 1
            if step_i + 1 < steps:  # prefetch the next batch while this one is searched
                nb = b ^ 1
                with torch.cuda.stream(copy):
                    if step_i >= 1:
                        copy.wait_event(freed[nb])
                    q_bufs[nb].copy_(q_host, non_blocking=True)
                    up[nb].record(copy)
            comp.wait_event(up[b])
            if step_i >= 2:  # result buffer b is free once download step_i - 2 finished
                comp.wait_event(fetched[b])
            s, i = sharded.search(q_bufs[b], k, out=(r_s[b], r_i[b]))
            freed[b].record(comp)
            done[b].record(comp)
            with torch.cuda.stream(copy):
                copy.wait_event(done[b])
                h_s[b].copy_(s, non_blocking=True)
                h_i[b].copy_(i, non_blocking=True)
                fetched[b].record(copy)
        comp.wait_stream(copy)
        ev3.record(comp)
        barrier()
        return max_over_ranks(ev2.elapsed_time(ev3))

    # The two timed regions alternate in blocks, each bracketed by a barrier + synchronize, in
    # the order device|e2e, e2e|device, device|e2e, e2e|device: under the 1 kW cap the clock
    # falls during the first ~0.3 s of load, so timing one region after the other hands the
    # first one the higher clocks (measured: 16.0 vs 17.2 ms/step for the same work,
    # whichever runs first).
    clocks.mark()
    nblk = 4 if args.steps >= 8 else 1
    sizes = [args.steps // nblk + (1 if j < args.steps % nblk else 0) for j in range(nblk)]
    dev_ms = e2e_ms = scan_ms = 0.0
    launches = scan_launches = 0
    blocks = []
    for j, n_blk in enumerate(sizes):
        if j % 2:
            e_ms = e2e_region(n_blk)
            e2e_ms += e_ms
        d_ms, d_l, s_ms, s_l = device_region(n_blk)
        dev_ms += d_ms
        launches += d_l
        scan_ms += s_ms
        scan_launches += s_l
        if not j % 2:
            e_ms = e2e_region(n_blk)
            e2e_ms += e_ms
        blocks.append((n_blk, round(d_ms / n_blk, 3), round(e_ms / n_blk, 3)))
    if os.environ.get("BENCH_VERBOSE"):
        print(f"blocks (steps, device ms/step, e2e ms/step): {blocks}", file=sys.stderr)
    clk = clocks.stop()
    # sanity check on the last e2e result: every planted query finds its corpus row first
    last_ids = h_i[(sizes[-1] - 1) & 1]
    planted_top1 = float((last_ids[: planted.numel(), 0] == planted.cpu().to(torch.int32))
                         .float().mean())

    peaks, peak_src = load_peaks()
    # per-step device time of the scan kernel(s): k > 32 adds a 1/16-sample seeding pass, which
    # counts as time but not as algorithmic work
    avg_scan_ms = scan_ms / max(args.steps, 1)
    n_local = hi - lo
    flops = 2.0 * B * n_local * D
    bytes_alg = n_local * D * 2 + B * D * 2 + B * k * 8
    achieved_tf = flops / (avg_scan_ms / 1000.0) / 1e12
    achieved_gbs = bytes_alg / (avg_scan_ms / 1000.0) / 1e9
    peak_tf = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
    peak_tf_sus = float(peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"]))
    f32_peak_src = None
    if args.storage == "f32":
        # fp32 mode: 3 tf32 MMAs per product, so the algorithmic-fp32-flop ceiling is the
        # measured cuBLAS TF32 peak / 3 (scripts/tf32_peak.py -> profiles/tf32_peak.json);
        # without that file, the nominal tf32 = bf16 / 2 relation (bf16 / 6)
        # The tensor pipe's dense tf32 rate is half its bf16 rate; cuBLAS's own TF32 GEMM
        # reaches less than that on this part (722 / 605 TFLOP/s burst / sustained vs bf16
        # 1629 / 1374), so the ceiling is the larger of the two per regime.
        tp = ROOT / "profiles" / "tf32_peak.json"
        cublas = json.loads(tp.read_text()) if tp.exists() else None
        peak_tf = max(peak_tf / 6.0, cublas["fp32_mode_ceiling_tflops"] if cublas else 0.0)
        peak_tf_sus = max(peak_tf_sus / 6.0,
                          cublas["fp32_mode_ceiling_tflops_sustained"] if cublas else 0.0)
        f32_peak_src = ("max(measured bf16 / 2, measured cuBLAS TF32 GEMM "
                        "[profiles/tf32_peak.json]) / 3 tf32 MMAs per product")
        bytes_alg = n_local * D * 8 + B * D * 4 + B * k * 8
    peak_bw = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
    # The timed kernels run after >= 1 s of continuous load, i.e. at the settled power-capped
    # clock: the sustained bf16 figure is the denominator for that (MEASURED_PEAKS: "burst for a
    # kernel timed alone, sustained for a kernel timed inside a long step"); with
    # --min-warmup-s below 1 the burst figure is used. Both fractions are reported.
    long_step = args.min_warmup_s >= 1.0
    peak_tc = peak_tf_sus if long_step else peak_tf
    t_tc = flops / (peak_tc * 1e12)
    t_bw = bytes_alg / (peak_bw * 1e9)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            key = f"{n_local}x{D}xB{B}k{k}"
            traffic = tj.get(key)
        except (ValueError, OSError):
            traffic = None
    if t_tc >= t_bw:
        roof = {"bound": "tensor", "achieved": achieved_tf, "peak": peak_tc, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tc, "traffic": traffic,
                "frac_of_burst": achieved_tf / peak_tf,
                "frac_of_sustained": achieved_tf / peak_tf_sus}
    else:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak_bw, "unit": "GB/s",
                "frac": achieved_gbs / peak_bw, "traffic": traffic}
    # the north star's per-kernel pair: both utilisations, whichever bounds
    roof.update({"tensor_tflops": achieved_tf, "tensor_frac": achieved_tf / peak_tc,
                 "hbm_gbs": achieved_gbs, "hbm_frac": achieved_gbs / peak_bw,
                 "corpus_bytes_frac_at_peak": achieved_gbs / peak_bw})
    roof.update({"kernel": "scan_topk_pair_kernel / scan_topk_kernel (K1, tcgen05 fused IP + "
                           "top-k)",
                 "avg_launch_ms": avg_scan_ms, "scan_ms_per_step": avg_scan_ms,
                 "launches_timed": scan_launches,
                 "algorithmic_flops_per_launch": flops,
                 "algorithmic_bytes_per_launch": bytes_alg,
                 "peak_source": (f"{peak_src} (MEASURED_PEAKS.json "
                                 f"{'sustained' if long_step else 'burst'} bf16 / copy GB/s)"
                                 if peak_src == "measured" else "fallback (B200_PROFILING.md)")
                 + (f"; fp32 mode: {f32_peak_src}" if args.storage == "f32" else "")})

    value = B * args.steps / (dev_ms / 1000.0)
    e2e_value = B * args.steps / (e2e_ms / 1000.0)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        qb, cb, n_s, threads, variant = cpu_sample(D, B, k, min(args.cpu_seconds, 3.0),
                                                   rows_dev=idx.data(),
                                                   max_rows=min(N, 2_000_000))
        # repeat the bounded sample until ~cpu_seconds of CPU work were timed (the sample
        # size is capped to keep the host copy of the rows small)
        reps, total = 0, 0.0
        while reps == 0 or total < args.cpu_seconds:
            total += time_cpu(qb, cb, k, threads)
            reps += 1
        dt = total / reps
        cpu_qps = B / (dt * N / n_s)
        cpu = {"value": cpu_qps, "unit": "queries/s", "cores": threads, "kind": "port",
               "variant": variant, "cpu_model": cpu_model(), "rows_timed": n_s,
               "extrapolated": n_s != N,
               "sample": f"{B} queries x first {n_s} corpus rows (of {N}); time scaled by "
                         f"{N / n_s:.1f}; C oracle ({variant}), fp32 accumulate, OpenMP; "
                         f"{reps} repetitions, {total:.1f} s measured",
               "torch_cpu": torch_cpu_baseline(qb, cb, k, threads, N)}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": "vector-search queries/s (10Mx1024 corpus, k=10)",
            "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_extra_steps": warm_extra,
            "world": {"ranks": world, "process_group": group_world, "backend": backend if world > 1 else None,
                      "spawned_by_bench": os.environ.get("BENCH_SPAWNED") == "1",
                      "devices": device_names,
                      "nccl_log": os.environ.get("NCCL_DEBUG_FILE") if world > 1 else None},
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (3xTF32)" if args.storage == "f32" else "bf16",
            "data": "synthetic (seeded N(0,1) rows; queries: B/2 planted = corpus row + "
                    "N(0,0.05^2), B/2 fresh N(0,1); L2-normalised on device)",
            "planted_top1": planted_top1,
            "simulated_reference_ms": simulated_reference_ms(B),
            "config": _config(args),
            "exchange_used": (None if world == 1 else sharded.exchange
                              + (f" (p2p unavailable: {sharded.p2p_error})"
                                 if sharded.p2p_error else "")),
            "exchange_check": getattr(sharded, "p2p_checked", None),
            "e2e": {"value": e2e_value, "unit": "queries/s",
                    "h2d_bytes_per_step": B * D * 2, "d2h_bytes_per_step": B * k * 8,
                    "ms_per_step": e2e_ms / args.steps,
                    "copies": "pinned host buffers, H2D/D2H on a copy stream overlapping the "
                              "previous/next batch (double-buffered)",
                    "path": "ShardedSearch.search -> DeviceIndex.search (C ABI tsv_search) "
                            "[+ tsv_peer_allgather_merge over NVLink (or NCCL all-gather + "
                            "tsv_merge_topk) when sharded], pinned host buffers"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
