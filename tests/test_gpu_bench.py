"""bench.py contract on the GPU: one JSON line with the driver's keys, and the N>1 sharded path
(two ranks sharing this GPU over gloo; the driver's scaling run uses NCCL across GPUs) finds
every planted neighbour with its global id."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline",
        "gpu_launches", "clocks"}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_one_gpu_line(cuda):
    r = subprocess.run([sys.executable, "bench.py", "--rows", "1000000", "--steps", "8",
                        "--warmup", "3", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["planted_top1"] == 1.0
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 1024 * 1024 * 2
    assert d["roofline"]["bound"] in ("tensor", "hbm") and d["roofline"]["frac"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("world,exchange", [(2, "p2p"), (4, "p2p"), (2, "nccl")])
def test_bench_ranks_sharded(cuda, world, exchange):
    """p2p: fused peer exchange + merge kernel; nccl: the collective all-gather + K4 merge path
    (run over gloo here, since the ranks share one GPU)."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                        "--master-port", str(_port()), "bench.py", "--gpus", str(world),
                        "--rows", "1000000", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0", "--exchange", exchange], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == world and d["config"]["shard_rows"] == 1_000_000 // world
    assert d["config"]["exchange"] == exchange
    assert d["planted_top1"] == 1.0  # global ids survive the exchange + merge
    if exchange == "p2p":  # the first fused exchange matched NCCL all-gather + K4 on every rank
        assert d["exchange_used"] == "p2p" and d["exchange_check"]


def test_bench_spawns_its_own_ranks(cuda):
    """`bench.py --gpus 2` with no launcher starts 2 ranks itself and reports them (ranks share
    this GPU over gloo; on an 8-GPU node the same command runs one NCCL rank per GPU)."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--rows", "1000000",
                        "--steps", "4", "--warmup", "3", "--min-warmup-s", "0"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["world"]["process_group"] == 2
    assert d["world"]["spawned_by_bench"] and d["config"]["shard_rows"] == 500_000
    assert d["planted_top1"] == 1.0
