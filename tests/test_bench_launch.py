"""bench.py's N-rank launch on CPU: `bench.py --gpus N` with no external launcher starts N
ranks itself (torch.distributed.run re-exec), every rank joins one process group, and the
shard plan covers the corpus exactly once; a launcher that starts a different number of
ranks than --gpus is refused (the scaling run must measure N GPUs)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None, timeout=180):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", **(env_extra or {}))
    env.pop("WORLD_SIZE", None)
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout, env=env)


def _json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_gpus_2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json(r.stdout)
    assert d["n_gpus"] == 2 and d["world_size_from_group"] == 2 and d["spawned"]
    assert d["shards"] == [[0, 5_000_000], [5_000_000, 10_000_000]]
    assert d["config"]["shard_rows"] == 10_000_000 // 2
    assert d["config"]["parallelism"] == "corpus-shard x2"


def test_gpus_3_ragged_shards_cover_corpus():
    r = _run(["--gpus", "3", "--dry-run", "--rows", "1000"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json(r.stdout)
    assert d["n_gpus"] == 3 and d["world_size_from_group"] == 3
    assert d["shards"][0][0] == 0 and d["shards"][-1][1] == 1000
    assert all(a[1] == b[0] for a, b in zip(d["shards"], d["shards"][1:]))


def test_world_mismatch_refused():
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0
    assert "refusing" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_nccl_more_gpus_than_present_fails_clearly():
    import torch

    n = torch.cuda.device_count()
    env = dict(os.environ)
    env.pop("BENCH_DIST_BACKEND", None)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n + 2), "--steps", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 2
    assert f"needs {n + 2} GPUs" in r.stderr
