"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/tsv.h
declares; the product path has no CPU fallback. No compute call needs a GPU here."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    hdr = (ROOT / "include" / "tsv.h").read_text()
    return sorted(set(re.findall(r"TSV_API\s+[\w\s\*]+?\b(tsv_\w+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("tsv_search", "tsv_search_segmented", "tsv_rerank", "tsv_merge_topk",
                 "tsv_index_create", "tsv_index_append", "tsv_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2407_00326_b200 import _native

    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_native.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tsv_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_code():
    from paper_2407_00326_b200 import _native

    out = subprocess.run(["cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA, tcgen05.ld
        assert mnemonic in sass, mnemonic
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_abi_version_and_error_channel():
    from paper_2407_00326_b200 import _native

    lib = _native.load()
    assert lib.tsv_abi_version() == 1
    assert isinstance(lib.tsv_last_error(), bytes)
    assert lib.tsv_launch_count() >= 0


def test_argument_errors_map_to_teola_errors_without_a_gpu():
    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.errors import CapacityExceeded, ConfigParse, TeolaError

    lib = _native.load()
    # null index / empty merge are rejected before touching the device
    with pytest.raises(ConfigParse):
        _native.check(lib.tsv_search(None, None, 0, 1, 1, 0, 0, 0, None, None, None))
    with pytest.raises(CapacityExceeded):
        _native.check(lib.tsv_merge_topk(None, None, 0, 1, 1, 1, 0, None, None, None))
    with pytest.raises(ConfigParse):
        _native.check(lib.tsv_normalize_rows(None, 0, 1, 7, 1, None, None))
    assert issubclass(ConfigParse, TeolaError) and ConfigParse.exit_code == 2


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2407_00326_b200.errors import DeviceError
    from paper_2407_00326_b200.index import DeviceIndex

    with pytest.raises(DeviceError):
        DeviceIndex(64, 10, device=0)
    from paper_2407_00326_b200.index import normalize_rows

    with pytest.raises(DeviceError):
        normalize_rows(torch.zeros((2, 64)))


def test_missing_library_fails_loudly(tmp_path):
    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.errors import DeviceError

    saved = _native._lib
    try:
        _native._lib = None
        with pytest.raises(DeviceError):
            _native.load(tmp_path / "nope.so")
    finally:
        _native._lib = saved


def _build_c_example(out_dir):
    import shutil
    import subprocess

    root = Path(__file__).resolve().parents[1]
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    cuda = Path("/usr/local/cuda")
    exe = Path(out_dir) / "tsv_example"
    lib = root / "paper_2407_00326_b200" / "lib"
    cmd = [cc, "-O2", "-Wall", "-Werror", "-I", str(root / "include"), "-I", str(cuda / "include"),
           str(root / "examples" / "tsv_example.c"), "-L", str(lib), "-ltsv",
           "-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{lib}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_builds_against_the_abi(tmp_path):
    """examples/tsv_example.c uses only include/tsv.h + libtsv.so + the CUDA runtime: the C ABI
    is usable without Python or torch (a cgo / JNI / N-API binding links the same way)."""
    if not (Path("/usr/local/cuda") / "include" / "cuda_runtime.h").exists():
        pytest.skip("CUDA headers not present")
    _build_c_example(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import subprocess

    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "64/64 queries found their row first" in r.stdout
