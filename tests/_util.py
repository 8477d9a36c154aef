"""Shared helpers for the parity tests (test infrastructure)."""

from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def to_dev_bf16(x: np.ndarray, device):
    """bf16-rounded float32 numpy matrix -> CUDA bfloat16 tensor with identical values."""
    import torch

    bits = orc.bf16_bits(x).view(np.int16)
    return torch.from_numpy(bits.copy()).to(device).view(torch.bfloat16)


def from_dev(t) -> np.ndarray:
    import torch

    if isinstance(t, np.ndarray):
        return t
    if t.dtype == torch.bfloat16:
        return orc.bf16_to_f32(t.view(torch.int16).cpu().numpy().view(np.uint16))
    return t.cpu().numpy()


def assert_topk(g_s, g_i, q, c, k, tol=1e-3, id_offset=0, oracle=None):
    problems = orc.check_topk(from_dev(g_s), from_dev(g_i), q, c, k, tol, id_offset=id_offset,
                              oracle=oracle)
    assert not problems, "\n".join(problems[:20])
