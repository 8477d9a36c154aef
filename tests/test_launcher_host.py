"""Host-side checks of the CUDA-graph wrappers (no GPU needed)."""

from __future__ import annotations

import pytest
import torch

from paper_2407_00326_b200.errors import ConfigParse
from paper_2407_00326_b200.launcher import _same_shape


def test_same_shape_accepts_the_captured_shape():
    _same_shape(torch.zeros(16, 8), torch.zeros(16, 8), "queries")


@pytest.mark.parametrize("shape", [(1, 8), (15, 8), (16, 4), (16,)])
def test_same_shape_rejects_broadcastable_and_other_shapes(shape):
    # copy_ would broadcast (1, 8) into the captured (16, 8) buffer without complaint
    with pytest.raises(ConfigParse):
        _same_shape(torch.zeros(shape), torch.zeros(16, 8), "queries")
