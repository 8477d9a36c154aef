"""Error hierarchy of the retrieval backend.

Mirrors the reference's convention (pkg/src/teola_sim/errors.py:7-67): every error is a
``TeolaError`` subclass carrying the CLI exit code it maps to. ``DeviceError`` is new: it
surfaces CUDA failures of the B200 path (the reference has no device).
"""

from __future__ import annotations


class TeolaError(Exception):
    exit_code = 1


class CapacityExceeded(TeolaError):
    """Batch load is empty or exceeds engine / arena capacity (errors.py:34-35)."""


class EmptyProfile(TeolaError):
    """Engine latency table has no breakpoints (errors.py:30-31)."""


class UnknownNode(TeolaError):
    pass


class DuplicateQueryId(TeolaError):
    pass


class NonQuiescent(TeolaError):
    """Event loop exceeded its safety bound without quiescing (errors.py:46-47)."""


class ConfigParse(TeolaError):
    exit_code = 2


class ProfileMissing(TeolaError):
    exit_code = 4


class DeviceError(TeolaError):
    """CUDA / NCCL failure, or the native library is missing on a GPU host."""

    exit_code = 6


# C-ABI status code (include/tsv.h) -> exception class.
STATUS_ERRORS = {
    1: CapacityExceeded,
    2: ConfigParse,
    3: DeviceError,
    4: ConfigParse,
}
