"""The C-ABI library loads and exports every symbol include/corridor_b200.h declares (no GPU needed)."""

import re
from pathlib import Path

from paper_2504_10783_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "corridor_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\**\s+\**(ez_[a-z0-9_]+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, name


def test_abi_version_and_device_count_without_gpu():
    lib = N.load_library()
    assert lib.ez_abi_version() == 3
    assert lib.ez_device_count() >= 0


def test_status_mapping():
    import pytest

    from paper_2504_10783_b200 import errors as E

    for code, exc in ((1, E.DimensionMismatch), (2, E.EmptyChord), (3, E.SeedOutside), (4, E.GradientUndefined),
                      (5, E.SegmentInCollision), (6, E.SeedOutsideDomain), (7, E.GridMismatch), (8, ValueError),
                      (9, E.NativeError), (10, NotImplementedError)):
        with pytest.raises(exc):
            E.raise_for_status(code, "x")
    E.raise_for_status(0)


def test_gpu_entry_points_fail_loudly_without_device():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2504_10783_b200 import fixtures as fx
    from paper_2504_10783_b200.errors import NativeError

    with pytest.raises(NativeError):
        fx.arm3_world().checker().check_batch([[1.0, 0.0, 0.0]])
