"""Shared test configuration.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU (``pytest -m "not gpu"``).
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def inflate_index():
    z = golden("inflate.npz")
    return z, json.loads(str(z["index"]))
