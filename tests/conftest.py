import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_cache = {}


def golden(name: str):
    if name not in _cache:
        _cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
    return _cache[name]


def golden_bcsc(d, prefix):
    """Reference-layout matrix (oracle.Bcsc) stored in a golden file."""
    import oracle
    rows, cols, b = (int(v) for v in d[f"{prefix}_meta"])
    return oracle.Bcsc(rows, cols, b, d[f"{prefix}_col_ptr"], d[f"{prefix}_row_idx"],
                       d[f"{prefix}_values"])
