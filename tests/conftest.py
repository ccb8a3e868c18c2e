import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")
    # the sm_100a library cross-compiles without a GPU; build it once if this checkout lacks it
    lib = ROOT / "paper_2304_06835_b200" / "libens.so"
    if not lib.exists():
        from paper_2304_06835_b200 import _build
        _build.build()


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
