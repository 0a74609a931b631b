"""Test configuration: `gpu` marks tests that need a B200 (run with -m gpu)."""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer parity runs")


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


@pytest.fixture(scope="session")
def lib_built():
    """Build (if stale) and load the C-ABI library."""
    from paper_2201_05555_b200 import _build, _lib
    _build.build()
    return _lib.load()


@pytest.fixture
def parity_report(request):
    """rec(**values): append the measured errors of a parity test as one JSON
    line to $PICROM_PARITY_REPORT (no-op when unset) -- the numbers DESIGN.md
    quotes come from this file (profiles/)."""
    import json
    path = os.environ.get("PICROM_PARITY_REPORT")

    def rec(**kv):
        if path:
            row = {"test": request.node.name}
            row.update({k: (float(v) if not isinstance(v, (list, str)) else v) for k, v in kv.items()})
            with open(path, "a") as f:
                f.write(json.dumps(row) + "\n")

    return rec
