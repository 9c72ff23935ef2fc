import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "reference: needs the reference package mounted at /root/reference")


def pytest_collection_modifyitems(config, items):
    if REFERENCE_SRC.exists():
        return
    skip = pytest.mark.skip(reason="/root/reference not mounted (build container only)")
    for item in items:
        if "reference" in item.keywords:
            item.add_marker(skip)
