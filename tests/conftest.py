import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
if str(ROOT / "tests") not in sys.path:
    sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session", autouse=True)
def _guarded_allocations():
    """HW_TEST_GUARD=1|2 runs the whole GPU suite with the library's guarded device allocations
    (option "guard": every buffer between unmapped pages, start- or end-aligned), so an
    out-of-bounds access of any kernel faults instead of passing unnoticed.  The variable is read
    here, by the tests; the library itself reads no environment."""
    g = int(os.environ.get("HW_TEST_GUARD", "0"))
    if g:
        import paper_2310_00236_b200 as hw

        hw.set_option("guard", g)
    yield


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


@pytest.fixture
def hwopt():
    """Set library kernel-path options (hw_set_option) for one test; restored afterwards."""
    import paper_2310_00236_b200 as hw

    saved = {}

    def set_(**kw):
        for k, v in kw.items():
            if k not in saved:
                saved[k] = hw.get_option(k)
            hw.set_option(k, v)

    yield set_
    for k, v in saved.items():
        hw.set_option(k, v)
