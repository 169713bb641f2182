import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "ref: needs the compiled reference oracle/_ref")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure)."""
    from oracle import oracle

    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def dfx():
    import paper_2507_13833_b200 as d

    return d


def pytest_terminal_summary(terminalreporter):
    """Print the achieved maximum relative error of every loss scalar checked this session (tests/helpers.py)."""
    try:
        from tests.helpers import ACHIEVED
    except Exception:  # noqa: BLE001
        return
    if not ACHIEVED:
        return
    terminalreporter.write_sep("-", "achieved max relative error of loss scalars (bound 1e-5, plain relative)")
    for k in sorted(ACHIEVED):
        err, where = ACHIEVED[k]
        terminalreporter.write_line(f"{k:>12s}  {err:.3e}   ({where[:110]})")
