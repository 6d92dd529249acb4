import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size parity cases")


def golden_lines(name):
    """Non-comment lines of a golden fixture (each fixture cites its source in its header)."""
    out = []
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line)
    return out


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def full_grid(G, D, batch=0):
    """Every cell of a G^D grid (fully occupied: C = Z^D restricted to the box)."""
    idx = np.stack(np.meshgrid(*[np.arange(G)] * D, indexing="ij"), axis=-1).reshape(-1, D)
    return np.concatenate([idx, np.full((idx.shape[0], 1), batch)], axis=1).astype(np.int32)


def pytest_collection_modifyitems(config, items):
    """GPU tests get a per-test timeout (pytest-timeout, thread method): a kernel that hangs
    ends the run with a stack dump instead of blocking it until an outer limit."""
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(600, method="thread"))
