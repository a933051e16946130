import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfram.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def rng():
    import numpy as np
    return np.random.Generator(np.random.PCG64(12345))


@pytest.fixture
def errlog(request):
    """Record an observed parity error next to its tolerance: printed (pytest -s / -rA) and, when
    FRAM_PARITY_LOG names a file, appended to it as one JSON line per record."""
    import json

    def rec(quantity, observed, tol, **extra):
        d = {"test": request.node.nodeid, "quantity": quantity, "observed": float(observed), "tol": float(tol),
             **extra}
        print("PARITY", json.dumps(d))
        path = os.environ.get("FRAM_PARITY_LOG")
        if path:
            with open(path, "a") as f:
                f.write(json.dumps(d) + "\n")
        return observed

    return rec
