import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.join(ROOT, "tests")
if TESTS not in sys.path:  # test helpers (wan_weights, peer_worker)
    sys.path.insert(0, TESTS)

_PARITY = {}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test scheduled without a GPU")
    return torch.device("cuda:0")


@pytest.fixture
def parity_log(request):
    """record measured errors of a parity test: parity_log(key=value, ...). With
    SPX_PARITY_LOG=<path> the session writes every record there as JSON (the committed
    profiles/parity_*.json come from such a run)."""
    def log(**kw):
        _PARITY.setdefault(request.node.nodeid, {}).update(
            {k: (float(v) if isinstance(v, (int, float)) or hasattr(v, "__float__") else v)
             for k, v in kw.items()})
    return log


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("SPX_PARITY_LOG")
    if path and _PARITY:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(_PARITY, f, indent=1, sort_keys=True)
