import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")


def opts_to_ref(opts):
    """The product's BlockSolverOptions and the oracle harness's struct share
    one layout (include/elastodyn_b200.h, oracle/ref_harness.cpp)."""
    from oracle import ref
    return ref.SolverOptions.from_buffer_copy(bytes(opts))


@pytest.fixture(scope="session")
def oracle():
    from oracle import ref
    ref.lib()
    return ref


_PARITY = []


@pytest.fixture(scope="session")
def parity_log():
    """Collects per-case parity figures (counts, max history deviation, x error);
    written as JSON to $PARITY_LOG at the end of the session (committed under
    profiles/ as the evidence behind the GPU parity claims)."""
    return _PARITY


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PARITY_LOG")
    if path and _PARITY:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(_PARITY, f, indent=1, default=float)
