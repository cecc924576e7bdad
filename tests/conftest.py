import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def device():
    import paper_2412_09584_b200 as bp

    return bp.Device(0)


@pytest.fixture(autouse=True)
def _rollout_path_reset(request):
    """A failing test that forced a rollout kernel must not leave it forced for the next."""
    yield
    if "device" in request.fixturenames:
        request.getfixturevalue("device").rollout_path("auto")
