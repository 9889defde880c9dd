import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")


@pytest.fixture(scope="session")
def gpu_lib():
    from paper_2112_13169_b200 import _native

    lib = _native.load()
    if lib.vxm_device_count() == 0:
        pytest.fail("gpu test ran without a visible sm_100 device (no CPU fallback exists)")
    return lib
