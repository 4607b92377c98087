import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: large CPU-side reference builds")


def _gpu_available() -> bool:
    try:
        from paper_2605_06472_b200 import api

        return api.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _gpu_available():
        pytest.fail("GPU test selected but no sm_100 device / libpbkv.so unavailable (no CPU fallback exists)")
    return True
