import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA render path)")
    config.addinivalue_line("markers", "slow: full-size configuration")


@pytest.fixture(scope="session", autouse=True)
def _native_built():
    """Build the in-tree native libraries (incremental) and the oracle before any test."""
    from paper_2501_17792_b200.build import build, build_oracle

    build()
    build_oracle()
    yield


def has_gpu() -> bool:
    try:
        import ctypes as C

        from paper_2501_17792_b200 import native as N

        n = C.c_int(0)
        N.gscg().gscg_device_count(C.byref(n))
        return n.value > 0
    except Exception:
        return False
