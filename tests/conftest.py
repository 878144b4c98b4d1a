import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libbp.so")
    config.addinivalue_line("markers", "slow: large-instance test")


@pytest.fixture(scope="session")
def oracle_built():
    """Builds oracle/_ref (port always; reference shim when /root/reference exists)."""
    from oracle import bind
    if not bind.PORT_SO.exists() or (not bind.REF_SO.exists()
                                     and Path("/root/reference/proj/include/pulse").is_dir()):
        bind.build()
    return bind
