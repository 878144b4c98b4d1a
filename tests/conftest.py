import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

# The reference's parallel_for (parallel.hpp:100-129) can destroy its mutex / condition variable
# while its last worker is about to lock them (seen once as a segfault inside the reference's
# propagation_round in this suite). The reference is thread-count independent by design, so the
# parity tests run it on one thread (read once, at its first parallel_for): the checker must not
# crash. bench.py's CPU baselines still use every host thread.
os.environ.setdefault("PULSE_THREADS", "1")


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
