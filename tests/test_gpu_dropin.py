"""GPU: the C++ drop-in (include/pulse_gpu.hpp) against the unmodified reference, side by side in
one C++ process (tests/cpp/test_dropin.cpp, built by oracle/Makefile into oracle/_ref/test_dropin
from the reference headers; the binary travels with the repo snapshot). Every pulse:: hot-path
function — compute_activities, tighten_bounds, propagate, prioritize_probe_vars, probe_variable,
build_cache, assemble_bulk_warm_start, parallel_propagate, propagation_round — is compared bitwise."""
import subprocess

import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu
BIN = ROOT / "oracle" / "_ref" / "test_dropin"


def test_cpp_dropin_matches_reference():
    assert BIN.exists(), "oracle/_ref/test_dropin not built (run __graft_entry__.build() where /root/reference exists)"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
