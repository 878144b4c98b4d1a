"""Shared test utilities: golden-case loading, bitwise comparisons, instance streams."""
from __future__ import annotations

import math
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(GOLDEN))

from golden_io import unpack  # noqa: E402
from paper_2510_20499_b200.problem import problem_from_csr  # noqa: E402


@dataclass
class Lim:
    max_rounds: int = 64
    time_limit: float = math.inf
    abs_threshold: float = 1e-7
    rel_threshold: float = 1e-4
    incremental: bool = True


def golden(name):
    return unpack(GOLDEN / f"{name}.npz")


def case_problem(c):
    n, m = int(c["n"][0]), int(c["m"][0])
    return problem_from_csr(n, m, c["row_start"], c["row_col"], c["row_val"], c["var_lower"],
                            c["var_upper"], c["is_integer"], c["cons_lower"], c["cons_upper"],
                            apply_integral=False, validate=False)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    """IEEE == (the reference's own criterion, test_propagation.cpp:239) AND identical bits
    (sign of zero included)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    eq = (a == b) | (np.isnan(a) & np.isnan(b))
    if not eq.all():
        i = int(np.nonzero(~eq)[0][0])
        raise AssertionError(f"{what}: {int((~eq).sum())} value mismatches, first at {i}: {a[i]!r} vs {b[i]!r}")
    bb = bits(a) == bits(b)
    if not bb.all():
        i = int(np.nonzero(~bb)[0][0])
        raise AssertionError(f"{what}: {int((~bb).sum())} sign-of-zero mismatches, first at {i}: {a[i]!r} vs {b[i]!r}")
