"""CPU: pins the plain-C oracle port (oracle/bp_oracle.c) against the reference's golden vectors
(tests/golden/*.npz, produced by the reference itself) and, when present, against the
reference library directly. No GPU needed."""
import numpy as np
import pytest

from helpers import Lim, assert_bitwise, case_problem, golden


@pytest.mark.parametrize("name", ["prop_accept", "prop_cont", "prop_thr0"])
def test_port_matches_golden_propagation(oracle_built, name):
    from oracle.bind import PortProblem
    lim = Lim(abs_threshold=0.0, rel_threshold=0.0) if name == "prop_thr0" else Lim()
    for idx, c in enumerate(golden(name)):
        p = case_problem(c)
        pp = PortProblem(p)
        root = p.root_bounds()
        b, inf, st, rounds, cr = pp.propagate(root, lim=lim)
        info = c["inc_info"]
        assert [int(inf), st, rounds, cr] == list(info), f"{name}[{idx}] inc info"
        assert_bitwise(b, c["inc_bounds"], f"{name}[{idx}] inc bounds")
        lf = Lim(**vars(lim))
        lf.incremental = False
        b, inf, st, rounds, cr = pp.propagate(root, lim=lf)
        assert [int(inf), st, rounds, cr] == list(c["full_info"]), f"{name}[{idx}] full info"
        assert_bitwise(b, c["full_bounds"], f"{name}[{idx}] full bounds")
        act, nmin, nmax = pp.compute_activities(root)
        assert_bitwise(act, c["act"], f"{name}[{idx}] act")
        assert np.array_equal(nmin, c["nmin"]) and np.array_equal(nmax, c["nmax"])
        tb, tinf, changed, crossed = pp.tighten_bounds(root, False, act, nmin, nmax, lim=lim)
        assert_bitwise(tb, c["t_bounds"], f"{name}[{idx}] tighten bounds")
        assert changed == list(c["t_changed"])
        assert [int(tinf), crossed] == list(c["t_info"])


def test_port_matches_golden_probing(oracle_built):
    from oracle.bind import PortProblem
    for idx, c in enumerate(golden("probe")):
        p = case_problem(c)
        pp = PortProblem(p)
        root = p.root_bounds()
        hdr = c["hdr"].reshape(-1, 7)
        doff = c["doff"]
        for v in range(p.n_vars):
            kind, br = pp.probe_variable(root, v)
            for side in range(2):
                feas, dv, dl, du = br[side]
                if kind == 0:  # no spec: default entry, both branches "feasible", no deltas
                    assert hdr[v][3 + side] == 1 and hdr[v][5 + side] == 0
                    continue
                j = 2 * v + side
                assert int(feas) == hdr[v][3 + side], f"probe[{idx}] v{v} side{side} feasible"
                sl = slice(doff[j], doff[j + 1])
                assert list(dv) == list(c["dvar"][sl])
                assert_bitwise(dl, c["dlo"][sl], f"probe[{idx}] lo")
                assert_bitwise(du, c["dup"][sl], f"probe[{idx}] up")


def test_port_matches_reference_on_c1(oracle_built):
    """Large mixed instance (configs[0] shape) — port vs the reference library, bitwise."""
    from oracle.bind import PortProblem, Ref, RefProblem, ref_propagate
    from paper_2510_20499_b200 import synth
    if not Ref.available():
        pytest.skip("reference library not built here")
    p = synth.c1()
    b1, i1, s1, r1, c1 = ref_propagate(RefProblem.from_def(p), p.root_bounds())
    b2, i2, s2, r2, c2 = PortProblem(p).propagate(p.root_bounds())
    assert (i1, s1, r1, c1) == (i2, s2, r2, c2)
    assert_bitwise(b1, b2, "C1 bounds")


def test_branch_spec_known_answers(oracle_built):
    """test_probing.cpp:15-64: [0,10] -> [0,4]/[5,10]; [0,inf) -> {0}/[1,inf); binary {0}/{1}."""
    import ctypes as C
    from oracle.bind import Port
    s = np.zeros(4)
    assert Port.lib().orc_make_branch_spec(0.0, 10.0, s.ctypes.data_as(C.c_void_p)) == 1
    assert list(s) == [0.0, 4.0, 5.0, 10.0]
    assert Port.lib().orc_make_branch_spec(0.0, np.inf, s.ctypes.data_as(C.c_void_p)) == 2
    assert list(s) == [0.0, 0.0, 1.0, np.inf]
    assert Port.lib().orc_make_branch_spec(0.0, 1.0, s.ctypes.data_as(C.c_void_p)) == 1
    assert s[1] == 0.0 and s[2] == 1.0
    assert Port.lib().orc_make_branch_spec(-np.inf, np.inf, s.ctypes.data_as(C.c_void_p)) == 0
    assert Port.lib().orc_make_branch_spec(3.0, 3.0, s.ctypes.data_as(C.c_void_p)) == 0
