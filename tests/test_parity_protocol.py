"""The margin-aware parity protocol itself (tests/parity.py track_parity),
checked on the CPU with the oracle standing in for both sides.

A GPU/oracle difference in an iteration's advantage set A = {k : E_k < E_base} is
accepted only as a *tie* -- the oracle's fitness-decision margin (ora_track_ex emargin) below
E_TIE -- and then the oracle is re-run *shadowed* with the other side's membership.  These tests
pin the machinery: forcing the natural membership changes nothing, a genuine tie is shadowed and
accepted, a difference with a large margin is rejected."""
import dataclasses

import numpy as np
import pytest

import oracle
from tests.fixtures import f_track_inputs
from tests.parity import E_TIE, selection, track_parity


def _ftrack():
    f = f_track_inputs()
    ov = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    return f, ov


def _fake_gpu(ov, f, params, force, tie_low=()):
    """A stand-in 'GPU': the oracle with a forced membership.  tie_low = ((iteration, k), ...): the
    tied particles the fake counted as members report E_k one ulp below E_base in that iteration
    (as a real GPU's rounding would), so its E_k are consistent with its membership."""
    def run(iters):
        p = dataclasses.replace(params, iters=iters)
        r = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], p, force=force[:iters])
        for it, k in tie_low:
            if it == iters - 1:
                r["E"] = r["E"].copy()
                r["E"][k] = np.nextafter(r["trace"][it, 0], 0.0)
        return r
    return run


def test_emargin_reports_the_exact_tie_of_the_identity_row():
    # F-track's template row 0 is the identity: its candidate IS the current pose, E_0 = E_base
    # bit for bit, so iteration 1's fitness margin is exactly 0 (strict <: not a member, L12)
    f, ov = _ftrack()
    o = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    assert o["emargin"][0] == 0.0
    assert o["trace"][0, 1] == 1   # only row 1 improves (E = 0 < 0.0833)


def test_forcing_the_natural_membership_changes_nothing():
    f, ov = _ftrack()
    p = f["params"]
    o = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], p)
    K = len(f["pst"])
    force = np.full((p.iters, K), -1, dtype=np.int8)
    for i in range(p.iters):
        oi = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], dataclasses.replace(p, iters=i + 1))
        force[i] = selection(oi["E"], o["trace"][i, 0], K, p)
    of = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], p, force=force)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(o[k], of[k]), k


def test_a_tie_is_shadowed_and_accepted():
    f, ov = _ftrack()
    p = f["params"]
    K = len(f["pst"])
    force = np.full((p.iters, K), -1, dtype=np.int8)
    force[0, 0] = 1                        # the other side counted the tied identity row as a member
    run = _fake_gpu(ov, f, p, force, tie_low=((0, 0),))
    r = run(p.iters)
    o0 = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], p)
    assert r["trace"][0, 1] == 2 and o0["trace"][0, 1] == 1   # the advantage sets really differ
    r2, o2, ties = track_parity(run, ov, f["depth"], f["intr"], f["T_init"], f["pst"], p, "shadow")
    assert ties == 1
    assert np.array_equal(r2["trace"], o2["trace"])


def test_a_difference_with_a_real_margin_is_rejected():
    """Iteration 1 holds a tie (row 0, margin 0), but the other side dropped row 1 (E_1 = 0 vs
    E_base = 0.0833): the per-particle check rejects it although the iteration's smallest margin is 0."""
    f, ov = _ftrack()
    p = f["params"]
    K = len(f["pst"])
    force = np.full((p.iters, K), -1, dtype=np.int8)
    force[0, 1] = 0
    run = _fake_gpu(ov, f, p, force)
    o = ov.track(f["depth"], f["intr"], f["T_init"], f["pst"], p)
    assert o["emargin"][0] < E_TIE
    with pytest.raises(AssertionError, match="not a tie"):
        track_parity(run, ov, f["depth"], f["intr"], f["T_init"], f["pst"], p, "real")


def test_margin_threshold_rejects_large_margins():
    """With a template whose iteration-1 margin is large (no identity row), any membership
    difference is rejected as 'not a tie'."""
    f, ov = _ftrack()
    pst = f["pst"][1:].copy()              # row (0,0,0, 0,0,-0.25) only: E_1 = 0 vs E_base 0.0833
    p = f["params"]
    o = ov.track(f["depth"], f["intr"], f["T_init"], pst, p)
    assert o["emargin"][0] > 0.5
    force = np.full((p.iters, 1), -1, dtype=np.int8)
    force[0, 0] = 0

    def run(iters):
        return ov.track(f["depth"], f["intr"], f["T_init"], pst, dataclasses.replace(p, iters=iters),
                        force=force[:iters])
    with pytest.raises(AssertionError, match="not a tie"):
        track_parity(run, ov, f["depth"], f["intr"], f["T_init"], pst, p, "large margin")
