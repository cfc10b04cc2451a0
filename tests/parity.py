"""Parity helpers: GPU (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star): in-band counts bit-exact; E within
1e-5 relative (1e-9 absolute floor); TSDF voxels within 1e-5 absolute (here: bit-exact, since
the fusion arithmetic is evaluated in the same fp64 operation order on both sides); poses
within 1e-4 m and 1e-4 rad.  A count mismatch is accepted only as a "tie": the oracle's cell
decision margin (distance of a grid coordinate to an integer) below 1e-9 voxel units.
"""
import dataclasses

import numpy as np

import oracle

E_REL, E_ABS = 1e-5, 1e-9
POSE_M, POSE_RAD = 1e-4, 1e-4
TIE_MARGIN = 1e-9   # cell decisions: distance of a grid coordinate to an integer (voxel units)
# fitness decisions: relative distance of E_k to E_base (oracle emargin).  Derived from the GPU's
# fitness arithmetic (DESIGN.md §6 "Tie handling"): fp32 record coefficients, fp32 lerp and a 2^-23
# fraction grid give per-evaluation errors of a few 2^-24 |v|; the mean over a candidate's in-band
# points measured 1.7e-8 relative at most over the 2048 converged candidates of config Q frame 1
# (test_gpu_fullsize.py::test_fitness_error_budget pins it below E_TIE / 3).  Round 1-2's 1e-8 sat
# below that measured error and held only because no candidate happened to fall closer.
E_TIE = 1e-7


def close_E(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.abs(a - b) <= np.maximum(E_REL * np.abs(b), E_ABS)


def assert_eval_parity(E_gpu, n_gpu, ora, what=""):
    """ora: dict(E, n, margin) from OracleVolume.eval_poses."""
    n_gpu = np.asarray(n_gpu)
    bad_n = n_gpu != ora["n"]
    ties = bad_n & (ora["margin"] < TIE_MARGIN)
    real = bad_n & ~ties
    assert not real.any(), f"{what}: in-band count mismatch at {np.nonzero(real)[0][:10]} " \
                           f"gpu={n_gpu[real][:5]} oracle={ora['n'][real][:5]} margin={ora['margin'][real][:5]}"
    ok = close_E(E_gpu, ora["E"]) | bad_n
    assert ok.all(), f"{what}: E mismatch at {np.nonzero(~ok)[0][:10]}: gpu={np.asarray(E_gpu)[~ok][:5]} " \
                     f"oracle={ora['E'][~ok][:5]}"
    return int(ties.sum())


def assert_pose_close(Ta, Tb, what=""):
    Ta, Tb = np.asarray(Ta).reshape(3, 4), np.asarray(Tb).reshape(3, 4)
    dt = np.abs(Ta[:, 3] - Tb[:, 3]).max()
    dr = oracle.rotation_error_rad(Ta, Tb)
    assert dt <= POSE_M and dr <= POSE_RAD, f"{what}: pose differs by {dt:.3e} m / {dr:.3e} rad"


def assert_trace_parity(tr_gpu, tr_ora, what=""):
    """Per-iteration: |A| exact, E_base / E(P) 1e-5 rel, s 1e-6 rel, P 1e-4, flags exact; the
    24-double rows' n_c, N, K_i and point-set code exact.  Rows after a stop rule fired are
    "not run" (flag bit 5, include/pft.h): all zeros except the flag, on both sides."""
    tr_gpu = np.asarray(tr_gpu)
    for i in range(tr_ora.shape[0]):
        g, o = tr_gpu[i], tr_ora[i]
        w = f"{what} iter {i + 1}"
        if int(o[19]) & 32:
            assert np.array_equal(g, o), f"{w}: not-run row gpu={g} oracle={o}"
            continue
        assert g[1] == o[1], f"{w}: |A| gpu={g[1]} oracle={o[1]}"
        if len(o) > 20:
            assert np.array_equal(g[20:24], o[20:24]), f"{w}: n_c/N/K_i/code gpu={g[20:24]} oracle={o[20:24]}"
        assert close_E(g[0], o[0]) and close_E(g[16], o[16]), f"{w}: E gpu={g[[0, 16]]} oracle={o[[0, 16]]}"
        for j in (2, 3, 17, 18):
            assert abs(g[j] - o[j]) <= 1e-6 * abs(o[j]) + 1e-12, f"{w}: s[{j}] gpu={g[j]} oracle={o[j]}"
        assert_pose_close(g[4:16], o[4:16], w)
        assert g[19] == o[19], f"{w}: flags gpu={g[19]} oracle={o[19]}"


def assert_last_iter_counts(n_gpu, E_gpu, o, ov, depth, intr, pst, params, T_init, what=""):
    """Last-iteration per-particle n_k exact and E_k within tolerance, except decision ties: a
    particle whose count differs must have, at the oracle's last-iteration candidate pose, a cell
    decision margin below TIE_MARGIN.  Returns the number of ties."""
    n_gpu, E_gpu = np.asarray(n_gpu), np.asarray(E_gpu)
    bad = np.nonzero(n_gpu != o["n"])[0]
    if len(bad):
        tr = o["trace"]
        # the last iteration that ran (rows after a stop rule are "not run", flag bit 5): its
        # search size, and the pose it started from (the row before it, or T_init)
        ran = [i for i in range(len(tr)) if not (int(tr[i, 19]) & 32)]
        last = ran[-1]
        P_last = tr[last - 1, 4:16].reshape(3, 4) if last > 0 else np.asarray(T_init).reshape(3, 4)
        om, v = tr[last, 2], tr[last, 3]
        poses = []
        for k in bad:
            dR, _, u = oracle.delta(pst[k], om, v)
            poses.append(oracle.apply_delta(dR, u, P_last, params.delta_conv))
        e = ov.eval_poses(depth, intr, np.stack(poses), stride=params.stride, rho=params.min_inband_frac)
        assert np.array_equal(e["n"], o["n"][bad]), f"{what}: oracle recomputation inconsistent"
        assert np.all(e["margin"] < TIE_MARGIN), \
            f"{what}: count mismatch at {bad[:8]} with decision margins {e['margin'][:8]} (not ties)"
        assert len(bad) <= max(2, len(n_gpu) // 1000), f"{what}: {len(bad)} ties is implausibly many"
    ok = close_E(E_gpu, o["E"]) | (n_gpu != o["n"])
    assert ok.all(), f"{what}: E mismatch at {np.nonzero(~ok)[0][:10]}"
    return len(bad)


# ------------------------------------------------------------------ fitness-decision ties
def selection(E, Ebase, Ki, params):
    """The membership include/pft.h defines for one iteration, from that side's E_k and E_base:
    A = {k < K_i : E_k < E_base}; for the top-k rule the topk smallest (E_k, k) of A."""
    E = np.asarray(E, dtype=np.float64)
    m = np.zeros(len(E), dtype=bool)
    m[:Ki] = E[:Ki] < Ebase
    if getattr(params, "update_rule", 0) == 2 and m.sum() > params.topk:
        idx = np.nonzero(m)[0]
        keep = idx[np.lexsort((idx, E[idx]))[:params.topk]]
        m[:] = False
        m[keep] = True
    return m


def first_selection_mismatch(tr_gpu, tr_ora):
    """Index of the first run iteration whose |A| differs, or None."""
    for i in range(tr_ora.shape[0]):
        if int(tr_ora[i, 19]) & 32 or int(tr_gpu[i, 19]) & 32:
            return None
        if tr_gpu[i, 1] != tr_ora[i, 1]:
            return i
    return None


def selection_margins(E, Ebase, Ki, params):
    """Per particle k < K_i: the relative distance of E_k to the thresholds its selection depends on
    (E_base; for the top-k rule also the topk-th and the next member's E)."""
    E = np.asarray(E, dtype=np.float64)[:Ki]
    m = np.abs(E - Ebase)
    if getattr(params, "update_rule", 0) == 2:
        mem = np.sort(E[E < Ebase])
        if len(mem) > params.topk:
            for c in (mem[params.topk - 1], mem[params.topk]):
                m = np.minimum(m, np.abs(E - c))
    return m / (Ebase if Ebase > 0 else 1.0)


def track_parity(run_gpu, ov, depth, intr, T_init, pst, params, what="", max_ties=2):
    """Whole-run parity with the margin-aware protocol.

    run_gpu(iters) -> dict(T, E, n, trace) of the GPU path run with `iters` iterations (the API is
    prefix-stable, include/pft.h).  The full GPU run is compared with the oracle; when the advantage
    set first differs (iteration i), both sides' per-particle E_k of iteration i are taken from
    prefix re-runs, and every particle whose selection differs must be a tie: its oracle E_k within
    E_TIE (relative) of a threshold it is compared with.  The oracle is then re-run *shadowed* --
    forced to the GPU's membership at i -- and everything downstream must agree again.  Returns
    (gpu, oracle, number of tied iterations)."""
    r = run_gpu(params.iters)
    K = np.asarray(pst).shape[0]
    force = np.full((params.iters, K), -1, dtype=np.int8)
    o = ov.track(depth, intr, T_init, pst, params)
    ties = 0
    while True:
        i = first_selection_mismatch(r["trace"], o["trace"])
        if i is None:
            break
        assert ties < max_ties, f"{what}: more than {max_ties} tied iterations"
        Ki = int(o["trace"][i, 22]) if o["trace"].shape[1] > 22 else K
        ri = run_gpu(i + 1)
        oi = ov.track(depth, intr, T_init, pst, dataclasses.replace(params, iters=i + 1), force=force[:i + 1])
        m_gpu = selection(ri["E"], r["trace"][i, 0], Ki, params)
        m_ora = selection(oi["E"], o["trace"][i, 0], Ki, params)
        diff = np.nonzero(m_gpu[:Ki] != m_ora[:Ki])[0]
        marg = selection_margins(oi["E"], o["trace"][i, 0], Ki, params)[diff]
        assert len(diff) and np.all(marg < E_TIE), \
            f"{what} iter {i + 1}: |A| gpu={r['trace'][i, 1]} oracle={o['trace'][i, 1]}; particles {diff[:8]} " \
            f"differ with fitness margins {marg[:8]} (not a tie)"
        # and the GPU's own E_k of a tied particle is within the same bar of the oracle's
        Eg, Eo = np.asarray(ri["E"], float)[diff], np.asarray(oi["E"], float)[diff]
        assert np.all(np.abs(Eg - Eo) <= E_TIE * np.abs(Eo)), \
            f"{what} iter {i + 1}: tied particles {diff[:8]} have E_k gpu={Eg[:4]} oracle={Eo[:4]}"
        force[i, :] = 0
        force[i, :Ki] = m_gpu[:Ki]
        o = ov.track(depth, intr, T_init, pst, params, force=force)
        ties += 1
    assert_trace_parity(r["trace"], o["trace"], what)
    return r, o, ties
