"""Pins of the oracle's NEXT-row extensions: F1 the paper's schedule
(K and point-rate alternation, max iterations, convergence stop) and F3 the
update-rule / acceptance variants (weighted mean w_k = E_base - E_k).
CPU only.  Each pin is a closed form, a reduction to the already-pinned plain run, or an invariant."""
import dataclasses

import numpy as np

import oracle
from synth.configs import TrackParams, config_tiny, make_pst
from tests.fixtures import f_track_inputs


def _run(c, params, pst=None):
    vol = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    return vol, vol.track(c["depth"], c["intr"], c["T_init"], c["pst"] if pst is None else pst, params)


def test_backproject_2d_strides_brute_force():
    """O2 with 2-D strides (sx on columns, sy on rows; L20 for the 1/8 and 1/32 rates): the list
    equals a brute-force row-major walk over pixels (sx*c, sy*r)."""
    c = config_tiny(seed=1)
    depth, K = c["depth"], c["intr"]
    for sx, sy in [(4, 2), (8, 4), (3, 5)]:
        pts = oracle.backproject(depth, K, sx, stride_y=sy)
        exp = []
        for v in range(0, K.height, sy):
            for u in range(0, K.width, sx):
                raw = int(depth[v, u])
                d = raw * 0.001
                if raw > 0 and d < 8.0:
                    exp.append(((u - K.cx) * d / K.fx, (v - K.cy) * d / K.fy, d))
        assert np.array_equal(pts, np.array(exp))


def test_single_entry_schedule_equals_plain_run():
    """F1 with one schedule entry (K, s, s) is the plain run bit for bit (trace columns 0-21),
    and records K_i and the stride code."""
    c = config_tiny(seed=2)
    plain = TrackParams(iters=3, stride=2)
    sch = dataclasses.replace(plain, nsched=1, sched_K=(64, 0, 0, 0), sched_sx=(2, 0, 0, 0), sched_sy=(2, 0, 0, 0))
    _, a = _run(c, plain)
    _, b = _run(c, sch)
    assert np.array_equal(a["trace"][:, :22], b["trace"][:, :22])
    assert np.array_equal(a["T"], b["T"]) and np.array_equal(a["E"], b["E"])
    assert np.all(b["trace"][:, 22] == 64) and np.all(b["trace"][:, 23] == 2 + 1000 * 2)


def test_schedule_uses_template_prefix():
    """Iteration i evaluates the first K_i template rows: a run whose schedule uses 24 of 64 rows
    equals the plain run on the 24-row template; rows >= K_i report E = 1, n = 0."""
    c = config_tiny(seed=3)
    sch = TrackParams(iters=3, stride=2, nsched=1, sched_K=(24, 0, 0, 0), sched_sx=(2, 0, 0, 0), sched_sy=(2, 0, 0, 0))
    _, a = _run(c, sch)
    _, b = _run(c, TrackParams(iters=3, stride=2), pst=c["pst"][:24].copy())
    assert np.array_equal(a["trace"][:, :22], b["trace"][:, :22])
    assert np.array_equal(a["E"][:24], b["E"]) and np.all(a["E"][24:] == 1.0) and np.all(a["n"][24:] == 0)


def test_schedule_baseline_recomputed_on_new_point_set():
    """L11 under F1: when the point set changes, E_base of iteration i is E(P^(i-1)) on X_i (an
    independent fitness call on the iteration's own strided points), and N_i is that set's size."""
    c = config_tiny(seed=4)
    sch = TrackParams(iters=4, stride=1, nsched=2, sched_K=(64, 32, 0, 0), sched_sx=(2, 4, 0, 0), sched_sy=(1, 2, 0, 0))
    vol, r = _run(c, sch)
    tr = r["trace"]
    P_prev = c["T_init"]
    for i in range(4):
        sx, sy = (2, 1) if i % 2 == 0 else (4, 2)
        pts = oracle.backproject(c["depth"], c["intr"], sx, stride_y=sy)
        E, _, _ = vol.fitness(pts, P_prev)
        assert tr[i, 0] == E and tr[i, 21] == len(pts) and tr[i, 22] == (64 if i % 2 == 0 else 32)
        P_prev = tr[i, 4:16].reshape(3, 4)


def test_min_search_stop():
    """F1 convergence stop: the run stops after the first iteration whose new search size is below
    (min_search_deg, min_search_cm); later rows are flagged not-run; T_out is that row's pose."""
    c = config_tiny(seed=1)
    full = TrackParams(iters=6, stride=2)
    _, a = _run(c, full)
    s_next = a["trace"][:, 17]
    stop_at = int(np.argmax(s_next < 4.0))
    assert s_next[stop_at] < 4.0 and stop_at < 5
    _, b = _run(c, dataclasses.replace(full, min_search_deg=4.0, min_search_cm=1e9))
    tb = b["trace"]
    assert np.array_equal(tb[:stop_at + 1, :19], a["trace"][:stop_at + 1, :19])
    assert int(tb[stop_at, 19]) & 16 and np.all(tb[stop_at + 1:, 19] == 32)
    assert np.array_equal(b["T"].reshape(12), tb[stop_at, 4:16])


def test_guard_monotone_and_rejection_keeps_pose():
    """F3 guard: with the guard every iteration's E_c <= E_base on the same
    point set; a rejected iteration (flag bit 3) keeps the previous pose and E_c = E_base."""
    c = config_tiny(seed=1)
    _, r = _run(c, TrackParams(iters=6, stride=1, guard=1))
    tr = r["trace"]
    assert np.all(tr[:, 16] <= tr[:, 0])
    prev = c["T_init"].reshape(12)
    for row in tr:
        if int(row[19]) & 8:
            assert np.array_equal(row[4:16], prev) and row[16] == row[0]
        prev = row[4:16]
    # the unguarded paper rule is not monotone on this seed; the guard matters
    _, u = _run(c, TrackParams(iters=6, stride=1))
    assert np.any(u["trace"][:, 16] > u["trace"][:, 0]) or np.any(tr[:, 19].astype(int) & 8)


def test_stall_limit_on_f_track():
    """F3 stall stop on fixture F-track: iteration 2 has an empty advantage set (a stall), so with
    stall_limit = 1 the run stops there; with 2 it runs on."""
    f = f_track_inputs()
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    p = dataclasses.replace(f["params"], iters=3, stall_limit=1)
    r = vol.track(f["depth"], f["intr"], f["T_init"], f["pst"], p)
    tr = r["trace"]
    assert tr[0, 1] == 1 and tr[1, 1] == 0
    assert int(tr[1, 19]) & 16 and tr[2, 19] == 32
    r2 = vol.track(f["depth"], f["intr"], f["T_init"], f["pst"], dataclasses.replace(p, stall_limit=2))
    assert not (int(r2["trace"][1, 19]) & 16) and int(r2["trace"][2, 19]) & 16


def test_weighted_mean_closed_form_on_plane():
    """F3 weighted rule on the F-track plane: rows u_z = -2.5 cm (E = 0) and -1.25 cm
    (E = 1.25/30) improve on E_base = 2.5/30; weights E_base - E_k give u = -2.0833 cm, while the
    paper's plain mean gives -1.875 cm (camera-centred, t' = t + u)."""
    f = f_track_inputs()
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    pst = np.array([[0, 0, 0, 0, 0, -0.25], [0, 0, 0, 0, 0, -0.125]], np.float32)
    p = dataclasses.replace(f["params"], iters=1)
    w = vol.track(f["depth"], f["intr"], f["T_init"], pst, dataclasses.replace(p, update_rule=1))
    m = vol.track(f["depth"], f["intr"], f["T_init"], pst, p)
    z0 = f["T_init"][2, 3]
    Eb, E1 = 0.025 / 0.3, 0.0125 / 0.3
    u_w = (Eb * -0.025 + (Eb - E1) * -0.0125) / (Eb + (Eb - E1))
    assert abs(w["T"][2, 3] - (z0 + u_w)) < 1e-7
    assert abs(m["T"][2, 3] - (z0 - 0.01875)) < 1e-7
    assert w["trace"][0, 1] == m["trace"][0, 1] == 2


def test_paper_schedule_runs_and_converges_on_tiny():
    """The paper's schedule on config T with its own K alternation (template of 10240 rows): the
    search size never grows, K_i cycles 10240/3072/1024, and it stops by min_search within 20."""
    from synth.configs import PAPER_SCHEDULE
    c = config_tiny(seed=1)
    p = TrackParams(stride=1, **PAPER_SCHEDULE)
    _, r = _run(c, p, pst=make_pst(1, 10240))
    tr = r["trace"]
    ran = tr[:, 19].astype(int) & 32 == 0
    assert np.all(np.diff(tr[ran, 2]) <= 0)
    assert list(tr[:3, 22]) == [10240, 3072, 1024]
    assert int(tr[ran][-1, 19]) & 16 or ran.sum() == 20


# ------------------------------------------------------------------ F4 surface points
def test_extract_fresh_volume_is_empty():
    """a fresh (unobserved) volume has no surface points."""
    from synth.configs import VolumeDesc
    vol = oracle.OracleVolume(VolumeDesc(12, 10, 8, 0.1, (0.0, 0.0, 0.0), 0.3))
    assert len(vol.extract()) == 0


def test_extract_plane_closed_form():
    """A linear field V = (z - z0)/tau (analytic fill, W = 1) crosses zero exactly at z0: every
    extracted point lies on z = z0 (up to the fp32 rounding of the stored values), only z-edges
    cross, and there is one crossing per (i, j) column."""
    from synth.configs import VolumeDesc
    n, s, tau, z0 = 16, 0.1, 0.3, 0.83
    desc = VolumeDesc(n, n, n, s, (0.0, 0.0, 0.0), tau)
    z = (np.arange(n) + 0.5) * s
    col = np.clip((z - z0) / tau, -1, 1).astype(np.float32)
    V = np.broadcast_to(col[:, None, None], (n, n, n)).astype(np.float32).ravel()
    W = np.ones_like(V)
    pts = oracle.OracleVolume(desc, V, W).extract()
    assert len(pts) == n * n
    assert np.abs(pts[:, 2] - z0).max() < 1e-6
    xs = np.sort(np.unique(np.round(pts[:, 0], 9)))
    assert np.allclose(xs, (np.arange(n) + 0.5) * s)


def test_extract_sphere_radii():
    """SPEC.md:262 analytic sphere (config T fill): extracted points lie within one voxel of the
    sphere or the ground plane."""
    c = config_tiny(seed=1)
    pts = oracle.OracleVolume(c["desc"], c["V"], c["W"]).extract()
    assert len(pts) > 1000
    d = np.abs(c["scene"].sdf(pts))
    assert d.max() < c["desc"].voxel_m and np.sqrt(np.mean(d ** 2)) < c["desc"].voxel_m / 2


def test_extract_ignores_unobserved_and_brute_force_small():
    """Brute force on a random 5x4x3 grid with unobserved voxels: the oracle's list equals a direct
    enumeration of the definition (edges between observed voxels with a sign change)."""
    from synth.configs import VolumeDesc
    rng = np.random.default_rng(3)
    nx, ny, nz, s = 5, 4, 3, 0.1
    desc = VolumeDesc(nx, ny, nz, s, (0.1, -0.2, 0.3), 0.3)
    V = rng.choice([-0.75, -0.25, 0.0, 0.5, 1.0], size=nx * ny * nz).astype(np.float32)
    W = rng.choice([0.0, 1.0, 2.0], size=nx * ny * nz).astype(np.float32)
    got = oracle.OracleVolume(desc, V, W).extract()
    Vg, Wg = V.reshape(nz, ny, nx).astype(float), W.reshape(nz, ny, nx)
    exp = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                for a, (di, dj, dk) in enumerate([(1, 0, 0), (0, 1, 0), (0, 0, 1)]):
                    i1, j1, k1 = i + di, j + dj, k + dk
                    if i1 >= nx or j1 >= ny or k1 >= nz or Wg[k, j, i] <= 0 or Wg[k1, j1, i1] <= 0:
                        continue
                    v0, v1 = Vg[k, j, i], Vg[k1, j1, i1]
                    if (v0 > 0) == (v1 > 0) or (v0 == 0 and v1 == 0):
                        continue
                    p = [0.1 + s * (i + 0.5), -0.2 + s * (j + 0.5), 0.3 + s * (k + 0.5)]
                    p[a] = p[a] + (v0 / (v0 - v1)) * s
                    exp.append(p)
    assert np.array_equal(got, np.array(exp).reshape(-1, 3))


def test_topk_reductions_and_closed_form():
    """F3 top-k (north_star "fused top-k/weighted-mean pose update"): topk >= |A| is the paper's
    mean bit for bit; topk = 1 moves by exactly the best member's delta (smallest E_k, lowest k on
    ties) -- on the F-track plane the 2.5 cm row (E = 0) wins over the 1.25 cm row."""
    f = f_track_inputs()
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    pst = np.array([[0, 0, 0, 0, 0, -0.125], [0, 0, 0, 0, 0, -0.25], [0, 0, 0, 0, 0, 0.1]], np.float32)
    p = dataclasses.replace(f["params"], iters=1)
    m = vol.track(f["depth"], f["intr"], f["T_init"], pst, p)
    big = vol.track(f["depth"], f["intr"], f["T_init"], pst, dataclasses.replace(p, update_rule=2, topk=5))
    assert np.array_equal(m["trace"], big["trace"]) and np.array_equal(m["T"], big["T"])
    one = vol.track(f["depth"], f["intr"], f["T_init"], pst, dataclasses.replace(p, update_rule=2, topk=1))
    assert one["trace"][0, 1] == 1
    assert abs(one["T"][2, 3] - (f["T_init"][2, 3] - 0.025)) < 1e-12
    # on config T, topk = 8 averages exactly the 8 best members of iteration 1
    c = config_tiny(seed=1)
    ct = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    p8 = TrackParams(iters=1, stride=2, update_rule=2, topk=8)
    r8 = ct.track(c["depth"], c["intr"], c["T_init"], c["pst"], p8)
    Eb = r8["trace"][0, 0]
    order = sorted([k for k in range(64) if r8["E"][k] < Eb], key=lambda k: (r8["E"][k], k))[:8]
    Q, U = np.zeros(4), np.zeros(3)
    for k in sorted(order):
        _, q, u = oracle.delta(c["pst"][k], 10.0, 10.0)
        Q, U = Q + q, U + u
    Pn = oracle.apply_delta(oracle.quat_to_R(Q / np.linalg.norm(Q)), U / 8, c["T_init"], 0)
    assert r8["trace"][0, 1] == 8 and np.abs(r8["T"] - Pn).max() < 1e-12


def test_f_mean_non_coaxial_quaternion_average():
    """O7 average over a two-member advantage set with non-coaxial rotations (rotX(10 deg) and
    rotY(10 deg)) against the hand-derived axis-angle closed form (tests/golden/f_mean.json): pins
    the L13 reading (normalised quaternion sum; a rotation-vector mean differs by 2.8e-5 rad), the
    left-multiplied camera-centred composition and the sense of the rotation."""
    from tests.fixtures import f_mean_closed_form, f_mean_inputs
    f = f_mean_inputs()
    cf = f_mean_closed_form()
    o = oracle.OracleVolume(f["desc"], f["V"], f["W"]).track(f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    tr = o["trace"][0]
    assert tr[1] == 2
    assert abs(tr[0] - cf["E_base"]) < 1e-7
    np.testing.assert_allclose(o["E"], cf["E"], atol=1e-7)
    np.testing.assert_allclose(o["T"], cf["P"], atol=1e-12)
    np.testing.assert_allclose(tr[4:16].reshape(3, 4), cf["P"], atol=1e-12)
    assert abs(tr[16] - cf["E_c"]) < 1e-7
    assert abs(tr[17] - cf["s_next"][0]) < 2e-6 and abs(tr[18] - cf["s_next"][1]) < 1e-6
    # the reading matters at this size: the rotation-vector mean is a different pose
    assert abs(cf["phi"] - np.deg2rad(10.0) / np.sqrt(2.0)) > 2e-5
