"""Pins of the fp64 CPU oracle against what the paper and the mathematics fix (CPU only).

Each test names the oracle step and the pin kind:
closed form, special case reducing to a library routine, invariant, brute force
or a hand-derived golden fixture (tests/golden/, each with its citation).
"""
import math

import numpy as np
import pytest
from scipy.linalg import expm
from scipy.spatial.transform import Rotation

import oracle
from synth.configs import VolumeDesc, TrackParams
from synth.scene import Intrinsics, Scene, analytic_fill, look_at, render_depth
from tests.fixtures import f_track_inputs, golden


# ----------------------------------------------------------------------------- O1/O2 back-projection
def test_backproject_principal_ray():
    """pixel (cx, cy, d=2.0) -> (0, 0, 2.0)."""
    intr = Intrinsics(100.0, 100.0, 1.0, 1.0, 3, 3)
    depth = np.zeros((3, 3), np.uint16)
    depth[1, 1] = 2000
    p = oracle.backproject(depth, intr, 1)
    assert p.shape == (1, 3)
    assert np.array_equal(p[0], [0.0, 0.0, 2.0])


def test_backproject_unit_tangent():
    """fx=fy=100, cx=cy=50, pixel (150, 50, d=1.0) -> (1, 0, 1)."""
    intr = Intrinsics(100.0, 100.0, 50.0, 50.0, 160, 100)
    depth = np.zeros((100, 160), np.uint16)
    depth[50, 150] = 1000
    p = oracle.backproject(depth, intr, 1)
    assert np.allclose(p, [[1.0, 0.0, 1.0]], atol=1e-15)


def test_backproject_stride_order_validity():
    """O2 reading L20: 2-D stride over rows then columns, row-major, ceil(H/s) x ceil(W/s) candidates;
    raw 0 and d >= max_depth are invalid (O1)."""
    intr = Intrinsics(50.0, 60.0, 4.5, 3.5, 10, 7)
    rng = np.random.default_rng(0)
    depth = rng.integers(500, 4000, size=(7, 10)).astype(np.uint16)
    depth[0, 3] = 0            # invalid: raw 0 (kept pixel, stride 3 -> column 3 is sampled)
    depth[3, 6] = 9000         # invalid: beyond 8 m
    p = oracle.backproject(depth, intr, 3, max_depth_m=8.0)
    want = []
    for v in range(0, 7, 3):
        for u in range(0, 10, 3):
            raw = int(depth[v, u])
            d = raw * 0.001
            if raw == 0 or d >= 8.0:
                continue
            want.append(((u - 4.5) * d / 50.0, (v - 3.5) * d / 60.0, d))
    assert len(want) == 3 * 4 - 2
    assert np.allclose(p, np.array(want), rtol=0, atol=1e-15)
    # round trip project(backproject(.)) = source pixel centre
    u = 50.0 * p[:, 0] / p[:, 2] + 4.5
    v = 60.0 * p[:, 1] / p[:, 2] + 3.5
    assert np.all(np.abs(u - np.round(u)) < 1e-9) and np.all(np.abs(v - np.round(v)) < 1e-9)


# ----------------------------------------------------------------------------- O3 query
def _vol(n, voxel, origin, trunc, V):
    desc = VolumeDesc(n, n, n, voxel, origin, trunc)
    return oracle.OracleVolume(desc, V.astype(np.float32), np.ones(n ** 3, np.float32))


def test_query_affine_and_multilinear_fields_exact():
    """Trilinear interpolation reproduces affine and multilinear (xyz) fields exactly.  Values are
    dyadic (exact in fp32), so any wrong weight, swapped axis, dropped cross term or missing
    half-voxel offset shows up as an O(1e-3) error instead of 1e-15."""
    n = 12
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    # affine with distinct per-axis coefficients + a trilinear cross term, |V| < 1
    V = (3 * i - 5 * j + 7 * k) / 256.0 + (i * j * k) / 4096.0 - 0.125
    assert np.abs(V).max() < 1
    vol = _vol(n, 0.05, (-0.3, 0.2, 1.0), 0.2, V.ravel())
    rng = np.random.default_rng(1)
    for _ in range(300):
        g = rng.uniform(0, n - 1, 3)
        q = np.array([-0.3, 0.2, 1.0]) + 0.05 * (g + 0.5)
        ok, v, _ = vol.query(q)
        gx, gy, gz = (q - np.array([-0.3, 0.2, 1.0])) / 0.05 - 0.5
        want = (3 * gx - 5 * gy + 7 * gz) / 256.0 + gx * gy * gz / 4096.0 - 0.125
        assert ok
        assert abs(v - want) < 1e-12


def test_query_voxel_centre_and_midpoint():
    """a voxel-centre query returns the stored value; midway between two centres
    along x gives (a+b)/2."""
    n = 8
    rng = np.random.default_rng(2)
    V = rng.uniform(-0.9, 0.9, n ** 3).astype(np.float32)
    vol = _vol(n, 0.125, (0, 0, 0), 0.3, V)       # dyadic voxel: g is exact
    Vc = V.reshape(n, n, n).astype(np.float64)
    for (i, j, k) in [(0, 0, 0), (3, 4, 5), (6, 6, 6), (2, 6, 1)]:
        ok, v, _ = vol.query(0.125 * (np.array([i, j, k]) + 0.5))
        assert ok and v == Vc[k, j, i]
        ok, v, _ = vol.query(0.125 * (np.array([i + 0.5, j, k]) + 0.5))
        assert ok and abs(v - 0.5 * (Vc[k, j, i] + Vc[k, j, i + 1])) < 1e-15


def test_query_bounds_and_band():
    """L5: cells with floor(g) in [0, n-2] only (the exact last sample plane is excluded);
    L3: all 8 corners must satisfy |V| < 1 strictly; a fresh (reset) volume has nothing in band."""
    n = 8
    V = np.zeros(n ** 3, np.float32)
    vol = _vol(n, 0.1, (0, 0, 0), 0.3, V)
    c = lambda g: 0.1 * (np.asarray(g, float) + 0.5)
    assert vol.query(c([0, 0, 0]))[0]
    assert not vol.query(c([-1e-9, 3, 3]))[0]
    assert vol.query(c([n - 1 - 1e-9, 3, 3]))[0]
    assert not vol.query(c([n - 1, 3, 3]))[0]
    assert not vol.query(c([3, 3, n - 1]))[0]
    Vb = V.reshape(n, n, n).copy()
    Vb[4, 4, 4] = 1.0                       # one corner exactly 1 -> cells touching it leave the band
    vol2 = _vol(n, 0.1, (0, 0, 0), 0.3, Vb.ravel())
    assert not vol2.query(c([3.5, 3.5, 3.5]))[0]
    assert vol2.query(c([4.5, 4.5, 4.5]))[0] is False
    assert vol2.query(c([5.5, 5.5, 5.5]))[0]
    Vb[4, 4, 4] = np.float32(0.99999994)    # largest fp32 below 1 is in band
    vol3 = _vol(n, 0.1, (0, 0, 0), 0.3, Vb.ravel())
    assert vol3.query(c([3.5, 3.5, 3.5]))[0]
    fresh = oracle.OracleVolume(VolumeDesc(n, n, n, 0.1, (0, 0, 0), 0.3))
    assert all(not fresh.query(c(g))[0] for g in np.random.default_rng(3).uniform(0, n - 1, (50, 3)))


def test_query_sphere_surface_closed_form_bound():
    """Analytic sphere SDF (north_star): points on the sphere read |v| <= (3/8)s^2/(rho tau)
    (trilinear error of a smooth SDF), here 2.5e-4 m / tau.  A missing half-voxel offset or a
    swapped corner would read ~0.17 instead."""
    scene = Scene(spheres=[(0.64, 0.64, 0.64, 0.4)])
    desc = VolumeDesc(64, 64, 64, 0.02, (0.0, 0.0, 0.0), 0.06)
    V, W = analytic_fill(scene, 64, 64, 64, 0.02, desc.origin_m, desc.trunc_m)
    vol = oracle.OracleVolume(desc, V, W)
    rng = np.random.default_rng(4)
    dirs = rng.normal(size=(400, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    pts = np.array([0.64, 0.64, 0.64]) + 0.4 * dirs
    worst = 0.0
    for p in pts:
        ok, v, _ = vol.query(p)
        assert ok
        worst = max(worst, abs(v))
    bound = (3.0 / 8.0) * 0.02 ** 2 / 0.4 / 0.06 + 1e-6
    assert worst <= bound
    # points 1 cm outside the sphere read +1cm/tau up to the same bound
    ok, v, _ = vol.query(np.array([0.64, 0.64, 0.64]) + 0.41 * dirs[0])
    assert ok and abs(v - 0.01 / 0.06) <= bound


# ----------------------------------------------------------------------------- O4 fitness
def _plane_volume(z0=0.8, n=16, voxel=0.1, tau=0.3):
    z = voxel * (np.arange(n) + 0.5)
    col = np.clip((z - z0) / tau, -1.0, 1.0).astype(np.float32)
    V = np.broadcast_to(col[:, None, None], (n, n, n)).astype(np.float32).ravel()
    return oracle.OracleVolume(VolumeDesc(n, n, n, voxel, (0, 0, 0), tau), V, np.ones_like(V))


@pytest.mark.parametrize("delta", [-0.18, -0.05, -0.005, 0.0, 0.005, 0.07, 0.19])
def test_fitness_plane_closed_form(delta):
    """PAPER.md:201 eq. E on a plane: points displaced delta along the normal read E = |delta|/tau
    while every trilinear corner stays in band (|delta| <= tau - voxel).  Tolerance covers the fp32
    rounding of the stored V (L23)."""
    vol = _plane_volume()
    rng = np.random.default_rng(5)
    pts = np.column_stack([rng.uniform(0.3, 1.2, 200), rng.uniform(0.3, 1.2, 200), np.full(200, 0.8 + delta)])
    E, n, _ = vol.fitness(pts, np.hstack([np.eye(3), np.zeros((3, 1))]))
    assert n == 200
    assert abs(E - abs(delta) / 0.3) < 2e-7


def test_fitness_empty_and_min_fraction():
    """L6: no in-band point -> E = 1, n = 0; with rho > 0, n < rho N -> E = 1 (n still reported)."""
    vol = _plane_volume()
    I = np.hstack([np.eye(3), np.zeros((3, 1))])
    far = np.array([[5.0, 5.0, 5.0], [-1.0, 0.5, 0.8]])
    E, n, _ = vol.fitness(far, I)
    assert E == 1.0 and n == 0
    pts = np.array([[0.5, 0.5, 0.8], [5.0, 5.0, 5.0], [6.0, 6.0, 6.0]])
    E, n, _ = vol.fitness(pts, I, rho=0.5)
    assert E == 1.0 and n == 1
    E, n, _ = vol.fitness(pts, I, rho=0.3)
    assert n == 1 and E < 1e-6


def test_fitness_permutation_invariant():
    vol = _plane_volume()
    rng = np.random.default_rng(6)
    pts = np.column_stack([rng.uniform(0.2, 1.3, 300), rng.uniform(0.2, 1.3, 300), rng.uniform(0.6, 1.0, 300)])
    T = np.hstack([Rotation.from_rotvec([0.02, -0.01, 0.03]).as_matrix(), [[0.01], [0.0], [-0.02]]])
    E1, n1, _ = vol.fitness(pts, T)
    E2, n2, _ = vol.fitness(pts[rng.permutation(300)], T)
    assert n1 == n2 and abs(E1 - E2) < 1e-13


# ----------------------------------------------------------------------------- O5 / O6 delta poses
def test_delta_zero_is_identity():
    """s = (0,0) or a zero template row -> identity delta and q = (1,0,0,0)."""
    dR, q, u = oracle.delta(np.array([0.3, -0.7, 1.0, 0.2, -1.0, 0.5]), 0.0, 0.0)
    assert np.array_equal(dR, np.eye(3)) and np.array_equal(q, [1, 0, 0, 0]) and np.array_equal(u, [0, 0, 0])
    dR, q, u = oracle.delta(np.zeros(6), 10.0, 10.0)
    assert np.array_equal(dR, np.eye(3)) and np.array_equal(u, [0, 0, 0])


def test_delta_rotz90():
    """r = (0,0,pi/2) -> rotZ(90 deg)."""
    dR, q, u = oracle.delta(np.array([0, 0, 1, 0, 0, 0], np.float32), 90.0, 0.0)
    assert np.allclose(dR, [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    assert np.allclose(q, [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)], atol=1e-15)


def test_delta_matches_matrix_exponential_and_quaternion():
    """Rodrigues (L9) equals the matrix exponential of [r]x (scipy.linalg.expm) and the
    Hamilton quaternion's matrix (O5 self-check, 4e-15); box bounds: angle <= sqrt(3) omega,
    |u_a| <= v/100."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        a = rng.uniform(-1, 1, 6).astype(np.float32)
        om, v = rng.uniform(0, 100), rng.uniform(0, 20)
        dR, q, u = oracle.delta(a, om, v)
        r = a[:3].astype(np.float64) * (om * np.pi / 180.0)
        S = np.array([[0, -r[2], r[1]], [r[2], 0, -r[0]], [-r[1], r[0], 0]])
        assert np.abs(dR - expm(S)).max() < 1e-13
        assert np.abs(dR - oracle.quat_to_R(q)).max() < 4e-15
        assert abs(np.linalg.norm(q) - 1) < 1e-15 and q[0] > 0
        assert np.linalg.norm(r) <= math.sqrt(3) * om * np.pi / 180 + 1e-15
        assert np.all(np.abs(u) <= v / 100 + 1e-17)
        assert np.allclose(u, a[3:].astype(np.float64) * v / 100, rtol=0, atol=1e-16)


def test_apply_delta_conventions():
    """L10: camera-centred (R', t') = (dR R, t + u) equals the literal left product conjugated to
    the camera centre; world-literal equals the 4x4 homogeneous product [dR u; 0 1][R t; 0 1]."""
    rng = np.random.default_rng(8)
    for _ in range(50):
        P = np.hstack([Rotation.random(random_state=rng).as_matrix(), rng.normal(size=(3, 1))])
        dR = Rotation.from_rotvec(rng.normal(size=3) * 0.2).as_matrix()
        u = rng.normal(size=3) * 0.1
        H = lambda R, t: np.vstack([np.hstack([R, np.reshape(t, (3, 1))]), [0, 0, 0, 1]])
        lit = (H(dR, u) @ H(P[:, :3], P[:, 3]))[:3]
        assert np.allclose(oracle.apply_delta(dR, u, P, conv=1), lit, atol=1e-14)
        c = P[:, 3]
        cam = (H(np.eye(3), c + u) @ H(dR, np.zeros(3)) @ H(np.eye(3), -c) @ H(P[:, :3], P[:, 3]))[:3]
        assert np.allclose(oracle.apply_delta(dR, u, P, conv=0), cam, atol=1e-14)


def test_rotation_error_matches_quaternion_angle():
    """PAPER.md:174 l_R = arccos((tr(R^T R') - 1)/2) equals the quaternion angle 2 acos|q.q'|."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        a, b = Rotation.random(random_state=rng), Rotation.random(random_state=rng)
        want = 2 * math.acos(min(1.0, abs(float(np.dot(a.as_quat(), b.as_quat())))))
        assert abs(oracle.rotation_error_rad(a.as_matrix(), b.as_matrix()) - want) < 1e-6


# ----------------------------------------------------------------------------- O7 / O8 tracking
def test_track_golden_f_track():
    """Golden fixture F-track (tests/golden/f_track.json, derived from PAPER.md:205-207)."""
    f = f_track_inputs()
    a = float(np.float32(1.0 / 6.0))
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    r = vol.track(f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    tol = f["g"]["expect"]["tol"]
    tr = r["trace"]
    assert r["N"] == 4
    # iteration 1
    assert abs(tr[0, 0] - 0.5 * a) < tol and tr[0, 1] == 1 and tr[0, 2] == 10 and tr[0, 3] == 10
    assert np.abs(tr[0, 4:16].reshape(3, 4) - f["T_gt"]).max() < tol
    assert abs(tr[0, 16]) < tol and abs(tr[0, 17] - 1.0) < tol and abs(tr[0, 18] - 1.0) < tol and tr[0, 19] == 0
    # iteration 2
    assert abs(tr[1, 0]) < tol and tr[1, 1] == 0 and abs(tr[1, 2] - 1) < tol
    assert abs(tr[1, 17] - 0.1) < tol and abs(tr[1, 18] - 0.1) < tol and tr[1, 19] == 1
    assert abs(r["E"][0]) < tol and abs(r["E"][1] - 0.05 * a) < tol
    assert list(r["n"]) == [4, 4]
    assert np.abs(r["T"] - f["T_gt"]).max() < tol


def test_track_symmetric_pair_averages_to_identity():
    """SPEC.md:95-96 / PAPER.md:206: a symmetric advantage set {rotZ(+a), rotZ(-a)} with equal
    translations averages to no rotation; the plane scene makes both rows improve equally
    (rotation about the optical axis keeps points on the plane)."""
    f = f_track_inputs()
    pst = np.array([[0, 0, 0.5, 0, 0, -0.25], [0, 0, -0.5, 0, 0, -0.25], [0, 0, 0, 0, 0, 0]], np.float32)
    p = TrackParams(iters=1, stride=2)
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    r = vol.track(f["depth"], f["intr"], f["T_init"], pst, p)
    assert r["trace"][0, 1] == 2
    assert np.abs(r["T"] - f["T_gt"]).max() < 1e-12


def test_track_permutation_invariant():
    """Advantage-set membership is order independent and the mean is a sum (1e-12)."""
    f = f_track_inputs()
    rng = np.random.default_rng(10)
    pst = rng.uniform(-1, 1, (40, 6)).astype(np.float32)
    perm = rng.permutation(40)
    p = TrackParams(iters=3, stride=1, omega0_deg=2.0, v0_cm=3.0)
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    depth = np.full((3, 3), 800, np.uint16)
    r1 = vol.track(depth, f["intr"], f["T_init"], pst, p)
    r2 = vol.track(depth, f["intr"], f["T_init"], pst[perm], p)
    assert np.abs(r1["T"] - r2["T"]).max() < 1e-12
    assert np.abs(r1["E"][perm] - r2["E"]).max() < 1e-12
    assert np.array_equal(r1["trace"][:, 1], r2["trace"][:, 1])


def test_track_search_size_law_and_lost():
    """PAPER.md:207 s-law examples: E = 1 leaves s unchanged (here: every point
    outside the grid -> lost flag, |A| = 0); s never grows; EMPTY cloud returns T_init, E = 1."""
    f = f_track_inputs()
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    T_far = f["T_init"].copy()
    T_far[:, 3] += 50.0
    r = vol.track(f["depth"], f["intr"], T_far, f["pst"], TrackParams(iters=3, stride=2))
    tr = r["trace"]
    assert np.all(tr[:, 0] == 1.0) and np.all(tr[:, 1] == 0) and np.all(tr[:, 2] == 10) and np.all(tr[:, 17] == 10)
    assert np.all(tr[:, 19] == 3)
    assert np.array_equal(r["T"], T_far)
    # empty cloud
    r = vol.track(np.zeros((3, 3), np.uint16), f["intr"], f["T_init"], f["pst"], TrackParams(iters=2, stride=2))
    assert r["N"] == 0 and np.array_equal(r["T"], f["T_init"]) and np.all(r["E"] == 1) and np.all(r["n"] == 0)
    # never grows, with E in [0,1]
    rng = np.random.default_rng(11)
    pst = rng.uniform(-1, 1, (64, 6)).astype(np.float32)
    r = vol.track(np.full((3, 3), 800, np.uint16), f["intr"], f["T_init"], pst, TrackParams(iters=5, stride=1))
    tr = r["trace"]
    assert np.all(tr[:, 17] <= tr[:, 2]) and np.all(tr[:, 16] <= 1) and np.all(tr[:, 16] >= 0)
    fac = 0.1 + 0.9 * tr[:, 16]
    assert np.allclose(tr[:, 17], fac * tr[:, 2], rtol=1e-15)


def test_track_deterministic():
    """Bit-identical repeat runs, also with a different thread count."""
    f = f_track_inputs()
    rng = np.random.default_rng(12)
    pst = rng.uniform(-1, 1, (100, 6)).astype(np.float32)
    vol = oracle.OracleVolume(f["desc"], f["V"], f["W"])
    p = TrackParams(iters=4, stride=1)
    depth = np.full((3, 3), 800, np.uint16)
    r1 = vol.track(depth, f["intr"], f["T_init"], pst, p, nthreads=1)
    r2 = vol.track(depth, f["intr"], f["T_init"], pst, p, nthreads=4)
    assert np.array_equal(r1["T"], r2["T"]) and np.array_equal(r1["E"], r2["E"]) and np.array_equal(r1["trace"], r2["trace"])


# ----------------------------------------------------------------------------- O9 integration
def test_integrate_golden_f_integrate():
    """Golden fixture F-integrate (tests/golden/f_integrate.json; L22)."""
    f = f_track_inputs()
    g = golden("f_integrate.json")
    vol = oracle.OracleVolume(f["desc"])
    n = vol.integrate(f["depth"], f["intr"], f["T_gt"])
    assert n == g["updated_voxels"]
    V = vol.values_f64().reshape(16, 16, 16)
    W = vol.weights_f64().reshape(16, 16, 16)
    i, j = g["column_ij"]
    want = np.array([eval(s) for s in g["V"]], dtype=np.float64)
    assert np.abs(V[:, j, i] - want).max() < g["value_tol"]
    assert np.array_equal(W[:, j, i], np.array(g["W"], np.float64))
    assert int((W > 0).sum()) == g["updated_voxels"]
    # the same frame again: V unchanged, W = 2
    V1 = vol.V.copy()
    vol.integrate(f["depth"], f["intr"], f["T_gt"])
    assert np.array_equal(vol.V, V1)
    assert set(np.unique(vol.weights_f64())) == {0.0, 2.0}


def test_integrate_frontal_plane_closed_form():
    """Frontal plane at depth D seen by a camera looking along +z: every voxel well inside the
    image gets V = min(1, (D - z_c)/tau) if z_c < D + tau and stays untouched beyond."""
    n, vox, tau, D = 24, 0.05, 0.15, 0.8
    desc = VolumeDesc(n, n, n, vox, (-0.6, -0.6, 0.0), tau)
    intr = Intrinsics(40.0, 40.0, 19.5, 19.5, 40, 40)
    depth = np.full((40, 40), int(D * 1000), np.uint16)
    T = np.hstack([np.eye(3), np.zeros((3, 1))])
    vol = oracle.OracleVolume(desc)
    vol.integrate(depth, intr, T)
    V = vol.values_f64().reshape(n, n, n)
    W = vol.weights_f64().reshape(n, n, n)
    checked = 0
    for k in range(n):
        zc = vox * (k + 0.5)
        for j in range(n):
            for i in range(n):
                x, y = -0.6 + vox * (i + 0.5), -0.6 + vox * (j + 0.5)
                u, v = 40 * x / zc + 19.5, 40 * y / zc + 19.5
                if not (0.5 < u < 38.5 and 0.5 < v < 38.5):
                    continue
                checked += 1
                if zc < D + tau - 1e-9:
                    assert W[k, j, i] == 1
                    assert abs(V[k, j, i] - min(1.0, (D - zc) / tau)) < 1e-7
                elif zc > D + tau + 1e-9:
                    assert W[k, j, i] == 0 and V[k, j, i] == 1
    assert checked > 1000


def test_integrate_bounds_cap_and_order():
    """Invariants: V in [-1,1], W in [0, W_max] (cap reached), and fusing A then B
    equals B then A below the cap (1e-6)."""
    scene = Scene(spheres=[(0.0, 0.0, 1.2, 0.3)], plane_z=None, room_half=2.0)
    intr = Intrinsics(60.0, 60.0, 31.5, 23.5, 64, 48)
    desc = VolumeDesc(32, 32, 32, 0.05, (-0.8, -0.8, 0.4), 0.15, max_weight=3.0)
    poses = [look_at([0.1 * s, -0.6 - 0.05 * s, 0.0], [0.0, 0.0, 1.2]) for s in (-1, 0, 1, 2, -2)]
    frames = [render_depth(scene, intr, T) for T in poses]
    volA = oracle.OracleVolume(desc)
    for T, dpt in zip(poses, frames):
        volA.integrate(dpt, intr, T)
    V, W = volA.values_f64(), volA.weights_f64()
    assert V.min() >= -1 and V.max() <= 1 and W.min() >= 0 and W.max() == 3.0
    descB = VolumeDesc(32, 32, 32, 0.05, (-0.8, -0.8, 0.4), 0.15, max_weight=128.0)
    a, b = oracle.OracleVolume(descB), oracle.OracleVolume(descB)
    a.integrate(frames[0], intr, poses[0]); a.integrate(frames[1], intr, poses[1])
    b.integrate(frames[1], intr, poses[1]); b.integrate(frames[0], intr, poses[0])
    assert np.abs(a.values_f64() - b.values_f64()).max() < 1e-6
    assert np.array_equal(a.W, b.W)


def test_fp16_storage_rounding_matches_numpy():
    """L23 fp16 storage: the oracle's one RNE rounding equals numpy's float64 -> float16 cast,
    including exact ties."""
    rng = np.random.default_rng(13)
    xs = list(rng.uniform(-1, 1, 2000)) + list(rng.uniform(0, 130, 200))
    # exact ties between consecutive fp16 values in [0.5, 1): spacing 2^-11
    xs += [0.5 + (2 * m + 1) * 2.0 ** -12 for m in range(0, 1000, 7)]
    for x in xs:
        assert oracle.round_to_storage(x, "f16") == float(np.float16(x))
        assert oracle.round_to_storage(x, "f32") == float(np.float32(x))
