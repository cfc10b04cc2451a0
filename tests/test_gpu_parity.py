"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by element, on
seeded synthetic inputs (BASELINE.json configs) and the hand-derived golden fixtures."""
import os

import numpy as np
import pytest

import oracle
from synth.configs import (KINECT_VGA, TrackParams, VolumeDesc, config_single, config_tiny, init_noise, make_pst,
                           with_desc)
from synth.rng import Stream
from synth.scene import Intrinsics, analytic_fill, box_room, perturb, render_depth
from tests.fixtures import f_track_inputs, golden
from tests.parity import (assert_eval_parity, assert_last_iter_counts, assert_pose_close, assert_trace_parity,
                          close_E, track_parity)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pft():
    import paper_2509_24236_b200 as m
    m.lib()
    return m


def dev():
    return torch.device("cuda", torch.cuda.current_device())


def T(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t if dtype is None else t.to(dtype)).to(dev())


def gpu_volume(pft, desc, V=None, W=None):
    vol = pft.Volume(desc, dev())
    if V is None:
        vol.reset()
    else:
        vol.upload(V, W)
    return vol


def run_track(pft, vol, depth, intr, T_init, pst, params):
    r = vol.track(T(depth), intr, T(T_init), T(pst), params)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in r.items() if k != "ws"}


def storage_bits(x):
    x = np.asarray(x)
    return x.view(np.uint32) if x.dtype.itemsize == 4 else x.view(np.uint16)


# ------------------------------------------------------------------ golden fixtures
def test_f_track_golden(pft):
    f = f_track_inputs()
    vol = gpu_volume(pft, f["desc"], f["V"], f["W"])
    r = run_track(pft, vol, f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    a = float(np.float32(1.0 / 6.0))
    tr = r["trace"]
    # iteration 1: E_base = 0.5a, |A| = 1, P = GT, E_c = 0, s -> (1, 1)
    assert abs(tr[0, 0] - 0.5 * a) < 1e-8 and tr[0, 1] == 1 and tr[0, 16] == 0.0
    assert tr[0, 17] == pytest.approx(1.0, abs=1e-12) and tr[0, 18] == pytest.approx(1.0, abs=1e-12)
    # iteration 2: |A| = 0, s -> (0.1, 0.1)
    assert tr[1, 1] == 0 and tr[1, 17] == pytest.approx(0.1, abs=1e-12)
    np.testing.assert_allclose(r["T"], f["T_gt"], atol=1e-12)
    np.testing.assert_array_equal(r["n"], [4, 4])
    np.testing.assert_allclose(r["E"], [0.0, 0.05 * a], atol=1e-8)
    # and against the oracle
    o = oracle.OracleVolume(f["desc"], f["V"], f["W"]).track(f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    assert_trace_parity(tr, o["trace"], "F-track")
    vol.close()


def test_f_mean_golden(pft):
    """Fixture F-mean (tests/golden/f_mean.json): a two-member advantage set of non-coaxial
    rotations; the GPU's averaged pose, E_k, |A|, E(P') and s against the hand-derived closed form
    and the oracle."""
    from tests.fixtures import f_mean_closed_form, f_mean_inputs
    f = f_mean_inputs()
    cf = f_mean_closed_form()
    vol = gpu_volume(pft, f["desc"], f["V"], f["W"])
    r = run_track(pft, vol, f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    tr = r["trace"][0]
    assert tr[1] == 2
    np.testing.assert_allclose(r["E"], cf["E"], atol=1e-7)
    np.testing.assert_allclose(r["T"], cf["P"], atol=1e-12)
    assert abs(tr[16] - cf["E_c"]) < 1e-7
    assert abs(tr[17] - cf["s_next"][0]) < 2e-6
    o = oracle.OracleVolume(f["desc"], f["V"], f["W"]).track(f["depth"], f["intr"], f["T_init"], f["pst"], f["params"])
    assert_trace_parity(r["trace"], o["trace"], "F-mean")
    np.testing.assert_array_equal(r["n"], o["n"])
    vol.close()


def test_f_integrate_golden(pft):
    f = f_track_inputs()
    g = golden("f_integrate.json")
    for full in (False, True):
        vol = gpu_volume(pft, f["desc"])
        vol.integrate(T(f["depth"]), f["intr"], T(f["T_gt"]), full_sweep=full)
        V, W = [x.cpu().numpy().reshape(16, 16, 16) for x in vol.download()]
        i, j = g["column_ij"]
        exp_V = [float(eval(s)) for s in g["V"]]
        np.testing.assert_allclose(V[:, j, i], exp_V, atol=1e-7)
        np.testing.assert_array_equal(W[:, j, i], g["W"])
        assert int((W > 0).sum()) == g["updated_voxels"]
        ov = oracle.OracleVolume(f["desc"])
        ov.integrate(f["depth"], f["intr"], f["T_gt"])
        assert np.array_equal(storage_bits(V.ravel()), storage_bits(ov.V))
        assert np.array_equal(storage_bits(W.ravel()), storage_bits(ov.W))
        vol.close()


# ------------------------------------------------------------------ eval_poses (K2 in isolation)
def _pose_cloud(T_gt, seed, M, deg, cm):
    st = Stream(seed, 77)
    ab = st.symmetric(6 * M).reshape(M, 6)
    return np.stack([perturb(T_gt, a[:3], a[3:], deg, cm) for a in ab])


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_eval_poses_tiny(pft, storage):
    c = config_tiny(seed=1)
    desc = with_desc(c, storage=storage)["desc"]
    V, W = c["V"], c["W"]
    if storage == "f16":
        V, W = V.astype(np.float16), W.astype(np.float16)
    poses = np.concatenate([c["T_gt"][None], _pose_cloud(c["T_gt"], 1, 300, 3.0, 3.0),
                            _pose_cloud(c["T_gt"], 2, 60, 40.0, 60.0)])
    vol = gpu_volume(pft, desc, V, W)
    params = TrackParams(stride=1)
    r = vol.eval_poses(T(c["depth"]), c["intr"], T(poses), params)
    torch.cuda.synchronize()
    ov = oracle.OracleVolume(desc, V.view(np.uint16) if storage == "f16" else V,
                             W.view(np.uint16) if storage == "f16" else W)
    o = ov.eval_poses(c["depth"], c["intr"], poses, stride=1)
    assert vol.npoints(r["ws"]) == o["N"] == 4800
    assert_eval_parity(r["E"].cpu().numpy(), r["n"].cpu().numpy(), o, f"tiny {storage}")
    assert (o["n"] > 0).sum() > 200   # the cloud really exercises the band
    vol.close()


def test_eval_poses_single_room(pft):
    """Config S geometry (256^3 @ 1 cm, 640x480 -> 160x120 points); poses span in-band,
    partially-outside and fully-outside cases, several 8x4 tiles and the ragged last CTA."""
    c = config_single(seed=1)
    poses = np.concatenate([c["T_gt"][None], _pose_cloud(c["T_gt"], 3, 96, 8.0, 8.0),
                            _pose_cloud(c["T_gt"], 4, 31, 90.0, 150.0)])
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    r = vol.eval_poses(T(c["depth"]), c["intr"], T(poses), c["params"])
    torch.cuda.synchronize()
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).eval_poses(c["depth"], c["intr"], poses, stride=4)
    assert o["N"] == vol.npoints(r["ws"])
    assert_eval_parity(r["E"].cpu().numpy(), r["n"].cpu().numpy(), o, "single")
    vol.close()


@pytest.mark.parametrize("stride", [1, 3, 5])
def test_eval_poses_strides_and_ragged_image(pft, stride):
    """Ragged strided grids (ceil(H/s) x ceil(W/s) not multiples of the 8x4 tile) and a
    depth map with invalid pixels (0 and >= max_depth)."""
    c = config_tiny(seed=2)
    depth = c["depth"].copy()
    st = Stream(9, 9)
    holes = st.uniform(depth.size).reshape(depth.shape)
    depth[holes < 0.1] = 0
    depth[(holes >= 0.1) & (holes < 0.15)] = 9000  # 9 m >= max_depth 8 m: invalid
    depth = depth[:57, :75].copy()
    intr = Intrinsics(131.25, 131.25, 37.0, 28.0, 75, 57)
    poses = np.concatenate([c["T_gt"][None], _pose_cloud(c["T_gt"], 5, 40, 3.0, 3.0)])
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    r = vol.eval_poses(T(depth), intr, T(poses), TrackParams(stride=stride, min_inband_frac=0.3))
    torch.cuda.synchronize()
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).eval_poses(depth, intr, poses, stride=stride, rho=0.3)
    assert o["N"] == vol.npoints(r["ws"])
    assert_eval_parity(r["E"].cpu().numpy(), r["n"].cpu().numpy(), o, f"stride {stride}")
    vol.close()


# ------------------------------------------------------------------ track (whole RO loop)
@pytest.mark.parametrize("conv", [0, 1])
def test_track_tiny(pft, conv):
    c = config_tiny(seed=1)
    params = TrackParams(iters=3, stride=1, delta_conv=conv)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    r = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"], params)
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], c["pst"], params)
    assert_trace_parity(r["trace"], o["trace"], f"tiny conv={conv}")
    np.testing.assert_array_equal(r["n"], o["n"])
    assert close_E(r["E"], o["E"]).all()
    assert_pose_close(r["T"], o["T"], "tiny final")
    assert np.all(r["trace"][:, 21] == 4800)
    vol.close()


@pytest.mark.parametrize("variant", ["plain", "schedule", "high"])
def test_track_min_inband_fraction(pft, variant):
    """Reading L6 with rho = min_inband_frac > 0 through pft_track: E = 1 for a candidate whose
    in-band count is below rho N -- plain, with the F1 schedule (N changes per point set), and a rho
    high enough that many candidates (and some centres) are rejected -- every trace row and the last
    E_k / n_k against the oracle."""
    import dataclasses
    c = config_tiny(seed=2)
    base = TrackParams(iters=5, stride=1, min_inband_frac=0.3)
    params = {"plain": base, "schedule": dataclasses.replace(base, **SCHED_TINY),
              "high": dataclasses.replace(base, min_inband_frac=0.62)}[variant]
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    ov = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    r, o, _ = track_parity(lambda it: run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"],
                                                dataclasses.replace(params, iters=it)),
                           ov, c["depth"], c["intr"], c["T_init"], c["pst"], params, f"rho {variant}")
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], c["pst"], params, c["T_init"], variant)
    assert_pose_close(r["T"], o["T"], variant)
    if variant == "high":  # the fraction rule really decides something here (|A| differs from rho = 0)
        o0 = ov.track(c["depth"], c["intr"], c["T_init"], c["pst"], dataclasses.replace(params, min_inband_frac=0.0))
        assert not np.array_equal(o0["trace"][:, 1], o["trace"][:, 1])
    vol.close()


@pytest.mark.parametrize("seed", [1, 2])
def test_track_single(pft, seed):
    """Config S in full: 256^3 @1 cm, 1024 particles, 10 iterations, +-8 deg/cm init."""
    c = config_single(seed=seed)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    r = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"], c["params"])
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], c["pst"], c["params"])
    assert_trace_parity(r["trace"], o["trace"], f"single seed {seed}")
    ov = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], c["pst"], c["params"], c["T_init"],
                            f"single seed {seed}")
    assert_pose_close(r["T"], o["T"], "single final")
    vol.close()


def test_track_ragged_K_and_prefix_stable_and_deterministic(pft):
    c = config_tiny(seed=3)
    pst = make_pst(3, 37)  # not a multiple of the 32-particle CTA chunk
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    p3 = TrackParams(iters=3, stride=1)
    p2 = TrackParams(iters=2, stride=1)
    a = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, p3)
    b = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, p3)
    d = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, p2)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k]), f"non-deterministic {k}"
    assert np.array_equal(a["trace"][:2], d["trace"]), "not prefix-stable"
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], pst, p3)
    assert_trace_parity(a["trace"], o["trace"], "K=37")
    np.testing.assert_array_equal(a["n"], o["n"])
    vol.close()


def test_track_single_particle_and_empty_cloud(pft):
    c = config_tiny(seed=1)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    p = TrackParams(iters=2, stride=1)
    one = make_pst(5, 1)
    a = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], one, p)
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], one, p)
    assert_trace_parity(a["trace"], o["trace"], "K=1")
    # empty cloud: T_out = T_init, E = 1, n = 0, trace flag bit 2
    z = np.zeros_like(c["depth"])
    e = run_track(pft, vol, z, c["intr"], c["T_init"], c["pst"], p)
    np.testing.assert_array_equal(e["T"], c["T_init"])
    assert np.all(e["E"] == 1.0) and np.all(e["n"] == 0)
    assert all(int(f) & 4 for f in e["trace"][:, 19])
    vol.close()


@pytest.mark.parametrize("persistent", [True, False])
def test_track_fresh_volume_is_lost(pft, persistent):
    """Degenerate map: a reset volume (V = 1, W = 0) has no in-band cell, so every E_k = E_c = 1
    (reading L6), no particle improves on the baseline (strict <, L12), the pose never moves and
    the search size never shrinks (s-law factor 1 at E = 1): trace flags 'A empty' and 'lost' on
    every iteration, equal to the oracle -- on both tracker paths (K = 61, ragged)."""
    import subprocess
    import sys
    c = config_tiny(seed=2)
    pst = make_pst(2, 61)
    p = TrackParams(iters=3, stride=1)
    vol = gpu_volume(pft, c["desc"])
    if persistent:
        r = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, p)
    else:
        env = dict(os.environ, PFT_TRACK_PERSISTENT="0")
        code = ("import sys; sys.path.insert(0, %r); import numpy as np, torch, tests.test_gpu_parity as t; "
                "import paper_2509_24236_b200 as pft; from synth.configs import config_tiny, make_pst, TrackParams; "
                "c = config_tiny(seed=2); v = t.gpu_volume(pft, c['desc']); "
                "r = t.run_track(pft, v, c['depth'], c['intr'], c['T_init'], make_pst(2, 61), TrackParams(iters=3, stride=1)); "
                "np.savez(sys.argv[1], **{k: r[k] for k in ('T', 'E', 'n', 'trace')})") % ROOT
        out = os.path.join(os.environ.get("TMPDIR", "/tmp"), "pft_fresh_ml.npz")
        subprocess.check_call([sys.executable, "-c", code, out], env=env)
        r = dict(np.load(out))
    o = oracle.OracleVolume(c["desc"]).track(c["depth"], c["intr"], c["T_init"], pst, p)
    assert_trace_parity(r["trace"], o["trace"], "fresh volume")
    np.testing.assert_array_equal(r["T"], c["T_init"])
    assert np.all(r["E"] == 1.0) and np.all(r["n"] == 0)
    assert all((int(f) & 3) == 3 for f in r["trace"][:, 19])
    assert np.all(r["trace"][:, 17] == p.omega0_deg) and np.all(r["trace"][:, 18] == p.v0_cm)
    vol.close()


# ------------------------------------------------------------------ integration
@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_integrate_room_bit_exact(pft, storage):
    """Three frames of the room fused into a reset 128^3 volume @2 cm (GPU culled path and
    full sweep vs oracle): stored values and weights bit-identical."""
    scene = box_room(seed=4)
    desc = VolumeDesc(128, 128, 128, 0.02, (-1.28, -1.28, -1.28), 0.06, storage=storage)
    intr = Intrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    from synth.configs import room_gt_pose
    T_gt = room_gt_pose(scene, 4)
    vol = gpu_volume(pft, desc)
    vol_full = gpu_volume(pft, desc)
    ov = oracle.OracleVolume(desc)
    for f in range(3):
        Tf = perturb(T_gt, [0.0, 0.0, 0.1 * f], [0.05 * f, 0.0, 0.0], 10.0, 10.0)
        depth = render_depth(scene, intr, Tf, Stream(4, 4_000_000 + f))
        vol.integrate(T(depth), intr, T(Tf))
        vol_full.integrate(T(depth), intr, T(Tf), full_sweep=True)
        n_ora = ov.integrate(depth, intr, Tf)
        st = vol.integrate_stats()  # the culled path's work counters: updated voxels = the definition's
        assert st["updated_voxels"] == n_ora, (st, n_ora)
        assert 0 < st["free_bricks"] <= st["kept_bricks"] and st["dirty_cell_bricks"] > 0
        assert vol_full.integrate_stats()["updated_voxels"] == -1
    V, W = [x.cpu().numpy() for x in vol.download()]
    Vf, Wf = [x.cpu().numpy() for x in vol_full.download()]
    assert np.array_equal(storage_bits(V), storage_bits(Vf)) and np.array_equal(storage_bits(W), storage_bits(Wf))
    assert np.array_equal(storage_bits(V), storage_bits(ov.V)), \
        f"{int((storage_bits(V) != storage_bits(ov.V)).sum())} voxel values differ"
    assert np.array_equal(storage_bits(W), storage_bits(ov.W))
    assert vol.checksum() == vol_full.checksum()
    assert (ov.weights_f64() > 0).sum() > 10000
    vol.close()
    vol_full.close()


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_integrate_camera_plane_cone(pft, storage):
    """The cull of boxes straddling the camera plane (integrate.cu box_class: culled only when
    laterally outside the frustum cone at their far depth): the camera sits inside a 64^3 @ 1 cm
    volume, rotated off the grid axes, facing a surface 3-20 cm away, so voxels with 0 < z < 20 cm
    near the optical axis are updated while their bricks straddle z = 0.  Culled path and full sweep
    against the oracle bit for bit, and the culled path's updated-voxel count equals the oracle's."""
    desc = VolumeDesc(64, 64, 64, 0.01, (-0.32, -0.32, -0.32), 0.03, storage=storage)
    intr = Intrinsics(80.0, 80.0, 39.5, 29.5, 80, 60)
    T0 = perturb(np.hstack([np.eye(3), np.zeros((3, 1))]), [0.3, -0.2, 0.1], [0.3, -0.2, 0.1], 25.0, 0.5)
    v, u = np.mgrid[0:60, 0:80]
    depth = (30 + (u + 2 * v) % 171).astype(np.uint16)  # 3 .. 20 cm, a ramp with steps
    depth[::7, ::5] = 0                                  # scattered invalid pixels
    vol = gpu_volume(pft, desc)
    vfull = gpu_volume(pft, desc)
    ov = oracle.OracleVolume(desc)
    for f in range(2):
        vol.integrate(T(depth), intr, T(T0))
        vfull.integrate(T(depth), intr, T(T0), full_sweep=True)
        n_ora = ov.integrate(depth, intr, T0)
        assert vol.integrate_stats()["updated_voxels"] == n_ora > 100
    for v_ in (vol, vfull):
        V, W = [x.cpu().numpy() for x in v_.download()]
        assert np.array_equal(storage_bits(V), storage_bits(ov.V)), \
            f"{int((storage_bits(V) != storage_bits(ov.V)).sum())} voxel values differ"
        assert np.array_equal(storage_bits(W), storage_bits(ov.W))
    vol.close()
    vfull.close()


@pytest.mark.parametrize("voxel", [0.0625, 0.05])
@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_integrate_grid_aligned_pixel_ties(pft, voxel, storage):
    """Adversarial projection decisions (integrate.cu pixel_of): a camera at the world origin with
    identity rotation looking along +z over voxel centres x = s(i - 24), z = s k, fx = fy = 60,
    cx = cy = 31.5, so fx x / z + cx + 1/2 = 60 (i - 24)/k + 32 lands exactly on (s = 1/16, binary)
    or within ulps of (s = 0.05) integer pixel boundaries for many voxels: the guarded reciprocal
    path must hand every such voxel to the exact division and decide the same pixel as the oracle.
    A frontal plane at 1.5 m, fused 3 times (free space carved to V = 1, then the V' = 1 shortcut),
    culled and full sweep, against the oracle bit for bit."""
    n = 48
    desc = VolumeDesc(n, n, n, voxel, (-voxel * 24.5, -voxel * 24.5, -voxel * 0.5), 2.5 * voxel, storage=storage)
    intr = Intrinsics(60.0, 60.0, 31.5, 31.5, 64, 64)
    T0 = np.zeros((3, 4))
    T0[:, :3] = np.eye(3)
    depth = np.full((64, 64), 1500, dtype=np.uint16)
    depth[:, :7] = 0            # an invalid band
    depth[40:, 30:] = 2200      # a step
    vol = gpu_volume(pft, desc)
    vfull = gpu_volume(pft, desc)
    ov = oracle.OracleVolume(desc)
    for _ in range(3):
        vol.integrate(T(depth), intr, T(T0))
        vfull.integrate(T(depth), intr, T(T0), full_sweep=True)
        ov.integrate(depth, intr, T0)
    for v in (vol, vfull):
        V, W = [x.cpu().numpy() for x in v.download()]
        assert np.array_equal(storage_bits(V), storage_bits(ov.V)), \
            f"{int((storage_bits(V) != storage_bits(ov.V)).sum())} voxel values differ"
        assert np.array_equal(storage_bits(W), storage_bits(ov.W))
    assert (ov.weights_f64() == 3).sum() > 5000
    vol.close()
    vfull.close()


def test_upload_download_roundtrip_and_checksum(pft):
    desc = VolumeDesc(37, 18, 23, 0.05, (0.0, 0.0, 0.0), 0.2)   # ragged bricks on every axis
    st = Stream(11, 11)
    V = st.symmetric(37 * 18 * 23).astype(np.float32)
    W = np.floor(st.uniform(37 * 18 * 23) * 5).astype(np.float32)
    vol = gpu_volume(pft, desc, V, W)
    V2, W2 = [x.cpu().numpy() for x in vol.download()]
    assert np.array_equal(V, V2) and np.array_equal(W, W2)
    h1 = vol.checksum()
    vol2 = gpu_volume(pft, desc, V, W)
    assert vol2.checksum() == h1
    W[5] += 1
    vol2.upload(V, W)
    assert vol2.checksum() != h1
    vol.close()
    vol2.close()


def test_sequence_track_then_integrate(pft):
    """Config-Q-like loop at reduced size: frame 0 integrated at GT, then 3 frames of
    track (K=256, 5 iterations) + integrate at the tracked pose, GPU and oracle in lock step;
    voxels bit-exact after every frame, poses within 1e-4."""
    from synth.configs import shaky_trajectory
    from synth.scene import compose, inverse
    scene = box_room(seed=6)
    desc = VolumeDesc(160, 160, 160, 0.02, (-1.6, -1.6, -1.6), 0.06)
    intr = Intrinsics(262.5, 262.5, 159.5, 119.5, 320, 240)
    gt = shaky_trajectory(scene, 40, seed=6)
    pst = make_pst(6, 256)
    params = TrackParams(iters=5, stride=4)
    vol = gpu_volume(pft, desc)
    ov = oracle.OracleVolume(desc)
    d0 = render_depth(scene, intr, gt[0], Stream(6, 4_000_000))
    vol.integrate(T(d0), intr, T(gt[0]))
    ov.integrate(d0, intr, gt[0])
    P_prev = gt[0]
    for t in range(1, 4):
        depth = render_depth(scene, intr, gt[t], Stream(6, 4_000_000 + t))
        rel = init_noise(6, t, compose(inverse(gt[t - 1]), gt[t]), 5.0, 5.0)
        T_init = compose(P_prev, rel)
        r = run_track(pft, vol, depth, intr, T_init, pst, params)
        o = ov.track(depth, intr, T_init, pst, params)
        assert_trace_parity(r["trace"], o["trace"], f"frame {t}")
        P_prev = o["T"]
        vol.integrate(T(depth), intr, T(P_prev))
        ov.integrate(depth, intr, P_prev)
        V, W = [x.cpu().numpy() for x in vol.download()]
        assert np.array_equal(storage_bits(V), storage_bits(ov.V)), f"frame {t}: values differ"
        assert np.array_equal(storage_bits(W), storage_bits(ov.W)), f"frame {t}: weights differ"
    vol.close()


@pytest.mark.parametrize("cfg", ["tiny", "tiny16", "single", "tiny_sched", "single_topk", "tiny_bigK"])
def test_persistent_tracker_bit_identical_to_multilaunch(cfg, tmp_path):
    """The single-launch persistent tracker (G = 1 default) and the multi-launch path (used for
    G > 1) share their arithmetic helpers and fixed reduction trees: outputs must be bit-identical."""
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_track.py")
    outs = {}
    for mode in ("0", "1"):
        env = dict(os.environ, PFT_TRACK_PERSISTENT=mode)
        f = str(tmp_path / f"{cfg}_{mode}.npz")
        subprocess.check_call([sys.executable, helper, cfg, "1", f], env=env)
        outs[mode] = np.load(f)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(outs["0"][k], outs["1"][k]), k
    # and the multi-launch run (the G > 1 code path) against the oracle
    from tests.helpers.run_track import make_case
    c, params = make_case(cfg, 1)
    _assert_vs_oracle(dict(outs["0"]), c, c["pst"], params, f"multi-launch {cfg}")


@pytest.mark.parametrize("cfg", ["single", "tiny_bigK"])
def test_persistent_item_order_bit_identical(cfg, tmp_path):
    """P2's work order does not change any result (every evaluation term is its own fixed-point
    integer): the SM-paired static item positions (default) and the plain CTA order
    (PFT_PAIR_SM=0) give bit-identical outputs.  tiny_bigK (K = 70000: >= 1 static item per warp
    at 296 CTAs) exercises the static items themselves; the persistent run of the
    same case is compared with the multi-launch path and the oracle above."""
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_track.py")
    outs = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"{cfg}_pair{mode}.npz")
        subprocess.check_call([sys.executable, helper, cfg, "1", f], env=dict(os.environ, PFT_PAIR_SM=mode))
        outs[mode] = np.load(f)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(outs["0"][k], outs["1"][k]), k


_ORACLE_CACHE = {}


def _oracle_run(key, c, pst, params):
    """The oracle's run of a case (cached per key: the sharded tests compare several G with it)."""
    if key not in _ORACLE_CACHE:
        V, W = c["V"], c["W"]
        if c["desc"].storage == "f16":
            V, W = np.asarray(V).view(np.uint16), np.asarray(W).view(np.uint16)
        ov = oracle.OracleVolume(c["desc"], V, W)
        _ORACLE_CACHE[key] = (ov, ov.track(c["depth"], c["intr"], c["T_init"], pst, params))
    return _ORACLE_CACHE[key]


def _assert_vs_oracle(r, c, pst, params, what, key=None):
    """Trace, last-iteration E_k / n_k and pose of a GPU run against the oracle (north_star bar)."""
    ov, o = _oracle_run(key or what, c, pst, params)
    assert_trace_parity(r["trace"], o["trace"], what)
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], pst, params, c["T_init"], what)
    assert_pose_close(r["T"], o["T"], what)


# ------------------------------------------------------------------ NEXT rows F1 / F3
SCHED_TINY = dict(nsched=3, sched_K=(64, 40, 24, 0), sched_sx=(2, 2, 4, 0), sched_sy=(1, 2, 2, 0))


@pytest.mark.parametrize("variant", ["schedule", "schedule_guard", "weighted", "weighted_guard_world", "topk",
                                     "topk_schedule_guard"])
def test_track_next_rows_tiny(pft, variant):
    """F1 (cycled K / 2-D stride schedule, baseline recomputed on a new point set) and F3 (guard,
    weighted mean) against the oracle: every iteration's trace row and the last E_k / n_k."""
    import dataclasses
    c = config_tiny(seed=2)
    base = TrackParams(iters=7, stride=1)
    kw = {"schedule": dict(SCHED_TINY), "schedule_guard": dict(SCHED_TINY, guard=1),
          "weighted": dict(update_rule=1), "weighted_guard_world": dict(update_rule=1, guard=1, delta_conv=1),
          "topk": dict(update_rule=2, topk=8), "topk_schedule_guard": dict(SCHED_TINY, update_rule=2, topk=5, guard=1)}[variant]
    params = dataclasses.replace(base, **kw)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    r = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"], params)
    ov = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    o = ov.track(c["depth"], c["intr"], c["T_init"], c["pst"], params)
    assert_trace_parity(r["trace"], o["trace"], variant)
    np.testing.assert_array_equal(r["trace"][:, 20:24], o["trace"][:, 20:24])
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], c["pst"], params, c["T_init"], variant)
    assert_pose_close(r["T"], o["T"], variant)
    vol.close()


@pytest.mark.parametrize("stop", ["min_search", "stall"])
def test_track_stop_rules(pft, stop):
    """F1 min-search stop and F3 stall stop: the same stop iteration as the oracle, later trace rows
    flagged not-run (bit 5), T_out = the last row's pose."""
    import dataclasses
    if stop == "stall":
        f = f_track_inputs()
        desc, V, W, depth, intr, T0, pst = f["desc"], f["V"], f["W"], f["depth"], f["intr"], f["T_init"], f["pst"]
        params = dataclasses.replace(f["params"], iters=4, stall_limit=1)
    else:
        c = config_tiny(seed=1)
        desc, V, W, depth, intr, T0, pst = c["desc"], c["V"], c["W"], c["depth"], c["intr"], c["T_init"], c["pst"]
        params = TrackParams(iters=8, stride=2, min_search_deg=4.0, min_search_cm=1e9)
    vol = gpu_volume(pft, desc, V, W)
    r = run_track(pft, vol, depth, intr, T0, pst, params)
    o = oracle.OracleVolume(desc, V, W).track(depth, intr, T0, pst, params)
    ran = (o["trace"][:, 19].astype(int) & 32) == 0
    assert 0 < ran.sum() < params.iters
    assert np.array_equal(r["trace"][:, 19], o["trace"][:, 19])
    assert_trace_parity(r["trace"][ran], o["trace"][ran], stop)
    assert np.all(r["trace"][~ran] == o["trace"][~ran])
    assert_pose_close(r["T"], o["T"], stop)
    vol.close()


# ------------------------------------------------------------------ NEXT row F4
def _sorted_rows(p):
    p = np.asarray(p)
    return p[np.lexsort((p[:, 2], p[:, 1], p[:, 0]))] if len(p) else p.reshape(0, 3)


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_extract_surface_bit_exact(pft, storage):
    """F4 zero-crossing points of a fused room volume (and of config T's analytic fill): the GPU's
    unordered list equals the oracle's, sorted, bit for bit; a fresh volume yields none."""
    from synth.configs import room_gt_pose
    scene = box_room(seed=5)
    desc = VolumeDesc(96, 96, 96, 0.03, (-1.44, -1.44, -1.44), 0.09, storage=storage)
    intr = Intrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    T0 = room_gt_pose(scene, 5)
    vol = gpu_volume(pft, desc)
    assert len(vol.extract_surface()) == 0
    ov = oracle.OracleVolume(desc)
    for f in range(3):
        Tf = perturb(T0, [0.0, 0.0, 0.15 * f], [0.0, 0.04 * f, 0.0], 10.0, 10.0)
        depth = render_depth(scene, intr, Tf, Stream(5, 4_000_000 + f))
        vol.integrate(T(depth), intr, T(Tf))
        ov.integrate(depth, intr, Tf)
    g = vol.extract_surface().cpu().numpy()
    o = ov.extract()
    assert len(o) > 2000 and len(g) == len(o)
    assert np.array_equal(_sorted_rows(g), _sorted_rows(o))
    # truncated output: the count still reports every crossing
    cnt_only = vol.extract_surface(max_points=100)
    assert len(cnt_only) == 100
    vol.close()
    c = config_tiny(seed=1)
    vt = gpu_volume(pft, c["desc"], c["V"], c["W"])
    assert np.array_equal(_sorted_rows(vt.extract_surface().cpu().numpy()),
                          _sorted_rows(oracle.OracleVolume(c["desc"], c["V"], c["W"]).extract()))
    vt.close()


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_extract_surface_dense_crossings(pft, storage):
    """A checkerboard volume (every voxel pair with a sign change, ragged 18 x 13 x 11 grid): up to 3
    crossings per voxel, more than a warp's 64-point shared-memory buffer holds for one brick (the
    kernel's direct-append path) and several buffer flushes per warp; bit-equal to the oracle."""
    nx, ny, nz = 18, 13, 11
    desc = VolumeDesc(nx, ny, nz, 0.05, (-0.4, -0.3, -0.2), 0.15, storage=storage)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    V = np.where((i + j + k) % 2 == 0, 0.5, -0.25).astype(np.float32)
    V[2, 3, 4] = 0.0  # a zero value: crossings with it count only against a non-zero neighbour
    W = np.ones_like(V)
    W[5, 6, 7] = 0.0  # an unobserved voxel breaks its crossings
    if storage == "f16":
        V, W = V.astype(np.float16), W.astype(np.float16)
    vol = gpu_volume(pft, desc, V, W)
    g = vol.extract_surface().cpu().numpy()
    o = oracle.OracleVolume(desc, V, W).extract()
    assert len(o) > 3 * nx * ny * nz // 2 and len(g) == len(o)
    assert np.array_equal(_sorted_rows(g), _sorted_rows(o))
    vol.close()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_bit_identical(pft, G):  # noqa: C901
    """SURVEY.md §4 "virtual shards": the multi-GPU code path (rank q evaluates template rows
    [q*ceil(K/G), ...), per-particle records all-gathered, identical update everywhere), emulated on
    one GPU with sequential shards, equals the 1-rank result bit for bit -- on config S and on a
    scheduled/guarded/weighted run with a ragged K."""
    import dataclasses
    for name in ("single", "tiny_sched", "single_topk"):
        if name == "single":
            c = config_single(seed=1)
            pst, params = c["pst"], c["params"]
        elif name == "single_topk":
            c = config_single(seed=2)
            pst, params = c["pst"], dataclasses.replace(c["params"], update_rule=2, topk=32, iters=4)
        else:
            c = config_tiny(seed=2)
            pst = make_pst(2, 61)
            params = dataclasses.replace(TrackParams(iters=7, stride=1, guard=1, update_rule=1), **SCHED_TINY)
        ref = gpu_volume(pft, c["desc"], c["V"], c["W"])
        a = run_track(pft, ref, c["depth"], c["intr"], c["T_init"], pst, params)
        ref.close()
        vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
        vol.comm_init_virtual(G)
        b = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, params)
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(a[k], b[k]), (name, G, k)
        _assert_vs_oracle(b, c, pst, params, f"virtual shards G={G} {name}", key=name)
        vol.close()


def _fused_cases():
    import dataclasses
    out = []
    c = config_single(seed=1)
    out.append(("single", c, c["pst"], c["params"]))
    c = config_single(seed=2)
    out.append(("single_topk", c, c["pst"], dataclasses.replace(c["params"], update_rule=2, topk=32, iters=4)))
    c = config_tiny(seed=2)
    out.append(("tiny_sched", c, make_pst(2, 61),
                dataclasses.replace(TrackParams(iters=7, stride=1, guard=1, update_rule=1), **SCHED_TINY)))
    c = config_tiny(seed=1)
    out.append(("tiny_stop", c, c["pst"], TrackParams(iters=8, stride=2, min_search_deg=4.0, min_search_cm=1e9)))
    c = dict(with_desc(config_tiny(seed=3), storage="f16"))
    c["V"], c["W"] = c["V"].astype(np.float16), c["W"].astype(np.float16)
    out.append(("tiny16_world", c, c["pst"], TrackParams(iters=4, stride=1, delta_conv=1)))
    return out


@pytest.mark.parametrize("G", [2, 3, 8])
def test_fused_exchange_bit_identical(pft, G):
    """F2 fused exchange (include/pft.h pft_comm_init_virtual_fused): G rank groups of CTAs in ONE
    persistent launch, each evaluating its shard and pushing its per-particle records into every
    group's exchange buffer, waiting on the same monotone counters the multi-GPU path uses.  Equals
    the 1-rank run bit for bit (T, every E_k / n_k, every trace row), including a top-k run, a
    scheduled ragged-K weighted/guarded run (K = 61: empty and ragged shards) and an early stop."""
    for name, c, pst, params in _fused_cases():
        ref = gpu_volume(pft, c["desc"], c["V"], c["W"])
        a = run_track(pft, ref, c["depth"], c["intr"], c["T_init"], pst, params)
        ref.close()
        vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
        vol.comm_init_virtual(G, fused=True)
        ws_bytes = vol.workspace(c["intr"], pst.shape[0], params).numel()
        b = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, params)
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(a[k], b[k]), (name, G, k)
        _assert_vs_oracle(b, c, pst, params, f"fused exchange G={G} {name}", key="fused " + name)
        # a second call on the same workspace: the exchange counters continue from the stored
        # round count (no reset handshake) and the results repeat
        b2 = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, params)
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(a[k], b2[k]), (name, G, k, "second call")
        assert vol.workspace(c["intr"], pst.shape[0], params).numel() == ws_bytes
        vol.close()


def test_fused_exchange_one_launch(pft):
    """The fused G-rank emulation is one kernel launch per pft_track call (no per-iteration
    collective or host round trip)."""
    c = config_single(seed=1)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    vol.comm_init_virtual(4, fused=True)
    run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"], c["params"])
    n0 = pft.launch_count()
    run_track(pft, vol, c["depth"], c["intr"], c["T_init"], c["pst"], c["params"])
    assert pft.launch_count() - n0 == 1
    vol.close()


def test_fused_exchange_counters_follow_the_layout(pft):
    """F2 emulation: consecutive calls on ONE workspace buffer with different K (so the exchange
    counters move) -- each call still equals its 1-rank run (the counters are re-zeroed whenever
    the layout changes, include/pft.h)."""
    c = config_single(seed=1)
    ref = gpu_volume(pft, c["desc"], c["V"], c["W"])
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    vol.comm_init_virtual(3, fused=True)
    big = torch.empty(1 << 28, dtype=torch.uint8, device=dev())
    vol.workspace = lambda intr, K, params: big
    for K in (1024, 1000, 1024, 517):
        pst = make_pst(4, K)
        a = run_track(pft, ref, c["depth"], c["intr"], c["T_init"], pst, c["params"])
        b = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, c["params"])
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(a[k], b[k]), (K, k)
    ref.close()
    vol.close()


def test_debug_build_bounds_checked(tmp_path):
    """The PFT_DEBUG build (every mask / record address bounds- and alignment-checked in the
    evaluation, every brick entry, depth pixel and dirty cell-brick in the integration, a trap on a
    bad one; DESIGN.md §9's stale-register hazard would show up here) runs config S, a top-k run, the
    fp16 volume and fp32 / fp16 integrations with results bit-identical to the product build."""
    import subprocess
    import sys
    lib = str(tmp_path / "libpft_debug.so")
    subprocess.check_call(["sh", os.path.join(ROOT, "paper_2509_24236_b200", "csrc", "build.sh"), lib, "-DPFT_DEBUG"])
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_track.py")
    for cfg in ("single", "single_topk", "tiny16"):
        outs = {}
        for name, env in (("prod", dict(os.environ)), ("debug", dict(os.environ, PFT_LIB=lib))):
            f = str(tmp_path / f"{cfg}_{name}.npz")
            subprocess.check_call([sys.executable, helper, cfg, "1", f], env=env)
            outs[name] = np.load(f)
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(outs["prod"][k], outs["debug"][k]), (cfg, k)
    # and the culled integration (brick entries, pixel indices and dirty cell-bricks checked)
    ihelper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_integrate.py")
    for storage in ("f32", "f16"):
        outs = {}
        for name, env in (("prod", dict(os.environ)), ("debug", dict(os.environ, PFT_LIB=lib))):
            f = str(tmp_path / f"integ_{storage}_{name}.npz")
            subprocess.check_call([sys.executable, ihelper, storage, f], env=env)
            outs[name] = np.load(f)
        for k in ("V", "W", "stats", "checksum"):
            assert np.array_equal(outs["prod"][k], outs["debug"][k]), (storage, k)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_point_shards_bit_identical(pft, G):
    """F2b point-sharded partition (include/pft.h pft_comm_set_partition), emulated on one GPU with G
    virtual ranks: every rank evaluates all K_i particles on its contiguous slice of point tiles and
    the fixed-point sums -- per particle and of the centre -- are added across the slices (what the
    NCCL all-reduce does across GPUs).  Equals the 1-rank run bit for bit (config S, top-k, a
    scheduled ragged-K weighted/guarded run) and the oracle."""
    import dataclasses
    cases = []
    c = config_single(seed=1)
    cases.append(("single", c, c["pst"], c["params"]))
    c = config_single(seed=2)
    cases.append(("single_topk", c, c["pst"], dataclasses.replace(c["params"], update_rule=2, topk=32, iters=4)))
    c = config_tiny(seed=2)
    cases.append(("tiny_sched", c, make_pst(2, 61),
                  dataclasses.replace(TrackParams(iters=7, stride=1, guard=1, update_rule=1), **SCHED_TINY)))
    for name, c, pst, params in cases:
        ref = gpu_volume(pft, c["desc"], c["V"], c["W"])
        a = run_track(pft, ref, c["depth"], c["intr"], c["T_init"], pst, params)
        ref.close()
        vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
        vol.comm_init_virtual(G)
        vol.set_partition(True)
        b = run_track(pft, vol, c["depth"], c["intr"], c["T_init"], pst, params)
        for k in ("T", "E", "n", "trace"):
            assert np.array_equal(a[k], b[k]), (name, G, k)
        _assert_vs_oracle(b, c, pst, params, f"point shards G={G} {name}", key="pts " + name)
        vol.close()


def test_point_partition_rejected_with_peer_exchange(pft):
    c = config_tiny(seed=1)
    vol = gpu_volume(pft, c["desc"], c["V"], c["W"])
    vol.comm_init_virtual(4, fused=True)
    with pytest.raises(pft.PftError, match="UNSUPPORTED"):
        vol.set_partition(True)
    vol.close()


def test_pose_compose(pft):
    """pft_pose_compose (device-side chaining of the sequence driver's T_init = P_{t-1} rel_t) against
    the rigid-transform product."""
    from synth.scene import compose
    st = Stream(21, 21)
    for _ in range(5):
        A = perturb(np.eye(3, 4), st.symmetric(3), st.symmetric(3), 60.0, 200.0)
        B = perturb(np.eye(3, 4), st.symmetric(3), st.symmetric(3), 60.0, 200.0)
        out = pft.pose_compose(T(A), T(B)).cpu().numpy()
        np.testing.assert_allclose(out, compose(A, B), atol=1e-14)
        a_dev = T(A)
        pft.pose_compose(a_dev, T(B), out=a_dev)  # in place
        np.testing.assert_allclose(a_dev.cpu().numpy(), compose(A, B), atol=1e-14)


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_integrate_fused_launch_identical(storage, tmp_path):
    """The opt-in single cooperative integration launch (PFT_INTEGRATE_FUSED=1: pyramid, both cull
    levels, fusion and record refresh separated by grid barriers) and the default separate kernels
    run the same device functions: bit-identical volumes, checksums and work counters."""
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_integrate.py")
    outs = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"{storage}_{mode}.npz")
        subprocess.check_call([sys.executable, helper, storage, f], env=dict(os.environ, PFT_INTEGRATE_FUSED=mode))
        outs[mode] = np.load(f)
    for k in ("V", "W", "stats", "checksum"):
        assert np.array_equal(outs["0"][k], outs["1"][k]), k
    assert outs["0"]["stats"][:, 2].min() > 1000


@pytest.mark.parametrize("storage", ["f32", "f16"])
def test_integrate_pdl_launch_identical(storage, tmp_path):
    """The integration chain launched with programmatic dependent launch (default) and as plain
    stream-ordered kernels (PFT_PDL=0): bit-identical volumes, checksums and work counters (each
    kernel waits on griddepcontrol before reading its predecessor's output)."""
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "run_integrate.py")
    outs = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"{storage}_pdl{mode}.npz")
        subprocess.check_call([sys.executable, helper, storage, f], env=dict(os.environ, PFT_PDL=mode))
        outs[mode] = np.load(f)
    for k in ("V", "W", "stats", "checksum"):
        assert np.array_equal(outs["0"][k], outs["1"][k]), k
    assert outs["0"]["stats"][:, 2].min() > 1000


@pytest.mark.parametrize("case", ["ragged", "far_principal_point", "tiny_image", "huge_image"])
def test_integrate_edge_cases(pft, case):
    """Culled integration edge cases against the full sweep and the oracle, bit for bit:
    ragged volume dims (partial bricks and super-bricks on every axis), a principal point beyond
    2^19 px (pixel_of's fast path off: every projection decided by the exact division, all outside
    the image), a 7 x 5 image (a single pyramid tile), and a 2048 x 1536 image (the pyramid does not
    fit: full-sweep fallback)."""
    scene = box_room(seed=7)
    from synth.configs import room_gt_pose
    T0 = room_gt_pose(scene, 7)
    if case == "ragged":
        desc = VolumeDesc(37, 50, 45, 0.06, (-1.11, -1.5, -1.35), 0.15)
        intr = Intrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    elif case == "far_principal_point":
        desc = VolumeDesc(64, 64, 64, 0.04, (-1.28, -1.28, -1.28), 0.12)
        intr = Intrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    elif case == "tiny_image":
        desc = VolumeDesc(64, 64, 64, 0.04, (-1.28, -1.28, -1.28), 0.12)
        intr = Intrinsics(3.0, 3.0, 3.0, 2.0, 7, 5)
    else:
        desc = VolumeDesc(64, 64, 64, 0.04, (-1.28, -1.28, -1.28), 0.12)
        intr = Intrinsics(1680.0, 1680.0, 1023.5, 767.5, 2048, 1536)
    depth = render_depth(scene, intr, T0, Stream(7, 4_000_000))
    if case == "far_principal_point":
        intr = Intrinsics(131.25, 131.25, 79.5 + 600000.0, 59.5, 160, 120)
    vol, vfull = gpu_volume(pft, desc), gpu_volume(pft, desc)
    ov = oracle.OracleVolume(desc)
    n_ora = 0
    for f in range(2):
        Tf = perturb(T0, [0.0, 0.05 * f, 0.0], [0.0, 0.0, 0.03 * f], 10.0, 10.0)
        vol.integrate(T(depth), intr, T(Tf))
        vfull.integrate(T(depth), intr, T(Tf), full_sweep=True)
        n_ora = ov.integrate(depth, intr, Tf)
        st = vol.integrate_stats()
        assert st["updated_voxels"] in (n_ora, -1), (st, n_ora)
    for v in (vol, vfull):
        V, W = [x.cpu().numpy() for x in v.download()]
        assert np.array_equal(storage_bits(V), storage_bits(ov.V)), f"{case}: {int((storage_bits(V) != storage_bits(ov.V)).sum())} values differ"
        assert np.array_equal(storage_bits(W), storage_bits(ov.W))
    if case == "far_principal_point":
        assert (ov.weights_f64() > 0).sum() == 0
    else:
        assert (ov.weights_f64() > 0).sum() > 0
    vol.close()
    vfull.close()


@pytest.mark.parametrize("partition", ["particles", "points"])
@pytest.mark.parametrize("cfg", ["single", "tiny_sched", "single_topk"])
def test_single_rank_nccl_collectives(cfg, partition, tmp_path):
    """The NCCL plumbing on real collectives: a single-rank communicator (torch.distributed world
    size 1) makes pft_track take the multi-launch collective path -- ncclAllGather of the particle
    records, or (F2b) ncclAllReduce of the per-particle and centre fixed-point sums, with the async
    error polled after each -- and its results equal the plain run bit for bit."""
    import socket
    import subprocess
    import sys
    helpers = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers")
    ref = str(tmp_path / "ref.npz")
    subprocess.check_call([sys.executable, os.path.join(helpers, "run_track.py"), cfg, "1", ref])
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = str(sk.getsockname()[1])
    sk.close()
    f = str(tmp_path / "nccl.npz")
    subprocess.check_call([sys.executable, os.path.join(helpers, "run_nccl1.py"), cfg, partition, f, port])
    a, b = np.load(ref), np.load(f)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k]), k
    assert int(b["launches"][0]) > 10   # the multi-launch path (kernels + collectives per iteration)
