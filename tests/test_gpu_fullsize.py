"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
config W (512^3 fp32, K = 4096 full 10-iteration trace; K = 65536 sampled), config Q (512^3 fp32)
and config L (1024^3 fp16) as short GPU/oracle lock-step sequences (track + integrate)."""
import dataclasses

import numpy as np
import pytest

import oracle
from synth.configs import Sequence, TrackParams, config_sweep, init_noise
from synth.rng import Stream
from synth.scene import compose, inverse
from tests.parity import (E_TIE, assert_eval_parity, assert_last_iter_counts, assert_pose_close, assert_trace_parity,
                          close_E, track_parity)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev():
    return torch.device("cuda", torch.cuda.current_device())


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev())


def bits(x):
    x = np.asarray(x)
    return x.view(np.uint32) if x.dtype.itemsize == 4 else x.view(np.uint16)


@pytest.fixture(scope="module")
def sweep():
    c = config_sweep(seed=1, K=65536, iters=10)     # 512^3 analytic fill of the room (~20 s on the host)
    import paper_2509_24236_b200 as pft
    vol = pft.Volume(c["desc"], dev())
    vol.upload(c["V"], c["W"])
    ov = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    yield c, vol, ov
    vol.close()


_W4096 = {}


def _w4096_oracle(c, ov):
    """The oracle's config-W K = 4096 run (shared by the tests of the sharded paths)."""
    if "o" not in _W4096:
        _W4096["o"] = ov.track(c["depth"], c["intr"], c["T_init"], c["pst"][:4096].copy(), TrackParams(iters=10, stride=4))
    return _W4096["o"]


def _np(r):
    return {k: r[k].cpu().numpy() for k in ("T", "E", "n", "trace")}


def _w4096_vs_oracle(r, c, ov, what):
    pst = c["pst"][:4096].copy()
    params = TrackParams(iters=10, stride=4)
    o = _w4096_oracle(c, ov)
    assert_trace_parity(r["trace"], o["trace"], what)
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], pst, params, c["T_init"], what)
    assert_pose_close(r["T"], o["T"], what)


def test_sweep_W_k4096_full_trace(sweep):
    """Config W, K = 4096: the whole 10-iteration RO run, every iteration's |A|, E, s and pose and the
    last iteration's per-particle E_k / n_k against the oracle (margin-aware: an advantage-set
    difference must be a fitness tie, then the oracle is shadowed, tests/parity.py)."""
    c, vol, ov = sweep
    pst = c["pst"][:4096].copy()
    params = TrackParams(iters=10, stride=4)

    def run(iters):
        p = TrackParams(iters=iters, stride=4)
        r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(pst), p)
        torch.cuda.synchronize()
        return _np(r)
    r, o, _ = track_parity(run, ov, c["depth"], c["intr"], c["T_init"], pst, params, "W K=4096")
    assert_last_iter_counts(r["n"], r["E"], o, ov, c["depth"], c["intr"], pst, params, c["T_init"], "W K=4096")
    assert_pose_close(r["T"], o["T"])


def test_sweep_W_k65536_sampled(sweep):
    """Config W, K = 65536 in the bench's launch configuration: all 65536 E_k / n_k of the first
    iteration computed on the GPU; 1024 of them (every 64th particle) recomputed one by one by the
    oracle from the paper's definition (candidate = dP_k(s1) T_init, eq. E)."""
    c, vol, ov = sweep
    params = TrackParams(iters=1, stride=4)
    r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(c["pst"]), params)
    torch.cuda.synchronize()
    E, n = r["E"].cpu().numpy(), r["n"].cpu().numpy()
    ks = np.arange(0, 65536, 64)
    poses = []
    for k in ks:
        dR, _, u = oracle.delta(c["pst"][k], params.omega0_deg, params.v0_cm)
        poses.append(oracle.apply_delta(dR, u, c["T_init"], 0))
    o = ov.eval_poses(c["depth"], c["intr"], np.stack(poses), stride=4)
    assert_eval_parity(E[ks], n[ks], o, "W K=65536 sampled")
    # the centre and the advantage-set size of the iteration, from the same definitions
    pts = oracle.backproject(c["depth"], c["intr"], 4)
    Ec, _, _ = ov.fitness(pts, c["T_init"])
    tr = r["trace"].cpu().numpy()[0]
    assert close_E(tr[0], Ec)
    assert tr[1] == int((E < tr[0]).sum())
    assert (n > 0).sum() > 1000


def _ate_cm(traj, gt):
    """ATE-RMSE in cm of the camera centres (no alignment; SPEC.md:98-115 raw variant)."""
    d = np.array([np.linalg.norm(np.asarray(a)[:, 3] - np.asarray(g)[:, 3]) for a, g in zip(traj, gt)])
    return float(np.sqrt(np.mean(d ** 2)) * 100.0)


def _lockstep(kind, n_frames, K, check_frames, iters=10):
    """GPU and oracle in lock step over the first n_frames of the sequence (SURVEY.md §8(c-4) item 5,
    §8(d-6)): frame 0 fused at GT (L24); then per frame t, T_init = P_{t-1} (GT_{t-1}^-1 GT_t (+) noise)
    -- config Q's chained network stand-in (L25) on the oracle's previous pose -- tracked by both
    (whole-run parity, margin-aware), and both fuse the frame at the oracle's pose.  Voxel bits are
    compared after the frames in check_frames; the ATE of both trajectories must agree."""
    import paper_2509_24236_b200 as pft
    seq = Sequence(kind, seed=1, n_frames=max(n_frames, 8), K=K, iters=iters)
    vol = pft.Volume(seq.desc, dev())
    vol.reset()
    ov = oracle.OracleVolume(seq.desc)
    d0 = seq.depth(0)
    vol.integrate(T(d0), seq.intr, T(seq.gt[0]))
    ov.integrate(d0, seq.intr, seq.gt[0])
    P_prev = seq.gt[0]
    traj_gpu, traj_ora = [seq.gt[0]], [seq.gt[0]]
    ties = 0
    pst_dev = T(seq.pst)
    for t in range(1, n_frames):
        depth = seq.depth(t)
        T_init = compose(P_prev, seq.rel_init(t))
        d_dev, ti_dev = T(depth), T(T_init)

        def run(it):
            r = vol.track(d_dev, seq.intr, ti_dev, pst_dev, dataclasses.replace(seq.params, iters=it))
            torch.cuda.synchronize()
            return {k: r[k].cpu().numpy() for k in ("T", "E", "n", "trace")}
        r, o, nt = track_parity(run, ov, depth, seq.intr, T_init, seq.pst, seq.params, f"{kind} frame {t}")
        ties += nt
        assert_last_iter_counts(r["n"], r["E"], o, ov, depth, seq.intr, seq.pst, seq.params, T_init, f"{kind} frame {t}")
        assert_pose_close(r["T"], o["T"], f"{kind} frame {t}")
        traj_gpu.append(r["T"])
        traj_ora.append(o["T"])
        P_prev = o["T"]
        # both sides fuse at the same (oracle) pose; the GPU pose is within 1e-4 of it
        vol.integrate(d_dev, seq.intr, T(P_prev))
        ov.integrate(depth, seq.intr, P_prev)
        if t in check_frames:
            V, W = [x.cpu().numpy() for x in vol.download()]
            assert np.array_equal(bits(V), bits(ov.V)), f"{kind} frame {t}: {int((bits(V) != bits(ov.V)).sum())} values differ"
            assert np.array_equal(bits(W), bits(ov.W)), f"{kind} frame {t}: weights differ"
            del V, W
    gt = [seq.gt[t] for t in range(n_frames)]
    ate_gpu, ate_ora = _ate_cm(traj_gpu, gt), _ate_cm(traj_ora, gt)
    assert abs(ate_gpu - ate_ora) <= 1e-2, f"{kind}: ATE gpu {ate_gpu:.6f} cm vs oracle {ate_ora:.6f} cm"  # 1e-4 m
    vol.close()
    return dict(ate_gpu_cm=ate_gpu, ate_oracle_cm=ate_ora, ties=ties)


def test_sequence_Q_512_lockstep():
    """Config Q: 512^3 @ 1 cm fp32, K = 2048, 10 iterations, 640x480 frames, the first 31 frames
    (30 tracked) with the chained L25 init; voxel bits at frames 1, 2, 10 and 30; ATE of both."""
    _lockstep("Q", 31, 2048, check_frames={1, 2, 10, 30})


def test_fitness_error_budget():
    """The tie bar E_TIE (tests/parity.py) against the fitness arithmetic it covers: config Q frame 1
    (map = frame 0 fused at GT, chained L25 init), the oracle's 2048 candidates of its last
    (converged) iteration -- where near-ties are dense -- evaluated by pft_eval_poses and by the
    oracle from eq. E: counts exact, and the relative E_k error of every candidate below E_TIE / 3."""
    import paper_2509_24236_b200 as pft
    seq = Sequence("Q", seed=1, n_frames=8, K=2048, iters=10)
    vol = pft.Volume(seq.desc, dev())
    vol.reset()
    ov = oracle.OracleVolume(seq.desc)
    d0 = seq.depth(0)
    vol.integrate(T(d0), seq.intr, T(seq.gt[0]))
    ov.integrate(d0, seq.intr, seq.gt[0])
    depth = seq.depth(1)
    T_init = compose(seq.gt[0], seq.rel_init(1))
    o = ov.track(depth, seq.intr, T_init, seq.pst, seq.params)
    row = o["trace"][seq.params.iters - 2]          # the pose and search size entering the last iteration
    P, om, v = row[4:16].reshape(3, 4), row[2], row[3]
    poses = []
    for k in range(seq.pst.shape[0]):
        dR, _, u = oracle.delta(seq.pst[k], om, v)
        poses.append(oracle.apply_delta(dR, u, P, 0))
    poses = np.stack(poses)
    e = ov.eval_poses(depth, seq.intr, poses, stride=seq.params.stride)
    r = vol.eval_poses(T(depth), seq.intr, T(poses), seq.params)
    torch.cuda.synchronize()
    E, n = r["E"].cpu().numpy(), r["n"].cpu().numpy()
    assert_eval_parity(E, n, e, "Q frame 1 last-iteration candidates")
    ok = n == e["n"]
    rel = np.abs(E - e["E"])[ok] / np.abs(e["E"][ok])
    assert ok.sum() >= 2040 and rel.max() < E_TIE / 3, f"max relative E_k error {rel.max():.3e}"
    vol.close()


def test_sequence_L_1024_fp16_lockstep():
    """Config L: 1024^3 @ 5 mm, tau 2 cm, fp16 values and weights (bit-exact fp16 rounding), K = 4096,
    the first 6 frames (5 tracked); voxel bits at frames 1, 2 and 5; ATE of both."""
    _lockstep("L", 6, 4096, check_frames={1, 2, 5})


def test_sweep_W_k4096_fused_exchange_G8(sweep):
    """Config W, K = 4096, 10 iterations: the F2 fused exchange emulated with 8 rank groups in one
    launch (37 CTAs each) equals the 1-rank persistent run bit for bit."""
    import paper_2509_24236_b200 as pft
    c, vol, ov = sweep
    pst = T(c["pst"][:4096].copy())
    params = TrackParams(iters=10, stride=4)
    a = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params)
    a = {k: a[k].cpu().numpy() for k in ("T", "E", "n", "trace")}
    v8 = pft.Volume(c["desc"], dev())
    v8.upload(c["V"], c["W"])
    v8.comm_init_virtual(8, fused=True)
    b = v8.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params)
    torch.cuda.synchronize()
    b = _np(b)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k]), k
    _w4096_vs_oracle(b, c, ov, "W K=4096 fused exchange G=8")
    v8.close()


@pytest.mark.parametrize("variant", ["topk", "weighted_guard"])
def test_sweep_W_k4096_update_variants(sweep, variant):
    """NEXT row F3 at full size: config W, K = 4096, 10 iterations, with the top-32 mean or the
    weighted mean + acceptance guard + stall stop -- the whole trace and the last iteration's
    per-particle E_k / n_k against the oracle."""
    import dataclasses
    c, vol, ov = sweep
    pst = c["pst"][:4096].copy()
    extra = dict(update_rule=2, topk=32) if variant == "topk" else dict(update_rule=1, guard=1, stall_limit=3)
    params = dataclasses.replace(TrackParams(iters=10, stride=4), **extra)
    r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(pst), params)
    torch.cuda.synchronize()
    o = ov.track(c["depth"], c["intr"], c["T_init"], pst, params)
    assert_trace_parity(r["trace"].cpu().numpy(), o["trace"], f"W {variant}")
    assert_last_iter_counts(r["n"].cpu().numpy(), r["E"].cpu().numpy(), o, ov, c["depth"], c["intr"], pst, params,
                            c["T_init"], f"W {variant}")
    assert_pose_close(r["T"].cpu().numpy(), o["T"])


def test_sweep_W_paper_schedule(sweep):
    """NEXT row F1 at full size: the paper's schedule on config W -- K cycling
    10240 / 3072 / 1024 with 2-D strides (8,4) / (4,4) / (4,2), up to 20 iterations with the
    min-search stop -- every trace row (incl. K_i, the stride code, n_c, the stop iteration) and
    the last iteration's counts against the oracle."""
    import dataclasses
    from synth.configs import PAPER_SCHEDULE
    c, vol, ov = sweep
    pst = c["pst"][:10240].copy()
    params = dataclasses.replace(TrackParams(iters=20, stride=4), **PAPER_SCHEDULE)
    r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(pst), params)
    torch.cuda.synchronize()
    o = ov.track(c["depth"], c["intr"], c["T_init"], pst, params)
    tr = r["trace"].cpu().numpy()
    assert_trace_parity(tr, o["trace"], "W paper schedule")
    n, E = r["n"].cpu().numpy(), r["E"].cpu().numpy()
    mism = int((n != o["n"]).sum())
    assert mism == 0, f"{mism} last-iteration count mismatches"
    assert close_E(E, o["E"]).all()
    assert_pose_close(r["T"].cpu().numpy(), o["T"])


@pytest.mark.parametrize("variant", ["mean", "topk", "weighted_guard"])
def test_sweep_W_k65536_two_iterations(sweep, variant):
    """Config W at the largest K (65536: 256 update blocks, the top-k merge over 256 sorted
    lists), 2 iterations of each update rule: both trace rows and all 65536 last-iteration E_k /
    n_k against the oracle."""
    import dataclasses
    c, vol, ov = sweep
    extra = {"mean": {}, "topk": dict(update_rule=2, topk=32),
             "weighted_guard": dict(update_rule=1, guard=1)}[variant]
    params = dataclasses.replace(TrackParams(iters=2, stride=4), **extra)
    r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(c["pst"]), params)
    torch.cuda.synchronize()
    o = ov.track(c["depth"], c["intr"], c["T_init"], c["pst"], params)
    assert_trace_parity(r["trace"].cpu().numpy(), o["trace"], f"W K=65536 {variant}")
    assert_last_iter_counts(r["n"].cpu().numpy(), r["E"].cpu().numpy(), o, ov, c["depth"], c["intr"], c["pst"],
                            params, c["T_init"], f"W K=65536 {variant}")
    assert_pose_close(r["T"].cpu().numpy(), o["T"])


def test_sweep_W_k4096_virtual_shards_G4(sweep):
    """The multi-launch sharded path (NCCL all-gather replaced by device copies, 4 virtual ranks)
    at config W, K = 4096, 10 iterations: bit-identical to the 1-rank persistent run."""
    import paper_2509_24236_b200 as pft
    c, vol, ov = sweep
    pst = T(c["pst"][:4096].copy())
    params = TrackParams(iters=10, stride=4)
    a = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params)
    a = {k: a[k].cpu().numpy() for k in ("T", "E", "n", "trace")}
    v4 = pft.Volume(c["desc"], dev())
    v4.upload(c["V"], c["W"])
    v4.comm_init_virtual(4)
    b = v4.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params)
    torch.cuda.synchronize()
    b = _np(b)
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k]), k
    _w4096_vs_oracle(b, c, ov, "W K=4096 virtual shards G=4")
    v4.close()


def test_sweep_W_k4096_point_shards_G4(sweep):
    """F2b at full size: config W, K = 4096, 10 iterations with the point-sharded partition over 4
    virtual ranks (each a contiguous slice of point tiles; sums added across slices): bit-identical
    to the 1-rank persistent run and equal to the oracle."""
    import paper_2509_24236_b200 as pft
    c, vol, ov = sweep
    pst = T(c["pst"][:4096].copy())
    params = TrackParams(iters=10, stride=4)
    a = _np(vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params))
    v4 = pft.Volume(c["desc"], dev())
    v4.upload(c["V"], c["W"])
    v4.comm_init_virtual(4)
    v4.set_partition(True)
    b = _np(v4.track(T(c["depth"]), c["intr"], T(c["T_init"]), pst, params))
    torch.cuda.synchronize()
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k]), k
    _w4096_vs_oracle(b, c, ov, "W K=4096 point shards G=4")
    v4.close()
