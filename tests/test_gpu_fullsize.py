"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
config W (512^3 fp32, K = 4096 full 10-iteration trace; K = 65536 sampled), config Q (512^3 fp32)
and config L (1024^3 fp16) as short GPU/oracle lock-step sequences (track + integrate)."""
import numpy as np
import pytest

import oracle
from synth.configs import Sequence, TrackParams, config_sweep, init_noise
from synth.rng import Stream
from synth.scene import compose, inverse
from tests.parity import (assert_eval_parity, assert_last_iter_counts, assert_pose_close, assert_trace_parity,
                          close_E)

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


def test_sweep_W_k4096_full_trace(sweep):
    """Config W, K = 4096: the whole 10-iteration RO run, every iteration's |A|, E, s and pose and the
    last iteration's per-particle E_k / n_k against the oracle."""
    c, vol, ov = sweep
    pst = c["pst"][:4096].copy()
    params = TrackParams(iters=10, stride=4)
    r = vol.track(T(c["depth"]), c["intr"], T(c["T_init"]), T(pst), params)
    torch.cuda.synchronize()
    o = ov.track(c["depth"], c["intr"], c["T_init"], pst, params)
    assert_trace_parity(r["trace"].cpu().numpy(), o["trace"], "W K=4096")
    assert_last_iter_counts(r["n"].cpu().numpy(), r["E"].cpu().numpy(), o, ov, c["depth"], c["intr"], pst, params,
                            c["T_init"], "W K=4096")
    assert_pose_close(r["T"].cpu().numpy(), o["T"])


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


def _lockstep(kind, n_frames, K, iters=10):
    import paper_2509_24236_b200 as pft
    seq = Sequence(kind, seed=1, n_frames=max(n_frames, 8), K=K, iters=iters)
    vol = pft.Volume(seq.desc, dev())
    vol.reset()
    ov = oracle.OracleVolume(seq.desc)
    d0 = seq.depth(0)
    vol.integrate(T(d0), seq.intr, T(seq.gt[0]))
    ov.integrate(d0, seq.intr, seq.gt[0])
    P_prev = seq.gt[0]
    for t in range(1, n_frames):
        depth = seq.depth(t)
        T_init = compose(P_prev, seq.rel_init(t))
        r = vol.track(T(depth), seq.intr, T(T_init), T(seq.pst), seq.params)
        torch.cuda.synchronize()
        o = ov.track(depth, seq.intr, T_init, seq.pst, seq.params)
        assert_trace_parity(r["trace"].cpu().numpy(), o["trace"], f"{kind} frame {t}")
        assert_last_iter_counts(r["n"].cpu().numpy(), r["E"].cpu().numpy(), o, ov, depth, seq.intr, seq.pst,
                                seq.params, T_init, f"{kind} frame {t}")
        P_prev = o["T"]
        # both sides fuse at the same (oracle) pose; the GPU pose is within 1e-4 of it
        vol.integrate(T(depth), seq.intr, T(P_prev))
        ov.integrate(depth, seq.intr, P_prev)
    V, W = [x.cpu().numpy() for x in vol.download()]
    assert np.array_equal(bits(V), bits(ov.V)), f"{kind}: {int((bits(V) != bits(ov.V)).sum())} values differ"
    assert np.array_equal(bits(W), bits(ov.W))
    vol.close()


def test_sequence_Q_512_lockstep():
    """Config Q geometry: 512^3 @ 1 cm fp32, K = 2048, 10 iterations, 640x480 frames."""
    _lockstep("Q", 3, 2048)


def test_sequence_L_1024_fp16_lockstep():
    """Config L: 1024^3 @ 5 mm, tau 2 cm, fp16 values and weights (bit-exact fp16 rounding), K = 4096."""
    _lockstep("L", 3, 4096)


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
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k].cpu().numpy()), k
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
    for k in ("T", "E", "n", "trace"):
        assert np.array_equal(a[k], b[k].cpu().numpy()), k
    v4.close()
