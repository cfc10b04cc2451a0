"""Multi-rank (world_size 2, gloo, CPU) check of the particle-sharded RO decomposition the GPU path
uses: rank r evaluates template rows [r*ceil(K/G), ...) with the
oracle, the per-particle (E_k, n_k) are all-gathered, and every rank applies the identical
advantage-set update.  The sharded run must reproduce the unsharded oracle trace bit for bit."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_range(K, G, r):
    kloc = -(-K // G)
    b = r * kloc
    return b, max(0, min(K, b + kloc) - b)


def sharded_track(rank, world, c, pst, params, out):
    """PAPER.md:192-208 with the evaluation of the K candidates sharded over the ranks."""
    import oracle
    vol = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    pts = oracle.backproject(c["depth"], c["intr"], params.stride)
    P = np.array(c["T_init"], dtype=np.float64)
    omega, v = params.omega0_deg, params.v0_cm
    Ec, _, _ = vol.fitness(pts, P)
    K = len(pst)
    b, n_loc = shard_range(K, world, rank)
    kloc = -(-K // world)
    trace = []
    for it in range(params.iters):
        E_loc = np.ones(kloc)
        n_loc_arr = np.zeros(kloc, np.int32)
        qs, us = np.zeros((K, 4)), np.zeros((K, 3))
        for k in range(K):
            _, qs[k], us[k] = oracle.delta(pst[k], omega, v)
        for j in range(n_loc):
            dR, _, u = oracle.delta(pst[b + j], omega, v)
            Tk = oracle.apply_delta(dR, u, P, params.delta_conv)
            E_loc[j], n_loc_arr[j], _ = vol.fitness(pts, Tk)
        # the exchange step (a6): all-gather of the per-particle results
        gE = [torch.zeros(kloc, dtype=torch.float64) for _ in range(world)]
        gn = [torch.zeros(kloc, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gE, torch.from_numpy(E_loc))
        dist.all_gather(gn, torch.from_numpy(n_loc_arr))
        E = torch.cat(gE).numpy()[:K]
        n = torch.cat(gn).numpy()[:K]
        # identical update on every rank, ascending k
        Ebase = Ec
        Q, U, nA = np.zeros(4), np.zeros(3), 0
        for k in range(K):
            if E[k] < Ebase:
                Q = Q + qs[k]
                U = U + us[k]
                nA += 1
        if nA > 0:
            qn = np.sqrt(Q[0] * Q[0] + Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3])
            Rb = oracle.quat_to_R(Q / qn)
            P = oracle.apply_delta(Rb, U / nA, P, params.delta_conv).reshape(12)
            Ec, _, _ = vol.fitness(pts, P)
        f = params.beta + (1.0 - params.beta) * Ec
        trace.append([Ebase, nA, omega, v] + list(np.asarray(P).reshape(12)) + [Ec, f * omega, f * v])
        omega, v = f * omega, f * v
    out[rank] = dict(trace=np.array(trace), E=E, n=n)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth.configs import TrackParams, config_tiny, make_pst
    c = config_tiny(seed=2)
    pst = make_pst(2, 37)       # ragged: 37 = 19 + 18 over 2 ranks
    params = TrackParams(iters=3, stride=2)
    out = {}
    sharded_track(rank, world, c, pst, params, out)
    q.put((rank, out[rank]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_ro_equals_unsharded_oracle():
    import oracle
    from synth.configs import TrackParams, config_tiny, make_pst
    oracle.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = config_tiny(seed=2)
    pst = make_pst(2, 37)
    params = TrackParams(iters=3, stride=2)
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], pst, params)
    for r in range(world):
        tr = res[r]["trace"]
        assert np.array_equal(tr, o["trace"][:, :19]), (r, np.abs(tr - o["trace"][:, :19]).max())
        assert np.array_equal(res[r]["E"], o["E"]) and np.array_equal(res[r]["n"], o["n"])
    assert np.array_equal(res[0]["trace"], res[1]["trace"])


def test_shard_ranges_cover_exactly_once():
    """Rows [r*ceil(K/G), min(K, (r+1)*ceil(K/G))) partition [0, K) for every K, G (include/pft.h)."""
    import paper_2509_24236_b200 as pft
    for K in (1, 7, 37, 64, 2048, 65536):
        for G in (1, 2, 3, 4, 8):
            seen = np.zeros(K, int)
            for r in range(G):
                b, n = pft.shard_range(K, G, r)
                assert (b, n) == shard_range(K, G, r)
                seen[b:b + n] += 1
            assert np.all(seen == 1)


def _handles_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_24236_b200.api import gather_handles
    mine = bytes((rank * 37 + i) % 256 for i in range(64))
    q.put((rank, gather_handles(mine)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_handle_gather(world):
    """Host plumbing of the F2 peer exchange (api.Volume.comm_init_p2p): every rank receives all
    ranks' 64-byte CUDA IPC handles, concatenated in rank order, over torch.distributed (gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = b"".join(bytes((r * 37 + i) % 256 for i in range(64)) for r in range(world))
    for r in range(world):
        assert res[r] == want


def _p2p_consensus_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C
    import types
    import paper_2509_24236_b200 as pft
    from paper_2509_24236_b200 import api
    from synth.configs import config_tiny
    L = pft.lib()
    d = api.make_desc(config_tiny(seed=1)["desc"])
    n = C.c_size_t()
    L.pft_volume_bytes(C.byref(d), C.byref(n))
    h = C.c_void_p()
    assert L.pft_volume_create(C.byref(d), C.c_void_p(1 << 40), n.value, C.byref(h)) == 0  # never dereferenced
    fake = types.SimpleNamespace(handle=h, device=torch.device("cpu"), nranks=1, rank=0, _ws={})
    # no GPU here: pft_comm_p2p_init fails on every rank (cudaMalloc), the ranks agree, all detach
    ok = api.Volume.comm_init_p2p(fake, 64)
    q.put((rank, ok, fake.nranks))
    L.pft_volume_destroy(h)
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_init_consensus_falls_back_together():
    """Volume.comm_init_p2p: when any rank cannot attach, every rank detaches and reports False
    (bench.py then uses the NCCL path on all ranks) -- no rank is left waiting on peers."""
    if torch.cuda.is_available():
        pytest.skip("exercises the failure path (no device memory)")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_consensus_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (ok, nr)) for r, ok, nr in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: (False, 1), 1: (False, 1)}


def _p2p_attach_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2509_24236_b200 as pft
    from synth.configs import config_tiny
    torch.cuda.set_device(0)
    c = config_tiny(seed=1)
    vol = pft.Volume(c["desc"], torch.device("cuda", 0))
    ok = vol.comm_init_p2p(4096)  # real CUDA IPC between two processes (same device here)
    state = (ok, vol.nranks, vol.rank)
    if ok:
        vol.comm_detach_p2p()
        state = state + (vol.nranks,)
    vol.close()
    q.put((rank, state))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_p2p_ipc_attach_two_processes():
    """F2 plumbing on real CUDA IPC: two processes (ranks) each allocate an exchange buffer, trade
    IPC handles over torch.distributed, open each other's buffer and agree; then detach.  Only the
    mapping is exercised -- no tracker kernels, so nothing waits on a peer (one GPU here)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_attach_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: (True, 2, 0, 1), 1: (True, 2, 1, 1)}, res


def _preflight_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C
    import paper_2509_24236_b200 as pft
    from paper_2509_24236_b200 import api
    from synth.configs import config_tiny
    torch.cuda.set_device(0)
    vol = pft.Volume(config_tiny(seed=1)["desc"], torch.device("cuda", 0))
    L = pft.lib()
    h = (C.c_uint8 * api.IPC_HANDLE_BYTES)()
    assert L.pft_comm_p2p_init(vol.handle, world, rank, 64, h) == 0
    handles = api.gather_handles(bytes(h), None)
    raw = (C.c_uint8 * (api.IPC_HANDLE_BYTES * world))(*handles)
    assert L.pft_comm_p2p_attach(vol.handle, raw) == 0
    dist.barrier()
    res = None
    if rank == 0:
        # rank 1 never writes its token: the pre-flight must time out and report failure (no trap,
        # no hang) -- rank 0's kernel waits on memory only, never on another kernel
        okp = C.c_int32(7)
        st = L.pft_comm_p2p_preflight(vol.handle, 200, C.byref(okp), None)
        res = (st, okp.value, int(torch.cuda.is_available()))
        # the context is still usable afterwards
        vol.reset()
        torch.cuda.synchronize()
    dist.barrier()
    assert L.pft_comm_p2p_detach(vol.handle) == 0
    q.put((rank, res))
    vol.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_p2p_preflight_times_out_without_trapping():
    """The F2 pre-flight (include/pft.h pft_comm_p2p_preflight) on real CUDA IPC between two
    processes: with the peer silent, it returns ok = 0 within its timeout instead of trapping, and
    the CUDA context stays usable (the caller then falls back to NCCL, api.Volume.comm_init_p2p)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_preflight_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == (0, 0, 1), res


def _points_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from synth.configs import TrackParams, config_tiny, make_pst
    c = config_tiny(seed=2)
    pst = make_pst(2, 37)
    params = TrackParams(iters=3, stride=2)
    vol = oracle.OracleVolume(c["desc"], c["V"], c["W"])
    pts = oracle.backproject(c["depth"], c["intr"], params.stride)
    N = len(pts)
    per = -(-N // world)
    mine = pts[rank * per:(rank + 1) * per]  # this rank's slice of the points (F2b)

    def fit(T):
        """(S, n) of this rank's slice, summed across the ranks (the all-reduce), -> E, n."""
        E, n, _ = vol.fitness(mine, T) if len(mine) else (1.0, 0, 1.0)
        S = E * n if n > 0 else 0.0
        t = torch.tensor([S, float(n)], dtype=torch.float64)
        dist.all_reduce(t)
        S, n = float(t[0]), int(t[1])
        return (S / n if n > 0 else 1.0), n

    P = np.array(c["T_init"], dtype=np.float64)
    omega, v = params.omega0_deg, params.v0_cm
    Ec, _ = fit(P)
    K = len(pst)
    trace = []
    for it in range(params.iters):
        E, n = np.ones(K), np.zeros(K, np.int32)
        qs, us = np.zeros((K, 4)), np.zeros((K, 3))
        for k in range(K):
            dR, qs[k], us[k] = oracle.delta(pst[k], omega, v)
            E[k], n[k] = fit(oracle.apply_delta(dR, us[k], P, params.delta_conv))
        Ebase = Ec
        Q, U, nA = np.zeros(4), np.zeros(3), 0
        for k in range(K):
            if E[k] < Ebase:
                Q, U, nA = Q + qs[k], U + us[k], nA + 1
        if nA > 0:
            qn = np.sqrt(Q[0] * Q[0] + Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3])
            P = oracle.apply_delta(oracle.quat_to_R(Q / qn), U / nA, P, params.delta_conv).reshape(12)
            Ec, _ = fit(P)
        f = params.beta + (1.0 - params.beta) * Ec
        trace.append([Ebase, nA, omega, v] + list(np.asarray(P).reshape(12)) + [Ec, f * omega, f * v])
        omega, v = f * omega, f * v
    q.put((rank, dict(trace=np.array(trace), E=E, n=n)))
    dist.barrier()
    dist.destroy_process_group()


def test_point_sharded_ro_equals_unsharded_oracle():
    """F2b decomposition on 2 gloo ranks: each rank evaluates every candidate on its half of the
    points, the (S, n) sums are all-reduced, every rank applies the identical update; the in-band
    counts and |A| equal the unsharded oracle exactly and E / poses within 1e-12 (the sums are fp64
    here, in a different order; the GPU sums exact fixed-point integers instead)."""
    import oracle
    from synth.configs import TrackParams, config_tiny, make_pst
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_points_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = config_tiny(seed=2)
    pst = make_pst(2, 37)
    params = TrackParams(iters=3, stride=2)
    o = oracle.OracleVolume(c["desc"], c["V"], c["W"]).track(c["depth"], c["intr"], c["T_init"], pst, params)
    for r in (0, 1):
        tr = res[r]["trace"]
        np.testing.assert_array_equal(tr[:, 1], o["trace"][:, 1])
        np.testing.assert_allclose(tr[:, [0, 16]], o["trace"][:, [0, 16]], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(tr[:, 4:16], o["trace"][:, 4:16], atol=1e-12)
        np.testing.assert_array_equal(res[r]["n"], o["n"])
        np.testing.assert_allclose(res[r]["E"], o["E"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(res[0]["trace"], res[1]["trace"])
