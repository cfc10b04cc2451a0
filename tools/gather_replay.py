"""Gather-replay ceiling of the evaluation (SURVEY.md §8(d-3) denominator (4)).

Builds the bench map (config Q, 512^3 fp32, 8 fused frames), tracks one frame (argv: init noise
in deg/cm, default 5 as in the bench; frame, default 9) and, from the tracker's trace, rebuilds all
10 iterations' K = 2048 candidate poses (template rows scaled by s_i around P^(i-1),
camera-centred); computes on the host, in fp64, every (particle, point) cell and its in-band bit
-- the address stream the tracker's P2 phase issues (checked: the host in-band count of the final
centre equals the tracker's n_c).  tools/microbench/libreplay.so
then replays exactly those mask-word and record loads on the GPU in the tracker's item order,
without the transform or the lerp.  Prints one JSON line: the replay's evaluations/s (the gather
ceiling for this access pattern) next to the tracker's.  A second replay generates the same
stream on the device (fp32 cells from fp32 folded poses, the real in-band mask: no 157 MB/iteration
index stream from HBM); the ceiling is the faster of the two."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence, init_noise


def rodrigues(r):
    th = np.linalg.norm(r)
    K = np.array([[0.0, -r[2], r[1]], [r[2], 0.0, -r[0]], [-r[1], r[0], 0.0]])
    if th < 1e-12:
        return np.eye(3) + K
    return np.eye(3) + np.sin(th) / th * K + (1.0 - np.cos(th)) / th ** 2 * (K @ K)


TILES = int(os.environ.get("REPLAY_TILES", "6"))  # the tracker's item width (points per lane)


def main():
    dev = torch.device("cuda", 0)
    seq = Sequence("Q", seed=1, n_frames=16, K=2048, iters=10)
    d, intr = seq.desc, seq.intr
    vol = pft.Volume(d, dev)
    vol.reset()
    for t in range(8):
        vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
    t = int(sys.argv[2]) if len(sys.argv) > 2 else 9
    noise = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0  # init box (deg, cm); the bench uses 5
    depth = seq.depth(t)
    T0 = init_noise(1, t, seq.gt[t], noise, noise).reshape(3, 4)
    V, _ = vol.download()
    torch.cuda.synchronize()
    nx, ny, nz = d.nx, d.ny, d.nz
    A = (V.abs() < 1.0).reshape(nz, ny, nx)
    inb = torch.ones(nz - 1, ny - 1, nx - 1, dtype=torch.bool, device=dev)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                inb &= A[dz:nz - 1 + dz, dy:ny - 1 + dy, dx:nx - 1 + dx]
    inb = inb.cpu().numpy()
    del V, A
    # strided points in the tracker's slot order (8 x 4 pixel tiles of 32 slots)
    s = seq.params.stride
    nr, ncol = -(-intr.height // s), -(-intr.width // s)
    ntx, nty = -(-ncol // 8), -(-nr // 4)
    npad = ntx * nty * 32
    i = np.arange(npad)
    tt, ll = i >> 5, i & 31
    r = (tt // ntx) * 4 + (ll >> 3)
    c = (tt % ntx) * 8 + (ll & 7)
    ok = (r < nr) & (c < ncol)
    u, v = np.minimum(c * s, intr.width - 1), np.minimum(r * s, intr.height - 1)
    raw = depth[v, u].astype(np.float64)
    dd = raw * intr.depth_unit_m
    ok &= (raw > 0) & (dd < getattr(d, "max_depth", 8.0))
    P = np.stack([(u - intr.cx) * dd / intr.fx, (v - intr.cy) * dd / intr.fy, dd])  # 3 x npad
    pst = seq.pst.astype(np.float64)
    K = pst.shape[0]
    o = np.array(d.origin_m)
    nbx, nby = -(-nx // 4), -(-ny // 4)
    sy, sz = 64 * nbx, 64 * nbx * nby
    nrec = 64 * nbx * nby * -(-nz // 4)
    # the tracker on this frame: its trace gives every iteration's centre P^(i-1) and size s_i
    pst_d = torch.from_numpy(seq.pst).to(dev)
    dep_d = torch.from_numpy(depth).to(dev)
    Ti = torch.from_numpy(T0.reshape(12).copy()).to(dev)
    for _ in range(2):
        r0 = vol.track(dep_d, intr, Ti, pst_d, seq.params)
    torch.cuda.synchronize()
    trace = r0["trace"].cpu().numpy()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    vol.track(dep_d, intr, Ti, pst_d, seq.params)
    e1.record()
    torch.cuda.synchronize()
    track_ms = e0.elapsed_time(e1)
    rec = torch.rand(nrec * 8, device=dev)
    mask = torch.full((nrec // 32,), -1, dtype=torch.int32, device=dev)
    queue = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.zeros(296, dtype=torch.float32, device=dev)
    lib = C.CDLL(os.path.join(ROOT, "tools", "microbench", "libreplay.so"))
    replay_ms, n_inb = 0.0, 0
    # device-generated replay (no index stream): the REAL in-band mask in brick-order bits, fp32
    # points (invalid slots z = 0) and per-iteration fp32 folded poses
    zc, yc, xc = np.nonzero(inb)
    bit = (((xc >> 2) << 6) | (xc & 3)) + (yc >> 2) * sy + ((yc & 3) << 2) + (zc >> 2) * sz + ((zc & 3) << 4)
    words = np.zeros(nrec // 32 + 1, dtype=np.uint32)
    np.bitwise_or.at(words, bit >> 5, (np.uint32(1) << (bit & 31).astype(np.uint32)))
    real_mask = torch.from_numpy(words.view(np.int32)).to(dev)
    del zc, yc, xc, bit, words
    pts32 = torch.from_numpy(np.where(ok[None, :], P, 0.0).astype(np.float32).copy()).to(dev)
    out_gen = torch.zeros(1 + 296, dtype=torch.int64, device=dev)
    gen_ms, gen_inb = 0.0, 0
    n_valid = int(ok.sum())
    # sanity: the in-band count of the final centre pose, host-computed, against the tracker's n_c
    Pf = trace[seq.params.iters - 1, 4:16].reshape(3, 4)
    gf = (Pf[:, :3] @ P + (Pf[:, 3] - o)[:, None]) / d.voxel_m - 0.5
    cf = np.floor(gf).astype(np.int64)
    vf = ok & (cf[0] >= 0) & (cf[0] <= nx - 2) & (cf[1] >= 0) & (cf[1] <= ny - 2) & (cf[2] >= 0) & (cf[2] <= nz - 2)
    nf = int((vf & inb[np.where(vf, cf[2], 0), np.where(vf, cf[1], 0), np.where(vf, cf[0], 0)]).sum())
    print(json.dumps({"check_centre_inband_host": nf, "tracker_n_c": float(trace[seq.params.iters - 1, 20]),
                      "N": float(trace[0, 21]), "cells_inband_frac": float(inb.mean())}))
    for it in range(seq.params.iters):
        Pc = T0 if it == 0 else trace[it - 1, 4:16].reshape(3, 4)
        om, vv = trace[it, 2], trace[it, 3]
        idx = np.zeros((K, npad), dtype=np.uint32)
        fold = np.zeros((K, 12), dtype=np.float64)
        for k in range(K):
            dR = rodrigues(pst[k, :3] * om * np.pi / 180.0)
            R = dR @ Pc[:, :3]
            tk = Pc[:, 3] + pst[k, 3:] * vv / 100.0
            fold[k] = np.concatenate([R / d.voxel_m, ((tk - o) / d.voxel_m - 0.5)[:, None]], axis=1).reshape(12)
            g = (R @ P + (tk - o)[:, None]) / d.voxel_m - 0.5
            cl = np.floor(g).astype(np.int64)
            valid = ok & (cl[0] >= 0) & (cl[0] <= nx - 2) & (cl[1] >= 0) & (cl[1] <= ny - 2) & (cl[2] >= 0) & (cl[2] <= nz - 2)
            x, y, z = np.where(valid, cl[0], 0), np.where(valid, cl[1], 0), np.where(valid, cl[2], 0)
            off = ((x >> 2) << 6) | (x & 3)
            off = off + (y >> 2) * sy + ((y & 3) << 2) + (z >> 2) * sz + ((z & 3) << 4)
            b = valid & inb[z, y, x]
            n_inb += int(b.sum())
            idx[k] = (np.where(valid, off, 0).astype(np.uint32)) | (b.astype(np.uint32) << 31)
        idx_d = torch.from_numpy(idx.view(np.int32)).to(dev)
        ms = C.c_float()
        rc = lib.replay_run(C.c_void_p(idx_d.data_ptr()), K, npad, C.c_void_p(rec.data_ptr()),
                            C.c_void_p(mask.data_ptr()), 5, C.c_void_p(queue.data_ptr()), C.c_void_p(out.data_ptr()),
                            C.byref(ms), TILES)
        assert rc == 0, rc
        replay_ms += ms.value
        del idx_d
        poses_d = torch.from_numpy(fold.astype(np.float32)).to(dev)
        rc = lib.replay_gen_run(C.c_void_p(poses_d.data_ptr()), C.c_void_p(pts32.data_ptr()), K, npad, nx, ny, nz,
                                C.c_uint(sy), C.c_uint(sz), C.c_void_p(rec.data_ptr()), C.c_void_p(real_mask.data_ptr()), 5,
                                C.c_void_p(queue.data_ptr()), C.c_void_p(out_gen.data_ptr()), C.byref(ms), TILES)
        assert rc == 0, rc
        gen_ms += ms.value
        gen_inb += int(out_gen[0].item())
    evals = K * n_valid * seq.params.iters
    res = {"tool": "gather_replay", "tiles": TILES, "frame": t, "init_noise_deg_cm": noise, "K": K, "npad": npad, "n_valid": n_valid, "iters": seq.params.iters,
           "inband_frac": n_inb / (K * npad * seq.params.iters),
           "replay_ms": replay_ms, "replay_evals_per_s": evals / (replay_ms * 1e-3),
           "index_stream_bytes_per_iter": K * npad * 4,
           "track_ms": track_ms, "track_evals_per_s": evals / (track_ms * 1e-3),
           "track_over_replay": replay_ms / track_ms,
           "gen_replay_ms": gen_ms, "gen_replay_evals_per_s": evals / (gen_ms * 1e-3),
           "gen_inband_evals": gen_inb, "host_inband_evals": n_inb,
           "ceiling_evals_per_s": evals / (min(replay_ms, gen_ms) * 1e-3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
