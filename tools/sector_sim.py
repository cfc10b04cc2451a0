"""Mask-sector count per warp request under brick-group layouts (host simulation, no GPU): the
strided points of bench frame 12 in the tracker's 8x4-tile slot order, 64 random candidates around
the ground-truth pose at three search sizes; for each warp (32 slots) the number of distinct 32-B
sectors of the 1-bit in-band mask when a sector holds 4 bricks of 4^3 cells in a row along x (the
layout used), 2x2 along x-y, x-z or y-z.  DESIGN.md section 7."""
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from synth.configs import Sequence, init_noise
seq = Sequence("Q", seed=1, n_frames=16, K=2048, iters=10)
d, intr = seq.desc, seq.intr
t = 12
depth = seq.depth(t)
s = seq.params.stride
nr, ncol = -(-intr.height // s), -(-intr.width // s)
ntx, nty = -(-ncol // 8), -(-nr // 4)
npad = ntx * nty * 32
i = np.arange(npad); tt, ll = i >> 5, i & 31
r = (tt // ntx) * 4 + (ll >> 3); c = (tt % ntx) * 8 + (ll & 7)
ok = (r < nr) & (c < ncol)
u, v = np.minimum(c * s, intr.width - 1), np.minimum(r * s, intr.height - 1)
dd = depth[v, u].astype(np.float64) * intr.depth_unit_m
ok &= dd > 0
P = np.stack([(u - intr.cx) * dd / intr.fx, (v - intr.cy) * dd / intr.fy, dd])
o = np.array(d.origin_m); nx, ny, nz = d.nx, d.ny, d.nz
nbx, nby = -(-nx // 4), -(-ny // 4)
rng = np.random.default_rng(1)
def rod(w):
    th = np.linalg.norm(w)
    if th < 1e-12: return np.eye(3)
    k = w / th; Kx = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx
Tgt = seq.gt[t].reshape(3, 4)
for deg, cm in [(10, 10), (1, 1), (0.1, 0.1)]:
    res = {"A_x4": [], "B_xy2x2": [], "C_xz2x2": [], "D_yz": []}
    for k in range(64):
        R = rod(np.deg2rad(deg) * rng.uniform(-1, 1, 3)) @ Tgt[:, :3]
        tk = Tgt[:, 3] + rng.uniform(-1, 1, 3) * cm / 100
        g = (R @ P + (tk - o)[:, None]) / d.voxel_m - 0.5
        cl = np.floor(g).astype(np.int64)
        val = ok & (cl[0] >= 0) & (cl[0] <= nx - 2) & (cl[1] >= 0) & (cl[1] <= ny - 2) & (cl[2] >= 0) & (cl[2] <= nz - 2)
        bx, by, bz = [np.where(val, cl[a], 0) >> 2 for a in range(3)]
        secs = {"A_x4": (bx >> 2) + 1000 * (by + 1000 * bz), "B_xy2x2": (bx >> 1) + 1000 * ((by >> 1) + 1000 * bz),
                "C_xz2x2": (bx >> 1) + 1000 * (by + 1000 * (bz >> 1)), "D_yz": bx + 1000 * ((by >> 1) + 1000 * (bz >> 1))}
        for name, sec in secs.items():
            sec = np.where(val, sec, -1).reshape(-1, 32)
            res[name].append(np.mean([len(np.unique(w)) for w in sec]))
    print(deg, cm, {k2: round(float(np.mean(v2)), 2) for k2, v2 in res.items()})
