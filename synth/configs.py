"""BASELINE.json workloads T, S, Q, W, L as seeded synthetic inputs.

These stand in for the paper's FastCaMo-Synth / TUM / ETH3D sequences, which
are not available: room-scale analytic scenes, fast shaky motion, a dense TSDF.
Everything returned here is an *input* (volume fill, depth, poses, template);
nothing here evaluates fitness, integrates or updates a pose.
"""
from dataclasses import dataclass, replace
import numpy as np

from .rng import Stream
from .scene import (Intrinsics, analytic_fill, box_room, compose, inverse, look_at, perturb,
                    render_depth, rot_z, rotvec_to_matrix, pose, sphere_on_plane)


@dataclass
class VolumeDesc:
    nx: int
    ny: int
    nz: int
    voxel_m: float
    origin_m: tuple
    trunc_m: float
    max_weight: float = 128.0
    max_depth_m: float = 8.0
    storage: str = "f32"          # "f32" | "f16" (value AND weight precision)


@dataclass
class TrackParams:
    omega0_deg: float = 10.0
    v0_cm: float = 10.0
    beta: float = 0.1
    iters: int = 10
    stride: int = 4               # 1/16 rate as a 4x4 stride
    min_inband_frac: float = 0.0
    delta_conv: int = 0           # 0 camera-centred (default), 1 world-literal
    update_rule: int = 0          # 0 plain mean (paper, L14); 1 weighted (NEXT F3)
    topk: int = 0
    nsched: int = 0               # NEXT F1: cycled (K, sx, sy) schedule
    sched_K: tuple = (0, 0, 0, 0)
    sched_sx: tuple = (0, 0, 0, 0)
    sched_sy: tuple = (0, 0, 0, 0)
    min_search_deg: float = 0.0   # F1 convergence stop; 0 = off
    min_search_cm: float = 0.0
    guard: int = 0                # F3 acceptance guard
    stall_limit: int = 0          # F3 stall stop; 0 = off


# The paper's schedule as SPEC.md:371 pairs it: largest K with the coarsest rate;
# rates 1/32, 1/16, 1/8 as 2-D strides (8,4), (4,4), (4,2) (L20).
PAPER_SCHEDULE = dict(nsched=3, sched_K=(10240, 3072, 1024, 0), sched_sx=(8, 4, 4, 0), sched_sy=(4, 4, 2, 0),
                      iters=20, min_search_deg=0.1, min_search_cm=0.1)


KINECT_VGA = Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
TINY_CAM = Intrinsics(131.25, 131.25, 39.5, 29.5, 80, 60)


def make_pst(seed: int, K: int, order: str = "none") -> np.ndarray:
    """Particle-swarm template: K x 6 uniform in [-1,1], rounded to fp32 (stream 3).
    order="morton" returns the same set of rows sorted along a 6-D Morton curve (10 bits per
    axis), so neighbouring rows are similar delta poses (an input layout choice: the sample set,
    and hence the method, is unchanged)."""
    pst = Stream(seed, 3).symmetric(6 * K).astype(np.float32).reshape(K, 6)
    if order == "morton":
        q = np.clip(((pst.astype(np.float64) + 1.0) * 512.0).astype(np.int64), 0, 1023)
        key = np.zeros(K, dtype=np.int64)
        for bit in range(9, -1, -1):
            for ax in range(6):
                key = (key << 1) | ((q[:, ax] >> bit) & 1)
        pst = pst[np.argsort(key, kind="stable")]
    return pst


def init_noise(seed: int, t: int, T_gt, deg, cm):
    """GT perturbed by a seeded uniform box of +-deg / +-cm (stream 2e6+t; L26)."""
    st = Stream(seed, 2_000_000 + t)
    ab = st.symmetric(6)
    return perturb(T_gt, ab[:3], ab[3:], deg, cm)


# ----------------------------------------------------------------------------- config T
def tiny_gt_pose(seed=1):
    st = Stream(seed, 1)
    u = st.uniform(3)
    dist = 1.8 + 0.4 * u[0]
    el = np.deg2rad(20.0 + 30.0 * u[1])
    az = 2.0 * np.pi * u[2]
    c = np.array([0.64, 0.64, 0.64])
    C = c + dist * np.array([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
    return look_at(C, c)


def config_tiny(seed=1, K=64, iters=3):
    scene = sphere_on_plane()
    desc = VolumeDesc(64, 64, 64, 0.02, (0.0, 0.0, 0.0), 0.06)
    T_gt = tiny_gt_pose(seed)
    depth = render_depth(scene, TINY_CAM, T_gt)
    V, W = analytic_fill(scene, 64, 64, 64, 0.02, desc.origin_m, desc.trunc_m)
    return dict(name="tiny", scene=scene, desc=desc, intr=TINY_CAM, depth=depth, T_gt=T_gt,
                T_init=init_noise(seed, 0, T_gt, 3.0, 3.0), pst=make_pst(seed, K),
                params=TrackParams(iters=iters, stride=1), V=V, W=W)


# ----------------------------------------------------------------------------- room configs
def room_gt_pose(scene, seed=1, clearance=0.35):
    """Camera inside the room >= clearance from every surface, looking at a random sphere."""
    st = Stream(seed, 1)
    while True:
        C = st.symmetric(3) * 1.25
        if scene.sdf(C[None])[0] >= clearance:
            break
    j = int(st.uniform(1)[0] * len(scene.spheres))
    target = np.array(scene.spheres[j][:3])
    return look_at(C, target)


def config_single(seed=1, K=1024, iters=10, n=256, voxel=0.01, half=1.28, deg=8.0):
    scene = box_room(seed)
    desc = VolumeDesc(n, n, n, voxel, (-half, -half, -half), 0.04)
    T_gt = room_gt_pose(scene, seed)
    depth = render_depth(scene, KINECT_VGA, T_gt, Stream(seed, 4_000_000))
    V, W = analytic_fill(scene, n, n, n, voxel, desc.origin_m, desc.trunc_m)
    return dict(name="single", scene=scene, desc=desc, intr=KINECT_VGA, depth=depth, T_gt=T_gt,
                T_init=init_noise(seed, 0, T_gt, deg, deg), pst=make_pst(seed, K),
                params=TrackParams(iters=iters, stride=4), V=V, W=W)


def config_sweep(seed=1, K=4096, iters=10):
    """Config W: the S room filled analytically into 512^3 @1 cm, one frame, init +-15/15."""
    c = config_single(seed, K=K, iters=iters, n=512, voxel=0.01, half=2.56, deg=15.0)
    c["name"] = f"sweep{K}"
    return c


# ----------------------------------------------------------------------------- sequences
def _catmull_rom_closed(P, s):
    """Closed uniform Catmull-Rom through control points P (m,3) at parameters s (in [0,m))."""
    m = len(P)
    i = np.floor(s).astype(int) % m
    u = (s - np.floor(s))[:, None]
    p0, p1, p2, p3 = P[(i - 1) % m], P[i], P[(i + 1) % m], P[(i + 2) % m]
    return 0.5 * ((2 * p1) + (-p0 + p2) * u + (2 * p0 - 5 * p1 + 4 * p2 - p3) * u ** 2
                  + (-p0 + 3 * p1 - 3 * p2 + p3) * u ** 3)


def shaky_trajectory(scene, n_frames, seed=1, loops=2.0):
    """Smooth spline + per-frame non-accumulating jitter (<=10 deg / <=5 cm) + persistent
    +-30 deg in-place yaw bursts (per-frame probability 0.03).  Returns (n,3,4) GT poses."""
    st = Stream(seed, 1)
    ctrl = []
    while len(ctrl) < 6:
        C = st.symmetric(3) * 1.25
        if scene.sdf(C[None])[0] >= 0.5:
            ctrl.append(C)
    ctrl = np.array(ctrl)
    tgt = np.array([s[:3] for s in scene.spheres[:6]]) if len(scene.spheres) >= 6 else st.symmetric(18).reshape(6, 3)
    s = np.arange(n_frames) * (6.0 * loops / n_frames)
    Cs = _catmull_rom_closed(ctrl, s)
    Ts = _catmull_rom_closed(tgt, (s * 0.7 + 1.5) % 6.0)
    yaw = 0.0
    out = np.zeros((n_frames, 3, 4))
    for f in range(n_frames):
        j = st.uniform(7)
        if j[0] < 0.03:
            yaw += np.deg2rad(30.0) * (1.0 if j[1] < 0.5 else -1.0)
        T = look_at(Cs[f], Ts[f])
        R = rot_z(yaw) @ T[:, :3]
        axis = st.normal(3)
        axis /= np.linalg.norm(axis)
        ang = np.deg2rad(10.0) * j[2]
        R = rotvec_to_matrix(axis * ang) @ R
        tdir = st.normal(3)
        tdir /= np.linalg.norm(tdir)
        out[f] = pose(R, Cs[f] + tdir * (0.05 * j[3]))
    return out


class Sequence:
    """Config Q (512^3 @1 cm fp32, K=2048) or L (1024^3 @5 mm fp16, tau 2 cm, K=4096).

    Frame t (0-based): depth D_t, GT pose; the PR stand-in (L25) gives
    rel_init_t = (GT_{t-1}^-1 GT_t) (+) U+-5deg/+-5cm so that
    T_init_t = P_hat_{t-1} * rel_init_t.  Frame 0 gets P_hat_0 = GT_0 (L24)."""

    def __init__(self, kind="Q", seed=1, n_frames=300, K=None, iters=10):
        self.kind, self.seed = kind, seed
        self.scene = box_room(seed)
        if kind == "Q":
            self.desc = VolumeDesc(512, 512, 512, 0.01, (-2.56, -2.56, -2.56), 0.04)
            self.K = K or 2048
        elif kind == "L":
            self.desc = VolumeDesc(1024, 1024, 1024, 0.005, (-2.56, -2.56, -2.56), 0.02, storage="f16")
            self.K = K or 4096
        else:
            raise ValueError(kind)
        self.intr = KINECT_VGA
        self.n_frames = n_frames
        self.gt = shaky_trajectory(self.scene, n_frames, seed)
        self.pst = make_pst(seed, self.K)
        self.params = TrackParams(iters=iters, stride=4)

    def depth(self, t):
        return render_depth(self.scene, self.intr, self.gt[t], Stream(self.seed, 4_000_000 + t))

    def rel_init(self, t):
        rel = compose(inverse(self.gt[t - 1]), self.gt[t])
        return init_noise(self.seed, t, rel, 5.0, 5.0)


def with_desc(c, **kw):
    c = dict(c)
    c["desc"] = replace(c["desc"], **kw)
    return c
