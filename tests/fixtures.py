"""Builders for the hand-derived golden fixtures (inputs only; expected values live in tests/golden/)."""
import json
import os

import numpy as np

from synth.configs import VolumeDesc, TrackParams
from synth.scene import Intrinsics

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def f_track_inputs():
    g = golden("f_track.json")
    v = g["volume"]
    desc = VolumeDesc(v["nx"], v["ny"], v["nz"], v["voxel_m"], tuple(v["origin_m"]), v["trunc_m"])
    k = g["intrinsics"]
    intr = Intrinsics(k["fx"], k["fy"], k["cx"], k["cy"], k["width"], k["height"])
    # analytic fill of the plane z = plane_z: V = clamp((z - z0)/tau, -1, 1) -> fp32, W = 1
    z = v["origin_m"][2] + v["voxel_m"] * (np.arange(v["nz"]) + 0.5)
    col = np.clip((z - v["plane_z"]) / v["trunc_m"], -1.0, 1.0).astype(np.float32)
    V = np.broadcast_to(col[:, None, None], (v["nz"], v["ny"], v["nx"])).astype(np.float32).ravel()
    W = np.ones_like(V)
    depth = np.full((k["height"], k["width"]), g["depth_mm"], dtype=np.uint16)
    T_gt = np.array(g["T_gt"], dtype=np.float64)
    T_init = T_gt.copy()
    T_init[2, 3] += g["T_init_dz"]
    pst = np.array(g["pst"], dtype=np.float32)
    params = TrackParams(omega0_deg=g["omega0_deg"], v0_cm=g["v0_cm"], beta=g["beta"], iters=g["iters"],
                         stride=g["stride"])
    return dict(desc=desc, intr=intr, V=V, W=W, depth=depth, T_gt=T_gt, T_init=T_init, pst=pst, params=params, g=g)


def f_mean_inputs():
    """Fixture F-mean (tests/golden/f_mean.json): F-track's scene with a two-member, non-coaxial
    advantage set."""
    import dataclasses
    f = f_track_inputs()
    g = golden("f_mean.json")
    f["pst"] = np.array(g["pst"], dtype=np.float32)
    f["params"] = dataclasses.replace(f["params"], omega0_deg=g["omega0_deg"], v0_cm=g["v0_cm"], beta=g["beta"],
                                      iters=g["iters"])
    f["gm"] = g
    return f


def f_mean_closed_form():
    """The hand-derived expectations of F-mean (tests/golden/f_mean.json "_derivation"), evaluated
    from their closed forms: the advantage set's fitness, the averaged pose P' as an axis-angle
    rotation (scipy), E(P') and the next search size."""
    from scipy.spatial.transform import Rotation
    a = np.deg2rad(10.0)
    tau = 0.3
    E_base = 0.025 / tau
    E_member = 0.1 * np.sin(a) / tau
    phi = 2.0 * np.arctan(np.tan(a / 2.0) / np.sqrt(2.0))
    n = np.array([1.0, 1.0, 0.0]) / np.sqrt(2.0)
    Rm = Rotation.from_rotvec(n * phi).as_matrix()
    P = np.zeros((3, 4))
    P[:, :3] = Rm @ np.diag([1.0, -1.0, -1.0])
    P[:, 3] = [0.8, 0.8, 1.6]
    c, s = np.cos(phi), np.sin(phi)
    vals = [0.8 * (1.0 - c) + (s / np.sqrt(2.0)) * d for d in (-0.2, 0.0, 0.0, 0.2)]
    E_c = float(np.mean(np.abs(vals))) / tau
    f = 0.1 + 0.9 * E_c
    return dict(E_base=E_base, E=[E_member, E_member, 0.05 / tau], P=P, E_c=E_c, s_next=(20.0 * f, 10.0 * f),
                phi=phi)
