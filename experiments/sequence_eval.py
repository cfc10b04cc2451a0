#!/usr/bin/env python
"""NEXT row F4: sequence-level evaluation on the GPU path (PAPER.md:562-572,
:595-605 analogs on synthetic data; the paper's datasets are not available).

Runs a config-Q-like sequence (512^3 @ 1 cm fp32, K = 2048, 10 iterations by default) through
libpft: frame 0 is fused at GT (reading L24), every later kept frame is tracked from an initial
pose and fused at the tracked pose.  Reports
  - ATE RMSE (cm) of the tracked trajectory, raw and after Horn rigid alignment;
  - completeness: % of ground-truth surface samples with a reconstructed point within 10 cm, and
    accuracy: mean distance (cm) of reconstructed points to the ground-truth surface
    (PAPER.md:562-563), with the reconstruction = pft_extract_surface and the ground truth = the
    analytic scene (distance = |scene SDF|).
Variants:
  --init pr        P_hat_{t-1} * (GT relative pose (+) U+-5deg/+-5cm): the PR-network stand-in (L25)
  --init ro_alone  P_hat_{t-1} (no relative-pose prior: "RO alone")
  --drop R         drop a fraction R of the frames (seeded; PAPER.md:442, :506 frame-drop protocol)
  --tracker paper | guard_weighted | schedule | topk | schedule_topk | topk_guard   (F3 / F1 variants;
                   topk = the north_star "top-k" rule with the 32 best members)
  --init local     no chaining: the map is fused at GT from --map frames, every later frame starts
                   from GT_t (+) U+-noise and is tracked but not fused -- RO's local convergence alone
Per frame it also records the pose error of the initial pose and of the RO result against GT, so
that it shows whether a reading of the update rule actually improves on its initialisation
(characterisation; the default rule is not changed).
"""
import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def horn_align(A, B):
    """Rigid (R, t) minimising sum |R a + t - b|^2 (Horn / Kabsch via SVD)."""
    ca, cb = A.mean(0), B.mean(0)
    H = (A - ca).T @ (B - cb)
    U, _, Vt = np.linalg.svd(H)
    D = np.diag([1.0, 1.0, np.sign(np.linalg.det(Vt.T @ U.T))])
    R = Vt.T @ D @ U.T
    return R, cb - R @ ca


def ate_cm(est, gt):
    e, g = est[:, :, 3], gt[:, :, 3]
    raw = np.sqrt(np.mean(np.sum((e - g) ** 2, axis=1))) * 100.0
    R, t = horn_align(e, g)
    al = np.sqrt(np.mean(np.sum(((e @ R.T) + t - g) ** 2, axis=1))) * 100.0
    return raw, al


def scene_surface_samples(scene, spacing=0.02, lo=-2.56, hi=2.56):
    """Points on the analytic scene's surfaces: the room's 6 walls on a grid and each sphere by a
    Fibonacci lattice, kept inside the volume."""
    pts = []
    h = scene.room_half
    g = np.arange(-h, h + 1e-9, spacing)
    A, B = np.meshgrid(g, g, indexing="ij")
    A, B = A.ravel(), B.ravel()
    for ax in range(3):
        for sgn in (-1.0, 1.0):
            P = np.zeros((A.size, 3))
            o = [a for a in range(3) if a != ax]
            P[:, ax] = sgn * h
            P[:, o[0]], P[:, o[1]] = A, B
            pts.append(P)
    for (cx, cy, cz, r) in scene.spheres:
        n = max(64, int(4 * np.pi * r * r / spacing ** 2))
        i = np.arange(n) + 0.5
        phi = np.arccos(1 - 2 * i / n)
        th = np.pi * (1 + 5 ** 0.5) * i
        P = np.stack([cx + r * np.cos(th) * np.sin(phi), cy + r * np.sin(th) * np.sin(phi), cz + r * np.cos(phi)], 1)
        pts.append(P)
    P = np.concatenate(pts)
    P = P[np.all((P > lo) & (P < hi), axis=1)]
    return P[np.abs(scene.sdf(P)) < 1e-6]  # drop wall samples hidden inside spheres


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--init", default="pr", choices=["pr", "ro_alone", "local"])
    ap.add_argument("--noise", type=float, default=5.0, help="--init local: GT (+) U+-noise deg / cm")
    ap.add_argument("--drop", type=float, default=0.0)
    ap.add_argument("--tracker", default="paper",
                    choices=["paper", "guard_weighted", "schedule", "topk", "schedule_topk", "topk_guard"])
    ap.add_argument("--topk", type=int, default=32)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--map", type=int, default=8, help="--init local: frames fused at GT first")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from scipy.spatial import cKDTree
    import paper_2509_24236_b200 as pft
    from synth.configs import PAPER_SCHEDULE, Sequence, init_noise, make_pst
    from synth.rng import Stream
    from synth.scene import compose, inverse

    dev = torch.device("cuda", 0)
    seq = Sequence("Q", seed=args.seed, n_frames=args.frames, K=2048, iters=10)
    params = seq.params
    pst = seq.pst
    if args.tracker == "guard_weighted":
        params = dataclasses.replace(params, guard=1, update_rule=1)
    elif args.tracker == "schedule":
        params = dataclasses.replace(params, **PAPER_SCHEDULE)
        pst = make_pst(args.seed, 10240)
    elif args.tracker == "topk":
        params = dataclasses.replace(params, update_rule=2, topk=args.topk)
    elif args.tracker == "topk_guard":
        params = dataclasses.replace(params, update_rule=2, topk=args.topk, guard=1)
    elif args.tracker == "schedule_topk":
        params = dataclasses.replace(params, update_rule=2, topk=args.topk, **PAPER_SCHEDULE)
        pst = make_pst(args.seed, 10240)
    keep = np.ones(args.frames, bool)
    if args.drop > 0:
        u = Stream(args.seed, 5).uniform(args.frames)
        keep = u >= args.drop
        keep[0] = True
    frames = np.nonzero(keep)[0]
    vol = pft.Volume(seq.desc, dev)
    vol.reset()
    pst_d = torch.from_numpy(pst).to(dev)
    d0 = seq.depth(0)
    vol.integrate(torch.from_numpy(d0).to(dev), seq.intr, torch.from_numpy(seq.gt[0].copy()).to(dev))
    if args.init == "local":
        for t in range(1, args.map):
            vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
        frames = np.array([0] + [t for t in frames if t >= args.map])
    est = [seq.gt[0]]
    P_prev, t_prev = seq.gt[0], 0
    t_track = []
    err_init, err_fin = [], []

    def pose_err(A, B):
        c = (np.trace(A[:, :3].T @ B[:, :3]) - 1.0) / 2.0
        return float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))), float(np.linalg.norm(A[:, 3] - B[:, 3]) * 100.0)
    for t in frames[1:]:
        depth = torch.from_numpy(seq.depth(t)).to(dev)
        if args.init == "pr":
            rel = init_noise(args.seed, int(t), compose(inverse(seq.gt[t_prev]), seq.gt[t]), 5.0, 5.0)
            T_init = compose(P_prev, rel)
        elif args.init == "local":
            T_init = init_noise(args.seed, int(t), seq.gt[t], args.noise, args.noise)
        else:
            T_init = P_prev
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = vol.track(depth, seq.intr, torch.from_numpy(np.ascontiguousarray(T_init)).to(dev), pst_d, params)
        if args.init != "local":
            vol.integrate(depth, seq.intr, r["T"])
        e1.record()
        torch.cuda.synchronize()
        t_track.append(e0.elapsed_time(e1))
        P_prev, t_prev = r["T"].cpu().numpy(), int(t)
        est.append(P_prev)
        err_init.append(pose_err(np.asarray(T_init), seq.gt[t]))
        err_fin.append(pose_err(P_prev, seq.gt[t]))
    est = np.stack(est)
    gt = seq.gt[frames]
    raw, aligned = ate_cm(est, gt)
    pts = vol.extract_surface().cpu().numpy()
    gt_pts = scene_surface_samples(seq.scene)
    acc = float(np.mean(np.abs(seq.scene.sdf(pts))) * 100.0) if len(pts) else None
    comp = float(np.mean(cKDTree(pts).query(gt_pts, k=1)[0] < 0.10) * 100.0) if len(pts) else 0.0
    ei, ef = np.array(err_init), np.array(err_fin)
    better = (ef[:, 0] < ei[:, 0]) & (ef[:, 1] < ei[:, 1])
    res = dict(frames=int(len(frames)), init=args.init, drop=args.drop, tracker=args.tracker,
               noise=args.noise if args.init == "local" else None,
               topk=int(params.topk) if params.update_rule == 2 else None,
               init_err_median_deg_cm=[float(np.median(ei[:, 0])), float(np.median(ei[:, 1]))],
               ro_err_median_deg_cm=[float(np.median(ef[:, 0])), float(np.median(ef[:, 1]))],
               ro_improves_both_frac=float(better.mean()),
               ate_cm_raw=raw, ate_cm_aligned=aligned, completeness_pct_10cm=comp, accuracy_cm=acc,
               surface_points=int(len(pts)), gt_samples=int(len(gt_pts)),
               ms_per_frame_median=float(np.median(t_track)))
    print(json.dumps(res))
    if args.out:
        with open(args.out, "a") as f:
            f.write(json.dumps(res) + "\n")
    vol.close()


if __name__ == "__main__":
    main()
