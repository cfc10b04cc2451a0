#!/usr/bin/env python
"""Benchmark of the PROFusion tracking-and-fusion hot path on B200 (BASELINE.json metric:
particle-point TSDF evals/s; ms per 640x480 frame, track + integrate).

One step = one frame of BASELINE config 3 ("Q"), as the sequence driver runs it (SURVEY.md §8(c-1)
O11, reading L25): T_init = P_{t-1} * (GT_{t-1}^-1 GT_t (+) U+-5 deg/+-5 cm) -- the network stand-in
chained on the previous *tracked* pose, composed on the device (pft_pose_compose) -- then track the
640x480 depth frame (160x120 strided points, K = 2048 particles per GPU, 10 iterations) against the
512^3 @ 1 cm fp32 TSDF and integrate the frame at the tracked pose.  The TSDF is the sequence's own:
frame 0 fused at GT (L24), frames 1 .. map_frames-1 tracked and fused the same way (untimed), then
the warm-up frames, then the timed frames, all chained.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path (libpft.so)
  python bench.py --impl reference [...]                   # the fp64 CPU oracle, same workload

Multi-GPU (torchrun, one rank per GPU): particles are sharded (K = 2048 * N in total, weak
scaling), the volume is replicated, and each iteration's per-particle records reach every rank
through the F2 exchange inside the persistent tracker (P2P stores over NVLink after a pre-flight;
`--exchange nccl` for the ncclAllGather path, and the automatic fallback).  The config-W particle
sweep (K = 4096 / 16384 / 65536 in total, strong scaling) runs at every N, and every rank's poses
and volume checksum are compared (replica identity).  Timing: CUDA events around each step on the
launching stream, L2 flushed (256 MiB write) between steps outside the events, max over ranks;
each frame is replayed as a CUDA graph (`--no-graph` for eager calls).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_PER_GPU = 2048
ITERS = 10
BYTES_PER_EVAL = 32          # one 32-byte cell record gathered per particle-point evaluation
DP_PER_EVAL = 18             # fp64 pipe instructions per evaluation: 9 DFMA transform + 9 DADD exact floor/fraction
DFMA_PER_CLK_SM = 61.7       # measured fp64 issue rate per SM (tools/microbench/pipes.cu)
INTEG_BYTES_PER_VOXEL = {"f32": 16, "f16": 8}   # V + W read and written per updated voxel


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--map-frames", type=int, default=8)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-large", action="store_true", help="skip the config-L (1024^3 fp16) measurement")
    p.add_argument("--no-graph", action="store_true", help="time eager library calls instead of CUDA-graph replay")
    p.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                   help="N>1: F2 fused P2P exchange inside the persistent tracker (default) or ncclAllGather")
    return p.parse_args()


def config_of(args, world, K):
    """The line's `config` (identical for both arms)."""
    return {"workload": "Q: 640x480 frames, 160x120 points, K=2048/GPU, 10 iters, 512^3 @1cm fp32 TSDF, "
                        "track + integrate, init chained on the previous tracked pose (L25)",
            "particles": K, "iters": ITERS, "volume": "512^3 fp32", "map_frames": args.map_frames,
            "seed": args.seed, "l2": "flushed (256 MiB write) between steps",
            "parallelism": f"particles sharded x{world}, volume replicated"}


# ---------------------------------------------------------------------------- workload
def make_workload(args, n_steps, world):
    """The sequence (config Q) and per-frame inputs: depth and the network stand-in's relative
    init rel_t = GT_{t-1}^-1 GT_t (+) U+-5/+-5 (L25).  Frames [0, map_frames) build the map."""
    from synth.configs import Sequence
    nf = args.map_frames + n_steps
    seq = Sequence("Q", seed=args.seed, n_frames=max(nf, 48), K=K_PER_GPU * world, iters=ITERS)
    frames = [dict(t=t, depth=seq.depth(t), rel=seq.rel_init(t) if t > 0 else None) for t in range(nf)]
    return seq, frames


def strided_valid(depth, stride, max_depth=8.0):
    d = depth[::stride, ::stride].astype(np.float64) * 0.001
    return int(((depth[::stride, ::stride] > 0) & (d < max_depth)).sum())


def ate_cm(poses, gts):
    d = [np.linalg.norm(np.asarray(a)[:, 3] - np.asarray(g)[:, 3]) for a, g in zip(poses, gts)]
    return float(np.sqrt(np.mean(np.square(d))) * 100.0)


def load_jsonl(name):
    path = os.path.join(ROOT, "profiles", name)
    return [json.loads(x) for x in open(path) if x.strip()] if os.path.exists(path) else []


# ---------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.lines, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                pw.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(sm)}


# ---------------------------------------------------------------------------- our path
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2509_24236_b200 as pft

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_run = args.warmup + args.steps
    seq, frames = make_workload(args, n_run, world)
    desc, intr, params = seq.desc, seq.intr, seq.params
    K = K_PER_GPU * world
    M = args.map_frames

    vol = pft.Volume(desc, dev)
    vol.reset()
    exchange = args.exchange
    if world > 1:
        if exchange == "p2p" and not vol.comm_init_p2p(max(K, 65536)):
            # no peer access, or the pre-flight failed on some rank: every rank detached; NCCL path
            print("bench: P2P exchange unavailable on some rank; using ncclAllGather", file=sys.stderr)
            exchange = "nccl"
        if exchange == "nccl":
            vol.comm_init()
    pst = torch.from_numpy(seq.pst).to(dev)
    stream = torch.cuda.current_stream()
    out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(K, dtype=torch.float64, device=dev),
               n=torch.empty(K, dtype=torch.int32, device=dev),
               trace=torch.zeros(ITERS, pft.TRACE_DOUBLES, dtype=torch.float64, device=dev))
    T_prev = torch.from_numpy(seq.gt[0].copy()).to(dev)     # P_0 = GT_0 (L24)
    T_init = torch.empty(3, 4, dtype=torch.float64, device=dev)

    def step(depth, rel):
        """One sequence frame: T_init = P_{t-1} rel_t; track; integrate at the tracked pose; P_t."""
        pft.pose_compose(T_prev, rel, out=T_init)
        vol.track(depth, intr, T_init, pst, params, out=out)
        vol.integrate(depth, intr, out["T"])
        T_prev.copy_(out["T"])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- the map: frame 0 fused at GT, frames 1..M-1 tracked and fused (chained), then warm-up
    vol.integrate(torch.from_numpy(frames[0]["depth"]).to(dev), intr, T_prev)
    dev_in = {}
    for t in range(1, M + n_run):
        dev_in[t] = (torch.from_numpy(frames[t]["depth"]).to(dev), torch.from_numpy(frames[t]["rel"].copy()).to(dev))
    for t in range(1, M + args.warmup):
        step(*dev_in[t])
    barrier()
    idx = list(range(M + args.warmup, M + n_run))          # the timed frames
    n_valid = {t: strided_valid(frames[t]["depth"], params.stride) for t in idx}
    evals = [K * n_valid[t] * ITERS for t in idx]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    snap = vol.storage.clone()          # every timed run below starts from this map state and pose
    snap_T = T_prev.clone()
    poses = {}                          # run name -> (steps, 3, 4) tracked poses

    def restore():
        vol.storage.copy_(snap)
        T_prev.copy_(snap_T)

    # ---- eager timed run: the per-kernel breakdown (CUDA events around every launch) and launch count
    Tq = torch.empty(len(idx), 3, 4, dtype=torch.float64, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
    barrier()
    pft.profile_start()
    l0 = pft.launch_count()
    for j, t in enumerate(idx):
        flush.zero_()
        ev[j][0].record(stream)
        step(*dev_in[t])
        ev[j][1].record(stream)
        Tq[j].copy_(out["T"])
    barrier()
    launches = pft.launch_count() - l0
    prof = pft.profile_stop()
    per_step_eager = [a.elapsed_time(b) for a, b in ev]
    poses["eager"] = Tq.cpu().numpy()
    n_chk = int(out["trace"][-1, 21].item())
    assert n_chk == n_valid[idx[-1]], (n_chk, n_valid[idx[-1]])

    # ---- CUDA-graph replay (the headline): one graph per input-buffer pair, captured once
    graphs = None
    with Clocks(local) as clk:
        if not args.no_graph:
            gd = [torch.empty_like(dev_in[idx[0]][0]) for _ in range(2)]
            gr = [torch.empty_like(dev_in[idx[0]][1]) for _ in range(2)]
            graphs = []
            for b in range(2):
                gd[b].copy_(dev_in[idx[0]][0])
                gr[b].copy_(dev_in[idx[0]][1])
                step(gd[b], gr[b])             # warm-up on these buffers (state restored below)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(gd[b], gr[b])
                graphs.append(g)
            restore()
            barrier()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
            for j, t in enumerate(idx):
                flush.zero_()
                ev[j][0].record(stream)
                gd[0].copy_(dev_in[t][0])       # the graph's static inputs (D2D, inside the window)
                gr[0].copy_(dev_in[t][1])
                graphs[0].replay()
                ev[j][1].record(stream)
                Tq[j].copy_(out["T"])
            barrier()
            poses["graph"] = Tq.cpu().numpy()
    per_step = [a.elapsed_time(b) for a, b in ev] if graphs else per_step_eager
    t_ms = sum(per_step)
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    tot_evals = sum(evals)
    value = tot_evals / (t_max * 1e-3)

    # ---- end-to-end through the public API with host buffers: per step the H2D of the frame's
    # depth and relative init from pinned memory and the D2H of the tracked pose, inside the window
    host_depth = {t: torch.from_numpy(frames[t]["depth"]).pin_memory() for t in idx}
    host_rel = {t: torch.from_numpy(frames[t]["rel"].copy()).pin_memory() for t in idx}
    host_T = [torch.empty(3, 4, dtype=torch.float64).pin_memory() for _ in idx]
    eye = torch.zeros(3, 4, dtype=torch.float64, device=dev)
    eye[0, 0] = eye[1, 1] = eye[2, 2] = 1.0
    d_buf = gd if graphs else [torch.empty_like(dev_in[idx[0]][0]) for _ in range(2)]
    r_buf = gr if graphs else [torch.empty_like(dev_in[idx[0]][1]) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)

    def prefetch(j):
        # double-buffered inputs: frame j+1's H2D runs on a copy stream while frame j computes (a
        # user's capture pipeline); every copy lies inside some step's event window
        t, b = idx[j], j & 1
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(used[b])
            d_buf[b].copy_(host_depth[t], non_blocking=True)
            r_buf[b].copy_(host_rel[t], non_blocking=True)
            ready[b].record(cs)

    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
    restore()
    barrier()
    for j, t in enumerate(idx):
        flush.zero_()
        ev2[j][0].record(stream)
        if j == 0:
            cs.wait_event(ev2[0][0])
            prefetch(0)
        b = j & 1
        stream.wait_event(ready[b])
        if j + 1 < len(idx):
            prefetch(j + 1)
        if graphs:
            graphs[b].replay()
        else:
            step(d_buf[b], r_buf[b])
        used[b].record(stream)
        # the tracked pose to pinned host memory: written by a library kernel through the pinned
        # buffer's unified-address mapping (pft_pose_compose with an identity right factor, an exact
        # copy) -- 96 B over PCIe per step; ~9 us less than a memcpy node (3 bench runs each:
        # e2e 1.505 vs 1.514 ms per step; tools/e2e_split.py)
        pft.pose_compose(out["T"], eye, out=host_T[j])
        ev2[j][1].record(stream)
    barrier()
    poses["e2e"] = np.stack([h.numpy() for h in host_T])
    e2e_ms = sum(a.elapsed_time(b) for a, b in ev2)
    if world > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = host_depth[idx[0]].numel() * 2 + 96
    d2h = 96
    runs_agree = all(np.array_equal(poses["eager"], p) for p in poses.values())
    checksum = vol.checksum()

    # ---- replica identity (N > 1): every rank's tracked poses (bits) and final volume checksum
    identity = None
    if world > 1:
        bits = torch.from_numpy(poses["e2e"].view(np.int64).ravel().copy()).to(dev)
        lo, hi = bits.clone(), bits.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        cs_t = torch.tensor([checksum & 0x7FFFFFFFFFFFFFFF, checksum >> 63], dtype=torch.int64, device=dev)
        cl, ch = cs_t.clone(), cs_t.clone()
        dist.all_reduce(cl, op=dist.ReduceOp.MIN)
        dist.all_reduce(ch, op=dist.ReduceOp.MAX)
        identity = {"identity_ok": bool(torch.equal(lo, hi) and torch.equal(cl, ch)),
                    "poses_compared": len(idx), "volume_checksum_compared": True}

    # ---- accuracy of the timed frames (characterisation of the paper-literal rule)
    gts = [seq.gt[t] for t in idx]
    rot_err, tr_err = [], []
    for Tt, Tg in zip(poses["e2e"], gts):
        c = (np.trace(Tg[:, :3].T @ Tt[:, :3]) - 1.0) / 2.0
        rot_err.append(float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))))
        tr_err.append(float(np.linalg.norm(Tg[:, 3] - Tt[:, 3]) * 100.0))

    # ---- integration work per frame (an untimed replay of the timed frames, reading the counters)
    integ = {}
    restore()
    st_rows = []
    for t in idx:
        step(*dev_in[t])
        st_rows.append(vol.integrate_stats())
    upd = statistics.mean(r["updated_voxels"] for r in st_rows)
    esz = getattr(desc, "storage", "f32")
    ms_int = prof["integrate"][0] / max(prof["integrate"][1], 1)
    ms_cull = prof["cull"][0] / max(prof["integrate"][1], 1)
    ms_rec = prof["records"][0] / max(prof["integrate"][1], 1)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    integ = {"updated_voxels_per_frame": upd,
             "kept_bricks_per_frame": statistics.mean(r["kept_bricks"] for r in st_rows),
             "free_space_bricks_per_frame": statistics.mean(r["free_bricks"] for r in st_rows),
             "rebuilt_cell_bricks_per_frame": statistics.mean(r["dirty_cell_bricks"] for r in st_rows),
             "us_fusion": ms_int * 1e3, "us_cull": ms_cull * 1e3, "us_records": ms_rec * 1e3,
             "gvox_per_s_fusion_kernel": upd / (ms_int * 1e-3) / 1e9,
             "gvox_per_s_with_cull_and_records": upd / ((ms_int + ms_cull + ms_rec) * 1e-3) / 1e9,
             "hbm_frac_fusion_kernel": upd * INTEG_BYTES_PER_VOXEL[esz] / (ms_int * 1e-3) / 1e9 / hbm_peak,
             "basis": f"{INTEG_BYTES_PER_VOXEL[esz]} B (V + W read + write) per updated voxel (pft_integrate_stats) "
                      "/ CUDA-event kernel time; peak MEASURED_PEAKS.json hbm_gbs"}

    # ---- roofline of the dominant kernel (the persistent tracker: one launch per frame)
    if prof["eval"][1] > 0:       # multi-launch tracker: k_particle_eval is the dominant kernel
        kname, (eval_ms, eval_n) = "k_particle_eval", prof["eval"]
        evals_per_launch = K_PER_GPU * statistics.mean(n_valid[t] for t in idx)
    else:
        kname, (eval_ms, eval_n) = "k_track_persistent (eval+update+centre phases)", prof["track"]
        evals_per_launch = K_PER_GPU * ITERS * statistics.mean(n_valid[t] for t in idx)
    avg_launch_s = eval_ms / eval_n * 1e-3
    kernel_evals_s = evals_per_launch / avg_launch_s
    gather_gbs = kernel_evals_s * BYTES_PER_EVAL / 1e9
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    gth = [r for r in load_jsonl("r02_gather.jsonl") if r.get("test") == "gather32"]
    band = [r for r in gth if r["footprint_bytes"] == 32 << 20]
    gather_peak = band[0]["gathers_per_s"] * BYTES_PER_EVAL / 1e9 if band else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "r02_track_traffic.json")
    if os.path.exists(tf):
        tj = json.load(open(tf))
        traffic = tj.get("dram_bytes_per_eval", 0) * evals_per_launch
    # the replay in the tracker's own item shape (6 tiles x 16 particles since round 2; earlier lines: 4 tiles)
    rep = [x for x in load_jsonl("r02_gather_replay.jsonl")
           if x.get("init_noise_deg_cm") == 5.0 and x.get("frame") == 12 and x.get("tiles", 4) == 6]
    gather_view = None
    if rep:
        x = rep[-1]  # the latest measurement
        ceil = x.get("ceiling_evals_per_s", x["replay_evals_per_s"])
        gather_view = {"replay_evals_per_s": ceil, "frac": kernel_evals_s / ceil,
                       "index_stream_replay_evals_per_s": x["replay_evals_per_s"],
                       "device_generated_replay_evals_per_s": x.get("gen_replay_evals_per_s"),
                       "inband_frac": x["inband_frac"],
                       "source": "profiles/r02_gather_replay.jsonl: the evaluation's mask + record address stream of a "
                                 "bench frame replayed without the fp64 transform and the lerp in the tracker's item "
                                 "order (6-tile x 16-particle warp items; frame 12, +-5 deg/cm init); the faster of "
                                 "the host-built index stream and its on-device fp32 regeneration"}
    roofline = {"bound": "gather", "achieved": gather_gbs, "peak": gather_peak, "unit": "GB/s",
                "frac": gather_gbs / gather_peak if gather_peak else None, "traffic": traffic, "kernel": kname,
                "basis": f"{BYTES_PER_EVAL} B cell record gathered per particle-point evaluation (the record holds the "
                         f"8 trilinear corners) x {evals_per_launch:.0f} evaluations/launch / the launch's CUDA-event "
                         "time; peak = the measured rate of independent random 32-B gathers over a 32 MB (band-sized, "
                         "L2-resident) footprint, profiles/r02_gather.jsonl (tools/microbench/gather.cu)",
                "evals_per_s_kernel": kernel_evals_s,
                "gather_view": gather_view,
                "hbm_view": {"logical_gather_gbs": gather_gbs, "peak_gbs": hbm_peak, "frac": gather_gbs / hbm_peak,
                             "note": "served from L2/L1: DRAM bytes are 'traffic'"},
                "fp64_view": {"dp_instr_per_eval": DP_PER_EVAL, "peak_per_clk_sm": DFMA_PER_CLK_SM,
                              "frac": kernel_evals_s * DP_PER_EVAL / (n_sm * DFMA_PER_CLK_SM * sm_mhz * 1e6)}}

    # ---- config-W particle sweep (strong scaling: K in total, sharded over the N ranks), 1 frame
    sweep = {}
    t0_ = idx[0]
    for Ks in (4096, 16384, 65536):
        from synth.configs import make_pst
        pst_s = torch.from_numpy(make_pst(args.seed, Ks)).to(dev)
        o2 = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(Ks, dtype=torch.float64, device=dev),
                  n=torch.empty(Ks, dtype=torch.int32, device=dev), trace=None)
        restore()
        pft.pose_compose(T_prev, dev_in[t0_][1], out=T_init)
        vol.track(dev_in[t0_][0], intr, T_init, pst_s, params, out=o2)
        ts = []
        for _ in range(3):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            vol.track(dev_in[t0_][0], intr, T_init, pst_s, params, out=o2)
            e1.record(stream)
            barrier()
            ts.append(e0.elapsed_time(e1))
        tm = min(ts)
        if world > 1:
            tt = torch.tensor([tm], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tm = float(tt.item())
        sweep[str(Ks)] = {"evals_per_s": Ks * n_valid[t0_] * ITERS / (tm * 1e-3), "ms_track": tm}
        del pst_s, o2
    vol._ws = {}

    # ---- N > 1: the two partitions over NCCL at config W's smallest K (strong scaling, where the
    # per-rank work is smallest): particles sharded + all-gather vs points sharded + all-reduce (F2b)
    partitions = {}
    if world > 1:
        from synth.configs import make_pst
        if exchange == "p2p":
            vol.comm_detach_p2p()
            vol.comm_init()
        Ks = 4096
        pst_s = torch.from_numpy(make_pst(args.seed, Ks)).to(dev)
        o2 = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(Ks, dtype=torch.float64, device=dev),
                  n=torch.empty(Ks, dtype=torch.int32, device=dev), trace=None)
        restore()
        pft.pose_compose(T_prev, dev_in[t0_][1], out=T_init)
        for name, pts_part in (("particles_allgather", False), ("points_allreduce", True)):
            vol.set_partition(pts_part)
            vol.track(dev_in[t0_][0], intr, T_init, pst_s, params, out=o2)
            ts = []
            for _ in range(3):
                flush.zero_()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                vol.track(dev_in[t0_][0], intr, T_init, pst_s, params, out=o2)
                e1.record(stream)
                barrier()
                ts.append(e0.elapsed_time(e1))
            tm = min(ts)
            tt = torch.tensor([tm], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tm = float(tt.item())
            partitions[name] = {"K": Ks, "ms_track": tm, "evals_per_s": Ks * n_valid[t0_] * ITERS / (tm * 1e-3)}
        vol.set_partition(False)
        vol._ws = {}
        del pst_s, o2

    # ---- F4 surface extraction on the final map: reads W everywhere and V where observed
    extract = {}
    if world == 1:
        restore()
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        npts = len(vol.extract_surface())
        pts_buf = torch.empty(max(npts, 1), 3, dtype=torch.float64, device=dev)
        import ctypes as C
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pft.check(pft.lib().pft_extract_surface(vol.handle, C.c_void_p(pts_buf.data_ptr()), npts,
                                                    C.c_void_p(cnt.data_ptr()), C.c_void_p(stream.cuda_stream)))
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms_x = statistics.median(ts)
        esz_b = 4 if esz == "f32" else 2
        W_all = vol.download()[1]
        observed = int((W_all > 0).sum().item())
        del W_all
        nbytes = esz_b * vol.nvox + esz_b * observed + 24 * npts
        extract = {"ms": ms_x, "points": npts, "observed_voxels": observed, "algorithmic_bytes": nbytes,
                   "achieved_gbs": nbytes / (ms_x * 1e-3) / 1e9, "frac_of_hbm": nbytes / (ms_x * 1e-3) / 1e9 / hbm_peak,
                   "basis": "W of every voxel + V of every observed voxel read once + 24 B per point written"}
        del pts_buf

    # ---- F2 fused exchange and F2b point shards, emulated on this GPU (one frame)
    fused = {}
    if world == 1:
        o3 = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(K, dtype=torch.float64, device=dev),
                  n=torch.empty(K, dtype=torch.int32, device=dev), trace=None)
        restore()
        pft.pose_compose(T_prev, dev_in[t0_][1], out=T_init)
        for mode, G in [("fused", 1), ("fused", 2), ("fused", 4), ("fused", 8), ("points", 2), ("points", 8)]:
            vol.comm_init_virtual(G, fused=(mode == "fused"))
            if mode == "points":
                vol.set_partition(True)
            vol.track(dev_in[t0_][0], intr, T_init, pst, params, out=o3)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                vol.track(dev_in[t0_][0], intr, T_init, pst, params, out=o3)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            fused[f"{mode}_G{G}"] = {"ms_track": statistics.median(ts)}
            vol.set_partition(False)
        vol.comm_init_virtual(1)
        vol._ws = {}
        del o3

    # ---- config L: 1024^3 @ 5 mm fp16 volume, built by its own sequence, K = 4096 track + integrate
    large = {}
    if world == 1 and not args.no_large:
        large = run_large(args, pft, dev, flush, stream)

    res = {
        "metric": "particle-point TSDF evals/s (track) with ms per 640x480 frame (track+integrate)",
        "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 transform/decisions, f32 TSDF + lerp, int64 fixed-point sums",
        "data": "synthetic (seeded box room + shaky trajectory, BASELINE config 3)",
        "config": config_of(args, world, K),
        "points_per_frame": statistics.mean(n_valid.values()),
        "frame_ms": {"median": statistics.median(per_step), "p99": float(np.percentile(per_step, 99)),
                     "max": max(per_step)},
        "launch": "CUDA graph per frame (compose + track + integrate), replayed" if graphs else "eager library calls",
        "eager_ms_per_step": sum(per_step_eager) / args.steps,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]},
        "e2e": {"value": tot_evals / (e2e_ms * 1e-3), "unit": "evals/s", "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "runs_agree": runs_agree,
        "roofline": roofline,
        "integration": integ,
        "clocks": clk.summary(),
        "particle_sweep": sweep,
        "extract_surface": extract,
        "fused_exchange_emulation": fused,
        "large_volume": large,
        "tracking_accuracy": {"ate_cm_timed_frames": ate_cm(poses["e2e"], gts),
                              "rot_deg_median": statistics.median(rot_err), "rot_deg_p90": float(np.percentile(rot_err, 90)),
                              "trans_cm_median": statistics.median(tr_err), "trans_cm_p90": float(np.percentile(tr_err, 90)),
                              "note": "paper-literal RO, init chained on the previous tracked pose with +-5 deg/cm "
                                      "stand-in noise (L25); characterisation, SURVEY.md 8(c-5)"},
    }
    if world > 1:
        res["scaling_check"] = identity
        res["partition_sweep_nccl"] = partitions
        res["config"]["parallelism"] += f", {exchange} exchange"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the contract: rank 0 at N=1 only
        res["cpu_baseline"] = cpu_baseline(args, seq, frames, idx)
    if rank == 0:
        print(json.dumps(res), flush=True)
    vol.close()
    if world > 1:
        dist.destroy_process_group()


def run_large(args, pft, dev, flush, stream):
    """Config L: its own sequence, frame 0 at GT then tracked + fused frames (chained, K = 4096)."""
    import torch
    from synth.configs import Sequence
    nmap = args.map_frames
    sl = Sequence("L", seed=args.seed, n_frames=max(nmap + 8, 16), K=4096, iters=ITERS)
    voll = pft.Volume(sl.desc, dev)
    voll.reset()
    pst_l = torch.from_numpy(sl.pst).to(dev)
    ol = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(4096, dtype=torch.float64, device=dev),
              n=torch.empty(4096, dtype=torch.int32, device=dev), trace=None)
    Tp = torch.from_numpy(sl.gt[0].copy()).to(dev)
    Ti = torch.empty(3, 4, dtype=torch.float64, device=dev)
    voll.integrate(torch.from_numpy(sl.depth(0)).to(dev), sl.intr, Tp)
    ms, stats = [], []
    for t in range(1, nmap + 6):
        d = torch.from_numpy(sl.depth(t)).to(dev)
        rel = torch.from_numpy(sl.rel_init(t).copy()).to(dev)
        timed = t >= nmap + 1
        if timed:
            flush.zero_()
            torch.cuda.synchronize()
            pft.profile_start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        pft.pose_compose(Tp, rel, out=Ti)
        voll.track(d, sl.intr, Ti, pst_l, sl.params, out=ol)
        voll.integrate(d, sl.intr, ol["T"])
        Tp.copy_(ol["T"])
        if timed:
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            pl = pft.profile_stop()
            stats.append((voll.integrate_stats(), {k: v[0] for k, v in pl.items() if v[1]}))
    nvl = strided_valid(sl.depth(nmap + 1), 4)
    kern = {k: statistics.mean(s[1].get(k, 0.0) for s in stats) for k in stats[0][1]}
    upd = statistics.mean(s[0]["updated_voxels"] for s in stats)
    voll.close()
    return {"workload": "L: 1024^3 @5 mm fp16 V+W, tau 2 cm, K=4096, 10 iters, 640x480, chained init",
            "ms_per_frame_median": statistics.median(ms),
            "evals_per_s": 4096 * nvl * ITERS / (statistics.median(ms) * 1e-3),
            "kernel_ms_per_frame": kern,
            "integration": {"updated_voxels_per_frame": upd,
                            "gvox_per_s_fusion_kernel": upd / (kern["integrate"] * 1e-3) / 1e9,
                            "us_fusion": kern["integrate"] * 1e3, "us_cull": kern.get("cull", 0) * 1e3,
                            "us_records": kern.get("records", 0) * 1e3}}


# ---------------------------------------------------------------------------- oracle arms
def oracle_sequence(seq, frames, t_end, nthreads, on_frame=None):
    """The sequence driver (O11) on the oracle: frame 0 fused at GT, then T_init = P_{t-1} rel_t,
    track, fuse at the tracked pose, for frames 1 .. t_end-1.  on_frame(t, seconds, result)."""
    import oracle
    from synth.scene import compose
    ov = oracle.OracleVolume(seq.desc)
    ov.integrate(frames[0]["depth"], seq.intr, seq.gt[0], nthreads=nthreads)
    P = seq.gt[0]
    for t in range(1, t_end):
        t0 = time.perf_counter()
        T_init = compose(P, frames[t]["rel"])
        r = ov.track(frames[t]["depth"], seq.intr, T_init, seq.pst, seq.params, nthreads=nthreads)
        ov.integrate(frames[t]["depth"], seq.intr, r["T"], nthreads=nthreads)
        P = r["T"]
        if on_frame and on_frame(t, time.perf_counter() - t0, r):
            break
    return ov


def cores():
    return len(os.sched_getaffinity(0))


def cpu_baseline(args, seq, frames, idx, budget_s=12.0):
    """The oracle as it stands, on this host's cores: the sequence driver (track K particles x 10
    iterations + fuse per frame) over the first timed frames after building its own map, until
    ~budget_s of CPU work (>= 1 frame), in evals/s."""
    acc = {"ev": 0, "dt": 0.0, "nf": 0, "N": 0}
    first = idx[0]

    def on_frame(t, dt, r):
        if t < first:
            return False
        acc["ev"] += len(seq.pst) * r["N"] * seq.params.iters
        acc["dt"] += dt
        acc["nf"] += 1
        acc["N"] = r["N"]
        return acc["dt"] >= budget_s
    ov = oracle_sequence(seq, frames, idx[-1] + 1, cores(), on_frame)
    # effective parallelism: one frame's track on a 128-particle subset, one
    # thread vs all cores (sandboxed hosts may expose more cores than they deliver)
    from synth.scene import compose
    t = idx[0]
    T_init = compose(seq.gt[t - 1], frames[t]["rel"])
    sub = seq.pst[:128].copy()
    t1 = time.perf_counter()
    ov.track(frames[t]["depth"], seq.intr, T_init, sub, seq.params, nthreads=1)
    t1 = time.perf_counter() - t1
    tn = time.perf_counter()
    ov.track(frames[t]["depth"], seq.intr, T_init, sub, seq.params, nthreads=cores())
    tn = time.perf_counter() - tn
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": acc["ev"] / acc["dt"], "unit": "evals/s", "cores": cores(), "kind": "oracle", "cpu_model": model,
            "effective_parallelism": t1 / tn,
            "sample": f"{acc['nf']} timed frame(s) of the chained sequence (track {len(seq.pst)} particles x "
                      f"{seq.params.iters} iterations x {acc['N']} points + fusion into 512^3 fp32) after the oracle's "
                      f"own map (frames 0..{first - 1}, untimed); {acc['dt']:.1f} s"}


def run_reference(args):
    """The fp64 CPU oracle as the reference arm (this tier has no reference implementation): the
    same chained sequence and per-step workload as our arm (K = 2048 x N particles, 10 iterations,
    160x120 points, fusion into the 512^3 map), on this host's cores, each step a frame; the map
    frames are untimed.  Under torchrun only rank 0 runs."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_run = args.warmup + args.steps
    seq, frames = make_workload(args, n_run, world)
    first_timed = args.map_frames + args.warmup
    per, evs = [], []

    def on_frame(t, dt, r):
        if t >= first_timed:
            per.append(dt)
            evs.append(len(seq.pst) * r["N"] * seq.params.iters)
        return False
    oracle_sequence(seq, frames, args.map_frames + n_run, cores(), on_frame)
    value = sum(evs) / sum(per)
    res = {"impl": "reference",
           "metric": "particle-point TSDF evals/s (track) with ms per 640x480 frame (track+integrate)",
           "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(per) / len(per), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded box room + shaky trajectory, BASELINE config 3)",
           "config": config_of(args, world, len(seq.pst)),
           "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores(), "kind": "oracle",
                            "sample": f"full workload: {len(per)} timed frames (+{args.warmup} warm-up, "
                                      f"{args.map_frames} map frames untimed), {len(seq.pst)} particles x "
                                      f"{seq.params.iters} iterations + fusion"},
           "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
