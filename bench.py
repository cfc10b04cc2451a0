#!/usr/bin/env python
"""Benchmark of the PROFusion tracking-and-fusion hot path on B200 (BASELINE.json metric:
particle-point TSDF evals/s; ms per 640x480 frame, track + integrate).

One step = one frame of BASELINE config 3 ("Q"): track the 640x480 depth frame (160x120 strided
points, K = 2048 particles per GPU, 10 iterations, init = GT (+) U+-5 deg/+-5 cm standing in for the
regression network) against a 512^3 @ 1 cm fp32 TSDF, then integrate the frame at the tracked
pose.  The TSDF is first built by integrating `--map-frames` frames of the trajectory at GT.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path (libpft.so)
  python bench.py --impl reference [...]                   # the fp64 CPU oracle on a bounded sample

Multi-GPU (torchrun, one rank per GPU): particles are sharded (K = 2048 * N in total, weak
scaling), the volume is replicated, and each iteration's per-particle records reach every rank
through the F2 exchange inside the persistent tracker (P2P stores over NVLink; `--exchange nccl`
for the ncclAllGather path).  Each frame is replayed as a CUDA graph (`--no-graph` for eager
calls).  Timing: CUDA events around each step on the launching stream, L2 flushed (256 MiB
write) between steps outside the events, max over ranks.
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
BYTES_PER_EVAL = 32          # 8 trilinear corners x fp32 value
OPS_PER_EVAL = 32            # algorithmic thread-level operations per particle-point evaluation
LANES_PER_SM = 128           # 4 SM sub-partitions x 32 lanes, one instruction issue per clock each


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


# ---------------------------------------------------------------------------- workload
def make_workload(args, n_steps, world):
    from synth.configs import Sequence, init_noise
    from synth.scene import Intrinsics  # noqa: F401
    nf = args.map_frames + n_steps
    seq = Sequence("Q", seed=args.seed, n_frames=max(nf, 48), K=K_PER_GPU * world, iters=ITERS)
    if os.environ.get("PFT_BENCH_PST_ORDER"):
        from synth.configs import make_pst
        seq.pst = make_pst(args.seed, seq.K, os.environ["PFT_BENCH_PST_ORDER"])
    map_depth = [seq.depth(t) for t in range(args.map_frames)]
    steps = []
    for i in range(n_steps):
        t = args.map_frames + i
        steps.append(dict(t=t, depth=seq.depth(t), T_init=init_noise(args.seed, t, seq.gt[t], 5.0, 5.0)))
    return seq, map_depth, steps


def strided_valid(depth, stride, max_depth=8.0):
    d = depth[::stride, ::stride].astype(np.float64) * 0.001
    return int(((depth[::stride, ::stride] > 0) & (d < max_depth)).sum())


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
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


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
    seq, map_depth, steps_in = make_workload(args, args.warmup + args.steps, world)
    desc, intr, params = seq.desc, seq.intr, seq.params
    K = K_PER_GPU * world

    vol = pft.Volume(desc, dev)
    vol.reset()
    for t, d in enumerate(map_depth):
        vol.integrate(torch.from_numpy(d).to(dev), intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
    exchange = args.exchange
    if world > 1:
        if exchange == "p2p" and not vol.comm_init_p2p(K):
            # e.g. GPUs without peer access: every rank detached; fall back to the NCCL path
            print("bench: P2P exchange unavailable on some rank; using ncclAllGather", file=sys.stderr)
            exchange = "nccl"
        if exchange == "nccl":
            vol.comm_init()
    pst = torch.from_numpy(seq.pst).to(dev)
    depth_dev = [torch.from_numpy(s["depth"]).to(dev) for s in steps_in]
    tinit_dev = [torch.from_numpy(s["T_init"]).to(dev) for s in steps_in]
    n_valid = [strided_valid(s["depth"], params.stride) for s in steps_in]
    evals = [K * n * ITERS for n in n_valid]
    out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(K, dtype=torch.float64, device=dev),
               n=torch.empty(K, dtype=torch.int32, device=dev),
               trace=torch.zeros(ITERS, pft.TRACE_DOUBLES, dtype=torch.float64, device=dev))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(i, depth, T_init):
        vol.track(depth, intr, T_init, pst, params, out=out)
        vol.integrate(depth, intr, out["T"])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i, depth_dev[i], tinit_dev[i])
    barrier()

    # the e2e run below replays the same frames from the same map state (integration changes the map)
    snap = vol.storage.clone()

    # ---- device-resident timed region
    idx = list(range(args.warmup, args.warmup + args.steps))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
    with Clocks(local) as clk:
        barrier()
        pft.profile_start()
        l0 = pft.launch_count()
        for j, i in enumerate(idx):
            flush.zero_()
            ev[j][0].record(stream)
            step(i, depth_dev[i], tinit_dev[i])
            ev[j][1].record(stream)
        barrier()
        launches = pft.launch_count() - l0
        prof = pft.profile_stop()
        per_step_eager = [a.elapsed_time(b) for a, b in ev]
        n_chk = int(out["trace"][-1, 21].item())
        assert n_chk == n_valid[idx[-1]], (n_chk, n_valid[idx[-1]])
        graphs = None
        if not args.no_graph:
            # one frame (pft_track + pft_integrate: memsets, the cooperative tracker, the cull and
            # fusion kernels) captured as a CUDA graph per input-buffer pair, replayed per step;
            # the eager loop above supplies the per-kernel breakdown and the launch count
            gd = [torch.empty_like(depth_dev[0]) for _ in range(2)]
            gt = [torch.empty_like(tinit_dev[0]) for _ in range(2)]
            graphs = []
            for b in range(2):
                gd[b].copy_(depth_dev[0])
                gt[b].copy_(tinit_dev[0])
                step(0, gd[b], gt[b])  # warm-up on these buffers (the map is restored below)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(0, gd[b], gt[b])
                graphs.append(g)
            vol.storage.copy_(snap)
            barrier()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
            for j, i in enumerate(idx):
                flush.zero_()
                ev[j][0].record(stream)
                gd[0].copy_(depth_dev[i])  # the graph's static inputs (D2D, inside the window)
                gt[0].copy_(tinit_dev[i])
                graphs[0].replay()
                ev[j][1].record(stream)
            barrier()
            n_chk = int(out["trace"][-1, 21].item())
            assert n_chk == n_valid[idx[-1]], (n_chk, n_valid[idx[-1]])
    per_step = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(per_step)
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    tot_evals = sum(evals[i] for i in idx)
    value = tot_evals / (t_max * 1e-3)

    # ---- end-to-end through the public API with host buffers
    host_depth = [torch.from_numpy(s["depth"]).pin_memory() for s in steps_in]
    host_tinit = [torch.from_numpy(s["T_init"]).pin_memory() for s in steps_in]
    host_T = [torch.empty(3, 4, dtype=torch.float64).pin_memory() for _ in idx]
    # double-buffered inputs: frame j+1's H2D runs on a copy stream while frame j computes (a
    # user's pipeline); every copy lies inside some step's event window (frame 0's inside its own)
    d_buf = gd if graphs else [torch.empty_like(depth_dev[0]) for _ in range(2)]
    t_buf = gt if graphs else [torch.empty_like(tinit_dev[0]) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)

    def prefetch(j):
        i, b = idx[j], j & 1
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(used[b])
            d_buf[b].copy_(host_depth[i], non_blocking=True)
            t_buf[b].copy_(host_tinit[i], non_blocking=True)
            ready[b].record(cs)

    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
    vol.storage.copy_(snap)
    del snap
    barrier()
    for j, i in enumerate(idx):
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
            step(i, d_buf[b], t_buf[b])
        used[b].record(stream)
        host_T[j].copy_(out["T"], non_blocking=True)
        ev2[j][1].record(stream)
    barrier()
    # tracked pose vs GT per frame (characterisation of the paper-literal rule)
    rot_err, tr_err = [], []
    for j, i in enumerate(idx):
        Tg, Tt = seq.gt[steps_in[i]["t"]], host_T[j].numpy()
        c = (np.trace(Tg[:, :3].T @ Tt[:, :3]) - 1.0) / 2.0
        rot_err.append(float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))))
        tr_err.append(float(np.linalg.norm(Tg[:, 3] - Tt[:, 3]) * 100.0))
    e2e_ms = sum(a.elapsed_time(b) for a, b in ev2)
    if world > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = host_depth[0].numel() * 2 + 96
    d2h = 96

    # ---- roofline of the dominant kernel (k_particle_eval)
    if prof["eval"][1] > 0:       # multi-launch tracker: k_particle_eval is the dominant kernel
        kname, (eval_ms, eval_n) = "k_particle_eval", prof["eval"]
        evals_per_launch = K_PER_GPU * statistics.mean(n_valid[i] for i in idx)
    else:                         # persistent tracker: one launch per frame holds all 10 iterations
        kname, (eval_ms, eval_n) = "k_track_persistent (eval+update+centre phases)", prof["track"]
        evals_per_launch = K_PER_GPU * ITERS * statistics.mean(n_valid[i] for i in idx)
    avg_launch_s = eval_ms / eval_n * 1e-3
    gather_gbs = evals_per_launch * BYTES_PER_EVAL / avg_launch_s / 1e9
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # issue-slot ceiling from unit counts and clocks: SMs x 128 lanes x f_max
    alu_peak = n_sm * LANES_PER_SM * sm_mhz * 1e6 / 1e12
    achieved = evals_per_launch * OPS_PER_EVAL / avg_launch_s / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "eval_traffic.json")
    if os.path.exists(tf):
        tj = json.load(open(tf))
        traffic = tj.get("dram_bytes_per_eval", 0) * evals_per_launch

    # gather-replay ceiling (tools/gather_replay.py on the bench map): the evaluation's exact mask +
    # record address stream replayed without arithmetic, next to the tracker on the same frame
    gather_view = None
    gr = os.path.join(ROOT, "profiles", "r01_gather_replay.jsonl")
    if os.path.exists(gr):
        rows = [json.loads(x) for x in open(gr) if x.strip()]
        ref = [x for x in rows if x.get("init_noise_deg_cm") == 5.0 and x.get("frame") == 12] or rows
        x = ref[0]
        gather_view = {"replay_evals_per_s": x["replay_evals_per_s"], "track_evals_per_s": x["track_evals_per_s"],
                       "frac": x["track_evals_per_s"] / x["replay_evals_per_s"], "inband_frac": x["inband_frac"],
                       "source": "profiles/r01_gather_replay.jsonl (frame %d, +-%g deg/cm init)" % (
                           x["frame"], x["init_noise_deg_cm"])}

    # ---- particle sweep (BASELINE config 4 sizes) on the same 512^3 map, one frame, 10 iterations
    sweep = {}
    if world == 1:
        for Ks in (4096, 16384, 65536):
            from synth.configs import make_pst
            pst_s = torch.from_numpy(make_pst(args.seed, Ks)).to(dev)
            o2 = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev),
                      E=torch.empty(Ks, dtype=torch.float64, device=dev), n=torch.empty(Ks, dtype=torch.int32, device=dev),
                      trace=None)
            i0 = idx[0]
            vol.track(depth_dev[i0], intr, tinit_dev[i0], pst_s, params, out=o2)
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                vol.track(depth_dev[i0], intr, tinit_dev[i0], pst_s, params, out=o2)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            sweep[str(Ks)] = {"evals_per_s": Ks * n_valid[i0] * ITERS / (min(ts) * 1e-3), "ms_track": min(ts)}
            del pst_s, o2
        vol._ws = {}

    # ---- F4 surface extraction on the bench map (NEXT row F4): one full pass over V and W
    extract = {}
    if world == 1:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        lib_ = pft.lib()
        import ctypes as C
        lib_.pft_extract_surface(vol.handle, C.c_void_p(0), 0, C.c_void_p(cnt.data_ptr()),
                                 C.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        npts = int(cnt.item())
        pts_buf = torch.empty(max(npts, 1), 3, dtype=torch.float64, device=dev)
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lib_.pft_extract_surface(vol.handle, C.c_void_p(pts_buf.data_ptr()), npts, C.c_void_p(cnt.data_ptr()),
                                     C.c_void_p(stream.cuda_stream))
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms_x = statistics.median(ts)
        esz = 4 if getattr(desc, "storage", "f32") == "f32" else 2
        nbytes = 2 * esz * vol.nvox + 24 * npts  # V + W once, the points written
        extract = {"ms": ms_x, "points": npts, "algorithmic_bytes": nbytes,
                   "achieved_gbs": nbytes / (ms_x * 1e-3) / 1e9, "frac_of_hbm": nbytes / (ms_x * 1e-3) / 1e9 / hbm_peak}
        del pts_buf

    # ---- F2 fused exchange, emulated on this GPU: G rank groups in one persistent launch (same K)
    fused = {}
    if world == 1:
        i0 = idx[0]
        o3 = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(K, dtype=torch.float64, device=dev),
                  n=torch.empty(K, dtype=torch.int32, device=dev), trace=None)
        for G in (1, 2, 4, 8):
            vol.comm_init_virtual(G, fused=True)
            vol.track(depth_dev[i0], intr, tinit_dev[i0], pst, params, out=o3)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                vol.track(depth_dev[i0], intr, tinit_dev[i0], pst, params, out=o3)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            fused[str(G)] = {"ms_track": statistics.median(ts)}
        vol.comm_init_virtual(1)
        vol._ws = {}
        del o3

    # ---- config L: 1024^3 @ 5 mm fp16 volume built by integration, K = 4096 track + integrate per frame
    large = {}
    if world == 1 and not args.no_large:
        from synth.configs import Sequence
        sl = Sequence("L", seed=args.seed, n_frames=max(len(map_depth) + 8, 16), K=4096, iters=ITERS)
        voll = pft.Volume(sl.desc, dev)
        voll.reset()
        for t in range(len(map_depth)):
            voll.integrate(torch.from_numpy(sl.depth(t)).to(dev), sl.intr, torch.from_numpy(sl.gt[t].copy()).to(dev))
        pst_l = torch.from_numpy(sl.pst).to(dev)
        frames = [len(map_depth) + f for f in range(6)]
        dl = [torch.from_numpy(sl.depth(t)).to(dev) for t in frames]
        from synth.configs import init_noise
        tl = [torch.from_numpy(init_noise(args.seed, t, sl.gt[t], 5.0, 5.0)).to(dev) for t in frames]
        ol = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(4096, dtype=torch.float64, device=dev),
                  n=torch.empty(4096, dtype=torch.int32, device=dev), trace=None)
        voll.track(dl[0], sl.intr, tl[0], pst_l, sl.params, out=ol)
        voll.integrate(dl[0], sl.intr, ol["T"])
        torch.cuda.synchronize()
        pft.profile_start()
        ms = []
        for f in range(1, len(frames)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            voll.track(dl[f], sl.intr, tl[f], pst_l, sl.params, out=ol)
            voll.integrate(dl[f], sl.intr, ol["T"])
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        pl = pft.profile_stop()
        nvl = strided_valid(sl.depth(frames[1]), 4)
        large = {"workload": "L: 1024^3 @5 mm fp16 V+W, tau 2 cm, K=4096, 10 iters, 640x480",
                 "ms_per_frame_median": statistics.median(ms),
                 "evals_per_s": 4096 * nvl * ITERS / (statistics.median(ms) * 1e-3),
                 "kernel_ms_per_frame": {k: v[0] / len(ms) for k, v in pl.items() if v[1]}}
        voll.close()
        del pst_l, dl, tl, ol

    res = {
        "metric": "particle-point TSDF evals/s (track) with ms per 640x480 frame (track+integrate)",
        "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 transform/decisions, f32 TSDF + lerp, int64 fixed-point sums",
        "data": "synthetic (seeded box room + shaky trajectory, BASELINE config 3)",
        "config": {"workload": "Q: 640x480 frame, 160x120 points, K=2048/GPU, 10 iters, 512^3 @1cm fp32 TSDF, "
                               "track + integrate", "particles": K, "points_per_frame": statistics.mean(n_valid),
                   "iters": ITERS, "volume": "512^3 fp32", "l2": "flushed (256 MiB write) between steps",
                   "parallelism": f"particles sharded x{world}, volume replicated"
                   + (f", {exchange} exchange" if world > 1 else "")},
        "frame_ms": {"median": statistics.median(per_step), "p99": float(np.percentile(per_step, 99)),
                     "max": max(per_step)},
        "launch": "CUDA graph per frame (track + integrate), replayed" if graphs else "eager library calls",
        "eager_ms_per_step": sum(per_step_eager) / args.steps,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]},
        "e2e": {"value": tot_evals / (e2e_ms * 1e-3), "unit": "evals/s", "ms_per_step": e2e_ms / args.steps,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "Tops/s",
                     "frac": achieved / alu_peak, "traffic": traffic, "kernel": kname,
                     "basis": f"{OPS_PER_EVAL} algorithmic ops/eval x {evals_per_launch:.0f} evals/launch / event time; "
                              f"peak = {n_sm} SMs x {LANES_PER_SM} lanes x {sm_mhz:.0f} MHz issue slots (DESIGN.md §7)",
                     "evals_per_s_kernel": evals_per_launch / avg_launch_s,
                     "gather_view": gather_view,
                     "hbm_view": {"logical_gather_gbs": gather_gbs, "peak_gbs": hbm_peak, "frac": gather_gbs / hbm_peak,
                                  "note": f"{BYTES_PER_EVAL} B corner gather/eval, served from L2/L1 (DRAM traffic "
                                          "is 'traffic'); not the binding resource"}},
        "clocks": clk.summary(),
        "particle_sweep": sweep,
        "fused_exchange_emulation": fused,
        "extract_surface": extract,
        "large_volume": large,
        "pose_err_vs_gt": {"rot_deg_median": statistics.median(rot_err), "rot_deg_p90": float(np.percentile(rot_err, 90)),
                           "trans_cm_median": statistics.median(tr_err), "trans_cm_p90": float(np.percentile(tr_err, 90)),
                           "note": "paper-literal RO from GT (+) U+-5deg/+-5cm, per frame (SURVEY.md 8(c-5))"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the contract: rank 0 at N=1 only
        res["cpu_baseline"] = cpu_baseline(args, seq, map_depth, [steps_in[i] for i in idx])
    if rank == 0:
        print(json.dumps(res), flush=True)
    vol.close()
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- oracle arms
def oracle_map(seq, map_depth):
    import oracle
    ov = oracle.OracleVolume(seq.desc)
    for t, d in enumerate(map_depth):
        ov.integrate(d, seq.intr, seq.gt[t])
    return ov


def cores():
    return len(os.sched_getaffinity(0))


def cpu_baseline(args, seq, map_depth, steps, budget_s=10.0):
    """The oracle as it stands, on this host's cores: full RO tracking (K particles, 10 iterations)
    of consecutive timed frames until ~budget_s of CPU work (>= 1 frame), in evals/s."""
    ov = oracle_map(seq, map_depth)
    ev, dt, nf = 0, 0.0, 0
    for s in steps:
        t0 = time.perf_counter()
        r = ov.track(s["depth"], seq.intr, s["T_init"], seq.pst, seq.params, nthreads=cores())
        dt += time.perf_counter() - t0
        ev += len(seq.pst) * r["N"] * seq.params.iters
        nf += 1
        if dt >= budget_s:
            break
    # effective parallelism: the same one-frame track on 1 thread vs all cores,
    # on a small particle subset
    s0 = steps[0]
    sub = seq.pst[:128].copy()
    t1 = time.perf_counter()
    ov.track(s0["depth"], seq.intr, s0["T_init"], sub, seq.params, nthreads=1)
    t1 = time.perf_counter() - t1
    tn = time.perf_counter()
    ov.track(s0["depth"], seq.intr, s0["T_init"], sub, seq.params, nthreads=cores())
    tn = time.perf_counter() - tn
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": ev / dt, "unit": "evals/s", "cores": cores(), "kind": "oracle",
            "cpu_model": model, "effective_parallelism": t1 / tn,
            "sample": f"{nf} frame(s) of full RO tracking ({len(seq.pst)} particles x {seq.params.iters} iterations "
                      f"x {r['N']} points) on a 512^3 fp32 map fused by the oracle from {len(map_depth)} frames; "
                      f"{dt:.1f} s"}


def run_reference(args):
    """The fp64 CPU oracle as the reference arm (this tier has no reference implementation): the
    same workload per step as our arm (K = 2048 x N particles, 10 iterations, 160x120 points, then
    fusion into the 512^3 map), on this host's cores.  Under torchrun only rank 0 runs."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    seq, map_depth, steps_in = make_workload(args, args.warmup + args.steps, world)
    ov = oracle_map(seq, map_depth)
    per, evs = [], []
    for i, s in enumerate(steps_in):
        t0 = time.perf_counter()
        r = ov.track(s["depth"], seq.intr, s["T_init"], seq.pst, seq.params, nthreads=cores())
        ov.integrate(s["depth"], seq.intr, r["T"], nthreads=cores())
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            per.append(dt)
            evs.append(len(seq.pst) * r["N"] * seq.params.iters)
    value = sum(evs) / sum(per)
    res = {"impl": "reference",
           "metric": "particle-point TSDF evals/s (track) with ms per 640x480 frame (track+integrate)",
           "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(per) / len(per), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded box room + shaky trajectory, config 3)",
           "config": {"workload": f"Q: 640x480 frame, 160x120 points, K={len(seq.pst)}, 10 iters, 512^3 @1cm fp32 "
                                  "TSDF, track + integrate (full workload per step, fp64 CPU oracle)"},
           "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores(), "kind": "oracle",
                            "sample": f"full workload: {len(per)} timed frames (+{args.warmup} warm-up), "
                                      f"{len(seq.pst)} particles x {seq.params.iters} iterations + fusion"},
           "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
