"""Where the bench's end-to-end step (host depth / relative init in, tracked pose out) loses time
against the device-resident graph step: the bench's double-buffered e2e loop timed with CUDA events
under variants -- (a) as bench.py (H2D of frame j+1 on a copy stream during frame j, D2H of the
pose on the compute stream); (b) without the D2H; (c) without the cross-stream wait (inputs already
on the device); (d) the pose written to mapped pinned host memory by a kernel (pft_pose_compose
with an identity right factor) instead of a memcpy."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence

dev = torch.device("cuda", 0)
seq = Sequence("Q", seed=1, n_frames=48, K=2048, iters=10)
vol = pft.Volume(seq.desc, dev)
vol.reset()
intr, params = seq.intr, seq.params
pst = torch.from_numpy(seq.pst).to(dev)
out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(2048, dtype=torch.float64, device=dev),
           n=torch.empty(2048, dtype=torch.int32, device=dev),
           trace=torch.zeros(10, pft.TRACE_DOUBLES, dtype=torch.float64, device=dev))
T_prev = torch.from_numpy(seq.gt[0].copy()).to(dev)
T_init = torch.empty(3, 4, dtype=torch.float64, device=dev)
eye = torch.zeros(3, 4, dtype=torch.float64, device=dev)
eye[0, 0] = eye[1, 1] = eye[2, 2] = 1.0


def step(depth, rel):
    pft.pose_compose(T_prev, rel, out=T_init)
    vol.track(depth, intr, T_init, pst, params, out=out)
    vol.integrate(depth, intr, out["T"])
    T_prev.copy_(out["T"])


vol.integrate(torch.from_numpy(seq.depth(0)).to(dev), intr, T_prev)
for t in range(1, 12):
    step(torch.from_numpy(seq.depth(t)).to(dev), torch.from_numpy(seq.rel_init(t).copy()).to(dev))
torch.cuda.synchronize()
idx = list(range(12, 32))
host_depth = {t: torch.from_numpy(seq.depth(t)).pin_memory() for t in idx}
host_rel = {t: torch.from_numpy(seq.rel_init(t).copy()).pin_memory() for t in idx}
dev_depth = {t: host_depth[t].to(dev) for t in idx}
dev_rel = {t: host_rel[t].to(dev) for t in idx}
host_T = torch.empty(len(idx), 3, 4, dtype=torch.float64).pin_memory()
snap, snap_T = vol.storage.clone(), T_prev.clone()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
stream = torch.cuda.current_stream()
gd = [torch.empty_like(dev_depth[idx[0]]) for _ in range(2)]
gr = [torch.empty_like(dev_rel[idx[0]]) for _ in range(2)]
graphs = []
for b in range(2):
    gd[b].copy_(dev_depth[idx[0]])
    gr[b].copy_(dev_rel[idx[0]])
    step(gd[b], gr[b])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(gd[b], gr[b])
    graphs.append(g)

# (d) mapped pinned host memory for the pose, written by a kernel
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
mapped_ptr = mapped_dev = None
if cudart is not None:
    hp = C.c_void_p()
    if cudart.cudaHostAlloc(C.byref(hp), C.c_size_t(96 * len(idx)), C.c_uint(2)) == 0:  # cudaHostAllocMapped
        dp = C.c_void_p()
        if cudart.cudaHostGetDevicePointer(C.byref(dp), hp, C.c_uint(0)) == 0:
            mapped_ptr, mapped_dev = hp.value, dp.value


def run(label, d2h="memcpy", h2d=True):
    vol.storage.copy_(snap)
    T_prev.copy_(snap_T)
    torch.cuda.synchronize()
    ready = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)

    def prefetch(j):
        t, b = idx[j], j & 1
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(used[b])
            gd[b].copy_(host_depth[t], non_blocking=True)
            gr[b].copy_(host_rel[t], non_blocking=True)
            ready[b].record(cs)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in idx]
    for j, t in enumerate(idx):
        flush.zero_()
        ev[j][0].record(stream)
        b = j & 1
        if h2d:
            if j == 0:
                cs.wait_event(ev[0][0])
                prefetch(0)
            stream.wait_event(ready[b])
            if j + 1 < len(idx):
                prefetch(j + 1)
        else:
            gd[b].copy_(dev_depth[t])
            gr[b].copy_(dev_rel[t])
        graphs[b].replay()
        used[b].record(stream)
        if d2h == "memcpy":
            host_T[j].copy_(out["T"], non_blocking=True)
        elif d2h == "pinned_kernel":  # torch's pinned tensor written by a kernel through its UVA mapping
            pft.pose_compose(out["T"], eye, out=host_T[j])
        elif d2h == "mapped":
            pft.check(pft.lib().pft_pose_compose(C.c_void_p(out["T"].data_ptr()), C.c_void_p(eye.data_ptr()),
                                                 C.c_void_p(mapped_dev + 96 * j), C.c_void_p(stream.cuda_stream)))
        ev[j][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    print(f"{label:48s} mean {np.mean(ms):.4f} ms  median {np.median(ms):.4f}")


for rep in range(2):
    run("graph, inputs D2D (bench value)", d2h="none", h2d=False)
    run("e2e as bench (H2D copy stream + D2H memcpy)")
    run("e2e without the D2H", d2h="none")
    run("D2D inputs + D2H memcpy", d2h="memcpy", h2d=False)
    if mapped_dev:
        run("e2e with the pose to mapped host memory", d2h="mapped")
    run("e2e with the pose to torch pinned memory by a kernel", d2h="pinned_kernel")
    ref = out["T"].cpu()
    assert torch.equal(host_T[len(idx) - 1], ref), (host_T[len(idx) - 1], ref)
