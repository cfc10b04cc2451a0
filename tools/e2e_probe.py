"""Where does the end-to-end step (host depth/T_init in, T_out back) lose time against the
device-resident step?  Times the config-Q frame (track + integrate) with CUDA events under variants:
resident inputs; H2D depth+T on the compute stream; + D2H of T; H2D on a side stream one frame ahead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence, init_noise

dev = torch.device("cuda", 0)
seq = Sequence("Q", seed=1, n_frames=40, K=2048, iters=10)
vol = pft.Volume(seq.desc, dev)
vol.reset()
for t in range(8):
    vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
frames = list(range(8, 28))
hd = [torch.from_numpy(seq.depth(t)).pin_memory() for t in frames]
ht = [torch.from_numpy(init_noise(1, t, seq.gt[t], 5.0, 5.0)).pin_memory() for t in frames]
dd = [x.to(dev) for x in hd]
dt = [x.to(dev) for x in ht]
pst = torch.from_numpy(seq.pst).to(dev)
out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(2048, dtype=torch.float64, device=dev),
           n=torch.empty(2048, dtype=torch.int32, device=dev), trace=None)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
hT = [torch.empty(3, 4, dtype=torch.float64).pin_memory() for _ in frames]
d_buf, t_buf = torch.empty_like(dd[0]), torch.empty_like(dt[0])


def step(d, t):
    vol.track(d, seq.intr, t, pst, seq.params, out=out)
    vol.integrate(d, seq.intr, out["T"])


def timed(body, label):
    for i in range(3):
        body(i)
    torch.cuda.synchronize()
    ms = []
    for i in range(len(frames)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        body(i)
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"{label:40s} median {np.median(ms):.3f} ms  mean {np.mean(ms):.3f}")


timed(lambda i: step(dd[i], dt[i]), "resident")
timed(lambda i: step(dd[i], dt[i]) or hT[i].copy_(out["T"], non_blocking=True), "resident + D2H T")


def h2d(i):
    d_buf.copy_(hd[i], non_blocking=True)
    t_buf.copy_(ht[i], non_blocking=True)
    step(d_buf, t_buf)


timed(h2d, "H2D depth+T")


def full(i):
    h2d(i)
    hT[i].copy_(out["T"], non_blocking=True)


timed(full, "H2D + D2H (bench e2e)")
timed(lambda i: step(dd[i], dt[i]), "resident again")
