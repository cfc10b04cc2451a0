"""Can one frame (pft_track + pft_integrate: the cooperative persistent tracker, the cull kernels,
memsets) be captured into a CUDA graph and replayed?  Compares the replay time per frame with the
eager stream of library calls, and checks the replayed results equal the eager ones."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence, init_noise

dev = torch.device("cuda", 0)
seq = Sequence("Q", seed=1, n_frames=24, K=2048, iters=10)
vol = pft.Volume(seq.desc, dev)
vol.reset()
for t in range(8):
    vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
pst = torch.from_numpy(seq.pst).to(dev)
frames = list(range(8, 20))
dd = [torch.from_numpy(seq.depth(t)).to(dev) for t in frames]
tt = [torch.from_numpy(init_noise(1, t, seq.gt[t], 5.0, 5.0)).to(dev) for t in frames]
d_buf, t_buf = torch.empty_like(dd[0]), torch.empty_like(tt[0])
K = 2048
out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=dev), E=torch.empty(K, dtype=torch.float64, device=dev),
           n=torch.empty(K, dtype=torch.int32, device=dev), trace=None)
snap = vol.storage.clone()


def step():
    vol.track(d_buf, seq.intr, t_buf, pst, seq.params, out=out)
    vol.integrate(d_buf, seq.intr, out["T"])


# eager reference
s = torch.cuda.Stream()
res_eager, ms_eager = [], []
with torch.cuda.stream(s):
    for i in range(len(frames)):
        d_buf.copy_(dd[i])
        t_buf.copy_(tt[i])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        step()
        e1.record(s)
        s.synchronize()
        ms_eager.append(e0.elapsed_time(e1))
        res_eager.append(out["T"].cpu().numpy().copy())
# graph capture of one frame (after a warm-up call on the same stream)
vol.storage.copy_(snap)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
err = None
try:
    with torch.cuda.stream(s):
        d_buf.copy_(dd[0])
        t_buf.copy_(tt[0])
        step()
        s.synchronize()
        vol.storage.copy_(snap)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            step()
except Exception as e:  # noqa: BLE001
    err = repr(e)
res = {"capture_error": err}
if err is None:
    vol.storage.copy_(snap)
    torch.cuda.synchronize()
    ms_graph, same = [], True
    with torch.cuda.stream(s):
        for i in range(len(frames)):
            d_buf.copy_(dd[i])
            t_buf.copy_(tt[i])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            s.synchronize()
            ms_graph.append(e0.elapsed_time(e1))
            same = same and np.array_equal(out["T"].cpu().numpy(), res_eager[i])
    res.update({"eager_ms_median": float(np.median(ms_eager[2:])), "graph_ms_median": float(np.median(ms_graph[2:])),
                "graph_results_equal_eager": bool(same)})
print(json.dumps(res))
