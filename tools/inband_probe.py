"""Tracker throughput versus the in-band fraction of the evaluations: the bench frame (config Q map,
K = 2048, 10 iterations) tracked from inits at decreasing distance to GT (+-5 deg/cm as in the bench
down to +-0.2), reporting the centre's in-band fraction (trace n_c / N) and evaluations/s."""
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
snap = vol.storage.clone()
pst = torch.from_numpy(seq.pst).to(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for noise in (5.0, 2.0, 1.0, 0.5, 0.2):
    ms, fr = [], []
    vol.storage.copy_(snap)
    for t in range(8, 16):
        d = torch.from_numpy(seq.depth(t)).to(dev)
        Ti = torch.from_numpy(init_noise(1, t, seq.gt[t], noise, noise)).to(dev)
        vol.track(d, seq.intr, Ti, pst, seq.params)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = vol.track(d, seq.intr, Ti, pst, seq.params)
        e1.record()
        torch.cuda.synchronize()
        tr = r["trace"].cpu().numpy()
        ms.append(e0.elapsed_time(e1))
        fr.append(float(np.mean(tr[:, 20] / np.maximum(tr[:, 21], 1))))
        N = float(tr[0, 21])
        vol.integrate(d, seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
    print(json.dumps({"init_noise_deg_cm": noise, "centre_inband_frac": float(np.mean(fr)),
                      "track_ms_median": float(np.median(ms)),
                      "evals_per_s": 2048 * N * 10 / (float(np.median(ms)) * 1e-3)}))
