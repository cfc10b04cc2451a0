"""Runs the bench frame (config Q map, K particles, 10 iterations) with PFT_PHASE_TIMING=1 so the
persistent tracker prints per-phase device times (debug aid)."""
import os
import sys

os.environ["PFT_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence, init_noise, make_pst

dev = torch.device("cuda", 0)
seq = Sequence("Q", seed=1, n_frames=16, K=2048, iters=10)
vol = pft.Volume(seq.desc, dev)
vol.reset()
for t in range(8):
    vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
d = torch.from_numpy(seq.depth(9)).to(dev)
Ti = torch.from_numpy(init_noise(1, 9, seq.gt[9], 5.0, 5.0)).to(dev)
for K in [int(x) for x in sys.argv[1:]] or [2048]:
    pst = torch.from_numpy(make_pst(1, K)).to(dev)
    for rep in range(2):
        vol.track(d, seq.intr, Ti, pst, seq.params)
        torch.cuda.synchronize()
