"""Integration work per frame on the bench map (config Q, 512^3 fp32): bricks kept by the cull,
voxels actually updated, cell-bricks marked dirty, and per-kernel device times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_24236_b200 as pft
from synth.configs import Sequence

kind = sys.argv[1] if len(sys.argv) > 1 else "Q"
dev = torch.device("cuda", 0)
seq = Sequence(kind, seed=1, n_frames=16, K=2048, iters=10)
vol = pft.Volume(seq.desc, dev)
vol.reset()
for t in range(8):
    vol.integrate(torch.from_numpy(seq.depth(t)).to(dev), seq.intr, torch.from_numpy(seq.gt[t].copy()).to(dev))
torch.cuda.synchronize()
for t in range(8, 12):
    d = torch.from_numpy(seq.depth(t)).to(dev)
    T = torch.from_numpy(seq.gt[t].copy()).to(dev)
    V0, W0 = [x.clone() for x in vol.download()]
    pft.profile_start()
    vol.integrate(d, seq.intr, T)
    prof = pft.profile_stop()
    torch.cuda.synchronize()
    V1, W1 = vol.download()
    sc = vol.storage[:256].view(torch.int32).cpu().numpy()
    changed_w = int((W1 != W0).sum())
    changed_v = int((V1 != V0).sum())
    wmax = float(getattr(seq.desc, "max_weight", 128.0))
    sat = int(((W1 == W0) & (W1 == wmax)).sum())
    print(f"frame {t}: kept bricks {sc[16]} ({sc[16] * 64} voxels), super-bricks {sc[48]}, dirty cell-bricks {sc[32]}, "
          f"W changed {changed_w}, V changed {changed_v}, W saturated+unchanged {sat}; "
          + " ".join(f"{k} {v[0] * 1e3:.1f}us/{v[1]}" for k, v in prof.items() if v[1]))
