"""Diagnostic: config L lock-step; for any n_k mismatch report the oracle's decision margin."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle, paper_2509_24236_b200 as pft
from synth.configs import Sequence
from synth.scene import compose
dev = torch.device("cuda", 0)
def T(x): return torch.from_numpy(np.ascontiguousarray(x)).to(dev)
seq = Sequence("L", seed=1, n_frames=8, K=4096, iters=10)
vol = pft.Volume(seq.desc, dev); vol.reset(); ov = oracle.OracleVolume(seq.desc)
d0 = seq.depth(0); vol.integrate(T(d0), seq.intr, T(seq.gt[0])); ov.integrate(d0, seq.intr, seq.gt[0])
P_prev = seq.gt[0]
for t in range(1, 3):
    depth = seq.depth(t); T_init = compose(P_prev, seq.rel_init(t))
    r = vol.track(T(depth), seq.intr, T(T_init), T(seq.pst), seq.params); torch.cuda.synchronize()
    o = ov.track(depth, seq.intr, T_init, seq.pst, seq.params)
    n = r["n"].cpu().numpy(); bad = np.nonzero(n != o["n"])[0]
    print("frame", t, "mismatches", bad, "gpu", n[bad], "ora", o["n"][bad], "track min margin", o["margin"])
    tr = o["trace"]
    P_last = tr[-2, 4:16].reshape(3, 4) if len(tr) > 1 else T_init
    om, v = tr[-1, 2], tr[-1, 3]
    for k in bad:
        dR, _, u = oracle.delta(seq.pst[k], om, v)
        Tk = oracle.apply_delta(dR, u, P_last, 0)
        e = ov.eval_poses(depth, seq.intr, Tk[None], stride=4)
        print("  k", k, "oracle n", e["n"], "E", e["E"], "margin", e["margin"], "gpu E", r["E"].cpu().numpy()[k], "ora E", o["E"][k])
    P_prev = o["T"]
    vol.integrate(T(depth), seq.intr, T(P_prev)); ov.integrate(depth, seq.intr, P_prev)
