"""Runs pft_track on a seeded config and saves T, E, n, trace (used by tests that compare
library code paths across processes, e.g. PFT_TRACK_PERSISTENT=0 vs 1)."""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def make_case(cfg, seed):
    """(config dict, params) of a named case (shared with the tests that compare it to the oracle)."""
    from synth.configs import config_single, config_tiny, with_desc
    import dataclasses
    c = config_tiny(seed=seed) if cfg.startswith("tiny") else config_single(seed=seed)
    c = dict(c)
    if cfg == "single_topk":
        c["params"] = dataclasses.replace(c["params"], update_rule=2, topk=16, iters=5)
    if cfg == "tiny_sched":
        c["params"] = dataclasses.replace(c["params"], iters=7, nsched=3, sched_K=(64, 40, 24, 0),
                                          sched_sx=(1, 2, 4, 0), sched_sy=(1, 2, 2, 0), guard=1, update_rule=1,
                                          stall_limit=3, min_search_deg=0.05, min_search_cm=0.05)
    if cfg == "tiny_bigK":
        # more than 256 update blocks of 256 particles: the combine's general path (K > 65536)
        from synth.configs import make_pst
        c["pst"] = make_pst(seed, 70000)
        c["params"] = dataclasses.replace(c["params"], iters=2)
    if cfg == "tiny16":
        c = with_desc(c, storage="f16")
        c["V"], c["W"] = c["V"].astype(np.float16), c["W"].astype(np.float16)
    return c, c["params"]


def main(cfg, seed, out):
    import torch
    import paper_2509_24236_b200 as pft
    c, params = make_case(cfg, seed)
    dev = torch.device("cuda", 0)
    vol = pft.Volume(c["desc"], dev)
    vol.upload(c["V"], c["W"])
    r = vol.track(torch.from_numpy(c["depth"]).to(dev), c["intr"], torch.from_numpy(c["T_init"]).to(dev),
                  torch.from_numpy(c["pst"]).to(dev), params)
    torch.cuda.synchronize()
    np.savez(out, **{k: r[k].cpu().numpy() for k in ("T", "E", "n", "trace")})


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
