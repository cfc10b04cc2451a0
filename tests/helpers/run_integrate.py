"""Fuses three frames of the room into a reset volume and saves V, W and the work counters (used
to compare library integration paths across processes, e.g. PFT_INTEGRATE_FUSED=1 vs default)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main(storage, out):
    import torch
    import paper_2509_24236_b200 as pft
    from synth.configs import VolumeDesc, room_gt_pose
    from synth.rng import Stream
    from synth.scene import Intrinsics, box_room, perturb, render_depth
    scene = box_room(seed=4)
    desc = VolumeDesc(128, 128, 128, 0.02, (-1.28, -1.28, -1.28), 0.06, storage=storage)
    intr = Intrinsics(131.25, 131.25, 79.5, 59.5, 160, 120)
    T_gt = room_gt_pose(scene, 4)
    dev = torch.device("cuda", 0)
    vol = pft.Volume(desc, dev)
    vol.reset()
    stats = []
    for f in range(3):
        Tf = perturb(T_gt, [0.0, 0.0, 0.1 * f], [0.05 * f, 0.0, 0.0], 10.0, 10.0)
        depth = render_depth(scene, intr, Tf, Stream(4, 4_000_000 + f))
        vol.integrate(torch.from_numpy(depth).to(dev), intr, torch.from_numpy(Tf).to(dev))
        s = vol.integrate_stats()
        stats.append([s["kept_bricks"], s["free_bricks"], s["updated_voxels"], s["dirty_cell_bricks"]])
    V, W = [x.cpu().numpy() for x in vol.download()]
    np.savez(out, V=V, W=W, stats=np.array(stats), checksum=np.array([vol.checksum()], dtype=np.uint64))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
