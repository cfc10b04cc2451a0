"""Single-rank NCCL communicator (torch.distributed world_size 1): runs pft_track through the
collective path -- ncclAllGather of the particle records, or with the point partition ncclAllReduce
of the per-particle and centre sums -- and saves T, E, n, trace and the launch count per call."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main(cfg, partition, out, port):
    import torch
    import torch.distributed as dist
    from tests.helpers.run_track import make_case
    import paper_2509_24236_b200 as pft
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = port
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    c, params = make_case(cfg, 1)
    vol = pft.Volume(c["desc"], dev)
    vol.upload(c["V"], c["W"])
    vol.comm_init()
    if partition == "points":
        vol.set_partition(True)
    args = (torch.from_numpy(c["depth"]).to(dev), c["intr"], torch.from_numpy(c["T_init"]).to(dev),
            torch.from_numpy(c["pst"]).to(dev), params)
    vol.track(*args)
    torch.cuda.synchronize()
    n0 = pft.launch_count()
    r = vol.track(*args)
    torch.cuda.synchronize()
    launches = pft.launch_count() - n0
    np.savez(out, launches=np.array([launches]), **{k: r[k].cpu().numpy() for k in ("T", "E", "n", "trace")})
    vol.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(*sys.argv[1:5])
