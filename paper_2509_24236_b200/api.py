"""Thin Python binding over libpft.so (include/pft.h): argument marshalling only.

PyTorch provides device memory, streams and process groups; every step of the path runs in
the library's CUDA kernels.  Tensors passed in must already live on the current CUDA device.
"""
import ctypes as C

import torch

from ._lib import (INTEGRATE_FULL_SWEEP, IPC_HANDLE_BYTES, TRACE_DOUBLES, Intrinsics, TrackParams, VolumeDesc, check, lib)

STORE = {"f32": 0, "f16": 1, 0: 0, 1: 1}


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_desc(d):
    return VolumeDesc(int(d.nx), int(d.ny), int(d.nz), float(d.voxel_m), (C.c_double * 3)(*d.origin_m),
                      float(d.trunc_m), float(getattr(d, "max_weight", 128.0)), float(getattr(d, "max_depth_m", 8.0)),
                      STORE[getattr(d, "storage", "f32")])


def make_intr(k):
    return Intrinsics(float(k.fx), float(k.fy), float(k.cx), float(k.cy), int(k.width), int(k.height),
                      float(getattr(k, "depth_unit_m", 0.001)))


def make_params(p):
    def arr(name):
        v = [int(x) for x in getattr(p, name, (0, 0, 0, 0))] + [0, 0, 0, 0]
        return (C.c_int32 * 4)(*v[:4])
    return TrackParams(float(p.omega0_deg), float(p.v0_cm), float(p.beta), int(p.iters), int(p.stride),
                       float(p.min_inband_frac), int(p.delta_conv), int(p.update_rule), int(p.topk),
                       int(getattr(p, "nsched", 0)), arr("sched_K"), arr("sched_sx"), arr("sched_sy"),
                       float(getattr(p, "min_search_deg", 0.0)), float(getattr(p, "min_search_cm", 0.0)),
                       int(getattr(p, "guard", 0)), int(getattr(p, "stall_limit", 0)))


def _dev_tensor(x, dtype, device):
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=dtype)
    else:
        t = torch.as_tensor(x, dtype=dtype).to(device)
    return t.contiguous()


class Volume:
    """A TSDF volume whose storage is a torch uint8 tensor on `device`, borrowed by the library."""

    def __init__(self, desc, device=None):
        self.desc = desc
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._cdesc = make_desc(desc)
        nbytes = C.c_size_t()
        check(lib().pft_volume_bytes(C.byref(self._cdesc), C.byref(nbytes)))
        self.nbytes = nbytes.value
        self.storage = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        h = C.c_void_p()
        check(lib().pft_volume_create(C.byref(self._cdesc), _vp(self.storage), self.nbytes, C.byref(h)))
        self.handle = h
        self._ws = {}
        self.nranks, self.rank = 1, 0

    @property
    def storage_dtype(self):
        return torch.float32 if STORE[getattr(self.desc, "storage", "f32")] == 0 else torch.float16

    @property
    def nvox(self):
        return int(self.desc.nx) * int(self.desc.ny) * int(self.desc.nz)

    # --------------------------------------------------------------- volume
    def reset(self, stream=None):
        check(lib().pft_volume_reset(self.handle, _stream(stream)))

    def upload(self, V, W, stream=None):
        """Canonical x-fastest arrays (numpy or torch) in the storage precision; fp16 may be
        given as float16 or as raw uint16 bit patterns."""
        dt = self.storage_dtype
        def conv(x):
            if not isinstance(x, torch.Tensor):
                x = torch.from_numpy(x.reshape(-1).copy())
            if dt == torch.float16 and x.dtype in (torch.uint16, torch.int16):
                x = x.view(torch.float16)
            return x.reshape(-1).to(device=self.device, dtype=dt).contiguous()
        v, w = conv(V), conv(W)
        assert v.numel() == self.nvox and w.numel() == self.nvox
        check(lib().pft_volume_upload(self.handle, _vp(v), _vp(w), _stream(stream)))
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()

    def download(self, stream=None):
        v = torch.empty(self.nvox, dtype=self.storage_dtype, device=self.device)
        w = torch.empty_like(v)
        check(lib().pft_volume_download(self.handle, _vp(v), _vp(w), _stream(stream)))
        return v, w

    def checksum(self, stream=None):
        h = C.c_uint64()
        check(lib().pft_volume_checksum(self.handle, C.byref(h), _stream(stream)))
        return h.value

    # --------------------------------------------------------------- fusion
    def integrate(self, depth, intr, T, full_sweep=False, stream=None):
        """depth: (H, W) uint16 device tensor; T: 3x4 (or 12) fp64 device tensor."""
        ci = make_intr(intr)
        check(lib().pft_integrate_ex(self.handle, _vp(depth), C.byref(ci), _vp(T),
                                     INTEGRATE_FULL_SWEEP if full_sweep else 0, _stream(stream)))

    def integrate_stats(self, stream=None):
        """Work counters of the last culled integrate (include/pft.h pft_integrate_stats): dict of
        kept bricks, free-space bricks, updated voxels, rebuilt cell-bricks.  Syncs."""
        out = (C.c_int64 * 4)()
        check(lib().pft_integrate_stats(self.handle, out, _stream(stream)))
        return dict(kept_bricks=out[0], free_bricks=out[1], updated_voxels=out[2], dirty_cell_bricks=out[3])

    def extract_surface(self, max_points=None, stream=None):
        """F4 zero-crossing surface points -> (N, 3) fp64 device tensor (unordered)."""
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        if max_points is None:
            check(lib().pft_extract_surface(self.handle, C.c_void_p(0), 0, _vp(cnt), _stream(stream)))
            max_points = int(cnt.item())
        pts = torch.empty(max(max_points, 1), 3, dtype=torch.float64, device=self.device)
        check(lib().pft_extract_surface(self.handle, _vp(pts), int(max_points), _vp(cnt), _stream(stream)))
        n = int(cnt.item())
        return pts[:min(n, max_points)]

    # --------------------------------------------------------------- tracking
    def workspace(self, intr, nparticles, params):
        ci, cp = make_intr(intr), make_params(params)
        n = C.c_size_t()
        check(lib().pft_track_workspace_bytes(self.handle, C.byref(ci), int(nparticles), C.byref(cp), C.byref(n)))
        key = n.value
        ws = self._ws.get(key)
        if ws is None:
            ws = torch.empty(key, dtype=torch.uint8, device=self.device)
            self._ws = {key: ws}
        return ws

    def track(self, depth, intr, T_init, pst, params, trace=True, out=None, stream=None):
        """Randomized optimisation.  Returns dict(T, E, n, trace) of device
        tensors (asynchronous; nothing is synchronised here)."""
        K = int(pst.shape[0])
        ci, cp = make_intr(intr), make_params(params)
        ws = self.workspace(intr, K, params)
        if out is None:
            out = dict(T=torch.empty(3, 4, dtype=torch.float64, device=self.device),
                       E=torch.empty(K, dtype=torch.float64, device=self.device),
                       n=torch.empty(K, dtype=torch.int32, device=self.device),
                       trace=torch.zeros(int(params.iters), TRACE_DOUBLES, dtype=torch.float64, device=self.device)
                       if trace else None)
        check(lib().pft_track(self.handle, _vp(depth), C.byref(ci), _vp(T_init), _vp(pst), K, C.byref(cp),
                              _vp(ws), ws.numel(), _vp(out["T"]), _vp(out["E"]), _vp(out["n"]),
                              _vp(out.get("trace")), _stream(stream)))
        out["ws"] = ws
        return out

    def eval_poses(self, depth, intr, poses, params, stream=None):
        """E and in-band count of M explicit poses (M x 3 x 4 fp64 device tensor)."""
        M = int(poses.shape[0])
        ci, cp = make_intr(intr), make_params(params)
        ws = self.workspace(intr, M, params)
        E = torch.empty(M, dtype=torch.float64, device=self.device)
        n = torch.empty(M, dtype=torch.int32, device=self.device)
        check(lib().pft_eval_poses(self.handle, _vp(depth), C.byref(ci), C.byref(cp), _vp(poses), M, _vp(ws),
                                   ws.numel(), _vp(E), _vp(n), _stream(stream)))
        return dict(E=E, n=n, ws=ws)

    def npoints(self, ws, stream=None):
        n = C.c_int32()
        check(lib().pft_track_info(_vp(ws), C.byref(n), _stream(stream)))
        return n.value

    # --------------------------------------------------------------- multi-GPU
    def comm_init(self, group=None):
        """Attach an NCCL communicator over the ranks of torch.distributed `group` (one GPU each)."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            check(lib().pft_comm_get_unique_id(buf))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            uid = uid.to(self.device)
        dist.broadcast(uid, 0, group=group)
        raw = (C.c_uint8 * 128)(*uid.cpu().tolist())
        check(lib().pft_comm_init(self.handle, raw, world, rank))
        self.nranks, self.rank = world, rank
        self._ws = {}

    def comm_init_virtual(self, nranks, fused=False):
        """Test/debug: run the multi-GPU path with nranks shards on this GPU -- sequential shard
        launches + device copies (fused=False), or the F2 fused exchange with nranks rank groups
        of CTAs in one persistent launch (fused=True)."""
        fn = lib().pft_comm_init_virtual_fused if fused else lib().pft_comm_init_virtual
        check(fn(self.handle, int(nranks)))
        self.nranks, self.rank = int(nranks), 0
        self._ws = {}

    def comm_init_p2p(self, max_particles, group=None, preflight_ms=2000):
        """F2 fused exchange over NVLink peer memory: allocate this rank's exchange buffer, gather
        every rank's CUDA IPC handle over torch.distributed `group`, open the peers', then run the
        pre-flight token exchange (include/pft.h pft_comm_p2p_preflight; no trap on failure).  All
        ranks agree on the outcome (all-reduces of a success flag): returns True when every rank is
        attached and every pre-flight succeeded; otherwise every rank has detached again and False
        is returned (use comm_init)."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        h = (C.c_uint8 * IPC_HANDLE_BYTES)()
        ok = lib().pft_comm_p2p_init(self.handle, world, rank, int(max_particles), h) == 0
        handles = gather_handles(bytes(h), group)
        if ok:
            raw = (C.c_uint8 * (IPC_HANDLE_BYTES * world))(*handles)
            ok = lib().pft_comm_p2p_attach(self.handle, raw) == 0
        if not _all_ranks(ok, group, self.device):
            check(lib().pft_comm_p2p_detach(self.handle))
            return False
        dist.barrier(group=group)
        okp = C.c_int32(0)
        ok = lib().pft_comm_p2p_preflight(self.handle, int(preflight_ms), C.byref(okp), _stream(None)) == 0
        if not _all_ranks(ok and okp.value == 1, group, self.device):
            check(lib().pft_comm_p2p_detach(self.handle))
            return False
        self.nranks, self.rank = world, rank
        self._ws = {}
        return True

    def set_partition(self, points):
        """F2b: shard the points (True) or the particles (False, default) across the ranks of the
        NCCL communicator / virtual shards (include/pft.h pft_comm_set_partition)."""
        check(lib().pft_comm_set_partition(self.handle, 1 if points else 0))
        self._ws = {}

    def comm_detach_p2p(self):
        """Undo comm_init_p2p on this rank (single-rank again)."""
        check(lib().pft_comm_p2p_detach(self.handle))
        self.nranks, self.rank = 1, 0
        self._ws = {}

    def close(self):
        if getattr(self, "handle", None):
            lib().pft_volume_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _all_ranks(ok, group, device):
    """True iff `ok` holds on every rank of `group` (an all-reduce MIN of a flag)."""
    import torch.distributed as dist
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32)
    if dist.get_backend(group) == "nccl":
        flag = flag.to(device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return int(flag.item()) == 1


def pose_compose(A, B, out=None, stream=None):
    """out = A * B for 3x4 rigid poses on the device (include/pft.h pft_pose_compose)."""
    if out is None:
        out = torch.empty(3, 4, dtype=torch.float64, device=A.device)
    check(lib().pft_pose_compose(_vp(A), _vp(B), _vp(out), _stream(stream)))
    return out


def gather_handles(mine, group=None):
    """All ranks' IPC handles (IPC_HANDLE_BYTES each) concatenated in rank order, as a byte string.
    Host-side plumbing only (tests/test_multirank.py exercises it over gloo)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    assert len(mine) == IPC_HANDLE_BYTES
    t = torch.tensor(list(mine), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.to(torch.device("cuda", torch.cuda.current_device()))
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return b"".join(bytes(o.cpu().tolist()) for o in out)


def shard_range(K, nranks, rank):
    """Particles rank `rank` evaluates (include/pft.h: rows [r*ceil(K/G), ...))."""
    kloc = -(-K // nranks)
    b = rank * kloc
    return b, max(0, min(K, b + kloc) - b)
