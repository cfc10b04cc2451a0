"""ctypes declarations of libpft.so (include/pft.h).  Argument marshalling only.

The shared library is built in-tree (``paper_2509_24236_b200/libpft.so``) by
``__graft_entry__.build()`` / ``csrc/build.sh``.  There is no fallback: if the library is
missing or fails to load, every call raises.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PFT_LIB") or os.path.join(HERE, "libpft.so")
TRACE_DOUBLES = 24
IPC_HANDLE_BYTES = 64          # include/pft.h PFT_IPC_HANDLE_BYTES
MAX_FUSED_RANKS = 8            # include/pft.h PFT_MAX_FUSED_RANKS
INTEGRATE_FULL_SWEEP = 1

STATUS = {0: "PFT_OK", -1: "PFT_ERR_INVALID_ARG", -2: "PFT_ERR_BUFFER_TOO_SMALL", -3: "PFT_ERR_EMPTY_CLOUD",
          -4: "PFT_ERR_CUDA", -5: "PFT_ERR_NCCL", -6: "PFT_ERR_UNSUPPORTED", -7: "PFT_ERR_STATE"}

# every symbol include/pft.h declares (checked by tests/test_abi.py)
EXPORTS = ["pft_volume_bytes", "pft_volume_create", "pft_volume_reset", "pft_volume_upload", "pft_volume_download",
           "pft_volume_checksum", "pft_volume_destroy", "pft_integrate", "pft_integrate_ex", "pft_integrate_stats", "pft_extract_surface",
           "pft_track_workspace_bytes", "pft_track", "pft_eval_poses", "pft_track_info", "pft_pose_compose", "pft_comm_get_unique_id",
           "pft_comm_init", "pft_comm_init_virtual", "pft_comm_init_virtual_fused", "pft_comm_p2p_init",
           "pft_comm_p2p_attach", "pft_comm_p2p_detach", "pft_comm_p2p_preflight", "pft_comm_set_partition", "pft_last_error", "pft_abi_version", "pft_launch_count", "pft_profile_start",
           "pft_profile_stop"]
PROF_CLASSES = ["eval", "centre", "update", "prep", "integrate", "cull", "comm", "other", "records", "track"]


class PftError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class VolumeDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("voxel_m", C.c_double),
                ("origin_m", C.c_double * 3), ("trunc_m", C.c_double), ("max_weight", C.c_double),
                ("max_depth_m", C.c_double), ("storage", C.c_int32)]


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_unit_m", C.c_double)]


class TrackParams(C.Structure):
    _fields_ = [("omega0_deg", C.c_double), ("v0_cm", C.c_double), ("beta", C.c_double),
                ("iters", C.c_int32), ("stride", C.c_int32), ("min_inband_frac", C.c_double),
                ("delta_conv", C.c_int32), ("update_rule", C.c_int32), ("topk", C.c_int32),
                ("nsched", C.c_int32), ("sched_K", C.c_int32 * 4), ("sched_sx", C.c_int32 * 4),
                ("sched_sy", C.c_int32 * 4), ("min_search_deg", C.c_double), ("min_search_cm", C.c_double),
                ("guard", C.c_int32), ("stall_limit", C.c_int32)]


_lib = None


def lib():
    """Load libpft.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (or csrc/build.sh) first")
    L = C.CDLL(LIB_PATH)
    P, I32, SZ, D = C.c_void_p, C.c_int32, C.c_size_t, C.c_double
    sig = {
        "pft_volume_bytes": [P, P],
        "pft_volume_create": [P, P, SZ, P],
        "pft_volume_reset": [P, P],
        "pft_volume_upload": [P, P, P, P],
        "pft_volume_download": [P, P, P, P],
        "pft_volume_checksum": [P, P, P],
        "pft_volume_destroy": [P],
        "pft_integrate": [P, P, P, P, P],
        "pft_integrate_ex": [P, P, P, P, I32, P],
        "pft_integrate_stats": [P, P, P],
        "pft_extract_surface": [P, P, C.c_int64, P, P],
        "pft_track_workspace_bytes": [P, P, I32, P, P],
        "pft_track": [P, P, P, P, P, I32, P, P, SZ, P, P, P, P, P],
        "pft_eval_poses": [P, P, P, P, P, I32, P, SZ, P, P, P],
        "pft_track_info": [P, P, P],
        "pft_comm_get_unique_id": [P],
        "pft_comm_init": [P, P, I32, I32],
        "pft_comm_init_virtual": [P, I32],
        "pft_comm_init_virtual_fused": [P, I32],
        "pft_comm_p2p_init": [P, I32, I32, I32, P],
        "pft_comm_p2p_attach": [P, P],
        "pft_comm_p2p_detach": [P],
        "pft_comm_p2p_preflight": [P, I32, P, P],
        "pft_comm_set_partition": [P, I32],
        "pft_pose_compose": [P, P, P, P],
        "pft_profile_start": [],
        "pft_profile_stop": [P, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.pft_last_error.restype = C.c_char_p
    L.pft_last_error.argtypes = []
    L.pft_abi_version.restype = C.c_int32
    L.pft_abi_version.argtypes = []
    L.pft_launch_count.restype = C.c_uint64
    L.pft_launch_count.argtypes = []
    _lib = L
    return L


def launch_count():
    return int(lib().pft_launch_count())


def profile_start():
    check(lib().pft_profile_start())


def profile_stop():
    """-> {class: (total_ms, launches)} of the library's kernels since profile_start (syncs)."""
    ms = (C.c_double * len(PROF_CLASSES))()
    n = (C.c_int64 * len(PROF_CLASSES))()
    check(lib().pft_profile_stop(ms, n))
    return {c: (ms[i], n[i]) for i, c in enumerate(PROF_CLASSES)}


def check(status):
    if status != 0:
        raise PftError(status, lib().pft_last_error().decode(errors="replace"))
    return status
