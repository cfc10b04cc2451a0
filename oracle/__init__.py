"""fp64 CPU oracle for the PROFusion RO-tracking + TSDF-fusion hot path.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never from the product package
(paper_2509_24236_b200/).  The arithmetic lives in pft_oracle.c (plain C, fp64,
-O2 -ffp-contract=off); this module is argument marshalling via ctypes.
See pft_oracle.c for the per-function paper citations.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pft_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
TRACE_DOUBLES = 24


def build(force=False):
    """Compile liboracle.so (gcc, fp64, no FMA contraction, OpenMP over independent items)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=gnu11",
                           "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


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
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.ora_backproject.restype = C.c_int32
        _lib.ora_backproject.argtypes = [P, P, C.c_int32, C.c_double, P]
        _lib.ora_backproject2.restype = C.c_int32
        _lib.ora_backproject2.argtypes = [P, P, C.c_int32, C.c_int32, C.c_double, P]
        _lib.ora_query.restype = C.c_int32
        _lib.ora_query.argtypes = [P, P, P, P, P]
        _lib.ora_fitness.restype = C.c_double
        _lib.ora_fitness.argtypes = [P, P, P, C.c_int32, P, C.c_double, P, P]
        _lib.ora_delta.restype = None
        _lib.ora_delta.argtypes = [P, C.c_double, C.c_double, P, P, P]
        _lib.ora_apply_delta.restype = None
        _lib.ora_apply_delta.argtypes = [P, P, P, C.c_int32, P]
        _lib.ora_quat_to_R.restype = None
        _lib.ora_quat_to_R.argtypes = [P, P]
        _lib.ora_track.restype = C.c_int32
        _lib.ora_track.argtypes = [P, P, P, P, P, P, C.c_int32, P, P, P, P, P, P, P, C.c_int32]
        _lib.ora_track_ex.restype = C.c_int32
        _lib.ora_track_ex.argtypes = [P, P, P, P, P, P, C.c_int32, P, P, P, P, P, P, P, P, P, C.c_int32]
        _lib.ora_eval_poses.restype = C.c_int32
        _lib.ora_eval_poses.argtypes = [P, P, P, P, C.c_int32, C.c_double, P, C.c_int32, P, P, P, P, C.c_int32]
        _lib.ora_integrate.restype = C.c_int64
        _lib.ora_integrate.argtypes = [P, P, P, P, P, P, C.c_int32]
        _lib.ora_reset.restype = None
        _lib.ora_reset.argtypes = [P, P, P]
        _lib.ora_extract.restype = C.c_int64
        _lib.ora_extract.argtypes = [P, P, P, P, C.c_int64]
        _lib.ora_round_to_storage.restype = C.c_double
        _lib.ora_round_to_storage.argtypes = [C.c_double, C.c_int32]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def default_threads():
    return max(1, len(os.sched_getaffinity(0)))


def make_desc(d):
    """From a synth VolumeDesc (or any object with the same fields)."""
    out = VolumeDesc(d.nx, d.ny, d.nz, d.voxel_m, (C.c_double * 3)(*d.origin_m), d.trunc_m,
                     d.max_weight, d.max_depth_m, 0 if d.storage == "f32" else 1)
    return out


def make_intr(k):
    return Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_unit_m)


def make_params(p):
    def arr(name):
        v = list(getattr(p, name, (0, 0, 0, 0))) + [0, 0, 0, 0]
        return (C.c_int32 * 4)(*v[:4])
    return TrackParams(p.omega0_deg, p.v0_cm, p.beta, p.iters, p.stride, p.min_inband_frac,
                       p.delta_conv, p.update_rule, p.topk, getattr(p, "nsched", 0), arr("sched_K"), arr("sched_sx"),
                       arr("sched_sy"), getattr(p, "min_search_deg", 0.0), getattr(p, "min_search_cm", 0.0),
                       getattr(p, "guard", 0), getattr(p, "stall_limit", 0))


def densest_slots(intr, params):
    """Point slots of the densest point set a run uses (workspace size)."""
    sets = [(params.stride, params.stride)]
    for j in range(getattr(params, "nsched", 0)):
        sets.append((params.sched_sx[j], params.sched_sy[j]))
    return max((-(-intr.height // sy)) * (-(-intr.width // sx)) for sx, sy in sets)


def storage_dtype(desc):
    return np.float32 if desc.storage == "f32" else np.uint16


class OracleVolume:
    """Canonical x-fastest V/W arrays in the storage precision (fp16 as raw uint16 bits)."""

    def __init__(self, desc, V=None, W=None):
        self.desc = desc
        self.cdesc = make_desc(desc)
        n = desc.nx * desc.ny * desc.nz
        dt = storage_dtype(desc)
        if V is None:
            self.V = np.empty(n, dtype=dt)
            self.W = np.empty(n, dtype=dt)
            lib().ora_reset(_p(self.V), _p(self.W), C.byref(self.cdesc))
        else:
            self.V = np.ascontiguousarray(V).view(dt).ravel().copy()
            self.W = np.ascontiguousarray(W).view(dt).ravel().copy()

    def values_f64(self):
        if self.desc.storage == "f32":
            return self.V.astype(np.float64)
        return self.V.view(np.float16).astype(np.float64)

    def weights_f64(self):
        if self.desc.storage == "f32":
            return self.W.astype(np.float64)
        return self.W.view(np.float16).astype(np.float64)

    def query(self, q):
        """O3 at world point q -> (in_band, v, margin)."""
        v = np.zeros(1)
        m = np.ones(1)
        q = np.ascontiguousarray(q, dtype=np.float64)
        ok = lib().ora_query(_p(self.V), C.byref(self.cdesc), _p(q), _p(v), _p(m))
        return bool(ok), float(v[0]), float(m[0])

    def fitness(self, pts, T, rho=0.0):
        """O4 -> (E, n, margin)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        T = np.ascontiguousarray(T, dtype=np.float64)
        n = np.zeros(1, dtype=np.int32)
        m = np.ones(1)
        E = lib().ora_fitness(_p(self.V), C.byref(self.cdesc), _p(pts), len(pts), _p(T), rho, _p(n), _p(m))
        return E, int(n[0]), float(m[0])

    def integrate(self, depth, intr, T, nthreads=None):
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        T = np.ascontiguousarray(T, dtype=np.float64)
        ci = make_intr(intr)
        return int(lib().ora_integrate(_p(self.V), _p(self.W), C.byref(self.cdesc), _p(depth), C.byref(ci),
                                       _p(T), nthreads or default_threads()))

    def track(self, depth, intr, T_init, pst, params, nthreads=None, force=None):
        """O7/O8 -> dict(T, E, n, trace, N, margin, emargin).  emargin[i]: iteration i's smallest
        relative distance of a fitness decision to its threshold (inf for iterations not run);
        force (iters x K int8, -1 = decide): the shadowed re-run with a given membership
        (pft_oracle.c ora_track_ex)."""
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        T_init = np.ascontiguousarray(T_init, dtype=np.float64)
        pst = np.ascontiguousarray(pst, dtype=np.float32)
        K = pst.shape[0]
        ws = np.zeros(3 * densest_slots(intr, params))
        T = np.zeros(12)
        E = np.zeros(K)
        n = np.zeros(K, dtype=np.int32)
        tr = np.zeros((params.iters, TRACE_DOUBLES))
        m = np.ones(1)
        em = np.full(params.iters, np.inf)
        ci, cp = make_intr(intr), make_params(params)
        fp = None
        if force is not None:
            force = np.ascontiguousarray(force, dtype=np.int8).reshape(params.iters, K)
            fp = _p(force)
        N = lib().ora_track_ex(_p(self.V), C.byref(self.cdesc), _p(depth), C.byref(ci), _p(T_init), _p(pst), K,
                               C.byref(cp), _p(ws), _p(T), _p(E), _p(n), _p(tr), _p(m), _p(em), fp,
                               nthreads or default_threads())
        return dict(T=T.reshape(3, 4), E=E, n=n, trace=tr, N=N, margin=float(m[0]), emargin=em)

    def extract(self, max_pts=None):
        """F4 zero-crossing surface points (N x 3, canonical voxel/axis order)."""
        n = lib().ora_extract(_p(self.V), _p(self.W), C.byref(self.cdesc), None, 0)
        pts = np.zeros((max(n, 1), 3))
        lib().ora_extract(_p(self.V), _p(self.W), C.byref(self.cdesc), _p(pts), n)
        return pts[:n]

    def eval_poses(self, depth, intr, poses, stride, rho=0.0, nthreads=None):
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 12)
        M = poses.shape[0]
        ws = np.zeros(3 * (-(-intr.height // stride)) * (-(-intr.width // stride)))
        E = np.zeros(M)
        n = np.zeros(M, dtype=np.int32)
        mg = np.ones(M)
        ci = make_intr(intr)
        N = lib().ora_eval_poses(_p(self.V), C.byref(self.cdesc), _p(depth), C.byref(ci), stride, rho, _p(poses), M,
                                 _p(ws), _p(E), _p(n), _p(mg), nthreads or default_threads())
        return dict(E=E, n=n, N=N, margin=mg)


def backproject(depth, intr, stride, max_depth_m=8.0, stride_y=None):
    """O2 strided points; stride_y given: 2-D strides (stride on columns, stride_y on rows)."""
    depth = np.ascontiguousarray(depth, dtype=np.uint16)
    sy = stride if stride_y is None else stride_y
    ws = np.zeros(3 * (-(-intr.height // sy)) * (-(-intr.width // stride)))
    ci = make_intr(intr)
    N = lib().ora_backproject2(_p(depth), C.byref(ci), stride, sy, max_depth_m, _p(ws))
    return ws[: 3 * N].reshape(N, 3)


def delta(a, omega_deg, v_cm):
    a = np.ascontiguousarray(a, dtype=np.float32)
    dR = np.zeros(9)
    q = np.zeros(4)
    u = np.zeros(3)
    lib().ora_delta(_p(a), omega_deg, v_cm, _p(dR), _p(q), _p(u))
    return dR.reshape(3, 3), q, u


def apply_delta(dR, u, P, conv=0):
    dR = np.ascontiguousarray(dR, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    P = np.ascontiguousarray(P, dtype=np.float64)
    out = np.zeros(12)
    lib().ora_apply_delta(_p(dR), _p(u), _p(P), conv, _p(out))
    return out.reshape(3, 4)


def quat_to_R(q):
    q = np.ascontiguousarray(q, dtype=np.float64)
    R = np.zeros(9)
    lib().ora_quat_to_R(_p(q), _p(R))
    return R.reshape(3, 3)


def round_to_storage(x, storage):
    return lib().ora_round_to_storage(float(x), 0 if storage == "f32" else 1)


def rotation_error_rad(Ra, Rb):
    """l_R = arccos((tr(Ra^T Rb) - 1)/2), argument clamped to [-1,1]."""
    c = (np.trace(np.asarray(Ra)[:3, :3].T @ np.asarray(Rb)[:3, :3]) - 1.0) / 2.0
    return float(np.arccos(np.clip(c, -1.0, 1.0)))
