"""CPU checks of the C ABI boundary (no GPU needed): libpft.so builds for sm_100a, loads, exports
every symbol include/pft.h declares, and rejects invalid arguments before touching a device.
Also: the product package must not import the oracle."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pft():
    import paper_2509_24236_b200 as m
    if not os.path.exists(m.LIB_PATH):
        subprocess.check_call(["sh", os.path.join(ROOT, "paper_2509_24236_b200", "csrc", "build.sh")])
    m.lib()
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pft.h")).read()
    return sorted(set(re.findall(r"^\s*(?:pft_status|const char\*|int32_t|uint64_t)\s+(pft_\w+)\s*\(", src, re.M)))


def test_header_matches_binding_exports(pft):
    assert header_symbols() == sorted(pft.EXPORTS)


def test_library_exports_every_header_symbol(pft):
    out = subprocess.check_output(["nm", "-D", "--defined-only", pft.LIB_PATH]).decode()
    defined = set(re.findall(r"\sT\s(pft_\w+)", out))
    missing = [s for s in header_symbols() if s not in defined]
    assert not missing, missing


def test_library_is_sm100a(pft):
    out = subprocess.check_output(["cuobjdump", "--list-elf", pft.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_abi_version(pft):
    assert pft.lib().pft_abi_version() == 4


def _desc(pft, **kw):
    from paper_2509_24236_b200._lib import VolumeDesc
    d = dict(nx=64, ny=64, nz=64, voxel_m=0.02, origin=(0.0, 0.0, 0.0), trunc_m=0.06, max_weight=128.0,
             max_depth_m=8.0, storage=0)
    d.update(kw)
    return VolumeDesc(d["nx"], d["ny"], d["nz"], d["voxel_m"], (C.c_double * 3)(*d["origin"]), d["trunc_m"],
                      d["max_weight"], d["max_depth_m"], d["storage"])


def test_volume_bytes_and_validation(pft):
    L = pft.lib()
    n = C.c_size_t()
    assert L.pft_volume_bytes(C.byref(_desc(pft)), C.byref(n)) == 0
    # 64^3 fp32 values + weights + scratch + brick list + tile scratch
    assert n.value >= 2 * 64 ** 3 * 4
    n16 = C.c_size_t()
    assert L.pft_volume_bytes(C.byref(_desc(pft, storage=1)), C.byref(n16)) == 0
    assert n16.value < n.value
    bad = [dict(nx=1), dict(nz=4097), dict(voxel_m=0.0), dict(trunc_m=0.03), dict(max_weight=0.5), dict(storage=7),
           dict(max_depth_m=0.0)]
    for b in bad:
        assert L.pft_volume_bytes(C.byref(_desc(pft, **b)), C.byref(n)) == -1, b
        assert L.pft_last_error()
    assert L.pft_volume_bytes(C.byref(_desc(pft, nx=2048, ny=2048, nz=1024)), C.byref(n)) == -6  # > 2^31 voxels
    assert L.pft_volume_bytes(None, C.byref(n)) == -1


def test_create_workspace_and_argument_errors(pft):
    """Host-only paths: create on a fake (never dereferenced) aligned pointer, size queries and
    argument validation all return before any device work."""
    from paper_2509_24236_b200._lib import Intrinsics, TrackParams
    L = pft.lib()
    d = _desc(pft)
    n = C.c_size_t()
    L.pft_volume_bytes(C.byref(d), C.byref(n))
    h = C.c_void_p()
    fake = C.c_void_p(1 << 40)
    assert L.pft_volume_create(C.byref(d), fake, n.value - 1, C.byref(h)) == -2
    assert L.pft_volume_create(C.byref(d), C.c_void_p((1 << 40) + 8), n.value, C.byref(h)) == -1  # misaligned
    assert L.pft_volume_create(C.byref(d), fake, n.value, C.byref(h)) == 0
    K = Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480, 0.001)
    p = TrackParams(10.0, 10.0, 0.1, 10, 4, 0.0, 0, 0, 0)
    ws = C.c_size_t()
    assert L.pft_track_workspace_bytes(h, C.byref(K), 1024, C.byref(p), C.byref(ws)) == 0
    # points (160 x 120 strided grid padded to 8x4 tiles) as 3 fp64 + 16 B per particle
    assert ws.value >= 160 * 120 * 24 + 1024 * 16
    assert L.pft_track_workspace_bytes(h, C.byref(K), 0, C.byref(p), C.byref(ws)) == -1
    nul = C.c_void_p(0)
    dummy = C.c_void_p(1 << 41)
    def track(prm, ws_bytes=1 << 30, Kp=1024):
        return L.pft_track(h, dummy, C.byref(K), dummy, dummy, Kp, C.byref(prm), dummy, ws_bytes, dummy, dummy,
                           dummy, nul, nul)
    assert track(TrackParams(10.0, 10.0, 1.0, 10, 4, 0.0, 0, 0, 0)) == -1      # beta = 1
    assert track(TrackParams(10.0, 10.0, 0.1, 0, 4, 0.0, 0, 0, 0)) == -1       # iters = 0
    assert track(TrackParams(120.0, 10.0, 0.1, 10, 4, 0.0, 0, 0, 0)) == -1     # omega > 100
    assert track(TrackParams(10.0, 10.0, 0.1, 10, 0, 0.0, 0, 0, 0)) == -1      # stride 0
    assert track(TrackParams(10.0, 10.0, 0.1, 10, 4, 0.0, 0, 2, 0)) == -1      # top-k needs 1 <= topk <= 32
    assert track(TrackParams(10.0, 10.0, 0.1, 10, 4, 0.0, 0, 2, 33)) == -1
    assert track(TrackParams(10.0, 10.0, 0.1, 10, 4, 0.0, 0, 3, 0)) == -1      # unknown rule
    assert track(p, ws_bytes=16) == -2                                          # workspace too small
    assert track(p, Kp=0) == -1
    badK = Intrinsics(0.0, 525.0, 319.5, 239.5, 640, 480, 0.001)
    assert L.pft_track(h, dummy, C.byref(badK), dummy, dummy, 16, C.byref(p), dummy, 1 << 30, dummy, dummy, dummy,
                       nul, nul) == -1
    assert L.pft_integrate(h, nul, C.byref(K), dummy, nul) == -1
    # F2 exchange: argument and state validation happens before any device call
    hbuf = (C.c_uint8 * 64)()
    assert L.pft_comm_p2p_init(nul, 2, 0, 1024, hbuf) == -1
    assert L.pft_comm_p2p_init(h, 1, 0, 1024, hbuf) == -1          # needs >= 2 ranks
    assert L.pft_comm_p2p_init(h, 9, 0, 1024, hbuf) == -1          # <= PFT_MAX_FUSED_RANKS
    assert L.pft_comm_p2p_init(h, 2, 2, 1024, hbuf) == -1          # rank out of range
    assert L.pft_comm_p2p_init(h, 2, 0, 0, hbuf) == -1             # max_particles >= 1
    assert L.pft_comm_p2p_attach(h, hbuf) == -7                    # init not called
    assert L.pft_comm_p2p_detach(h) == 0 and L.pft_comm_p2p_detach(nul) == -1
    assert L.pft_comm_init_virtual_fused(h, 0) == -1
    assert L.pft_comm_init_virtual_fused(h, 9) == -1
    assert L.pft_comm_init_virtual_fused(h, 4) == 0
    ws8 = C.c_size_t()
    assert L.pft_track_workspace_bytes(h, C.byref(K), 1024, C.byref(p), C.byref(ws8)) == 0
    assert ws8.value >= 4 * ws.value                               # one region per emulated rank
    assert L.pft_comm_init_virtual(h, 1) == 0
    assert L.pft_volume_destroy(h) == 0


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2509_24236_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".sh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle/)", "").lower() or f == "__init__.py", f
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "pft_oracle" not in src and "liboracle" not in src, f


def test_no_cs2r_short_distance_reads(pft):
    """Regression guard for the stale-register hazard seen on B200: no
    'CS2R Rx, SRZ' whose destination is read fewer than 6 issue-stall cycles later."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_hazard_scan
    hits = sass_hazard_scan.scan(pft.LIB_PATH, 6)
    assert not hits, hits[:5]
