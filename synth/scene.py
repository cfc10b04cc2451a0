"""Analytic scenes, closed-form depth rendering and camera poses (input generation only).

World is z-up; the camera is x right, y down, z forward; a pose is a 3x4
row-major [R|t] mapping camera to world (p_w = R p_c + t).
Depth is the z-depth along the optical axis in uint16 millimetres
(BASELINE.json configs), rounded half-to-even and clamped to [1, 65535];
pixels whose ray hits nothing are 0.  Noise (configs S/Q/W/L) is
z += N(0, (0.0012 z^2)^2) before rounding.
"""
from dataclasses import dataclass, field
import numpy as np

from .rng import Stream


# ----------------------------------------------------------------------------- rotations
def rotvec_to_matrix(r):
    """Rotation matrix of a rotation vector (generator-side Rodrigues)."""
    r = np.asarray(r, dtype=np.float64)
    th = float(np.sqrt(r @ r))
    if th < 1e-12:
        K = _skew(r)
        return np.eye(3) + K
    k = r / th
    K = _skew(k)
    return np.eye(3) + np.sin(th) * K + (1.0 - np.cos(th)) * (K @ K)


def _skew(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def rot_z(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def pose(R, t):
    T = np.zeros((3, 4))
    T[:, :3] = R
    T[:, 3] = t
    return T


def compose(A, B):
    """A*B for 3x4 rigid poses."""
    return pose(A[:, :3] @ B[:, :3], A[:, :3] @ B[:, 3] + A[:, 3])


def inverse(A):
    Rt = A[:, :3].T
    return pose(Rt, -Rt @ A[:, 3])


def look_at(C, target):
    """Camera->world pose at centre C looking at target, world up = +z."""
    f = np.asarray(target, float) - np.asarray(C, float)
    f /= np.linalg.norm(f)
    right = np.cross(f, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    return pose(np.stack([right, down, f], axis=1), np.asarray(C, float))


def perturb(T, a, b, deg, cm):
    """Box perturbation of a pose, camera-centred convention:
    r = a*deg*pi/180, u = b*cm/100, result = (Rodrigues(r) R, t + u)."""
    dR = rotvec_to_matrix(np.asarray(a, float) * (deg * np.pi / 180.0))
    return pose(dR @ T[:, :3], T[:, 3] + np.asarray(b, float) * (cm / 100.0))


# ----------------------------------------------------------------------------- scenes
@dataclass
class Scene:
    """Union of primitives; signed distance is positive in free space."""
    spheres: list = field(default_factory=list)      # [(cx, cy, cz, r)]
    plane_z: float = None                             # ground plane z = plane_z (free space above)
    room_half: float = None                           # box room interior |x|,|y|,|z| < room_half

    def sdf(self, p):
        """p: (..., 3) fp64 -> (...) signed distance in metres."""
        p = np.asarray(p, dtype=np.float64)
        d = np.full(p.shape[:-1], np.inf)
        if self.room_half is not None:
            h = self.room_half
            d = np.minimum(d, np.minimum(np.minimum(h - np.abs(p[..., 0]), h - np.abs(p[..., 1])), h - np.abs(p[..., 2])))
        if self.plane_z is not None:
            d = np.minimum(d, p[..., 2] - self.plane_z)
        for (cx, cy, cz, r) in self.spheres:
            q0, q1, q2 = p[..., 0] - cx, p[..., 1] - cy, p[..., 2] - cz
            d = np.minimum(d, np.sqrt(q0 * q0 + q1 * q1 + q2 * q2) - r)
        return d

    def ray_hit(self, C, D):
        """First positive hit parameter t of rays C + t*D (D: (n,3), C: (3,)); inf if none."""
        C = np.asarray(C, float)
        t = np.full(D.shape[0], np.inf)
        with np.errstate(divide="ignore", invalid="ignore"):
            if self.room_half is not None:
                h = self.room_half
                for a in range(3):
                    da = D[:, a]
                    ta = np.where(da > 0, (h - C[a]) / da, np.where(da < 0, (-h - C[a]) / da, np.inf))
                    t = np.minimum(t, np.where(ta > 0, ta, np.inf))
            if self.plane_z is not None:
                tz = (self.plane_z - C[2]) / D[:, 2]
                t = np.minimum(t, np.where(np.isfinite(tz) & (tz > 0), tz, np.inf))
            for (cx, cy, cz, r) in self.spheres:
                oc = C - np.array([cx, cy, cz])
                a = np.einsum("ij,ij->i", D, D)
                b = D @ oc
                c = oc @ oc - r * r
                disc = b * b - a * c
                sq = np.sqrt(np.maximum(disc, 0.0))
                t1 = (-b - sq) / a
                t2 = (-b + sq) / a
                ts = np.where(t1 > 0, t1, np.where(t2 > 0, t2, np.inf))
                t = np.minimum(t, np.where(disc >= 0, ts, np.inf))
        return t


def sphere_on_plane():
    """Config T scene: sphere r=0.4 at the centre of [0,1.28]^3 on its tangent ground plane."""
    return Scene(spheres=[(0.64, 0.64, 0.64, 0.4)], plane_z=0.24)


def box_room(seed=1, n_spheres=8):
    """Configs S/Q/W/L scene: 2.5 m box room centred at 0 with seeded spheres r in U[0.1,0.4]."""
    st = Stream(seed, 0)
    sph = []
    for _ in range(n_spheres):
        r = 0.1 + 0.3 * st.uniform(1)[0]
        c = st.symmetric(3) * (1.25 - r)
        sph.append((float(c[0]), float(c[1]), float(c[2]), float(r)))
    return Scene(spheres=sph, room_half=1.25)


# ----------------------------------------------------------------------------- rendering
@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    depth_unit_m: float = 0.001


def render_depth(scene, K: Intrinsics, T, noise_stream: Stream = None):
    """Closed-form ray cast through pixel centres (u, v) -> uint16 mm z-depth (H, W)."""
    v, u = np.mgrid[0:K.height, 0:K.width]
    dc = np.stack([(u.ravel() - K.cx) / K.fx, (v.ravel() - K.cy) / K.fy, np.ones(u.size)], axis=1)
    dw = dc @ T[:, :3].T
    z = scene.ray_hit(T[:, 3], dw)          # ray parameter == z-depth because dc.z == 1
    hit = np.isfinite(z)
    if noise_stream is not None:
        g = noise_stream.normal(z.size)
        z = np.where(hit, z + g * (0.0012 * z * z), z)
    raw = np.where(hit, np.clip(np.rint(z / K.depth_unit_m), 1, 65535), 0)
    return raw.astype(np.uint16).reshape(K.height, K.width)


def analytic_fill(scene, nx, ny, nz, voxel, origin, trunc, storage="f32"):
    """Test utility (not in the paper): V = clamp(sdf/tau, -1, 1)
    rounded to storage precision, W = 1, canonical x-fastest arrays of nx*ny*nz."""
    dt = np.float32 if storage == "f32" else np.float16
    V = np.empty((nz, ny, nx), dtype=dt)
    xs = origin[0] + voxel * (np.arange(nx) + 0.5)
    ys = origin[1] + voxel * (np.arange(ny) + 0.5)
    gy, gx = np.meshgrid(ys, xs, indexing="ij")
    for k in range(nz):
        zc = origin[2] + voxel * (k + 0.5)
        p = np.stack([gx, gy, np.full_like(gx, zc)], axis=-1)
        V[k] = np.clip(scene.sdf(p) / trunc, -1.0, 1.0).astype(dt)
    W = np.ones((nz, ny, nx), dtype=dt)
    return V.ravel(), W.ravel()
