"""Counter-based SplitMix64 streams shared by the oracle side and the CUDA side.

Input generation only: nothing here computes any part of the method.  Every
random number the generator draws comes from ``stream(seed, sid)``; the k-th
output is ``mix(state0 + (k+1)*GAMMA)`` (SplitMix64 is counter based), so a
stream can be sliced without replaying it.  Stream ids:
0 scene, 1 GT pose / trajectory, 2 init perturbation (2e6+t per frame),
3 particle template, 4 depth noise (4e6+t per frame).
"""
import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_u64(seed: int, sid: int, n: int, offset: int = 0) -> np.ndarray:
    """n raw 64-bit outputs of stream (seed, sid) starting at counter ``offset``."""
    with np.errstate(over="ignore"):
        s0 = _mix(np.array([(int(seed) * 0x100000001B3 + int(sid)) & ((1 << 64) - 1)], dtype=np.uint64))[0]
        k = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix(s0 + k * GAMMA)


class Stream:
    """Sequential reader over one SplitMix64 stream."""

    def __init__(self, seed: int, sid: int):
        self.seed, self.sid, self.pos = int(seed), int(sid), 0

    def u64(self, n: int) -> np.ndarray:
        out = stream_u64(self.seed, self.sid, n, self.pos)
        self.pos += n
        return out

    def uniform(self, n: int) -> np.ndarray:
        """fp64 uniforms in [0,1): (x >> 11) * 2^-53."""
        return (self.u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def symmetric(self, n: int) -> np.ndarray:
        """fp64 uniforms in [-1,1)."""
        return self.uniform(n) * 2.0 - 1.0

    def normal(self, n: int) -> np.ndarray:
        """fp64 standard normals by Box-Muller (one normal per uniform pair)."""
        u1 = self.uniform(n)
        u2 = self.uniform(n)
        return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
