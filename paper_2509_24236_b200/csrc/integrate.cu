// integrate.cu — KinectFusion TSDF fusion of one depth frame ("The fusion process
// remains the same as KinectFusion"; reading L22/L23 in DESIGN.md §3).
//
// Per voxel, in this exact fp64 operation order (no FMA contraction, IEEE division), so the
// stored bits equal a plain fp64 evaluation of the same formulas:
//   g_w = o + s*(i + 1/2);  p_c = R^T (g_w - t);  skip unless z_c > 0;
//   u = fx*x/z + cx, v = fy*y/z + cy;  pixel = (floor(u + 1/2), floor(v + 1/2)) inside and valid;
//   sdf = d - z_c;  skip unless sdf > -tau;  v_new = min(1, sdf/tau);
//   V' = (V W + v_new)/(W + 1), W' = min(W + 1, W_max), each rounded once (RNE) to storage.
//
// B200 design: the update set of a frame is the camera frustum up to the
// surface + tau, a few % of a room-scale grid.  A per-brick cull (conservative, fp32 with
// margins) compacts the 4^3 bricks that can contain an updated voxel; the fusion kernel then
// sweeps only those bricks, 64 consecutive elements (one brick = 2 x 128 B lines per array
// at fp32) per pair of warps, fully coalesced.  The full sweep is kept for verification.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "pft_internal.cuh"
#include "records.cuh"

namespace pft {

struct Intr {
  double fx, fy, cx, cy, unit;
  int W, H;
  bool c_small;  // |cx|, |cy| < 2^19: pixel_of's guarded fast path applies
};

template <typename T> __device__ __forceinline__ double to_double(T x);
template <> __device__ __forceinline__ double to_double<float>(float x) { return (double)x; }
template <> __device__ __forceinline__ double to_double<__half>(__half x) { return (double)__half2float(x); }
template <typename T> __device__ __forceinline__ T store_rn(double x);
template <> __device__ __forceinline__ float store_rn<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __half store_rn<__half>(double x) { return __double2half(x); }

template <typename T> __device__ __forceinline__ bool same_bits(T a, T b);
template <> __device__ __forceinline__ bool same_bits<float>(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }
template <> __device__ __forceinline__ bool same_bits<__half>(__half a, __half b) { return __half_as_ushort(a) == __half_as_ushort(b); }

// Exact int -> double without the conversion pipe (XU): 2^52 + i has i in its low mantissa bits.
__device__ __forceinline__ double i2d(int i) {  // 0 <= i < 2^31
  return __dsub_rn(__hiloint2double(0x43300000, i), 4503599627370496.0);
}
// floor(x) as an int for |x| < 2^30 (exact; no FRND): x + 1.5*2^52 rounded toward -inf holds
// floor(x) in its low word.
__device__ __forceinline__ int floor_lo(double x) { return __double2loint(__dadd_rd(x, 6755399441055744.0)); }

// Pixel index floor(u2) of u2 = RN(RN(RN(p / z) + c) + 1/2), the definition's expression (O9) (p = RN(f x)),
// given rz = RN(1/z) shared by both image axes.  Fast path: qa = RN(p rz) differs from RN(p/z) by
// at most 1.5 ulp, so for |qa| < 2^19 and |c| < 2^19 the approximate u2a is within 2^-30 of u2
// (two more roundings of values < 2^21, ulp 2^-32 each); whenever the fraction of u2a is at least
// 2^-26 away from an integer, floor(u2a) = floor(u2) -- the same decision.  Otherwise (a guard-band
// hit, ~1e-8 of the voxels, or a huge |qa|) the exact IEEE division decides.  Returns false when the
// pixel is outside [0, n) (also for |u2| >= 2^30 and NaN).
__device__ __forceinline__ bool pixel_of(double p, double z, double rz, double c, bool c_small, int n, int& pix) {
  const double qa = __dmul_rn(p, rz);
  if (c_small && fabs(qa) < 524288.0) {
    const double u2a = __dadd_rn(__dadd_rn(qa, c), 0.5);
    const double t = __dadd_rd(u2a, 6755399441055744.0);         // floor(u2a) in the low word
    const double fr = __dsub_rn(u2a, __dsub_rn(t, 6755399441055744.0));  // exact: |u2a| < 2^20
    if (fr >= 1.4901161193847656e-08 && fr <= 1.0 - 1.4901161193847656e-08) {
      pix = __double2loint(t);
      return (unsigned)pix < (unsigned)n;
    }
  }
  const double u2 = __dadd_rn(__dadd_rn(__ddiv_rn(p, z), c), 0.5);
  if (!(fabs(u2) < 1073741824.0)) return false;
  pix = floor_lo(u2);
  return (unsigned)pix < (unsigned)n;
}

// Per-frame axis tables (fusion step 1, computed by k_frame_prep).  The definition's camera coordinates (O9) are
//   x = RN(RN(RN(R00 d0) + RN(R10 d1)) + RN(R20 d2)),  d_a = RN(g_a - t_a),  g_a = RN(o_a + RN(s RN(i_a + 1/2)))
// (T = [R|t] row-major, so x pairs with T[0], T[4], T[8]; y with T[1], T[5], T[9]; z with T[2], T[6],
// T[10]).  Each product depends on one axis index only, so the 9 rounded products are tabulated once
// per frame per axis index, {RN(T[4a] d_a), RN(T[4a+1] d_a), RN(T[4a+2] d_a)} for axis a, and a voxel
// needs 3 table loads and 6 additions in the definition's order -- the same bits.
template <typename T> __device__ __forceinline__ T ldcs_t(const T* p);
template <> __device__ __forceinline__ float ldcs_t<float>(const float* p) { return __ldcs(p); }
template <> __device__ __forceinline__ __half ldcs_t<__half>(const __half* p) {
  return __ushort_as_half(__ldcs(reinterpret_cast<const unsigned short*>(p)));
}

__device__ __forceinline__ double4 ld_axis(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// Vs, Ws: the voxel's stored value and weight, loaded by the caller ahead of the dependent chain
// (their addresses depend on nothing computed here).  Returns true iff the stored value V changed
// (its cell records must then be refreshed).  Stored bits equal those of the plain fp64 definition (O9): every value that reaches storage (z, sdf, v_new, V', W') is
// computed with the exact operations of the definition (O9) (x, y, z from the axis tables in its order); the
// projection only decides a pixel (pixel_of's guarded reciprocal), and two divisions are skipped
// where their correctly rounded result is known exactly: v_new = 1 when sdf >= tau (then
// sdf/tau >= 1, rounded >= 1, clamped to 1), and V' = 1 when V = 1 and v_new = 1 (numerator
// RN(1*W + 1) and denominator RN(W + 1) are the same finite a >= 1, and a/a = 1) -- the free space
// in front of the surface, most updated voxels.
template <typename T>
__device__ __forceinline__ bool fuse_voxel(const Geom& g, const Intr& K, const uint16_t* __restrict__ depth,
                                           const double4& A, const double4& B, const double4& C, T Vs, T Ws,
                                           T* __restrict__ V, T* __restrict__ W, uint32_t o, bool& updated) {
  updated = false;
  const double z = __dadd_rn(__dadd_rn(A.z, B.z), C.z);
  if (!(z > 0.0)) return false;
  const double x = __dadd_rn(__dadd_rn(A.x, B.x), C.x);
  const double y = __dadd_rn(__dadd_rn(A.y, B.y), C.y);
  const double rz = __drcp_rn(z);
  int ui, vi;
  if (!pixel_of(__dmul_rn(K.fx, x), z, rz, K.cx, K.c_small, K.W, ui)) return false;
  if (!pixel_of(__dmul_rn(K.fy, y), z, rz, K.cy, K.c_small, K.H, vi)) return false;
#ifdef PFT_DEBUG
  if ((unsigned)ui >= (unsigned)K.W || (unsigned)vi >= (unsigned)K.H) {
    printf("pft debug: pixel (%d, %d) outside %dx%d\n", ui, vi, K.W, K.H);
    __trap();
  }
#endif
  const uint16_t raw = __ldg(depth + (size_t)vi * K.W + (size_t)ui);
  const double d = __dmul_rn(i2d((int)raw), K.unit);
  if (raw == 0 || !(d < g.max_depth)) return false;
  const double sdf = __dsub_rn(d, z);
  if (!(sdf > -g.trunc)) return false;
  double vnew = 1.0;
  if (!(sdf >= g.trunc)) {
    vnew = __ddiv_rn(sdf, g.trunc);
    if (vnew > 1.0) vnew = 1.0;
  }
  const double Vo = to_double<T>(Vs), Wo = to_double<T>(Ws);
  const double Wp = __dadd_rn(Wo, 1.0);
  const double Vn = (vnew == 1.0 && Vo == 1.0 && Wo >= 0.0 && Wo <= 1e300)
                        ? 1.0
                        : __ddiv_rn(__dadd_rn(__dmul_rn(Vo, Wo), vnew), Wp);
  const double Wn = Wp > g.max_weight ? g.max_weight : Wp;
  const T Vnew = store_rn<T>(Vn);
  V[o] = Vnew;
  W[o] = store_rn<T>(Wn);
  updated = true;
  return !same_bits<T>(Vs, Vnew);
}

// Full sweep: one thread per brick element (the verification path).
template <typename T>
__global__ __launch_bounds__(256) void k_integrate_sweep(Geom g, Intr K, const uint16_t* __restrict__ depth,
                                                         const double4* __restrict__ tab, T* __restrict__ V,
                                                         T* __restrict__ W, size_t nelem) {
  const int n0 = 4 * g.nbx, n1 = 4 * g.nby;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nelem; e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(e >> 6), w = (uint32_t)(e & 63);
    const int bx = (int)(b % (uint32_t)g.nbx);
    const uint32_t r = b / (uint32_t)g.nbx;
    const int by = (int)(r % (uint32_t)g.nby), bz = (int)(r / (uint32_t)g.nby);
    const int i = bx * 4 + (int)(w & 3), j = by * 4 + (int)((w >> 2) & 3), k = bz * 4 + (int)(w >> 4);
    if (i >= g.nx || j >= g.ny || k >= g.nz) continue;
    bool updated;
    fuse_voxel<T>(g, K, depth, ld_axis(tab + i), ld_axis(tab + n0 + j), ld_axis(tab + n0 + n1 + k), V[e], W[e], V, W,
                  (uint32_t)e, updated);
  }
}

// ---- culling ---------------------------------------------------------------------------------
// Depth pyramid: level l holds, per tile of (8 << l) x (8 << l) pixels, {max valid raw depth,
// ~min over the tile's pixels of (valid ? raw : 0)} (validity is the exact fp64 test of O1,
// raw > 0 and raw * unit < max_depth; the minimum is stored complemented so that both halves are
// maxima with identity 0).  A box's footprint is bounded by at most 4 x 4 tiles of the finest
// level whose tiles it spans at most 4 of per axis: 16 independent loads in one round trip.  Four
// levels (8..64 px tiles): a footprint wider than 4 x 64 px is kept without a test.
constexpr int kTile = 8;
constexpr int kLevels = 4;
struct Pyr {
  int W, H;   // image size; level l has nx(l) x ny(l) tiles starting at element off(l)
  int total;  // elements (uint2) of all levels
  __host__ __device__ __forceinline__ int nx(int l) const { return (W + (kTile << l) - 1) >> (3 + l); }
  __host__ __device__ __forceinline__ int ny(int l) const { return (H + (kTile << l) - 1) >> (3 + l); }
  __host__ __device__ __forceinline__ int off(int l) const {
    int o = 0;
    for (int q = 0; q < l; ++q) o += nx(q) * ny(q);
    return o;
  }
};

static Pyr make_pyr(int W, int H) {
  Pyr p{W, H, 0};
  p.total = p.off(kLevels);
  return p;
}

__device__ __forceinline__ uint2 tmax(uint2 a, uint2 b) { return make_uint2(max(a.x, b.x), max(a.y, b.y)); }

// Axis tables (fuse_voxel): entry e of the three axes' 4*(nbx+nby+nbz) entries.
__device__ __forceinline__ void axis_entry(const Geom& g, const double* __restrict__ Tdev, double4* __restrict__ tab,
                                           int e) {
  const int n0 = 4 * g.nbx, n1 = 4 * g.nby, n2 = 4 * g.nbz;
  if (e >= n0 + n1 + n2) return;
  const int a = e < n0 ? 0 : (e < n0 + n1 ? 1 : 2);
  const int i = e - (a == 0 ? 0 : (a == 1 ? n0 : n0 + n1));
  const double o = a == 0 ? g.ox : (a == 1 ? g.oy : g.oz);
  const double gw = __dadd_rn(o, __dmul_rn(g.voxel, __dadd_rn((double)i, 0.5)));
  const double d = __dsub_rn(gw, Tdev[3 + 4 * a]);
  tab[e] = make_double4(__dmul_rn(Tdev[4 * a], d), __dmul_rn(Tdev[4 * a + 1], d), __dmul_rn(Tdev[4 * a + 2], d), 0.0);
}

// Frame preparation of one 64 x 64-pixel region (a level-3 tile; the whole CTA): its 64 level-0 tiles
// by warps, levels 1-3 from shared memory.
__device__ __forceinline__ void prep_region(const Intr& K, double max_depth, const uint16_t* __restrict__ depth,
                                            uint2* __restrict__ tiles, const Pyr& P, int v, uint2* s0, uint2* s1,
                                            uint2* s2) {
  const int nx3 = P.nx(3);
  const int rx = v % nx3, ry = v / nx3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nx0 = P.nx(0), ny0 = P.ny(0);
  int raw[16];  // all 16 pixel loads of this lane in flight together; -1: outside the image
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int ti = warp * 8 + (q >> 1), p = lane + 32 * (q & 1);
    const int u = (rx * 8 + (ti & 7)) * kTile + (p & 7), vv = (ry * 8 + (ti >> 3)) * kTile + (p >> 3);
    raw[q] = (u < K.W && vv < K.H) ? (int)__ldg(depth + (size_t)vv * K.W + u) : -1;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int ti = warp * 8 + q;
    const int tx = rx * 8 + (ti & 7), ty = ry * 8 + (ti >> 3);
    uint2 m = make_uint2(0u, 0u);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = raw[2 * q + h];
      if (r >= 0) {
        const bool valid = r != 0 && __dmul_rn((double)r, K.unit) < max_depth;
        m = tmax(m, make_uint2(valid ? (uint32_t)r : 0u, ~(valid ? (uint32_t)r : 0u)));
      }
    }
    for (int sft = 16; sft > 0; sft >>= 1)
      m = tmax(m, make_uint2(__shfl_xor_sync(0xffffffffu, m.x, sft), __shfl_xor_sync(0xffffffffu, m.y, sft)));
    if (lane == 0) {
      s0[ti] = m;
      if (tx < nx0 && ty < ny0) tiles[ty * nx0 + tx] = m;
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < 16) {
    const int a = t & 3, b = t >> 2;
    const uint2 m = tmax(tmax(s0[16 * b + 2 * a], s0[16 * b + 2 * a + 1]), tmax(s0[16 * b + 8 + 2 * a], s0[16 * b + 9 + 2 * a]));
    s1[t] = m;
    const int X = rx * 4 + a, Y = ry * 4 + b;
    if (X < P.nx(1) && Y < P.ny(1)) tiles[P.off(1) + Y * P.nx(1) + X] = m;
  }
  __syncthreads();
  if (t < 4) {
    const int a = t & 1, b = t >> 1;
    const uint2 m = tmax(tmax(s1[8 * b + 2 * a], s1[8 * b + 2 * a + 1]), tmax(s1[8 * b + 4 + 2 * a], s1[8 * b + 5 + 2 * a]));
    s2[t] = m;
    const int X = rx * 2 + a, Y = ry * 2 + b;
    if (X < P.nx(2) && Y < P.ny(2)) tiles[P.off(2) + Y * P.nx(2) + X] = m;
  }
  __syncthreads();
  if (t == 0) tiles[P.off(3) + ry * nx3 + rx] = tmax(tmax(s2[0], s2[1]), tmax(s2[2], s2[3]));
  __syncthreads();  // (s0..s2 are reused by the next region of this CTA)
}

// Frame preparation, one launch: CTAs [0, nreg) build the pyramid (one region each), the remaining
// CTAs compute the axis tables (the full sweep: tables only, nreg = 0).
__global__ __launch_bounds__(256) void k_frame_prep(Intr K, double max_depth, const uint16_t* __restrict__ depth,
                                                    uint2* __restrict__ tiles, Pyr P, int nreg, Geom g,
                                                    const double* __restrict__ Tdev, double4* __restrict__ tab,
                                                    uint32_t* __restrict__ zero, int nzero) {
  __shared__ uint2 s0[64], s1[16], s2[4];
  pdl_wait();  // the pose (tracker output) and the previous frame's counters
  pdl_trigger();
  if (blockIdx.x == 0 && (int)threadIdx.x < nzero) zero[threadIdx.x] = 0u;  // the frame's counters
  if ((int)blockIdx.x >= nreg) {
    axis_entry(g, Tdev, tab, ((int)blockIdx.x - nreg) * 256 + threadIdx.x);
    return;
  }
  prep_region(K, max_depth, depth, tiles, P, blockIdx.x, s0, s1, s2);
}

// Conservative classification of a box of voxel centres given by its centre (world, fp64) and
// bounding-sphere radius, in fp32 with margins (1 mm, 2 px) far above fp32 rounding at room scale:
//   CULL  no voxel centre inside can pass the voxel-level tests (all z_c <= 0, the projection misses
//         the image, or every pixel it can project to is invalid or has d + tau <= z_c);
//   FREE  every voxel centre inside projects into the image onto a valid pixel with d - z_c >= tau:
//         each is updated with v_new = 1, whatever its exact pixel (the "free space" class);
//   KEEP  otherwise (incl. boxes straddling the camera plane or wider than 4 coarsest tiles).
enum { kCull = 0, kKeep = 1, kFree = 2 };

__device__ __forceinline__ int box_class(const Geom& g, const Intr& K, const double* __restrict__ Tdev,
                                         const uint2* __restrict__ tiles, const Pyr& P, double cxw, double cyw,
                                         double czw, float rad, int lane16) {
  const float cwx = (float)(cxw - Tdev[3]), cwy = (float)(cyw - Tdev[7]), cwz = (float)(czw - Tdev[11]);
  const float x = (float)Tdev[0] * cwx + (float)Tdev[4] * cwy + (float)Tdev[8] * cwz;
  const float y = (float)Tdev[1] * cwx + (float)Tdev[5] * cwy + (float)Tdev[9] * cwz;
  const float z = (float)Tdev[2] * cwx + (float)Tdev[6] * cwy + (float)Tdev[10] * cwz;
  if (!(z + rad > 0.f)) return kCull;
  const float fx = (float)K.fx, fy = (float)K.fy, cx = (float)K.cx, cy = (float)K.cy;
  if (z - rad <= 1e-3f) {
    // straddles the camera plane: no projection bound, but the frustum there is a thin cone from
    // the camera centre.  A voxel (xv, yv, zv), zv > 0, lands on a pixel only if |xv| <= zv * ax
    // (ax = the larger half-width of the image in pixels / fx, +1/2 pixel for the rounding) and
    // |yv| <= zv * ay; every voxel here has zv <= z + rad and |xv| >= |x| - rad, so a box laterally
    // beyond the cone at its far depth cannot be updated (1% + 1 mm of slack for the fp32 transform)
    const float zf = z + rad;
    const float ax = fmaxf(cx + 0.5f, (float)K.W - 0.5f - cx) / fx, ay = fmaxf(cy + 0.5f, (float)K.H - 0.5f - cy) / fy;
    if (fabsf(x) - rad > 1.01f * zf * ax + 1e-3f || fabsf(y) - rad > 1.01f * zf * ay + 1e-3f) return kCull;
    return kKeep;
  }
  const float zn = z - rad, zf = z + rad;
  const float izn = __frcp_rn(zn), izf = __frcp_rn(zf);  // (a few ulp: far inside the 2 px margin)
  const float u0 = fx * fminf((x - rad) * izn, (x - rad) * izf) + cx - 2.f;
  const float u1 = fx * fmaxf((x + rad) * izn, (x + rad) * izf) + cx + 2.f;
  const float v0 = fy * fminf((y - rad) * izn, (y - rad) * izf) + cy - 2.f;
  const float v1 = fy * fmaxf((y + rad) * izn, (y + rad) * izf) + cy + 2.f;
  if (!(u1 >= -0.5f && v1 >= -0.5f && u0 < (float)K.W && v0 < (float)K.H)) return kCull;
  const bool inside = u0 >= 0.f && v0 >= 0.f && u1 < (float)K.W - 1.f && v1 < (float)K.H - 1.f;
  const int pu0 = max(0, (int)floorf(u0 + 0.5f)), pu1 = min(K.W - 1, (int)floorf(u1 + 0.5f));
  const int pv0 = max(0, (int)floorf(v0 + 0.5f)), pv1 = min(K.H - 1, (int)floorf(v1 + 0.5f));
  int l = 0;
  while (l < kLevels && ((pu1 >> (3 + l)) - (pu0 >> (3 + l)) > 3 || (pv1 >> (3 + l)) - (pv0 >> (3 + l)) > 3)) ++l;
  if (l == kLevels) return kKeep;
  const int s = 3 + l;
  const uint2* lvl = tiles + P.off(l);
  const int stride = P.nx(l), t0x = pu0 >> s, t1x = pu1 >> s, t0y = pv0 >> s, t1y = pv1 >> s;
  uint2 m = make_uint2(0u, 0u);
  if (lane16 < 0) {  // this thread alone: all 16 tiles (clamped into the footprint: repeats are harmless)
    uint2 tv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) tv[q] = __ldg(lvl + min(t0y + (q >> 2), t1y) * stride + min(t0x + (q & 3), t1x));
#pragma unroll
    for (int q = 0; q < 16; ++q) m = tmax(m, tv[q]);
  } else {  // the warp (uniform box): lane q < 16 loads tile q
    if (lane16 < 16) m = __ldg(lvl + min(t0y + (lane16 >> 2), t1y) * stride + min(t0x + (lane16 & 3), t1x));
    for (int sft = 16; sft > 0; sft >>= 1)
      m = tmax(m, make_uint2(__shfl_xor_sync(0xffffffffu, m.x, sft), __shfl_xor_sync(0xffffffffu, m.y, sft)));
  }
  if (m.x == 0) return kCull;  // no valid pixel
  if (!(zn - 1e-3f < (float)((double)m.x * K.unit) + (float)g.trunc)) return kCull;
  const uint32_t mn = ~m.y;      // min raw over the tiles, 0 if any pixel is invalid
  if (inside && mn != 0 && (float)((double)mn * K.unit) - (zf + 1e-3f) >= (float)g.trunc) return kFree;
  return kKeep;
}

// Kept-brick list entries carry the brick coordinates packed 10:10:10 bits (grids up to 4096
// voxels per axis, checked at volume creation) and the FREE class in bit 31, so the sweep decodes
// them with shifts instead of two runtime integer divisions per thread.
constexpr uint32_t kFreeBit = 1u << 31;
__device__ __forceinline__ uint32_t pack_brick(int bx, int by, int bz) {
  return ((uint32_t)bz << 20) | ((uint32_t)by << 10) | (uint32_t)bx;
}

__device__ __forceinline__ void append_warp(bool keep, uint32_t v, uint32_t* __restrict__ list,
                                            uint32_t* __restrict__ count) {
  const unsigned ball = __ballot_sync(0xffffffffu, keep);
  if (ball) {
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(count, (uint32_t)__popc(ball));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) list[base + __popc(ball & ((1u << lane) - 1))] = v;
  }
}

constexpr int kSuper = 4;  // super-brick = 4^3 bricks = 16^3 voxels

// Level 1: one thread per super-brick (its 16 tile loads issued together); survivors appended
// warp-aggregated.  Whole warps iterate together (warp w of nwarps takes super-bricks 32 w + lane, ...).
__device__ __forceinline__ void cull_super_pass(const Geom& g, const Intr& K, const double* __restrict__ Tdev,
                                                const uint2* __restrict__ tiles, const Pyr& P, int nsx, int nsy, int nsz,
                                                uint32_t* __restrict__ slist, uint32_t* __restrict__ scount,
                                                uint32_t warp, uint32_t nwarps) {
  const uint32_t ns = (uint32_t)nsx * nsy * nsz;
  const int lane = threadIdx.x & 31;
  for (uint32_t b0 = warp * 32; b0 < ns; b0 += nwarps * 32) {
    const uint32_t sb = b0 + lane;
    int c = kCull;
    if (sb < ns) {
      const int sx = (int)(sb % (uint32_t)nsx);
      const uint32_t r = sb / (uint32_t)nsx;
      const int sy = (int)(r % (uint32_t)nsy), sz = (int)(r / (uint32_t)nsy);
      // voxel-centre box of the super-brick: voxels [16 s, 16 s + 15] per axis
      c = box_class(g, K, Tdev, tiles, P, g.ox + g.voxel * (16.0 * sx + 8.0), g.oy + g.voxel * (16.0 * sy + 8.0),
                    g.oz + g.voxel * (16.0 * sz + 8.0), (float)(7.5 * 1.7320508 * g.voxel) + 1e-3f, -1);
    }
    append_warp(c != kCull, sb, slist, scount);
  }
}

// Level 2: one warp per surviving super-brick, two of its 64 bricks per lane.
__device__ __forceinline__ void cull_bricks_pass(const Geom& g, const Intr& K, const double* __restrict__ Tdev,
                                                 const uint2* __restrict__ tiles, const Pyr& P, int nsx, int nsy,
                                                 const uint32_t* __restrict__ slist, uint32_t n,
                                                 uint32_t* __restrict__ list, uint32_t* __restrict__ count,
                                                 uint32_t* __restrict__ nfree_out, uint32_t warp, uint32_t nwarps) {
  const int lane = threadIdx.x & 31;
  for (uint32_t li = warp; li < n; li += nwarps) {
    const uint32_t sb = slist[li];
    const int sx = (int)(sb % (uint32_t)nsx);
    const uint32_t r = sb / (uint32_t)nsx;
    const int sy = (int)(r % (uint32_t)nsy), sz = (int)(r / (uint32_t)nsy);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = lane + 32 * h;
      const int bx = sx * kSuper + (t & 3), by = sy * kSuper + ((t >> 2) & 3), bz = sz * kSuper + (t >> 4);
      int c = kCull;
      if (bx < g.nbx && by < g.nby && bz < g.nbz)
        c = box_class(g, K, Tdev, tiles, P, g.ox + g.voxel * (4.0 * bx + 2.0), g.oy + g.voxel * (4.0 * by + 2.0),
                      g.oz + g.voxel * (4.0 * bz + 2.0), (float)(1.5 * 1.7320508 * g.voxel) + 1e-3f, -1);
      append_warp(c != kCull, pack_brick(bx, by, bz) | (c == kFree ? kFreeBit : 0u), list, count);
      const unsigned nfree = __popc(__ballot_sync(0xffffffffu, c == kFree));
      if (lane == 0 && nfree) atomicAdd(nfree_out, nfree);
    }
  }
}

__global__ __launch_bounds__(256) void k_cull_super(Geom g, Intr K, const double* __restrict__ Tdev,
                                                    const uint2* __restrict__ tiles, Pyr P, int nsx, int nsy, int nsz,
                                                    uint32_t* __restrict__ slist, uint32_t* __restrict__ scount) {
  pdl_wait();
  pdl_trigger();
  cull_super_pass(g, K, Tdev, tiles, P, nsx, nsy, nsz, slist, scount, (blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                  (gridDim.x * blockDim.x) >> 5);
}

__global__ __launch_bounds__(256) void k_cull_bricks(Geom g, Intr K, const double* __restrict__ Tdev,
                                                     const uint2* __restrict__ tiles, Pyr P, int nsx, int nsy,
                                                     const uint32_t* __restrict__ slist,
                                                     const uint32_t* __restrict__ scount, uint32_t* __restrict__ list,
                                                     uint32_t* __restrict__ count, uint32_t* __restrict__ nfree_out) {
  pdl_wait();
  pdl_trigger();
  cull_bricks_pass(g, K, Tdev, tiles, P, nsx, nsy, slist, *scount, list, count, nfree_out,
                   (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
}

// A FREE-class voxel (box_class): v_new = 1, so V' = (V W + 1)/(W + 1) (= 1 exactly when V = 1, see
// fuse_voxel) and W' = min(W + 1, W_max), each rounded once -- the definition's update without its
// projection, whose every possible outcome was proven to be "updated with v_new = 1".
template <typename T>
__device__ __forceinline__ bool fuse_free(const Geom& g, T Vs, T Ws, T* __restrict__ V, T* __restrict__ W, uint32_t o) {
  const double Vo = to_double<T>(Vs), Wo = to_double<T>(Ws);
  const double Wp = __dadd_rn(Wo, 1.0);
  const double Wn = Wp > g.max_weight ? g.max_weight : Wp;
  W[o] = store_rn<T>(Wn);
  if (Vo == 1.0 && Wo >= 0.0 && Wo <= 1e300) return false;  // V' = 1: bits unchanged, not stored
  const T Vnew = store_rn<T>(__ddiv_rn(__dadd_rn(__dmul_rn(Vo, Wo), 1.0), Wp));
  V[o] = Vnew;
  return !same_bits<T>(Vs, Vnew);
}

// Sweep of the compacted bricks: a warp covers half a brick (one voxel per lane), 4 bricks per
// 256-thread CTA and iteration, CTA-stride over the list (CTAs block, block + nblocks, ...).  The
// next brick's list entry is loaded one iteration ahead and the voxel's stored value/weight before
// the projection chain (their addresses depend only on the list).  *sUpd (shared, zeroed by the
// caller) collects the CTA's updated voxels.
template <typename T>
__device__ __forceinline__ void fuse_pass(const Geom& g, const Intr& K, const uint16_t* __restrict__ depth,
                                          const double4* __restrict__ tab, const uint32_t* __restrict__ list, uint32_t n,
                                          T* __restrict__ V, T* __restrict__ W, uint32_t* __restrict__ dirty,
                                          uint32_t* __restrict__ dlist, uint32_t* __restrict__ dcount, unsigned* sUpd,
                                          uint32_t block, uint32_t nblocks) {
  unsigned upd = 0u;  // voxels this thread updated (work counter, pft_integrate_stats)
  const int n0 = 4 * g.nbx, n1 = 4 * g.nby;
  const uint32_t w = threadIdx.x & 63;
  const uint32_t step = nblocks * 4;
  uint32_t li = block * 4 + (threadIdx.x >> 6);
  uint32_t e = li < n ? __ldg(list + li) : 0u;
  for (; li < n; li += step) {
    const int bx = (int)(e & 1023u), by = (int)((e >> 10) & 1023u), bz = (int)((e >> 20) & 1023u);
    const bool free_class = (e & kFreeBit) != 0u;  // brick-uniform
    if (li + step < n) e = __ldg(list + li + step);  // the next brick's entry, in flight during this one
    const uint32_t b = ((uint32_t)bz * g.nby + (uint32_t)by) * g.nbx + (uint32_t)bx;
    const int i = bx * 4 + (int)(w & 3), j = by * 4 + (int)((w >> 2) & 3), k = bz * 4 + (int)(w >> 4);
    bool changed = false;
    if (i < g.nx && j < g.ny && k < g.nz) {
      const uint32_t o = b * 64u + w;
#ifdef PFT_DEBUG
      if (b >= (uint32_t)g.nbx * g.nby * g.nbz || i >= 4 * g.nbx || j >= 4 * g.nby || k >= 4 * g.nbz) {
        printf("pft debug: bad brick entry %08x (b=%u i=%d j=%d k=%d)\n", e, b, i, j, k);
        __trap();
      }
#endif
      // issued first (independent of the projection chain), streamed past L1 (ld.global.cs) so the
      // axis tables and depth stay L1-resident: Q 37.9 -> 34.3 us, L 165 -> 143 us per frame
      const T Vs = ldcs_t(V + o), Ws = ldcs_t(W + o);
      bool updated = true;
      changed = free_class ? fuse_free<T>(g, Vs, Ws, V, W, o)
                           : fuse_voxel<T>(g, K, depth, ld_axis(tab + i), ld_axis(tab + n0 + j),
                                           ld_axis(tab + n0 + n1 + k), Vs, Ws, V, W, o, updated);
      upd += updated ? 1u : 0u;
    }
    // cell-bricks whose records read this voxel: (b - d) for d in {0,1}^3, the -1 neighbours
    // only from the brick's low faces
    unsigned nbm = 0u;
    if (changed) {
      const unsigned ex = (w & 3) == 0, ey = ((w >> 2) & 3) == 0, ez = (w >> 4) == 0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if ((!(q & 1) || ex) && (!(q & 2) || ey) && (!(q & 4) || ez)) nbm |= 1u << q;
    }
    nbm = __reduce_or_sync(0xffffffffu, nbm);
    if (nbm) mark_dirty_cells_warp(g, bx, by, bz, nbm, dirty, dlist, dcount);  // warp-uniform
  }
  upd = __reduce_add_sync(0xffffffffu, upd);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(sUpd, upd);
}

template <typename T>
#ifndef PFT_INTEG_MINB
#define PFT_INTEG_MINB 5  // 48 registers, 40 warps/SM (6: 40 registers with spills, 36.1 vs 34.3 us at Q)
#endif
__global__ __launch_bounds__(256, PFT_INTEG_MINB) void k_integrate_list(Geom g, Intr K, const uint16_t* __restrict__ depth,
                                                        const double4* __restrict__ tab, const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ count, T* __restrict__ V,
                                                        T* __restrict__ W, uint32_t* __restrict__ dirty,
                                                        uint32_t* __restrict__ dlist, uint32_t* __restrict__ dcount,
                                                        unsigned long long* __restrict__ nupd) {
  __shared__ unsigned sUpd;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) sUpd = 0u;
  __syncthreads();
  fuse_pass<T>(g, K, depth, tab, list, *count, V, W, dirty, dlist, dcount, &sUpd, blockIdx.x, gridDim.x);
  __syncthreads();
  if (threadIdx.x == 0 && sUpd) atomicAdd(nupd, (unsigned long long)sUpd);
}

// ---- the whole culled integration in ONE cooperative launch (co-resident CTAs): frame preparation
// | cull level 1 | cull level 2 | fusion | record refresh, separated by a grid barrier (a monotone
// arrival counter in the volume scratch, zeroed with the frame's counters) instead of 4 kernel
// boundaries.  Same device functions as the separate kernels (the fallback), so the same bits.
struct FusedArgs {
  Geom g;
  Intr K;
  Pyr P;
  const uint16_t* depth;
  const double* T;
  uint2* tiles;
  double4* tab;
  int nreg, ntab, nsx, nsy, nsz;
  uint32_t *slist, *scount, *list, *count, *dirty, *dlist, *dcount, *nfree;
  unsigned long long *nupd, *bar;
  void *V, *W, *R;
  uint32_t* mask;
};

__device__ __forceinline__ void coop_barrier(unsigned long long* ctr, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

template <typename T>
__global__ __launch_bounds__(256, 5) void k_integrate_fused(FusedArgs a) {
  __shared__ uint2 s0[64], s1[16], s2[4];
  __shared__ unsigned sUpd;
  unsigned long long target = 0ull;
  if (threadIdx.x == 0) sUpd = 0u;
  // frame preparation: pyramid regions and axis-table blocks over the CTAs
  for (int v = blockIdx.x; v < a.nreg + a.ntab; v += gridDim.x) {
    if (v < a.nreg) prep_region(a.K, a.g.max_depth, a.depth, a.tiles, a.P, v, s0, s1, s2);
    else axis_entry(a.g, a.T, a.tab, (v - a.nreg) * 256 + threadIdx.x);
  }
  coop_barrier(a.bar, target);
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  cull_super_pass(a.g, a.K, a.T, a.tiles, a.P, a.nsx, a.nsy, a.nsz, a.slist, a.scount, warp, nwarps);
  coop_barrier(a.bar, target);
  cull_bricks_pass(a.g, a.K, a.T, a.tiles, a.P, a.nsx, a.nsy, a.slist, __ldcg(a.scount), a.list, a.count, a.nfree,
                   warp, nwarps);
  coop_barrier(a.bar, target);
  fuse_pass<T>(a.g, a.K, a.depth, a.tab, a.list, __ldcg(a.count), (T*)a.V, (T*)a.W, a.dirty, a.dlist, a.dcount, &sUpd,
               blockIdx.x, gridDim.x);
  __syncthreads();
  if (threadIdx.x == 0 && sUpd) atomicAdd(a.nupd, (unsigned long long)sUpd);
  coop_barrier(a.bar, target);
  records_dirty_pass<T>(a.g, (const T*)a.V, (T*)a.R, a.mask, a.dirty, a.dlist, __ldcg(a.dcount), blockIdx.x, gridDim.x);
}

__global__ void k_mark_sweep(uint32_t* flag) { *flag = 1u; }

// Co-resident CTAs of `kern` at `threads` per CTA on the current device (cached per kernel and device).
template <typename K>
static int resident_grid(K kern, int threads) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<const void*, int> key((const void*)kern, dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& c : cache)
    if (c.first == key) return c.second;
  int per_sm = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0);
  const int v = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
  cache.push_back({key, v});
  return v;
}

// The single cooperative launch is measured slower than the 5 graph-replayed kernels (Q: 69 vs 66 us
// of kernel time, 1.634 vs 1.626 ms per bench frame; L: 240 vs 200 us -- 740 CTAs through 4 grid
// barriers cost more than the kernel boundaries they replace), so it is opt-in: PFT_INTEGRATE_FUSED=1.
static bool use_fused_integrate() {
  static const bool on = [] {
    const char* e = getenv("PFT_INTEGRATE_FUSED");
    return e && e[0] == '1';
  }();
  return on;
}

pft_status integrate_impl(pft_volume* vol, const uint16_t* depth, const pft_intrinsics* Kp, const double* T,
                          int full_sweep, cudaStream_t st) {
  Intr K{Kp->fx, Kp->fy, Kp->cx, Kp->cy, Kp->depth_unit_m, Kp->width, Kp->height,
         fabs(Kp->cx) < 524288.0 && fabs(Kp->cy) < 524288.0};
  const Geom& g = vol->g;
  const Pyr P = make_pyr(K.W, K.H);
  if ((size_t)P.total * sizeof(uint2) > vol->L.tiles_bytes) full_sweep = 1;
  double4* tab = (double4*)(vol->base + vol->L.axis_off);
  if (full_sweep) {
    const int ntab = (4 * (g.nbx + g.nby + g.nbz) + 255) / 256;
    PFT_LAUNCH(PFT_PROF_CULL, st, k_frame_prep<<<ntab, 256, 0, st>>>(K, g.max_depth, depth, nullptr, P, 0, g, T, tab, nullptr, 0));
    size_t n = vol->L.elems;
    size_t blocks = (n + 255) / 256;
    int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
    if (vol->esize == 4)
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_sweep<float><<<grid, 256, 0, st>>>(g, K, depth, tab, (float*)(vol->base + vol->L.v_off),
                                                     (float*)(vol->base + vol->L.w_off), n));
    else
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_sweep<__half><<<grid, 256, 0, st>>>(g, K, depth, tab, (__half*)(vol->base + vol->L.v_off),
                                                      (__half*)(vol->base + vol->L.w_off), n));
    records_rebuild_all(vol, st);
    // pft_integrate_stats: the full sweep does not maintain the counters (scratch +268 = 1)
    k_mark_sweep<<<1, 1, 0, st>>>((uint32_t*)(vol->base + vol->L.scratch_off + 268));
    return cuda_check("integrate (full sweep)");
  }
  uint2* tiles = (uint2*)(vol->base + vol->L.tiles_off);
  uint32_t* list = (uint32_t*)(vol->base + vol->L.list_off);
  uint32_t* count = (uint32_t*)(vol->base + vol->L.scratch_off + 64);
  uint32_t* dcount = (uint32_t*)(vol->base + vol->L.scratch_off + 128);
  uint32_t* dirty = (uint32_t*)(vol->base + vol->L.dirty_off);
  uint32_t* dlist = (uint32_t*)(vol->base + vol->L.dlist_off);
  unsigned long long* nupd = (unsigned long long*)(vol->base + vol->L.scratch_off + 256);
  uint32_t* nfree = (uint32_t*)(vol->base + vol->L.scratch_off + 264);
  unsigned long long* bar = (unsigned long long*)(vol->base + vol->L.scratch_off + 320);
  // kept, dirty, super-brick counts, updated voxels, free bricks, sweep flag, barrier (+64..+327):
  // zeroed by k_frame_prep (the fused path: here)
  uint32_t* zero = count;
  const int nzero = 264 / 4;
  if (use_fused_integrate()) cudaMemsetAsync(count, 0, 264, st);
  const int nreg = P.nx(3) * P.ny(3);
  const int ntab = (4 * (g.nbx + g.nby + g.nbz) + 255) / 256;
  const int nsx = (g.nbx + kSuper - 1) / kSuper, nsy = (g.nby + kSuper - 1) / kSuper, nsz = (g.nbz + kSuper - 1) / kSuper;
  const uint32_t ns = (uint32_t)nsx * nsy * nsz;
  uint32_t* slist = (uint32_t*)(vol->base + vol->L.slist_off);
  uint32_t* scount = (uint32_t*)(vol->base + vol->L.scratch_off + 192);
  if (use_fused_integrate()) {
    FusedArgs fa{g, K, P, depth, T, tiles, tab, nreg, ntab, nsx, nsy, nsz, slist, scount, list, count, dirty, dlist,
                 dcount, nfree, nupd, bar, vol->base + vol->L.v_off, vol->base + vol->L.w_off, vol->base + vol->L.r_off,
                 (uint32_t*)(vol->base + vol->L.m_off)};
    void* args[] = {&fa};
    cudaError_t e = cudaSuccess;
    if (vol->esize == 4) {
      const int grid = resident_grid(k_integrate_fused<float>, 256);
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st,
                 e = cudaLaunchCooperativeKernel((const void*)k_integrate_fused<float>, dim3(grid), dim3(256), args, 0, st));
    } else {
      const int grid = resident_grid(k_integrate_fused<__half>, 256);
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st,
                 e = cudaLaunchCooperativeKernel((const void*)k_integrate_fused<__half>, dim3(grid), dim3(256), args, 0, st));
    }
    if (e == cudaSuccess) return cuda_check("integrate (fused)");
    if (e != cudaErrorCooperativeLaunchTooLarge) return fail(PFT_ERR_CUDA, "integrate launch: %s", cudaGetErrorString(e));
    cudaGetLastError();  // not sticky (SMs partly taken): the separate kernels below, same results
  }
  PFT_LAUNCH(PFT_PROF_CULL, st, launch_pdl(k_frame_prep, dim3(nreg + ntab), dim3(256), 0, st, K, g.max_depth, depth, tiles, P, nreg, g, T, tab, zero, nzero));
  PFT_LAUNCH(PFT_PROF_CULL, st, launch_pdl(k_cull_super, dim3((ns + 255) / 256), dim3(256), 0, st, g, K, T, (const uint2*)tiles, P, nsx, nsy, nsz, slist, scount));
  PFT_LAUNCH(PFT_PROF_CULL, st, launch_pdl(k_cull_bricks, dim3(resident_grid(k_cull_bricks, 256)), dim3(256), 0, st, g, K, T, (const uint2*)tiles, P, nsx, nsy, (const uint32_t*)slist, (const uint32_t*)scount, list, count, nfree));
  // grid = the resident capacity (one wave: no partial second wave of CTAs, the CTA-stride loop
  // balances the bricks)
  const int grid = vol->esize == 4 ? resident_grid(k_integrate_list<float>, 256) : resident_grid(k_integrate_list<__half>, 256);
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_INTEGRATE, st, launch_pdl(k_integrate_list<float>, dim3(grid), dim3(256), 0, st, g, K, depth, (const double4*)tab,
                                                  (const uint32_t*)list, (const uint32_t*)count, (float*)(vol->base + vol->L.v_off),
                                                  (float*)(vol->base + vol->L.w_off), dirty, dlist, dcount, nupd));
  else
    PFT_LAUNCH(PFT_PROF_INTEGRATE, st, launch_pdl(k_integrate_list<__half>, dim3(grid), dim3(256), 0, st, g, K, depth, (const double4*)tab,
                                                  (const uint32_t*)list, (const uint32_t*)count, (__half*)(vol->base + vol->L.v_off),
                                                  (__half*)(vol->base + vol->L.w_off), dirty, dlist, dcount, nupd));
  records_rebuild_dirty(vol, st);
  return cuda_check("integrate");
}

}  // namespace pft

using namespace pft;

extern "C" {

pft_status pft_integrate_ex(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K, const double* dev_T,
                            int32_t flags, void* stream) {
  if (!vol || !dev_depth || !dev_T) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  pft_status s = check_intrinsics(K);
  if (s != PFT_OK) return s;
  return integrate_impl(vol, dev_depth, K, dev_T, flags & 1, (cudaStream_t)stream);
}

pft_status pft_integrate_stats(const pft_volume* vol, int64_t out[4], void* stream) {
  if (!vol || !out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  uint32_t w[80];
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(w, vol->base + vol->L.scratch_off, sizeof w, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check("integrate_stats");
  if (w[268 / 4]) {
    for (int i = 0; i < 4; ++i) out[i] = -1;
    return PFT_OK;
  }
  unsigned long long upd;
  memcpy(&upd, (const char*)w + 256, 8);
  out[0] = w[64 / 4];
  out[1] = w[264 / 4];
  out[2] = (int64_t)upd;
  out[3] = w[128 / 4];
  return PFT_OK;
}

pft_status pft_integrate(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K, const double* dev_T,
                         void* stream) {
  return pft_integrate_ex(vol, dev_depth, K, dev_T, 0, stream);
}

}  // extern "C"
