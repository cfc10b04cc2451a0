// track.cu — randomized-optimisation tracking (§III-B) on the TSDF.
//
// Step map:
//   k_track_init     a: state <- (T_init, s^(1)); zero accumulators
//   k_backproject    a1/a2: uint16 depth -> strided fp64 points, 8x4-pixel tile order
//   k_centre         a5: E(P) of the current pose (+ s-law a8 and the trace in its last block)
//   k_particle_eval  a3/a4: candidate poses dP_k P built per CTA in smem; particle x point
//                    tile, TSDF trilinear gathers from brick-ordered storage, per-warp
//                    reductions (REDUX) -> per-CTA smem -> one global atomic per particle
//   [ncclAllGather]  a6 (multi-GPU)
//   k_update         a7: E_k, advantage set, quaternion/translation mean, pose update; the
//                    last CTA to finish combines the per-CTA partials in a fixed order
//
// Numerics: every discrete decision (cell floor, bounds,
// in-band, E_k < E_c) is made from fp64 transforms of fp64 points; lerps are fp32; sums are
// fixed-point integers (2^-29) so per-particle totals are exact and independent of order,
// CTA shape and sharding.
#include <cmath>
#include <cstdlib>

#include "pft_internal.cuh"

namespace pft {

constexpr int kThreads = 256;  // 8 warps
constexpr int kPPT = 4;        // points per thread in k_particle_eval (one 8x4 tile per warp per p)
constexpr int kCentrePPT = 1;  // points per thread in k_centre (latency-bound: more CTAs)
constexpr int kPC = 32;        // particles per CTA chunk
constexpr double kFixScale = 536870912.0;            // 2^29
constexpr double kFixInv = 1.0 / 536870912.0;        // 2^-29


// ------------------------------------------------------------------ pose algebra (fp64)
// Rodrigues (reading L9): dR = I + (sin th/th)[r]x + ((1-cos th)/th^2)[r]x^2, th < 1e-12: I + [r]x.
__device__ __forceinline__ void rodrigues(const double r[3], double dR[9]) {
  const double th = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  double A, B;
  if (th < 1e-12) {
    A = 1.0; B = 0.0;
  } else {
    double s, c;
    sincos(th, &s, &c);
    A = s / th;
    B = (1.0 - c) / (th * th);
  }
  const double K[9] = {0.0, -r[2], r[1], r[2], 0.0, -r[0], -r[1], r[0], 0.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double k2 = K[3 * i + 0] * K[0 + j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
      dR[3 * i + j] = (i == j ? 1.0 : 0.0) + A * K[3 * i + j] + B * k2;
    }
}

// Unit quaternion (w,x,y,z) of rotation vector r (Hamilton, active): (cos th/2, r sin(th/2)/th).
__device__ __forceinline__ void rotvec_quat(const double r[3], double q[4]) {
  const double th = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (th < 1e-12) {
    q[0] = 1.0; q[1] = r[0] * 0.5; q[2] = r[1] * 0.5; q[3] = r[2] * 0.5;
  } else {
    double s, c;
    sincos(0.5 * th, &s, &c);
    const double sh = s / th;
    q[0] = c; q[1] = r[0] * sh; q[2] = r[1] * sh; q[3] = r[2] * sh;
  }
}

__device__ __forceinline__ void quat_to_R(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z);       R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);       R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);       R[7] = 2.0 * (y * z + w * x);       R[8] = 1.0 - 2.0 * (x * x + y * y);
}

// Delta (dR, u) applied to pose P (reading L10): camera-centred (dR R, t + u) or world-literal
// (dR R, dR t + u).
__device__ __forceinline__ void apply_delta(const double dR[9], const double u[3], const double* P, int conv,
                                            double out[12]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out[4 * i + j] = dR[3 * i + 0] * P[j] + dR[3 * i + 1] * P[4 + j] + dR[3 * i + 2] * P[8 + j];
    double ti = P[4 * i + 3];
    if (conv == 1) ti = dR[3 * i + 0] * P[3] + dR[3 * i + 1] * P[7] + dR[3 * i + 2] * P[11];
    out[4 * i + 3] = ti + u[i];
  }
}

// Fold pose T into voxel-grid coordinates: g = (T p - o)/s - 1/2 = (R/s) p + ((t - o)/s - 1/2).
// Returns false for non-finite or absurd poses (then every point is "outside").
__device__ __forceinline__ bool fold_pose(const double T[12], const Geom& g, double m[12]) {
  const double o[3] = {g.ox, g.oy, g.oz};
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) m[4 * i + j] = T[4 * i + j] / g.voxel;
    m[4 * i + 3] = (T[4 * i + 3] - o[i]) / g.voxel - 0.5;
  }
#pragma unroll
  for (int i = 0; i < 12; ++i) ok = ok && fabs(m[i]) < 1e30;
  return ok;
}

// Template row k scaled by s = (omega deg, v cm) (reading L8): r = a*omega*pi/180, u = b*v/100.
__device__ __forceinline__ void template_delta(const float* __restrict__ a, double omega, double v, double r[3],
                                               double u[3]) {
  const double ws = omega * (M_PI / 180.0), vs = v / 100.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    r[i] = (double)__ldg(a + i) * ws;
    u[i] = (double)__ldg(a + 3 + i) * vs;
  }
}

// ------------------------------------------------------------------ shared, non-inlined steps
// Both tracker implementations (multi-launch and persistent) call these exact functions, so their
// fp64 arithmetic (including FMA contraction) is identical and results are bit-identical.
__device__ __forceinline__ bool fast_ok(const double m[12], double pmax);

// a3: folded pose of candidate k = (dR_k R, t + u_k) (or world-literal) in grid coordinates.
// Returns 0 (invalid pose), 1 (general floor path) or 2 (fast floor path, |g| < 2^30).
__device__ __noinline__ int candidate_pose(const float* __restrict__ pst_row, double omega, double v, const double* P,
                                           int conv, const Geom& g, double pmax, double* m) {
  double r[3], u[3], dR[9], T_[12];
  template_delta(pst_row, omega, v, r, u);
  rodrigues(r, dR);
  apply_delta(dR, u, P, conv, T_);
  double mm[12];
  const bool ok = fold_pose(T_, g, mm);
  for (int i = 0; i < 12; ++i) m[i] = mm[i];
  return !ok ? 0 : (fast_ok(mm, pmax) ? 2 : 1);
}

// Folded explicit pose (pft_eval_poses rows, and the centre pose P).
__device__ __noinline__ int explicit_pose(const double* T_, const Geom& g, double pmax, double* m) {
  double t[12], mm[12];
  for (int i = 0; i < 12; ++i) t[i] = T_[i];
  const bool ok = fold_pose(t, g, mm);
  for (int i = 0; i < 12; ++i) m[i] = mm[i];
  return !ok ? 0 : (fast_ok(mm, pmax) ? 2 : 1);
}

// a7: unit quaternion and translation of template row k at search size s (advantage-set member).
__device__ __noinline__ void member_delta(const float* __restrict__ pst_row, double omega, double v, double* q,
                                          double* u) {
  double r[3], uu[3], qq[4];
  template_delta(pst_row, omega, v, r, uu);
  rotvec_quat(r, qq);
  for (int i = 0; i < 4; ++i) q[i] = qq[i];
  for (int i = 0; i < 3; ++i) u[i] = uu[i];
}

// a7: P <- (R(Q/|Q|), U/|A|) P, Q and U the sums over the advantage set.
__device__ __noinline__ void apply_mean(const double* Q, const double* U, int nA, const double* P, int conv,
                                        double* Pn) {
  const double qn = sqrt(Q[0] * Q[0] + Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3]);
  const double qb[4] = {Q[0] / qn, Q[1] / qn, Q[2] / qn, Q[3] / qn};
  const double ub[3] = {U[0] / nA, U[1] / nA, U[2] / nA};
  double Rb[9], PP[12], out[12];
  quat_to_R(qb, Rb);
  for (int i = 0; i < 12; ++i) PP[i] = P[i];
  apply_delta(Rb, ub, PP, conv, out);
  for (int i = 0; i < 12; ++i) Pn[i] = out[i];
}

// 256-thread fixed-shape tree over red[8][256] (result in red[c][0]); all threads must call.
__device__ __forceinline__ void tree8(double (*red)[256], int tid) {
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s)
#pragma unroll
      for (int c = 0; c < 8; ++c) red[c][tid] += red[c][tid + s];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ the gather-and-lerp core
// One 256-bit (fp32) / 128-bit (fp16) load per evaluation: the cell record of the 8 corners.
__device__ __forceinline__ void ld_rec(const float* p, float (&v)[8]) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
      : "l"(p));
}
__device__ __forceinline__ void ld_rec(const __half* p, float (&v)[8]) {
  unsigned u0, u1, u2, u3;
  asm("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3) : "l"(p));
  const unsigned u[4] = {u0, u1, u2, u3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __half2float(__ushort_as_half((unsigned short)(u[i] & 0xffffu)));
    v[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(u[i] >> 16)));
  }
}

// Cell index and fraction of grid coordinate g: n = floor(g), f = g - n (exact in fp64, then
// rounded to fp32 for the lerp).  FAST (|g| < 2^30 guaranteed by the caller's bound):
// t = g + 1.5*2^52 rounded toward -inf holds floor(g) in its low 32 bits and t - 1.5*2^52 is
// floor(g) exactly, so the decision is the exact floor with three DADDs and no conversion-pipe
// (XU) instruction.  Otherwise: FRND.FLOOR + saturating F2I.
template <bool FAST>
__device__ __forceinline__ int cell_split(double g, float& f) {
  if (FAST) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double t = __dadd_rd(g, M);
    f = __double2float_rn(__dsub_rn(g, __dsub_rn(t, M)));
    return __double2loint(t);
  } else {
    const double fl = floor(g);
    f = __double2float_rn(g - fl);
    return (int)fl;  // saturates; finite by fold_pose
  }
}

// PPT particle-point evaluations (O3/O4) of one pose, batched so the loads of all PPT points are
// in flight together: (1) transforms, cell splits and bounds; (2) the in-band mask words;
// (3) the 32-byte records, out-of-band lanes reading record 0 (one broadcast sector) instead
// of branching; (4) trilinear lerps.  In-band points add round(|v| * 2^29) to fix and 1 to cnt:
// each term is converted to fixed point on its own, so every sum is an exact integer whatever
// the grouping of points into threads, warps, CTAs or ranks.
template <typename T, bool FAST, int PPT>
__device__ __forceinline__ void eval_points(const T* __restrict__ R, const unsigned long long* __restrict__ mask,
                                            const Geom& g, const double (&m)[12], const double (&px)[PPT],
                                            const double (&py)[PPT], const double (&pz)[PPT], unsigned& fix,
                                            unsigned& cnt) {
  static_assert(PPT <= 7, "per-thread fixed-point sum must stay below 2^32");
  uint32_t o[PPT];
  float fx[PPT], fy[PPT], fz[PPT];
  bool ok[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const double gx = fma(m[0], px[p], fma(m[1], py[p], fma(m[2], pz[p], m[3])));
    const double gy = fma(m[4], px[p], fma(m[5], py[p], fma(m[6], pz[p], m[7])));
    const double gz = fma(m[8], px[p], fma(m[9], py[p], fma(m[10], pz[p], m[11])));
    const int ix = cell_split<FAST>(gx, fx[p]), iy = cell_split<FAST>(gy, fy[p]), iz = cell_split<FAST>(gz, fz[p]);
    ok[p] = pz[p] != 0.0 && (unsigned)ix <= (unsigned)(g.nx - 2) && (unsigned)iy <= (unsigned)(g.ny - 2) &&
            (unsigned)iz <= (unsigned)(g.nz - 2);
    // computed unconditionally and masked (no branch): out-of-range lanes use cell 0
    o[p] = (offx(ix) + offy(iy, g.sy) + offz(iz, g.sz)) & (0u - (uint32_t)ok[p]);
  }
  // in band iff all 8 corners |V| < 1 (reading L3): one bit per cell, precomputed from the
  // same stored values by the record builder
  unsigned long long mw[PPT];
#ifdef PFT_DEBUG
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const size_t nrec = (size_t)g.sz * (size_t)g.nbz;
    if (o[p] >= nrec || ((uintptr_t)(mask + (o[p] >> 6)) & 7) || ((uintptr_t)(R + (size_t)o[p] * 8) & (8 * sizeof(T) - 1))) {
      printf("pft debug: bad address p=%d o=%u nrec=%zu mask=%p R=%p ok=%d\n", p, o[p], nrec, (void*)mask, (void*)R, (int)ok[p]);
      __trap();
    }
  }
#endif
  // Addresses are formed as byte offsets from integer-selected indices (one IMAD.WIDE each):
  // the predicated "CS2R; @!P IMAD.WIDE; IADD3 r,UR,r" idiom ptxas 12.9 emitted for
  // base + (ok ? o : 0) * size read a stale register on B200.
  const char* mbase = reinterpret_cast<const char*>(mask);
  const char* rbase = reinterpret_cast<const char*>(R);
#pragma unroll
  for (int p = 0; p < PPT; ++p)
    mw[p] = __ldg(reinterpret_cast<const unsigned long long*>(mbase + (size_t)(o[p] >> 6) * 8u));
  float v[PPT][8];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ok[p] = ok[p] && ((mw[p] >> (o[p] & 63)) & 1ull);
    const uint32_t orec = o[p] & (0u - (uint32_t)ok[p]);
    ld_rec(reinterpret_cast<const T*>(rbase + (size_t)orec * (8u * sizeof(T))), v[p]);
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    float val;
    if (sizeof(T) == 4) {  // polynomial coefficients [a b c d e f g h]
      const float* k = v[p];
      const float t1 = fmaf(fz[p], k[7], k[4]);          // e + h fz
      float t2 = fmaf(fy[p], t1, k[1]);                   // b + fy (e + h fz)
      t2 = fmaf(fz[p], k[5], t2);                         //   + f fz
      const float t3 = fmaf(fz[p], k[6], k[2]);           // c + g fz
      float acc = fmaf(fz[p], k[3], k[0]);                // a + d fz
      acc = fmaf(fy[p], t3, acc);
      val = fmaf(fx[p], t2, acc);
    } else {               // corner values
      const float c00 = fmaf(fx[p], v[p][1] - v[p][0], v[p][0]), c10 = fmaf(fx[p], v[p][3] - v[p][2], v[p][2]);
      const float c01 = fmaf(fx[p], v[p][5] - v[p][4], v[p][4]), c11 = fmaf(fx[p], v[p][7] - v[p][6], v[p][6]);
      const float c0 = fmaf(fy[p], c10 - c00, c00), c1 = fmaf(fy[p], c11 - c01, c01);
      val = fmaf(fz[p], c1 - c0, c0);
    }
    fix += ok[p] ? __float2uint_rn(fabsf(val) * (float)kFixScale) : 0u;
    cnt += ok[p] ? 1u : 0u;
  }
}

// The centre E(P) (a5) drives the search-size law (a8), so its value is reproduced to fp64
// accuracy: same decisions and loads as eval_points, fp64 lerps, and each |v| rounded to a
// 2^-44 fixed-point uint64 (exact sums; < 2^63 for N < 2^19 points).
constexpr double kFixScaleC = 17592186044416.0;   // 2^44
constexpr double kFixInvC = 1.0 / 17592186044416.0;
template <typename T> __device__ __forceinline__ float ldv(const T* p);
template <> __device__ __forceinline__ float ldv<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ldv<__half>(const __half* p) { return __half2float(__ldg(p)); }
template <typename T, bool FAST, int PPT>
__device__ __forceinline__ void eval_points_f64(const T* __restrict__ V, const unsigned long long* __restrict__ mask,
                                                const Geom& g, const double (&m)[12], const double (&px)[PPT],
                                                const double (&py)[PPT], const double (&pz)[PPT],
                                                unsigned long long& fix, unsigned& cnt) {
  uint32_t o[PPT];
  double fx[PPT], fy[PPT], fz[PPT];
  bool ok[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const double gx = fma(m[0], px[p], fma(m[1], py[p], fma(m[2], pz[p], m[3])));
    const double gy = fma(m[4], px[p], fma(m[5], py[p], fma(m[6], pz[p], m[7])));
    const double gz = fma(m[8], px[p], fma(m[9], py[p], fma(m[10], pz[p], m[11])));
    float f32;
    const int ix = cell_split<FAST>(gx, f32), iy = cell_split<FAST>(gy, f32), iz = cell_split<FAST>(gz, f32);
    fx[p] = gx - floor(gx); fy[p] = gy - floor(gy); fz[p] = gz - floor(gz);
    ok[p] = pz[p] != 0.0 && (unsigned)ix <= (unsigned)(g.nx - 2) && (unsigned)iy <= (unsigned)(g.ny - 2) &&
            (unsigned)iz <= (unsigned)(g.nz - 2);
    o[p] = ok[p] ? offx(ix) + offy(iy, g.sy) + offz(iz, g.sz) : 0u;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const unsigned long long mw = __ldg(mask + (o[p] >> 6));
    ok[p] = ok[p] && ((mw >> (o[p] & 63)) & 1ull);
    // exact stored corner values (brick order), not the record
    const uint32_t b = ok[p] ? o[p] : 0u;
    const uint32_t dx = ((b & 3u) == 3u) ? 64u - 3u : 1u;              // x + 1 crosses into the next brick?
    const uint32_t dy = (((b >> 2) & 3u) == 3u) ? g.sy - 12u : 4u;
    const uint32_t dz = (((b >> 4) & 3u) == 3u) ? g.sz - 48u : 16u;
    double w[8];
    w[0] = ldv(V + b);           w[1] = ldv(V + b + dx);
    w[2] = ldv(V + b + dy);      w[3] = ldv(V + b + dx + dy);
    w[4] = ldv(V + b + dz);      w[5] = ldv(V + b + dx + dz);
    w[6] = ldv(V + b + dy + dz); w[7] = ldv(V + b + dx + dy + dz);
    const double c00 = __fma_rn(fx[p], w[1] - w[0], w[0]), c10 = __fma_rn(fx[p], w[3] - w[2], w[2]);
    const double c01 = __fma_rn(fx[p], w[5] - w[4], w[4]), c11 = __fma_rn(fx[p], w[7] - w[6], w[6]);
    const double c0 = __fma_rn(fy[p], c10 - c00, c00), c1 = __fma_rn(fy[p], c11 - c01, c01);
    const double val = __fma_rn(fz[p], c1 - c0, c0);
    fix += ok[p] ? __double2ull_rn(fabs(val) * kFixScaleC) : 0ull;
    cnt += ok[p] ? 1u : 0u;
  }
}

// Warp total of a 64-bit fixed-point sum and a count (butterfly; same value in every lane).
__device__ __forceinline__ void warp_total64(unsigned long long fix, unsigned cnt, unsigned long long& S, unsigned& n) {
  for (int sft = 16; sft > 0; sft >>= 1) {
    fix += __shfl_xor_sync(0xffffffffu, fix, sft);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, sft);
  }
  S = fix;
  n = cnt;
}

// Warp total of (fix, cnt) -> 64-bit fixed-point total (same value in every lane).  All lanes must call.
__device__ __forceinline__ void warp_total(unsigned fix, unsigned cnt, unsigned long long& S, unsigned& n) {
  const unsigned lo = __reduce_add_sync(0xffffffffu, fix & 0xffffu);
  const unsigned hi = __reduce_add_sync(0xffffffffu, fix >> 16);
  n = __reduce_add_sync(0xffffffffu, cnt);
  S = ((unsigned long long)hi << 16) + lo;
}

// FAST-path bound for pose m on points with max |coordinate| <= pmax: every |g| < 2^30.
__device__ __forceinline__ bool fast_ok(const double m[12], double pmax) {
  bool ok = true;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    ok = ok && (fabs(m[4 * r]) + fabs(m[4 * r + 1]) + fabs(m[4 * r + 2])) * pmax + fabs(m[4 * r + 3]) < 1073741824.0;
  return ok;
}

struct Points { const double *x, *y, *z; int npad; };

// Block-wide max of v (blockDim.x == kThreads); all threads get the result.
__device__ __forceinline__ double block_max(double v, double* red) {
  for (int s = 16; s > 0; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, s));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int w = 1; w < kThreads / 32; ++w) r = fmax(r, red[w]);
  return r;
}

// ------------------------------------------------------------------ kernels
struct EvalArgs {
  const void* R;             // cell records
  const unsigned long long* mask;  // in-band bits
  Geom g;
  Points pts;
  int mode;                  // 0: template particles, 1: explicit poses
  const float* pst;          // mode 0: full K x 6 template
  int k_begin, k_count;      // particle range of this launch (absolute template rows / pose rows)
  const TrackState* st;      // mode 0: P and s
  int conv;
  const double* poses;       // mode 1: M x 12
  PartRec* acc;              // indexed by k - k_begin
};

template <typename T, int PPT, bool FAST>
__device__ __forceinline__ void eval_chunk(const EvalArgs& a, const double2 (*sPose)[6], const int* sFlag,
                                          unsigned long long* sS, unsigned* sN, int kc, const double (&px)[PPT],
                                          const double (&py)[PPT], const double (&pz)[PPT]) {
  const T* R = (const T*)a.R;
  for (int j = 0; j < kc; ++j) {
    if (sFlag[j] != (FAST ? 2 : 1)) continue;  // block-uniform
    double m[12];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const double2 q = sPose[j][i];
      m[2 * i] = q.x;
      m[2 * i + 1] = q.y;
    }
    unsigned sum = 0u;
    unsigned cnt = 0u;
    eval_points<T, FAST, PPT>(R, a.mask, a.g, m, px, py, pz, sum, cnt);
    unsigned long long S;
    unsigned n;
    warp_total(sum, cnt, S, n);
    if ((threadIdx.x & 31) == 0 && n) {
      atomicAdd(&sS[j], S);
      atomicAdd(&sN[j], n);
    }
  }
}

// a3/a4: CTA = kThreads x PPT points (PPT 8x4-pixel tiles per warp) x kPC particles.
template <typename T, int PPT>
#ifndef PFT_MINB
#define PFT_MINB 2
#endif
__global__ __launch_bounds__(kThreads, PFT_MINB) void k_particle_eval(EvalArgs a) {
  __shared__ double2 sPose[kPC][6];
  __shared__ unsigned long long sS[kPC];
  __shared__ unsigned sN[kPC];
  __shared__ int sFlag[kPC];  // 0 invalid pose, 1 general path, 2 fast path
  __shared__ double sRed[kThreads / 32];
  const int c0 = blockIdx.y * kPC;
  const int kc = min(kPC, a.k_count - c0);
  const int tid = threadIdx.x;
  // this thread's points (8x4 tiles; z == 0 marks an invalid / padding slot)
  double px[PPT], py[PPT], pz[PPT];
  double pm = 0.0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int i = (blockIdx.x * PPT + p) * kThreads + tid;
    if (i < a.pts.npad) {
      px[p] = a.pts.x[i]; py[p] = a.pts.y[i]; pz[p] = a.pts.z[i];
    } else {
      px[p] = py[p] = pz[p] = 0.0;
    }
    pm = fmax(pm, fmax(fabs(px[p]), fmax(fabs(py[p]), fabs(pz[p]))));
  }
  const double pmax = block_max(pm, sRed);
  if (tid < kc) {
    const int k = a.k_begin + c0 + tid;
    double m[12];
    sFlag[tid] = a.mode == 0 ? candidate_pose(a.pst + 6 * (size_t)k, a.st->omega, a.st->v, a.st->P, a.conv, a.g, pmax, m)
                             : explicit_pose(a.poses + 12 * (size_t)k, a.g, pmax, m);
#pragma unroll
    for (int i = 0; i < 6; ++i) sPose[tid][i] = make_double2(m[2 * i], m[2 * i + 1]);
    sS[tid] = 0ull;
    sN[tid] = 0u;
  }
  __syncthreads();
  eval_chunk<T, PPT, true>(a, sPose, sFlag, sS, sN, kc, px, py, pz);
  eval_chunk<T, PPT, false>(a, sPose, sFlag, sS, sN, kc, px, py, pz);
  __syncthreads();
  if (tid < kc && sN[tid]) {
    PartRec* r = a.acc + (c0 + tid);
    atomicAdd(&r->S, sS[tid]);
    atomicAdd(&r->n, sN[tid]);
  }
}

// E from a fixed-point record (O4; reading L6): S/n if n > 0 and n >= rho N, else 1.
__device__ __forceinline__ double fitness_of(unsigned long long S, unsigned n, double rho, int N) {
  if (n > 0u && (double)n >= rho * (double)N) return ((double)S * kFixInv) / (double)n;
  return 1.0;
}
// Same for the fp64 centre sums (2^-44 units).
__device__ __forceinline__ double fitness_c(unsigned long long S, unsigned n, double rho, int N) {
  if (n > 0u && (double)n >= rho * (double)N) return ((double)S * kFixInvC) / (double)n;
  return 1.0;
}

struct TrackArgs {
  TrackState* st;
  const double* T_init;
  double omega0, v0, beta, rho;
  int conv;
  PartRec* acc_local;
  int kloc;
};

__global__ void k_track_init(TrackArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    TrackState* s = a.st;
    for (int j = 0; j < 12; ++j) s->P[j] = a.T_init[j];
    s->omega = a.omega0; s->v = a.v0;
    s->Ec = 1.0; s->Ebase = 1.0;
    s->Sc_acc = 0ull; s->nc_acc = 0u; s->nc = 0u;
    s->nA = 0; s->iter = 0; s->Nvalid = 0;
    s->ticket_upd = 0u; s->ticket_ctr = 0u;
  }
  for (int k = i; k < a.kloc; k += gridDim.x * blockDim.x) {
    a.acc_local[k].S = 0ull;
    a.acc_local[k].n = 0u;
    a.acc_local[k].pad = 0u;
  }
}

// O1/O2: points of the strided pixel grid (sigma c, sigma r), r < nr, c < nc, in 8x4 tiles.
struct BPArgs {
  const uint16_t* depth;
  double fx, fy, cx, cy, unit, max_depth;
  int W, H, stride, nr, nc, ntx, npad;
  double *x, *y, *z;
  int* Nvalid;
};

__global__ void k_backproject(BPArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npad) return;
  const int t = i >> 5, l = i & 31;
  const int r = (t / a.ntx) * 4 + (l >> 3), c = (t % a.ntx) * 8 + (l & 7);
  double X = 0.0, Y = 0.0, Z = 0.0;
  bool valid = false;
  if (r < a.nr && c < a.nc) {
    const int u = c * a.stride, v = r * a.stride;
    const uint16_t raw = a.depth[(size_t)v * a.W + u];
    const double d = __dmul_rn((double)raw, a.unit);
    if (raw != 0 && d < a.max_depth) {
      valid = true;
      X = __ddiv_rn(__dmul_rn(__dsub_rn((double)u, a.cx), d), a.fx);
      Y = __ddiv_rn(__dmul_rn(__dsub_rn((double)v, a.cy), d), a.fy);
      Z = d;
    }
  }
  a.x[i] = X; a.y[i] = Y; a.z[i] = Z;
  const unsigned b = __ballot_sync(0xffffffffu, valid);
  if (l == 0 && b) atomicAdd(a.Nvalid, __popc(b));
}

// a5 + a8: E(P) of the current pose; the last CTA closes the iteration (s-law, trace).
struct CentreArgs {
  const void* V;                    // stored values (the centre lerps exact corner values in fp64)
  const unsigned long long* mask;
  Geom g;
  Points pts;
  TrackState* st;
  int initial;          // 1: baseline E(T_init) before iteration 1 (no s-update, no trace)
  double beta, rho;
  double* trace;        // NULL or iters x PFT_TRACE_DOUBLES
  double* T_out;        // written by the last CTA of every call
};

template <typename T>
__global__ __launch_bounds__(kThreads) void k_centre(CentreArgs a) {
  __shared__ double sm[12];
  __shared__ int sOk;
  __shared__ bool sLast;
  __shared__ double sRed[kThreads / 32];
  TrackState* st = a.st;
  const bool do_eval = a.initial || st->nA > 0;
  const int tid = threadIdx.x;
  if (do_eval) {
    double px[kCentrePPT], py[kCentrePPT], pz[kCentrePPT], pm = 0.0;
#pragma unroll
    for (int p = 0; p < kCentrePPT; ++p) {
      const int i = (blockIdx.x * kCentrePPT + p) * kThreads + tid;
      px[p] = py[p] = pz[p] = 0.0;
      if (i < a.pts.npad) { px[p] = a.pts.x[i]; py[p] = a.pts.y[i]; pz[p] = a.pts.z[i]; }
      pm = fmax(pm, fmax(fabs(px[p]), fmax(fabs(py[p]), fabs(pz[p]))));
    }
    const double pmax = block_max(pm, sRed);
    if (tid == 0) {
      double m[12];
      sOk = explicit_pose(st->P, a.g, pmax, m);
      for (int i = 0; i < 12; ++i) sm[i] = m[i];
    }
    __syncthreads();
    unsigned long long sum = 0ull;
    unsigned cnt = 0u;
    if (sOk) {
      double m[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) m[i] = sm[i];
      if (sOk == 2) eval_points_f64<T, true, kCentrePPT>((const T*)a.V, a.mask, a.g, m, px, py, pz, sum, cnt);
      else eval_points_f64<T, false, kCentrePPT>((const T*)a.V, a.mask, a.g, m, px, py, pz, sum, cnt);
    }
    unsigned long long S;
    unsigned n;
    warp_total64(sum, cnt, S, n);
    if ((tid & 31) == 0 && n) {
      atomicAdd(&st->Sc_acc, S);
      atomicAdd(&st->nc_acc, n);
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) sLast = atomicAdd(&st->ticket_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sLast || tid != 0) return;
  __threadfence();
  volatile TrackState* vs = st;
  double Ec = vs->Ec;
  unsigned nc = vs->nc;
  if (do_eval) {
    const unsigned long long S = vs->Sc_acc;
    nc = vs->nc_acc;
    Ec = fitness_c(S, nc, a.rho, vs->Nvalid);
  }
  st->Sc_acc = 0ull;
  st->nc_acc = 0u;
  st->ticket_ctr = 0u;
  st->Ec = Ec;
  st->nc = nc;
  if (!a.initial) {
    // s^(i+1) = beta s^(i) + (1 - beta) E(P^(i)) s^(i), as (beta + (1-beta)E) s
    const double om = vs->omega, v = vs->v;
    const double factor = __dadd_rn(a.beta, __dmul_rn(__dsub_rn(1.0, a.beta), Ec));
    const double om1 = __dmul_rn(factor, om), v1 = __dmul_rn(factor, v);
    st->omega = om1;
    st->v = v1;
    const int it = vs->iter;
    if (a.trace) {
      double* r = a.trace + (size_t)it * PFT_TRACE_DOUBLES;
      const int nA = vs->nA;
      const int N = vs->Nvalid;
      r[0] = vs->Ebase; r[1] = (double)nA; r[2] = om; r[3] = v;
      for (int i = 0; i < 12; ++i) r[4 + i] = vs->P[i];
      r[16] = Ec; r[17] = om1; r[18] = v1;
      r[19] = (double)((nA == 0 ? 1 : 0) | (vs->Ebase == 1.0 ? 2 : 0) | (N == 0 ? 4 : 0));
      r[20] = (double)nc; r[21] = (double)N; r[22] = 0.0; r[23] = 0.0;
    }
    st->iter = it + 1;
  }
  if (a.T_out)
    for (int i = 0; i < 12; ++i) a.T_out[i] = vs->P[i];
}

// a7: E_k, advantage set A = {k : E_k < E_c}, mean delta over A,
// P <- (R(q), u) P.  nblk CTAs of 256 threads, one particle per thread; each CTA
// reduces its members in a fixed tree, the last CTA combines the CTA partials in a fixed tree.
struct UpdArgs {
  TrackState* st;
  const PartRec* full;       // K records (all ranks)
  PartRec* local;            // this rank's records, zeroed for the next iteration
  int K, k_begin, kloc;      // local covers global [k_begin, k_begin + kloc)
  const float* pst;
  int conv;
  double rho;
  double* E_out;
  int* n_out;
  double* partials;          // nblk x 8
};

__global__ __launch_bounds__(256) void k_update(UpdArgs a) {
  __shared__ double red[8][256];
  __shared__ bool sLast;
  TrackState* st = a.st;
  const int tid = threadIdx.x;
  const int k = blockIdx.x * 256 + tid;
  const double Ec = st->Ec;
  const int N = st->Nvalid;
  double q[4] = {0.0, 0.0, 0.0, 0.0}, u[3] = {0.0, 0.0, 0.0}, member = 0.0;
  if (k < a.K) {
    const PartRec rec = a.full[k];
    const double E = fitness_of(rec.S, rec.n, a.rho, N);
    a.E_out[k] = E;
    a.n_out[k] = (int)rec.n;
    if (E < Ec) {
      member_delta(a.pst + 6 * (size_t)k, st->omega, st->v, q, u);
      member = 1.0;
    }
    const int j = k - a.k_begin;
    if (j >= 0 && j < a.kloc) {
      a.local[j].S = 0ull;
      a.local[j].n = 0u;
    }
  }
  red[0][tid] = q[0]; red[1][tid] = q[1]; red[2][tid] = q[2]; red[3][tid] = q[3];
  red[4][tid] = u[0]; red[5][tid] = u[1]; red[6][tid] = u[2]; red[7][tid] = member;
  tree8(red, tid);
  if (tid < 8) a.partials[blockIdx.x * 8 + tid] = red[tid][0];
  __threadfence();
  __syncthreads();
  if (tid == 0) sLast = atomicAdd(&st->ticket_upd, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sLast) return;
  __threadfence();
  // fixed-order combine of the CTA partials
#pragma unroll
  for (int c = 0; c < 8; ++c) red[c][tid] = 0.0;
  for (int b = tid; b < (int)gridDim.x; b += 256)
#pragma unroll
    for (int c = 0; c < 8; ++c) red[c][tid] += __ldcg(a.partials + b * 8 + c);
  tree8(red, tid);
  if (tid == 0) {
    const int nA = (int)red[7][0];
    st->nA = nA;
    st->Ebase = Ec;
    st->ticket_upd = 0u;
    if (nA > 0) {
      const double Q[4] = {red[0][0], red[1][0], red[2][0], red[3][0]};
      const double U[3] = {red[4][0], red[5][0], red[6][0]};
      double Pn[12];
      apply_mean(Q, U, nA, st->P, a.conv, Pn);
      for (int i = 0; i < 12; ++i) st->P[i] = Pn[i];
    }
  }
}


// ------------------------------------------------------------------ persistent tracker (G = 1)
// The whole RO loop of one frame in ONE cooperative launch (all CTAs co-resident): phases are
// separated by a software grid barrier instead of kernel boundaries, which removes ~3 launches
// and their tail/latency per iteration.  Phase structure per iteration i:
//   P1 candidate-pose table (K rows, each CTA a slice)                    | barrier
//   P2 particle x point evaluation: warp-granular items (4 tiles x 16
//      particles) handed out by an atomic counter -> no CTA barriers, no
//      wave tail; warp totals -> global integer atomics                   | barrier
//   P3 update partials: 256-particle blocks, the same tree as k_update    | barrier
//   P4 every CTA combines the partials in the same fixed tree (identical
//      P everywhere), then evaluates E(P) on its slice of the points      | barrier
//   P5 every CTA sums the centre partials (integers) -> E_c, s-law; CTA 0
//      writes the trace.
// Results are bit-identical to the multi-launch path (same helpers, integer sums, same trees).
constexpr int kItemTiles = 4;     // 8x4 tiles per warp item (= PPT 4 points per lane)
constexpr int kItemParticles = 16;

struct PArgs {
  const void* R;
  const void* V;
  const unsigned long long* mask;
  Geom g;
  BPArgs bp;
  Points pts;
  const float* pst;
  int K, conv, iters, nblk_upd, ngroups, nchunks, sched;
  double beta, rho, omega0, v0;
  const double* T_init;
  TrackState* st;
  PartRec* acc;
  double* E_out;
  int* n_out;
  double* trace;
  double* T_out;
  double* ptab;
  int* pflag;
  double* upart;
  unsigned long long* cpart;
  unsigned* work;
};

// Sense-reversing grid barrier over co-resident CTAs; the gpu-scope fences also invalidate L1
// (CCTL.IVALL) so data written by other CTAs before the barrier is read fresh after it.
__device__ __forceinline__ void grid_barrier(TrackState* st, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&st->bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      st->bar_count = 0u;
      __threadfence();
      atomicExch(&st->bar_gen, gen + 1u);
    } else {
      while (*(volatile unsigned*)&st->bar_gen == gen) __nanosleep(32);
    }
    __threadfence();
  }
  gen += 1u;
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ void centre_slice(const PArgs& a, const double* m, int flag, unsigned long long& sum,
                                             unsigned& cnt) {
  const int per = (a.pts.npad + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(a.pts.npad, b0 + per);
  for (int base = b0; base < b1; base += kThreads) {
    const int i = base + threadIdx.x;
    double px[1] = {0.0}, py[1] = {0.0}, pz[1] = {0.0};
    if (i < b1) { px[0] = __ldcg(a.pts.x + i); py[0] = __ldcg(a.pts.y + i); pz[0] = __ldcg(a.pts.z + i); }
    double mm[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) mm[q] = m[q];
    if (flag == 2) eval_points_f64<T, true, 1>((const T*)a.V, a.mask, a.g, mm, px, py, pz, sum, cnt);
    else if (flag == 1) eval_points_f64<T, false, 1>((const T*)a.V, a.mask, a.g, mm, px, py, pz, sum, cnt);
  }
}

// CTA total of the centre's (sum, cnt) -> thread 0.
__device__ __forceinline__ void block_total(unsigned long long sum, unsigned cnt, unsigned long long* sS, unsigned* sN,
                                            unsigned long long& S, unsigned& n) {
  unsigned long long ws;
  unsigned wn;
  warp_total64(sum, cnt, ws, wn);
  if ((threadIdx.x & 31) == 0) { sS[threadIdx.x >> 5] = ws; sN[threadIdx.x >> 5] = wn; }
  __syncthreads();
  S = 0ull; n = 0u;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) { S += sS[w]; n += sN[w]; }
  __syncthreads();
}

template <typename T>
__global__ __launch_bounds__(kThreads, 2) void k_track_persistent(PArgs a) {
  // red (update phases) and sPart (evaluation phase) are never live at the same time
  constexpr size_t kRedBytes = 8 * 256 * sizeof(double);
  constexpr size_t kPartBytes = (kThreads / 32) * kItemParticles * 33 * sizeof(unsigned long long);
  __shared__ __align__(16) unsigned char sUnion[kRedBytes > kPartBytes ? kRedBytes : kPartBytes];
  double (*red)[256] = reinterpret_cast<double (*)[256]>(sUnion);
  __shared__ double sP[12], sM[12];
  __shared__ double sState[4];  // omega, v, Ec, Ebase
  __shared__ int sFlagC, sNA, sN, sItem;
  __shared__ unsigned sNc;
  __shared__ unsigned long long sS[kThreads / 32];
  __shared__ unsigned sNw[kThreads / 32];
  __shared__ double2 sWPose[kThreads / 32][kItemParticles * 6];
  __shared__ int sWFlag[kThreads / 32][kItemParticles];
  // per-lane partials of the item's particles: (fix | cnt << 32), rows padded against bank conflicts
  unsigned long long (*sPart)[kItemParticles][33] =
      reinterpret_cast<unsigned long long (*)[kItemParticles][33]>(sUnion);
  TrackState* st = a.st;
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned gen = 0u;
  if (tid == 0) gen = *(volatile unsigned*)&st->bar_gen;
  // ---- P0: points (a1/a2), accumulators, pmax
  {
    const int stride = gridDim.x * kThreads;
    double pm = 0.0;
    for (int i0 = blockIdx.x * kThreads; i0 < a.pts.npad; i0 += stride) {
      const int i = i0 + tid;  // npad is a multiple of 32: whole warps stay converged
      const int t = i >> 5, l = i & 31;
      const int r = (t / a.bp.ntx) * 4 + (l >> 3), c = (t % a.bp.ntx) * 8 + (l & 7);
      double X = 0.0, Y = 0.0, Z = 0.0;
      bool valid = false;
      if (i < a.pts.npad && r < a.bp.nr && c < a.bp.nc) {
        const int u = c * a.bp.stride, v = r * a.bp.stride;
        const uint16_t raw = a.bp.depth[(size_t)v * a.bp.W + u];
        const double d = __dmul_rn((double)raw, a.bp.unit);
        if (raw != 0 && d < a.bp.max_depth) {
          valid = true;
          X = __ddiv_rn(__dmul_rn(__dsub_rn((double)u, a.bp.cx), d), a.bp.fx);
          Y = __ddiv_rn(__dmul_rn(__dsub_rn((double)v, a.bp.cy), d), a.bp.fy);
          Z = d;
        }
      }
      if (i < a.pts.npad) { a.bp.x[i] = X; a.bp.y[i] = Y; a.bp.z[i] = Z; }
      pm = fmax(pm, fmax(fabs(X), fmax(fabs(Y), fabs(Z))));
      const unsigned b = __ballot_sync(0xffffffffu, valid);
      if (l == 0 && b) atomicAdd(&st->Nvalid, __popc(b));
    }
    for (int sft = 16; sft > 0; sft >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, sft));
    if (lane == 0 && pm > 0.0) atomicMax(&st->pmax_bits, (unsigned long long)__double_as_longlong(pm));
    for (int k = blockIdx.x * kThreads + tid; k < a.K; k += stride) { a.acc[k].S = 0ull; a.acc[k].n = 0u; }
  }
  grid_barrier(st, gen);
  const double pmax = __longlong_as_double((long long)__ldcg(&st->pmax_bits));
  const int N = __ldcg(&st->Nvalid);
  // ---- initial centre E(T_init)
  if (tid == 0) {
    for (int q = 0; q < 12; ++q) sP[q] = a.T_init[q];
    sFlagC = explicit_pose(sP, a.g, pmax, sM);
  }
  __syncthreads();
  {
    unsigned long long sum = 0ull;
    unsigned cnt = 0u;
    centre_slice<T>(a, sM, sFlagC, sum, cnt);
    unsigned long long S;
    unsigned n;
    block_total(sum, cnt, sS, sNw, S, n);
    if (tid == 0) { a.cpart[2 * blockIdx.x] = S; a.cpart[2 * blockIdx.x + 1] = n; }
  }
  grid_barrier(st, gen);
  if (tid == 0) {
    unsigned long long S = 0ull, n = 0ull;
    for (int b = 0; b < (int)gridDim.x; ++b) { S += __ldcg(a.cpart + 2 * b); n += __ldcg(a.cpart + 2 * b + 1); }
    sState[0] = a.omega0; sState[1] = a.v0;
    sState[2] = fitness_c(S, (unsigned)n, a.rho, N);
    sNc = (unsigned)n;
    sN = N;
  }
  __syncthreads();
  for (int it = 0; it < a.iters; ++it) {
    // ---- P1: candidate-pose table
    for (int k = blockIdx.x * kThreads + tid; k < a.K; k += gridDim.x * kThreads) {
      double m[12];
      a.pflag[k] = candidate_pose(a.pst + 6 * (size_t)k, sState[0], sState[1], sP, a.conv, a.g, pmax, m);
      double2* row = (double2*)(a.ptab + 12 * (size_t)k);
#pragma unroll
      for (int q = 0; q < 6; ++q) row[q] = make_double2(m[2 * q], m[2 * q + 1]);
    }
    grid_barrier(st, gen);
    // ---- P2: particle x point evaluation, warp-granular items (group-major: item = group * nchunks
    // + chunk).  sched 0: one global dynamic queue; sched 1: CTA c owns the contiguous range
    // [c*n/G, (c+1)*n/G) (its warps share one image region -> L1 reuse), handed out by a CTA counter.
    {
      const int nitems = a.ngroups * a.nchunks;
      const int r0 = (int)((long long)nitems * blockIdx.x / gridDim.x);
      const int r1 = (int)((long long)nitems * (blockIdx.x + 1) / gridDim.x);
      if (tid == 0) sItem = 0;
      __syncthreads();
      for (;;) {
        int item = 0;
        if (lane == 0) item = a.sched == 1 ? r0 + atomicAdd(&sItem, 1) : (int)atomicAdd(a.work + it, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= (a.sched == 1 ? r1 : nitems)) break;
        const int group = item / a.nchunks, chunk = item - group * a.nchunks;
        double px[kItemTiles], py[kItemTiles], pz[kItemTiles];
#pragma unroll
        for (int p = 0; p < kItemTiles; ++p) {
          const int i = (group * kItemTiles + p) * 32 + lane;
          px[p] = py[p] = pz[p] = 0.0;
          if (i < a.pts.npad) { px[p] = __ldcg(a.pts.x + i); py[p] = __ldcg(a.pts.y + i); pz[p] = __ldcg(a.pts.z + i); }
        }
        const int k0 = chunk * kItemParticles, k1 = min(a.K, k0 + kItemParticles);
        // stage the item's poses in this warp's shared slot (6 x 16 B per pose, 3 per lane)
        double2* wp = sWPose[tid >> 5];
        int* wf = sWFlag[tid >> 5];
        __syncwarp();
        for (int q = lane; q < (k1 - k0) * 6; q += 32) wp[q] = __ldcg((const double2*)(a.ptab + 12 * (size_t)k0) + q);
        if (lane < k1 - k0) wf[lane] = __ldcg(a.pflag + k0 + lane);
        __syncwarp();
        unsigned long long (*part)[33] = sPart[tid >> 5];
        for (int k = k0; k < k1; ++k) {
          const int flag = wf[k - k0];
          unsigned sum = 0u;
          unsigned cnt = 0u;
          if (flag != 0) {  // warp-uniform
            double m[12];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const double2 v = wp[(k - k0) * 6 + q];
              m[2 * q] = v.x;
              m[2 * q + 1] = v.y;
            }
            if (flag == 2) eval_points<T, true, kItemTiles>((const T*)a.R, a.mask, a.g, m, px, py, pz, sum, cnt);
            else eval_points<T, false, kItemTiles>((const T*)a.R, a.mask, a.g, m, px, py, pz, sum, cnt);
          }
          part[k - k0][lane] = (unsigned long long)sum | ((unsigned long long)cnt << 32);
        }
        __syncwarp();
        // lane j < #particles reduces particle j's row (exact integers) and issues its atomics
        if (lane < k1 - k0) {
          unsigned long long S = 0ull;
          unsigned n = 0u;
          for (int l = 0; l < 32; ++l) {
            const unsigned long long w = part[lane][l];
            S += w & 0xffffffffull;
            n += (unsigned)(w >> 32);
          }
          if (n) {
            atomicAdd(&a.acc[k0 + lane].S, S);
            atomicAdd(&a.acc[k0 + lane].n, n);
          }
        }
        __syncwarp();
      }
    }
    grid_barrier(st, gen);
    // ---- P3: E_k, advantage set, per-block partials (same tree as k_update)
    const double Ec = sState[2];
    for (int b = blockIdx.x; b < a.nblk_upd; b += gridDim.x) {
      const int k = b * 256 + tid;
      double q[4] = {0.0, 0.0, 0.0, 0.0}, u[3] = {0.0, 0.0, 0.0}, member = 0.0;
      if (k < a.K) {
        const unsigned long long S = __ldcg(&a.acc[k].S);
        const unsigned n = __ldcg(&a.acc[k].n);
        const double E = fitness_of(S, n, a.rho, N);
        a.E_out[k] = E;
        a.n_out[k] = (int)n;
        if (E < Ec) {
          member_delta(a.pst + 6 * (size_t)k, sState[0], sState[1], q, u);
          member = 1.0;
        }
        a.acc[k].S = 0ull;
        a.acc[k].n = 0u;
      }
      red[0][tid] = q[0]; red[1][tid] = q[1]; red[2][tid] = q[2]; red[3][tid] = q[3];
      red[4][tid] = u[0]; red[5][tid] = u[1]; red[6][tid] = u[2]; red[7][tid] = member;
      tree8(red, tid);
      if (tid < 8) a.upart[b * 8 + tid] = red[tid][0];
      __syncthreads();
    }
    grid_barrier(st, gen);
    // ---- P4: combine partials (fixed tree, identical in every CTA) -> P; centre slice
#pragma unroll
    for (int c = 0; c < 8; ++c) red[c][tid] = 0.0;
    for (int b = tid; b < a.nblk_upd; b += 256)
#pragma unroll
      for (int c = 0; c < 8; ++c) red[c][tid] += __ldcg(a.upart + b * 8 + c);
    tree8(red, tid);
    if (tid == 0) {
      const int nA = (int)red[7][0];
      sNA = nA;
      sState[3] = Ec;
      if (nA > 0) {
        const double Q[4] = {red[0][0], red[1][0], red[2][0], red[3][0]};
        const double U[3] = {red[4][0], red[5][0], red[6][0]};
        double Pn[12];
        apply_mean(Q, U, nA, sP, a.conv, Pn);
        for (int q = 0; q < 12; ++q) sP[q] = Pn[q];
        sFlagC = explicit_pose(sP, a.g, pmax, sM);
      }
    }
    __syncthreads();
    if (sNA > 0) {
      unsigned long long sum = 0ull;
      unsigned cnt = 0u;
      centre_slice<T>(a, sM, sFlagC, sum, cnt);
      unsigned long long S;
      unsigned n;
      block_total(sum, cnt, sS, sNw, S, n);
      if (tid == 0) { a.cpart[2 * blockIdx.x] = S; a.cpart[2 * blockIdx.x + 1] = n; }
      grid_barrier(st, gen);  // sNA is identical in every CTA: uniform barrier
    }
    // ---- P5: E(P), s-law, trace
    if (tid == 0) {
      double Ecn = sState[2];
      unsigned nc = sNc;
      if (sNA > 0) {
        unsigned long long S = 0ull, n = 0ull;
        for (int b = 0; b < (int)gridDim.x; ++b) { S += __ldcg(a.cpart + 2 * b); n += __ldcg(a.cpart + 2 * b + 1); }
        nc = (unsigned)n;
        Ecn = fitness_c(S, nc, a.rho, N);
      }
      const double om = sState[0], v = sState[1];
      const double factor = __dadd_rn(a.beta, __dmul_rn(__dsub_rn(1.0, a.beta), Ecn));
      const double om1 = __dmul_rn(factor, om), v1 = __dmul_rn(factor, v);
      if (blockIdx.x == 0 && a.trace) {
        double* r = a.trace + (size_t)it * PFT_TRACE_DOUBLES;
        const int nA = sNA;
        r[0] = sState[3]; r[1] = (double)nA; r[2] = om; r[3] = v;
        for (int q = 0; q < 12; ++q) r[4 + q] = sP[q];
        r[16] = Ecn; r[17] = om1; r[18] = v1;
        r[19] = (double)((nA == 0 ? 1 : 0) | (sState[3] == 1.0 ? 2 : 0) | (N == 0 ? 4 : 0));
        r[20] = (double)nc; r[21] = (double)N; r[22] = 0.0; r[23] = 0.0;
      }
      sState[0] = om1; sState[1] = v1; sState[2] = Ecn; sNc = nc;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    for (int q = 0; q < 12; ++q) { a.T_out[q] = sP[q]; st->P[q] = sP[q]; }
    st->omega = sState[0]; st->v = sState[1]; st->Ec = sState[2]; st->nA = sNA; st->nc = sNc;
    st->iter = a.iters;
  }
}

// ------------------------------------------------------------------ host side
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

pft_status track_layout(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles, int32_t stride,
                        int nranks, TrackLayout* L) {
  (void)vol;
  if (nparticles < 1) return fail(PFT_ERR_INVALID_ARG, "number of particles/poses must be >= 1");
  if (stride < 1) return fail(PFT_ERR_INVALID_ARG, "stride must be >= 1");
  pft_status s = check_intrinsics(K);
  if (s != PFT_OK) return s;
  L->nr = (K->height + stride - 1) / stride;
  L->nc = (K->width + stride - 1) / stride;
  L->ntx = (L->nc + 7) / 8;
  L->nty = (L->nr + 3) / 4;
  L->npad = L->ntx * L->nty * 32;
  L->kloc = (nparticles + nranks - 1) / nranks;
  L->kfull = L->kloc * nranks;
  L->nblk_upd = (nparticles + 255) / 256;
  size_t off = 0;
  L->state_off = off; off = align_up(off + sizeof(TrackState), 256);
  L->pts_off = off; off = align_up(off + 3 * sizeof(double) * (size_t)L->npad, 256);
  L->acc_local_off = off; off = align_up(off + sizeof(PartRec) * (size_t)L->kloc, 256);
  if (nranks > 1) { L->acc_full_off = off; off = align_up(off + sizeof(PartRec) * (size_t)L->kfull, 256); }
  else L->acc_full_off = L->acc_local_off;
  L->part_off = off; off = align_up(off + 8 * sizeof(double) * (size_t)L->nblk_upd, 256);
  L->ptab_off = off; off = align_up(off + (12 * sizeof(double) + sizeof(int)) * (size_t)nparticles, 256);
  L->cpart_off = off; off = align_up(off + 2 * sizeof(unsigned long long) * 148 * 8, 256);
  L->work_off = off; off = align_up(off + sizeof(unsigned) * 1024, 256);
  L->total = off;
  return PFT_OK;
}

pft_status comm_allgather(pft_volume* vol, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st);

struct Launch {
  pft_volume* vol;
  TrackLayout L;
  char* ws;
  cudaStream_t st;
  TrackState* state() const { return (TrackState*)(ws + L.state_off); }
  Points pts() const {
    double* p = (double*)(ws + L.pts_off);
    return Points{p, p + L.npad, p + 2 * (size_t)L.npad, L.npad};
  }
};

static void launch_prologue(const Launch& c, const uint16_t* depth, const pft_intrinsics* K, int stride,
                            const double* T_init, double omega0, double v0, int conv) {
  TrackArgs ta{c.state(), T_init, omega0, v0, 0.0, 0.0, conv, (PartRec*)(c.ws + c.L.acc_local_off), c.L.kloc};
  int gi = (c.L.kloc + 255) / 256;
  PFT_LAUNCH(PFT_PROF_PREP, c.st, k_track_init<<<gi < 148 ? gi : 148, 256, 0, c.st>>>(ta));
  Points P = c.pts();
  BPArgs b{depth, K->fx, K->fy, K->cx, K->cy, K->depth_unit_m, c.vol->g.max_depth, K->width, K->height, stride,
           c.L.nr, c.L.nc, c.L.ntx, c.L.npad, (double*)P.x, (double*)P.y, (double*)P.z, &c.state()->Nvalid};
  PFT_LAUNCH(PFT_PROF_PREP, c.st, k_backproject<<<(c.L.npad + 255) / 256, 256, 0, c.st>>>(b));
}

template <typename T>
static void launch_centre(const Launch& c, int initial, double beta, double rho, double* trace, double* T_out) {
  CentreArgs ca{c.vol->base + c.vol->L.v_off, (const unsigned long long*)(c.vol->base + c.vol->L.m_off), c.vol->g, c.pts(), c.state(), initial, beta, rho, trace, T_out};
  int grid = (c.L.npad + kThreads * kCentrePPT - 1) / (kThreads * kCentrePPT);
  PFT_LAUNCH(PFT_PROF_CENTRE, c.st, k_centre<T><<<grid, kThreads, 0, c.st>>>(ca));
}

template <typename T>
static void launch_eval(const Launch& c, int mode, const float* pst, int k_begin, int k_count, int conv,
                        const double* poses, PartRec* acc) {
  if (k_count <= 0) return;
  EvalArgs ea{c.vol->base + c.vol->L.r_off, (const unsigned long long*)(c.vol->base + c.vol->L.m_off), c.vol->g, c.pts(), mode, pst, k_begin, k_count, c.state(), conv, poses, acc};
  dim3 grid((c.L.npad + kThreads * kPPT - 1) / (kThreads * kPPT), (k_count + kPC - 1) / kPC);
  static const int ppt = [] {  // tuning knob for experiments: PFT_EVAL_PPT=2|4
    const char* e = getenv("PFT_EVAL_PPT");
    return e && atoi(e) == 2 ? 2 : kPPT;
  }();
  if (ppt == 2) {
    grid.x = (c.L.npad + kThreads * 2 - 1) / (kThreads * 2);
    PFT_LAUNCH(PFT_PROF_EVAL, c.st, k_particle_eval<T, 2><<<grid, kThreads, 0, c.st>>>(ea));
  } else {
    PFT_LAUNCH(PFT_PROF_EVAL, c.st, k_particle_eval<T, kPPT><<<grid, kThreads, 0, c.st>>>(ea));
  }
}

// Persistent single-launch tracker (G = 1): cooperative launch, all CTAs co-resident.
template <typename T>
static pft_status track_persistent(Launch& c, const uint16_t* depth, const pft_intrinsics* K, const double* T_init,
                                   const float* pst, int Kp, const pft_track_params* prm, double* T_out, double* E,
                                   int32_t* n_out, double* trace) {
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_track_persistent<T>, kThreads, 0);
    grid = per_sm * sms;
    if (grid > 148 * 8) grid = 148 * 8;
    if (grid < 1) return fail(PFT_ERR_CUDA, "persistent tracker does not fit on the device");
  }
  cudaMemsetAsync(c.state(), 0, sizeof(TrackState), c.st);
  cudaMemsetAsync(c.ws + c.L.work_off, 0, sizeof(unsigned) * (size_t)prm->iters, c.st);
  Points P = c.pts();
  PArgs pa;
  pa.R = c.vol->base + c.vol->L.r_off;
  pa.V = c.vol->base + c.vol->L.v_off;
  pa.mask = (const unsigned long long*)(c.vol->base + c.vol->L.m_off);
  pa.g = c.vol->g;
  pa.bp = BPArgs{depth, K->fx, K->fy, K->cx, K->cy, K->depth_unit_m, c.vol->g.max_depth, K->width, K->height,
                 prm->stride, c.L.nr, c.L.nc, c.L.ntx, c.L.npad, (double*)P.x, (double*)P.y, (double*)P.z,
                 &c.state()->Nvalid};
  pa.pts = P;
  pa.pst = pst;
  pa.K = Kp; pa.conv = prm->delta_conv; pa.iters = prm->iters; pa.nblk_upd = c.L.nblk_upd;
  pa.ngroups = (c.L.npad + 32 * kItemTiles - 1) / (32 * kItemTiles);
  pa.nchunks = (Kp + kItemParticles - 1) / kItemParticles;
  static const int sched = [] { const char* e = getenv("PFT_EVAL_SCHED"); return e ? atoi(e) : 0; }();
  pa.sched = sched;
  pa.beta = prm->beta; pa.rho = prm->min_inband_frac; pa.omega0 = prm->omega0_deg; pa.v0 = prm->v0_cm;
  pa.T_init = T_init;
  pa.st = c.state();
  pa.acc = (PartRec*)(c.ws + c.L.acc_local_off);
  pa.E_out = E; pa.n_out = n_out; pa.trace = trace; pa.T_out = T_out;
  pa.ptab = (double*)(c.ws + c.L.ptab_off);
  pa.pflag = (int*)(c.ws + c.L.ptab_off + 12 * sizeof(double) * (size_t)Kp);
  pa.upart = (double*)(c.ws + c.L.part_off);
  pa.cpart = (unsigned long long*)(c.ws + c.L.cpart_off);
  pa.work = (unsigned*)(c.ws + c.L.work_off);
  void* args[] = {&pa};
  cudaError_t e = cudaSuccess;
  PFT_LAUNCH(PFT_PROF_TRACK, c.st,
             e = cudaLaunchCooperativeKernel((const void*)k_track_persistent<T>, dim3(grid), dim3(kThreads), args, 0, c.st));
  if (e != cudaSuccess) return fail(PFT_ERR_CUDA, "persistent tracker launch: %s", cudaGetErrorString(e));
  return cuda_check("track (persistent)");
}

static bool use_persistent() {
  static const bool on = [] {
    const char* e = getenv("PFT_TRACK_PERSISTENT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T>
static pft_status track_run(Launch& c, const uint16_t* depth, const pft_intrinsics* K, const double* T_init,
                            const float* pst, int Kp, const pft_track_params* prm, double* T_out, double* E,
                            int32_t* n_out, double* trace) {
  const int G = c.vol->nranks, r = c.vol->rank;
  if (G == 1 && use_persistent() && prm->iters <= 1024)
    return track_persistent<T>(c, depth, K, T_init, pst, Kp, prm, T_out, E, n_out, trace);
  const int kloc = c.L.kloc;
  const int k_begin = r * kloc;
  const int k_count = max(0, min(Kp, k_begin + kloc) - k_begin);
  PartRec* local = (PartRec*)(c.ws + c.L.acc_local_off);
  PartRec* full = (PartRec*)(c.ws + c.L.acc_full_off);
  launch_prologue(c, depth, K, prm->stride, T_init, prm->omega0_deg, prm->v0_cm, prm->delta_conv);
  launch_centre<T>(c, 1, prm->beta, prm->min_inband_frac, nullptr, nullptr);
  for (int it = 0; it < prm->iters; ++it) {
    launch_eval<T>(c, 0, pst, k_begin, k_count, prm->delta_conv, nullptr, local);
    if (G > 1) {
      pft_status s = comm_allgather(c.vol, local, full, sizeof(PartRec) * (size_t)kloc, c.st);
      if (s != PFT_OK) return s;
    }
    UpdArgs ua{c.state(), full, local, Kp, k_begin, kloc, pst, prm->delta_conv, prm->min_inband_frac, E, n_out,
               (double*)(c.ws + c.L.part_off)};
    PFT_LAUNCH(PFT_PROF_UPDATE, c.st, k_update<<<c.L.nblk_upd, 256, 0, c.st>>>(ua));
    launch_centre<T>(c, 0, prm->beta, prm->min_inband_frac, trace, it == prm->iters - 1 ? T_out : nullptr);
  }
  return cuda_check("track");
}

// per-pose results of an eval_poses call
__global__ void k_finish_poses(const PartRec* acc, int M, const TrackState* st, double rho, double* E, int* n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  const PartRec r = acc[k];
  E[k] = fitness_of(r.S, r.n, rho, st->Nvalid);
  n[k] = (int)r.n;
}

static pft_status check_params(const pft_track_params* p) {
  if (!p) return fail(PFT_ERR_INVALID_ARG, "params is NULL");
  if (!(p->beta >= 0.0 && p->beta < 1.0)) return fail(PFT_ERR_INVALID_ARG, "beta must be in [0,1) (SPEC.md:313)");
  if (p->iters < 1) return fail(PFT_ERR_INVALID_ARG, "iters must be >= 1");
  if (!(p->omega0_deg >= 0.0 && p->omega0_deg <= 100.0)) return fail(PFT_ERR_INVALID_ARG, "omega0_deg must be in [0,100]");
  if (!(p->v0_cm >= 0.0 && p->v0_cm < 1e6)) return fail(PFT_ERR_INVALID_ARG, "v0_cm must be in [0,1e6)");
  if (p->stride < 1) return fail(PFT_ERR_INVALID_ARG, "stride must be >= 1");
  if (!(p->min_inband_frac >= 0.0 && p->min_inband_frac <= 1.0)) return fail(PFT_ERR_INVALID_ARG, "min_inband_frac must be in [0,1]");
  if (p->delta_conv != PFT_DELTA_CAMERA_CENTRED && p->delta_conv != PFT_DELTA_WORLD_LITERAL)
    return fail(PFT_ERR_INVALID_ARG, "bad delta_conv");
  if (p->update_rule != PFT_UPDATE_MEAN) return fail(PFT_ERR_UNSUPPORTED, "only PFT_UPDATE_MEAN is implemented");
  return PFT_OK;
}

}  // namespace pft

using namespace pft;

extern "C" {

pft_status pft_track_workspace_bytes(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles,
                                     const pft_track_params* prm, size_t* bytes_out) {
  if (!vol || !bytes_out || !prm) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  TrackLayout L;
  pft_status s = track_layout(vol, K, nparticles, prm->stride, vol->nranks, &L);
  if (s != PFT_OK) return s;
  *bytes_out = L.total;
  return PFT_OK;
}

pft_status pft_track(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K, const double* dev_T_init,
                     const float* dev_pst, int32_t nparticles, const pft_track_params* prm, void* dev_ws,
                     size_t ws_bytes, double* dev_T_out, double* dev_E, int32_t* dev_inband, double* dev_trace,
                     void* stream) {
  if (!vol || !dev_depth || !dev_T_init || !dev_pst || !dev_ws || !dev_T_out || !dev_E || !dev_inband)
    return fail(PFT_ERR_INVALID_ARG, "NULL required argument");
  pft_status s = check_params(prm);
  if (s != PFT_OK) return s;
  Launch c;
  c.vol = vol;
  c.ws = (char*)dev_ws;
  c.st = (cudaStream_t)stream;
  s = track_layout(vol, K, nparticles, prm->stride, vol->nranks, &c.L);
  if (s != PFT_OK) return s;
  if (ws_bytes < c.L.total) return fail(PFT_ERR_BUFFER_TOO_SMALL, "workspace %zu B < required %zu B", ws_bytes, c.L.total);
  if (((uintptr_t)dev_ws) % 256) return fail(PFT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (vol->esize == 4)
    return track_run<float>(c, dev_depth, K, dev_T_init, dev_pst, nparticles, prm, dev_T_out, dev_E, dev_inband, dev_trace);
  return track_run<__half>(c, dev_depth, K, dev_T_init, dev_pst, nparticles, prm, dev_T_out, dev_E, dev_inband, dev_trace);
}

pft_status pft_eval_poses(const pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K,
                          const pft_track_params* prm, const double* dev_poses, int32_t M, void* dev_ws,
                          size_t ws_bytes, double* dev_E, int32_t* dev_inband, void* stream) {
  if (!vol || !dev_depth || !prm || !dev_poses || !dev_ws || !dev_E || !dev_inband)
    return fail(PFT_ERR_INVALID_ARG, "NULL required argument");
  if (prm->stride < 1) return fail(PFT_ERR_INVALID_ARG, "stride must be >= 1");
  if (!(prm->min_inband_frac >= 0.0 && prm->min_inband_frac <= 1.0)) return fail(PFT_ERR_INVALID_ARG, "min_inband_frac must be in [0,1]");
  Launch c;
  c.vol = (pft_volume*)vol;
  c.ws = (char*)dev_ws;
  c.st = (cudaStream_t)stream;
  // eval_poses is rank-local: lay the workspace out for one rank
  pft_status s = track_layout(vol, K, M, prm->stride, 1, &c.L);
  if (s != PFT_OK) return s;
  if (ws_bytes < c.L.total) return fail(PFT_ERR_BUFFER_TOO_SMALL, "workspace %zu B < required %zu B", ws_bytes, c.L.total);
  if (((uintptr_t)dev_ws) % 256) return fail(PFT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  // (the state's pose is initialised from pose 0; eval_poses never reads it)
  launch_prologue(c, dev_depth, K, prm->stride, dev_poses, 0.0, 0.0, 0);
  PartRec* acc = (PartRec*)(c.ws + c.L.acc_local_off);
  if (vol->esize == 4) launch_eval<float>(c, 1, nullptr, 0, M, 0, dev_poses, acc);
  else launch_eval<__half>(c, 1, nullptr, 0, M, 0, dev_poses, acc);
  PFT_LAUNCH(PFT_PROF_UPDATE, c.st, k_finish_poses<<<(M + 255) / 256, 256, 0, c.st>>>(acc, M, c.state(), prm->min_inband_frac, dev_E, dev_inband));
  return cuda_check("eval_poses");
}

pft_status pft_track_info(const void* dev_ws, int32_t* npoints_out, void* stream) {
  if (!dev_ws || !npoints_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  int n = 0;
  const TrackState* s = (const TrackState*)dev_ws;  // state is at offset 0 of every layout
  if (cudaMemcpyAsync(&n, &s->Nvalid, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check("track_info");
  *npoints_out = n;
  return PFT_OK;
}

}  // extern "C"
