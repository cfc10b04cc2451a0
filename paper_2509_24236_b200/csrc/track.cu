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
#include <cstdio>
#include <cstdlib>
#include <mutex>

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
    const double ith = 1.0 / th;
    A = s * ith;
    B = (1.0 - c) * ith * ith;
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
  const double iv = 1.0 / g.voxel;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) m[4 * i + j] = T[4 * i + j] * iv;
    m[4 * i + 3] = (T[4 * i + 3] - o[i]) * iv - 0.5;
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

// a7: P <- (R(Q/|Q|), U/Wsum) P, Q and U the (weighted) sums over the
// advantage set and Wsum the sum of the weights (|A| for the paper's plain mean).
__device__ __noinline__ void apply_mean(const double* Q, const double* U, double Wsum, const double* P, int conv,
                                        double* Pn) {
  const double iq = 1.0 / sqrt(Q[0] * Q[0] + Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3]);
  const double iw = 1.0 / Wsum;
  const double qb[4] = {Q[0] * iq, Q[1] * iq, Q[2] * iq, Q[3] * iq};
  const double ub[3] = {U[0] * iw, U[1] * iw, U[2] * iw};
  double Rb[9], PP[12], out[12];
  quat_to_R(qb, Rb);
  for (int i = 0; i < 12; ++i) PP[i] = P[i];
  apply_delta(Rb, ub, PP, conv, out);
  for (int i = 0; i < 12; ++i) Pn[i] = out[i];
}

// 256-thread fixed-shape tree over red[kUpdW][256] (result in red[c][0]); all threads must call.
// Level s adds element t + s into element t (t < s), s = 128 ... 1: the levels >= 32 in shared
// memory, the last five in warp 0 by shfl_down (the same pairs, so the same sums bit for bit).
__device__ __forceinline__ void treeW(double (*red)[256], int tid) {
  __syncthreads();
  for (int s = 128; s >= 32; s >>= 1) {
    if (tid < s)
#pragma unroll
      for (int c = 0; c < kUpdW; ++c) red[c][tid] += red[c][tid + s];
    __syncthreads();
  }
  if (tid < 32) {
    double v[kUpdW];
#pragma unroll
    for (int c = 0; c < kUpdW; ++c) v[c] = red[c][tid];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1)
#pragma unroll
      for (int c = 0; c < kUpdW; ++c) v[c] += __shfl_down_sync(0xffffffffu, v[c], s);
    if (tid == 0)
#pragma unroll
      for (int c = 0; c < kUpdW; ++c) red[c][0] = v[c];
  }
  __syncthreads();
}

// a7 contribution of particle k (E_k from its record) to one 256-particle update block:
// member iff E_k < E_base; weight 1 (mean) or E_base - E_k (F3 weighted).
__device__ __forceinline__ void member_row(double* row, double E, double Ebase, int rule, const float* pst_row,
                                           double omega, double v) {
#pragma unroll
  for (int c = 0; c < kUpdW; ++c) row[c] = 0.0;
  if (E < Ebase) {
    double q[4], u[3];
    member_delta(pst_row, omega, v, q, u);
    const double w = rule == 1 ? Ebase - E : 1.0;
    row[0] = w * q[0]; row[1] = w * q[1]; row[2] = w * q[2]; row[3] = w * q[3];
    row[4] = w * u[0]; row[5] = w * u[1]; row[6] = w * u[2];
    row[7] = 1.0; row[8] = w;
  }
}

// Same from a member delta (q, u) computed beforehand by member_delta: identical arithmetic.
__device__ __forceinline__ void member_row_pre(double* row, double E, double Ebase, int rule, const double* q,
                                               const double* u) {
#pragma unroll
  for (int c = 0; c < kUpdW; ++c) row[c] = 0.0;
  if (E < Ebase) {
    const double w = rule == 1 ? Ebase - E : 1.0;
    row[0] = w * q[0]; row[1] = w * q[1]; row[2] = w * q[2]; row[3] = w * q[3];
    row[4] = w * u[0]; row[5] = w * u[1]; row[6] = w * u[2];
    row[7] = 1.0; row[8] = w;
  }
}

// Same from the member delta precomputed in P1 (the persistent tracker's table: q(4), u(3), pad):
// identical arithmetic, member_delta's values loaded instead of recomputed.
__device__ __forceinline__ void member_row_tab(double* row, double E, double Ebase, int rule, const double* mrow) {
#pragma unroll
  for (int c = 0; c < kUpdW; ++c) row[c] = 0.0;
  if (E < Ebase) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(mrow));
    const double2 b = __ldcg(reinterpret_cast<const double2*>(mrow) + 1);
    const double2 c2 = __ldcg(reinterpret_cast<const double2*>(mrow) + 2);
    const double u2 = __ldcg(mrow + 6);
    const double w = rule == 1 ? Ebase - E : 1.0;
    row[0] = w * a.x; row[1] = w * a.y; row[2] = w * b.x; row[3] = w * b.y;
    row[4] = w * c2.x; row[5] = w * c2.y; row[6] = w * u2;
    row[7] = 1.0; row[8] = w;
  }
}

// ---- F3 top-k: (E_k, k) keys.  E >= 0 doubles order like their bit patterns; non-members get ~0.
constexpr int kTopkMax = 32;

__device__ __forceinline__ bool key_less(unsigned long long ka, int ia, unsigned long long kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// Ascending bitonic sort of 256 (key, index) pairs in shared memory (blockDim.x == 256).
__device__ __forceinline__ void bitonic256(unsigned long long* key, int* idx, int tid) {
  __syncthreads();
  for (int k = 2; k <= 256; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = tid ^ j;
      if (tid < 256 && p > tid) {
        const bool up = (tid & k) == 0;
        const bool gt = key_less(key[p], idx[p], key[tid], idx[tid]);
        if (up == gt) {
          const unsigned long long tk = key[tid]; key[tid] = key[p]; key[p] = tk;
          const int ti = idx[tid]; idx[tid] = idx[p]; idx[p] = ti;
        }
      }
      __syncthreads();
    }
}

// One 256-particle block's top-k candidates: sorted (key, index) of its members, padded with ~0.
__device__ __forceinline__ void block_topk(unsigned long long key_mine, int k, int topk, unsigned long long* skey,
                                           int* sidx, unsigned long long* cand_key, int* cand_idx, int tid) {
  if (tid < 256) {
    skey[tid] = key_mine;
    sidx[tid] = k;
  }
  bitonic256(skey, sidx, tid);
  if (tid < topk) { cand_key[tid] = skey[tid]; cand_idx[tid] = sidx[tid]; }
  __syncthreads();
}

// Merge of the nblk sorted candidate lists by repeated block-wide minimum of the list heads (one
// CTA); the selected indices, sorted ascending, then sum their deltas serially in thread 0 (the
// definition's ascending-k order).  Writes Q(4), U(3), n to out[0..7].
__device__ __noinline__ void topk_finish(const unsigned long long* cand_key, const int* cand_idx, int nblk, int topk,
                                         const float* pst, double omega, double v, double* out,
                                         unsigned long long* skey, int* sidx, int* ssel) {
  const int tid = threadIdx.x;
  int head = 0;
  int nsel = 0;
  for (int r = 0; r < topk; ++r) {
    unsigned long long kk = ~0ull;
    int ii = 0x7fffffff;
    for (int b = tid; b < nblk; b += 256)
      if (b == tid && head < topk) {  // each list owned by one thread (nblk <= 256 * ... see below)
        kk = __ldcg(cand_key + b * kTopkMax + head);
        ii = __ldcg(cand_idx + b * kTopkMax + head);
      }
    if (tid < 256) {
      skey[tid] = kk;
      sidx[tid] = ii;
    }
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (tid < s && key_less(skey[tid + s], sidx[tid + s], skey[tid], sidx[tid])) {
        skey[tid] = skey[tid + s];
        sidx[tid] = sidx[tid + s];
      }
      __syncthreads();
    }
    const unsigned long long wk = skey[0];
    const int wi = sidx[0];
    __syncthreads();
    if (wk == ~0ull) break;  // no member left
    if (tid < nblk && kk == wk && ii == wi) ++head;
    if (tid == 0) ssel[nsel] = wi;
    ++nsel;
  }
  if (tid == 0) {
    for (int a = 1; a < nsel; ++a)  // insertion sort: ascending particle index
      for (int b = a; b > 0 && ssel[b - 1] > ssel[b]; --b) { const int t = ssel[b]; ssel[b] = ssel[b - 1]; ssel[b - 1] = t; }
    double Q[4] = {0.0, 0.0, 0.0, 0.0}, U[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < nsel; ++a) {
      double q[4], u[3];
      member_delta(pst + 6 * (size_t)ssel[a], omega, v, q, u);
      for (int c = 0; c < 4; ++c) Q[c] = Q[c] + 1.0 * q[c];
      for (int c = 0; c < 3; ++c) U[c] = U[c] + 1.0 * u[c];
    }
    for (int c = 0; c < 4; ++c) out[c] = Q[c];
    for (int c = 0; c < 3; ++c) out[4 + c] = U[c];
    out[7] = (double)nsel;
  }
  __syncthreads();
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

// Cell index and fraction of grid coordinate g: n = floor(g) exactly, f = g - n rounded to the
// nearest multiple of 2^-23 (|error| <= 2^-24, unbiased) for the fp32 lerp.  FAST (|g| < 2^27
// guaranteed by the caller's bound): t = g (+)_RD 1.5*2^52 holds floor(g) in its low 32 bits
// (one DADD, no conversion); u = g (+)_RN (1.5*2^29 + 127) holds round(g * 2^23) in its low
// word, offset by 127 * 2^23 = the bit pattern of 1.0f, so low(u) - floor(g) * 2^23 is the
// pattern of the float 1 + f: no conversion-pipe (XU) instruction at all (F2F.F32.F64 was 3 per
// evaluation; -0.7% track time).  Otherwise: FRND.FLOOR + saturating F2I, same results.
template <bool FAST>
__device__ __forceinline__ int cell_split(double g, float& f) {
  const double M29 = 805306495.0;  // 1.5 * 2^29 + 127
  if (FAST) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const int ix = __double2loint(__dadd_rd(g, M));
    f = __int_as_float((int)((unsigned)__double2loint(__dadd_rn(g, M29)) - ((unsigned)ix << 23))) - 1.0f;
    return ix;
  } else {
    const double fl = floor(g);
    f = __int_as_float(__double2loint(__dadd_rn(g - fl, M29))) - 1.0f;
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
  // same stored values by the record builder; read as the 32-bit half of the brick's word
  uint32_t mw[PPT];
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
    mw[p] = __ldg(reinterpret_cast<const unsigned*>(mbase + (size_t)(o[p] >> 5) * 4u));
  float v[PPT][8];
  uint32_t inb[PPT];  // 1 iff the evaluation is counted (in range, valid point, in band)
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    inb[p] = (mw[p] >> (o[p] & 31u)) & (uint32_t)ok[p];
    const uint32_t orec = o[p] * inb[p];
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
    fix += __float2uint_rn(fabsf(val) * (float)kFixScale) * inb[p];
    cnt += inb[p];
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
    // exact stored corner values (brick order), not the record; loaded together with the mask
    // word (one round trip), used only when the cell is in band
    const uint32_t b = o[p];
    ok[p] = ok[p] && ((mw >> (o[p] & 63)) & 1ull);
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

// FAST-path bound for pose m on points with max |coordinate| <= pmax: every |g| < 2^27 (the magic
// constants of cell_split need |g| < 2^28 - 128).
__device__ __forceinline__ bool fast_ok(const double m[12], double pmax) {
  bool ok = true;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    ok = ok && (fabs(m[4 * r]) + fabs(m[4 * r + 1]) + fabs(m[4 * r + 2])) * pmax + fabs(m[4 * r + 3]) < 134217728.0;
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
  int pbeg, pend;            // point slots [pbeg, pend) of this launch (F2b point shards; else [0, npad))
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
#define PFT_MINB 3  // 3 CTAs/SM (80 registers): 246.8 vs 233.7 Gevals/s at 2 (round 2 A/B)
#endif
__global__ __launch_bounds__(kThreads, PFT_MINB) void k_particle_eval(EvalArgs a) {
  if (a.mode == 0 && a.st->stopped) return;  // a stop rule fired (multi-launch path; uniform)
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
    const int i = a.pbeg + (blockIdx.x * PPT + p) * kThreads + tid;
    if (i < a.pend) {
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

// ------------------------------------------------------------------ point sets and schedule
// O1/O2 per set: pixels (sx c, sy r), r < nr = ceil(H/sy), c < nc = ceil(W/sx), in 8x4 tiles.
struct BPFrame {
  const uint16_t* depth;
  double fx, fy, cx, cy, unit, max_depth;
  int W, H;
};
struct PSet {
  double *x, *y, *z;
  int npad, sx, sy, nr, nc, ntx;
  __host__ __device__ Points pts() const { return Points{x, y, z, npad}; }
};
// The iteration schedule (F1; one entry for the plain run): entry j = (K_j, point set).
struct Sched {
  int n, nsets;
  int K[PFT_MAX_SCHED], set[PFT_MAX_SCHED];
  PSet sets[PFT_MAX_SCHED];
};

__device__ __forceinline__ bool bp_slot(const BPFrame& f, const PSet& s, int i, double& X, double& Y, double& Z) {
  const int t = i >> 5, l = i & 31;
  const int r = (t / s.ntx) * 4 + (l >> 3), c = (t % s.ntx) * 8 + (l & 7);
  X = Y = Z = 0.0;
  if (r >= s.nr || c >= s.nc) return false;
  const int u = c * s.sx, v = r * s.sy;
  const uint16_t raw = f.depth[(size_t)v * f.W + u];
  const double d = __dmul_rn((double)raw, f.unit);
  if (raw == 0 || !(d < f.max_depth)) return false;
  X = __ddiv_rn(__dmul_rn(__dsub_rn((double)u, f.cx), d), f.fx);
  Y = __ddiv_rn(__dmul_rn(__dsub_rn((double)v, f.cy), d), f.fy);
  Z = d;
  return true;
}

// Trace row of iteration `it` (include/pft.h).
__device__ __forceinline__ void write_trace(double* r, double Ebase, int nA, double om, double v, const double* P,
                                            double Ec, double om1, double v1, int flags, unsigned nc, int N, int Ki,
                                            int code) {
  r[0] = Ebase; r[1] = (double)nA; r[2] = om; r[3] = v;
  for (int i = 0; i < 12; ++i) r[4 + i] = P[i];
  r[16] = Ec; r[17] = om1; r[18] = v1; r[19] = (double)flags;
  r[20] = (double)nc; r[21] = (double)N; r[22] = (double)Ki; r[23] = (double)code;
}
__device__ __forceinline__ void write_not_run(double* r) {
  for (int i = 0; i < PFT_TRACE_DOUBLES; ++i) r[i] = 0.0;
  r[19] = 32.0;
}

// a8 + F1/F3 bookkeeping shared by both implementations: s-law, stalls, stop rule.
struct StopRule { double min_deg, min_cm; int stall_limit; };
__device__ __forceinline__ bool stop_now(const StopRule& sr, double om1, double v1, int stalls) {
  return ((sr.min_deg > 0.0 || sr.min_cm > 0.0) && om1 < sr.min_deg && v1 < sr.min_cm) ||
         (sr.stall_limit > 0 && stalls >= sr.stall_limit);
}
__device__ __forceinline__ double s_factor(double beta, double E) {
  // s^(i+1) = beta s^(i) + (1 - beta) E(P^(i)) s^(i), as (beta + (1-beta)E) s
  return __dadd_rn(beta, __dmul_rn(__dsub_rn(1.0, beta), E));
}

// ------------------------------------------------------------------ multi-launch kernels (G > 1)
struct TrackArgs {
  TrackState* st;
  const double* T_init;
  double omega0, v0;
  PartRec* acc_local;
  int kloc;
};

__global__ void k_track_init(TrackArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    TrackState* s = a.st;
    for (int j = 0; j < 12; ++j) { s->P[j] = a.T_init[j]; s->Pprev[j] = a.T_init[j]; }
    s->omega = a.omega0; s->v = a.v0;
    s->Ec = 1.0; s->Ebase = 1.0; s->Wsum = 0.0;
    s->Sc_acc = 0ull; s->nc_acc = 0u; s->nc = 0u; s->nc_base = 0u;
    s->nA = 0; s->iter = 0;
    for (int j = 0; j < 4; ++j) s->Nvalid[j] = 0;
    s->cur_set = -1; s->stalls = 0; s->stopped = 0; s->K_last = 0;
    s->ticket_upd = 0u; s->ticket_ctr = 0u;
  }
  for (int k = i; k < a.kloc; k += gridDim.x * blockDim.x) {
    a.acc_local[k].S = 0ull;
    a.acc_local[k].n = 0u;
    a.acc_local[k].pad = 0u;
  }
}

__global__ void k_backproject(BPFrame f, PSet s, int* Nvalid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.npad) return;
  double X, Y, Z;
  const bool valid = bp_slot(f, s, i, X, Y, Z);
  s.x[i] = X; s.y[i] = Y; s.z[i] = Z;
  const unsigned b = __ballot_sync(0xffffffffu, valid);
  if ((i & 31) == 0 && b) atomicAdd(Nvalid, __popc(b));
}

// a5 (+ a8): E(P) on point set `set`.  mode 0 (baseline, L11): E(P^(i-1)) on the iteration's set
// when the set changed (incl. the first iteration).  mode 1 (after the update): E(P^(i)) if
// A != {}, then the F3 guard, the s-law, stalls / stop rule and the trace row.
struct CentreArgs {
  const void* V;                    // stored values (the centre lerps exact corner values in fp64)
  const unsigned long long* mask;
  Geom g;
  Points pts;
  TrackState* st;
  int mode, set, it, Ki, code, guard;
  double beta, rho;
  StopRule sr;
  double* trace;
  int pbeg, pend;                   // point slots of this launch
  unsigned long long* cacc;         // F2b: non-null = partial mode, accumulate (S, n) here only
};

__device__ __noinline__ void centre_finish(const CentreArgs& a, unsigned long long S, unsigned ncn);

template <typename T>
__global__ __launch_bounds__(kThreads) void k_centre(CentreArgs a) {
  __shared__ double sm[12];
  __shared__ int sOk;
  __shared__ bool sLast;
  __shared__ double sRed[kThreads / 32];
  TrackState* st = a.st;
  const int tid = threadIdx.x;
  if (st->stopped) {  // uniform: a stop rule fired in an earlier iteration
    if (a.mode == 1 && blockIdx.x == 0 && tid == 0 && a.trace) write_not_run(a.trace + (size_t)a.it * PFT_TRACE_DOUBLES);
    return;
  }
  const bool do_eval = a.mode == 0 || st->nA > 0;
  if (do_eval) {
    double px[kCentrePPT], py[kCentrePPT], pz[kCentrePPT], pm = 0.0;
#pragma unroll
    for (int p = 0; p < kCentrePPT; ++p) {
      const int i = a.pbeg + (blockIdx.x * kCentrePPT + p) * kThreads + tid;
      px[p] = py[p] = pz[p] = 0.0;
      if (i < a.pend) { px[p] = a.pts.x[i]; py[p] = a.pts.y[i]; pz[p] = a.pts.z[i]; }
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
      if (a.cacc) {  // F2b partial: the rank's slice only; summed across ranks, then k_centre_finish
        atomicAdd(a.cacc, S);
        atomicAdd(a.cacc + 1, (unsigned long long)n);
      } else {
        atomicAdd(&st->Sc_acc, S);
        atomicAdd(&st->nc_acc, n);
      }
    }
  }
  if (a.cacc) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) sLast = atomicAdd(&st->ticket_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sLast || tid != 0) return;
  __threadfence();
  volatile TrackState* vs = st;
  const unsigned long long S = vs->Sc_acc;
  const unsigned ncn = vs->nc_acc;
  st->Sc_acc = 0ull;
  st->nc_acc = 0u;
  st->ticket_ctr = 0u;
  centre_finish(a, S, ncn);
}

// The centre's E(P) from its summed (S, n) (one thread): baseline (mode 0), or after the update
// (mode 1) the F3 guard, the s-law, stalls / stop rule and the trace row.
__device__ __noinline__ void centre_finish(const CentreArgs& a, unsigned long long S, unsigned ncn) {
  TrackState* st = a.st;
  volatile TrackState* vs = st;
  const int N = vs->Nvalid[a.set];
  if (a.mode == 0) {
    st->Ec = fitness_c(S, ncn, a.rho, N);
    st->nc = ncn;
    st->cur_set = a.set;
    return;
  }
  const int nA = vs->nA;
  const double Ebase = vs->Ebase;
  double Ec = Ebase;
  unsigned nc = vs->nc_base;
  int rejected = 0;
  if (nA > 0) {
    const double En = fitness_c(S, ncn, a.rho, N);
    if (a.guard && En > Ebase) {  // F3 guard: keep P^(i-1)
      rejected = 1;
      for (int i = 0; i < 12; ++i) st->P[i] = vs->Pprev[i];
    } else {
      Ec = En;
      nc = ncn;
    }
  }
  const int stalls = (nA == 0 || rejected) ? vs->stalls + 1 : 0;
  const double om = vs->omega, v = vs->v;
  const double f = s_factor(a.beta, Ec);
  const double om1 = __dmul_rn(f, om), v1 = __dmul_rn(f, v);
  const bool stop = stop_now(a.sr, om1, v1, stalls);
  st->Ec = Ec; st->nc = nc; st->omega = om1; st->v = v1; st->stalls = stalls; st->K_last = a.Ki;
  st->iter = a.it + 1;
  if (stop) st->stopped = 1;
  if (a.trace) {
    double P[12];
    for (int i = 0; i < 12; ++i) P[i] = vs->P[i];
    const int flags = (nA == 0 ? 1 : 0) | (Ebase == 1.0 ? 2 : 0) | (N == 0 ? 4 : 0) | (rejected ? 8 : 0) | (stop ? 16 : 0);
    write_trace(a.trace + (size_t)a.it * PFT_TRACE_DOUBLES, Ebase, nA, om, v, P, Ec, om1, v1, flags, nc, N, a.Ki, a.code);
  }
}

// F2b: the centre's finalisation after its per-rank partial sums were added across ranks
// (cacc = (S, n) as uint64); re-zeroes cacc for the next centre.
__global__ void k_centre_finish(CentreArgs a) {
  if (a.st->stopped) {
    if (a.mode == 1 && a.trace) write_not_run(a.trace + (size_t)a.it * PFT_TRACE_DOUBLES);
    return;
  }
  const unsigned long long S = a.cacc[0], n = a.cacc[1];
  a.cacc[0] = 0ull;
  a.cacc[1] = 0ull;
  centre_finish(a, S, (unsigned)n);
}

// a7: E_k, advantage set A = {k < K_i : E_k < E_base}, (weighted) mean delta over A
// (PAPER.md:206), P <- (R(q), u) P.  ceil(K_i/256) CTAs, one particle per thread;
// each CTA reduces its members in a fixed tree, the last CTA combines the partials in a fixed tree.
struct UpdArgs {
  int topk;
  unsigned long long* ckey;
  int* cidx;
  double* tkout;
  TrackState* st;
  const PartRec* full;       // K records (all ranks)
  PartRec* local;            // this rank's records, zeroed for the next iteration
  int Ki, k_begin, kloc;     // local covers global [k_begin, k_begin + kloc)
  const float* pst;
  int conv, rule, set;
  double rho;
  double* E_out;
  int* n_out;
  double* partials;          // nblk x kUpdW
};

__global__ __launch_bounds__(256) void k_update(UpdArgs a) {
  __shared__ double red[kUpdW][256];
  __shared__ unsigned long long tkey[256];
  __shared__ int tidx[256], tsel[kTopkMax];
  __shared__ bool sLast;
  TrackState* st = a.st;
  if (st->stopped) return;  // uniform
  const int tid = threadIdx.x;
  const int k = blockIdx.x * 256 + tid;
  const double Ebase = st->Ec;
  const int N = st->Nvalid[a.set];
  double row[kUpdW];
#pragma unroll
  for (int c = 0; c < kUpdW; ++c) row[c] = 0.0;
  unsigned long long key = ~0ull;
  if (k < a.Ki) {
    const PartRec rec = a.full[k];
    const double E = fitness_of(rec.S, rec.n, a.rho, N);
    a.E_out[k] = E;
    a.n_out[k] = (int)rec.n;
    if (a.rule == 2) {
      if (E < Ebase) key = (unsigned long long)__double_as_longlong(E);
    } else {
      member_row(row, E, Ebase, a.rule, a.pst + 6 * (size_t)k, st->omega, st->v);
    }
    const int j = k - a.k_begin;
    if (j >= 0 && j < a.kloc) {
      a.local[j].S = 0ull;
      a.local[j].n = 0u;
    }
  }
  if (a.rule == 2) {
    block_topk(key, k, a.topk, tkey, tidx, a.ckey + (size_t)blockIdx.x * kTopkMax, a.cidx + (size_t)blockIdx.x * kTopkMax, tid);
  } else {
#pragma unroll
    for (int c = 0; c < kUpdW; ++c) red[c][tid] = row[c];
    treeW(red, tid);
    if (tid < kUpdW) a.partials[blockIdx.x * kUpdW + tid] = red[tid][0];
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) sLast = atomicAdd(&st->ticket_upd, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sLast) return;
  __threadfence();
  if (a.rule == 2) {
    topk_finish(a.ckey, a.cidx, gridDim.x, a.topk, a.pst, st->omega, st->v, a.tkout, tkey, tidx, tsel);
    if (tid < 8) red[tid][0] = __ldcg(a.tkout + tid);
    if (tid == 8) red[8][0] = __ldcg(a.tkout + 7);
    __syncthreads();
  } else {
    // fixed-order combine of the CTA partials
#pragma unroll
    for (int c = 0; c < kUpdW; ++c) red[c][tid] = 0.0;
    for (int b = tid; b < (int)gridDim.x; b += 256)
#pragma unroll
      for (int c = 0; c < kUpdW; ++c) red[c][tid] += __ldcg(a.partials + b * kUpdW + c);
    treeW(red, tid);
  }
  if (tid == 0) {
    const int nA = (int)red[7][0];
    st->nA = nA;
    st->Ebase = Ebase;
    st->nc_base = st->nc;
    st->Wsum = red[8][0];
    st->ticket_upd = 0u;
    for (int i = 0; i < 12; ++i) st->Pprev[i] = st->P[i];
    if (nA > 0) {
      const double Q[4] = {red[0][0], red[1][0], red[2][0], red[3][0]};
      const double U[3] = {red[4][0], red[5][0], red[6][0]};
      double Pn[12];
      apply_mean(Q, U, red[8][0], st->P, a.conv, Pn);
      for (int i = 0; i < 12; ++i) st->P[i] = Pn[i];
    }
  }
}

// End of the multi-launch run: T_out; rows k >= K_last of the outputs report E = 1, n = 0.
__global__ void k_track_finalize(const TrackState* st, int K, double* E_out, int* n_out, double* T_out) {
  const int k0 = st->K_last;
  for (int k = k0 + blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    E_out[k] = 1.0;
    n_out[k] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x < 12) T_out[threadIdx.x] = st->P[threadIdx.x];
}

// ------------------------------------------------------------------ persistent tracker (G = 1)
// The whole RO loop of one frame in ONE cooperative launch (all CTAs co-resident): phases are
// separated by a software grid barrier instead of kernel boundaries.  Per iteration i (schedule
// entry j = i mod n, particles K_j, point set X_j):
//   P0 (once) points of every set, pmax                                    | barrier
//   B  baseline E(P) on X_j if the set changed (L11)                      | barrier
//   P1 candidate-pose table (K_j rows, each CTA a slice)                  | barrier
//   P2 particle x point evaluation: warp-granular items (6 tiles x 16
//      particles) handed out by an atomic counter -> no CTA barriers, no
//      wave tail                                                          | barrier
//   P3 update partials: 256-particle blocks, the same tree as k_update    | barrier
//   P4 every CTA combines the partials in the same fixed tree (identical
//      P everywhere), then evaluates E(P) on its slice of X_j             | barrier
//   P5 every CTA: E(P), F3 guard, s-law, stalls, stop rule (identical
//      decisions); CTA 0 writes the trace.
// Results are bit-identical to the multi-launch path (same helpers, integer sums, same trees).
#ifndef PFT_ITEM_TILES
#define PFT_ITEM_TILES 6
#endif
constexpr int kItemTiles = PFT_ITEM_TILES;  // 8x4 tiles per warp item (= points per lane); 6: DESIGN.md §7
#ifndef PFT_ITEM_PARTICLES
#define PFT_ITEM_PARTICLES 16
#endif
constexpr int kItemParticles = PFT_ITEM_PARTICLES;
// CTA size of the persistent tracker: 512 threads at 1 CTA/SM (16 warps, 128 registers each, the
// same warps per SM as 2 x 256) halves the CTAs that take part in every grid barrier and serial phase
#ifndef PFT_PERSIST_THREADS
#define PFT_PERSIST_THREADS 256
#endif
constexpr int kPT = PFT_PERSIST_THREADS;
static_assert(kPT % 256 == 0, "update blocks are 256 particles");
// dynamic shared memory: red (update phases) and sPart (evaluation phase) are never live at the
// same time (the union), then the warps' pose slots
constexpr size_t kRedBytes = kUpdW * 256 * sizeof(double);
constexpr size_t kTopBytes = 256 * (sizeof(unsigned long long) + sizeof(int));
constexpr size_t kPartBytes = (kPT / 32) * kItemParticles * 33 * sizeof(unsigned long long);
constexpr size_t kUnionBytes = kPartBytes > kRedBytes + kTopBytes ? kPartBytes : kRedBytes + kTopBytes;
constexpr size_t kWPoseBytes = (kPT / 32) * kItemParticles * 6 * sizeof(double2);
constexpr size_t kPersistDynSmem = kUnionBytes + kWPoseBytes;

struct PArgs {
  const void* R;
  const void* V;
  const unsigned long long* mask;
  Geom g;
  BPFrame f;
  Sched sc;
  const float* pst;
  int K, conv, iters, rule, guard, sched, tail_pct, pair_sm;
  double beta, rho, omega0, v0;
  StopRule sr;
  const double* T_init;
  double* E_out;
  int* n_out;
  double* trace;
  double* T_out;
  unsigned long long* tdone;   // PFT_PHASE_TIMING: per-CTA P2 finish times (nullptr: off)
  int topk;
  // workspace: rank r's region starts at ws + r * rank_stride in one-GPU emulation (emul = 1),
  // at ws on its own GPU otherwise; the o_* are byte offsets inside a region
  char* ws;
  size_t rank_stride;
  size_t o_state, o_acc, o_ptab, o_pflag, o_upart, o_cpart, o_work, o_mtab;
  size_t o_ckey, o_cidx, o_tkout;  // F3 top-k candidates nblk x kTopkMax (key, index); result Q(4), U(3), n
  // F2 fused exchange (G > 1): xbuf[r] = rank r's exchange buffer (Kpad PartRec records, then
  // kXchgWords counter words), a peer pointer on a real multi-GPU node
  int G, rank, emul;
  char* xbuf[kMaxFusedRanks];
  size_t o_xcnt;
  size_t xhalf;  // records per exchange half: fixed per buffer (a peer may still read the previous call's half)
  unsigned long long watchdog_ns;  // grid-barrier / exchange wait before a trap (PFT_WATCHDOG_MS)
};

// Peer-exchange buffers of one rank's job (pre-flight).
struct PArgsX {
  int G, rank;
  char* xbuf[kMaxFusedRanks];
  size_t pre_off;
};

#ifdef PFT_WARP_UTIL
// diagnostic build only: per-warp P2 time split (claim -> staged, evaluation loop, row reduction,
// idle after the queue ran dry until the P2 barrier released), ns summed over the launch
__device__ unsigned long long g_wutil[4096][4];
#endif
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier over the nb co-resident CTAs of one rank: a monotone arrival counter (zeroed with
// the state before every launch).  Thread 0 adds 1 with release semantics (MEMBAR.GPU + RED)
// and polls until all nb CTAs of this round arrived: 1.3 us vs 2.2 us for a sense-reversing
// barrier at 296 CTAs (tools/microbench/barrier.cu).  The poll is a relaxed load (LDG.STRONG.GPU)
// and ONE acquire load follows it (LDG.STRONG.GPU + CCTL.IVALL, so data other CTAs wrote before
// the barrier is read fresh after it): an acquire in the poll loop itself invalidated the SM's L1
// on every poll, under the records the co-resident CTA was still gathering in P2
// (PFT_POLL_ACQUIRE=1 restores it, for A/B).
#ifndef PFT_POLL_ACQUIRE
#define PFT_POLL_ACQUIRE 0
#endif
#ifndef PFT_POLL_NS
#define PFT_POLL_NS 32  // poll backoff
#endif
__device__ __forceinline__ unsigned long long ld_poll_gpu(const unsigned long long* p) {
  unsigned long long v;
#if PFT_POLL_ACQUIRE
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#else
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#endif
  return v;
}
// Watchdog: a CTA that waits longer than watchdog_ns (PFT_WATCHDOG_MS, default 5 s) traps (a launch
// error instead of a hung GPU).
__device__ __forceinline__ void grid_barrier(TrackState* st, unsigned long long& target, int nb,
                                             unsigned long long watchdog_ns) {
  __syncthreads();
  target += (unsigned long long)nb;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&st->bar_mono) : "memory");
    unsigned long long v, t0 = 0ull;
    for (;;) {
      v = ld_poll_gpu(&st->bar_mono);
      if (v >= target) break;
      if (PFT_POLL_NS > 0) __nanosleep(PFT_POLL_NS);
      const unsigned long long now = global_ns();
      if (t0 == 0ull) t0 = now;
      else if (now - t0 > watchdog_ns) {
        printf("pft: grid barrier timeout (CTA %d, target %llu)\n", blockIdx.x, target);
        __trap();
      }
    }
#if !PFT_POLL_ACQUIRE
    // the acquire half: reads a value >= target of the same monotone counter, i.e. the release
    // sequence of every arrival of this round
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&st->bar_mono) : "memory");
#endif
  }
  __syncthreads();
}

template <typename T, int NT>
__device__ __forceinline__ void centre_slice(const T* __restrict__ V, const unsigned long long* __restrict__ mask,
                                             const Geom& g, const Points& pts, const double* m, int flag,
                                             int nb, int lb, unsigned long long& sum, unsigned& cnt,
                                             const double* pre = nullptr) {
  const int per = (pts.npad + nb - 1) / nb;
  const int b0 = lb * per, b1 = min(pts.npad, b0 + per);
  for (int base = b0; base < b1; base += NT) {
    const int i = base + threadIdx.x;
    double px[1] = {0.0}, py[1] = {0.0}, pz[1] = {0.0};
    if (pre && base == b0) { px[0] = pre[0]; py[0] = pre[1]; pz[0] = pre[2]; }  // first pass, loaded early
    else if (i < b1) { px[0] = __ldcg(pts.x + i); py[0] = __ldcg(pts.y + i); pz[0] = __ldcg(pts.z + i); }
    double mm[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) mm[q] = m[q];
    if (flag == 2) eval_points_f64<T, true, 1>(V, mask, g, mm, px, py, pz, sum, cnt);
    else if (flag == 1) eval_points_f64<T, false, 1>(V, mask, g, mm, px, py, pz, sum, cnt);
  }
}

// CTA total of the centre's (sum, cnt) -> thread 0 (NT threads).
template <int NT>
__device__ __forceinline__ void block_total(unsigned long long sum, unsigned cnt, unsigned long long* sS, unsigned* sN,
                                            unsigned long long& S, unsigned& n) {
  unsigned long long ws;
  unsigned wn;
  warp_total64(sum, cnt, ws, wn);
  if ((threadIdx.x & 31) == 0) { sS[threadIdx.x >> 5] = ws; sN[threadIdx.x >> 5] = wn; }
  __syncthreads();
  S = 0ull; n = 0u;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) { S += sS[w]; n += sN[w]; }
  __syncthreads();
}

template <typename T>
#ifndef PFT_PERSIST_MINB
#define PFT_PERSIST_MINB (512 / PFT_PERSIST_THREADS)
#endif
__global__ __launch_bounds__(kPT, PFT_PERSIST_MINB) void k_track_persistent(PArgs a) {
  extern __shared__ __align__(16) unsigned char sDyn[];
  unsigned char* const sUnion = sDyn;
  double (*red)[256] = reinterpret_cast<double (*)[256]>(sUnion);
  __shared__ double sP[12], sM[12], sPprev[12];
  __shared__ double sState[4];  // omega, v, Ec, Ebase
  __shared__ int sFlagC, sNA, sItem, sPos, sStalls, sStop, sSet, sKlast, sRej;
  __shared__ unsigned sNc, sNcBase;
  __shared__ unsigned long long sS[kPT / 32];
  __shared__ unsigned sNw[kPT / 32];
  double2 (*sWPose)[kItemParticles * 6] = reinterpret_cast<double2 (*)[kItemParticles * 6]>(sDyn + kUnionBytes);
  __shared__ int sTopSel[kTopkMax];
  // per-lane partials of the item's particles: (fix | cnt << 32), rows padded against bank conflicts
  unsigned long long (*sPart)[kItemParticles][33] =
      reinterpret_cast<unsigned long long (*)[kItemParticles][33]>(sUnion);
  // the schedule lives in shared memory: dynamically indexing the kernel-parameter copy would
  // make the compiler spill the whole parameter block to local memory
  __shared__ PSet sSets[PFT_MAX_SCHED];
  __shared__ int sSchedK[PFT_MAX_SCHED], sSchedSet[PFT_MAX_SCHED];
  // F2 rank groups: G ranks; in one-GPU emulation the grid holds all G groups of nb CTAs each and
  // every group owns a workspace region (a real multi-GPU run has one group per GPU)
  const int G = a.G;
  const int nb = a.emul ? (int)gridDim.x / G : (int)gridDim.x;   // CTAs of this rank
  const int grp = a.emul ? (int)blockIdx.x / nb : a.rank;       // this rank
  const int lb = a.emul ? (int)blockIdx.x - grp * nb : (int)blockIdx.x;
  char* const wsb = a.ws + (a.emul ? (size_t)grp * a.rank_stride : 0);
  const size_t wsoff = (size_t)(wsb - a.ws);
  TrackState* st = (TrackState*)(wsb + a.o_state);
  PartRec* const acc = (PartRec*)(wsb + a.o_acc);                // this rank's shard accumulators
  double* const ptab = (double*)(wsb + a.o_ptab);
  double* const mtab = (double*)(wsb + a.o_mtab);  // member deltas (q, u) of all K_i rows
  int* const pflag = (int*)(wsb + a.o_pflag);
  double* const upart = (double*)(wsb + a.o_upart);
  unsigned long long* const cpart = (unsigned long long*)(wsb + a.o_cpart);
  // centre-sum ring slot q: S at CSLOT(q)[0], n at CSLOT(q)[CN] (S and n on separate 128-B lines
  // measured the same)
#define CN 1
#define CSLOT(q) (cpart + 2 * (q))
  unsigned* const work = (unsigned*)(wsb + a.o_work);
  unsigned long long* const ckey = (unsigned long long*)(wsb + a.o_ckey);
  int* const cidx = (int*)(wsb + a.o_cidx);
  double* const tkout = (double*)(wsb + a.o_tkout);
  const bool out_rank = !a.emul || grp == 0;                     // writes the caller's outputs
  const int kloc = (a.K + G - 1) / G, kb = grp * kloc;            // shard: rows [kb, kb + kloc)
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long gen = 0ull;  // grid-barrier arrival target
  // centre sums: every CTA adds its (S, n) into slot cev % 3 of a 3-slot ring (exact integers, any
  // order); CTA 0 zeroes slot (cev + 1) % 3 during evaluation cev -- its last readers (evaluation
  // cev - 2) all passed the barrier of evaluation cev - 1 -- and the barrier of evaluation cev orders
  // that store before evaluation cev + 1's atomics.  Slot 0 is zeroed in P0.
  int cev = 0;
  // PFT_PHASE_TIMING accumulators (CTA 0, thread 0): B, P1, P2, P3, P4, P5, P2 tail, P0
  // (zero-initialised from a value ptxas cannot fold, a.K >= 1: a constant 0 was materialised
  // with 'CS2R Rx, SRZ' and spilled 5 cycles later, the idiom of DESIGN.md §9)
  const unsigned long long z0 = (unsigned long long)(a.K < 0);
  unsigned long long tph[8] = {z0, z0, z0, z0, z0, z0, z0, z0}, tmark = z0;
  const bool timing = a.tdone != nullptr;
  if (timing && tid == 0) tmark = global_ns();
  __shared__ unsigned long long sXround;
  __shared__ char* sXbuf[kMaxFusedRanks];  // (dynamic indexing of the parameter copy would spill it)
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < kMaxFusedRanks; ++q) sXbuf[q] = a.xbuf[q];
  }
  __syncthreads();
  if (tid == 0) {
    sXround = G > 1 ? *(volatile unsigned long long*)(sXbuf[grp] + a.o_xcnt + kMaxFusedRanks * sizeof(unsigned long long)) : 0ull;
#pragma unroll
    for (int q = 0; q < PFT_MAX_SCHED; ++q) {
      PSet p = a.sc.sets[q];
      if (p.x) { p.x = (double*)((char*)p.x + wsoff); p.y = (double*)((char*)p.y + wsoff); p.z = (double*)((char*)p.z + wsoff); }
      sSets[q] = p;
      sSchedK[q] = a.sc.K[q];
      sSchedSet[q] = a.sc.set[q];
    }
  }
  __syncthreads();
  const int nsched = a.sc.n, nsets = a.sc.nsets;
  const unsigned long long xround0 = sXround;
#ifndef PFT_CENTRE_CTAS
#define PFT_CENTRE_CTAS 148  // one slice per SM: 1.4233 vs 1.4249 ms (all 296 CTAs) and 1.4241 (96), A/B
#endif
  // CTAs that evaluate the centre E(P) (slices of the point set); the others add nothing
  const int ncc = PFT_CENTRE_CTAS > 0 ? min(nb, PFT_CENTRE_CTAS) : nb;
  // ---- P0: points of every set (a1/a2), accumulators, pmax
  {
    const int stride = nb * kPT;
    double pm = 0.0;
    for (int sidx = 0; sidx < nsets; ++sidx) {
      const PSet ps = sSets[sidx];
      for (int i0 = lb * kPT; i0 < ps.npad; i0 += stride) {
        const int i = i0 + tid;  // npad is a multiple of 32: whole warps stay converged
        double X = 0.0, Y = 0.0, Z = 0.0;
        bool valid = false;
        if (i < ps.npad) {
          valid = bp_slot(a.f, ps, i, X, Y, Z);
          ps.x[i] = X; ps.y[i] = Y; ps.z[i] = Z;
        }
        pm = fmax(pm, fmax(fabs(X), fmax(fabs(Y), fabs(Z))));
        const unsigned b = __ballot_sync(0xffffffffu, valid);
        if (lane == 0 && b) atomicAdd(&st->Nvalid[sidx], __popc(b));
      }
    }
    for (int sft = 16; sft > 0; sft >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, sft));
    if (lane == 0 && pm > 0.0) atomicMax(&st->pmax_bits, (unsigned long long)__double_as_longlong(pm));
    for (int k = lb * kPT + tid; k < kloc; k += stride) { acc[k].S = 0ull; acc[k].n = 0u; }
    if (lb == 0 && tid == 0) { CSLOT(0)[0] = 0ull; CSLOT(0)[CN] = 0ull; }
    // P2's static items go to CTA positions; with exactly two co-resident CTAs on every SM
    // (a.pair_sm: grid = 2 x SMs, so each SM holds two) the two CTAs of an SM take adjacent
    // positions, so its 16 warps share one point group in their L1.  Pairing: the SM's first CTA
    // draws a pair index and publishes it, the second waits for it.  (No watchdog on that wait:
    // at most two CTAs fit on an SM and all 2 x SMs are co-resident, so every SM's first CTA exists
    // and publishes; a watchdog here measured +0.15% from the allocation.)
    if (tid == 0) {
      int pos = lb;
      unsigned smid, nsm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsm));
      if (a.pair_sm && nsm <= 256u) {
        const unsigned sl = atomicAdd(&st->sm_cnt[smid], 1u);
        unsigned pr;
        if (sl == 0u) {
          pr = atomicAdd(&st->npairs, 1u);
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&st->sm_pair[smid]), "r"(pr + 1u) : "memory");
        } else {
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(pr) : "l"(&st->sm_pair[smid]) : "memory");
            if (pr) break;
            __nanosleep(32);
          }
          pr -= 1u;
        }
        pos = (int)(pr * 2u + (sl & 1u));
      }
      sPos = pos;
    }
  }
  if (tid == 0) {
    for (int q = 0; q < 12; ++q) sP[q] = a.T_init[q];
    sState[0] = a.omega0; sState[1] = a.v0; sState[2] = 1.0;
    sStalls = 0; sStop = 0; sSet = -1; sKlast = 0; sNc = 0u; sNA = 0;
  }
  grid_barrier(st, gen, nb, a.watchdog_ns);
#define PFT_TMARK(slot)                                        \
  if (timing && tid == 0) {                                    \
    const unsigned long long now_ = global_ns();               \
    tph[slot] += now_ - tmark;                                 \
    tmark = now_;                                              \
  }
  PFT_TMARK(7);
  const double pmax = __longlong_as_double((long long)__ldcg(&st->pmax_bits));
  __shared__ int sNv[4];  // valid points per set (final after P0's barrier): one read per CTA, not
  if (tid < 4) sNv[tid] = __ldcg(&st->Nvalid[tid]);  // one per warp of every CTA and iteration
  __syncthreads();
  int it = 0;
  for (; it < a.iters; ++it) {
    const int j = it % nsched;
    const int Ki = sSchedK[j], set = sSchedSet[j];
    const PSet ps = sSets[set];
    const Points pts = ps.pts();
    const int N = sNv[set];
    // ---- B: baseline E(P^(i-1)) on this iteration's point set when it changed (L11)
    if (set != sSet) {
      if (tid == 0) sFlagC = explicit_pose(sP, a.g, pmax, sM);
      __syncthreads();
      unsigned long long sum = 0ull;
      unsigned cnt = 0u;
      centre_slice<T, kPT>((const T*)a.V, a.mask, a.g, pts, sM, sFlagC, ncc, lb, sum, cnt);
      unsigned long long S;
      unsigned n;
      block_total<kPT>(sum, cnt, sS, sNw, S, n);
      unsigned long long* slot = CSLOT(cev % 3);
      if (tid == 0) {
        if (lb == 0) { CSLOT((cev + 1) % 3)[0] = 0ull; CSLOT((cev + 1) % 3)[CN] = 0ull; }
        if (lb < ncc) {
          atomicAdd(slot, S);
          atomicAdd(slot + CN, (unsigned long long)n);
        }
      }
      grid_barrier(st, gen, nb, a.watchdog_ns);
      ++cev;
      unsigned long long S2 = 0ull, n2 = 0ull;
      if (tid == 0) { S2 = __ldcg(slot); n2 = __ldcg(slot + CN); }
      if (tid == 0) {
        sState[2] = fitness_c(S2, (unsigned)n2, a.rho, N);
        sNc = (unsigned)n2;
        sSet = set;
      }
      __syncthreads();
    }
    PFT_TMARK(0);
    // ---- P1: candidate-pose table (K_i rows), interleaved over all CTAs (row kb + tid*nb + lb):
    // each pose is a ~2500-cycle fp64 chain, so K = 2048 rows on 296 CTAs x ~7 threads is one
    // chain's latency, where contiguous 256-row slices put them all on 8 SMs' fp64 pipes
    for (int k = kb + tid * nb + lb; k < min(Ki, kb + kloc); k += nb * kPT) {
      double m[12];
      pflag[k] = candidate_pose(a.pst + 6 * (size_t)k, sState[0], sState[1], sP, a.conv, a.g, pmax, m);
      double2* row = (double2*)(ptab + 12 * (size_t)k);
#pragma unroll
      for (int q = 0; q < 6; ++q) row[q] = make_double2(m[2 * q], m[2 * q + 1]);
    }
    // and, on threads the pose rows leave idle, the member deltas (q_k, u_k) of all K_i rows for P3
    // (plain / weighted mean), so P3 loads them instead of running the sincos chain on the 256-row
    // blocks' few SMs
#ifdef PFT_MEMBER_TABLE
    if (a.rule != 2)
      for (int k = (kPT - 1 - tid) * nb + lb; k < Ki; k += nb * kPT) {
        double q[4], u[3];
        member_delta(a.pst + 6 * (size_t)k, sState[0], sState[1], q, u);
        double2* mrow = (double2*)(mtab + 8 * (size_t)k);
        mrow[0] = make_double2(q[0], q[1]);
        mrow[1] = make_double2(q[2], q[3]);
        mrow[2] = make_double2(u[0], u[1]);
        mtab[8 * (size_t)k + 6] = u[2];
      }
#endif
    grid_barrier(st, gen, nb, a.watchdog_ns);
    PFT_TMARK(1);
    // F2: this rank's shard of the K_i particles, local rows [0, Ks) = global rows [kb, kb + Ks)
    const int Ks = max(0, min(Ki, kb + kloc) - kb);
    // ---- P2: particle x point evaluation, warp-granular items (group-major: item = group * nchunks
    // + chunk).  sched 0: one global dynamic queue; sched 1: CTA c owns the contiguous range
    // [c*n/G, (c+1)*n/G) (its warps share one image region -> L1 reuse), handed out by a CTA counter.
    {
      // Items: the first ~80% of the particle chunks as 16-particle items, the rest as 4-particle
      // items handed out last, so the queue drains on small items (short cross-CTA tail).
      const int ngroups = (pts.npad + 32 * kItemTiles - 1) / (32 * kItemTiles);
      const int nch16 = (Ks + kItemParticles - 1) / kItemParticles;
      // (only when there are few items per warp: with many, the tail is already negligible)
      const bool few = (long long)ngroups * nch16 < 64LL * nb * (kPT / 32);
      const int cb = (a.sched == 1 || !few) ? nch16 : nch16 - (nch16 * a.tail_pct + 99) / 100;  // big chunks
      const int ksmall = cb * kItemParticles;                           // first particle of the small part
      const int nch4 = (Ks - ksmall + 3) / 4;
      const int nbig = ngroups * cb;
      const int nitems = nbig + ngroups * nch4;
      const int r0 = (int)((long long)nitems * lb / nb);
      const int r1 = (int)((long long)nitems * (lb + 1) / nb);
      if (tid == 0) sItem = 0;
      __syncthreads();
#ifdef PFT_WARP_UTIL
      unsigned long long wu0 = global_ns(), wu[4] = {0ull, 0ull, 0ull, 0ull};
#endif
      // sched 0: the first ~static_pct % of the big items are handed out statically, warp w taking
      // items w, w + nw, w + 2 nw, ... (no atomic round trip per claim, and the 8 warps of a CTA --
      // consecutive items -- work on the same point group, sharing its points and nearby records
      // in L1); the rest, and the small tail items, come from the dynamic queue, whose counter is
      // offset by the static items
      const int nwq = nb * (kPT / 32), gwq = sPos * (kPT / 32) + (tid >> 5);
#ifndef PFT_STATIC_ITEMS
#define PFT_STATIC_ITEMS 4  // at most, per warp (config Q: 4 of ~6.3 items; 2 / 3 / 5: slower, A/B)
#endif
#ifndef PFT_STATIC_PCT
#define PFT_STATIC_PCT 80   // at most this share of the big items (5 at config Q = 98%: slower)
#endif
      const int nstat = a.sched == 1 ? 0 : min(PFT_STATIC_ITEMS, (int)((long long)nbig * PFT_STATIC_PCT / 100) / nwq);
      int nst = 0;
      for (;;) {
#ifdef PFT_WARP_UTIL
        const unsigned long long wa = global_ns();
#endif
        int item = 0;
        if (lane == 0)
          item = a.sched == 1                ? r0 + atomicAdd(&sItem, 1)
                 : nst < nstat ? gwq + nst * nwq
                                : nstat * nwq + (int)atomicAdd(work + it, 1u);
        ++nst;
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= (a.sched == 1 ? r1 : nitems)) break;
        int group, k0, k1;
        if (item < nbig) {
          group = item / cb;
          const int chunk = item - group * cb;
          k0 = chunk * kItemParticles;
          k1 = min(Ks, k0 + kItemParticles);
        } else {
          const int it2 = item - nbig;
          group = it2 / nch4;
          const int chunk = it2 - group * nch4;
          k0 = ksmall + chunk * 4;
          k1 = min(Ks, k0 + 4);
        }
        double px[kItemTiles], py[kItemTiles], pz[kItemTiles];
#pragma unroll
        for (int p = 0; p < kItemTiles; ++p) {
          const int i = (group * kItemTiles + p) * 32 + lane;
          px[p] = py[p] = pz[p] = 0.0;
          if (i < pts.npad) { px[p] = __ldcg(pts.x + i); py[p] = __ldcg(pts.y + i); pz[p] = __ldcg(pts.z + i); }
        }
        // stage the item's poses in this warp's shared slot (6 x 16 B per pose, 3 per lane); the
        // item's pose flags as two warp-uniform bit masks (no per-particle shared-memory load)
        double2* wp = sWPose[tid >> 5];
        __syncwarp();
        for (int q = lane; q < (k1 - k0) * 6; q += 32) wp[q] = __ldcg((const double2*)(ptab + 12 * (size_t)(kb + k0)) + q);
        const int myflag = lane < k1 - k0 ? __ldcg(pflag + kb + k0 + lane) : 0;
        const unsigned fvalid = __ballot_sync(0xffffffffu, myflag != 0), ffast = __ballot_sync(0xffffffffu, myflag == 2);
        __syncwarp();
#ifdef PFT_WARP_UTIL
        const unsigned long long wb = global_ns();
#endif
        unsigned long long (*part)[33] = sPart[tid >> 5];
        for (int k = k0; k < k1; ++k) {
          unsigned sum = 0u;
          unsigned cnt = 0u;
          if ((fvalid >> (k - k0)) & 1u) {  // warp-uniform
            double m[12];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const double2 v = wp[(k - k0) * 6 + q];
              m[2 * q] = v.x;
              m[2 * q + 1] = v.y;
            }
            if ((ffast >> (k - k0)) & 1u) eval_points<T, true, kItemTiles>((const T*)a.R, a.mask, a.g, m, px, py, pz, sum, cnt);
            else eval_points<T, false, kItemTiles>((const T*)a.R, a.mask, a.g, m, px, py, pz, sum, cnt);
          }
          part[k - k0][lane] = (unsigned long long)sum | ((unsigned long long)cnt << 32);
        }
        __syncwarp();
#ifdef PFT_WARP_UTIL
        const unsigned long long wc = global_ns();
#endif
        // particle j's row is reduced by lanes j and j + 16, half a row each (exact integers),
        // combined by one shuffle; lane j issues the atomics
        static_assert(kItemParticles <= 16, "two lanes per particle row");
        {
          const int pj = lane & 15, h = lane >> 4;
          unsigned long long S = 0ull;
          unsigned n = 0u;
          if (pj < k1 - k0) {
#pragma unroll
            for (int l = 0; l < 16; ++l) {
              const unsigned long long w = part[pj][h * 16 + l];
              S += w & 0xffffffffull;
              n += (unsigned)(w >> 32);
            }
          }
          S += __shfl_down_sync(0xffffffffu, S, 16);
          n += __shfl_down_sync(0xffffffffu, n, 16);
          if (lane < k1 - k0 && n) {
            atomicAdd(&acc[k0 + lane].S, S);
            atomicAdd(&acc[k0 + lane].n, n);
          }
        }
        __syncwarp();
#ifdef PFT_WARP_UTIL
        wu[0] += wb - wa; wu[1] += wc - wb; wu[2] += global_ns() - wc;
#endif
      }
#ifdef PFT_WARP_UTIL
      wu0 = global_ns();
      if (lane == 0) {
        const int gw = (lb * kPT + tid) >> 5;
        g_wutil[gw][0] += wu[0]; g_wutil[gw][1] += wu[1]; g_wutil[gw][2] += wu[2];
        g_wutil[gw][3] -= wu0;  // + the P2 barrier release time below
      }
#endif
    }
    // the member deltas of this CTA's first P3 block depend only on s and the template rows, so
    // they are computed here, while the other CTAs still finish P2
    double mq[4] = {0.0, 0.0, 0.0, 0.0}, mu[3] = {0.0, 0.0, 0.0};
    if (a.rule != 2 && tid < 256 && lb * 256 + tid < Ki)
      member_delta(a.pst + 6 * (size_t)(lb * 256 + tid), sState[0], sState[1], mq, mu);
    if (timing) {
      __syncthreads();
      if (tid == 0) a.tdone[lb] = global_ns();
    }
    grid_barrier(st, gen, nb, a.watchdog_ns);
#ifdef PFT_WARP_UTIL
    if ((tid & 31) == 0) g_wutil[(lb * kPT + tid) >> 5][3] += global_ns();
#endif
    if (timing && tid == 0 && lb == 0) {
      unsigned long long lo = ~0ull, hi = 0ull;
      for (int b = 0; b < (int)nb; ++b) {
        const unsigned long long v = __ldcg(a.tdone + b);
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
      }
      tph[6] += hi - lo;
    }
    PFT_TMARK(2);
    // ---- X (F2, G > 1): every CTA pushes its slice of this rank's shard records into every rank's
    // exchange buffer (P2P stores) in the half of the round's parity -- a peer may still be reading
    // the other half in its P3 of the previous round, possibly of the previous call, but not this
    // half's previous round (it signalled round R-1 after finishing P3 of round R-2) -- then the
    // rank signals each peer once and every CTA waits until all G shards of the round arrived.
    const PartRec* recs = acc;
    if (G > 1) {
      const size_t half = (size_t)((xround0 + (unsigned long long)it) & 1ull) * a.xhalf;  // global round parity
      for (int j = lb * kPT + tid; j < Ks; j += nb * kPT) {
        const ulonglong2 r = __ldcg(reinterpret_cast<const ulonglong2*>(acc + j));  // (S, n | pad)
        for (int q = 0; q < G; ++q) __stcg(reinterpret_cast<ulonglong2*>((PartRec*)sXbuf[q] + half + kb + j), r);
        acc[j].S = 0ull;
        acc[j].n = 0u;
      }
      __threadfence_system();
      grid_barrier(st, gen, nb, a.watchdog_ns);
      if (lb == 0 && tid < G) {
        __threadfence_system();
        atomicAdd_system((unsigned long long*)(sXbuf[tid] + a.o_xcnt) + grp, 1ull);
      }
      if (tid == 0) {
        const unsigned long long* cnt = (const unsigned long long*)(sXbuf[grp] + a.o_xcnt);
        const unsigned long long target = xround0 + (unsigned long long)it + 1ull;
        const unsigned long long t0 = global_ns();
        for (int q = 0; q < G; ++q)
          while (ld_acquire_sys(cnt + q) < target) {
            __nanosleep(32);
            if (global_ns() - t0 > a.watchdog_ns) {
              printf("pft: exchange timeout (rank %d CTA %d source %d round %llu)\n", grp, lb, q, target);
              __trap();
            }
          }
        __threadfence_system();
      }
      __syncthreads();
      recs = (const PartRec*)sXbuf[grp] + half;
    }
    // ---- P3: E_k, advantage set, per-block partials (same tree as k_update)
    const double Ebase = sState[2];
    const int nblk = (Ki + 255) / 256;
    unsigned long long* tkey = reinterpret_cast<unsigned long long*>(sUnion + kRedBytes);  // top-k scratch
    int* tidx = reinterpret_cast<int*>(sUnion + kRedBytes + 256 * sizeof(unsigned long long));
    for (int b = lb; b < nblk; b += nb) {
      const int k = tid < 256 ? b * 256 + tid : Ki;  // (threads >= 256 of a 512-thread CTA idle)
      double row[kUpdW];
#pragma unroll
      for (int c = 0; c < kUpdW; ++c) row[c] = 0.0;
      unsigned long long key = ~0ull;
      if (k < Ki) {
        const unsigned long long S = __ldcg(&recs[k].S);
        const unsigned n = __ldcg(&recs[k].n);
        const double E = fitness_of(S, n, a.rho, N);
        if (out_rank) {
          a.E_out[k] = E;
          a.n_out[k] = (int)n;
        }
        if (a.rule == 2) {
          if (E < Ebase) key = (unsigned long long)__double_as_longlong(E);
        } else {
#ifdef PFT_MEMBER_TABLE
          member_row_tab(row, E, Ebase, a.rule, mtab + 8 * (size_t)k);
#else
          if (b == lb) member_row_pre(row, E, Ebase, a.rule, mq, mu);
          else
          member_row(row, E, Ebase, a.rule, a.pst + 6 * (size_t)k, sState[0], sState[1]);
#endif
        }
        if (G == 1) {
          acc[k].S = 0ull;
          acc[k].n = 0u;
        }
      }
      if (a.rule == 2) {
        block_topk(key, k, a.topk, tkey, tidx, ckey + (size_t)b * kTopkMax, cidx + (size_t)b * kTopkMax, tid);
      } else {
        if (tid < 256)
#pragma unroll
          for (int c = 0; c < kUpdW; ++c) red[c][tid] = row[c];
        treeW(red, tid);
        if (tid < kUpdW) upart[b * kUpdW + tid] = red[tid][0];
        __syncthreads();
      }
    }
    // the centre slice's first-pass points, loaded now: their L2 round trip overlaps the barrier
    double cpre[3] = {0.0, 0.0, 0.0};
    {
      const int per = (pts.npad + ncc - 1) / ncc, i = lb * per + tid;
      if (i < min(pts.npad, lb * per + per)) { cpre[0] = __ldcg(pts.x + i); cpre[1] = __ldcg(pts.y + i); cpre[2] = __ldcg(pts.z + i); }
    }
    grid_barrier(st, gen, nb, a.watchdog_ns);
    PFT_TMARK(3);
    // ---- P4: combine partials (fixed tree, identical in every CTA) -> P; centre slice
    if (a.rule == 2) {
      // F3 top-k: CTA 0 merges the blocks' sorted candidates and sums the selected deltas
      if (lb == 0)
        topk_finish(ckey, cidx, nblk, a.topk, a.pst, sState[0], sState[1], tkout, tkey, tidx, sTopSel);
      grid_barrier(st, gen, nb, a.watchdog_ns);
      if (tid < 8) red[tid][0] = __ldcg(tkout + tid);
      if (tid == 8) red[8][0] = __ldcg(tkout + 7);  // weight sum = number selected
      __syncthreads();
    } else {
      if (nblk <= 256) {
        // every CTA reads the same nblk x kUpdW partials right after the barrier: read them as one
        // flat array, consecutive threads on consecutive doubles (a few 128-B requests per CTA
        // instead of ~45 scattered ones on the same 5 L2 lines, x 296 CTAs); red[c][b] = 0 + p
        if (tid < 256)
#pragma unroll
          for (int c = 0; c < kUpdW; ++c) red[c][tid] = 0.0;
        __syncthreads();
        for (int e = tid; e < nblk * kUpdW; e += kPT) {
          const int b = e / kUpdW, c = e - b * kUpdW;
          red[c][b] += __ldcg(upart + e);
        }
      } else if (tid < 256) {
#pragma unroll
        for (int c = 0; c < kUpdW; ++c) red[c][tid] = 0.0;
        for (int b = tid; b < nblk; b += 256)
#pragma unroll
          for (int c = 0; c < kUpdW; ++c) red[c][tid] += __ldcg(upart + b * kUpdW + c);
      }
      treeW(red, tid);
    }
    if (tid == 0) {
      const int nA = (int)red[7][0];
      sNA = nA;
      sState[3] = Ebase;
      sNcBase = sNc;
      for (int q = 0; q < 12; ++q) sPprev[q] = sP[q];
      if (nA > 0) {
        const double Q[4] = {red[0][0], red[1][0], red[2][0], red[3][0]};
        const double U[3] = {red[4][0], red[5][0], red[6][0]};
        double Pn[12];
        apply_mean(Q, U, red[8][0], sP, a.conv, Pn);
        for (int q = 0; q < 12; ++q) sP[q] = Pn[q];
        sFlagC = explicit_pose(sP, a.g, pmax, sM);
      }
    }
    __syncthreads();
    if (sNA > 0) {
      unsigned long long sum = 0ull;
      unsigned cnt = 0u;
      centre_slice<T, kPT>((const T*)a.V, a.mask, a.g, pts, sM, sFlagC, ncc, lb, sum, cnt, cpre);
      unsigned long long S;
      unsigned n;
      block_total<kPT>(sum, cnt, sS, sNw, S, n);
      if (tid == 0) {
        if (lb == 0) { CSLOT((cev + 1) % 3)[0] = 0ull; CSLOT((cev + 1) % 3)[CN] = 0ull; }
        if (lb < ncc) {
          atomicAdd(CSLOT(cev % 3), S);
          atomicAdd(CSLOT(cev % 3) + CN, (unsigned long long)n);
        }
      }
      grid_barrier(st, gen, nb, a.watchdog_ns);  // sNA is identical in every CTA: uniform barrier
    }
    PFT_TMARK(4);
    // ---- P5: E(P), F3 guard, s-law, stalls, stop rule, trace
    unsigned long long S5 = 0ull, n5 = 0ull;
    if (sNA > 0) {
      if (tid == 0) { S5 = __ldcg(CSLOT(cev % 3)); n5 = __ldcg(CSLOT(cev % 3) + CN); }
      ++cev;
    }
    if (tid == 0) {
      double Ec = sState[3];
      unsigned nc = sNcBase;
      int rejected = 0;
      if (sNA > 0) {
        const unsigned long long S = S5, n = n5;
        const double En = fitness_c(S, (unsigned)n, a.rho, N);
        if (a.guard && En > sState[3]) {  // F3 guard: keep P^(i-1)
          rejected = 1;
          for (int q = 0; q < 12; ++q) sP[q] = sPprev[q];
        } else {
          Ec = En;
          nc = (unsigned)n;
        }
      }
      const int stalls = (sNA == 0 || rejected) ? sStalls + 1 : 0;
      const double om = sState[0], v = sState[1];
      const double f = s_factor(a.beta, Ec);
      const double om1 = __dmul_rn(f, om), v1 = __dmul_rn(f, v);
      const bool stop = stop_now(a.sr, om1, v1, stalls);
      if (lb == 0 && out_rank && a.trace) {
        const int flags = (sNA == 0 ? 1 : 0) | (sState[3] == 1.0 ? 2 : 0) | (N == 0 ? 4 : 0) | (rejected ? 8 : 0) |
                          (stop ? 16 : 0);
        write_trace(a.trace + (size_t)it * PFT_TRACE_DOUBLES, sState[3], sNA, om, v, sP, Ec, om1, v1, flags, nc, N, Ki,
                    ps.sx + 1000 * ps.sy);
      }
      sState[0] = om1; sState[1] = v1; sState[2] = Ec; sNc = nc; sStalls = stalls; sStop = stop ? 1 : 0;
      sKlast = Ki; sRej = rejected;
    }
    __syncthreads();
    PFT_TMARK(5);
    if (sStop) { ++it; break; }  // identical decision in every CTA
  }
  if (timing && tid == 0 && lb == 0)
    printf("pft phase timing (us, %d iterations, %d CTAs): P0 %.1f  B %.1f  P1 %.1f  P2 %.1f (tail %.1f)  P3 %.1f  P4 %.1f  P5 %.1f\n",
           it, (int)nb, tph[7] * 1e-3, tph[0] * 1e-3, tph[1] * 1e-3, tph[2] * 1e-3, tph[6] * 1e-3,
           tph[3] * 1e-3, tph[4] * 1e-3, tph[5] * 1e-3);
#undef PFT_TMARK
#undef CSLOT
#undef CN
  // ---- outputs
  if (lb == 0 && tid == 0) {
    for (int q = 0; q < 12; ++q) st->P[q] = sP[q];
    st->omega = sState[0]; st->v = sState[1]; st->Ec = sState[2]; st->nA = sNA; st->nc = sNc;
    st->iter = it; st->K_last = sKlast; st->stopped = sStop;
    if (G > 1) *(unsigned long long*)(sXbuf[grp] + a.o_xcnt + kMaxFusedRanks * sizeof(unsigned long long)) =
        xround0 + (unsigned long long)it;  // exchange rounds completed (every CTA read xround0 before P0's barrier)
    if (out_rank) {
      for (int q = 0; q < 12; ++q) a.T_out[q] = sP[q];
      if (a.trace)
        for (int r = it; r < a.iters; ++r) write_not_run(a.trace + (size_t)r * PFT_TRACE_DOUBLES);
    }
  }
  if (out_rank)
    for (int k = sKlast + lb * kPT + tid; k < a.K; k += nb * kPT) {
      a.E_out[k] = 1.0;
      a.n_out[k] = 0;
    }
}

// ------------------------------------------------------------------ host side
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

pft_status track_layout(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles,
                        const pft_track_params* prm, int nranks, TrackLayout* L) {
  if (nparticles < 1) return fail(PFT_ERR_INVALID_ARG, "number of particles/poses must be >= 1");
  if (prm->stride < 1) return fail(PFT_ERR_INVALID_ARG, "stride must be >= 1");
  if (prm->nsched < 0 || prm->nsched > PFT_MAX_SCHED) return fail(PFT_ERR_INVALID_ARG, "nsched must be in [0,%d]", PFT_MAX_SCHED);
  pft_status s = check_intrinsics(K);
  if (s != PFT_OK) return s;
  int n = prm->nsched > 0 ? prm->nsched : 1;
  L->nsched = n;
  L->nsets = 0;
  L->npad_max = 0;
  size_t off = 0;
  L->state_off = off; off = align_up(off + sizeof(TrackState), 256);
  for (int j = 0; j < n; ++j) {
    int sx = prm->stride, sy = prm->stride, Kj = nparticles;
    if (prm->nsched > 0) {
      sx = prm->sched_sx[j]; sy = prm->sched_sy[j];
      if (prm->sched_K[j] < 1) return fail(PFT_ERR_INVALID_ARG, "sched_K[%d] must be >= 1", j);
      Kj = prm->sched_K[j] < nparticles ? prm->sched_K[j] : nparticles;
    }
    if (sx < 1 || sy < 1) return fail(PFT_ERR_INVALID_ARG, "schedule strides must be >= 1");
    L->sched_K[j] = Kj;
    int found = -1;
    for (int q = 0; q < L->nsets; ++q)
      if (L->sets[q].sx == sx && L->sets[q].sy == sy) found = q;
    if (found < 0) {
      PointSetL& p = L->sets[L->nsets];
      p.sx = sx; p.sy = sy;
      p.nr = (K->height + sy - 1) / sy;
      p.nc = (K->width + sx - 1) / sx;
      p.ntx = (p.nc + 7) / 8;
      p.nty = (p.nr + 3) / 4;
      p.npad = p.ntx * p.nty * 32;
      p.off = off;
      off = align_up(off + 3 * sizeof(double) * (size_t)p.npad, 256);
      if (p.npad > L->npad_max) L->npad_max = p.npad;
      found = L->nsets++;
    }
    L->sched_set[j] = found;
  }
  // F2b point shards (virtual or NCCL, G > 1): every rank holds all K records
  L->points_part = vol && vol->partition == PFT_PARTITION_POINTS && (nranks > 1 || vol->nccl_comm) && !vol->virtual_fused &&
                   !vol->p2p;
  L->kloc = L->points_part ? nparticles : (nparticles + nranks - 1) / nranks;
  L->kfull = L->kloc * nranks;
  L->nblk_upd = (nparticles + 255) / 256;
  L->acc_local_off = off; off = align_up(off + sizeof(PartRec) * (size_t)L->kloc, 256);
  if (nranks > 1 && !L->points_part) { L->acc_full_off = off; off = align_up(off + sizeof(PartRec) * (size_t)L->kfull, 256); }
  else L->acc_full_off = L->acc_local_off;  // (point shards: the records are all-reduced in place)
  L->cacc_off = off; off = align_up(off + 2 * sizeof(unsigned long long), 256);
  L->part_off = off; off = align_up(off + kUpdW * sizeof(double) * (size_t)L->nblk_upd, 256);
  L->ptab_off = off; off = align_up(off + (12 * sizeof(double) + sizeof(int)) * (size_t)nparticles, 256);
  L->mtab_off = off; off = align_up(off + 8 * sizeof(double) * (size_t)nparticles, 256);
  L->cpart_off = off; off = align_up(off + 2 * 2 * sizeof(unsigned long long) * 148 * 8, 256);  // centre-sum ring (3 x (S, n))
  L->work_off = off; off = align_up(off + sizeof(unsigned) * 1024 + sizeof(unsigned long long) * 148 * 8, 256);
  L->topk_off = off;
  off = align_up(off + (sizeof(unsigned long long) + sizeof(int)) * kTopkMax * (size_t)L->nblk_upd + 16 * sizeof(double), 256);
  L->xch_off = 0;
  L->xcnt_rel = 0;
  if (vol && vol->virtual_fused && nranks > 1) {
    // two halves of G * kloc records, then the counters
    L->xch_off = off;
    L->xcnt_rel = align_up(2 * sizeof(PartRec) * (size_t)L->kfull, 256);
    off = align_up(off + L->xcnt_rel + (kMaxFusedRanks + 1) * sizeof(unsigned long long), 256);
  }
  L->region = off;
  L->total = (vol && vol->virtual_fused && nranks > 1) ? off * (size_t)nranks : off;
  return PFT_OK;
}

pft_status comm_allgather(pft_volume* vol, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st);
pft_status comm_allreduce_u64(pft_volume* vol, void* buf, size_t count, cudaStream_t st);

// F2b: point slots of rank q of G -- whole 8x4 tiles (32 slots), contiguous.
static void point_slice(int npad, int G, int q, int& b, int& e) {
  const int tiles = npad / 32, per = (tiles + G - 1) / G;
  b = min(npad, q * per * 32);
  e = min(npad, (q + 1) * per * 32);
}

struct Launch {
  pft_volume* vol;
  TrackLayout L;
  char* ws;
  cudaStream_t st;
  TrackState* state() const { return (TrackState*)(ws + L.state_off); }
  PSet set(int q) const {
    const PointSetL& p = L.sets[q];
    double* b = (double*)(ws + p.off);
    return PSet{b, b + p.npad, b + 2 * (size_t)p.npad, p.npad, p.sx, p.sy, p.nr, p.nc, p.ntx};
  }
  Sched sched() const {
    Sched s;
    s.n = L.nsched;
    s.nsets = L.nsets;
    for (int j = 0; j < PFT_MAX_SCHED; ++j) { s.K[j] = j < L.nsched ? L.sched_K[j] : 0; s.set[j] = j < L.nsched ? L.sched_set[j] : 0; }
    for (int q = 0; q < PFT_MAX_SCHED; ++q) s.sets[q] = q < L.nsets ? set(q) : PSet{};
    return s;
  }
};

static BPFrame frame_of(const Launch& c, const uint16_t* depth, const pft_intrinsics* K) {
  return BPFrame{depth, K->fx, K->fy, K->cx, K->cy, K->depth_unit_m, c.vol->g.max_depth, K->width, K->height};
}

static void launch_prologue(const Launch& c, const uint16_t* depth, const pft_intrinsics* K, const double* T_init,
                            double omega0, double v0) {
  TrackArgs ta{c.state(), T_init, omega0, v0, (PartRec*)(c.ws + c.L.acc_local_off), c.L.kloc};
  int gi = (c.L.kloc + 255) / 256;
  PFT_LAUNCH(PFT_PROF_PREP, c.st, k_track_init<<<gi < 148 ? gi : 148, 256, 0, c.st>>>(ta));
  const BPFrame f = frame_of(c, depth, K);
  for (int q = 0; q < c.L.nsets; ++q) {
    const PSet s = c.set(q);
    PFT_LAUNCH(PFT_PROF_PREP, c.st, k_backproject<<<(s.npad + 255) / 256, 256, 0, c.st>>>(f, s, &c.state()->Nvalid[q]));
  }
}

template <typename T>
static pft_status launch_centre(const Launch& c, int mode, int set, int it, int Ki, const pft_track_params* prm,
                                double* trace) {
  const PSet s = c.set(set);
  CentreArgs ca{c.vol->base + c.vol->L.v_off, (const unsigned long long*)(c.vol->base + c.vol->L.m_off), c.vol->g,
                s.pts(), c.state(), mode, set, it, Ki, s.sx + 1000 * s.sy, prm->guard, prm->beta,
                prm->min_inband_frac, StopRule{prm->min_search_deg, prm->min_search_cm, prm->stall_limit}, trace,
                0, s.npad, nullptr};
  if (!c.L.points_part) {
    const int grid = (s.npad + kThreads * kCentrePPT - 1) / (kThreads * kCentrePPT);
    PFT_LAUNCH(PFT_PROF_CENTRE, c.st, k_centre<T><<<grid, kThreads, 0, c.st>>>(ca));
    return PFT_OK;
  }
  // F2b: this rank's slice (virtual shards: every slice in turn) into the partial sums, their sum
  // across the ranks (NCCL all-reduce; the virtual slices already share one accumulator), finish
  ca.cacc = (unsigned long long*)(c.ws + c.L.cacc_off);
  const int G = c.vol->nranks;
  for (int q = 0; q < G; ++q) {
    if (c.vol->virtual_ranks <= 1 && q != c.vol->rank) continue;
    point_slice(s.npad, G, q, ca.pbeg, ca.pend);
    const int grid = (ca.pend - ca.pbeg + kThreads * kCentrePPT - 1) / (kThreads * kCentrePPT);
    if (grid > 0) PFT_LAUNCH(PFT_PROF_CENTRE, c.st, k_centre<T><<<grid, kThreads, 0, c.st>>>(ca));
  }
  if (c.vol->virtual_ranks <= 1) {
    const pft_status r = comm_allreduce_u64(c.vol, ca.cacc, 2, c.st);
    if (r != PFT_OK) return r;
  }
  PFT_LAUNCH(PFT_PROF_CENTRE, c.st, k_centre_finish<<<1, 1, 0, c.st>>>(ca));
  return PFT_OK;
}

template <typename T>
static void launch_eval(const Launch& c, int mode, const float* pst, int k_begin, int k_count, int conv,
                        const double* poses, PartRec* acc, int set, int pbeg = 0, int pend = -1) {
  if (k_count <= 0) return;
  const PSet s = c.set(set);
  if (pend < 0) pend = s.npad;
  if (pend <= pbeg) return;
  EvalArgs ea{c.vol->base + c.vol->L.r_off, (const unsigned long long*)(c.vol->base + c.vol->L.m_off), c.vol->g,
              s.pts(), pbeg, pend, mode, pst, k_begin, k_count, c.state(), conv, poses, acc};
  dim3 grid((pend - pbeg + kThreads * kPPT - 1) / (kThreads * kPPT), (k_count + kPC - 1) / kPC);
  static const int ppt = [] {  // tuning knob for experiments: PFT_EVAL_PPT=2|4
    const char* e = getenv("PFT_EVAL_PPT");
    return e && atoi(e) == 2 ? 2 : kPPT;
  }();
  if (ppt == 2) {
    grid.x = (pend - pbeg + kThreads * 2 - 1) / (kThreads * 2);
    PFT_LAUNCH(PFT_PROF_EVAL, c.st, k_particle_eval<T, 2><<<grid, kThreads, 0, c.st>>>(ea));
  } else {
    PFT_LAUNCH(PFT_PROF_EVAL, c.st, k_particle_eval<T, kPPT><<<grid, kThreads, 0, c.st>>>(ea));
  }
}

// Co-resident CTAs of k_track_persistent<T> on the current device (cached per device; the carveout
// attribute is set once per device before the occupancy query).  Shared-memory carveout: the
// smallest that keeps 2 CTAs/SM resident, so the rest of the unified 256 KB stays L1 for the record
// and mask gathers (measured: 1.584 vs 1.597 ms with the driver's default; PFT_CARVEOUT=<percent>
// overrides).
template <typename T>
static int persistent_cap() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& cap = cache[dev & 63];
  if (cap != 0) return cap;
  int per_sm = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int carve = -1;
  if (const char* e = getenv("PFT_CARVEOUT")) {
    carve = atoi(e);
  } else {
    cudaFuncAttributes fa;
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (cudaFuncGetAttributes(&fa, k_track_persistent<T>) == cudaSuccess && smem_sm > 0)
      carve = (int)((100.0 * PFT_PERSIST_MINB * ((double)fa.sharedSizeBytes + (double)kPersistDynSmem + 1024.0) + smem_sm - 1) /
                    smem_sm);
  }
  cudaFuncSetAttribute(k_track_persistent<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPersistDynSmem);
  if (carve >= 0 && carve <= 100)
    cudaFuncSetAttribute(k_track_persistent<T>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_track_persistent<T>, kPT, kPersistDynSmem);
  cap = per_sm * sms;
  if (cap > 148 * 8) cap = 148 * 8;
  if (cap < 1) cap = -1;
  return cap;
}

static unsigned long long watchdog_ns() {
  static const unsigned long long ns = [] {
    const char* e = getenv("PFT_WATCHDOG_MS");
    const long long ms = e ? atoll(e) : 5000;
    return (unsigned long long)(ms > 0 ? ms : 5000) * 1000000ull;
  }();
  return ns;
}

// Persistent single-launch tracker: cooperative launch, all CTAs co-resident.  G = 1; or G rank
// groups of CTAs in one launch (fused one-GPU emulation of F2, each group in its own workspace
// region); or one group per GPU with the peers' exchange buffers attached (pft_comm_p2p_attach).
template <typename T>
static pft_status track_persistent(Launch& c, const uint16_t* depth, const pft_intrinsics* K, const double* T_init,
                                   const float* pst, int Kp, const pft_track_params* prm, double* T_out, double* E,
                                   int32_t* n_out, double* trace) {
  const int cap = persistent_cap<T>();
  if (cap < 1) return fail(PFT_ERR_CUDA, "persistent tracker does not fit on the device");
  pft_volume* vol = c.vol;
  const bool emul = vol->virtual_fused && vol->nranks > 1;
  const int G = (emul || vol->p2p) ? vol->nranks : 1;
  const int nb = emul ? cap / G : cap;
  if (nb < 1) return fail(PFT_ERR_INVALID_ARG, "%d rank groups do not fit in %d co-resident CTAs", G, cap);
  const int grid = emul ? nb * G : nb;
  const size_t region = c.L.region;
  for (int q = 0; q < (emul ? G : 1); ++q) {
    char* w = c.ws + (size_t)q * region;
    cudaMemsetAsync(w + c.L.state_off, 0, sizeof(TrackState), c.st);
    cudaMemsetAsync(w + c.L.work_off, 0, sizeof(unsigned) * (size_t)prm->iters, c.st);
  }
  PArgs pa;
  pa.R = vol->base + vol->L.r_off;
  pa.V = vol->base + vol->L.v_off;
  pa.mask = (const unsigned long long*)(vol->base + vol->L.m_off);
  pa.g = vol->g;
  pa.f = frame_of(c, depth, K);
  pa.sc = c.sched();
  pa.pst = pst;
  pa.K = Kp; pa.conv = prm->delta_conv; pa.iters = prm->iters; pa.rule = prm->update_rule; pa.guard = prm->guard;
  static const int sched = [] { const char* e = getenv("PFT_EVAL_SCHED"); return e ? atoi(e) : 0; }();
  pa.sched = sched;
  static const int tail_pct = [] { const char* e = getenv("PFT_TAIL_PCT"); return e ? atoi(e) : 5; }();
  pa.tail_pct = tail_pct;
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const bool pair_env = [] { const char* e = getenv("PFT_PAIR_SM"); return !(e && e[0] == '0'); }();
    pa.pair_sm = (pair_env && !emul && G == 1 && grid == 2 * sms) ? 1 : 0;
  }
  pa.beta = prm->beta; pa.rho = prm->min_inband_frac; pa.omega0 = prm->omega0_deg; pa.v0 = prm->v0_cm;
  pa.sr = StopRule{prm->min_search_deg, prm->min_search_cm, prm->stall_limit};
  pa.T_init = T_init;
  pa.E_out = E; pa.n_out = n_out; pa.trace = trace; pa.T_out = T_out;
  static const bool timing = [] { const char* e = getenv("PFT_PHASE_TIMING"); return e && e[0] == '1'; }();
  pa.tdone = (timing && !emul) ? (unsigned long long*)(c.ws + c.L.work_off + 1024 * sizeof(unsigned)) : nullptr;
  pa.topk = prm->topk;
  pa.watchdog_ns = watchdog_ns();
  pa.ws = c.ws;
  pa.rank_stride = region;
  pa.o_state = c.L.state_off;
  pa.o_acc = c.L.acc_local_off;
  pa.o_ptab = c.L.ptab_off;
  pa.o_pflag = c.L.ptab_off + 12 * sizeof(double) * (size_t)Kp;
  pa.o_mtab = c.L.mtab_off;
  pa.o_upart = c.L.part_off;
  pa.o_cpart = c.L.cpart_off;
  pa.o_work = c.L.work_off;
  pa.o_ckey = c.L.topk_off;
  pa.o_cidx = c.L.topk_off + sizeof(unsigned long long) * kTopkMax * (size_t)c.L.nblk_upd;
  pa.o_tkout = c.L.topk_off + (sizeof(unsigned long long) + sizeof(int)) * kTopkMax * (size_t)c.L.nblk_upd;
  pa.G = G;
  pa.rank = emul ? 0 : (G > 1 ? vol->rank : 0);
  pa.emul = emul ? 1 : 0;
  for (int q = 0; q < kMaxFusedRanks; ++q) pa.xbuf[q] = nullptr;
  pa.o_xcnt = 0;
  pa.xhalf = 0;
  if (emul) {
    for (int q = 0; q < G; ++q) pa.xbuf[q] = c.ws + (size_t)q * region + c.L.xch_off;
    pa.o_xcnt = c.L.xcnt_rel;
    pa.xhalf = (size_t)c.L.kfull;  // emulation: one launch at a time, so a per-call stride is safe
    // the counters are monotone across calls (pft.h: F2 exchange); a new workspace starts them at 0
    // the counters' location depends on the layout (K, G), not only on the workspace pointer
    if (vol->xws_last != c.ws || vol->xws_total != c.L.total || vol->xws_region != region ||
        vol->xws_xcnt != c.L.xch_off + c.L.xcnt_rel) {
      for (int q = 0; q < G; ++q)
        cudaMemsetAsync(pa.xbuf[q] + pa.o_xcnt, 0, (kMaxFusedRanks + 1) * sizeof(unsigned long long), c.st);
      vol->xws_last = c.ws;
      vol->xws_total = c.L.total;
      vol->xws_region = region;
      vol->xws_xcnt = c.L.xch_off + c.L.xcnt_rel;
    }
  } else if (G > 1) {
    if (Kp > vol->xmax_particles)
      return fail(PFT_ERR_INVALID_ARG, "%d particles exceed the exchange buffer's %d", Kp, vol->xmax_particles);
    for (int q = 0; q < G; ++q) pa.xbuf[q] = vol->xbuf[q];
    pa.o_xcnt = vol->xcnt_off;
    pa.xhalf = (size_t)G * (size_t)((vol->xmax_particles + G - 1) / G);
  }
  void* args[] = {&pa};
  cudaError_t e = cudaSuccess;
  PFT_LAUNCH(PFT_PROF_TRACK, c.st,
             e = cudaLaunchCooperativeKernel((const void*)k_track_persistent<T>, dim3(grid), dim3(kPT), args,
                                             kPersistDynSmem, c.st));
  if (e == cudaErrorCooperativeLaunchTooLarge && G == 1 && !emul) {
    cudaGetLastError();  // not sticky: the SMs are partly taken (e.g. by another context)
    return PFT_ERR_UNSUPPORTED;  // the caller falls back to the multi-launch tracker
  }
  if (e != cudaSuccess) return fail(PFT_ERR_CUDA, "persistent tracker launch: %s", cudaGetErrorString(e));
#ifdef PFT_WARP_UTIL
  {
    static unsigned long long h[4096][4];
    cudaStreamSynchronize(c.st);
    cudaMemcpyFromSymbol(h, g_wutil, sizeof h);
    const int nw = grid * (kPT / 32);
    double t[4] = {0, 0, 0, 0};
    for (int w = 0; w < nw; ++w)
      for (int q = 0; q < 4; ++q) t[q] += (double)h[w][q];
    const double tot = t[0] + t[1] + t[2] + t[3];
    printf("pft warp util (P2, per warp, us per launch): staging %.1f  eval %.1f  reduce %.1f  idle-at-end %.1f  (eval share %.3f)\n",
           t[0] / nw * 1e-3, t[1] / nw * 1e-3, t[2] / nw * 1e-3, t[3] / nw * 1e-3, t[1] / tot);
    static unsigned long long zero[4096][4];
    cudaMemcpyToSymbol(g_wutil, zero, sizeof zero);
  }
#endif
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
  // (a communicator attached -- even a single-rank one -- selects the collective multi-launch path)
  if (((G == 1 && !c.vol->nccl_comm) || c.vol->virtual_fused || c.vol->p2p) && use_persistent() && prm->iters <= 1024) {
    const pft_status s = track_persistent<T>(c, depth, K, T_init, pst, Kp, prm, T_out, E, n_out, trace);
    if (s != PFT_ERR_UNSUPPORTED) return s;
    // the cooperative grid does not fit right now (G = 1): same results from the multi-launch path
  }
  const int kloc = c.L.kloc;
  const int k_begin = c.L.points_part ? 0 : r * kloc;
  PartRec* local = (PartRec*)(c.ws + c.L.acc_local_off);
  PartRec* full = (PartRec*)(c.ws + c.L.acc_full_off);
  launch_prologue(c, depth, K, T_init, prm->omega0_deg, prm->v0_cm);
  if (c.L.points_part) cudaMemsetAsync(c.ws + c.L.cacc_off, 0, 2 * sizeof(unsigned long long), c.st);
  int prev_set = -1;
  for (int it = 0; it < prm->iters; ++it) {
    const int j = it % c.L.nsched;
    const int Ki = c.L.sched_K[j], set = c.L.sched_set[j];
    if (set != prev_set) {  // baseline on the new set (L11)
      const pft_status s = launch_centre<T>(c, 0, set, it, Ki, prm, trace);
      if (s != PFT_OK) return s;
    }
    prev_set = set;
    if (c.L.points_part) {
      // F2b: all K_i particles on this rank's point slice (virtual: every slice in turn into the same
      // accumulators), the per-particle sums added across the ranks in place (exact integers)
      const int npad = c.set(set).npad;
      for (int q = 0; q < G; ++q) {
        if (c.vol->virtual_ranks <= 1 && q != r) continue;
        int pb, pe;
        point_slice(npad, G, q, pb, pe);
        launch_eval<T>(c, 0, pst, 0, Ki, prm->delta_conv, nullptr, local, set, pb, pe);
      }
      if (c.vol->virtual_ranks <= 1) {
        const pft_status s = comm_allreduce_u64(c.vol, local, 2 * (size_t)Ki, c.st);
        if (s != PFT_OK) return s;
      }
    } else if (c.vol->virtual_ranks > 1) {
      // virtual shards: rank q's evaluation, then its all-gather slot filled by a device copy
      for (int q = 0; q < G; ++q) {
        const int kb = q * kloc, kc = max(0, min(Ki, kb + kloc) - kb);
        launch_eval<T>(c, 0, pst, kb, kc, prm->delta_conv, nullptr, local, set);
        cudaMemcpyAsync(full + kb, local, sizeof(PartRec) * (size_t)kloc, cudaMemcpyDeviceToDevice, c.st);
        cudaMemsetAsync(local, 0, sizeof(PartRec) * (size_t)kloc, c.st);
      }
    } else {
      const int k_count = max(0, min(Ki, k_begin + kloc) - k_begin);
      launch_eval<T>(c, 0, pst, k_begin, k_count, prm->delta_conv, nullptr, local, set);
      if (G > 1 || c.vol->nccl_comm) {
        pft_status s = comm_allgather(c.vol, local, full, sizeof(PartRec) * (size_t)kloc, c.st);
        if (s != PFT_OK) return s;
      }
    }
    UpdArgs ua{prm->topk, (unsigned long long*)(c.ws + c.L.topk_off),
               (int*)(c.ws + c.L.topk_off + sizeof(unsigned long long) * kTopkMax * (size_t)c.L.nblk_upd),
               (double*)(c.ws + c.L.topk_off + (sizeof(unsigned long long) + sizeof(int)) * kTopkMax * (size_t)c.L.nblk_upd),
               c.state(), full, local, Ki, k_begin, kloc, pst, prm->delta_conv, prm->update_rule, set,
               prm->min_inband_frac, E, n_out, (double*)(c.ws + c.L.part_off)};
    PFT_LAUNCH(PFT_PROF_UPDATE, c.st, k_update<<<(Ki + 255) / 256, 256, 0, c.st>>>(ua));
    const pft_status s = launch_centre<T>(c, 1, set, it, Ki, prm, trace);
    if (s != PFT_OK) return s;
  }
  PFT_LAUNCH(PFT_PROF_UPDATE, c.st, k_track_finalize<<<(Kp + 255) / 256, 256, 0, c.st>>>(c.state(), Kp, E, n_out, T_out));
  return cuda_check("track");
}

// per-pose results of an eval_poses call
__global__ void k_finish_poses(const PartRec* acc, int M, const TrackState* st, double rho, double* E, int* n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  const PartRec r = acc[k];
  E[k] = fitness_of(r.S, r.n, rho, st->Nvalid[0]);
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
  if (p->update_rule != PFT_UPDATE_MEAN && p->update_rule != PFT_UPDATE_WEIGHTED && p->update_rule != PFT_UPDATE_TOPK)
    return fail(PFT_ERR_INVALID_ARG, "bad update_rule");
  if (p->update_rule == PFT_UPDATE_TOPK && (p->topk < 1 || p->topk > kTopkMax))
    return fail(PFT_ERR_INVALID_ARG, "topk must be in [1, %d]", kTopkMax);
  if (p->nsched < 0 || p->nsched > PFT_MAX_SCHED) return fail(PFT_ERR_INVALID_ARG, "nsched must be in [0,%d]", PFT_MAX_SCHED);
  if (!(p->min_search_deg >= 0.0) || !(p->min_search_cm >= 0.0)) return fail(PFT_ERR_INVALID_ARG, "min_search must be >= 0");
  if (p->stall_limit < 0) return fail(PFT_ERR_INVALID_ARG, "stall_limit must be >= 0");
  return PFT_OK;
}

// F2 pre-flight: one block; thread q < G stores this rank's token into slot [rank] of rank q's
// preflight array (system-scope release store over NVLink), then thread 0 polls its own array until
// every slot holds the round's token of its writer (acquire loads), for at most timeout_ns.
__global__ void k_p2p_preflight(PArgsX x, unsigned long long round, unsigned long long timeout_ns, int* ok) {
  const int q = threadIdx.x;
  if (q < x.G) {
    unsigned long long* dst = (unsigned long long*)(x.xbuf[q] + x.pre_off) + x.rank;
    const unsigned long long tok = (round << 8) | (unsigned long long)(x.rank + 1);
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(tok) : "memory");
  }
  __syncthreads();
  if (q != 0) return;
  const unsigned long long* mine = (const unsigned long long*)(x.xbuf[x.rank] + x.pre_off);
  const unsigned long long t0 = global_ns();
  int good = 1;
  for (int r = 0; r < x.G && good; ++r) {
    const unsigned long long want = (round << 8) | (unsigned long long)(r + 1);
    for (;;) {
      const unsigned long long v = ld_acquire_sys(mine + r);
      if (v == want) break;
      if (global_ns() - t0 > timeout_ns) { good = 0; break; }
      __nanosleep(64);
    }
  }
  *ok = good;
}

pft_status p2p_preflight(pft_volume* vol, int timeout_ms, int32_t* ok_out, cudaStream_t st) {
  PArgsX x;
  x.G = vol->nranks;
  x.rank = vol->rank;
  for (int q = 0; q < kMaxFusedRanks; ++q) x.xbuf[q] = q < vol->nranks ? vol->xbuf[q] : nullptr;
  x.pre_off = vol->xcnt_off + (kMaxFusedRanks + 1) * sizeof(unsigned long long);
  // the result word follows the kMaxFusedRanks tokens in this rank's own buffer
  int* d_ok = (int*)(vol->xown + x.pre_off + kMaxFusedRanks * sizeof(unsigned long long));
  int h_ok = 0;
  const unsigned long long round = ++vol->preflight_round;
  k_p2p_preflight<<<1, 32, 0, st>>>(x, round, (unsigned long long)timeout_ms * 1000000ull, d_ok);
  cudaMemcpyAsync(&h_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check("preflight");
  *ok_out = h_ok;
  return cuda_check("preflight");
}

// out = A * B for rigid 3x4 row-major [R|t] poses: (R_A R_B, R_A t_B + t_A).
__global__ void k_pose_compose(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ out) {
  const int i = threadIdx.x;  // threads 0..11: element (r, c)
  const int r = (i >> 2) % 3, c = i & 3;
  double v = A[4 * r + 0] * B[c] + A[4 * r + 1] * B[4 + c] + A[4 * r + 2] * B[8 + c];
  if (c == 3) v += A[4 * r + 3];
  __syncthreads();
  if (i < 12) out[i] = v;  // (out may alias A or B: every read happens before the barrier)
}

}  // namespace pft

using namespace pft;

extern "C" {

pft_status pft_pose_compose(const double* dev_A, const double* dev_B, double* dev_out, void* stream) {
  if (!dev_A || !dev_B || !dev_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  PFT_LAUNCH(PFT_PROF_OTHER, st, k_pose_compose<<<1, 32, 0, st>>>(dev_A, dev_B, dev_out));
  return cuda_check("pose_compose");
}

pft_status pft_track_workspace_bytes(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles,
                                     const pft_track_params* prm, size_t* bytes_out) {
  if (!vol || !bytes_out || !prm) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  TrackLayout L;
  pft_status s = track_layout(vol, K, nparticles, prm, vol->nranks, &L);
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
  s = track_layout(vol, K, nparticles, prm, vol->nranks, &c.L);
  if (s != PFT_OK) return s;
  if (ws_bytes < c.L.total) return fail(PFT_ERR_BUFFER_TOO_SMALL, "workspace %zu B < required %zu B", ws_bytes, c.L.total);
  if (((uintptr_t)dev_ws) % 256) return fail(PFT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (prm->update_rule == PFT_UPDATE_TOPK && nparticles > 256 * 256)
    return fail(PFT_ERR_UNSUPPORTED, "PFT_UPDATE_TOPK supports at most 65536 particles");
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
  // eval_poses is rank-local and uses the plain stride (no schedule)
  pft_track_params p1 = *prm;
  p1.nsched = 0;
  pft_status s = track_layout(vol, K, M, &p1, 1, &c.L);
  if (s != PFT_OK) return s;
  if (ws_bytes < c.L.total) return fail(PFT_ERR_BUFFER_TOO_SMALL, "workspace %zu B < required %zu B", ws_bytes, c.L.total);
  if (((uintptr_t)dev_ws) % 256) return fail(PFT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  // (the state's pose is initialised from pose 0; eval_poses never reads it)
  launch_prologue(c, dev_depth, K, dev_poses, 0.0, 0.0);
  PartRec* acc = (PartRec*)(c.ws + c.L.acc_local_off);
  if (vol->esize == 4) launch_eval<float>(c, 1, nullptr, 0, M, 0, dev_poses, acc, 0);
  else launch_eval<__half>(c, 1, nullptr, 0, M, 0, dev_poses, acc, 0);
  PFT_LAUNCH(PFT_PROF_UPDATE, c.st, k_finish_poses<<<(M + 255) / 256, 256, 0, c.st>>>(acc, M, c.state(), prm->min_inband_frac, dev_E, dev_inband));
  return cuda_check("eval_poses");
}

pft_status pft_track_info(const void* dev_ws, int32_t* npoints_out, void* stream) {
  if (!dev_ws || !npoints_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  int n = 0;
  const TrackState* s = (const TrackState*)dev_ws;  // state is at offset 0 of every layout
  if (cudaMemcpyAsync(&n, &s->Nvalid[0], sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check("track_info");
  *npoints_out = n;
  return PFT_OK;
}

}  // extern "C"
