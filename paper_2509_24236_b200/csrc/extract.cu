// extract.cu — NEXT row F4: zero-crossing surface points of the TSDF, the input
// of the completeness / accuracy metrics of PAPER.md:562-563.  For every voxel and axis whose +1
// neighbour is inside the grid, both observed (W > 0), values of different sign (not both 0):
//   t = V0 / (V0 - V1),  p = c0 + (t * s) e_a,   c0 = o + s (i + 1/2, j + 1/2, k + 1/2)
// evaluated in fp64 in this exact operation order (bit-identical to a plain evaluation).  Points
// are appended in no particular order (warp-aggregated atomics).
#include "pft_internal.cuh"

namespace pft {

template <typename T> __device__ __forceinline__ double ld64(const T* p);
template <> __device__ __forceinline__ double ld64<float>(const float* p) { return (double)__ldg(p); }
template <> __device__ __forceinline__ double ld64<__half>(const __half* p) { return (double)__half2float(__ldg(p)); }

// q = n / d for n < 2^31, d <= 4096: a double reciprocal estimate corrected by one step (exact,
// no integer-division loop)
__device__ __forceinline__ uint32_t udiv_small(uint32_t n, uint32_t d, double inv_d) {
  uint32_t q = (uint32_t)((double)n * inv_d);
  if (q * d > n) --q;
  else if ((q + 1) * d <= n) ++q;
  return q;
}

// The brick's 64 weights as two per lane in one 8-byte (fp32) / 4-byte (fp16) load: a brick is 64
// consecutive elements, so a warp reads it with one coalesced request.
template <typename T> __device__ __forceinline__ void ld_w2(const T* p, float& a, float& b);
template <> __device__ __forceinline__ void ld_w2<float>(const float* p, float& a, float& b) {
  const float2 v = __ldcs(reinterpret_cast<const float2*>(p));
  a = v.x;
  b = v.y;
}
template <> __device__ __forceinline__ void ld_w2<__half>(const __half* p, float& a, float& b) {
  const unsigned u = __ldcs(reinterpret_cast<const unsigned*>(p));
  a = __half2float(__ushort_as_half((unsigned short)(u & 0xffffu)));
  b = __half2float(__ushort_as_half((unsigned short)(u >> 16)));
}

// Brick-centric sweep: a warp streams the weights of kB bricks at once (one coalesced request per
// brick, all in flight together; evict-first: W is read once), and only bricks with an observed
// voxel (ballot) do the per-voxel work -- a few % of a room-scale grid -- with all of a voxel's
// loads (V, and W and V of its three +1 neighbours) in one round trip.  Points go to a per-warp
// shared-memory buffer flushed with one global atomic per 64 points.  Lane l owns voxels 2l and
// 2l + 1 of the brick (x = 2l & 3 and x + 1, y = (l >> 1) & 3, z = l >> 3).  Round 2: 0.40 ->
// 0.25 ms on the bench map (0.21 -> 0.35 of HBM for W of every voxel + V of the observed ones);
// the rest is the observed bricks' round trips, one brick at a time per warp.
#ifndef PFT_EXTRACT_MINB
#define PFT_EXTRACT_MINB 6  // 40 registers, 48 warps/SM: 0.250 ms vs 0.301 at 8 CTAs/SM (32 registers) on the bench map
#endif
template <typename T>
__global__ __launch_bounds__(256, PFT_EXTRACT_MINB) void k_extract(Geom g, const T* __restrict__ V, const T* __restrict__ W,
                                                 double* __restrict__ pts, unsigned long long max_pts,
                                                 unsigned long long* __restrict__ count, uint32_t nbricks) {
  constexpr int kB = 8;
  const double inv_nbx = 1.0 / g.nbx, inv_nby = 1.0 / g.nby;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr unsigned kBuf = 64;  // points per warp buffer
  __shared__ double sbuf[8][kBuf][3];
  double (*buf)[3] = sbuf[threadIdx.x >> 5];
  unsigned nbuf = 0;  // warp-uniform
  auto flush = [&]() {
    if (nbuf == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    for (unsigned q = lane; q < nbuf; q += 32)
      if (base + q < max_pts) {
        pts[3 * (base + q)] = buf[q][0]; pts[3 * (base + q) + 1] = buf[q][1]; pts[3 * (base + q) + 2] = buf[q][2];
      }
    __syncwarp();
    nbuf = 0;
  };
  for (uint32_t b00 = warp * kB; b00 < nbricks; b00 += nwarps * kB) {
    float wa[kB], wb[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      wa[q] = wb[q] = 0.f;
      if (b00 + q < nbricks) ld_w2(W + (size_t)(b00 + q) * 64 + 2 * lane, wa[q], wb[q]);
    }
#pragma unroll 1
    for (int q = 0; q < kB; ++q) {
      const uint32_t b = b00 + q;
      if (b >= nbricks) break;  // warp-uniform
      const bool obs0 = wa[q] > 0.f, obs1 = wb[q] > 0.f;
      if (!__any_sync(0xffffffffu, obs0 || obs1)) continue;  // no observed voxel in this brick
      const uint32_t r = udiv_small(b, (uint32_t)g.nbx, inv_nbx);
      const int bx = (int)(b - r * (uint32_t)g.nbx);
      const uint32_t bz_ = udiv_small(r, (uint32_t)g.nby, inv_nby);
      const int by = (int)(r - bz_ * (uint32_t)g.nby), bz = (int)bz_;
      double p[6][3];
      int np = 0;
      // all loads of the brick's observed voxels first (V of the voxel, W and V of its three +1
      // neighbours: one round trip instead of a V -> W -> V chain per axis), then the decisions
      float v0f[2], w1f[2][3], v1f[2][3];
      bool ok[2];
      int cc[2][3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t w = 2u * (uint32_t)lane + (uint32_t)h;
        const size_t e = (size_t)b * 64 + w;
        cc[h][0] = bx * 4 + (int)(w & 3); cc[h][1] = by * 4 + (int)((w >> 2) & 3); cc[h][2] = bz * 4 + (int)(w >> 4);
        ok[h] = (h == 0 ? obs0 : obs1) && cc[h][0] < g.nx && cc[h][1] < g.ny && cc[h][2] < g.nz;
        const uint32_t step[3] = {(w & 3u) == 3u ? 64u - 3u : 1u, ((w >> 2) & 3u) == 3u ? g.sy - 12u : 4u,
                                  (w >> 4) == 3u ? g.sz - 48u : 16u};
        const int n[3] = {g.nx, g.ny, g.nz};
        v0f[h] = ok[h] ? (float)ld64(V + e) : 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const bool in = ok[h] && cc[h][a] + 1 < n[a];
          const size_t e1 = in ? e + step[a] : e;
          w1f[h][a] = in ? (float)ld64(W + e1) : 0.f;
          v1f[h][a] = in ? (float)ld64(V + e1) : 0.f;
        }
      }
      const double o[3] = {g.ox, g.oy, g.oz};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!ok[h]) continue;
        const double v0 = (double)v0f[h];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!((double)w1f[h][a] > 0.0)) continue;  // unobserved or outside the grid
          const double v1 = (double)v1f[h][a];
          if ((v0 > 0.0) == (v1 > 0.0) || (v0 == 0.0 && v1 == 0.0)) continue;
          const double t = __ddiv_rn(v0, __dsub_rn(v0, v1));
#pragma unroll
          for (int d = 0; d < 3; ++d) p[np][d] = __dadd_rn(o[d], __dmul_rn(g.voxel, __dadd_rn((double)cc[h][d], 0.5)));
          p[np][a] = __dadd_rn(p[np][a], __dmul_rn(t, g.voxel));
          ++np;
        }
      }
      // append into the warp's shared-memory buffer; one global atomic per 64 buffered points
      // (one per brick with points was a hot spot: every warp of the grid on one counter)
      if (!__any_sync(0xffffffffu, np > 0)) continue;
      unsigned incl = (unsigned)np;
      for (int s = 1; s < 32; s <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
      }
      const unsigned warp_sum = __shfl_sync(0xffffffffu, incl, 31);
      if (nbuf + warp_sum > kBuf) flush();
      if (warp_sum > kBuf) {  // (rare: more points than the buffer holds) straight to global memory
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(count, (unsigned long long)warp_sum);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long at = base + incl - (unsigned)np;
        for (int q2 = 0; q2 < np; ++q2, ++at)
          if (at < max_pts) { pts[3 * at] = p[q2][0]; pts[3 * at + 1] = p[q2][1]; pts[3 * at + 2] = p[q2][2]; }
        continue;
      }
      for (int q2 = 0; q2 < np; ++q2) {
        const unsigned at = nbuf + incl - (unsigned)np + (unsigned)q2;
        buf[at][0] = p[q2][0]; buf[at][1] = p[q2][1]; buf[at][2] = p[q2][2];
      }
      nbuf += warp_sum;
      __syncwarp();
    }
  }
  flush();
}

}  // namespace pft

using namespace pft;

extern "C" pft_status pft_extract_surface(const pft_volume* vol, double* dev_points, int64_t max_points,
                                          int64_t* dev_count, void* stream) {
  if (!vol || !dev_count || (max_points > 0 && !dev_points)) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (max_points < 0) return fail(PFT_ERR_INVALID_ARG, "max_points must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(dev_count, 0, sizeof(int64_t), st);
  const uint32_t nb = (uint32_t)(vol->L.elems / 64);
  // one wave of co-resident CTAs (the loop strides over the bricks), 8 bricks of weights in flight per warp
  const int grid = 148 * PFT_EXTRACT_MINB;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_extract<float><<<grid, 256, 0, st>>>(vol->g, (const float*)(vol->base + vol->L.v_off),
        (const float*)(vol->base + vol->L.w_off), dev_points, (unsigned long long)max_points, (unsigned long long*)dev_count, nb));
  else
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_extract<__half><<<grid, 256, 0, st>>>(vol->g, (const __half*)(vol->base + vol->L.v_off),
        (const __half*)(vol->base + vol->L.w_off), dev_points, (unsigned long long)max_points, (unsigned long long*)dev_count, nb));
  return cuda_check("extract_surface");
}
