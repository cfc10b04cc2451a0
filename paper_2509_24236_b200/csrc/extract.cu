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

template <typename T>
__global__ __launch_bounds__(256) void k_extract(Geom g, const T* __restrict__ V, const T* __restrict__ W,
                                                 double* __restrict__ pts, unsigned long long max_pts,
                                                 unsigned long long* __restrict__ count, size_t nelem) {
  const double inv_nbx = 1.0 / g.nbx, inv_nby = 1.0 / g.nby;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int kU = 4;  // elements per thread per round: their weight loads are in flight together
  for (size_t e00 = blockIdx.x * (size_t)blockDim.x; e00 < nelem; e00 += kU * stride) {
    double wts[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t e = e00 + u * stride + threadIdx.x;
      wts[u] = e < nelem ? ld64(W + e) : 0.0;
    }
#pragma unroll 1
    for (int u = 0; u < kU; ++u) {
      const size_t e0 = e00 + u * stride;
      if (e0 >= nelem) break;  // uniform across the block
      const size_t e = e0 + threadIdx.x;
      double p[3][3];
      int np = 0;
      // most voxels are unobserved (W = 0): the weight was loaded above
      if (e < nelem && wts[u] > 0.0) {
        const uint32_t b = (uint32_t)(e >> 6), w = (uint32_t)(e & 63);
        const uint32_t r = udiv_small(b, (uint32_t)g.nbx, inv_nbx);
        const int bx = (int)(b - r * (uint32_t)g.nbx);
        const uint32_t bz_ = udiv_small(r, (uint32_t)g.nby, inv_nby);
        const int by = (int)(r - bz_ * (uint32_t)g.nby), bz = (int)bz_;
        const int c[3] = {bx * 4 + (int)(w & 3), by * 4 + (int)((w >> 2) & 3), bz * 4 + (int)(w >> 4)};
        const int n[3] = {g.nx, g.ny, g.nz};
        if (c[0] < g.nx && c[1] < g.ny && c[2] < g.nz) {
          const double v0 = ld64(V + e);
          // +1 neighbour offsets in brick order
          const uint32_t step[3] = {(w & 3u) == 3u ? 64u - 3u : 1u, ((w >> 2) & 3u) == 3u ? g.sy - 12u : 4u,
                                    (w >> 4) == 3u ? g.sz - 48u : 16u};
          const double o[3] = {g.ox, g.oy, g.oz};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (c[a] + 1 >= n[a]) continue;
            const size_t e1 = e + step[a];
            if (!(ld64(W + e1) > 0.0)) continue;
            const double v1 = ld64(V + e1);
            if ((v0 > 0.0) == (v1 > 0.0) || (v0 == 0.0 && v1 == 0.0)) continue;
            const double t = __ddiv_rn(v0, __dsub_rn(v0, v1));
#pragma unroll
            for (int q = 0; q < 3; ++q) p[np][q] = __dadd_rn(o[q], __dmul_rn(g.voxel, __dadd_rn((double)c[q], 0.5)));
            p[np][a] = __dadd_rn(p[np][a], __dmul_rn(t, g.voxel));
            ++np;
          }
        }
      }
      // warp-aggregated append of up to 3 points per lane (skipped by warps without a point)
      if (!__any_sync(0xffffffffu, np > 0)) continue;
      unsigned long long total = np;
      const int lane = threadIdx.x & 31;
      unsigned long long incl = total;
      for (int s = 1; s < 32; s <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
      }
      const unsigned long long warp_sum = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long base = 0;
      if (lane == 31 && warp_sum) base = atomicAdd(count, warp_sum);
      base = __shfl_sync(0xffffffffu, base, 31);
      unsigned long long at = base + incl - total;
      for (int q = 0; q < np; ++q, ++at)
        if (at < max_pts) { pts[3 * at] = p[q][0]; pts[3 * at + 1] = p[q][1]; pts[3 * at + 2] = p[q][2]; }
    }
  }
}

}  // namespace pft

using namespace pft;

extern "C" pft_status pft_extract_surface(const pft_volume* vol, double* dev_points, int64_t max_points,
                                          int64_t* dev_count, void* stream) {
  if (!vol || !dev_count || (max_points > 0 && !dev_points)) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (max_points < 0) return fail(PFT_ERR_INVALID_ARG, "max_points must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(dev_count, 0, sizeof(int64_t), st);
  const size_t n = vol->L.elems;
  const int grid = 148 * 16;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_extract<float><<<grid, 256, 0, st>>>(vol->g, (const float*)(vol->base + vol->L.v_off),
        (const float*)(vol->base + vol->L.w_off), dev_points, (unsigned long long)max_points, (unsigned long long*)dev_count, n));
  else
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_extract<__half><<<grid, 256, 0, st>>>(vol->g, (const __half*)(vol->base + vol->L.v_off),
        (const __half*)(vol->base + vol->L.w_off), dev_points, (unsigned long long)max_points, (unsigned long long*)dev_count, n));
  return cuda_check("extract_surface");
}
