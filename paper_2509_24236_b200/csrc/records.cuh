// records.cuh — the tracker's cell records and in-band mask, rebuilt from stored V:
// shared by the volume kernels (volume.cu) and the fused integration kernel (integrate.cu).
#pragma once
#include <cstdio>

#include "pft_internal.cuh"

namespace pft {

// Record of cell (cx,cy,cz): its 8 corner values, x fastest (exact copies of stored bits).
template <typename T> __device__ __forceinline__ float tof(T x);
template <> __device__ __forceinline__ float tof<float>(float x) { return x; }
template <> __device__ __forceinline__ float tof<__half>(__half x) { return __half2float(x); }

// Writes the record of cell (cx,cy,cz); returns whether the cell is in band (all |V| < 1).
template <typename T>
__device__ __forceinline__ bool build_record(const Geom& g, const T* __restrict__ V, T* __restrict__ R, int cx, int cy,
                                             int cz) {
  const uint32_t x0 = offx(cx), x1 = offx(cx + 1), y0 = offy(cy, g.sy), y1 = offy(cy + 1, g.sy);
  const uint32_t z0 = offz(cz, g.sz), z1 = offz(cz + 1, g.sz);
  T r[8] = {V[x0 + y0 + z0], V[x1 + y0 + z0], V[x0 + y1 + z0], V[x1 + y1 + z0],
            V[x0 + y0 + z1], V[x1 + y0 + z1], V[x0 + y1 + z1], V[x1 + y1 + z1]};
  T* dst = R + (size_t)(x0 + y0 + z0) * 8;
  if (sizeof(T) == 4) {
    // fp32 volumes: trilinear polynomial coefficients, computed in fp64 and rounded once:
    // v(f) = a + b fx + c fy + d fz + e fx fy + f fx fz + g fy fz + h fx fy fz
    double w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (double)*(const float*)&r[i];
    const double ca = w[0], cb = w[1] - w[0], cc = w[2] - w[0], cd = w[4] - w[0];
    const double ce = (w[3] - w[2]) - (w[1] - w[0]);
    const double cf = (w[5] - w[4]) - (w[1] - w[0]);
    const double cg = (w[6] - w[4]) - (w[2] - w[0]);
    const double ch = ((w[7] - w[6]) - (w[5] - w[4])) - ((w[3] - w[2]) - (w[1] - w[0]));
    float4* d = (float4*)dst;
    d[0] = make_float4((float)ca, (float)cb, (float)cc, (float)cd);
    d[1] = make_float4((float)ce, (float)cf, (float)cg, (float)ch);
  } else {
    uint4 u;
    u.x = (uint32_t)*(unsigned short*)&r[0] | ((uint32_t)*(unsigned short*)&r[1] << 16);
    u.y = (uint32_t)*(unsigned short*)&r[2] | ((uint32_t)*(unsigned short*)&r[3] << 16);
    u.z = (uint32_t)*(unsigned short*)&r[4] | ((uint32_t)*(unsigned short*)&r[5] << 16);
    u.w = (uint32_t)*(unsigned short*)&r[6] | ((uint32_t)*(unsigned short*)&r[7] << 16);
    *(uint4*)dst = u;
  }
  bool in = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) in = in && fabsf(tof<T>(r[i])) < 1.0f;
  return in;
}

// Dirty cell-bricks: 64 threads (two warps) rebuild the brick's 64 cell records and write the
// two 32-bit halves of its mask word by ballot; then the dirty flag is cleared.  Blocks
// [block, block + nblocks, ...) of 4 cell-bricks each.
template <typename T>
__device__ __forceinline__ void records_dirty_pass(const Geom& g, const T* __restrict__ V, T* __restrict__ R,
                                                   uint32_t* __restrict__ mask, uint32_t* __restrict__ dirty,
                                                   const uint32_t* __restrict__ dlist, uint32_t n, uint32_t block,
                                                   uint32_t nblocks) {
  const uint32_t w = threadIdx.x & 63;
  const uint32_t step = nblocks * 4;
  uint32_t li = block * 4 + (threadIdx.x >> 6);
  uint32_t bn = li < n ? __ldcg(dlist + li) : 0u;
  for (; li < n; li += step) {
    const uint32_t b = bn;
    if (li + step < n) bn = __ldcg(dlist + li + step);  // the next cell-brick, in flight during this one
#ifdef PFT_DEBUG
    if (b >= (uint32_t)g.nbx * g.nby * g.nbz) {
      printf("pft debug: bad dirty cell-brick %u\n", b);
      __trap();
    }
#endif
    const int bx = (int)(b % (uint32_t)g.nbx);
    const uint32_t r = b / (uint32_t)g.nbx;
    const int by = (int)(r % (uint32_t)g.nby), bz = (int)(r / (uint32_t)g.nby);
    const int cx = bx * 4 + (int)(w & 3), cy = by * 4 + (int)((w >> 2) & 3), cz = bz * 4 + (int)(w >> 4);
    bool in = false;
    if (cx <= g.nx - 2 && cy <= g.ny - 2 && cz <= g.nz - 2) in = build_record<T>(g, V, R, cx, cy, cz);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if ((threadIdx.x & 31) == 0) mask[b * 2 + (w >> 5)] = bal;
    if (w == 0) dirty[b] = 0u;
  }
}

}  // namespace pft
