// Gather-replay ceiling (SURVEY.md §8(d-3) roofline denominator (4)): replays the evaluation's
// exact address stream -- per (particle, point) the cell's in-band mask word and then its 32-byte
// record (record 0 when out of band), in the tracker's work-item order (TILES tiles x 16 particles per
// warp item from one dynamic queue, TILES points per lane batched; the tracker uses 6 since round 2) -- with no transform and no lerp.
// The packed index stream (bit 31 in-band, bits 0..30 the record index) is precomputed on the host
// by tools/gather_replay.py and streamed with evict-first loads (157 MB per iteration at config Q),
// prefetched two particles ahead so that its HBM latency is not part of the replayed chain (r01
// loaded it in line, which put an HBM round trip in front of every mask -> record pair and made the
// ceiling pessimistic).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o libreplay.so replay.cu
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ void ld32(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

template <int TILES>
__global__ __launch_bounds__(256, 2) void k_replay(const uint32_t* __restrict__ idx, int K, int npad,
                                                   const float* __restrict__ rec, const unsigned* __restrict__ mask,
                                                   unsigned* __restrict__ queue, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int ngroups = (npad + 32 * TILES - 1) / (32 * TILES), nch = (K + 15) / 16;
  const int nitems = ngroups * nch;
  float acc = 0.f;
  for (;;) {
    int item = 0;
    if (lane == 0) item = (int)atomicAdd(queue, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= nitems) break;
    const int group = item / nch, chunk = item - group * nch;
    const int k0 = chunk * 16, k1 = min(K, k0 + 16);
    // the index stream is prefetched two particles ahead (registers), so its HBM latency is off the
    // replayed chain: what remains is the tracker's own dependent pair, mask word -> record
    const uint32_t* base = idx + (group * TILES) * 32 + lane;
    bool in[TILES];  // slots beyond npad (the last group) replay as out of range (index word 0)
#pragma unroll
    for (int p = 0; p < TILES; ++p) in[p] = (group * TILES + p) * 32 + lane < npad;
    uint32_t wn[2][TILES];
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int p = 0; p < TILES; ++p) wn[d][p] = k0 + d < k1 && in[p] ? __ldcs(base + (size_t)(k0 + d) * npad + p * 32) : 0u;
    for (int k = k0; k < k1; ++k) {
      uint32_t w[TILES], mw[TILES];
#pragma unroll
      for (int p = 0; p < TILES; ++p) { w[p] = wn[0][p]; wn[0][p] = wn[1][p]; }
#pragma unroll
      for (int p = 0; p < TILES; ++p) wn[1][p] = k + 2 < k1 && in[p] ? __ldcs(base + (size_t)(k + 2) * npad + p * 32) : 0u;
#pragma unroll
      for (int p = 0; p < TILES; ++p) mw[p] = __ldg(mask + ((w[p] & 0x7fffffffu) >> 5));
#pragma unroll
      for (int p = 0; p < TILES; ++p) {
        const uint32_t o = w[p] & 0x7fffffffu;
        const uint32_t inb = (w[p] >> 31) & (mw[p] >> (o & 31u));  // the mask is all ones: inb, with the dependency
        float v[8];
        ld32(rec + (size_t)(o * inb) * 8, v);
        acc += inb ? fabsf(v[0] + v[7]) : 0.f;
      }
    }
  }
  if (acc == 1234.5f) out[blockIdx.x] = acc;
}
}  // namespace

extern "C" int replay_run(const uint32_t* idx, int K, int npad, const float* rec, const unsigned* mask, int reps,
                          unsigned* queue, float* out, float* ms_out, int tiles) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaMemset(queue, 0, 4);
    cudaEventRecord(e0);
    if (tiles == 6) k_replay<6><<<296, 256>>>(idx, K, npad, rec, mask, queue, out);
    else k_replay<4><<<296, 256>>>(idx, K, npad, rec, mask, queue, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;  // the first run is a warm-up
  }
  *ms_out = best;
  return (int)cudaGetLastError();
}
