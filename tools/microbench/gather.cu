// Random-gather ceiling microbenchmark (SURVEY.md §8(d-3) roofline denominator (1)): independent
// 32-byte (ld.global.nc.v8.f32, the tracker's record load) and 4-byte gathers at hashed addresses
// over footprints from L1-resident to HBM-resident, 296 CTAs x 256 threads with 8 loads in flight
// per thread.  Also the dependent pair the evaluation issues: a 4-byte mask word, then a 32-byte
// record at an address derived from it.  Prints one JSON object per line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void ld32(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// MODE 0: 32-B gathers; 1: 4-B gathers; 2: dependent 4-B -> 32-B pair
template <int MODE>
__global__ __launch_bounds__(256, 2) void k_gather(const float* __restrict__ base, uint32_t nrec, int iters,
                                                   float* __restrict__ out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  uint32_t h = hash32(tid * 0x9e3779b9U + 1u);
  for (int it = 0; it < iters; ++it) {
    uint32_t idx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { h = hash32(h + j); idx[j] = h % nrec; }
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v[8];
        ld32(base + (size_t)idx[j] * 8, v);
        acc += v[0] + v[7];
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += __ldg(base + idx[j]);
    } else {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = __float_as_uint(__ldg(base + (idx[j] & ~7u)));
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v[8];
        ld32(base + (size_t)((idx[j] ^ (w[j] & 1u)) % nrec) * 8, v);
        acc += v[0] + v[7];
      }
    }
  }
  if (acc == 1234.5f) out[tid] = acc;
}

template <int MODE>
static void run(const char* name, const float* d, size_t bytes, float* out) {
  const uint32_t nrec = (uint32_t)((MODE == 1 ? bytes / 4 : bytes / 32));
  const int grid = 296, iters = 64;
  k_gather<MODE><<<grid, 256>>>(d, nrec, 4, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_gather<MODE><<<grid, 256>>>(d, nrec, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)grid * 256 * iters * 8;  // gathers (pairs for MODE 2)
  printf("{\"test\": \"%s\", \"footprint_bytes\": %zu, \"gathers_per_s\": %.4e, \"ms\": %.3f, \"err\": \"%s\"}\n", name,
         bytes, n / (ms * 1e-3), ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t maxb = (size_t)4 << 30;
  float* d;
  float* out;
  if (cudaMalloc(&d, maxb) != cudaSuccess) return 1;
  cudaMalloc(&out, 296 * 256 * 4);
  cudaMemset(d, 0, maxb);
  const size_t fps[] = {(size_t)64 << 10, (size_t)1 << 20, (size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20,
                        (size_t)1 << 30, maxb};
  for (size_t b : fps) {
    run<0>("gather32", d, b, out);
    run<1>("gather4", d, b, out);
    run<2>("mask4_then_record32", d, b, out);
  }
  return 0;
}
