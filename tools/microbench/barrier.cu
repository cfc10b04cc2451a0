// Grid-barrier latency microbenchmark (DESIGN.md §7 "barriers"): 296 co-resident CTAs x 256
// threads (the persistent tracker's launch shape) pass NB barriers back to back.
//  V0: the tracker's sense-reversing barrier (fence; atomicAdd; last arriver flips a generation word)
//  V1: monotone counter: red.release.gpu add, every CTA polls ld.acquire.gpu until count >= target
//  V2: V1 without the nanosleep in the poll loop
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Bar { unsigned count, gen; unsigned long long mono; };

__device__ __forceinline__ void bar_v0(Bar* b, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&b->count, 1u);
    if (arrived == gridDim.x - 1) {
      b->count = 0u;
      __threadfence();
      atomicExch(&b->gen, gen + 1u);
    } else {
      while (*(volatile unsigned*)&b->gen == gen) __nanosleep(64);
    }
    __threadfence();
  }
  gen += 1u;
  __syncthreads();
}

template <bool SLEEP>
__device__ __forceinline__ void bar_v1(Bar* b, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&b->mono) : "memory");
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&b->mono) : "memory");
      if (v >= target) break;
      if (SLEEP) __nanosleep(32);
    }
  }
  __syncthreads();
}

template <int V>
__global__ void kern(Bar* b, int nb, int* out) {
  unsigned gen = 0;
  unsigned long long target = 0;
  int acc = 0;
  for (int i = 0; i < nb; ++i) {
    acc += threadIdx.x ^ i;
    if (V == 0) bar_v0(b, gen);
    if (V == 1) bar_v1<true>(b, target);
    if (V == 2) bar_v1<false>(b, target);
  }
  if (acc == 12345678) out[0] = acc;
}

template <int V>
void run(const char* name, Bar* b, int* o) {
  const int grid = 296, nb = 2000;
  cudaMemset(b, 0, sizeof(Bar));
  void* args[] = {&b, (void*)&nb, &o};
  int nbv = nb;
  args[1] = &nbv;
  cudaLaunchCooperativeKernel((const void*)kern<V>, dim3(grid), dim3(256), args, 0, 0);
  cudaDeviceSynchronize();
  cudaMemset(b, 0, sizeof(Bar));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((const void*)kern<V>, dim3(grid), dim3(256), args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s %.3f us per barrier (%s)\n", name, ms * 1e3 / nb, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Bar* b;
  int* o;
  cudaMalloc(&b, sizeof(Bar));
  cudaMalloc(&o, 4);
  run<0>("V0 sense-reversing (tracker)", b, o);
  run<1>("V1 monotone red.release/ld.acquire", b, o);
  run<2>("V2 monotone, no nanosleep", b, o);
  return 0;
}
