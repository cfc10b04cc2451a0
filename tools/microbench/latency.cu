// Dependent-chain latency of fp64 operations on one thread (cycles per op, clock64): DFMA, DADD,
// sqrt, IEEE division, sincos -- the serial pose-algebra phases of the tracker are such chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, double seed, int n, long long* cyc) {
  double x = seed, y = 1.0000001;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = fma(x, y, 0.5);
    if (OP == 1) x = x + y;
    if (OP == 2) x = sqrt(x) + 1.0;
    if (OP == 3) x = y / x + 1.0;
    if (OP == 4) { double s, c; sincos(x, &s, &c); x = s + c; }
    if (OP == 5) { float f = (float)x; x = (double)(f * 1.0001f); }
    if (OP == 6) x = fmaf((float)x, 1.0001f, 0.5f);
  }
  const long long t1 = clock64();
  out[0] = x;
  *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, double* d, long long* c) {
  const int n = 1000;
  k<OP><<<1, 1>>>(d, 1.5, n, c);
  k<OP><<<1, 1>>>(d, 1.5, n, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %.1f cycles per dependent step\n", name, (double)h / n);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  run<0>("DFMA", d, c);
  run<1>("DADD", d, c);
  run<2>("sqrt + DADD", d, c);
  run<3>("IEEE div + DADD", d, c);
  run<4>("sincos + DADD", d, c);
  run<5>("F2F.F32.F64 + FMUL + F2F.F64.F32", d, c);
  run<6>("F2F + FFMA + F2F", d, c);
  return 0;
}
