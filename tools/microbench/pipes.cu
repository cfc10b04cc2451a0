// Pipe-throughput microbenchmark for the design decisions in DESIGN.md:
// fp64 FMA, fp32->fp64 conversion, fp64->int conversion, fp64 floor, fp32 FMA.
// Measured on B200 (r01): DFMA/DADD 62 op/clk/SM; every conversion (F2F either way, F2I from
// fp32 or fp64, FRND) 14-16 op/clk/SM (the XU pipe); FFMA 114 op/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
template <int OP>
__global__ void kern(double* out, float seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  float f0 = seed * threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  long long acc = 0;
  #pragma unroll 16
  for (int i = 0; i < N_IT; ++i) {
    if (OP == 0) { a0 = fma(a0, 1.0000001, 0.5); a1 = fma(a1, 1.0000001, 0.5); a2 = fma(a2, 1.0000001, 0.5); a3 = fma(a3, 1.0000001, 0.5); }
    if (OP == 1) { a0 += (double)f0; a1 += (double)f1; a2 += (double)f2; a3 += (double)f3; f0 += 1.f; f1 += 1.f; f2+=1.f; f3+=1.f; }
    if (OP == 2) { acc += __double2ll_rn(a0) + __double2ll_rn(a1) + __double2ll_rn(a2) + __double2ll_rn(a3); a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0; }
    if (OP == 3) { a0 = floor(a0) + 0.75; a1 = floor(a1) + 0.75; a2 = floor(a2) + 0.75; a3 = floor(a3) + 0.75; }
    if (OP == 4) { f0 = fmaf(f0, 1.0001f, 0.5f); f1 = fmaf(f1, 1.0001f, 0.5f); f2 = fmaf(f2, 1.0001f, 0.5f); f3 = fmaf(f3, 1.0001f, 0.5f); }
    if (OP == 6) { f0 += __double2float_rn(a0); f1 += __double2float_rn(a1); f2 += __double2float_rn(a2); f3 += __double2float_rn(a3); a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0; }
    if (OP == 7) { acc += __float2uint_rn(f0) + __float2uint_rn(f1) + __float2uint_rn(f2) + __float2uint_rn(f3); f0 += 1.f; f1 += 1.f; f2 += 1.f; f3 += 1.f; }
    if (OP == 8) { a0 = a0 + 1.0000001; a1 = a1 + 1.0000001; a2 = a2 + 1.0000001; a3 = a3 + 1.0000001; }
    if (OP == 5) { acc += __double2int_rd(a0) + __double2int_rd(a1) + __double2int_rd(a2) + __double2int_rd(a3); a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + f0 + f1 + f2 + f3 + (double)acc;
}
template <int OP> void run(const char* name, double ops_per_it, double* d) {
  int blocks = 148 * 8, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<OP><<<blocks, threads>>>(d, 1.f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<OP><<<blocks, threads>>>(d, 1.f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * blocks * threads * (double)N_IT * ops_per_it;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s %10.3f Gop/s  %.2f op/clk/SM (at max clk %d MHz)\n", name, ops / ms / 1e6, ops / (ms * 1e-3) / (148.0 * clk * 1e3), clk / 1000);
}
int main() {
  double* d; cudaMalloc(&d, 148 * 8 * 256 * 8);
  run<0>("DFMA", 4, d);
  run<1>("F2F.F64.F32 (+DADD)", 4, d);
  run<2>("F2I.S64.F64 (+DADD)", 4, d);
  run<3>("FRND.F64.FLOOR (+DADD)", 4, d);
  run<4>("FFMA", 4, d);
  run<5>("F2I.S32.F64.RM (+DADD)", 4, d);
  run<6>("F2F.F32.F64 (+FADD+DADD)", 4, d);
  run<7>("F2I.U32.F32 (+FADD+IADD)", 4, d);
  run<8>("DADD", 4, d);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("L2 bytes %d  SMs %d\n", l2, sms);
  return 0;
}
