// Microbenchmark: FP64 tensor-core (mma.sync m8n8k4 f64, DMMA) vs DFMA issue
// rate on this GPU (decides DMMA vs DFMA formulations of the 1-D contractions).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) c[r] = fma(c[r], b, a);
  }
  double s = 0;
  for (int r = 0; r < 16; ++r) s += c[r];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 4; warps <= 32; warps *= 2) {
    k_dmma<<<sms, 32 * warps>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma<<<sms, 32 * warps>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * warps * sms;
    printf("DMMA warps/SM=%2d: %.1f TFLOP/s  (%.2f clk/DMMA/SM at 1.965 GHz)\n", warps, fl / ms / 1e9,
           ms * 1e-3 * 1.965e9 / ((double)iters * 8 * warps));
    k_dfma<<<sms, 32 * warps>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<<<sms, 32 * warps>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 32 * 16 * (double)iters * warps * sms;
    printf("DFMA warps/SM=%2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
