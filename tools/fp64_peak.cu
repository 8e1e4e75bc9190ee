// Microbenchmark: sustained FP64 throughput of DMMA (mma.sync f64) vs DFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double c[8][4];
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, b0 = a0 * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0; for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 123.456) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double c[8]; for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-3 + j;
  double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 123.456) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    int iters = 20000; dim3 grid(sms * 2), block(32 * warps);
    dmma_loop<<<grid, block>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); dmma_loop<<<grid, block>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
    printf("DMMA m16n8k4 warps/cta=%d ctas=%d: %.2f TFLOP/s\n", warps, grid.x, flops / ms / 1e9);
    dfma_loop<<<grid, block>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); dfma_loop<<<grid, block>>>(d, iters * 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * iters * 4.0 * (double)grid.x * block.x;
    printf("DFMA warps/cta=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
