// Dependent-chain latencies on B200: DFMA, DMUL, cvt f64<->f32, MUFU.RSQ, LDS, __syncthreads.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) :: "memory"); return t; }
#define PIN_D(x) asm volatile("" : "+d"(x) :: "memory")
#define PIN_F(x) asm volatile("" : "+f"(x) :: "memory")
#define PIN_I(x) asm volatile("" : "+r"(x) :: "memory")
__global__ void k(double* out, long long* t, double a, double b, int nthreads_active) {
  __shared__ double sm[1024];
  sm[threadIdx.x] = a + threadIdx.x;
  __syncthreads();
  double x = a; float f = (float)b; int idx = threadIdx.x;
  long long t0, t1;
  // DFMA chain
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = fma(x, b, a);
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[0] = t1 - t0;
  // DMUL chain
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = x * b;
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[1] = t1 - t0;
  // cvt chain d->f->d
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 128; ++i) x = (double)((float)x) + 0.0;
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[2] = t1 - t0;
  // rsqrtf chain (float)
  f = (float)x;
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 256; ++i) f = rsqrtf(f) + 1.0f;
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[3] = t1 - t0;
  // FFMA chain
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 256; ++i) f = fmaf(f, 1.0001f, 0.5f);
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[4] = t1 - t0;
  // LDS dependent chain
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 128; ++i) idx = (int)sm[idx & 1023] & 1023;
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[5] = t1 - t0;
  // barrier
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 128; ++i) __syncthreads();
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[6] = t1 - t0;
  // double division chain
  PIN_D(x); PIN_F(f); PIN_I(idx); t0 = clk();
#pragma unroll
  for (int i = 0; i < 64; ++i) x = a / (x + 1.5);
  PIN_D(x); PIN_F(f); PIN_I(idx); t1 = clk();
  if (threadIdx.x == 0) t[7] = t1 - t0;
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* out; long long* t;
  cudaMalloc(&out, 8192); cudaMalloc(&t, 64);
  for (int nt : {32, 128, 512}) {
    k<<<1, nt>>>(out, t, 1.0000001, 0.9999999, nt);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %.1f  DMUL %.1f  cvt d->f->d+add %.1f  rsqrtf+fadd %.1f  FFMA %.1f  LDS-chain(+cvt) %.1f  syncthreads %.1f  ddiv+add %.1f cycles\n", nt,
           h[0] / 256.0, h[1] / 256.0, h[2] / 128.0, h[3] / 256.0, h[4] / 256.0, h[5] / 128.0, h[6] / 128.0, h[7] / 64.0);
  }
  return 0;
}
