// Shared device/host definitions for the ttgpu sm_100a library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ttg {

// Complex128 as an interleaved (re, im) pair, the layout of std::complex<double>
// and of the reference's Tensor3 storage (tensor.hpp:13-86).
struct __align__(16) cplx {
  double x, y;
};

template <typename T> struct Scalar;
template <> struct Scalar<double> {
  static constexpr bool is_complex = false;
  __host__ __device__ static double zero() { return 0.0; }
  __host__ __device__ static double one() { return 1.0; }
};
template <> struct Scalar<cplx> {
  static constexpr bool is_complex = true;
  __host__ __device__ static cplx zero() { return {0.0, 0.0}; }
  __host__ __device__ static cplx one() { return {1.0, 0.0}; }
};

__host__ __device__ inline double conj_(double a) { return a; }
__host__ __device__ inline cplx conj_(cplx a) { return {a.x, -a.y}; }
__host__ __device__ inline double abs2(double a) { return a * a; }
__host__ __device__ inline double abs2(cplx a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ inline double add(double a, double b) { return a + b; }
__host__ __device__ inline cplx add(cplx a, cplx b) { return {a.x + b.x, a.y + b.y}; }
__host__ __device__ inline double sub(double a, double b) { return a - b; }
__host__ __device__ inline cplx sub(cplx a, cplx b) { return {a.x - b.x, a.y - b.y}; }
__host__ __device__ inline double mul(double a, double b) { return a * b; }
__host__ __device__ inline cplx mul(cplx a, cplx b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__host__ __device__ inline double scale(double a, double s) { return a * s; }
__host__ __device__ inline cplx scale(cplx a, double s) { return {a.x * s, a.y * s}; }
// conj(a) * b
__host__ __device__ inline double cmul(double a, double b) { return a * b; }
__host__ __device__ inline cplx cmul(cplx a, cplx b) { return {a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x}; }
__host__ __device__ inline bool finite_(double a) { return isfinite(a); }
__host__ __device__ inline bool finite_(cplx a) { return isfinite(a.x) && isfinite(a.y); }

// A matrix dimension that is either a host constant or `mult` times a bond
// dimension read from device memory (`bonds[chain * ld + idx]`).  Truncation
// ranks are produced on the device, so kernels that follow an SVD read their
// shapes instead of having the host wait for them.
struct DimExpr {
  int idx;   // < 0: constant
  int mult;  // multiplier (or the constant)
  __host__ __device__ int eval(const int* bonds, int chain, int ld) const {
    return idx < 0 ? mult : mult * bonds[chain * ld + idx];
  }
};
__host__ inline DimExpr dconst(int v) { return DimExpr{-1, v}; }
__host__ inline DimExpr dbond(int idx, int mult = 1) { return DimExpr{idx, mult}; }

// Per-chain run state for batched sweeps (one entry per chain).
struct ChainState {
  double target_norm2;  // <T,T>
  double err2;          // canonical-form truncation ledger (sum of squares)
  double dist2;         // last sweep's |T|^2 - |psi|^2
  double prev_dist2;
  int sweeps;
  int active;           // 1 while the variational loop runs for this chain
  int converged;
  int status;           // 0 ok, else TTG_NUMERIC bit flags
};

enum StatusBits { ST_NONFINITE = 1, ST_NOCONV = 2, ST_RETRY = 4 };  // ST_RETRY: split pending a jitter retry

}  // namespace ttg

// Debug build switch -DTTG_SMEM_POISON: kernels with a dynamic shared-memory panel start by filling it with NaN
// bit patterns, so a read of shared memory the kernel did not write shows up at once instead of depending on
// what the previous kernel on that SM left behind.
__device__ __forceinline__ void ttg_smem_poison(void* dyn) {
#ifdef TTG_SMEM_POISON
  unsigned nbytes;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(nbytes));
  unsigned long long* q = static_cast<unsigned long long*>(dyn);
  for (unsigned i = threadIdx.x; i < nbytes / 8; i += blockDim.x) q[i] = 0xFFFFFFFFFFFFFFFFull;
  __syncthreads();
#else
  (void)dyn;
#endif
}

