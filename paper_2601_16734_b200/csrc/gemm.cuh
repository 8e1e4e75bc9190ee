// Batched FP64 / complex128 GEMM on the sm_100a DMMA tensor pipe.
//
// Replaces the Eigen products of the hot path: environment updates
// (environments.hpp:18-31), the two-site projection (forms.hpp:13-32), the
// QR/SVD carries (mps.hpp:202, 246, 261) and the scalar product chain
// (mps.hpp:416-423).  tcgen05.mma has no f64 kind, so the FP64 tensor path on
// B200 is the warp-level `mma.sync.m16n8k4.f64` (SASS: DMMA.8x8x4).
#pragma once

#include "common.cuh"

namespace ttg {

enum Op { OP_N = 0, OP_T = 1, OP_C = 2, OP_R = 3 };  // R = elementwise conjugate, no transpose

struct GemmParams {
  const void* A;
  const void* B;
  void* C;
  long long sA, sB, sC;  // per-chain strides in elements (0 = shared operand)
  DimExpr M, N, K;
  const int* bonds;
  int bonds_ld;
  const ChainState* st;  // nullable: chains with st[c].active == 0 are skipped
  double alpha;
  int beta;  // 0: C = alpha*op(A)op(B); 1: C += alpha*op(A)op(B)
  // leading dimensions (row strides, elements) of the stored A, B, C; 0 = compact
  long long lda = 0, ldb = 0, ldc = 0;
  // split-K partial tiles (set by gemm(): [chain][split][mmax][nmax], reduced in fixed order)
  void* ws = nullptr;
  int ws_m = 0, ws_n = 0;
  // 1: op(A) = A (OP_N / OP_R) is upper triangular or trapezoidal (A[i][k] = 0 for k < i), e.g. the R
  // factor carried into the next site (mps.hpp:202): output row tiles skip the k range left of the diagonal
  int a_upper = 0;
  int raster = 0;  // set by gemm(): tile rows per raster group (<= 1: row-major)
};

// Host launcher.  mmax/nmax bound M and N over all chains (grid sizing only);
// kmax (an upper bound of K, 0 = unknown) enables split-K for long, narrow products.
template <typename T>
cudaError_t gemm(const GemmParams& p, int opA, int opB, int mmax, int nmax, int chains, cudaStream_t s, int kmax = 0);

}  // namespace ttg
