// Householder QR with explicit thin Q (mps.hpp:193-205 HouseholderQR).
#pragma once

#include "common.cuh"

namespace ttg {

struct QrParams {
  const void* A;  // row-major m x n per chain
  long long sA;
  void* Q;        // row-major m x k
  long long sQ;
  void* R;        // row-major k x n
  long long sR;
  void* work;     // global scratch, qr_workspace_elems(m, n) per chain (used when it exceeds smem)
  long long s_work;
  int m, n;
};

template <typename T> size_t qr_workspace_elems(int m, int n);
template <typename T> cudaError_t householder_qr(const QrParams& p, int chains, cudaStream_t s);

}  // namespace ttg

namespace ttg {

// Blocked Householder QR (xGEQRF + xUNGQR structure) for panels that do not fit
// one CTA's shared memory: per 32-column panel one CTA per chain factors the
// panel and forms the compact-WY factor T (xLARFT), then the trailing matrix is
// updated with three batched DMMA GEMMs, A <- A - V T^H (V^H A); Q is built the
// same way backwards, Q <- Q - V T (V^H Q).  A is not modified (copied first).
struct QrBlockedWork {
  void* A;   // m x n working copy
  void* V;   // m x k unit lower-trapezoidal reflectors
  void* T;   // ceil(k/32) x 32 x 32 WY factors
  void* W1;  // 32 x n
  void* W2;  // 32 x n
  void* P;   // panel scratch m x 32 (global fallback of the panel kernel)
  long long sA, sV, sT, sW, sP;  // per-chain strides
};
constexpr int QR_NB = 32;
template <typename T> size_t qr_blocked_elems(int m, int n, size_t* sA, size_t* sV, size_t* sT, size_t* sW, size_t* sP);
template <typename T>
cudaError_t householder_qr_blocked(const QrParams& p, const QrBlockedWork& w, int chains, cudaStream_t s,
                                   long long* launches);

}  // namespace ttg
