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
