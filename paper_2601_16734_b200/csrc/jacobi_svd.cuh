// Truncated split on the device: one-sided (Hestenes) Jacobi SVD with
// on-device truncation rank and dropped weight.
//
// Replaces schmidt_split + svd_with_retry + truncation_rank + dropped_weight
// (schmidt.hpp:18-89) as used by move_center_left (mps.hpp:253-265) and
// split_pair (mps.hpp:164-173).
#pragma once

#include "common.cuh"

namespace ttg {

struct SvdParams {
  const void* theta;  // row-major m x n per chain
  long long s_theta;
  DimExpr M, N;
  int* bonds;         // shapes are read from here; the truncation rank is written to bonds[c*ld + out_idx]
  int ld;
  int out_idx;
  void* iso;          // mode 0: U_r (m x r, row-major); mode 1: V_r^H (r x n, row-major)
  long long s_iso;
  double* svals;      // nullable: sorted singular values, min(m,n) per chain
  long long s_svals;
  ChainState* st;     // err2 ledger and status flags
  int check_active;   // skip chains with st.active == 0
  int accumulate_err; // st.err2 += dropped weight^2
  double tol;         // relative cutoff (strict >, schmidt.hpp:45)
  long long max_bond;
  int mode;           // 0 = LEFT_TO_RIGHT, 1 = RIGHT_TO_LEFT (schmidt.hpp:81-87)
  void* work;         // global scratch (l*k elements per chain) when the panel exceeds shared memory
  long long s_work;
};

template <typename T>
cudaError_t jacobi_svd(const SvdParams& p, int lmax, int kmax, int chains, cudaStream_t s);

}  // namespace ttg
