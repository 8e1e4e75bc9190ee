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
  int* sweeps_out;    // nullable: Jacobi sweeps executed per chain (diagnostics)
  double tol_rot;     // rotation threshold |a^H b| > tol_rot |a||b|; 0 = default l*eps
  int no_early;       // 1: iterate until a sweep rotates nothing (no early stop, see early_stop2)
  // Warm start.  theta_pre = theta F for mode 0 (F = V frame of the previous
  // split at this bond) or F^H theta for mode 1 (F = U frame); it has the same
  // singular values and the same isometry as theta.  It is used only when
  // frame_in[c*frame_ld] == m == n, i.e. the frame was square and complete.
  const void* theta_pre;
  long long s_pre;
  const int* frame_in;
  int* frame_out;     // written: m if the full orthonormal frame was stored, else 0
  int frame_ld;
  void* frame;        // full normalised frame (l x k row-major, columns sorted by singular value)
  long long s_frame;
  // retry policy (schmidt.hpp:23-35, see svd_jitter)
  int retry;          // 1: a non-converged first attempt flags ST_RETRY instead of ST_NOCONV
  int attempt;        // 0: first attempt; 1: relaunch for the chains flagged ST_RETRY
  int first_budget;   // > 0: sweep budget of the first attempt (forced-failure test hook)
};

// Shared-memory plan of the SVD kernel: per-column metadata plus, when it fits,
// the whole l x k working panel.  Otherwise the panel lives in `work`.
constexpr size_t SVD_SMEM_LIMIT = 220 * 1024;
inline size_t jacobi_svd_meta_bytes(long long kmax) { return (size_t)kmax * (2 * sizeof(double) + sizeof(int)) + 16; }
inline bool jacobi_svd_panel_in_smem(long long lmax, long long kmax, size_t es) {
  return jacobi_svd_meta_bytes(kmax) + (size_t)(lmax | 1) * kmax * es <= SVD_SMEM_LIMIT;
}

template <typename T>
cudaError_t jacobi_svd(const SvdParams& p, int lmax, int kmax, int chains, cudaStream_t s);

// Grid-cooperative variant for a few large splits: the columns are grouped in
// blocks, every CTA of a cooperative grid owns one block pair per block round
// (its whole CTA works on the pair: rows split over threads, one cross-warp
// reduction per sub-round), and rounds are separated by grid-wide barriers.
// `work` must hold, per chain, jacobi_grid_work_bytes(lmax, kmax) bytes.
size_t jacobi_grid_work_bytes(int lmax, int kmax, size_t es);
bool jacobi_grid_eligible(int lmax, int kmax, int chains, size_t es);
template <typename T>
cudaError_t jacobi_svd_grid(const SvdParams& p, int lmax, int kmax, int chains, void* work, cudaStream_t s);


// Block-Gram variant for one large real split (jacobi_bg.cu): a cluster per block pair keeps the
// pair's rows in shared memory, rotates the pair's Gram matrix and applies the accumulated
// rotations by DMMA.  Same workspace as jacobi_svd_grid.  cudaErrorNotSupported when the
// cooperative cluster launch is not available (the caller falls back to the grid kernels).
bool jacobi_bg_eligible(int lmax, int kmax, int chains, size_t es);
cudaError_t jacobi_svd_bg(const SvdParams& p, int lmax, int kmax, void* work, cudaStream_t s);

}  // namespace ttg

namespace ttg {
// Replace kept isometry vectors of numerically-zero singular values (sigma^2 <=
// l^2 eps^2 |theta|_F^2) by orthonormal completions; needs p.svals (sorted,
// min(m,n) per chain) from the preceding Jacobi launch.  lmax = isometry vector
// length bound, kmax = rank bound.
size_t iso_complete_smem(int lmax, int kmax, size_t es);
template <typename T>
cudaError_t iso_complete(const SvdParams& p, int lmax, int kmax, int chains, cudaStream_t s);
}  // namespace ttg

namespace ttg {
// In-place jitter of theta for the chains flagged ST_RETRY: theta[i][j] +=
// 1e-14 |theta|_F ((i + 31 j) % 7 / 7 + 1i ((3 i + j) % 5 / 5)) (schmidt.hpp:29-31;
// real theta takes the real part).  Chains without the flag are untouched.
template <typename T>
cudaError_t svd_jitter(void* theta, long long s_theta, DimExpr M, DimExpr N, const int* bonds, int ld,
                       const ChainState* st, int chains, cudaStream_t s);
}  // namespace ttg
