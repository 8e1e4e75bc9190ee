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

// R factor only, shapes read from the device bond table: for a tall m x n
// panel (m > n) writes the n x n upper-triangular R (the right singular vectors
// and singular values of A are those of R); otherwise copies A.  The effective
// row count (min(m, n)) is written to bonds[c*ld + out_idx].  One CTA per chain,
// panel in shared memory (bytes <= qr_r_smem_limit).
constexpr size_t QR_R_SMEM_LIMIT = 200 * 1024;  // + up to 16 KB static (reflector scalars)
// Preconditioner of the truncated split (Drmac-Veselic style): for the
// l x k matrix M = A (trans = 0) or A^H (trans = 1) compute M = Q1 R1 with
// r0 = min(l, k) and write Q1 (l x r0, row-major, nullable) and R1^H
// (k x r0, row-major); r0 goes to bonds[c*ld + out_idx].  Applied twice
// (the second time to R1^H without Q) it yields L = R2^H with
// M = Q1 L Q2, on which one-sided Jacobi needs a few sweeps instead of tens
// for the graded spectra of MPS splits.  Shared memory holds l*k elements.
template <typename T>
cudaError_t qr_precondition(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                            int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                            const ChainState* st, int chains, cudaStream_t s);

// Blocked variant of qr_precondition for l <= 256 and a panel that fits one
// CTA's shared memory (qr_small.cu): warp-level register panels + block
// reflector updates.  Returns cudaErrorInvalidValue when not applicable.
constexpr size_t QR_SMALL_SMEM_LIMIT = 216 * 1024;
size_t qr_small_bytes(int l, int k, bool cplx_);
template <typename T>
cudaError_t qr_precondition_unblocked(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                                      int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                                      const ChainState* st, int chains, cudaStream_t s);
template <typename T>
cudaError_t qr_precondition_small(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                                  int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                                  const ChainState* st, int chains, cudaStream_t s);

template <typename T>
cudaError_t qr_r_factor(const void* A, long long sA, DimExpr M, DimExpr N, int* bonds, int ld, int out_idx, void* R,
                        long long sR, int mmax, int nmax, int chains, cudaStream_t s);
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
  void* T;   // ceil(k/32) x 32 x 32 inner + (ceil(k/128) + 1) x 128 x 128 outer WY factors / S scratch
  void* W1;  // 128 x n
  void* W2;  // 128 x n
  void* P;   // panel scratch m x 32 (global fallback of the panel kernel)
  long long sA, sV, sT, sW, sP;  // per-chain strides
  int keep_wy = 0;  // R only, but complete every outer WY factor so V / T can apply Q later
  int two_level = -1;  // -1: by shape (qr_two_level); 0 / 1: force 32-column / 128-column trailing updates
};
constexpr int QR_NB = 32;
constexpr int QR_NBO = 128;  // outer block: trailing and Q updates use K = 128 (two-level blocking)
template <typename T> size_t qr_blocked_elems(int m, int n, size_t* sA, size_t* sV, size_t* sT, size_t* sW, size_t* sP);
// dst (cols x rows) = src^H (rows x cols), row-major, batched
template <typename T>
cudaError_t conj_transpose(const void* src, long long s_src, int rows, int cols, void* dst, long long s_dst, int chains,
                           cudaStream_t s);
// p.Q == nullptr: R only (no Q formation)
template <typename T>
cudaError_t householder_qr_blocked(const QrParams& p, const QrBlockedWork& w, int chains, cudaStream_t s,
                                   long long* launches);
// Two-level blocking is used for k = min(m, n) >= 512 (the only case householder_apply_q supports).
inline bool qr_two_level(int m, int n) { return (m < n ? m : n) >= 512; }
// X (m x r, row-major, ld r) <- Q X for the thin Q (m x k) of a two-level blocked QR run with
// keep_wy (V: m x k reflectors with ld k, Tw: its T workspace), i.e. Q M = H_1 .. H_k [M; 0]
// when X holds M (k x r) on top of zeros: the backward Q formation applied to X instead of the
// identity, 4 m k r flops instead of forming Q (about 2 m k^2) and multiplying.  W1, W2: 128 x r.
template <typename T>
cudaError_t householder_apply_q(const void* V, const void* Tw, int m, int k, void* X, int r, void* W1, void* W2,
                                cudaStream_t s, long long* launches);

}  // namespace ttg
