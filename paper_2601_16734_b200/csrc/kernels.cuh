// Expansion kernels (apply_raw, hadamard) and the small per-chain kernels of
// the sweep engine (norms, stop rules, copies).
#pragma once

#include "common.cuh"

namespace ttg {

// mpo.hpp:213-238.  C[(cb*Al+al), j, (cb2*Ar+ar)] = sum_i W[cb,j,i,cb2] A[al,i,ar]
template <typename T>
cudaError_t expand_mpo(const T* W, const T* A, T* C, int Dl, int dout, int din, int Dr, int Al, int Ar, int chains,
                       long long sA, long long sC, cudaStream_t s);

// blas.hpp:45-67.  C[(a*Bl+b), s, (a2*Br+b2)] = A[a,s,a2] B[b,s,b2]
template <typename T>
cudaError_t expand_hadamard(const T* A, const T* B, T* C, int Al, int d, int Ar, int Bl, int Br, int chains,
                            long long sA, long long sB, long long sC, cudaStream_t s);

// out[c] = |X_c|_F^2 with X_c having rows*cols elements
template <typename T>
cudaError_t frob2(const T* X, long long sX, DimExpr rows, DimExpr cols, const int* bonds, int ld, double* out,
                  long long s_out, int chains, cudaStream_t s);

// out[c * s_out] = max(0, Re X_c[0]) (a closed <T,T> environment chain, simplify.hpp:37-41)
template <typename T>
cudaError_t env_real(const T* X, long long sX, double* out, long long s_out, int chains, cudaStream_t s);

// End of a variational sweep (simplify.hpp:90, 114-125): dist2 from the
// centre tensor psi_0 (size elems), convergence + plateau rules.
template <typename T>
cudaError_t sweep_end(const T* psi0, long long s_psi0, DimExpr elems, const int* bonds, int ld, ChainState* st,
                      double simplification_tolerance, int sweep_index, int chains, cudaStream_t s);

// dst[c][0:rows*cols] = src[c][0:rows*cols]
template <typename T>
cudaError_t copy_dims(const T* src, long long s_src, T* dst, long long s_dst, DimExpr rows, DimExpr cols,
                        const int* bonds, int ld, const ChainState* st, int check_active, long long max_elems,
                        int chains, cudaStream_t s);

template <typename T>
cudaError_t fill_one(T* dst, long long s_dst, int chains, cudaStream_t s);

cudaError_t real_to_complex(const double* src, cplx* dst, long long n, cudaStream_t s);
// *flag |= 1 when any element of x has a non-zero imaginary part
cudaError_t any_imag(const cplx* x, long long n, int* flag, cudaStream_t s);
cudaError_t complex_to_real(const cplx* src, double* dst, long long n, cudaStream_t s);

// MPSSum::join block (mps.hpp:352-405): dst[offl + a, s, offr + b] += f * src[a, s, b]
// for a src tensor (a_dim x d x b_dim) inside dst (. x d x dst_right).
template <typename TS, typename TD>
cudaError_t join_block(const TS* src, int a_dim, int d, int b_dim, TD* dst, int dst_right, int offl, int offr,
                       double f_re, double f_im, cudaStream_t s);

// gather per-chain device tensors into one packed site buffer
template <typename T>
cudaError_t gather(const T* const* srcs, T* dst, long long elems, long long s_dst, int chains, cudaStream_t s);

cudaError_t init_state(ChainState* st, int chains, cudaStream_t s);
// active = |T| > fp_error_floor(1) (simplify.hpp:107-112)
cudaError_t begin_sweeps(ChainState* st, int chains, cudaStream_t s);
// x[c][0:elems] *= factors[c]
template <typename T>
cudaError_t scale_chains(T* x, long long s_x, long long elems, const double* factors, int chains, cudaStream_t s);
// bonds[c*ld + to] = bonds[c*ld + from]
cudaError_t copy_bond(int* bonds, int ld, int from, int to, int chains, cudaStream_t s);
cudaError_t set_bonds(int* bonds, const int* values, int ld, int count, int chains, cudaStream_t s);

}  // namespace ttg
