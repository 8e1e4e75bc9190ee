// Householder QR with explicit thin Q, one CTA per chain.
//
// Replaces Eigen::HouseholderQR in the exact left-to-right pass of the
// CanonicalMPS constructor (mps.hpp:193-205): for the (left*phys) x right
// unfolding A = Q R with k = min(m, n), Q (m x k, isometry) and R (k x n,
// upper trapezoidal).  Reflectors follow LAPACK's xGEQR2/xUNG2R conventions
// (beta = -sign(Re alpha) |x|, H = I - tau v v^H, v_0 = 1).  The working copy
// is column-major so that every reflector touches contiguous memory; it lives
// in shared memory when it fits, else in an L2-resident global workspace.
#include "qr.cuh"

#include <algorithm>
#include <cfloat>
#include <cstdlib>

namespace ttg {
namespace {

constexpr int QR_THREADS = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < nw ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

template <typename T>
__global__ void __launch_bounds__(QR_THREADS) qr_kernel(QrParams p, int in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[33];
  __shared__ T s_tau;
  const int chain = blockIdx.x;
  const int m = p.m, n = p.n, k = min(m, n);
  ttg_smem_poison(smem_raw);
  T* Wk = in_smem ? reinterpret_cast<T*>(smem_raw) : static_cast<T*>(p.work) + p.s_work * chain;
  T* E = Wk + (size_t)m * n;
  T* tau = E + (size_t)m * k;
  const T* A = static_cast<const T*>(p.A) + p.sA * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  for (int idx = tid; idx < m * n; idx += blockDim.x) {
    const int i = idx / n, c = idx % n;
    Wk[(size_t)c * m + i] = A[idx];
  }
  __syncthreads();

  for (int j = 0; j < k; ++j) {
    T* v = Wk + (size_t)j * m;
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += blockDim.x) part += abs2(v[i]);
    const double xn2 = block_sum(part, red);
    if (tid == 0) {
      const T alpha = v[j];
      double ar, ai;
      if constexpr (Scalar<T>::is_complex) {
        ar = alpha.x;
        ai = alpha.y;
      } else {
        ar = alpha;
        ai = 0.0;
      }
      T t = Scalar<T>::zero();
      if (!(xn2 == 0.0 && ai == 0.0)) {
        const double beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        if constexpr (Scalar<T>::is_complex) {
          t = cplx{(beta - ar) / beta, -ai / beta};
          // scal = 1 / (alpha - beta)
          const double dr = ar - beta, di = ai, den = dr * dr + di * di;
          const cplx sc{dr / den, -di / den};
          red[0] = sc.x;
          red[1] = sc.y;
          v[j] = cplx{beta, 0.0};
        } else {
          t = (beta - ar) / beta;
          red[0] = 1.0 / (ar - beta);
          red[1] = 0.0;
          v[j] = beta;
        }
      } else {
        red[0] = 1.0;
        red[1] = 0.0;
      }
      s_tau = t;
      tau[j] = t;
    }
    __syncthreads();
    T sc;
    if constexpr (Scalar<T>::is_complex)
      sc = cplx{red[0], red[1]};
    else
      sc = red[0];
    for (int i = j + 1 + tid; i < m; i += blockDim.x) v[i] = mul(v[i], sc);
    __syncthreads();
    const T ct = conj_(s_tau);
    // A[j:, c] -= conj(tau) v (v^H A[j:, c]) for c > j
    for (int c = j + 1 + warp; c < n; c += nwarps) {
      T* a = Wk + (size_t)c * m;
      T w = Scalar<T>::zero();
      for (int i = j + lane; i < m; i += 32) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
        w = add(w, cmul(vi, a[i]));
      }
      if constexpr (Scalar<T>::is_complex) {
        w.x = warp_sum(w.x);
        w.y = warp_sum(w.y);
      } else {
        w = warp_sum(w);
      }
      const T f = mul(ct, w);
      for (int i = j + lane; i < m; i += 32) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
        a[i] = sub(a[i], mul(vi, f));
      }
    }
    __syncthreads();
  }

  // R (k x n, row-major, explicit zeros below the diagonal)
  T* R = static_cast<T*>(p.R) + p.sR * chain;
  for (int idx = tid; idx < k * n; idx += blockDim.x) {
    const int i = idx / n, c = idx % n;
    R[idx] = (c >= i) ? Wk[(size_t)c * m + i] : Scalar<T>::zero();
  }
  // Q = H_0 ... H_{k-1} I[:, :k], accumulated backwards (xUNG2R)
  for (int idx = tid; idx < m * k; idx += blockDim.x) {
    const int c = idx / m, i = idx % m;
    E[idx] = (i == c) ? Scalar<T>::one() : Scalar<T>::zero();
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const T* v = Wk + (size_t)j * m;
    const T tj = tau[j];
    for (int c = j + warp; c < k; c += nwarps) {
      T* e = E + (size_t)c * m;
      T w = Scalar<T>::zero();
      for (int i = j + lane; i < m; i += 32) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
        w = add(w, cmul(vi, e[i]));
      }
      if constexpr (Scalar<T>::is_complex) {
        w.x = warp_sum(w.x);
        w.y = warp_sum(w.y);
      } else {
        w = warp_sum(w);
      }
      const T f = mul(tj, w);
      for (int i = j + lane; i < m; i += 32) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
        e[i] = sub(e[i], mul(vi, f));
      }
    }
    __syncthreads();
  }
  T* Q = static_cast<T*>(p.Q) + p.sQ * chain;
  for (int idx = tid; idx < m * k; idx += blockDim.x) {
    const int i = idx / k, c = idx % k;
    Q[idx] = E[(size_t)c * m + i];
  }
}

template <typename T>
__global__ void __launch_bounds__(QR_THREADS) qr_r_kernel(const T* A, long long sA, DimExpr M, DimExpr N, int* bonds,
                                                           int ld, int out_idx, T* R, long long sR) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[33];
  __shared__ T s_tau;
  const int chain = blockIdx.x;
  const int m = M.eval(bonds, chain, ld), n = N.eval(bonds, chain, ld);
  ttg_smem_poison(smem_raw);
  A += sA * chain;
  R += sR * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (m <= n) {
    for (int idx = tid; idx < m * n; idx += blockDim.x) R[idx] = A[idx];
    if (tid == 0) bonds[chain * ld + out_idx] = m;
    return;
  }
  T* Wk = reinterpret_cast<T*>(smem_raw);
  for (int idx = tid; idx < m * n; idx += blockDim.x) {
    const int i = idx / n, c = idx % n;
    Wk[c * m + i] = A[idx];
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    T* v = Wk + j * m;
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += blockDim.x) part += abs2(v[i]);
    const double xn2 = block_sum(part, red);
    if (tid == 0) {
      const T alpha = v[j];
      double ar, ai;
      if constexpr (Scalar<T>::is_complex) {
        ar = alpha.x;
        ai = alpha.y;
      } else {
        ar = alpha;
        ai = 0.0;
      }
      T t = Scalar<T>::zero();
      red[0] = 1.0;
      red[1] = 0.0;
      if (!(xn2 == 0.0 && ai == 0.0)) {
        const double beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        if constexpr (Scalar<T>::is_complex) {
          t = cplx{(beta - ar) / beta, -ai / beta};
          const double dr = ar - beta, di = ai, den = dr * dr + di * di;
          red[0] = dr / den;
          red[1] = -di / den;
          v[j] = cplx{beta, 0.0};
        } else {
          t = (beta - ar) / beta;
          red[0] = 1.0 / (ar - beta);
          v[j] = beta;
        }
      }
      s_tau = t;
    }
    __syncthreads();
    T sc;
    if constexpr (Scalar<T>::is_complex)
      sc = cplx{red[0], red[1]};
    else
      sc = red[0];
    for (int i = j + 1 + tid; i < m; i += blockDim.x) v[i] = mul(v[i], sc);
    __syncthreads();
    const T ct = conj_(s_tau);
    for (int c = j + 1 + warp; c < n; c += nwarps) {
      T* a = Wk + c * m;
      T w = Scalar<T>::zero();
      for (int i = j + lane; i < m; i += 32) w = add(w, cmul(i == j ? Scalar<T>::one() : v[i], a[i]));
      if constexpr (Scalar<T>::is_complex) {
        w.x = warp_sum(w.x);
        w.y = warp_sum(w.y);
      } else {
        w = warp_sum(w);
      }
      const T f = mul(ct, w);
      for (int i = j + lane; i < m; i += 32) a[i] = sub(a[i], mul(i == j ? Scalar<T>::one() : v[i], f));
    }
    __syncthreads();
  }
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int i = idx / n, c = idx % n;
    R[idx] = (c >= i) ? Wk[c * m + i] : Scalar<T>::zero();
  }
  if (tid == 0) bonds[chain * ld + out_idx] = n;
}

// a_c[j:] -= f v (v^H a_c[j:]) for the columns c in [c0, c1) handled by this
// warp, four at a time so that the four reductions overlap.
template <typename T>
__device__ __forceinline__ void apply_reflector_cols(T* Wk, int l, int lw, const T* v, int j, T f_scale, int c0,
                                                     int c1, int warp, int nwarps, int lane) {
  for (int cb = c0 + warp; cb < c1; cb += 4 * nwarps) {
    T w[4];
    T* a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = cb + u * nwarps;
      a[u] = Wk + (c < c1 ? c : c0) * lw;
      w[u] = Scalar<T>::zero();
    }
    for (int i = j + lane; i < l; i += 32) {
      const T vi = (i == j) ? Scalar<T>::one() : v[i];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = add(w[u], cmul(vi, a[u][i]));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if constexpr (Scalar<T>::is_complex) {
        w[u].x = warp_sum(w[u].x);
        w[u].y = warp_sum(w[u].y);
      } else {
        w[u] = warp_sum(w[u]);
      }
      w[u] = mul(f_scale, w[u]);
    }
    for (int i = j + lane; i < l; i += 32) {
      const T vi = (i == j) ? Scalar<T>::one() : v[i];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (cb + u * nwarps < c1) a[u][i] = sub(a[u][i], mul(vi, w[u]));
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(QR_THREADS) qr_pre_kernel(const T* A, long long sA, DimExpr Md, DimExpr Nd, int trans,
                                                             int* bonds, int ld, int out_idx, T* Q, long long sQ,
                                                             T* RH, long long sRH, const ChainState* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T s_tau;
  __shared__ T taus[1024];
  const int chain = blockIdx.x;
  if (st && !st[chain].active) return;
  ttg_smem_poison(smem_raw);
  const int mi = Md.eval(bonds, chain, ld), ni = Nd.eval(bonds, chain, ld);
  const bool out_r = (trans & 2) != 0;  // write R (r0 x k) instead of R^H
  trans &= 1;
  const int l = trans ? ni : mi, k = trans ? mi : ni, r0 = min(l, k);
  const int lw = l | 1;  // odd column stride: transposing loads/stores are bank-conflict free
  A += sA * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  T* Wk = reinterpret_cast<T*>(smem_raw);
  // W[c*l + i] = M[i, c]
  for (int idx = tid; idx < mi * ni; idx += blockDim.x) {
    const int r = idx / ni, c = idx % ni;
    if (trans)
      Wk[r * lw + c] = conj_(A[idx]);
    else
      Wk[c * lw + r] = A[idx];
  }
  __syncthreads();
  // Column j: warp 0 forms the reflector (norm, beta, tau, scaling of v) without
  // a block-wide reduction; one barrier publishes it, all warps update the
  // trailing columns, one barrier closes the step.
  for (int j = 0; j < r0; ++j) {
    T* v = Wk + j * lw;
    if (warp == 0) {
      double part = 0.0;
      for (int i = j + 1 + lane; i < l; i += 32) part += abs2(v[i]);
      const double xn2 = warp_sum(part);
      const T alpha = v[j];
      double ar, ai;
      if constexpr (Scalar<T>::is_complex) {
        ar = alpha.x;
        ai = alpha.y;
      } else {
        ar = alpha;
        ai = 0.0;
      }
      T t = Scalar<T>::zero();
      T sc = Scalar<T>::one();
      double beta = ar;
      const bool refl = !(xn2 == 0.0 && ai == 0.0);
      if (refl) {
        beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        if constexpr (Scalar<T>::is_complex) {
          t = cplx{(beta - ar) / beta, -ai / beta};
          const double dr = ar - beta, di = ai, den = dr * dr + di * di;
          sc = cplx{dr / den, -di / den};
        } else {
          t = (beta - ar) / beta;
          sc = 1.0 / (ar - beta);
        }
      }
      for (int i = j + 1 + lane; i < l; i += 32) v[i] = mul(v[i], sc);
      if (lane == 0) {
        if (refl) {
          if constexpr (Scalar<T>::is_complex)
            v[j] = cplx{beta, 0.0};
          else
            v[j] = beta;
        }
        s_tau = t;
        taus[j] = t;
      }
    }
    __syncthreads();
    apply_reflector_cols<T>(Wk, l, lw, v, j, conj_(s_tau), j + 1, k, warp, nwarps, lane);
    __syncthreads();
  }
  // R1^H (k x r0): RH[c, i] = conj(R1[i, c]) for c >= i; with trans & 2: R1 itself (r0 x k)
  T* rh = RH + sRH * chain;
  if (out_r) {
    for (int idx = tid; idx < r0 * k; idx += blockDim.x) {
      const int i = idx / k, c = idx % k;
      rh[idx] = (c >= i) ? Wk[c * lw + i] : Scalar<T>::zero();
    }
  } else {
    for (int idx = tid; idx < k * r0; idx += blockDim.x) {
      const int c = idx / r0, i = idx % r0;
      rh[idx] = (c >= i) ? conj_(Wk[c * lw + i]) : Scalar<T>::zero();
    }
  }
  if (tid == 0) bonds[chain * ld + out_idx] = r0;
  if (!Q) return;
  __syncthreads();
  // Q1 in place over the reflectors (xORG2R), columns 0..r0-1
  for (int j = r0 - 1; j >= 0; --j) {
    T* v = Wk + j * lw;
    const T tj = taus[j];
    apply_reflector_cols<T>(Wk, l, lw, v, j, tj, j + 1, r0, warp, nwarps, lane);  // (xORG2R)
    __syncthreads();
    for (int i = tid; i < l; i += blockDim.x) {
      if (i < j)
        v[i] = Scalar<T>::zero();
      else if (i == j)
        v[i] = sub(Scalar<T>::one(), tj);
      else
        v[i] = mul(sub(Scalar<T>::zero(), tj), v[i]);
    }
    __syncthreads();
  }
  T* q = Q + sQ * chain;
  for (int idx = tid; idx < l * r0; idx += blockDim.x) {
    const int i = idx / r0, c = idx % r0;
    q[idx] = Wk[c * lw + i];
  }
}

}  // namespace

template <typename T>
cudaError_t qr_precondition(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                            int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                            const ChainState* st, int chains, cudaStream_t s) {
  static const bool small_off = [] {
    const char* e = std::getenv("TTG_QR_SMALL");
    return e && e[0] == '0';
  }();
  if (!small_off && lmax <= 256 && qr_small_bytes(lmax, kmax, Scalar<T>::is_complex) <= QR_SMALL_SMEM_LIMIT)
    return qr_precondition_small<T>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH, lmax, kmax, st, chains, s);
  return qr_precondition_unblocked<T>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH, lmax, kmax, st, chains,
                                      s);
}

template <typename T>
cudaError_t qr_precondition_unblocked(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                                      int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                                      const ChainState* st, int chains, cudaStream_t s) {
  const size_t bytes = (size_t)(lmax | 1) * kmax * sizeof(T);
  if (bytes > QR_R_SMEM_LIMIT || (lmax < kmax ? lmax : kmax) > 1024) return cudaErrorInvalidValue;
  cudaError_t e =
      cudaFuncSetAttribute(qr_pre_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_R_SMEM_LIMIT);
  if (e != cudaSuccess) return e;
  qr_pre_kernel<T><<<chains, QR_THREADS, bytes, s>>>(static_cast<const T*>(A), sA, M, N, trans, bonds, ld, out_idx,
                                                    static_cast<T*>(Q), sQ, static_cast<T*>(RH), sRH, st);
  return cudaGetLastError();
}

template cudaError_t qr_precondition_unblocked<double>(const void*, long long, DimExpr, DimExpr, int, int*, int, int,
                                                       void*, long long, void*, long long, int, int,
                                                       const ChainState*, int, cudaStream_t);
template cudaError_t qr_precondition_unblocked<cplx>(const void*, long long, DimExpr, DimExpr, int, int*, int, int,
                                                     void*, long long, void*, long long, int, int, const ChainState*,
                                                     int, cudaStream_t);
template cudaError_t qr_precondition<double>(const void*, long long, DimExpr, DimExpr, int, int*, int, int, void*,
                                             long long, void*, long long, int, int, const ChainState*, int,
                                             cudaStream_t);
template cudaError_t qr_precondition<cplx>(const void*, long long, DimExpr, DimExpr, int, int*, int, int, void*,
                                           long long, void*, long long, int, int, const ChainState*, int,
                                           cudaStream_t);

template <typename T>
cudaError_t qr_r_factor(const void* A, long long sA, DimExpr M, DimExpr N, int* bonds, int ld, int out_idx, void* R,
                        long long sR, int mmax, int nmax, int chains, cudaStream_t s) {
  const size_t bytes = (size_t)mmax * nmax * sizeof(T);
  if (bytes > QR_R_SMEM_LIMIT) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(qr_r_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_R_SMEM_LIMIT);
  if (e != cudaSuccess) return e;
  qr_r_kernel<T><<<chains, QR_THREADS, bytes, s>>>(static_cast<const T*>(A), sA, M, N, bonds, ld, out_idx,
                                                  static_cast<T*>(R), sR);
  return cudaGetLastError();
}

template cudaError_t qr_r_factor<double>(const void*, long long, DimExpr, DimExpr, int*, int, int, void*, long long,
                                         int, int, int, cudaStream_t);
template cudaError_t qr_r_factor<cplx>(const void*, long long, DimExpr, DimExpr, int*, int, int, void*, long long,
                                       int, int, int, cudaStream_t);

template <typename T>
size_t qr_workspace_elems(int m, int n) {
  const int k = m < n ? m : n;
  return (size_t)m * n + (size_t)m * k + (size_t)k + 2;
}

template <typename T>
cudaError_t householder_qr(const QrParams& p, int chains, cudaStream_t s) {
  if (chains <= 0 || p.m <= 0 || p.n <= 0) return cudaSuccess;
  const size_t bytes = qr_workspace_elems<T>(p.m, p.n) * sizeof(T);
  const size_t limit = 200 * 1024;
  const int in_smem = bytes <= limit;
  if (!in_smem && p.work == nullptr) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(qr_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
  if (e != cudaSuccess) return e;
  qr_kernel<T><<<chains, QR_THREADS, in_smem ? bytes : 0, s>>>(p, in_smem);
  return cudaGetLastError();
}

template size_t qr_workspace_elems<double>(int, int);
template size_t qr_workspace_elems<cplx>(int, int);
template cudaError_t householder_qr<double>(const QrParams&, int, cudaStream_t);
template cudaError_t householder_qr<cplx>(const QrParams&, int, cudaStream_t);

}  // namespace ttg

// ---------------------------------------------------------------------------
// blocked QR
// ---------------------------------------------------------------------------
#include <cooperative_groups.h>

#include "gemm.cuh"

namespace ttg {
namespace {

namespace cg = cooperative_groups;
constexpr int PANEL_THREADS = 512;

// xLARFT (forward, columnwise) by one warp: T[i,i] = tau_i,
// T[0:i,i] = -tau_i T[0:i,0:i] S[0:i,i]; lane r owns row r of T and only reads
// back its own row (global Tp, no shared-memory copy).
template <typename T>
__device__ __forceinline__ void warp_larft(const T (&S)[QR_NB][QR_NB + 1], const T* taus, int jr, int lane, T* Tp) {
  T* row = Tp + lane * QR_NB;
  for (int c = 0; c < QR_NB; ++c) row[c] = Scalar<T>::zero();
  for (int i = 0; i < jr; ++i) {
    const T ti = taus[i];
    if (lane < i) {
      T acc = Scalar<T>::zero();
      for (int c = lane; c < i; ++c) acc = add(acc, mul(row[c], S[c][i]));
      row[i] = mul(sub(Scalar<T>::zero(), ti), acc);
    } else if (lane == i) {
      row[i] = ti;
    }
  }
}

// Factor the mp x jb panel A[j0:, j0:j0+jb] (row stride lda) in place, write the
// unit lower-trapezoidal V into Vall[j0:, j0:j0+jb] (row stride k) and the
// jb x jb upper-triangular WY factor into Tp.
template <typename T>
__global__ void __launch_bounds__(PANEL_THREADS) qr_panel_kernel(T* A, long long sA, int lda, int mp, int jb, T* Vall,
                                                                  long long sV, int ldv, T* Tall, long long sT,
                                                                  T* Pg, long long sP, int in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[33];
  __shared__ T s_tau;
  __shared__ T taus[QR_NB];
  __shared__ T S[QR_NB][QR_NB + 1];
  const int chain = blockIdx.x;
  A += sA * chain;
  Vall += sV * chain;
  T* Tp = Tall + sT * chain;
  T* P = in_smem ? reinterpret_cast<T*>(smem_raw) : Pg + sP * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  for (int idx = tid; idx < mp * jb; idx += blockDim.x) {
    const int r = idx / jb, c = idx % jb;
    P[(size_t)c * mp + r] = A[(size_t)r * lda + c];
  }
  __syncthreads();
  for (int j = 0; j < jb && j < mp; ++j) {
    T* v = P + (size_t)j * mp;
    double part = 0.0;
    for (int i = j + 1 + tid; i < mp; i += blockDim.x) part += abs2(v[i]);
    const double xn2 = block_sum(part, red);
    if (tid == 0) {
      const T alpha = v[j];
      double ar, ai;
      if constexpr (Scalar<T>::is_complex) {
        ar = alpha.x;
        ai = alpha.y;
      } else {
        ar = alpha;
        ai = 0.0;
      }
      T t = Scalar<T>::zero();
      if (!(xn2 == 0.0 && ai == 0.0)) {
        const double beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        if constexpr (Scalar<T>::is_complex) {
          t = cplx{(beta - ar) / beta, -ai / beta};
          const double dr = ar - beta, di = ai, den = dr * dr + di * di;
          red[0] = dr / den;
          red[1] = -di / den;
          v[j] = cplx{beta, 0.0};
        } else {
          t = (beta - ar) / beta;
          red[0] = 1.0 / (ar - beta);
          red[1] = 0.0;
          v[j] = beta;
        }
      } else {
        red[0] = 1.0;
        red[1] = 0.0;
      }
      s_tau = t;
      taus[j] = t;
    }
    __syncthreads();
    T sc;
    if constexpr (Scalar<T>::is_complex)
      sc = cplx{red[0], red[1]};
    else
      sc = red[0];
    for (int i = j + 1 + tid; i < mp; i += blockDim.x) v[i] = mul(v[i], sc);
    __syncthreads();
    const T ct = conj_(s_tau);
    for (int c = j + 1 + warp; c < jb; c += nwarps) {
      T* a = P + (size_t)c * mp;
      T w = Scalar<T>::zero();
      for (int i = j + lane; i < mp; i += 32) w = add(w, cmul(i == j ? Scalar<T>::one() : v[i], a[i]));
      if constexpr (Scalar<T>::is_complex) {
        w.x = warp_sum(w.x);
        w.y = warp_sum(w.y);
      } else {
        w = warp_sum(w);
      }
      const T f = mul(ct, w);
      for (int i = j + lane; i < mp; i += 32) a[i] = sub(a[i], mul(i == j ? Scalar<T>::one() : v[i], f));
    }
    __syncthreads();
  }
  const int jr = jb < mp ? jb : mp;  // reflectors actually formed
  // write back R (upper part) and V (unit lower trapezoid, zeros above)
  for (int idx = tid; idx < mp * jb; idx += blockDim.x) {
    const int r = idx / jb, c = idx % jb;
    const T x = P[(size_t)c * mp + r];
    A[(size_t)r * lda + c] = x;
    Vall[(size_t)r * ldv + c] = (c >= jr) ? Scalar<T>::zero()
                                          : (r > c ? x : (r == c ? Scalar<T>::one() : Scalar<T>::zero()));
  }
  // S = V^H V (upper part), V read from P
  for (int pr = warp; pr < jr * jr; pr += nwarps) {
    const int a = pr / jr, b = pr % jr;
    if (a >= b) continue;
    T w = Scalar<T>::zero();
    for (int i = b + lane; i < mp; i += 32) {
      const T va = (i == a) ? Scalar<T>::one() : (i > a ? P[(size_t)a * mp + i] : Scalar<T>::zero());
      const T vb = (i == b) ? Scalar<T>::one() : P[(size_t)b * mp + i];
      w = add(w, cmul(va, vb));
    }
    if constexpr (Scalar<T>::is_complex) {
      w.x = warp_sum(w.x);
      w.y = warp_sum(w.y);
    } else {
      w = warp_sum(w);
    }
    if (lane == 0) S[a][b] = w;
  }
  __syncthreads();
  // xLARFT (forward, columnwise): T[i,i] = tau_i, T[0:i,i] = -tau_i T[0:i,0:i] S[0:i,i]
  if (warp == 0) warp_larft<T>(S, taus, jr, lane, Tp);
}

// Tall panels (not in shared memory): rows are spread over 1024 threads, the
// panel lives column-major in an L2-resident scratch, and for every column all
// trailing dot products are reduced together (one block reduction of <= 31
// values per column instead of one per column pair).
constexpr int PANEL_ROWS_THREADS = 512;

template <typename T>
__global__ void __launch_bounds__(PANEL_ROWS_THREADS) qr_panel_rows_kernel(T* A, long long sA, int lda, int mp, int jb,
                                                                           T* Vall, long long sV, int ldv, T* Tall,
                                                                           long long sT, T* Pg, long long sP) {
  constexpr bool CPX = Scalar<T>::is_complex;
  constexpr int NW = PANEL_ROWS_THREADS / 32;
  __shared__ double red[NW][QR_NB][CPX ? 2 : 1];
  __shared__ double rs[NW];
  __shared__ T bc[QR_NB];
  __shared__ T s_sc, s_tau;
  __shared__ T taus[QR_NB];
  __shared__ T S[QR_NB][QR_NB + 1];
  const int chain = blockIdx.x;
  A += sA * chain;
  Vall += sV * chain;
  T* Tp = Tall + sT * chain;
  T* P = Pg + sP * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (long long idx = tid; idx < (long long)mp * jb; idx += PANEL_ROWS_THREADS) {
    const int c = (int)(idx / mp), r = (int)(idx % mp);
    P[idx] = A[(size_t)r * lda + c];
  }
  __syncthreads();
  const int jr = jb < mp ? jb : mp;
  for (int j = 0; j < jr; ++j) {
    T* v = P + (size_t)j * mp;
    double part = 0.0;
    for (int i = j + 1 + tid; i < mp; i += PANEL_ROWS_THREADS) part += abs2(v[i]);
    part = warp_sum(part);
    if (lane == 0) rs[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double xn2 = 0.0;
      for (int w = 0; w < NW; ++w) xn2 += rs[w];
      const T alpha = v[j];
      double ar, ai;
      if constexpr (CPX) {
        ar = alpha.x;
        ai = alpha.y;
      } else {
        ar = alpha;
        ai = 0.0;
      }
      T t = Scalar<T>::zero();
      T sc = Scalar<T>::one();
      if (!(xn2 == 0.0 && ai == 0.0)) {
        const double beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
        if constexpr (CPX) {
          t = cplx{(beta - ar) / beta, -ai / beta};
          const double dr = ar - beta, di = ai, den = dr * dr + di * di;
          sc = cplx{dr / den, -di / den};
          v[j] = cplx{beta, 0.0};
        } else {
          t = (beta - ar) / beta;
          sc = 1.0 / (ar - beta);
          v[j] = beta;
        }
      }
      s_tau = t;
      s_sc = sc;
      taus[j] = t;
    }
    __syncthreads();
    const T sc = s_sc;
    for (int i = j + 1 + tid; i < mp; i += PANEL_ROWS_THREADS) v[i] = mul(v[i], sc);
    // all trailing dots w_c = v^H P[:, c] at once (own rows; v_j = 1)
    const int nc = jb - j - 1;
    if (nc > 0) {
      double pr[QR_NB], pi[QR_NB];
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) {
        pr[c] = 0.0;
        pi[c] = 0.0;
      }
      for (int i = j + tid; i < mp; i += PANEL_ROWS_THREADS) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
#pragma unroll
        for (int c = 0; c < QR_NB; ++c) {
          if (c < nc) {
            const T x = cmul(vi, P[(size_t)(j + 1 + c) * mp + i]);
            if constexpr (CPX) {
              pr[c] += x.x;
              pi[c] += x.y;
            } else {
              pr[c] += x;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) {
        if (c < nc) {
          pr[c] = warp_sum(pr[c]);
          if constexpr (CPX) pi[c] = warp_sum(pi[c]);
          if (lane == 0) {
            red[warp][c][0] = pr[c];
            if constexpr (CPX) red[warp][c][1] = pi[c];
          }
        }
      }
      __syncthreads();
      if (tid < nc) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < NW; ++w) {
          a += red[w][tid][0];
          if constexpr (CPX) b += red[w][tid][1];
        }
        T wc;
        if constexpr (CPX)
          wc = cplx{a, b};
        else
          wc = a;
        bc[tid] = mul(conj_(s_tau), wc);
      }
      __syncthreads();
      for (int i = j + tid; i < mp; i += PANEL_ROWS_THREADS) {
        const T vi = (i == j) ? Scalar<T>::one() : v[i];
        for (int c = 0; c < nc; ++c) {
          T* a = P + (size_t)(j + 1 + c) * mp;
          a[i] = sub(a[i], mul(vi, bc[c]));
        }
      }
    }
    __syncthreads();
  }
  // write back R / V, then S = V^H V and the WY factor (as qr_panel_kernel)
  for (long long idx = tid; idx < (long long)mp * jb; idx += PANEL_ROWS_THREADS) {
    const int c = (int)(idx / mp), r = (int)(idx % mp);
    const T x = P[idx];
    A[(size_t)r * lda + c] = x;
    Vall[(size_t)r * ldv + c] = (c >= jr) ? Scalar<T>::zero()
                                          : (r > c ? x : (r == c ? Scalar<T>::one() : Scalar<T>::zero()));
  }
  for (int pr2 = warp; pr2 < jr * jr; pr2 += NW) {
    const int a = pr2 / jr, b = pr2 % jr;
    if (a >= b) continue;
    T w = Scalar<T>::zero();
    for (int i = b + lane; i < mp; i += 32) {
      const T va = (i == a) ? Scalar<T>::one() : (i > a ? P[(size_t)a * mp + i] : Scalar<T>::zero());
      const T vb = (i == b) ? Scalar<T>::one() : P[(size_t)b * mp + i];
      w = add(w, cmul(va, vb));
    }
    if constexpr (CPX) {
      w.x = warp_sum(w.x);
      w.y = warp_sum(w.y);
    } else {
      w = warp_sum(w);
    }
    if (lane == 0) S[a][b] = w;
  }
  __syncthreads();
  if (warp == 0) warp_larft<T>(S, taus, jr, lane, Tp);
}

// Tall panels of a single chain: the rows are split over a cooperative grid,
// each CTA keeps its row block of the panel in shared memory, and every column
// costs two grid barriers (norm reduction, then the batched trailing dots).
constexpr int COOP_THREADS = 256;
constexpr int COOP_MAX_CTAS = 148;

template <bool CLUSTER>
__device__ __forceinline__ void panel_barrier() {
  if constexpr (CLUSTER) {
    __threadfence();
    cg::this_cluster().sync();
  } else {
    cg::this_grid().sync();
  }
}

// CLUSTER: the CTAs form one thread-block cluster (<= 16) and synchronise with
// the hardware cluster barrier; otherwise a cooperative grid barrier.
template <typename T, bool CLUSTER>
__global__ void __launch_bounds__(COOP_THREADS) qr_panel_coop_kernel(T* A, int lda, int mp, int jb, T* Vall, int ldv,
                                                                     T* Tp, double* gpart, int rows_per) {
  constexpr bool CPX = Scalar<T>::is_complex;
  constexpr int NW = COOP_THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* P = reinterpret_cast<T*>(smem_raw);  // rows_per x jb, column-major (ld = rows_per)
  __shared__ double wred[NW][QR_NB][CPX ? 2 : 1];
  __shared__ double rs[NW];
  __shared__ T wcs[QR_NB];
  __shared__ T taus[QR_NB];
  __shared__ T S[QR_NB][QR_NB + 1];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = b * rows_per, r1 = min(mp, r0 + rows_per), nr = max(0, r1 - r0);
  // global scratch: [0, G) norm partials | alpha (2 doubles) | [G][QR_NB][2] dot partials | [G][QR_NB^2][2] gram
  double* gnorm = gpart;
  double* galpha = gpart + G;
  double* gdot = gpart + G + 2;
  double* ggram = gdot + (size_t)G * QR_NB * 2;
  for (int idx = tid; idx < nr * jb; idx += COOP_THREADS) {
    const int c = idx / nr, r = idx % nr;
    P[c * rows_per + r] = A[(size_t)(r0 + r) * lda + c];
  }
  __syncthreads();
  const int jr = jb < mp ? jb : mp;
  for (int j = 0; j < jr; ++j) {
    T* v = P + j * rows_per;  // local rows r0..r1-1 of column j
    double part = 0.0;
    for (int r = tid; r < nr; r += COOP_THREADS)
      if (r0 + r > j) part += abs2(v[r]);
    part = warp_sum(part);
    if (lane == 0) rs[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += rs[w];
      gnorm[b] = t;
      if (j >= r0 && j < r1) {
        const T a = v[j - r0];
        if constexpr (CPX) {
          galpha[0] = a.x;
          galpha[1] = a.y;
        } else {
          galpha[0] = a;
          galpha[1] = 0.0;
        }
      }
    }
    panel_barrier<CLUSTER>();
    // every CTA forms the same reflector
    double xn2 = 0.0;
    for (int g = 0; g < G; ++g) xn2 += gnorm[g];
    const double ar = galpha[0], ai = galpha[1];
    T tau = Scalar<T>::zero(), sc = Scalar<T>::one();
    double beta = ar;
    const bool refl = !(xn2 == 0.0 && ai == 0.0);
    if (refl) {
      beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
      if constexpr (CPX) {
        tau = cplx{(beta - ar) / beta, -ai / beta};
        const double dr = ar - beta, di = ai, den = dr * dr + di * di;
        sc = cplx{dr / den, -di / den};
      } else {
        tau = (beta - ar) / beta;
        sc = 1.0 / (ar - beta);
      }
    }
    if (tid == 0) taus[j] = tau;
    for (int r = tid; r < nr; r += COOP_THREADS) {
      const int gi = r0 + r;
      if (gi > j) v[r] = mul(v[r], sc);
      if (gi == j && refl) {
        if constexpr (CPX)
          v[r] = cplx{beta, 0.0};
        else
          v[r] = beta;
      }
    }
    __syncthreads();
    const int nc = jb - j - 1;
    if (nc > 0) {
      double pr[QR_NB], pi[QR_NB];
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) {
        pr[c] = 0.0;
        pi[c] = 0.0;
      }
      for (int r = tid; r < nr; r += COOP_THREADS) {
        const int gi = r0 + r;
        if (gi < j) continue;
        const T vi = (gi == j) ? Scalar<T>::one() : v[r];
#pragma unroll
        for (int c = 0; c < QR_NB; ++c)
          if (c < nc) {
            const T x = cmul(vi, P[(j + 1 + c) * rows_per + r]);
            if constexpr (CPX) {
              pr[c] += x.x;
              pi[c] += x.y;
            } else {
              pr[c] += x;
            }
          }
      }
#pragma unroll
      for (int c = 0; c < QR_NB; ++c)
        if (c < nc) {
          pr[c] = warp_sum(pr[c]);
          if constexpr (CPX) pi[c] = warp_sum(pi[c]);
          if (lane == 0) {
            wred[warp][c][0] = pr[c];
            if constexpr (CPX) wred[warp][c][1] = pi[c];
          }
        }
      __syncthreads();
      if (tid < nc) {
        double a = 0.0, bb = 0.0;
        for (int w = 0; w < NW; ++w) {
          a += wred[w][tid][0];
          if constexpr (CPX) bb += wred[w][tid][1];
        }
        gdot[((size_t)b * QR_NB + tid) * 2] = a;
        gdot[((size_t)b * QR_NB + tid) * 2 + 1] = bb;
      }
    }
    panel_barrier<CLUSTER>();
    if (nc > 0) {
      if (tid < nc) {
        double a = 0.0, bb = 0.0;
        for (int g = 0; g < G; ++g) {
          a += gdot[((size_t)g * QR_NB + tid) * 2];
          bb += gdot[((size_t)g * QR_NB + tid) * 2 + 1];
        }
        T wc;
        if constexpr (CPX)
          wc = cplx{a, bb};
        else
          wc = a;
        wcs[tid] = mul(conj_(tau), wc);
      }
      __syncthreads();
      for (int r = tid; r < nr; r += COOP_THREADS) {
        const int gi = r0 + r;
        if (gi < j) continue;
        const T vi = (gi == j) ? Scalar<T>::one() : v[r];
        for (int c = 0; c < nc; ++c) {
          T* a = P + (j + 1 + c) * rows_per;
          a[r] = sub(a[r], mul(vi, wcs[c]));
        }
      }
      __syncthreads();
    }
  }
  // write back R and V; Gram of V for the WY factor
  for (int idx = tid; idx < nr * jb; idx += COOP_THREADS) {
    const int c = idx / nr, r = idx % nr, gi = r0 + r;
    const T x = P[c * rows_per + r];
    A[(size_t)gi * lda + c] = x;
    Vall[(size_t)gi * ldv + c] =
        (c >= jr) ? Scalar<T>::zero() : (gi > c ? x : (gi == c ? Scalar<T>::one() : Scalar<T>::zero()));
  }
  for (int pr2 = warp; pr2 < jr * jr; pr2 += NW) {
    const int a = pr2 / jr, c = pr2 % jr;
    T w = Scalar<T>::zero();
    if (a < c) {
      for (int r = lane; r < nr; r += 32) {
        const int gi = r0 + r;
        const T va = (gi == a) ? Scalar<T>::one() : (gi > a ? P[a * rows_per + r] : Scalar<T>::zero());
        const T vb = (gi == c) ? Scalar<T>::one() : (gi > c ? P[c * rows_per + r] : Scalar<T>::zero());
        w = add(w, cmul(va, vb));
      }
      if constexpr (CPX) {
        w.x = warp_sum(w.x);
        w.y = warp_sum(w.y);
      } else {
        w = warp_sum(w);
      }
    }
    if (lane == 0) {
      double* gg = ggram + ((size_t)b * QR_NB * QR_NB + a * QR_NB + c) * 2;
      if constexpr (CPX) {
        gg[0] = w.x;
        gg[1] = w.y;
      } else {
        gg[0] = w;
        gg[1] = 0.0;
      }
    }
  }
  panel_barrier<CLUSTER>();
  if (b == 0) {
    for (int pr2 = tid; pr2 < jr * jr; pr2 += COOP_THREADS) {
      const int a = pr2 / jr, c = pr2 % jr;
      double x = 0.0, y = 0.0;
      for (int g = 0; g < G; ++g) {
        x += ggram[((size_t)g * QR_NB * QR_NB + a * QR_NB + c) * 2];
        y += ggram[((size_t)g * QR_NB * QR_NB + a * QR_NB + c) * 2 + 1];
      }
      if constexpr (CPX)
        S[a][c] = cplx{x, y};
      else
        S[a][c] = x;
    }
    __syncthreads();
    if (warp == 0) warp_larft<T>(S, taus, jr, lane, Tp);
  }
}

template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src) {
  if constexpr (Scalar<T>::is_complex)
    return cplx{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
  else
    return __shfl_sync(0xffffffffu, v, src);
}
__device__ __forceinline__ double fma_c(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ cplx fma_c(cplx a, cplx b, cplx c) {
  return cplx{fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
__device__ __forceinline__ double re_of(double a) { return a; }
__device__ __forceinline__ double re_of(cplx a) { return a.x; }

// Single-chain panels, one thread-block cluster (C <= 16 CTAs): lanes own the
// panel's columns (lane c = column c) and every warp a contiguous slab of RW
// rows, all in registers, so column j is simply lane j (shuffles, no dynamic
// register indexing).  Per column ONE 32-value reduction: lane c accumulates
// q_c = sum_{rows > j} conj(P_c) x over its rows (x = column j): q_j = |x|^2,
// q_c (c > j) = conj(x^H a_c), q_c (c < j) = V_c^H x (the Gram column of the
// WY factor).  Warp partials -> CTA partial (shared) -> pushed into every
// CTA of the cluster (DSMEM), one cluster barrier, then every warp forms the
// same reflector (xLARFG convention) and updates its rows.  Partial slots are
// double-buffered by column parity, so one barrier per column suffices.
// RS > 0: each warp keeps RW of its rows in registers and RS more in (dynamic) shared memory
// ([warp][row][lane], one element per lane): the 8192-row complex panels, whose 32 register
// rows per lane would not fit in the 128-register budget of 512 threads.
template <typename T, int RW, int NT, int RS = 0>
__global__ void __launch_bounds__(NT, 1) qr_panel_cl_kernel(T* A, int lda, int mp, int jb, T* Vall, int ldv, T* Tp) {
  constexpr bool CPX = Scalar<T>::is_complex;
  constexpr int NW = NT / 32;
  constexpr int RT = RW + RS;  // rows per warp
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), b = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ T wpart[NW][32];
  __shared__ T slot[2][16][32];
  __shared__ T rowj[2][32];
  __shared__ T taus[QR_NB];
  __shared__ T S[QR_NB][QR_NB + 1];
  const int g0 = (b * NW + warp) * RT;  // first row of this warp's slab
  const bool colv = lane < jb;
  T a[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) a[r] = Scalar<T>::zero();  // (overwritten by the load below)
  extern __shared__ __align__(16) unsigned char qr_cl_dyn[];
  T* srow = reinterpret_cast<T*>(qr_cl_dyn) + (size_t)warp * (RS > 0 ? RS : 1) * 32 + lane;
  // row r of the slab: a register for r < RW, shared memory otherwise (r is a constant after unrolling)
  auto getv = [&](int r) -> T { return r < RW ? a[r < RW ? r : 0] : srow[(r - RW) * 32]; };
  auto setv = [&](int r, T v) {
    if (r < RW)
      a[r < RW ? r : 0] = v;
    else
      srow[(r - RW) * 32] = v;
  };
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int g = g0 + r;
    setv(r, (colv && g < mp) ? A[(size_t)g * lda + lane] : Scalar<T>::zero());
  }
  const int jr = jb < mp ? jb : mp;
  for (int j = 0; j < jr; ++j) {
    const int par = j & 1;
    // ---- partials
    T q = Scalar<T>::zero(), q2 = Scalar<T>::zero();
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const T ar = getv(r);
      const T x = shfl_t(ar, j);
      const T y = (g0 + r > j) ? x : Scalar<T>::zero();
      if (r & 1)
        q2 = fma_c(conj_(ar), y, q2);
      else
        q = fma_c(conj_(ar), y, q);
    }
    q = add(q, q2);
    // the owner of row j publishes it to every CTA
    if (j >= g0 && j < g0 + RT) {
      T rv = Scalar<T>::zero();
#pragma unroll
      for (int r = 0; r < RT; ++r)
        if (g0 + r == j) rv = getv(r);
      for (int g = 0; g < C; ++g) cl.map_shared_rank(&rowj[par][0], g)[lane] = rv;
    }
    wpart[warp][lane] = q;
    __syncthreads();
    if (warp == 0) {
      T s = wpart[0][lane];
#pragma unroll
      for (int w = 1; w < NW; ++w) s = add(s, wpart[w][lane]);
      for (int g = 0; g < C; ++g) cl.map_shared_rank(&slot[par][0][0], g)[b * 32 + lane] = s;
    }
    cl.sync();
    // ---- reflector (every warp, redundantly)
    T t = slot[par][0][lane];
    for (int g = 1; g < C; ++g) t = add(t, slot[par][g][lane]);
    const double xn2 = re_of(shfl_t(t, j));
    const T alpha = rowj[par][j];
    double ar, ai;
    if constexpr (CPX) {
      ar = alpha.x;
      ai = alpha.y;
    } else {
      ar = alpha;
      ai = 0.0;
    }
    T tau = Scalar<T>::zero(), sc = Scalar<T>::one();
    double beta = ar;
    const bool refl = !(xn2 == 0.0 && ai == 0.0);
    if (refl) {
      beta = -copysign(sqrt(ar * ar + ai * ai + xn2), ar);
      const double rb = 1.0 / beta;
      if constexpr (CPX) {
        tau = cplx{(beta - ar) * rb, -ai * rb};
        const double dr = ar - beta, di = ai, rden = 1.0 / (dr * dr + di * di);
        sc = cplx{dr * rden, -di * rden};
      } else {
        tau = (beta - ar) * rb;
        sc = 1.0 / (ar - beta);
      }
    }
    const T pj = rowj[par][lane];  // P(j, c)
    // f_c = conj(tau) (a_c(j) + conj(sc) d_c), d_c = conj(t_c)  (c > j)
    const T f = mul(conj_(tau), add(pj, mul(conj_(sc), conj_(t))));
    if (warp == 0 && lane < j) S[lane][j] = add(conj_(pj), mul(sc, t));  // V_c^H v_j
    if (tid == 0) taus[j] = tau;
    // ---- update: lane j stores v (rows > j) and beta; lanes c > j: a_c -= v f_c
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int g = g0 + r;
      const T ar = getv(r);
      const T x = shfl_t(ar, j);
      const T v = (g > j) ? mul(x, sc) : (g == j ? Scalar<T>::one() : Scalar<T>::zero());
      T nv = ar;
      if (lane > j) nv = sub(ar, mul(v, f));
      if (lane == j) {
        if (g > j) nv = v;
        else if (g == j && refl) {
          if constexpr (CPX)
            nv = cplx{beta, 0.0};
          else
            nv = beta;
        }
      }
      setv(r, nv);
    }
  }
  // ---- write back R (upper part) and V (unit lower trapezoid)
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int g = g0 + r;
    if (colv && g < mp) {
      const T ar = getv(r);
      A[(size_t)g * lda + lane] = ar;
      Vall[(size_t)g * ldv + lane] =
          (lane >= jr) ? Scalar<T>::zero() : (g > lane ? ar : (g == lane ? Scalar<T>::one() : Scalar<T>::zero()));
    }
  }
  if (b == 0) {
    __syncthreads();
    if (warp == 0) warp_larft<T>(S, taus, jr, lane, Tp);
  }
  cl.sync();  // no CTA leaves while peers may still write into its shared memory
}

template <typename T, int RW, int RS = 0>
cudaError_t launch_panel_cl(T* Ap, int lda, int mp, int jb, T* Vp, int ldv, T* Tp, cudaStream_t s) {
  constexpr int NT = 512;
  const int rows_cta = (NT / 32) * (RW + RS);
  const int C = (mp + rows_cta - 1) / rows_cta;
  if (C > 16) return cudaErrorInvalidValue;
  const size_t dyn = (size_t)RS * NT * sizeof(T);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(qr_panel_cl_kernel<T, RW, NT, RS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess && dyn > 0)
      e = cudaFuncSetAttribute(qr_panel_cl_kernel<T, RW, NT, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qr_panel_cl_kernel<T, RW, NT, RS>, Ap, lda, mp, jb, Vp, ldv, Tp);
}

// Rows per warp for an mp-row panel: the smallest slab that keeps the cluster
// at <= 8 CTAs (<= 16 for the tallest panels); 0 = not eligible.
template <typename T>
cudaError_t panel_cl(T* Ap, int lda, int mp, int jb, T* Vp, int ldv, T* Tp, cudaStream_t s) {
  if (mp <= 8 * 16 * 4) return launch_panel_cl<T, 4>(Ap, lda, mp, jb, Vp, ldv, Tp, s);
  if (mp <= 8 * 16 * 8) return launch_panel_cl<T, 8>(Ap, lda, mp, jb, Vp, ldv, Tp, s);
  if (mp <= 16 * 16 * 16) return launch_panel_cl<T, 16>(Ap, lda, mp, jb, Vp, ldv, Tp, s);
  // 32 rows per warp: all in registers for real panels; complex: 16 in registers + 16 in shared memory
  static const int rs_real = [] {  // TTG_QR_RS=1: real panels split 16 + 16 as well
    const char* e = getenv("TTG_QR_RS");
    return e ? atoi(e) : 0;
  }();
  if constexpr (Scalar<T>::is_complex)
    return launch_panel_cl<T, 16, 16>(Ap, lda, mp, jb, Vp, ldv, Tp, s);
  else
    return rs_real ? launch_panel_cl<T, 16, 16>(Ap, lda, mp, jb, Vp, ldv, Tp, s)
                   : launch_panel_cl<T, 32>(Ap, lda, mp, jb, Vp, ldv, Tp, s);
}

bool panel_cl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TTG_QR_CL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T> int panel_cl_max_rows() { return 16 * 16 * 32; }

template <typename T>
__global__ void conj_transpose_kernel(const T* src, long long s_src, int rows, int cols, T* dst, long long s_dst) {
  __shared__ T tile[32][33];
  const int chain = blockIdx.z;
  src += s_src * chain;
  dst += s_dst * chain;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const int r = by + yy, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[yy][threadIdx.x] = src[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += 8) {
    const int c = bx + yy, r = by + threadIdx.x;  // dst[c, r] = conj(src[r, c])
    if (r < rows && c < cols) dst[(size_t)c * rows + r] = conj_(tile[threadIdx.x][yy]);
  }
}

template <typename T>
__global__ void copy_in_kernel(const T* src, long long s_src, T* dst, long long s_dst, long long n) {
  const int chain = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[s_dst * chain + i] = src[s_src * chain + i];
}

template <typename T>
__global__ void upper_kernel(const T* A, long long sA, int n, T* R, long long sR, int k) {
  const int chain = blockIdx.y;
  const long long tot = (long long)k * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), c = (int)(idx % n);
    R[sR * chain + idx] = (c >= i) ? A[sA * chain + idx] : Scalar<T>::zero();
  }
}

template <typename T>
__global__ void eye_kernel(T* Q, long long sQ, int m, int k) {
  const int chain = blockIdx.y;
  const long long tot = (long long)m * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / k), c = (int)(idx % k);
    Q[sQ * chain + idx] = (i == c) ? Scalar<T>::one() : Scalar<T>::zero();
  }
}

int blocks_for(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

template <typename T>
size_t qr_blocked_elems(int m, int n, size_t* sA, size_t* sV, size_t* sT, size_t* sW, size_t* sP) {
  const int k = m < n ? m : n;
  const int nblk = (k + QR_NB - 1) / QR_NB;
  const int nblko = (k + QR_NBO - 1) / QR_NBO;
  *sA = (size_t)m * n;
  *sV = (size_t)m * k;
  // inner 32 x 32 WY factors | outer 128 x 128 WY factors | S = V_O^H V_O scratch
  *sT = (size_t)nblk * QR_NB * QR_NB + (size_t)(nblko + 1) * QR_NBO * QR_NBO;
  *sW = (size_t)QR_NBO * n;
  *sP = (size_t)m * QR_NB;
  return *sA + *sV + *sT + 2 * *sW + *sP;
}

// WY factor of an outer block of nbi inner 32-column blocks (xLARFT, blocked):
// T_O = [[T_A, -T_A (V_A^H V_b) T_b], [0, T_b]] appended block by block, with
// S = V_O^H V_O precomputed by one GEMM.  One CTA; T_O (row-major, ld QR_NBO)
// in global memory (L2), Z = S[0:n0, n0:n0+32] T_b staged in shared memory.
// T_O is upper triangular: it is built in shared memory with its upper triangle packed by rows
// (row r holds columns r .. QR_NBO-1; 66 KB real, 132 KB complex) and written out once, so the
// triangular products read shared memory instead of L2.
__host__ __device__ constexpr int tri_off(int r) { return r * QR_NBO - r * (r - 1) / 2; }

// S[0:n0, n0:n0+w] and T_b are staged in shared memory before the products (they were read from L2
// inside dependent loops), and the dot products run on four partial accumulators.
template <typename T>
__global__ void __launch_bounds__(256) t_combine_kernel(const T* S, int lds, const T* Tin, T* TO, int jbo,
                                                        long long stride) {
  constexpr int ZS = QR_NB + 1;
  constexpr int NTH = 256;
  constexpr int MAXI = (QR_NBO - QR_NB) * QR_NB / NTH;  // items per thread of the largest block
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Z = reinterpret_cast<T*>(smem_raw);        // (QR_NBO - QR_NB) x ZS: S block, then Z
  T* Tbs = Z + (QR_NBO - QR_NB) * ZS;           // QR_NB x ZS: T_b
  T* Tp = Tbs + QR_NB * ZS;                     // packed upper triangle of T_O
  const int tid = threadIdx.x;
  S += stride * blockIdx.x;  // one CTA per chain
  Tin += stride * blockIdx.x;
  TO += stride * blockIdx.x;
  const int nbi = (jbo + QR_NB - 1) / QR_NB;
  for (int r = tid / 32; r < QR_NBO; r += NTH / 32)  // diagonal blocks T_b, zero elsewhere
    for (int c = r + (tid & 31); c < QR_NBO; c += 32) {
      const int br = r / QR_NB, bc = c / QR_NB;
      Tp[tri_off(r) + c - r] = (br == bc && r < jbo && c < jbo)
                                   ? Tin[(size_t)br * QR_NB * QR_NB + (r % QR_NB) * QR_NB + (c % QR_NB)]
                                   : Scalar<T>::zero();
    }
  for (int b = 1; b < nbi; ++b) {
    const int n0 = b * QR_NB, w = min(QR_NB, jbo - n0);
    const T* Tb = Tin + (size_t)b * QR_NB * QR_NB;
    __syncthreads();  // previous block's products are done with Z / T_b
    for (int idx = tid; idx < n0 * w; idx += NTH) {
      const int r = idx / w, c = idx % w;
      Z[r * ZS + c] = S[(size_t)r * lds + n0 + c];
    }
    for (int idx = tid; idx < w * w; idx += NTH) {
      const int r = idx / w, c = idx % w;
      Tbs[r * ZS + c] = Tb[r * QR_NB + c];
    }
    __syncthreads();
    T zr[MAXI];
#pragma unroll
    for (int it = 0; it < MAXI; ++it) {  // Z = S[0:n0, n0:n0+w] T_b (T_b upper triangular)
      const int idx = tid + it * NTH;
      zr[it] = Scalar<T>::zero();
      if (idx < n0 * w) {
        const int r = idx / w, c = idx % w;
        const T* srow = Z + r * ZS;
        T z0 = Scalar<T>::zero(), z1 = Scalar<T>::zero();
        int q = 0;
        for (; q + 1 <= c; q += 2) {
          z0 = add(z0, mul(srow[q], Tbs[q * ZS + c]));
          z1 = add(z1, mul(srow[q + 1], Tbs[(q + 1) * ZS + c]));
        }
        if (q <= c) z0 = add(z0, mul(srow[q], Tbs[q * ZS + c]));
        zr[it] = add(z0, z1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < MAXI; ++it) {
      const int idx = tid + it * NTH;
      if (idx < n0 * w) Z[(idx / w) * ZS + idx % w] = zr[it];
    }
    __syncthreads();
    for (int idx = tid; idx < n0 * w; idx += NTH) {  // T_O[0:n0, n0:n0+w] = -T_O[0:n0, 0:n0] Z
      const int r = idx / w, c = idx % w;
      const T* row = Tp + tri_off(r) - r;  // row[q] = T_O[r][q], q >= r
      T a0 = Scalar<T>::zero(), a1 = Scalar<T>::zero(), a2 = Scalar<T>::zero(), a3 = Scalar<T>::zero();
      int q = r;
      for (; q + 3 < n0; q += 4) {
        a0 = add(a0, mul(row[q], Z[q * ZS + c]));
        a1 = add(a1, mul(row[q + 1], Z[(q + 1) * ZS + c]));
        a2 = add(a2, mul(row[q + 2], Z[(q + 2) * ZS + c]));
        a3 = add(a3, mul(row[q + 3], Z[(q + 3) * ZS + c]));
      }
      for (; q < n0; ++q) a0 = add(a0, mul(row[q], Z[q * ZS + c]));
      Tp[tri_off(r) + n0 + c - r] = sub(Scalar<T>::zero(), add(add(a0, a1), add(a2, a3)));
    }
  }
  __syncthreads();
  for (int idx = tid; idx < QR_NBO * QR_NBO; idx += NTH) {
    const int r = idx / QR_NBO, c = idx % QR_NBO;
    TO[idx] = c >= r ? Tp[tri_off(r) + c - r] : Scalar<T>::zero();
  }
}

template <typename T>
constexpr size_t t_combine_smem() {
  return ((size_t)(QR_NBO - QR_NB) * (QR_NB + 1) + (size_t)QR_NB * (QR_NB + 1) + (size_t)tri_off(QR_NBO)) * sizeof(T);
}

template <typename T>
cudaError_t householder_qr_blocked(const QrParams& p, const QrBlockedWork& w, int chains, cudaStream_t s,
                                   long long* launches) {
  const int m = p.m, n = p.n, k = m < n ? m : n;
  if (chains <= 0 || m <= 0 || n <= 0) return cudaSuccess;
  T* A = static_cast<T*>(w.A);
  T* V = static_cast<T*>(w.V);
  T* Tt = static_cast<T*>(w.T);
  cudaError_t e;
  long long nl = 0;
  copy_in_kernel<T><<<dim3(blocks_for((long long)m * n), chains), 256, 0, s>>>(static_cast<const T*>(p.A), p.sA, A,
                                                                             w.sA, (long long)m * n);
  ++nl;
  // two-level blocking: 32-column panels, trailing/Q updates per 128-column outer block (K = 128)
  static const int two_level_env = [] {
    const char* ev = std::getenv("TTG_QR_2L");
    return ev ? std::atoi(ev) : -1;
  }();
  // (narrow matrices: the outer T factor (t_combine) costs more than the K = 128 updates save; C2's
  // 384 x 192 exact-pass QRs measured 1.5 ms per call faster without it.  Complex: C3 3.36 -> 2.57 s
  // once t_combine keeps T_O in shared memory; the rank-32 updates stream the trailing matrix
  // from HBM four times as often)
  const bool two_level = w.keep_wy ? true
                         : two_level_env >= 0 ? two_level_env != 0
                         : w.two_level >= 0 ? w.two_level != 0
                                            : qr_two_level(m, n);
  const int nblk_in = (k + QR_NB - 1) / QR_NB;
  T* To_all = Tt + (size_t)nblk_in * QR_NB * QR_NB;  // outer WY factors, QR_NBO x QR_NBO each
  T* Sbuf = To_all + (size_t)((k + QR_NBO - 1) / QR_NBO) * QR_NBO * QR_NBO;
  if (two_level) {
    if ((e = cudaMemsetAsync(V, 0, (size_t)w.sV * (chains - 1) * sizeof(T) + (size_t)m * k * sizeof(T), s)) !=
        cudaSuccess)
      return e;
    e = cudaFuncSetAttribute(t_combine_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)t_combine_smem<T>());
    if (e != cudaSuccess) return e;
  }
  // Panel lookahead (single chain, two-level, tall and wide): see `outer`.  TTG_QR_LOOKAHEAD=0 disables.
  struct Lookahead {
    bool on = false, pending = false;
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_block = nullptr, ev_far = nullptr;
    void *W1 = nullptr, *W2 = nullptr;
  } la;
  {
    static const bool la_env = [] {
      const char* ev = std::getenv("TTG_QR_LOOKAHEAD");
      return !(ev && ev[0] == '0');
    }();
    static cudaStream_t aux_stream = nullptr;  // one process per GPU: one auxiliary stream per process
    static cudaEvent_t evs[2] = {nullptr, nullptr};
    static const int la1_rows = [] {  // rank-32 (single-level) lookahead from this many rows on; 0 = off
      const char* ev = std::getenv("TTG_QR_LOOKAHEAD1");
      return ev ? std::atoi(ev) : 0;  // measured: C4 2078 -> 2087 ms with 512 (tiny updates, event traffic)
    }();
    const bool la2 = two_level && m >= 2048 && n >= 4 * QR_NBO;
    const bool la1 = !two_level && la1_rows > 0 && m >= la1_rows && n >= 8 * QR_NB;
    if (la_env && chains == 1 && (la2 || la1)) {
      if (!aux_stream) {
        // lowest priority: the panel stream's cluster kernels are placed before pending update CTAs
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&aux_stream, cudaStreamNonBlocking, lo) != cudaSuccess) aux_stream = nullptr;
        if (aux_stream && (cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming) != cudaSuccess ||
                           cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming) != cudaSuccess)) {
          cudaStreamDestroy(aux_stream);
          aux_stream = nullptr;
        }
        cudaGetLastError();
      }
      if (aux_stream) {
        const size_t wb = (size_t)QR_NBO * n * sizeof(T);
        if (cudaMallocAsync(&la.W1, wb, s) == cudaSuccess && cudaMallocAsync(&la.W2, wb, s) == cudaSuccess) {
          la.on = true;
          la.aux = aux_stream;
          la.ev_block = evs[0];
          la.ev_far = evs[1];
        } else {
          if (la.W1) cudaFreeAsync(la.W1, s);
          la.W1 = la.W2 = nullptr;
          cudaGetLastError();
        }
      }
    }
  }
  // outer block: S = V_O^H V_O, T_O (t_combine); far columns [jend, n) -= V_O T_O^H V_O^H A
  auto outer = [&](int J0, int jend, bool far) -> cudaError_t {
    const int jbo = jend - J0, mpo = m - J0;
    T* To = To_all + (size_t)(J0 / QR_NBO) * QR_NBO * QR_NBO;
    GemmParams gs{V + (size_t)J0 * k + J0, V + (size_t)J0 * k + J0, Sbuf, w.sV, w.sV, w.sT, dconst(jbo), dconst(jbo),
                  dconst(mpo), nullptr, 0, nullptr, 1.0, 0};
    gs.lda = k;
    gs.ldb = k;
    gs.ldc = jbo;
    cudaError_t e2;
    if ((e2 = gemm<T>(gs, OP_C, OP_N, jbo, jbo, chains, s, mpo)) != cudaSuccess) return e2;
    t_combine_kernel<T><<<chains, 256, t_combine_smem<T>(), s>>>(
        Sbuf, jbo, Tt + (size_t)(J0 / QR_NB) * QR_NB * QR_NB, To, jbo, w.sT);
    nl += 2;
    if (!far || n - jend <= 0) return cudaGetLastError();
    // columns [c0, c1) -= V_O T_O^H V_O^H A on stream `st` with the scratch pair (W1_, W2_)
    auto far_update = [&](int c0, int c1, void* W1_, void* W2_, cudaStream_t st) -> cudaError_t {
      const int nt = c1 - c0;
      cudaError_t e3;
      GemmParams g1{V + (size_t)J0 * k + J0, A + (size_t)J0 * n + c0, W1_, w.sV, w.sA, w.sW, dconst(jbo), dconst(nt),
                    dconst(mpo), nullptr, 0, nullptr, 1.0, 0};
      g1.lda = k;
      g1.ldb = n;
      g1.ldc = nt;
      if ((e3 = gemm<T>(g1, OP_C, OP_N, jbo, nt, chains, st, mpo)) != cudaSuccess) return e3;
      GemmParams g2{To, W1_, W2_, w.sT, w.sW, w.sW, dconst(jbo), dconst(nt), dconst(jbo), nullptr, 0, nullptr, 1.0, 0};
      g2.lda = QR_NBO;
      g2.ldb = nt;
      g2.ldc = nt;
      if ((e3 = gemm<T>(g2, OP_C, OP_N, jbo, nt, chains, st)) != cudaSuccess) return e3;
      GemmParams g3{V + (size_t)J0 * k + J0, W2_, A + (size_t)J0 * n + c0, w.sV, w.sW, w.sA, dconst(mpo), dconst(nt),
                    dconst(jbo), nullptr, 0, nullptr, -1.0, 1};
      g3.lda = k;
      g3.ldb = nt;
      g3.ldc = n;
      if ((e3 = gemm<T>(g3, OP_N, OP_N, mpo, nt, chains, st)) != cudaSuccess) return e3;
      nl += 3;
      return cudaSuccess;
    };
    if (!la.on) return far_update(jend, n, w.W1, w.W2, s);
    // Lookahead: the next outer block's columns are updated on the panel stream; the rest of the
    // trailing matrix is updated on the auxiliary stream while the next block's panels are factored.
    const int jn = jend + QR_NBO < n ? jend + QR_NBO : n;
    if (la.pending && (e2 = cudaStreamWaitEvent(s, la.ev_far, 0)) != cudaSuccess) return e2;  // previous far update
    la.pending = false;
    if ((e2 = far_update(jend, jn, w.W1, w.W2, s)) != cudaSuccess) return e2;
    if (jn < n) {
      if ((e2 = cudaEventRecord(la.ev_block, s)) != cudaSuccess) return e2;
      if ((e2 = cudaStreamWaitEvent(la.aux, la.ev_block, 0)) != cudaSuccess) return e2;
      if ((e2 = far_update(jn, n, la.W1, la.W2, la.aux)) != cudaSuccess) return e2;
      if ((e2 = cudaEventRecord(la.ev_far, la.aux)) != cudaSuccess) return e2;
      la.pending = true;
    }
    return cudaSuccess;
  };
  const size_t panel_bytes_max = (size_t)m * QR_NB * sizeof(T);
  const size_t smem_limit = 200 * 1024;
  e = cudaFuncSetAttribute(qr_panel_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit);
  if (e != cudaSuccess) return e;
  (void)panel_bytes_max;
  // cooperative tall-panel path (single chain): one CTA per SM at most, <= 200 KB
  // of panel rows per CTA (occupancy checked for the largest launch below)
  double* coop_part = nullptr;
  int coop_ctas = 0;
  const size_t coop_smem_max = 200 * 1024;
  if (chains == 1 && (size_t)m * QR_NB * sizeof(T) > smem_limit) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(qr_panel_coop_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)coop_smem_max);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(qr_panel_coop_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)coop_smem_max);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(qr_panel_coop_kernel<T, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_panel_coop_kernel<T, false>, COOP_THREADS,
                                                        coop_smem_max);
    if (e == cudaSuccess && per_sm > 0) {
      coop_ctas = std::min(COOP_MAX_CTAS, sms);
      const size_t words = (size_t)COOP_MAX_CTAS + 2 + (size_t)COOP_MAX_CTAS * QR_NB * 2 +
                           (size_t)COOP_MAX_CTAS * QR_NB * QR_NB * 2;
      e = cudaMallocAsync(&coop_part, words * sizeof(double), s);
      if (e != cudaSuccess) coop_part = nullptr;
    }
    cudaGetLastError();
    e = cudaSuccess;
  }
  for (int j0 = 0; j0 < k; j0 += QR_NB) {
    const int jb = (k - j0) < QR_NB ? (k - j0) : QR_NB;
    const int mp = m - j0;
    const size_t pbytes = (size_t)mp * jb * sizeof(T);
    const int in_smem = pbytes <= smem_limit;
    if (chains == 1 && panel_cl_enabled() && mp <= panel_cl_max_rows<T>()) {
      e = panel_cl<T>(A + (size_t)j0 * n + j0, n, mp, jb, V + (size_t)j0 * k + j0, k,
                      Tt + (size_t)(j0 / QR_NB) * QR_NB * QR_NB, s);
      if (e != cudaSuccess) return e;
    } else if (in_smem) {
      qr_panel_kernel<T><<<chains, PANEL_THREADS, pbytes, s>>>(
          A + (size_t)j0 * n + j0, w.sA, n, mp, jb, V + (size_t)j0 * k + j0, w.sV, k,
          Tt + (size_t)(j0 / QR_NB) * QR_NB * QR_NB, w.sT, static_cast<T*>(w.P), w.sP, 1);
    } else if (chains == 1 && coop_part &&
               (size_t)((mp + coop_ctas - 1) / coop_ctas) * QR_NB * sizeof(T) <= coop_smem_max) {
      // at least 128 rows per CTA: fewer CTAs make the two grid barriers per column cheaper
      const int G = std::max(1, std::min(coop_ctas, (mp + 127) / 128));
      int rows_per = (mp + G - 1) / G;
      const int Gu = (mp + rows_per - 1) / rows_per;
      T* Ap = A + (size_t)j0 * n + j0;
      T* Vp = V + (size_t)j0 * k + j0;
      T* Tp = Tt + (size_t)(j0 / QR_NB) * QR_NB * QR_NB;
      int lda_ = n, mp_ = mp, jb_ = jb, ldv_ = k;
      double* gp = coop_part;
      const size_t pbytes2 = (size_t)rows_per * QR_NB * sizeof(T);
      bool launched = false;
      if (Gu <= 16) {  // one thread-block cluster: hardware cluster barrier
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(Gu);
        cfg.blockDim = dim3(COOP_THREADS);
        cfg.dynamicSmemBytes = pbytes2;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = Gu;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, qr_panel_coop_kernel<T, true>, Ap, lda_, mp_, jb_, Vp, ldv_, Tp, gp, rows_per);
        if (e == cudaSuccess)
          launched = true;
        else
          cudaGetLastError();
      }
      if (!launched) {
        void* args[] = {&Ap, &lda_, &mp_, &jb_, &Vp, &ldv_, &Tp, &gp, &rows_per};
        e = cudaLaunchCooperativeKernel((void*)qr_panel_coop_kernel<T, false>, dim3(Gu), dim3(COOP_THREADS), args,
                                        pbytes2, s);
        if (e != cudaSuccess) return e;
      }
    } else
      qr_panel_rows_kernel<T><<<chains, PANEL_ROWS_THREADS, 0, s>>>(
          A + (size_t)j0 * n + j0, w.sA, n, mp, jb, V + (size_t)j0 * k + j0, w.sV, k,
          Tt + (size_t)(j0 / QR_NB) * QR_NB * QR_NB, w.sT, static_cast<T*>(w.P), w.sP);
    ++nl;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int J0 = (j0 / QR_NBO) * QR_NBO;
    const int jend = two_level ? (J0 + QR_NBO < k ? J0 + QR_NBO : k) : n;  // inner updates stop at the block end
    const int nt = jend - j0 - jb;
    if (nt > 0) {
      // columns [c0, c1) -= V T^H V^H A for this panel's reflectors
      auto panel_update = [&](int c0, int c1, void* W1_, void* W2_, cudaStream_t st) -> cudaError_t {
        const int ntc = c1 - c0;
        cudaError_t e3;
        // W1 = V^H A_trail (jb x ntc)
        GemmParams g1{V + (size_t)j0 * k + j0, A + (size_t)j0 * n + c0, W1_, w.sV, w.sA, w.sW, dconst(jb), dconst(ntc),
                      dconst(mp), nullptr, 0, nullptr, 1.0, 0};
        g1.lda = k;
        g1.ldb = n;
        g1.ldc = ntc;
        if ((e3 = gemm<T>(g1, OP_C, OP_N, jb, ntc, chains, st, mp)) != cudaSuccess) return e3;
        // W2 = T^H W1
        GemmParams g2{Tt + (size_t)(j0 / QR_NB) * QR_NB * QR_NB, W1_, W2_, w.sT, w.sW, w.sW, dconst(jb), dconst(ntc),
                      dconst(jb), nullptr, 0, nullptr, 1.0, 0};
        g2.lda = QR_NB;
        g2.ldb = ntc;
        g2.ldc = ntc;
        if ((e3 = gemm<T>(g2, OP_C, OP_N, jb, ntc, chains, st)) != cudaSuccess) return e3;
        // A_trail -= V W2
        GemmParams g3{V + (size_t)j0 * k + j0, W2_, A + (size_t)j0 * n + c0, w.sV, w.sW, w.sA, dconst(mp), dconst(ntc),
                      dconst(jb), nullptr, 0, nullptr, -1.0, 1};
        g3.lda = k;
        g3.ldb = ntc;
        g3.ldc = n;
        if ((e3 = gemm<T>(g3, OP_N, OP_N, mp, ntc, chains, st)) != cudaSuccess) return e3;
        nl += 3;
        return cudaSuccess;
      };
      const int c_lo = j0 + jb;
      if (la.on && !two_level) {
        // rank-32 lookahead: the next panel's columns on the panel stream, the rest behind it
        const int jn = c_lo + QR_NB < jend ? c_lo + QR_NB : jend;
        if (la.pending && (e = cudaStreamWaitEvent(s, la.ev_far, 0)) != cudaSuccess) return e;
        la.pending = false;
        if ((e = panel_update(c_lo, jn, w.W1, w.W2, s)) != cudaSuccess) return e;
        if (jn < jend) {
          if ((e = cudaEventRecord(la.ev_block, s)) != cudaSuccess) return e;
          if ((e = cudaStreamWaitEvent(la.aux, la.ev_block, 0)) != cudaSuccess) return e;
          if ((e = panel_update(jn, jend, la.W1, la.W2, la.aux)) != cudaSuccess) return e;
          if ((e = cudaEventRecord(la.ev_far, la.aux)) != cudaSuccess) return e;
          la.pending = true;
        }
      } else if ((e = panel_update(c_lo, jend, w.W1, w.W2, s)) != cudaSuccess) {
        return e;
      }
    }
    if (two_level && j0 + jb == jend && (jend < n || p.Q || w.keep_wy))
      if ((e = outer(J0, jend, jend < n)) != cudaSuccess) return e;
  }
  if (la.on) {  // join the auxiliary stream before R / Q are formed and the scratch is released
    if (la.pending && (e = cudaStreamWaitEvent(s, la.ev_far, 0)) != cudaSuccess) return e;
    cudaFreeAsync(la.W1, s);
    cudaFreeAsync(la.W2, s);
  }
  if (coop_part) cudaFreeAsync(coop_part, s);
  upper_kernel<T><<<dim3(blocks_for((long long)k * n), chains), 256, 0, s>>>(A, w.sA, n, static_cast<T*>(p.R), p.sR, k);
  T* Q = static_cast<T*>(p.Q);
  if (!Q) {  // R only
    if (launches) *launches += nl + 1;
    return cudaGetLastError();
  }
  eye_kernel<T><<<dim3(blocks_for((long long)m * k), chains), 256, 0, s>>>(Q, p.sQ, m, k);
  nl += 2;
  const int NBQ = two_level ? QR_NBO : QR_NB;
  const int nblk = (k + NBQ - 1) / NBQ;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * NBQ;
    const int jb = (k - j0) < NBQ ? (k - j0) : NBQ;
    const int mp = m - j0, kq = k - j0;
    // W1 = V^H Q_sub (jb x kq)
    GemmParams g1{V + (size_t)j0 * k + j0, Q + (size_t)j0 * k + j0, w.W1, w.sV, p.sQ, w.sW, dconst(jb), dconst(kq),
                  dconst(mp), nullptr, 0, nullptr, 1.0, 0};
    g1.lda = k;
    g1.ldb = k;
    g1.ldc = kq;
    if ((e = gemm<T>(g1, OP_C, OP_N, jb, kq, chains, s, mp)) != cudaSuccess) return e;
    // W2 = T W1
    GemmParams g2{two_level ? To_all + (size_t)b * QR_NBO * QR_NBO : Tt + (size_t)b * QR_NB * QR_NB, w.W1, w.W2, w.sT,
                  w.sW, w.sW, dconst(jb), dconst(kq), dconst(jb), nullptr, 0, nullptr, 1.0, 0};
    g2.lda = NBQ;
    g2.ldb = kq;
    g2.ldc = kq;
    if ((e = gemm<T>(g2, OP_N, OP_N, jb, kq, chains, s)) != cudaSuccess) return e;
    // Q_sub -= V W2
    GemmParams g3{V + (size_t)j0 * k + j0, w.W2, Q + (size_t)j0 * k + j0, w.sV, w.sW, p.sQ, dconst(mp), dconst(kq),
                  dconst(jb), nullptr, 0, nullptr, -1.0, 1};
    g3.lda = k;
    g3.ldb = kq;
    g3.ldc = k;
    if ((e = gemm<T>(g3, OP_N, OP_N, mp, kq, chains, s)) != cudaSuccess) return e;
    nl += 3;
  }
  if (launches) *launches += nl;
  return cudaGetLastError();
}

template <typename T>
cudaError_t householder_apply_q(const void* Vv, const void* Tw, int m, int k, void* Xv, int r, void* W1, void* W2,
                                cudaStream_t s, long long* launches) {
  if (m <= 0 || k <= 0 || r <= 0) return cudaSuccess;
  const T* V = static_cast<const T*>(Vv);
  T* X = static_cast<T*>(Xv);
  const int nblk_in = (k + QR_NB - 1) / QR_NB;
  const T* To_all = static_cast<const T*>(Tw) + (size_t)nblk_in * QR_NB * QR_NB;
  const int nblk = (k + QR_NBO - 1) / QR_NBO;
  cudaError_t e;
  long long nl = 0;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * QR_NBO;
    const int jb = (k - j0) < QR_NBO ? (k - j0) : QR_NBO;
    const int mp = m - j0;
    // W1 = V_b^H X[j0:, :] (jb x r)
    GemmParams g1{V + (size_t)j0 * k + j0, X + (size_t)j0 * r, W1, 0, 0, 0, dconst(jb), dconst(r), dconst(mp), nullptr,
                  0, nullptr, 1.0, 0};
    g1.lda = k;
    g1.ldb = r;
    g1.ldc = r;
    if ((e = gemm<T>(g1, OP_C, OP_N, jb, r, 1, s, mp)) != cudaSuccess) return e;
    // W2 = T_b W1
    GemmParams g2{To_all + (size_t)b * QR_NBO * QR_NBO, W1, W2, 0, 0, 0, dconst(jb), dconst(r), dconst(jb), nullptr, 0,
                  nullptr, 1.0, 0};
    g2.lda = QR_NBO;
    g2.ldb = r;
    g2.ldc = r;
    if ((e = gemm<T>(g2, OP_N, OP_N, jb, r, 1, s)) != cudaSuccess) return e;
    // X[j0:, :] -= V_b W2
    GemmParams g3{V + (size_t)j0 * k + j0, W2, X + (size_t)j0 * r, 0, 0, 0, dconst(mp), dconst(r), dconst(jb), nullptr,
                  0, nullptr, -1.0, 1};
    g3.lda = k;
    g3.ldb = r;
    g3.ldc = r;
    if ((e = gemm<T>(g3, OP_N, OP_N, mp, r, 1, s)) != cudaSuccess) return e;
    nl += 3;
  }
  if (launches) *launches += nl;
  return cudaGetLastError();
}
template cudaError_t householder_apply_q<double>(const void*, const void*, int, int, void*, int, void*, void*,
                                                 cudaStream_t, long long*);
template cudaError_t householder_apply_q<cplx>(const void*, const void*, int, int, void*, int, void*, void*,
                                               cudaStream_t, long long*);

template <typename T>
cudaError_t conj_transpose(const void* src, long long s_src, int rows, int cols, void* dst, long long s_dst, int chains,
                           cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || chains <= 0) return cudaSuccess;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, chains);
  conj_transpose_kernel<T><<<grid, dim3(32, 8), 0, s>>>(static_cast<const T*>(src), s_src, rows, cols,
                                                        static_cast<T*>(dst), s_dst);
  return cudaGetLastError();
}
template cudaError_t conj_transpose<double>(const void*, long long, int, int, void*, long long, int, cudaStream_t);
template cudaError_t conj_transpose<cplx>(const void*, long long, int, int, void*, long long, int, cudaStream_t);

template size_t qr_blocked_elems<double>(int, int, size_t*, size_t*, size_t*, size_t*, size_t*);
template size_t qr_blocked_elems<cplx>(int, int, size_t*, size_t*, size_t*, size_t*, size_t*);
template cudaError_t householder_qr_blocked<double>(const QrParams&, const QrBlockedWork&, int, cudaStream_t,
                                                    long long*);
template cudaError_t householder_qr_blocked<cplx>(const QrParams&, const QrBlockedWork&, int, cudaStream_t,
                                                  long long*);

}  // namespace ttg
