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

#include <cfloat>

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

}  // namespace

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
