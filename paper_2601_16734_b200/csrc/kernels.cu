#include "kernels.cuh"

#include <algorithm>

namespace ttg {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v) {
  __shared__ double red[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < nw ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Expansions are pure HBM writes (the inputs are tiny and L2/L1 resident), so
// they are organised by OUTPUT ROW: one CTA per row of the fused-bond target,
// the row's indices decoded once per CTA (no per-element div/mod), and each
// thread writes VEC consecutive elements (16-byte stores: VEC = 2 for f64,
// 1 for complex128) for every right block, reusing the input values it holds
// in registers across the blocks.

template <typename T, int VEC> struct Vec;
template <> struct Vec<double, 2> { using type = double2; };
template <> struct Vec<double, 1> { using type = double; };
template <> struct Vec<cplx, 1> { using type = cplx; };

template <typename T, int VEC>
__device__ __forceinline__ void store_vec(T* dst, const T (&v)[VEC]) {
  if constexpr (VEC == 2)
    *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
  else
    *dst = v[0];
}

// apply_raw (mpo.hpp:213-238): C[(cb*Al + al), j, (cb2*Ar + ar)] = sum_i W[cb, j, i, cb2] A[al, i, ar].
// Row r = (cb*Al + al)*dout + j; columns (cb2, ar).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) expand_mpo_kernel(const T* __restrict__ W, const T* __restrict__ A,
                                                          T* __restrict__ C, int Dl, int dout, int din, int Dr, int Al,
                                                          int Ar, long long sA, long long sC) {
  const int chain = blockIdx.z;
  A += sA * chain;
  C += sC * chain;
  const int rows = Dl * Al * dout;
  const long long cols = (long long)Dr * Ar;
  for (int row = blockIdx.y * gridDim.x + blockIdx.x; row < rows; row += gridDim.x * gridDim.y) {
    const int j = row % dout, ra = row / dout;
    const int cb = ra / Al, al = ra - cb * Al;
    T* crow = C + (long long)row * cols;
    for (int ar = threadIdx.x * VEC; ar < Ar; ar += blockDim.x * VEC) {
      T a[4][VEC];  // the first four physical indices in registers
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < din)
#pragma unroll
          for (int v = 0; v < VEC; ++v) a[i][v] = A[((long long)al * din + i) * Ar + ar + v];
      for (int cb2 = 0; cb2 < Dr; ++cb2) {
        T out[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) out[v] = Scalar<T>::zero();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < din) {
            const T w = W[(((long long)cb * dout + j) * din + i) * Dr + cb2];
#pragma unroll
            for (int v = 0; v < VEC; ++v) out[v] = add(out[v], mul(w, a[i][v]));
          }
        for (int i = 4; i < din; ++i) {  // physical dimensions > 4: straight from L1/L2
          const T w = W[(((long long)cb * dout + j) * din + i) * Dr + cb2];
#pragma unroll
          for (int v = 0; v < VEC; ++v) out[v] = add(out[v], mul(w, A[((long long)al * din + i) * Ar + ar + v]));
        }
        store_vec<T, VEC>(crow + (long long)cb2 * Ar + ar, out);
      }
    }
  }
}

// hadamard (blas.hpp:45-67): C[(a*Bl + b), s, (a2*Br + b2)] = A[a, s, a2] B[b, s, b2].
// Row r = (a*Bl + b)*d + s; columns (a2, b2).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) expand_hadamard_kernel(const T* __restrict__ A, const T* __restrict__ B,
                                                               T* __restrict__ C, int Al, int d, int Ar, int Bl,
                                                               int Br, long long sA, long long sB, long long sC) {
  const int chain = blockIdx.z;
  A += sA * chain;
  B += sB * chain;
  C += sC * chain;
  const int rows = Al * Bl * d;
  const long long cols = (long long)Ar * Br;
  for (int row = blockIdx.y * gridDim.x + blockIdx.x; row < rows; row += gridDim.x * gridDim.y) {
    const int s = row % d, ab = row / d;
    const int a = ab / Bl, b = ab - a * Bl;
    T* crow = C + (long long)row * cols;
    const T* arow = A + ((long long)a * d + s) * Ar;
    const T* brow = B + ((long long)b * d + s) * Br;
    for (int b2 = threadIdx.x * VEC; b2 < Br; b2 += blockDim.x * VEC) {
      T bv[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) bv[v] = brow[b2 + v];
      for (int a2 = 0; a2 < Ar; ++a2) {
        const T x = arow[a2];
        T out[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) out[v] = mul(x, bv[v]);
        store_vec<T, VEC>(crow + (long long)a2 * Br + b2, out);
      }
    }
  }
}

template <typename T>
__global__ void frob2_kernel(const T* X, long long sX, DimExpr rows, DimExpr cols, const int* bonds, int ld,
                             double* out, long long s_out) {
  const int chain = blockIdx.x;
  const long long n = (long long)rows.eval(bonds, chain, ld) * cols.eval(bonds, chain, ld);
  const T* x = X + sX * chain;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += abs2(x[i]);
  acc = block_sum(acc);
  if (threadIdx.x == 0) out[s_out * chain] = acc;
}

template <typename T>
__global__ void sweep_end_kernel(const T* psi0, long long s_psi0, DimExpr elems, const int* bonds, int ld,
                                 ChainState* st, double simp_tol, int sweep_index) {
  const int chain = blockIdx.x;
  ChainState* c = st + chain;
  if (!c->active) return;
  const long long n = elems.eval(bonds, chain, ld);
  const T* x = psi0 + s_psi0 * chain;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += abs2(x[i]);
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    // CanonicalMPS::norm_squared = |center|_F^2 (mps.hpp:222-224); sweep returns
    // max(0, target_norm2 - |psi|^2) (simplify.hpp:90)
    const double prev = c->dist2;
    const double dist2 = fmax(0.0, c->target_norm2 - acc);
    c->prev_dist2 = prev;
    c->dist2 = dist2;
    c->sweeps += 1;
    const double target_norm = sqrt(c->target_norm2);
    if (sqrt(dist2) <= simp_tol * target_norm) {  // simplify.hpp:118
      c->converged = 1;
      c->active = 0;
    } else if (sweep_index > 0 && fabs(prev - dist2) <= 1e-15 * c->target_norm2) {  // simplify.hpp:123
      c->active = 0;
    }
  }
}

template <typename T>
__global__ void copy_dims_kernel(const T* src, long long s_src, T* dst, long long s_dst, DimExpr rows,
                                   DimExpr cols, const int* bonds, int ld, const ChainState* st, int check_active) {
  const int chain = blockIdx.y;
  if (check_active && st && !st[chain].active) return;
  const long long n = (long long)rows.eval(bonds, chain, ld) * cols.eval(bonds, chain, ld);
  const T* s = src + s_src * chain;
  T* d = dst + s_dst * chain;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}

template <typename T>
__global__ void fill_one_kernel(T* dst, long long s_dst, int chains) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < chains) dst[s_dst * c] = Scalar<T>::one();
}

__global__ void any_imag_kernel(const cplx* x, long long n, int* flag) {
  int hit = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    hit |= x[i].y != 0.0;
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void complex_to_real_kernel(const cplx* src, double* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i].x;
}

__global__ void real_to_complex_kernel(const double* src, cplx* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = cplx{src[i], 0.0};
}

template <typename T>
__global__ void gather_kernel(const T* const* srcs, T* dst, long long elems, long long s_dst) {
  const int chain = blockIdx.y;
  const T* s = srcs[chain];
  T* d = dst + s_dst * chain;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < elems;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void init_state_kernel(ChainState* st, int chains) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < chains) {
    ChainState z{};
    z.active = 1;
    st[c] = z;
  }
}

__global__ void begin_sweeps_kernel(ChainState* st, int chains) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < chains) {
    const double tn = sqrt(fmax(0.0, st[c].target_norm2));
    st[c].active = tn > 32.0 * 2.220446049250313e-16 ? 1 : 0;
    st[c].dist2 = st[c].target_norm2;
  }
}

__global__ void set_bonds_kernel(int* bonds, const int* values, int ld, int count, int chains) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count * chains) bonds[(idx / count) * ld + idx % count] = values[idx % count];
}

template <typename T>
__global__ void scale_chains_kernel(T* x, long long s_x, long long elems, const double* f) {
  const int chain = blockIdx.y;
  T* p = x + s_x * chain;
  const double a = f[chain];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < elems; i += (long long)gridDim.x * blockDim.x)
    p[i] = scale(p[i], a);
}

__global__ void copy_bond_kernel(int* bonds, int ld, int from, int to, int chains) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < chains) bonds[c * ld + to] = bonds[c * ld + from];
}

template <typename TS, typename TD>
__global__ void join_block_kernel(const TS* src, int a_dim, int d, int b_dim, TD* dst, int dst_right, int offl, int offr,
                                  double f_re, double f_im) {
  const long long total = (long long)a_dim * d * b_dim;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx % b_dim);
    const long long as = idx / b_dim;
    const int sp = (int)(as % d), a = (int)(as / d);
    TD* o = dst + ((long long)(offl + a) * d + sp) * dst_right + offr + b;
    if constexpr (Scalar<TD>::is_complex) {
      cplx x;
      if constexpr (Scalar<TS>::is_complex)
        x = src[idx];
      else
        x = cplx{src[idx], 0.0};
      const cplx y = *o;  // accumulate: blocks are disjoint except for the summed one-site case
      *o = cplx{y.x + f_re * x.x - f_im * x.y, y.y + f_re * x.y + f_im * x.x};
    } else {
      *o += f_re * src[idx];
    }
  }
}

template <typename T>
__global__ void env_real_kernel(const T* X, long long sX, double* out, long long s_out, int chains) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= chains) return;
  double v;
  if constexpr (Scalar<T>::is_complex)
    v = X[c * sX].x;
  else
    v = X[c * sX];
  out[c * s_out] = v > 0.0 ? v : 0.0;
}

int grid_for(long long total, int threads) {
  long long b = (total + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

template <typename T>
cudaError_t expand_mpo(const T* W, const T* A, T* C, int Dl, int dout, int din, int Dr, int Al, int Ar, int chains,
                       long long sA, long long sC, cudaStream_t s) {
  const int rows = Dl * Al * dout;
  const dim3 grid(std::min(rows, 32768), (rows + 32767) / 32768, chains);
  // threads per row: enough for one pass over Ar
  const bool vec2 = !Scalar<T>::is_complex && (Ar % 2 == 0);
  const int per = vec2 ? (Ar / 2) : Ar;
  const int nt = per >= 256 ? 256 : std::max(32, (per + 31) / 32 * 32);
  if constexpr (!Scalar<T>::is_complex) {
    if (vec2) {
      expand_mpo_kernel<T, 2><<<grid, nt, 0, s>>>(W, A, C, Dl, dout, din, Dr, Al, Ar, sA, sC);
      return cudaGetLastError();
    }
  }
  expand_mpo_kernel<T, 1><<<grid, nt, 0, s>>>(W, A, C, Dl, dout, din, Dr, Al, Ar, sA, sC);
  return cudaGetLastError();
}

template <typename T>
cudaError_t expand_hadamard(const T* A, const T* B, T* C, int Al, int d, int Ar, int Bl, int Br, int chains,
                            long long sA, long long sB, long long sC, cudaStream_t s) {
  const int rows = Al * Bl * d;
  const dim3 grid(std::min(rows, 32768), (rows + 32767) / 32768, chains);
  const bool vec2 = !Scalar<T>::is_complex && (Br % 2 == 0);
  const int per = vec2 ? (Br / 2) : Br;
  const int nt = per >= 256 ? 256 : std::max(32, (per + 31) / 32 * 32);
  if constexpr (!Scalar<T>::is_complex) {
    if (vec2) {
      expand_hadamard_kernel<T, 2><<<grid, nt, 0, s>>>(A, B, C, Al, d, Ar, Bl, Br, sA, sB, sC);
      return cudaGetLastError();
    }
  }
  expand_hadamard_kernel<T, 1><<<grid, nt, 0, s>>>(A, B, C, Al, d, Ar, Bl, Br, sA, sB, sC);
  return cudaGetLastError();
}

template <typename T>
cudaError_t frob2(const T* X, long long sX, DimExpr rows, DimExpr cols, const int* bonds, int ld, double* out,
                  long long s_out, int chains, cudaStream_t s) {
  frob2_kernel<T><<<chains, 512, 0, s>>>(X, sX, rows, cols, bonds, ld, out, s_out);
  return cudaGetLastError();
}

template <typename T>
cudaError_t sweep_end(const T* psi0, long long s_psi0, DimExpr elems, const int* bonds, int ld, ChainState* st,
                      double simp_tol, int sweep_index, int chains, cudaStream_t s) {
  sweep_end_kernel<T><<<chains, 256, 0, s>>>(psi0, s_psi0, elems, bonds, ld, st, simp_tol, sweep_index);
  return cudaGetLastError();
}

template <typename T>
cudaError_t copy_dims(const T* src, long long s_src, T* dst, long long s_dst, DimExpr rows, DimExpr cols,
                        const int* bonds, int ld, const ChainState* st, int check_active, long long max_elems,
                        int chains, cudaStream_t s) {
  copy_dims_kernel<T><<<dim3(grid_for(max_elems, 256), chains), 256, 0, s>>>(src, s_src, dst, s_dst, rows, cols,
                                                                               bonds, ld, st, check_active);
  return cudaGetLastError();
}

template <typename T>
cudaError_t fill_one(T* dst, long long s_dst, int chains, cudaStream_t s) {
  fill_one_kernel<T><<<(chains + 255) / 256, 256, 0, s>>>(dst, s_dst, chains);
  return cudaGetLastError();
}

cudaError_t any_imag(const cplx* x, long long n, int* flag, cudaStream_t s) {
  any_imag_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, flag);
  return cudaGetLastError();
}

cudaError_t complex_to_real(const cplx* src, double* dst, long long n, cudaStream_t s) {
  complex_to_real_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

cudaError_t real_to_complex(const double* src, cplx* dst, long long n, cudaStream_t s) {
  real_to_complex_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

template <typename T>
cudaError_t gather(const T* const* srcs, T* dst, long long elems, long long s_dst, int chains, cudaStream_t s) {
  gather_kernel<T><<<dim3(grid_for(elems, 256), chains), 256, 0, s>>>(srcs, dst, elems, s_dst);
  return cudaGetLastError();
}

cudaError_t init_state(ChainState* st, int chains, cudaStream_t s) {
  init_state_kernel<<<(chains + 255) / 256, 256, 0, s>>>(st, chains);
  return cudaGetLastError();
}

template <typename TS, typename TD>
cudaError_t join_block(const TS* src, int a_dim, int d, int b_dim, TD* dst, int dst_right, int offl, int offr,
                       double f_re, double f_im, cudaStream_t s) {
  const long long total = (long long)a_dim * d * b_dim;
  join_block_kernel<TS, TD><<<grid_for(total, 256), 256, 0, s>>>(src, a_dim, d, b_dim, dst, dst_right, offl, offr,
                                                                 f_re, f_im);
  return cudaGetLastError();
}
template cudaError_t join_block<double, double>(const double*, int, int, int, double*, int, int, int, double, double,
                                                cudaStream_t);
template cudaError_t join_block<double, cplx>(const double*, int, int, int, cplx*, int, int, int, double, double,
                                              cudaStream_t);
template cudaError_t join_block<cplx, cplx>(const cplx*, int, int, int, cplx*, int, int, int, double, double,
                                            cudaStream_t);

template <typename T>
cudaError_t env_real(const T* X, long long sX, double* out, long long s_out, int chains, cudaStream_t s) {
  env_real_kernel<T><<<(chains + 127) / 128, 128, 0, s>>>(X, sX, out, s_out, chains);
  return cudaGetLastError();
}
template cudaError_t env_real<double>(const double*, long long, double*, long long, int, cudaStream_t);
template cudaError_t env_real<cplx>(const cplx*, long long, double*, long long, int, cudaStream_t);

cudaError_t begin_sweeps(ChainState* st, int chains, cudaStream_t s) {
  begin_sweeps_kernel<<<(chains + 255) / 256, 256, 0, s>>>(st, chains);
  return cudaGetLastError();
}

template <typename T>
cudaError_t scale_chains(T* x, long long s_x, long long elems, const double* factors, int chains, cudaStream_t s) {
  scale_chains_kernel<T><<<dim3(grid_for(elems, 256), chains), 256, 0, s>>>(x, s_x, elems, factors);
  return cudaGetLastError();
}

cudaError_t copy_bond(int* bonds, int ld, int from, int to, int chains, cudaStream_t s) {
  copy_bond_kernel<<<(chains + 255) / 256, 256, 0, s>>>(bonds, ld, from, to, chains);
  return cudaGetLastError();
}

cudaError_t set_bonds(int* bonds, const int* values, int ld, int count, int chains, cudaStream_t s) {
  set_bonds_kernel<<<(count * chains + 255) / 256, 256, 0, s>>>(bonds, values, ld, count, chains);
  return cudaGetLastError();
}

#define TTG_INST(T)                                                                                               \
  template cudaError_t expand_mpo<T>(const T*, const T*, T*, int, int, int, int, int, int, int, long long,       \
                                     long long, cudaStream_t);                                                   \
  template cudaError_t expand_hadamard<T>(const T*, const T*, T*, int, int, int, int, int, int, long long,       \
                                          long long, long long, cudaStream_t);                                   \
  template cudaError_t frob2<T>(const T*, long long, DimExpr, DimExpr, const int*, int, double*, long long, int,  \
                                cudaStream_t);                                                                   \
  template cudaError_t sweep_end<T>(const T*, long long, DimExpr, const int*, int, ChainState*, double, int, int, \
                                    cudaStream_t);                                                               \
  template cudaError_t copy_dims<T>(const T*, long long, T*, long long, DimExpr, DimExpr, const int*, int,     \
                                      const ChainState*, int, long long, int, cudaStream_t);                     \
  template cudaError_t fill_one<T>(T*, long long, int, cudaStream_t);                                            \
  template cudaError_t scale_chains<T>(T*, long long, long long, const double*, int, cudaStream_t);              \
  template cudaError_t gather<T>(const T* const*, T*, long long, long long, int, cudaStream_t);
TTG_INST(double)
TTG_INST(cplx)

}  // namespace ttg
