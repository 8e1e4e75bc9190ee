// Blocked Householder QR of one shared-memory-resident panel per CTA: the
// preconditioner of the truncated two-site split (see qr.cuh, qr_precondition)
// for the panel sizes of the sweeps (l*k*sizeof(T) <= ~190 KB).
//
// The unblocked kernel (qr_pre_kernel) pays two CTA barriers and a pass over
// the whole trailing matrix per column.  Here warp 0 factors an NB-column
// panel entirely in registers (LAPACK xGEQR2 on the panel: one warp reduction
// per column norm, the trailing panel dots reduced together), and the whole
// CTA then applies the block reflector H_1..H_nb = I - V T V^H to the trailing
// columns in three register-blocked passes (W = V^H A, W = T^H W, A -= V W;
// xLARFT/xLARFB).  Q, when requested, is formed in place backwards
// (xORGQR): the block reflector is applied to the already formed columns and
// the panel's own columns are written directly as E - V (T V1^H).
#include "qr.cuh"

#include <cstdlib>

namespace ttg {
namespace {

constexpr int QRS_THREADS = 256;
constexpr int QRS_NW = QRS_THREADS / 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double shfl_(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ cplx shfl_(cplx v, int src) {
  return cplx{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
}
__device__ __forceinline__ double wsum_t(double v) { return wsum(v); }
__device__ __forceinline__ cplx wsum_t(cplx v) { return cplx{wsum(v.x), wsum(v.y)}; }
__device__ __forceinline__ double sum4(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}
__device__ __forceinline__ cplx sum4(cplx v) { return cplx{sum4(v.x), sum4(v.y)}; }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ cplx fma_(cplx a, cplx b, cplx c) {
  return cplx{fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
// c + conj(a) b
__device__ __forceinline__ double cfma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ cplx cfma_(cplx a, cplx b, cplx c) {
  return cplx{fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y))};
}

struct SmallLayout {
  int lw, k, npan;
  // element offsets
  long long vs, wb, w2, tall, z;
  long long total;
};

__host__ __device__ inline SmallLayout small_layout(int l, int k, int nb) {
  SmallLayout L;
  L.lw = l | 1;
  L.k = k;
  const int r0 = l < k ? l : k;
  L.npan = (r0 + nb - 1) / nb;
  L.vs = (long long)L.lw * k;          // Wk: l x k, column-major, stride lw
  L.wb = L.vs + (long long)L.lw * nb;  // Vs: l x nb, column-major, stride lw
  L.w2 = L.wb + (long long)nb * (k + nb + 1);
  L.tall = L.w2 + (long long)nb * (k + nb + 1);
  L.z = L.tall + (long long)L.npan * nb * nb;
  L.total = L.z + (long long)nb * nb;
  return L;
}

__device__ __forceinline__ void dmma_(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}
__device__ __forceinline__ double re_(double a) { return a; }
__device__ __forceinline__ double re_(cplx a) { return a.x; }
__device__ __forceinline__ double im_(double) { return 0.0; }
__device__ __forceinline__ double im_(cplx a) { return a.y; }

// acc (+)= A B for one m16n8k4 step; complex as four real DMMAs.  ar/ai: A fragment
// (rows g, g+8 at column t4), br/bi: B fragment (row t4, column g).
template <typename T>
__device__ __forceinline__ void cstep(double (&acc)[4], double (&acci)[4], double ar0, double ar1, double ai0,
                                      double ai1, double br, double bi) {
  dmma_(acc, ar0, ar1, br);
  if constexpr (Scalar<T>::is_complex) {
    dmma_(acc, -ai0, -ai1, bi);
    dmma_(acci, ar0, ar1, bi);
    dmma_(acci, ai0, ai1, br);
  }
}

// W[a][cc] = sum_{i in [j0, l)} conj(V[i][a]) X_cc[i] on the DMMA pipe, a < NB (one
// 16-row tile), cc < ncol.  Column cc of X is column col(cc) of the column-major
// smem block at Wk (stride lw): the panel's V (Vs == Wk + k*lw) for cc < nv, else
// Wk column xc0 + cc - nv.  V is zero above its unit diagonal and in columns >= nb.
template <typename T, int NB>
__device__ __forceinline__ void vh_times(const T* Wk, int k, int lw, int l, int j0, int nb, int nv, int xc0, int ncol,
                                         T* W, int ldw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const T* Vs = Wk + (long long)k * lw;
  const int ntiles = (nv + ncol + 7) >> 3;
  for (int nt_ = warp; nt_ < ntiles; nt_ += QRS_NW) {
    const int cc = nt_ * 8 + g;
    const bool con = cc < nv + ncol;
    const T* xc = Wk + (long long)(!con ? 0 : (cc < nv ? k + cc : xc0 + cc - nv)) * lw;
    const T* va = Vs + (long long)(g < NB ? g : 0) * lw;
    const T* vb = Vs + (long long)(g + 8 < NB ? g + 8 : 0) * lw;
    double acc[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
    for (int i0 = j0; i0 < l; i0 += 4) {
      const int i = i0 + t4;
      const bool ok = i < l;
      const T x = (ok && con) ? xc[i] : Scalar<T>::zero();
      const T a0 = (ok && g < nb) ? va[i] : Scalar<T>::zero();
      const T a1 = (ok && g + 8 < nb) ? vb[i] : Scalar<T>::zero();
      // conj(V): imaginary parts negated
      cstep<T>(acc, acci, re_(a0), re_(a1), -im_(a0), -im_(a1), re_(x), im_(x));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int a = g + (r >= 2 ? 8 : 0), c = nt_ * 8 + 2 * t4 + (r & 1);
      if (a < nb && c < nv + ncol) {
        if constexpr (Scalar<T>::is_complex)
          W[a * ldw + c] = cplx{acc[r], acci[r]};
        else
          W[a * ldw + c] = acc[r];
      }
    }
  }
}

// X[i][c] -= sum_{a < NB} V[i][a] Wt[a][wc0 + c] for i in [j0, l), c < ncol, X column
// c = Wk column xc0 + c.  DMMA tiles of 16 rows x 8 columns, K = NB.
template <typename T, int NB>
__device__ __forceinline__ void minus_v_times(T* Wk, int k, int lw, int l, int j0, int nb, int xc0, int ncol,
                                              const T* Wt, int ldw, int wc0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const T* Vs = Wk + (long long)k * lw;
  const int mp = l - j0;
  const int mt = (mp + 15) >> 4, ntl = (ncol + 7) >> 3;
  for (int tile = warp; tile < mt * ntl; tile += QRS_NW) {
    const int m0 = j0 + (tile % mt) * 16, n0 = (tile / mt) * 8;
    const int r0 = m0 + g, r1 = m0 + g + 8;
    double acc[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const int a = k0 + t4;
      const T* vcol = Vs + (long long)a * lw;
      const T v0 = (r0 < l && a < nb) ? vcol[r0] : Scalar<T>::zero();
      const T v1 = (r1 < l && a < nb) ? vcol[r1] : Scalar<T>::zero();
      const int c = n0 + g;
      const T w = (c < ncol && a < nb) ? Wt[a * ldw + wc0 + c] : Scalar<T>::zero();
      cstep<T>(acc, acci, re_(v0), re_(v1), im_(v0), im_(v1), re_(w), im_(w));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = r >= 2 ? r1 : r0, c = n0 + 2 * t4 + (r & 1);
      if (i < l && c < ncol) {
        T* xp = Wk + (long long)(xc0 + c) * lw + i;
        if constexpr (Scalar<T>::is_complex)
          *xp = cplx{xp->x - acc[r], xp->y - acci[r]};
        else
          *xp -= acc[r];
      }
    }
  }
}

// C[a][cc0 + c] = sum_{b < nb} op(T)[a][b] B[b][bc0 + c] for a < nb, c < ncol on the DMMA
// pipe; op(T) = T^H (CONJT) or T, T an NB x NB row-major block.
template <typename T, int NB, bool CONJT>
__device__ __forceinline__ void t_times(const T* Tp, int nb, const T* B, int ldb, int bc0, T* Cm, int ldc, int cc0,
                                        int ncol) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int ntl = (ncol + 7) >> 3;
  for (int tile = warp; tile < ntl; tile += QRS_NW) {
    const int n0 = tile * 8;
    double acc[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const int b = k0 + t4;
      T a0 = Scalar<T>::zero(), a1 = Scalar<T>::zero();
      if (b < nb) {
        if (g < nb) a0 = CONJT ? conj_(Tp[b * NB + g]) : Tp[g * NB + b];
        if (g + 8 < nb) a1 = CONJT ? conj_(Tp[b * NB + g + 8]) : Tp[(g + 8) * NB + b];
      }
      const int c = n0 + g;
      const T w = (b < nb && c < ncol) ? B[b * ldb + bc0 + c] : Scalar<T>::zero();
      cstep<T>(acc, acci, re_(a0), re_(a1), im_(a0), im_(a1), re_(w), im_(w));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int a = g + (r >= 2 ? 8 : 0), c = n0 + 2 * t4 + (r & 1);
      if (a < nb && c < ncol) {
        if constexpr (Scalar<T>::is_complex)
          Cm[a * ldc + cc0 + c] = cplx{acc[r], acci[r]};
        else
          Cm[a * ldc + cc0 + c] = acc[r];
      }
    }
  }
}

// Transposed warp reduction of NV (power of two, <= 32) values per lane: after
// log2(NV) halving exchanges (xor 16, 8, ...) each lane holds the warp total of
// one value, index treduce_index(lane); remaining xor steps finish the sum.
template <int NV>
__device__ __forceinline__ void treduce(double (&p)[NV], int lane) {
  int m = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h /= 2) {
    const bool up = lane & m;
#pragma unroll
    for (int q = 0; q < h; ++q) {
      const double send = up ? p[q] : p[q + h];
      const double keep = up ? p[q + h] : p[q];
      p[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
    m >>= 1;
  }
  for (; m >= 1; m >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], m);
}
template <int NV> __device__ __forceinline__ int treduce_index(int lane) {
  int idx = 0, m = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h /= 2) {
    if (lane & m) idx += h;
    m >>= 1;
  }
  return idx;
}
// lanes that differ only in these bits hold the same value
template <int NV> __host__ __device__ constexpr int treduce_dup_mask() { return 32 / NV - 1; }

// All-warp panel factorisation (real, NB <= 16): the panel's NB columns are
// spread over the lanes (two lanes per column, lane = 2c + h) and its rows over
// the 8 warps (lane half h of warp w holds rows 8 (2r + h) + w), so every
// warp holds a row slab of every column.  Per column ONE CTA reduction: each
// lane forms the partial x^H a_c over its rows (x = the pivot column, fetched
// from the lanes of the same warp that own it, which hold the same rows), the
// two halves combine by one shuffle and the 8 warp partials meet in shared
// memory behind one barrier; every lane then forms the same reflector (xLARFG)
// and updates its rows.  Row j + 1 of the panel (the next alpha and the
// a_c(j) terms) is published through shared memory for the next column; all
// scratch is double-buffered by column parity, so one barrier per column
// suffices.  Replaces the one-warp register panel, during which the other
// seven warps idled (profiles/r01_qrs.hot.txt: 42% of the stall samples).
template <int RS, int NB>
__device__ __forceinline__ void panel_allwarps(double* Wk, double* Vs, int lw, int l, int j0, int nb, double* taus,
                                               double (*part)[QRS_NW][NB], double (*srow)[NB]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane >> 1, h = lane & 1;
  const bool cv = c < nb;
  double a[RS];
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const int i = 8 * (2 * r + h) + warp;
    a[r] = (cv && i < l) ? Wk[(long long)(j0 + c) * lw + i] : 0.0;
    if (cv && i == j0) srow[0][c] = a[r];
  }
  __syncthreads();
#pragma unroll 1
  for (int jj = 0; jj < nb; ++jj) {
    const int j = j0 + jj, buf = jj & 1;
    // pivot column values at my rows (lanes 2 jj + h hold the same rows)
    double x[RS];
    double q = 0.0;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      x[r] = __shfl_sync(0xffffffffu, a[r], 2 * jj + h);
      const int i = 8 * (2 * r + h) + warp;
      if (i > j && i < l) q = fma(x[r], a[r], q);
    }
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    if (h == 0 && cv) part[buf][warp][c] = q;
    __syncthreads();
    double qc = 0.0, xn2 = 0.0;
#pragma unroll
    for (int w = 0; w < QRS_NW; ++w) {
      qc += cv ? part[buf][w][c] : 0.0;
      xn2 += part[buf][w][jj];
    }
    const double alpha = srow[buf][jj];
    double tau = 0.0, beta = alpha, sc = 0.0;
    if (xn2 != 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
      tau = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    if (c > jj && cv) {
      // v^H a_c = a_c(j) + sc * x^H a_c (v_j = 1, v_i = sc x_i below)
      const double f = tau * fma(sc, qc, srow[buf][c]);
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int i = 8 * (2 * r + h) + warp;
        if (i > j && i < l)
          a[r] = fma(-f, x[r] * sc, a[r]);
        else if (i == j)
          a[r] -= f;
      }
    } else if (c == jj) {
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        const int i = 8 * (2 * r + h) + warp;
        if (i > j && i < l)
          a[r] *= sc;
        else if (i == j)
          a[r] = beta;
      }
    }
    // row j + 1 of the remaining columns for the next column step
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int i = 8 * (2 * r + h) + warp;
      if (i == j + 1 && cv) srow[buf ^ 1][c] = a[r];
    }
    if (threadIdx.x == 0) taus[jj] = tau;
  }
  // factored panel back to Wk (R on/above the diagonal, v below) and the explicit V to Vs
#pragma unroll
  for (int r = 0; r < RS; ++r) {
    const int i = 8 * (2 * r + h) + warp;
    if (cv && i < l) {
      const int jc = j0 + c;
      Wk[(long long)jc * lw + i] = a[r];
      Vs[(long long)c * lw + i] = i > jc ? a[r] : (i == jc ? 1.0 : 0.0);
    }
  }
}

template <typename T, int RT, int NB, bool ALLW>
__global__ void __launch_bounds__(QRS_THREADS, 1)
    qr_small_kernel(const T* A, long long sA, DimExpr Md, DimExpr Nd, int trans, int* bonds, int ld, int out_idx,
                    T* Q, long long sQ, T* RH, long long sRH, const ChainState* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T S[NB][NB + 1];
  __shared__ T taus[NB];
  __shared__ T srow[NB];
  __shared__ double red[Scalar<T>::is_complex ? 2 * NB : NB];
  const int chain = blockIdx.x;
  if (st && !st[chain].active) return;
  ttg_smem_poison(smem_raw);
  const int mi = Md.eval(bonds, chain, ld), ni = Nd.eval(bonds, chain, ld);
  const bool out_r = (trans & 2) != 0;  // write R (r0 x k) instead of R^H
  trans &= 1;
  const int l = trans ? ni : mi, k = trans ? mi : ni, r0 = min(l, k);
  const SmallLayout Ly = small_layout(l, k, NB);
  const int lw = Ly.lw;
  T* Wk = reinterpret_cast<T*>(smem_raw);
  T* Vs = Wk + Ly.vs;
  T* Wb = Wk + Ly.wb;
  T* W2 = Wk + Ly.w2;
  T* Tall = Wk + Ly.tall;
  T* Z = Wk + Ly.z;
  const int ldw = k + NB + 1;  // odd: conflict-free fragment loads
  A += sA * chain;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < mi * ni; idx += QRS_THREADS) {
    const int r = idx / ni, c = idx % ni;
    if (trans)
      Wk[r * lw + c] = conj_(A[idx]);
    else
      Wk[c * lw + r] = A[idx];
  }
  __syncthreads();
  for (int j0 = 0, p = 0; j0 < r0; j0 += NB, ++p) {
    const int nb = min(NB, r0 - j0);
    T* Tp = Tall + (long long)p * NB * NB;
    if constexpr (ALLW) {
      __shared__ double s_part[2][QRS_NW][NB];
      __shared__ double s_row[2][NB];
      panel_allwarps<2 * RT, NB>(Wk, Vs, lw, l, j0, nb, taus, s_part, s_row);
    } else if (warp == 0) {
      // ---- panel factorisation in registers: lane holds rows j0 + lane + 32 t of
      // a rolling window of NB columns (a[t][0] = the current column; the window
      // shifts left after every column, so the loop body is the same code for all
      // columns and stays in the instruction cache).  One transposed warp
      // reduction per column yields |x|^2 (rows > j) and the raw dots
      // d_c = x^H a_c of the trailing panel columns; with v = sc x (v_j = 1):
      // v^H a_c = a_c(j) + conj(sc) d_c.
      T a[RT][NB];
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = j0 + lane + 32 * t;
#pragma unroll
        for (int c = 0; c < NB; ++c) a[t][c] = (i < l && c < nb) ? Wk[(long long)(j0 + c) * lw + i] : Scalar<T>::zero();
      }
      constexpr int NV = Scalar<T>::is_complex ? 2 * NB : NB;
      const int my_idx = treduce_index<NV>(lane);
#pragma unroll 1
      for (int jj = 0; jj < nb; ++jj) {
        const int j = j0 + jj;
        double pv[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) pv[q] = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j0 + lane + 32 * t;
          if (i > j && i < l) {
            const T x = a[t][0];
            if constexpr (Scalar<T>::is_complex) {
              pv[0] += abs2(x);
#pragma unroll
              for (int c = 1; c < NB; ++c) {
                const cplx d = cmul(x, a[t][c]);
                pv[2 * c] += d.x;
                pv[2 * c + 1] += d.y;
              }
            } else {
              pv[0] += x * x;
#pragma unroll
              for (int c = 1; c < NB; ++c) pv[c] += x * a[t][c];
            }
          }
          if (i == j) {
#pragma unroll
            for (int c = 0; c < NB; ++c) srow[c] = a[t][c];
          }
        }
        treduce<NV>(pv, lane);
        if ((lane & treduce_dup_mask<NV>()) == 0) red[my_idx] = pv[0];
        __syncwarp();
        const double xn2 = red[0];
        const T alpha = srow[0];
        double ar, ai;
        if constexpr (Scalar<T>::is_complex) {
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
          if constexpr (Scalar<T>::is_complex) {
            tau = cplx{(beta - ar) * rb, -ai * rb};
            const double dr = ar - beta, di = ai, rden = 1.0 / (dr * dr + di * di);
            sc = cplx{dr * rden, -di * rden};
          } else {
            tau = (beta - ar) * rb;
            sc = 1.0 / (ar - beta);
          }
        }
        // f_c = conj(tau) (a_c(j) + conj(sc) d_c); a_c -= v f_c
        T f[NB];
#pragma unroll
        for (int c = 1; c < NB; ++c) {
          T d;
          if constexpr (Scalar<T>::is_complex)
            d = cplx{red[2 * c], red[2 * c + 1]};
          else
            d = red[c];
          f[c] = mul(conj_(tau), add(srow[c], mul(conj_(sc), d)));
        }
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j0 + lane + 32 * t;
          if (i > j && i < l) {
            const T v = mul(a[t][0], sc);
            a[t][0] = v;
#pragma unroll
            for (int c = 1; c < NB; ++c) a[t][c] = sub(a[t][c], mul(v, f[c]));
          } else if (i == j) {
#pragma unroll
            for (int c = 1; c < NB; ++c) a[t][c] = sub(a[t][c], f[c]);
            if (refl) {
              if constexpr (Scalar<T>::is_complex)
                a[t][0] = cplx{beta, 0.0};
              else
                a[t][0] = beta;
            }
          }
          // column j done: R (rows <= j) and V (rows > j) to Wk, explicit V to Vs
          if (i < l) {
            Wk[(long long)j * lw + i] = a[t][0];
            Vs[(long long)jj * lw + i] = i > j ? a[t][0] : (i == j ? Scalar<T>::one() : Scalar<T>::zero());
          }
#pragma unroll
          for (int c = 0; c + 1 < NB; ++c) a[t][c] = a[t][c + 1];
          a[t][NB - 1] = Scalar<T>::zero();
        }
        if (lane == 0) taus[jj] = tau;
        __syncwarp();
      }
    }
    __syncthreads();
    const int nt = k - (j0 + nb);
    // S = V^H V (the nb x nb Gram of the reflectors) and W = V^H A_trail
    vh_times<T, NB>(Wk, k, lw, l, j0, nb, nb, j0 + nb, nt, Wb, ldw);
    __syncthreads();
    if (warp == 0 && lane < NB) {
      // xLARFT in registers, lane r owns row r of T:
      // T[i][i] = tau_i, T[r][i] = -tau_i sum_{r <= c < i} T[r][c] S[c][i]  (S = V^H V)
      T trow[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        T v = Scalar<T>::zero();
        if (i < nb) {
          const T ti = taus[i];
          if (lane < i) {
            T acc = Scalar<T>::zero();
#pragma unroll
            for (int c = 0; c < i; ++c)
              if (c >= lane) acc = add(acc, mul(trow[c], Wb[c * ldw + i]));
            v = mul(sub(Scalar<T>::zero(), ti), acc);
          } else if (lane == i) {
            v = ti;
          }
        }
        trow[i] = v;
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) Tp[lane * NB + c] = trow[c];
    }
    __syncthreads();
    // W2 = T^H W on the trailing columns (DMMA)
    t_times<T, NB, true>(Tp, nb, Wb, ldw, nb, W2, ldw, 0, nt);
    __syncthreads();
    minus_v_times<T, NB>(Wk, k, lw, l, j0, nb, j0 + nb, nt, W2, ldw, 0);
    __syncthreads();
  }
  // R1^H (k x r0): RH[c, i] = conj(R1[i, c]) for c >= i; with trans & 2: R1 itself (r0 x k)
  T* rh = RH + sRH * chain;
  if (out_r) {
    for (int idx = tid; idx < r0 * k; idx += QRS_THREADS) {
      const int i = idx / k, c = idx % k;
      rh[idx] = (c >= i) ? Wk[(long long)c * lw + i] : Scalar<T>::zero();
    }
  } else {
    for (int idx = tid; idx < k * r0; idx += QRS_THREADS) {
      const int c = idx / r0, i = idx % r0;
      rh[idx] = (c >= i) ? conj_(Wk[(long long)c * lw + i]) : Scalar<T>::zero();
    }
  }
  if (tid == 0) bonds[chain * ld + out_idx] = r0;
  if (!Q) return;
  __syncthreads();
  // ---- Q1 = H_1 ... H_r0 [I; 0] in place (blocked xORGQR), panels backwards
  for (int p = Ly.npan - 1; p >= 0; --p) {
    const int j0 = p * NB, nb = min(NB, r0 - j0);
    const T* Tp = Tall + (long long)p * NB * NB;
    for (int idx = tid; idx < nb * (l - j0); idx += QRS_THREADS) {
      const int c = idx / (l - j0), i = j0 + idx % (l - j0), j = j0 + c;
      Vs[(long long)c * lw + i] =
          i > j ? Wk[(long long)j * lw + i] : (i == j ? Scalar<T>::one() : Scalar<T>::zero());
    }
    __syncthreads();
    const int nt = r0 - (j0 + nb);
    if (nt > 0) vh_times<T, NB>(Wk, k, lw, l, j0, nb, 0, j0 + nb, nt, Wb, ldw);
    __syncthreads();
    // W2 = [Z | T W]: Z = T V1^H for the panel's own columns (V1[c][b] = V[j0+c][b]),
    // T W for the formed columns to the right
    if (nt > 0) t_times<T, NB, false>(Tp, nb, Wb, ldw, 0, W2, ldw, nb, nt);
    for (int idx = tid; idx < nb * nb; idx += QRS_THREADS) {
      const int a_ = idx / nb, c = idx % nb;
      T acc = Scalar<T>::zero();
      for (int b = a_; b < nb; ++b) acc = fma_(Tp[a_ * NB + b], conj_(Vs[(long long)b * lw + j0 + c]), acc);
      W2[a_ * ldw + c] = acc;
    }
    // panel columns start as E (rows >= j0), zero above
    for (int idx = tid; idx < nb * l; idx += QRS_THREADS) {
      const int c = idx / l, i = idx % l;
      Wk[(long long)(j0 + c) * lw + i] = (i == j0 + c) ? Scalar<T>::one() : Scalar<T>::zero();
    }
    __syncthreads();
    minus_v_times<T, NB>(Wk, k, lw, l, j0, nb, j0, nb + nt, W2, ldw, 0);
    __syncthreads();
  }
  T* q = Q + sQ * chain;
  for (int idx = tid; idx < l * r0; idx += QRS_THREADS) {
    const int i = idx / r0, c = idx % r0;
    q[idx] = Wk[(long long)c * lw + i];
  }
}

bool qr_panel_allwarps() {
  static const bool on = [] {
    const char* e = std::getenv("TTG_QR_PANEL_ALL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T, int RT, int NB>
cudaError_t launch_small(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld, int out_idx,
                         void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax, const ChainState* st,
                         int chains, cudaStream_t s) {
  const SmallLayout L = small_layout(lmax, kmax, NB);
  const size_t bytes = (size_t)L.total * sizeof(T);
  constexpr bool CAN_ALLW = !Scalar<T>::is_complex && NB == 16;  // two lanes per panel column
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    kern<<<chains, QRS_THREADS, bytes, s>>>(static_cast<const T*>(A), sA, M, N, trans, bonds, ld, out_idx,
                                           static_cast<T*>(Q), sQ, static_cast<T*>(RH), sRH, st);
    return cudaGetLastError();
  };
  if constexpr (CAN_ALLW) {
    if (qr_panel_allwarps()) return go(qr_small_kernel<T, RT, NB, true>);
  }
  return go(qr_small_kernel<T, RT, NB, false>);
}

}  // namespace

template <typename T> constexpr int small_nb(int rt) {
  return Scalar<T>::is_complex ? (rt <= 2 ? 16 : (rt <= 4 ? 8 : 4)) : (rt <= 4 ? 16 : 8);
}

size_t qr_small_bytes(int l, int k, bool cplx_) {
  const int rt = l <= 32 ? 1 : l <= 64 ? 2 : l <= 128 ? 4 : 8;
  const int nb = cplx_ ? small_nb<cplx>(rt) : small_nb<double>(rt);
  return (size_t)small_layout(l, k, nb).total * (cplx_ ? 16 : 8);
}

template <typename T>
cudaError_t qr_precondition_small(const void* A, long long sA, DimExpr M, DimExpr N, int trans, int* bonds, int ld,
                                  int out_idx, void* Q, long long sQ, void* RH, long long sRH, int lmax, int kmax,
                                  const ChainState* st, int chains, cudaStream_t s) {
  if (lmax > 256 || qr_small_bytes(lmax, kmax, Scalar<T>::is_complex) > QR_SMALL_SMEM_LIMIT) return cudaErrorInvalidValue;
  if (lmax <= 32) return launch_small<T, 1, small_nb<T>(1)>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH,
                                                             lmax, kmax, st, chains, s);
  if (lmax <= 64) return launch_small<T, 2, small_nb<T>(2)>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH,
                                                             lmax, kmax, st, chains, s);
  if (lmax <= 128) return launch_small<T, 4, small_nb<T>(4)>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH,
                                                              lmax, kmax, st, chains, s);
  return launch_small<T, 8, small_nb<T>(8)>(A, sA, M, N, trans, bonds, ld, out_idx, Q, sQ, RH, sRH, lmax, kmax, st,
                                            chains, s);
}

template cudaError_t qr_precondition_small<double>(const void*, long long, DimExpr, DimExpr, int, int*, int, int,
                                                   void*, long long, void*, long long, int, int, const ChainState*, int,
                                                   cudaStream_t);
template cudaError_t qr_precondition_small<cplx>(const void*, long long, DimExpr, DimExpr, int, int*, int, int, void*,
                                                 long long, void*, long long, int, int, const ChainState*, int,
                                                 cudaStream_t);

}  // namespace ttg
