// Helpers shared by the Jacobi SVD kernels (jacobi_svd.cu, jacobi_bg.cu): retry policy,
// rotation angle, stop rules, and the workspace layout / epilogue of the grid-cooperative kernels.
#pragma once

#include "jacobi_svd.cuh"

#include <cfloat>
#include <cooperative_groups.h>

namespace ttg {
namespace {

constexpr int SVD_THREADS = 256;
constexpr int MAX_SWEEPS = 60;

// Retry policy of svd_with_retry (schmidt.hpp:23-35): a split whose sweeps do
// not converge within the budget is not an error on the first attempt.  The
// kernel flags the chain ST_RETRY (no ledger update), the engine jitters theta
// by 1e-14 |theta|_F times a fixed pattern (svd_jitter_kernel) and relaunches
// the split with attempt = 1, which runs only for flagged chains; a second
// failure is ST_NOCONV (numeric_error).  first_budget > 0 shortens the first
// attempt (forced-failure test hook, TTG_SVD_FORCE_RETRY).
__device__ __forceinline__ int sweep_budget(const SvdParams& p) {
  return (p.attempt == 0 && p.first_budget > 0) ? p.first_budget : MAX_SWEEPS;
}
__device__ __forceinline__ bool retry_skip(const SvdParams& p, const ChainState* st) {
  return p.attempt != 0 && !(st && (st->status & ST_RETRY));
}
__device__ __forceinline__ bool will_retry(const SvdParams& p, bool noconv) {
  return noconv && p.attempt == 0 && p.retry;
}
__device__ __forceinline__ void finish_status(const SvdParams& p, ChainState* st, bool bad, bool noconv) {
  if (!st) return;
  int v = st->status & ~ST_RETRY;
  if (bad) v |= ST_NONFINITE;
  if (noconv) v |= will_retry(p, noconv) ? ST_RETRY : ST_NOCONV;
  st->status = v;
}

// Early stop.  Cyclic Jacobi converges quadratically: after a sweep whose
// largest rotated cosine is c, the next sweep starts from cosines of order c^2
// (measured on C2 splits: c 2e-9 .. 6e-7 -> next sweep 0 .. 7e-14 = below
// tol_rot).  A sweep that rotates nothing with cos^2 > tol_rot / 100 ends the
// iteration, which drops the final all-skipped check sweep in most splits
// (C2: 7.8 -> 6.9 sweeps per split, same singular values and isometries).
// TTG_SVD_EARLY=0 (p.no_early) restores the check sweep.
// Ring kernels (one CTA or one cluster per chain, unpreconditioned or small splits): clustered
// singular values (sigma = 1 +- 1e-9 blocks, tools/orth_probe.py) left cosines of 6000 cos^2 behind a
// sweep that looked quadratic, so their early stop keeps a factor 1e4 instead of 100.
__device__ __forceinline__ double early_stop2_ring(const SvdParams& p, double tol_rot) {
  return p.no_early == 1 ? tol_rot * tol_rot : fmax(tol_rot * tol_rot, 1.0e-4 * tol_rot);
}
__device__ __forceinline__ double early_stop2(const SvdParams& p, double tol_rot) {
  // no_early: 0 = default margin (cos^2 <= tol_rot / 100), 1 = no early stop, 2 = cos^2 <= tol_rot / 10 (experiment)
  return p.no_early == 1 ? tol_rot * tol_rot : fmax(tol_rot * tol_rot, (p.no_early == 2 ? 0.1 : 0.01) * tol_rot);
}

// 1/sqrt(w) for w in [1, 2]: single-precision seed + two Newton steps (full double)
__device__ __forceinline__ double rsqrt_12(double w) {
  double y = (double)rsqrtf((float)w);
  y = y * fma(-0.5 * w, y * y, 1.5);
  y = y * fma(-0.5 * w, y * y, 1.5);
  return y;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Rotation angle without divergent branches or double-precision divisions:
// alpha, beta, g are scaled into float range by an exact power of two and
// t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (beta - alpha) / (2g),
// is formed in float (only the orthogonality of the rotation matters, and
// c = (1 + t^2)^-1/2 is formed in double).  Tiny angles (2g/scale < 1e-30,
// i.e. |alpha - beta| ~ scale) use t = g / (beta - alpha) with a refined
// float reciprocal.  Requires g > 0.
__device__ __forceinline__ double ring_tan(double alpha, double beta, double g) {
  const double sc = fmax(fmax(alpha, beta), g);
  int eb = (__double2hiint(sc) >> 20) & 0x7ff;
  eb = eb > 2045 ? 2045 : eb;
  const double f = __hiloint2double((2046 - eb) << 20, 0);  // 2^-(eb - 1023)
  const double num = (beta - alpha) * f, den = 2.0 * g * f;  // |num| < 2, 0 <= den < 4
  const float fn = (float)num, fd = (float)den;
  const float an = fabsf(fn);
  const bool big = an >= fd;
  const float u = big ? __fdividef(fd, an) : __fdividef(fn, fd);  // 1/|zeta| or zeta
  const float w = fmaf(u, u, 1.0f);
  const float sq = w * rsqrtf(w);  // sqrt(1 + u^2)
  const float tb = __fdividef(u, 1.0f + sq);            // |zeta| >= 1
  const float ts = __fdividef(1.0f, fabsf(u) + sq);     // |zeta| < 1
  const float tf = copysignf(big ? tb : ts, big ? fn : u);
  double r = (double)__frcp_rn(fn);
  r = r * fma(-num, r, 2.0);
  const double tt = 0.5 * den * r;
  return den < 1e-30 ? tt : (double)tf;
}

__device__ __forceinline__ float bg_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float bg_rsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Rotation of a pair from (alpha, beta, g = |inner product| > 0): tangent t (signed like beta - alpha)
// and cosine c = (1 + t^2)^-1/2 with c accurate to double precision (the rotation must be orthogonal
// to rounding; the angle itself only needs single precision).  alpha, beta, g are scaled into float
// range by an exact power of two (g <= sqrt(alpha beta) <= max(alpha, beta), so the larger high word
// gives the exponent).  With fn = (beta - alpha) f, fd = 2 g f and r = sqrt(fn^2 + fd^2):
//   t = fd / (|fn| + r)           (= 1 / (|zeta| + sqrt(1 + zeta^2)), zeta = fn / fd; no case split,
//                                  and the tiny-angle limit g / (beta - alpha) comes out by itself)
//   c^2 = (|fn| + r) / (2 r)      (half-angle), so the seed of c needs no extra dependent MUFU:
//                                  rcp(|fn| + r) and rsqrt(c^2) issue together
// followed by one Halley step for c in double (seed error 2^-22 -> ~1e-20).
__device__ __forceinline__ void bg_rotation(double alpha, double beta, double g, double& t, double& c) {
  int eb = (max(__double2hiint(alpha), __double2hiint(beta)) >> 20) & 0x7ff;
  eb = eb > 2045 ? 2045 : eb;
  const double f = __hiloint2double((2046 - eb) << 20, 0);
  const float fn = (float)((beta - alpha) * f), fd = (float)(2.0 * g * f);  // |fn| < 2, 0 <= fd < 4
  const float an = fabsf(fn);
  const float s2 = fmaf(fn, fn, fd * fd);
  const float rs = bg_rsqrt(s2);           // 1 / r
  const float den = fmaf(s2, rs, an);      // |fn| + r
  const float tf = fd * bg_rcp(den);
  const float c2 = 0.5f * den * rs;        // cos^2 in [1/2, 1]
  const float cf = c2 * bg_rsqrt(c2);
  t = (double)copysignf(tf, fn);
  const double w = fma(t, t, 1.0), y = (double)cf;
  const double e = fma(-w, y * y, 1.0);
  c = fma(y * e, fma(0.375, e, 0.5), y);
}

namespace cg = cooperative_groups;

constexpr int GRID_NT = 256;
constexpr int GRID_MAX_CHAINS = 16;

struct GridLayout {  // per-chain layout of the grid kernel's workspace (bytes)
  size_t w, nrm, sig, perm, meta, total;
};

__host__ __device__ inline GridLayout grid_layout(int lmax, int kmax, size_t es) {
  GridLayout g;
  g.w = 0;
  g.nrm = ((size_t)lmax * kmax * es + 255) & ~(size_t)255;
  g.sig = g.nrm + (((size_t)kmax * 8 + 255) & ~(size_t)255);
  g.perm = g.sig + (((size_t)kmax * 8 + 255) & ~(size_t)255);
  g.meta = g.perm + (((size_t)kmax * 4 + 255) & ~(size_t)255);
  g.total = g.meta + 256;
  return g;
}

// Transposed warp reduction of NV (power of two, <= 32) values per lane: after
// it lane L holds in p[0] the warp total of value grid_treduce_index<NV>(L).
template <int NV>
__device__ __forceinline__ void grid_treduce(double (&p)[NV], int lane) {
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
#pragma unroll
  for (; m >= 1; m >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], m);
}
template <int NV>
__device__ __forceinline__ int grid_treduce_index(int lane) {
  int idx = 0, m = 16;
#pragma unroll
  for (int h = NV / 2; h >= 1; h /= 2) {
    if (lane & m) idx += h;
    m >>= 1;
  }
  return idx;
}

// per-chain meta block: [0] f2 (double) | [8] bad (int) | [12] rank | [16] flag0 | [20] flag1 | [24] sweeps | [28] full
struct GridMeta {
  double f2;
  int bad, rank, flag[2], sweeps, full;
  unsigned c2bits[3];  // largest rotated cos^2 of sweep s in slot s % 3 (float bits, atomicMax)
  unsigned tc2bits[3]; // largest (t cos)^2 of the sweep's rotations, same slots (kernels that track it)
};

// Stop rule of the grid kernels.  A sweep whose rotations all had cos^2 <= tol^2
// rotated nothing: converged.  The early stop (largest rotated cos^2 <= big2, see
// early_stop2) assumes quadratic convergence; it is taken only when the sweep's
// largest cos^2 is also <= 1e4 x (previous sweep's)^2, i.e. when the decay was
// quadratic: cos_next <= 100 cos^2.  Measured on the C4 splits (1024 columns,
// TTG_BG_DEBUG): cos^2 per sweep ... 8.9e-6, 7.0e-10, 9.5e-17, 0, i.e. cos_next =
// 3 .. 20 cos^2, and a factor of 100 on cos^2 (10 on the cosine) sent most splits
// into an all-skipped check sweep.  Clustered singular values converge linearly
// (cos^2_next ~ rho cos^2, ratio to the square >> 1e4 at this level) and keep
// sweeping until a sweep rotates nothing above the threshold.
__device__ __forceinline__ bool grid_converged(const GridMeta* mt, int sweep, double tol2, double big2,
                                               double tol_rot = 0.0, bool guarded = false) {
  const double c2 = (double)__uint_as_float(mt->c2bits[sweep % 3]);
  const double prev = sweep > 0 ? (double)__uint_as_float(mt->c2bits[(sweep + 2) % 3]) : 1.0;
  // Early stop only for kernels that track (t cos)^2 (guarded): small rotation angles are what
  // near-degenerate singular values violate (see sweep_stop in jacobi_svd.cu); the others always end
  // with a sweep that rotates nothing.
  if (c2 <= tol2) return true;
  if (!guarded) return false;
  const double tc2 = (double)__uint_as_float(mt->tc2bits[sweep % 3]);
  return c2 <= big2 && c2 <= 1.0e4 * prev * prev && tc2 <= 0.01 * tol_rot * tol_rot;
}

// Epilogue of the grid Jacobi kernels: exact column norms, descending order, truncation
// rank + dropped weight (schmidt.hpp:40-59), singular values and isometry.
template <typename T, typename Skip>
__device__ void grid_epilogue(const SvdParams& p, cg::grid_group& grid, unsigned char* work, size_t chain_bytes,
                              const GridLayout& lay, int chains, Skip skip) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int NT = blockDim.x;
  const int gthreads = gridDim.x * NT, gtid = blockIdx.x * NT + tid;
  const int gwarp = gtid >> 5, gwarps = gthreads >> 5;
  auto chain_base = [&](int c) { return work + chain_bytes * c; };
  auto W_of = [&](int c) { return reinterpret_cast<T*>(chain_base(c) + lay.w); };
  auto sig_of = [&](int c) { return reinterpret_cast<double*>(chain_base(c) + lay.sig); };
  auto perm_of = [&](int c) { return reinterpret_cast<int*>(chain_base(c) + lay.perm); };
  auto meta_of = [&](int c) { return reinterpret_cast<GridMeta*>(chain_base(c) + lay.meta); };
  auto dims = [&](int c, int& m, int& n, int& l, int& k) {
    m = p.M.eval(p.bonds, c, p.ld);
    n = p.N.eval(p.bonds, c, p.ld);
    l = p.mode == 0 ? m : n;
    k = p.mode == 0 ? n : m;
  };
  // ---- epilogue: exact norms, order, rank, outputs
  for (int c = 0; c < chains; ++c) {
    if (skip(c)) continue;
    int m, n, l, k;
    dims(c, m, n, l, k);
    const T* W = W_of(c);
    double* sig = sig_of(c);
    for (int col = gwarp; col < k; col += gwarps) {
      double acc = 0.0;
      for (int i = lane; i < l; i += 32) acc += abs2(W[(size_t)col * l + i]);
      acc = warp_sum(acc);
      if (lane == 0) sig[col] = sqrt(acc);
    }
  }
  grid.sync();
  for (int c = 0; c < chains; ++c) {
    if (skip(c)) continue;
    int m, n, l, k;
    dims(c, m, n, l, k);
    const double* sig = sig_of(c);
    int* perm = perm_of(c);
    for (int col = gtid; col < k; col += gthreads) {
      const double v = sig[col];
      int pos = 0;
      for (int c2 = 0; c2 < k; ++c2) {
        const double u = sig[c2];
        pos += (u > v) || (u == v && c2 < col);
      }
      perm[pos] = col;
    }
  }
  grid.sync();
  for (int c = blockIdx.x; c < chains; c += gridDim.x) {
    if (skip(c) || tid != 0) continue;
    int m, n, l, k;
    dims(c, m, n, l, k);
    const int kmin = min(m, n);
    const double* sig = sig_of(c);
    const int* perm = perm_of(c);
    GridMeta* mt = meta_of(c);
    ChainState* st = p.st ? p.st + c : nullptr;
    int r = 1;
    if (!mt->bad && kmin > 0) {
      r = 0;
      const double cutoff = p.tol * sig[perm[0]];
      while (r < kmin && sig[perm[r]] > cutoff) ++r;
      if (r < 1) r = 1;
      if (p.max_bond > 0 && r > p.max_bond) r = (int)p.max_bond;
      double drop = 0.0;
      for (int j = r; j < kmin; ++j) drop += sig[perm[j]] * sig[perm[j]];
      if (st && p.accumulate_err && !will_retry(p, mt->flag[0] == 2)) st->err2 += drop;
    }
    const double negligible = (double)l * l * DBL_EPSILON * DBL_EPSILON * mt->f2;
    mt->rank = r;
    mt->full = (m == n && !mt->bad && sig[perm[k - 1]] * sig[perm[k - 1]] > negligible) ? 1 : 0;
    p.bonds[c * p.ld + p.out_idx] = r;
    if (p.frame_out) p.frame_out[c * p.frame_ld] = (p.frame && mt->full) ? m : 0;
    if (p.sweeps_out) p.sweeps_out[c] = mt->sweeps;
    finish_status(p, st, mt->bad, mt->flag[0] == 2);
    if (p.svals)
      for (int j = 0; j < kmin; ++j) p.svals[p.s_svals * c + j] = sig[perm[j]];
  }
  grid.sync();
  for (int c = 0; c < chains; ++c) {
    if (skip(c)) continue;
    int m, n, l, k;
    dims(c, m, n, l, k);
    const T* W = W_of(c);
    const double* sig = sig_of(c);
    const int* perm = perm_of(c);
    const GridMeta* mt = meta_of(c);
    const int r = mt->rank;
    T* iso = static_cast<T*>(p.iso) + p.s_iso * c;
    const long long tot = p.mode == 0 ? (long long)m * r : (long long)r * n;
    for (long long idx = gtid; idx < tot; idx += gthreads) {
      int i, j;
      if (p.mode == 0) {
        i = (int)(idx / r);
        j = (int)(idx - (long long)i * r);
      } else {
        j = (int)(idx / n);
        i = (int)(idx - (long long)j * n);
      }
      const double sv = sig[perm[j]];
      T v;
      if (sv > 0.0) {
        v = scale(W[(size_t)perm[j] * l + i], 1.0 / sv);
        if (p.mode == 1) v = conj_(v);
      } else {
        v = (i == j) ? Scalar<T>::one() : Scalar<T>::zero();
      }
      iso[idx] = v;
    }
    if (p.frame && mt->full) {
      T* fr = static_cast<T*>(p.frame) + p.s_frame * c;
      for (long long idx = gtid; idx < (long long)l * k; idx += gthreads) {
        const int i = (int)(idx / k), j = (int)(idx - (long long)(idx / k) * k);
        fr[idx] = scale(W[(size_t)perm[j] * l + i], 1.0 / sig[perm[j]]);
      }
    }
  }
}

}  // namespace
}  // namespace ttg
