// Host side of the ttgpu C ABI: device MPS/MPO containers and the sweep
// engine that drives the sm_100a kernels.
//
// The engine restates, for a batch of independent chains with one shared
// shape, the reference's
//   CanonicalMPS(const MPS&, center, Strategy)      mps.hpp:188-218
//   CompressionEngine + variational_compress         simplify.hpp:15-131
//   simplify(MPS, Strategy, guess)                  simplify.hpp:182-195
// Every truncation rank is produced on the device and written into a per-chain
// bond table that the following kernels read, so the host never waits inside a
// call: a whole simplify is one stream-ordered sequence of launches, with one
// host read of the per-chain "active" flags per sweep (early stop) and one at
// the end.
#include <algorithm>
#include <cstddef>
#include <memory>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the library is bound with dlopen (ttg_comm_*)

#include "../../include/ttgpu.h"
#include "common.cuh"
#include "gemm.cuh"
#include "jacobi_svd.cuh"
#include "kernels.cuh"
#include "qr.cuh"

using namespace ttg;

// Per-kernel-class profile (enabled by ttg_profile_enable): CUDA events around
// every launch of the engine on the context stream, plus the executed flops of
// each GEMM / SVD evaluated from the device bond table (which costs a host sync
// per launch, so profiled runs are separate from timed runs).
struct ProfileRec {
  int cls;
  cudaEvent_t e0, e1;
  double flops;
};

struct ttg_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  int profile = 0;
  std::vector<ProfileRec> pending;
  int64_t prof_count[TTG_PROF_CLASSES] = {};
  double prof_ms[TTG_PROF_CLASSES] = {};
  double prof_flops[TTG_PROF_CLASSES] = {};
  int64_t prof_svd_sweeps = 0;
  int* d_sweeps = nullptr;  // device counter target for the SVD kernel (profiling)
  // pinned double buffer of the TTLAB1 file I/O (allocated on first use)
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // NCCL communicator of the batched configs (one rank per GPU), see ttg_comm_init
  void* comm = nullptr;
  int comm_rank = 0, comm_size = 1;
  void flush_profile() {
    if (pending.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& r : pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.e0, r.e1);
      prof_count[r.cls] += 1;
      prof_ms[r.cls] += ms;
      prof_flops[r.cls] += r.flops;
      cudaEventDestroy(r.e0);
      cudaEventDestroy(r.e1);
    }
    pending.clear();
  }
};

// RAII: brackets one launch with events when profiling.
struct ProfScope {
  ttg_ctx* ctx;
  ProfileRec rec{};
  ProfScope(ttg_ctx* c, int cls, double flops = 0.0) : ctx(c) {
    if (!ctx->profile) return;
    rec.cls = cls;
    rec.flops = flops;
    cudaEventCreate(&rec.e0);
    cudaEventCreate(&rec.e1);
    cudaEventRecord(rec.e0, ctx->stream);
  }
  ~ProfScope() {
    if (!ctx->profile) return;
    cudaEventRecord(rec.e1, ctx->stream);
    ctx->pending.push_back(rec);
  }
};

struct ttg_dmps {
  int n = 0, dtype = TTG_F64, count = 1;
  std::vector<int> phys;          // n
  std::vector<int> bonds;         // count * (n + 1), host mirror
  std::vector<long long> cap;     // elements per chain per site
  std::vector<void*> site;        // n device buffers of count * cap[k] elements
  std::vector<double> error;      // per chain
  int center = -1;
  cudaStream_t stream = nullptr;  // allocation stream
  ~ttg_dmps() {
    for (void* p : site)
      if (p) cudaFreeAsync(p, stream);
  }
  int bond(int chain, int k) const { return bonds[(size_t)chain * (n + 1) + k]; }
  bool uniform() const {
    for (int c = 1; c < count; ++c)
      for (int k = 0; k <= n; ++k)
        if (bond(c, k) != bond(0, k)) return false;
    return true;
  }
};

struct ttg_dmpo {
  int n = 0, dtype = TTG_F64;
  std::vector<int> bonds, dout, din;
  std::vector<void*> site;
  cudaStream_t stream = nullptr;
  ~ttg_dmpo() {
    for (void* p : site)
      if (p) cudaFreeAsync(p, stream);
  }
};

namespace {

struct Error {
  ttg_status st;
  std::string msg;
};

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) throw Error{TTG_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

size_t esize(int dtype) { return dtype == TTG_C128 ? 16 : 8; }

// Stream-ordered device allocation (the default pool keeps freed blocks, so
// repeated calls do not reach cudaMalloc).
// debug (TTG_WATCH_ADDR=0x..., TTG_WATCH_BYTES=n): checksum of a device range, printed with the split / GEMM traces
inline void debug_watch(const char* where) {
  static const unsigned long long addr = getenv("TTG_WATCH_ADDR") ? strtoull(getenv("TTG_WATCH_ADDR"), nullptr, 16) : 0ull;
  static const size_t nb = getenv("TTG_WATCH_BYTES") ? (size_t)atoll(getenv("TTG_WATCH_BYTES")) : 0;
  if (!addr || !nb) return;
  std::vector<double> h(nb / 8);
  cudaDeviceSynchronize();
  if (cudaMemcpy(h.data(), reinterpret_cast<const void*>(addr), nb, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();  // range not allocated (yet): nothing to report, no error left behind
    return;
  }
  double a = 0.0;
  for (double x : h) a += x * x;
  fprintf(stderr, "    watch %s: %.15e\n", where, std::sqrt(a));
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error{TTG_CAPACITY, "device allocation of " + std::to_string(bytes) + " bytes failed"};
    }
    // TTG_POISON=1 (debug): every workspace starts as NaN bit patterns, so a read of memory the call did
    // not write shows up at once instead of depending on what the pool block held before
    static const bool poison = getenv("TTG_POISON") != nullptr;
    if (poison) cudaMemsetAsync(p, 0xFF, bytes, st);
    static const bool dbg_alloc = getenv("TTG_DEBUG_SPLITS") != nullptr;
    if (dbg_alloc) fprintf(stderr, "  alloc DevBuf %p .. %p (%zu bytes)\n", p, static_cast<char*>(p) + bytes, bytes);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(s, o.s);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

void* dev_alloc(size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{TTG_CAPACITY, "device allocation of " + std::to_string(bytes) + " bytes failed"};
  }
  static const bool poison = getenv("TTG_POISON") != nullptr;  // debug: see DevBuf
  if (poison) cudaMemsetAsync(p, 0xFF, bytes, s);
  static const bool dbg_alloc = getenv("TTG_DEBUG_SPLITS") != nullptr;
  if (dbg_alloc) fprintf(stderr, "  alloc dev %p .. %p (%zu bytes)\n", p, static_cast<char*>(p) + bytes, bytes);
  return p;
}

ttg_dmps* new_dmps(int n, int dtype, int count, const std::vector<int>& phys, const std::vector<long long>& cap,
                   cudaStream_t s) {
  auto* m = new ttg_dmps();
  m->n = n;
  m->dtype = dtype;
  m->count = count;
  m->phys = phys;
  m->cap = cap;
  m->stream = s;
  m->bonds.assign((size_t)count * (n + 1), 1);
  m->error.assign(count, 0.0);
  m->site.assign(n, nullptr);
  try {
    for (int k = 0; k < n; ++k) m->site[k] = dev_alloc((size_t)count * cap[k] * esize(dtype), s);
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

inline int clamp_bond(int64_t mb) {
  if (mb <= 0 || mb >= std::numeric_limits<int>::max()) return std::numeric_limits<int>::max();
  return (int)mb;
}

inline double fp_error_floor(double scale) { return 32.0 * std::numeric_limits<double>::epsilon() * scale; }

// ---------------------------------------------------------------------------
// sweep engine
// ---------------------------------------------------------------------------

template <typename T>
struct Engine {
  ttg_ctx* ctx;
  cudaStream_t st;
  int L, B;
  std::vector<int> d, t, g, q, pb, bound;
  int* d_bonds = nullptr;  // B x (L+1) psi bonds
  void* svd_grid_work = nullptr;  // workspace of the grid-cooperative SVD (few large splits)
  // QR-preconditioned split (Q1, R1^H, L, U_L per chain, `pre_cap` elements each)
  void* pre_buf = nullptr;
  long long pre_cap = 0;
  int pre_slot = 0;
  int ld = 0;
  ChainState* d_state = nullptr;
  double* svals = nullptr;  // sorted singular values of the last split (isometry completion)
  long long svals_cap = 0;

  Engine(ttg_ctx* c, int L_, int B_) : ctx(c), st(c->stream), L(L_), B(B_) {}

  int ub(DimExpr e) const { return e.idx < 0 ? e.mult : e.mult * bound[e.idx]; }

  // Host mirror of the single chain's bond table (host_dims): refreshed once per sweep step (the sync the
  // large split needs anyway), so the step's projection GEMMs X = L T, Y = X T, theta = Y R^T get host
  // shapes and run on the tensor-map TMA kernel.  Entries written on the device since the last refresh
  // are marked invalid and keep their device-side DimExpr.
  bool host_dims = false;
  std::vector<int> hostb;
  std::vector<char> hostb_ok;
  void refresh_bonds() {
    if (!host_dims) return;
    hostb.resize(ld);
    CK(cudaMemcpyAsync(hostb.data(), d_bonds, ld * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    hostb_ok.assign(ld, 1);
  }
  void invalidate_bond(int idx) {
    if (host_dims && idx >= 0 && idx < (int)hostb_ok.size()) hostb_ok[idx] = 0;
  }
  DimExpr resolve(DimExpr e) const {
    if (host_dims && e.idx >= 0 && e.idx < (int)hostb_ok.size() && hostb_ok[e.idx]) return dconst(e.mult * hostb[e.idx]);
    return e;
  }

  // host copies of the bond table / chain states (profiling only)
  std::vector<int> hb;
  std::vector<ChainState> hs;
  bool live_dims(bool check_active) {
    if (!ctx->profile) return false;
    CK(cudaStreamSynchronize(st));
    hb.resize((size_t)B * ld);
    CK(cudaMemcpy(hb.data(), d_bonds, hb.size() * sizeof(int), cudaMemcpyDeviceToHost));
    hs.resize(B);
    if (check_active && d_state) CK(cudaMemcpy(hs.data(), d_state, B * sizeof(ChainState), cudaMemcpyDeviceToHost));
    return true;
  }
  bool chain_on(int c, bool check_active) const { return !(check_active && d_state) || hs[c].active; }

  void G(const void* A, long long sA, const void* Bm, long long sB, void* C, long long sC, DimExpr M, DimExpr N,
         DimExpr K, int opA, int opB, bool check_active, int beta = 0, bool a_upper = false) {
    double flops = 0.0;
    if (live_dims(check_active))
      for (int c = 0; c < B; ++c)
        if (chain_on(c, check_active)) {
          const double m = M.eval(hb.data(), c, ld), kk = K.eval(hb.data(), c, ld);
          // upper triangular / trapezoidal A: row i multiplies k >= i only
          const double mk = a_upper ? (m <= kk ? m * kk - m * (m - 1) / 2.0 : kk * (kk + 1) / 2.0) : m * kk;
          flops += (Scalar<T>::is_complex ? 8.0 : 2.0) * mk * (double)N.eval(hb.data(), c, ld);
        }
    // single chain with a host mirror: the chain is active whenever the sweep loop is running
    GemmParams p{A,      Bm,   C,  sA, sB, sC, resolve(M), resolve(N), resolve(K),
                 d_bonds, ld, (check_active && !host_dims) ? d_state : nullptr, 1.0, beta};
    p.a_upper = a_upper ? 1 : 0;
    ProfScope ps(ctx, TTG_PROF_GEMM, flops);
    CK(gemm<T>(p, opA, opB, ub(p.M), ub(p.N), B, st, ub(p.K)));
    ++ctx->launches;
    static const bool dbg_gemm = getenv("TTG_DEBUG_SPLITS") != nullptr;  // debug: live shape and |C|_F of chain 0
    if (dbg_gemm) {
      std::vector<int> hbd(ld);
      cudaStreamSynchronize(st);
      cudaMemcpy(hbd.data(), d_bonds, ld * sizeof(int), cudaMemcpyDeviceToHost);
      const int m = M.eval(hbd.data(), 0, ld), n = N.eval(hbd.data(), 0, ld), k = K.eval(hbd.data(), 0, ld);
      std::vector<T> hc((size_t)m * n);
      cudaMemcpy(hc.data(), C, hc.size() * sizeof(T), cudaMemcpyDeviceToHost);
      double t2 = 0.0;
      for (auto& x : hc) t2 += abs2(x);
      std::vector<T> ha((size_t)m * k), hbm((size_t)k * n);
      cudaMemcpy(ha.data(), A, ha.size() * sizeof(T), cudaMemcpyDeviceToHost);
      cudaMemcpy(hbm.data(), Bm, hbm.size() * sizeof(T), cudaMemcpyDeviceToHost);
      double a2 = 0.0, b2 = 0.0, wa = 0.0, wb = 0.0;
      for (size_t i = 0; i < ha.size(); ++i) {
        a2 += abs2(ha[i]);
        wa += abs2(ha[i]) * (double)(i % 97 + 1);
      }
      for (size_t i = 0; i < hbm.size(); ++i) {
        b2 += abs2(hbm[i]);
        wb += abs2(hbm[i]) * (double)(i % 89 + 1);
      }
      debug_watch("after gemm");
      fprintf(stderr, "  gemm op %d %d live %d x %d x %d (bounds %d %d %d) |C| %.15e |A| %.12e (%.12e) |B| %.12e (%.12e) A %p B %p C %p\n",
              opA, opB, m, n, k, ub(p.M), ub(p.N), ub(p.K), std::sqrt(t2), std::sqrt(a2), wa, std::sqrt(b2), wb, A, Bm, C);
    }
  }

  struct Warm {
    const void* pre = nullptr;
    long long s_pre = 0;
    const int* fin = nullptr;
    int* fout = nullptr;
    int fld = 0;
    void* frame = nullptr;
    long long s_frame = 0;
  };

  void split_large(const void* theta, long long s_theta, DimExpr M, DimExpr N, int out_idx, void* iso,
                   long long s_iso, int mode, double tol, int max_bond, bool check_active, bool accumulate,
                   void* work, long long s_work);

  void split_preconditioned(const void* theta, long long s_theta, DimExpr M, DimExpr N, int out_idx, void* iso,
                            long long s_iso, int mode, double tol, int max_bond, bool check_active, bool accumulate,
                            void* work, long long s_work);

  void S(const void* theta, long long s_theta, DimExpr M, DimExpr N, int out_idx, void* iso, long long s_iso,
         int mode, double tol, int max_bond, bool check_active, bool accumulate, void* work, long long s_work,
         const Warm& w = Warm(), bool no_pre = false) {
    const DimExpr M_dev = M, N_dev = N;  // the split kernels read their shapes from the device table
    (void)M_dev;
    (void)N_dev;
    struct Inval {  // the rank is written on the device: the host mirror of this bond is stale afterwards
      Engine* e;
      int idx;
      ~Inval() {
        e->invalidate_bond(idx);
        e->invalidate_bond(e->pre_slot);
      }
    } inval{this, out_idx};
    // TTG_DEBUG_SPLITS=1: one line per split on stderr (bounds, live shape, resulting rank of chain 0)
    static const bool dbg_splits = getenv("TTG_DEBUG_SPLITS") != nullptr;
    struct DbgSplit {
      Engine* e;
      DimExpr M, N;
      int idx, mode, pre;
      bool on;
      int m = 0, n = 0;
      void live(int& a, int& b, int& r) {
        std::vector<int> hb(e->ld);
        cudaStreamSynchronize(e->st);
        cudaMemcpy(hb.data(), e->d_bonds, e->ld * sizeof(int), cudaMemcpyDeviceToHost);
        a = M.eval(hb.data(), 0, e->ld);
        b = N.eval(hb.data(), 0, e->ld);
        r = hb[idx];
      }
      DbgSplit(Engine* e_, DimExpr M_, DimExpr N_, int idx_, int mode_, int pre_, bool on_)
          : e(e_), M(M_), N(N_), idx(idx_), mode(mode_), pre(pre_), on(on_) {
        int r;
        if (on) live(m, n, r);
      }
      const void* theta = nullptr;
      const void* iso = nullptr;
      ~DbgSplit() {
        if (!on) return;
        int a, b, r;
        live(a, b, r);
        // |theta|_F and the orthonormality defect of the isometry (chain 0), computed on the host
        double tn = 0.0, defect = 0.0;
        {
          std::vector<T> th((size_t)m * n), is((size_t)(mode == 0 ? m : n) * r);
          cudaMemcpy(th.data(), theta, th.size() * sizeof(T), cudaMemcpyDeviceToHost);
          cudaMemcpy(is.data(), iso, is.size() * sizeof(T), cudaMemcpyDeviceToHost);
          for (auto& x : th) tn += abs2(x);
          const int len = mode == 0 ? m : n;  // mode 0: iso is len x r (columns); mode 1: r x len (rows)
          for (int p = 0; p < r; ++p)
            for (int q = 0; q < r; ++q) {
              double gr = 0.0, gi = 0.0;
              for (int i = 0; i < len; ++i) {
                const T u = mode == 0 ? is[(size_t)i * r + p] : is[(size_t)p * len + i];
                const T v = mode == 0 ? is[(size_t)i * r + q] : is[(size_t)q * len + i];
                if constexpr (Scalar<T>::is_complex) {
                  gr += u.x * v.x + u.y * v.y;
                  gi += u.x * v.y - u.y * v.x;
                } else {
                  gr += u * v;
                }
              }
              defect = std::max(defect, std::hypot(gr - (p == q ? 1.0 : 0.0), gi));
            }
          // weight of theta outside the span of the isometry: |theta|^2 - |U^H theta|^2 (mode 0) or - |theta V|^2
          double kept = 0.0;
          for (int p = 0; p < r; ++p)
            for (int j = 0; j < (mode == 0 ? n : m); ++j) {
              double gr = 0.0, gi = 0.0;
              for (int i = 0; i < len; ++i) {
                const T u = mode == 0 ? is[(size_t)i * r + p] : is[(size_t)p * len + i];
                const T x = mode == 0 ? th[(size_t)i * n + j] : th[(size_t)j * n + i];
                if constexpr (Scalar<T>::is_complex) {
                  // mode 0: conj(u) x; mode 1: x conj(v^H row) = x * conj(u)
                  gr += u.x * x.x + u.y * x.y;
                  gi += u.x * x.y - u.y * x.x;
                } else {
                  gr += u * x;
                }
              }
              kept += gr * gr + gi * gi;
            }
          fprintf(stderr, "   outside weight %.6e of |theta|^2 %.6e\n", tn - kept, tn);
        }
        debug_watch("after split");
        fprintf(stderr, "split mode %d no_pre %d bounds %d x %d live %d x %d -> bond[%d] = %d  |theta| %.15e iso defect %.2e\n",
                mode, pre, e->ub(M), e->ub(N), m, n, idx, r, std::sqrt(tn), defect);
      }
    } dbg_split(this, M, N, out_idx, mode, no_pre ? 1 : 0, dbg_splits);
    dbg_split.theta = theta;
    dbg_split.iso = iso;
    SvdParams p{};
    static const int no_early = [] {
      const char* e = getenv("TTG_SVD_EARLY");
      return (e && e[0] == '0') ? 1 : (e && e[0] == '2') ? 2 : 0;
    }();
    p.no_early = no_early;
    p.theta_pre = w.pre;
    p.s_pre = w.s_pre;
    p.frame_in = w.fin;
    p.frame_out = w.fout;
    p.frame_ld = w.fld;
    p.frame = w.frame;
    p.s_frame = w.s_frame;
    p.theta = theta;
    p.s_theta = s_theta;
    p.M = M;
    p.N = N;
    p.bonds = d_bonds;
    p.ld = ld;
    p.out_idx = out_idx;
    p.iso = iso;
    p.s_iso = s_iso;
    p.svals = nullptr;
    p.s_svals = 0;
    p.st = d_state;
    p.check_active = check_active ? 1 : 0;
    p.accumulate_err = accumulate ? 1 : 0;
    p.tol = tol;
    p.max_bond = max_bond == std::numeric_limits<int>::max() ? 0 : max_bond;
    p.mode = mode;
    p.work = work;
    p.s_work = s_work;
    const int mu = ub(M), nu = ub(N);
    static const bool pre_ok = [] {
      const char* e = getenv("TTG_SVD_PRECOND");
      return !(e && e[0] == '0');
    }();
    const bool grid_path = svd_grid_work && jacobi_grid_eligible(mode == 0 ? mu : nu, mode == 0 ? nu : mu, B, sizeof(T));
    if (!no_pre && pre_ok && B == 1 && w.pre == nullptr && std::min(mu, nu) >= 24 &&
        (std::max(mu, nu) > 160 || (size_t)(std::max(mu, nu) | 1) * std::max(mu, nu) * sizeof(T) > QR_R_SMEM_LIMIT)) {
      split_large(theta, s_theta, M, N, out_idx, iso, s_iso, mode, tol, max_bond, check_active, accumulate, work,
                  s_work);
      return;
    }
    // splits within 32 x 32: the two preconditioning QRs cost more than the
    // Jacobi sweeps they save (tools/split_probe.py, C1)
    static const int pre_skip = [] {
      const char* e = getenv("TTG_PRE_SKIP");
      return e ? atoi(e) : 32;
    }();
    if (!no_pre && pre_ok && pre_buf && !grid_path && w.pre == nullptr && std::min(mu, nu) >= 24 &&
        std::max(mu, nu) > pre_skip &&
        (size_t)(std::max(mu, nu) | 1) * std::max(mu, nu) * sizeof(T) <= QR_R_SMEM_LIMIT && std::min(mu, nu) <= 1024 &&
        (long long)std::max(mu, nu) * std::max(mu, nu) <= pre_cap) {
      split_preconditioned(theta, s_theta, M, N, out_idx, iso, s_iso, mode, tol, max_bond, check_active, accumulate,
                           work, s_work);
      return;
    }
    double flops = 0.0;  // Golub-Van Loan R-SVD count (U, S, V): 4m^2n + 8mn^2 + 9n^3, m >= n
    if (live_dims(check_active))
      for (int c = 0; c < B; ++c)
        if (chain_on(c, check_active)) {
          double a = M.eval(hb.data(), c, ld), b = N.eval(hb.data(), c, ld);
          if (a < b) std::swap(a, b);
          flops += (Scalar<T>::is_complex ? 4.0 : 1.0) * (4 * a * a * b + 8 * a * b * b + 9 * b * b * b);
        }
    const int m = ub(M), n = ub(N);
    const int l = mode == 0 ? m : n, k = mode == 0 ? n : m;
    if (ctx->profile) {
      if (!ctx->d_sweeps) CK(cudaMalloc(&ctx->d_sweeps, 4096 * sizeof(int)));
      CK(cudaMemsetAsync(ctx->d_sweeps, 0, B * sizeof(int), st));
      p.sweeps_out = B <= 4096 ? ctx->d_sweeps : nullptr;
    }
    // kept near-zero singular values (sigma <= 100 l eps |theta|_F <= 100 l sqrt(k) eps sigma_0, see
    // iso_complete) are possible only when tol < 100 l sqrt(k) eps: then the isometry is checked and
    // completed after the sweeps
    const bool complete = svals && std::min(l, k) <= svals_cap && tol < 100.0 * l * std::sqrt((double)k) * 2.3e-16 &&
                          iso_complete_smem(l, std::min(l, k), sizeof(T)) <= 200 * 1024;
    if (complete) {
      p.svals = svals;
      p.s_svals = svals_cap;
    }
    // retry policy (schmidt.hpp:23-35): a split that does not converge is jittered in place and
    // relaunched once for the flagged chains (two launches that exit at once otherwise)
    static const int force_retry = [] {
      const char* e = getenv("TTG_SVD_FORCE_RETRY");  // test hook: sweeps allowed in the first attempt
      return e ? atoi(e) : 0;
    }();
    p.retry = 1;
    p.first_budget = force_retry;
    {
      ProfScope ps(ctx, TTG_PROF_SVD, flops);
      static const bool grid_ok = [] {
        const char* e = getenv("TTG_SVD_GRID");
        return !(e && e[0] == '0');
      }();
      const bool grid = grid_ok && svd_grid_work && jacobi_grid_eligible(l, k, B, sizeof(T));
      for (int attempt = 0; attempt < 2; ++attempt) {
        p.attempt = attempt;
        if (attempt == 1) {
          p.theta_pre = nullptr;
          CK(svd_jitter<T>(const_cast<void*>(theta), s_theta, M, N, d_bonds, ld, d_state, B, st));
          ++ctx->launches;
        }
        if (grid)
          CK(jacobi_svd_grid<T>(p, l, k, B, svd_grid_work, st));
        else
          CK(jacobi_svd<T>(p, l, k, B, st));
        ++ctx->launches;
      }
      if (complete) {
        CK(iso_complete<T>(p, l, std::min(l, k), B, st));
        ++ctx->launches;
      }
    }
    if (ctx->profile && p.sweeps_out) {
      std::vector<int> hsw(B);
      CK(cudaMemcpyAsync(hsw.data(), ctx->d_sweeps, B * sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int c = 0; c < B; ++c) ctx->prof_svd_sweeps += hsw[c];
      static const bool print_sweeps = getenv("TTG_PRINT_SWEEPS") != nullptr;
      if (print_sweeps)
        fprintf(stderr, "svd mode=%d l<=%d k<=%d warm=%d sweeps=%d\n", mode, l, k, w.pre != nullptr ? 1 : 0, hsw[0]);
    }
  }
};

template <typename T>
void Engine<T>::split_preconditioned(const void* theta, long long s_theta, DimExpr M, DimExpr N, int out_idx,
                                     void* iso, long long s_iso, int mode, double tol, int max_bond,
                                     bool check_active, bool accumulate, void* work, long long s_work) {
  // M_ = theta (mode 0) or theta^H (mode 1), l x k.  M_ = Q1 R1, R1 = L Q2 (QR of R1^H);
  // one-sided Jacobi on L's columns gives U_L, and U_M = Q1 U_L is the isometry.
  T* base = static_cast<T*>(pre_buf);
  T* Qb = base;
  T* R1h = base + pre_cap;
  T* Lb = base + 2 * pre_cap;
  T* Ub = base + 3 * pre_cap;
  const long long sp = 4 * pre_cap;
  const DimExpr Lr = mode == 0 ? M : N;  // column length l
  const DimExpr Kc = mode == 0 ? N : M;  // number of columns k
  const DimExpr R0 = dbond(pre_slot);
  const int lu = ub(Lr), ku = ub(Kc);
  // The preconditioner rank r0 <= min(l, k) of THIS split: the inner split below sizes its kernel (panel in
  // shared memory or in the global workspace) from the bound of the rank slot, which otherwise is the largest
  // d * bond of the whole chain.  With that loose bound a 32 x 32 inner split of a chain with one 256-wide
  // bond elsewhere chose the global-workspace kernel although the plan (sized from the outer shapes, which do
  // fit shared memory) had reserved no workspace: its panel overran the 16-byte placeholder into neighbouring
  // allocations (found by tools/fuzz_parity.py: results depended on what the pool had placed there).
  struct BoundGuard {
    std::vector<int>& b;
    int idx, saved;
    BoundGuard(std::vector<int>& b_, int idx_, int v) : b(b_), idx(idx_), saved(b_[idx_]) { b[idx] = std::min(saved, v); }
    ~BoundGuard() { b[idx] = saved; }
  } rank_bound(bound, pre_slot, std::min(lu, ku));
  const ChainState* stp = check_active ? d_state : nullptr;
  double qflops = 0.0;  // QR with Q: 4n^2(m - n/3); R only: 2n^2(m - n/3)
  if (live_dims(check_active))
    for (int c = 0; c < B; ++c)
      if (chain_on(c, check_active)) {
        const double a = std::max(Lr.eval(hb.data(), c, ld), Kc.eval(hb.data(), c, ld));
        const double b = std::min(Lr.eval(hb.data(), c, ld), Kc.eval(hb.data(), c, ld));
        qflops += (Scalar<T>::is_complex ? 4.0 : 1.0) * 6.0 * b * b * (a - b / 3.0);
      }
  // TTG_PRE_SMALL=1: one R-only QR as for the large splits (split_large): mode 0 factors theta^H = Q R
  // and rotates the columns of L = R^H (same left singular vectors as theta), mode 1 factors theta = Q R
  // and rotates R in mode 1 (same right singular vectors); the isometry comes straight out of the Jacobi
  // epilogue, no Q, no second QR, no isometry GEMM.
  // Measured: single chains (C2) 125.1 -> 116.3 ms per call; batches (C5) 1347 -> 1447 ms (21% more
  // Jacobi sweeps, and the batched splits are Jacobi-bound), so batches keep the two-QR form.
  static const int pre_small = [] {
    const char* e = getenv("TTG_PRE_SMALL");
    return e ? atoi(e) : 0;
  }();
  if (pre_small == 1 || (pre_small == 0 && B == 1)) {
    {
      ProfScope ps(ctx, TTG_PROF_QR, qflops / 3.0);
      // mode 0: M_ = theta^H (n x m), output R^H = L (m x r0); mode 1: M_ = theta (m x n), output R (r0 x n)
      CK(qr_precondition<T>(theta, s_theta, M, N, mode == 0 ? 1 : 2, d_bonds, ld, pre_slot, nullptr, 0, Lb, sp,
                            mode == 0 ? ub(N) : ub(M), mode == 0 ? ub(M) : ub(N), stp, B, st));
    }
    ++ctx->launches;
    if (mode == 0)
      S(Lb, sp, M, R0, out_idx, iso, s_iso, 0, tol, max_bond, check_active, accumulate, work, s_work, Warm(), true);
    else
      S(Lb, sp, R0, N, out_idx, iso, s_iso, 1, tol, max_bond, check_active, accumulate, work, s_work, Warm(), true);
    return;
  }
  {
    ProfScope ps(ctx, TTG_PROF_QR, qflops);
    CK(qr_precondition<T>(theta, s_theta, M, N, mode, d_bonds, ld, pre_slot, Qb, sp, R1h, sp, lu, ku, stp, B, st));
    CK(qr_precondition<T>(R1h, sp, Kc, R0, 0, d_bonds, ld, pre_slot, nullptr, 0, Lb, sp, ku, std::min(lu, ku), stp, B,
                          st));
  }
  ctx->launches += 2;
  S(Lb, sp, R0, R0, out_idx, Ub, sp, 0, tol, max_bond, check_active, accumulate, work, s_work, Warm(), true);
  if (mode == 0)
    G(Qb, sp, Ub, sp, iso, s_iso, M, dbond(out_idx), R0, OP_N, OP_N, check_active);
  else
    G(Ub, sp, Qb, sp, iso, s_iso, dbond(out_idx), N, R0, OP_C, OP_C, check_active);
}

// Large split of a single chain: shapes are read back from the device (one sync;
// each such split is milliseconds of work), M_ = theta or theta^H is reduced by
// two blocked Householder QRs (M_ = Q1 R1, R1^H = Q2 R2, so M_ = Q1 R2^H Q2^H)
// and one-sided Jacobi runs on the square R2 (mode 1 orthogonalises the
// columns of R2^H = L).  Isometry: U_M = Q1 U_L.
template <typename T>
void Engine<T>::split_large(const void* theta, long long s_theta, DimExpr M, DimExpr N, int out_idx, void* iso,
                            long long s_iso, int mode, double tol, int max_bond, bool check_active, bool accumulate,
                            void* work, long long s_work) {
  (void)s_theta;
  (void)s_iso;
  std::vector<int> hb(ld);
  ChainState hs{};
  const DimExpr Mr = resolve(M), Nr = resolve(N);
  if (host_dims && Mr.idx < 0 && Nr.idx < 0) {
    // shapes from the host mirror refreshed at the start of the sweep step (the chain is active there)
  } else {
    CK(cudaMemcpyAsync(hb.data(), d_bonds, ld * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (check_active) CK(cudaMemcpyAsync(&hs, d_state, sizeof(ChainState), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (check_active && !hs.active) return;
  }
  const int m = Mr.idx < 0 && host_dims ? Mr.mult : M.eval(hb.data(), 0, ld);
  const int n = Nr.idx < 0 && host_dims ? Nr.mult : N.eval(hb.data(), 0, ld);
  const int l = mode == 0 ? m : n, k = mode == 0 ? n : m, r0 = std::min(l, k);
  const size_t es = sizeof(T);
  // TTG_PRE=2: the two-QR preconditioner below.  Default: one R-only QR (C4 A/B on one B200:
  // 3029 -> 2715 ms per call with the CTA-pair grid kernel; the Jacobi needs ~13% more sweeps
  // on L = R^H than on R2^H, the second QR with its explicit Q costs more than that)
  static const int single = [] {
    const char* e = getenv("TTG_PRE");
    return e ? atoi(e) != 2 : 1;
  }();
  if (single) {
    // One R-only QR: mode 0: theta^H = Q R, theta = R^H Q^H, so the left singular vectors of
    // theta are those of L = R^H (m x r0): Jacobi mode 0 on L writes U_r straight into iso.
    // mode 1: theta = Q R, the right singular vectors of theta are those of R (r0 x n): Jacobi
    // mode 1 on R writes V_r^H straight into iso.  No Q, no isometry GEMM.
    const int rr = std::min(m, n);
    DevBuf Mb((size_t)m * n * es, st), R((size_t)rr * std::max(m, n) * es, st), Lb((size_t)rr * std::max(m, n) * es, st);
    const int qr_rows = mode == 0 ? n : m, qr_cols = mode == 0 ? m : n;
    if (mode == 0)
      CK(conj_transpose<T>(theta, 0, m, n, Mb.p, 0, 1, st));
    else
      CK(cudaMemcpyAsync(Mb.p, theta, (size_t)m * n * es, cudaMemcpyDeviceToDevice, st));
    ++ctx->launches;
    {
      size_t a, v, t2, w2, pp;
      qr_blocked_elems<T>(qr_rows, qr_cols, &a, &v, &t2, &w2, &pp);
      DevBuf wa(a * es, st), wv(v * es, st), wt(t2 * es, st), w1b(w2 * es, st), w2b(w2 * es, st), wp(pp * es, st);
      QrParams qp{Mb.p, 0, nullptr, 0, R.p, 0, nullptr, 0, qr_rows, qr_cols};
      QrBlockedWork qw{wa.p, wv.p, wt.p, w1b.p, w2b.p, wp.p, 0, 0, 0, 0, 0};
      // R-only QR of a matrix with few rows: the outer WY factor (S product + t_combine per 128 columns)
      // costs more than the rank-128 updates save (C4 A/B: 1024 x 1024 splits 50 ms per call faster with
      // rank-32 updates, 4096 x 1024 truncating-pass splits another 7 ms).  TTG_QR_PRE2L: two-level from this many rows on.
      static const int pre2l = [] {
        const char* e = getenv("TTG_QR_PRE2L");
        return e ? atoi(e) : (1 << 30);
      }();
      qw.two_level = qr_rows >= pre2l ? -1 : 0;
      long long nl = 0;
      const double big = std::max(qr_rows, qr_cols), sm = std::min(qr_rows, qr_cols);
      ProfScope ps(ctx, TTG_PROF_QR, (Scalar<T>::is_complex ? 4.0 : 1.0) * 2.0 * sm * sm * (big - sm / 3.0));
      CK(householder_qr_blocked<T>(qp, qw, 1, st, &nl));
      ctx->launches += nl;
    }
    if (mode == 0) {  // L = R^H (m x rr)
      CK(conj_transpose<T>(R.p, 0, rr, m, Lb.p, 0, 1, st));
      ++ctx->launches;
      S(Lb.p, 0, dconst(m), dconst(rr), out_idx, iso, 0, 0, tol, max_bond, check_active, accumulate, work, s_work,
        Warm(), true);
    } else {
      S(R.p, 0, dconst(rr), dconst(n), out_idx, iso, 0, 1, tol, max_bond, check_active, accumulate, work, s_work,
        Warm(), true);
    }
    return;
  }
  DevBuf Mb((size_t)l * k * es, st), Q1((size_t)l * r0 * es, st), R1((size_t)r0 * k * es, st),
      R1h((size_t)k * r0 * es, st), R2((size_t)r0 * r0 * es, st), Ut((size_t)r0 * r0 * es, st);
  if (mode == 0)
    CK(cudaMemcpyAsync(Mb.p, theta, (size_t)m * n * es, cudaMemcpyDeviceToDevice, st));
  else
    CK(conj_transpose<T>(theta, 0, m, n, Mb.p, 0, 1, st));
  ++ctx->launches;
  auto blocked = [&](void* A, int rows, int cols, void* Q, void* R) {
    size_t a, v, t2, w2, pp;
    qr_blocked_elems<T>(rows, cols, &a, &v, &t2, &w2, &pp);
    DevBuf wa(a * es, st), wv(v * es, st), wt(t2 * es, st), w1b(w2 * es, st), w2b(w2 * es, st), wp(pp * es, st);
    QrParams qp{A, 0, Q, 0, R, 0, nullptr, 0, rows, cols};
    const QrBlockedWork qw{wa.p, wv.p, wt.p, w1b.p, w2b.p, wp.p, 0, 0, 0, 0, 0};
    long long nl = 0;
    const double big = std::max(rows, cols), sm = std::min(rows, cols);
    ProfScope ps(ctx, TTG_PROF_QR, (Scalar<T>::is_complex ? 4.0 : 1.0) * (Q ? 4.0 : 2.0) * sm * sm * (big - sm / 3.0));
    CK(householder_qr_blocked<T>(qp, qw, 1, st, &nl));
    ctx->launches += nl;
  };
  blocked(Mb.p, l, k, Q1.p, R1.p);
  CK(conj_transpose<T>(R1.p, 0, r0, k, R1h.p, 0, 1, st));
  ++ctx->launches;
  blocked(R1h.p, k, r0, nullptr, R2.p);
  // Jacobi (mode 1) on R2: iso_tmp = U_L^H (r x r0), rank -> bonds[out_idx]
  S(R2.p, 0, dconst(r0), dconst(r0), out_idx, Ut.p, 0, 1, tol, max_bond, check_active, accumulate, work, s_work, Warm(),
    true);
  if (mode == 0)  // psi_n = Q1 U_L = Q1 (U_L^H)^H  (m x r)
    G(Q1.p, 0, Ut.p, 0, iso, 0, dconst(m), dbond(out_idx), dconst(r0), OP_N, OP_C, check_active);
  else  // psi_{n+1} = (Q1 U_L)^H = U_L^H Q1^H  (r x n)
    G(Ut.p, 0, Q1.p, 0, iso, 0, dbond(out_idx), dconst(n), dconst(r0), OP_N, OP_C, check_active);
}

// Host-side bookkeeping shared by simplify / canonicalize.
struct Plan {
  std::vector<long long> psi_cap;
  long long ccap = 1, rcap = 1, bcap = 1, svd_work = 0, qr_work = 0;
  long long qb_A = 0, qb_V = 0, qb_T = 0, qb_W = 0, qb_P = 0;  // blocked-QR workspaces
  long long xz = 1, yw = 1, th = 1;
  std::vector<long long> env_cap;
};

template <typename T>
void run_simplify(ttg_ctx* ctx, const ttg_dmps& target, const ttg_dmps& guess, const ttg_strategy& s,
                  bool variational, int center, ttg_dmps** out, ttg_report* reports) {
  const int L = target.n, B = target.count;
  cudaStream_t st = ctx->stream;
  Engine<T> E(ctx, L, B);
  E.ld = L + 3;  // column L+1: old bond during pass 3; column L+2: preconditioner rank
  E.d = target.phys;
  E.t.assign(target.bonds.begin(), target.bonds.begin() + (L + 1));
  E.g.assign(guess.bonds.begin(), guess.bonds.begin() + (L + 1));
  const int mb = clamp_bond(s.max_bond);
  auto& d = E.d;
  auto& t = E.t;
  auto& g = E.g;
  auto& q = E.q;
  auto& pb = E.pb;
  auto& bound = E.bound;
  q.assign(L + 1, 1);
  for (int k = 0; k + 1 < L; ++k) q[k + 1] = std::min((long long)q[k] * d[k], (long long)g[k + 1]);
  q[L] = 1;
  std::vector<long long> dl(L + 1, 1), dr(L + 1, 1);
  const long long BIG = 1LL << 30;
  for (int k = 1; k <= L; ++k) dl[k] = std::min(BIG, dl[k - 1] * d[k - 1]);
  for (int k = L - 1; k >= 0; --k) dr[k] = std::min(BIG, dr[k + 1] * d[k]);
  pb.assign(L + 3, 1);
  bound.assign(L + 3, 1);
  for (int k = 0; k <= L; ++k) {
    pb[k] = (int)std::max(1LL, std::min({(long long)mb, dl[k], dr[k]}));
    bound[k] = std::max(q[k], pb[k]);
  }
  pb[0] = pb[L] = bound[0] = bound[L] = 1;
  bound[L + 1] = *std::max_element(bound.begin(), bound.end());
  bound[L + 2] = 1;
  for (int k = 0; k < L; ++k) bound[L + 2] = std::max({bound[L + 2], d[k] * bound[k], d[k] * bound[k + 1], q[k]});

  Plan P;
  P.psi_cap.resize(L);
  for (int k = 0; k < L; ++k) P.psi_cap[k] = (long long)bound[k] * d[k] * bound[k + 1];
  for (int k = 0; k < L; ++k) {
    const long long gk1 = g[k + 1];
    P.ccap = std::max(P.ccap, (long long)q[k] * d[k] * std::max<long long>(gk1, bound[k + 1]));
    if (k + 1 < L) {
      P.rcap = std::max(P.rcap, (long long)q[k + 1] * gk1);
      const long long qw = (long long)qr_workspace_elems<T>(q[k] * d[k], (int)gk1);
      if (qw * (long long)sizeof(T) > 200 * 1024) {  // blocked path (panel kernel + DMMA WY updates)
        size_t a, v, t2, w, pp;
        qr_blocked_elems<T>(q[k] * d[k], (int)gk1, &a, &v, &t2, &w, &pp);
        P.qb_A = std::max(P.qb_A, (long long)a);
        P.qb_V = std::max(P.qb_V, (long long)v);
        P.qb_T = std::max(P.qb_T, (long long)t2);
        P.qb_W = std::max(P.qb_W, (long long)w);
        P.qb_P = std::max(P.qb_P, (long long)pp);
      }
    }
    P.bcap = std::max(P.bcap, (long long)q[k] * std::min<long long>(q[k], (long long)d[k] * bound[k + 1]));
    P.bcap = std::max(P.bcap, (long long)bound[k + 1] * bound[k + 1]);
    // R->L pass panels: theta = q_k x d p_{k+1}
    const long long l1 = (long long)d[k] * bound[k + 1], k1 = q[k];
    if (!jacobi_svd_panel_in_smem(l1, k1, sizeof(T))) P.svd_work = std::max(P.svd_work, (l1 + 1) * k1);
    // pass 3 (centre > 0): left unfolding (bound_k d) x bound_{k+1}
    const long long l3 = (long long)bound[k] * d[k], k3 = bound[k + 1];
    if (!jacobi_svd_panel_in_smem(l3, k3, sizeof(T))) P.svd_work = std::max(P.svd_work, (l3 + 1) * (k3 + 1));
  }
  for (int n = 0; n + 1 < L; ++n) {
    const long long dn = d[n], dn1 = d[n + 1];
    P.xz = std::max({P.xz, (long long)pb[n] * dn * t[n + 1], (long long)t[n + 1] * dn1 * pb[n + 2],
                     (long long)t[n] * dn * pb[n + 1]});
    P.yw = std::max({P.yw, (long long)pb[n] * dn * dn1 * t[n + 2], (long long)t[n] * dn * dn1 * pb[n + 2]});
    P.th = std::max(P.th, (long long)pb[n] * dn * dn1 * pb[n + 2]);
    const long long l = (long long)bound[n] * dn, kk = (long long)dn1 * bound[n + 2];
    if (!jacobi_svd_panel_in_smem(l, kk, sizeof(T)) || !jacobi_svd_panel_in_smem(kk, l, sizeof(T)))
      P.svd_work = std::max(P.svd_work, (l + 1) * (kk + 1));
  }
  if (L >= 1) P.xz = std::max(P.xz, (long long)t[L - 1] * d[L - 1] * pb[L]);
  // largest split panel (either orientation) for the grid-cooperative SVD workspace
  long long svd_l = 1, svd_k = 1;
  for (int k = 0; k < L; ++k) {
    svd_l = std::max({svd_l, (long long)d[k] * bound[k + 1], (long long)bound[k] * d[k]});
    svd_k = std::max({svd_k, (long long)q[k], (long long)bound[k + 1], (long long)d[k] * bound[k + 1],
                      (long long)bound[k] * d[k]});
  }
  const long long svd_lk = std::max(svd_l, svd_k);
  P.env_cap.resize(L + 1);
  for (int k = 0; k <= L; ++k) P.env_cap[k] = (long long)pb[k] * t[k];

  // ---- output container and workspaces
  ttg_dmps* psi = new_dmps(L, target.dtype, B, d, P.psi_cap, st);
  std::unique_ptr<ttg_dmps> psi_guard(psi);
  const size_t es = sizeof(T);
  DevBuf bonds_buf((size_t)B * (L + 3) * sizeof(int), st);
  DevBuf state_buf((size_t)B * sizeof(ChainState), st);
  E.d_bonds = bonds_buf.as<int>();
  E.d_state = state_buf.as<ChainState>();
  {
    std::vector<int> hb((size_t)B * (L + 3));
    for (int c = 0; c < B; ++c)
      for (int k = 0; k <= L + 2; ++k) hb[(size_t)c * (L + 3) + k] = k <= L ? q[k] : 1;
    CK(cudaMemcpyAsync(E.d_bonds, hb.data(), hb.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // hb goes out of scope
  }
  CK(init_state(E.d_state, B, st));
  ++ctx->launches;
  DevBuf C0((size_t)B * P.ccap * es, st), C1((size_t)B * P.ccap * es, st);
  DevBuf Rb((size_t)B * P.rcap * es, st), Bb((size_t)B * P.bcap * es, st);
  DevBuf qrw(P.qr_work ? (size_t)B * P.qr_work * es : 0, st);
  const bool any_blocked = P.qb_A > 0;
  DevBuf qbA(any_blocked ? (size_t)B * P.qb_A * es : 0, st), qbV(any_blocked ? (size_t)B * P.qb_V * es : 0, st),
      qbT(any_blocked ? (size_t)B * P.qb_T * es : 0, st), qbW1(any_blocked ? (size_t)B * P.qb_W * es : 0, st),
      qbW2(any_blocked ? (size_t)B * P.qb_W * es : 0, st), qbP(any_blocked ? (size_t)B * P.qb_P * es : 0, st);
  const QrBlockedWork qbw{qbA.p, qbV.p, qbT.p, qbW1.p, qbW2.p, qbP.p, P.qb_A, P.qb_V, P.qb_T, P.qb_W, P.qb_P};
  DevBuf svdw(P.svd_work ? (size_t)B * P.svd_work * es : 0, st);
  DevBuf svdg(B <= 16 ? (size_t)B * jacobi_grid_work_bytes((int)svd_lk, (int)svd_lk, es) : 0, st);
  E.svd_grid_work = B <= 16 ? svdg.p : nullptr;
  E.pre_cap = std::min(svd_lk, 256LL) * std::min(svd_lk, 256LL);  // small preconditioned splits only
  DevBuf prebuf((size_t)B * 4 * E.pre_cap * es, st);
  DevBuf svbuf((size_t)B * svd_lk * sizeof(double), st);
  E.svals = svbuf.as<double>();
  E.svals_cap = svd_lk;
  E.pre_buf = prebuf.p;
  E.pre_slot = L + 2;
  const long long sC = P.ccap, sR = P.rcap, sBb = P.bcap;
  T* cbuf[2] = {C0.as<T>(), C1.as<T>()};
  const double tol = s.tolerance;

  // TTG_PHASES=1: device time of the call's phases on stderr (diagnostics)
  static const bool phases = getenv("TTG_PHASES") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  auto mark = [&](const char* name) {
    if (!phases) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.emplace_back(name, e);
  };
  mark("start");
  // Q-free exact pass (single chains, two-level blocked QRs): the thin Q of site k is applied to
  // the carried U S of pass 2 from its WY form (4 m k r flops) instead of being formed (2 m k^2)
  // and multiplied (2 m k r).  TTG_QFREE=0 forms Q as before.
  static const bool qfree_ok = [] {
    const char* e = getenv("TTG_QFREE");
    return !(e && e[0] == '0');
  }();
  std::vector<char> qfree(L, 0);
  std::vector<DevBuf> wy(L);
  for (int k = 0; k + 1 < L; ++k)
    qfree[k] = qfree_ok && B == 1 && (long long)qr_workspace_elems<T>(q[k] * d[k], g[k + 1]) * (long long)sizeof(T) >
                                           200 * 1024 && qr_two_level(q[k] * d[k], g[k + 1]) &&
               q[k + 1] == std::min(q[k] * d[k], g[k + 1]);
  // ---- pass 1: exact left-to-right QR (mps.hpp:193-205)
  int cur = 0;
  const T* curp = static_cast<const T*>(guess.site[0]);
  long long s_cur = guess.cap[0];
  if (L == 1) {
    CK(cudaMemcpy2DAsync(cbuf[0], sC * es, curp, s_cur * es, (size_t)d[0] * es, B, cudaMemcpyDeviceToDevice, st));
    curp = cbuf[0];
    s_cur = sC;
  }
  for (int k = 0; k + 1 < L; ++k) {
    QrParams qp{};
    qp.A = curp;
    qp.sA = s_cur;
    qp.Q = psi->site[k];
    qp.sQ = P.psi_cap[k];
    qp.R = Rb.p;
    qp.sR = sR;
    qp.work = qrw.p;
    qp.s_work = P.qr_work;
    qp.m = q[k] * d[k];
    qp.n = g[k + 1];
    {
      const double a = std::max(qp.m, qp.n), b = std::min(qp.m, qp.n);
      ProfScope ps(ctx, TTG_PROF_QR, (Scalar<T>::is_complex ? 4.0 : 1.0) * B * 4.0 * b * b * (a - b / 3.0));
      if ((long long)qr_workspace_elems<T>(qp.m, qp.n) * (long long)sizeof(T) > 200 * 1024) {
        long long nl = 0;
        if (qfree[k]) {
          // Q is never formed: the reflectors stay in the psi site (ld = q_{k+1} = min(m, n)) and the
          // WY factors in wy[k]; pass 2 applies Q to the carried U S (householder_apply_q)
          size_t a_, v_, t_, w_, p_;
          qr_blocked_elems<T>(qp.m, qp.n, &a_, &v_, &t_, &w_, &p_);
          wy[k] = DevBuf(t_ * sizeof(T), st);
          QrBlockedWork wk = qbw;
          wk.V = psi->site[k];
          wk.T = wy[k].p;
          wk.keep_wy = 1;
          QrParams qr = qp;
          qr.Q = nullptr;
          CK(householder_qr_blocked<T>(qr, wk, B, st, &nl));
        } else {
          CK(householder_qr_blocked<T>(qp, qbw, B, st, &nl));
        }
        ctx->launches += nl - 1;
      } else {
        CK(householder_qr<T>(qp, B, st));
      }
    }
    ++ctx->launches;
    // carried = R * next.right_matrix()  (mps.hpp:202)
    const int nxt = (k == 0 && curp != cbuf[0]) ? 0 : cur ^ 1;
    E.G(Rb.p, sR, guess.site[k + 1], guess.cap[k + 1], cbuf[nxt], sC, dconst(q[k + 1]), dconst(d[k + 1] * g[k + 2]),
        dconst(g[k + 1]), OP_N, OP_N, false, 0, true);  // R is upper triangular: half the product
    cur = nxt;
    curp = cbuf[cur];
    s_cur = sC;
  }
  // <T,T>: with the default guess the QR pass is an exact orthogonalisation of
  // T itself, so |T|^2 = |carried centre|_F^2 (= scprod(T,T), simplify.hpp:37-41)
  const bool default_guess = (&guess == &target);
  if (variational) {
    double* tn2 = reinterpret_cast<double*>(E.d_state) + offsetof(ChainState, target_norm2) / sizeof(double);
    const long long s_st = sizeof(ChainState) / sizeof(double);
    if (default_guess) {
      CK(frob2<T>(curp, s_cur, dconst(q[L - 1] * d[L - 1]), dconst(1), E.d_bonds, E.ld, tn2, s_st, B, st));
      ++ctx->launches;
    } else {
      // env chain <T,T> (mps.hpp:416-423)
      long long ecap = 1, xcap = 1;
      for (int k = 0; k < L; ++k) {
        ecap = std::max(ecap, (long long)t[k] * t[k]);
        xcap = std::max(xcap, (long long)t[k] * d[k] * t[k + 1]);
      }
      DevBuf e0((size_t)B * ecap * es, st), e1((size_t)B * ecap * es, st), xb((size_t)B * xcap * es, st);
      CK(fill_one<T>(e0.as<T>(), ecap, B, st));
      ++ctx->launches;
      T* eb[2] = {e0.as<T>(), e1.as<T>()};
      for (int k = 0; k < L; ++k) {
        E.G(eb[k & 1], ecap, target.site[k], target.cap[k], xb.p, xcap, dconst(t[k]), dconst(d[k] * t[k + 1]),
            dconst(t[k]), OP_N, OP_N, false);
        E.G(target.site[k], target.cap[k], xb.p, xcap, eb[(k + 1) & 1], ecap, dconst(t[k + 1]), dconst(t[k + 1]),
            dconst(t[k] * d[k]), OP_C, OP_N, false);
      }
      CK(env_real<T>(eb[L & 1], ecap, tn2, s_st, B, st));  // <T,T>
      ++ctx->launches;
    }
  }

  // Frames of the previous split at a bond as a warm start: off by default (for
  // graded spectra a slightly stale frame does not cut the Jacobi sweeps; the
  // QR preconditioner does), TTG_SVD_WARM=1 enables it.
  static const bool warm_frames = [] {
    const char* e = getenv("TTG_SVD_WARM");
    return e && e[0] == '1';
  }();
  // warm-start frames per two-site block n: U (after L->R) and V (after R->L)
  DevBuf TH2(variational && warm_frames ? (size_t)B * P.th * es : 0, st);
  std::vector<long long> fcap(L, 1);
  std::vector<DevBuf> frameU, frameV;
  frameU.reserve(L);
  frameV.reserve(L);
  for (int n = 0; n + 1 < L; ++n) {
    const long long side = std::max((long long)pb[n] * d[n], (long long)d[n + 1] * pb[n + 2]);
    fcap[n] = side * side;
    frameU.emplace_back(warm_frames ? (size_t)B * fcap[n] * es : 0, st);  // placeholders unless TTG_SVD_WARM=1
    frameV.emplace_back(warm_frames ? (size_t)B * fcap[n] * es : 0, st);
  }
  DevBuf fmeta((size_t)2 * B * L * sizeof(int), st);
  CK(cudaMemsetAsync(fmeta.p, 0, (size_t)2 * B * L * sizeof(int), st));
  int* fU = fmeta.as<int>();
  int* fV = fU + (size_t)B * L;
  mark("qr_pass");
  // ---- pass 2: truncating right-to-left sweep (mps.hpp:206-210, 253-265)
  for (int k = L - 1; k >= 1; --k) {
    const DimExpr rows = dconst(q[k]);
    const DimExpr cols = dbond(k + 1, d[k]);
    E.S(curp, s_cur, rows, cols, k, psi->site[k], P.psi_cap[k], 1, tol, mb, false, true, svdw.p, P.svd_work);
    // U S = theta V_r  (q_k x r)
    E.G(curp, s_cur, psi->site[k], P.psi_cap[k], Bb.p, sBb, rows, dbond(k), cols, OP_N, OP_C, false);
    // prev.left_matrix() * (U S)  (mps.hpp:261)
    const int nxt = cur ^ 1;
    if (qfree[k - 1]) {  // Q_{k-1} [U S; 0] from the WY form of the exact-pass QR
      int r = 0;
      CK(cudaMemcpyAsync(&r, E.d_bonds + k, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const int mq = q[k - 1] * d[k - 1];
      T* X = cbuf[nxt];
      CK(cudaMemcpyAsync(X, Bb.p, (size_t)q[k] * r * es, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemsetAsync(X + (size_t)q[k] * r, 0, (size_t)(mq - q[k]) * r * es, st));
      long long nl = 0;
      ProfScope ps(ctx, TTG_PROF_GEMM, (Scalar<T>::is_complex ? 16.0 : 4.0) * mq * (double)q[k] * r);
      CK(householder_apply_q<T>(psi->site[k - 1], wy[k - 1].p, mq, q[k], X, r, qbW1.p, qbW2.p, st, &nl));
      ctx->launches += nl;
      wy[k - 1] = DevBuf();
    } else {
      E.G(psi->site[k - 1], P.psi_cap[k - 1], Bb.p, sBb, cbuf[nxt], sC, dconst(q[k - 1] * d[k - 1]), dbond(k),
          dconst(q[k]), OP_N, OP_N, false);
    }
    cur = nxt;
    curp = cbuf[cur];
    s_cur = sC;
  }
  // centre tensor at site 0
  CK(copy_dims<T>(curp, s_cur, static_cast<T*>(psi->site[0]), P.psi_cap[0], dconst(d[0]), dbond(1), E.d_bonds, E.ld,
                  nullptr, 0, (long long)d[0] * bound[1], B, st));
  ++ctx->launches;
  // pass 3: move to the requested centre (mps.hpp:211-213, 238-250)
  for (int c = 0; c < center; ++c) {
    CK(copy_dims<T>(static_cast<T*>(psi->site[c]), P.psi_cap[c], cbuf[0], sC, dbond(c, d[c]), dbond(c + 1),
                    E.d_bonds, E.ld, nullptr, 0, P.psi_cap[c], B, st));
    ++ctx->launches;
    CK(copy_bond(E.d_bonds, E.ld, c + 1, L + 1, B, st));  // keep the old bond p_{c+1}
    ++ctx->launches;
    E.S(cbuf[0], sC, dbond(c, d[c]), dbond(c + 1), c + 1, psi->site[c], P.psi_cap[c], 0, tol, mb, false, true,
        svdw.p, P.svd_work);
    // S V^H = U_r^H theta (r x p_old), then carried into the next site (mps.hpp:246)
    E.G(psi->site[c], P.psi_cap[c], cbuf[0], sC, Bb.p, sBb, dbond(c + 1), dbond(L + 1), dbond(c, d[c]), OP_C, OP_N,
        false);
    E.G(Bb.p, sBb, psi->site[c + 1], P.psi_cap[c + 1], cbuf[1], sC, dbond(c + 1), dbond(c + 2, d[c + 1]),
        dbond(L + 1), OP_N, OP_N, false);
    CK(copy_dims<T>(cbuf[1], sC, static_cast<T*>(psi->site[c + 1]), P.psi_cap[c + 1], dbond(c + 1),
                    dbond(c + 2, d[c + 1]), E.d_bonds, E.ld, nullptr, 0, P.psi_cap[c + 1], B, st));
    ++ctx->launches;
  }
  const int out_center = variational ? 0 : center;

  if (variational && L >= 2) {
    mark("truncating_pass");
    // ---- environments (simplify.hpp:28-36)
    std::vector<DevBuf> lenv, renv;
    lenv.reserve(L + 1);
    renv.reserve(L + 1);
    for (int k = 0; k <= L; ++k) {
      lenv.emplace_back((size_t)B * P.env_cap[k] * es, st);
      renv.emplace_back((size_t)B * P.env_cap[k] * es, st);
    }
    DevBuf XZ((size_t)B * P.xz * es, st), YW((size_t)B * P.yw * es, st), TH((size_t)B * P.th * es, st);
    const long long sxz = P.xz, syw = P.yw, sth = P.th;
    CK(fill_one<T>(lenv[0].as<T>(), P.env_cap[0], B, st));
    CK(fill_one<T>(renv[L].as<T>(), P.env_cap[L], B, st));
    ctx->launches += 2;
    auto Ts = [&](int k) { return (const void*)target.site[k]; };
    auto Tc = [&](int k) { return target.count == 1 ? 0LL : target.cap[k]; };
    for (int k = L - 1; k >= 1; --k) {
      // Z = T_k (t_k d x t_{k+1}) . renv[k+1]^T ; renv[k] = conj(psi_k) . Z^T
      E.G(Ts(k), Tc(k), renv[k + 1].p, P.env_cap[k + 1], XZ.p, sxz, dconst(t[k] * d[k]), dbond(k + 1),
          dconst(t[k + 1]), OP_N, OP_T, false);
      E.G(psi->site[k], P.psi_cap[k], XZ.p, sxz, renv[k].p, P.env_cap[k], dbond(k), dconst(t[k]), dbond(k + 1, d[k]),
          OP_R, OP_T, false);
    }
    CK(begin_sweeps(E.d_state, B, st));
    // from here on psi bonds are <= pb (truncated canonical form): tighter launch bounds
    for (int k = 0; k <= L; ++k) bound[k] = pb[k];
    bound[L + 1] = *std::max_element(pb.begin(), pb.begin() + L + 1);
    bound[L + 2] = 1;
    for (int k = 0; k < L; ++k) bound[L + 2] = std::max({bound[L + 2], d[k] * pb[k], d[k] * pb[k + 1]});
    ++ctx->launches;

    mark("right_envs");
    // ---- sweeps (simplify.hpp:66-91, 114-125)
    const int nsweeps = std::max(1, s.max_sweeps);
    std::vector<ChainState> hstate(B);
    // host mirror of the bond table for one chain with large bonds (TTG_HOST_DIMS=0 disables): the sweep
    // splits of such chains synchronise once per step anyway (split_large)
    static const bool host_dims_env = [] {
      const char* ev = getenv("TTG_HOST_DIMS");
      return !(ev && ev[0] == '0');
    }();
    E.host_dims = host_dims_env && B == 1 && !Scalar<T>::is_complex && bound[L + 1] >= 256;
    for (int sw = 0; sw < nsweeps; ++sw) {
      for (int n = 0; n + 1 < L; ++n) {  // left to right
        const int dn = d[n], dn1 = d[n + 1];
        E.refresh_bonds();
        E.G(lenv[n].p, P.env_cap[n], Ts(n), Tc(n), XZ.p, sxz, dbond(n), dconst(dn * t[n + 1]), dconst(t[n]), OP_N,
            OP_N, true);
        E.G(XZ.p, sxz, Ts(n + 1), Tc(n + 1), YW.p, syw, dbond(n, dn), dconst(dn1 * t[n + 2]), dconst(t[n + 1]),
            OP_N, OP_N, true);
        E.G(YW.p, syw, renv[n + 2].p, P.env_cap[n + 2], TH.p, sth, dbond(n, dn * dn1), dbond(n + 2),
            dconst(t[n + 2]), OP_N, OP_T, true);
        // optional warm start: theta V_prev (same singular values, same U)
        typename Engine<T>::Warm wl;
        if (warm_frames)
          E.G(TH.p, sth, frameV[n].p, fcap[n], TH2.p, sth, dbond(n, dn), dbond(n + 2, dn1), dbond(n + 2, dn1), OP_N,
              OP_N, true);
        wl.pre = warm_frames ? TH2.p : nullptr;
        wl.s_pre = sth;
        wl.fin = warm_frames ? fV + n : nullptr;
        wl.fout = warm_frames ? fU + n : nullptr;
        wl.fld = L;
        wl.frame = warm_frames ? frameU[n].p : nullptr;
        wl.s_frame = fcap[n];
        E.S(TH.p, sth, dbond(n, dn), dbond(n + 2, dn1), n + 1, psi->site[n], P.psi_cap[n], 0, tol, mb, true, false,
            svdw.p, P.svd_work, wl);
        E.G(psi->site[n], P.psi_cap[n], TH.p, sth, psi->site[n + 1], P.psi_cap[n + 1], dbond(n + 1),
            dbond(n + 2, dn1), dbond(n, dn), OP_C, OP_N, true);
        E.G(psi->site[n], P.psi_cap[n], XZ.p, sxz, lenv[n + 1].p, P.env_cap[n + 1], dbond(n + 1),
            dconst(t[n + 1]), dbond(n, dn), OP_C, OP_N, true);
      }
      for (int n = L - 2; n >= 0; --n) {  // right to left
        const int dn = d[n], dn1 = d[n + 1];
        E.refresh_bonds();
        E.G(Ts(n + 1), Tc(n + 1), renv[n + 2].p, P.env_cap[n + 2], XZ.p, sxz, dconst(t[n + 1] * dn1), dbond(n + 2),
            dconst(t[n + 2]), OP_N, OP_T, true);
        E.G(Ts(n), Tc(n), XZ.p, sxz, YW.p, syw, dconst(t[n] * dn), dbond(n + 2, dn1), dconst(t[n + 1]), OP_N, OP_N,
            true);
        E.G(lenv[n].p, P.env_cap[n], YW.p, syw, TH.p, sth, dbond(n), dbond(n + 2, dn * dn1), dconst(t[n]), OP_N,
            OP_N, true);
        // optional warm start: U_prev^H theta (same singular values, same V)
        typename Engine<T>::Warm wr;
        if (warm_frames)
          E.G(frameU[n].p, fcap[n], TH.p, sth, TH2.p, sth, dbond(n, dn), dbond(n + 2, dn1), dbond(n, dn), OP_C, OP_N,
              true);
        wr.pre = warm_frames ? TH2.p : nullptr;
        wr.s_pre = sth;
        wr.fin = warm_frames ? fU + n : nullptr;
        wr.fout = warm_frames ? fV + n : nullptr;
        wr.fld = L;
        wr.frame = warm_frames ? frameV[n].p : nullptr;
        wr.s_frame = fcap[n];
        E.S(TH.p, sth, dbond(n, dn), dbond(n + 2, dn1), n + 1, psi->site[n + 1], P.psi_cap[n + 1], 1, tol, mb, true,
            false, svdw.p, P.svd_work, wr);
        E.G(TH.p, sth, psi->site[n + 1], P.psi_cap[n + 1], psi->site[n], P.psi_cap[n], dbond(n, dn), dbond(n + 1),
            dbond(n + 2, dn1), OP_N, OP_C, true);
        E.G(psi->site[n + 1], P.psi_cap[n + 1], XZ.p, sxz, renv[n + 1].p, P.env_cap[n + 1], dbond(n + 1),
            dconst(t[n + 1]), dbond(n + 2, dn1), OP_R, OP_T, true);
      }
      CK(sweep_end<T>(static_cast<T*>(psi->site[0]), P.psi_cap[0], dbond(1, d[0]), E.d_bonds, E.ld, E.d_state,
                      s.simplification_tolerance, sw, B, st));
      ++ctx->launches;
      if (sw + 1 < nsweeps) {
        CK(cudaMemcpyAsync(hstate.data(), E.d_state, B * sizeof(ChainState), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        bool any = false;
        for (int c = 0; c < B && !any; ++c) any = hstate[c].active != 0;
        if (!any) break;
      }
    }
  } else if (variational) {
    // L == 1: the sweep copies the target (simplify.hpp:68-76)
    CK(cudaMemcpy2DAsync(psi->site[0], P.psi_cap[0] * es, target.site[0], target.cap[0] * es, (size_t)d[0] * es, B,
                         cudaMemcpyDeviceToDevice, st));
  }

  mark("sweeps");
  if (phases) {
    cudaEventSynchronize(marks.back().second);
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
      fprintf(stderr, "phase %-16s %9.2f ms\n", marks[i].first, ms);
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
  // ---- finalize: norms, ledger, zero states, normalisation
  DevBuf norms((size_t)B * sizeof(double), st);
  {
    // centre = out_center; its shape is p_c x d x p_{c+1}
    std::vector<int> hb((size_t)B * (L + 3));
    CK(cudaMemcpyAsync(hb.data(), E.d_bonds, hb.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int c = 0; c < B; ++c)
      for (int k = 0; k <= L; ++k) psi->bonds[(size_t)c * (L + 1) + k] = hb[(size_t)c * (L + 3) + k];
  }
  const int cc = out_center;
  CK(frob2<T>(static_cast<T*>(psi->site[cc]), P.psi_cap[cc], dbond(cc, d[cc]), dbond(cc + 1), E.d_bonds, E.ld,
              norms.as<double>(), 1, B, st));
  ++ctx->launches;
  std::vector<ChainState> hs(B);
  std::vector<double> hn(B);
  CK(cudaMemcpyAsync(hs.data(), E.d_state, B * sizeof(ChainState), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hn.data(), norms.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < B; ++c) {
    if (hs[c].status & ST_NONFINITE) throw Error{TTG_NUMERIC, "schmidt_split: non-finite input"};
    if (hs[c].status & ST_NOCONV) throw Error{TTG_NUMERIC, "SVD failed to converge"};
  }
  std::vector<double> scale(B, 1.0);
  bool any_scale = false, any_zero = false;
  std::vector<int> zero(B, 0);
  for (int c = 0; c < B; ++c) {
    const double nrm = std::sqrt(std::max(0.0, hn[c]));
    ttg_report r{};
    if (variational) {
      const double tn2 = L == 1 ? hn[c] : hs[c].target_norm2;
      const double tn = std::sqrt(std::max(0.0, tn2));
      double residual;
      int sweeps = hs[c].sweeps;
      int conv = hs[c].converged;
      if (L == 1) {
        residual = fp_error_floor(tn);
        sweeps = 1;
        conv = 1;
      } else if (tn <= fp_error_floor(1.0)) {  // simplify.hpp:107-112
        residual = tn;
        conv = 1;
        zero[c] = 1;
      } else {
        residual = std::sqrt(std::max(0.0, hs[c].dist2)) + fp_error_floor(tn);
      }
      if (nrm == 0.0) zero[c] = 1;  // simplify.hpp:128-129
      r.sweeps = sweeps;
      r.converged = conv;
      r.residual = residual;
      r.target_norm2 = tn2;
      psi->error[c] = target.error[c] + residual;  // simplify.hpp:191
    } else {
      // CanonicalMPS ctor ledger (mps.hpp:214-215)
      psi->error[c] = guess.error[c] + std::sqrt(hs[c].err2) + fp_error_floor(nrm);
      r.residual = std::sqrt(hs[c].err2);
      r.target_norm2 = hn[c];
    }
    double final_norm = zero[c] ? 0.0 : nrm;
    if (s.normalize && final_norm > 0.0) {  // mps.hpp:227-235
      scale[c] = 1.0 / final_norm;
      any_scale = true;
      psi->error[c] /= final_norm;
      final_norm = 1.0;
    }
    r.norm = final_norm;
    r.error = psi->error[c];
    if (reports) reports[c] = r;
    any_zero |= zero[c] != 0;
  }
  if (any_zero) {
    for (int c = 0; c < B; ++c) {
      if (!zero[c]) continue;
      for (int k = 0; k <= L; ++k) psi->bonds[(size_t)c * (L + 1) + k] = 1;
      for (int k = 0; k < L; ++k)
        CK(cudaMemsetAsync(static_cast<char*>(psi->site[k]) + (size_t)c * P.psi_cap[k] * es, 0, (size_t)d[k] * es,
                           st));
    }
  }
  if (any_scale) {
    DevBuf f((size_t)B * sizeof(double), st);
    CK(cudaMemcpyAsync(f.p, scale.data(), B * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(scale_chains<T>(static_cast<T*>(psi->site[cc]), P.psi_cap[cc], P.psi_cap[cc], f.as<double>(), B, st));
    ++ctx->launches;
    CK(cudaStreamSynchronize(st));
  }
  psi->center = out_center;
  CK(cudaStreamSynchronize(st));
  *out = psi_guard.release();
}

// ---------------------------------------------------------------------------
// helpers for the ABI
// ---------------------------------------------------------------------------

ttg_status fail(ttg_ctx* ctx, ttg_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return st;
}

template <typename F>
ttg_status guarded(ttg_ctx* ctx, F&& f) {
  if (!ctx) return TTG_INVALID;
  try {
    f();
    return TTG_OK;
  } catch (const Error& e) {
    return fail(ctx, e.st, e.msg);
  } catch (const std::exception& e) {
    return fail(ctx, TTG_INVALID, e.what());
  }
}

// Convert a batch to complex128 (promotion of real inputs, types.hpp:12-16).
ttg_dmps* to_complex(ttg_ctx* ctx, const ttg_dmps& m) {
  std::vector<long long> cap = m.cap;
  ttg_dmps* o = new_dmps(m.n, TTG_C128, m.count, m.phys, cap, ctx->stream);
  o->bonds = m.bonds;
  o->error = m.error;
  o->center = m.center;
  for (int k = 0; k < m.n; ++k) {
    CK(real_to_complex(static_cast<const double*>(m.site[k]), static_cast<cplx*>(o->site[k]),
                       (long long)m.count * m.cap[k], ctx->stream));
    ++ctx->launches;
  }
  return o;
}

void check_strategy(const ttg_strategy* s) {
  if (!s) throw Error{TTG_INVALID, "null strategy"};
}

void dispatch_simplify(ttg_ctx* ctx, const ttg_dmps* target, const ttg_dmps* guess, const ttg_strategy& s,
                       bool variational, int center, ttg_dmps** out, ttg_report* reports) {
  if (!target || !out) throw Error{TTG_INVALID, "null argument"};
  if (target->n < 1) throw Error{TTG_SHAPE, "empty MPS"};
  if (!target->uniform()) throw Error{TTG_SHAPE, "batched simplify needs chains of identical shape"};
  std::unique_ptr<ttg_dmps> promoted_t, promoted_g;
  const ttg_dmps* T_ = target;
  const ttg_dmps* G_ = guess ? guess : target;
  if (guess) {
    if (guess->n != target->n || guess->count != target->count) throw Error{TTG_SHAPE, "guess/target mismatch"};
    if (!guess->uniform()) throw Error{TTG_SHAPE, "guess chains must share one shape"};
    for (int k = 0; k < target->n; ++k)
      if (guess->phys[k] != target->phys[k]) throw Error{TTG_SHAPE, "guess/target physical dimension mismatch"};
    if (guess->dtype != target->dtype) {
      if (target->dtype == TTG_F64) {
        promoted_t.reset(to_complex(ctx, *target));
        T_ = promoted_t.get();
      } else {
        promoted_g.reset(to_complex(ctx, *guess));
        G_ = promoted_g.get();
      }
    }
  }
  if (!guess) G_ = T_;
  if (T_->dtype == TTG_F64)
    run_simplify<double>(ctx, *T_, *G_, s, variational, center, out, reports);
  else
    run_simplify<cplx>(ctx, *T_, *G_, s, variational, center, out, reports);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

const char* ttg_version(void) { return "ttgpu 0.1 (sm_100a)"; }

ttg_status ttg_create(int device, ttg_ctx** out) {
  if (!out) return TTG_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return TTG_CUDA;
  }
  if (device < 0 || device >= n) return TTG_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return TTG_CUDA;
  auto* c = new ttg_ctx();
  c->device = device;
  // highest priority: the context stream carries the latency-critical chain (panels, splits); the
  // blocked QR's far updates run on a lowest-priority auxiliary stream (qr.cu, lookahead)
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&c->own, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    delete c;
    return TTG_CUDA;
  }
  c->stream = c->own;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return TTG_OK;
}

void ttg_destroy(ttg_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  ttg_comm_free(ctx);
  ctx->flush_profile();
  if (ctx->d_sweeps) cudaFree(ctx->d_sweeps);
  for (int i = 0; i < 2; ++i) {
    if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
    if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
  }
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
}

// ---------------------------------------------------------------------------
// NCCL communicator owned by the context.  The batched configs shard independent
// chains over one rank per GPU; the only exchange is one all-gather of per-chain scalars per batch.
// libnccl is bound at run time (dlopen by soname: inside a torch process that is torch's own copy), so
// single-GPU users never need it and the library has no link-time dependency on it.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  void* handle = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string why;
};
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = getenv("TTG_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n || !*n) continue;
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      a.why = "libnccl.so.2 not found (set TTG_NCCL_LIB)";
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.handle, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.handle, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.handle, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.handle, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.handle, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllGather || !a.CommDestroy || !a.GetErrorString) {
      a.why = "libnccl lacks a required symbol";
      a.handle = nullptr;
    }
    return a;
  }();
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error{TTG_CUDA, std::string(what) + ": " + nccl_api().GetErrorString(r)};
}
NcclApi& nccl_required() {
  NcclApi& a = nccl_api();
  if (!a.handle) throw Error{TTG_CUDA, "NCCL unavailable: " + a.why};
  return a;
}
}  // namespace

static_assert(sizeof(ncclUniqueId) == TTG_COMM_ID_BYTES, "ttgpu.h: TTG_COMM_ID_BYTES must match ncclUniqueId");

ttg_status ttg_comm_unique_id(ttg_ctx* ctx, void* id) {
  return guarded(ctx, [&] {
    if (!id) throw Error{TTG_INVALID, "ttg_comm_unique_id: null id"};
    ncclUniqueId u;
    nccl_check(nccl_required().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
  });
}

ttg_status ttg_comm_init(ttg_ctx* ctx, int nranks, int rank, const void* id) {
  return guarded(ctx, [&] {
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) throw Error{TTG_INVALID, "ttg_comm_init: bad rank / size / id"};
    if (ctx->comm) throw Error{TTG_INVALID, "ttg_comm_init: the context already owns a communicator"};
    CK(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    nccl_check(nccl_required().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
    ctx->comm = c;
    ctx->comm_rank = rank;
    ctx->comm_size = nranks;
  });
}

ttg_status ttg_comm_info(const ttg_ctx* ctx, int* nranks, int* rank) {
  if (!ctx) return TTG_INVALID;
  if (nranks) *nranks = ctx->comm ? ctx->comm_size : 1;
  if (rank) *rank = ctx->comm ? ctx->comm_rank : 0;
  return TTG_OK;
}

ttg_status ttg_comm_allgather_f64(ttg_ctx* ctx, const double* send, int64_t count, double* recv) {
  return guarded(ctx, [&] {
    if (count < 0 || (count > 0 && (!send || !recv))) throw Error{TTG_INVALID, "ttg_comm_allgather_f64: bad arguments"};
    if (count == 0) return;
    if (!ctx->comm) {  // no communicator: a world of one
      std::memcpy(recv, send, (size_t)count * sizeof(double));
      return;
    }
    CK(cudaSetDevice(ctx->device));
    const size_t nb = (size_t)count * sizeof(double);
    DevBuf ds(nb, ctx->stream), dr(nb * ctx->comm_size, ctx->stream);
    CK(cudaMemcpyAsync(ds.p, send, nb, cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(nccl_api().AllGather(ds.p, dr.p, (size_t)count, ncclFloat64, static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllGather");
    CK(cudaMemcpyAsync(recv, dr.p, nb * ctx->comm_size, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

ttg_status ttg_comm_free(ttg_ctx* ctx) {
  if (!ctx) return TTG_INVALID;
  if (ctx->comm) {
    nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
    ctx->comm_rank = 0;
    ctx->comm_size = 1;
  }
  return TTG_OK;
}

const char* ttg_last_error(const ttg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

ttg_status ttg_set_stream(ttg_ctx* ctx, void* stream) {
  if (!ctx) return TTG_INVALID;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return TTG_OK;
}

ttg_status ttg_synchronize(ttg_ctx* ctx) {
  return guarded(ctx, [&] { CK(cudaStreamSynchronize(ctx->stream)); });
}

int64_t ttg_kernel_launches(const ttg_ctx* ctx) { return ctx ? ctx->launches : 0; }

ttg_status ttg_profile_enable(ttg_ctx* ctx, int on) {
  if (!ctx) return TTG_INVALID;
  ctx->flush_profile();
  ctx->profile = on ? 1 : 0;
  ctx->prof_svd_sweeps = 0;
  for (int c = 0; c < TTG_PROF_CLASSES; ++c) {
    ctx->prof_count[c] = 0;
    ctx->prof_ms[c] = 0.0;
    ctx->prof_flops[c] = 0.0;
  }
  return TTG_OK;
}

ttg_status ttg_profile_svd_sweeps(ttg_ctx* ctx, int64_t* total) {
  if (!ctx || !total) return TTG_INVALID;
  *total = ctx->prof_svd_sweeps;
  return TTG_OK;
}

ttg_status ttg_profile_read(ttg_ctx* ctx, int cls, int64_t* launches, double* ms, double* flops) {
  if (!ctx || cls < 0 || cls >= TTG_PROF_CLASSES) return TTG_INVALID;
  ctx->flush_profile();
  if (launches) *launches = ctx->prof_count[cls];
  if (ms) *ms = ctx->prof_ms[cls];
  if (flops) *flops = ctx->prof_flops[cls];
  return TTG_OK;
}

// pinned staging buffers of the context (shared with the TTLAB1 I/O path), allocated on first use
static size_t mps_stage_bytes() { return size_t(32) << 20; }
static void mps_stage_init(ttg_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (!ctx->stage[i]) CK(cudaMallocHost(&ctx->stage[i], mps_stage_bytes()));
    if (!ctx->stage_ev[i]) CK(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
  }
}

ttg_status ttg_mps_upload(ttg_ctx* ctx, const ttg_mps_view* views, int count, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!views || !out || count < 1) throw Error{TTG_INVALID, "null argument"};
    const int n = views[0].n, dtype = views[0].dtype;
    if (n < 1) throw Error{TTG_SHAPE, "empty MPS"};
    if (dtype != TTG_F64 && dtype != TTG_C128) throw Error{TTG_INVALID, "unknown dtype"};
    std::vector<int> phys(n);
    std::vector<long long> cap(n, 1);
    for (int k = 0; k < n; ++k) phys[k] = (int)views[0].phys[k];
    for (int c = 0; c < count; ++c) {
      const ttg_mps_view& v = views[c];
      if (v.n != n || v.dtype != dtype) throw Error{TTG_SHAPE, "batch chains differ in length or dtype"};
      if (v.bonds[0] != 1 || v.bonds[n] != 1) throw Error{TTG_SHAPE, "MPS boundary bonds must have size one"};
      if (v.error < 0) throw Error{TTG_SHAPE, "MPS error bound must be non-negative"};
      for (int k = 0; k < n; ++k) {
        if (v.phys[k] != phys[k]) throw Error{TTG_SHAPE, "batch chains differ in physical dimensions"};
        if (v.bonds[k] < 1 || v.phys[k] < 1 || v.bonds[k + 1] < 1) throw Error{TTG_SHAPE, "Tensor3 dimensions must be >= 1"};
        cap[k] = std::max(cap[k], (long long)(v.bonds[k] * v.phys[k] * v.bonds[k + 1]));
      }
    }
    ttg_dmps* m = new_dmps(n, dtype, count, phys, cap, ctx->stream);
    std::unique_ptr<ttg_dmps> guard(m);
    const size_t es = esize(dtype);
    for (int c = 0; c < count; ++c) {
      const ttg_mps_view& v = views[c];
      m->error[c] = v.error;
      for (int k = 0; k <= n; ++k) m->bonds[(size_t)c * (n + 1) + k] = (int)v.bonds[k];
    }
    // Batches go through the two pinned staging buffers: the chains' site-k tensors are packed
    // in the device layout (chain c at c * cap[k]) and cross PCIe as one copy per staging
    // chunk, the packing of chunk i+1 overlapping the DMA of chunk i.  Single chains and
    // tensors larger than a staging buffer are copied directly.
    const bool staged = count > 1 && [&] {
      for (int k = 0; k < n; ++k)
        if ((size_t)cap[k] * es > mps_stage_bytes()) return false;
      return true;
    }();
    if (staged) {
      mps_stage_init(ctx);
      int cur = 0;
      for (int k = 0; k < n; ++k) {
        const size_t cb = (size_t)cap[k] * es;
        const int per = (int)std::max<size_t>(1, mps_stage_bytes() / cb);
        for (int c0 = 0; c0 < count; c0 += per) {
          const int c1 = std::min(count, c0 + per);
          CK(cudaEventSynchronize(ctx->stage_ev[cur]));
          char* stg = static_cast<char*>(ctx->stage[cur]);
          for (int c = c0; c < c1; ++c) {
            const ttg_mps_view& v = views[c];
            std::memcpy(stg + (size_t)(c - c0) * cb, v.sites[k], (size_t)(v.bonds[k] * v.phys[k] * v.bonds[k + 1]) * es);
          }
          CK(cudaMemcpyAsync(static_cast<char*>(m->site[k]) + (size_t)c0 * cb, stg, (size_t)(c1 - c0) * cb,
                             cudaMemcpyHostToDevice, ctx->stream));
          CK(cudaEventRecord(ctx->stage_ev[cur], ctx->stream));
          cur ^= 1;
        }
      }
    } else {
      for (int c = 0; c < count; ++c) {
        const ttg_mps_view& v = views[c];
        for (int k = 0; k < n; ++k) {
          const size_t bytes = (size_t)(v.bonds[k] * v.phys[k] * v.bonds[k + 1]) * es;
          CK(cudaMemcpyAsync(static_cast<char*>(m->site[k]) + (size_t)c * cap[k] * es, v.sites[k], bytes,
                             cudaMemcpyHostToDevice, ctx->stream));
        }
      }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    *out = guard.release();
  });
}

ttg_status ttg_mps_from_device(ttg_ctx* ctx, int n, int dtype, int count, const int64_t* bonds, const int64_t* phys,
                               const void* const* dev_sites, const double* errors, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!bonds || !phys || !dev_sites || !out || count < 1 || n < 1) throw Error{TTG_INVALID, "bad argument"};
    if (dtype != TTG_F64 && dtype != TTG_C128) throw Error{TTG_INVALID, "unknown dtype"};
    if (bonds[0] != 1 || bonds[n] != 1) throw Error{TTG_SHAPE, "MPS boundary bonds must have size one"};
    std::vector<int> ph(n);
    std::vector<long long> cap(n);
    for (int k = 0; k < n; ++k) {
      if (bonds[k] < 1 || phys[k] < 1 || bonds[k + 1] < 1 || !dev_sites[k])
        throw Error{TTG_SHAPE, "Tensor3 dimensions must be >= 1"};
      ph[k] = (int)phys[k];
      cap[k] = bonds[k] * phys[k] * bonds[k + 1];
    }
    if (errors)
      for (int c = 0; c < count; ++c)
        if (!(errors[c] >= 0)) throw Error{TTG_SHAPE, "MPS error bound must be non-negative"};
    // the source buffers belong to the caller (e.g. torch tensors on another stream): order the copy after
    // all work already submitted to the device and finish it before returning (calls are synchronous)
    CK(cudaDeviceSynchronize());
    ttg_dmps* m = new_dmps(n, dtype, count, ph, cap, ctx->stream);
    std::unique_ptr<ttg_dmps> guard(m);
    for (int c = 0; c < count; ++c) {
      for (int k = 0; k <= n; ++k) m->bonds[(size_t)c * (n + 1) + k] = (int)bonds[k];
      m->error[c] = errors ? errors[c] : 0.0;
    }
    for (int k = 0; k < n; ++k)
      CK(cudaMemcpyAsync(m->site[k], dev_sites[k], (size_t)count * cap[k] * esize(dtype), cudaMemcpyDeviceToDevice,
                         ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *out = guard.release();
  });
}

void ttg_mps_free(ttg_dmps* m) { delete m; }

ttg_status ttg_mps_info(const ttg_dmps* m, int chain, int* n, int* dtype, int* count, int64_t* bonds, int64_t* phys,
                        double* error, int* center) {
  if (!m || chain < 0 || chain >= m->count) return TTG_INVALID;
  if (n) *n = m->n;
  if (dtype) *dtype = m->dtype;
  if (count) *count = m->count;
  if (bonds)
    for (int k = 0; k <= m->n; ++k) bonds[k] = m->bond(chain, k);
  if (phys)
    for (int k = 0; k < m->n; ++k) phys[k] = m->phys[k];
  if (error) *error = m->error[chain];
  if (center) *center = m->center;
  return TTG_OK;
}

ttg_status ttg_mps_download(ttg_ctx* ctx, const ttg_dmps* m, int chain, void* const* sites) {
  return guarded(ctx, [&] {
    if (!m || !sites || chain < 0 || chain >= m->count) throw Error{TTG_INVALID, "bad argument"};
    const size_t es = esize(m->dtype);
    for (int k = 0; k < m->n; ++k) {
      const size_t bytes = (size_t)m->bond(chain, k) * m->phys[k] * m->bond(chain, k + 1) * es;
      CK(cudaMemcpyAsync(sites[k], static_cast<const char*>(m->site[k]) + (size_t)chain * m->cap[k] * es, bytes,
                         cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

ttg_status ttg_mps_download_batch(ttg_ctx* ctx, const ttg_dmps* m, void* const* sites) {
  return guarded(ctx, [&] {
    if (!m || !sites) throw Error{TTG_INVALID, "bad argument"};
    const size_t es = esize(m->dtype);
    const int n = m->n, count = m->count;
    bool staged = count > 1;
    for (int k = 0; k < n; ++k) staged = staged && (size_t)m->cap[k] * es <= mps_stage_bytes();
    if (!staged) {
      for (int c = 0; c < count; ++c)
        for (int k = 0; k < n; ++k) {
          const size_t bytes = (size_t)m->bond(c, k) * m->phys[k] * m->bond(c, k + 1) * es;
          CK(cudaMemcpyAsync(sites[(size_t)c * n + k], static_cast<const char*>(m->site[k]) + (size_t)c * m->cap[k] * es,
                             bytes, cudaMemcpyDeviceToHost, ctx->stream));
        }
      CK(cudaStreamSynchronize(ctx->stream));
      return;
    }
    // one D2H per staging chunk (chains [c0, c1) of site k in the device layout); the copy of
    // the next chunk is in flight while the current one is scattered into the caller's buffers
    mps_stage_init(ctx);
    struct Chunk { int k, c0, c1; };
    std::vector<Chunk> chunks;
    for (int k = 0; k < n; ++k) {
      const size_t cb = (size_t)m->cap[k] * es;
      const int per = (int)std::max<size_t>(1, mps_stage_bytes() / cb);
      for (int c0 = 0; c0 < count; c0 += per) chunks.push_back({k, c0, std::min(count, c0 + per)});
    }
    auto issue = [&](size_t i) {
      const Chunk& q = chunks[i];
      const size_t cb = (size_t)m->cap[q.k] * es;
      CK(cudaMemcpyAsync(ctx->stage[i & 1], static_cast<const char*>(m->site[q.k]) + (size_t)q.c0 * cb,
                         (size_t)(q.c1 - q.c0) * cb, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaEventRecord(ctx->stage_ev[i & 1], ctx->stream));
    };
    issue(0);
    for (size_t i = 0; i < chunks.size(); ++i) {
      if (i + 1 < chunks.size()) issue(i + 1);
      CK(cudaEventSynchronize(ctx->stage_ev[i & 1]));
      const Chunk& q = chunks[i];
      const size_t cb = (size_t)m->cap[q.k] * es;
      const char* stg = static_cast<const char*>(ctx->stage[i & 1]);
      for (int c = q.c0; c < q.c1; ++c)
        std::memcpy(sites[(size_t)c * n + q.k], stg + (size_t)(c - q.c0) * cb,
                    (size_t)m->bond(c, q.k) * m->phys[q.k] * m->bond(c, q.k + 1) * es);
    }
  });
}

ttg_status ttg_mps_site_ptr(const ttg_dmps* m, int chain, int k, void** ptr, int64_t* elems) {
  if (!m || chain < 0 || chain >= m->count || k < 0 || k >= m->n) return TTG_INVALID;
  if (ptr) *ptr = static_cast<char*>(m->site[k]) + (size_t)chain * m->cap[k] * esize(m->dtype);
  if (elems) *elems = (int64_t)m->bond(chain, k) * m->phys[k] * m->bond(chain, k + 1);
  return TTG_OK;
}

ttg_status ttg_mpo_upload(ttg_ctx* ctx, const ttg_mpo_view* v, ttg_dmpo** out) {
  return guarded(ctx, [&] {
    if (!v || !out || v->n < 1) throw Error{TTG_INVALID, "bad argument"};
    if (v->dtype != TTG_F64 && v->dtype != TTG_C128) throw Error{TTG_INVALID, "unknown dtype"};
    const int n = v->n;
    if (v->bonds[0] != 1 || v->bonds[n] != 1) throw Error{TTG_SHAPE, "MPO boundary bonds must have size one"};
    auto* w = new ttg_dmpo();
    std::unique_ptr<ttg_dmpo> guard(w);
    w->n = n;
    w->dtype = v->dtype;
    w->stream = ctx->stream;
    for (int k = 0; k <= n; ++k) w->bonds.push_back((int)v->bonds[k]);
    for (int k = 0; k < n; ++k) {
      w->dout.push_back((int)v->phys_out[k]);
      w->din.push_back((int)v->phys_in[k]);
      const size_t bytes = (size_t)(v->bonds[k] * v->phys_out[k] * v->phys_in[k] * v->bonds[k + 1]) * esize(v->dtype);
      w->site.push_back(dev_alloc(bytes, ctx->stream));
      CK(cudaMemcpyAsync(w->site.back(), v->sites[k], bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    *out = guard.release();
  });
}

void ttg_mpo_free(ttg_dmpo* w) { delete w; }

ttg_status ttg_apply_raw(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* v, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!op || !v || !out) throw Error{TTG_INVALID, "null argument"};
    if (op->n != v->n) throw Error{TTG_SHAPE, "apply: operator and state sizes differ"};  // mpo.hpp:214-215
    for (int k = 0; k < v->n; ++k)
      if (op->din[k] != v->phys[k]) throw Error{TTG_SHAPE, "apply: physical dimension mismatch"};  // mpo.hpp:221-222
    if (!v->uniform()) throw Error{TTG_SHAPE, "apply on a batch needs chains of identical shape"};
    const int n = v->n, B = v->count;
    const int dtype = (op->dtype == TTG_C128 || v->dtype == TTG_C128) ? TTG_C128 : TTG_F64;
    std::unique_ptr<ttg_dmps> vc;
    const ttg_dmps* V = v;
    if (dtype == TTG_C128 && v->dtype == TTG_F64) {
      vc.reset(to_complex(ctx, *v));
      V = vc.get();
    }
    std::vector<int> phys(n);
    std::vector<long long> cap(n);
    for (int k = 0; k < n; ++k) {
      phys[k] = op->dout[k];
      cap[k] = (long long)op->bonds[k] * V->bond(0, k) * op->dout[k] * op->bonds[k + 1] * V->bond(0, k + 1);
    }
    ttg_dmps* o = new_dmps(n, dtype, B, phys, cap, ctx->stream);
    std::unique_ptr<ttg_dmps> guard(o);
    for (int c = 0; c < B; ++c) {
      for (int k = 0; k <= n; ++k) o->bonds[(size_t)c * (n + 1) + k] = op->bonds[k] * V->bond(0, k);
      o->error[c] = v->error[c];  // mpo.hpp:237
    }
    for (int k = 0; k < n; ++k) {
      const size_t welems = (size_t)op->bonds[k] * op->dout[k] * op->din[k] * op->bonds[k + 1];
      ProfScope ps(ctx, TTG_PROF_EXPAND, 0.0);
      if (dtype == TTG_F64) {
        CK(expand_mpo<double>(static_cast<const double*>(op->site[k]), static_cast<const double*>(V->site[k]),
                              static_cast<double*>(o->site[k]), op->bonds[k], op->dout[k], op->din[k],
                              op->bonds[k + 1], V->bond(0, k), V->bond(0, k + 1), B, V->cap[k], cap[k], ctx->stream));
      } else {
        DevBuf wc;
        const cplx* W = static_cast<const cplx*>(op->site[k]);
        if (op->dtype == TTG_F64) {
          wc = DevBuf(welems * sizeof(cplx), ctx->stream);
          CK(real_to_complex(static_cast<const double*>(op->site[k]), wc.as<cplx>(), (long long)welems, ctx->stream));
          ++ctx->launches;
          W = wc.as<cplx>();
        }
        CK(expand_mpo<cplx>(W, static_cast<const cplx*>(V->site[k]), static_cast<cplx*>(o->site[k]), op->bonds[k],
                            op->dout[k], op->din[k], op->bonds[k + 1], V->bond(0, k), V->bond(0, k + 1), B, V->cap[k],
                            cap[k], ctx->stream));
      }
      ++ctx->launches;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    *out = guard.release();
  });
}

ttg_status ttg_hadamard(ttg_ctx* ctx, const ttg_dmps* u, const ttg_dmps* v, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!u || !v || !out) throw Error{TTG_INVALID, "null argument"};
    if (u->n != v->n) throw Error{TTG_SHAPE, "hadamard: states of different length"};  // blas.hpp:46-47
    for (int k = 0; k < u->n; ++k)
      if (u->phys[k] != v->phys[k]) throw Error{TTG_SHAPE, "hadamard: physical dimension mismatch"};  // blas.hpp:53-54
    if (u->count != v->count) throw Error{TTG_SHAPE, "hadamard: batch sizes differ"};
    if (!u->uniform() || !v->uniform()) throw Error{TTG_SHAPE, "hadamard on a batch needs identical shapes"};
    const int n = u->n, B = u->count;
    const int dtype = (u->dtype == TTG_C128 || v->dtype == TTG_C128) ? TTG_C128 : TTG_F64;
    std::unique_ptr<ttg_dmps> uc, vc;
    const ttg_dmps* U = u;
    const ttg_dmps* V = v;
    if (dtype == TTG_C128 && u->dtype == TTG_F64) {
      uc.reset(to_complex(ctx, *u));
      U = uc.get();
    }
    if (dtype == TTG_C128 && v->dtype == TTG_F64) {
      vc.reset(to_complex(ctx, *v));
      V = vc.get();
    }
    std::vector<long long> cap(n);
    for (int k = 0; k < n; ++k)
      cap[k] = (long long)U->bond(0, k) * V->bond(0, k) * u->phys[k] * U->bond(0, k + 1) * V->bond(0, k + 1);
    ttg_dmps* o = new_dmps(n, dtype, B, u->phys, cap, ctx->stream);
    std::unique_ptr<ttg_dmps> guard(o);
    for (int c = 0; c < B; ++c) {
      for (int k = 0; k <= n; ++k) o->bonds[(size_t)c * (n + 1) + k] = U->bond(0, k) * V->bond(0, k);
      o->error[c] = u->error[c] + v->error[c];  // blas.hpp:66
    }
    for (int k = 0; k < n; ++k) {
      ProfScope ps(ctx, TTG_PROF_EXPAND, 0.0);
      if (dtype == TTG_F64)
        CK(expand_hadamard<double>(static_cast<const double*>(U->site[k]), static_cast<const double*>(V->site[k]),
                                   static_cast<double*>(o->site[k]), U->bond(0, k), u->phys[k], U->bond(0, k + 1),
                                   V->bond(0, k), V->bond(0, k + 1), B, U->cap[k], V->cap[k], cap[k], ctx->stream));
      else
        CK(expand_hadamard<cplx>(static_cast<const cplx*>(U->site[k]), static_cast<const cplx*>(V->site[k]),
                                 static_cast<cplx*>(o->site[k]), U->bond(0, k), u->phys[k], U->bond(0, k + 1),
                                 V->bond(0, k), V->bond(0, k + 1), B, U->cap[k], V->cap[k], cap[k], ctx->stream));
      ++ctx->launches;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    *out = guard.release();
  });
}

ttg_status ttg_simplify(ttg_ctx* ctx, const ttg_dmps* target, const ttg_strategy* strategy, const ttg_dmps* guess,
                        ttg_dmps** out, ttg_report* reports) {
  return guarded(ctx, [&] {
    check_strategy(strategy);
    if (strategy->method == TTG_SVD_TRUNCATE)  // simplify.hpp:184-187
      dispatch_simplify(ctx, target, nullptr, *strategy, false, 0, out, reports);
    else
      dispatch_simplify(ctx, target, guess, *strategy, true, 0, out, reports);
  });
}

ttg_status ttg_apply(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* v, const ttg_strategy* strategy, ttg_dmps** out,
                     ttg_report* reports) {
  ttg_dmps* raw = nullptr;
  ttg_status st = ttg_apply_raw(ctx, op, v, &raw);
  if (st != TTG_OK) return st;
  st = ttg_simplify(ctx, raw, strategy, nullptr, out, reports);
  ttg_mps_free(raw);
  return st;
}

ttg_status ttg_canonicalize(ttg_ctx* ctx, const ttg_dmps* v, int center, const ttg_strategy* strategy, ttg_dmps** out,
                            ttg_report* reports) {
  return guarded(ctx, [&] {
    check_strategy(strategy);
    if (!v) throw Error{TTG_INVALID, "null argument"};
    if (center < 0 || center >= v->n) throw Error{TTG_SHAPE, "canonical center out of range"};  // mps.hpp:190-191
    dispatch_simplify(ctx, v, nullptr, *strategy, false, center, out, reports);
  });
}

// MPSSum::join (mps.hpp:352-405).  sum_single: for a one-site chain the terms are
// added into one 1 x d x 1 tensor (the L == 1 branch of CompressionEngine::sweep,
// simplify.hpp:62-70) instead of being rejected.
static ttg_dmps* join_states(ttg_ctx* ctx, int nterms, const double* w_re, const double* w_im,
                             const ttg_dmps* const* states, bool sum_single) {
    if (nterms < 1 || !w_re || !states) throw Error{TTG_SHAPE, "MPSSum: weights and states must be non-empty and match"};
    const ttg_dmps* s0 = states[0];
    if (!s0) throw Error{TTG_INVALID, "null state"};
    const int n = s0->n;
    bool cplx_out = false;
    for (int l = 0; l < nterms; ++l) {
      const ttg_dmps* st = states[l];
      if (!st || st->count != 1) throw Error{TTG_INVALID, "join takes single chains"};
      if (st->n != n) throw Error{TTG_SHAPE, "MPSSum: states must share physical dimensions"};
      for (int k = 0; k < n; ++k)
        if (st->phys[k] != s0->phys[k]) throw Error{TTG_SHAPE, "MPSSum: states must share physical dimensions"};
      cplx_out = cplx_out || st->dtype == TTG_C128 || (w_im && w_im[l] != 0.0) ;
    }
    if (n == 1 && nterms > 1 && !sum_single) throw Error{TTG_SHAPE, "MPS boundary bonds must have size one"};
    const int dtype = cplx_out ? TTG_C128 : TTG_F64;
    // MPS::scaled(w) (mps.hpp:98-117): |w|^(1/n) on every site, phase on site 0; w = 0 -> zero_like
    std::vector<double> mag(nterms);
    std::vector<std::vector<int>> bl(nterms, std::vector<int>(n + 1, 1));
    for (int l = 0; l < nterms; ++l) {
      mag[l] = std::hypot(w_re[l], w_im ? w_im[l] : 0.0);
      for (int k = 0; k <= n; ++k) bl[l][k] = mag[l] == 0.0 ? 1 : states[l]->bond(0, k);
    }
    std::vector<int> bonds(n + 1, 0);
    for (int k = 0; k <= n; ++k)
      for (int l = 0; l < nterms; ++l) bonds[k] += bl[l][k];
    bonds[0] = bonds[n] = 1;
    if (nterms == 1 || n == 1) bonds = bl[0];
    std::vector<long long> cap(n);
    for (int k = 0; k < n; ++k) cap[k] = (long long)bonds[k] * s0->phys[k] * bonds[k + 1];
    ttg_dmps* o = new_dmps(n, dtype, 1, s0->phys, cap, ctx->stream);
    std::unique_ptr<ttg_dmps> guard(o);
    for (int k = 0; k <= n; ++k) o->bonds[k] = bonds[k];
    double err = 0.0;
    for (int l = 0; l < nterms; ++l) err += mag[l] * states[l]->error[0];  // MPSSum::error (mps.hpp:344-349)
    o->error[0] = err;
    const size_t es = esize(dtype);
    for (int k = 0; k < n; ++k) {
      CK(cudaMemsetAsync(o->site[k], 0, (size_t)cap[k] * es, ctx->stream));
      int offl = 0, offr = 0;
      for (int l = 0; l < nterms; ++l) {
        const ttg_dmps* st = states[l];
        const int a = bl[l][k], b = bl[l][k + 1], d = s0->phys[k];
        const int ol = (k == 0 || nterms == 1) ? 0 : offl, orr = (k == n - 1 || nterms == 1) ? 0 : offr;
        if (mag[l] != 0.0) {
          const double root = std::pow(mag[l], 1.0 / n);
          double fr = root, fi = 0.0;
          if (k == 0) {
            fr = root * w_re[l] / mag[l];
            fi = root * (w_im ? w_im[l] : 0.0) / mag[l];
          }
          if (dtype == TTG_F64)
            CK((join_block<double, double>(static_cast<const double*>(st->site[k]), a, d, b,
                                          static_cast<double*>(o->site[k]), bonds[k + 1], ol, orr, fr, fi,
                                          ctx->stream)));
          else if (st->dtype == TTG_F64)
            CK((join_block<double, cplx>(static_cast<const double*>(st->site[k]), a, d, b,
                                        static_cast<cplx*>(o->site[k]), bonds[k + 1], ol, orr, fr, fi, ctx->stream)));
          else
            CK((join_block<cplx, cplx>(static_cast<const cplx*>(st->site[k]), a, d, b, static_cast<cplx*>(o->site[k]),
                                      bonds[k + 1], ol, orr, fr, fi, ctx->stream)));
          ++ctx->launches;
        }
        offl += a;
        offr += b;
      }
    }
    return guard.release();
}

ttg_status ttg_mps_join(ttg_ctx* ctx, int nterms, const double* w_re, const double* w_im,
                        const ttg_dmps* const* states, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!out) throw Error{TTG_INVALID, "null argument"};
    *out = join_states(ctx, nterms, w_re, w_im, states, false);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

ttg_status ttg_simplify_sum(ttg_ctx* ctx, int nterms, const double* w_re, const double* w_im,
                            const ttg_dmps* const* states, const ttg_strategy* strategy, const ttg_dmps* guess,
                            ttg_dmps** out, ttg_report* report) {
  return guarded(ctx, [&] {
    check_strategy(strategy);
    if (!out) throw Error{TTG_INVALID, "null argument"};
    if (strategy->method == TTG_SVD_TRUNCATE) {  // simplify.hpp:200-206: canonical form of the joined tensors
      std::unique_ptr<ttg_dmps> joined(join_states(ctx, nterms, w_re, w_im, states, false));
      dispatch_simplify(ctx, joined.get(), nullptr, *strategy, false, 0, out, report);
      return;
    }
    // Variational (simplify.hpp:207-214).  The summand environments of
    // CompressionEngine are the diagonal blocks of the joined target's
    // environments, so the sweep runs on the joined tensors; <T,T> comes from the
    // env chain of the join (= sum_lm conj(w_l) w_m <T_l,T_m>, simplify.hpp:37-41).
    std::unique_ptr<ttg_dmps> joined(join_states(ctx, nterms, w_re, w_im, states, true));
    std::unique_ptr<ttg_dmps> def_guess;
    const ttg_dmps* G = guess;
    if (joined->n == 1) {
      G = nullptr;  // one-site chains: the summed tensor itself (simplify.hpp:62-70)
    } else if (!G) {
      // default_guess (simplify.hpp:132-143): the term with the largest |w_l| |T_l|, scaled by w_l
      int best = 0;
      double best_w = -1.0;
      for (int l = 0; l < nterms; ++l) {
        double re = 0.0, im = 0.0;
        const ttg_status st = ttg_scprod(ctx, states[l], states[l], &re, &im);
        if (st != TTG_OK) throw Error{st, ttg_last_error(ctx)};
        const double w = std::hypot(w_re[l], w_im ? w_im[l] : 0.0) * std::sqrt(std::max(0.0, re));
        if (w > best_w) {
          best_w = w;
          best = l;
        }
      }
      const double wi = w_im ? w_im[best] : 0.0;
      def_guess.reset(join_states(ctx, 1, &w_re[best], &wi, &states[best], false));
      G = def_guess.get();
    }
    dispatch_simplify(ctx, joined.get(), G, *strategy, true, 0, out, report);
  });
}

// blas.hpp:128-138 expectation_mpo(op, u, v): <u, W v>.  The operator
// environment chain of the reference (environments.hpp:42-63) contracts the
// same network as the bra/ket chain over W v with the MPO bond fused into the
// ket bond, so this is the expansion kernel (apply_raw) followed by the DMMA
// environment chain of scprod.  Per chain; v NULL = u.
ttg_status ttg_expectation_mpo(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* u, const ttg_dmps* v, double* out_re,
                               double* out_im) {
  return guarded(ctx, [&] {
    if (!op || !u || !out_re) throw Error{TTG_INVALID, "null argument"};
    const ttg_dmps* ket = v ? v : u;
    if (op->n != u->n || ket->n != u->n) throw Error{TTG_SHAPE, "expectation_mpo: size mismatch"};
    ttg_dmps* raw = nullptr;
    ttg_status st = ttg_apply_raw(ctx, op, ket, &raw);
    if (st != TTG_OK) throw Error{st, ttg_last_error(ctx)};
    std::unique_ptr<ttg_dmps> guard(raw);
    st = ttg_scprod(ctx, u, raw, out_re, out_im);
    if (st != TTG_OK) throw Error{st, ttg_last_error(ctx)};
  });
}

ttg_status ttg_scprod(ttg_ctx* ctx, const ttg_dmps* u, const ttg_dmps* v, double* out_re, double* out_im) {
  return guarded(ctx, [&] {
    if (!u || !v || !out_re) throw Error{TTG_INVALID, "null argument"};
    if (u->n != v->n) throw Error{TTG_SHAPE, "scprod: states of different length"};  // mps.hpp:417-418
    if (u->count != v->count) throw Error{TTG_SHAPE, "scprod: batch sizes differ"};
    for (int k = 0; k < u->n; ++k)
      if (u->phys[k] != v->phys[k]) throw Error{TTG_SHAPE, "scprod: physical dimensions differ"};
    if (!u->uniform() || !v->uniform()) throw Error{TTG_SHAPE, "scprod on a batch needs identical shapes"};
    const int dtype = (u->dtype == TTG_C128 || v->dtype == TTG_C128) ? TTG_C128 : TTG_F64;
    std::unique_ptr<ttg_dmps> uc, vc;
    const ttg_dmps* U = u;
    const ttg_dmps* V = v;
    if (dtype == TTG_C128 && u->dtype == TTG_F64) {
      uc.reset(to_complex(ctx, *u));
      U = uc.get();
    }
    if (dtype == TTG_C128 && v->dtype == TTG_F64) {
      vc.reset(to_complex(ctx, *v));
      V = vc.get();
    }
    const int n = u->n, B = u->count;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      Engine<T> E(ctx, n, B);
      E.ld = n + 1;
      DevBuf bb((size_t)B * (n + 1) * sizeof(int), ctx->stream);
      E.d_bonds = bb.as<int>();
      E.bound.assign(n + 1, 1);
      long long ecap = 1, xcap = 1;
      for (int k = 0; k <= n; ++k) ecap = std::max(ecap, (long long)U->bond(0, k) * V->bond(0, k));
      for (int k = 0; k < n; ++k) xcap = std::max(xcap, (long long)U->bond(0, k) * v->phys[k] * V->bond(0, k + 1));
      const size_t es = sizeof(T);
      DevBuf e0((size_t)B * ecap * es, ctx->stream), e1((size_t)B * ecap * es, ctx->stream),
          xb((size_t)B * xcap * es, ctx->stream);
      CK(fill_one<T>(e0.as<T>(), ecap, B, ctx->stream));
      ++ctx->launches;
      T* eb[2] = {e0.as<T>(), e1.as<T>()};
      for (int k = 0; k < n; ++k) {
        const int pu = U->bond(0, k), pv = V->bond(0, k), pu1 = U->bond(0, k + 1), pv1 = V->bond(0, k + 1);
        const int dk = v->phys[k];
        E.G(eb[k & 1], ecap, V->site[k], V->cap[k], xb.p, xcap, dconst(pu), dconst(dk * pv1), dconst(pv), OP_N, OP_N,
            false);
        E.G(U->site[k], U->cap[k], xb.p, xcap, eb[(k + 1) & 1], ecap, dconst(pu1), dconst(pv1), dconst(pu * dk),
            OP_C, OP_N, false);
      }
      std::vector<T> h((size_t)B * ecap);
      CK(cudaMemcpyAsync(h.data(), eb[n & 1], h.size() * es, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      for (int c = 0; c < B; ++c) {
        if constexpr (std::is_same<T, double>::value) {
          out_re[c] = h[(size_t)c * ecap];
          if (out_im) out_im[c] = 0.0;
        } else {
          out_re[c] = h[(size_t)c * ecap].x;
          if (out_im) out_im[c] = h[(size_t)c * ecap].y;
        }
      }
    };
    if (dtype == TTG_F64)
      run(double{});
    else
      run(cplx{});
  });
}

// ---------------------------------------------------------------------------
// TTLAB1 container on the device boundary (serialize.hpp:13-121): magic
// "TTLAB1\0", u32 version 1, u32 tensor count, per tensor u8 rank + u64 dims
// + complex128 row-major payload; MPS files end with the f64 error bound.
// Payloads stream through two pinned 32 MB buffers straight into (out of)
// the device allocations, so a file is read once and crosses PCIe once.
// ---------------------------------------------------------------------------

}  // extern "C"

namespace {

constexpr size_t TTLAB_STAGE = size_t(32) << 20;
const char TTLAB_MAGIC[7] = {'T', 'T', 'L', 'A', 'B', '1', '\0'};

struct File {
  FILE* f = nullptr;
  long long remaining = 0;  // bytes left to read (read mode)
  File(const char* path, bool write) {
    if (!path) throw Error{TTG_INVALID, "null path"};
    f = std::fopen(path, write ? "wb" : "rb");
    if (!f)
      throw Error{TTG_NUMERIC, std::string(write ? "cannot open file for writing: " : "cannot open file for reading: ") +
                                   path};
    if (!write) {
      std::fseek(f, 0, SEEK_END);
      remaining = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
    }
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void read(void* p, size_t n) {
    if ((long long)n > remaining || std::fread(p, 1, n, f) != n)
      throw Error{TTG_NUMERIC, "ttlab container: truncated file"};
    remaining -= (long long)n;
  }
  template <typename T> T pod() {
    T v;
    read(&v, sizeof(T));
    return v;
  }
  void write(const void* p, size_t n) {
    if (std::fwrite(p, 1, n, f) != n) throw Error{TTG_NUMERIC, "ttlab container: write failed"};
  }
  template <typename T> void put(T v) { write(&v, sizeof(T)); }
  void close() {
    if (f && std::fclose(f) != 0) {
      f = nullptr;
      throw Error{TTG_NUMERIC, "ttlab container: write failed"};
    }
    f = nullptr;
  }
};

void stage_init(ttg_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (!ctx->stage[i]) CK(cudaMallocHost(&ctx->stage[i], TTLAB_STAGE));
    if (!ctx->stage_ev[i]) CK(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
  }
}

// file -> device, double-buffered: the read of chunk k+1 overlaps the copy of chunk k
void stream_in(ttg_ctx* ctx, File& fl, void* dst, size_t bytes, int& cur) {
  for (size_t off = 0; off < bytes; off += TTLAB_STAGE) {
    const size_t n = std::min(TTLAB_STAGE, bytes - off);
    CK(cudaEventSynchronize(ctx->stage_ev[cur]));
    fl.read(ctx->stage[cur], n);
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->stage[cur], n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->stage_ev[cur], ctx->stream));
    cur ^= 1;
  }
}

// device -> file: the copy of chunk k+1 is in flight while chunk k is written
void stream_out(ttg_ctx* ctx, File& fl, const void* src, size_t bytes) {
  if (bytes == 0) return;
  const size_t chunks = (bytes + TTLAB_STAGE - 1) / TTLAB_STAGE;
  auto issue = [&](size_t k) {
    const size_t off = k * TTLAB_STAGE, n = std::min(TTLAB_STAGE, bytes - off);
    CK(cudaMemcpyAsync(ctx->stage[k & 1], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(ctx->stage_ev[k & 1], ctx->stream));
  };
  issue(0);
  for (size_t k = 0; k < chunks; ++k) {
    if (k + 1 < chunks) issue(k + 1);
    CK(cudaEventSynchronize(ctx->stage_ev[k & 1]));
    fl.write(ctx->stage[k & 1], std::min(TTLAB_STAGE, bytes - k * TTLAB_STAGE));
  }
}

uint32_t read_header(File& fl) {
  char magic[7];
  fl.read(magic, sizeof(magic));
  if (std::memcmp(magic, TTLAB_MAGIC, sizeof(magic)) != 0) throw Error{TTG_NUMERIC, "ttlab container: bad magic"};
  if (fl.pod<uint32_t>() != 1u) throw Error{TTG_NUMERIC, "ttlab container: unsupported version"};
  return fl.pod<uint32_t>();
}

void write_header(File& fl, uint32_t count) {
  fl.write(TTLAB_MAGIC, sizeof(TTLAB_MAGIC));
  fl.put<uint32_t>(1u);
  fl.put<uint32_t>(count);
}

// dims of one tensor record, validated against the bytes left in the file
std::vector<long long> read_dims(File& fl, int rank) {
  if (fl.pod<uint8_t>() != rank)
    throw Error{TTG_NUMERIC, rank == 3 ? "ttlab container: expected rank-3 tensor"
                                       : "ttlab container: expected rank-4 tensor"};
  std::vector<long long> d(rank);
  long long elems = 1;
  for (int i = 0; i < rank; ++i) {
    const uint64_t x = fl.pod<uint64_t>();
    if (x < 1) throw Error{TTG_SHAPE, rank == 3 ? "Tensor3 dimensions must be >= 1" : "Tensor4 dimensions must be >= 1"};
    if (x > (uint64_t)fl.remaining || (elems *= (long long)x) > fl.remaining / 16)
      throw Error{TTG_NUMERIC, "ttlab container: truncated file"};
    d[i] = (long long)x;
  }
  return d;
}

// complex128 sites -> float64 when every imaginary part is zero (types.hpp:12-16: the
// reference promotes real data to complex; the real device path gives the same
// gauge-invariant results at a quarter of the arithmetic)
bool all_real(ttg_ctx* ctx, const std::vector<void*>& sites, const std::vector<long long>& elems) {
  DevBuf flag(sizeof(int), ctx->stream);
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  for (size_t k = 0; k < sites.size(); ++k) {
    CK(any_imag(static_cast<const cplx*>(sites[k]), elems[k], flag.as<int>(), ctx->stream));
    ++ctx->launches;
  }
  int h = 0;
  CK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}

void* demote_site(ttg_ctx* ctx, void* site, long long elems) {
  void* r = dev_alloc((size_t)elems * sizeof(double), ctx->stream);
  CK(complex_to_real(static_cast<const cplx*>(site), static_cast<double*>(r), elems, ctx->stream));
  ++ctx->launches;
  cudaFreeAsync(site, ctx->stream);
  return r;
}

}  // namespace

extern "C" {

ttg_status ttg_mps_load(ttg_ctx* ctx, const char* path, int real_if_possible, ttg_dmps** out) {
  return guarded(ctx, [&] {
    if (!out) throw Error{TTG_INVALID, "null argument"};
    File fl(path, false);
    const uint32_t count = read_header(fl);
    stage_init(ctx);
    std::vector<int> bonds{1}, phys;
    std::vector<long long> cap;
    auto* m = new ttg_dmps();
    std::unique_ptr<ttg_dmps> guard(m);
    m->dtype = TTG_C128;
    m->count = 1;
    m->stream = ctx->stream;
    int cur = 0;
    for (uint32_t k = 0; k < count; ++k) {
      const auto d = read_dims(fl, 3);
      if (k == 0) bonds[0] = (int)d[0];
      if (k > 0 && d[0] != bonds.back()) throw Error{TTG_SHAPE, "MPS bond mismatch between neighboring tensors"};
      if (d[0] > INT32_MAX || d[1] > INT32_MAX || d[2] > INT32_MAX) throw Error{TTG_CAPACITY, "tensor dimension too large"};
      bonds.push_back((int)d[2]);
      phys.push_back((int)d[1]);
      cap.push_back(d[0] * d[1] * d[2]);
      m->site.push_back(dev_alloc((size_t)cap.back() * sizeof(cplx), ctx->stream));
      stream_in(ctx, fl, m->site.back(), (size_t)cap.back() * sizeof(cplx), cur);
    }
    const double error = fl.pod<double>();
    if (count > 0 && (bonds.front() != 1 || bonds.back() != 1))  // mps.hpp:129-133
      throw Error{TTG_SHAPE, "MPS boundary bonds must have size one"};
    if (error < 0) throw Error{TTG_SHAPE, "MPS error bound must be non-negative"};
    m->n = (int)count;
    m->phys = phys;
    m->cap = cap;
    m->bonds = bonds;
    m->error.assign(1, error);
    CK(cudaStreamSynchronize(ctx->stream));
    if (real_if_possible && count > 0 && all_real(ctx, m->site, cap)) {
      for (uint32_t k = 0; k < count; ++k) m->site[k] = demote_site(ctx, m->site[k], cap[k]);
      m->dtype = TTG_F64;
      CK(cudaStreamSynchronize(ctx->stream));
    }
    *out = guard.release();
  });
}

ttg_status ttg_mps_save(ttg_ctx* ctx, const ttg_dmps* m, int chain, const char* path) {
  return guarded(ctx, [&] {
    if (!m) throw Error{TTG_INVALID, "null argument"};
    if (chain < 0 || chain >= m->count) throw Error{TTG_INVALID, "chain index out of range"};
    File fl(path, true);
    stage_init(ctx);
    write_header(fl, (uint32_t)m->n);
    long long maxe = 0;
    for (int k = 0; k < m->n; ++k) maxe = std::max(maxe, (long long)m->bond(chain, k) * m->phys[k] * m->bond(chain, k + 1));
    std::unique_ptr<DevBuf> promo;
    if (m->dtype == TTG_F64) promo.reset(new DevBuf((size_t)std::max(1LL, maxe) * sizeof(cplx), ctx->stream));
    for (int k = 0; k < m->n; ++k) {
      const long long a = m->bond(chain, k), d = m->phys[k], b = m->bond(chain, k + 1), e = a * d * b;
      fl.put<uint8_t>(3);
      fl.put<uint64_t>((uint64_t)a);
      fl.put<uint64_t>((uint64_t)d);
      fl.put<uint64_t>((uint64_t)b);
      const char* src = static_cast<const char*>(m->site[k]) + (size_t)chain * m->cap[k] * esize(m->dtype);
      if (m->dtype == TTG_F64) {
        CK(real_to_complex(reinterpret_cast<const double*>(src), promo->as<cplx>(), e, ctx->stream));
        ++ctx->launches;
        src = static_cast<const char*>(promo->p);
      }
      stream_out(ctx, fl, src, (size_t)e * sizeof(cplx));
    }
    fl.put<double>(m->error[chain]);
    fl.close();
  });
}

ttg_status ttg_mpo_load(ttg_ctx* ctx, const char* path, int real_if_possible, ttg_dmpo** out) {
  return guarded(ctx, [&] {
    if (!out) throw Error{TTG_INVALID, "null argument"};
    File fl(path, false);
    const uint32_t count = read_header(fl);
    stage_init(ctx);
    auto* w = new ttg_dmpo();
    std::unique_ptr<ttg_dmpo> guard(w);
    w->dtype = TTG_C128;
    w->stream = ctx->stream;
    w->bonds.push_back(1);
    std::vector<long long> elems;
    int cur = 0;
    for (uint32_t k = 0; k < count; ++k) {
      const auto d = read_dims(fl, 4);
      if (k == 0) w->bonds[0] = (int)d[0];
      if (k > 0 && d[0] != w->bonds.back()) throw Error{TTG_SHAPE, "MPO bond mismatch between neighboring tensors"};
      for (long long x : d)
        if (x > INT32_MAX) throw Error{TTG_CAPACITY, "tensor dimension too large"};
      w->dout.push_back((int)d[1]);
      w->din.push_back((int)d[2]);
      w->bonds.push_back((int)d[3]);
      elems.push_back(d[0] * d[1] * d[2] * d[3]);
      w->site.push_back(dev_alloc((size_t)elems.back() * sizeof(cplx), ctx->stream));
      stream_in(ctx, fl, w->site.back(), (size_t)elems.back() * sizeof(cplx), cur);
    }
    if (count > 0 && (w->bonds.front() != 1 || w->bonds.back() != 1))
      throw Error{TTG_SHAPE, "MPO boundary bonds must have size one"};
    w->n = (int)count;
    CK(cudaStreamSynchronize(ctx->stream));
    if (real_if_possible && count > 0 && all_real(ctx, w->site, elems)) {
      for (uint32_t k = 0; k < count; ++k) w->site[k] = demote_site(ctx, w->site[k], elems[k]);
      w->dtype = TTG_F64;
      CK(cudaStreamSynchronize(ctx->stream));
    }
    *out = guard.release();
  });
}

ttg_status ttg_mpo_save(ttg_ctx* ctx, const ttg_dmpo* w, const char* path) {
  return guarded(ctx, [&] {
    if (!w) throw Error{TTG_INVALID, "null argument"};
    File fl(path, true);
    stage_init(ctx);
    write_header(fl, (uint32_t)w->n);
    for (int k = 0; k < w->n; ++k) {
      const long long e = (long long)w->bonds[k] * w->dout[k] * w->din[k] * w->bonds[k + 1];
      fl.put<uint8_t>(4);
      fl.put<uint64_t>((uint64_t)w->bonds[k]);
      fl.put<uint64_t>((uint64_t)w->dout[k]);
      fl.put<uint64_t>((uint64_t)w->din[k]);
      fl.put<uint64_t>((uint64_t)w->bonds[k + 1]);
      std::unique_ptr<DevBuf> promo;
      const void* src = w->site[k];
      if (w->dtype == TTG_F64) {
        promo.reset(new DevBuf((size_t)e * sizeof(cplx), ctx->stream));
        CK(real_to_complex(static_cast<const double*>(src), promo->as<cplx>(), e, ctx->stream));
        ++ctx->launches;
        src = promo->p;
      }
      stream_out(ctx, fl, src, (size_t)e * sizeof(cplx));
    }
    fl.close();
  });
}

}  // extern "C"


// ---------------------------------------------------------------------------
// Two-site effective operator matvec (eigensolvers.hpp:15-64, apply_effective_two_site):
//   y[a', s1', s2', b'] = sum L[c0](a', a) W1[c0, s1', s1, c1] W2[c1, s2', s2, c2] R[c2](b', B)
//                         x[a, s1, s2, B]
// B200 form: one DMMA GEMM for the left environment over all c0 at once (L stacked
// (D0 chiAo) x chiA), one memory-bound kernel that contracts both MPO sites together
// (the MPO entries live in shared memory, outputs written along B so loads and stores
// coalesce), then D2 accumulating DMMA GEMMs against R[c2]^T.
// ---------------------------------------------------------------------------
namespace ttg {
namespace {
// Both MPO sites at once: V[a'][s1'][s2'][c2][B] = sum_{c0,s1,s2} W12[c0,s1',s1,s2',s2,c2] XL[c0][a'][s1][s2][B]
// with W12 = sum_{c1} W1[c0,s1',s1,c1] W2[c1,s2',s2,c2] formed once per CTA in shared memory.  One thread
// per (a', B) reads its D0 d1 d2 values of XL once (coalesced over B) and writes all d1o d2o D2 outputs,
// so XL is read once and V written once (memory-bound).
template <typename T>
__global__ void heff_mix_kernel(const T* XL, const T* W1, const T* W2, T* V, int D0, int D1, int D2, int d1o, int d1,
                                int d2o, int d2, int chiAo, int chiB) {
  extern __shared__ __align__(16) unsigned char heff_smem[];
  T* w12 = reinterpret_cast<T*>(heff_smem);  // [c0][s1o][s1][s2o][s2][c2]
  const int n12 = D0 * d1o * d1 * d2o * d2 * D2;
  for (int i = threadIdx.x; i < n12; i += blockDim.x) {
    int t = i;
    const int c2 = t % D2;
    t /= D2;
    const int s2 = t % d2;
    t /= d2;
    const int s2o = t % d2o;
    t /= d2o;
    const int s1 = t % d1;
    t /= d1;
    const int s1o = t % d1o;
    const int c0 = t / d1o;
    T acc = Scalar<T>::zero();
    for (int c1 = 0; c1 < D1; ++c1)
      acc = add(acc, mul(W1[((c0 * d1o + s1o) * d1 + s1) * D1 + c1], W2[((c1 * d2o + s2o) * d2 + s2) * D2 + c2]));
    w12[i] = acc;
  }
  __syncthreads();
  const int nin = D0 * d1 * d2;
  const long long total = (long long)chiAo * chiB;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int B = (int)(idx % chiB), a = (int)(idx / chiB);
    for (int s1o = 0; s1o < d1o; ++s1o)
      for (int s2o = 0; s2o < d2o; ++s2o)
        for (int c2 = 0; c2 < D2; ++c2) {
          T acc = Scalar<T>::zero();
          for (int c0 = 0; c0 < D0; ++c0)
            for (int s1 = 0; s1 < d1; ++s1)
              for (int s2 = 0; s2 < d2; ++s2) {
                const T x = XL[((((size_t)c0 * chiAo + a) * d1 + s1) * d2 + s2) * chiB + B];
                acc = add(acc, mul(w12[((((c0 * d1o + s1o) * d1 + s1) * d2o + s2o) * d2 + s2) * D2 + c2], x));
              }
          V[((((size_t)a * d1o + s1o) * d2o + s2o) * D2 + c2) * chiB + B] = acc;
        }
    (void)nin;
  }
}

// y = H_eff x on device buffers (stream-ordered, no host synchronisation).
template <typename T>
void heff_two_site_dev(ttg_ctx* ctx, const int* dm, const void* L, const void* W1, const void* W2, const void* R,
                       const void* x, void* y) {
  const int D0 = dm[0], D1 = dm[1], D2 = dm[2], d1o = dm[3], d1 = dm[4], d2o = dm[5], d2 = dm[6];
  const int chiAo = dm[7], chiA = dm[8], chiBo = dm[9], chiB = dm[10];
  cudaStream_t st = ctx->stream;
  const size_t es = sizeof(T);
  const size_t nW1 = (size_t)D0 * d1o * d1 * D1, nW2 = (size_t)D1 * d2o * d2 * D2;
  const size_t nXL = (size_t)D0 * chiAo * d1 * d2 * chiB, nV = (size_t)chiAo * d1o * d2o * D2 * chiB;
  DevBuf XL(nXL * es, st), V(nV * es, st);
  // XL = [L[0]; ...; L[D0-1]] x  ((D0 chiAo) x chiA times chiA x (d1 d2 chiB))
  const int M1 = D0 * chiAo, N1 = d1 * d2 * chiB;
  GemmParams g1{L, x, XL.p, 0, 0, 0, dconst(M1), dconst(N1), dconst(chiA), nullptr, 0, nullptr, 1.0, 0};
  {
    ProfScope ps(ctx, TTG_PROF_GEMM, (Scalar<T>::is_complex ? 8.0 : 2.0) * M1 * (double)N1 * chiA);
    CK(gemm<T>(g1, OP_N, OP_N, M1, N1, 1, st, chiA));
  }
  const size_t smem = (size_t)D0 * d1o * d1 * d2o * d2 * D2 * es;  // fused W12
  // the fused pair W12 lives in shared memory: up to 200 KB (e.g. D = 8 with d = 4 on both sites: 8 * 16 * 16 * 8
  // complex values = 256 KB does not fit; D = 4, d = 4: 64 KB does)
  if (smem > 200 * 1024) throw Error{TTG_CAPACITY, "apply_effective_two_site: MPO sites too large"};
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(heff_mix_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  (void)nW1;
  (void)nW2;
  const long long tot = (long long)chiAo * chiB;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(148 * 8, (tot + 255) / 256));
  {
    ProfScope ps(ctx, TTG_PROF_EXPAND);
    heff_mix_kernel<T><<<blocks, 256, smem, st>>>(static_cast<const T*>(XL.p), static_cast<const T*>(W1),
                                                   static_cast<const T*>(W2), static_cast<T*>(V.p), D0, D1, D2, d1o,
                                                   d1, d2o, d2, chiAo, chiB);
    CK(cudaGetLastError());
  }
  // y += V[:, c2, :] R[c2]^T for every c2  ((chiAo d1o d2o) x chiB times chiB x chiBo)
  const int M3 = chiAo * d1o * d2o;
  for (int c2 = 0; c2 < D2; ++c2) {
    GemmParams g3{static_cast<const T*>(V.p) + (size_t)c2 * chiB, static_cast<const T*>(R) + (size_t)c2 * chiBo * chiB,
                  y, 0, 0, 0, dconst(M3), dconst(chiBo), dconst(chiB), nullptr, 0, nullptr, 1.0, c2 > 0 ? 1 : 0};
    g3.lda = (long long)D2 * chiB;
    g3.ldb = chiB;
    g3.ldc = chiBo;
    ProfScope ps(ctx, TTG_PROF_GEMM, (Scalar<T>::is_complex ? 8.0 : 2.0) * M3 * (double)chiBo * chiB);
    CK(gemm<T>(g3, OP_N, OP_T, M3, chiBo, 1, st, chiB));
  }
  ctx->launches += 2 + D2;
}

template <typename T>
void heff_two_site(ttg_ctx* ctx, const int* dm, const void* hL, const void* hW1, const void* hW2, const void* hR,
                   const void* hx, void* hy) {
  const int D0 = dm[0], D1 = dm[1], D2 = dm[2], d1o = dm[3], d1 = dm[4], d2o = dm[5], d2 = dm[6];
  const int chiAo = dm[7], chiA = dm[8], chiBo = dm[9], chiB = dm[10];
  cudaStream_t st = ctx->stream;
  const size_t es = sizeof(T);
  const size_t nL = (size_t)D0 * chiAo * chiA, nW1 = (size_t)D0 * d1o * d1 * D1, nW2 = (size_t)D1 * d2o * d2 * D2;
  const size_t nR = (size_t)D2 * chiBo * chiB, nx = (size_t)chiA * d1 * d2 * chiB;
  const size_t ny = (size_t)chiAo * d1o * d2o * chiBo;
  DevBuf L(nL * es, st), W1(nW1 * es, st), W2(nW2 * es, st), R(nR * es, st), X(nx * es, st), Y(ny * es, st);
  CK(cudaMemcpyAsync(L.p, hL, nL * es, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(W1.p, hW1, nW1 * es, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(W2.p, hW2, nW2 * es, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(R.p, hR, nR * es, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(X.p, hx, nx * es, cudaMemcpyHostToDevice, st));
  heff_two_site_dev<T>(ctx, dm, L.p, W1.p, W2.p, R.p, X.p, Y.p);
  CK(cudaMemcpyAsync(hy, Y.p, ny * es, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

// Operator-environment mixing (memory-bound, W in shared memory).
// left:  Y[c'][a][s'][b'] = sum_{c,s} W[c,s',s,c'] X[c][a][s][b']          (X: D x P x d x Q)
// right: Y[c][s'][a'][b] = sum_{c',s} W[c,s',s,c'] Z[c'][a'][b][s]          (Z: D' x P x Q x d)
template <typename T, bool LEFT>
__global__ void openv_mix_kernel(const T* X, const T* W, T* Y, int Dl, int dout, int din, int Dr, int P, int Q) {
  extern __shared__ __align__(16) unsigned char openv_smem[];
  T* w = reinterpret_cast<T*>(openv_smem);
  const int nw = Dl * dout * din * Dr;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) w[i] = W[i];
  __syncthreads();
  const int Dout = LEFT ? Dr : Dl, Din = LEFT ? Dl : Dr;
  const long long total = (long long)Dout * P * dout * Q;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    int co, p, sp, q;
    if constexpr (LEFT) {  // idx = ((c' P + a) dout + s') Q + b'
      q = (int)(t % Q);
      t /= Q;
      sp = (int)(t % dout);
      t /= dout;
      p = (int)(t % P);
      co = (int)(t / P);
    } else {  // idx = ((c dout + s') P + a') Q + b
      q = (int)(t % Q);
      t /= Q;
      p = (int)(t % P);
      t /= P;
      sp = (int)(t % dout);
      co = (int)(t / dout);
    }
    T acc = Scalar<T>::zero();
    for (int ci = 0; ci < Din; ++ci)
      for (int s = 0; s < din; ++s) {
        const int c = LEFT ? ci : co, cp = LEFT ? co : ci;
        const T wv = w[((c * dout + sp) * din + s) * Dr + cp];
        const T xv = LEFT ? X[(((long long)ci * P + p) * din + s) * Q + q] : X[(((long long)ci * P + p) * Q + q) * din + s];
        acc = add(acc, mul(wv, xv));
      }
    Y[idx] = acc;
  }
}

// update_left_op_environment / update_right_op_environment (environments.hpp:42-83) on device
// buffers.  dims = {Dl, dout, din, Dr, bra_l, bra_r, ket_l, ket_r}; env / out are stacked
// matrices E[c](a, b) as [c][a][b] (left: env over Dl with a, b = bra_l, ket_l; out over Dr with
// bra_r, ket_r.  right: env over Dr with bra_r, ket_r; out over Dl with bra_l, ket_l).
template <typename T>
void openv_update(ttg_ctx* ctx, bool left, const int* dm, const void* env, const void* bra, const void* op,
                  const void* ket, void* out) {
  const int Dl = dm[0], dout = dm[1], din = dm[2], Dr = dm[3], al = dm[4], ar = dm[5], bl = dm[6], br = dm[7];
  cudaStream_t st = ctx->stream;
  const size_t es = sizeof(T);
  const double fm = Scalar<T>::is_complex ? 8.0 : 2.0;
  const size_t smem = (size_t)Dl * dout * din * Dr * es;
  if (smem > 48 * 1024) throw Error{TTG_CAPACITY, "op environment: MPO site too large"};
  if (left) {
    // X[c][a][s][b'] = E[c](a, b) B[b, s, b']: (Dl al) x bl times bl x (din br)
    DevBuf X((size_t)Dl * al * din * br * es, st), Y((size_t)Dr * al * dout * br * es, st);
    GemmParams g1{env, ket, X.p, 0, 0, 0, dconst(Dl * al), dconst(din * br), dconst(bl), nullptr, 0, nullptr, 1.0, 0};
    {
      ProfScope ps(ctx, TTG_PROF_GEMM, fm * Dl * al * (double)din * br * bl);
      CK(gemm<T>(g1, OP_N, OP_N, Dl * al, din * br, 1, st, bl));
    }
    const long long tot = (long long)Dr * al * dout * br;
    openv_mix_kernel<T, true><<<(int)std::max<long long>(1, std::min<long long>(148 * 8, (tot + 255) / 256)), 256,
                                smem, st>>>(static_cast<const T*>(X.p), static_cast<const T*>(op), Y.as<T>(), Dl, dout,
                                            din, Dr, al, br);
    CK(cudaGetLastError());
    // out[c'] = A^H (ar x (al dout)) Y[c'] ((al dout) x br), batched over c'
    GemmParams g3{bra, Y.p, out, 0, (long long)al * dout * br, (long long)ar * br, dconst(ar), dconst(br),
                  dconst(al * dout), nullptr, 0, nullptr, 1.0, 0};
    ProfScope ps(ctx, TTG_PROF_GEMM, fm * Dr * (double)ar * br * al * dout);
    CK(gemm<T>(g3, OP_C, OP_N, ar, br, Dr, st, al * dout));
  } else {
    // Z[c'][a'][b][s] = E[c'](a', b') B[b, s, b']: (Dr ar) x br times (bl din x br)^T
    DevBuf Z((size_t)Dr * ar * bl * din * es, st), Y((size_t)Dl * dout * ar * bl * es, st);
    GemmParams g1{env, ket, Z.p, 0, 0, 0, dconst(Dr * ar), dconst(bl * din), dconst(br), nullptr, 0, nullptr, 1.0, 0};
    {
      ProfScope ps(ctx, TTG_PROF_GEMM, fm * Dr * ar * (double)bl * din * br);
      CK(gemm<T>(g1, OP_N, OP_T, Dr * ar, bl * din, 1, st, br));
    }
    const long long tot = (long long)Dl * dout * ar * bl;
    openv_mix_kernel<T, false><<<(int)std::max<long long>(1, std::min<long long>(148 * 8, (tot + 255) / 256)), 256,
                                 smem, st>>>(static_cast<const T*>(Z.p), static_cast<const T*>(op), Y.as<T>(), Dl, dout,
                                             din, Dr, ar, bl);
    CK(cudaGetLastError());
    // out[c] = conj(A) (al x (dout ar)) Y[c] ((dout ar) x bl), batched over c
    GemmParams g3{bra, Y.p, out, 0, (long long)dout * ar * bl, (long long)al * bl, dconst(al), dconst(bl),
                  dconst(dout * ar), nullptr, 0, nullptr, 1.0, 0};
    ProfScope ps(ctx, TTG_PROF_GEMM, fm * Dl * (double)al * bl * dout * ar);
    CK(gemm<T>(g3, OP_R, OP_N, al, bl, Dl, st, dout * ar));
  }
  ctx->launches += 3;
}
}  // namespace
}  // namespace ttg

ttg_status ttg_apply_effective_two_site_dev(ttg_ctx* ctx, int dtype, const int* dims, const void* L, const void* W1,
                                            const void* W2, const void* R, const void* x, void* y) {
  return guarded(ctx, [&] {
    if (!dims || !L || !W1 || !W2 || !R || !x || !y) throw Error{TTG_INVALID, "null argument"};
    for (int i = 0; i < 11; ++i)
      if (dims[i] <= 0) throw Error{TTG_SHAPE, "apply_effective_two_site: bad dimension"};
    CK(cudaSetDevice(ctx->device));
    if (dtype == TTG_C128)
      ttg::heff_two_site_dev<ttg::cplx>(ctx, dims, L, W1, W2, R, x, y);
    else if (dtype == TTG_F64)
      ttg::heff_two_site_dev<double>(ctx, dims, L, W1, W2, R, x, y);
    else
      throw Error{TTG_INVALID, "apply_effective_two_site: dtype"};
  });
}

ttg_status ttg_op_env_update(ttg_ctx* ctx, int dtype, int side, const int* dims, const void* env, const void* bra,
                             const void* op, const void* ket, void* out) {
  return guarded(ctx, [&] {
    if (!dims || !env || !bra || !op || !ket || !out) throw Error{TTG_INVALID, "null argument"};
    for (int i = 0; i < 8; ++i)
      if (dims[i] <= 0) throw Error{TTG_SHAPE, "op environment: bad dimension"};
    if (side != TTG_LEFT_TO_RIGHT && side != TTG_RIGHT_TO_LEFT) throw Error{TTG_INVALID, "op environment: side"};
    CK(cudaSetDevice(ctx->device));
    const bool left = side == TTG_LEFT_TO_RIGHT;
    if (dtype == TTG_C128)
      ttg::openv_update<ttg::cplx>(ctx, left, dims, env, bra, op, ket, out);
    else if (dtype == TTG_F64)
      ttg::openv_update<double>(ctx, left, dims, env, bra, op, ket, out);
    else
      throw Error{TTG_INVALID, "op environment: dtype"};
  });
}

ttg_status ttg_apply_effective_two_site(ttg_ctx* ctx, int dtype, const int* dims, const void* L, const void* W1,
                                        const void* W2, const void* R, const void* x, void* y) {
  return guarded(ctx, [&] {
    if (!dims || !L || !W1 || !W2 || !R || !x || !y) throw Error{TTG_INVALID, "null argument"};
    for (int i = 0; i < 11; ++i)
      if (dims[i] <= 0) throw Error{TTG_SHAPE, "apply_effective_two_site: bad dimension"};
    CK(cudaSetDevice(ctx->device));
    if (dtype == TTG_C128)
      ttg::heff_two_site<ttg::cplx>(ctx, dims, L, W1, W2, R, x, y);
    else if (dtype == TTG_F64)
      ttg::heff_two_site<double>(ctx, dims, L, W1, W2, R, x, y);
    else
      throw Error{TTG_INVALID, "apply_effective_two_site: dtype"};
  });
}

// ---------------------------------------------------------------------------
// CanonicalMPS centre moves and the truncated split on the device
// (mps.hpp:238-297, schmidt.hpp:72-89)
// ---------------------------------------------------------------------------
namespace {

// Split workspaces for an Engine that runs isolated splits of at most lmax x kmax.
template <typename T>
struct SplitWork {
  DevBuf svdw, svdg, prebuf, svbuf;
  long long svd_work = 0;
  SplitWork(Engine<T>& E, long long lmax, long long kmax, int B, cudaStream_t st) {
    const size_t es = sizeof(T);
    const long long lk = std::max({lmax, kmax, 1LL});
    svd_work = (lk + 1) * (lk + 1);  // any panel orientation outside shared memory
    svdw = DevBuf((size_t)B * svd_work * es, st);
    svdg = DevBuf(B <= 16 ? (size_t)B * jacobi_grid_work_bytes((int)lk, (int)lk, es) : 0, st);
    E.svd_grid_work = B <= 16 ? svdg.p : nullptr;
    E.pre_cap = std::min(lk, 256LL) * std::min(lk, 256LL);
    prebuf = DevBuf((size_t)B * 4 * E.pre_cap * es, st);
    E.pre_buf = prebuf.p;
    E.pre_slot = E.ld - 1;
    svbuf = DevBuf((size_t)B * lk * sizeof(double), st);
    E.svals = svbuf.as<double>();
    E.svals_cap = lk;
  }
};

template <typename T>
int read_bond(Engine<T>& E, int idx) {
  int r = 0;
  CK(cudaMemcpyAsync(&r, E.d_bonds + idx, sizeof(int), cudaMemcpyDeviceToHost, E.st));
  CK(cudaStreamSynchronize(E.st));
  return r;
}

// Move the centre of a canonical single chain from `center` to `target`,
// truncating per strategy (recenter, mps.hpp:268-279, built from
// move_center_right / move_center_left, mps.hpp:238-265).  Returns the
// moved copy and sqrt(sum of the squared dropped weights).
template <typename T>
ttg_dmps* run_recenter(ttg_ctx* ctx, const ttg_dmps& in, int center, int target, const ttg_strategy& s, double* err) {
  const int L = in.n;
  cudaStream_t st = ctx->stream;
  const size_t es = sizeof(T);
  ttg_dmps* o = new_dmps(L, in.dtype, 1, in.phys, in.cap, st);
  std::unique_ptr<ttg_dmps> guard(o);
  o->bonds.assign(in.bonds.begin(), in.bonds.begin() + (L + 1));
  o->error[0] = in.error[0];
  for (int k = 0; k < L; ++k)
    CK(cudaMemcpyAsync(o->site[k], in.site[k], (size_t)in.cap[k] * es, cudaMemcpyDeviceToDevice, st));
  std::vector<int> b(o->bonds.begin(), o->bonds.end());
  Engine<T> E(ctx, L, 1);
  E.ld = L + 3;
  long long lmax = 1, cmax = 1;
  for (int k = 0; k < L; ++k) {
    lmax = std::max({lmax, (long long)b[k] * in.phys[k], (long long)in.phys[k] * b[k + 1]});
    cmax = std::max(cmax, in.cap[k]);
  }
  E.bound.assign(E.ld, (int)lmax);
  DevBuf bonds_buf((size_t)E.ld * sizeof(int), st), state_buf(sizeof(ChainState), st);
  E.d_bonds = bonds_buf.as<int>();
  E.d_state = state_buf.as<ChainState>();
  {
    std::vector<int> hb(E.ld, 1);
    for (int k = 0; k <= L; ++k) hb[k] = b[k];
    CK(cudaMemcpyAsync(E.d_bonds, hb.data(), hb.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(init_state(E.d_state, 1, st));
  SplitWork<T> work(E, lmax, lmax, 1, st);
  DevBuf Th((size_t)cmax * es, st), Bb((size_t)lmax * lmax * es, st), X((size_t)cmax * es, st);
  const int mb = clamp_bond(s.max_bond);
  const double tol = s.tolerance;
  int c = center;
  while (c < target) {  // move_center_right (mps.hpp:238-250): theta = left unfolding of site c
    const int m = b[c] * o->phys[c], n = b[c + 1];
    CK(cudaMemcpyAsync(Th.p, o->site[c], (size_t)m * n * es, cudaMemcpyDeviceToDevice, st));
    E.S(Th.p, 0, dconst(m), dconst(n), c + 1, o->site[c], 0, 0, tol, mb, false, true, work.svdw.p, work.svd_work);
    const int r = read_bond(E, c + 1);
    // S V^H = U_r^H theta (r x n), carried into site c+1 (mps.hpp:246)
    E.G(o->site[c], 0, Th.p, 0, Bb.p, 0, dconst(r), dconst(n), dconst(m), OP_C, OP_N, false);
    const int w = o->phys[c + 1] * b[c + 2];
    E.G(Bb.p, 0, o->site[c + 1], 0, X.p, 0, dconst(r), dconst(w), dconst(n), OP_N, OP_N, false);
    CK(cudaMemcpyAsync(o->site[c + 1], X.p, (size_t)r * w * es, cudaMemcpyDeviceToDevice, st));
    b[c + 1] = r;
    ++c;
  }
  while (c > target) {  // move_center_left (mps.hpp:253-265): theta = right unfolding of site c
    const int m = b[c], n = o->phys[c] * b[c + 1];
    CK(cudaMemcpyAsync(Th.p, o->site[c], (size_t)m * n * es, cudaMemcpyDeviceToDevice, st));
    E.S(Th.p, 0, dconst(m), dconst(n), c, o->site[c], 0, 1, tol, mb, false, true, work.svdw.p, work.svd_work);
    const int r = read_bond(E, c);
    // U S = theta V_r (m x r), carried into site c-1 (mps.hpp:261)
    E.G(Th.p, 0, o->site[c], 0, Bb.p, 0, dconst(m), dconst(r), dconst(n), OP_N, OP_C, false);
    const int h = b[c - 1] * o->phys[c - 1];
    E.G(o->site[c - 1], 0, Bb.p, 0, X.p, 0, dconst(h), dconst(r), dconst(m), OP_N, OP_N, false);
    CK(cudaMemcpyAsync(o->site[c - 1], X.p, (size_t)h * r * es, cudaMemcpyDeviceToDevice, st));
    b[c] = r;
    --c;
  }
  ChainState hs{};
  CK(cudaMemcpyAsync(&hs, E.d_state, sizeof hs, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hs.status & ST_NONFINITE) throw Error{TTG_NUMERIC, "schmidt_split: non-finite input"};
  if (hs.status & ST_NOCONV) throw Error{TTG_NUMERIC, "SVD failed to converge"};
  for (int k = 0; k <= L; ++k) o->bonds[k] = b[k];
  o->center = target;
  if (err) *err = std::sqrt(std::max(0.0, hs.err2));
  return guard.release();
}

// schmidt_split (schmidt.hpp:72-89) of one host matrix on the device.
template <typename T>
void run_schmidt_split(ttg_ctx* ctx, int m, int n, const void* theta, int direction, const ttg_strategy& s, void* a,
                       void* bout, int64_t* rank, double* err) {
  cudaStream_t st = ctx->stream;
  const size_t es = sizeof(T);
  const int kmin = std::min(m, n);
  Engine<T> E(ctx, 1, 1);
  E.ld = 4;
  E.bound.assign(E.ld, std::max(m, n));
  DevBuf bonds_buf((size_t)E.ld * sizeof(int), st), state_buf(sizeof(ChainState), st);
  E.d_bonds = bonds_buf.as<int>();
  E.d_state = state_buf.as<ChainState>();
  CK(cudaMemsetAsync(E.d_bonds, 0, E.ld * sizeof(int), st));
  CK(init_state(E.d_state, 1, st));
  SplitWork<T> work(E, std::max(m, n), std::max(m, n), 1, st);
  DevBuf th((size_t)m * n * es, st), iso((size_t)std::max(m, n) * kmin * es, st), other((size_t)std::max(m, n) * kmin * es, st);
  CK(cudaMemcpyAsync(th.p, theta, (size_t)m * n * es, cudaMemcpyHostToDevice, st));
  const int mode = direction == TTG_RIGHT_TO_LEFT ? 1 : 0;
  E.S(th.p, 0, dconst(m), dconst(n), 0, iso.p, 0, mode, s.tolerance, clamp_bond(s.max_bond), false, true,
      work.svdw.p, work.svd_work);
  const int r = read_bond(E, 0);
  if (mode == 0) {  // a = U_r (m x r), b = S V^H = U_r^H theta (r x n)
    E.G(iso.p, 0, th.p, 0, other.p, 0, dconst(r), dconst(n), dconst(m), OP_C, OP_N, false);
    CK(cudaMemcpyAsync(a, iso.p, (size_t)m * r * es, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(bout, other.p, (size_t)r * n * es, cudaMemcpyDeviceToHost, st));
  } else {  // b = V_r^H (r x n), a = U S = theta V_r (m x r)
    E.G(th.p, 0, iso.p, 0, other.p, 0, dconst(m), dconst(r), dconst(n), OP_N, OP_C, false);
    CK(cudaMemcpyAsync(a, other.p, (size_t)m * r * es, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(bout, iso.p, (size_t)r * n * es, cudaMemcpyDeviceToHost, st));
  }
  ChainState hs{};
  CK(cudaMemcpyAsync(&hs, E.d_state, sizeof hs, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hs.status & ST_NONFINITE) throw Error{TTG_NUMERIC, "schmidt_split: non-finite input"};
  if (hs.status & ST_NOCONV) throw Error{TTG_NUMERIC, "SVD failed to converge"};
  *rank = r;
  if (err) *err = std::sqrt(std::max(0.0, hs.err2));
}

}  // namespace

extern "C" {

ttg_status ttg_recenter(ttg_ctx* ctx, const ttg_dmps* v, int center, int target, const ttg_strategy* strategy,
                        ttg_dmps** out, double* err) {
  return guarded(ctx, [&] {
    check_strategy(strategy);
    if (!v || !out) throw Error{TTG_INVALID, "null argument"};
    if (v->count != 1) throw Error{TTG_SHAPE, "recenter: single chains only"};
    if (center < 0 || center >= v->n) throw Error{TTG_SHAPE, "recenter: center out of range"};
    if (target < 0 || target >= v->n) throw Error{TTG_SHAPE, "recenter: center out of range"};  // mps.hpp:269-270
    if (v->dtype == TTG_F64)
      *out = run_recenter<double>(ctx, *v, center, target, *strategy, err);
    else
      *out = run_recenter<cplx>(ctx, *v, center, target, *strategy, err);
  });
}

ttg_status ttg_schmidt_split(ttg_ctx* ctx, int dtype, int64_t m, int64_t n, const void* theta, int direction,
                             const ttg_strategy* strategy, void* a, void* b, int64_t* rank, double* err) {
  return guarded(ctx, [&] {
    check_strategy(strategy);
    if (!theta || !a || !b || !rank) throw Error{TTG_INVALID, "null argument"};
    if (m < 1 || n < 1 || m > (1 << 30) / std::max<int64_t>(n, 1)) throw Error{TTG_SHAPE, "schmidt_split: bad shape"};
    if (dtype == TTG_F64)
      run_schmidt_split<double>(ctx, (int)m, (int)n, theta, direction, *strategy, a, b, rank, err);
    else if (dtype == TTG_C128)
      run_schmidt_split<cplx>(ctx, (int)m, (int)n, theta, direction, *strategy, a, b, rank, err);
    else
      throw Error{TTG_INVALID, "unknown dtype"};
  });
}

}  // extern "C"
