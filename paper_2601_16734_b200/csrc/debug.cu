// Kernel-level test hooks of the C ABI (host buffers in, host buffers out).
// They run exactly the kernels the engine uses, one call each, so the parity
// tests can pin the GEMM fragment layouts, the QR and the truncated SVD in
// isolation before the sweep engine is involved.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ttgpu.h"
#include "common.cuh"
#include "gemm.cuh"
#include "jacobi_svd.cuh"
#include "qr.cuh"

using namespace ttg;

namespace {

struct Buf {
  void* p = nullptr;
  explicit Buf(size_t bytes) { cudaMalloc(&p, bytes ? bytes : 16); }
  ~Buf() { cudaFree(p); }
};

ttg_status cuda_status(cudaError_t e) { return e == cudaSuccess ? TTG_OK : TTG_CUDA; }

template <typename T>
ttg_status do_gemm(int opA, int opB, int M, int N, int K, const void* A, const void* B, void* Cout, int batch) {
  const size_t es = sizeof(T);
  const size_t na = (size_t)M * K, nb = (size_t)K * N, nc = (size_t)M * N;
  Buf a(na * es * batch), b(nb * es * batch), c(nc * es * batch);
  cudaMemcpy(a.p, A, na * es * batch, cudaMemcpyHostToDevice);
  cudaMemcpy(b.p, B, nb * es * batch, cudaMemcpyHostToDevice);
  GemmParams p{a.p, b.p, c.p, (long long)na, (long long)nb, (long long)nc, dconst(M), dconst(N), dconst(K),
               nullptr, 0, nullptr, 1.0, 0};
  cudaError_t e = gemm<T>(p, opA, opB, M, N, batch, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(Cout, c.p, nc * es * batch, cudaMemcpyDeviceToHost);
  return cuda_status(e);
}

template <typename T>
ttg_status do_svd(int m, int n, const void* theta, int mode, double tol, int64_t max_bond, void* iso, double* svals,
                  int* rank, double* err2, int* sweeps, double* ms, double tol_rot) {
  const size_t es = sizeof(T);
  const int kmin = m < n ? m : n;
  Buf th((size_t)m * n * es), is((size_t)m * n * es + (size_t)kmin * kmin * es), sv((size_t)kmin * 8),
      bonds(4 * sizeof(int)), st(sizeof(ChainState)), work((size_t)(m + 1) * (n + 1) * es);
  cudaMemcpy(th.p, theta, (size_t)m * n * es, cudaMemcpyHostToDevice);
  ChainState z{};
  z.active = 1;
  cudaMemcpy(st.p, &z, sizeof z, cudaMemcpyHostToDevice);
  int hb[4] = {m, n, 0, 0};
  cudaMemcpy(bonds.p, hb, sizeof hb, cudaMemcpyHostToDevice);
  SvdParams p{};
  {
    const char* e = getenv("TTG_SVD_EARLY");
    p.no_early = (e && e[0] == '0') ? 1 : 0;
  }
  p.theta = th.p;
  p.M = dbond(0);
  p.N = dbond(1);
  p.bonds = static_cast<int*>(bonds.p);
  p.ld = 4;
  p.out_idx = 2;
  p.iso = is.p;
  p.svals = static_cast<double*>(sv.p);
  p.st = static_cast<ChainState*>(st.p);
  p.check_active = 0;
  p.accumulate_err = 1;
  p.tol = tol;
  p.max_bond = max_bond;
  p.mode = mode;
  p.work = work.p;
  p.s_work = (long long)(m + 1) * (n + 1);  // capacity of `work` in elements (checked by jacobi_svd)
  Buf sw(sizeof(int));
  p.sweeps_out = static_cast<int*>(sw.p);
  p.tol_rot = tol_rot;
  const int l = mode == 0 ? m : n, k = mode == 0 ? n : m;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, nullptr);
  const char* ge = getenv("TTG_DEBUG_SVD_GRID");
  const bool use_grid = ge && ge[0] == '1' && jacobi_grid_eligible(l, k, 1, sizeof(T));
  Buf gw(use_grid ? jacobi_grid_work_bytes(l, k, sizeof(T)) : 16);
  p.retry = 1;
  {
    const char* fr = getenv("TTG_SVD_FORCE_RETRY");
    p.first_budget = fr ? atoi(fr) : 0;
  }
  cudaError_t e = cudaSuccess;
  for (int attempt = 0; attempt < 2 && e == cudaSuccess; ++attempt) {
    p.attempt = attempt;
    if (attempt == 1) e = svd_jitter<T>(th.p, 0, p.M, p.N, p.bonds, p.ld, p.st, 1, nullptr);
    if (e == cudaSuccess)
      e = use_grid ? jacobi_svd_grid<T>(p, l, k, 1, gw.p, nullptr) : jacobi_svd<T>(p, l, k, 1, nullptr);
  }
  if (e == cudaSuccess && iso_complete_smem(l, kmin, sizeof(T)) <= 200 * 1024)
    e = iso_complete<T>(p, l, kmin, 1, nullptr);
  cudaEventRecord(e1, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return TTG_CUDA;
  float fms = 0.f;
  cudaEventElapsedTime(&fms, e0, e1);
  if (ms) *ms = fms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (sweeps) cudaMemcpy(sweeps, sw.p, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, bonds.p, sizeof hb, cudaMemcpyDeviceToHost);
  cudaMemcpy(&z, st.p, sizeof z, cudaMemcpyDeviceToHost);
  const int r = hb[2];
  *rank = r;
  *err2 = z.err2;
  cudaMemcpy(svals, sv.p, (size_t)kmin * 8, cudaMemcpyDeviceToHost);
  const size_t iso_elems = mode == 0 ? (size_t)m * r : (size_t)r * n;
  cudaMemcpy(iso, is.p, iso_elems * es, cudaMemcpyDeviceToHost);
  if (z.status) return TTG_NUMERIC;
  return TTG_OK;
}

template <typename T>
ttg_status do_qr(int m, int n, const void* A, void* Q, void* R) {
  const size_t es = sizeof(T);
  const int k = m < n ? m : n;
  Buf a((size_t)m * n * es), q((size_t)m * k * es), r((size_t)k * n * es),
      w(qr_workspace_elems<T>(m, n) * es);
  cudaMemcpy(a.p, A, (size_t)m * n * es, cudaMemcpyHostToDevice);
  QrParams p{a.p, 0, q.p, 0, r.p, 0, w.p, 0, m, n};
  cudaError_t e = householder_qr<T>(p, 1, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return TTG_CUDA;
  cudaMemcpy(Q, q.p, (size_t)m * k * es, cudaMemcpyDeviceToHost);
  cudaMemcpy(R, r.p, (size_t)k * n * es, cudaMemcpyDeviceToHost);
  return TTG_OK;
}

template <typename T>
ttg_status do_qr_blocked(int m, int n, const void* A, void* Q, void* R) {
  const size_t es = sizeof(T);
  const int k = m < n ? m : n;
  size_t sA, sV, sT, sW, sP;
  qr_blocked_elems<T>(m, n, &sA, &sV, &sT, &sW, &sP);
  Buf a((size_t)m * n * es), q((size_t)m * k * es), r((size_t)k * n * es), wa(sA * es), wv(sV * es), wt(sT * es),
      w1(sW * es), w2(sW * es), wp(sP * es);
  cudaMemcpy(a.p, A, (size_t)m * n * es, cudaMemcpyHostToDevice);
  QrParams p{a.p, 0, q.p, 0, r.p, 0, nullptr, 0, m, n};
  QrBlockedWork w{wa.p, wv.p, wt.p, w1.p, w2.p, wp.p, 0, 0, 0, 0, 0};
  cudaError_t e = householder_qr_blocked<T>(p, w, 1, nullptr, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return TTG_CUDA;
  cudaMemcpy(Q, q.p, (size_t)m * k * es, cudaMemcpyDeviceToHost);
  cudaMemcpy(R, r.p, (size_t)k * n * es, cudaMemcpyDeviceToHost);
  return TTG_OK;
}

// qr_precondition on one l x k matrix M = A (trans 0) or A^H (trans 1), A m x n row-major
template <typename T>
ttg_status do_qr_pre(int m, int n, int trans, const void* A, void* Q, void* RH, int small, double* ms) {
  const size_t es = sizeof(T);
  const int l = trans ? n : m, k = trans ? m : n, r0 = l < k ? l : k;
  Buf a((size_t)m * n * es), q((size_t)l * r0 * es), rh((size_t)k * r0 * es), bonds(4 * sizeof(int));
  cudaMemcpy(a.p, A, (size_t)m * n * es, cudaMemcpyHostToDevice);
  cudaMemset(bonds.p, 0, 4 * sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, nullptr);
  cudaError_t e = small ? qr_precondition_small<T>(a.p, 0, dconst(m), dconst(n), trans, static_cast<int*>(bonds.p), 4,
                                                   0, Q ? q.p : nullptr, 0, rh.p, 0, l, k, nullptr, 1, nullptr)
                        : qr_precondition_unblocked<T>(a.p, 0, dconst(m), dconst(n), trans,
                                                       static_cast<int*>(bonds.p), 4, 0, Q ? q.p : nullptr, 0, rh.p, 0,
                                                       l, k, nullptr, 1, nullptr);
  cudaEventRecord(e1, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  float f = 0.f;
  cudaEventElapsedTime(&f, e0, e1);
  if (ms) *ms = f;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return TTG_CUDA;
  if (Q) cudaMemcpy(Q, q.p, (size_t)l * r0 * es, cudaMemcpyDeviceToHost);
  cudaMemcpy(RH, rh.p, (size_t)k * r0 * es, cudaMemcpyDeviceToHost);
  return TTG_OK;
}

}  // namespace

extern "C" {

ttg_status ttg_debug_qr_pre(int dtype, int m, int n, int trans, const void* A, void* Q, void* RH, int small,
                            double* ms) {
  if (m < 1 || n < 1) return TTG_INVALID;
  return dtype == TTG_F64 ? do_qr_pre<double>(m, n, trans, A, Q, RH, small, ms)
                          : do_qr_pre<cplx>(m, n, trans, A, Q, RH, small, ms);
}

ttg_status ttg_debug_qr_blocked(int dtype, int m, int n, const void* A, void* Q, void* R) {
  if (m < 1 || n < 1) return TTG_INVALID;
  return dtype == TTG_F64 ? do_qr_blocked<double>(m, n, A, Q, R) : do_qr_blocked<cplx>(m, n, A, Q, R);
}


ttg_status ttg_debug_gemm(int dtype, int opA, int opB, int M, int N, int K, int batch, const void* A, const void* B,
                          void* C) {
  if (M < 1 || N < 1 || K < 0 || batch < 1) return TTG_INVALID;
  return dtype == TTG_F64 ? do_gemm<double>(opA, opB, M, N, K, A, B, C, batch)
                          : do_gemm<cplx>(opA, opB, M, N, K, A, B, C, batch);
}

ttg_status ttg_debug_gemm_dev(int dtype, int opA, int opB, int M, int N, int K, int batch, const void* A,
                              const void* B, void* C, int reps, double* ms) {
  if (M < 1 || N < 1 || K < 0 || batch < 1 || reps < 1) return TTG_INVALID;
  const long long na = (long long)M * K, nb = (long long)K * N, nc = (long long)M * N;
  GemmParams p{A, B, C, na, nb, nc, dconst(M), dconst(N), dconst(K), nullptr, 0, nullptr, 1.0, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaError_t e = cudaSuccess;
  cudaEventRecord(e0, nullptr);
  for (int r = 0; r < reps && e == cudaSuccess; ++r)
    e = dtype == TTG_F64 ? gemm<double>(p, opA, opB, M, N, batch, nullptr) : gemm<cplx>(p, opA, opB, M, N, batch, nullptr);
  cudaEventRecord(e1, nullptr);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float f = 0.f;
  cudaEventElapsedTime(&f, e0, e1);
  if (ms) *ms = f / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return e == cudaSuccess ? TTG_OK : TTG_CUDA;
}

ttg_status ttg_debug_svd(int dtype, int m, int n, const void* theta, int mode, double tol, int64_t max_bond,
                         void* iso, double* svals, int* rank, double* err2) {
  return ttg_debug_svd_ex(dtype, m, n, theta, mode, tol, max_bond, iso, svals, rank, err2, nullptr, nullptr, 0.0);
}

ttg_status ttg_debug_svd_ex(int dtype, int m, int n, const void* theta, int mode, double tol, int64_t max_bond,
                            void* iso, double* svals, int* rank, double* err2, int* sweeps, double* ms,
                            double tol_rot) {
  if (m < 1 || n < 1) return TTG_INVALID;
  return dtype == TTG_F64
             ? do_svd<double>(m, n, theta, mode, tol, max_bond, iso, svals, rank, err2, sweeps, ms, tol_rot)
             : do_svd<cplx>(m, n, theta, mode, tol, max_bond, iso, svals, rank, err2, sweeps, ms, tol_rot);
}

ttg_status ttg_debug_qr(int dtype, int m, int n, const void* A, void* Q, void* R) {
  if (m < 1 || n < 1) return TTG_INVALID;
  return dtype == TTG_F64 ? do_qr<double>(m, n, A, Q, R) : do_qr<cplx>(m, n, A, Q, R);
}

}  // extern "C"
