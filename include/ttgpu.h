/* ttgpu — C ABI of the B200 (sm_100a) MPO·MPS apply / Hadamard + canonical
 * simplification hot path.
 *
 * This is the boundary the drop-in C++ headers (include/ttlab/*.hpp) call in
 * place of the reference's Eigen implementation.  Every entry point names the
 * reference function it replaces (paths relative to
 * /root/reference/proj/include/ttlab/).  Plain C types only: pointers, sizes,
 * integers and doubles.
 *
 * Conventions
 *   - Tensors are row-major, Tensor3 A[left, phys, right] (tensor.hpp:13-86) and
 *     Tensor4 B[left, out, in, right] (tensor.hpp:89-149).  dtype TTG_F64 holds
 *     doubles, TTG_C128 interleaved (re, im) pairs = std::complex<double>.
 *   - A ttg_dmps is a device-resident batch of `count` chains with identical
 *     length and physical dimensions (count = 1 for an ordinary MPS).
 *   - Every call returns a ttg_status; on failure ttg_last_error(ctx) holds the
 *     message.  TTG_SHAPE / TTG_CAPACITY / TTG_NUMERIC map to the reference's
 *     shape_error / capacity_error / numeric_error (types.hpp:22-37).
 *   - One context per host thread; calls are stream-ordered on the context's
 *     stream and synchronous at return unless documented otherwise.
 */
#ifndef TTGPU_H
#define TTGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  TTG_OK = 0,
  TTG_SHAPE = 1,    /* shape_error   (types.hpp:22-25) */
  TTG_CAPACITY = 2, /* capacity_error (types.hpp:28-31) */
  TTG_NUMERIC = 3,  /* numeric_error (types.hpp:34-37) */
  TTG_CUDA = 4,     /* CUDA runtime failure / no device */
  TTG_INVALID = 5   /* bad argument (null pointer, unknown dtype, ...) */
} ttg_status;

typedef enum { TTG_F64 = 0, TTG_C128 = 1 } ttg_dtype;
typedef enum { TTG_SVD_TRUNCATE = 0, TTG_VARIATIONAL = 1 } ttg_truncation; /* types.hpp:39 */
typedef enum { TTG_LEFT_TO_RIGHT = 0, TTG_RIGHT_TO_LEFT = 1 } ttg_direction; /* types.hpp:41 */

/* types.hpp:50-88 Strategy.  max_bond <= 0 or >= INT32_MAX means unbounded. */
typedef struct {
  int method;
  double tolerance;
  double simplification_tolerance;
  int64_t max_bond;
  int max_sweeps;
  int normalize;
} ttg_strategy;

/* Per-chain outcome of simplify / apply (simplify.hpp:94-99 CompressionResult). */
typedef struct {
  int sweeps;
  int converged;
  double residual;     /* sqrt(dist2) + fp_error_floor(|T|)   (simplify.hpp:126) */
  double error;        /* error ledger of the output state      (simplify.hpp:191) */
  double norm;         /* |psi| = Frobenius norm of the centre  (mps.hpp:225)      */
  double target_norm2; /* <T, T>                                (simplify.hpp:37-41) */
} ttg_report;

/* Host view of one MPS (mps.hpp:21-143): n sites, bonds[n+1], phys[n],
 * sites[k] -> bonds[k]*phys[k]*bonds[k+1] elements of `dtype`. */
typedef struct {
  int n;
  int dtype;
  const int64_t* bonds;
  const int64_t* phys;
  const void* const* sites;
  double error;
} ttg_mps_view;

/* Host view of one MPO (mpo.hpp:14-105): sites[k] -> bonds[k]*out[k]*in[k]*bonds[k+1]. */
typedef struct {
  int n;
  int dtype;
  const int64_t* bonds;
  const int64_t* phys_out;
  const int64_t* phys_in;
  const void* const* sites;
} ttg_mpo_view;

typedef struct ttg_ctx ttg_ctx;
typedef struct ttg_dmps ttg_dmps;
typedef struct ttg_dmpo ttg_dmpo;

/* ---- context ------------------------------------------------------------ */
ttg_status ttg_create(int device, ttg_ctx** out);
void ttg_destroy(ttg_ctx* ctx);
const char* ttg_last_error(const ttg_ctx* ctx);
/* Run on an external cudaStream_t (e.g. torch's current stream); NULL = own stream. */
ttg_status ttg_set_stream(ttg_ctx* ctx, void* cuda_stream);
ttg_status ttg_synchronize(ttg_ctx* ctx);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t ttg_kernel_launches(const ttg_ctx* ctx);
const char* ttg_version(void);

/* ---- communicator (batched configs, one rank per GPU) --------------------------
 * The reference has no multi-process path; its batched use is a host loop over simplify
 * (simplify.hpp:182-195).  Here independent chains are sharded over ranks with no exchange during the
 * sweeps, and the context owns the NCCL communicator for the one collective of a batch: the all-gather
 * of per-chain scalars (norm, error, sweeps).  libnccl.so.2 is bound at run time (TTG_NCCL_LIB overrides
 * the name); contexts without a communicator behave as a world of one.
 *   rank 0: ttg_comm_unique_id -> ship the TTG_COMM_ID_BYTES to every rank by the host's own means
 *   every rank: ttg_comm_init(ctx, nranks, rank, id)      (collective: ncclCommInitRank on ctx's device)
 *   ttg_comm_allgather_f64: send[count] of every rank -> recv[nranks * count] in rank order, host
 *   buffers, on the context stream, synchronous at return. */
#define TTG_COMM_ID_BYTES 128
ttg_status ttg_comm_unique_id(ttg_ctx* ctx, void* id /* TTG_COMM_ID_BYTES */);
ttg_status ttg_comm_init(ttg_ctx* ctx, int nranks, int rank, const void* id);
ttg_status ttg_comm_info(const ttg_ctx* ctx, int* nranks, int* rank);
ttg_status ttg_comm_allgather_f64(ttg_ctx* ctx, const double* send, int64_t count, double* recv);
ttg_status ttg_comm_free(ttg_ctx* ctx);

/* Per-kernel-class timing: when enabled, every launch is bracketed by CUDA
 * events on the context stream and GEMM/SVD/QR launches record their executed
 * flops (read from the device bond table, one host sync per launch: use a
 * separate pass, not the timed one).  Enabling resets the counters. */
enum { TTG_PROF_GEMM = 0, TTG_PROF_SVD = 1, TTG_PROF_QR = 2, TTG_PROF_EXPAND = 3, TTG_PROF_CLASSES = 4 };
ttg_status ttg_profile_enable(ttg_ctx* ctx, int on);
ttg_status ttg_profile_read(ttg_ctx* ctx, int cls, int64_t* launches, double* ms, double* flops);
/* Jacobi sweeps executed by all SVD launches since profiling was enabled. */
ttg_status ttg_profile_svd_sweeps(ttg_ctx* ctx, int64_t* total);

/* ---- device MPS / MPO ---------------------------------------------------- */
/* Upload `count` host MPS of identical length/physical dims/bonds as one batch. */
ttg_status ttg_mps_upload(ttg_ctx* ctx, const ttg_mps_view* views, int count, ttg_dmps** out);
/* Wrap device-resident site tensors (copied, stream-ordered):
 * dev_sites[k] holds count * bonds[k]*phys[k]*bonds[k+1] contiguous elements. */
ttg_status ttg_mps_from_device(ttg_ctx* ctx, int n, int dtype, int count, const int64_t* bonds,
                               const int64_t* phys, const void* const* dev_sites, const double* errors,
                               ttg_dmps** out);
void ttg_mps_free(ttg_dmps* m);
/* Shape of chain `chain`: n, dtype, count, bonds[n+1], phys[n], error, centre (-1 if not canonical). */
ttg_status ttg_mps_info(const ttg_dmps* m, int chain, int* n, int* dtype, int* count, int64_t* bonds, int64_t* phys,
                        double* error, int* center);
/* Copy chain `chain` to caller-allocated host buffers sized from ttg_mps_info. */
ttg_status ttg_mps_download(ttg_ctx* ctx, const ttg_dmps* m, int chain, void* const* sites);
/* Copy every chain of the batch to caller-allocated host buffers: sites[c * n + k] receives site k
 * of chain c (shapes from ttg_mps_info).  Batches stream through pinned staging buffers (one D2H
 * per staging chunk instead of one per chain and site). */
ttg_status ttg_mps_download_batch(ttg_ctx* ctx, const ttg_dmps* m, void* const* sites);
/* Device pointer of site k of chain `chain` and its element count (for zero-copy readers). */
ttg_status ttg_mps_site_ptr(const ttg_dmps* m, int chain, int k, void** ptr, int64_t* elems);

ttg_status ttg_mpo_upload(ttg_ctx* ctx, const ttg_mpo_view* view, ttg_dmpo** out);
void ttg_mpo_free(ttg_dmpo* w);

/* ---- hot path ------------------------------------------------------------- */
/* mpo.hpp:213-238 detail::apply_raw — exact MPO·MPS, fused bond (mpo, mps). */
ttg_status ttg_apply_raw(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* v, ttg_dmps** out);
/* blas.hpp:45-67 hadamard — exact element-wise product, bonds multiply. */
ttg_status ttg_hadamard(ttg_ctx* ctx, const ttg_dmps* u, const ttg_dmps* v, ttg_dmps** out);
/* simplify.hpp:182-195 simplify(MPS, Strategy, optional guess); guess may be NULL.
 * Returns a canonical batch (centre 0); reports[count] may be NULL. */
ttg_status ttg_simplify(ttg_ctx* ctx, const ttg_dmps* target, const ttg_strategy* strategy, const ttg_dmps* guess,
                        ttg_dmps** out, ttg_report* reports);
/* blas.hpp:8-11 apply(MPO, MPS, Strategy) = simplify(apply_raw(op, v)). */
ttg_status ttg_apply(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* v, const ttg_strategy* strategy,
                     ttg_dmps** out, ttg_report* reports);
/* mps.hpp:310-313 canonicalize(MPS, centre, Strategy) (QR pass + truncating sweep). */
ttg_status ttg_canonicalize(ttg_ctx* ctx, const ttg_dmps* v, int center, const ttg_strategy* strategy,
                            ttg_dmps** out, ttg_report* reports);
/* CanonicalMPS::recenter (mps.hpp:268-279) on the device: `v` is a single chain canonical at
 * `center`; the copy in *out is moved to `target` with the truncating moves move_center_right /
 * move_center_left (mps.hpp:238-265) under `strategy`.  *err (may be NULL) = sqrt(sum of the squared
 * dropped weights) of the moves; the error ledger of *out is NOT updated (the caller decides, as
 * recenter and the single moves do differently).  Also canonicalize(const CanonicalMPS&)
 * (mps.hpp:316-323). */
ttg_status ttg_recenter(ttg_ctx* ctx, const ttg_dmps* v, int center, int target, const ttg_strategy* strategy,
                        ttg_dmps** out, double* err);
/* schmidt_split (schmidt.hpp:72-89) of one host m x n matrix (row-major, `dtype`) on the device:
 * rank r = #{s_k > tolerance s_0} clamped to [1, max_bond]; LEFT_TO_RIGHT: a = U_r (m x r),
 * b = S_r V_r^H (r x n); RIGHT_TO_LEFT: a = U_r S_r, b = V_r^H.  a needs m*min(m,n) and b
 * min(m,n)*n elements of space; written compactly.  *err = sqrt(sum_{k>=r} s_k^2).  Used by
 * CanonicalMPS::update_two_site / detail::split_pair (mps.hpp:164-173, 283-297). */
ttg_status ttg_schmidt_split(ttg_ctx* ctx, int dtype, int64_t m, int64_t n, const void* theta, int direction,
                             const ttg_strategy* strategy, void* a, void* b, int64_t* rank, double* err);
/* mps.hpp:326-405 MPSSum(weights, states).join(): block-diagonal concatenation of the scaled
 * single-chain states (MPS::scaled semantics, mps.hpp:98-117); nterms = 1 gives states[0].scaled(w).
 * error = sum |w_l| err_l.  With the variational simplify this is combine / simplify(MPSSum)
 * (simplify.hpp:151-215). w_im may be NULL. */
ttg_status ttg_mps_join(ttg_ctx* ctx, int nterms, const double* w_re, const double* w_im,
                        const ttg_dmps* const* states, ttg_dmps** out);
/* simplify.hpp:151-215 simplify(MPSSum, strategy, guess) == combine(weights, states, strategy):
 * closest MPS under `strategy` to sum_l w_l states[l] (single chains).  guess NULL = default_guess
 * (largest |w_l| |states[l]|, scaled).  One report. */
ttg_status ttg_simplify_sum(ttg_ctx* ctx, int nterms, const double* w_re, const double* w_im,
                            const ttg_dmps* const* states, const ttg_strategy* strategy, const ttg_dmps* guess,
                            ttg_dmps** out, ttg_report* report);
/* TTLAB1 container on the device boundary (serialize.hpp:61-121).  Files hold complex128;
 * real_if_possible = 1 stores the loaded object as float64 when every imaginary part is zero.
 * Errors: unreadable / bad magic / bad version / truncated / wrong rank -> TTG_NUMERIC
 * (numeric_error), inconsistent bonds -> TTG_SHAPE.  Saving a float64 object writes
 * complex128 with zero imaginary parts; ttg_mps_save writes one chain of a batch. */
ttg_status ttg_mps_load(ttg_ctx* ctx, const char* path, int real_if_possible, ttg_dmps** out);
ttg_status ttg_mps_save(ttg_ctx* ctx, const ttg_dmps* m, int chain, const char* path);
ttg_status ttg_mpo_load(ttg_ctx* ctx, const char* path, int real_if_possible, ttg_dmpo** out);
ttg_status ttg_mpo_save(ttg_ctx* ctx, const ttg_dmpo* op, const char* path);
/* eigensolvers.hpp:15-64 detail::apply_effective_two_site(lenv, w1, w2, renv, x): y = H_eff x without
 * forming H_eff.  dims = {D0, D1, D2, d1o, d1, d2o, d2, chiAo, chiA, chiBo, chiB} (w1: D0 x d1o x d1 x D1,
 * w2: D1 x d2o x d2 x D2, Tensor4 row-major).  Host buffers, all of `dtype`: L[c0](a', a) as
 * [D0][chiAo][chiA], R[c2](b', B) as [D2][chiBo][chiB], x[a][s1][s2][B], y[a'][s1'][s2'][b']. */
ttg_status ttg_apply_effective_two_site(ttg_ctx* ctx, int dtype, const int* dims, const void* L, const void* W1,
                                        const void* W2, const void* R, const void* x, void* y);
/* Device-pointer variant of ttg_apply_effective_two_site: L, W1, W2, R, x, y are device buffers with
 * the same layouts; stream-ordered on the context stream and NOT synchronised at return (a Lanczos
 * loop chains calls without host round trips; ttg_synchronize waits). */
ttg_status ttg_apply_effective_two_site_dev(ttg_ctx* ctx, int dtype, const int* dims, const void* L, const void* W1,
                                            const void* W2, const void* R, const void* x, void* y);
/* detail::update_left_op_environment (side TTG_LEFT_TO_RIGHT) / update_right_op_environment
 * (TTG_RIGHT_TO_LEFT) of environments.hpp:42-83 on device buffers (stream-ordered, not synchronised).
 * dims = {Dl, dout, din, Dr, bra_l, bra_r, ket_l, ket_r}: bra (Tensor3 bra_l x dout x bra_r),
 * op (Tensor4 Dl x dout x din x Dr), ket (Tensor3 ket_l x din x ket_r).  Environments are stacked
 * matrices E[c](a, b) stored [c][a][b]: left: env Dl x bra_l x ket_l -> out Dr x bra_r x ket_r;
 * right: env Dr x bra_r x ket_r -> out Dl x bra_l x ket_l. */
ttg_status ttg_op_env_update(ttg_ctx* ctx, int dtype, int side, const int* dims, const void* env, const void* bra,
                             const void* op, const void* ket, void* out);
/* blas.hpp:128-138 expectation_mpo(op, u, v) = <u, op v> per chain (v NULL: v = u). */
ttg_status ttg_expectation_mpo(ttg_ctx* ctx, const ttg_dmpo* op, const ttg_dmps* u, const ttg_dmps* v, double* out_re,
                               double* out_im);
/* mps.hpp:416-423 scprod(u, v) per chain: out_re/out_im[count]. */
ttg_status ttg_scprod(ttg_ctx* ctx, const ttg_dmps* u, const ttg_dmps* v, double* out_re, double* out_im);

/* ---- kernel-level test hooks (host buffers; one kernel each) ------------- */
/* C[b] = op(A[b]) op(B[b]) for b < batch; op: 0 = N, 1 = T, 2 = C (conj-transpose), 3 = conj. */
ttg_status ttg_debug_gemm(int dtype, int opA, int opB, int M, int N, int K, int batch, const void* A, const void* B,
                          void* C);
/* Same GEMM on device buffers, `reps` back-to-back launches; average kernel time in ms. */
ttg_status ttg_debug_gemm_dev(int dtype, int opA, int opB, int M, int N, int K, int batch, const void* A,
                              const void* B, void* C, int reps, double* ms);
/* schmidt_split (schmidt.hpp:72-89) of one m x n theta: mode 0 = LEFT_TO_RIGHT writes U_r (m x r),
 * mode 1 = RIGHT_TO_LEFT writes V_r^H (r x n); svals[min(m,n)] descending, rank, dropped weight^2. */
ttg_status ttg_debug_svd(int dtype, int m, int n, const void* theta, int mode, double tol, int64_t max_bond,
                         void* iso, double* svals, int* rank, double* err2);
/* As ttg_debug_svd, plus Jacobi sweeps executed, kernel time (ms) and the rotation threshold (0 = default). */
ttg_status ttg_debug_svd_ex(int dtype, int m, int n, const void* theta, int mode, double tol, int64_t max_bond,
                            void* iso, double* svals, int* rank, double* err2, int* sweeps, double* ms,
                            double tol_rot);
/* Thin Householder QR (mps.hpp:196-199): Q (m x k), R (k x n), k = min(m, n). */
ttg_status ttg_debug_qr(int dtype, int m, int n, const void* A, void* Q, void* R);
/* Same factorisation through the blocked path (panel kernel + DMMA WY updates). */
ttg_status ttg_debug_qr_blocked(int dtype, int m, int n, const void* A, void* Q, void* R);
/* Split preconditioner: M = A (trans 0) or A^H (trans 1) = Q R; writes Q (l x r0, nullable) and
 * R^H (k x r0).  small = 1: blocked shared-memory kernel (qr_small.cu); 0: the unblocked kernel. */
ttg_status ttg_debug_qr_pre(int dtype, int m, int n, int trans, const void* A, void* Q, void* RH, int small,
                            double* ms);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* TTGPU_H */
