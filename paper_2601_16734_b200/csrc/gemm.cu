// Batched DMMA GEMM (see gemm.cuh).  Tiles: 64x64x16 per CTA, 4 warps in a
// 2x2 layout, each warp 32x32 = 2 x 4 m16n8 accumulator tiles.  Operands are
// staged k-major in shared memory by a 2-stage cp.async pipeline (zero-filled
// at the ragged edges), rows padded so that the 64-bit (f64) and 128-bit
// (complex) fragment loads are bank-conflict free.
#include "gemm.cuh"

#include <cuda.h>  // CUtensorMap and its enums (types only; the encoder is fetched through the runtime)

#include <algorithm>
#include <cstdint>
#include <cstdlib>

namespace ttg {
namespace {

constexpr int BM = 64, BN = 64, NTHREADS = 128, STAGES = 2;

template <typename T> struct Pad { static constexpr int value = 4; };
template <> struct Pad<cplx> { static constexpr int value = 2; };
// k-depth per stage: 16 (f64) / 8 (complex) keeps both stages under 48 KB static smem
template <typename T> struct Depth { static constexpr int value = 16; };
template <> struct Depth<cplx> { static constexpr int value = 8; };

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool valid, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src = valid ? bytes : 0;
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// Grouped raster: consecutive CTAs walk RASTER_G tile rows of one tile column before moving to the
// next column, so a B tile column (K x 64) is reused from L2 by the group's rows and the group's A
// rows stay resident while the columns stream (row-major order re-read all of B once per tile row:
// 3.33 GB of DRAM reads for the 0.37 GB operands of the C4 product Y = X T, profiles/r01_gemm_c4Y).
__device__ __forceinline__ void tile_of(int bid, int tiles_m, int tiles_n, int RASTER_G, int& tm, int& tn) {
  if (RASTER_G <= 1) {  // row-major
    tm = bid / tiles_n;
    tn = bid - tm * tiles_n;
    return;
  }
  const int gsz = RASTER_G * tiles_n;
  const int g = bid / gsz, r = bid - g * gsz;
  const int first = g * RASTER_G;
  const int gm = min(RASTER_G, tiles_m - first);
  tn = r / gm;
  tm = first + (r - tn * gm);
}

// ---- TMA (bulk asynchronous copy) + mbarrier helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TTG_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra TTG_DONE;\n"
      "bra TTG_WAIT;\n"
      "TTG_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one contiguous row segment global -> shared through the TMA engine (SASS UBLKCP); completion is
// counted in bytes on the stage's mbarrier
__device__ __forceinline__ void tma_row(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int TMA_STAGES = 4;

// TMA-staged variant of gemm_kernel for products whose shapes are known on the host and satisfy
// gemm_tma_ok(): same 64 x 64 x BK tiles, warp layout and padded (bank-conflict free) shared-memory
// layouts, but the operand rows of a stage are moved by bulk asynchronous copies (one per tile row,
// 128 B .. 1 KB each, issued by the lanes of warp 0) that complete on the stage's mbarrier, four
// stages deep.  No ragged K (K % BK == 0); rows / columns beyond M / N are never copied and their
// (garbage) products are discarded by the epilogue's bounds check.
template <typename T, int OPA, int OPB>
__global__ void __launch_bounds__(NTHREADS) gemm_tma_kernel(GemmParams p, int tiles_m, int tiles_n) {
  constexpr int PAD = Pad<T>::value;
  constexpr int BK = Depth<T>::value;
  constexpr int SA = BM + PAD, SB = BN + PAD;
  constexpr bool CPX = Scalar<T>::is_complex;
  constexpr bool AK = (OPA == OP_N || OPA == OP_R);
  constexpr bool BK_ = (OPB == OP_T || OPB == OP_C);
  constexpr int SK = BK + 4;
  constexpr int A_ELEMS = AK ? BM * SK : BK * SA;
  constexpr int B_ELEMS = BK_ ? BN * SK : BK * SB;
  extern __shared__ __align__(16) unsigned char tma_smem[];
  T* const As = reinterpret_cast<T*>(tma_smem);
  T* const Bs = As + TMA_STAGES * A_ELEMS;
  __shared__ __align__(8) unsigned long long full[TMA_STAGES];
  auto a_at = [&](int st, int k, int m) -> T& { return AK ? As[st * A_ELEMS + m * SK + k] : As[st * A_ELEMS + k * SA + m]; };
  auto b_at = [&](int st, int k, int n) -> T& { return BK_ ? Bs[st * B_ELEMS + n * SK + k] : Bs[st * B_ELEMS + k * SB + n]; };

  const int chain = blockIdx.y;
  if (p.st && !p.st[chain].active) return;
  const int M = p.M.eval(p.bonds, chain, p.bonds_ld);
  const int N = p.N.eval(p.bonds, chain, p.bonds_ld);
  const int K = p.K.eval(p.bonds, chain, p.bonds_ld);
  int tm, tn;
  tile_of(blockIdx.x, tiles_m, tiles_n, p.raster, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  if (m0 >= M || n0 >= N) return;

  const long long lda = p.lda ? p.lda : (AK ? K : M);
  const long long ldb = p.ldb ? p.ldb : (BK_ ? K : N);
  const long long ldc = p.ldc ? p.ldc : N;
  const T* A = static_cast<const T*>(p.A) + p.sA * chain;
  const T* B = static_cast<const T*>(p.B) + p.sB * chain;
  T* C = static_cast<T*>(p.C) + p.sC * chain;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int mrows = min(BM, M - m0), ncols = min(BN, N - n0);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TMA_STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  double acc[2][4][4];
  double acci[CPX ? 2 : 1][CPX ? 4 : 1][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
  if constexpr (CPX) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acci[i][j][r] = 0.0;
  }

  // warp 0: expected bytes of the stage, then one bulk copy per operand row
  const unsigned a_bytes = (AK ? (unsigned)mrows * BK : (unsigned)BK * mrows) * (unsigned)sizeof(T);
  const unsigned b_bytes = (BK_ ? (unsigned)ncols * BK : (unsigned)BK * ncols) * (unsigned)sizeof(T);
  auto issue = [&](int stage, int k0) {
    if (lane == 0) mbar_expect_tx(&full[stage], a_bytes + b_bytes);
    __syncwarp();
    if constexpr (AK) {
      for (int m = lane; m < mrows; m += 32)
        tma_row(&a_at(stage, 0, m), A + (m0 + m) * lda + k0, BK * sizeof(T), &full[stage]);
    } else {
      for (int k = lane; k < BK; k += 32)
        tma_row(&a_at(stage, k, 0), A + (k0 + k) * lda + m0, mrows * sizeof(T), &full[stage]);
    }
    if constexpr (BK_) {
      for (int n = lane; n < ncols; n += 32)
        tma_row(&b_at(stage, 0, n), B + (n0 + n) * ldb + k0, BK * sizeof(T), &full[stage]);
    } else {
      for (int k = lane; k < BK; k += 32)
        tma_row(&b_at(stage, k, 0), B + (k0 + k) * ldb + n0, ncols * sizeof(T), &full[stage]);
    }
  };

  const int ktiles_all = K / BK;
  const int splits = gridDim.z;
  const int per = (ktiles_all + splits - 1) / splits;
  int kt0 = blockIdx.z * per;
  const int kt1 = min(ktiles_all, kt0 + per);
  if constexpr (AK)
    if (p.a_upper) kt0 = max(kt0, m0 / BK);
  const int ktiles = max(0, kt1 - kt0);
  if (warp == 0)
    for (int s = 0; s < TMA_STAGES - 1 && s < ktiles; ++s) issue(s, (kt0 + s) * BK);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int stage = kt % TMA_STAGES;
    // the stage of tile kt + STAGES - 1 was read in iteration kt - 1 (all warps are past its barrier)
    if (warp == 0 && kt + TMA_STAGES - 1 < ktiles) issue((kt + TMA_STAGES - 1) % TMA_STAGES, (kt0 + kt + TMA_STAGES - 1) * BK);
    mbar_wait(&full[stage], (kt / TMA_STAGES) & 1);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if constexpr (!CPX) {
        double a[2][2], b[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          a[i][0] = a_at(stage, kk + t4, wm + i * 16 + g);
          a[i][1] = a_at(stage, kk + t4, wm + i * 16 + g + 8);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = b_at(stage, kk + t4, wn + j * 8 + g);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i][0], a[i][1], b[j]);
      } else {
        constexpr double sa = (OPA == OP_C || OPA == OP_R) ? -1.0 : 1.0;
        constexpr double sb = (OPB == OP_C || OPB == OP_R) ? -1.0 : 1.0;
        double ar[2][2], ai[2][2], nai[2][2], br[4], bi[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const cplx x0 = a_at(stage, kk + t4, wm + i * 16 + g);
          const cplx x1 = a_at(stage, kk + t4, wm + i * 16 + g + 8);
          ar[i][0] = x0.x; ai[i][0] = sa * x0.y; nai[i][0] = -ai[i][0];
          ar[i][1] = x1.x; ai[i][1] = sa * x1.y; nai[i][1] = -ai[i][1];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const cplx y = b_at(stage, kk + t4, wn + j * 8 + g);
          br[j] = y.x; bi[j] = sb * y.y;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dmma(acc[i][j], ar[i][0], ar[i][1], br[j]);
            dmma(acc[i][j], nai[i][0], nai[i][1], bi[j]);
            dmma(acci[i][j], ar[i][0], ar[i][1], bi[j]);
            dmma(acci[i][j], ai[i][0], ai[i][1], br[j]);
          }
      }
    }
    __syncthreads();
  }

  const double alpha = p.alpha;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + wm + i * 16 + g + (r >= 2 ? 8 : 0);
        const int n = n0 + wn + j * 8 + 2 * t4 + (r & 1);
        if (m < M && n < N) {
          T* dst = C + m * ldc + n;
          if (splits > 1) {
            T* w = static_cast<T*>(p.ws) + (((long long)chain * splits + blockIdx.z) * p.ws_m + m) * p.ws_n + n;
            if constexpr (!CPX)
              *w = alpha * acc[i][j][r];
            else
              *w = cplx{alpha * acc[i][j][r], alpha * acci[i][j][r]};
          } else if constexpr (!CPX) {
            const double v = alpha * acc[i][j][r];
            *dst = p.beta ? *dst + v : v;
          } else {
            cplx v{alpha * acc[i][j][r], alpha * acci[i][j][r]};
            if (p.beta) v = add(*dst, v);
            *dst = v;
          }
        }
      }
}

template <typename T, int OPA, int OPB>
constexpr size_t gemm_tma_smem() {
  constexpr int PAD = Pad<T>::value, BK = Depth<T>::value, SK = BK + 4;
  constexpr bool AK = (OPA == OP_N || OPA == OP_R), BK_ = (OPB == OP_T || OPB == OP_C);
  return (size_t)TMA_STAGES * ((AK ? BM * SK : BK * (BM + PAD)) + (BK_ ? BN * SK : BK * (BN + PAD))) * sizeof(T);
}

template <typename T, int OPA, int OPB>
__global__ void __launch_bounds__(NTHREADS) gemm_kernel(GemmParams p, int tiles_m, int tiles_n) {
  constexpr int PAD = Pad<T>::value;
  constexpr int BK = Depth<T>::value;
  constexpr int KSH = BK == 16 ? 4 : 3;
  constexpr int SA = BM + PAD, SB = BN + PAD;
  constexpr bool CPX = Scalar<T>::is_complex;
  // Operands whose global layout is contiguous along k are staged [row][k]
  // (stride BK + 4: conflict-free fragment loads and conflict-free cp.async
  // stores); the others [k][row] (stride BM + PAD).
  constexpr bool AK = (OPA == OP_N || OPA == OP_R);
  constexpr bool BK_ = (OPB == OP_T || OPB == OP_C);
  constexpr int SK = BK + 4;
  constexpr int A_ELEMS = AK ? BM * SK : BK * SA;
  constexpr int B_ELEMS = BK_ ? BN * SK : BK * SB;
  __shared__ __align__(16) T As[STAGES][A_ELEMS];
  __shared__ __align__(16) T Bs[STAGES][B_ELEMS];
  auto a_at = [&](int st, int k, int m) -> T& { return AK ? As[st][m * SK + k] : As[st][k * SA + m]; };
  auto b_at = [&](int st, int k, int n) -> T& { return BK_ ? Bs[st][n * SK + k] : Bs[st][k * SB + n]; };

  const int chain = blockIdx.y;
  if (p.st && !p.st[chain].active) return;
  const int M = p.M.eval(p.bonds, chain, p.bonds_ld);
  const int N = p.N.eval(p.bonds, chain, p.bonds_ld);
  const int K = p.K.eval(p.bonds, chain, p.bonds_ld);
  int tm, tn;
  tile_of(blockIdx.x, tiles_m, tiles_n, p.raster, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  if (m0 >= M || n0 >= N) return;

  const long long lda = p.lda ? p.lda : ((OPA == OP_N || OPA == OP_R) ? K : M);
  const long long ldb = p.ldb ? p.ldb : ((OPB == OP_N || OPB == OP_R) ? N : K);
  const long long ldc = p.ldc ? p.ldc : N;
  const T* A = static_cast<const T*>(p.A) + p.sA * chain;
  const T* B = static_cast<const T*>(p.B) + p.sB * chain;
  T* C = static_cast<T*>(p.C) + p.sC * chain;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  double acc[2][4][4];
  double acci[CPX ? 2 : 1][CPX ? 4 : 1][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
  if constexpr (CPX) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acci[i][j][r] = 0.0;
  }

  auto load_tile = [&](int stage, int k0) {
    // A tile: BM x BK, element (m, k) -> As[k][m]
    if constexpr (OPA == OP_N || OPA == OP_R) {
      const int kk = tid & (BK - 1), mb = tid >> KSH;
#pragma unroll
      for (int i = 0; i < BM * BK / NTHREADS; ++i) {
        const int m = mb + (NTHREADS / BK) * i;
        const bool v = (m0 + m < M) && (k0 + kk < K);
        const T* src = v ? A + (m0 + m) * lda + (k0 + kk) : A;
        cp_async(&a_at(stage, kk, m), src, v, sizeof(T));
      }
    } else {
      const int m = tid & 63, kb = tid >> 6;
#pragma unroll
      for (int i = 0; i < BK / 2; ++i) {
        const int kk = kb + 2 * i;
        const bool v = (m0 + m < M) && (k0 + kk < K);
        const T* src = v ? A + (k0 + kk) * lda + (m0 + m) : A;
        cp_async(&a_at(stage, kk, m), src, v, sizeof(T));
      }
    }
    // B tile: BK x BN, element (k, n) -> Bs[k][n]
    if constexpr (OPB == OP_N || OPB == OP_R) {
      const int n = tid & 63, kb = tid >> 6;
#pragma unroll
      for (int i = 0; i < BK / 2; ++i) {
        const int kk = kb + 2 * i;
        const bool v = (n0 + n < N) && (k0 + kk < K);
        const T* src = v ? B + (k0 + kk) * ldb + (n0 + n) : B;
        cp_async(&b_at(stage, kk, n), src, v, sizeof(T));
      }
    } else {
      const int kk = tid & (BK - 1), nb = tid >> KSH;
#pragma unroll
      for (int i = 0; i < BN * BK / NTHREADS; ++i) {
        const int n = nb + (NTHREADS / BK) * i;
        const bool v = (n0 + n < N) && (k0 + kk < K);
        const T* src = v ? B + (n0 + n) * ldb + (k0 + kk) : B;
        cp_async(&b_at(stage, kk, n), src, v, sizeof(T));
      }
    }
  };

  // split-K: blockIdx.z owns k-tiles [kt0, kt1); its partial tile goes to the workspace
  const int ktiles_all = (K + BK - 1) / BK;
  const int splits = gridDim.z;
  const int per = (ktiles_all + splits - 1) / splits;
  int kt0 = blockIdx.z * per;
  const int kt1 = min(ktiles_all, kt0 + per);
  if constexpr (OPA == OP_N || OPA == OP_R)
    if (p.a_upper) kt0 = max(kt0, m0 / BK);
  const int ktiles = max(0, kt1 - kt0);
  if (ktiles > 0) load_tile(0, kt0 * BK);
  cp_commit();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int stage = kt & 1;
    if (kt + 1 < ktiles) load_tile(stage ^ 1, (kt0 + kt + 1) * BK);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if constexpr (!CPX) {
        double a[2][2], b[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          a[i][0] = a_at(stage, kk + t4, wm + i * 16 + g);
          a[i][1] = a_at(stage, kk + t4, wm + i * 16 + g + 8);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = b_at(stage, kk + t4, wn + j * 8 + g);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i][0], a[i][1], b[j]);
      } else {
        constexpr double sa = (OPA == OP_C || OPA == OP_R) ? -1.0 : 1.0;
        constexpr double sb = (OPB == OP_C || OPB == OP_R) ? -1.0 : 1.0;
        double ar[2][2], ai[2][2], nai[2][2], br[4], bi[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const cplx x0 = a_at(stage, kk + t4, wm + i * 16 + g);
          const cplx x1 = a_at(stage, kk + t4, wm + i * 16 + g + 8);
          ar[i][0] = x0.x; ai[i][0] = sa * x0.y; nai[i][0] = -ai[i][0];
          ar[i][1] = x1.x; ai[i][1] = sa * x1.y; nai[i][1] = -ai[i][1];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const cplx y = b_at(stage, kk + t4, wn + j * 8 + g);
          br[j] = y.x; bi[j] = sb * y.y;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dmma(acc[i][j], ar[i][0], ar[i][1], br[j]);
            dmma(acc[i][j], nai[i][0], nai[i][1], bi[j]);
            dmma(acci[i][j], ar[i][0], ar[i][1], bi[j]);
            dmma(acci[i][j], ai[i][0], ai[i][1], br[j]);
          }
      }
    }
    __syncthreads();
  }

  // epilogue: c0,c1 -> (g, 2t..2t+1), c2,c3 -> (g+8, 2t..2t+1)
  const double alpha = p.alpha;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + wm + i * 16 + g + (r >= 2 ? 8 : 0);
        const int n = n0 + wn + j * 8 + 2 * t4 + (r & 1);
        if (m < M && n < N) {
          T* dst = C + m * ldc + n;
          if (splits > 1) {  // partial tile of split z; reduced in order by splitk_reduce_kernel
            T* w = static_cast<T*>(p.ws) + (((long long)chain * splits + blockIdx.z) * p.ws_m + m) * p.ws_n + n;
            if constexpr (!CPX)
              *w = alpha * acc[i][j][r];
            else
              *w = cplx{alpha * acc[i][j][r], alpha * acci[i][j][r]};
          } else if constexpr (!CPX) {
            const double v = alpha * acc[i][j][r];
            *dst = p.beta ? *dst + v : v;
          } else {
            cplx v{alpha * acc[i][j][r], alpha * acci[i][j][r]};
            if (p.beta) v = add(*dst, v);
            *dst = v;
          }
        }
      }
}

// Deterministic split-K: C (+)= sum over splits in split order.  One thread per output element
// (blockIdx.y = row, no index division), the partials of eight splits in flight before they are added
// in order.
template <typename T>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(GemmParams p, int splits) {
  const int chain = blockIdx.z;
  if (p.st && !p.st[chain].active) return;
  const int M = p.M.eval(p.bonds, chain, p.bonds_ld);
  const int N = p.N.eval(p.bonds, chain, p.bonds_ld);
  const int m = blockIdx.y, n = blockIdx.x * 256 + threadIdx.x;
  if (m >= M || n >= N) return;
  const long long ldc = p.ldc ? p.ldc : N;
  T* dst = static_cast<T*>(p.C) + p.sC * chain + m * ldc + n;
  const long long plane = (long long)p.ws_m * p.ws_n;
  const T* w = static_cast<const T*>(p.ws) + (long long)chain * splits * plane + (long long)m * p.ws_n + n;
  T acc = p.beta ? *dst : Scalar<T>::zero();
  int z = 0;
  for (; z + 8 <= splits; z += 8) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = w[(z + u) * plane];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = add(acc, v[u]);
  }
  for (; z < splits; ++z) acc = add(acc, w[z * plane]);
  *dst = acc;
}


// ---------------------------------------------------------------------------
// Tensor-map TMA variant (f64, one chain, A = OP_N): the stage's A tile (64 rows x 16 k) and B tile arrive
// by cp.async.bulk.tensor.2d (SASS UTMALDG) into unpadded 128-byte rows with the 128-byte swizzle
// (16-byte chunk index XOR (row & 7)); out-of-range rows / columns / k are zero-filled by the TMA unit, so
// ragged edges need no special case.  Fragment loads stay bank-conflict free without padding:
//   * lane t4 takes the k PAIR (2 t4, 2 t4 + 1) of an 8-k group: one MMA consumes the even, the next the odd
//     k of the pairs (A and B use the same assignment, the sum over k does not care);
//   * k-contiguous tiles (A; B for OP_T): one 128-bit load per fragment row gives the pair; fragment row g
//     maps to tile row phys(g) = ((g & 1) << 2) | (g >> 1), so the two rows of a quarter warp differ in
//     bit 2 and the XOR spreads the eight lanes over the eight chunks;
//   * n-contiguous B (OP_N): four boxes of 16 columns per stage; the two k rows of a pair are 64-bit loads
//     from rows k & 7 in {0, 2, 4, 6} (even MMA) or {1, 3, 5, 7} (odd MMA), which the XOR spreads as well.
// The output rows (and, for OP_T, columns) are un-permuted in the epilogue.
// ---------------------------------------------------------------------------
constexpr int TM_STAGES = 4;
constexpr int TM_TILE_BYTES = 64 * 128;  // 64 rows (or 4 boxes x 16 rows) of 128 bytes
constexpr size_t TM_SMEM = (size_t)TM_STAGES * 2 * TM_TILE_BYTES + 1024;  // + alignment slack

__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int tm_phys(int g) { return ((g & 1) << 2) | (g >> 1); }

template <int OPB>  // OP_N: B is K x N (n contiguous); OP_T: B is N x K (k contiguous)
__global__ void __launch_bounds__(NTHREADS) gemm_tm_kernel(GemmParams p, const __grid_constant__ CUtensorMap mapA,
                                                           const __grid_constant__ CUtensorMap mapB, int tiles_m,
                                                           int tiles_n) {
  constexpr int BK = 16;
  extern __shared__ unsigned char tm_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* As = base;                                  // [stage][64 rows][128 B]
  unsigned char* Bs = base + TM_STAGES * TM_TILE_BYTES;      // OP_N: [stage][4 boxes][16 k][128 B]; OP_T: as A
  __shared__ __align__(8) unsigned long long full[TM_STAGES];
  const int M = p.M.mult, N = p.N.mult, K = p.K.mult;  // host-shaped products only
  int tm, tn;
  tile_of(blockIdx.x, tiles_m, tiles_n, p.raster, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  if (m0 >= M || n0 >= N) return;
  const long long ldc = p.ldc ? p.ldc : N;
  double* C = static_cast<double*>(p.C);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int pg = tm_phys(g);

  if (tid == 0) {
#pragma unroll
    for (int st = 0; st < TM_STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

  auto issue = [&](int stage, int k0) {  // one elected thread
    mbar_expect_tx(&full[stage], 2 * TM_TILE_BYTES);
    tma_load_2d(As + stage * TM_TILE_BYTES, &mapA, k0, m0, &full[stage]);
    if constexpr (OPB == OP_N) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        tma_load_2d(Bs + stage * TM_TILE_BYTES + b * 2048, &mapB, n0 + 16 * b, k0, &full[stage]);
    } else {
      tma_load_2d(Bs + stage * TM_TILE_BYTES, &mapB, k0, n0, &full[stage]);
    }
  };

  const int ktiles_all = (K + BK - 1) / BK;
  const int splits = gridDim.z;
  const int per = (ktiles_all + splits - 1) / splits;
  int kt0 = blockIdx.z * per;
  const int kt1 = min(ktiles_all, kt0 + per);
  if (p.a_upper) kt0 = max(kt0, m0 / BK);
  const int ktiles = max(0, kt1 - kt0);
  if (tid == 0)
    for (int st = 0; st < TM_STAGES - 1 && st < ktiles; ++st) issue(st, (kt0 + st) * BK);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int stage = kt % TM_STAGES;
    if (tid == 0 && kt + TM_STAGES - 1 < ktiles) issue((kt + TM_STAGES - 1) % TM_STAGES, (kt0 + kt + TM_STAGES - 1) * BK);
    mbar_wait(&full[stage], (kt / TM_STAGES) & 1);
    const unsigned char* at = As + stage * TM_TILE_BYTES;
    const unsigned char* bt = Bs + stage * TM_TILE_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      const int ch = (kk >> 1) + t4;  // 16-byte chunk of this lane's k pair
      double2 a[2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = wm + i * 16 + h * 8 + pg;
          a[i][h] = *reinterpret_cast<const double2*>(at + row * 128 + ((ch ^ (row & 7)) << 4));
        }
      double2 b[4];
      if constexpr (OPB == OP_N) {
        const int ke = kk + 2 * t4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int n = wn + j * 8 + g;
          const unsigned char* bx = bt + (n >> 4) * 2048 + (n & 1) * 8;
          const int c2 = (n & 15) >> 1;
          b[j].x = *reinterpret_cast<const double*>(bx + ke * 128 + ((c2 ^ (ke & 7)) << 4));
          b[j].y = *reinterpret_cast<const double*>(bx + (ke + 1) * 128 + ((c2 ^ ((ke + 1) & 7)) << 4));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int row = wn + j * 8 + pg;
          b[j] = *reinterpret_cast<const double2*>(bt + row * 128 + ((ch ^ (row & 7)) << 4));
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(acc[i][j], a[i][0].x, a[i][1].x, b[j].x);
          dmma(acc[i][j], a[i][0].y, a[i][1].y, b[j].y);
        }
    }
    __syncthreads();
  }

  const double alpha = p.alpha;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + wm + i * 16 + (r >= 2 ? 8 : 0) + pg;
        const int fc = 2 * t4 + (r & 1);  // fragment column
        const int n = n0 + wn + j * 8 + (OPB == OP_N ? fc : tm_phys(fc));
        if (m < M && n < N) {
          double* dst = C + m * ldc + n;
          if (splits > 1) {
            double* w = static_cast<double*>(p.ws) + ((long long)blockIdx.z * p.ws_m + m) * p.ws_n + n;
            *w = alpha * acc[i][j][r];
          } else {
            const double v = alpha * acc[i][j][r];
            *dst = p.beta ? *dst + v : v;
          }
        }
      }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                   const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeTiledFn tm_encoder() {
  static const EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}
// f64 matrix with `inner` contiguous elements per row, `rows` rows, leading dimension ld: boxes of 16 x box_rows
inline bool tm_encode(CUtensorMap* map, const void* base, long long inner, long long rows, long long ld, int box_rows) {
  const EncodeTiledFn enc = tm_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1u, 1u};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int OPA, int OPB>
cudaError_t launch_one(const GemmParams& p, dim3 grid, int tiles_m, int tiles_n, bool tma, cudaStream_t s) {
  if (tma) {
    constexpr size_t smem = gemm_tma_smem<T, OPA, OPB>();
    static const cudaError_t attr = cudaFuncSetAttribute(gemm_tma_kernel<T, OPA, OPB>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (attr != cudaSuccess) return attr;
    gemm_tma_kernel<T, OPA, OPB><<<grid, NTHREADS, smem, s>>>(p, tiles_m, tiles_n);
  } else {
    gemm_kernel<T, OPA, OPB><<<grid, NTHREADS, 0, s>>>(p, tiles_m, tiles_n);
  }
  return cudaGetLastError();
}

template <typename T, int OPA>
cudaError_t launch_b(const GemmParams& p, int opB, dim3 grid, int tiles_m, int tiles_n, bool tma, cudaStream_t s) {
  switch (opB) {
    case OP_N: return launch_one<T, OPA, OP_N>(p, grid, tiles_m, tiles_n, tma, s);
    case OP_T: return launch_one<T, OPA, OP_T>(p, grid, tiles_m, tiles_n, tma, s);
    case OP_C: return launch_one<T, OPA, OP_C>(p, grid, tiles_m, tiles_n, tma, s);
    default: return launch_one<T, OPA, OP_R>(p, grid, tiles_m, tiles_n, tma, s);
  }
}

// The TMA kernel needs host-known shapes (constant DimExpr), no ragged K, and 16-byte aligned,
// 16-byte sized row segments: even leading dimensions / extents for f64 (complex elements are 16 B).
template <typename T>
bool gemm_tma_ok(const GemmParams& p, int opA, int opB) {
  static const bool enabled = [] {
    const char* e = getenv("TTG_GEMM_TMA");
    return !(e && e[0] == '0');
  }();
  if (!enabled || p.M.idx >= 0 || p.N.idx >= 0 || p.K.idx >= 0) return false;
  const long long M = p.M.mult, N = p.N.mult, K = p.K.mult;
  constexpr int BK = Depth<T>::value;
  if (K < 2 * BK || K % BK != 0 || M * N < 64 * 64) return false;
  const bool ak = (opA == OP_N || opA == OP_R), bk = (opB == OP_T || opB == OP_C);
  // k-contiguous operands would be staged in 128-byte row copies (64 per stage): measured 2x slower
  // than the cp.async kernel (17.9 vs 33.9 TF/s, 4096^3); m- / n-contiguous operands move in 512 B - 1 KB
  // rows (16 + 16 copies per stage) and win (psi^H X: 27.5 vs 25.9 TF/s).  TTG_GEMM_TMA=2 forces all.
  static const bool all_ops = [] {
    const char* e = getenv("TTG_GEMM_TMA");
    return e && e[0] == '2';
  }();
  if ((ak || bk) && !all_ops) return false;
  const long long lda = p.lda ? p.lda : (ak ? K : M), ldb = p.ldb ? p.ldb : (bk ? K : N);
  const long long unit = 16 / (long long)sizeof(T);  // elements per 16 bytes
  auto aligned = [&](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!aligned(p.A) || !aligned(p.B) || lda % unit || ldb % unit || p.sA % unit || p.sB % unit) return false;
  if (!ak && M % unit) return false;  // rows of the A stage are m-contiguous: partial rows copy M - m0 elements
  if (!bk && N % unit) return false;
  return true;
}

}  // namespace

template <typename T>
cudaError_t gemm(const GemmParams& p, int opA, int opB, int mmax, int nmax, int chains, cudaStream_t s, int kmax) {
  if (mmax <= 0 || nmax <= 0 || chains <= 0) return cudaSuccess;
  const int tiles_m = (mmax + BM - 1) / BM, tiles_n = (nmax + BN - 1) / BN;
  // split-K when the output tiles cannot fill the GPU but K is long (e.g. V^H A in the
  // blocked QR: 32 x n x m)
  int splits = 1;
  const long long tiles = (long long)tiles_m * tiles_n * chains;
  static const int splitk_min = [] {  // split-K from this K on (TTG_GEMM_SPLITK_MIN)
    const char* e = getenv("TTG_GEMM_SPLITK_MIN");
    return e ? atoi(e) : 256;
  }();
  if (kmax >= splitk_min && tiles < 2 * 148) {
    static const int splitk_div = [] {  // at least this much K per split (TTG_GEMM_SPLITK_DIV)
      const char* e = getenv("TTG_GEMM_SPLITK_DIV");
      return e ? atoi(e) : 64;  // C4 A/B (K >= / K per split): 1024/256 1913 ms, 512/128 1833 ms, 256/64 1816 ms, 128/32 1814 ms
    }();
    splits = (int)std::min<long long>((2 * 148 + tiles - 1) / tiles, kmax / splitk_div);
    splits = std::max(1, std::min(splits, 64));
  }
  dim3 grid(tiles_m * tiles_n, chains, splits);
  GemmParams q = p;
  // grouped raster only where a B tile column is worth keeping in L2 (long K): the K = 32 / 128
  // trailing updates of the blocked QR stream C and measured faster in row-major order
  static const int raster_env = [] {
    const char* e = getenv("TTG_GEMM_RASTER");
    return e ? atoi(e) : 16;
  }();
  static const int raster_kmin = [] {
    const char* e = getenv("TTG_GEMM_RASTER_KMIN");
    return e ? atoi(e) : 512;
  }();
  q.raster = (kmax >= raster_kmin || (p.K.idx < 0 && p.K.mult >= raster_kmin)) ? raster_env : 0;
  if (splits > 1) {  // partial tiles in a stream-ordered workspace, reduced in fixed order (deterministic)
    q.ws_m = mmax;
    q.ws_n = nmax;
    cudaError_t e = cudaMallocAsync(&q.ws, (size_t)chains * splits * mmax * nmax * sizeof(T), s);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e;
  // tensor-map TMA kernel: f64, one chain, host shapes, A = OP_N and B = OP_N / OP_T (the projection chain
  // X = L T, Y = X T, theta = Y R^T and the carry R T), 16-byte aligned bases and leading dimensions
  if constexpr (!Scalar<T>::is_complex) {
    static const int tm_mode = [] {
      const char* ev = getenv("TTG_GEMM_TM");
      return ev ? atoi(ev) : 1;
    }();
    const bool shapes = q.M.idx < 0 && q.N.idx < 0 && q.K.idx < 0;
    if (tm_mode && shapes && chains == 1 && q.st == nullptr && opA == OP_N && (opB == OP_N || opB == OP_T)) {
      const long long M = q.M.mult, N = q.N.mult, K = q.K.mult;
      const long long lda = q.lda ? q.lda : K, ldb = q.ldb ? q.ldb : (opB == OP_N ? N : K);
      auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
      const bool big = tm_mode == 2 || (K >= 256 && M * N >= 256 * 256);
      if (big && al16(q.A) && al16(q.B) && lda % 2 == 0 && ldb % 2 == 0 && M > 0 && N > 0 && K > 0) {
        CUtensorMap mapA, mapB;
        const bool okA = tm_encode(&mapA, q.A, K, M, lda, 64);
        const bool okB = opB == OP_N ? tm_encode(&mapB, q.B, N, K, ldb, 16) : tm_encode(&mapB, q.B, K, N, ldb, 64);
        if (okA && okB) {
          if (opB == OP_N) {
            static const cudaError_t at = cudaFuncSetAttribute(gemm_tm_kernel<OP_N>,
                                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TM_SMEM);
            if (at != cudaSuccess) return at;
            gemm_tm_kernel<OP_N><<<grid, NTHREADS, TM_SMEM, s>>>(q, mapA, mapB, tiles_m, tiles_n);
          } else {
            static const cudaError_t at = cudaFuncSetAttribute(gemm_tm_kernel<OP_T>,
                                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TM_SMEM);
            if (at != cudaSuccess) return at;
            gemm_tm_kernel<OP_T><<<grid, NTHREADS, TM_SMEM, s>>>(q, mapA, mapB, tiles_m, tiles_n);
          }
          e = cudaGetLastError();
          if (splits > 1) {
            if (e == cudaSuccess) {
              splitk_reduce_kernel<T><<<dim3((nmax + 255) / 256, mmax, chains), 256, 0, s>>>(q, splits);
              e = cudaGetLastError();
            }
            cudaFreeAsync(q.ws, s);
          }
          return e;
        }
      }
    }
  }
  const bool tma = gemm_tma_ok<T>(q, opA, opB);
  switch (opA) {
    case OP_N: e = launch_b<T, OP_N>(q, opB, grid, tiles_m, tiles_n, tma, s); break;
    case OP_T: e = launch_b<T, OP_T>(q, opB, grid, tiles_m, tiles_n, tma, s); break;
    case OP_C: e = launch_b<T, OP_C>(q, opB, grid, tiles_m, tiles_n, tma, s); break;
    default: e = launch_b<T, OP_R>(q, opB, grid, tiles_m, tiles_n, tma, s); break;
  }
  if (splits > 1) {
    if (e == cudaSuccess) {
      splitk_reduce_kernel<T><<<dim3((nmax + 255) / 256, mmax, chains), 256, 0, s>>>(q, splits);
      e = cudaGetLastError();
    }
    cudaFreeAsync(q.ws, s);
  }
  return e;
}

template cudaError_t gemm<double>(const GemmParams&, int, int, int, int, int, cudaStream_t, int);
template cudaError_t gemm<cplx>(const GemmParams&, int, int, int, int, int, cudaStream_t, int);

}  // namespace ttg
