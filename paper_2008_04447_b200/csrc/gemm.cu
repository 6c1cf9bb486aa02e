// fp64 tensor-core GEMMs for the RQRCP hot path (sm_100a, mma.sync f64 -> DMMA).
//
//  gemm_tn:  D(MxN) = alpha * X^T C + beta * E     (short M <= 144, long K, long N)
//            the sketch B = Omega A (sketch.py:70-71, X = Omega^T), the trailing
//            update's first sweep Y^T C (randomized.py:206), TRQRCP's Y2^T A
//            (randomized.py:322), W = T^T (.) (householder.py:109-110).
//  gemm_nn:  D(MxN) = alpha * X Y + beta * E        (long M, long N, short K)
//            the trailing update's second sweep C -= Y W (randomized.py:207),
//            TRQRCP panel/R-row materialisation (randomized.py:305,330), TUXV A V_k
//            (randomized.py:384).
//
// Both stage operands through a cp.async ring in padded shared memory
// (row pitch = 4 mod 16 doubles => conflict-free f64 fragment gathers) and
// accumulate with m16n8k4 f64 MMAs.  gemm_tn splits K across CTAs when the
// N-tiles cannot fill 148 SMs; partials are summed in a FIXED split order by
// a separate reduce kernel, so results are bitwise deterministic.
#include <algorithm>

#include <climits>

#include "common.cuh"

namespace sqr {

int splitk_reduce_launch(int M, int N, int MT, int nsplit, double alpha, const double* part, double beta,
                         const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, cudaStream_t s);


namespace {

// 4 warps per CTA and two CTAs per SM: a CTA waiting at __syncthreads or on
// its epilogue leaves the DMMA pipe to the other one (ptxas spaces a warp's
// DMMA.8x8x4 16 cycles apart, so the pipe needs >= 2 issuing warps per SMSP).
constexpr int kThreads = 128;
constexpr int kBK = 16;        // K per pipeline stage
constexpr int kPitchK = kBK + 4;
constexpr int kStages = 3;
// gemm_nn runs 4 CTAs/SM with a 2-deep ring: measured on the C5 rank-128
// update (32768 x 32640 x 128) 29.3 TF vs 24.2 TF at 2 CTAs x 3 stages and
// 27.0 at 3 x 3 -- the short-K update is latency- not bandwidth-limited, so
// resident warps beat pipeline depth (prefetching beta*E into registers
// before the K loop gained nothing and costs the 4th CTA).
#ifndef SQR_NN_STAGES
#define SQR_NN_STAGES 2
#endif
#ifndef SQR_NN_CTAS
#define SQR_NN_CTAS 4
#endif
constexpr int kStagesNN = SQR_NN_STAGES;
#ifndef SQR_NN_GROUP
#define SQR_NN_GROUP 16
#endif
constexpr int kNnGroup = SQR_NN_GROUP;  // M-tiles per raster group (gemm_nn)

// ---------------------------------------------------------------- gemm_tn
// Computed as D^T(N x M) = C^T(N x K) X(K x M): MMA rows = n, MMA cols = i.
// CTA tile: 64 n x MT i;  4 warps = 2 (n) x 2 (i);  warp tile 32 n x MT/2 i.
#ifndef SQR_TN_BK
#define SQR_TN_BK 16
#endif
#ifndef SQR_TN_STAGES
#define SQR_TN_STAGES 3
#endif
template <int MT, int VEC>
struct TnCfg {
  static constexpr int BN = 64;
  static constexpr int NI = MT / 16;  // n8 fragments per warp along i
  // K per stage / ring depth (two CTAs per SM must fit: the 144-row tile keeps 16 x 3)
  static constexpr int BK = MT <= 128 ? SQR_TN_BK : 16;
  static constexpr int NST = MT <= 128 ? SQR_TN_STAGES : 3;
  static constexpr int PK = BK + 4;   // pitch of a k-row (4 mod 16 doubles)
  static constexpr int A_ELEMS = BN * PK;
  static constexpr int B_ELEMS = MT * PK;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int SMEM = STAGE * NST * 8;
  static constexpr int ACC = 2 * NI * 4;
};

template <int MT, int VEC>
__device__ __forceinline__ void tn_load_stage(double* sA, double* sB, const double* __restrict__ X,
                                              int64_t ldx, const double* __restrict__ C, int64_t ldc,
                                              int M, int N, int n0, int k0, int kend, const GemmDyn& dyn) {
  using Cfg = TnCfg<MT, VEC>;
  constexpr int CPR = Cfg::BK / VEC;  // chunks per row
  const int tid = threadIdx.x;
#pragma unroll 4
  for (int c = tid; c < Cfg::BN * CPR; c += kThreads) {
    const int r = c / CPR, kc = (c % CPR) * VEC;
    const int n = n0 + r, k = k0 + kc;
    const bool ok = (n < N) && (k < kend);
    const double* src = !ok ? C
                            : (n < dyn.npre ? dyn.pre + (int64_t)n * dyn.ldpre + k
                                            : C + (int64_t)(n - dyn.npre) * ldc + k);
    double* dst = sA + r * Cfg::PK + kc;
    if constexpr (VEC == 2) {
      const int sz = ok ? ((k + 1 < kend) ? 16 : 8) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                   "r"(sz));
    } else {
      cp_async<8>(dst, src, ok);
    }
  }
#pragma unroll 4
  for (int c = tid; c < MT * CPR; c += kThreads) {
    const int r = c / CPR, kc = (c % CPR) * VEC;
    const int k = k0 + kc;
    const bool ok = (r < M) && (k < kend);
    const double* src = ok ? X + (int64_t)r * ldx + k : X;
    double* dst = sB + r * Cfg::PK + kc;
    if constexpr (VEC == 2) {
      const int sz = ok ? ((k + 1 < kend) ? 16 : 8) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                   "r"(sz));
    } else {
      cp_async<8>(dst, src, ok);
    }
  }
}

// Aligned (16-byte) fast path of tn_load_stage: the per-thread source rows
// (prefix / C selection, bounds) are resolved once per CTA, so a stage costs
// one add and one cp.async per 16-byte chunk.
template <int MT>
struct TnLoader2 {
  static constexpr int kBK = TnCfg<MT, 2>::BK, kPitchK = TnCfg<MT, 2>::PK;
  static constexpr int CPR = kBK / 2;             // 16-byte chunks per k-row
  static constexpr int RSTEP = kThreads / CPR;    // rows covered per pass
  static constexpr int NA = 64 / RSTEP;
  static constexpr int NB = (MT + RSTEP - 1) / RSTEP;
  const double* asrc[NA];
  const double* bsrc;
  int64_t bstep;
  uint32_t adst, bdst;
  int kc, r0, M;
  unsigned aok, bok;
  __device__ __forceinline__ void init(const double* X, int64_t ldx, const double* C, int64_t ldc, int M_,
                                       int N, int n0, const GemmDyn& dyn, const double* sA, const double* sB) {
    const int tid = threadIdx.x;
    r0 = tid / CPR;
    kc = (tid % CPR) * 2;
    M = M_;
    aok = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int n = n0 + r0 + RSTEP * i;
      const bool ok = n < N;
      aok |= (ok ? 1u : 0u) << i;
      asrc[i] = !ok ? C
                    : (n < dyn.npre ? dyn.pre + (int64_t)n * dyn.ldpre : C + (int64_t)(n - dyn.npre) * ldc);
    }
    bok = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i) bok |= ((r0 + RSTEP * i) < M ? 1u : 0u) << i;
    bsrc = X + (int64_t)r0 * ldx;
    bstep = (int64_t)RSTEP * ldx;
    adst = smem_u32(sA + r0 * kPitchK + kc);
    bdst = smem_u32(sB + r0 * kPitchK + kc);
  }
  __device__ __forceinline__ void load(uint32_t stage_off, int k0, int kend) const {
    const int k = k0 + kc;
    const int sz = k < kend ? (k + 1 < kend ? 16 : 8) : 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const bool ok = (aok >> i) & 1u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(adst + stage_off + i * RSTEP * kPitchK * 8),
                   "l"(ok ? asrc[i] + k : asrc[i]), "r"(ok ? sz : 0));
    }
    const double* b = bsrc + k;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const bool ok = (bok >> i) & 1u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(bdst + stage_off + i * RSTEP * kPitchK * 8),
                   "l"(ok ? b : bsrc), "r"(ok ? sz : 0));
      b += bstep;
    }
  }
};

#ifndef SQR_TN_MINB
#define SQR_TN_MINB 2   // resident CTAs per SM the register budget is sized for
#endif
template <int MT, int VEC>
__global__ void __launch_bounds__(kThreads, SQR_TN_MINB)
    gemm_tn_kernel(int M, int N, int K, double alpha, const double* __restrict__ X, int64_t ldx,
                   const double* __restrict__ C, int64_t ldc, double beta, const double* E,
                   int64_t lde, double* D, int64_t ldd, int kchunk, double* part, unsigned* sems,
                   GemmDyn dyn) {
  using Cfg = TnCfg<MT, VEC>;
  extern __shared__ __align__(16) double smem[];
  if (dyn.stop && *dyn.stop) return;
  if (dyn.shift) {
    const int sh = *dyn.shift;
    N -= sh;
    if (dyn.flags & kShiftB) C += (int64_t)sh * ldc;
    if (dyn.flags & kShiftD) {
      D += (int64_t)sh * ldd;
      if (E) E += (int64_t)sh * lde;
    }
  }
  const int Npart = N;  // split-K partial stride (before the limit, as in splitk_reduce)
  if (dyn.limit) N = min(N, *dyn.limit - dyn.limit_off);
  if ((int)blockIdx.x * Cfg::BN >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wn = (warp & 1) * 32, wi = (warp >> 1) * (MT / 2);
  const int n0 = blockIdx.x * Cfg::BN;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int kbeg = split * kchunk;
  const int kend = min(K, kbeg + kchunk);
  constexpr int kBK = Cfg::BK, kPitchK = Cfg::PK, kStages = Cfg::NST;
  const int nk = kend > kbeg ? (int)cdiv(kend - kbeg, kBK) : 0;

  double acc[2][Cfg::NI][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::NI; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;

  TnLoader2<MT> ld2;
  if constexpr (VEC == 2) ld2.init(X, ldx, C, ldc, M, N, n0, dyn, smem, smem + Cfg::A_ELEMS);
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) {
      double* st = smem + s * Cfg::STAGE;
      if constexpr (VEC == 2)
        ld2.load((uint32_t)(s * Cfg::STAGE * 8), kbeg + s * kBK, kend);
      else
        tn_load_stage<MT, VEC>(st, st + Cfg::A_ELEMS, X, ldx, C, ldc, M, N, n0, kbeg + s * kBK, kend, dyn);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int ls = kt + kStages - 1;
      if (ls < nk) {
        double* st = smem + (ls % kStages) * Cfg::STAGE;
        if constexpr (VEC == 2)
          ld2.load((uint32_t)((ls % kStages) * Cfg::STAGE * 8), kbeg + ls * kBK, kend);
        else
          tn_load_stage<MT, VEC>(st, st + Cfg::A_ELEMS, X, ldx, C, ldc, M, N, n0, kbeg + ls * kBK,
                                 kend, dyn);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % kStages) * Cfg::STAGE;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double a[2][2], b[Cfg::NI];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a[mi][0] = sA[(wn + mi * 16 + g) * kPitchK + kk + t];
        a[mi][1] = sA[(wn + mi * 16 + g + 8) * kPitchK + kk + t];
      }
#pragma unroll
      for (int ni = 0; ni < Cfg::NI; ++ni) b[ni] = sB[(wi + ni * 8 + g) * kPitchK + kk + t];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ++ni) dmma16x8x4(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
    }
  }
  cp_async_wait<0>();

  if (nsplit > 1) {
    // Split-K: store the raw partial as part[split][n][i] (ld MT); the
    // separate splitk_reduce kernel sums the splits in index order.
    double* mine = part + (int64_t)split * Npart * MT;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn + mi * 16 + g + h * 8;
        if (n >= N) continue;
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ++ni) {
          const int i = wi + ni * 8 + 2 * t;
          __stcg(reinterpret_cast<double2*>(mine + (int64_t)n * MT + i),
                 make_double2(acc[mi][ni][h * 2], acc[mi][ni][h * 2 + 1]));
        }
      }
    return;
  }

  // Epilogue: D(i, n) = alpha * acc + beta * E(i, n).
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = n0 + wn + mi * 16 + g + h * 8;
      if (n >= N) continue;
#pragma unroll
      for (int ni = 0; ni < Cfg::NI; ++ni) {
        const int i = wi + ni * 8 + 2 * t;
        double v0 = alpha * acc[mi][ni][h * 2], v1 = alpha * acc[mi][ni][h * 2 + 1];
        if (beta != 0.0) {
          if (i < M) v0 += beta * E[(int64_t)n * lde + i];
          if (i + 1 < M) v1 += beta * E[(int64_t)n * lde + i + 1];
        }
        if (i < M) D[(int64_t)n * ldd + i] = v0;
        if (i + 1 < M) D[(int64_t)n * ldd + i + 1] = v1;
      }
    }
}

// Deterministic split-K reduction: D(i, n) = alpha * sum_s part[s][n][i] +
// beta * E(i, n), splits summed in index order, all SMs participating.
__global__ void __launch_bounds__(256)
    splitk_reduce_kernel(int M, int N, int MT, int nsplit, double alpha, const double* __restrict__ part,
                         double beta, const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, int n_lo,
                         int n_hi, int64_t pstride, int ncol0) {
  if (dyn.stop && *dyn.stop) return;
  if (dyn.shift) {
    const int sh = *dyn.shift;
    N -= sh;
    if (dyn.flags & kShiftD) {
      D += (int64_t)sh * ldd;
      if (E) E += (int64_t)sh * lde;
    }
  }
  // partial layout [split][column - ncol0][MT]: pstride elements per split (0: N * MT, N before the limit)
  const int64_t stride = pstride ? pstride : (int64_t)N * MT;
  if (dyn.limit) N = min(N, *dyn.limit - dyn.limit_off);
  N = min(N, n_hi);  // columns [n_lo, n_hi) of the output
  const int64_t total = (int64_t)M * max(N - n_lo, 0);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % M), n = n_lo + (int)(e / M);
    const double* src = part + (int64_t)(n - ncol0) * MT + i;
    double s = 0.0;
    int sp = 0;
    for (; sp + 8 <= nsplit; sp += 8) {
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = __ldcg(src + (sp + q) * stride);
#pragma unroll
      for (int q = 0; q < 8; ++q) s += x[q];
    }
    for (; sp < nsplit; ++sp) s += __ldcg(src + sp * stride);
    double v = alpha * s;
    if (beta != 0.0) v += beta * E[(int64_t)n * lde + i];
    D[(int64_t)n * ldd + i] = v;
  }
}

// gemm_nn split-K reduction: D(m, n) = alpha * sum_z part[z](m, n) + beta * E(m, n).
__global__ void __launch_bounds__(256)
    nn_splitk_reduce_kernel(int M, int N, int nsplit, double alpha, const double* __restrict__ part, double beta,
                            const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn) {
  if (dyn.stop && *dyn.stop) return;
  const int64_t total = (int64_t)M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(e % M), n = (int)(e / M);
    double s = 0.0;
    for (int z = 0; z < nsplit; ++z) s += __ldcg(part + z * total + e);
    double v = alpha * s;
    if (beta != 0.0) v = fma(beta, E[(int64_t)n * lde + m], v);
    D[(int64_t)n * ldd + m] = v;
  }
}

// ---------------------------------------------------------------- gemm_nn
// CTA tile 64 m x 128 n; 4 warps = 2 (m) x 2 (n); warp tile 32 m x 64 n.
// beta * E is read in the epilogue in two halves (32 values per thread in
// flight each), its latency covered by the SM's other CTA.
template <int VEC, int BNT = 128>
struct NnCfg {
  static constexpr int BM = 64, BN = BNT;
  static constexpr int NJ = BN / 16;  // n8 fragments per warp (2 x 2 warps)
  static constexpr int PM = BM + 4;   // pitch of the m-contiguous X tile (4 mod 16)
  static constexpr int A_ELEMS = kBK * PM;
  static constexpr int B_ELEMS = BN * kPitchK;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int SMEM = STAGE * kStagesNN * 8;
};

template <int VEC, int BNT>
__device__ __forceinline__ void nn_load_stage(double* sA, double* sB, const double* __restrict__ X,
                                              int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                              int M, int N, int K, int m0, int n0, int k0) {
  using Cfg = NnCfg<VEC, BNT>;
  const int tid = threadIdx.x;
  constexpr int CPM = Cfg::BM / VEC;  // chunks per k-row of X
#pragma unroll 4
  for (int c = tid; c < kBK * CPM; c += kThreads) {
    const int kr = c / CPM, mc = (c % CPM) * VEC;
    const int k = k0 + kr, m = m0 + mc;
    const bool ok = (k < K) && (m < M);
    const double* src = ok ? X + (int64_t)k * ldx + m : X;
    double* dst = sA + kr * Cfg::PM + mc;
    if constexpr (VEC == 2) {
      const int sz = ok ? ((m + 1 < M) ? 16 : 8) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                   "r"(sz));
    } else {
      cp_async<8>(dst, src, ok);
    }
  }
  constexpr int CPK = kBK / VEC;
#pragma unroll 4
  for (int c = tid; c < Cfg::BN * CPK; c += kThreads) {
    const int r = c / CPK, kc = (c % CPK) * VEC;
    const int n = n0 + r, k = k0 + kc;
    const bool ok = (n < N) && (k < K);
    const double* src = ok ? Y + (int64_t)n * ldy + k : Y;
    double* dst = sB + r * kPitchK + kc;
    if constexpr (VEC == 2) {
      const int sz = ok ? ((k + 1 < K) ? 16 : 8) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                   "r"(sz));
    } else {
      cp_async<8>(dst, src, ok);
    }
  }
}

// Aligned fast path of nn_load_stage (addresses and bounds resolved once).
template <int BNT>
struct NnLoader2 {
  static constexpr int BM = 64;
  static constexpr int ACH = BM / 2;                 // 16-byte chunks per k-row of X
  static constexpr int AR = kThreads / ACH;          // k-rows per pass
  static constexpr int NA = kBK / AR;
  static constexpr int BCH = kBK / 2;                // chunks per n-row of Y
  static constexpr int BR = kThreads / BCH;          // n-rows per pass
  static constexpr int NB = BNT / BR;
  const double* asrc;
  int64_t astep;
  const double* bsrc;
  int64_t bstep;
  uint32_t adst, bdst;
  int akr, bkc, K, asz;
  bool aok;
  unsigned bok;
  __device__ __forceinline__ void init(const double* X, int64_t ldx, const double* Y, int64_t ldy, int M, int N,
                                       int K_, int m0, int n0, const double* sA, const double* sB, int pm) {
    const int tid = threadIdx.x;
    K = K_;
    akr = tid / ACH;
    const int mc = (tid % ACH) * 2;
    aok = m0 + mc < M;
    asz = m0 + mc + 1 < M ? 16 : 8;  // odd M: the last pair is half valid
    asrc = X + (int64_t)akr * ldx + m0 + mc;
    astep = (int64_t)AR * ldx;
    adst = smem_u32(sA + akr * pm + mc);
    const int br = tid / BCH;
    bkc = (tid % BCH) * 2;
    bok = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i) bok |= ((n0 + br + BR * i) < N ? 1u : 0u) << i;
    bsrc = Y + (int64_t)(n0 + br) * ldy + bkc;
    bstep = (int64_t)BR * ldy;
    bdst = smem_u32(sB + br * kPitchK + bkc);
  }
  // A chunk needs m < M and k < K.
  __device__ __forceinline__ void load(uint32_t stage_off, int pm, int k0, const double* X,
                                       const double* Y) const {
    const double* a = asrc + (int64_t)k0 * (astep / AR);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int k = k0 + akr + AR * i;
      const bool ok = aok && k < K;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(adst + stage_off + i * AR * pm * 8),
                   "l"(ok ? a : X), "r"(ok ? asz : 0));
      a += astep;
    }
    const int k = k0 + bkc;
    const int sz = k < K ? (k + 1 < K ? 16 : 8) : 0;
    const double* b = bsrc + k0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const bool ok = (bok >> i) & 1u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(bdst + stage_off + i * BR * kPitchK * 8),
                   "l"(ok ? b : Y), "r"(ok ? sz : 0));
      b += bstep;
    }
  }
};

// CTA tile 64 m x BN n; 4 warps = 2 (m) x 2 (n); warp tile 32 m x BN/2 n.
template <int VEC, int BNT>
__global__ void __launch_bounds__(kThreads, SQR_NN_CTAS)
    gemm_nn_kernel(int M, int N, int K, double alpha, const double* __restrict__ X, int64_t ldx,
                   const double* __restrict__ Y, int64_t ldy, double beta, const double* E,
                   int64_t lde, double* D, int64_t ldd, GemmDyn dyn, int kchunk, double* part) {
  using Cfg = NnCfg<VEC, BNT>;
  constexpr int NJ = Cfg::NJ;
    extern __shared__ __align__(16) double smem[];
  if (dyn.stop && *dyn.stop) return;
  if (dyn.shift) {
    const int sh = *dyn.shift;
    N -= sh;
    if (dyn.flags & kShiftB) Y += (int64_t)sh * ldy;
    if (dyn.flags & kShiftD) {
      D += (int64_t)sh * ldd;
      if (E) E += (int64_t)sh * lde;
    }
  }
  if (dyn.limit) N = min(N, *dyn.limit - dyn.limit_off);
  // Grouped raster: CTAs in launch order walk groups of kNnGroup M-tiles
  // down all N-tiles, so the ~600 co-resident CTAs touch ~16 M-panels of X
  // and ~37 N-panels of Y instead of every X panel (a 67 MB X at K = 2b
  // would otherwise be re-fetched from DRAM by every wave).
  int mt, nt_;
  {
    const int tm = gridDim.x, tn = gridDim.y;
    const int lin = blockIdx.y * tm + blockIdx.x;
    const int per = kNnGroup * tn;
    const int first = (lin / per) * kNnGroup;
    const int gsz = min(tm - first, kNnGroup);
    const int r = lin % per;
    mt = first + r % gsz;
    nt_ = r / gsz;
  }
  const int m0 = mt * Cfg::BM, n0 = nt_ * Cfg::BN;
  if (n0 >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * (Cfg::BN / 2);
  // split-K (blockIdx.z): this CTA's K range [kbeg, kend); X and Y are
  // advanced so the loaders see a K-range starting at 0
  const int kbeg = blockIdx.z * kchunk;
  K = min(K, kbeg + kchunk) - kbeg;
  X += (int64_t)kbeg * ldx;
  Y += kbeg;
  const int nk = K > 0 ? (int)cdiv(K, kBK) : 0;
  double acc[2][NJ][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NJ; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;

  NnLoader2<BNT> ld2;
  if constexpr (VEC == 2) ld2.init(X, ldx, Y, ldy, M, N, K, m0, n0, smem, smem + Cfg::A_ELEMS, Cfg::PM);
#pragma unroll
  for (int s = 0; s < kStagesNN - 1; ++s) {
    if (s < nk) {
      double* st = smem + s * Cfg::STAGE;
      if constexpr (VEC == 2)
        ld2.load((uint32_t)(s * Cfg::STAGE * 8), Cfg::PM, s * kBK, X, Y);
      else
        nn_load_stage<VEC, BNT>(st, st + Cfg::A_ELEMS, X, ldx, Y, ldy, M, N, K, m0, n0, s * kBK);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<kStagesNN - 2>();
    __syncthreads();
    {
      const int ls = kt + kStagesNN - 1;
      if (ls < nk) {
        double* st = smem + (ls % kStagesNN) * Cfg::STAGE;
        if constexpr (VEC == 2)
          ld2.load((uint32_t)((ls % kStagesNN) * Cfg::STAGE * 8), Cfg::PM, ls * kBK, X, Y);
        else
          nn_load_stage<VEC, BNT>(st, st + Cfg::A_ELEMS, X, ldx, Y, ldy, M, N, K, m0, n0, ls * kBK);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % kStagesNN) * Cfg::STAGE;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double a[2][2], b[NJ];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a[mi][0] = sA[(kk + t) * Cfg::PM + wm + mi * 16 + g];
        a[mi][1] = sA[(kk + t) * Cfg::PM + wm + mi * 16 + g + 8];
      }
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) b[nj] = sB[(wn + nj * 8 + g) * kPitchK + kk + t];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) dmma16x8x4(acc[mi][nj], a[mi][0], a[mi][1], b[nj]);
    }
  }
  cp_async_wait<0>();

  if (part != nullptr) {
    // split-K: raw partial tile to part[z] (column-major M x N); the reduce
    // kernel sums the splits in index order (bitwise deterministic)
    double* mine = part + (int64_t)blockIdx.z * M * N;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + mi * 16 + g + h * 8;
        if (m >= M) continue;
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = n0 + wn + nj * 8 + 2 * t + e;
            if (n < N) __stcg(mine + (int64_t)n * M + m, acc[mi][nj][h * 2 + e]);
          }
      }
    return;
  }

  // Epilogue in 4 row chunks (mi, h); the beta*E loads of chunk c+1 are issued
  // before the stores of chunk c (E and D may alias in place, so the compiler
  // cannot hoist them itself: without this the chunks pay 4 serial round trips).
  auto load_e = [&](int c, double (&el)[NJ][2]) {
    const int mi = c >> 1, h = c & 1;
    const int m = m0 + wm + mi * 16 + g + h * 8;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn + nj * 8 + 2 * t + e;
        el[nj][e] = (beta != 0.0 && m < M && n < N) ? E[(int64_t)n * lde + m] : 0.0;
      }
  };
  double ea[NJ][2], eb[NJ][2];
  load_e(0, ea);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double (&cur)[NJ][2] = (c & 1) ? eb : ea;
    double (&nxt)[NJ][2] = (c & 1) ? ea : eb;
    if (c + 1 < 4) load_e(c + 1, nxt);
    const int mi = c >> 1, h = c & 1;
    const int m = m0 + wm + mi * 16 + g + h * 8;
    if (m >= M) continue;
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn + nj * 8 + 2 * t + e;
        if (n >= N) continue;
        double v = alpha * acc[mi][nj][h * 2 + e];
        if (beta != 0.0) v = fma(beta, cur[nj][e], v);
        D[(int64_t)n * ldd + m] = v;
      }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int MT, int VEC>
int launch_tn(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* C,
              int64_t ldc, double beta, const double* E, int64_t lde, double* D, int64_t ldd,
              double* ws, int64_t ws_bytes, GemmDyn dyn, cudaStream_t s) {
  using Cfg = TnCfg<MT, VEC>;
  if (int rc = smem_optin((const void*)gemm_tn_kernel<MT, VEC>, Cfg::SMEM)) return rc;
  const int tiles = (int)cdiv(N, Cfg::BN);
  const int sms = SQR_TN_MINB * sm_count();  // resident CTAs
  // Pick the split count that minimises waves/split (i.e. the padded work),
  // keeping >= 512 K per split; ties go to fewer splits.
  int best = 1;
  double best_cost = 1e30;
  const int max_split = std::max(1, std::min(sms, K / 512));
  for (int sp = 1; sp <= max_split; ++sp) {
    if ((int64_t)tiles * sp > 8LL * sms) break;  // bounded partial workspace
    const double waves = (double)cdiv((int64_t)tiles * sp, sms);
    const double cost = waves / sp + 0.02 * (sp > 1);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  int kchunk = (int)rup(cdiv(K, best), Cfg::BK);
  int nsplit = (int)cdiv(K, kchunk);
  if (nsplit < 1) nsplit = 1;
  double* part = nullptr;
  if (nsplit > 1) {
    const int64_t need = (int64_t)nsplit * N * MT * 8;
    if (ws == nullptr || ws_bytes < need) {
      nsplit = 1;
      kchunk = K;
    } else {
      part = ws;
    }
  }
  if (nsplit == 1) kchunk = std::max(K, 1);
  dim3 grid(tiles, nsplit);
  ProfScope ps(kTagGemmTn, s);
  gemm_tn_kernel<MT, VEC><<<grid, kThreads, Cfg::SMEM, s>>>(M, N, K, alpha, X, ldx, C, ldc, beta, E,
                                                           lde, D, ldd, kchunk, part, nullptr, dyn);
  SQR_LAUNCH("gemm_tn_kernel");
  if (nsplit > 1) return splitk_reduce_launch(M, N, MT, nsplit, alpha, part, beta, E, lde, D, ldd, dyn, s);
  if (dyn.pre_ready) SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
  return SQR_OK;
}

template <int MT>
int dispatch_tn_vec(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* C,
                    int64_t ldc, double beta, const double* E, int64_t lde, double* D, int64_t ldd,
                    double* ws, int64_t ws_bytes, GemmDyn dyn, cudaStream_t s) {
  const bool v2 = aligned16(X) && aligned16(C) && (ldx % 2 == 0) && (ldc % 2 == 0) &&
                  (dyn.npre == 0 || (aligned16(dyn.pre) && dyn.ldpre % 2 == 0));
  if (v2)
    return launch_tn<MT, 2>(M, N, K, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, ws, ws_bytes, dyn, s);
  return launch_tn<MT, 1>(M, N, K, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, ws, ws_bytes, dyn, s);
}

#ifndef SQR_NN_BN
#define SQR_NN_BN 64
#endif
template <int VEC>
int launch_nn(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* Y,
              int64_t ldy, double beta, const double* E, int64_t lde, double* D, int64_t ldd,
              GemmDyn dyn, cudaStream_t s, double* ws, int64_t ws_bytes) {
  using Cfg = NnCfg<VEC, SQR_NN_BN>;
  if (int rc = smem_optin((const void*)gemm_nn_kernel<VEC, SQR_NN_BN>, Cfg::SMEM)) return rc;
  const int64_t tiles = cdiv(M, Cfg::BM) * cdiv(N, Cfg::BN);
  // Split K when the tiles fill less than ~3 waves of resident CTAs and K is
  // long (skinny products such as TUXV's A V_k): splits of >= 1024 K, chosen
  // to minimise the padded waves; needs a caller workspace (static shapes
  // only: no dynamic shift / limit).
  int nsplit = 1;
  const int64_t slots = (int64_t)SQR_NN_CTAS * sm_count();
  if (ws != nullptr && dyn.shift == nullptr && dyn.limit == nullptr && K >= 2048 && tiles < 3 * slots) {
    double best = (double)cdiv(tiles, slots);
    for (int sp = 2; sp <= 16 && (int64_t)K / sp >= 1024; ++sp) {
      if ((int64_t)sp * M * N * 8 > ws_bytes) break;
      const double cost = (double)cdiv(tiles * sp, slots) / sp + 0.03;
      if (cost < best - 1e-9) {
        best = cost;
        nsplit = sp;
      }
    }
  }
  const int kchunk = nsplit > 1 ? (int)rup(cdiv(K, nsplit), kBK) : std::max(K, 1);
  nsplit = nsplit > 1 ? (int)cdiv(K, kchunk) : 1;
  dim3 grid((unsigned)cdiv(M, Cfg::BM), (unsigned)cdiv(N, Cfg::BN), (unsigned)nsplit);
  ProfScope ps(dyn.prof_tag >= 0 ? dyn.prof_tag : kTagGemmNn, s);
  gemm_nn_kernel<VEC, SQR_NN_BN><<<grid, kThreads, Cfg::SMEM, s>>>(M, N, K, alpha, X, ldx, Y, ldy, beta, E, lde,
                                                                  D, ldd, dyn, kchunk, nsplit > 1 ? ws : nullptr);
  SQR_LAUNCH("gemm_nn_kernel");
  if (nsplit > 1) {
    const int blocks = (int)std::min<int64_t>(cdiv((int64_t)M * N, 256), (int64_t)sm_count() * 8);
    nn_splitk_reduce_kernel<<<blocks, 256, 0, s>>>(M, N, nsplit, alpha, ws, beta, E, lde, D, ldd, dyn);
    SQR_LAUNCH("nn_splitk_reduce_kernel");
  }
  return SQR_OK;
}

}  // namespace

// Fixed-order split-K reduction shared with the TMA kernel (gemm_tma.cu).
int splitk_reduce_range(int M, int N, int MT, int nsplit, double alpha, const double* part, double beta,
                        const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, int n_lo, int n_hi,
                        int64_t pstride, int ncol0, cudaStream_t s) {
  const int64_t cols = std::max<int64_t>(1, (int64_t)std::min(N, n_hi) - n_lo);
  const int blocks = (int)std::min<int64_t>(cdiv((int64_t)M * cols, 256), (int64_t)sm_count() * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, s>>>(M, N, MT, nsplit, alpha, part, beta, E, lde, D, ldd, dyn, n_lo, n_hi,
                                              pstride, ncol0);
  SQR_LAUNCH("splitk_reduce_kernel");
  return SQR_OK;
}

int splitk_reduce_launch(int M, int N, int MT, int nsplit, double alpha, const double* part, double beta,
                         const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, cudaStream_t s) {
  int n_lo = 0;
  if (dyn.pre_ready && dyn.npre > 0 && dyn.npre < N) {
    // the Gram prefix first: T is built beside the reduction of the other columns
    if (int rc = splitk_reduce_range(M, N, MT, nsplit, alpha, part, beta, E, lde, D, ldd, dyn, 0, dyn.npre, 0, 0, s))
      return rc;
    SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
    n_lo = dyn.npre;
  }
  if (int rc = splitk_reduce_range(M, N, MT, nsplit, alpha, part, beta, E, lde, D, ldd, dyn, n_lo, INT_MAX, 0, 0, s))
    return rc;
  if (dyn.pre_ready && n_lo == 0) SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
  return SQR_OK;
}

int gemm_tn_tma(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* C, int64_t ldc,
                double beta, const double* E, int64_t lde, double* D, int64_t ldd, double* ws, int64_t ws_bytes,
                cudaStream_t s, GemmDyn dyn);

int gemm_tn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
            const double* C, int64_t ldc, double beta, const double* E, int64_t lde, double* D,
            int64_t ldd, double* ws, int64_t ws_bytes, cudaStream_t s, GemmDyn dyn) {
  if (M <= 0 || N <= 0) return SQR_OK;
  if (M > 144 || K < 0) {
    set_error("gemm_tn: M=%lld must be in [1,144]", (long long)M);
    return SQR_EINVAL;
  }
  if (beta != 0.0 && E == nullptr) E = D;
  const int m = (int)M, n = (int)N, k = (int)K;
  {
    const int rc = gemm_tn_tma(m, n, k, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, ws, ws_bytes, s, dyn);
    if (rc != -1) return rc;
  }
#define SQR_TN(MT)                                                                                  \
  if (M <= MT)                                                                                      \
    return dispatch_tn_vec<MT>(m, n, k, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, ws, ws_bytes, dyn, s);
  SQR_TN(16) SQR_TN(32) SQR_TN(48) SQR_TN(64) SQR_TN(80) SQR_TN(96) SQR_TN(112) SQR_TN(128) SQR_TN(144)
#undef SQR_TN
  return SQR_EINVAL;
}

int gemm_nn_tma(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                double beta, const double* E, int64_t lde, double* D, int64_t ldd, cudaStream_t s, GemmDyn dyn);

int gemm_nn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
            const double* Y, int64_t ldy, double beta, const double* E, int64_t lde, double* D,
            int64_t ldd, cudaStream_t s, GemmDyn dyn, double* ws, int64_t ws_bytes) {
  if (M <= 0 || N <= 0) return SQR_OK;
  if (beta != 0.0 && E == nullptr) E = D;
  // TMA path unless launch_nn would split K (skinny long-K products with a workspace)
  if (!(ws != nullptr && dyn.shift == nullptr && dyn.limit == nullptr && K >= 2048)) {
    const int rc = gemm_nn_tma((int)M, (int)N, (int)K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd, s, dyn);
    if (rc != -1) return rc;
  }
  const bool v2 = aligned16(X) && aligned16(Y) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                  (beta == 0.0 || (aligned16(E) && lde % 2 == 0));
  if (v2)
    return launch_nn<2>((int)M, (int)N, (int)K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd, dyn, s, ws, ws_bytes);
  return launch_nn<1>((int)M, (int)N, (int)K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd, dyn, s, ws, ws_bytes);
}

int64_t gemm_tn_workspace(int64_t N, int64_t /*K*/) {
  const int64_t tiles = cdiv(N, 128);
  return tiles * 148 * (2 * 9 * 4) * kThreads * 8 / 8 + tiles * 4 + 64;
}

}  // namespace sqr

extern "C" int sqr_gemm_tn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                           const double* C, int64_t ldc, double beta, const double* E, int64_t lde,
                           double* D, int64_t ldd, double* workspace, int64_t workspace_bytes,
                           void* stream) {
  return sqr::gemm_tn(M, N, K, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, workspace,
                      workspace_bytes, static_cast<cudaStream_t>(stream), sqr::GemmDyn{});
}

extern "C" int sqr_gemm_nn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                           const double* Y, int64_t ldy, double beta, const double* E, int64_t lde,
                           double* D, int64_t ldd, void* stream) {
  return sqr::gemm_nn(M, N, K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd,
                      static_cast<cudaStream_t>(stream), sqr::GemmDyn{});
}

extern "C" int sqr_gemm_nn_ws(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                              const double* Y, int64_t ldy, double beta, const double* E, int64_t lde,
                              double* D, int64_t ldd, double* workspace, int64_t workspace_bytes, void* stream) {
  return sqr::gemm_nn(M, N, K, alpha, X, ldx, Y, ldy, beta, E, lde, D, ldd, static_cast<cudaStream_t>(stream),
                      sqr::GemmDyn{}, workspace, workspace_bytes);
}
