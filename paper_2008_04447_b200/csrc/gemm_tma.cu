// gemm_tn with TMA-staged operands and a warp-specialised mbarrier pipeline
// (sm_100a).  Same contract and arithmetic as gemm_tn_kernel in gemm.cu
// (randomized.py:206 first sweep Y^T [Y | C], sketch.py:70-71 Omega A,
// randomized.py:322 Y2^T A):
//
//   D(MxN) = alpha * X^T C + beta * E,  computed as D^T = C^T X,
//   CTA tile 64 n x MT i, 4 consumer warps (2 n x 2 i, warp tile 32 n x MT/2 i)
//   issuing m16n8k4 f64 MMAs (SASS DMMA.8x8x4; fp64 has no tcgen05 path),
//   plus one producer warp whose elected lane streams K-stages of 16 with
//   cp.async.bulk.tensor (2-D tensor maps, SWIZZLE_128B: a 16-double k-row
//   is one 128-byte line, its 16-byte chunks XOR-permuted by row % 8, so the
//   fragment gathers -- 8 rows x 2 chunks per warp -- are conflict-free
//   without padding) into an NST-deep ring of full / empty mbarriers.
//   Consumers never meet at a CTA barrier: each waits on the stage's full
//   barrier and releases it with one arrive per warp.
//
// Out-of-range rows / columns / k are zero-filled by the TMA unit, so the
// kernel has no bounds predicates in its loads.  The device-side dynamic
// shape of GemmDyn (stop, shift of the C operand / of D and E, limit, and a
// 64-aligned prefix taken from a second operand) is honoured: the C tensor
// map covers the whole unshifted operand and the shift moves the TMA
// coordinate.  Split-K partials go to the same workspace layout as
// gemm_tn_kernel and are reduced by its fixed-order splitk_reduce kernel, so
// results are bitwise identical to that kernel's.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstdio>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace sqr {

int splitk_reduce_launch(int M, int N, int MT, int nsplit, double alpha, const double* part, double beta,
                         const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, cudaStream_t s);
int splitk_reduce_range(int M, int N, int MT, int nsplit, double alpha, const double* part, double beta,
                        const double* E, int64_t lde, double* D, int64_t ldd, GemmDyn dyn, int n_lo, int n_hi,
                        int64_t pstride, int ncol0, cudaStream_t s);

namespace {

constexpr int kTmaBN = 64;       // n rows per CTA tile
constexpr int kTmaBK = 16;       // k per stage: one 128-byte swizzle line per row
constexpr int kTmaConsumers = 4;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;

template <int MT>
struct TmaCfg {
  static constexpr int NI = MT / 16;
  static constexpr int A_BYTES = kTmaBN * kTmaBK * 8;  // 8 KB
  static constexpr int B_BYTES = MT * kTmaBK * 8;      // MT rows of 128 B
  static constexpr int STAGE = A_BYTES + B_BYTES;      // multiple of 1024 (MT % 8 == 0)
  static constexpr int NST = MT <= 128 ? 4 : 4;
  static constexpr int SMEM = STAGE * NST + 1024;      // + alignment slack
};

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  while (!mbar_try_wait(a, parity)) {
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

template <int MT>
__global__ void __launch_bounds__(kTmaThreads, 2)
    gemm_tn_tma_kernel(const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapP,
                       const __grid_constant__ CUtensorMap mapX, int M, int N, int K, double alpha, double beta,
                       const double* E, int64_t lde, double* D, int64_t ldd, int kchunk, double* part,
                       GemmDyn dyn, int tile0, int64_t pstride, int ncol0) {
  using Cfg = TmaCfg<MT>;
  constexpr int NST = Cfg::NST;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  if (dyn.stop && *dyn.stop) return;
  int sh = 0;
  if (dyn.shift) {
    sh = *dyn.shift;
    N -= sh;
    if (dyn.flags & kShiftD) {
      D += (int64_t)sh * ldd;
      if (E) E += (int64_t)sh * lde;
    }
  }
  const int Npart = N;  // split-K partial stride (before the limit, as in splitk_reduce)
  if (dyn.limit) N = min(N, *dyn.limit - dyn.limit_off);
  const int n0 = (blockIdx.x + tile0) * kTmaBN;  // tile0: this launch covers the tiles from tile0 on
  if (n0 >= N) return;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int kbeg = split * kchunk;
  const int kend = min(K, kbeg + kchunk);
  const int nk = kend > kbeg ? (int)cdiv(kend - kbeg, kTmaBK) : 0;
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kTmaConsumers) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const bool pre = n0 < dyn.npre;  // the prefix is 64-aligned: a tile is all prefix or all C
      const CUtensorMap* ma = pre ? &mapP : &mapC;
      const int an = pre ? n0 : n0 - dyn.npre + ((dyn.flags & kShiftB) ? sh : 0);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % NST;
        if (kt >= NST) mbar_wait(smem_u32(&empty[s]), ((kt / NST) & 1) ^ 1);
        const uint32_t fb = smem_u32(&full[s]);
        mbar_expect_tx(fb, Cfg::STAGE);
        const uint32_t dst = sbase + s * Cfg::STAGE;
        const int k = kbeg + kt * kTmaBK;
        tma_load_2d(dst, ma, k, an, fb);
        tma_load_2d(dst + Cfg::A_BYTES, &mapX, k, 0, fb);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int g = lane >> 2, t = lane & 3;
  const int wn = (warp & 1) * 32, wi = (warp >> 1) * (MT / 2);
  double acc[2][Cfg::NI][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::NI; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  // swizzled byte offset of (row, k) inside a tile: row * 128 + ((k / 2) ^ (row % 8)) * 16 + (k % 2) * 8,
  // with row % 8 == g for every fragment row (row bases are multiples of 8)
  uint32_t koff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = 4 * q + t;
    koff[q] = (uint32_t)((((k >> 1) ^ g) << 4) | ((k & 1) << 3));
  }
  const uint32_t arow0 = (uint32_t)(wn + g) * 128u, brow0 = (uint32_t)(wi + g) * 128u;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % NST;
    mbar_wait(smem_u32(&full[s]), (kt / NST) & 1);
    const uint32_t sa = sbase + s * Cfg::STAGE, sb = sa + Cfg::A_BYTES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double a[2][2], b[Cfg::NI];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const uint32_t ra = sa + arow0 + (uint32_t)(mi * 16) * 128u + koff[q];
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a[mi][0]) : "r"(ra));
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a[mi][1]) : "r"(ra + 8u * 128u));
      }
#pragma unroll
      for (int ni = 0; ni < Cfg::NI; ++ni) {
        const uint32_t rb = sb + brow0 + (uint32_t)(ni * 8) * 128u + koff[q];
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(b[ni]) : "r"(rb));
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ++ni) dmma16x8x4(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
  }

  if (nsplit > 1) {
    // partial layout [split][column - ncol0][MT]; pstride = elements per split (0: N * MT)
    double* mine = part + (int64_t)split * (pstride ? pstride : (int64_t)Npart * MT) - (int64_t)ncol0 * MT;
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


// ------------------------------------------------------------------ gemm_nn
// D(MxN) = alpha * X Y + beta * E (randomized.py:207 second sweep C -= Y W,
// merged over a block pair with K = 2b).  CTA tile 64 m x 128 n, 4 consumer
// warps (2 m x 2 n, warp tile 32 m x 64 n), one producer warp.  X is
// m-contiguous: a stage holds it as 8 boxes of {8 m, 16 k} (64-byte rows,
// SWIZZLE_64B: chunk ^= (k / 2) % 4), which makes the A-fragment gather --
// 4 k-rows x 8 consecutive m per warp -- conflict-free; Y is k-contiguous and
// staged like gemm_tn's operands (128-byte rows, SWIZZLE_128B).  The beta * E
// tile (64 m x 128 n, 64 KB) is fetched by the producer into ring slots as
// they drain after the last K-stage, so the epilogue reads E from shared
// memory (no exposed global latency, no E registers: the 168-register
// budget of two 5-warp CTAs per SM holds only the accumulators).
constexpr int kNnXBox = 8 * kTmaBK * 8;                          // 1 KB per {8 m, 16 k} box
constexpr int kNnEBoxM = 64, kNnEBoxN = 32;                     // E box {64 m, 32 n} = 16 KB
constexpr int kNnEBox = kNnEBoxM * kNnEBoxN * 8;
#ifndef SQR_NN_TMA_GROUP
#define SQR_NN_TMA_GROUP 16
#endif
#ifndef SQR_NN_E_PREFETCH
#define SQR_NN_E_PREFETCH 1
#endif
constexpr bool kNnEPrefetch = SQR_NN_E_PREFETCH != 0;
// Tile BM x BN, consumer warps (BM / 32) x (BN / WTN) with warp tile 32 x WTN,
// NST-deep ring, CTAS resident per SM.
template <int BM, int BN, int WTN, int NST, int CTAS>
struct NnTma {
  static constexpr int CW = (BM / 32) * (BN / WTN);  // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int XBYTES = (BM / 8) * kNnXBox;
  static constexpr int YBYTES = BN * kTmaBK * 8;
  static constexpr int STAGE = XBYTES + YBYTES;
  static constexpr int EBOXES = (BM / kNnEBoxM) * (BN / kNnEBoxN);
  static constexpr int SMEM = STAGE * NST + 1024;
  static_assert(EBOXES <= NST && kNnEBox <= STAGE, "E tile must fit the drained ring");
};

template <int BM, int BN, int WTN, int NST, int CTAS>
__global__ void __launch_bounds__(NnTma<BM, BN, WTN, NST, CTAS>::THREADS, CTAS)
    gemm_nn_tma_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapY,
                       const __grid_constant__ CUtensorMap mapE, int M, int N, int K, double alpha, double beta,
                       double* D, int64_t ldd, GemmDyn dyn, int x3d) {
  using Cfg = NnTma<BM, BN, WTN, NST, CTAS>;
  constexpr int NJ = WTN / 8, CW = Cfg::CW, STAGE = Cfg::STAGE, EBOXES = Cfg::EBOXES;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], ebar;
  if (dyn.stop && *dyn.stop) return;
  int sh = 0;
  if (dyn.shift) {
    sh = *dyn.shift;
    N -= sh;
    if (dyn.flags & kShiftD) D += (int64_t)sh * ldd;
  }
  if (dyn.limit) N = min(N, *dyn.limit - dyn.limit_off);
  // grouped raster (as gemm_nn_kernel): a wave touches ~16 M-panels of X
  int mt, ntile;
  {
    const int tm = gridDim.x, tn = gridDim.y;
    const int lin = blockIdx.y * tm + blockIdx.x;
    const int per = SQR_NN_TMA_GROUP * tn;
    const int first = (lin / per) * SQR_NN_TMA_GROUP;
    const int gsz = min(tm - first, SQR_NN_TMA_GROUP);
    const int r = lin % per;
    mt = first + r % gsz;
    ntile = r / gsz;
  }
  const int m0 = mt * BM, n0 = ntile * BN;
  if (n0 >= N) return;
  const int nk = K > 0 ? (int)cdiv(K, kTmaBK) : 0;
  const bool use_e = beta != 0.0;
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), CW);
    }
    mbar_init(smem_u32(&ebar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    if (lane == 0) {
      const int yn = n0 + ((dyn.flags & kShiftB) ? sh : 0);
      if (use_e && kNnEPrefetch) {
        // the beta E tile is read after the last stage: start pulling it from
        // HBM into L2 now, so its epilogue TMA is an L2 hit
        const int en = n0 + ((dyn.flags & kShiftD) ? sh : 0);
        for (int e = 0; e < EBOXES; ++e)
          tma_prefetch_2d(&mapE, m0 + (e % (BM / kNnEBoxM)) * kNnEBoxM, en + (e / (BM / kNnEBoxM)) * kNnEBoxN);
      }
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % NST;
        if (kt >= NST) mbar_wait(smem_u32(&empty[s]), ((kt / NST) & 1) ^ 1);
        const uint32_t fb = smem_u32(&full[s]);
        mbar_expect_tx(fb, STAGE);
        const uint32_t dst = sbase + s * STAGE;
        const int k = kt * kTmaBK;
        if (x3d) {
          // one 3-D box {8 m, 16 k, BM / 8 groups} lands as the BM / 8 boxes of the 2-D path
          tma_load_3d(dst, &mapX, 0, k, m0 / 8, fb);
        } else {
#pragma unroll
          for (int q = 0; q < BM / 8; ++q) tma_load_2d(dst + q * kNnXBox, &mapX, m0 + 8 * q, k, fb);
        }
        tma_load_2d(dst + Cfg::XBYTES, &mapY, k, yn, fb);
      }
      if (use_e) {
        // E box e = (m half, n quarter) goes to the e-th slot to drain after the last stage
        const uint32_t eb = smem_u32(&ebar);
        mbar_expect_tx(eb, EBOXES * kNnEBox);
        const int en = n0 + ((dyn.flags & kShiftD) ? sh : 0);
        for (int e = 0; e < EBOXES; ++e) {
          const int kt = nk + e;
          const int s = kt % NST;
          if (kt >= NST) mbar_wait(smem_u32(&empty[s]), ((kt / NST) & 1) ^ 1);
          const int em = e % (BM / kNnEBoxM), enq = e / (BM / kNnEBoxM);
          tma_load_2d(sbase + s * STAGE, &mapE, m0 + em * kNnEBoxM, en + enq * kNnEBoxN, eb);
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % (BM / 32)) * 32, wn = (warp / (BM / 32)) * WTN;
  double acc[2][NJ][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NJ; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
  // X box row k holds 8 m; byte offset of (m % 8 = g, k):
  //   k * 64 + ((g / 2) ^ ((k / 2) % 4)) * 16 + (g % 2) * 8
  uint32_t xoff[4], yoff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = 4 * q + t;
    xoff[q] = (uint32_t)(k * 64 + ((((g >> 1) ^ ((k >> 1) & 3))) << 4) + ((g & 1) << 3));
    yoff[q] = (uint32_t)((((k >> 1) ^ g) << 4) | ((k & 1) << 3));
  }
  const uint32_t xbox0 = (uint32_t)(wm / 8) * kNnXBox;  // box of rows wm .. wm + 7
  const uint32_t yrow0 = (uint32_t)(wn + g) * 128u;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % NST;
    mbar_wait(smem_u32(&full[s]), (kt / NST) & 1);
    const uint32_t sx = sbase + s * STAGE, sy = sx + Cfg::XBYTES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double a[2][2], b[NJ];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const uint32_t ra = sx + xbox0 + (uint32_t)(mi * 2) * kNnXBox + xoff[q];
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a[mi][0]) : "r"(ra));
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a[mi][1]) : "r"(ra + kNnXBox));
      }
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        const uint32_t rb = sy + yrow0 + (uint32_t)(nj * 8) * 128u + yoff[q];
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(b[nj]) : "r"(rb));
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj) dmma16x8x4(acc[mi][nj], a[mi][0], a[mi][1], b[nj]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
  }
  // epilogue: D = alpha acc + beta E, E from the drained ring (box (ml / 64,
  // nl / 32) in slot (nk + box) % NST, element at (nl % 32) * 512 + (ml % 64) * 8)
  if (use_e) mbar_wait(smem_u32(&ebar), 0);
  // alpha == 1 (the trailing updates) skips the multiply: epilogue fp64 ops
  // issue on the same pipe as the DMMAs of the SM's other CTAs
  auto epilogue = [&](auto unit) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ml = wm + mi * 16 + g + h * 8;
        const int m = m0 + ml;
        if (m >= M) continue;
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nl = wn + nj * 8 + 2 * t + e;
            const int n = n0 + nl;
            if (n >= N) continue;
            double v = decltype(unit)::value ? acc[mi][nj][h * 2 + e] : alpha * acc[mi][nj][h * 2 + e];
            if (use_e) {
              const int box = (ml / kNnEBoxM) + (BM / kNnEBoxM) * (nl / kNnEBoxN);
              const uint32_t ea = sbase + ((nk + box) % NST) * STAGE +
                                  (uint32_t)((nl % kNnEBoxN) * kNnEBoxM + ml % kNnEBoxM) * 8u;
              double ev;
              asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(ev) : "r"(ea));
              v = fma(beta, ev, v);
            }
            D[(int64_t)n * ldd + m] = v;
          }
      }
  };
  if (alpha == 1.0)
    epilogue(std::true_type{});
  else
    epilogue(std::false_type{});
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

// 2-D map over a column-major operand: dims {rows (k, contiguous), cols}, box
// {16 k, box_cols}, 128-byte swizzle, zero fill out of range.
bool make_map(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
              int box_rows = kTmaBK, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn || rows < 1 || cols < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int MT>
int launch_tn_tma(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* C, int64_t ldc,
                  double beta, const double* E, int64_t lde, double* D, int64_t ldd, double* ws, int64_t ws_bytes,
                  GemmDyn dyn, cudaStream_t s) {
  using Cfg = TmaCfg<MT>;
  CUtensorMap mC, mP, mX;
  const int ncols = N - dyn.npre;  // columns taken from C (before any device-side shift)
  if (!make_map(&mX, X, K, M, ldx, MT)) return -1;
  if (ncols > 0) {
    if (!make_map(&mC, C, K, ncols, ldc, kTmaBN)) return -1;
  } else {
    mC = mX;  // never read
  }
  if (dyn.npre > 0) {
    if (!make_map(&mP, dyn.pre, K, dyn.npre, dyn.ldpre, kTmaBN)) return -1;
  } else {
    mP = mX;  // never read
  }
  if (int rc = smem_optin((const void*)gemm_tn_tma_kernel<MT>, Cfg::SMEM)) return rc;
  const int tiles = (int)cdiv(N, kTmaBN);
  const int sms = 2 * sm_count();  // resident CTAs
  int best = 1;
  double best_cost = 1e30;
  const int max_split = std::max(1, std::min(sms, K / 512));
  for (int sp = 1; sp <= max_split; ++sp) {
    if ((int64_t)tiles * sp > 8LL * sms) break;
    const double waves = (double)cdiv((int64_t)tiles * sp, sms);
    const double cost = waves / sp + 0.02 * (sp > 1);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = sp;
    }
  }
  // Two launches for long sweeps: with equal-length CTAs the last wave of tiles * sp CTAs leaves part of
  // the chip idle for a whole CTA duration (3.2% of the C5 first sweeps).  The tiles that fill whole
  // waves at split sp go first; the rest run at a higher split sp2, one more wave of shorter CTAs
  // (0.5% left).  Only for wide outputs (the drivers' sweeps); other shapes keep the single launch,
  // whose results are bitwise those of the cp.async kernel.
  static const bool no_two = env_flag("SQR_NO_TN_TAIL_SPLIT");
  constexpr int kTailMinK = 512;       // shortest K chunk of the tail launch (1024: same; measured)
  constexpr double kTailCost = 0.03;   // second launch + longer reduction, in CTA durations (0.01-0.06: +-2 ms)
  int t1 = tiles, t2 = 0, sp2 = 1;
  if (!no_two && dyn.limit == nullptr && tiles >= sms / 2 && ws != nullptr) {
    const int pre_tiles = (int)cdiv(dyn.npre, kTmaBN);
    for (int sp = 1; sp <= max_split; ++sp) {
      if ((int64_t)tiles * sp > 8LL * sms) break;
      const int full = (int)(((int64_t)tiles * sp) / sms);
      if (full == 0) continue;
      const int c1 = std::min(tiles, (int)(((int64_t)full * sms) / sp)), c2 = tiles - c1;
      if (c2 == 0 || c1 < pre_tiles) continue;
      const int s2 = std::min(std::min(max_split, sms / c2), std::max(1, K / kTailMinK));
      if (s2 <= sp) continue;
      const double cost = (double)full / sp + 1.0 / s2 + kTailCost;
      const int64_t need = ((int64_t)sp * c1 + (int64_t)s2 * c2) * kTmaBN * MT * 8;
      if (cost < best_cost - 1e-9 && need <= ws_bytes) {
        best_cost = cost;
        best = sp;
        t1 = c1;
        t2 = c2;
        sp2 = s2;
      }
    }
  }
  auto chunk_of = [&](int sp, int* nsp) {
    int kc = (int)rup(cdiv(K, sp), kTmaBK);
    *nsp = std::max(1, (int)cdiv(K, kc));
    if (*nsp == 1) kc = std::max(K, 1);
    return kc;
  };
  if (t2 > 0) {
    int ns1 = 1, ns2 = 1;
    const int kc1 = chunk_of(best, &ns1), kc2 = chunk_of(sp2, &ns2);
    const int64_t ps1 = (int64_t)t1 * kTmaBN * MT, ps2 = (int64_t)t2 * kTmaBN * MT;
    double* part2 = ws + (int64_t)ns1 * ps1;
    const int n1 = t1 * kTmaBN;
    ProfScope ps(kTagGemmTn, s);
    gemm_tn_tma_kernel<MT><<<dim3(t1, ns1), kTmaThreads, Cfg::SMEM, s>>>(mC, mP, mX, M, N, K, alpha, beta, E, lde, D,
                                                                         ldd, kc1, ns1 > 1 ? ws : nullptr, dyn, 0,
                                                                         ps1, 0);
    SQR_LAUNCH("gemm_tn_tma_kernel");
    if (ns1 == 1 && dyn.pre_ready) SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
    gemm_tn_tma_kernel<MT><<<dim3(t2, ns2), kTmaThreads, Cfg::SMEM, s>>>(mC, mP, mX, M, N, K, alpha, beta, E, lde, D,
                                                                         ldd, kc2, ns2 > 1 ? part2 : nullptr, dyn,
                                                                         t1, ps2, n1);
    SQR_LAUNCH("gemm_tn_tma_kernel");
    if (ns1 > 1) {
      int lo = 0;
      if (dyn.pre_ready && dyn.npre > 0 && dyn.npre < n1) {
        if (int rc = splitk_reduce_range(M, N, MT, ns1, alpha, ws, beta, E, lde, D, ldd, dyn, 0, dyn.npre, ps1, 0, s))
          return rc;
        SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
        lo = dyn.npre;
      }
      if (int rc = splitk_reduce_range(M, N, MT, ns1, alpha, ws, beta, E, lde, D, ldd, dyn, lo, n1, ps1, 0, s))
        return rc;
      if (dyn.pre_ready && lo == 0) SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
    }
    if (ns2 > 1)
      return splitk_reduce_range(M, N, MT, ns2, alpha, part2, beta, E, lde, D, ldd, dyn, n1, INT_MAX, ps2, n1, s);
    return SQR_OK;
  }
  int kchunk = (int)rup(cdiv(K, best), kTmaBK);
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
  gemm_tn_tma_kernel<MT><<<grid, kTmaThreads, Cfg::SMEM, s>>>(mC, mP, mX, M, N, K, alpha, beta, E, lde, D, ldd,
                                                               kchunk, part, dyn, 0, 0, 0);
  SQR_LAUNCH("gemm_tn_tma_kernel");
  if (nsplit > 1) return splitk_reduce_launch(M, N, MT, nsplit, alpha, part, beta, E, lde, D, ldd, dyn, s);
  if (dyn.pre_ready) SQR_CUDA(cudaEventRecord(dyn.pre_ready, s));
  return SQR_OK;
}

}  // namespace

// Returns SQR_OK / an error code when it handled the call, -1 when the operands
// do not qualify (unaligned, prefix not 64-aligned, no tensor-map entry point):
// the caller then runs the cp.async kernel.
int gemm_tn_tma(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* C, int64_t ldc,
                double beta, const double* E, int64_t lde, double* D, int64_t ldd, double* ws, int64_t ws_bytes,
                cudaStream_t s, GemmDyn dyn) {
  if (env_flag("SQR_NO_TMA") || K < kTmaBK) return -1;  // read per call (A/B tests)
  if (!al16(X) || (ldx & 1) || ldx < 2) return -1;
  if (N - dyn.npre > 0 && (!al16(C) || (ldc & 1))) return -1;
  if (dyn.npre > 0 && (dyn.npre % kTmaBN != 0 || !al16(dyn.pre) || (dyn.ldpre & 1))) return -1;
#define SQR_TMA(MT) \
  if (M <= MT) return launch_tn_tma<MT>(M, N, K, alpha, X, ldx, C, ldc, beta, E, lde, D, ldd, ws, ws_bytes, dyn, s);
  SQR_TMA(16) SQR_TMA(32) SQR_TMA(48) SQR_TMA(64) SQR_TMA(80) SQR_TMA(96) SQR_TMA(112) SQR_TMA(128)
#undef SQR_TMA
  // M in (128, 144] (the sketch, l = b + p rows) stays on the cp.async kernel:
  // measured 31.4 vs 32.1 TFLOP/s on the C5 sketch (the 144-row tile spills at
  // the 2-CTA register budget of the 5-warp CTA)
  return -1;
}


template <int BM, int BN, int WTN, int NST, int CTAS>
int launch_nn_tma(const CUtensorMap& mX, const CUtensorMap& mY, const CUtensorMap& mE, int M, int N, int K,
                  double alpha, double beta, double* D, int64_t ldd, cudaStream_t s, GemmDyn dyn, int x3d) {
  using Cfg = NnTma<BM, BN, WTN, NST, CTAS>;
  auto kern = gemm_nn_tma_kernel<BM, BN, WTN, NST, CTAS>;
  if (int rc = smem_optin((const void*)kern, Cfg::SMEM)) return rc;
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN));
  ProfScope ps(dyn.prof_tag >= 0 ? dyn.prof_tag : kTagGemmNn, s);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(mX, mY, mE, M, N, K, alpha, beta, D, ldd, dyn, x3d);
  SQR_LAUNCH("gemm_nn_tma_kernel");
  return SQR_OK;
}

#ifndef SQR_NN_TMA_CFG
#define SQR_NN_TMA_CFG 0
#endif

int gemm_nn_tma(int M, int N, int K, double alpha, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                double beta, const double* E, int64_t lde, double* D, int64_t ldd, cudaStream_t s, GemmDyn dyn) {
  if (env_flag("SQR_NO_TMA") || K < 1 || M < 1 || N < 1) return -1;
  if (!al16(X) || (ldx & 1) || !al16(Y) || (ldy & 1)) return -1;
  if (beta != 0.0 && (!al16(E) || (lde & 1))) return -1;
  // config: 0 = 64 x 64 (4 warps, 3 stages, 4 CTAs/SM); 1 = 128 x 64 (8 warps, 4 stages, 2 CTAs/SM);
  //         2 = 64 x 128 (8 warps, 4 stages, 2 CTAs/SM)
  const int cfg = SQR_NN_TMA_CFG;
  const int bm = cfg == 1 ? 128 : 64, bn = cfg == 2 ? 128 : 64;
  CUtensorMap mX, mY, mE;
  // X: M % 8 == 0 -> one 3-D map {8 m, k, m / 8} (strides ldx, 64 bytes) loaded with one TMA per stage;
  // otherwise 2-D boxes {8 m, 16 k}
  int x3d = (M % 8 == 0 && !env_flag("SQR_NN_X2D")) ? 1 : 0;
  if (x3d) {
    auto fn = encode_fn();
    cuuint64_t dims[3] = {8, (cuuint64_t)K, (cuuint64_t)(M / 8)};
    cuuint64_t strides[2] = {(cuuint64_t)ldx * 8, 64};
    cuuint32_t box[3] = {8, (cuuint32_t)kTmaBK, (cuuint32_t)(bm / 8)};
    cuuint32_t estr[3] = {1, 1, 1};
    if (!fn || fn(&mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      x3d = 0;
  }
  if (!x3d && !make_map(&mX, X, M, K, ldx, kTmaBK, 8, CU_TENSOR_MAP_SWIZZLE_64B)) return -1;
  if (env_flag("SQR_TMA_DEBUG")) fprintf(stderr, "gemm_nn_tma M=%d N=%d K=%d x3d=%d\n", M, N, K, x3d);
  if (!make_map(&mY, Y, K, N, ldy, bn)) return -1;
  if (beta != 0.0) {
    if (!make_map(&mE, E, M, N, lde, kNnEBoxN, kNnEBoxM, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  } else {
    mE = mX;  // never read
  }
    if (cfg == 1) return launch_nn_tma<128, 64, 32, 4, 2>(mX, mY, mE, M, N, K, alpha, beta, D, ldd, s, dyn, x3d);
  if (cfg == 2) return launch_nn_tma<64, 128, 32, 4, 2>(mX, mY, mE, M, N, K, alpha, beta, D, ldd, s, dyn, x3d);
  return launch_nn_tma<64, 64, 32, 3, 4>(mX, mY, mE, M, N, K, alpha, beta, D, ldd, s, dyn, x3d);
}

}  // namespace sqr
