// Bandwidth / latency kernels around the GEMMs:
//   * counter-based Gaussian Omega (rng.py:38-70)                     [L0]
//   * block column moves (randomized.py:194-195, :299-302)            [K3]
//   * sample update B_next = [S12 - S11 R11^-1 R12; S22]
//     with the R11 diagonal guard (sketch.py:122-149, randomized.py:133-135) [K7]
//   * per-block bookkeeping of the driver loop (randomized.py:211-213)
// and the library's error state / device queries.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sqr {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_cuda(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return SQR_ECUDA;
}

unsigned long long* g_trace_host_ptr = nullptr;

// ------------------------------------------------------------ accounting
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> tags;
  size_t used = 0;
  cudaEvent_t pending[kNumTags] = {};
  double flops[kNumTags] = {};
  unsigned mask = ~0u;  // classes that get events (sqr_profile_select)
};
Profiler g_prof;
std::mutex g_prof_mu;  // bench-only instrumentation, but callable from any thread
}  // namespace

void prof_begin(int tag, cudaStream_t s) {
  if (!g_prof.on || !((g_prof.mask >> tag) & 1u)) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (!g_prof.on || g_prof.used + 2 > g_prof.ev.size()) return;
  cudaEvent_t e = g_prof.ev[g_prof.used];
  cudaEventRecord(e, s);
  g_prof.pending[tag] = e;
}
void prof_end(int tag, cudaStream_t s) {
  if (!g_prof.on || !((g_prof.mask >> tag) & 1u)) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (!g_prof.on || g_prof.pending[tag] == nullptr || g_prof.used + 2 > g_prof.ev.size()) return;
  cudaEvent_t e = g_prof.ev[g_prof.used + 1];
  cudaEventRecord(e, s);
  g_prof.tags.push_back(tag);
  g_prof.used += 2;
  g_prof.pending[tag] = nullptr;
}

void prof_add_flops(int tag, double flops) {
  if (!g_prof.on) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_prof.flops[tag] += flops;
}

// Device attributes, cached per device (thread-safe: atomics, idempotent fill).
namespace {
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev], g_smem[kMaxDev];
int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDev ? 0 : dev;
}
}  // namespace

int sm_count() {
  const int dev = cur_dev();
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    g_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int max_smem_optin() {
  const int dev = cur_dev();
  int n = g_smem[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
    g_smem[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int smem_optin(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  const int dev = cur_dev();
  std::lock_guard<std::mutex> lock(mu);
  int& cur = done[{fn, dev}];
  if (bytes > cur) {
    SQR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
  }
  return SQR_OK;
}

namespace {

// ------------------------------------------------------------------ Gaussian
__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + (ctr + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double open_uniform(uint64_t seed, uint64_t ctr) {
  return ((double)(mix64(seed, ctr) >> 11) + 0.5) * 0x1p-53;
}

__global__ void gaussian_kernel(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed,
                                uint64_t offset, int transpose, const int32_t* gate) {
  if (gate && *gate) return;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    // e enumerates the stream order: i fastest (column-major fill).
    const int64_t i = e % rows, t = e / rows;
    const uint64_t pos = offset + (uint64_t)e;
    const uint64_t base = (pos >> 1) << 1;
    const double u1 = open_uniform(seed, base);
    const double u2 = open_uniform(seed, base + 1);
    const double r = sqrt(-2.0 * log(u1));
    const double ang = (2.0 * 3.141592653589793) * u2;
    const double v = (pos & 1) ? r * sin(ang) : r * cos(ang);
    if (transpose)
      out[i * ld + t] = v;
    else
      out[t * ld + i] = v;
  }
}

// ------------------------------------------------------------- column moves
constexpr int kMoveRows = 32;
__global__ void apply_moves_kernel(double* X, int64_t ld, int64_t rows, int64_t col0, int64_t* perm,
                                   const int32_t* moves, const sqr_status* st) {
  extern __shared__ __align__(16) double buf[];  // [nmoves][kMoveRows]
  if (st->stop) return;
  const int nm = st->nmoves;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kMoveRows;
  const int64_t r = r0 + lane;
  // 8 moves per thread in flight (the loads are independent; storing each to
  // shared memory before issuing the next would serialise on HBM latency)
  for (int m0 = warp; m0 < nm; m0 += 8 * nw) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int m = m0 + u * nw;
      v[u] = (m < nm && r < rows && moves[2 * m] >= 0) ? __ldcs(X + (col0 + moves[2 * m + 1]) * ld + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int m = m0 + u * nw;
      if (m < nm) buf[m * kMoveRows + lane] = v[u];
    }
  }
  __syncthreads();
  for (int m = warp; m < nm; m += nw) {
    const int dst = moves[2 * m];
    if (r < rows && dst >= 0) X[(col0 + dst) * ld + r] = buf[m * kMoveRows + lane];
  }
  if (perm != nullptr && blockIdx.x == 0) {
    __syncthreads();
    int64_t* pb = reinterpret_cast<int64_t*>(buf);
    for (int m = threadIdx.x; m < nm; m += blockDim.x)
      if (moves[2 * m] >= 0) pb[m] = perm[col0 + moves[2 * m + 1]];
    __syncthreads();
    for (int m = threadIdx.x; m < nm; m += blockDim.x)
      if (moves[2 * m] >= 0) perm[col0 + moves[2 * m]] = pb[m];
  }
}

// Register-staged variant for <= 256 moves: warp w of a 256-thread CTA owns
// moves w, w+8, ..., w+248 of the CTA's 32 rows (one row per lane), issues
// all of its <= 32 source loads before any store (every read of the CTA's
// rows precedes every write after the barrier), then stores.  No shared
// memory, ~8 CTAs/SM, so one wave covers m = 32768 rows with a single DRAM
// round trip per CTA.
__global__ void __launch_bounds__(256) apply_moves_reg_kernel(double* X, int64_t ld, int64_t rows, int64_t col0,
                                                              int64_t* perm, const int32_t* moves,
                                                              const sqr_status* st) {
  if (st->stop) return;
  const int nm = st->nmoves;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + lane;
  const bool live = r < rows;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int mv = warp + 8 * i;
    v[i] = (mv < nm && live && moves[2 * mv] >= 0) ? __ldcs(X + (col0 + moves[2 * mv + 1]) * ld + r) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int mv = warp + 8 * i;
    if (mv < nm && live && moves[2 * mv] >= 0) __stcs(X + (col0 + moves[2 * mv]) * ld + r, v[i]);
  }
  if (perm != nullptr && blockIdx.x == 0) {
    __shared__ int64_t pb[256];
    for (int mv = threadIdx.x; mv < nm; mv += blockDim.x)
      if (moves[2 * mv] >= 0) pb[mv] = perm[col0 + moves[2 * mv + 1]];
    __syncthreads();
    for (int mv = threadIdx.x; mv < nm; mv += blockDim.x)
      if (moves[2 * mv] >= 0) perm[col0 + moves[2 * mv]] = pb[mv];
  }
}

// ------------------------------------------------------------ sample update
// B_next = [S12 - S11 R11^{-1} R12 ; S22]  (sketch.py:132-149).
// su_prep (one CTA): the R11 diagonal guard (randomized.py:133-135) and
// M = S11 R11^{-1} (sketch.py:132-149: the sample update's S11 R11^{-1}),
// M R11 = S11 with M upper triangular like S11.  One warp per row i of M,
// right-looking: lane l keeps the running sums p[c] = sum_{l' < c} M(i,l') R(l',c)
// for c = l + 32q; each step finishes M(i,c) = (S11(i,c) - p[c]) / R(c,c) in
// the owning lane, broadcasts it with one shuffle and folds it into the
// remaining sums (4 FMAs per lane) -- ~1 shuffle + 1 division per step
// instead of a warp reduction.  Every CTA also evaluates the reference's
// diagonal test (randomized.py:217-219); CTA 0 records the stop.
constexpr int kSuThreads = 256;
constexpr int kSuRows = kSuThreads / 32;
__global__ void __launch_bounds__(kSuThreads, 1)
    su_prep_kernel(const double* Bf, int64_t ldbf, const double* R, int64_t ldr, double* Mout, int64_t ldm,
                   int bmax, sqr_status* st, int32_t* guard) {
  extern __shared__ __align__(16) double Rs[];  // R11 transposed: Rs[l * P + c] = R(l, c), P odd
  __shared__ double rdiag[128];
  __shared__ double wmin[kSuRows];
  if (st->stop) return;
  const int bh = st->sample_achieved;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = bh | 1;
  double dm = INFINITY;
  for (int i = tid; i < bh; i += kSuThreads) {
    const double d = R[(int64_t)i * ldr + i];
    rdiag[i] = d;
    if (i > 0) dm = fmin(dm, fabs(d));
  }
  for (int e0 = tid; e0 < bh * bh; e0 += 8 * kSuThreads) {  // 8 loads in flight per thread
    double rv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kSuThreads;
      const int l = e % bh, c = e / bh;  // coalesced along l
      rv[u] = (e < bh * bh && l < c) ? R[(int64_t)c * ldr + l] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kSuThreads;
      const int l = e % bh, c = e / bh;
      if (e < bh * bh && l < c) Rs[l * P + c] = rv[u];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmin(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if (lane == 0) wmin[warp] = dm;
  __syncthreads();
  double dmin = wmin[0];
  for (int w = 1; w < kSuRows; ++w) dmin = fmin(dmin, wmin[w]);
  const double d0 = bh > 0 ? fabs(rdiag[0]) : 0.0;
  dmin = fmin(dmin, d0);
  const bool ok = (bh > 0) && (dmin > 0x1p-52 * d0);
  // With a guard word (su_prep launched early on a side stream, concurrent
  // with the trailing update that reads st->stop) the verdict is only
  // recorded; finish_block folds it into st->stop after the update, in the
  // reference's order (randomized.py:212-219).
  if (guard != nullptr && blockIdx.x == 0 && tid == 0) *guard = ok ? 0 : 1;
  if (!ok) {
    if (guard == nullptr && blockIdx.x == 0 && tid == 0) {
      st->stop = 1;
      st->reason = SQR_STOP_R11_SINGULAR;
    }
    return;
  }
  const int i = blockIdx.x * kSuRows + warp;
  if (i >= bmax) return;
  double p[4], sv[4], mv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = lane + 32 * q;
    p[q] = 0.0;
    mv[q] = 0.0;
    sv[q] = (i < bh && c >= i && c < bh) ? Bf[(int64_t)c * ldbf + i] : 0.0;
  }
  if (i < bh) {
    for (int c = i; c < bh; ++c) {
      const int qc = c >> 5, lc = c & 31;
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q == qc) v = (sv[q] - p[q]) / rdiag[c];  // meaningful in lane lc
      v = __shfl_sync(0xffffffffu, v, lc);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int cc = lane + 32 * q;
        if (q == qc && lane == lc) mv[q] = v;
        if (cc > c && cc < bh) p[q] = fma(v, Rs[c * P + cc], p[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = lane + 32 * q;
    if (c < bmax) Mout[(int64_t)c * ldm + i] = (i < bh && c >= i && c < bh) ? mv[q] : 0.0;
  }
}

// Rows [rows0, ell) of the sample: B_next(r, c) = Bf(r, bh + c).
__global__ void copy_s22_kernel(const double* Bf, int64_t ldbf, int ell, int nt, double* Bn, int64_t ldbn,
                                const sqr_status* st) {
  if (st->stop) return;
  const int bh = st->sample_achieved;
  const int rows = ell - bh;
  const int64_t total = (int64_t)rows * nt;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = bh + (int)(e % rows), c = (int)(e / rows);
    Bn[(int64_t)c * ldbn + r] = Bf[(int64_t)(bh + c) * ldbf + r];
  }
}

// ----------------------------------------------------------- bookkeeping
__global__ void finish_block_kernel(sqr_status* st, int32_t* widths, int i0, int bb, int k, int n,
                                    const int32_t* guard) {
  if (st->stop) return;
  const int bhat = st->bhat;
  const int achieved = i0 + bhat;
  st->achieved = achieved;
  if (widths) widths[st->nblocks] = bhat;
  st->nblocks += 1;
  if (bhat < bb) {
    st->stop = 1;
    st->reason = SQR_STOP_SHORT_BLOCK;
  } else if (achieved >= k) {
    st->stop = 1;
    st->reason = SQR_STOP_K_REACHED;
  } else if (n - achieved == 0) {
    st->stop = 1;
    st->reason = SQR_STOP_NO_TRAILING;
  } else if (guard != nullptr && *guard) {
    st->stop = 1;
    st->reason = SQR_STOP_R11_SINGULAR;
  }
}

// dst(r, c) = (r <= c) ? src(r, c) : 0 for an n x n block (R11 into Rg, randomized.py:316).
__global__ void copy_upper_kernel(const double* src, int64_t lds, double* dst, int64_t ldd, int n,
                                  const int32_t* gate) {
  if (gate && *gate) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int r = e % n, c = e / n;
    dst[(int64_t)c * ldd + r] = (r <= c) ? src[(int64_t)c * lds + r] : 0.0;
  }
}

// dst[:, dst_idx[j]] = src[:, src_idx[j]] for j < n (rows [0, rows)); NULL
// index arrays mean the identity.  Used by the multi-GPU driver to pack /
// unpack moved columns and to assemble block-cyclic slabs.
__global__ void copy_columns_kernel(const double* src, int64_t lds, int64_t rows, const int64_t* sidx, double* dst,
                                    int64_t ldd, const int64_t* didx, int64_t n) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    const int64_t cs = sidx ? sidx[j] : j, cd = didx ? didx[j] : j;
    const double* s = src + cs * lds;
    double* d = dst + cd * ldd;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
      d[r] = s[r];
  }
}

// One thread holds its stream until a chain kernel on another stream has
// signalled that all its CTAs are resident (ResidentSig, common.cuh); the
// timeout bounds the wait if that kernel cannot start first.
__global__ void wait_resident_kernel(const unsigned* flag, unsigned val, unsigned long long timeout_ns) {
  const unsigned long long t0 = gtimer();
  while ((int)(ld_acquire_u32(flag) - val) < 0) {
    if (gtimer() - t0 > timeout_ns) break;
    __nanosleep(200);
  }
}
__global__ void signal_resident_kernel(ResidentSig sig) { signal_resident(sig); }

// W[0:rows, c] = 0 for c < min(ncols, *lim) (gated on *gate): retires the
// columns of a deferred block update that were already applied in place.
__global__ void zero_columns_kernel(double* W, int64_t ld, int rows, int ncols, const int32_t* lim,
                                    const int32_t* gate) {
  if (gate && *gate) return;
  const int nc = lim ? min(ncols, *lim) : ncols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * nc; e += gridDim.x * blockDim.x)
    W[(int64_t)(e / rows) * ld + e % rows] = 0.0;
}

// dst = src (m x n, column-major; dst may be NULL) and *nonfinite += the
// number of NaN / Inf entries: the input contract's copy + finite scan
// (validation.py:21-37) in one read of A.  Warp-aggregated atomics.
__global__ void copy_check_kernel(const double* __restrict__ src, int64_t lds, int64_t m, int64_t n,
                                  double* __restrict__ dst, int64_t ldd, unsigned long long* nonfinite) {
  unsigned bad = 0;
  const int64_t rows_per = (int64_t)blockDim.x * 2;
  const int64_t rchunks = (m + rows_per - 1) / rows_per;
  for (int64_t w = blockIdx.x; w < rchunks * n; w += gridDim.x) {
    const int64_t c = w / rchunks, r0 = (w % rchunks) * rows_per;
    const double* s = src + c * lds + r0;
    double* d = dst ? dst + c * ldd + r0 : nullptr;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t r = threadIdx.x + u * (int64_t)blockDim.x;
      if (r0 + r < m) {
        const double v = __ldcs(s + r);
        bad += isfinite(v) ? 0u : 1u;
        if (d) __stcs(d + r, v);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, (unsigned long long)bad);
}

// Row-major source (element (r, c) at src[r * lds + c]) into column-major
// dst, + the non-finite count: 32 x 32 tiles through padded shared memory so
// both the reads (along c) and the writes (along r) are coalesced.
__global__ void __launch_bounds__(256) copy_check_t_kernel(const double* __restrict__ src, int64_t lds, int64_t m,
                                                           int64_t n, double* __restrict__ dst, int64_t ldd,
                                                           unsigned long long* nonfinite) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int64_t tiles_c = (n + 31) / 32, tiles = ((m + 31) / 32) * tiles_c;
  unsigned bad = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      const int64_t r = r0 + ty + i, c = c0 + tx;
      double v = 0.0;
      if (r < m && c < n) {
        v = __ldcs(src + r * lds + c);
        bad += isfinite(v) ? 0u : 1u;
      }
      tile[ty + i][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      const int64_t c = c0 + ty + i, r = r0 + tx;
      if (r < m && c < n) __stcs(dst + c * ldd + r, tile[tx][ty + i]);
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, (unsigned long long)bad);
}

__global__ void iota_kernel(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

}  // namespace

int gaussian(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed, uint64_t offset,
             int transpose, const int32_t* gate, cudaStream_t s) {
  const int64_t total = rows * cols;
  if (total <= 0) return SQR_OK;
  const int blocks = (int)std::min<int64_t>(cdiv(total, 256), (int64_t)sm_count() * 16);
  ProfScope ps(kTagGaussian, s);
  gaussian_kernel<<<blocks, 256, 0, s>>>(out, ld, rows, cols, seed, offset, transpose, gate);
  SQR_LAUNCH("gaussian_kernel");
  return SQR_OK;
}

int apply_moves(double* X, int64_t ld, int64_t rows, int64_t col0, int64_t* perm, const int32_t* moves,
                const sqr_status* st, int64_t max_moves, cudaStream_t s) {
  if (rows <= 0 && perm == nullptr) return SQR_OK;
  if (max_moves <= 256) {
    const int blocks = (int)std::max<int64_t>(1, cdiv(rows, 32));
    ProfScope ps(kTagMoves, s);
    apply_moves_reg_kernel<<<blocks, 256, 0, s>>>(X, ld, rows, col0, perm, moves, st);
    SQR_LAUNCH("apply_moves_reg_kernel");
    return SQR_OK;
  }
  const int64_t smem = std::max<int64_t>(max_moves, 1) * kMoveRows * 8;
  if (int rc = smem_optin((const void*)apply_moves_kernel, (int)smem)) return rc;
  const int blocks = (int)std::max<int64_t>(1, cdiv(rows, kMoveRows));
  ProfScope ps(kTagMoves, s);
  apply_moves_kernel<<<blocks, 256, smem, s>>>(X, ld, rows, col0, perm, moves, st);
  SQR_LAUNCH("apply_moves_kernel");
  return SQR_OK;
}

int su_prep(const double* Bf, int64_t ldbf, const double* R, int64_t ldr, int64_t bmax, double* mbuf,
            sqr_status* st, int32_t* guard, cudaStream_t s) {
  if (bmax > 128) {
    set_error("sample_update: block size %lld > 128", (long long)bmax);
    return SQR_EINVAL;
  }
  const int64_t smem = (bmax | 1) * bmax * 8;
  if (int rc = smem_optin((const void*)su_prep_kernel, (int)smem)) return rc;
  // The early (guard-word) launch overlaps the trailing update on a side
  // stream: it is not event-timed (its span would mostly be queueing).
  if (guard == nullptr) prof_begin(kTagSampleUpd, s);
  su_prep_kernel<<<(unsigned)cdiv(bmax, (int64_t)kSuRows), kSuThreads, smem, s>>>(Bf, ldbf, R, ldr, mbuf, bmax,
                                                                                (int)bmax, st, guard);
  if (guard == nullptr) prof_end(kTagSampleUpd, s);
  SQR_LAUNCH("su_prep_kernel");
  return SQR_OK;
}

int sample_update(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr, int64_t nt,
                  int64_t bmax, double* Bn, int64_t ldbn, sqr_status* st, double* mbuf, cudaStream_t s,
                  bool prepped) {
  if (nt <= 0) return SQR_OK;
  if (!prepped) {
    const int rc = su_prep(Bf, ldbf, R, ldr, bmax, mbuf, st, nullptr, s);
    if (rc) return rc;
  }
  // B_top = S12 - M R12 with the block size read on the device (== bmax
  // whenever the loop continues: a short block stops the factorization).
  int rc = gemm_nn(bmax, nt, bmax, -1.0, mbuf, bmax, R + bmax * ldr, ldr, 1.0, Bf + bmax * ldbf, ldbf, Bn, ldbn, s,
                   GemmDyn{&st->stop, nullptr, 0});
  if (rc) return rc;
  if (ell > bmax) {
    ProfScope ps(kTagSampleUpd, s);
    const int blocks = (int)std::min<int64_t>(cdiv((ell - bmax) * nt, 256), (int64_t)sm_count() * 4);
    copy_s22_kernel<<<std::max(blocks, 1), 256, 0, s>>>(Bf, ldbf, (int)ell, (int)nt, Bn, ldbn, st);
    SQR_LAUNCH("copy_s22_kernel");
  }
  return SQR_OK;
}

int finish_block(sqr_status* st, int32_t* widths, int i0, int bb, int k, int n, cudaStream_t s,
                 const int32_t* guard) {
  ProfScope ps(kTagMisc, s);
  finish_block_kernel<<<1, 1, 0, s>>>(st, widths, i0, bb, k, n, guard);
  SQR_LAUNCH("finish_block_kernel");
  return SQR_OK;
}

int copy_upper(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, const int32_t* gate,
               cudaStream_t s) {
  if (n <= 0) return SQR_OK;
  ProfScope ps(kTagMisc, s);
  copy_upper_kernel<<<(unsigned)std::min<int64_t>(cdiv(n * n, 256), 256), 256, 0, s>>>(src, lds, dst, ldd, (int)n,
                                                                                     gate);
  SQR_LAUNCH("copy_upper_kernel");
  return SQR_OK;
}

int copy_columns(const double* src, int64_t lds, int64_t rows, const int64_t* sidx, double* dst, int64_t ldd,
                 const int64_t* didx, int64_t n, cudaStream_t s) {
  if (rows <= 0 || n <= 0) return SQR_OK;
  ProfScope ps(kTagMisc, s);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(rows, 256), 64), (unsigned)std::min<int64_t>(n, 4096));
  copy_columns_kernel<<<grid, 256, 0, s>>>(src, lds, rows, sidx, dst, ldd, didx, n);
  SQR_LAUNCH("copy_columns_kernel");
  return SQR_OK;
}

int wait_resident(ResidentSig sig, int timeout_us, cudaStream_t s) {
  if (sig.flag == nullptr) return SQR_OK;
  wait_resident_kernel<<<1, 1, 0, s>>>(sig.flag, sig.val, (unsigned long long)timeout_us * 1000ull);
  SQR_LAUNCH("wait_resident_kernel");
  return SQR_OK;
}

int signal_resident_host(ResidentSig sig, cudaStream_t s) {
  if (sig.flag == nullptr) return SQR_OK;
  signal_resident_kernel<<<1, 1, 0, s>>>(sig);
  SQR_LAUNCH("signal_resident_kernel");
  return SQR_OK;
}

int zero_columns(double* W, int64_t ld, int64_t rows, int64_t ncols, const int32_t* lim, const int32_t* gate,
                 cudaStream_t s) {
  if (rows <= 0 || ncols <= 0) return SQR_OK;
  ProfScope ps(kTagMisc, s);
  zero_columns_kernel<<<(unsigned)std::min<int64_t>(cdiv(rows * ncols, 256), 512), 256, 0, s>>>(
      W, ld, (int)rows, (int)ncols, lim, gate);
  SQR_LAUNCH("zero_columns_kernel");
  return SQR_OK;
}

int iota(int64_t* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return SQR_OK;
  ProfScope ps(kTagMisc, s);
  iota_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 1024), 256, 0, s>>>(p, n);
  SQR_LAUNCH("iota_kernel");
  return SQR_OK;
}

}  // namespace sqr

extern "C" const char* sqr_version(void) { return "libsqr 0.1.0 (sm_100a, fp64 DMMA)"; }
extern "C" const char* sqr_last_error(void) { return sqr::g_err; }
extern "C" int sqr_device_sm_count(void) { return sqr::sm_count(); }

extern "C" int sqr_gaussian(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed,
                            uint64_t offset, int transpose, void* stream) {
  return sqr::gaussian(out, ld, rows, cols, seed, offset, transpose, nullptr,
                       static_cast<cudaStream_t>(stream));
}

extern "C" int sqr_apply_moves(double* X, int64_t ld, int64_t rows, int64_t col0, int64_t* perm,
                               const int32_t* moves, const sqr_status* st, int64_t max_moves, void* stream) {
  return sqr::apply_moves(X, ld, rows, col0, perm, moves, st, max_moves, static_cast<cudaStream_t>(stream));
}

extern "C" int sqr_sample_update(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr,
                                 int64_t nt, double* Bnext, int64_t ldbn, sqr_status* st, void* stream) {
  // stand-alone entry: the block size is the sample QRCP's (st->sample_achieved)
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sqr_status hs;
  if (cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return sqr::check_cuda(cudaGetLastError(), "sqr_sample_update");
  const int64_t bh = hs.sample_achieved;
  double* mbuf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&mbuf), std::max<int64_t>(bh * bh, 1) * 8, s) != cudaSuccess)
    return sqr::check_cuda(cudaGetLastError(), "cudaMallocAsync");
  int rc = sqr::sample_update(Bf, ldbf, ell, R, ldr, nt, bh, Bnext, ldbn, st, mbuf, s);
  cudaFreeAsync(mbuf, s);
  return rc;
}

// Same update with the block size b supplied by the caller (the sample
// QRCP's sample_achieved, already known to a host orchestrator) and a
// caller-owned b*b scratch: no host synchronisation (multi-GPU driver).
extern "C" int sqr_sample_update_b(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr,
                                   int64_t nt, int64_t b, double* Bnext, int64_t ldbn, sqr_status* st, double* mbuf,
                                   void* stream) {
  if (b < 1 || b > ell || mbuf == nullptr) {
    sqr::set_error("sqr_sample_update_b: need 1 <= b <= ell and a b*b scratch");
    return SQR_EINVAL;
  }
  return sqr::sample_update(Bf, ldbf, ell, R, ldr, nt, b, Bnext, ldbn, st, mbuf, static_cast<cudaStream_t>(stream));
}

extern "C" int sqr_copy_check(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                              unsigned long long* nonfinite, void* stream) {
  if (m <= 0 || n <= 0) return SQR_OK;
  if (lds < m || (dst != nullptr && ldd < m) || nonfinite == nullptr) {
    sqr::set_error("sqr_copy_check: bad leading dimension or NULL counter");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t work = sqr::cdiv(m, 512) * n;
  const int blocks = (int)std::min<int64_t>(work, (int64_t)sqr::sm_count() * 16);
  sqr::ProfScope ps(sqr::kTagMisc, s);
  sqr::copy_check_kernel<<<blocks, 256, 0, s>>>(src, lds, m, n, dst, ldd, nonfinite);
  SQR_LAUNCH("copy_check_kernel");
  return SQR_OK;
}

extern "C" int sqr_copy_check_t(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                                unsigned long long* nonfinite, void* stream) {
  if (m <= 0 || n <= 0) return SQR_OK;
  if (lds < n || dst == nullptr || ldd < m || nonfinite == nullptr) {
    sqr::set_error("sqr_copy_check_t: bad leading dimension or NULL argument");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t tiles = sqr::cdiv(m, 32) * sqr::cdiv(n, 32);
  const int blocks = (int)std::min<int64_t>(tiles, (int64_t)sqr::sm_count() * 8);
  sqr::ProfScope ps(sqr::kTagMisc, s);
  sqr::copy_check_t_kernel<<<blocks, 256, 0, s>>>(src, lds, m, n, dst, ldd, nonfinite);
  SQR_LAUNCH("copy_check_t_kernel");
  return SQR_OK;
}

// The two halves of sqr_sample_update_b for an orchestrator that overlaps the
// prep with the trailing update: prep = R11 guard + M = S11 R11^-1 (b x b,
// into mbuf; S11 = the first b columns of Bf, R11 at R with ld ldr), apply =
// Bnext = [S12 - M R12 ; S22] (R = [R11 | R12], gated on st->stop).
extern "C" int sqr_sample_update_prep(const double* Bf, int64_t ldbf, const double* R11, int64_t ldr, int64_t b,
                                      double* mbuf, sqr_status* st, void* stream) {
  if (b < 1 || mbuf == nullptr) {
    sqr::set_error("sqr_sample_update_prep: need b >= 1 and a b*b scratch");
    return SQR_EINVAL;
  }
  return sqr::su_prep(Bf, ldbf, R11, ldr, b, mbuf, st, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" int sqr_sample_update_apply(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr,
                                       int64_t nt, int64_t b, double* Bnext, int64_t ldbn, sqr_status* st,
                                       const double* mbuf, void* stream) {
  if (b < 1 || b > ell || mbuf == nullptr) {
    sqr::set_error("sqr_sample_update_apply: need 1 <= b <= ell and the prep's scratch");
    return SQR_EINVAL;
  }
  return sqr::sample_update(Bf, ldbf, ell, R, ldr, nt, b, Bnext, ldbn, st, const_cast<double*>(mbuf),
                            static_cast<cudaStream_t>(stream), true);
}

extern "C" int64_t sqr_launch_count(void) { return sqr::g_launches.load(); }

extern "C" int sqr_profile_enable(int64_t max_launches) {
  using sqr::g_prof;
  std::lock_guard<std::mutex> lock(sqr::g_prof_mu);
  for (auto e : g_prof.ev) cudaEventDestroy(e);
  g_prof.ev.clear();
  g_prof.tags.clear();
  g_prof.used = 0;
  for (auto& p : g_prof.pending) p = nullptr;
  for (auto& f : g_prof.flops) f = 0.0;
  g_prof.on = max_launches > 0;
  if (!g_prof.on) return SQR_OK;
  g_prof.ev.resize(2 * max_launches);
  for (auto& e : g_prof.ev)
    if (cudaEventCreate(&e) != cudaSuccess) return sqr::check_cuda(cudaGetLastError(), "cudaEventCreate");
  return SQR_OK;
}

// Sum of device time (ms) and launch count per kernel class since
// sqr_profile_enable; synchronises on the recorded events, then resets.
extern "C" int sqr_profile_collect(double* ms_per_tag, int64_t* count_per_tag, int ntags) {
  using sqr::g_prof;
  std::lock_guard<std::mutex> lock(sqr::g_prof_mu);
  for (int t = 0; t < ntags; ++t) {
    ms_per_tag[t] = 0.0;
    count_per_tag[t] = 0;
  }
  for (size_t i = 0; i < g_prof.tags.size(); ++i) {
    float ms = 0.f;
    cudaEventSynchronize(g_prof.ev[2 * i + 1]);
    if (cudaEventElapsedTime(&ms, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]) != cudaSuccess) continue;
    const int t = g_prof.tags[i];
    if (t < ntags) {
      ms_per_tag[t] += ms;
      count_per_tag[t] += 1;
    }
  }
  g_prof.tags.clear();
  g_prof.used = 0;
  return SQR_OK;
}

// Restrict the per-launch events to the classes in tag_mask (bit t = class t;
// the two event records cost ~2 us each per launch, ~20 ms per C5 step when
// every class is timed).  Takes effect for launches enqueued afterwards.
extern "C" int sqr_profile_select(uint32_t tag_mask) {
  std::lock_guard<std::mutex> lock(sqr::g_prof_mu);
  sqr::g_prof.mask = tag_mask;
  return SQR_OK;
}

// Flops the drivers attributed to a class since sqr_profile_enable (only the
// launches whose share of a class the caller cannot derive from the shapes:
// class 9, the bulk updates running beside a chain kernel).
extern "C" int sqr_profile_flops(double* flops_per_tag, int ntags) {
  using sqr::g_prof;
  std::lock_guard<std::mutex> lock(sqr::g_prof_mu);
  for (int t = 0; t < ntags; ++t) flops_per_tag[t] = t < sqr::kNumTags ? g_prof.flops[t] : 0.0;
  return SQR_OK;
}

// Debug: device buffer (>= 8 * steps u64) receiving %globaltimer stamps of
// the next cooperative kernels' phases (CTA 0); NULL disables.
extern "C" int sqr_debug_trace(void* device_buffer) {
  sqr::g_trace_host_ptr = static_cast<unsigned long long*>(device_buffer);
  return SQR_OK;
}

extern "C" int sqr_copy_columns(const double* src, int64_t lds, int64_t rows, const int64_t* src_idx, double* dst,
                                int64_t ldd, const int64_t* dst_idx, int64_t n, void* stream) {
  return sqr::copy_columns(src, lds, rows, src_idx, dst, ldd, dst_idx, n, static_cast<cudaStream_t>(stream));
}
