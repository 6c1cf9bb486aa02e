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
};
Profiler g_prof;
}  // namespace

void prof_begin(int tag, cudaStream_t s) {
  if (!g_prof.on || g_prof.used + 2 > g_prof.ev.size()) return;
  cudaEvent_t e = g_prof.ev[g_prof.used];
  cudaEventRecord(e, s);
  g_prof.pending[tag] = e;
}
void prof_end(int tag, cudaStream_t s) {
  if (!g_prof.on || g_prof.pending[tag] == nullptr || g_prof.used + 2 > g_prof.ev.size()) return;
  cudaEvent_t e = g_prof.ev[g_prof.used + 1];
  cudaEventRecord(e, s);
  g_prof.tags.push_back(tag);
  g_prof.used += 2;
  g_prof.pending[tag] = nullptr;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int max_smem_optin() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
  }
  return n;
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
  for (int m = warp; m < nm; m += nw) {
    const int src = moves[2 * m + 1];
    buf[m * kMoveRows + lane] = (r < rows) ? X[(col0 + src) * ld + r] : 0.0;
  }
  __syncthreads();
  for (int m = warp; m < nm; m += nw) {
    const int dst = moves[2 * m];
    if (r < rows) X[(col0 + dst) * ld + r] = buf[m * kMoveRows + lane];
  }
  if (perm != nullptr && blockIdx.x == 0) {
    __syncthreads();
    int64_t* pb = reinterpret_cast<int64_t*>(buf);
    for (int m = threadIdx.x; m < nm; m += blockDim.x) pb[m] = perm[col0 + moves[2 * m + 1]];
    __syncthreads();
    for (int m = threadIdx.x; m < nm; m += blockDim.x) perm[col0 + moves[2 * m]] = pb[m];
  }
}

// ------------------------------------------------------------ sample update
// CTA = 32 trailing columns; 8 threads per column.  Phase 1 solves
// X = R11^{-1} R12 by row-oriented back substitution (sketch.py:122-129);
// phase 2 forms S12 - S11 X (sketch.py:147) and copies S22.
constexpr int kSuCols = 32;
constexpr int kSuThreads = 256;
__global__ void __launch_bounds__(kSuThreads, 1)
    sample_update_kernel(const double* Bf, int64_t ldbf, int ell, const double* R, int64_t ldr,
                         int nt, double* Bn, int64_t ldbn, sqr_status* st) {
  extern __shared__ __align__(16) double sm[];
  if (st->stop) return;
  const int bh = st->sample_achieved;
  const int ldt = bh | 1;
  double* Tm = sm;                        // bh x bh (R11, then S11), pitch ldt
  double* Xs = sm + (size_t)bh * ldt;     // bh x kSuCols, pitch bh+1
  const int ldx = bh + 1;
  const int tid = threadIdx.x;
  // _diag_ok (randomized.py:133-135): every CTA checks redundantly.
  {
    __shared__ int ok;
    if (tid == 0) {
      const double d0 = fabs(R[0]);
      double dmin = d0;
      for (int i = 1; i < bh; ++i) dmin = fmin(dmin, fabs(R[(int64_t)i * ldr + i]));
      ok = (bh > 0) && (dmin > 0x1p-52 * d0);
    }
    __syncthreads();
    if (!ok) {
      if (blockIdx.x == 0 && tid == 0) {
        st->stop = 1;
        st->reason = SQR_STOP_R11_SINGULAR;
      }
      return;
    }
  }
  const int c0 = blockIdx.x * kSuCols;
  const int nc = min(kSuCols, nt - c0);
  if (nc <= 0) return;
  for (int e = tid; e < bh * bh; e += kSuThreads) {
    const int i = e % bh, j = e / bh;
    Tm[j * ldt + i] = (i <= j) ? R[(int64_t)j * ldr + i] : 0.0;
  }
  for (int e = tid; e < bh * nc; e += kSuThreads) {
    const int i = e % bh, c = e / bh;
    Xs[c * ldx + i] = R[(int64_t)(bh + c0 + c) * ldr + i];  // R12
  }
  __syncthreads();
  const int col = tid >> 3, q = tid & 7;
  // Back substitution, 8 lanes per column, fixed shuffle tree.
  for (int i = bh - 1; i >= 0; --i) {
    double s = 0.0;
    if (col < nc)
      for (int l = i + 1 + q; l < bh; l += 8) s = fma(Tm[l * ldt + i], Xs[col * ldx + l], s);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (col < nc && q == 0) Xs[col * ldx + i] = (Xs[col * ldx + i] - s) / Tm[i * ldt + i];
    __syncwarp();
  }
  __syncthreads();
  // S11 replaces R11.
  for (int e = tid; e < bh * bh; e += kSuThreads) {
    const int i = e % bh, j = e / bh;
    Tm[j * ldt + i] = (i <= j) ? Bf[(int64_t)j * ldbf + i] : 0.0;
  }
  __syncthreads();
  // top = S12 - S11 X
  for (int e = tid; e < bh * nc; e += kSuThreads) {
    const int i = e % bh, c = e / bh;
    double s = 0.0;
    for (int l = i; l < bh; ++l) s = fma(Tm[l * ldt + i], Xs[c * ldx + l], s);
    Bn[(int64_t)(c0 + c) * ldbn + i] = Bf[(int64_t)(bh + c0 + c) * ldbf + i] - s;
  }
  for (int e = tid; e < (ell - bh) * nc; e += kSuThreads) {
    const int i = bh + e % (ell - bh), c = e / (ell - bh);
    Bn[(int64_t)(c0 + c) * ldbn + i] = Bf[(int64_t)(bh + c0 + c) * ldbf + i];
  }
}

// ----------------------------------------------------------- bookkeeping
__global__ void finish_block_kernel(sqr_status* st, int32_t* widths, int i0, int bb, int k, int n) {
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
  const int64_t smem = std::max<int64_t>(max_moves, 1) * kMoveRows * 8;
  static int64_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    SQR_CUDA(cudaFuncSetAttribute(apply_moves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  const int blocks = (int)std::max<int64_t>(1, cdiv(rows, kMoveRows));
  ProfScope ps(kTagMoves, s);
  apply_moves_kernel<<<blocks, 256, smem, s>>>(X, ld, rows, col0, perm, moves, st);
  SQR_LAUNCH("apply_moves_kernel");
  return SQR_OK;
}

int sample_update(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr, int64_t nt,
                  int64_t bmax, double* Bn, int64_t ldbn, sqr_status* st, cudaStream_t s) {
  if (nt <= 0) return SQR_OK;
  const int64_t smem = ((bmax | 1) * bmax + (bmax + 1) * kSuCols) * 8;
  static int64_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    SQR_CUDA(cudaFuncSetAttribute(sample_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    configured = smem;
  }
  ProfScope ps(kTagSampleUpd, s);
  sample_update_kernel<<<(unsigned)cdiv(nt, kSuCols), kSuThreads, smem, s>>>(Bf, ldbf, (int)ell, R, ldr,
                                                                           (int)nt, Bn, ldbn, st);
  SQR_LAUNCH("sample_update_kernel");
  return SQR_OK;
}

int finish_block(sqr_status* st, int32_t* widths, int i0, int bb, int k, int n, cudaStream_t s) {
  ProfScope ps(kTagMisc, s);
  finish_block_kernel<<<1, 1, 0, s>>>(st, widths, i0, bb, k, n);
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
  return sqr::sample_update(Bf, ldbf, ell, R, ldr, nt, ell, Bnext, ldbn, st, static_cast<cudaStream_t>(stream));
}

extern "C" int64_t sqr_launch_count(void) { return sqr::g_launches.load(); }

extern "C" int sqr_profile_enable(int64_t max_launches) {
  using sqr::g_prof;
  for (auto e : g_prof.ev) cudaEventDestroy(e);
  g_prof.ev.clear();
  g_prof.tags.clear();
  g_prof.used = 0;
  for (auto& p : g_prof.pending) p = nullptr;
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

// Debug: device buffer (>= 8 * steps u64) receiving %globaltimer stamps of
// the next cooperative kernels' phases (CTA 0); NULL disables.
extern "C" int sqr_debug_trace(void* device_buffer) {
  sqr::g_trace_host_ptr = static_cast<unsigned long long*>(device_buffer);
  return SQR_OK;
}
