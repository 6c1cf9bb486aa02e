// Shared device helpers for libsqr (sm_100a): fp64 DMMA wrappers, cp.async,
// a reusable grid barrier for cooperative persistent kernels, reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/sqr.h"

namespace sqr {

constexpr int kWarp = 32;

// Debug / A-B switches: set, non-empty and not "0".
inline bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e != nullptr && *e != '\0' && !(e[0] == '0' && e[1] == '\0');
}

// ----------------------------------------------------------------- error state
void set_error(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
int sm_count();
int max_smem_optin();
// Dynamic shared-memory opt-in of `fn` on the CURRENT device (raised, never
// lowered), once per (kernel, device); thread-safe (process-wide mutex).
int smem_optin(const void* fn, int bytes);

#define SQR_CUDA(call)                                              \
  do {                                                              \
    cudaError_t e__ = (call);                                       \
    if (e__ != cudaSuccess) return ::sqr::check_cuda(e__, #call);   \
  } while (0)
#define SQR_LAUNCH(what)                                            \
  do {                                                              \
    ::sqr::count_launch();                                          \
    cudaError_t e__ = cudaGetLastError();                           \
    if (e__ != cudaSuccess) return ::sqr::check_cuda(e__, what);    \
  } while (0)

// Launch accounting + optional per-kernel-class CUDA-event timing (bench.py
// reads it through sqr_launch_count / sqr_profile_*).
enum ProfTag { kTagGemmTn = 0, kTagGemmNn, kTagSample, kTagPanel, kTagBuildT, kTagMoves, kTagSampleUpd,
               kTagGaussian, kTagMisc, kTagGemmNnBeside, kNumTags };
void count_launch();
void prof_begin(int tag, cudaStream_t s);
void prof_end(int tag, cudaStream_t s);
void prof_add_flops(int tag, double flops);  // only counted while profiling is on
struct ProfScope {
  int tag;
  cudaStream_t s;
  ProfScope(int t, cudaStream_t st) : tag(t), s(st) { prof_begin(tag, s); }
  ~ProfScope() { prof_end(tag, s); }
};

// ------------------------------------------------------------------- fp64 MMA
// m16n8k4 f64 tensor-core MMA (SASS: 2x DMMA.8x8x4).  Fragment layout
// (lane = 4*g + t):  a0 = A[g][t], a1 = A[g+8][t];  b0 = B[t][g];
// d0,d1 = D[g][2t,2t+1];  d2,d3 = D[g+8][2t,2t+1].
__device__ __forceinline__ void dmma16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// ------------------------------------------------------------------ cp.async
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool pred) {
  const int sz = pred ? BYTES : 0;  // src-size 0 => zero fill
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(sz));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "n"(BYTES), "r"(sz));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ------------------------------------------------------ memory-model helpers
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// L1-bypassing loads for data other CTAs wrote during this launch.
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }

// Grid barrier for cooperative persistent kernels: a monotonic arrival
// counter (zeroed by the host with cudaMemsetAsync before every launch),
// release-add to arrive, relaxed polling, one acquire fence to leave.
// Measured ~1.2 us per barrier at 148 CTAs on B200 (tools/barrier_bench.cu).
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
struct GridBarrier {
  unsigned* ctr;
  unsigned target;
  unsigned nblocks;
  __device__ void init(unsigned* c) {
    ctr = c;
    target = 0;
    nblocks = gridDim.x * gridDim.y * gridDim.z;
  }
  // Split phases: arrive() publishes this CTA's prior writes; wait() (any
  // one warp may call it, the caller's thread 0 polls) returns once every
  // CTA has arrived.  sync() = arrive + wait.
  // red.release is cumulative over the CTA's writes ordered before it by
  // the bar.sync (one MEMBAR.GPU in SASS; an explicit fence.acq_rel in front
  // of it only adds a second one), and the acquire poll (LDG.STRONG.GPU +
  // L1 invalidate, no MEMBAR) synchronises with every arrival through the
  // counter's release sequence.  SQR_GB_FENCE builds the fenced variant.
  __device__ void arrive() {
    __syncthreads();
    target += nblocks;
    if (threadIdx.x == 0) {
#ifdef SQR_GB_FENCE
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
#endif
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    }
  }
  __device__ void wait_lane0() {  // call from lane 0 of one warp
    while ((int)(ld_acquire_u32(ctr) - target) < 0) {
    }
  }
  __device__ void sync() {
    __syncthreads();
    target += nblocks;
    if (threadIdx.x == 0) {
#ifdef SQR_GB_FENCE
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
#endif
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
      while ((int)(ld_acquire_u32(ctr) - target) < 0) {
      }
    }
    __syncthreads();
  }
};

// Debug phase trace (sqr_debug_trace): CTA 0 / thread 0 of the cooperative
// kernels stamps %globaltimer at phase boundaries when a buffer is set.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SQR_TRACE(buf, idx)                                                      \
  do {                                                                           \
    if ((buf) != nullptr && blockIdx.x == 0 && threadIdx.x == 0) (buf)[idx] = gtimer(); \
  } while (0)
extern unsigned long long* g_trace_host_ptr;

// ------------------------------------------------------------ fp64 division
// a / b correctly rounded from ry = RN(1/b) (Markstein: q = RN(a ry) is
// within an ulp, the remainder a - b q is exact under fma, and one
// correction q + (a - b q) ry rounds to RN(a / b)) for quotients in the
// normal range -- the reflector tails a_r / (a_0 - beta) (|.| <= 1) and the
// panel's s_c / y0.  Bitwise equal to a / b there, without the IEEE
// division's per-quotient iteration and slow-path branch: one drcp per
// reflector instead of one division per entry.
__device__ __forceinline__ double div_rn(double a, double b, double ry) {
  const double q = a * ry;
  const double r = fma(-q, b, a);
  return fma(r, ry, q);
}


// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree): every thread gets the result.
// `red` must hold >= 32 doubles.  Contains __syncthreads.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

// Device-side dynamic shape for GEMMs enqueued ahead of the data that sizes
// them: skip when *stop != 0; shrink N by *shift and advance the flagged
// operands by *shift columns (trailing update after a panel of bhat columns).
constexpr int kShiftB = 1;  // tn: C operand, nn: Y operand
constexpr int kShiftD = 2;  // D and E
struct GemmDyn {
  const int32_t* stop = nullptr;
  const int32_t* shift = nullptr;
  int flags = 0;
  // gemm_tn only: the first npre columns of the C operand come from pre
  // (ld ldpre) and are never shifted -- lets the trailing-update sweep
  // Y^T [Y | C] produce the Gram matrix Y^T Y for T in the same launch.
  const double* pre = nullptr;
  int64_t ldpre = 0;
  int npre = 0;
  // optional cap: N <= *limit - limit_off (dynamic panel width)
  const int32_t* limit = nullptr;
  int limit_off = 0;
  // profiling class of this launch when >= 0 (gemm_nn: kTagGemmNnBeside for the
  // bulk updates that share the chip with a chain kernel, whose event times
  // measure the shared run)
  int prof_tag = -1;
  // gemm_tn only, host side: recorded on the launch stream as soon as the
  // first npre output columns (the Gram prefix) are final -- before the
  // split-K reduction of the other columns -- so T can be built beside it
  cudaEvent_t pre_ready = nullptr;
};

// "Every CTA of this launch is resident" signal of the whole-SM chain kernels
// (sample QRCP, panel): the last CTA stores val to *flag when it starts (CTAs
// are dispatched in index order; CTA 0 on an early exit).  The driver holds a GEMM on
// another stream behind wait_resident() until then, so the chain kernel
// takes its SMs first and the GEMM's CTAs fill the rest (driver.cu, Overlap).
struct ResidentSig {
  unsigned* flag = nullptr;
  unsigned val = 0;
};
__device__ __forceinline__ void signal_resident(const ResidentSig& s) {
  if (s.flag != nullptr) st_release_u32(s.flag, s.val);
}

__host__ __device__ constexpr int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

}  // namespace sqr

// ------------------------------------------------------ internal entry points
namespace sqr {
int gemm_tn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx, const double* C,
            int64_t ldc, double beta, const double* E, int64_t lde, double* D, int64_t ldd, double* ws,
            int64_t ws_bytes, cudaStream_t s, GemmDyn dyn);
int gemm_nn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx, const double* Y,
            int64_t ldy, double beta, const double* E, int64_t lde, double* D, int64_t ldd, cudaStream_t s,
            GemmDyn dyn, double* ws = nullptr, int64_t ws_bytes = 0);
int64_t sample_qrcp_workspace(int64_t ell, int64_t nt);
int sample_qrcp(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf, int64_t ldbf,
                int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st, void* ws,
                int64_t ws_bytes, cudaStream_t s, ResidentSig sig = {});
// Holds stream s until *sig.flag == sig.val (bounded by timeout_us).
int wait_resident(ResidentSig sig, int timeout_us, cudaStream_t s);
int signal_resident_host(ResidentSig sig, cudaStream_t s);
int64_t panel_workspace(int64_t w);
int64_t panel_block_max_rows();
int64_t panel_block_workspace();
int panel_block(double* P, int64_t ldp, int64_t mr, int64_t w, int64_t wmax, double* Y, int64_t ldy,
                double* taus, int stop_at_zero, sqr_status* st, void* ws, int64_t ws_bytes, cudaStream_t s,
                ResidentSig sig = {});
int panel_qr(double* P, int64_t ldp, int64_t mr, int64_t w, int64_t wmax, double* Y, int64_t ldy,
             double* taus, int stop_at_zero, sqr_status* st, void* ws, int64_t ws_bytes, cudaStream_t s,
             int64_t c0 = 0);
int build_t_fast(const double* Gm, int64_t ldg, const double* taus, int64_t j, double* T, int64_t ldt,
                 const int32_t* gate, cudaStream_t s);
int build_t(const double* Gm, int64_t ldg, const double* taus, int64_t j, double* T, int64_t ldt,
            const int32_t* gate, cudaStream_t s);
int gaussian(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed, uint64_t offset,
             int transpose, const int32_t* gate, cudaStream_t s);
int apply_moves(double* X, int64_t ld, int64_t rows, int64_t col0, int64_t* perm, const int32_t* moves,
                const sqr_status* st, int64_t max_moves, cudaStream_t s);
int su_prep(const double* Bf, int64_t ldbf, const double* R, int64_t ldr, int64_t bmax, double* mbuf,
            sqr_status* st, int32_t* guard, cudaStream_t s);
int sample_update(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr, int64_t nt,
                  int64_t bmax, double* Bn, int64_t ldbn, sqr_status* st, double* mbuf, cudaStream_t s,
                  bool prepped = false);
int finish_block(sqr_status* st, int32_t* widths, int i0, int bb, int k, int n, cudaStream_t s,
                 const int32_t* guard = nullptr);
int iota(int64_t* p, int64_t n, cudaStream_t s);
int zero_columns(double* W, int64_t ld, int64_t rows, int64_t ncols, const int32_t* lim, const int32_t* gate,
                 cudaStream_t s);
int copy_columns(const double* src, int64_t lds, int64_t rows, const int64_t* sidx, double* dst, int64_t ldd,
                 const int64_t* didx, int64_t n, cudaStream_t s);
int copy_upper(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t n, const int32_t* gate,
               cudaStream_t s);
}  // namespace sqr
