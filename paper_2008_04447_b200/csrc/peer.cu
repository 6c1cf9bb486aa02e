// Device-initiated collectives over NVLink peer memory (the "B200-native
// upgrade" of the multi-GPU driver): instead of host-launched
// NCCL broadcast / all-gather calls, the producing rank's kernels store the
// data straight into every peer's copy of a symmetric buffer (P2P stores
// through NVLink / NVSwitch) and publish an epoch into each peer's flag word
// with a system-scope release; consumers gate their stream on a device-side
// acquire wait.  Peer base pointers come from the caller (e.g. the
// buffer_ptrs of torch.distributed._symmetric_memory); on one GPU any set of
// device buffers works, which is how the kernels are unit-tested.
//
//   sqr_peer_put          the panel record (Y | taus | R11 | status) of the
//                         block owner into every peer (randomized.py:203-207
//                         needs it on every rank: the block reflection)
//   sqr_peer_put_columns  the sample-update slab of this rank, scattered to
//                         its GLOBAL column positions in every peer's
//                         replicated sample (sketch.py:132-149) -- all-gather
//                         and assembly in one kernel
//   sqr_peer_wait         device-side wait for the epochs of a set of flags
#include <algorithm>

#include "common.cuh"

namespace sqr {
namespace {

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// The last CTA to finish publishes `epoch` into every peer's flag word: each
// CTA's stores are fenced system-wide before its arrival, so the release
// store orders after all of them.
__device__ __forceinline__ void publish(unsigned* counter, unsigned long long* const* flags, int npeers, int slot,
                                       unsigned long long epoch) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0u;  // reusable by the next call on this stream
      __threadfence_system();
      for (int q = 0; q < npeers; ++q) st_release_sys_u64(flags[q] + slot, epoch);
    }
  }
}

__global__ void __launch_bounds__(256) peer_put_kernel(const int4* __restrict__ src, int64_t n16,
                                                       char* const* __restrict__ dst, int64_t dst_off, int npeers,
                                                       unsigned long long* const* flags, int slot,
                                                       unsigned long long epoch, unsigned* counter) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = __ldg(src + i);
    for (int q = 0; q < npeers; ++q) reinterpret_cast<int4*>(dst[q] + dst_off)[i] = v;
  }
  publish(counter, flags, npeers, slot, epoch);
}

// dst_q[didx[j] * ldd + r] = src[j * lds + r], r < rows, for every peer q.
__global__ void __launch_bounds__(256) peer_put_columns_kernel(const double* __restrict__ src, int64_t lds, int rows,
                                                               int64_t ncols, const int64_t* __restrict__ didx,
                                                               double* const* __restrict__ dst, int64_t ldd,
                                                               int npeers, unsigned long long* const* flags,
                                                               int slot, unsigned long long epoch,
                                                               unsigned* counter) {
  const int64_t total = ncols * rows;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows;
    const int r = (int)(e - j * rows);
    const double v = src[j * lds + r];
    const int64_t o = __ldg(didx + j) * ldd + r;
    for (int q = 0; q < npeers; ++q) dst[q][o] = v;
  }
  publish(counter, flags, npeers, slot, epoch);
}

__global__ void peer_wait_kernel(const unsigned long long* flags, int nflags, unsigned long long epoch) {
  for (int i = threadIdx.x; i < nflags; i += blockDim.x)
    while (ld_acquire_sys_u64(flags + i) < epoch) {
    }
  __syncthreads();
}

int put_grid(int64_t work) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(work, 256), 4LL * sm_count())); }

}  // namespace
}  // namespace sqr

using namespace sqr;

/* Copy `bytes` (a multiple of 16) from src into dst_ptrs[q] + dst_offset for
 * every q < npeers (dst_ptrs / flag_ptrs: DEVICE arrays of peer pointers),
 * then store epoch into flag_ptrs[q][slot] with system-scope release.
 * counter: a device u32, zero before the first call, left at zero. */
extern "C" int sqr_peer_put(const void* src, int64_t bytes, void* const* dst_ptrs, int64_t dst_offset, int npeers,
                            unsigned long long* const* flag_ptrs, int slot, unsigned long long epoch,
                            unsigned* counter, void* stream) {
  if (bytes < 0 || (bytes & 15) || npeers < 1 || dst_ptrs == nullptr || flag_ptrs == nullptr || counter == nullptr ||
      (bytes && src == nullptr) || (reinterpret_cast<uintptr_t>(src) & 15) || (dst_offset & 15)) {
    set_error("sqr_peer_put: need 16-byte aligned buffers / sizes and peer arrays");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n16 = bytes / 16;
  ProfScope ps(kTagMisc, s);
  peer_put_kernel<<<put_grid(n16), 256, 0, s>>>(static_cast<const int4*>(src), n16,
                                                 reinterpret_cast<char* const*>(dst_ptrs), dst_offset, npeers,
                                                 flag_ptrs, slot, epoch, counter);
  SQR_LAUNCH("peer_put_kernel");
  return SQR_OK;
}

/* dst_ptrs[q][didx[j] * ldd + r] = src[j * lds + r] (r < rows, j < ncols) for
 * every peer q, then the epoch into flag_ptrs[q][slot] (release). */
extern "C" int sqr_peer_put_columns(const double* src, int64_t lds, int64_t rows, int64_t ncols, const int64_t* didx,
                                    double* const* dst_ptrs, int64_t ldd, int npeers,
                                    unsigned long long* const* flag_ptrs, int slot, unsigned long long epoch,
                                    unsigned* counter, void* stream) {
  if (rows < 0 || ncols < 0 || npeers < 1 || dst_ptrs == nullptr || flag_ptrs == nullptr || counter == nullptr ||
      (ncols && (src == nullptr || didx == nullptr)) || lds < rows || ldd < rows) {
    set_error("sqr_peer_put_columns: bad arguments");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps(kTagMisc, s);
  peer_put_columns_kernel<<<put_grid(rows * ncols), 256, 0, s>>>(src, lds, (int)rows, ncols, didx, dst_ptrs, ldd,
                                                                 npeers, flag_ptrs, slot, epoch, counter);
  SQR_LAUNCH("peer_put_columns_kernel");
  return SQR_OK;
}

/* Gate the stream until flags[i] >= epoch for every i < nflags (this rank's
 * own flag words, written by peers; acquire, system scope). */
extern "C" int sqr_peer_wait(const unsigned long long* flags, int nflags, unsigned long long epoch, void* stream) {
  if (nflags <= 0) return SQR_OK;
  if (flags == nullptr) {
    set_error("sqr_peer_wait: NULL flags");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  peer_wait_kernel<<<1, 32 * (int)std::min<int64_t>(cdiv(nflags, 32), 32), 0, s>>>(flags, nflags, epoch);
  SQR_LAUNCH("peer_wait_kernel");
  return SQR_OK;
}
