// Result-assembly kernels: the reference builds its result objects with
// NumPy slicing (np.triu, fancy-index gathers, explicit reflector matrices);
// here they are bandwidth kernels on the device, so a factorization's result
// is materialised without ATen glue:
//   * sqr_transpose / upper rows   R = triu(work[:achieved]) as row-major rows
//                                  (randomized.py:223, 338; reference.py:262)
//   * sqr_unpack_reflectors        explicit unit-lower Y of a block from the
//                                  LAPACK-packed work matrix
//                                  (randomized.py:199-201; reference.py:153-159)
//   * sqr_gather/scatter_rows      Z0^T = (R P^T)^T and P^T V_k row permutations
//                                  (randomized.py:374, 384; validation.py:56-59)
#include <algorithm>

#include "common.cuh"

namespace sqr {
namespace {

// dst (n x m, column-major, ld ldd) = src^T for src m x n (ld lds); mode 1
// keeps only src's upper trapezoid (r <= c) and zeroes the rest.  32 x 32
// tiles through padded shared memory: reads along r, writes along c, both
// coalesced.
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ src, int64_t lds, int64_t m,
                                                        int64_t n, double* __restrict__ dst, int64_t ldd, int upper) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t tiles_r = (m + 31) / 32, tiles = tiles_r * ((n + 31) / 32);
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = (t % tiles_r) * 32, c0 = (t / tiles_r) * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      const int64_t c = c0 + ty + i, r = r0 + tx;
      double v = 0.0;
      if (r < m && c < n && (!upper || r <= c)) v = src[c * lds + r];
      tile[ty + i][tx] = v;  // tile[c][r]
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      const int64_t r = r0 + ty + i, c = c0 + tx;
      if (r < m && c < n) dst[r * ldd + c] = tile[tx][ty + i];
    }
    __syncthreads();
  }
}

// Y (m x w, ld ldy) = explicit unit-lower reflectors of packed columns
// [i0, i0+w) of W: Y[r, c] = W[r, i0+c] below the diagonal (r > i0+c), 1 on
// it, 0 above -- the reference's Yfull with zeros above the block offset.
__global__ void unpack_reflectors_kernel(const double* __restrict__ W, int64_t ldw, int64_t m, int64_t i0, int w,
                                         double* __restrict__ Y, int64_t ldy) {
  for (int c = blockIdx.y; c < w; c += gridDim.y) {
    const int64_t d = i0 + c;
    const double* src = W + d * ldw;
    double* out = Y + (int64_t)c * ldy;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
      out[r] = r > d ? src[r] : (r == d ? 1.0 : 0.0);
  }
}

// gather: dst[i, j] = src[idx[i], j];  scatter: dst[idx[i], j] = src[i, j]
// (i < rows, j < cols; column-major both).
template <bool kScatter>
__global__ void permute_rows_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                    const int64_t* __restrict__ idx, double* __restrict__ dst, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const double* s = src + j * lds;
    double* d = dst + j * ldd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
      if (kScatter)
        d[__ldg(idx + i)] = s[i];
      else
        d[i] = s[__ldg(idx + i)];
    }
  }
}

template <bool kScatter>
int permute_rows(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx, double* dst,
                 int64_t ldd, cudaStream_t s, const char* what) {
  if (rows <= 0 || cols <= 0) return SQR_OK;
  if (src == nullptr || dst == nullptr || idx == nullptr || ldd < rows || lds < rows) {
    set_error("%s: bad arguments", what);
    return SQR_EINVAL;
  }
  dim3 grid((unsigned)std::min<int64_t>(cdiv(rows, 256), 64), (unsigned)std::min<int64_t>(cols, 4096));
  ProfScope ps(kTagMisc, s);
  permute_rows_kernel<kScatter><<<grid, 256, 0, s>>>(src, lds, rows, cols, idx, dst, ldd);
  SQR_LAUNCH(what);
  return SQR_OK;
}

}  // namespace
}  // namespace sqr

using namespace sqr;

extern "C" int sqr_transpose(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                             int upper, void* stream) {
  if (m <= 0 || n <= 0) return SQR_OK;
  if (src == nullptr || dst == nullptr || lds < m || ldd < n) {
    set_error("sqr_transpose: bad leading dimension or NULL argument");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t tiles = cdiv(m, 32) * cdiv(n, 32);
  ProfScope ps(kTagMisc, s);
  transpose_kernel<<<(unsigned)std::min<int64_t>(tiles, (int64_t)sm_count() * 8), 256, 0, s>>>(src, lds, m, n, dst,
                                                                                            ldd, upper ? 1 : 0);
  SQR_LAUNCH("transpose_kernel");
  return SQR_OK;
}

extern "C" int sqr_unpack_reflectors(const double* W, int64_t ldw, int64_t m, int64_t i0, int64_t w, double* Y,
                                     int64_t ldy, void* stream) {
  if (m <= 0 || w <= 0) return SQR_OK;
  if (W == nullptr || Y == nullptr || ldw < m || ldy < m || i0 < 0 || i0 + w > m) {
    set_error("sqr_unpack_reflectors: bad arguments");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(m, 256), 64), (unsigned)std::min<int64_t>(w, 4096));
  ProfScope ps(kTagMisc, s);
  unpack_reflectors_kernel<<<grid, 256, 0, s>>>(W, ldw, m, i0, (int)w, Y, ldy);
  SQR_LAUNCH("unpack_reflectors_kernel");
  return SQR_OK;
}

extern "C" int sqr_gather_rows(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx,
                               double* dst, int64_t ldd, void* stream) {
  return permute_rows<false>(src, lds, rows, cols, idx, dst, ldd, static_cast<cudaStream_t>(stream),
                             "sqr_gather_rows");
}

extern "C" int sqr_scatter_rows(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx,
                                double* dst, int64_t ldd, void* stream) {
  return permute_rows<true>(src, lds, rows, cols, idx, dst, ldd, static_cast<cudaStream_t>(stream),
                            "sqr_scatter_rows");
}

// X R = S for X (rows x n), R upper triangular n x n (ld ldr): the sample
// update's S11 R11^{-1} for blocks wider than su_prep's 128 (sketch.py:122-149
// as the row form of its back substitution).  One warp per row, left-looking:
// X(i, c) = (S(i, c) - sum_{l < c} X(i, l) R(l, c)) / R(c, c), fixed-order
// warp reduction (deterministic).  upper_s: S is upper triangular (entries
// below its diagonal, e.g. reflector tails, are read as zero).
namespace sqr {
namespace {
__global__ void __launch_bounds__(256) trsm_ru_kernel(const double* __restrict__ S, int64_t lds, int rows, int n,
                                                      const double* __restrict__ R, int64_t ldr,
                                                      double* __restrict__ X, int64_t ldx, int upper_s) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= rows) return;
  for (int c = 0; c < n; ++c) {
    if (upper_s && c < i) {
      if (lane == 0) X[(int64_t)c * ldx + i] = 0.0;
      continue;
    }
    double acc = 0.0;
    for (int l = (upper_s ? i : 0) + lane; l < c; l += 32) acc = fma(X[(int64_t)l * ldx + i], R[(int64_t)c * ldr + l], acc);
    acc = warp_sum(acc);
    if (lane == 0) X[(int64_t)c * ldx + i] = (S[(int64_t)c * lds + i] - acc) / R[(int64_t)c * ldr + c];
    __syncwarp();
  }
}
}  // namespace
}  // namespace sqr

extern "C" int sqr_trsm_right_upper(const double* S, int64_t lds, int64_t rows, int64_t n, const double* R,
                                    int64_t ldr, double* X, int64_t ldx, int upper_s, void* stream) {
  if (rows <= 0 || n <= 0) return SQR_OK;
  if (S == nullptr || R == nullptr || X == nullptr || lds < rows || ldx < rows || ldr < n) {
    set_error("sqr_trsm_right_upper: bad arguments");
    return SQR_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps(kTagSampleUpd, s);
  trsm_ru_kernel<<<(unsigned)cdiv(rows, 8), 256, 0, s>>>(S, lds, (int)rows, (int)n, R, ldr, X, ldx, upper_s);
  SQR_LAUNCH("trsm_ru_kernel");
  return SQR_OK;
}
