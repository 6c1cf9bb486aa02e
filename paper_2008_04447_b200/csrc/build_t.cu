// Compact-WY T factor from G = Y^T Y and taus (householder.py:52-61), one
// CTA, latency-oriented:
//   1. 16 x 16 diagonal blocks, one warp each, right-looking form of the
//      reference recurrence T[:c, c] = -tau_c T[:c, :c] G[:c, c]: lane i keeps
//      row i and, once T[i][c] is final, folds it into the running sums of
//      all later columns (one FMA per column, no reduction chain);
//   2. blocks merged pairwise, 16 -> 32 -> 64 -> 128, by the composition rule
//      of wy_compose (householder.py:94-104):
//          T_AB = -T_AA (G_AB T_BB)
//      as two DMMA (m16n8k4) products over shared memory, all merges of a
//      level at once, tiles spread over the 8 warps.
// Storage: one row-major array, T in the upper triangle, G(r, c) (r > c) in
// the strict lower one (G is symmetric), pitch 132 (4 mod 32: conflict-free
// fragment gathers).  Widths are padded to 16/32/64/128 with tau = 0, which
// gives zero rows and columns, as in the recurrence.
#include "common.cuh"

namespace sqr {
namespace {

constexpr int kBtThreads = 256;
constexpr int kBtP = 132;  // pitch of the 128 x 128 array
constexpr int kBtXP = 68;  // pitch of the merge scratch (64 x 64 max)

__global__ void __launch_bounds__(kBtThreads, 1)
    build_t_fast_kernel(const double* Gm, int64_t ldg, const double* taus, int j, int jp, double* T, int64_t ldt,
                        const int32_t* gate) {
  extern __shared__ __align__(16) double smb[];
  double* M = smb;                  // jp x kBtP
  double* Xs = M + 128 * kBtP;      // merge scratch, 4 blocks of (<= 32 x 32) or one 64 x 64
  __shared__ double tau_s[128];
  if (gate && *gate) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  // 8 loads in flight per thread (a load -> store loop would pay the full
  // L2 latency per element)
  for (int e0 = tid; e0 < jp * jp; e0 += 8 * kBtThreads) {
    double gv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kBtThreads;
      const int r = e % jp, c = e / jp;  // coalesced along r
      gv[u] = (e < jp * jp && r > c && r < j && c < j) ? Gm[(int64_t)c * ldg + r] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kBtThreads;
      if (e < jp * jp) M[(e % jp) * kBtP + e / jp] = gv[u];  // lower: G(r, c); upper (T) zero
    }
  }
  for (int i = tid; i < jp; i += kBtThreads) tau_s[i] = i < j ? taus[i] : 0.0;
  __syncthreads();
  // ---- 1. diagonal 16-blocks (lanes 0..15 of warp w own rows of block w)
  if (warp < jp / 16 && lane < 16) {
    const int o = warp * 16, i = lane;
    double tr[16], p[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) p[c] = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const double tc = tau_s[o + c];
      tr[c] = c == i ? tc : (c > i ? -tc * p[c] : 0.0);
#pragma unroll
      for (int c2 = c + 1; c2 < 16; ++c2) p[c2] = fma(tr[c], M[(o + c2) * kBtP + o + c], p[c2]);  // G(c, c2)
    }
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c >= i) M[(o + i) * kBtP + o + c] = tr[c];
  }
  __syncthreads();
  // ---- 2. merges: level s merges blocks [a0, a0+s) and [a0+s, a0+2s)
  for (int s = 16; s < jp; s *= 2) {
    const int nm = jp / (2 * s);           // merges at this level
    const int tm = s / 16, tn = s / 8;     // 16 x 8 tiles per s x s product
    const int ntiles = nm * tm * tn;
    // X = G_AB T_BB  (G_AB[i][l] = G(a0+s+l, a0+i) from the lower part; T_BB upper)
    for (int tile = warp; tile < ntiles; tile += kBtThreads / 32) {
      const int mg = tile / (tm * tn), tt = tile % (tm * tn);
      const int ti = (tt / tn) * 16, tc = (tt % tn) * 8;
      const int a0 = mg * 2 * s, b0 = a0 + s;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k0 = 0; k0 < min(s, tc + 8); k0 += 4) {  // T_BB[l][c] = 0 for l > c
        const int l = k0 + tq;
        const double a0v = M[(b0 + l) * kBtP + a0 + ti + gq];
        const double a1v = M[(b0 + l) * kBtP + a0 + ti + gq + 8];
        const int cc = tc + gq;
        const double bv = l <= cc ? M[(b0 + l) * kBtP + b0 + cc] : 0.0;
        dmma16x8x4(acc, a0v, a1v, bv);
      }
      double* X = Xs + mg * s * kBtXP;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) X[(ti + gq + 8 * h) * kBtXP + tc + 2 * tq + e] = acc[2 * h + e];
    }
    __syncthreads();
    // T_AB = -T_AA X  (T_AA upper: rows i use l >= i)
    for (int tile = warp; tile < ntiles; tile += kBtThreads / 32) {
      const int mg = tile / (tm * tn), tt = tile % (tm * tn);
      const int ti = (tt / tn) * 16, tc = (tt % tn) * 8;
      const int a0 = mg * 2 * s, b0 = a0 + s;
      const double* X = Xs + mg * s * kBtXP;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k0 = (ti / 4) * 4; k0 < s; k0 += 4) {
        const int l = k0 + tq;
        const int r0 = ti + gq, r1 = ti + gq + 8;
        const double a0v = l >= r0 ? M[(a0 + r0) * kBtP + a0 + l] : 0.0;
        const double a1v = l >= r1 ? M[(a0 + r1) * kBtP + a0 + l] : 0.0;
        const double bv = X[l * kBtXP + tc + gq];
        dmma16x8x4(acc, a0v, a1v, bv);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) M[(a0 + ti + gq + 8 * h) * kBtP + b0 + tc + 2 * tq + e] = -acc[2 * h + e];
    }
    __syncthreads();
  }
  for (int e = tid; e < j * j; e += kBtThreads) {
    const int r = e % j, c = e / j;
    T[(int64_t)c * ldt + r] = r <= c ? M[r * kBtP + c] : 0.0;
  }
}

}  // namespace

int build_t_fast(const double* Gm, int64_t ldg, const double* taus, int64_t j, double* T, int64_t ldt,
                 const int32_t* gate, cudaStream_t s) {
  if (j <= 0) return SQR_OK;
  if (j > 128) {
    set_error("build_t: %lld reflectors > 128", (long long)j);
    return SQR_EINVAL;
  }
  const int jp = j <= 16 ? 16 : j <= 32 ? 32 : j <= 64 ? 64 : 128;
  const int smem = (128 * kBtP + 64 * kBtXP) * 8;
  if (int rc = smem_optin((const void*)build_t_fast_kernel, smem)) return rc;
  ProfScope ps(kTagBuildT, s);
  build_t_fast_kernel<<<1, kBtThreads, smem, s>>>(Gm, ldg, taus, (int)j, jp, T, ldt, gate);
  SQR_LAUNCH("build_t_fast_kernel");
  return SQR_OK;
}

}  // namespace sqr
