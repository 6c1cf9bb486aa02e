// K2 + K12: halted column-pivoted QR of the l x nt sketch B on one persistent
// cooperative kernel (reference: sketch.py:97-119 -> reference.py:107-150).
//
// Layout: the nt sample columns are split into G contiguous chunks, one per
// CTA, held in shared memory (odd pitch => conflict-free thread-per-column
// access); columns beyond the smem capacity live in an L2-resident spill
// buffer.  Columns never move: pivoting is tracked with per-column
// "position" tags, reproducing the reference's swap sequence exactly
// (np.argmax over the swapped order => ties to the lowest POSITION).
//
// One grid barrier per pivot step: each CTA publishes its best (norm^2,
// position) candidate together with the candidate's column; after the
// barrier every CTA picks the same global winner, rebuilds the same
// reflector from the published column (deterministic fixed-order
// reductions), and applies it to its own columns while downdating norms
// with the reference's 2^-40 guard and exact recompute.
#include <float.h>
#include <math.h>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kSqThreads = 256;
constexpr int kMaxRowsPerLane = 5;  // spill path: ell <= 160
constexpr double kNormGuard = 0x1p-40;   // reference.py:40
constexpr double kRankFloor = 0x1p-52;   // reference.py:44
constexpr double kSampleFloor = 0x1p-48; // sketch.py:38

struct Cand {
  double val;
  int pos;
  int lc;
};

__device__ __forceinline__ bool better(double v1, int p1, double v2, int p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// Block-wide argmax of (val, pos) with ties to the lowest pos.  Result in out[0].
__device__ Cand block_argmax(Cand c, Cand* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v = __shfl_xor_sync(0xffffffffu, c.val, o);
    int p = __shfl_xor_sync(0xffffffffu, c.pos, o);
    int l = __shfl_xor_sync(0xffffffffu, c.lc, o);
    if (better(v, p, c.val, c.pos)) {
      c.val = v;
      c.pos = p;
      c.lc = l;
    }
  }
  __syncthreads();
  if (lane == 0) red[wid] = c;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    Cand d = lane < nw ? red[lane] : Cand{-1.0, INT_MAX, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v = __shfl_xor_sync(0xffffffffu, d.val, o);
      int p = __shfl_xor_sync(0xffffffffu, d.pos, o);
      int l = __shfl_xor_sync(0xffffffffu, d.lc, o);
      if (better(v, p, d.val, d.pos)) {
        d.val = v;
        d.pos = p;
        d.lc = l;
      }
    }
    if (lane == 0) red[0] = d;
  }
  __syncthreads();
  Cand r = red[0];
  __syncthreads();
  return r;
}

struct SampleArgs {
  const double* B;
  int64_t ldb;
  int ell, nt, bb, w, cap, ldS, first, warp_spill;
  double* Bf;
  int64_t ldbf;
  int64_t* lperm;
  int32_t* moves;
  double* taus;
  sqr_status* st;
  unsigned* bar;
  double* cval;    // [2][G]
  int* cpos;       // [2][G]
  double* ccol;    // [2][G][ell]
  double* psum;    // [G]
  double* pmax;    // [G]
  double* spill;   // [nt][ell] for columns beyond cap
};

__global__ void __launch_bounds__(kSqThreads, 1) sample_qrcp_kernel(SampleArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Cand red[32];
  __shared__ double sred[32];
  __shared__ int s_stop;
  if (a.st->stop) return;  // uniform: no CTA enters the barrier

  GridBarrier gb;
  gb.init(a.bar);
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int ell = a.ell;
  const int col0 = g * a.w;
  const int ncols = max(0, min(a.w, a.nt - col0));
  double* cols = sm;                                   // cap x ldS
  double* nsq = sm + (size_t)a.cap * a.ldS;            // w
  double* rsq = nsq + a.w;                             // w
  double* yv = rsq + a.w;                              // ell (+pad)
  int* pos = reinterpret_cast<int*>(yv + ell + 2);     // w

  auto colp = [&](int lc) -> double* {
    return lc < a.cap ? cols + (size_t)lc * a.ldS : a.spill + (size_t)(col0 + lc) * ell;
  };

  if (g == 0 && tid == 0) a.st->nmoves = 0;
  // Load my columns (coalesced along rows).
  for (int64_t e = tid; e < (int64_t)ncols * ell; e += kSqThreads) {
    const int lc = (int)(e / ell), r = (int)(e % ell);
    colp(lc)[r] = a.B[(int64_t)(col0 + lc) * a.ldb + r];
  }
  __syncthreads();
  double my_sum = 0.0, my_max = 0.0;
  for (int lc = tid; lc < ncols; lc += kSqThreads) {
    const double* d = colp(lc);
    double s = 0.0;
    for (int r = 0; r < ell; ++r) s = fma(d[r], d[r], s);
    nsq[lc] = s;
    rsq[lc] = s;
    pos[lc] = col0 + lc;
    my_sum += s;
    my_max = fmax(my_max, s);
  }
  // Deterministic CTA partials of sum / max of column norms^2.
  {
    double s = block_sum(my_sum, sred);
    double mx = my_max;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) sred[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < (kSqThreads >> 5); ++i) mx = fmax(mx, sred[i]);
      mx = fmax(mx, sred[0]);
      a.psum[g] = s;
      a.pmax[g] = mx;
    }
    __syncthreads();
  }
  gb.sync();
  double total = 0.0, gmax = 0.0;
  for (int i = 0; i < G; ++i) {
    total += __ldcg(a.psum + i);
    gmax = fmax(gmax, __ldcg(a.pmax + i));
  }
  const double fro = sqrt(total);
  const double rank_floor_sq = (kRankFloor * fro) * (kRankFloor * fro);
  double sample_floor;
  if (a.first) {
    sample_floor = kSampleFloor * kSampleFloor * gmax;
  } else {
    sample_floor = __ldcg(&a.st->floor_sq);
  }
  // Everyone must have read floor_sq before CTA 0 overwrites it.
  gb.sync();
  if (g == 0 && tid == 0 && a.first) a.st->floor_sq = sample_floor;
  if (a.nt == 0 || gmax <= sample_floor) {
    if (g == 0 && tid == 0) {
      a.st->stop = 1;
      a.st->reason = SQR_STOP_SAMPLE_FLOOR;
      a.st->sample_achieved = 0;
    }
    return;
  }

  int achieved = 0;
  for (int j = 0; j < a.bb; ++j) {
    const int par = j & 1;
    // Local candidate among active columns.
    Cand c{-1.0, INT_MAX, -1};
    for (int lc = tid; lc < ncols; lc += kSqThreads) {
      const int p = pos[lc];
      if (p >= 0 && better(nsq[lc], p, c.val, c.pos)) c = Cand{nsq[lc], p, lc};
    }
    c = block_argmax(c, red);
    if (tid == 0) {
      a.cval[par * G + g] = c.val;
      a.cpos[par * G + g] = c.pos;
    }
    if (c.lc >= 0) {
      const double* d = colp(c.lc);
      for (int r = j + tid; r < ell; r += kSqThreads) a.ccol[((size_t)par * G + g) * ell + r] = d[r];
    }
    gb.sync();
    // Global winner (identical on every CTA).
    Cand wbest{-1.0, INT_MAX, -1};
    for (int i = tid; i < G; i += kSqThreads) {
      const double v = __ldcg(a.cval + par * G + i);
      const int p = __ldcg(a.cpos + par * G + i);
      if (better(v, p, wbest.val, wbest.pos)) wbest = Cand{v, p, i};
    }
    wbest = block_argmax(wbest, red);
    if (wbest.val <= rank_floor_sq) break;  // reference.py:123-124
    const int pc = wbest.pos, gw = wbest.lc;
    const int len = ell - j;
    // Reflector from the published winner column (rows j..ell-1).
    const double* u = a.ccol + ((size_t)par * G + gw) * ell + j;
    double part = 0.0;
    for (int r = 1 + tid; r < len; r += kSqThreads) {
      const double x = __ldcg(u + r);
      part = fma(x, x, part);
    }
    const double s1 = block_sum(part, sred);
    const double u0 = __ldcg(u);
    const double nrm = sqrt(fma(u0, u0, s1));
    double beta = 0.0, tau = 0.0, y0 = 1.0;
    if (nrm != 0.0) {
      beta = (u0 >= 0.0 ? -1.0 : 1.0) * nrm;
      y0 = u0 - beta;
      tau = 2.0 / (1.0 + s1 / (y0 * y0));
    }
    for (int r = tid; r < len; r += kSqThreads) yv[r] = (r == 0) ? 1.0 : (nrm != 0.0 ? __ldcg(u + r) / y0 : 0.0);
    if (g == 0 && tid == 0) a.taus[j] = tau;
    __syncthreads();
    // Apply H_j to my active columns, downdate norms (reference.py:131-149).
    // Shared-memory columns: one thread per column.
    const int nsm = a.warp_spill ? min(ncols, a.cap) : ncols;
    for (int lc = tid; lc < nsm; lc += kSqThreads) {
      const int p = pos[lc];
      if (p < 0) continue;
      double* d = colp(lc);
      if (p == pc) {
        // The winner: final column j of the factored sample.
        for (int r = 0; r < j; ++r) a.Bf[(int64_t)j * a.ldbf + r] = d[r];
        a.Bf[(int64_t)j * a.ldbf + j] = beta;
        for (int r = 1; r < len; ++r) a.Bf[(int64_t)j * a.ldbf + j + r] = yv[r];
        a.lperm[j] = col0 + lc;
        if (col0 + lc != j) {
          const int slot = atomicAdd(&a.st->nmoves, 1);
          a.moves[2 * slot] = j;
          a.moves[2 * slot + 1] = col0 + lc;
        }
        pos[lc] = -1;
        continue;
      }
      if (p == j) pos[lc] = pc;  // the column that sat at position j moves to pc
      double dot = 0.0;
      int r = 0;
      for (; r + 4 <= len; r += 4) {
        dot = fma(yv[r], d[j + r], dot);
        dot = fma(yv[r + 1], d[j + r + 1], dot);
        dot = fma(yv[r + 2], d[j + r + 2], dot);
        dot = fma(yv[r + 3], d[j + r + 3], dot);
      }
      for (; r < len; ++r) dot = fma(yv[r], d[j + r], dot);
      const double wv = tau * dot;
      for (r = 0; r < len; ++r) d[j + r] = fma(-yv[r], wv, d[j + r]);
      const double rj = d[j];
      double ns = nsq[lc] - rj * rj;
      if (ns < kNormGuard * rsq[lc]) {
        double ex = 0.0;
        for (int q = j + 1; q < ell; ++q) ex = fma(d[q], d[q], ex);
        nsq[lc] = ex;
        rsq[lc] = ex;
      } else {
        nsq[lc] = fmax(ns, 0.0);
      }
    }
    // Spilled (L2-resident) columns: one warp per column, coalesced rows.
    for (int lc = a.cap + warp; a.warp_spill && lc < ncols; lc += kSqThreads / 32) {
      const int p = pos[lc];
      if (p < 0) continue;
      double* d = a.spill + (size_t)(col0 + lc) * ell;
      if (p == pc) {
        for (int r = lane; r < ell; r += 32)
          a.Bf[(int64_t)j * a.ldbf + r] = r < j ? __ldcg(d + r) : (r == j ? beta : yv[r - j]);
        if (lane == 0) {
          a.lperm[j] = col0 + lc;
          if (col0 + lc != j) {
            const int slot = atomicAdd(&a.st->nmoves, 1);
            a.moves[2 * slot] = j;
            a.moves[2 * slot + 1] = col0 + lc;
          }
          pos[lc] = -1;
        }
        __syncwarp();
        continue;
      }
      __syncwarp();
      if (p == j && lane == 0) pos[lc] = pc;
      double x[kMaxRowsPerLane];
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        x[i] = r < ell ? __ldcg(d + r) : 0.0;
      }
      double part = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        if (r < ell) part = fma(yv[r - j], x[i], part);
      }
      const double wv = tau * warp_sum(part);
      double ex = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        if (r < ell) {
          x[i] = fma(-yv[r - j], wv, x[i]);
          d[r] = x[i];
          if (r > j) ex = fma(x[i], x[i], ex);
        }
      }
      const double rj = __shfl_sync(0xffffffffu, x[0], 0);
      const double ns = nsq[lc] - rj * rj;
      const bool recompute = ns < kNormGuard * rsq[lc];
      ex = warp_sum(ex);
      __syncwarp();
      if (lane == 0) {
        if (recompute) {
          nsq[lc] = ex;
          rsq[lc] = ex;
        } else {
          nsq[lc] = fmax(ns, 0.0);
        }
      }
      __syncwarp();
    }
    achieved = j + 1;
    __syncthreads();
  }
  // Remaining (trailing) columns go to their final positions.
  for (int lc = tid; lc < ncols; lc += kSqThreads) {
    const int p = pos[lc];
    if (p < 0) continue;
    const double* d = colp(lc);
    for (int r = 0; r < ell; ++r) a.Bf[(int64_t)p * a.ldbf + r] = d[r];
    a.lperm[p] = col0 + lc;
    if (p != col0 + lc) {
      const int slot = atomicAdd(&a.st->nmoves, 1);
      a.moves[2 * slot] = p;
      a.moves[2 * slot + 1] = col0 + lc;
    }
  }
  if (g == 0 && tid == 0) {
    a.st->sample_achieved = achieved;
    if (achieved == 0) {
      a.st->stop = 1;
      a.st->reason = SQR_STOP_SAMPLE_RANK;
    }
  }
  (void)s_stop;
}

}  // namespace

struct SampleWorkspace {
  static int64_t bytes(int64_t ell, int64_t nt) {
    const int64_t G = 148;
    return 64 + 2 * G * 8 + 2 * G * 4 + 2 * G * ell * 8 + 2 * G * 8 + nt * ell * 8 + 1024;
  }
};

int64_t sample_qrcp_workspace(int64_t ell, int64_t nt) { return SampleWorkspace::bytes(ell, nt); }

int sample_qrcp(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st,
                void* ws, int64_t ws_bytes, cudaStream_t s) {
  if (ell <= 0 || nt < 0 || bb < 0 || bb > ell || bb > nt) {
    set_error("sample_qrcp: bad shape ell=%lld nt=%lld bb=%lld", (long long)ell, (long long)nt,
              (long long)bb);
    return SQR_EINVAL;
  }
  if (ws_bytes < SampleWorkspace::bytes(ell, nt)) {
    set_error("sample_qrcp: workspace too small");
    return SQR_EINVAL;
  }
  const int sms = sm_count();
  // At least 32 columns per CTA (amortise the per-step barrier), enough CTAs
  // to keep every column in shared memory when possible, one CTA per SM.
  const int ldS = (int)(ell | 1);
  const int64_t fixed_per_col = 16 + 4;
  const int64_t smem_avail = std::min<int64_t>(max_smem_optin(), 220 * 1024) - (ell + 2) * 8 - 64;
  const int64_t fit = std::max<int64_t>(1, smem_avail / ((int64_t)ldS * 8 + fixed_per_col));
  const int64_t ntc = std::max<int64_t>(nt, 1);
  int G = (int)std::min<int64_t>(sms, std::max<int64_t>(cdiv(ntc, 32), cdiv(ntc, fit)));
  G = std::max(G, 1);
  const int w = (int)cdiv(ntc, G);
  G = (int)cdiv(ntc, w);
  const int64_t fixed = (int64_t)w * 16 + (ell + 2) * 8 + (int64_t)w * 4 + 64;
  const int64_t budget = std::min<int64_t>(max_smem_optin(), 220 * 1024) - fixed;
  int cap = (int)std::max<int64_t>(0, std::min<int64_t>(w, budget / ((int64_t)ldS * 8)));
  const int64_t smem = (int64_t)cap * ldS * 8 + fixed;

  char* p = static_cast<char*>(ws);
  SampleArgs a;
  a.B = B;
  a.ldb = ldb;
  a.ell = (int)ell;
  a.nt = (int)nt;
  a.bb = (int)bb;
  a.w = w;
  a.cap = cap;
  a.ldS = ldS;
  a.first = first;
  a.warp_spill = ell <= 32 * kMaxRowsPerLane;
  a.Bf = Bf;
  a.ldbf = ldbf;
  a.lperm = lperm;
  a.moves = moves;
  a.taus = taus;
  a.st = st;
  a.bar = reinterpret_cast<unsigned*>(p);
  p += 64;
  a.cval = reinterpret_cast<double*>(p);
  p += 2 * 148 * 8;
  a.cpos = reinterpret_cast<int*>(p);
  p += 2 * 148 * 4;
  a.ccol = reinterpret_cast<double*>(p);
  p += 2 * 148 * ell * 8;
  a.psum = reinterpret_cast<double*>(p);
  p += 148 * 8;
  a.pmax = reinterpret_cast<double*>(p);
  p += 148 * 8;
  a.spill = reinterpret_cast<double*>(p);

  static int configured_smem = 0;
  if (smem > configured_smem) {
    SQR_CUDA(cudaFuncSetAttribute(sample_qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    configured_smem = (int)smem;
  }
  void* args[] = {&a};
  SQR_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  ProfScope ps(kTagSample, s);
  count_launch();
  SQR_CUDA(cudaLaunchCooperativeKernel((const void*)sample_qrcp_kernel, dim3(G), dim3(kSqThreads), args,
                                       (size_t)smem, s));
  return SQR_OK;
}

}  // namespace sqr

extern "C" int sqr_sample_qrcp(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb,
                               double* Bf, int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus,
                               int first, sqr_status* st, void* stream) {
  // Stand-alone entry: allocate its own scratch (tests / tools).  The drivers
  // use the workspace-taking internal entry.
  void* ws = nullptr;
  const int64_t bytes = sqr::sample_qrcp_workspace(ell, nt);
  if (cudaMallocAsync(&ws, bytes, static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    sqr::set_error("sqr_sample_qrcp: cudaMallocAsync failed");
    return SQR_ECUDA;
  }
  cudaMemsetAsync(ws, 0, 64, static_cast<cudaStream_t>(stream));
  int rc = sqr::sample_qrcp(B, ldb, ell, nt, bb, Bf, ldbf, lperm, moves, taus, first, st, ws, bytes,
                            static_cast<cudaStream_t>(stream));
  cudaFreeAsync(ws, static_cast<cudaStream_t>(stream));
  return rc;
}
