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
#include <stdlib.h>

#include <cooperative_groups.h>
#include <map>
#include <mutex>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kSqThreads = 256;
constexpr int kMaxRowsPerLane = 5;  // warp paths: ell <= 160
constexpr int kSpillPerWarp = 5;    // register-resident spill columns per warp
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

struct SampleArgs {
  const double* B;
  int64_t ldb;
  int ell, nt, bb, w, cap, ldS, first, warp_spill, reg_spill;
  double* Bf;
  int64_t ldbf;
  int64_t* lperm;
  int32_t* moves;
  double* taus;
  sqr_status* st;
  unsigned* bar;
  double2* cand;   // [2][G] {norm^2, position bits}: one 16-byte record per CTA
  double* ccol;    // [2][G][ell]
  double* psum;    // [G]
  double* pmax;    // [G]
  double* spill;   // [nt][ell] for columns beyond cap
  unsigned long long* trace;
};

__device__ __forceinline__ void warp_argmax(double& v, int& p, int& l) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
    const int l2 = __shfl_xor_sync(0xffffffffu, l, o);
    if (better(v2, p2, v, p)) {
      v = v2;
      p = p2;
      l = l2;
    }
  }
}

// Pivot step j (one grid barrier):
//   pass 1  every column: w_c = tau (y . d_c), new row-j entry d_c[j] - w_c,
//           norm downdate (+ exact recompute under the 2^-40 guard), local
//           candidate for step j+1; the winner column is written out.
//   publish the CTA candidate for step j+1 (value, position, updated column)
//           and ARRIVE at the grid barrier;
//   overlap warps 1..7: pass 2, d_c[j:] -= w_c y  (the rank-1 update)
//           warp 0:     wait for the barrier, pick the global winner, load
//                       its column, build reflector j+1 (y, tau, beta)
//   __syncthreads.
// so the rank-1 update hides the barrier and the two L2 round trips.
__global__ void __launch_bounds__(kSqThreads, 1) sample_qrcp_kernel(SampleArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double wv_s[kSqThreads / 32];
  __shared__ int wp_s[kSqThreads / 32], wl_s[kSqThreads / 32];
  __shared__ double sred[32];
  struct Bcast {
    int go, pc;
    double beta, tau;
  };
  __shared__ Bcast bc_s;
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
  double* wcol = rsq + a.w;                            // w: tau * (y . d_c) of the current step
  double* ybuf = wcol + a.w;                           // [2][ell + 2]: reflectors by step parity
  int* pos = reinterpret_cast<int*>(ybuf + 2 * (ell + 2));  // w

  auto colp = [&](int lc) -> double* {
    return lc < a.cap ? cols + (size_t)lc * a.ldS : a.spill + (size_t)(col0 + lc) * ell;
  };

  if (g == 0 && tid == 0) a.st->nmoves = 0;
  const int nld = a.reg_spill ? min(ncols, a.cap) : ncols;
  for (int64_t e0 = tid; e0 < (int64_t)nld * ell; e0 += 8 * kSqThreads) {  // 8 loads in flight
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = e0 + u * kSqThreads;
      v[u] = e < (int64_t)nld * ell ? a.B[(int64_t)(col0 + (int)(e / ell)) * a.ldb + (int)(e % ell)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = e0 + u * kSqThreads;
      if (e < (int64_t)nld * ell) colp((int)(e / ell))[(int)(e % ell)] = v[u];
    }
  }
  double xs[kSpillPerWarp][kMaxRowsPerLane];  // this warp's spill columns (reg mode)
#pragma unroll
  for (int i = 0; i < kSpillPerWarp; ++i) {
    const int lc = a.cap + warp + 8 * i;
#pragma unroll
    for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
      const int r = lane + 32 * qq;
      xs[i][qq] = (a.reg_spill && lc < ncols && r < ell) ? a.B[(int64_t)(col0 + lc) * a.ldb + r] : 0.0;
    }
  }
  __syncthreads();
  double my_sum = 0.0, my_max = 0.0;
  double cbv = -1.0;
  int cbp = INT_MAX, cbl = -1;
  for (int lc = tid; lc < nld; lc += kSqThreads) {
    const double* d = colp(lc);
    double s0 = 0.0, s1 = 0.0;
    int r = 0;
    for (; r + 2 <= ell; r += 2) {
      s0 = fma(d[r], d[r], s0);
      s1 = fma(d[r + 1], d[r + 1], s1);
    }
    if (r < ell) s0 = fma(d[r], d[r], s0);
    const double s = s0 + s1;
    nsq[lc] = s;
    rsq[lc] = s;
    wcol[lc] = 0.0;
    pos[lc] = col0 + lc;
    my_sum += s;
    my_max = fmax(my_max, s);
    if (better(s, col0 + lc, cbv, cbp)) {
      cbv = s;
      cbp = col0 + lc;
      cbl = lc;
    }
  }
  if (a.reg_spill) {
#pragma unroll
    for (int i = 0; i < kSpillPerWarp; ++i) {
      const int lc = a.cap + warp + 8 * i;
      if (lc >= ncols) continue;
      double s = 0.0;
#pragma unroll
      for (int qq = 0; qq < kMaxRowsPerLane; ++qq) s = fma(xs[i][qq], xs[i][qq], s);
      s = warp_sum(s);
      if (lane == 0) {
        nsq[lc] = s;
        rsq[lc] = s;
        wcol[lc] = 0.0;
        pos[lc] = col0 + lc;
        my_sum += s;
        my_max = fmax(my_max, s);
        if (better(s, col0 + lc, cbv, cbp)) {
          cbv = s;
          cbp = col0 + lc;
          cbl = lc;
        }
      }
    }
  }
  {
    const double s = block_sum(my_sum, sred);
    double mx = my_max;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sred[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < (kSqThreads >> 5); ++i) mx = fmax(mx, sred[i]);
      mx = fmax(mx, sred[0]);
      a.psum[g] = s;
      a.pmax[g] = mx;
    }
  }
  gb.sync();
  double total = 0.0, gmax = 0.0;
  for (int i = 0; i < G; ++i) {
    total += __ldcg(a.psum + i);
    gmax = fmax(gmax, __ldcg(a.pmax + i));
  }
  const double fro = sqrt(total);
  const double rank_floor_sq = (kRankFloor * fro) * (kRankFloor * fro);
  const double sample_floor = a.first ? kSampleFloor * kSampleFloor * gmax : __ldcg(&a.st->floor_sq);
  if (a.nt == 0 || gmax <= sample_floor) {
    if (g == 0 && tid == 0) {
      if (a.first) a.st->floor_sq = sample_floor;
      a.st->stop = 1;
      a.st->reason = SQR_STOP_SAMPLE_FLOOR;
      a.st->sample_achieved = 0;
    }
    return;
  }
  if (g == 0 && tid == 0 && a.first) a.st->floor_sq = sample_floor;

  // CTA candidate -> publish (value, position, column rows jn.. updated by
  // reflector jn-1 with coefficient wcol / y of parity (jn-1)&1).
  auto publish = [&](int jn) {
    warp_argmax(cbv, cbp, cbl);
    if (lane == 0) {
      wv_s[warp] = cbv;
      wp_s[warp] = cbp;
      wl_s[warp] = cbl;
    }
    __syncthreads();
    double v = lane < (kSqThreads >> 5) ? wv_s[lane] : -1.0;
    int p = lane < (kSqThreads >> 5) ? wp_s[lane] : INT_MAX;
    int l = lane < (kSqThreads >> 5) ? wl_s[lane] : -1;
    warp_argmax(v, p, l);
    const int par = jn & 1;
    if (warp == 0 && lane == 0) a.cand[par * G + g] = make_double2(v, __longlong_as_double((long long)p));
    double* dst = a.ccol + ((size_t)par * G + g) * ell;
    if (l >= 0 && (!a.reg_spill || l < a.cap)) {
      if (warp == 0) {
        const double* d = colp(l);
        const bool lazy = !a.warp_spill || l < a.cap;  // columns updated by pass 2
        if (jn == 0 || !lazy) {
          for (int r = jn + lane; r < ell; r += 32) dst[r] = d[r];
        } else {  // pass 2 of step jn-1 has not run yet: apply it on the fly
          const double* yp = ybuf + ((jn - 1) & 1) * (ell + 2);
          const double wl = wcol[l];
          for (int r = jn + lane; r < ell; r += 32) dst[r] = fma(-yp[r - (jn - 1)], wl, d[r]);
        }
      }
    } else if (l >= 0 && warp == (l - a.cap) % 8) {
      const int iw = (l - a.cap) / 8;
#pragma unroll
      for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
        double vv = xs[0][qq];
#pragma unroll
        for (int i = 1; i < kSpillPerWarp; ++i) {
          const double c = xs[i][qq];
          asm("{ .reg .pred p; setp.eq.s32 p, %2, %3; selp.f64 %0, %1, %0, p; }" : "+d"(vv) : "d"(c), "r"(iw), "r"(i));
        }
        const int r = lane + 32 * qq;
        if (r >= jn && r < ell) dst[r] = vv;
      }
    }
  };

  // Global winner of step jn + reflector, by ONE warp (lane 0 waited).
  auto winner = [&](int jn) {
    const int par = jn & 1;
    double bv = -1.0;
    int bp = INT_MAX, bl = -1;
    {
      // all records in flight at once (G <= 160), then a local + warp argmax
      double2 rec[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        rec[k] = i < G ? __ldcg(a.cand + par * G + i) : make_double2(-1.0, __longlong_as_double((long long)INT_MAX));
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int p = (int)__double_as_longlong(rec[k].y);
        if (better(rec[k].x, p, bv, bp)) {
          bv = rec[k].x;
          bp = p;
          bl = lane + 32 * k;
        }
      }
    }
    warp_argmax(bv, bp, bl);
    if (lane == 0) SQR_TRACE(a.trace, 8 * (jn - 1) + 7);
    const int len = ell - jn;
    double* ysh = ybuf + par * (ell + 2);
    double x[kMaxRowsPerLane];
    double s1 = 0.0, nrm = 0.0, beta = 0.0, tau = 0.0, y0 = 1.0;
    const bool go = bv > rank_floor_sq;  // reference.py:123-124
    if (go) {
      const double* u = a.ccol + ((size_t)par * G + bl) * ell + jn;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = lane + 32 * i;
        x[i] = r < len ? __ldcg(u + r) : 0.0;
      }
      for (int r = lane + 32 * kMaxRowsPerLane; r < len; r += 32) {  // tall samples only
        const double v = __ldcg(u + r);
        s1 = fma(v, v, s1);
      }
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i)
        if (lane + 32 * i >= 1) s1 = fma(x[i], x[i], s1);
      s1 = warp_sum(s1);
      const double u0 = __shfl_sync(0xffffffffu, x[0], 0);
      nrm = sqrt(fma(u0, u0, s1));
      if (nrm != 0.0) {
        beta = (u0 >= 0.0 ? -1.0 : 1.0) * nrm;
        y0 = u0 - beta;
        tau = 2.0 / (1.0 + s1 / (y0 * y0));
      }
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = lane + 32 * i;
        if (r < len) ysh[r] = (r == 0) ? 1.0 : (nrm != 0.0 ? x[i] / y0 : 0.0);
      }
      for (int r = lane + 32 * kMaxRowsPerLane; r < len; r += 32) ysh[r] = nrm != 0.0 ? __ldcg(u + r) / y0 : 0.0;
    }
    if (lane == 0) {
      bc_s.go = go;
      bc_s.pc = bp;
      bc_s.beta = beta;
      bc_s.tau = tau;
    }
  };

  // Pass 2 of step j: d[j:] -= w y on shared-memory columns; threads
  // [t0, kSqThreads) cooperate, one column per thread.
  auto pass2 = [&](int j, int t0) {
    const double* yw = ybuf + (j & 1) * (ell + 2);
    const int nsm = a.warp_spill ? min(ncols, a.cap) : ncols;
    const int len = ell - j;
    for (int lc = tid - t0; lc < nsm; lc += kSqThreads - t0) {
      if (pos[lc] < 0) continue;
      const double wvv = wcol[lc];
      double* dj = (a.warp_spill ? cols + (size_t)lc * a.ldS : colp(lc)) + j;
      int r = 0;
      for (; r + 2 <= len; r += 2) {
        const double p0 = dj[r], p1 = dj[r + 1];
        dj[r] = fma(-yw[r], wvv, p0);
        dj[r + 1] = fma(-yw[r + 1], wvv, p1);
      }
      if (r < len) dj[r] = fma(-yw[r], wvv, dj[r]);
    }
  };

  publish(0);
  gb.sync();
  if (warp == 0) winner(0);
  __syncthreads();

  int achieved = 0;
  for (int j = 0; j < a.bb; ++j) {
    SQR_TRACE(a.trace, 8 * j + 0);
    if (!bc_s.go) break;  // uniform across the grid
    const int pc = bc_s.pc;
    const double beta = bc_s.beta, tau = bc_s.tau;
    const int len = ell - j;
    const double* yw = ybuf + (j & 1) * (ell + 2);
    if (g == 0 && tid == 0) a.taus[j] = tau;

    // ---- pass 1: dots, downdates, next candidate; winner column written out.
    cbv = -1.0;
    cbp = INT_MAX;
    cbl = -1;
    const int nsm = a.warp_spill ? min(ncols, a.cap) : ncols;
    for (int lc = tid; lc < nsm; lc += kSqThreads) {
      const int p = pos[lc];
      if (p < 0) continue;
      double* d = a.warp_spill ? cols + (size_t)lc * a.ldS : colp(lc);
      if (p == pc) {
        for (int r = 0; r < j; ++r) a.Bf[(int64_t)j * a.ldbf + r] = d[r];
        a.Bf[(int64_t)j * a.ldbf + j] = beta;
        for (int r = 1; r < len; ++r) a.Bf[(int64_t)j * a.ldbf + j + r] = yw[r];
        a.lperm[j] = col0 + lc;
        if (col0 + lc != j) {
          const int slot = atomicAdd(&a.st->nmoves, 1);
          a.moves[2 * slot] = j;
          a.moves[2 * slot + 1] = col0 + lc;
        }
        pos[lc] = -1;
        continue;
      }
      const int pn = (p == j) ? pc : p;  // the column that sat at position j moves to pc
      pos[lc] = pn;
      const double* dj = d + j;
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
      int r = 0;
      for (; r + 4 <= len; r += 4) {
        d0 = fma(yw[r], dj[r], d0);
        d1 = fma(yw[r + 1], dj[r + 1], d1);
        d2 = fma(yw[r + 2], dj[r + 2], d2);
        d3 = fma(yw[r + 3], dj[r + 3], d3);
      }
      for (; r < len; ++r) d0 = fma(yw[r], dj[r], d0);
      const double wvv = tau * ((d0 + d1) + (d2 + d3));
      wcol[lc] = wvv;
      const double rj = fma(-yw[0], wvv, dj[0]);
      double ns = nsq[lc] - rj * rj;
      if (ns < kNormGuard * rsq[lc]) {
        double e0 = 0.0, e1 = 0.0;
        for (int qn = 1; qn < len; ++qn) {
          const double v = fma(-yw[qn], wvv, dj[qn]);
          if (qn & 1) e1 = fma(v, v, e1); else e0 = fma(v, v, e0);
        }
        ns = e0 + e1;
        rsq[lc] = ns;
      } else {
        ns = fmax(ns, 0.0);
      }
      nsq[lc] = ns;
      if (better(ns, pn, cbv, cbp)) {
        cbv = ns;
        cbp = pn;
        cbl = lc;
      }
    }
    SQR_TRACE(a.trace, 8 * j + 1);
    // Register-resident spill columns: warp q owns columns cap + q + 8 i
    // (i < 5), lanes own rows.  The five columns' warp reductions are
    // interleaved (one shuffle chain of depth 5 instead of five), and the
    // exact-recompute reduction only runs when the guard fires.
    if (a.reg_spill) {
      int pcol[kSpillPerWarp];
      double dot[kSpillPerWarp];
#pragma unroll
      for (int i = 0; i < kSpillPerWarp; ++i) {
        const int lc = a.cap + warp + 8 * i;
        pcol[i] = lc < ncols ? pos[lc] : -1;
        dot[i] = 0.0;
#pragma unroll
        for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
          const int r = lane + 32 * qq;
          if (r >= j && r < ell) dot[i] = fma(yw[r - j], xs[i][qq], dot[i]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < kSpillPerWarp; ++i) dot[i] += __shfl_xor_sync(0xffffffffu, dot[i], o);
      double ex[kSpillPerWarp], rjv[kSpillPerWarp];
#pragma unroll
      for (int i = 0; i < kSpillPerWarp; ++i) {
        const int lc = a.cap + warp + 8 * i;
        ex[i] = 0.0;
        rjv[i] = 0.0;
        if (pcol[i] < 0) continue;
        if (pcol[i] == pc) {  // the winner: its final column goes to Bf (xs untouched)
#pragma unroll
          for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
            const int r = lane + 32 * qq;
            if (r < ell) a.Bf[(int64_t)j * a.ldbf + r] = r < j ? xs[i][qq] : (r == j ? beta : yw[r - j]);
          }
          if (lane == 0) {
            a.lperm[j] = col0 + lc;
            if (col0 + lc != j) {
              const int slot = atomicAdd(&a.st->nmoves, 1);
              a.moves[2 * slot] = j;
              a.moves[2 * slot + 1] = col0 + lc;
            }
          }
          continue;
        }
        const double wvv = tau * dot[i];
#pragma unroll
        for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
          const int r = lane + 32 * qq;
          if (r >= j && r < ell) {
            xs[i][qq] = fma(-yw[r - j], wvv, xs[i][qq]);
            if (r > j) ex[i] = fma(xs[i][qq], xs[i][qq], ex[i]);
          }
          // select, not xs[i][j >> 5]: a dynamic index would demote xs to local memory
          asm("{ .reg .pred p; setp.eq.s32 p, %2, %3; selp.f64 %0, %1, %0, p; }"
              : "+d"(rjv[i]) : "d"(xs[i][qq]), "r"(j >> 5), "r"(qq));
        }
      }
      bool need = false;
      double nsv[kSpillPerWarp];
#pragma unroll
      for (int i = 0; i < kSpillPerWarp; ++i) {
        const int lc = a.cap + warp + 8 * i;
        const double rj = __shfl_sync(0xffffffffu, rjv[i], j & 31);
        nsv[i] = 0.0;
        if (pcol[i] < 0 || pcol[i] == pc) continue;
        nsv[i] = nsq[lc] - rj * rj;
        need |= nsv[i] < kNormGuard * rsq[lc];
      }
      if (need) {  // warp-uniform
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int i = 0; i < kSpillPerWarp; ++i) ex[i] += __shfl_xor_sync(0xffffffffu, ex[i], o);
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kSpillPerWarp; ++i) {
          const int lc = a.cap + warp + 8 * i;
          const int p = pcol[i];
          if (p < 0) continue;
          if (p == pc) {
            pos[lc] = -1;
            continue;
          }
          const int pn = (p == j) ? pc : p;
          double ns = nsv[i];
          if (ns < kNormGuard * rsq[lc]) {
            ns = ex[i];
            rsq[lc] = ns;
          } else {
            ns = fmax(ns, 0.0);
          }
          nsq[lc] = ns;
          pos[lc] = pn;
          if (better(ns, pn, cbv, cbp)) {
            cbv = ns;
            cbp = pn;
            cbl = lc;
          }
        }
      }
      __syncwarp();
    }
    // Spilled (L2-resident) columns (no reg mode): one warp per column, full update.
    for (int lc = a.cap + warp; a.warp_spill && !a.reg_spill && lc < ncols; lc += kSqThreads / 32) {
      const int p = pos[lc];
      if (p < 0) continue;
      double* d = a.spill + (size_t)(col0 + lc) * ell;
      if (p == pc) {
        for (int r = lane; r < ell; r += 32)
          a.Bf[(int64_t)j * a.ldbf + r] = r < j ? __ldcg(d + r) : (r == j ? beta : yw[r - j]);
        __syncwarp();
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
      const int pn = (p == j) ? pc : p;
      double xg[kMaxRowsPerLane];
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        xg[i] = r < ell ? __ldcg(d + r) : 0.0;
      }
      double part = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        if (r < ell) part = fma(yw[r - j], xg[i], part);
      }
      const double wvv = tau * warp_sum(part);
      double ex = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = j + lane + 32 * i;
        if (r < ell) {
          xg[i] = fma(-yw[r - j], wvv, xg[i]);
          d[r] = xg[i];
          if (r > j) ex = fma(xg[i], xg[i], ex);
        }
      }
      const double rj = __shfl_sync(0xffffffffu, xg[0], 0);
      double ns = nsq[lc] - rj * rj;
      const bool recompute = ns < kNormGuard * rsq[lc];
      ex = warp_sum(ex);
      ns = recompute ? ex : fmax(ns, 0.0);
      __syncwarp();
      if (lane == 0) {
        if (recompute) rsq[lc] = ex;
        nsq[lc] = ns;
        pos[lc] = pn;
        if (better(ns, pn, cbv, cbp)) {
          cbv = ns;
          cbp = pn;
          cbl = lc;
        }
      }
      __syncwarp();
    }
    achieved = j + 1;
    SQR_TRACE(a.trace, 8 * j + 2);
    if (j + 1 < a.bb) {
      publish(j + 1);
      gb.arrive();
      SQR_TRACE(a.trace, 8 * j + 3);
      if (warp == 0) {
        if (lane == 0) gb.wait_lane0();
        if (lane == 0) SQR_TRACE(a.trace, 8 * j + 6);
        __syncwarp();
        winner(j + 1);
      } else {
        pass2(j, 32);
      }
      SQR_TRACE(a.trace, 8 * j + 4);
      __syncthreads();
    } else {
      pass2(j, 0);
      __syncthreads();
    }
    SQR_TRACE(a.trace, 8 * j + 5);
  }
  __syncthreads();
  if (a.reg_spill) {
#pragma unroll
    for (int i = 0; i < kSpillPerWarp; ++i) {
      const int lc = a.cap + warp + 8 * i;
      if (lc >= ncols) continue;
      const int p = pos[lc];
      if (p < 0) continue;
#pragma unroll
      for (int qq = 0; qq < kMaxRowsPerLane; ++qq) {
        const int r = lane + 32 * qq;
        if (r < ell) a.Bf[(int64_t)p * a.ldbf + r] = xs[i][qq];
      }
      if (lane == 0) {
        a.lperm[p] = col0 + lc;
        if (p != col0 + lc) {
          const int slot = atomicAdd(&a.st->nmoves, 1);
          a.moves[2 * slot] = p;
          a.moves[2 * slot + 1] = col0 + lc;
        }
      }
    }
  }
  // Remaining (trailing) columns go to their final positions.
  for (int lc = tid; lc < (a.reg_spill ? min(ncols, a.cap) : ncols); lc += kSqThreads) {
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
}

// ---------------------------------------------------------------------------
// Thread-per-column variant (nt <= 256 G, ell <= 144): thread t of CTA g owns
// sample column 256 g + t for the whole launch.  Rows [RS, ell) (the last 48,
// RS = ell - 48) live in REGISTERS, rows [0, RS) in shared memory (row-major
// over the 256 columns: conflict-free), so the dot / update / downdate of a
// step are thread-local.  The reflector is kept as a full-length vector (zeros
// above the pivot row) so the register loops need no predicate.  Register
// rows are updated at once; the shared-memory rows' rank-1 update is deferred
// to the barrier wait (warps 1-7, while warp 0 selects the winner), and the
// published candidate column gets it applied on the fly.  One grid barrier per
// step; same arithmetic, downdate guard / exact recompute and tie rule as
// sample_qrcp_kernel.
constexpr int kRT = 256;
constexpr int kRR = 48;  // register rows
constexpr int kMaxEllCl = 144;  // sample rows supported by the cluster variant

// shared-memory pair load the compiler may not CSE (keeps 64 y values from
// staying live across the dot and the update loops)
__device__ __forceinline__ double2 lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

struct RegArgs {
  const double* B;
  int64_t ldb;
  int ell, nt, bb, first, RS;
  double* Bf;
  int64_t ldbf;
  int64_t* lperm;
  int32_t* moves;
  double* taus;
  sqr_status* st;
  unsigned* bar;
  double2* cand;
  double* ccol;
  double* psum;
  double* pmax;
  unsigned long long* trace;
  ResidentSig sig;
};

__device__ __forceinline__ void add_move(const RegArgs& a, int dst, int src) {
  const int slot = atomicAdd(&a.st->nmoves, 1);
  a.moves[2 * slot] = dst;
  a.moves[2 * slot + 1] = src;
}

// CL = true: the whole grid is ONE thread-block cluster (<= 16 CTAs, n_t <=
// 4096): the per-step candidate exchange goes through distributed shared
// memory (each CTA's record and candidate column stay in its own shared
// memory, readers map them with map_shared_rank) and the grid barrier is
// the hardware cluster barrier (arrive.release / wait.acquire), instead of
// L2 records, a fence and an atomic counter.
template <bool CL>
__global__ void __launch_bounds__(kRT, 1) sample_qrcp_reg_kernel(RegArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) double2 crec_s[2][16];    // CL: every CTA's candidate record (pushed), per parity
  __shared__ __align__(16) double ccol_s[2][kMaxEllCl];  // CL: my candidate column per step parity
  __shared__ double xs_s[2];                         // CL: my (sum, max) of the initial norms
  const int ell = a.ell, RS = a.RS;
  const int YP = ((max(ell, RS + kRR) + 1) | 1) + 1;  // even pitch of a reflector buffer
  double* cs = sm;                                     // [RS][kRT]
  double* ybase = cs + (size_t)RS * kRT;               // [2][YP]: reflectors by step parity
  const int yoff = RS & 1;                             // makes &y[RS] 16-byte aligned
  double* wcol = ybase + 2 * YP + 2;                   // [kRT]: tau (y . d_c) of the current step
  __shared__ __align__(16) double stg[kRR];            // publish staging of register rows
  __shared__ double wv_s[kRT / 32];
  __shared__ int wp_s[kRT / 32], wl_s[kRT / 32];
  __shared__ double sred[32];
  struct Bcast {
    int go, pc;
    double beta, tau;
  };
  __shared__ Bcast bc_s;
  if (a.st->stop) {
    if (blockIdx.x == 0 && threadIdx.x == 0) signal_resident(a.sig);
    return;
  }
  GridBarrier gb;
  if (!CL) gb.init(a.bar);
  namespace cg = cooperative_groups;
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  // CTAs are dispatched in index order: once the last one runs, all are resident
  if (g == G - 1 && tid == 0) signal_resident(a.sig);
  const int lane = tid & 31, warp = tid >> 5;
  const int col = g * kRT + tid;
  const bool own = col < a.nt;
  auto ybuf = [&](int par) -> double* { return ybase + par * YP + yoff; };
  // Moves without atomics (an atomicAdd round trip in the pivot's CTA sat on
  // the critical path of every step): slot j <- the pivot of step j, slot
  // bb + j <- the column displaced at step j if that is where it ends; -1
  // marks a no-op.  CTA 0 pre-fills 2*bb slots before the first barrier.
  if (g == 0) {
    for (int e = tid; e < 4 * a.bb; e += kRT) a.moves[e] = -1;
    if (tid == 0) a.st->nmoves = 2 * a.bb;
  }
  int disp = -1;  // step at which my column was last displaced
  int pj = -1;     // step at which my column became the pivot
  double pbeta = 0.0;
  for (int e = tid; e < 2 * YP; e += kRT) ybase[e] = 0.0;  // zero rows beyond ell (ell < 64)

  // ---- load my column: rows [0, RS) to shared memory, [RS, ell) to registers
  double xr[kRR];
  {
    const double* src = a.B + (int64_t)col * a.ldb;
    for (int r = 0; r < RS; ++r) cs[r * kRT + tid] = own ? src[r] : 0.0;
#pragma unroll
    for (int q = 0; q < kRR; ++q) xr[q] = (own && RS + q < ell) ? src[RS + q] : 0.0;
  }
  double nsq = 0.0;
  {
    double s0 = 0.0, s1 = 0.0;
    for (int r = 0; r < RS; ++r) {
      const double v = cs[r * kRT + tid];
      s0 = fma(v, v, s0);
    }
#pragma unroll
    for (int q = 0; q < kRR; q += 2) {
      s0 = fma(xr[q], xr[q], s0);
      s1 = fma(xr[q + 1], xr[q + 1], s1);
    }
    nsq = s0 + s1;
  }
  double rsq = nsq;
  int pos = own ? col : -1;
  double cbv = own ? nsq : -1.0;
  int cbp = own ? col : INT_MAX;
  int cbl = own ? tid : -1;
  {
    const double s = block_sum(own ? nsq : 0.0, sred);
    double mx = own ? nsq : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sred[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < (kRT >> 5); ++i) mx = fmax(mx, sred[i]);
      mx = fmax(mx, sred[0]);
      if (CL) {
        xs_s[0] = s;
        xs_s[1] = mx;
      } else {
        a.psum[g] = s;
        a.pmax[g] = mx;
      }
    }
  }
  double total = 0.0, gmax = 0.0;
  if (CL) {
    cg::this_cluster().sync();
    for (int i = 0; i < G; ++i) {
      const double* rx = cg::this_cluster().map_shared_rank(xs_s, i);
      total += rx[0];
      gmax = fmax(gmax, rx[1]);
    }
  } else {
    gb.sync();
    for (int i = 0; i < G; ++i) {
      total += __ldcg(a.psum + i);
      gmax = fmax(gmax, __ldcg(a.pmax + i));
    }
  }
  const double fro = sqrt(total);
  const double rank_floor_sq = (kRankFloor * fro) * (kRankFloor * fro);
  const double sample_floor = a.first ? kSampleFloor * kSampleFloor * gmax : __ldcg(&a.st->floor_sq);
  if (a.nt == 0 || gmax <= sample_floor) {
    if (g == 0 && tid == 0) {
      if (a.first) a.st->floor_sq = sample_floor;
      a.st->stop = 1;
      a.st->reason = SQR_STOP_SAMPLE_FLOOR;
      a.st->sample_achieved = 0;
    }
    if (CL) cg::this_cluster().sync();  // peers may still be reading my xs_s
    return;
  }
  if (g == 0 && tid == 0 && a.first) a.st->floor_sq = sample_floor;

  // CTA candidate for step jn -> publish (value, position, column rows jn..).
  // Shared-memory rows still miss the deferred update of step jn-1 (w, y of
  // parity (jn-1)&1): it is applied on the fly.
  auto publish = [&](int jn) {
    warp_argmax(cbv, cbp, cbl);
    if (lane == 0) {
      wv_s[warp] = cbv;
      wp_s[warp] = cbp;
      wl_s[warp] = cbl;
    }
    __syncthreads();
    double v = lane < (kRT >> 5) ? wv_s[lane] : -1.0;
    int p = lane < (kRT >> 5) ? wp_s[lane] : INT_MAX;
    int l = lane < (kRT >> 5) ? wl_s[lane] : -1;
    warp_argmax(v, p, l);
    const int par = jn & 1;
    if (CL) {
      // push my record into every peer's shared memory (lane q -> CTA q):
      // after the cluster barrier each reader finds all records locally
      if (warp == 0 && lane < G)
        *cg::this_cluster().map_shared_rank(&crec_s[par][g], lane) =
            make_double2(v, __longlong_as_double((long long)p));
    } else if (tid == 0) {
      a.cand[par * G + g] = make_double2(v, __longlong_as_double((long long)p));
    }
    if (l >= 0 && warp == (l >> 5)) {
      double* dst = CL ? ccol_s[par] : a.ccol + ((size_t)par * G + g) * ell;
      if (tid == l) {
#pragma unroll
        for (int q = 0; q < kRR; q += 2) *reinterpret_cast<double2*>(stg + q) = make_double2(xr[q], xr[q + 1]);
      }
      __syncwarp();
      const double* yp = ybuf((jn - 1) & 1);
      const double wl = jn > 0 ? wcol[l] : 0.0;
      for (int r = jn + lane; r < RS; r += 32) dst[r] = fma(-yp[r], wl, cs[r * kRT + l]);
      for (int q = lane; q < kRR; q += 32)
        if (RS + q >= jn && RS + q < ell) dst[RS + q] = stg[q];
    }
  };
  // global winner of step jn + its reflector (warp 0, lane 0 waited)
  auto winner = [&](int jn) {
    const int par = jn & 1;
    double bv = -1.0;
    int bp = INT_MAX, bl = -1;
    {
      double2 rec[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (CL)
          rec[k] = i < G ? crec_s[par][i] : make_double2(-1.0, __longlong_as_double((long long)INT_MAX));
        else
          rec[k] = i < G ? __ldcg(a.cand + par * G + i)
                         : make_double2(-1.0, __longlong_as_double((long long)INT_MAX));
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int p = (int)__double_as_longlong(rec[k].y);
        if (better(rec[k].x, p, bv, bp)) {
          bv = rec[k].x;
          bp = p;
          bl = lane + 32 * k;
        }
      }
    }
    warp_argmax(bv, bp, bl);
    const int len = ell - jn;
    double x[kMaxRowsPerLane];
    double s1 = 0.0, nrm = 0.0, beta = 0.0, tau = 0.0, y0 = 1.0;
    const bool go = bv > rank_floor_sq;  // reference.py:123-124
    if (go) {
      const double* u = CL ? cg::this_cluster().map_shared_rank(ccol_s[par], bl) + jn
                           : a.ccol + ((size_t)par * G + bl) * ell + jn;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = lane + 32 * i;
        x[i] = r < len ? (CL ? u[r] : __ldcg(u + r)) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i)
        if (lane + 32 * i >= 1) s1 = fma(x[i], x[i], s1);
      s1 = warp_sum(s1);
      const double u0 = __shfl_sync(0xffffffffu, x[0], 0);
      nrm = sqrt(fma(u0, u0, s1));
      double ry = 1.0;
      if (nrm != 0.0) {
        beta = (u0 >= 0.0 ? -1.0 : 1.0) * nrm;
        y0 = u0 - beta;
        ry = __drcp_rn(y0);
        tau = 2.0 / (1.0 + s1 / (y0 * y0));
      }
      double* yf = ybuf(par);
      for (int r = lane; r < jn; r += 32) yf[r] = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRowsPerLane; ++i) {
        const int r = lane + 32 * i;
        if (r < len) yf[jn + r] = (r == 0) ? 1.0 : (nrm != 0.0 ? div_rn(x[i], y0, ry) : 0.0);
      }
    }
    if (lane == 0) {
      bc_s.go = go;
      bc_s.pc = bp;
      bc_s.beta = beta;
      bc_s.tau = tau;
    }
  };
  // deferred rank-1 update of the shared-memory rows [jd, RS) with step jd's
  // (wcol, y), by threads [t0, kRT): rows outer, columns inner (coalesced)
  auto smem_update = [&](int jd, int t0) {
    const double* yp = ybuf(jd & 1);
    if (t0 == 32) {
      // warps 1..7 (224 threads): thread t owns column t (its w in a
      // register) for all rows, and rows jd + w' + 7k of column 224 + lane
      // of the last 32 columns: 8/7 of a column per thread, 2 shared loads
      // + 1 store per cell (no per-cell w reload)
      const int t = tid - 32, lw = t >> 5;
      const double wc = wcol[t], wx = wcol[224 + lane];
      for (int r = jd; r < RS; ++r) cs[r * kRT + t] = fma(-yp[r], wc, cs[r * kRT + t]);
      for (int r = jd + lw; r < RS; r += 7) cs[r * kRT + 224 + lane] = fma(-yp[r], wx, cs[r * kRT + 224 + lane]);
      return;
    }
    const int nthr = kRT - t0;
    const int ncell = (RS - jd) * kRT;
    for (int e = tid - t0; e < ncell; e += nthr) {
      const int r = jd + e / kRT, c = e % kRT;
      cs[r * kRT + c] = fma(-yp[r], wcol[c], cs[r * kRT + c]);
    }
  };

  publish(0);
  if (CL)
    cg::this_cluster().sync();
  else
    gb.sync();
  if (warp == 0) winner(0);
  __syncthreads();

  int achieved = 0;
  for (int j = 0; j < a.bb; ++j) {
    SQR_TRACE(a.trace, 8 * j + 0);
    if (!bc_s.go) break;  // uniform across the grid
    const int pc = bc_s.pc;
    const double beta = bc_s.beta, tau = bc_s.tau;
    const double* yf = ybuf(j & 1);
    if (g == 0 && tid == 0) a.taus[j] = tau;
    cbv = -1.0;
    cbp = INT_MAX;
    cbl = -1;
    double wvv = 0.0;
    if (pos == pc) {
      // the pivot: its column is frozen from here on (w = 0 in every later
      // update), so Bf column j (R part, beta, reflector tail u / (u_j -
      // beta)) is written after the loop -- no global stores in the step
      // that the grid barrier's release would have to wait for
      pj = j;
      pbeta = beta;
      pos = -1;
    } else if (pos >= 0) {
      const int pn = (pos == j) ? pc : pos;  // the column at position j moves to pc
      if (pos == j) {
        if (disp >= 0) a.moves[2 * (a.bb + disp)] = -1;
        disp = j;
      }
      pos = pn;
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
      {
        int r = j;
        for (; r + 2 <= RS; r += 2) {
          d2 = fma(yf[r], cs[r * kRT + tid], d2);
          d3 = fma(yf[r + 1], cs[(r + 1) * kRT + tid], d3);
        }
        if (r < RS) d2 = fma(yf[r], cs[r * kRT + tid], d2);
      }
#pragma unroll
      for (int q = 0; q < kRR; q += 2) {
        const double2 yv = lds2(yf + RS + q);
        d0 = fma(yv.x, xr[q], d0);
        d1 = fma(yv.y, xr[q + 1], d1);
      }
      wvv = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
      for (int q = 0; q < kRR; q += 2) {
        const double2 yv = lds2(yf + RS + q);
        xr[q] = fma(-yv.x, wvv, xr[q]);
        xr[q + 1] = fma(-yv.y, wvv, xr[q + 1]);
      }
      double rj;
      if (j < RS) {
        rj = fma(-yf[j], wvv, cs[j * kRT + tid]);
      } else {
        rj = 0.0;
#pragma unroll
        for (int q = 0; q < kRR; ++q)
          if (RS + q == j) rj = xr[q];
      }
      double ns = nsq - rj * rj;
      if (ns < kNormGuard * rsq) {
        double e0 = 0.0, e1 = 0.0;
        for (int r = j + 1; r < RS; ++r) {
          const double v = fma(-yf[r], wvv, cs[r * kRT + tid]);
          e0 = fma(v, v, e0);
        }
#pragma unroll
        for (int q = 0; q < kRR; ++q)
          if (RS + q > j) e1 = fma(xr[q], xr[q], e1);
        ns = e0 + e1;
        rsq = ns;
      } else {
        ns = fmax(ns, 0.0);
      }
      nsq = ns;
      cbv = ns;
      cbp = pn;
      cbl = tid;
    }
    wcol[tid] = wvv;  // 0 for the pivot and for finished / absent columns
    achieved = j + 1;
    SQR_TRACE(a.trace, 8 * j + 1);
    if (j + 1 < a.bb) {
      publish(j + 1);
      SQR_TRACE(a.trace, 8 * j + 2);
      if (CL) {
        __syncthreads();  // publish read the candidate's shared-memory rows
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      } else {
        gb.arrive();
      }
      SQR_TRACE(a.trace, 8 * j + 3);
      if (warp == 0) {
        if (CL)
          asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        else if (lane == 0)
          gb.wait_lane0();
        if (lane == 0) SQR_TRACE(a.trace, 8 * j + 6);
        __syncwarp();
        winner(j + 1);
        if (a.trace && g == 0 && tid == 0) a.trace[8 * j + 7] = gtimer();  // winner + reflector done
      } else {
        smem_update(j, 32);
        if (a.trace && g == 0 && tid == 32) a.trace[8 * j + 5] = gtimer();  // deferred update done
        if (CL) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
      }
      __syncthreads();
      SQR_TRACE(a.trace, 8 * j + 4);
    } else {
      __syncthreads();
      smem_update(j, 0);
      __syncthreads();
    }
  }
  __syncthreads();
  if (CL) cg::this_cluster().sync();  // no CTA leaves while a peer may read its records
  if (pj >= 0) {
    // pivot of step pj -> Bf column pj, exactly as the winner built it
    // (y_r = u_r / y0 with y0 = u_pj - beta; y = 0 for a zero column)
    double* bfj = a.Bf + (int64_t)pj * a.ldbf;
    const double u0 = pj < RS ? cs[pj * kRT + tid] : [&] {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kRR; ++q)
        if (RS + q == pj) v = xr[q];
      return v;
    }();
    const double y0 = u0 - pbeta;
    for (int r = 0; r < RS; ++r) {
      const double u = cs[r * kRT + tid];
      bfj[r] = r < pj ? u : (r == pj ? pbeta : (pbeta != 0.0 ? u / y0 : 0.0));
    }
#pragma unroll
    for (int q = 0; q < kRR; ++q) {
      const int r = RS + q;
      if (r < ell) bfj[r] = r < pj ? xr[q] : (r == pj ? pbeta : (pbeta != 0.0 ? xr[q] / y0 : 0.0));
    }
    a.lperm[pj] = col;
    if (col != pj) {
      a.moves[2 * pj] = pj;
      a.moves[2 * pj + 1] = col;
    }
    if (disp >= 0) a.moves[2 * (a.bb + disp)] = -1;  // superseded displacement
  }
  // remaining columns go to their final positions
  if (pos >= 0) {
    double* dst = a.Bf + (int64_t)pos * a.ldbf;
    for (int r = 0; r < RS; ++r) dst[r] = cs[r * kRT + tid];
#pragma unroll
    for (int q = 0; q < kRR; ++q)
      if (RS + q < ell) dst[RS + q] = xr[q];
    a.lperm[pos] = col;
    if (disp >= 0 && pos != col) {
      a.moves[2 * (a.bb + disp)] = pos;
      a.moves[2 * (a.bb + disp) + 1] = col;
    } else if (disp >= 0) {
      a.moves[2 * (a.bb + disp)] = -1;
    }
  }
  if (g == 0 && tid == 0) {
    a.st->sample_achieved = achieved;
    if (achieved == 0) {
      a.st->stop = 1;
      a.st->reason = SQR_STOP_SAMPLE_RANK;
    }
  }
}

}  // namespace

int64_t sample_epoch_workspace(int64_t ell, int64_t nt, int64_t bb);
bool sample_epoch_eligible(int64_t ell, int64_t nt);
int sample_epoch(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf, int64_t ldbf,
                 int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st, void* ws,
                 int64_t ws_bytes, cudaStream_t s);

struct SampleWorkspace {
  static int64_t bytes(int64_t ell, int64_t nt) {
    const int64_t G = 148;
    return std::max<int64_t>(64 + 2 * G * 16 + 2 * G * ell * 8 + 2 * G * 8 + nt * ell * 8 + 1024,
                             sample_epoch_workspace(ell, nt, ell));
  }
};

// Largest cluster the register sample kernel can be launched with (16 with
// the non-portable opt-in where the GPCs allow it, else 8), probed once.
int cluster_max_probe();
int cluster_max() {
  // per device, probed once under a process-wide lock
  static std::mutex mu;
  static std::map<int, int> probed;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = probed.find(dev);
  if (it != probed.end()) return it->second;
  const int c = cluster_max_probe();
  probed[dev] = c;
  return c;
}

int cluster_max_probe() {
  int cmax = 0;
  const int smem = (int)(((int64_t)(144 - kRR) * kRT + 2 * 152 + 2 + kRT) * 8);
  if (cudaFuncSetAttribute(sample_qrcp_reg_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return cmax;
  }
  cudaFuncSetAttribute(sample_qrcp_reg_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  for (int c : {16, 8}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kRT);
    cfg.dynamicSmemBytes = (size_t)smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, sample_qrcp_reg_kernel<true>, &cfg) == cudaSuccess && n > 0) {
      cmax = c;
      break;
    }
    cudaGetLastError();
  }
  return cmax;
}

int64_t sample_qrcp_workspace(int64_t ell, int64_t nt) { return SampleWorkspace::bytes(ell, nt); }

int sample_qrcp(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st,
                void* ws, int64_t ws_bytes, cudaStream_t s, ResidentSig sig) {
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
  static const bool no_reg = env_flag("SQR_NO_REGSAMPLE");
  const bool reg_path = !sample_epoch_eligible(ell, nt) && !no_reg && ell <= 144 &&
                        nt <= (int64_t)std::min(sms, 148) * kRT;
  // kernels without the in-kernel signal: release the waiter up front
  if (sig.flag != nullptr && !reg_path)
    if (int rc = signal_resident_host(sig, s)) return rc;
  if (sample_epoch_eligible(ell, nt))
    return sample_epoch(B, ldb, ell, nt, bb, Bf, ldbf, lperm, moves, taus, first, st, ws, ws_bytes, s);
  if (reg_path) {
    RegArgs a{};
    a.sig = sig;
    a.B = B;
    a.ldb = ldb;
    a.ell = (int)ell;
    a.nt = (int)nt;
    a.bb = (int)bb;
    a.first = first;
    a.RS = (int)std::max<int64_t>(0, ell - kRR);
    a.Bf = Bf;
    a.ldbf = ldbf;
    a.lperm = lperm;
    a.moves = moves;
    a.taus = taus;
    a.st = st;
    char* p = static_cast<char*>(ws);
    a.bar = reinterpret_cast<unsigned*>(p);
    p += 64;
    a.cand = reinterpret_cast<double2*>(p);
    p += 2 * 148 * 16;
    a.ccol = reinterpret_cast<double*>(p);
    p += 2 * 148 * ell * 8;
    a.psum = reinterpret_cast<double*>(p);
    p += 148 * 8;
    a.pmax = reinterpret_cast<double*>(p);
    a.trace = g_trace_host_ptr;
    const int G = (int)std::max<int64_t>(1, cdiv(nt, (int64_t)kRT));
    const int YP = (int)(((std::max<int64_t>(ell, a.RS + kRR) + 1) | 1) + 1);
    const int smem = (int)(((int64_t)a.RS * kRT + 2 * YP + 2 + kRT) * 8);
    if (int rc = smem_optin((const void*)sample_qrcp_reg_kernel<false>, smem)) return rc;
    // One cluster when the sample fits 16 CTAs (the hardware cluster
    // barrier and DSMEM exchange; measured per-step cost in DESIGN.md).
    static const bool no_cl = env_flag("SQR_NO_CLUSTER_SAMPLE");
    if (!no_cl && G <= cluster_max() && ell <= kMaxEllCl) {
      if (int rc = smem_optin((const void*)sample_qrcp_reg_kernel<true>, smem)) return rc;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(kRT);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = G;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      ProfScope ps(kTagSample, s);
      count_launch();
      SQR_CUDA(cudaLaunchKernelEx(&cfg, sample_qrcp_reg_kernel<true>, a));
      return SQR_OK;
    }
    void* args[] = {&a};
    SQR_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
    ProfScope ps(kTagSample, s);
    count_launch();
    SQR_CUDA(cudaLaunchCooperativeKernel((const void*)sample_qrcp_reg_kernel<false>, dim3(G), dim3(kRT), args,
                                         (size_t)smem, s));
    return SQR_OK;
  }
  // At least 32 columns per CTA (amortise the per-step barrier), enough CTAs
  // to keep every column in shared memory when possible, one CTA per SM.
  const int ldS = (int)(ell | 1);
  const int64_t fixed_per_col = 24 + 4;
  const int64_t smem_avail = (int64_t)max_smem_optin() - 2048 - 2 * (ell + 2) * 8 - 64;
  const int64_t fit = std::max<int64_t>(1, smem_avail / ((int64_t)ldS * 8 + fixed_per_col));
  const int64_t ntc = std::max<int64_t>(nt, 1);
  int G = (int)std::min<int64_t>(std::min(sms, 148), std::max<int64_t>(cdiv(ntc, 32), cdiv(ntc, fit)));
  G = std::max(G, 1);
  const int w = (int)cdiv(ntc, G);
  G = (int)cdiv(ntc, w);
  const int64_t fixed = (int64_t)w * 24 + 2 * (ell + 2) * 8 + (int64_t)w * 4 + 64;
  const int64_t budget = (int64_t)max_smem_optin() - 2048 - fixed;
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
  a.reg_spill = a.warp_spill && (w - cap) <= 8 * kSpillPerWarp;
  a.Bf = Bf;
  a.ldbf = ldbf;
  a.lperm = lperm;
  a.moves = moves;
  a.taus = taus;
  a.st = st;
  a.bar = reinterpret_cast<unsigned*>(p);
  p += 64;
  a.cand = reinterpret_cast<double2*>(p);
  p += 2 * 148 * 16;
  a.ccol = reinterpret_cast<double*>(p);
  p += 2 * 148 * ell * 8;
  a.psum = reinterpret_cast<double*>(p);
  p += 148 * 8;
  a.pmax = reinterpret_cast<double*>(p);
  p += 148 * 8;
  a.spill = reinterpret_cast<double*>(p);
  a.trace = g_trace_host_ptr;

  if (int rc = smem_optin((const void*)sample_qrcp_kernel, (int)smem)) return rc;
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

extern "C" int64_t sqr_sample_qrcp_workspace(int64_t ell, int64_t nt) { return sqr::sample_qrcp_workspace(ell, nt); }

extern "C" int sqr_sample_qrcp_ws(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                                  int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first,
                                  sqr_status* st, void* workspace, int64_t workspace_bytes, void* stream) {
  return sqr::sample_qrcp(B, ldb, ell, nt, bb, Bf, ldbf, lperm, moves, taus, first, st, workspace, workspace_bytes,
                          static_cast<cudaStream_t>(stream));
}

// The same with a residency signal: *resident_flag = resident_val once every
// CTA of the sample QRCP is on the chip, so a caller can hold a GEMM on
// another stream (sqr_wait_resident) until the whole-SM kernel has taken its
// SMs and run the GEMM beside it (driver.cu Overlap; the multi-GPU driver's
// deferred second-sweep rows).
extern "C" int sqr_sample_qrcp_ws_sig(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                                      int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first,
                                      sqr_status* st, void* workspace, int64_t workspace_bytes,
                                      uint32_t* resident_flag, uint32_t resident_val, void* stream) {
  return sqr::sample_qrcp(B, ldb, ell, nt, bb, Bf, ldbf, lperm, moves, taus, first, st, workspace, workspace_bytes,
                          static_cast<cudaStream_t>(stream), sqr::ResidentSig{resident_flag, resident_val});
}

extern "C" int sqr_wait_resident(uint32_t* resident_flag, uint32_t resident_val, int timeout_us, void* stream) {
  return sqr::wait_resident(sqr::ResidentSig{resident_flag, resident_val}, timeout_us,
                            static_cast<cudaStream_t>(stream));
}
