// K4/K5: unpivoted Householder QR of a tall panel (randomized.py:107-130 for
// the randomized drivers, reference.py:281-291 for qr_blocked) on one
// persistent cooperative kernel, plus the compact-WY T factor
// (householder.py:52-61).
//
// The mr x w panel is split by rows over G CTAs; each CTA keeps its row slab
// of the current sub-panel (<= sw columns) in shared memory.  A column step
// needs ONE grid-wide reduction: every CTA publishes, over its rows below the
// pivot row, [sum a_r^2, sum a_r P_rc for the remaining sub-panel columns];
// after the barrier every CTA sums the partials in the same fixed order and
// rebuilds the identical reflector:
//     nrm = sqrt(a_t^2 + s_a), beta = -sign(a_t) nrm, y0 = a_t - beta,
//     y_r = a_r / y0, tau = 2 / (1 + s_a / y0^2),
//     w_c = tau (P_tc + s_c / y0),   P_rc -= y_r w_c
// (house_gen, householder.py:44-48, with y^T P expanded so one reduction
// suffices).  Between sub-panels the finished sub-panel's reflectors are
// applied to the rest of the panel in compact-WY form with one fixed-order
// two-phase reduction of [Y_s^T Y_s | Y_s^T P_rest].  An exactly zero column
// stops the panel (randomized.py:120-121) after the remaining panel columns
// have received every earlier reflector, as in the reference loop.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kMaxG = 152;  // >= SM count, multiple of 8
constexpr int kRowsPerLane = 8;             // row chunk = 256 rows
constexpr int kColsPerWarp = 128 / kPWarps;  // sub-panel width <= 128

struct PanelArgs {
  double* P;
  int64_t ldp;
  int mr;      // panel rows
  int wstat;   // panel width (<0: st->sample_achieved)
  int wmax;    // columns of Y / taus to define (zero beyond bhat)
  int sw, h, hp, stop_at_zero;
  double* Y;
  int64_t ldy;
  double* taus;
  sqr_status* st;
  unsigned* bar;
  double* part;   // [2][sw+1][G]   per-step partials (value-major)
  double* rowt;   // [2][sw+1]      pivot-row values
  double* wpart;  // [G][sw*wmax]   WY partials
  double* wred;   // [sw*wmax]      WY reduced
  unsigned long long* trace;
  int c0;         // leaf offset: this launch factors panel columns [c0, c0 + wmax), rows [c0, mr)
};

__global__ void __launch_bounds__(kPThreads, 1) panel_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double vals[136];
  __shared__ double rowv[136];
  __shared__ double wv[136];
  if (a.st->stop) return;
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // Leaf view: columns [c0, c0 + wmax) of the panel, rows [c0, mr).
  const int lc0 = a.c0;
  const int wglob = a.wstat < 0 ? a.st->sample_achieved : a.wstat;
  const bool prior_stop = lc0 > 0 && a.st->bhat < lc0;  // an earlier leaf hit a zero column
  const int w = prior_stop ? 0 : max(0, min(wglob - lc0, a.wmax));
  if (lc0 > 0) {
    if (g == 0)  // explicit Y is zero above the leaf's first row
      for (int e = tid; e < lc0 * a.wmax; e += kPThreads)
        a.Y[(int64_t)(lc0 + e / lc0) * a.ldy + (e % lc0)] = 0.0;
    a.P += lc0 + (int64_t)lc0 * a.ldp;
    a.Y += lc0 + (int64_t)lc0 * a.ldy;
    a.taus += lc0;
    a.mr -= lc0;
  }
  const int row0 = g * a.h;
  const int nrows = max(0, min(a.h, a.mr - row0));
  GridBarrier gb;
  gb.init(a.bar);
  double* slab = sm;                              // sw x hp
  double* Ts = slab + (size_t)a.sw * a.hp;        // sw x sw
  double* GS = Ts + (size_t)a.sw * a.sw;          // swe x (swe + rest)
  int bhat = w;
  bool stopped = false;
  int written = 0;  // Y columns [0, written) defined on my rows

  for (int c0 = 0; c0 < w; c0 += a.sw) {
    const int c1 = min(w, c0 + a.sw);
    const int swe = c1 - c0;
    for (int c = 0; c < swe; ++c)
      for (int r = tid; r < nrows; r += kPThreads)
        slab[c * a.hp + r] = a.P[(int64_t)(c0 + c) * a.ldp + row0 + r];
    __syncthreads();

    // Partial sums of step tcur over my rows > tcur, for the columns
    // tcur..c1-1 (value v <-> column tcur + v; v = 0 gives |a|^2), fused with
    // the rank-1 update of the previous step (y in slab column tcur-1, w in
    // wv[1 + v]) when upd.  Lanes own rows (stride-1 shared-memory access for
    // any pitch); warp q owns columns v = q, q+8, ...; each warp reduces its
    // columns with shuffles, so no cross-warp pass is needed.
    auto fused = [&](int tcur, bool upd) {
      const int tl = tcur - c0;
      const int Lc = c1 - tcur;
      const int par = (tcur - c0) & 1;
      const double* yprev = slab + (tl - 1) * a.hp;
      const double* acol = slab + tl * a.hp;
      const double wa = upd ? wv[1] : 0.0;
      const int rsum = tcur + 1 - row0;   // summed rows: local index >= rsum
      const int rupd = tcur - row0;       // updated rows: local index >= rupd
      double acc[kColsPerWarp];
#pragma unroll
      for (int k = 0; k < kColsPerWarp; ++k) acc[k] = 0.0;
      for (int rc = 0; rc < nrows; rc += 32 * kRowsPerLane) {
        double yv[kRowsPerLane], av[kRowsPerLane];
#pragma unroll
        for (int i = 0; i < kRowsPerLane; ++i) {
          const int r = rc + lane + 32 * i;
          const bool in = r < nrows;
          const double yr = (upd && in && r >= rupd) ? yprev[r] : 0.0;
          yv[i] = yr;
          av[i] = (in && r >= rsum) ? fma(-yr, wa, acol[r]) : 0.0;  // 0 => excluded from sums
        }
#pragma unroll
        for (int k = 0; k < kColsPerWarp; ++k) {
          const int v = warp + kPWarps * k;
          if (v < Lc) {
            double* pc = slab + (tl + v) * a.hp;
            const double wc = upd ? wv[1 + v] : 0.0;
#pragma unroll
            for (int i = 0; i < kRowsPerLane; ++i) {
              const int r = rc + lane + 32 * i;
              if (r < nrows) {
                double pv = pc[r];
                if (upd && r >= rupd) {
                  pv = fma(-yv[i], wc, pv);
                  pc[r] = pv;
                }
                acc[k] = fma(av[i], pv, acc[k]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kColsPerWarp; ++k) acc[k] = warp_sum(acc[k]);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kColsPerWarp; ++k) {
          const int v = warp + kPWarps * k;
          if (v < Lc) a.part[((size_t)par * (a.sw + 1) + v) * G + g] = acc[k];
        }
      }
      __syncthreads();
      // the owner of row tcur publishes it (already updated above)
      if (tcur >= row0 && tcur < row0 + nrows) {
        for (int v = tid; v < Lc; v += kPThreads)
          a.rowt[par * (a.sw + 1) + v] = slab[(tl + v) * a.hp + (tcur - row0)];
      }
    };

    fused(c0, false);
    for (int t = c0; t < c1; ++t) {
      const int tl = t - c0;
      const int L = c1 - t;
      const int par = (t - c0) & 1;
      SQR_TRACE(a.trace, 8 * t + 1);
      gb.sync();
      SQR_TRACE(a.trace, 8 * t + 2);
      // Fixed-order reduction of the G partials of every value: 4 lanes per
      // value, each summing G/4 partials whose loads are all in flight at
      // once; the pivot-row values are fetched in the same round.
      for (int v = tid; v < L; v += kPThreads) rowv[v] = __ldcg(a.rowt + par * (a.sw + 1) + v);
      for (int v0 = 0; v0 < L; v0 += kPThreads / 4) {
        const int v = v0 + (tid >> 2), q = tid & 3;
        double x[kMaxG / 4];
        const double* src = a.part + ((size_t)par * (a.sw + 1) + v) * G;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) {
          const int gi = q + 4 * i;
          x[i] = (v < L && gi < G) ? __ldcg(src + gi) : 0.0;
        }
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < kMaxG / 4; ++i) sacc += x[i];
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
        if (v < L && q == 0) vals[v] = sacc;
      }
      __syncthreads();
      SQR_TRACE(a.trace, 8 * t + 3);
      const double at = rowv[0], sa = vals[0];
      const double nrm = sqrt(fma(at, at, sa));
      if (nrm == 0.0 && a.stop_at_zero) {
        bhat = t;
        stopped = true;
        break;
      }
      double beta = 0.0, tau = 0.0, y0 = 1.0;
      if (nrm != 0.0) {
        beta = (at >= 0.0 ? -1.0 : 1.0) * nrm;
        y0 = at - beta;
        tau = 2.0 / (1.0 + sa / (y0 * y0));
      }
      for (int v = 1 + tid; v < L; v += kPThreads) wv[v] = tau * (rowv[v] + vals[v] / y0);
      if (g == 0 && tid == 0) a.taus[t] = tau;
      // y for my rows below t; row t keeps beta and its R entries.
      const int rbeg = max(0, t + 1 - row0);
      for (int r = rbeg + tid; r < nrows; r += kPThreads) {
        const double yr = nrm != 0.0 ? slab[tl * a.hp + r] / y0 : 0.0;
        slab[tl * a.hp + r] = yr;
      }
      __syncthreads();
      if (t >= row0 && t < row0 + nrows) {
        const int rt = t - row0;
        for (int v = 1 + tid; v < L; v += kPThreads) slab[(tl + v) * a.hp + rt] -= wv[v];
        if (tid == 0) slab[tl * a.hp + rt] = beta;
      }
      SQR_TRACE(a.trace, 8 * t + 4);
      if (t + 1 < c1) {
        fused(t + 1, true);
      } else if (c1 < w) {
        // last step of a sub-panel that is followed by others: nothing left
        // to update inside the sub-panel.
      }
      __syncthreads();
      SQR_TRACE(a.trace, 8 * t + 5);
    }
    __syncthreads();
    // Write the sub-panel back (packed R / reflector tails) and explicit Y.
    for (int c = 0; c < swe; ++c) {
      const int gc = c0 + c;
      for (int r = tid; r < nrows; r += kPThreads) {
        const int R = row0 + r;
        const double v = slab[c * a.hp + r];
        a.P[(int64_t)gc * a.ldp + R] = v;
        double y = 0.0;
        if (gc < bhat) y = R > gc ? v : (R == gc ? 1.0 : 0.0);
        a.Y[(int64_t)gc * a.ldy + R] = y;
      }
    }
    written = c1;
    if (c1 >= w) break;
    // ---- compact-WY update of panel columns [c1, w) with this sub-panel.
    const int rest = w - c1;
    const int ncoef = swe * (swe + rest);
    for (int e = tid; e < ncoef; e += kPThreads) {
      const int ai = e % swe, cj = e / swe;
      const int gca = c0 + ai;
      double s = 0.0;
      if (gca < bhat) {
        if (cj < swe) {
          const int gcb = c0 + cj;
          if (gcb < bhat) {
            for (int r = max(0, max(gca, gcb) - row0); r < nrows; ++r) {
              const int R = row0 + r;
              const double ya = R > gca ? slab[ai * a.hp + r] : 1.0;
              const double yb = R > gcb ? slab[cj * a.hp + r] : 1.0;
              s = fma(ya, yb, s);
            }
          }
        } else {
          const double* pcol = a.P + (int64_t)(c1 + cj - swe) * a.ldp + row0;
          for (int r = max(0, gca - row0); r < nrows; ++r) {
            const int R = row0 + r;
            const double ya = R > gca ? slab[ai * a.hp + r] : 1.0;
            s = fma(ya, pcol[r], s);
          }
        }
      }
      a.wpart[(size_t)g * ncoef + e] = s;
    }
    gb.sync();
    {
      const int per = (int)cdiv(ncoef, G);
      for (int e = g * per + tid; e < min(ncoef, (g + 1) * per); e += kPThreads) {
        double s = 0.0;
        int i = 0;
        for (; i + 8 <= G; i += 8) {  // 8 loads in flight, summed in index order
          double x[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) x[q] = __ldcg(a.wpart + (size_t)(i + q) * ncoef + e);
#pragma unroll
          for (int q = 0; q < 8; ++q) s += x[q];
        }
        for (; i < G; ++i) s += __ldcg(a.wpart + (size_t)i * ncoef + e);
        a.wred[e] = s;
      }
    }
    gb.sync();
    for (int e = tid; e < ncoef; e += kPThreads) GS[e] = __ldcg(a.wred + e);
    for (int e = tid; e < a.sw * a.sw; e += kPThreads) Ts[e] = 0.0;
    __syncthreads();
    // T_s recurrence (householder.py:56-60): T[i,c] = -tau_c sum_{l=i}^{c-1} T[i,l] G[l,c].
    for (int c = 0; c < swe; ++c) {
      const double tc = (c0 + c < bhat) ? __ldcg(a.taus + c0 + c) : 0.0;
      for (int i = warp; i < c; i += kPWarps) {
        double s = 0.0;
        for (int l = i + lane; l < c; l += 32) s = fma(Ts[l * a.sw + i], GS[c * swe + l], s);
        s = warp_sum(s);
        if (lane == 0) Ts[c * a.sw + i] = -tc * s;
      }
      if (tid == 0) Ts[c * a.sw + c] = tc;
      __syncthreads();
    }
    // W = T^T S in place over S, one column at a time.
    for (int j = 0; j < rest; ++j) {
      double* Sj = GS + (size_t)(swe + j) * swe;
      double acc = 0.0;
      if (tid < swe)
        for (int l = 0; l <= tid; ++l) acc = fma(Ts[tid * a.sw + l], Sj[l], acc);
      __syncthreads();
      if (tid < swe) Sj[tid] = acc;
    }
    __syncthreads();
    // P_rest -= Y_s W on my rows.
    for (int j = 0; j < rest; ++j) {
      const double* Wj = GS + (size_t)(swe + j) * swe;
      double* pcol = a.P + (int64_t)(c1 + j) * a.ldp + row0;
      for (int r = tid; r < nrows; r += kPThreads) {
        const int R = row0 + r;
        if (R < c0) continue;
        double s = 0.0;
        const int amax = min(swe, min(bhat - c0, R - c0 + 1));
        for (int ai = 0; ai < amax; ++ai) {
          const double ya = (R > c0 + ai) ? slab[ai * a.hp + r] : 1.0;
          s = fma(ya, Wj[ai], s);
        }
        pcol[r] -= s;
      }
    }
    __syncthreads();
    if (stopped) break;
  }
  // Undefined Y columns (never reached, or beyond the dynamic width) are zero.
  for (int c = written; c < a.wmax; ++c)
    for (int r = tid; r < nrows; r += kPThreads) a.Y[(int64_t)c * a.ldy + row0 + r] = 0.0;
  if (g == 0 && tid == 0) {
    for (int c = bhat; c < a.wmax; ++c) a.taus[c] = 0.0;
    if (!prior_stop) {
      a.st->bhat = lc0 + bhat;
      if (lc0 == 0 && bhat == 0 && a.stop_at_zero) {
        a.st->stop = 1;
        a.st->reason = SQR_STOP_PANEL_ZERO;
      }
    }
  }
}

// Leaf kernel (w <= 32 columns): the same column step as panel_kernel with
// the CTA's rows held in REGISTERS, one row (RPT rows) per thread, all 32
// columns.  The step loop is fully unrolled so every column index is static;
// the per-step partials [sum a_r^2, sum a_r P_rc] are reduced inside a warp
// by a transpose butterfly (31 shuffles for 32 values, lane v ends with
// value v), across warps through shared memory, and across CTAs by the same
// fixed-order read of the G partials as panel_kernel.  Deterministic.
constexpr int kLThreads = 256;
constexpr int kLWarps = kLThreads / 32;
constexpr int kLW = 32;

// LW = leaf width (32, or 16 for very tall panels where RPT = 3..4 rows per
// thread must fit the register file).
template <int RPT, int LW>
__global__ void __launch_bounds__(kLThreads, 1) leaf_kernel(PanelArgs a) {
  __shared__ double red[kLWarps][LW];
  __shared__ double vals[LW];
  __shared__ double rowv[LW];
  __shared__ double wv[LW];
  if (a.st->stop) return;
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int lc0 = a.c0;
  const int wglob = a.wstat < 0 ? a.st->sample_achieved : a.wstat;
  const bool prior_stop = lc0 > 0 && a.st->bhat < lc0;  // an earlier leaf hit a zero column
  const int w = prior_stop ? 0 : max(0, min(wglob - lc0, a.wmax));
  if (lc0 > 0) {
    if (g == 0)  // explicit Y is zero above the leaf's first row
      for (int e = tid; e < lc0 * a.wmax; e += kLThreads)
        a.Y[(int64_t)(lc0 + e / lc0) * a.ldy + (e % lc0)] = 0.0;
    a.P += lc0 + (int64_t)lc0 * a.ldp;
    a.Y += lc0 + (int64_t)lc0 * a.ldy;
    a.taus += lc0;
    a.mr -= lc0;
  }
  SQR_TRACE(a.trace, 8 * 40 + 0);
  GridBarrier gb;
  gb.init(a.bar);
  int rows[RPT];
  double x[RPT][LW];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    rows[i] = g * kLThreads * RPT + i * kLThreads + tid;
#pragma unroll
    for (int c = 0; c < LW; ++c)
      x[i][c] = (rows[i] < a.mr && c < w) ? a.P[(int64_t)c * a.ldp + rows[i]] : 0.0;
  }
  int bhat = w;
  SQR_TRACE(a.trace, 8 * 40 + 1);
#pragma unroll
  for (int t = 0; t < LW; ++t) {
    if (t >= w) break;
    const int par = t & 1;
    // ---- partials of step t over my rows > t: q[0] = |a|^2, q[v] = a . P_{t+v}
    double q[LW];
#pragma unroll
    for (int v = 0; v < LW; ++v) q[v] = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const bool in = rows[i] > t;
      const double av = in ? x[i][t] : 0.0;
#pragma unroll
      for (int v = 0; v < LW - t; ++v) q[v] = fma(av, x[i][t + v], q[v]);
    }
    // ---- warp transpose butterfly: lane l ends with the warp sum of value
    // l mod LW (for LW = 16 the two 16-lane halves are added at the end)
#pragma unroll
    for (int k = LW / 2; k >= 1; k >>= 1) {
      const bool upper = (lane & k) != 0;
#pragma unroll
      for (int i = 0; i < k; ++i) {
        const double send = upper ? q[i] : q[i + k];
        const double keep = upper ? q[i + k] : q[i];
        q[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
      }
    }
    if (LW < 32) q[0] += __shfl_xor_sync(0xffffffffu, q[0], 16);
    if (lane < LW) red[warp][lane] = q[0];
    __syncthreads();
    if (tid < LW - t) {
      double s = 0.0;
#pragma unroll
      for (int wi = 0; wi < kLWarps; ++wi) s += red[wi][tid];
      a.part[((size_t)par * (LW + 1) + tid) * G + g] = s;
    }
    // the owner of row t (CTA 0, thread t) publishes it
    if (g == 0 && tid == t) {
#pragma unroll
      for (int v = 0; v < LW - t; ++v) a.rowt[par * (LW + 1) + v] = x[0][t + v];
    }
    SQR_TRACE(a.trace, 8 * t + 1);
    gb.sync();
    SQR_TRACE(a.trace, 8 * t + 2);
    {
      const int L = min(LW - t, w - t);
      if (tid < L) rowv[tid] = __ldcg(a.rowt + par * (LW + 1) + tid);
      // 8 lanes per value (32 values x 8 = 256 threads), G/8 loads each in flight
      const int v = tid >> 3, qd = tid & 7;
      if (v < L) {
        double xr[kMaxG / 8];
        const double* src = a.part + ((size_t)par * (LW + 1) + v) * G;
#pragma unroll
        for (int i = 0; i < kMaxG / 8; ++i) {
          const int gi = qd + 8 * i;
          xr[i] = gi < G ? __ldcg(src + gi) : 0.0;
        }
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < kMaxG / 8; ++i) sacc += xr[i];
        const unsigned gm = 0xffu << (lane & 24);  // this value's 8-lane group
        sacc += __shfl_xor_sync(gm, sacc, 4);
        sacc += __shfl_xor_sync(gm, sacc, 2);
        sacc += __shfl_xor_sync(gm, sacc, 1);
        if (qd == 0) vals[v] = sacc;
      }
    }
    __syncthreads();
    SQR_TRACE(a.trace, 8 * t + 3);
    const double at = rowv[0], sa = vals[0];
    const double nrm = sqrt(fma(at, at, sa));
    if (nrm == 0.0 && a.stop_at_zero) {
      bhat = t;
      break;
    }
    double beta = 0.0, tau = 0.0, y0 = 1.0, ry = 1.0;
    if (nrm != 0.0) {
      beta = (at >= 0.0 ? -1.0 : 1.0) * nrm;
      y0 = at - beta;
      ry = __drcp_rn(y0);
      tau = 2.0 / (1.0 + sa / (y0 * y0));
    }
    if (tid >= 1 && tid < min(LW - t, w - t)) wv[tid] = tau * (rowv[tid] + div_rn(vals[tid], y0, ry));
    if (g == 0 && tid == 0) a.taus[t] = tau;
    __syncthreads();
    // ---- apply reflector t to my rows (row t keeps beta and its R entries)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (rows[i] > t) {
        const double yr = nrm != 0.0 ? div_rn(x[i][t], y0, ry) : 0.0;
        x[i][t] = yr;
#pragma unroll
        for (int v = 1; v < LW - t; ++v) x[i][t + v] = fma(-yr, wv[v], x[i][t + v]);
      } else if (rows[i] == t) {
        x[i][t] = beta;
#pragma unroll
        for (int v = 1; v < LW - t; ++v) x[i][t + v] -= wv[v];
      }
    }
    SQR_TRACE(a.trace, 8 * t + 4);
  }
  // ---- write back: packed R / reflector tails into P, explicit Y
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int R = rows[i];
    if (R >= a.mr) continue;
#pragma unroll
    for (int c = 0; c < LW; ++c) {
      if (c < w) a.P[(int64_t)c * a.ldp + R] = x[i][c];
      if (c < a.wmax) {
        const double y = c < bhat ? (R > c ? x[i][c] : (R == c ? 1.0 : 0.0)) : 0.0;
        a.Y[(int64_t)c * a.ldy + R] = y;
      }
    }
  }
  SQR_TRACE(a.trace, 8 * 40 + 2);
  if (g == 0 && tid == 0) {
    for (int c = bhat; c < a.wmax; ++c) a.taus[c] = 0.0;
    if (!prior_stop) {
      a.st->bhat = lc0 + bhat;
      if (lc0 == 0 && bhat == 0 && a.stop_at_zero) {
        a.st->stop = 1;
        a.st->reason = SQR_STOP_PANEL_ZERO;
      }
    }
  }
}

}  // namespace

int64_t panel_workspace(int64_t w) {
  const int64_t G = 148, sw = 128;
  return std::max<int64_t>(panel_block_workspace(),
                           64 + 2 * G * (sw + 1) * 8 + 2 * (sw + 1) * 8 + G * sw * std::max<int64_t>(w, 1) * 8 +
                               sw * std::max<int64_t>(w, 1) * 8 + 4096);
}

// Rows per CTA >= 64 and at most one CTA per SM; the largest sub-panel width
// whose slab + WY scratch fits in shared memory.
int panel_qr(double* P, int64_t ldp, int64_t mr, int64_t w, int64_t wmax, double* Y, int64_t ldy,
             double* taus, int stop_at_zero, sqr_status* st, void* ws, int64_t ws_bytes,
             cudaStream_t s, int64_t c0) {
  if (mr - c0 <= 0 || wmax <= 0) return SQR_OK;
  if (wmax > 128) {
    set_error("panel_qr: width %lld > 128", (long long)wmax);
    return SQR_EINVAL;
  }
  if (ws_bytes < panel_workspace(wmax)) {
    set_error("panel_qr: workspace too small");
    return SQR_EINVAL;
  }
  const int sms = sm_count();
  const int64_t mrl0 = mr - c0;
  const int64_t rows1 = (int64_t)std::min(sms, 148) * kLThreads;  // one row per thread
  const bool narrow = wmax <= 16 && mrl0 > 2 * rows1 && mrl0 <= 4 * rows1;  // 16-wide leaves, 3-4 rows
  if ((narrow || (wmax <= kLW && mrl0 <= 2 * rows1)) && !env_flag("SQR_NO_LEAF")) {
    // register-resident leaf kernel: one to four rows per thread
    const int rpt = (int)cdiv(mrl0, rows1);
    const int G = (int)cdiv(mrl0, (int64_t)kLThreads * rpt);
    PanelArgs a{};
    a.P = P;
    a.ldp = ldp;
    a.mr = (int)mr;
    a.c0 = (int)c0;
    a.wstat = (int)w;
    a.wmax = (int)wmax;
    a.stop_at_zero = stop_at_zero;
    a.Y = Y;
    a.ldy = ldy;
    a.taus = taus;
    a.st = st;
    char* p = static_cast<char*>(ws);
    a.bar = reinterpret_cast<unsigned*>(p);
    p += 64;
    a.part = reinterpret_cast<double*>(p);
    p += 2 * 148 * (128 + 1) * 8;
    a.rowt = reinterpret_cast<double*>(p);
    a.trace = g_trace_host_ptr;
    void* args[] = {&a};
    SQR_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
    ProfScope ps(kTagPanel, s);
    count_launch();
    const void* fn = rpt == 1   ? (const void*)leaf_kernel<1, 32>
                     : rpt == 2 ? (const void*)leaf_kernel<2, 32>
                     : rpt == 3 ? (const void*)leaf_kernel<3, 16>
                                : (const void*)leaf_kernel<4, 16>;
    SQR_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kLThreads), args, 0, s));
    return SQR_OK;
  }
  const int64_t budget0 = (int64_t)max_smem_optin() - 4 * 1024;  // static smem of the kernel
  // Fewest CTAs whose row slabs still hold the whole panel in shared memory
  // (less cross-CTA reduction traffic per step), at least 64 rows each.
  const int64_t rows_fit = std::max<int64_t>(64, budget0 / (std::max<int64_t>(wmax, 1) * 8));
  // ~256 rows per CTA: enough work per step to cover the barrier, few enough
  // partials that the per-step reduction stays cheap.
  const int64_t mrl = mr - c0;
  const int64_t rows_target = std::max<int64_t>(64, std::min<int64_t>(rows_fit, 256));
  int G = (int)std::min<int64_t>(std::min(sms, kMaxG), std::max<int64_t>(1, cdiv(mrl, rows_target)));
  const int h = (int)cdiv(mrl, G);
  G = (int)cdiv(mrl, h);
  const int hp = h;  // lanes walk rows: stride-1, no padding needed
  const int64_t budget = budget0;
  int sw = 0;
  for (int cand : {128, 64, 32, 16, 8, 4, 2, 1}) {
    const int64_t swc = std::min<int64_t>(cand, wmax);
    // One sub-panel covering the whole width needs no compact-WY scratch.
    const int64_t need = swc == wmax ? swc * hp * 8 : (swc * hp + swc * swc + swc * wmax) * 8;
    if (need <= budget) {
      sw = (int)swc;
      break;
    }
  }
  if (sw == 0) {
    set_error("panel_qr: panel of %lld rows does not fit shared memory", (long long)mr);
    return SQR_EINVAL;
  }
  const int64_t smem = sw == wmax ? (int64_t)sw * hp * 8 : ((int64_t)sw * hp + (int64_t)sw * sw + (int64_t)sw * wmax) * 8;
  PanelArgs a;
  a.P = P;
  a.ldp = ldp;
  a.mr = (int)mr;
  a.c0 = (int)c0;
  a.wstat = (int)w;
  a.wmax = (int)wmax;
  a.sw = sw;
  a.h = h;
  a.hp = hp;
  a.stop_at_zero = stop_at_zero;
  a.Y = Y;
  a.ldy = ldy;
  a.taus = taus;
  a.st = st;
  char* p = static_cast<char*>(ws);
  a.bar = reinterpret_cast<unsigned*>(p);
  p += 64;
  a.part = reinterpret_cast<double*>(p);
  p += 2 * 148 * (128 + 1) * 8;
  a.rowt = reinterpret_cast<double*>(p);
  p += 2 * (128 + 1) * 8;
  a.wpart = reinterpret_cast<double*>(p);
  p += (int64_t)148 * 128 * wmax * 8;
  a.wred = reinterpret_cast<double*>(p);
  a.trace = g_trace_host_ptr;
  if (int rc = smem_optin((const void*)panel_kernel, (int)smem)) return rc;
  void* args[] = {&a};
  SQR_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  ProfScope ps(kTagPanel, s);
  count_launch();
  SQR_CUDA(cudaLaunchCooperativeKernel((const void*)panel_kernel, dim3(G), dim3(kPThreads), args,
                                       (size_t)smem, s));
  return SQR_OK;
}

int build_t(const double* Gm, int64_t ldg, const double* taus, int64_t j, double* T, int64_t ldt,
            const int32_t* gate, cudaStream_t s) {
  return build_t_fast(Gm, ldg, taus, j, T, ldt, gate, s);  // build_t.cu
}

}  // namespace sqr
