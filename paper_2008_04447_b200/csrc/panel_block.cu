// K4 (randomized.py:107-130): the whole <= 128-column panel QR of one block
// in ONE cooperative launch.  Replaces, for panels of <= 148 x 256 rows, the
// leaf-kernel + external-GEMM sequence of driver.cu:panel_factor.
//
//   * thread layout: CTA g, thread i owns panel row R = 256 g + i for the
//     whole launch; the current 32-column leaf of that row lives in
//     registers (as in panel.cu:leaf_kernel, same per-column step: one grid
//     barrier, transpose-butterfly warp reduction, fixed-order CTA reduction);
//   * leaf boundary (householder.py:52-61, 107-120 restated for one leaf):
//       M = Y_l^T [Y_l | P_rest]   per-CTA DMMA partials over its 256 rows,
//                                  then a distributed fixed-order grid
//                                  reduction (CTA g sums a slice, 2 barriers)
//       T_l from (diag(M), taus)   every CTA, one row of T per lane
//       W = T_l^T M[:, 32:]        every CTA
//       P_rest -= Y_l W            each thread on its own row (no barrier:
//                                  the next leaf loads rows it wrote itself)
//   An exactly zero column stops the panel after the remaining columns have
//   received every earlier reflector (randomized.py:120-121).
#include <math.h>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kBT = 256;            // threads = rows per CTA
constexpr int kBW = kBT / 32;       // warps
constexpr int kLf = 32;             // leaf width
constexpr int kYP = kBT + 4;        // smem pitch of a 256-row column (4 mod 32 doubles)
constexpr int kMaxGB = 152;

struct BlockPanelArgs {
  double* P;
  int64_t ldp;
  int mr, wstat, wmax, stop_at_zero;
  double* Y;
  int64_t ldy;
  double* taus;
  sqr_status* st;
  unsigned* bar;
  double* part;   // [2][33][G]       per-step partials
  double* rowt;   // [2][33]          pivot-row values
  double* mpart;  // [4096][G]        boundary partials (value-major)
  double* mred;   // [4096]           boundary sums
  unsigned long long* trace;
  ResidentSig sig;
};

constexpr int kWP = kLf + 4;        // W pitch (4 mod 32: conflict-free B fragments)
constexpr int kRP = kLf + 2;        // pitch of the per-warp M partials (conflict-free stores)
constexpr int kWsD = 96 * kWP + 96; // Ws + pad: Ms | Ts | Ws also holds 8 warps x 32 x kRP partials
// smem: ys[32][kYP] | ps[32][kYP] | Ms[128][32] | Ts[32][33] | Ws[96][kWP]+pad | taus[32]
constexpr int kSmemDoubles = 2 * kLf * kYP + 128 * kLf + kLf * (kLf + 1) + kWsD + kLf;
static_assert(128 * kLf + kLf * (kLf + 1) + kWsD >= kBW * kLf * kRP, "M partial scratch");

__global__ void __launch_bounds__(kBT, 1) panel_block_kernel(BlockPanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* ys = sm;
  double* ps = ys + kLf * kYP;
  double* Ms = ps + kLf * kYP;
  double* Ts = Ms + 128 * kLf;
  double* Ws = Ts + kLf * (kLf + 1);
  double* tau_s = Ws + kWsD;
  __shared__ double red[kBW][kLf];
  __shared__ double vals[kLf];
  __shared__ double rowv[kLf];
  __shared__ double wv[kLf];
  if (a.st->stop) {
    if (blockIdx.x == 0 && threadIdx.x == 0) signal_resident(a.sig);
    return;
  }
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  // CTAs are dispatched in index order: once the last one runs, all are resident
  if (g == G - 1 && tid == 0) signal_resident(a.sig);
  const int lane = tid & 31, warp = tid >> 5;
  const int w = max(0, min(a.wstat < 0 ? a.st->sample_achieved : a.wstat, a.wmax));
  const int R = g * kBT + tid;
  const bool live = R < a.mr;
  GridBarrier gb;
  gb.init(a.bar);
  int bhat = w;
  bool stopped = false;
  int step = 0;  // parity counter of the per-step partial buffers

  for (int c0 = 0; c0 < w && !stopped; c0 += kLf) {
    const int wl = min(kLf, w - c0);
    const int li = c0 / kLf;
    SQR_TRACE(a.trace, 8 * (40 + li) + 7);
    // Shift register: x[v] is panel column c0 + t + v of my row at step t, so
    // every register index is static without unrolling the step loop (the
    // finished column leaves through x[0] and is stored at once).
    double x[kLf];
#pragma unroll
    for (int c = 0; c < kLf; ++c) {
      x[c] = (live && c < wl) ? a.P[(int64_t)(c0 + c) * a.ldp + R] : 0.0;
      ys[c * kYP + tid] = 0.0;
    }
    int bl = wl;  // reflectors of this leaf
    int t = 0;
#pragma unroll 1
    for (; t < wl; ++t) {
      const int tc = c0 + t;
      const int par = step & 1;
      ++step;
      const int L = wl - t;  // live values this step: |a|^2 and L-1 dots
#ifdef SQR_PANEL_CK  // per-column cycle probe (tools/panel_cycles.py; build with -DSQR_PANEL_CK)
      const bool ck = a.trace != nullptr && g == 0 && tid == 0 && tc < 100;
#else
      constexpr bool ck = false;
#endif
      long long ck0 = ck ? clock64() : 0;
      double q[kLf];
      {
        const double av = R > tc ? x[0] : 0.0;
#pragma unroll
        for (int v = 0; v < kLf; ++v) q[v] = av * x[v];
      }
#pragma unroll
      for (int k = 16; k >= 1; k >>= 1) {
        const bool upper = (lane & k) != 0;
#pragma unroll
        for (int i = 0; i < k; ++i) {
          const double send = upper ? q[i] : q[i + k];
          const double keep = upper ? q[i + k] : q[i];
          q[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
        }
      }
      long long ck1 = ck ? clock64() + (long long)(q[0] * 0.0) : 0;
      red[warp][lane] = q[0];
      __syncthreads();
      if (tid < L) {
        double s = 0.0;
#pragma unroll
        for (int wi = 0; wi < kBW; ++wi) s += red[wi][tid];
        a.part[((size_t)par * (kLf + 1) + tid) * G + g] = s;
      }
      if (R == tc) {
#pragma unroll
        for (int v = 0; v < kLf; ++v)
          if (v < L) a.rowt[par * (kLf + 1) + v] = x[v];
      }
      long long ck2 = ck ? clock64() : 0;
      if (tc < 40) SQR_TRACE(a.trace, 8 * tc + 1);
      gb.sync();
      if (tc < 40) SQR_TRACE(a.trace, 8 * tc + 2);
      long long ck3 = ck ? clock64() : 0;
      {
        if (tid < L) rowv[tid] = __ldcg(a.rowt + par * (kLf + 1) + tid);
        const int v = tid >> 3, qd = tid & 7;
        if (v < L) {
          double xr[kMaxGB / 8];
          const double* src = a.part + ((size_t)par * (kLf + 1) + v) * G;
#pragma unroll
          for (int i = 0; i < kMaxGB / 8; ++i) {
            const int gi = qd + 8 * i;
            xr[i] = gi < G ? __ldcg(src + gi) : 0.0;
          }
          double sacc = 0.0;
#pragma unroll
          for (int i = 0; i < kMaxGB / 8; ++i) sacc += xr[i];
          const unsigned gm = 0xffu << (lane & 24);
          sacc += __shfl_xor_sync(gm, sacc, 4);
          sacc += __shfl_xor_sync(gm, sacc, 2);
          sacc += __shfl_xor_sync(gm, sacc, 1);
          if (qd == 0) vals[v] = sacc;
        }
      }
      __syncthreads();
      long long ck4 = ck ? clock64() : 0;
      const double at = rowv[0], sa = vals[0];
      const double nrm = sqrt(fma(at, at, sa));
      if (nrm == 0.0 && a.stop_at_zero) {
        bl = t;
        stopped = true;
        break;
      }
      double beta = 0.0, tau = 0.0, y0 = 1.0, ry = 1.0;
      if (nrm != 0.0) {
        beta = (at >= 0.0 ? -1.0 : 1.0) * nrm;
        y0 = at - beta;
        ry = __drcp_rn(y0);
        tau = 2.0 / (1.0 + sa / (y0 * y0));
      }
      // a / y0 as div_rn (correctly rounded, bitwise equal to the IEEE quotient)
      if (tid < kLf) wv[tid] = (tid >= 1 && tid < L) ? tau * (rowv[tid] + div_rn(vals[tid], y0, ry)) : 0.0;
      if (tid == 0) tau_s[t] = tau;
      if (g == 0 && tid == 0) a.taus[tc] = tau;
      __syncthreads();
      long long ck5 = ck ? clock64() : 0;
      double yst;  // explicit Y entry of my row in column tc
      if (R > tc) {
        const double yr = nrm != 0.0 ? div_rn(x[0], y0, ry) : 0.0;
        x[0] = yr;
        yst = yr;
#pragma unroll
        for (int v = 1; v < kLf; ++v) x[v] = fma(-yr, wv[v], x[v]);
      } else if (R == tc) {
        x[0] = beta;
        yst = 1.0;
#pragma unroll
        for (int v = 1; v < kLf; ++v) x[v] -= wv[v];
      } else {
        yst = 0.0;
      }
      ps[t * kYP + tid] = x[0];  // written back after the leaf (no stores before the barriers)
      ys[t * kYP + tid] = live ? yst : 0.0;
#pragma unroll
      for (int v = 0; v < kLf - 1; ++v) x[v] = x[v + 1];
      x[kLf - 1] = 0.0;
      if (ck) {
        long long* c = reinterpret_cast<long long*>(a.trace) + 1200 + 8 * tc;
        c[0] = ck1 - ck0;
        c[1] = ck2 - ck1;
        c[2] = ck3 - ck2;
        c[3] = ck4 - ck3;
        c[4] = ck5 - ck4;
        c[5] = clock64() - ck5 + (long long)(x[0] * 0.0);
      }
    }
    if (live) {
      for (int c = 0; c < t; ++c) {
        a.P[(int64_t)(c0 + c) * a.ldp + R] = ps[c * kYP + tid];
        a.Y[(int64_t)(c0 + c) * a.ldy + R] = ys[c * kYP + tid];
      }
    }
    if (stopped) {
      bhat = c0 + bl;
      // columns tc.. of the leaf keep their (updated) values and a zero Y
      if (live) {
#pragma unroll
        for (int v = 0; v < kLf; ++v)
          if (v < wl - t) {
            a.P[(int64_t)(c0 + t + v) * a.ldp + R] = x[v];
            a.Y[(int64_t)(c0 + t + v) * a.ldy + R] = 0.0;
          }
      }
    }
    // Y columns of a partial last leaf are zero (up to wmax)
    if (live)
      for (int c = c0 + wl; c < min(c0 + kLf, a.wmax); ++c) a.Y[(int64_t)c * a.ldy + R] = 0.0;
    SQR_TRACE(a.trace, 8 * (40 + li) + 0);
    const int rest = w - (c0 + kLf);
    if (rest <= 0 || bl == 0) continue;  // nothing right of the leaf / no reflector to apply
    // ---- leaf boundary: M = Y_l^T [Y_l | P_rest] over my CTA's rows (Y_l staged in ys)
    if (tid < kLf) tau_s[tid] = tid < bl ? tau_s[tid] : 0.0;
    const int nch = 1 + (rest + kLf - 1) / kLf;  // chunk 0 = Y_l itself
    const int V = kLf * (kLf + rest);
    const int gq = lane >> 2, tq = lane & 3;
    // my row of the next P_rest chunk, prefetched into registers while the
    // current chunk's DMMAs run (x is dead here)
    auto fetch = [&](int ch) {
      const int cb = c0 + kLf + (ch - 1) * kLf;
#pragma unroll
      for (int c = 0; c < kLf; ++c) {
        const int gc = cb + c;
        x[c] = (live && gc < w) ? a.P[(int64_t)gc * a.ldp + R] : 0.0;
      }
    };
    if (nch > 1) fetch(1);
    for (int ch = 0; ch < nch; ++ch) {
      const double* B = ys;
      if (ch > 0) {
#pragma unroll
        for (int c = 0; c < kLf; ++c) ps[c * kYP + tid] = x[c];
        if (ch + 1 < nch) fetch(ch + 1);
        B = ps;
      }
      __syncthreads();
      // K split over warps: warp q multiplies rows [32q, 32q + 32) into the
      // whole 32 x 32 chunk (A fragments reused across the 4 n-tiles), then
      // the 8 warp partials are summed in warp order through shared memory.
      double acc[2][4][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mi][nj][e] = 0.0;
      const int kb = warp * 32;
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 4) {
        const int kk = kb + k0 + tq;
        double af[2][2], bf[4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          af[mi][0] = ys[(16 * mi + gq) * kYP + kk];
          af[mi][1] = ys[(16 * mi + gq + 8) * kYP + kk];
        }
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) bf[nj] = B[(8 * nj + gq) * kYP + kk];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma16x8x4(acc[mi][nj], af[mi][0], af[mi][1], bf[nj]);
      }
      double* wred = Ms + warp * (kLf * kRP);  // scratch over Ms | Ts | Ws
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              wred[(8 * nj + 2 * tq + e) * kRP + 16 * mi + gq + 8 * h] = acc[mi][nj][2 * h + e];
      __syncthreads();
      // partial (a, c) -> value v = (32 ch + c) * 32 + a, stored value-major [v][G]
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int v = tid + kBT * k;
        const int c = v >> 5, ar = v & 31;
        double s = 0.0;
#pragma unroll
        for (int wi = 0; wi < kBW; ++wi) s += Ms[wi * (kLf * kRP) + c * kRP + ar];
        if (ch * kLf + c < kLf + rest) a.mpart[(size_t)(ch * kLf * kLf + v) * G + g] = s;
      }
      __syncthreads();
    }
    SQR_TRACE(a.trace, 8 * (40 + li) + 1);
    gb.sync();
    SQR_TRACE(a.trace, 8 * (40 + li) + 2);
    // distributed reduction: CTA g sums values [g per, (g+1) per), 8 lanes each
    {
      const int per = (V + G - 1) / G;
      const int vb = g * per, ve = min(V, vb + per);
      for (int v0 = vb; v0 < ve; v0 += kBT / 8) {
        const int v = v0 + (tid >> 3), qd = tid & 7;
        if (v < ve) {
          double xr[kMaxGB / 8];
          const double* src = a.mpart + (size_t)v * G;
#pragma unroll
          for (int i = 0; i < kMaxGB / 8; ++i) {
            const int gi = qd + 8 * i;
            xr[i] = gi < G ? __ldcg(src + gi) : 0.0;
          }
          double sacc = 0.0;
#pragma unroll
          for (int i = 0; i < kMaxGB / 8; ++i) sacc += xr[i];
          const unsigned gm = 0xffu << (lane & 24);
          sacc += __shfl_xor_sync(gm, sacc, 4);
          sacc += __shfl_xor_sync(gm, sacc, 2);
          sacc += __shfl_xor_sync(gm, sacc, 1);
          if (qd == 0) a.mred[v] = sacc;
        }
      }
    }
    SQR_TRACE(a.trace, 8 * (40 + li) + 3);
    gb.sync();
    for (int v = tid; v < V; v += kBT) Ms[v] = __ldcg(a.mred + v);
    __syncthreads();
    SQR_TRACE(a.trace, 8 * (40 + li) + 4);
    // T_l (householder.py:56-60): lane i of warp 0 builds row i,
    //   T[i][c] = -tau_c sum_{l<c} T[i][l] G[l][c]  (c > i),  T[i][i] = tau_i.
    if (warp == 0) {
      double tr[kLf];
#pragma unroll
      for (int c = 0; c < kLf; ++c) {
        // column c of G as broadcast LDS.128, all issued before the FMAs
        const double2* Gc = reinterpret_cast<const double2*>(Ms + c * kLf);
        double2 gv[kLf / 2];
#pragma unroll
        for (int l2 = 0; l2 < (c + 1) / 2; ++l2) gv[l2] = Gc[l2];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l2 = 0; l2 < (c + 1) / 2; ++l2) {
          const int l = 2 * l2;
          if (l2 & 1) {
            s2 = fma(tr[l], gv[l2].x, s2);
            if (l + 1 < c) s3 = fma(tr[l + 1], gv[l2].y, s3);
          } else {
            s0 = fma(tr[l], gv[l2].x, s0);
            if (l + 1 < c) s1 = fma(tr[l + 1], gv[l2].y, s1);
          }
        }
        const double tc = tau_s[c];
        tr[c] = c == lane ? tc : (c > lane ? -tc * ((s0 + s1) + (s2 + s3)) : 0.0);
      }
#pragma unroll
      for (int c = 0; c < kLf; ++c) Ts[lane * (kLf + 1) + c] = tr[c];
    }
    __syncthreads();
    SQR_TRACE(a.trace, 8 * (44 + li) + 0);
    // W = T^T S:  W[c][a] = sum_{i <= a} T[i][a] S[i][c],  S[i][c] = Ms[(32 + c) 32 + i];
    // lane a keeps column a of T in registers, warp q takes c = q, q + 8, ...
    // (zero rows up to the 32-column chunk boundary for the update GEMM).
    {
      double tcol[kLf];
#pragma unroll
      for (int i = 0; i < kLf; ++i) tcol[i] = i <= lane ? Ts[i * (kLf + 1) + lane] : 0.0;
      const int restp = (rest + kLf - 1) / kLf * kLf;
      for (int c = warp; c < restp; c += kBW) {
        double s0 = 0.0, s1 = 0.0;
        if (c < rest) {
          const double2* Sc = reinterpret_cast<const double2*>(Ms + (kLf + c) * kLf);
#pragma unroll
          for (int i = 0; i < kLf / 2; ++i) {
            const double2 sv = Sc[i];
            s0 = fma(tcol[2 * i], sv.x, s0);
            s1 = fma(tcol[2 * i + 1], sv.y, s1);
          }
        }
        Ws[c * kWP + lane] = s0 + s1;
      }
    }
    __syncthreads();
    SQR_TRACE(a.trace, 8 * (40 + li) + 5);
    // P_rest -= Y_l W with DMMA: warp q owns CTA rows [32q, 32q + 32), 32 columns per pass.
    {
      const int cb = c0 + kLf;
      const int rb = warp * 32;
      const int R0 = g * kBT;
      double pv[2][2][4][2];
      auto load_p = [&](int n0) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int Rr = R0 + rb + 16 * mi + gq + 8 * h;
            const bool rok = Rr < a.mr && Rr >= c0;
#pragma unroll
            for (int nj = 0; nj < 4; ++nj)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = n0 + 8 * nj + 2 * tq + e;
                pv[mi][h][nj][e] = (rok && c < rest) ? __ldcg(a.P + (int64_t)(cb + c) * a.ldp + Rr) : 0.0;
              }
          }
      };
      load_p(0);
      for (int n0 = 0; n0 < rest; n0 += kLf) {
        double acc[2][4][4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mi][nj][e] = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < kLf; k0 += 4) {
          double af[2][2], bf[4];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            af[mi][0] = ys[(k0 + tq) * kYP + rb + 16 * mi + gq];
            af[mi][1] = ys[(k0 + tq) * kYP + rb + 16 * mi + gq + 8];
          }
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) bf[nj] = Ws[(n0 + 8 * nj + gq) * kWP + k0 + tq];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 4; ++nj) dmma16x8x4(acc[mi][nj], af[mi][0], af[mi][1], bf[nj]);
        }
        double out[2][2][4][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nj = 0; nj < 4; ++nj)
#pragma unroll
              for (int e = 0; e < 2; ++e) out[mi][h][nj][e] = pv[mi][h][nj][e] - acc[mi][nj][2 * h + e];
        if (n0 + kLf < rest) load_p(n0 + kLf);  // next chunk's loads in flight during the stores
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int Rr = R0 + rb + 16 * mi + gq + 8 * h;
            const bool rok = Rr < a.mr && Rr >= c0;
#pragma unroll
            for (int nj = 0; nj < 4; ++nj)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = n0 + 8 * nj + 2 * tq + e;
                if (rok && c < rest) a.P[(int64_t)(cb + c) * a.ldp + Rr] = out[mi][h][nj][e];
              }
          }
      }
    }
    __syncthreads();
    SQR_TRACE(a.trace, 8 * (40 + li) + 6);
  }
  // columns never reached (zero-column stop) keep zero Y / tau
  if (stopped && live) {
    for (int c = ((bhat + kLf) / kLf) * kLf; c < a.wmax; ++c) a.Y[(int64_t)c * a.ldy + R] = 0.0;
  }
  if (live) {
    for (int c = ((w + kLf - 1) / kLf) * kLf; c < a.wmax; ++c) a.Y[(int64_t)c * a.ldy + R] = 0.0;
  }
  if (g == 0 && tid == 0) {
    for (int c = bhat; c < a.wmax; ++c) a.taus[c] = 0.0;
    a.st->bhat = bhat;
    if (bhat == 0 && a.stop_at_zero) {
      a.st->stop = 1;
      a.st->reason = SQR_STOP_PANEL_ZERO;
    }
  }
}

}  // namespace

int64_t panel_block_max_rows() { return (int64_t)148 * kBT; }

int64_t panel_block_workspace() {
  return 64 + 2 * 148 * 33 * 8 + 2 * 33 * 8 + (int64_t)4096 * 148 * 8 + 4096 * 8 + 4096;
}

int panel_block(double* P, int64_t ldp, int64_t mr, int64_t w, int64_t wmax, double* Y, int64_t ldy,
                double* taus, int stop_at_zero, sqr_status* st, void* ws, int64_t ws_bytes, cudaStream_t s,
                ResidentSig sig) {
  if (mr <= 0 || wmax <= 0) return sig.flag ? signal_resident_host(sig, s) : SQR_OK;
  if (wmax > 128 || mr > panel_block_max_rows() || ws_bytes < panel_block_workspace()) {
    set_error("panel_block: unsupported panel %lld x %lld", (long long)mr, (long long)wmax);
    return SQR_EINVAL;
  }
  const int G = (int)cdiv(mr, (int64_t)kBT);
  BlockPanelArgs a{};
  a.P = P;
  a.ldp = ldp;
  a.mr = (int)mr;
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
  p += 2 * 148 * 33 * 8;
  a.rowt = reinterpret_cast<double*>(p);
  p += 2 * 33 * 8;
  p = reinterpret_cast<char*>(rup(reinterpret_cast<uintptr_t>(p), 256));
  a.mpart = reinterpret_cast<double*>(p);
  p += (int64_t)4096 * 148 * 8;
  a.mred = reinterpret_cast<double*>(p);
  a.trace = g_trace_host_ptr;
  a.sig = sig;
  const int smem = kSmemDoubles * 8;
  if (int rc = smem_optin((const void*)panel_block_kernel, smem)) return rc;
  void* args[] = {&a};
  SQR_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  ProfScope ps(kTagPanel, s);
  count_launch();
  SQR_CUDA(cudaLaunchCooperativeKernel((const void*)panel_block_kernel, dim3(G), dim3(kBT), args, (size_t)smem, s));
  return SQR_OK;
}

}  // namespace sqr
