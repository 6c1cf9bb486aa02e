// Halted column-pivoted QR of the l x nt sample by PIVOT EPOCHS (reference:
// sketch.py:97-119 -> reference.py:107-150; same pivots, reflectors, norm
// downdates, 2^-40 guard with exact recompute, rank floor and tie rule as
// sample_qrcp_reg_kernel, whose per-column arithmetic this file repeats
// operation for operation).
//
// The per-pivot grid barrier of the thread-per-column kernel is replaced by a
// leader / worker split over G + 1 co-resident CTAs:
//
//   workers (CTAs 0..G-1)  thread t of CTA g owns sample column 256 g + t
//       (rows [RS, l) in registers, [0, RS) in shared memory, as in
//       sample_qrcp_reg_kernel).  They stream the reflectors the leader
//       publishes and apply them in order, batch by batch (one acquire poll +
//       one L2 read per batch, no grid barrier).  At an epoch boundary each
//       worker publishes its best q columns (by (norm^2, position)), their
//       values, and the bound "every other column of mine is <= ninth".
//   leader (CTA G)  gathers the published candidates, keeps the best <= 256
//       of them (threshold by bisection on the records), and runs the pivot
//       steps on its private copies of those columns: argmax, reflector,
//       update, downdate -- with the same code as the workers, so the copies
//       stay bitwise equal to the owners' columns.  A step is taken only
//       while its winner provably beats every column outside the candidate
//       set:  v > U + 2^-40 Uref,  U = the largest norm^2 left outside at the
//       epoch start (norms only shrink under the downdate; the guard's
//       exact recompute can exceed the downdated value by < 136 eps Uref,
//       far below the 2^-40 margin).  Otherwise the epoch ends and a new one
//       starts from fresh records; an epoch's first step is the exact global
//       argmax of the records (every worker's best column is among them), so
//       each epoch makes progress.
//
// A Gaussian 136 x 32768 sample needs ~7 epochs for 128 pivots
// (DESIGN.md §3), i.e. ~7 grid-wide exchanges instead of 128 barriers.
#include <float.h>
#include <limits.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace sqr {
namespace {

constexpr int kET = 256;     // threads per CTA: worker columns / leader candidate slots
constexpr int kER = 48;      // register rows per column
constexpr int kRing = 8;     // worker ring of reflectors (batch size cap)
constexpr int kEMaxEll = 144;
constexpr int kRecTarget = 1024;  // records per epoch (all workers together)
constexpr int kLW = 7;            // leader compute warps; warp kLW publishes
constexpr int kLC = kLW * 32;     // leader candidate slots
constexpr int kMaxRecPerThr = 6;  // leader: records per compute thread (G q <= 1280 <= 6 kLC)
constexpr int kBisect = 10;
constexpr int kPollNs = 100;   // worker poll back-off
constexpr double kGuardE = 0x1p-40;      // reference.py:40 (also the leader's margin)
constexpr double kRankFloorE = 0x1p-52;  // reference.py:44
constexpr double kSampleFloorE = 0x1p-48;  // sketch.py:38
constexpr int kPosNone = 1 << 30;        // + slot: unique key of an empty / dead entry

// progress word (leader -> workers): steps * 4 + kind
constexpr unsigned kMore = 0, kEpochEnd = 1, kFinished = 2;

struct EpochArgs {
  const double* B;
  int64_t ldb;
  int ell, nt, bb, first, RS, G, q, ldx;
  double* Bf;
  int64_t ldbf;
  int64_t* lperm;
  int32_t* moves;
  double* taus;
  sqr_status* st;
  unsigned* ectr;   // epoch arrivals of the workers (own 128-byte line)
  unsigned* word;   // leader progress word (own line)
  double2* rec;     // [G q] {norm^2, position bits}
  double* rrsq;     // [G q] the records' reference norms^2 (last exact recompute)
  double2* winfo;   // [G][2] {ninth, max rsq}, {sum norm^2, max norm^2} (initial)
  double* xcol;     // [G q][ldx] the records' columns (rows >= the epoch's step)
  double* yall;     // [bb][ldx] reflectors, zeros above the pivot row
  double4* meta;    // [bb] {tau, beta, pivot position bits, 0}
  unsigned long long* trace;
};

__device__ __forceinline__ bool better_e(double v1, int p1, double v2, int p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

__device__ __forceinline__ double2 lds2e(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// Shared rows are stored [row][column] with the column index XOR-swizzled by
// the row's low 4 bits: thread-per-column access of one row stays a
// permutation within each warp's 32 slots (conflict-free), and one column read
// across 32 rows (the pivot column, the coalesced staging copies) hits 16
// distinct 8-byte banks (2 wavefronts instead of 32).
__device__ __forceinline__ int cidx(int r, int c) { return r * kET + (c ^ (r & 15)); }

// Pending shared-memory-row update of a column: step pj's (y, w), applied to
// rows [pj, RS) by the NEXT step's pass (fused with its dot) or by flush().
// The arithmetic per entry is the per-pivot kernel's deferred update
// c = fma(-y_r, w, c), so values are bitwise the same.
struct Pending {
  const double* y;
  double w;
  int j;  // -1: none
};

__device__ __forceinline__ void flush(Pending& pd, int RS, double* cs, int c) {
  if (pd.j >= 0)
    for (int r = pd.j; r < RS; ++r) cs[cidx(r, c)] = fma(-pd.y[r], pd.w, cs[cidx(r, c)]);
  pd.j = -1;
}

// One reflector step on the calling thread's column (sample_qrcp_reg_kernel,
// "pos >= 0" branch): w = tau (y . d), d[j:] -= w y, downdate of the squared
// norm by the new row-j entry with the reference's guard and exact recompute.
// yf: full-length reflector (zeros above j and at rows >= ell), &yf[RS]
// 16-byte aligned; cs: this column's shared rows (stride kET).  The register
// rows are updated here; the shared rows' update of THIS step is left pending.
__device__ __forceinline__ void step_fused(Pending& pd, const double* yf, double tau, int j, int RS, double* cs,
                                           int c, double (&xr)[kER], double& nsq, double& rsq) {
  double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
  if (pd.j >= 0) {
    const double* py = pd.y;
    const double pw = pd.w;
    for (int r = pd.j; r < min(j, RS); ++r) cs[cidx(r, c)] = fma(-py[r], pw, cs[cidx(r, c)]);
    int r = j;
    for (; r + 2 <= RS; r += 2) {
      const double c0 = fma(-py[r], pw, cs[cidx(r, c)]);
      const double c1 = fma(-py[r + 1], pw, cs[cidx(r + 1, c)]);
      cs[cidx(r, c)] = c0;
      cs[cidx(r + 1, c)] = c1;
      d2 = fma(yf[r], c0, d2);
      d3 = fma(yf[r + 1], c1, d3);
    }
    if (r < RS) {
      const double c0 = fma(-py[r], pw, cs[cidx(r, c)]);
      cs[cidx(r, c)] = c0;
      d2 = fma(yf[r], c0, d2);
    }
  } else {
    int r = j;
    for (; r + 2 <= RS; r += 2) {
      d2 = fma(yf[r], cs[cidx(r, c)], d2);
      d3 = fma(yf[r + 1], cs[cidx(r + 1, c)], d3);
    }
    if (r < RS) d2 = fma(yf[r], cs[cidx(r, c)], d2);
  }
#pragma unroll
  for (int q = 0; q < kER; q += 2) {
    const double2 yv = lds2e(yf + RS + q);
    d0 = fma(yv.x, xr[q], d0);
    d1 = fma(yv.y, xr[q + 1], d1);
  }
  const double wvv = tau * ((d0 + d1) + (d2 + d3));
#pragma unroll
  for (int q = 0; q < kER; q += 2) {
    const double2 yv = lds2e(yf + RS + q);
    xr[q] = fma(-yv.x, wvv, xr[q]);
    xr[q + 1] = fma(-yv.y, wvv, xr[q + 1]);
  }
  double rj;
  if (j < RS) {
    rj = fma(-yf[j], wvv, cs[cidx(j, c)]);
  } else {
    rj = 0.0;
#pragma unroll
    for (int q = 0; q < kER; ++q)
      if (RS + q == j) rj = xr[q];
  }
  double ns = nsq - rj * rj;
  if (ns < kGuardE * rsq) {
    double e0 = 0.0, e1 = 0.0;
    for (int r = j + 1; r < RS; ++r) {
      const double v = fma(-yf[r], wvv, cs[cidx(r, c)]);
      e0 = fma(v, v, e0);
    }
#pragma unroll
    for (int q = 0; q < kER; ++q)
      if (RS + q > j) e1 = fma(xr[q], xr[q], e1);
    ns = e0 + e1;
    rsq = ns;
  } else {
    ns = fmax(ns, 0.0);
  }
  nsq = ns;
  pd.y = yf;
  pd.w = wvv;
  pd.j = j;
}

// Initial squared norm, same summation order as sample_qrcp_reg_kernel.
__device__ __forceinline__ double col_norm_sq(const double* cs, int c, int RS, const double (&xr)[kER]) {
  double s0 = 0.0, s1 = 0.0;
  for (int r = 0; r < RS; ++r) {
    const double v = cs[cidx(r, c)];
    s0 = fma(v, v, s0);
  }
#pragma unroll
  for (int q = 0; q < kER; q += 2) {
    s0 = fma(xr[q], xr[q], s0);
    s1 = fma(xr[q + 1], xr[q + 1], s1);
  }
  return s0 + s1;
}

__device__ __forceinline__ void warp_argmax_e(double& v, int& p, int& l) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
    const int l2 = __shfl_xor_sync(0xffffffffu, l, o);
    if (better_e(v2, p2, v, p)) {
      v = v2;
      p = p2;
      l = l2;
    }
  }
}

__device__ __forceinline__ double warp_max_e(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_isum(int v) { return __reduce_add_sync(0xffffffffu, v); }

__device__ __forceinline__ void st_release_word(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// leader compute warps (0 .. kLW-1) only; warp kLW publishes
__device__ __forceinline__ void lbar() { asm volatile("bar.sync 1, %0;\n" ::"n"(kLC) : "memory"); }

// Bitonic sort of one (v, p, i) entry per thread (kET threads), best (largest
// v, then smallest p) first.  Keys (v, p) must be distinct (empty entries
// carry p = kPosNone + tid).  Stages across warps go through shared memory.
__device__ void block_sort_desc(double& v, int& p, int& i, double* sv, int* sp, int* si) {
  const int tid = threadIdx.x;
  for (int k = 2; k <= kET; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      double pv;
      int pp, pi;
      if (jj >= 32) {
        sv[tid] = v;
        sp[tid] = p;
        si[tid] = i;
        __syncthreads();
        pv = sv[tid ^ jj];
        pp = sp[tid ^ jj];
        pi = si[tid ^ jj];
        __syncthreads();
      } else {
        pv = __shfl_xor_sync(0xffffffffu, v, jj);
        pp = __shfl_xor_sync(0xffffffffu, p, jj);
        pi = __shfl_xor_sync(0xffffffffu, i, jj);
      }
      const bool desc = (tid & k) == 0;
      const bool lower = (tid & jj) == 0;
      const bool mine = better_e(v, p, pv, pp);
      const bool keep = (lower == desc) ? mine : !mine;
      if (!keep) {
        v = pv;
        p = pp;
        i = pi;
      }
    }
  }
}

__global__ void __launch_bounds__(kET, 1) sample_epoch_kernel(EpochArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) double stg[kET / 32][kER];  // per-warp winner's register rows
  __shared__ double stg_w[kET / 32];                   // ... and its pending w
  __shared__ int stg_j[kET / 32];                      // ... and pending step
  __shared__ double sv[kET];
  __shared__ int sp[kET], si[kET];
  __shared__ __align__(16) double4 meta_s[kRing];
  __shared__ double rd[2][kET / 32];
  __shared__ int ri[2][kET / 32];
  __shared__ unsigned wsh;
  __shared__ int cand_src[kET];
  __shared__ double red[32];
  __shared__ volatile unsigned ready_word;  // leader compute -> publisher
  __shared__ volatile int pub_steps;        // publisher -> leader compute (ring back-pressure)
  __shared__ double u0_s;
  __shared__ double oy0[kET];

  if (a.st->stop) return;
  if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || (int)blockIdx.x == a.G))
    a.trace[1100 + 2 * ((int)blockIdx.x == a.G ? 1 : 0)] = gtimer();
  const int ell = a.ell, RS = a.RS, G = a.G, q = a.q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int YP = ((max(ell, RS + kER) + 1) | 1) + 1;  // even pitch of a reflector slot
  const int yoff = RS & 1;                            // &slot[RS] 16-byte aligned
  double* cs = sm;  // [max(RS, kER)][kET] swizzled (cidx); rows >= RS: staging
  double* ring = cs + (size_t)max(RS, kER) * kET;      // [kRing][YP] (+ yoff)
  auto slot = [&](int t) -> double* { return ring + (size_t)(t % kRing) * YP + yoff; };
  for (int e = tid; e < kRing * YP; e += kET) ring[e] = 0.0;  // rows >= ell stay zero
  const bool leader = (int)blockIdx.x == G;
  if (tid == 0) {
    ready_word = 0;
    pub_steps = 0;
  }
  __syncthreads();

  // ===================================================================== workers
  if (!leader) {
    const int g = blockIdx.x;
    const int col = g * kET + tid;
    const bool own = col < a.nt;
    double xr[kER];
    {
      // coalesced: a warp copies one column at a time (lanes over rows); the
      // register rows are staged through the (not yet used) shared-row area
      // gathers by cp.async (8-byte, zero-fill): the whole column block is in
      // flight at once -- register-staged loads cap the bytes in flight per
      // SM far below the L2 bandwidth.  Consecutive threads copy consecutive
      // rows of one column (coalesced); the register rows are staged through
      // the (not yet used) shared-row area.
      const int ncol = min(kET, a.nt - g * kET);
      const double* B0 = a.B + (int64_t)g * kET * a.ldb;
      for (int c = warp; c < kET; c += kET / 32) {
        const double* src = B0 + (int64_t)c * a.ldb;
        for (int qq = lane; qq < kER; qq += 32) {
          const bool ok = c < ncol && RS + qq < ell;
          cp_async<8>(cs + cidx(qq, c), ok ? src + RS + qq : B0, ok);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int qq = 0; qq < kER; ++qq) xr[qq] = cs[cidx(qq, tid)];
      __syncthreads();
      for (int c = warp; c < kET; c += kET / 32) {
        const double* src = B0 + (int64_t)c * a.ldb;
        for (int r = lane; r < RS; r += 32) cp_async<8>(cs + cidx(r, c), c < ncol ? src + r : B0, c < ncol);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
    if (a.trace && g == 0 && tid == 0) a.trace[1110] = gtimer();
    double nsq = col_norm_sq(cs, tid, RS, xr);
    double rsq = nsq;
    int pos = own ? col : -1;
    int disp = -1, pj = -1;
    double pbeta = 0.0;
    Pending pd{nullptr, 0.0, -1};
    double psum, pmax;
    {
      psum = block_sum(own ? nsq : 0.0, red);
      double mx = warp_max_e(own ? nsq : 0.0);
      if (lane == 0) rd[0][warp] = mx;
      __syncthreads();
      pmax = rd[0][0];
      for (int w = 1; w < kET / 32; ++w) pmax = fmax(pmax, rd[0][w]);
      __syncthreads();
    }
    // epoch boundary at step j: records, columns, bounds; arrive
    auto publish = [&](int j) {
      flush(pd, RS, cs, tid);
      double v = pos >= 0 ? nsq : -1.0;
      int p = pos >= 0 ? pos : kPosNone + tid;
      int i = tid;
      if (a.trace && g == 0 && tid == 0 && j == 0) a.trace[1111] = gtimer();
      block_sort_desc(v, p, i, sv, sp, si);
      __syncthreads();
      if (a.trace && g == 0 && tid == 0 && j == 0) a.trace[1112] = gtimer();
      si[i] = tid;  // sorted entry tid holds column i: its rank
      if (q < kET && tid == q) sv[0] = (p < kPosNone) ? v : -1.0;  // the (q+1)-th best
      double mr = warp_max_e(pos >= 0 ? rsq : 0.0);
      if (lane == 0) rd[1][warp] = mr;
      __syncthreads();
      const double ninth = q < kET ? sv[0] : -1.0;
      const int rank = si[tid];
      if (rank < q) {
        const int slot_i = g * q + rank;
        a.rec[slot_i] = make_double2(pos >= 0 ? nsq : -1.0,
                                     __longlong_as_double((long long)(pos >= 0 ? pos : kPosNone)));
        a.rrsq[slot_i] = rsq;
        if (pos >= 0) {
          double* dst = a.xcol + (size_t)slot_i * a.ldx;
          for (int r = j; r < RS; ++r) dst[r] = cs[cidx(r, tid)];
#pragma unroll
          for (int qq = 0; qq < kER; ++qq)
            if (RS + qq >= j && RS + qq < ell) dst[RS + qq] = xr[qq];
        }
      }
      if (tid == 0) {
        double m = rd[1][0];
        for (int w = 1; w < kET / 32; ++w) m = fmax(m, rd[1][w]);
        a.winfo[2 * g] = make_double2(ninth, m);
        a.winfo[2 * g + 1] = make_double2(psum, pmax);
      }
      __syncthreads();
      if (a.trace && g == 0 && tid == 0 && j == 0) a.trace[1113] = gtimer();
      if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(a.ectr) : "memory");
    };

    publish(0);
    if (a.trace && g == 0 && tid == 0) a.trace[1104] = gtimer();
    int jdone = 0, last_pub = 0;
    while (true) {
      if (tid == 0) {
        unsigned w;
        while (true) {
          w = ld_acquire_u32(a.word);
          const int s = (int)(w >> 2), kind = (int)(w & 3u);
          if (s > jdone || kind == (int)kFinished || (kind == (int)kEpochEnd && s != last_pub)) break;
          __nanosleep(kPollNs);  // keep 148 pollers off the L2 the leader reads
        }
        wsh = w;
      }
      __syncthreads();
      const unsigned w = wsh;
      const int s = (int)(w >> 2), kind = (int)(w & 3u);
      if (s > jdone) {
        // <= kRing - 1 per batch: the pending update still reads the slot of
        // step jdone - 1
        const int nb = min(s - jdone, kRing - 1);
        for (int e = tid; e < nb * ell; e += kET) {
          const int t = jdone + e / ell, r = e % ell;
          slot(t)[r] = __ldcg(a.yall + (size_t)t * a.ldx + r);
        }
        if (tid < nb) {
          const double2* mp = reinterpret_cast<const double2*>(a.meta + jdone + tid);
          const double2 m0 = __ldcg(mp), m1 = __ldcg(mp + 1);
          meta_s[tid] = make_double4(m0.x, m0.y, m1.x, m1.y);
        }
        __syncthreads();
        for (int t = jdone; t < jdone + nb; ++t) {
          const double4 m = meta_s[t - jdone];
          const int pc = (int)__double_as_longlong(m.z);
          if (pos == pc) {
            flush(pd, RS, cs, tid);  // frozen from here on
            pj = t;
            pbeta = m.y;
            pos = -1;
          } else if (pos >= 0) {
            if (pos == t) {
              if (disp >= 0) a.moves[2 * (a.bb + disp)] = -1;
              disp = t;
              pos = pc;
            }
            step_fused(pd, slot(t), m.x, t, RS, cs, tid, xr, nsq, rsq);
          }
        }
        __syncthreads();  // ring slots / meta_s reusable
        jdone += nb;
        continue;
      }
      if (kind == (int)kFinished) break;
      // kind == kEpochEnd, s == jdone, not yet published for this boundary
      publish(s);
      last_pub = s;
    }
    if (a.trace && g == 0 && tid == 0) a.trace[1105] = gtimer();
    flush(pd, RS, cs, tid);
    // ---- outputs (sample_qrcp_reg_kernel's tail).  A pivot column goes to Bf
    // column pj as (R part, beta, reflector tail u / (u_pj - beta)); every
    // other column to its final position.  Per column the destination, pivot
    // step, beta and y0 go to shared memory, then warps copy whole columns
    // (lanes over rows: coalesced), the register rows staged through the
    // shared-row area.
    {
      int dcol = -1, dpj = -1;
      double y0 = 1.0;
      if (pj >= 0) {
        const double u0 = pj < RS ? cs[cidx(pj, tid)] : [&] {
          double v = 0.0;
#pragma unroll
          for (int qq = 0; qq < kER; ++qq)
            if (RS + qq == pj) v = xr[qq];
          return v;
        }();
        y0 = u0 - pbeta;
        dcol = pj;
        dpj = pj;
        a.lperm[pj] = col;
        if (col != pj) {
          a.moves[2 * pj] = pj;
          a.moves[2 * pj + 1] = col;
        }
        if (disp >= 0) a.moves[2 * (a.bb + disp)] = -1;
      } else if (pos >= 0) {
        dcol = pos;
        a.lperm[pos] = col;
        if (disp >= 0 && pos != col) {
          a.moves[2 * (a.bb + disp)] = pos;
          a.moves[2 * (a.bb + disp) + 1] = col;
        } else if (disp >= 0) {
          a.moves[2 * (a.bb + disp)] = -1;
        }
      }
      sp[tid] = dcol;
      si[tid] = dpj;
      sv[tid] = pbeta;
      oy0[tid] = y0;
      __syncthreads();
      // warp per column, lanes over rows (coalesced stores)
      auto out_rows = [&](int r0, int r1, int soff) {
        for (int c = warp; c < kET; c += kET / 32) {
          const int d = sp[c];
          if (d < 0) continue;
          const int pjc = si[c];
          const double bc = sv[c], y0c = oy0[c];
          double* dst = a.Bf + (int64_t)d * a.ldbf;
          for (int r = r0 + lane; r < r1; r += 32) {
            const double u = cs[cidx(r - soff, c)];
            dst[r] = (pjc < 0 || r < pjc) ? u : (r == pjc ? bc : (bc != 0.0 ? u / y0c : 0.0));
          }
        }
      };
      out_rows(0, RS, 0);
      __syncthreads();
#pragma unroll
      for (int qq = 0; qq < kER; ++qq) cs[cidx(qq, tid)] = xr[qq];
      __syncthreads();
      out_rows(RS, ell, RS);
    }
    if (a.trace && g == 0 && tid == 0) a.trace[1101] = gtimer();
    return;
  }

  // ========================================================= leader: publisher
  // Copies each reflector / meta record from the shared ring to global memory
  // and releases the progress word, so the gpu-scope release (which waits
  // for the stores) is off the compute warps' critical path.
  if (warp == kLW) {
    unsigned done = 0;
    while (true) {
      unsigned rw = 0;
      if (lane == 0) {
        do {
          rw = ready_word;
#ifdef SQR_PUB_SLEEP
          if (rw == done) __nanosleep(SQR_PUB_SLEEP);
#endif
        } while (rw == done);
      }
      rw = __shfl_sync(0xffffffffu, rw, 0);
      __threadfence_block();
      const int s0 = (int)(done >> 2), s1 = (int)(rw >> 2);
      for (int t = s0; t < s1; ++t) {
        const double* ys = slot(t);
        double* yg = a.yall + (size_t)t * a.ldx;
        for (int r = lane; r < ell; r += 32) yg[r] = ys[r];
        if (lane == 0) {
          const double4 m = meta_s[t % kRing];
          double2* mp = reinterpret_cast<double2*>(a.meta + t);
          mp[0] = make_double2(m.x, m.y);
          mp[1] = make_double2(m.z, 0.0);
          a.taus[t] = m.x;
        }
      }
      __syncwarp();
      if (lane == 0) {
        st_release_word(a.word, rw);
        pub_steps = s1;
        if (a.trace && s1 > 0) a.trace[8 * (s1 - 1) + 6] = gtimer();
      }
      done = rw;
      if ((rw & 3u) == kFinished) break;
    }
    return;
  }

  // ====================================================== leader: compute warps
  for (int e = tid; e < 4 * a.bb; e += kLC) a.moves[e] = -1;
  if (tid == 0) a.st->nmoves = 2 * a.bb;
  auto post = [&](unsigned v) {  // thread 0 / lane 0 of warp 0
    __threadfence_block();
    ready_word = v;
  };
  double xr[kER];
  double nsq = -1.0, rsq = 0.0;
  int pos = -1;
  Pending pd{nullptr, 0.0, -1};
  double rank_floor_sq = 0.0, U = -1.0, Uref = 0.0;
  int j = 0;
  unsigned epoch = 0;
  const int NR = G * q;
  // block helpers over the compute warps (every thread gets the result;
  // alternating buffers: one barrier per call)
  int rbuf = 0;
  auto bsum_i = [&](int v) -> int {
    v = warp_isum(v);
    if (lane == 0) ri[rbuf][warp] = v;
    lbar();
    int s = 0;
#pragma unroll
    for (int w = 0; w < kLW; ++w) s += ri[rbuf][w];
    rbuf ^= 1;
    return s;
  };
  auto bmax_d = [&](double v) -> double {
    v = warp_max_e(v);
    if (lane == 0) rd[rbuf][warp] = v;
    lbar();
    double s = rd[rbuf][0];
#pragma unroll
    for (int w = 1; w < kLW; ++w) s = fmax(s, rd[rbuf][w]);
    rbuf ^= 1;
    return s;
  };

  while (true) {
    // ---------------------------------------------------------- epoch start
    if (tid == 0) {
      const unsigned target = (epoch + 1) * (unsigned)G;
      while ((int)(ld_acquire_u32(a.ectr) - target) < 0) {
      }
    }
    lbar();
    if (a.trace && tid == 0 && epoch < 64) a.trace[1024 + epoch] = gtimer();
    double L = -1.0, Ur = 0.0;
    if (epoch == 0) {
      // fro / max over the initial norms (fixed order over workers)
      // (loaded in parallel, summed in worker order)
      for (int g = tid; g < G; g += kLC) {
        const double2 wi = __ldcg(a.winfo + 2 * g + 1);
        sv[g] = wi.x;
        oy0[g] = wi.y;
      }
      lbar();
      double total = 0.0, gmax = 0.0;
      for (int g = 0; g < G; ++g) {
        total += sv[g];
        gmax = fmax(gmax, oy0[g]);
      }
      const double fro = sqrt(total);
      rank_floor_sq = (kRankFloorE * fro) * (kRankFloorE * fro);
      const double sample_floor = a.first ? kSampleFloorE * kSampleFloorE * gmax : __ldcg(&a.st->floor_sq);
      lbar();  // every thread has read st->floor_sq
      if (tid == 0 && a.first) a.st->floor_sq = sample_floor;
      if (a.nt == 0 || gmax <= sample_floor) {
        if (tid == 0) {
          a.st->stop = 1;
          a.st->reason = SQR_STOP_SAMPLE_FLOOR;
          a.st->sample_achieved = 0;
          post(kFinished);
        }
        return;
      }
    }
    for (int g = lane; g < G; g += 32) {
      const double2 wi = __ldcg(a.winfo + 2 * g);
      L = fmax(L, wi.x);
      Ur = fmax(Ur, wi.y);
    }
    L = warp_max_e(L);
    Ur = warp_max_e(Ur);
    // my records, in rank-major order (m = rank * G + worker): the compaction
    // below then gives the workers' best columns the lowest candidate slots,
    // so the candidates that stay active longest share warps
    auto rec_of = [&](int m) { return (m % G) * q + m / G; };
    double rv[kMaxRecPerThr];
    int rp[kMaxRecPerThr];
#pragma unroll
    for (int k = 0; k < kMaxRecPerThr; ++k) {
      const int i = tid + kLC * k;
      if (i < NR) {
        const double2 r = __ldcg(a.rec + rec_of(i));
        rv[k] = r.x;
        rp[k] = (int)__double_as_longlong(r.y);
      } else {
        rv[k] = -1.0;
        rp[k] = kPosNone;
      }
    }
    auto count_above = [&](double x) -> int {
      int c = 0;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k) c += rv[k] > x ? 1 : 0;
      return bsum_i(c);
    };
    double T = L;
    if (count_above(L) > kLC) {
      double lo = L;
      double hi = -1.0;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k) hi = fmax(hi, rv[k]);
      hi = bmax_d(hi);
      for (int it = 0; it < kBisect; ++it) {
        const double mid = lo + 0.5 * (hi - lo);
        if (count_above(mid) <= kLC)
          hi = mid;
        else
          lo = mid;
      }
      T = hi;
    }
    bool sel[kMaxRecPerThr];
    int mysel = 0;
#pragma unroll
    for (int k = 0; k < kMaxRecPerThr; ++k) {
      sel[k] = rv[k] > T;
      mysel += sel[k] ? 1 : 0;
    }
    int nsel = bsum_i(mysel);
    if (nsel == 0) {
      // ties at the top: the exact best record alone
      double bv = -1.0;
      int bp = INT_MAX, bl = -1;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k)
        if (better_e(rv[k], rp[k], bv, bp)) {
          bv = rv[k];
          bp = rp[k];
          bl = tid + kLC * k;
        }
      warp_argmax_e(bv, bp, bl);
      if (lane == 0) {
        sv[warp] = bv;
        sp[warp] = bp;
        si[warp] = bl;
      }
      lbar();
      for (int w = 0; w < kLW; ++w)
        if (better_e(sv[w], sp[w], bv, bp)) {
          bv = sv[w];
          bp = sp[w];
          bl = si[w];
        }
      mysel = 0;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k) {
        sel[k] = (tid + kLC * k) == bl;
        mysel += sel[k] ? 1 : 0;
      }
      nsel = 1;
      lbar();
    }
    {
      double ou = -1.0;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k)
        if (!sel[k]) ou = fmax(ou, rv[k]);
      U = fmax(L, bmax_d(ou));
      Uref = Ur;
    }
    // compaction: exclusive scan of mysel over the compute threads
    {
      int incl = mysel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) ri[rbuf][warp] = incl;
      lbar();
      int base = 0;
      for (int w = 0; w < warp; ++w) base += ri[rbuf][w];
      rbuf ^= 1;
      int o = base + incl - mysel;
#pragma unroll
      for (int k = 0; k < kMaxRecPerThr; ++k)
        if (sel[k]) cand_src[o++] = rec_of(tid + kLC * k);
    }
    lbar();
    // load my candidate (rows >= j; the rows above are zero: the reflectors
    // vanish there)
    if (a.trace && tid == 0 && epoch < 64) a.trace[1130 + epoch] = gtimer();
    pd.j = -1;
    // coalesced copy of the candidates' columns (rows >= j) from the
    // exchange area: warps copy whole columns, the register rows staged
    // through the shared-row area
    {
      const int nr = max(0, min(kER, ell - max(RS, j)));  // register rows >= j that exist
      const int r0 = max(0, j - RS);                      // first such register row
#pragma unroll
      for (int qq = 0; qq < kER; ++qq) cs[cidx(qq, tid)] = 0.0;
      lbar();
      for (int c = warp; c < nsel; c += kLW) {
        const double* x = a.xcol + (size_t)cand_src[c] * a.ldx + RS;
        for (int qq = r0 + lane; qq < r0 + nr; qq += 32) cp_async<8>(cs + cidx(qq, c), x + qq, true);
      }
      cp_async_commit();
      cp_async_wait<0>();
      lbar();
#pragma unroll
      for (int qq = 0; qq < kER; ++qq) xr[qq] = cs[cidx(qq, tid)];
      lbar();
      const int j0 = min(j, RS), ns = RS - j0;  // shared rows >= j (rows above are never read)
      for (int c = warp; c < nsel; c += kLW) {
        const double* x = a.xcol + (size_t)cand_src[c] * a.ldx;
        for (int r = j0 + lane; r < RS; r += 32) cp_async<8>(cs + cidx(r, c), x + r, true);
      }
      cp_async_commit();
    }
    if (tid < nsel) {
      const int src = cand_src[tid];
      const double2 r = __ldcg(a.rec + src);
      nsq = r.x;
      pos = (int)__double_as_longlong(r.y);
      rsq = __ldcg(a.rrsq + src);
    } else {
      nsq = -1.0;
      pos = -1;
    }
    cp_async_wait<0>();
    lbar();
    // ------------------------------------------------------------- steps
    bool first_step = true;
    while (true) {
      if (a.trace && tid == 0) a.trace[8 * j] = gtimer();
      long long ck_0 = clock64();
      double bv = pos >= 0 ? nsq : -1.0;
      int bp = pos >= 0 ? pos : INT_MAX;
      int bl = pos >= 0 ? tid : -1;
      warp_argmax_e(bv, bp, bl);
      if (bl >= 0 && tid == bl) {
#pragma unroll
        for (int qq = 0; qq < kER; ++qq) stg[warp][qq] = xr[qq];
        stg_w[warp] = pd.w;
        stg_j[warp] = pd.j;
      }
      if (lane == 0) {
        sv[warp] = bv;
        sp[warp] = bp;
        si[warp] = bl;
      }
      lbar();
      if (a.trace && tid == 0) a.trace[8 * j + 1] = gtimer();
      long long ck_1 = clock64();
      {
        double v7[kLW];
        int p7[kLW], l7[kLW];
#pragma unroll
        for (int w = 0; w < kLW; ++w) {
          v7[w] = sv[w];
          p7[w] = sp[w];
          l7[w] = si[w];
        }
#pragma unroll
        for (int w = 0; w < kLW; ++w)
          if (better_e(v7[w], p7[w], bv, bp)) {
            bv = v7[w];
            bp = p7[w];
            bl = l7[w];
          }
      }
      if (!first_step && !(bv > fma(kGuardE, Uref, U))) {
        // the winner is not provably global: new epoch from step j
        if (tid == 0) post((unsigned)j * 4u + kEpochEnd);
        break;
      }
      if (!(bv > rank_floor_sq)) {  // reference.py:123-124 (also: no candidate left)
        if (tid == 0) {
          a.st->sample_achieved = j;
          if (j == 0) {
            a.st->stop = 1;
            a.st->reason = SQR_STOP_SAMPLE_RANK;
          }
          post((unsigned)j * 4u + kFinished);
        }
        return;
      }
      // reflector j from candidate bl (house_gen, householder.py:28-49), built
      // by all compute warps: thread t takes row j + t of the winner's column
      // (its pending shared-row update applied on the fly), the squared norm
      // of rows > j is summed per warp then over warps in fixed order, every
      // thread derives (beta, y0, tau, 1 / y0) from the same values, and
      // writes its y entry.
      double* yf = slot(j);
      while (pub_steps + kRing <= j) {
      }  // slot of step j - kRing published
      const int len = ell - j;
      double xv = 0.0;
      {
        const int r = j + tid;
        const int wq = bl >> 5;
        if (tid < len) {
          if (r < RS) {
            xv = cs[cidx(r, bl)];
            if (stg_j[wq] >= 0) xv = fma(-slot(j > 0 ? j - 1 : 0)[r], stg_w[wq], xv);
          } else {
            xv = stg[wq][r - RS];
          }
        }
        const double part = warp_sum(tid >= 1 && tid < len ? xv * xv : 0.0);
        if (lane == 0) rd[rbuf][warp] = part;
        if (tid == 0) u0_s = xv;
      }
      lbar();
      long long ck_2 = clock64();
      double s1 = 0.0;
#pragma unroll
      for (int w = 0; w < kLW; ++w) s1 += rd[rbuf][w];
      rbuf ^= 1;
      const double u0 = u0_s;
      const double nrm = sqrt(fma(u0, u0, s1));
      double beta = 0.0, tau = 0.0, y0 = 1.0, ry = 1.0;
      if (nrm != 0.0) {
        beta = (u0 >= 0.0 ? -1.0 : 1.0) * nrm;
        y0 = u0 - beta;
        ry = __drcp_rn(y0);
        tau = 2.0 / (1.0 + s1 / (y0 * y0));
      }
      if (tid < len) yf[j + tid] = (tid == 0) ? 1.0 : (nrm != 0.0 ? div_rn(xv, y0, ry) : 0.0);
      for (int r = tid; r < j; r += kLC) yf[r] = 0.0;
      if (tid == 0) meta_s[j % kRing] = make_double4(tau, beta, __longlong_as_double((long long)bp), 0.0);
      lbar();
      if (tid == 0) post((unsigned)(j + 1) * 4u + kMore);
      if (a.trace && tid == 0) a.trace[8 * j + 4] = gtimer();
      long long ck_3 = clock64();
      // apply reflector j to the candidates
      if (pos == bp) {
        pos = -1;  // the pivot leaves the candidate set
        pd.j = -1;
      } else if (pos >= 0) {
        if (pos == j) pos = bp;
        step_fused(pd, yf, tau, j, RS, cs, tid, xr, nsq, rsq);
        // norms only shrink: a candidate at or below the bound can never win
        // in this epoch -- drop it (its warp skips the remaining steps once
        // all of its candidates are out)
        if (!(nsq > fma(kGuardE, Uref, U))) pos = -1;
      }
      if (a.trace && tid == 0) a.trace[8 * j + 5] = gtimer();
      if (a.trace && tid == 0 && j < 100) {
        long long* c = reinterpret_cast<long long*>(a.trace) + 1200 + 8 * j;
        c[0] = ck_1 - ck_0;
        c[1] = ck_2 - ck_1;
        c[2] = ck_3 - ck_2;
        c[3] = clock64() - ck_3;
      }
      if (a.trace && tid == 32 * (kLW - 1)) a.trace[8 * j + 7] = gtimer();
      ++j;
      first_step = false;
      if (j == a.bb) {
        if (tid == 0) {
          a.st->sample_achieved = j;
          post((unsigned)j * 4u + kFinished);
          if (a.trace) a.trace[1103] = gtimer();
        }
        return;
      }
    }
    ++epoch;
  }
}

}  // namespace

// ----------------------------------------------------------------- host side
int sample_epoch_records_per_worker(int G) {
  return std::min(kET, std::max(8, (int)cdiv(kRecTarget, G)));
}

int64_t sample_epoch_workspace(int64_t ell, int64_t nt, int64_t bb) {
  const int64_t G = std::max<int64_t>(1, cdiv(nt, kET));
  const int64_t q = sample_epoch_records_per_worker((int)G);
  const int64_t ldx = rup(ell, 2);
  return 256 + G * q * 16 + G * q * 8 + G * 32 + G * q * ldx * 8 + bb * ldx * 8 + bb * 32 + 256;
}

bool sample_epoch_eligible(int64_t ell, int64_t nt) {
  // opt-in (read per call): measured slower than the per-pivot-barrier kernel
  // in the C5 pipeline (207 vs 174 ms per step)
  if (!env_flag("SQR_EPOCH_SAMPLE")) return false;
  const int sms = std::min(sm_count(), 148);
  return ell <= kEMaxEll && nt >= 1 && cdiv(nt, kET) + 1 <= sms;
}

int sample_epoch(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf, int64_t ldbf,
                 int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st, void* ws,
                 int64_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < sample_epoch_workspace(ell, nt, bb)) {
    set_error("sample_qrcp (epoch): workspace too small");
    return SQR_EINVAL;
  }
  EpochArgs a{};
  a.B = B;
  a.ldb = ldb;
  a.ell = (int)ell;
  a.nt = (int)nt;
  a.bb = (int)bb;
  a.first = first;
  a.RS = (int)std::max<int64_t>(0, ell - kER);
  a.G = (int)std::max<int64_t>(1, cdiv(nt, kET));
  a.q = sample_epoch_records_per_worker(a.G);
  a.ldx = (int)rup(ell, 2);
  a.Bf = Bf;
  a.ldbf = ldbf;
  a.lperm = lperm;
  a.moves = moves;
  a.taus = taus;
  a.st = st;
  char* p = static_cast<char*>(ws);
  a.ectr = reinterpret_cast<unsigned*>(p);
  a.word = reinterpret_cast<unsigned*>(p + 128);
  p += 256;
  const int64_t NR = (int64_t)a.G * a.q;
  a.rec = reinterpret_cast<double2*>(p);
  p += NR * 16;
  a.winfo = reinterpret_cast<double2*>(p);
  p += (int64_t)a.G * 32;
  a.meta = reinterpret_cast<double4*>(p);
  p += bb * 32;
  a.rrsq = reinterpret_cast<double*>(p);
  p += NR * 8;
  a.xcol = reinterpret_cast<double*>(p);
  p += NR * a.ldx * 8;
  a.yall = reinterpret_cast<double*>(p);
  a.trace = g_trace_host_ptr;
  const int YP = (int)(((std::max<int64_t>(ell, a.RS + kER) + 1) | 1) + 1);
  const int smem = (int)(((int64_t)std::max(a.RS, kER) * kET + (int64_t)kRing * YP + 2) * 8);
  if (int rc = smem_optin((const void*)sample_epoch_kernel, smem)) return rc;
  void* args[] = {&a};
  SQR_CUDA(cudaMemsetAsync(ws, 0, 256, s));
  ProfScope ps(kTagSample, s);
  count_launch();
  SQR_CUDA(cudaLaunchCooperativeKernel((const void*)sample_epoch_kernel, dim3(a.G + 1), dim3(kET), args,
                                       (size_t)smem, s));
  return SQR_OK;
}

}  // namespace sqr
