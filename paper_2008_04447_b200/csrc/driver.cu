// Host-side drivers of libsqr: the whole factorization loop is enqueued on
// one stream with NO host synchronisation.  Every early exit of the
// reference loop (randomized.py:185-221, 287-336) is a device-side flag in
// sqr_status that the downstream kernels of the same and later blocks test,
// so the loop shape is static and can be captured in a CUDA graph.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace sqr {
namespace {

// Bump allocator over the caller's workspace; with base == nullptr it only
// measures (used by the *_workspace queries).
struct Carve {
  char* base;
  int64_t off = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(int64_t count) {
    off = rup(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += std::max<int64_t>(count, 1) * (int64_t)sizeof(T);
    return p;
  }
};

constexpr int64_t kLeaf = 32;
struct PanelScratch {
  double *GW, *W, *Tl;  // lw x (lw + bmax), lw x bmax, lw x lw
  static int64_t doubles(int64_t bmax) { return kLeaf * (kLeaf + bmax) + kLeaf * bmax + kLeaf * kLeaf + 64; }
};

constexpr int64_t kGemmWsBytes = (int64_t)8 * 148 * 72 * 256 * 8 + 8 * 148 * 8 * 4 + 4096;

struct RqrcpWs {
  double *Bcur, *Bnext, *Bf, *stau, *Ypan, *Gm, *Wt, *W, *OmT, *gemm, *pscr;
  int64_t* lperm;
  int32_t* moves;
  int32_t* snap;  // {stop .. bhat} of the block whose bulk update is in flight
  int32_t* guard; // R11 guard verdict of the early sample-update prep (EarlyPrep)
  double* Ypan2;  // second [Y_P | Y_J] buffer: pairs alternate (Overlap)
  unsigned* sig;  // ResidentSig word of the overlapped chain kernels
  int32_t* snap2; // {stop .. bhat} of a pair's first block (early rows, Overlap)
  void *sample, *panel;
  int64_t sample_bytes, panel_bytes;
  int64_t total;
};

RqrcpWs carve_rqrcp(void* ws, int64_t m, int64_t n, int64_t b, int64_t p, bool need_omega, bool resample) {
  const int64_t ell = b + p;
  Carve c(ws);
  RqrcpWs w;
  w.gemm = c.take<double>(kGemmWsBytes / 8);
  w.sample_bytes = sample_qrcp_workspace(ell, n);
  w.sample = c.take<char>(w.sample_bytes);
  w.panel_bytes = panel_workspace(b);
  w.panel = c.take<char>(w.panel_bytes);
  w.Bcur = c.take<double>(ell * n);
  w.Bnext = c.take<double>(ell * n);
  w.Bf = c.take<double>(ell * n);
  w.lperm = c.take<int64_t>(n);
  w.moves = c.take<int32_t>(4 * b + 8);
  w.stau = c.take<double>(b);
  w.Ypan = c.take<double>(m * 2 * b);  // [Y_P | Y_J] of a merged pair (PairedSweep)
  w.Gm = c.take<double>(b * b);
  w.Wt = c.take<double>(b * (n + 2 * b));
  w.W = c.take<double>(2 * b * n);      // [W_P ; W_J], ld 2b
  w.OmT = (need_omega || resample) ? c.take<double>(m * ell) : nullptr;
  w.pscr = c.take<double>(PanelScratch::doubles(b));
  w.snap = c.take<int32_t>(8);
  w.guard = c.take<int32_t>(8);
  w.sig = reinterpret_cast<unsigned*>(c.take<int32_t>(16));
  w.snap2 = c.take<int32_t>(8);
  w.Ypan2 = c.take<double>(m * 2 * b);
  w.total = c.off + 256;
  return w;
}

bool panel_is_block(int64_t mr, int64_t bb) {
  static const bool no_block = env_flag("SQR_NO_BLOCKPANEL");
  return !no_block && mr <= panel_block_max_rows() && bb <= 128;
}

// Panel QR (randomized.py:107-130 / reference.py:281-291) as 32-wide leaves
// on the cooperative panel kernel; between leaves the leaf's reflectors are
// applied to the rest of the panel in compact-WY form with the DMMA GEMMs:
//   [G_l | Wt] = Y_l^T [Y_l | P_rest];  T_l = build_t(G_l);  P_rest += Y_l (-T_l^T Wt).
// The panel width may be dynamic (wstat < 0: st->sample_achieved); leaves
// and WY updates never touch columns beyond it.
int panel_factor(double* P, int64_t lda, int64_t mr, int64_t bb, int64_t wstat, double* Y, int64_t ldy,
                 double* taus, int stop_at_zero, sqr_status* st, void* pws, int64_t pwsb, const PanelScratch& sc,
                 double* gws, cudaStream_t s, ResidentSig sig = {}) {
  if (panel_is_block(mr, bb))
    return panel_block(P, lda, mr, wstat, bb, Y, ldy, taus, stop_at_zero, st, pws, pwsb, s, sig);
  int rc;
  if ((rc = signal_resident_host(sig, s))) return rc;
  // 16-wide leaves when the panel needs 3-4 rows per thread (register file)
  const int64_t rows1 = (int64_t)std::min(sm_count(), 148) * 256;
  const int64_t leaf = (mr > 2 * rows1 && mr <= 4 * rows1) ? 16 : kLeaf;
  for (int64_t c0 = 0; c0 < bb; c0 += leaf) {
    const int64_t lwe = std::min(leaf, bb - c0);
    if ((rc = panel_qr(P, lda, mr, wstat, lwe, Y, ldy, taus, stop_at_zero, st, pws, pwsb, s, c0))) return rc;
    const int64_t rest = bb - (c0 + lwe);
    if (rest <= 0 || mr - c0 <= 0) continue;
    const double* Yl = Y + c0 + c0 * ldy;
    double* Prest = P + c0 + (c0 + lwe) * lda;
    const int32_t* lim = wstat < 0 ? &st->sample_achieved : nullptr;
    GemmDyn d1{&st->stop, nullptr, 0};
    d1.pre = Yl;
    d1.ldpre = ldy;
    d1.npre = (int)lwe;
    d1.limit = lim;
    d1.limit_off = (int)c0;
    const int64_t ld = kLeaf;
    if ((rc = gemm_tn(lwe, lwe + rest, mr - c0, 1.0, Yl, ldy, Prest, lda, 0.0, nullptr, 0, sc.GW, ld, gws,
                      kGemmWsBytes, s, d1)))
      return rc;
    if ((rc = build_t(sc.GW, ld, taus + c0, lwe, sc.Tl, kLeaf, &st->stop, s))) return rc;
    GemmDyn d2{&st->stop, nullptr, 0};
    d2.limit = lim;
    d2.limit_off = (int)(c0 + lwe);
    if ((rc = gemm_tn(lwe, rest, lwe, -1.0, sc.Tl, kLeaf, sc.GW + lwe * ld, ld, 0.0, nullptr, 0, sc.W, ld, gws,
                      kGemmWsBytes, s, d2)))
      return rc;
    if ((rc = gemm_nn(mr - c0, rest, lwe, 1.0, Yl, ldy, sc.W, ld, 1.0, Prest, lda, Prest, lda, s, d2))) return rc;
  }
  return SQR_OK;
}

// T of a block is built on a side stream as soon as the first sweep's Gram
// prefix is final (GemmDyn::pre_ready), beside the split-K reduction of the
// sweep's other columns (and, on merged blocks, the first-sweep correction):
// ~27 us per block off the critical path.
struct TBuild {
  cudaStream_t side = nullptr;
  cudaEvent_t pre = nullptr, done = nullptr;
  ~TBuild() {
    if (pre) cudaEventDestroy(pre);
    if (done) cudaEventDestroy(done);
    if (side) cudaStreamDestroy(side);
  }
  int init() {
    int lo = 0, hi = 0;
    SQR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SQR_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    SQR_CUDA(cudaEventCreateWithFlags(&pre, cudaEventDisableTiming));
    SQR_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    return SQR_OK;
  }
  // T = build_t(G, taus) on the side stream once `pre` has fired
  int build(const double* G, int64_t ldg, const double* taus, int64_t bb, double* T, int64_t ldt, sqr_status* st) {
    SQR_CUDA(cudaStreamWaitEvent(side, pre, 0));
    const int rc = build_t(G, ldg, taus, bb, T, ldt, &st->stop, side);
    if (rc) return rc;
    SQR_CUDA(cudaEventRecord(done, side));
    return SQR_OK;
  }
  int join(cudaStream_t s) {
    SQR_CUDA(cudaStreamWaitEvent(s, done, 0));
    return SQR_OK;
  }
};

// One compact-WY block reflection of the trailing matrix (randomized.py:203-210)
// plus the block's T (householder.py:52-61):
//   [G | Wt] = Y^T [Y | C]     one sweep; G = Y^T Y is free next to Y^T C
//   T        = build_t(G, tau)
//   W        = -T^T Wt;   C += Y W,
// with C starting bhat columns right of P (device-side shift).
int trailing_update(double* P, int64_t lda, int64_t mr, int64_t nt, int64_t bb, const double* Y,
                    int64_t ldy, const double* taus, double* T, int64_t ldt, double* GWt, double* W,
                    int64_t ldw, sqr_status* st, double* gws, cudaStream_t s, bool skip_pass2 = false) {
  GemmDyn d1{&st->stop, &st->bhat, kShiftB};
  d1.pre = Y;
  d1.ldpre = ldy;
  d1.npre = (int)bb;
  GemmDyn d2{&st->stop, &st->bhat, 0};
  GemmDyn d3{&st->stop, &st->bhat, kShiftD};
  int rc = gemm_tn(bb, bb + nt, mr, 1.0, Y, ldy, P, lda, 0.0, nullptr, 0, GWt, ldw, gws, kGemmWsBytes, s, d1);
  if (rc) return rc;
  if ((rc = build_t(GWt, ldw, taus, bb, T, ldt, &st->stop, s))) return rc;
  if (nt <= 1) return SQR_OK;
  const double* Wt = GWt + bb * ldw;
  rc = gemm_tn(bb, nt, bb, -1.0, T, ldt, Wt, ldw, 0.0, nullptr, 0, W, ldw, gws, kGemmWsBytes, s, d2);
  if (rc || skip_pass2) return rc;
  return gemm_nn(mr, nt, bb, 1.0, Y, ldy, W, ldw, 1.0, P, lda, P, lda, s, d3);
}

// Paired second sweep.  The reference applies every block reflection to the
// trailing matrix in two sweeps (randomized.py:203-207): Y^T C (long K =
// m - i0, ~93% of the fp64 tensor pipe) and C -= Y W (K = b = 128, ~84%:
// the short-K rank-b update is prologue/epilogue heavy).  Blocks are paired
// (P = 2q, J = 2q + 1) and P's second sweep is merged into J's, so the bulk
// rank update runs once per pair with K = 2b (33.5 vs 31.1 TFLOP/s on the C5
// shape, tools/nn_k_probe.py).  Arithmetic per column is unchanged:
//   P: [G|Wt] = Y_P^T [Y_P|C];  W_P = -T_P^T Wt;  only the R12 rows
//      C[0:b] += Y_P[0:b] W_P are applied (the sample update needs them);
//   J: sample QRCP on the updated sample; moves act on C and W_P alike;
//      the J panel columns get P's update (C_pan += Y_P W_P, then those W_P
//      columns are zeroed); panel;
//      [Y_J^T Y_P | G | Wt] = Y_J^T [Y_P | Y_J | C]  (one sweep, C lacking P),
//      Wt += (Y_J^T Y_P) W_P  (so Wt = Y_J^T (C + Y_P W_P) exactly as if P had
//      been applied), W_J = -T_J^T Wt, and finally
//      C[b:] += [Y_P | Y_J] [W_P ; W_J]  with K = 2b.
// Rows of Y are global rows offset by the pair's i0; Y_J sits in columns
// [b, 2b) of Ycat with its first b rows zero.
int trailing_first(double* P, int64_t lda, int64_t mr, int64_t nt, int64_t bb, const double* Ycat, int64_t ldy,
                   const double* taus, double* T, int64_t ldt, double* GWt, int64_t ldw, double* Wcat,
                   int64_t ldwc, sqr_status* st, double* gws, cudaStream_t s, TBuild* tb = nullptr) {
  GemmDyn d1{&st->stop, &st->bhat, kShiftB};
  d1.pre = Ycat;
  d1.ldpre = ldy;
  d1.npre = (int)bb;
  if (tb) d1.pre_ready = tb->pre;
  int rc = gemm_tn(bb, bb + nt, mr, 1.0, Ycat, ldy, P, lda, 0.0, nullptr, 0, GWt, ldw, gws, kGemmWsBytes, s, d1);
  if (rc) return rc;
  if (tb) {
    if ((rc = tb->build(GWt, ldw, taus, bb, T, ldt, st)) || (rc = tb->join(s))) return rc;
  } else if ((rc = build_t(GWt, ldw, taus, bb, T, ldt, &st->stop, s))) {
    return rc;
  }
  if (nt <= 1) return SQR_OK;
  // W_P (relative to column bhat_P = b: to i0_J), then the R12 rows only
  rc = gemm_tn(bb, nt, bb, -1.0, T, ldt, GWt + bb * ldw, ldw, 0.0, nullptr, 0, Wcat, ldwc, gws, kGemmWsBytes, s,
               GemmDyn{&st->stop, &st->bhat, 0});
  if (rc) return rc;
  return gemm_nn(bb, nt, bb, 1.0, Ycat, ldy, Wcat, ldwc, 1.0, P, lda, P, lda, s,
                 GemmDyn{&st->stop, &st->bhat, kShiftD});
}

// J's update of the panel columns by the pending P, before J's panel (the
// columns [0, sample_achieved) only; their W_P columns are then retired).
int pending_panel_update(double* P, int64_t lda, int64_t mr, int64_t bb, int64_t b, const double* Ycat,
                         int64_t ldy, double* Wcat, int64_t ldwc, sqr_status* st, cudaStream_t s) {
  GemmDyn d{&st->stop, nullptr, 0};
  d.limit = &st->sample_achieved;
  int rc = gemm_nn(mr, bb, b, 1.0, Ycat + b, ldy, Wcat, ldwc, 1.0, P, lda, P, lda, s, d);
  if (rc) return rc;
  return zero_columns(Wcat, ldwc, b, bb, &st->sample_achieved, &st->stop, s);
}

int trailing_second(double* P, int64_t lda, int64_t mr, int64_t nt, int64_t bb, int64_t b, const double* Ycat,
                    int64_t ldy, const double* taus, double* T, int64_t ldt, double* GWt, int64_t ldw,
                    double* Wcat, int64_t ldwc, sqr_status* st, double* gws, cudaStream_t s,
                    bool skip_merged = false, TBuild* tb = nullptr) {
  const double* Yj = Ycat + b * ldy + b;  // rows from i0_J
  GemmDyn d1{&st->stop, &st->bhat, kShiftB};
  d1.pre = Ycat + b;  // [Y_P | Y_J] rows from i0_J
  d1.ldpre = ldy;
  d1.npre = (int)(b + bb);
  if (tb) d1.pre_ready = tb->pre;
  int rc = gemm_tn(bb, b + bb + nt, mr, 1.0, Yj, ldy, P, lda, 0.0, nullptr, 0, GWt, ldw, gws, kGemmWsBytes, s, d1);
  if (rc) return rc;
  if (tb) {
    if ((rc = tb->build(GWt + b * ldw, ldw, taus, bb, T, ldt, st))) return rc;
  } else if ((rc = build_t(GWt + b * ldw, ldw, taus, bb, T, ldt, &st->stop, s))) {
    return rc;
  }
  if (nt <= 1) return tb ? tb->join(s) : SQR_OK;
  double* Wt = GWt + (b + bb) * ldw;
  rc = gemm_nn(bb, nt, b, 1.0, GWt, ldw, Wcat, ldwc, 1.0, Wt, ldw, Wt, ldw, s,
               GemmDyn{&st->stop, &st->bhat, kShiftB});
  if (rc) return rc;
  if (tb && (rc = tb->join(s))) return rc;  // T beside the reduction and the correction above
  rc = gemm_tn(bb, nt, bb, -1.0, T, ldt, Wt, ldw, 0.0, nullptr, 0, Wcat + b, ldwc, gws, kGemmWsBytes, s,
               GemmDyn{&st->stop, &st->bhat, kShiftD});
  if (rc || skip_merged) return rc;
  return gemm_nn(mr, nt, b + bb, 1.0, Ycat + b, ldy, Wcat, ldwc, 1.0, P, lda, P, lda, s,
                 GemmDyn{&st->stop, &st->bhat, kShiftB | kShiftD});
}

// Lookahead schedule of one block's second sweep (randomized.py:207-221):
// the R12 rows [0, bb) are updated first; then the bulk rows [bb, mr) run on
// the caller's stream while a high-priority side stream finishes the block
// (finish_block, sample update, next block's sample QRCP), which only reads
// R11/R12 and the sample.  The bulk GEMM gates on a snapshot of {stop, bhat}
// so the side stream's status writes cannot reach it.
struct Lookahead {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool on = false;
  ~Lookahead() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
  }
  int init() {
    // Opt-in (SQR_LOOKAHEAD=1): measured +1.1% on C5, because the side
    // stream's cooperative kernels need whole SMs and so mostly serialise
    // against the bulk GEMM anyway; off by default so per-kernel timings
    // (roofline) are not inflated by the overlap.
    static const bool enabled = [] {
      const char* e = getenv("SQR_LOOKAHEAD");
      return e && *e && *e != '0';
    }();
    if (!enabled) return SQR_OK;
    int lo = 0, hi = 0;
    SQR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SQR_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    SQR_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    SQR_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    on = true;
    return SQR_OK;
  }
};

// Chain / bulk overlap of the paired schedule.  The chain kernels (sample
// QRCP, panel) are latency-bound and hold their working set on chip: each of
// their CTAs takes a whole SM, but only ceil(n_t / 256) (sample) or
// ceil(m_r / 256) (panel) SMs -- the rest of the chip idles for ~1.2 ms per
// block.  The merged second sweep of a pair (the bulk rows below the R12
// rows, randomized.py:207) is therefore split by rows around the next
// block's chain:
//   R12 rows -> finish_block -> sample update
//   { next sample QRCP  ||  bulk rows A }          next pivots known
//   column moves on C and on [W_P ; W_J]; the next panel's columns get the
//   pair's update in rows B from their own K = 2b GEMM
//   { next panel        ||  bulk rows B of the other columns }
// Each chain kernel goes first (high-priority stream; the GEMM's stream is
// held until the kernel reports all CTAs resident, ResidentSig), the GEMM's
// CTAs fill the SMs it leaves free and spread over the chip when it ends.
// Per entry the arithmetic is that of the single merged sweep (same K order;
// the early rows below apply P and J one after the other, as the reference
// does).  The bulk GEMMs gate on a snapshot of {stop, bhat} taken before
// finish_block, like Lookahead.
struct Overlap {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  unsigned epoch = 0;
  ~Overlap() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
  }
  int init() {
    int lo = 0, hi = 0;
    SQR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SQR_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    SQR_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    SQR_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    return SQR_OK;
  }
  int fork_from(cudaStream_t s) {
    SQR_CUDA(cudaEventRecord(fork, s));
    SQR_CUDA(cudaStreamWaitEvent(side, fork, 0));
    return SQR_OK;
  }
  int mark_join() {
    SQR_CUDA(cudaEventRecord(join, side));
    return SQR_OK;
  }
  int join_to(cudaStream_t s) {
    SQR_CUDA(cudaStreamWaitEvent(s, join, 0));
    return SQR_OK;
  }
};
// bulk rows of a pair still to be applied when the next block starts
struct OverlapCarry {
  bool on = false;
  int64_t i0p = 0, bbp = 0, mrp = 0, rB = 0;  // the merging block's i0 / width / rows; first row of part B
  int64_t koff = 0;                           // b when rows B already hold P's update (early rows): K = bbp
  const double* Ycat = nullptr;               // the pair's [Y_P | Y_J]
};
// The second block's chain is hidden the same way behind the pair's FIRST
// block: while its sample QRCP runs, the bottom rows [ra, mr) of P's own
// second sweep are applied (K = b, every trailing column, before the column
// moves), and Y_P's rows there are zeroed -- so the pending panel update, the
// corrected first sweep (prefix Gram over the remaining rows only) and a
// K = 2b sweep would all skip them by themselves; the merged sweep then runs
// K = 2b above ra (beside the next sample QRCP) and K = b, Y_J only, below
// (beside the next panel).  ra is sized to the SMs the sample QRCP leaves.
struct EarlyRows {
  bool sample_launched = false;  // the second block's sample QRCP is already on the side stream
  int64_t ra = 0;                // first early row relative to the second block's i0 (0 = none)
};
constexpr double kEarlyRowsWork2 = 1.1 * 31.4e12 * 0.53e-3 / 2.0;  // ... one panel hides
// rows of P's second sweep to run beside the second block's panel (0 = none)
inline int64_t early_rows2(int64_t mr, int64_t nt, int64_t bb, int64_t b, int64_t ra) {
  static const bool off = env_flag("SQR_NO_EARLY_ROWS2");
  if (off || nt - bb <= 0) return 0;
  const int64_t sms = sm_count(), free_sms = std::max<int64_t>(0, sms - cdiv(mr, 256));
  int64_t a2 = (int64_t)(kEarlyRowsWork2 * (double)free_sms / (double)sms / (double)(b * (nt - bb))) / 64 * 64;
  static const bool force = env_flag("SQR_OVERLAP_FORCE");
  if (force) a2 = std::max<int64_t>(a2, 64);
  a2 = std::min(a2, (ra - bb) / 2 / 64 * 64);  // leave rows for the K = 2b part beside the next sample QRCP
  return a2 < (force ? 64 : 256) ? 0 : a2;
}
constexpr double kEarlyRowsWork = 1.0 * 31.4e12 * 0.66e-3 / 2.0;  // row x column x K products one sample QRCP hides
constexpr int kResidentTimeoutUs = 100;

// M = S11 R11^-1 and the R11 guard of the sample update (sketch.py:132-149,
// randomized.py:217-219) depend only on the block's factored sample and its
// R11, both final right after the panel: they run on a high-priority side
// stream concurrently with the trailing update (16 CTAs next to the GEMM)
// instead of on the critical path between the update and the next sample
// QRCP.  The guard verdict goes to a separate word that finish_block folds
// into st->stop after the update, as the reference orders it.
struct EarlyPrep {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~EarlyPrep() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
  }
  int init() {
    int lo = 0, hi = 0;
    SQR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SQR_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    SQR_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    SQR_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    return SQR_OK;
  }
  int launch(const double* Bf, int64_t ldbf, const double* R, int64_t ldr, int64_t bb, double* mbuf,
             sqr_status* st, int32_t* guard, cudaStream_t s) {
    SQR_CUDA(cudaEventRecord(fork, s));
    SQR_CUDA(cudaStreamWaitEvent(side, fork, 0));
    const int rc = su_prep(Bf, ldbf, R, ldr, bb, mbuf, st, guard, side);
    if (rc) return rc;
    SQR_CUDA(cudaEventRecord(join, side));
    return SQR_OK;
  }
  int wait(cudaStream_t s) {
    SQR_CUDA(cudaStreamWaitEvent(s, join, 0));
    return SQR_OK;
  }
};

int pass2_split(double* P, int64_t lda, int64_t mr, int64_t nt, int64_t bb, const double* Y, int64_t ldy,
                const double* W, int64_t ldw, sqr_status* st, int32_t* snap, cudaStream_t s, cudaEvent_t fork) {
  SQR_CUDA(cudaMemcpyAsync(snap, st, 6 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  GemmDyn d3{&snap[0], &snap[5], kShiftD};
  const int64_t top = std::min(bb, mr);
  int rc = gemm_nn(top, nt, bb, 1.0, Y, ldy, W, ldw, 1.0, P, lda, P, lda, s, d3);
  if (rc) return rc;
  SQR_CUDA(cudaEventRecord(fork, s));
  if (mr > top) rc = gemm_nn(mr - top, nt, bb, 1.0, Y + top, ldy, W, ldw, 1.0, P + top, lda, P + top, lda, s, d3);
  return rc;
}

}  // namespace
}  // namespace sqr

using namespace sqr;
static_assert(sizeof(sqr_status) == 72, "sqr_status layout is part of the ABI");

extern "C" int64_t sqr_rqrcp_workspace(int64_t m, int64_t n, int64_t /*k*/, int64_t b, int64_t p) {
  return carve_rqrcp(nullptr, m, n, b, p, true, true).total;
}

namespace sqr {
namespace {
// Streams the finished R columns to pinned host memory while later blocks run.
// Column block [i0, i0+bb) never changes after its block's trailing update
// (later column moves only touch columns >= the next block), so right after
// that update its rows above the block go out with one 2D copy and its
// diagonal block, with the reflector tails zeroed, through a per-block
// staging slot.
struct RSink {
  double* host = nullptr;
  int64_t ldh = 0;
  double* stage = nullptr;  // nblk x b x b
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  ~RSink() {
    if (ev) cudaEventDestroy(ev);
    if (cs) cudaStreamDestroy(cs);
  }
  int init(double* h, int64_t l, double* st) {
    host = h;
    ldh = l;
    stage = st;
    if (!host) return SQR_OK;
    SQR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SQR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    return SQR_OK;
  }
  int block(const double* A, int64_t lda, int64_t i0, int64_t bb, int64_t b, int64_t J, cudaStream_t s) {
    if (!host) return SQR_OK;
    double* slot = stage + J * b * b;
    int rc = copy_upper(A + i0 + i0 * lda, lda, slot, bb, bb, nullptr, s);
    if (rc) return rc;
    SQR_CUDA(cudaEventRecord(ev, s));
    SQR_CUDA(cudaStreamWaitEvent(cs, ev, 0));
    if (i0 > 0)
      SQR_CUDA(cudaMemcpy2DAsync(host + i0 * ldh, ldh * 8, A + i0 * lda, lda * 8, i0 * 8, bb,
                                 cudaMemcpyDeviceToHost, cs));
    SQR_CUDA(cudaMemcpy2DAsync(host + i0 + i0 * ldh, ldh * 8, slot, bb * 8, bb * 8, bb, cudaMemcpyDeviceToHost,
                               cs));
    return SQR_OK;
  }
  // rows [0, rows) of the columns [c0, n) left of no block (truncated runs), then join
  int finish(const double* A, int64_t lda, int64_t rows, int64_t c0, int64_t n, cudaStream_t s) {
    if (!host) return SQR_OK;
    if (c0 < n && rows > 0) {
      SQR_CUDA(cudaEventRecord(ev, s));
      SQR_CUDA(cudaStreamWaitEvent(cs, ev, 0));
      SQR_CUDA(cudaMemcpy2DAsync(host + c0 * ldh, ldh * 8, A + c0 * lda, lda * 8, rows * 8, n - c0,
                                 cudaMemcpyDeviceToHost, cs));
    }
    SQR_CUDA(cudaEventRecord(ev, cs));
    SQR_CUDA(cudaStreamWaitEvent(s, ev, 0));
    return SQR_OK;
  }
};

int rqrcp_impl(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p, uint64_t seed,
               const double* omegaT, int64_t ldo, int resample, int64_t* perm, double* taus, double* T,
               sqr_status* st, void* workspace, int64_t workspace_bytes, double* R_host, int64_t ldrh,
               cudaStream_t s) {
  const int64_t ell = b + p;
  if (m <= 0 || n <= 0 || k < 1 || k > std::min(m, n) || b < 1 || p < 0 || ell >= m || lda < m) {
    set_error("sqr_rqrcp: invalid arguments m=%lld n=%lld k=%lld b=%lld p=%lld", (long long)m, (long long)n,
              (long long)k, (long long)b, (long long)p);
    return SQR_EINVAL;
  }
  if (b > 128 || ell > 144) {
    set_error("sqr_rqrcp: b=%lld / l=%lld exceed the kernel limits (b<=128, b+p<=144)", (long long)b,
              (long long)ell);
    return SQR_EINVAL;
  }
  RqrcpWs w = carve_rqrcp(workspace, m, n, b, p, omegaT == nullptr, resample != 0);
  const int64_t stage_bytes = R_host ? cdiv(k, b) * b * b * 8 : 0;
  if (workspace == nullptr || workspace_bytes < w.total + stage_bytes) {
    set_error("sqr_rqrcp: workspace %lld < %lld bytes", (long long)workspace_bytes,
              (long long)(w.total + stage_bytes));
    return SQR_EINVAL;
  }
  RSink sink;
  int rcs = sink.init(R_host, ldrh, reinterpret_cast<double*>(static_cast<char*>(workspace) + w.total));
  if (rcs) return rcs;
  SQR_CUDA(cudaMemsetAsync(st, 0, sizeof(sqr_status), s));
  int rc = iota(perm, n, s);
  if (rc) return rc;
  if (omegaT == nullptr) {
    rc = gaussian(w.OmT, m, ell, m, seed, 0, 1, nullptr, s);
    if (rc) return rc;
    omegaT = w.OmT;
    ldo = m;
  }
  // Sketch B = Omega A (sketch.py:70-71).
  rc = gemm_tn(ell, n, m, 1.0, omegaT, ldo, A, lda, 0.0, nullptr, 0, w.Bcur, ell, w.gemm, kGemmWsBytes, s,
               GemmDyn{});
  if (rc) return rc;
  uint64_t stream_pos = (uint64_t)(ell * m);
  const int64_t nblk = cdiv(k, b);
  double* Bc = w.Bcur;
  double* Bn = w.Bnext;
  Lookahead la;
  if (!resample && (rc = la.init())) return rc;
  static const bool no_pair = env_flag("SQR_NO_PAIRED_SWEEP");
  const bool pair = !resample && !la.on && !no_pair;
  static const bool no_early = env_flag("SQR_NO_EARLY_PREP");
  EarlyPrep ep;
  const bool early = !resample && !la.on && !no_early;
  if (early && (rc = ep.init())) return rc;
  static const bool no_overlap = env_flag("SQR_NO_OVERLAP");
  const bool overlap = pair && !no_overlap;
  Overlap ov;
  OverlapCarry cy;
  EarlyRows er;
  TBuild tb;
  static const bool no_tside = env_flag("SQR_NO_T_SIDE");
  TBuild* tbp = (pair && !no_tside) ? &tb : nullptr;
  if (tbp && (rc = tb.init())) return rc;
  static const bool no_early_rows = env_flag("SQR_NO_EARLY_ROWS");
  static const bool force_overlap = env_flag("SQR_OVERLAP_FORCE");
  auto will_split = [&](int64_t Jn) {  // the merged sweep of second block Jn runs split around the next chain
    const int64_t i0n = Jn * b, bbn = std::min(b, k - i0n), ntn = n - i0n, mrn = m - i0n, topn = std::min(bbn, mrn);
    // worth it while the bulk rows outlast the chain kernels they hide (SQR_OVERLAP_FORCE: any size, tests),
    // and those leave an SM for the waiting thread
    const bool big = force_overlap ? mrn - topn >= 1
                                   : mrn - topn >= 1024 && (mrn - topn) * (ntn - bbn) >= (int64_t)3 << 22;
    const int64_t fit = (int64_t)(sm_count() - 1) * 256;  // chain kernels: 256 columns / rows per SM
    return overlap && (Jn & 1) && Jn + 1 < nblk && ntn > 1 && big && ntn - bbn <= fit && mrn - bbn <= fit;
  };
  if (overlap) {
    if ((rc = ov.init())) return rc;
    SQR_CUDA(cudaMemsetAsync(w.sig, 0, 64, s));
  }
  if (pair) {  // Y_J's zero top rows
    SQR_CUDA(cudaMemset2DAsync(w.Ypan + b * m, m * 8, 0, b * 8, b, s));
    if (overlap) SQR_CUDA(cudaMemset2DAsync(w.Ypan2 + b * m, m * 8, 0, b * 8, b, s));
  }
  for (int64_t J = 0; J < nblk; ++J) {
    const int64_t i0 = J * b, bb = std::min(b, k - i0), nt = n - i0, mr = m - i0;
    double* P = A + i0 + i0 * lda;
    double* TJ = T + J * b * b;
    const bool second = pair && (J & 1);                      // merges the pending block J-1
    const bool first = pair && !(J & 1) && J + 1 < nblk;      // second sweep deferred to J+1
    double* Ypair = (overlap && ((J >> 1) & 1)) ? w.Ypan2 : w.Ypan;  // this pair's [Y_P | Y_J]
    double* Yj = second ? Ypair + b * m + b : Ypair;          // ld m, rows from i0
    if (cy.on || er.sample_launched) {
      if ((rc = ov.join_to(s))) return rc;  // the sample QRCP launched behind the previous block's R12 rows
      er.sample_launched = false;
    } else if ((J == 0 || !la.on) &&
               (rc = sample_qrcp(Bc, ell, ell, nt, bb, w.Bf, ell, w.lperm, w.moves, w.stau, J == 0, st, w.sample,
                                 w.sample_bytes, s)))
      return rc;
    // the moves of the pending W rows (a few KB, latency-bound) beside the moves of A
    const bool wside = overlap && (second || cy.on);
    if (wside) {
      if ((rc = ov.fork_from(s))) return rc;
      const int64_t wrows = second ? b : b + cy.bbp - cy.koff;
      double* Wmv = second ? w.W : w.W + cy.bbp * 2 * b + cy.koff;
      if ((rc = apply_moves(Wmv, 2 * b, wrows, 0, nullptr, w.moves, st, 2 * bb, ov.side))) return rc;
      if ((rc = ov.mark_join())) return rc;
    }
    if ((rc = apply_moves(A, lda, m, i0, perm, w.moves, st, 2 * bb, s))) return rc;
    if (wside && (rc = ov.join_to(s))) return rc;
    if (second) {
      if (!wside && (rc = apply_moves(w.W, 2 * b, b, 0, nullptr, w.moves, st, 2 * bb, s))) return rc;
      if ((rc = pending_panel_update(P, lda, mr, bb, b, Ypair, m, w.W, 2 * b, st, s))) return rc;
    }
    PanelScratch sc{w.pscr, w.pscr + kLeaf * (kLeaf + b), w.pscr + kLeaf * (kLeaf + b) + kLeaf * b};
    if (cy.on) {
      // Rows B of the previous pair's merged sweep (see Overlap): W follows
      // the moves, the panel columns are updated on their own, the panel
      // runs beside the update of the other columns.
      cy.on = false;
      const int64_t kk = b + cy.bbp - cy.koff, mB = cy.mrp - cy.rB;
      double* Wm = w.W + cy.bbp * 2 * b + cy.koff;  // column i0 of A (its moves ran beside A's above)
      const double* YB = cy.Ycat + b + cy.rB + cy.koff * m;
      double* PB = A + (cy.i0p + cy.rB) + i0 * lda;
      const GemmDyn dsn{&w.snap[0], nullptr, 0};
      if (mB > 0 && (rc = gemm_nn(mB, bb, kk, 1.0, YB, m, Wm, 2 * b, 1.0, PB, lda, PB, lda, s, dsn))) return rc;
      if ((rc = ov.fork_from(s))) return rc;
      const ResidentSig sig{w.sig, ++ov.epoch};
      if ((rc = panel_factor(P, lda, mr, bb, -1, Yj, m, taus + i0, 1, st, w.panel, w.panel_bytes, sc, w.gemm,
                             ov.side, sig)))
        return rc;
      if ((rc = ov.mark_join())) return rc;
      if (mB > 0 && nt - bb > 0) {
        if ((rc = wait_resident(sig, kResidentTimeoutUs, s))) return rc;
        GemmDyn dsb = dsn;
        dsb.prof_tag = kTagGemmNnBeside;
        prof_add_flops(kTagGemmNnBeside, 2.0 * mB * (nt - bb) * kk);
        if ((rc = gemm_nn(mB, nt - bb, kk, 1.0, YB, m, Wm + bb * 2 * b, 2 * b, 1.0, PB + bb * lda, lda,
                          PB + bb * lda, lda, s, dsb)))
          return rc;
      }
      if ((rc = ov.join_to(s))) return rc;
    } else if (second && er.ra > 0 && panel_is_block(mr, bb) && early_rows2(mr, nt, bb, b, er.ra) > 0) {
      // the panel beside more of P's second sweep: the rows just above the
      // early rows, columns right of the panel (whose rows the pending update
      // above has already covered); Y_P's rows there are retired too
      const int64_t a2 = early_rows2(mr, nt, bb, b, er.ra), ra2 = er.ra - a2;
      SQR_CUDA(cudaMemcpyAsync(w.snap2, st, 6 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      if ((rc = ov.fork_from(s))) return rc;
      const ResidentSig sig{w.sig, ++ov.epoch};
      if ((rc = panel_factor(P, lda, mr, bb, -1, Yj, m, taus + i0, 1, st, w.panel, w.panel_bytes, sc, w.gemm,
                             ov.side, sig)))
        return rc;
      if ((rc = ov.mark_join())) return rc;
      if ((rc = wait_resident(sig, kResidentTimeoutUs, s))) return rc;
      double* Pa = P + ra2 + bb * lda;
      GemmDyn da{&w.snap2[0], nullptr, 0};
      da.prof_tag = kTagGemmNnBeside;
      prof_add_flops(kTagGemmNnBeside, 2.0 * a2 * (nt - bb) * b);
      if ((rc = gemm_nn(a2, nt - bb, b, 1.0, Ypair + b + ra2, m, w.W + bb * 2 * b, 2 * b, 1.0, Pa, lda, Pa, lda, s, da)))
        return rc;
      SQR_CUDA(cudaMemset2DAsync(Ypair + b + ra2, m * 8, 0, a2 * 8, b, s));
      if ((rc = ov.join_to(s))) return rc;
      er.ra = ra2;
    } else if ((rc = panel_factor(P, lda, mr, bb, -1, Yj, m, taus + i0, 1, st, w.panel, w.panel_bytes, sc, w.gemm,
                                  s)))
      return rc;
    const bool prep = early && J + 1 < nblk && nt - bb > 0;
    if (prep && (rc = ep.launch(w.Bf, ell, P, lda, bb, w.Gm, st, w.guard, s))) return rc;
    if (la.on) {
      // Second sweep split around the side stream (see Lookahead).
      if ((rc = trailing_update(P, lda, mr, nt, bb, w.Ypan, m, taus + i0, TJ, b, w.Wt, w.W, b, st, w.gemm, s,
                                true)))
        return rc;
      if (nt > 1 && (rc = pass2_split(P, lda, mr, nt, bb, w.Ypan, m, w.W, b, st, w.snap, s, la.fork))) return rc;
      if (nt <= 1) SQR_CUDA(cudaEventRecord(la.fork, s));
      if ((rc = sink.block(A, lda, i0, bb, b, J, s))) return rc;
      cudaStream_t s2 = la.side;
      SQR_CUDA(cudaStreamWaitEvent(s2, la.fork, 0));
      if ((rc = finish_block(st, nullptr, (int)i0, (int)bb, (int)k, (int)n, s2))) return rc;
      if (J + 1 < nblk) {
        std::swap(Bc, Bn);
        if ((rc = sample_update(w.Bf, ell, ell, P, lda, nt - bb, bb, Bc, ell, st, w.Gm, s2))) return rc;
        if ((rc = sample_qrcp(Bc, ell, ell, nt - bb, std::min(b, k - i0 - b), w.Bf, ell, w.lperm, w.moves, w.stau,
                              false, st, w.sample, w.sample_bytes, s2)))
          return rc;
      }
      SQR_CUDA(cudaEventRecord(la.join, s2));
      SQR_CUDA(cudaStreamWaitEvent(s, la.join, 0));
      continue;
    }
    const int64_t top = std::min(bb, mr);
    const bool split = will_split(J);
    if (first)
      rc = trailing_first(P, lda, mr, nt, bb, Ypair, m, taus + i0, TJ, b, w.Wt, b, w.W, 2 * b, st, w.gemm, s, tbp);
    else if (second)
      rc = trailing_second(P, lda, mr, nt, bb, b, Ypair, m, taus + i0, TJ, b, w.Wt, b, w.W, 2 * b, st, w.gemm, s,
                           split, tbp);
    else
      rc = trailing_update(P, lda, mr, nt, bb, Ypair, m, taus + i0, TJ, b, w.Wt, w.W, b, st, w.gemm, s);
    if (rc) return rc;
    if (split) {
      // R12 rows of the merged sweep now, the bulk rows around the next chain.
      SQR_CUDA(cudaMemcpyAsync(w.snap, st, 6 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      const GemmDyn dm{&w.snap[0], &w.snap[5], kShiftB | kShiftD};
      if ((rc = gemm_nn(top, nt, b + bb, 1.0, Ypair + b, m, w.W, 2 * b, 1.0, P, lda, P, lda, s, dm))) return rc;
      if ((rc = sink.block(A, lda, i0, bb, b, J, s))) return rc;
      if (prep && (rc = ep.wait(s))) return rc;
      if ((rc = finish_block(st, nullptr, (int)i0, (int)bb, (int)k, (int)n, s, prep ? w.guard : nullptr))) return rc;
      if ((rc = sample_update(w.Bf, ell, ell, P, lda, nt - bb, bb, Bn, ell, st, w.Gm, s, prep))) return rc;
      std::swap(Bc, Bn);
      if ((rc = ov.fork_from(s))) return rc;
      const ResidentSig sig{w.sig, ++ov.epoch};
      if ((rc = sample_qrcp(Bc, ell, ell, nt - bb, std::min(b, k - i0 - bb), w.Bf, ell, w.lperm, w.moves, w.stau, 0,
                            st, w.sample, w.sample_bytes, ov.side, sig)))
        return rc;
      if ((rc = ov.mark_join())) return rc;
      if ((rc = wait_resident(sig, kResidentTimeoutUs, s))) return rc;
      const int64_t rB = er.ra > 0 ? er.ra : std::min(mr, top + rup((mr - top) / 2, 64));
      GemmDyn dma = dm;
      dma.prof_tag = kTagGemmNnBeside;
      prof_add_flops(kTagGemmNnBeside, 2.0 * (rB - top) * (nt - bb) * (b + bb));
      if (rB > top && (rc = gemm_nn(rB - top, nt, b + bb, 1.0, Ypair + b + top, m, w.W, 2 * b, 1.0, P + top, lda,
                                    P + top, lda, s, dma)))
        return rc;
      cy.on = true;
      cy.i0p = i0;
      cy.bbp = bb;
      cy.mrp = mr;
      cy.rB = rB;
      cy.koff = er.ra > 0 ? b : 0;
      cy.Ycat = Ypair;
      er.ra = 0;
      continue;
    }
    // R columns [i0, i0+bb) go out only now: a short panel (bhat < bb) leaves
    // columns [i0+bhat, i0+bb) in the trailing matrix, whose R rows
    // [i0, i0+bhat) the update above has just rewritten (randomized.py:203-213).
    if ((rc = sink.block(A, lda, i0, bb, b, J, s))) return rc;
    if (prep && (rc = ep.wait(s))) return rc;
    int64_t early_rows = 0;
    if (first && !no_early_rows && will_split(J + 1)) {
      const int64_t ntj = nt - bb, mrj = mr - bb, sms = sm_count();
      const int64_t free_sms = std::max<int64_t>(0, sms - cdiv(ntj, 256));
      early_rows = (int64_t)(kEarlyRowsWork * (double)free_sms / (double)sms / (double)(b * ntj)) / 64 * 64;
      if (force_overlap) early_rows = std::max<int64_t>(early_rows, 64);
      early_rows = std::min(early_rows, (mrj - b) * 6 / 10 / 64 * 64);
      if (early_rows < (force_overlap ? 64 : 256)) early_rows = 0;
      if (early_rows) SQR_CUDA(cudaMemcpyAsync(w.snap2, st, 6 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
    if ((rc = finish_block(st, nullptr, (int)i0, (int)bb, (int)k, (int)n, s, prep ? w.guard : nullptr))) return rc;
    if (early_rows) {
      // the second block's sample QRCP beside P's own second sweep on the bottom rows (see EarlyRows)
      if ((rc = sample_update(w.Bf, ell, ell, P, lda, nt - bb, bb, Bn, ell, st, w.Gm, s, prep))) return rc;
      std::swap(Bc, Bn);
      if ((rc = ov.fork_from(s))) return rc;
      const ResidentSig sig{w.sig, ++ov.epoch};
      if ((rc = sample_qrcp(Bc, ell, ell, nt - bb, std::min(b, k - i0 - bb), w.Bf, ell, w.lperm, w.moves, w.stau, 0,
                            st, w.sample, w.sample_bytes, ov.side, sig)))
        return rc;
      if ((rc = ov.mark_join())) return rc;
      if ((rc = wait_resident(sig, kResidentTimeoutUs, s))) return rc;
      const int64_t ra = mr - early_rows;  // relative to i0
      GemmDyn de{&w.snap2[0], &w.snap2[5], kShiftD};
      de.prof_tag = kTagGemmNnBeside;
      prof_add_flops(kTagGemmNnBeside, 2.0 * early_rows * (nt - bb) * bb);
      if ((rc = gemm_nn(early_rows, nt, bb, 1.0, Ypair + ra, m, w.W, 2 * b, 1.0, P + ra, lda, P + ra, lda, s, de)))
        return rc;
      SQR_CUDA(cudaMemset2DAsync(Ypair + ra, m * 8, 0, early_rows * 8, bb, s));
      er.sample_launched = true;
      er.ra = ra - bb;
      continue;
    }
    if (J + 1 < nblk) {
      const int64_t a1 = i0 + bb;  // achieved if the block completed
      if (resample) {
        // Fresh draw of the trailing sample (randomized.py:214-215; rng.py:85-93).
        if ((rc = gaussian(w.OmT, m - a1, ell, m - a1, seed, stream_pos, 1, &st->stop, s))) return rc;
        if ((rc = gemm_tn(ell, n - a1, m - a1, 1.0, w.OmT, m - a1, A + a1 + a1 * lda, lda, 0.0, nullptr, 0, Bn,
                          ell, w.gemm, kGemmWsBytes, s, GemmDyn{&st->stop, nullptr, 0})))
          return rc;
        stream_pos += (uint64_t)(ell * (m - a1));
      } else {
        if ((rc = sample_update(w.Bf, ell, ell, P, lda, nt - bb, bb, Bn, ell, st, w.Gm, s, prep))) return rc;
      }
      std::swap(Bc, Bn);
    }
  }
  return sink.finish(A, lda, std::min(k, m), std::min(k, n), n, s);
}
}  // namespace
}  // namespace sqr

extern "C" int sqr_rqrcp(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
                         uint64_t seed, const double* omegaT, int64_t ldo, int resample, int64_t* perm,
                         double* taus, double* T, sqr_status* st, void* workspace, int64_t workspace_bytes,
                         void* stream) {
  return rqrcp_impl(A, lda, m, n, k, b, p, seed, omegaT, ldo, resample, perm, taus, T, st, workspace,
                    workspace_bytes, nullptr, 0, static_cast<cudaStream_t>(stream));
}

extern "C" int64_t sqr_rqrcp_stream_r_workspace(int64_t m, int64_t n, int64_t k, int64_t b, int64_t p) {
  return sqr_rqrcp_workspace(m, n, k, b, p) + cdiv(k, b) * b * b * 8;
}

extern "C" int sqr_rqrcp_stream_r(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
                                  uint64_t seed, const double* omegaT, int64_t ldo, int resample, int64_t* perm,
                                  double* taus, double* T, sqr_status* st, void* workspace,
                                  int64_t workspace_bytes, double* R_host, int64_t ldrh, void* stream) {
  if (R_host == nullptr || ldrh < std::min(k, m)) {
    set_error("sqr_rqrcp_stream_r: R_host missing or ldrh < min(k, m)");
    return SQR_EINVAL;
  }
  return rqrcp_impl(A, lda, m, n, k, b, p, seed, omegaT, ldo, resample, perm, taus, T, st, workspace,
                    workspace_bytes, R_host, ldrh, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------ TRQRCP
namespace {
struct TrqrcpWs {
  RqrcpWs r;
  double *Pn, *Gb, *Cr;
};
TrqrcpWs carve_trqrcp(void* ws, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p, bool need_omega) {
  TrqrcpWs w;
  w.r = carve_rqrcp(ws, m, n, b, p, need_omega, false);
  Carve c(ws);
  c.off = w.r.total;
  w.Pn = c.take<double>(m * b);
  w.Gb = c.take<double>(b * (n + b));
  w.Cr = c.take<double>(b * std::max<int64_t>(k, 1));
  w.r.total = c.off + 256;
  return w;
}
}  // namespace

extern "C" int64_t sqr_trqrcp_workspace(int64_t m, int64_t n, int64_t k, int64_t b, int64_t p) {
  return carve_trqrcp(nullptr, m, n, k, b, p, true).r.total;
}

// Truncated RQRCP (randomized.py:250-341): A is only permuted; per block the
// panel is materialised through the accumulated reflections, and the new
// W^T / R rows come from the adjusted inner products, so A is read about once
// per block (one GEMM sweep Y2^T A).
extern "C" int sqr_trqrcp(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
                          uint64_t seed, const double* omegaT, int64_t ldo, double* Yg, int64_t ldy, double* Wg,
                          int64_t ldw, double* Rg, int64_t ldr, int64_t* perm, double* taus, double* T,
                          sqr_status* st, void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t ell = b + p;
  if (m <= 0 || n <= 0 || k < 1 || k > std::min(m, n) || b < 1 || p < 0 || ell >= m || lda < m || ldy < m ||
      ldw < k || ldr < k) {
    set_error("sqr_trqrcp: invalid arguments");
    return SQR_EINVAL;
  }
  if (b > 128 || ell > 144) {
    set_error("sqr_trqrcp: b=%lld / l=%lld exceed the kernel limits (b<=128, b+p<=144)", (long long)b,
              (long long)ell);
    return SQR_EINVAL;
  }
  TrqrcpWs tw = carve_trqrcp(workspace, m, n, k, b, p, omegaT == nullptr);
  RqrcpWs& w = tw.r;
  if (workspace == nullptr || workspace_bytes < w.total) {
    set_error("sqr_trqrcp: workspace %lld < %lld bytes", (long long)workspace_bytes, (long long)w.total);
    return SQR_EINVAL;
  }
  SQR_CUDA(cudaMemsetAsync(st, 0, sizeof(sqr_status), s));
  int rc = iota(perm, n, s);
  if (rc) return rc;
  if (omegaT == nullptr) {
    if ((rc = gaussian(w.OmT, m, ell, m, seed, 0, 1, nullptr, s))) return rc;
    omegaT = w.OmT;
    ldo = m;
  }
  if ((rc = gemm_tn(ell, n, m, 1.0, omegaT, ldo, A, lda, 0.0, nullptr, 0, w.Bcur, ell, w.gemm, kGemmWsBytes, s,
                    GemmDyn{})))
    return rc;
  const int64_t nblk = cdiv(k, b);
  double* Bc = w.Bcur;
  double* Bn = w.Bnext;
  for (int64_t J = 0; J < nblk; ++J) {
    const int64_t i0 = J * b, bb = std::min(b, k - i0), nt = n - i0, mr = m - i0;
    double* TJ = T + J * b * b;
    double* Ypan = Yg + i0 + i0 * ldy;  // Yg[i0:, i0:i0+bb]
    GemmDyn gate{&st->stop, nullptr, 0};
    if ((rc = sample_qrcp(Bc, ell, ell, nt, bb, w.Bf, ell, w.lperm, w.moves, w.stau, J == 0, st, w.sample,
                          w.sample_bytes, s)))
      return rc;
    if ((rc = apply_moves(A, lda, m, i0, perm, w.moves, st, 2 * bb, s))) return rc;
    if (i0 > 0) {
      if ((rc = apply_moves(Wg, ldw, i0, i0, nullptr, w.moves, st, 2 * bb, s))) return rc;
      if ((rc = apply_moves(Rg, ldr, i0, i0, nullptr, w.moves, st, 2 * bb, s))) return rc;
    }
    // panel = A[i0:, sel] - Yg[i0:, :i0] Wg[:i0, sel]   (randomized.py:304-306)
    if ((rc = gemm_nn(mr, bb, i0, -1.0, Yg + i0, ldy, Wg + i0 * ldw, ldw, 1.0, A + i0 + i0 * lda, lda, tw.Pn, m,
                      s, gate)))
      return rc;
    {
      PanelScratch sc{w.pscr, w.pscr + kLeaf * (kLeaf + b), w.pscr + kLeaf * (kLeaf + b) + kLeaf * b};
      if ((rc = panel_factor(tw.Pn, m, mr, bb, -1, Ypan, ldy, taus + i0, 1, st, w.panel, w.panel_bytes, sc, w.gemm,
                             s)))
        return rc;
    }
    if ((rc = copy_upper(tw.Pn, m, Rg + i0 + i0 * ldr, ldr, bb, &st->stop, s))) return rc;
    // [Y2^T Y2 | G] = Y2^T [Y2 | A[i0:, tcols]]   (randomized.py:311,322) in one sweep
    GemmDyn shP{&st->stop, &st->bhat, kShiftB};
    shP.pre = Ypan;
    shP.ldpre = ldy;
    shP.npre = (int)bb;
    if ((rc = gemm_tn(bb, bb + nt, mr, 1.0, Ypan, ldy, A + i0 + i0 * lda, lda, 0.0, nullptr, 0, tw.Gb, b, w.gemm,
                      kGemmWsBytes, s, shP)))
      return rc;
    if ((rc = build_t(tw.Gb, b, taus + i0, bb, TJ, b, &st->stop, s))) return rc;
    if (nt > 1) {
      GemmDyn shB{&st->stop, &st->bhat, kShiftB};
      GemmDyn shD{&st->stop, &st->bhat, kShiftD};
      GemmDyn shBD{&st->stop, &st->bhat, kShiftB | kShiftD};
      double* Gbt = tw.Gb + bb * b;  // G = Y2^T A[i0:, tcols]
      if (i0 > 0) {
        // G -= (Y2^T Y1) W1^T   (randomized.py:325-326)
        if ((rc = gemm_tn(bb, i0, mr, 1.0, Ypan, ldy, Yg + i0, ldy, 0.0, nullptr, 0, tw.Cr, b, w.gemm, kGemmWsBytes,
                          s, gate)))
          return rc;
        if ((rc = gemm_nn(bb, nt, i0, -1.0, tw.Cr, b, Wg + i0 * ldw, ldw, 1.0, Gbt, b, Gbt, b, s, shB)))
          return rc;
      }
      // Wg[i0:i0+bb, tcols] = T2^T G   (randomized.py:327)
      if ((rc = gemm_tn(bb, nt, bb, 1.0, TJ, b, Gbt, b, 0.0, nullptr, 0, Wg + i0 + i0 * ldw, ldw, w.gemm,
                        kGemmWsBytes, s, shD)))
        return rc;
      // R12 = A[i0:i0+bb, tcols] - Yg[i0:i0+bb, :i0+bb] Wg[:i0+bb, tcols]   (randomized.py:329-330)
      if ((rc = gemm_nn(bb, nt, i0 + bb, -1.0, Yg + i0, ldy, Wg + i0 * ldw, ldw, 1.0, A + i0 + i0 * lda, lda,
                        Rg + i0 + i0 * ldr, ldr, s, shBD)))
        return rc;
    }
    if ((rc = finish_block(st, nullptr, (int)i0, (int)bb, (int)k, (int)n, s))) return rc;
    if (J + 1 < nblk) {
      if ((rc = sample_update(w.Bf, ell, ell, Rg + i0 + i0 * ldr, ldr, nt - bb, bb, Bn, ell, st, w.Gm, s))) return rc;
      std::swap(Bc, Bn);
    }
  }
  return SQR_OK;
}

// ------------------------------------------------------------ qr_blocked
extern "C" int64_t sqr_qr_blocked_workspace(int64_t m, int64_t n, int64_t /*k*/, int64_t b) {
  Carve c(nullptr);
  c.take<double>(kGemmWsBytes / 8);
  c.take<char>(panel_workspace(std::min<int64_t>(b, 128)));
  c.take<double>(m * b);        // Ypan
  c.take<double>(b * b);        // G
  c.take<double>(b * (n + b));  // [G | Wt]
  c.take<double>(b * n);        // W
  c.take<sqr_status>(1);
  c.take<double>(PanelScratch::doubles(b));
  return c.off + 256;
}

extern "C" int sqr_qr_blocked(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, double* taus,
                              double* T, void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (m <= 0 || n <= 0 || k < 1 || k > std::min(m, n) || b < 1 || b > 128 || lda < m) {
    set_error("sqr_qr_blocked: invalid arguments");
    return SQR_EINVAL;
  }
  if (workspace_bytes < sqr_qr_blocked_workspace(m, n, k, b)) {
    set_error("sqr_qr_blocked: workspace too small");
    return SQR_EINVAL;
  }
  Carve c(workspace);
  double* gws = c.take<double>(kGemmWsBytes / 8);
  const int64_t pb = panel_workspace(std::min<int64_t>(b, 128));
  void* pws = c.take<char>(pb);
  double* Ypan = c.take<double>(m * b);
  double* Gm = c.take<double>(b * b);
  double* Wt = c.take<double>(b * (n + b));
  double* W = c.take<double>(b * n);
  sqr_status* st = c.take<sqr_status>(1);
  double* pscr = c.take<double>(PanelScratch::doubles(b));
  (void)Gm;
  SQR_CUDA(cudaMemsetAsync(st, 0, sizeof(sqr_status), s));
  int rc;
  for (int64_t i0 = 0; i0 < k; i0 += b) {
    const int64_t bb = std::min(b, k - i0), mr = m - i0, nt = n - i0;
    double* P = A + i0 + i0 * lda;
    double* TJ = T + (i0 / b) * b * b;
    {
      PanelScratch sc{pscr, pscr + kLeaf * (kLeaf + b), pscr + kLeaf * (kLeaf + b) + kLeaf * b};
      if ((rc = panel_factor(P, lda, mr, bb, bb, Ypan, m, taus + i0, 0, st, pws, pb, sc, gws, s))) return rc;
    }
    if ((rc = trailing_update(P, lda, mr, nt, bb, Ypan, m, taus + i0, TJ, b, Wt, W, b, st, gws, s))) return rc;
  }
  return SQR_OK;
}

// ------------------------------------------------------------ WY helpers
extern "C" int sqr_build_t(const double* Y, int64_t ldy, int64_t m, int64_t j, const double* taus, double* T,
                           int64_t ldt, double* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (j <= 0) return SQR_OK;
  if (j > 144 || workspace_bytes < (int64_t)(j * j * 8) + kGemmWsBytes) {
    set_error("sqr_build_t: j > 144 or workspace too small");
    return SQR_EINVAL;
  }
  double* Gm = workspace;
  double* gws = workspace + rup(j * j, 32);
  int rc = gemm_tn(j, j, m, 1.0, Y, ldy, Y, ldy, 0.0, nullptr, 0, Gm, j, gws, kGemmWsBytes, s, GemmDyn{});
  if (rc) return rc;
  return build_t(Gm, j, taus, j, T, ldt, nullptr, s);
}

extern "C" int sqr_apply_wy(const double* Y, int64_t ldy, const double* T, int64_t ldt, int64_t m, int64_t j,
                            double* C, int64_t ldc, int64_t ncols, int transpose, double* workspace,
                            int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (j <= 0 || ncols <= 0) return SQR_OK;
  if (j > 144 || workspace_bytes < 2 * j * ncols * 8 + kGemmWsBytes + 1024) {
    set_error("sqr_apply_wy: j > 144 or workspace too small");
    return SQR_EINVAL;
  }
  double* Wt = workspace;
  double* W = workspace + rup(j * ncols, 32);
  double* gws = W + rup(j * ncols, 32);
  // Wt = Y^T C
  int rc = gemm_tn(j, ncols, m, 1.0, Y, ldy, C, ldc, 0.0, nullptr, 0, Wt, j, gws, kGemmWsBytes, s, GemmDyn{});
  if (rc) return rc;
  if (transpose) {
    // W = -T^T Wt
    rc = gemm_tn(j, ncols, j, -1.0, T, ldt, Wt, j, 0.0, nullptr, 0, W, j, gws, kGemmWsBytes, s, GemmDyn{});
  } else {
    // W = -T Wt
    rc = gemm_nn(j, ncols, j, -1.0, T, ldt, Wt, j, 0.0, nullptr, 0, W, j, s, GemmDyn{});
  }
  if (rc) return rc;
  return gemm_nn(m, ncols, j, 1.0, Y, ldy, W, j, 1.0, C, ldc, C, ldc, s, GemmDyn{});
}

extern "C" int sqr_panel_qr(double* P, int64_t ldp, int64_t mr, int64_t w, double* Y, int64_t ldy, double* taus,
                            double* T, int64_t ldt, int stop_at_zero, sqr_status* st, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t wmax = w < 0 ? 128 : w;
  const int64_t pb = panel_workspace(wmax);
  const int64_t total = pb + kGemmWsBytes + wmax * wmax * 8 + 1024;
  char* ws = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), total, s) != cudaSuccess) {
    set_error("sqr_panel_qr: cudaMallocAsync failed");
    return SQR_ECUDA;
  }
  cudaMemsetAsync(ws, 0, total, s);
  int rc = panel_qr(P, ldp, mr, w, wmax, Y, ldy, taus, stop_at_zero, st, ws, pb, s);
  double* Gm = reinterpret_cast<double*>(ws + rup(pb, 256));
  double* gws = Gm + rup(wmax * wmax, 32);
  if (!rc)
    rc = gemm_tn(wmax, wmax, mr, 1.0, Y, ldy, Y, ldy, 0.0, nullptr, 0, Gm, wmax, gws, kGemmWsBytes, s,
                 GemmDyn{&st->stop, nullptr, 0});
  if (!rc && T) rc = build_t(Gm, wmax, taus, wmax, T, ldt, &st->stop, s);
  cudaFreeAsync(ws, s);
  return rc;
}

// ------------------------------------------------------- multi-GPU building blocks
// Workspace for sqr_panel_factor / sqr_apply_block_update.
extern "C" int64_t sqr_block_workspace(int64_t m, int64_t ncols, int64_t b) {
  Carve c(nullptr);
  c.take<double>(kGemmWsBytes / 8);
  c.take<char>(panel_workspace(std::min<int64_t>(b, 128)));
  c.take<double>(PanelScratch::doubles(b));
  c.take<double>(b * (ncols + b));
  c.take<double>(b * std::max<int64_t>(ncols, 1));
  c.take<sqr_status>(1);
  return c.off + 256;
}

namespace {
struct BlockWs {
  double *gws, *pscr, *GWt, *W;
  void* pws;
  int64_t pwsb;
  sqr_status* st;
};
BlockWs carve_block(void* ws, int64_t ncols, int64_t b) {
  Carve c(ws);
  BlockWs w;
  w.gws = c.take<double>(kGemmWsBytes / 8);
  w.pwsb = panel_workspace(std::min<int64_t>(b, 128));
  w.pws = c.take<char>(w.pwsb);
  w.pscr = c.take<double>(PanelScratch::doubles(b));
  w.GWt = c.take<double>(b * (ncols + b));
  w.W = c.take<double>(b * std::max<int64_t>(ncols, 1));
  w.st = c.take<sqr_status>(1);
  return w;
}
}  // namespace

// Panel of width w (<= b) at P (mr rows) with the leaf kernel + WY updates;
// st receives bhat / stop (stop_at_zero semantics of randomized.py:120-121).
extern "C" int sqr_panel_factor(double* P, int64_t ldp, int64_t mr, int64_t w, double* Y, int64_t ldy,
                                double* taus, int stop_at_zero, sqr_status* st, void* workspace,
                                int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (w <= 0 || w > 128 || mr <= 0) {
    set_error("sqr_panel_factor: need 1 <= w <= 128");
    return SQR_EINVAL;
  }
  if (workspace_bytes < sqr_block_workspace(mr, 0, w)) {
    set_error("sqr_panel_factor: workspace too small");
    return SQR_EINVAL;
  }
  BlockWs bw = carve_block(workspace, 0, w);
  PanelScratch sc{bw.pscr, bw.pscr + kLeaf * (kLeaf + w), bw.pscr + kLeaf * (kLeaf + w) + kLeaf * w};
  return panel_factor(P, ldp, mr, w, w, Y, ldy, taus, stop_at_zero, st, bw.pws, bw.pwsb, sc, bw.gws, s);
}

// One block reflection of ncols columns C (mr rows): T from Y and taus
// (written to T, ld ldt), then C := (I - Y T Y^T)^T C  (randomized.py:203-207).
extern "C" int sqr_apply_block_update(double* C, int64_t ldc, int64_t mr, int64_t ncols, int64_t bb,
                                      const double* Y, int64_t ldy, const double* taus, double* T, int64_t ldt,
                                      void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bb <= 0 || bb > 128 || mr <= 0) {
    set_error("sqr_apply_block_update: need 1 <= bb <= 128");
    return SQR_EINVAL;
  }
  if (workspace_bytes < sqr_block_workspace(mr, ncols, bb)) {
    set_error("sqr_apply_block_update: workspace too small");
    return SQR_EINVAL;
  }
  BlockWs bw = carve_block(workspace, ncols, bb);
  SQR_CUDA(cudaMemsetAsync(bw.st, 0, sizeof(sqr_status), s));
  GemmDyn d1{nullptr, nullptr, 0};
  d1.pre = Y;
  d1.ldpre = ldy;
  d1.npre = (int)bb;
  int rc = gemm_tn(bb, bb + ncols, mr, 1.0, Y, ldy, C, ldc, 0.0, nullptr, 0, bw.GWt, bb, bw.gws, kGemmWsBytes, s, d1);
  if (rc) return rc;
  if ((rc = build_t(bw.GWt, bb, taus, bb, T, ldt, nullptr, s))) return rc;
  if (ncols <= 0) return SQR_OK;
  rc = gemm_tn(bb, ncols, bb, -1.0, T, ldt, bw.GWt + bb * bb, bb, 0.0, nullptr, 0, bw.W, bb, bw.gws, kGemmWsBytes, s,
               GemmDyn{});
  if (rc) return rc;
  return gemm_nn(mr, ncols, bb, 1.0, Y, ldy, bw.W, bb, 1.0, C, ldc, C, ldc, s, GemmDyn{});
}
