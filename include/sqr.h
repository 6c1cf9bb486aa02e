/*
 * sqr.h -- C ABI of libsqr.so, the B200 (sm_100a) implementation of the
 * randomized column-pivoted QR hot path of the reference package `sketchqr`
 * (Duersch & Gu, arXiv 2008.04447).
 *
 * The reference is pure Python; it has no FFI.  Its drop-in boundary is the
 * Python functions rqrcp / trqrcp / tuxv (pkg/src/sketchqr/randomized.py:227,
 * 250, 353).  This header is what a binding of those functions needs
 * underneath: every pointer is a DEVICE pointer to column-major fp64 (or
 * int64 / int32) storage, every size is an int64, and every call is
 * asynchronous on the given cudaStream_t (passed as void*).  No torch or
 * Python types cross this boundary.  INTEGRATION.md shows the ctypes stub.
 *
 * Return codes: SQR_OK, SQR_EINVAL (bad argument), SQR_ECUDA (CUDA error;
 * sqr_last_error() has the text).  Rank exhaustion is NOT an error: it shows
 * up as achieved < k in the status block, like the reference's achieved_rank.
 */
#ifndef SQR_H
#define SQR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SQR_OK 0
#define SQR_EINVAL 1
#define SQR_ECUDA 2

#define SQR_MAX_BLOCKS 65536

/* Device-resident progress / termination record of one factorization.
 * Mirrors the reference's loop state: achieved (randomized.py:183,211),
 * the list of ReflectorBlock widths (randomized.py:202), and the reason the
 * loop stopped (randomized.py:189-190,192-193,197-198,212-213,217-219). */
typedef struct sqr_status {
  int32_t stop;           /* 1 once the loop has terminated                       */
  int32_t reason;         /* SQR_STOP_* below                                     */
  int32_t achieved;       /* factored columns (achieved_rank)                     */
  int32_t nblocks;        /* completed ReflectorBlocks                            */
  int32_t sample_achieved;/* pivots found by the current block's sample QRCP      */
  int32_t bhat;           /* reflectors produced by the current block's panel     */
  int32_t nmoves;         /* column moves of the current block                    */
  int32_t pad_;
  double floor_sq;        /* SAMPLE_FLOOR^2 * max initial sample column norm^2     */
  double aux[4];
} sqr_status;

#define SQR_STOP_NONE 0
#define SQR_STOP_K_REACHED 1      /* achieved >= k                                   */
#define SQR_STOP_SAMPLE_FLOOR 2   /* max sample col norm^2 <= floor (randomized.py:189) */
#define SQR_STOP_SAMPLE_RANK 3    /* sample QRCP found 0 pivots (randomized.py:192)  */
#define SQR_STOP_PANEL_ZERO 4     /* panel beta == 0 at column 0 (randomized.py:197) */
#define SQR_STOP_SHORT_BLOCK 5    /* bhat < bb (randomized.py:212)                   */
#define SQR_STOP_NO_TRAILING 6    /* ncols == 0 (randomized.py:212)                  */
#define SQR_STOP_R11_SINGULAR 7   /* _diag_ok false (randomized.py:217-219)          */

/* ---------------------------------------------------------------- info */
const char* sqr_version(void);
const char* sqr_last_error(void);
int sqr_device_sm_count(void);

/* Kernels launched by this library since load (bench.py's gpu_launches). */
int64_t sqr_launch_count(void);
/* Per-kernel-class CUDA-event timing of the next <= max_launches launches
 * (0 disables).  Classes: 0 gemm_tn, 1 gemm_nn, 2 sample_qrcp, 3 panel,
 * 4 build_t, 5 apply_moves, 6 sample_update, 7 gaussian, 8 misc, 9 gemm_nn
 * launches that share the chip with a sample QRCP / panel kernel (their event
 * times measure the shared run; sqr_profile_flops gives their flops). */
int sqr_profile_enable(int64_t max_launches);
int sqr_profile_collect(double* ms_per_tag, int64_t* count_per_tag, int ntags);
int sqr_profile_flops(double* flops_per_tag, int ntags);
/* Time only the classes whose bit is set in tag_mask (default: all). */
int sqr_profile_select(uint32_t tag_mask);
/* Debug: %globaltimer phase stamps of the cooperative kernels (NULL = off). */
int sqr_debug_trace(void* device_buffer);

/* ------------------------------------------------------------ RNG (L0)
 * Omega[i, t] = normal(seed, offset + i + t*rows) for a rows x cols matrix
 * filled column-major (rng.py:49-70, NormalStream.matrix rng.py:90-93).
 * transpose=0 writes Omega (ld >= rows); transpose=1 writes Omega^T
 * (cols x rows, ld >= cols), the K-major operand the sketch GEMM reads. */
int sqr_gaussian(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed,
                 uint64_t offset, int transpose, void* stream);

/* ----------------------------------------------------------- GEMMs (K1, K6, K8-K11)
 * D(M x N) = alpha * X^T C + beta * E     X: K x M (ldx), C: K x N (ldc), E,D: M x N
 * (np: `Y.T @ C` sites: randomized.py:206,322,325; sketch.py:71 with X = Omega^T).
 * fp64 DMMA (mma.sync f64) tiles; deterministic split-K; E may alias D or be NULL. */
int sqr_gemm_tn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                const double* C, int64_t ldc, double beta, const double* E, int64_t lde,
                double* D, int64_t ldd, double* workspace, int64_t workspace_bytes, void* stream);

/* D(M x N) = alpha * X Y + beta * E         X: M x K (ldx), Y: K x N (ldy)
 * (np: `C -= Y @ W` sites: randomized.py:207,305,330,384). */
int sqr_gemm_nn(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                const double* Y, int64_t ldy, double beta, const double* E, int64_t lde,
                double* D, int64_t ldd, void* stream);
/* Same with a caller workspace: skinny products with long K (TUXV's A V_k,
 * randomized.py:384) split K across CTAs when the output tiles cannot fill
 * the GPU; partials are summed in a fixed order (deterministic).  Needs up to
 * 16 * M * N doubles; less workspace means fewer splits. */
int sqr_gemm_nn_ws(int64_t M, int64_t N, int64_t K, double alpha, const double* X, int64_t ldx,
                   const double* Y, int64_t ldy, double beta, const double* E, int64_t lde,
                   double* D, int64_t ldd, double* workspace, int64_t workspace_bytes, void* stream);

/* ------------------------------------------------- sample QRCP (K2, K12)
 * Halted pivoted QR of the l x nt sample B (sketch.py:97-119 -> reference.py
 * _qrcp_core:107-150) on a persistent cooperative kernel.  Writes the
 * factored sample in pivoted order to Bf (l x nt, ldbf), the local
 * permutation lperm[pos] = source column (int64, nt), the list of moved
 * positions moves[2*i] = dst, moves[2*i+1] = src (int32, <= 2*bb pairs; dst = -1 marks an unused slot) and
 * st->sample_achieved / st->nmoves.  first != 0 also sets st->floor_sq from
 * this sample (randomized.py:179-180).  Skipped when st->stop is set. */
int sqr_sample_qrcp(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb,
                    double* Bf, int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus,
                    int first, sqr_status* st, void* stream);
/* Same with caller-owned scratch (>= sqr_sample_qrcp_workspace(l, nt) bytes,
 * whose first 64 bytes -- the grid-barrier word -- the call resets on the
 * stream): no allocation, so it can be issued every block by an orchestrator. */
int64_t sqr_sample_qrcp_workspace(int64_t ell, int64_t nt);
int sqr_sample_qrcp_ws(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                       int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* sqr_sample_qrcp_ws that also stores resident_val to *resident_flag (device
 * memory, zeroed by the caller, values increasing) once all of its CTAs are
 * on the chip; sqr_wait_resident holds `stream` until then (at most
 * timeout_us).  The sample QRCP owns ceil(nt / 256) whole SMs for its ~0.7 ms:
 * a GEMM enqueued behind sqr_wait_resident on another stream runs on the
 * other SMs meanwhile (no reference counterpart: scheduling only). */
int sqr_sample_qrcp_ws_sig(const double* B, int64_t ldb, int64_t ell, int64_t nt, int64_t bb, double* Bf,
                           int64_t ldbf, int64_t* lperm, int32_t* moves, double* taus, int first, sqr_status* st,
                           void* workspace, int64_t workspace_bytes, uint32_t* resident_flag,
                           uint32_t resident_val, void* stream);
int sqr_wait_resident(uint32_t* resident_flag, uint32_t resident_val, int timeout_us, void* stream);

/* Apply the block's column moves to rows [0, rows) of X (ld) starting at
 * column col0, and to the int64 vector perm (may be NULL) starting at col0
 * (randomized.py:194-195; trqrcp also permutes Wg, Rg at :301-302). */
int sqr_apply_moves(double* X, int64_t ld, int64_t rows, int64_t col0, int64_t* perm,
                    const int32_t* moves, const sqr_status* st, int64_t max_moves, void* stream);

/* ----------------------------------------------------------- panel (K4, K5)
 * Unpivoted Householder QR of P (mr x w, ldp) in place (randomized.py:107-130,
 * householder.py:28-49), stopping at the first zero column when stop_at_zero
 * (the qr_blocked variant, reference.py:281-291, keeps identity reflectors).
 * w = st->sample_achieved when w < 0.  Outputs: the packed panel in P, the
 * explicit unit-lower Y (mr x w, ldy), taus, the compact-WY T (w x w, ldt,
 * householder.py:52-61) and st->bhat. */
int sqr_panel_qr(double* P, int64_t ldp, int64_t mr, int64_t w, double* Y, int64_t ldy,
                 double* taus, double* T, int64_t ldt, int stop_at_zero, sqr_status* st,
                 void* stream);

/* T factor only, from an explicit unit-lower Y (m x j) and taus. */
int sqr_build_t(const double* Y, int64_t ldy, int64_t m, int64_t j, const double* taus,
                double* T, int64_t ldt, double* workspace, int64_t workspace_bytes, void* stream);

/* ----------------------------------------------------- sample update (K7)
 * Bnext = [S12 - S11 R11^{-1} R12 ; S22] (sketch.py:122-149) for the nt
 * trailing columns, after the R11 diagonal guard (randomized.py:133-135,
 * 217-219).  Bf is the factored sample from sqr_sample_qrcp (l x (nt+b)). */
int sqr_sample_update(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr,
                      int64_t nt, double* Bnext, int64_t ldbn, sqr_status* st, void* stream);
/* Same, with the block size b (= the sample QRCP's sample_achieved) given by
 * the caller and a caller-owned b*b scratch `mbuf`: never synchronises the
 * host (the multi-GPU orchestrator already knows b). */
int sqr_sample_update_b(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr, int64_t nt,
                        int64_t b, double* Bnext, int64_t ldbn, sqr_status* st, double* mbuf, void* stream);
/* The same in two halves, so an orchestrator can run the prep (R11 guard +
 * M = S11 R11^-1, sketch.py:132-149 / randomized.py:217-219) concurrently with
 * the trailing update: prep reads S11 (first b columns of Bf) and R11 (ld ldr)
 * and writes M (b*b) to mbuf; apply forms Bnext from M, R = [R11 | R12] and Bf. */
int sqr_sample_update_prep(const double* Bf, int64_t ldbf, const double* R11, int64_t ldr, int64_t b,
                           double* mbuf, sqr_status* st, void* stream);
int sqr_sample_update_apply(const double* Bf, int64_t ldbf, int64_t ell, const double* R, int64_t ldr, int64_t nt,
                            int64_t b, double* Bnext, int64_t ldbn, sqr_status* st, const double* mbuf,
                            void* stream);

/* ------------------------------------------------------------- drivers
 * Full RQRCP (randomized.py:166-224, resample=0) / RSRQRCP (resample=1) on the
 * m x n device matrix A (lda), in place: R in the upper trapezoid of the
 * first `achieved` rows, reflector tails below the diagonal.  Omega^T (m x l,
 * ldo) is the sketch draw (or NULL to draw it from seed on the device).
 * Outputs: perm (int64, n), taus (k), T blocks (nblk x b x b, block J at
 * T + J*b*b, ld b), status.  All work is enqueued on `stream` with no host
 * synchronisation: early exits are device-side flags.  Workspace from
 * sqr_rqrcp_workspace(). */
int64_t sqr_rqrcp_workspace(int64_t m, int64_t n, int64_t k, int64_t b, int64_t p);
int sqr_rqrcp(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
              uint64_t seed, const double* omegaT, int64_t ldo, int resample, int64_t* perm,
              double* taus, double* T, sqr_status* st, void* workspace, int64_t workspace_bytes,
              void* stream);

/* sqr_rqrcp + R streamed to pinned host memory while the factorization runs:
 * each column block of R (rows [0, i0+bb), columns [i0, i0+bb)) is final right
 * after its panel (later column moves only touch later columns) and is copied
 * to R_host (column-major, ldrh >= min(k, m)) on an internal copy stream,
 * overlapping the remaining blocks; entries below the diagonal are not
 * written.  The copies are joined into `stream`.  Workspace:
 * sqr_rqrcp_stream_r_workspace() (adds one b x b staging slot per block).
 * Replaces the reference's host-resident result of randomized.py:227-229. */
int64_t sqr_rqrcp_stream_r_workspace(int64_t m, int64_t n, int64_t k, int64_t b, int64_t p);
int sqr_rqrcp_stream_r(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
                       uint64_t seed, const double* omegaT, int64_t ldo, int resample, int64_t* perm,
                       double* taus, double* T, sqr_status* st, void* workspace, int64_t workspace_bytes,
                       double* R_host, int64_t ldrh, void* stream);

/* Truncated RQRCP (randomized.py:250-341).  A is permuted in place but never
 * updated.  Outputs Yg (m x k, ldy), Wg (k x n, ldw: W^T rows), Rg (k x n,
 * ldr), perm, taus, T blocks, status. */
int64_t sqr_trqrcp_workspace(int64_t m, int64_t n, int64_t k, int64_t b, int64_t p);
int sqr_trqrcp(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b, int64_t p,
               uint64_t seed, const double* omegaT, int64_t ldo, double* Yg, int64_t ldy,
               double* Wg, int64_t ldw, double* Rg, int64_t ldr, int64_t* perm, double* taus,
               double* T, sqr_status* st, void* workspace, int64_t workspace_bytes, void* stream);

/* Unpivoted blocked QR (reference.py:266-311) in place on A (m x n), first k
 * columns; used by TUXV (randomized.py:375,387).  Outputs taus (k), T blocks
 * (ld b, block J at T + J*b*b). */
int64_t sqr_qr_blocked_workspace(int64_t m, int64_t n, int64_t k, int64_t b);
int sqr_qr_blocked(double* A, int64_t lda, int64_t m, int64_t n, int64_t k, int64_t b,
                   double* taus, double* T, void* workspace, int64_t workspace_bytes,
                   void* stream);

/* C := Q C (transpose=0) or Q^T C (transpose=1) for Q = I - Y T Y^T, Y m x j
 * explicit unit-lower (householder.py:107-120). */
int sqr_apply_wy(const double* Y, int64_t ldy, const double* T, int64_t ldt, int64_t m, int64_t j,
                 double* C, int64_t ldc, int64_t ncols, int transpose, double* workspace,
                 int64_t workspace_bytes, void* stream);

/* --------------------------------------------- multi-GPU building blocks
 * Used by the column block-cyclic driver (paper_2008_04447_b200/distributed.py)
 * where each rank owns a subset of the columns. */
int64_t sqr_block_workspace(int64_t m, int64_t ncols, int64_t b);
/* dst[:, dst_idx[j]] = src[:, src_idx[j]], j < n, rows [0, rows); NULL index = identity. */
/* Input contract (validation.py:21-37): dst = src (m x n, column-major; dst
 * may be NULL for a check only) and *nonfinite += #NaN/Inf entries, in one
 * read of src.  *nonfinite is a device counter the caller zeroes. */
int sqr_copy_check(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                   unsigned long long* nonfinite, void* stream);
/* Same for a ROW-major src (element (r, c) at src[r * lds + c], lds >= n, e.g. a
 * C-ordered torch tensor) into column-major dst (tiled transpose). */
int sqr_copy_check_t(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                     unsigned long long* nonfinite, void* stream);
int sqr_copy_columns(const double* src, int64_t lds, int64_t rows, const int64_t* src_idx, double* dst,
                     int64_t ldd, const int64_t* dst_idx, int64_t n, void* stream);
/* Panel QR of an mr x w panel (w <= 128), leaves + compact-WY updates; st->bhat/stop. */
int sqr_panel_factor(double* P, int64_t ldp, int64_t mr, int64_t w, double* Y, int64_t ldy, double* taus,
                     int stop_at_zero, sqr_status* st, void* workspace, int64_t workspace_bytes, void* stream);
/* T from (Y, taus), then C := Q^T C for ncols local columns (randomized.py:203-207). */
int sqr_apply_block_update(double* C, int64_t ldc, int64_t mr, int64_t ncols, int64_t bb, const double* Y,
                           int64_t ldy, const double* taus, double* T, int64_t ldt, void* workspace,
                           int64_t workspace_bytes, void* stream);

/* ------------------------------------------------------ result assembly
 * Bandwidth kernels that build the reference's result arrays on the device.
 * dst (n x m, ld ldd) = src^T for src m x n (ld lds); upper != 0 keeps only
 * src's upper trapezoid (r <= c) -- R = triu(work[:achieved, :]) as row-major
 * rows (randomized.py:223, 338). */
int sqr_transpose(const double* src, int64_t lds, int64_t m, int64_t n, double* dst, int64_t ldd,
                  int upper, void* stream);
/* Y (m x w, ldy) = the explicit unit-lower reflectors of packed columns
 * [i0, i0+w) of W (ldw): the reference's Yfull, zeros above the block
 * offset (randomized.py:199-201, reference.py:153-159). */
int sqr_unpack_reflectors(const double* W, int64_t ldw, int64_t m, int64_t i0, int64_t w, double* Y,
                          int64_t ldy, void* stream);
/* gather: dst[i, j] = src[idx[i], j]; scatter: dst[idx[i], j] = src[i, j]
 * (i < rows, j < cols, idx int64): TUXV's P^T V_k and Z0^T = (R P^T)^T
 * (randomized.py:374, 384; validation.py:56-59). */
int sqr_gather_rows(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx,
                    double* dst, int64_t ldd, void* stream);
int sqr_scatter_rows(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx,
                     double* dst, int64_t ldd, void* stream);
/* X R = S (X, S rows x n; R upper triangular n x n): S11 R11^{-1} of the
 * sample update for blocks wider than 128 (sketch.py:122-149); upper_s != 0
 * reads S as upper triangular (entries below its diagonal ignored). */
int sqr_trsm_right_upper(const double* S, int64_t lds, int64_t rows, int64_t n, const double* R, int64_t ldr,
                         double* X, int64_t ldx, int upper_s, void* stream);
/* ------------------------------------------------------------ Jacobi SVD
 * One-sided Jacobi SVD of W (m x n, m >= n, n <= 4096; jacobi.py:50-117) on
 * one CTA: W is rotated in place into U diag(sigma), V (n x n, ldv) gets
 * the accumulated rotations, sigma[c] the column norms (unsorted) and order
 * their stable descending order; info[0] = sweeps used, -1 if max_sweeps
 * did not converge.  tuxv(refine_sigma=True) uses it (randomized.py:402-403). */
int sqr_jacobi_svd(double* W, int64_t ldw, int64_t m, int64_t n, double* V, int64_t ldv, double* sigma,
                   int64_t* order, int max_sweeps, int32_t* info, void* stream);
/* ------------------------------------ device-initiated collectives (NVLink P2P)
 * The multi-GPU driver's fused collectives (SURVEY.md §8(e) B200-native
 * upgrade): the producing kernel stores straight into every peer's copy of a
 * symmetric buffer and publishes an epoch into each peer's flag word (system-
 * scope release); consumers gate their stream with sqr_peer_wait.  dst_ptrs /
 * flag_ptrs are DEVICE arrays of peer base pointers (e.g. the buffer_ptrs of
 * torch.distributed._symmetric_memory); counter is a device u32 owned by the
 * calling stream, zero before the first call and left at zero.
 * put: bytes (multiple of 16) from src to dst_ptrs[q] + dst_offset, q < npeers
 *      -- the panel record broadcast (randomized.py:203-207 on every rank);
 * put_columns: dst_ptrs[q][didx[j] * ldd + r] = src[j * lds + r] -- this
 *      rank's sample-update columns into their global positions of every
 *      replica (sketch.py:132-149): all-gather + assembly in one kernel;
 * wait: until flags[i] >= epoch, i < nflags (acquire, system scope). */
int sqr_peer_put(const void* src, int64_t bytes, void* const* dst_ptrs, int64_t dst_offset, int npeers,
                 unsigned long long* const* flag_ptrs, int slot, unsigned long long epoch, unsigned* counter,
                 void* stream);
int sqr_peer_put_columns(const double* src, int64_t lds, int64_t rows, int64_t ncols, const int64_t* didx,
                         double* const* dst_ptrs, int64_t ldd, int npeers, unsigned long long* const* flag_ptrs,
                         int slot, unsigned long long epoch, unsigned* counter, void* stream);
int sqr_peer_wait(const unsigned long long* flags, int nflags, unsigned long long epoch, void* stream);
#ifdef __cplusplus
}
#endif
#endif /* SQR_H */
