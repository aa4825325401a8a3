/*
 * pam_b200.h — C-ABI of the B200-native PAM hot path (libpam_b200.so).
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes (no torch
 * or C++ types), and returns an int status (PAM_OK on success).  Reals are
 * IEEE binary64 throughout; indices are int64 unless stated.
 *
 * Two layers:
 *
 *   1. Device-pointer, stream-ordered batch entry points (`pam_*_f64`).  All
 *      array arguments are DEVICE pointers; the call enqueues kernels on
 *      `stream` (a cudaStream_t passed as void*, NULL = legacy default stream)
 *      and returns without synchronising.  Data-dependent errors (non-positive
 *      field value, point outside all boxes, degenerate Shepard denominator)
 *      are reported through a caller-owned DEVICE int64[2] "error word"
 *      `err` = {code, first offending index}; initialise it with
 *      pam_err_reset() and read it after the stream is synchronised.
 *
 *   2. Host-pointer, synchronous seams (`pam_*_host_f64`) whose arguments
 *      mirror the reference function they replace one-for-one, so the
 *      reference package can bind them with ctypes.
 *
 * Ragged batches ("subdomains", reference partition.py:45-93) are described
 * by CSR-style offsets:
 *   row_off[S+1]  : cells (sample rows) of subdomain s are rows
 *                   [row_off[s], row_off[s+1]) of the packed point/value
 *                   arrays, ascending global cell index (fields.py:61-73).
 *   dict_off[S]   : first dictionary slot of subdomain s in the packed
 *                   centre/width/beta arrays; dict_cap[S] slots reserved.
 *   m_cur[S]      : current dictionary size M_s (int32, <= dict_cap[s]).
 *   w_off[S]      : offset (in doubles) of subdomain s's design matrix in
 *                   the packed W buffer; column-major with leading dimension
 *                   ld[s] (int32, multiple of 16): W_s[i, j] = W[w_off+j*ld+i].
 *
 * Concurrency: no entry point keeps mutable global state.  The batched CD and
 * evaluation kernels balance their work with a counter in the CALLER's
 * device workspace (`work`), so calls on different streams (or different
 * devices of one process) are independent as long as they use distinct
 * workspaces.  Kernel attributes are set per call, so one process may drive
 * several GPUs.  The host seams serialise per device on an internal arena.
 *
 * Citations are relative to the reference package root pkg/src/fieldfit/.
 */
#ifndef PAM_B200_H
#define PAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
#define PAM_OK 0
#define PAM_ERR_CUDA 1         /* CUDA runtime error (launch/alloc/copy)           */
#define PAM_ERR_ARG 2          /* invalid argument (sizes, dims, null pointers)    */
#define PAM_ERR_OUTSIDE 3      /* point outside all boxes  (geometry.py:255-257)   */
#define PAM_ERR_DEGENERATE 4   /* Shepard denominator degenerate (rbf.py:165-166)  */
#define PAM_ERR_NONPOSITIVE 5  /* field value not positive (elastic_net.py:200-204) */
#define PAM_ERR_UNSUPPORTED 6  /* shape outside the compiled kernel envelope       */
#define PAM_ERR_NONFINITE 7    /* non-finite design/target (elastic_net.py:81-82)  */
#define PAM_ERR_CLAIMED 8      /* point claimed by two boxes (geometry.py:249-251)  */

/* Version / capability probe: returns PAM_ABI_VERSION. */
#define PAM_ABI_VERSION 3
int pam_abi_version(void);
/* Last CUDA error string recorded by the library (host memory, static). */
const char* pam_last_error(void);
/* Largest subdomain sample count the CD kernels accept (rows per subdomain):
 * the reference has no limit; fits above 8192 rows run the CTA-per-fit
 * kernel with the residual in the workspace. */
int64_t pam_cd_max_rows(void);

/* CD kernel selection for pam_cd_tiles_f64 (`kernel`).  AUTO picks by batch
 * shape (see pam_cd_tiles_f64); the others force one implementation (tests
 * and A/B measurement).  Every choice computes the same CD up to the
 * rounding of the length-N dot products. */
#define PAM_CD_AUTO 0 /* by shape                                               */
#define PAM_CD_LEAN 1 /* one fit per warp                                       */
#define PAM_CD_DUAL 2 /* two fits per warp (257-512 rows)                       */
#define PAM_CD_PAIR 3 /* column pairs, few fits per SM (33-1024 rows)           */
#define PAM_CD_BLOCK 4 /* exact blocked CD, a solver + 8 worker warps per fit (<= 1024 rows) */

/* err[0] = 0 (no error), err[1] = INT64_MAX. Device pointer. */
int pam_err_reset(int64_t* err, void* stream);

/* ---- K0: log transform + positivity (elastic_net.py:197-205) ------------- */
/* y[i] = log(values[i]); first i with !(values[i] > 0) -> err {NONPOSITIVE, i}. */
int pam_log_values_f64(const double* values, int64_t n, double* y, int64_t* err,
                       void* stream);

/* ---- K1: Shepard design-matrix assembly ----------------------------------
 * Replaces RbfDictionary.log_features + assemble_features + shepard_normalize
 * = shepard_features (rbf.py:79-91, 123-149).  For every active subdomain s
 * and every row i < N_s, column j < m_cur[s]:
 *   L[i,j] = -(sum_k (x_ik - c_jk)^2) * (1 / (2 w_j^2))   (einsum order, F9)
 *   W[i,j] = exp(L[i,j] - max_j L[i,:]) / sum_j exp(L[i,j] - max_j L[i,:])
 * written column-major into W (see w_off/ld).  `active` may be NULL.
 * mode 0 = Shepard weights W (above); mode 1 = raw exponents L
 * (log_features); mode 2 = raw exp(L) (assemble_features values). */
int pam_assemble_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                     const int64_t* dict_off, const int32_t* m_cur,
                     const double* centres, const double* widths,
                     const int64_t* w_off, const int32_t* ld, const int32_t* active,
                     int32_t max_rows, int mode, double* W, void* stream);

/* Initial dictionaries into capacity slots (DictionarySpec.build /
 * centroid_dictionary, partition.py:96-112, rbf.py:195-214; RbfDictionary
 * generations default 0, rbf.py:28-60): entries src_off[s]..src_off[s+1]-1
 * of the packed source (centres (n, dim), widths or the per-subdomain
 * sigma[s], generations or 0) land in slots dict_off[s].. in order.  For the
 * per-cell dictionary the source is the gathered sample points themselves
 * (src_off = row_off). */
int pam_dict_scatter_f64(int dim, int64_t S, const int64_t* src_off, const double* src_centres,
                         const double* src_widths, const double* sigma, const int32_t* src_gens,
                         const int64_t* dict_off, double* centres, double* widths, int32_t* gens,
                         void* stream);

/* Row normalisation of a row-major (N, M) feature matrix (shepard_normalize,
 * rbf.py:131-144).  mode 1: input holds exponents L -> exp(L - rowmax) /
 * rowsum.  mode 0: input holds raw values -> v / rowsum; a row whose sum is
 * <= 0 reports err {DEGENERATE, row} ("row j ... sums to zero"). */
int pam_row_normalize_f64(int64_t N, int64_t M, const double* in, int mode, double* out,
                          int64_t* err, void* stream);

/* Subdomain batch gather from a structured mesh + make_partition grid
 * (FieldData.subdomain over Partition.boxes, fields.py:61-73,
 * partition.py:41-42, 73-92).  Cells of subdomain s = (sz*py+sy)*px+sx in
 * ascending global index (x fastest) land in rows [row_off[s], row_off[s+1]);
 * centroids are recomputed as lo_k + (i_k + 0.5) * d_k (geometry.py:122-132,
 * bit-identical), values gathered, global cell ids written to cell_idx. */
int pam_gather_cells_f64(int dim, const int64_t* counts, const int32_t* shape,
                         const double* lo, const double* d, const double* values,
                         int64_t S, const int64_t* row_off, double* pts_out,
                         double* vals_out, int64_t* cell_idx_out, void* stream);

/* On-device generator of BASELINE config 5 inputs (the
 * distributions of workloads.config5, counter-based random stream): boxes
 * first_box .. first_box + n_sub - 1 (a rank's shard; the data of a box do
 * not depend on the range) of the gx x gy x ... unit-box tiling (x fastest),
 * n_pts uniform samples
 * per box with values from 1-4 planar interfaces (levels 10^U[-3,3]), and
 * the jittered lx x ly x lz centre lattice per box (M = lx*ly*lz).  DEVICE
 * outputs: points (n_sub*n_pts, 3), values (n_sub*n_pts), centres
 * (n_sub*M, 3). */
int pam_c5_generate_f64(int64_t first_box, int64_t n_sub, int32_t n_pts, int32_t lx, int32_t ly, int32_t lz,
                        int32_t gx, int32_t gy, uint64_t seed, double* points, double* values, double* centres,
                        void* stream);

/* ---- K2b: batched cyclic coordinate descent -------------------------------
 * Replaces fit() + _cd_sweeps_jit (elastic_net.py:66-161) for every active
 * subdomain at once, one warp per subdomain fit, design-matrix columns
 * streamed HBM->SMEM with cp.async.bulk (TMA) + mbarrier.  Residual form:
 *   col_sq = sum_i W_ij^2, denom = col_sq + lam2, r = y - W beta0,
 *   sweeps in fixed order j = 0..M-1, soft threshold, stop when
 *   max|delta| <= tol * max(1, max|beta|) or max_iters sweeps have run.
 * beta (packed like centres, dict_off) is the warm start on entry and the
 * solution on exit.  Outputs per subdomain: sweeps, converged, objective
 * (= history[sweeps-1]).  hist/hist_off may be NULL; otherwise the per-sweep
 * objective of subdomain s is written to hist[hist_off[s] + sweep].
 * `work`: device workspace of pam_cd_workspace_bytes(S, sum N_s, total
 * dictionary slots, max_rows, kernel) bytes (work counter; residual scratch
 * for fits above 8192 rows; block descriptors and diagonal Gram blocks for
 * PAM_CD_BLOCK).  Fits of up to 8192 rows keep the residual in registers (one
 * warp, or a group of 4-8 warps when there are fewer than 4 fits per SM). */
int64_t pam_cd_workspace_bytes(int64_t S, int64_t total_rows, int64_t total_slots, int32_t max_rows,
                               int32_t kernel);
int pam_cd_f64(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
               const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
               const int32_t* ld, const double* W, const double* lam1, const double* lam2,
               const double* tol, const int32_t* max_iters, const int32_t* active,
               int32_t max_rows, double* beta, double* col_sq, int32_t* sweeps,
               int32_t* converged, double* objective, double* hist, const int64_t* hist_off,
               void* work, void* stream);
/* `order` (nullable): processing order of the S subdomains (longest first
 * balances the ragged batch); results do not depend on it.
 * pam_cd_ex_f64 adds `flags`: 1 = col_sq given (not recomputed), 2 = y holds
 * the initial residual r (no warm-start pass), 4 = write the final residual
 * back into y.  The host seam below uses 1|2|4. */
int pam_cd_ex_f64(int64_t S, const int64_t* order, const int64_t* row_off, double* y,
                  const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
                  const int32_t* ld, const double* W, const double* lam1, const double* lam2,
                  const double* tol, const int32_t* max_iters, const int32_t* active,
                  int32_t max_rows, double* beta, double* col_sq, int32_t* sweeps,
                  int32_t* converged, double* objective, double* hist, const int64_t* hist_off,
                  int flags, void* work, void* stream);

/* ---- K1t + K2b-tiles: tile-packed design matrices and their CD ------------
 * Same W as pam_assemble_f64 (mode 0) but stored for the CD stream as
 * column-major 32-row tiles in the row order perm (position p -> local row
 * perm[row_off[s] + p]; NULL = identity), keeping only tiles holding an entry
 * >= tau (tau = 0 keeps all).  tile_mask[slot] bit k = tile k stored;
 * col_off[slot] = column offset (doubles) inside the subdomain's packed block
 * at W + w_off[s]; packed_total[s] = doubles stored.  rowmax/rowsum are
 * per-row scratch (sum N_s doubles each); total_slots = size of the slot
 * arrays.  Requires N_s <= 1024.  Each column's mask is closed to ONE
 * contiguous run of tiles (holes stored as their exact small values).
 * pam_cd_tiles_f64 is pam_cd_f64 over that layout: one cp.async.bulk of
 * popcount(mask)*256 bytes per column; y is read through perm; max_m = the
 * largest m_cur of the batch (host-known; sizes the few-fit kernel's
 * staging).  kernel = PAM_CD_AUTO: 257-1024-row fits with <= 2 fits per SM
 * run the exact blocked CD (a CTA per fit: block dots, in-block updates
 * through the diagonal Gram block, one block AXPY, pipelined across blocks
 * with the previous-block Gram block), with <= 3 fits per SM the
 * column-pair kernel, 257-512-row fits with
 * >= 8 fits per SM two fits per warp, everything else one fit per warp;
 * results are the same either way up to dot-product rounding.  `work` as for
 * pam_cd_f64 (sized with the same `kernel`). */
int pam_assemble_tiles_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                           const int32_t* perm, const int64_t* dict_off, const int32_t* m_cur,
                           const double* centres, const double* widths, const int64_t* w_off,
                           const int32_t* active, int32_t max_rows, double tau, double* rowmax,
                           double* rowsum, uint64_t* tile_mask, int64_t* col_off,
                           int64_t* packed_total, int64_t total_slots, double* W, void* stream);
int pam_cd_tiles_f64(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
                     const int32_t* perm, const int64_t* dict_off, const int32_t* m_cur,
                     const int64_t* w_off, const uint64_t* tile_mask, const int64_t* col_off,
                     const double* W, const double* lam1, const double* lam2, const double* tol,
                     const int32_t* max_iters, const int32_t* active, int32_t max_rows,
                     int32_t max_m, double* beta, double* col_sq, int32_t* sweeps,
                     int32_t* converged, double* objective, double* hist, const int64_t* hist_off,
                     int32_t kernel, void* work, void* stream);

/* ---- K2 + K2b': Gram products and the Gram-form CD (M < N) -----------------
 * pam_gram_f64: G_s = W_s^T W_s (symmetric, column-major at G + g_off[s],
 * leading dimension ldg[s]), q = W^T y and col_sq = diag(G) per dictionary
 * slot, from the dense design matrices of pam_assemble_f64.
 * pam_cd_gram_f64: the reference's cyclic CD (elastic_net.py:113-161) in
 * covariance form c = q - G beta: z = col_sq_j beta_j + c_j, c -= d G[:, j];
 * same decisions and stop rule, M*M doubles streamed per sweep (vs N*M).
 * Writes beta, sweeps, converged (the objective is then evaluated exactly by
 * pam_cd_f64 with max_iters = 0, which computes 0.5|y - W beta|^2 + ...).
 * Requires M <= 3072 (> 512 only sensible for <= 1 fit per SM).  `work`: the
 * CD workspace (its first 4 bytes hold the work counter). */
int pam_gram_f64(int64_t S, const int64_t* row_off, const int32_t* m_cur, const int64_t* dict_off,
                 const int64_t* w_off, const int32_t* ld, const int64_t* g_off, const int32_t* ldg,
                 const int32_t* active, int32_t max_m, const double* W, const double* y,
                 double* G, double* q, double* col_sq, void* stream);
int pam_cd_gram_f64(int64_t S, const int64_t* order, const int64_t* dict_off, const int32_t* m_cur,
                    const int64_t* g_off, const int32_t* ldg, const double* G, const double* q,
                    const double* col_sq, const double* lam1, const double* lam2,
                    const double* tol, const int32_t* max_iters, const int32_t* active,
                    int32_t max_m, double* beta, int32_t* sweeps, int32_t* converged,
                    void* work, void* stream);

/* ---- K3: residual indicators + L2 misfit parts -----------------------------
 * Replaces residual_indicators (adaptive.py:133-138) with cell_quadrature
 * (geometry.py:204-224) and l2_misfit_parts (fields.py:113-121).  For each
 * active subdomain: R[i] = sum_l w_l (K*(x_i + off_l) - K_i)^2 with
 * K* = exp(shepard_eval) when log_flag, and parts[2s] = num, parts[2s+1] =
 * sum(w) * sum(K_i^2), rmax[s] = max_i R[i].  quad_order in {1, 2}. */
int pam_residual_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                     const double* values, const int64_t* dict_off,
                     const int32_t* m_cur, const double* centres,
                     const double* widths, const double* beta,
                     const int32_t* quad_order, const double* qoff, const double* qw,
                     int32_t log_flag, const int32_t* active, int32_t max_rows,
                     double* R, double* parts, double* rmax, int64_t* err, void* stream);
/* qoff: ((1 + 2^dim), dim) quadrature offsets from the centroid, row 0 the
 * order-1 point (zeros), rows 1.. the order-2 tensor Gauss points in the
 * reference's meshgrid('ij') order; qw: matching weights (cell measure / n_q).
 * Both are built on the host with the reference's own expressions. */

/* ---- K3b: stable top-K marking (adaptive.py:141-152) ----------------------
 * marked[s*kcap + t] = t-th cell (local row index) of subdomain s in
 * lexsort((idx, -R)) order restricted to R > 0, t < k_top[s]; n_marked[s]. */
int pam_mark_f64(int64_t S, const int64_t* row_off, const double* R,
                 const int32_t* k_top, const int32_t* active, int32_t kcap,
                 int32_t* marked, int32_t* n_marked, void* stream);

/* ---- K3c: enrichment (adaptive.py:155-210) --------------------------------
 * For marked cell t of subdomain s: parent = lexsort((idx, width, d2))[0]
 * with d2 = np.sum order, width = eta * w_parent, candidates
 * clamp(x_T + off_q * cell_size) dropped when an EXISTING entry matches to
 * <= 1e-12 on every coordinate and the width.  Survivors are appended in
 * (marked, offset) order at slot m_cur[s] onwards with generation `gen`;
 * beta of new slots is zeroed; m_cur[s] and n_added[s] are updated.
 * offsets: (S, mq_cap, dim) packed, m_q[s] used per subdomain.  A
 * subdomain whose survivors would overflow dict_cap reports
 * err {UNSUPPORTED, s} and adds nothing.
 * box_lo/box_hi: (S, dim). */
int pam_enrich_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                   const int32_t* marked, const int32_t* n_marked, int32_t kcap,
                   const double* eta, const int32_t* m_q, int32_t mq_cap,
                   const double* offsets, const double* cell_size,
                   const double* box_lo, const double* box_hi,
                   const int64_t* dict_off, const int32_t* dict_cap, int32_t* m_cur,
                   double* centres, double* widths, int32_t* gens, double* beta,
                   int32_t gen, const int32_t* active, int32_t* n_added,
                   int64_t* err, void* stream);

/* ---- K4: global evaluation ------------------------------------------------
 * Replaces GlobalSurrogate.evaluate (partition.py:132-143) = locate_many
 * (geometry.py:242-258) + LocalSurrogate.evaluate (rbf.py:152-192).
 * Boxes form a tensor grid: edges_k (shape[k]+1 values per axis, host-
 * identical to partition.py:59), open upper faces except the last box per
 * axis.  owner = (sz*py + sy)*px + sx.  Points outside -> err {OUTSIDE, j}.
 * out[j] = exp(v_j) (log_flag) or v_j, in input order.  `work` is scratch of
 * pam_eval_workspace_bytes(P, S) bytes. */
int64_t pam_eval_workspace_bytes(int64_t P, int64_t S);
int pam_locate_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                   const double* edges, int64_t* owner, int64_t* err, void* stream);
int pam_eval_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                 const double* edges, int64_t S, const int64_t* dict_off,
                 const int32_t* m_cur, const double* centres, const double* widths,
                 const double* beta, const int32_t* log_flag, double* out,
                 void* work, int64_t* err, void* stream);

/* The same for ARBITRARY half-open boxes (geometry.py:54-66, 242-258, the
 * reference's locate_many accepts any box set): box i = [lo, hi) per axis, the
 * upper face closed where box_open[i*dim + k] == 0; owner = the first box, in
 * order, containing the point.  Errors as the reference raises them: a point
 * inside two boxes -> err {CLAIMED, second box << 40 | point} (the first box,
 * in order, that re-claims a point; checked before coverage), a point in no
 * box -> err {OUTSIDE, j}.  S < 2^23, P < 2^40.  pam_locate_boxes_f64 needs
 * 16 bytes of scratch in `work`; pam_eval_boxes_f64 the scratch of
 * pam_eval_workspace_bytes(P, S). */
int pam_locate_boxes_f64(int dim, int64_t P, const double* pts, int64_t S,
                         const double* box_lo, const double* box_hi,
                         const int32_t* box_open, int64_t* owner, void* work,
                         int64_t* err, void* stream);
int pam_eval_boxes_f64(int dim, int64_t P, const double* pts, const double* box_lo,
                       const double* box_hi, const int32_t* box_open, int64_t S,
                       const int64_t* dict_off, const int32_t* m_cur,
                       const double* centres, const double* widths, const double* beta,
                       const int32_t* log_flag, double* out, void* work, int64_t* err,
                       void* stream);

/* Shepard evaluation of ONE dictionary at P points (rbf.py:152-167):
 * out[j] = (sum_m e_jm beta_m) / (sum_m e_jm), e = exp(L - rowmax). */
int pam_shepard_eval_f64(int dim, int64_t P, const double* pts, int64_t M,
                         const double* centres, const double* widths,
                         const double* beta, int32_t exp_out, double* out,
                         int64_t* err, void* stream);

/* FP64 pipe probe: launches 4*SMs x 256 threads, each running 8 independent
 * DFMA chains of `iters` steps (2 flops per DFMA); the caller times it to get
 * the measured FP64 peak (roofline denominator for the FP64-bound kernels). */
int pam_probe_fp64(int64_t iters, double* out, void* stream);

/* ---- host-pointer synchronous seams (drop-in for the reference) ---------- */

/* Exact signature of _cd_sweeps_jit (elastic_net.py:113): W is the (n, m)
 * Fortran-ordered design matrix, beta/r/history are updated in place.
 * Returns status; *sweeps, *converged receive the loop's return tuple. */
int pam_cd_sweeps_host_f64(const double* W_fortran, int64_t n, int64_t m,
                           const double* col_sq, const double* denom, double lam1,
                           double lam2, double tol, int64_t max_iters, double* beta,
                           double* r, double* history, int64_t* sweeps,
                           int32_t* converged);

/* shepard_eval(points, dictionary, beta) (rbf.py:152-167) on host arrays;
 * *err_index receives the first offending point on PAM_ERR_DEGENERATE. */
int pam_shepard_eval_host_f64(int dim, int64_t P, const double* pts, int64_t M,
                              const double* centres, const double* widths,
                              const double* beta, double* out, int64_t* err_index);

/* Surrogate text format fast path (partition.py:220-247 `save`): n entry
 * lines "<centre coords> <width> <beta> <generation>\n", reals as %.17g.
 * Returns bytes written into out[cap], or -1 when cap is too small. */
int64_t pam_format_entries_host(int dim, int64_t n, const double* centres, const double* widths,
                                const double* beta, const int64_t* gens, char* out, int64_t cap);

/* ---- Darcy consumer (reference darcy.py:238-375) -------
 * pam_p1_values_f64: CSR values of the P1 stiffness matrix (darcy.py:308-346
 * dim 2, 349-375 dim 1).  slot_ptr (nnz+1) / contrib list, per nonzero, the
 * element contributions c = e*9 + 3i + j (dim 2) or e*4 + 2i + j (dim 1) in
 * the reference's COO order; values are summed in that order (bit-identical
 * to its COO -> CSR sum).  elem_nodes (n_elem, dim+1), nodes (n_nodes, dim),
 * coef (n_elem) = coefficient at element centroids (validated by the caller).
 * pam_csr_spmv_f64: y = A x.
 * pam_pcg_f64: scipy.sparse.linalg.cg with M = diag(1/a_ii) (1 where
 * a_ii <= 0), x0 = 0, stop when ||r|| < rtol ||b|| (darcy.py:275-289); work
 * = pam_pcg_workspace_bytes(n) bytes of device memory.  Returns the completed
 * iterations, converged (0 = max_iter reached) and the recursive residual
 * ratio; fixed-order reductions (deterministic). */
int pam_p1_values_f64(int dim, int64_t nnz, const int64_t* slot_ptr, const int64_t* contrib,
                      const int64_t* elem_nodes, const double* nodes, const double* coef,
                      double* values, void* stream);
int pam_csr_spmv_f64(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                     const double* x, double* y, void* stream);
int64_t pam_pcg_workspace_bytes(int64_t n);
int pam_pcg_f64(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                const double* b, double* x, double rtol, int64_t max_iter, void* work,
                int64_t* iterations, int32_t* converged, double* rel_residual, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PAM_B200_H */
