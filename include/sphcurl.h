/*
 * sphcurl.h -- C ABI of libsphcurl.so, the B200 (sm_100a) kernels behind the
 * SpHcurlAMG setup + solve hot path (arxiv 2506.08284).
 *
 * The reference has no FFI: its boundary is the Python API
 *   build_hierarchy(A_e, S_e, A_n, D, cfg)      multigrid.py:119
 *   v_cycle_preconditioner(h)                    multigrid.py:191
 *   pcg_solve(A, b, precond, rtol, maxit)        multigrid.py:220
 *   build_edge_prolongator(A_n, A_e, S, D_h, cfg) edge_prolongator.py:184
 * which paper_2506_08284_b200/{multigrid,edge_prolongator}.py mirror (same
 * names, arguments, dataclass fields and ValueError texts). Every numeric call
 * those mirrors make lands here. Each entry point below names the reference
 * function (file:line) whose arithmetic it replaces.
 *
 * Conventions
 *  - Plain device pointers and sizes; no torch types. CSR = int64 row
 *    pointers, int32 column indices, fp64 values. Vectors are fp64.
 *  - `stream` is a cudaStream_t; every call is stream ordered and asynchronous
 *    unless documented otherwise. Scratch is stream-ordered (cudaMallocAsync).
 *  - Return 0 on success, a negative SPHC_ERR_* on a launch / argument error
 *    (message in sphc_last_error()).
 *  - Data-dependent failures (the reference's ValueErrors) are written to a
 *    caller-owned device array `status` of SPHC_STATUS_SLOTS int64 entries,
 *    initialised to INT64_MAX: slot k receives the lowest row that failed
 *    check k (SPHC_ST_*). The caller re-raises with the reference's message.
 */
#ifndef SPHCURL_H
#define SPHCURL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHC_OK 0
#define SPHC_ERR_CUDA (-1)
#define SPHC_ERR_ARG (-2)
#define SPHC_ERR_HOST (-3)

#define SPHC_STATUS_SLOTS 32
#define SPHC_ST_ZERO_DIAG 0        /* multigrid.py:38-40  zero diagonal entry in row r   */
#define SPHC_ST_NONPOS_DIAG 1      /* nodal_amg.py:41-43  nonpositive diagonal entry     */
#define SPHC_ST_NODAL_ZERO_DIAG 2  /* nodal_amg.py:147-148 zero diagonal in nodal operator */
#define SPHC_ST_ZERO_ROWSUM 3      /* nodal_amg.py:131-133 zero row sum before scaling   */
#define SPHC_ST_MALFORMED_GRAD 4   /* emin_setup.py:71-74 malformed gradient             */
#define SPHC_ST_EMPTY_I 5          /* emin_setup.py:292   row with empty prolongator pattern */
#define SPHC_ST_REDUCIBLE 6        /* emin_setup.py:304   block needs make_irreducible   */
#define SPHC_ST_RANK_LOW 7         /* emin_setup.py:233-237 rank below expected          */
#define SPHC_ST_EMIN_CAPACITY 8    /* row exceeds the emin kernel's |J|<=16, |I|<=128    */
#define SPHC_ST_EMPTY_J 9          /* emin_setup.py:125-127 empty constraint pattern     */
#define SPHC_ST_SPGEMM_CAPACITY 10 /* SpGEMM row exceeds the on-chip accumulator         */
#define SPHC_ST_SORT_CAPACITY 11   /* segmented sort row too long                        */
#define SPHC_ST_TRSV_STALL 12      /* triangular sweep dependency never resolved (bug)   */
#define SPHC_ST_PC_EMPTY_COLUMN 13 /* coarse_gradient.py:49-52 empty column (col id)     */
#define SPHC_ST_PC_EMPTY_ROW 14    /* coarse_gradient.py:82-83 row with no entries       */
#define SPHC_ST_PC_NO_DONOR 15     /* coarse_gradient.py:96-98 empty column after safeguard */
#define SPHC_ST_AGG_CAPACITY 16    /* aggregation row longer than the device kernel's buffer */
#define SPHC_ST_PC_NO_FIXPOINT 17  /* Algorithm 1 claiming pass did not converge (internal) */

/* emin constraint blocks: the on-chip default class (4 rows per CTA) and the
 * wide class its overflow rows are re-run through (one row per CTA); beyond
 * the wide class -> SPHC_ST_EMIN_CAPACITY */
#define SPHC_EMIN_JMAX 16
#define SPHC_EMIN_IMAX 128
#define SPHC_EMIN_JWIDE 32 /* one lane per coarse node                          */
#define SPHC_EMIN_IWIDE 592 /* 496 node pairs + 32 single-node edges + appended */
#define SPHC_DIMS_I 129 /* subproblem_dims histogram is [SPHC_DIMS_I][SPHC_DIMS_J] */
#define SPHC_DIMS_J 17

const char *sphc_last_error(void);
int sphc_abi_version(void);
/* number of kernels this library has launched in this process */
int64_t sphc_launch_count(void);

/* ---------------------------------------------------------------- primitives */

/* Exclusive scan of n counts into n+1 offsets (offsets[n] = total). Builds
 * every CSR row pointer (reference: scipy indptr construction). */
int sphc_scan_i64(int64_t n, const int64_t *counts, int64_t *offsets, void *stream);

/* *out = sum x_i y_i with a fixed two-pass tree (deterministic).
 * Replaces numpy dot in pcg_solve (multigrid.py:229,236,243,258,266). */
int sphc_dot(int64_t n, const double *x, const double *y, double *out, void *stream);

/* *out = sum x_i (fixed two-pass tree). Energies (edge_prolongator.py:154-156). */
int sphc_sum(int64_t n, const double *x, double *out, void *stream);

/* *out = max |x_i| (0 for n = 0). sparse_ops.py:116-119 max_abs. */
int sphc_maxabs(int64_t n, const double *x, double *out, void *stream);

/* *out = x . y in the OpenBLAS-Haswell ddot order (16 FMA chains, fixed
 * combine, plain tail): bit-identical to np.linalg.norm's dot under the
 * survey's BLAS pin. estimate_rho, nodal_amg.py:106-111. */
int sphc_hsw_dot(int64_t n, const double *x, const double *y, double *out, void *stream);

/* v = w / sqrt(*sq) elementwise (IEEE); writes sqrt(*sq) to *norm_out.
 * nodal_amg.py:107-115 (v /= norm). */
int sphc_scale_by_norm(int64_t n, const double *w, const double *sq, double *v,
                       double *norm_out, void *stream);

/* y = 1 / x elementwise, IEEE division (diags(1.0 / d), nodal_amg.py:150,
 * edge_prolongator.py:173). When zero_sub != NULL, zero entries of x are
 * replaced by *zero_sub first (_jacobi_diag, edge_prolongator.py:159-167). */
int sphc_reciprocal(int64_t n, const double *x, const double *zero_sub, double *y,
                    void *stream);

/* out_i = x[idx_i] (halo send staging of the partitioned solve). */
int sphc_gather(int64_t n, const int64_t *idx, const double *x, double *out, void *stream);

/* y = a x + b y */
int sphc_axpby(int64_t n, double a, const double *x, double b, double *y, void *stream);

/* ---------------------------------------------------------------- CSR utilities */

/* d_i = A_ii (0 if not stored); flags zero diagonals into status[ZERO_DIAG]
 * when status != NULL. multigrid.py:36-40, nodal_amg.py:40-43. */
int sphc_csr_diag(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                  double *d, int64_t *status, void *stream);

/* Sort every row of a CSR by column (stable for equal keys is not needed:
 * keys are unique per row), carrying fp64 values when v != NULL. */
int sphc_csr_sort_rows(int64_t n, const int64_t *rp, int32_t *ci, double *v,
                       int64_t *status, void *stream);

/* Transpose with sorted output rows (ascending original row index) -- the
 * CSC view scipy builds for A.T @ B (multigrid.py:150-152, coarse_gradient.py:46). */
int sphc_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t *rp,
                       const int32_t *ci, const double *v, int64_t *trp, int32_t *tci,
                       double *tv, int64_t *status, void *stream);

/* counts_i = number of nonzero stored values in row i */
int sphc_csr_count_nonzero(int64_t n, const int64_t *rp, const double *v, int64_t *counts,
                           void *stream);

/* C = alpha A + beta B on the union pattern of two canonical CSR matrices
 * (scipy csr_binop_csr, e.g. commutator_residual's P_e D_H - R_dp,
 * edge_prolongator.py:179-181): count pass, scan, fill. */
int sphc_csr_add_count(int64_t n, const int64_t *arp, const int32_t *aci, const int64_t *brp,
                       const int32_t *bci, int64_t *counts, void *stream);
int sphc_csr_add_fill(int64_t n, const int64_t *arp, const int32_t *aci, const double *av,
                      const int64_t *brp, const int32_t *bci, const double *bv, double alpha,
                      double beta, const int64_t *crp, int32_t *cci, double *cv, void *stream);

/* Drop exact zeros (sparse_ops.py:107-113 compress(A, 0)). new_rp from
 * sphc_csr_count_nonzero + sphc_scan_i64. */
int sphc_csr_compact(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                     const int64_t *new_rp, int32_t *nci, double *nv, void *stream);

/* out = dense row-major copy of A (coarsest level, multigrid.py:157 toarray) */
int sphc_csr_to_dense(int64_t n_rows, int64_t n_cols, const int64_t *rp, const int32_t *ci,
                      const double *v, double *out, void *stream);

/* ---------------------------------------------------------------- SpGEMM */

/* Structural nnz of each row of C = A B (unique columns). */
int sphc_spgemm_count(int64_t n, const int64_t *arp, const int32_t *aci, const int64_t *brp,
                      const int32_t *bci, int64_t *counts, int64_t *status, void *stream);

/* Numeric C = A B on the structural pattern, columns ascending.
 * ordered != 0: every entry is a sequential sum over k ascending of
 *   a_ik * b_kj with no FMA -- scipy csr_matmat's order, bit-identical for the
 *   nodal Galerkin product (multigrid.py:152).
 * ordered == 0: all lanes busy (sorted 32-product chunks, fixed shuffle-tree
 *   reduction); deterministic, TOL class. Used for the edge Galerkin products
 *   (:150-151), D^T A D (:103) and the null-space check (:111).
 * max_cols = the longest output row (max of the count pass; -1 if unknown):
 *   <= 64 selects a small-footprint, higher-occupancy variant. */
int sphc_spgemm_fill(int64_t n, const int64_t *arp, const int32_t *aci, const double *av,
                     const int64_t *brp, const int32_t *bci, const double *bv,
                     const int64_t *crp, int32_t *cci, double *cv, int ordered,
                     int64_t max_cols, int64_t *status, void *stream);

/* Two products on one pattern in one pass: C1 = A1 B1, C2 = A2 B2 where A1/A2
 * share arp/aci and B1/B2 share brp/bci (the A_e and S_e Galerkin products
 * P^T (A_e P) and P^T (S_e P), multigrid.py:150-151). Unordered (TOL). */
int sphc_spgemm_fill_pair(int64_t n, const int64_t *arp, const int32_t *aci, const double *av1,
                          const double *av2, const int64_t *brp, const int32_t *bci,
                          const double *bv1, const double *bv2, const int64_t *crp,
                          int32_t *cci, double *cv1, double *cv2, int64_t max_cols,
                          int64_t *status, void *stream);

/* Thin products (rows with few products and <= 32 distinct output columns:
 * A_e D, S_e D, D^T (A D) -- csr_matmat call sites multigrid.py:103,111): one
 * thread per output row with a private hash table in shared memory, products
 * in scipy's order (bitwise csr_matmat). sphc_spgemm_count_thin counts every
 * row (rows beyond 32 columns through the warp kernel; any_over: 1-int device
 * scratch). sphc_spgemm_fill_thin fills every row: av2 / bv2 / cv2 non-NULL =
 * the pair product on one pattern; `ordered` picks the warp kernels' ordered
 * sums for the rows beyond 32 columns; max_cols as in sphc_spgemm_fill. */
int sphc_spgemm_count_thin(int64_t n, const int64_t *arp, const int32_t *aci,
                           const int64_t *brp, const int32_t *bci, int64_t *counts,
                           int32_t *any_over, int64_t *status, void *stream);
int sphc_spgemm_fill_thin(int64_t n, const int64_t *arp, const int32_t *aci, const double *av1,
                          const double *av2, const int64_t *brp, const int32_t *bci,
                          const double *bv1, const double *bv2, const int64_t *crp,
                          int32_t *cci, double *cv1, double *cv2, int ordered,
                          int64_t max_cols, int64_t *status, void *stream);

/* Long-row variants (one CTA of 8 warps per output row) for products whose A
 * rows are long: the Galerkin R (A P) with R = P_e^T (150-2000 entries per
 * row, multigrid.py:150-151). Same outputs and capacity rule (<= 256 columns
 * per row) as sphc_spgemm_count / sphc_spgemm_fill(_pair), unordered (TOL);
 * av2 / bv2 / cv2 NULL for a single product. */
int sphc_spgemm_count_long(int64_t n, const int64_t *arp, const int32_t *aci,
                           const int64_t *brp, const int32_t *bci, int64_t *counts,
                           int64_t *status, void *stream);
int sphc_spgemm_fill_long(int64_t n, const int64_t *arp, const int32_t *aci, const double *av,
                          const double *av2, const int64_t *brp, const int32_t *bci,
                          const double *bv, const double *bv2, const int64_t *crp,
                          int32_t *cci, double *cv1, double *cv2, void *stream);

/* make_irreducible's main loop on the device (emin_setup.py:183-217,
 * 283-301): one warp per listed fine edge rows[r]; its coarse-node graph (J
 * from T, original pattern edges from prp/pci with endpoints ep_a/ep_b) is
 * joined greedily by the largest |R_dp[:, a] . R_dp[:, b]| over bridging
 * pairs (columns of R_dp = T^T in ttrp/ttci/ttv, summed in ascending fine
 * edge, unfused; ties: smallest (a, b)). ncnt[r] = number of joins, their
 * (a, b) in pairs[2 * (31 r + j)]; -1 single-node graph, -2 |J| > 32. */
int sphc_emin_repair(int64_t nrows, const int64_t *rows, const int64_t *trp, const int32_t *tci,
                     const int64_t *prp, const int32_t *pci, const int32_t *ep_a,
                     const int32_t *ep_b, const int64_t *ttrp, const int32_t *ttci,
                     const double *ttv, int32_t *ncnt, int32_t *pairs, int64_t *status,
                     void *stream);

/* ---------------------------------------------------------------- solve */

/* y = alpha * (A x) + beta * z  (z may be NULL; y may alias z).
 * `lanes` (1,2,4,8,16,32) = lanes per row; 256 = one CTA per row (few,
 * long rows: the explicit restrictions R = P_e^T of the coarse levels,
 * fixed-order block reduction). csr_matvec call sites
 * multigrid.py:46,51,168,171,183,186,242,252. */
int sphc_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v, int lanes,
              const double *x, double alpha, double beta, const double *z, double *y,
              void *stream);

/* SELL-32 mirror of a CSR operator (slices of 32 rows, column-major, padded
 * with value 0 / own column). sphc_sell_sizes writes the entry count of every
 * slice (ceil(n/32) values); after sphc_scan_i64 -> slice_ptr, sphc_sell_fill
 * writes the slices. */
int sphc_sell_sizes(int64_t n, const int64_t *rp, int64_t *slice_entries, void *stream);
int sphc_sell_fill(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   const int64_t *slice_ptr, int32_t *sci, double *sv, void *stream);
/* Delta-coded columns of a SELL mirror for the streamed operators: d16 holds
 * each stored entry's column as a 16-bit difference to the previous entry of
 * its row (SELL positions; padding: 0), c0 the row's 32-bit bases: nbase = 1,
 * the first column; nbase = 4, up to three more, a difference code 0xFFFF
 * meaning "this entry's column is the row's next base" (a jump beyond 16
 * bits: the next mesh plane at 256^3). *too_big is set when a row needs more
 * (the caller then keeps the 32-bit columns). rect = 1: an empty row's
 * column is 0, not the row index (A D). sphc_sell_spmv16 /
 * sphc_sell_cheb_step16 / sphc_sell_hipt_mid16: the same arithmetic as
 * sphc_sell_spmv / sphc_sell_cheb_step / sphc_sell_hipt_mid (bitwise) on 10
 * instead of 12 bytes per stored entry; one warp per slice (operators of at
 * least 148 * 48 slices). */
int sphc_sell_fill16(int64_t n, const int64_t *rp, const int32_t *ci, const int64_t *slice_ptr,
                     uint16_t *d16, int32_t *c0, int32_t *too_big, int rect, int nbase,
                     void *stream);
int sphc_sell_hipt_mid16(int64_t n, const int64_t *slice_ptr, const uint16_t *d16,
                         const int32_t *c0, const double *sv, const int64_t *drp,
                         const int32_t *dci, const double *dv, const double *dinv,
                         const double *r, const double *c, const double *x_in, double *x_out,
                         double *d, double cr, int nbase, void *stream);
int sphc_sell_spmv16(int64_t n, const int64_t *slice_ptr, const uint16_t *d16, const int32_t *c0,
                     const double *sv, const double *x, double alpha, double beta,
                     const double *z, double *y, int nbase, void *stream);
int sphc_sell_cheb_step16(int64_t n, const int64_t *slice_ptr, const uint16_t *d16,
                          const int32_t *c0, const double *sv, const double *dinv,
                          const double *b, const double *x_in, double *x_out, double *d,
                          double cd, double cr, int nbase, void *stream);
/* SELL fill for a rectangular operator (A_e D): padding entries repeat the
 * row's first column (0 for an empty row) instead of the row index. */
int sphc_sell_fill_rect(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                        const int64_t *slice_ptr, int32_t *sci, double *sv, void *stream);
/* Hiptmair mid step (hiptmair_smooth, multigrid.py:164-173): the nodal
 * correction x + D c and the first Chebyshev step of the second edge sweep
 * from the residual r = b - A x already held, b - A (x + D c) = r - (A D) c:
 *   d = cr dinv (r - (A D) c);  x_out = (x + D c) + d
 * (slice_ptr, sci, sv) = SELL mirror of A D (sphc_sell_fill_rect), (drp, dci,
 * dv) = CSR of D. Replaces one D pass and one A_e pass by one A D pass. */
int sphc_sell_hipt_mid(int64_t n, const int64_t *slice_ptr, const int32_t *sci,
                       const double *sv, const int64_t *drp, const int32_t *dci,
                       const double *dv, const double *dinv, const double *r,
                       const double *c, const double *x_in, double *x_out, double *d,
                       double cr, int64_t padded, void *stream);
/* y = alpha A x + beta z on the SELL mirror, one thread per row. `padded` =
 * stored entries (slice_ptr[n_slices]); operators above 48 MB are read with
 * evict-first loads, smaller ones stay L2-resident across the V-cycle. */
int sphc_sell_spmv(int64_t n, const int64_t *slice_ptr, const int32_t *sci, const double *sv,
                   const double *x, double alpha, double beta, const double *z, double *y,
                   int64_t padded, void *stream);
/* Fused Chebyshev step on the SELL mirror (same math as sphc_cheb_step). */
int sphc_sell_cheb_step(int64_t n, const int64_t *slice_ptr, const int32_t *sci,
                        const double *sv, const double *dinv, const double *b,
                        const double *x_in, double *x_out, double *d, double cd, double cr,
                        int x_zero, int64_t padded, void *stream);

/* One Chebyshev step, fused: d <- cd*d + cr*dinv*(b - A x_in); x_out = x_in + d.
 * x_zero != 0 means x_in == 0 (A x skipped). Replaces the reference's
 * Gauss-Seidel half sweeps (multigrid.py:45-59) in the smoother seam. */
int sphc_cheb_step(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   int lanes, const double *dinv, const double *b, const double *x_in,
                   double *x_out, double *d, double cd, double cr, int x_zero, void *stream);

/* One Gauss-Seidel half sweep of the reference's symmetric smoother
 * (multigrid.py:45-59): x_out = x_in + T^-1 (b - A x_in), T = tril(A)
 * (lower != 0) or triu(A) (lower == 0), read from the full CSR of A.
 * Sync-free substitution: a warp per row, rows claimed in dependency order
 * from *ticket; y (n doubles) is the solve's workspace, reset to a NaN
 * sentinel inside the call. x_in == NULL means x_in = 0. Zero diagonal rows
 * are reported in status[SPHC_ST_ZERO_DIAG]. */
int sphc_gs_half_sweep(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                       const double *b, const double *x_in, double *x_out, double *y,
                       int32_t *ticket, int lower, int64_t *status, void *stream);

/* y_i = d_i x_i (Jacobi scaling in the smoother's power iteration). */
int sphc_diag_scale(int64_t n, const double *d, const double *x, double *y, void *stream);

/* Deterministic start vector in [-1, 1) for the smoother's spectral bound
 * (splitmix64 of the index; oracle.cheb_start_vector computes the same). */
int sphc_cheb_start(int64_t n, double *x, void *stream);
/* One Lanczos step of the Chebyshev bound estimate (no reference
 * counterpart; the reference smoother is Gauss-Seidel, multigrid.py:32-66):
 * w = D^-1 u - alpha v - beta_prev v_prev (beta_prev == NULL: first step),
 * dw = D w; alpha, beta_prev are device scalars. */
int sphc_lanczos_update(int64_t n, const double *u, const double *dinv, const double *d,
                        const double *v, const double *vprev, const double *alpha,
                        const double *beta_prev, double *w, double *dw, void *stream);

/* PCG scalar slots of the device array `sc` (multigrid.py:220-274). */
#define SPHC_PCG_PAP 0  /* p . Ap        */
#define SPHC_PCG_RR 1   /* r . r         */
#define SPHC_PCG_RZ 2   /* r . z (current) */
#define SPHC_PCG_RZN 3  /* r . z (new)   */

/* alpha = sc[RZ] / sc[PAP]; if sc[PAP] > 0: x += alpha p, r -= alpha Ap and
 * *changed = 1 if any x_i changed (multigrid.py:244-257: the indefinite and
 * array_equal stagnation tests). No-op when p.Ap <= 0. */
int sphc_pcg_update(int64_t n, const double *sc, const double *p, const double *Ap, double *x,
                    double *r, int32_t *changed, void *stream);

/* sphc_pcg_update fused with sc[RR] = r . r of the updated residual, summed
 * exactly as sphc_dot(n, r, r) does (same grid, same order: bitwise equal).
 * sc[RR] is left untouched when p.Ap <= 0. */
int sphc_pcg_update_rr(int64_t n, double *sc, const double *p, const double *Ap, double *x,
                       double *r, int32_t *changed, void *stream);

/* p = z + (sc[RZN] / sc[RZ]) p (multigrid.py:268-270). */
int sphc_pcg_direction(int64_t n, const double *sc, const double *z, double *p, void *stream);

/* sc[RZ] = sc[RZN] */
int sphc_pcg_rotate(double *sc, void *stream);

/* One PCG iteration (the loop body of multigrid.py:241-270) captured from
 * `stream` into a CUDA graph and replayed per iteration. Plain runtime
 * stream capture (thread-local mode): the captured launches must not
 * allocate. sphc_graph_end writes the instantiated cudaGraphExec_t to
 * exec[0]. */
int sphc_graph_begin(void *stream);
int sphc_graph_end(void **exec, void *stream);
int sphc_graph_launch(void *exec, void *stream);
int sphc_graph_destroy(void *exec);

/* The whole PCG loop as ONE graph launch (device-side iteration control):
 * a WHILE conditional node whose body is captured from `stream` between
 * sphc_pcg_loop_begin and sphc_pcg_loop_end -- one PCG iteration followed by
 * sphc_pcg_check, which evaluates the reference's tests
 * (multigrid.py:244-266) on the device, records |r| and sqrt(r.z) in
 * hist[2 it], hist[2 it + 1], rotates r.z (sphc_pcg_rotate's update, so the
 * body omits that launch), and ends the loop. ctl[0] = rtol |b|,
 * ctl[1] = maxit, ctl[2] = iterations, ctl[3] = status (0 running,
 * 1 converged, 2 maxit, 3 stagnated, 4 indefinite). state[0] receives the
 * loop object. */
int sphc_pcg_loop_begin(void **state, void *stream);
int sphc_pcg_check(void *state, double *sc, double *ctl, double *hist, void *stream);
int sphc_pcg_loop_end(void *state, void *stream);
int sphc_pcg_loop_launch(void *state, int64_t *kernels_per_iteration, void *stream);
int sphc_pcg_loop_add_launches(int64_t n);
int sphc_pcg_loop_destroy(void *state);

/* Page-lock / release a caller's host range in place (uploads then DMA
 * straight from it); register fails (non-sticky) on overlapping ranges. */
int sphc_host_register(void *p, int64_t bytes);
int sphc_host_unregister(void *p);

/* dst (device) <- src (page-locked host), `bytes` bytes, asynchronous. */
int sphc_copy_h2d(void *dst, const void *src, int64_t bytes, void *stream);

/* dst (pinned host) <- src (device), `bytes` bytes, asynchronous on stream
 * (capturable; the PCG scalars' per-iteration readback). */
int sphc_copy_d2h(void *dst, const void *src, int64_t bytes, void *stream);

/* Wait for `stream` (the host side of a readback; other streams, e.g. an
 * upload streaming in behind the setup, keep running). */
int sphc_stream_sync(void *stream);

/* Readback gather: `count` (<= 16) device ranges -- desc holds host rows of
 * 3 int64 (device source pointer, bytes, byte offset into dst; bytes and
 * offsets multiples of 4) -- written by ONE kernel straight into `dst`, a
 * page-locked (device-mapped) host buffer. Replaces one copy-engine
 * transfer per range; visible on the host after sphc_stream_sync. */
int sphc_readback_gather(int32_t count, const int64_t *desc, void *dst, void *stream);

/* nsteps (2 or 3) consecutive Chebyshev steps (sphc_sell_cheb_step
 * semantics, step k: xout_k = xin_k + d, d <- cd_k d + cr_k D^-1 (b - A xin_k))
 * in ONE pass over the SELL matrix: row blocks of 256 in ascending order,
 * step k of a block once step k-1 is done within the matrix bandwidth L
 * (in blocks: ceil(max|col - row| / 256) + 1), so the block's rows are
 * re-read from L2. Bitwise identical to nsteps separate launches.
 * sync: int32 scratch of 1 + nsteps * ceil(n / 256) entries. x_zero applies
 * to step 0. */
int sphc_sell_cheb_fused(int64_t n, const int64_t *slice_ptr, const int32_t *sci,
                         const double *sv, const double *dinv, const double *b, double *d,
                         int nsteps, const double *xin0, double *xout0, double cd0, double cr0,
                         const double *xin1, double *xout1, double cd1, double cr1,
                         const double *xin2, double *xout2, double cd2, double cr2, int x_zero,
                         int L, int32_t *sync, void *stream);

/* *out = max |col - row| over the stored entries of a CSR with sorted rows. */
int sphc_csr_bandwidth(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *out,
                       void *stream);

/* The k-step Lanczos estimate behind the Chebyshev smoother's upper bound
 * (D^-1 A in the D inner product, deterministic start vector) in one
 * cooperative launch on the SELL mirror of A: writes alpha_1..k to sc[0..k)
 * and beta_0..k to sc[k..2k]. v, vprev, w, u are n-vectors of scratch. */
int sphc_lanczos_sell(int64_t n, const int64_t *slice_ptr, const int32_t *sci, const double *sv,
                      const double *d, const double *dinv, int k, double *v, double *vprev,
                      double *w, double *u, double *sc, void *stream);

/* y = A x for a dense row-major n x n A (coarsest level, explicit inverse of
 * the reference's lu_factor/lu_solve pair, multigrid.py:157,181). */
int sphc_dense_gemv(int64_t n, const double *A, const double *x, double *y, void *stream);

/* ---------------------------------------------------------------- nodal chain */

/* Strength pattern rows (nodal_amg.py:33-56): entries with
 * |a_ij| > drop_tol*sqrt(a_ii a_jj), plus the diagonal. Flags nonpositive
 * diagonals. Symmetrised afterwards with sphc_csr_transpose + union. */
int sphc_strength_count(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                        const double *diag, double drop_tol, int64_t *counts,
                        int64_t *status, void *stream);
int sphc_strength_fill(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                       const double *diag, double drop_tol, const int64_t *frp,
                       int32_t *fci, void *stream);
/* C = pattern(A) U pattern(B), sorted rows */
int sphc_pattern_union_count(int64_t n, const int64_t *arp, const int32_t *aci,
                             const int64_t *brp, const int32_t *bci, int64_t *counts,
                             void *stream);
int sphc_pattern_union_fill(int64_t n, const int64_t *arp, const int32_t *aci,
                            const int64_t *brp, const int32_t *bci, const int64_t *crp,
                            int32_t *cci, void *stream);

/* w = (diag(1/d) A) v with every row summed in DESCENDING column order, no FMA
 * -- the storage order scipy gives diags(1/d) @ A (nodal_amg.py:150-151,110). */
int sphc_nodal_powmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                     const double *dinv, const double *x, double *y, void *stream);

/* y_i = sum over row i IN STORAGE ORDER of fl(a_ij x_j), sequential from 0,
 * no FMA: scipy csr_matvec on any row order (estimate_rho(A_scaled),
 * nodal_amg.py:99-116, whose A_scaled rows scipy stores descending). */
int sphc_spmv_stored_order(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                           const double *x, double *y, void *stream);

/* normalize_rows (nodal_amg.py:119-135): out = fl(fl(1 / s_i) a_ij) with
 * s_i = a_i0 + pairwise(a_i1..) (np.add.reduceat); zero-sum rows (|s| <=
 * 1e-13 max(1, sum |a|)) -> status ZERO_ROWSUM; rows longer than 257 ->
 * SPGEMM_CAPACITY. Exact zeros are dropped by the caller (compact). */
int sphc_normalize_rows(int64_t n, const int64_t *rp, const double *v, double *out,
                        int64_t *status, void *stream);

/* Smoothed + normalised nodal prolongator rows (nodal_amg.py:119-155):
 * P = normalize((I - omega D^-1 A) P_tent), bit-faithful (Appendix A). */
int sphc_nodal_smooth_count(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                            const double *dinv, const int64_t *memb, double omega,
                            int64_t *counts, int64_t *status, void *stream);
int sphc_nodal_smooth_fill(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                           const double *dinv, const int64_t *memb, double omega,
                           const int64_t *prp, int32_t *pci, double *pv, int64_t *status,
                           void *stream);

/* ---------------------------------------------------------------- coarse topology */

/* Coarse edges (coarse_gradient.py:106-136): for every fine gradient row with
 * two entries whose endpoints lie in different aggregates a<b, bucket b under a.
 * count -> scan -> fill -> sphc_csr_sort_rows -> unique. */
int sphc_coarse_pairs_count(int64_t n_e, const int64_t *drp, const int32_t *dci,
                            const int64_t *assign, int64_t *counts, void *stream);
int sphc_coarse_pairs_fill(int64_t n_e, const int64_t *drp, const int32_t *dci,
                           const int64_t *assign, const int64_t *brp, int64_t *cursor,
                           int32_t *bcol, void *stream);
int sphc_unique_count(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *counts,
                      void *stream);
int sphc_unique_fill(int64_t n, const int64_t *rp, const int32_t *ci, const int64_t *urp,
                     int32_t *uci, void *stream);

/* flags[c] = 1 if aggregate c owns the free end of a one-entry gradient row
 * (coarse_gradient.py:139-160, augment_dirichlet_edges). */
int sphc_single_flags(int64_t n_e, const int64_t *drp, const int32_t *dci,
                      const int64_t *assign, int64_t *flags, void *stream);

/* D_H rows: interior edge e=(a,b): -1 at a, +1 at b; single-node edge: +1.
 * Also writes ep_a/ep_b (ep_a = -1 for single-node edges). */
int sphc_build_coarse_gradient(int64_t n_agg, int64_t n_int, const int64_t *adj_rp,
                               const int32_t *adj_col, const int64_t *single_off,
                               int64_t n_single, int64_t *dh_rp, int32_t *dh_ci,
                               double *dh_v, int32_t *ep_a, int32_t *ep_b,
                               int32_t *single_id, void *stream);

/* ---------------------------------------------------------------- emin */

/* Per fine edge (emin_setup.py:62-336, Appendix C): node set J (= T row),
 * coarse-edge set I (= prolongator pattern N row), |I|,|J|, the
 * subproblem_dims histogram [SPHC_DIMS_I][SPHC_DIMS_J] (rows with |I| > 0
 * inside the table; the caller adds the wider rows from icount / jcount) and
 * rmax2[0] = max |D_h P_n| over all rows (emin_setup.py:289),
 * rmax2[1] = the same over rows whose I is empty (emin_setup.py:292-295).
 * Capacity classes: rows with |J| > jcap or |I| > icap (<= 0 or above the
 * default class = SPHC_EMIN_JMAX / SPHC_EMIN_IMAX; tests lower them) are
 * counted in *over (caller zeroes it before the count pass) and handled by a
 * second launch of the wide class, which returns at once while *over == 0.
 * sphc_emin_fill and sphc_emin_step take the same jcap, icap and over. */
int sphc_emin_count(int64_t n_e, const int64_t *drp, const int32_t *dci, const double *dv,
                    const int64_t *prp, const int32_t *pci, const double *pv,
                    const int64_t *adj_rp, const int32_t *adj_col, int64_t n_int,
                    const int32_t *single_id, const int64_t *xrp, const int32_t *xeid,
                    const int32_t *ep_a, const int32_t *ep_b, int64_t *icount,
                    int64_t *jcount, double *rmax2, int64_t *dims, uint8_t *rowflag,
                    double *rowmax, int32_t jcap, int32_t icap, int64_t *over,
                    int64_t *status, void *stream);
/* Row extras: coarse edges appended by the host make_irreducible pass
 * (emin_setup.py:183-217,311-333) as a CSR over fine edges (xrp, xeid; NULL
 * xrp = none); ep_a/ep_b = endpoints of every coarse edge. The count pass only
 * sizes rows; with rowflag != NULL it writes bit 1 = empty pattern (rowmax =
 * that row's max |D_h P_n|). The fill pass factors every block; with rowflag
 * != NULL a reducible block sets bit 0 instead of failing. */

/* Writes T (J columns + commutator rhs r = D_h P_n on J) and the prolongator
 * row pattern I with the feasible guess p = 1 + G_k (G_k^T G_k)^-1 (r - G^T 1)_k
 * (edge_prolongator.py:104-126; Gram-Cholesky form of the QR least-norm solve). */
int sphc_emin_fill(int64_t n_e, const int64_t *drp, const int32_t *dci, const double *dv,
                   const int64_t *prp, const int32_t *pci, const double *pv,
                   const int64_t *adj_rp, const int32_t *adj_col, int64_t n_int,
                   const int32_t *single_id, const int64_t *xrp, const int32_t *xeid,
                   const int32_t *ep_a, const int32_t *ep_b, const int64_t *trp,
                   int32_t *tci, double *tv, const int64_t *erp, int32_t *eci, double *ev,
                   uint8_t *rowflag, int32_t jcap, int32_t icap, int64_t *over,
                   int64_t *status, void *stream);

/* One projected damped-Jacobi sweep (edge_prolongator.py:170-176) fused with
 * the masked product S P on the fixed pattern, the energy of the INPUT values
 * (:154-156) and the commutator residual of the OUTPUT (:179-181):
 *   g = (S P_in)|_I ; e_row[i] = p_in . g ; delta = dinv_i g ;
 *   delta -= G_k M^-1 G_k^T delta ; P_out = P_in - omega delta (update != 0)
 *   res_max = max |G^T p_out - r| over J.
 * With update == 0 only e_row and res_max (of P_in) are produced. Rows
 * [row0, row1) are processed (a row block of a sharded setup); every array
 * is indexed globally. */
int sphc_emin_step(int64_t row0, int64_t row1, const int64_t *srp, const int32_t *sci, const double *sv,
                   const double *dinv, const int64_t *trp, const int32_t *tci,
                   const double *tv, const int64_t *erp, const int32_t *eci,
                   const double *p_in, double *p_out, const int32_t *ep_a,
                   const int32_t *ep_b, double omega, int update, double *e_row,
                   double *res_max, int32_t jcap, int32_t icap, const int64_t *over,
                   int64_t *status, void *stream);

/* SpGEMM rows beyond the on-chip kernels' capacity (the count kernels
 * mark them with count -1: > 256 distinct columns, a B row longer than a
 * staging window, a hash overflow): one CTA per listed row, the row's hash
 * table in global scratch (hoff: per-row offsets, power-of-two sizes >= 2 x
 * the row's products, from sphc_spgemm_global_products). crp NULL: count
 * pass (counts[row]); else fill at crp[row] with sorted columns and
 * ascending-k unfused sums (bitwise scipy csr_matmat order); av2 non-NULL:
 * the pair product. Rows of more than 8192 columns -> SPGEMM_CAPACITY. */
int sphc_spgemm_global_products(int64_t nrows, const int64_t *rows, const int64_t *arp,
                                const int32_t *aci, const int64_t *brp, int64_t *prods,
                                void *stream);
int sphc_spgemm_global(int64_t nrows, const int64_t *rows, const int64_t *hoff, int32_t *hkeys,
                       int32_t *hslot, const int64_t *arp, const int32_t *aci, const double *av,
                       const double *av2, const int64_t *brp, const int32_t *bci,
                       const double *bv, const double *bv2, int64_t *counts, const int64_t *crp,
                       int32_t *cci, double *cv, double *cv2, int64_t *status, void *stream);

/* ---------------------------------------------------------------- host (C++) */

/* Greedy two-phase aggregation, exact reference semantics
 * (nodal_amg.py:59-88). Host arrays. Returns n_agg in *n_agg. */
int sphc_host_aggregate(int64_t n, const int64_t *rp, const int32_t *ci, int64_t *membership,
                        int64_t *n_agg);

/* Greedy root aggregation (nodal_amg.py:59-88) on the device, bit-identical
 * to the sequential loops. rp/ci: symmetric strength pattern incl. the
 * diagonal (n x n). Work buffers: state (n int32), ticket (1 int32), flags,
 * pos, list (n + 1 int64 each). memb (n int64) receives the aggregate of
 * every node and list[n] the number of aggregates. Both phases are sync-free
 * (nodes taken in ascending order from a ticket, each waiting only on lower
 * nodes within its dependency range). status[SPHC_ST_AGG_CAPACITY]: a
 * leftover node with more than 256 assigned neighbours. */
int sphc_aggregate(int64_t n, const int64_t *rp, const int32_t *ci, int32_t *state,
                   int32_t *ticket, int64_t *flags, int64_t *pos, int64_t *list, int64_t *memb,
                   int64_t *status, void *stream);

/* Algorithm 1 (coarse_gradient.py:36-103) on the device, bit-identical to
 * the reference's sequential column order. prp/pci/pv: P_n (m_h x m_H, CSR);
 * crp/crow/cval: its transpose (column view, rows ascending). Work buffers:
 * target, counts (m_H int64), srow (nnz int32), owner (2 m_h int32),
 * changed (1 int32), flags, pos, list (max(m_h, m_H) + 1 int64 each).
 * assign (m_h int64) receives the column of every row. Each claiming pass is
 * solved as a fixed point over all columns at once (one host sync per
 * iteration; a handful of iterations), see csrc/pconst.cu.
 * Errors: status[SPHC_ST_PC_*]. */
int sphc_piecewise_const(int64_t m_h, int64_t m_H, const int64_t *prp, const int32_t *pci,
                         const double *pv, const int64_t *crp, const int32_t *crow,
                         const double *cval, int n_passes, int64_t *target, int64_t *counts,
                         int32_t *srow, int32_t *owner, int32_t *changed, int64_t *flags,
                         int64_t *pos, int64_t *list, int64_t *assign, int64_t *status,
                         void *stream);

/* Algorithm 1 (coarse_gradient.py:36-103) on a host CSR copy of P_n.
 * On a data error returns SPHC_ERR_HOST with err[0] = kind (1 empty column,
 * 2 row with no entries, 3 empty column after safeguard), err[1] = index. */
int sphc_host_piecewise_const(int64_t m_h, int64_t m_H, const int64_t *rp, const int32_t *ci,
                              const double *v, int n_passes, int64_t *assign, int64_t *err);


/* ---- model-problem inputs on the device ----------
 * Replace the host generator's build_structured_mesh(3, 'hex', N + 1,
 * dirichlet) (meshing.py:61-131) and discretize(mesh, sigma)
 * (assembly.py:47-54, curl-curl assembly.py:135-144,231-290, edge mass
 * :297-306,346-366, nodal operator :373-386,404-434, gradient :62-79), with
 * two extensions the reference lacks: per-element sigma and curved
 * (jittered, isoparametric trilinear) hexes, integrated by 3x3x3 Gauss.
 * Numbering is the reference's (csrc/assemble.cu). Row kernels run in two
 * modes: rp == NULL writes per-row counts, otherwise fills col / values at
 * rp. X (n^3 x 3 node coordinates) == NULL means the uniform mesh (J = h I);
 * sigma == NULL means the constant sigma_const. */
int sphc_hex_node_counts(int N, int dirichlet, int64_t *edge_counts, int64_t *free_counts,
                         void *stream);
int sphc_hex_tables(int N, int dirichlet, const int64_t *edge_offsets,
                    const int64_t *free_offsets, int32_t *edge_of, int64_t *edge_code,
                    int32_t *free_id, int32_t *free_list, void *stream);
int sphc_hex_coords(int N, const double *jitter, double *X, void *stream);
/* A_e = S + sigma M and S on one pattern (edges sharing a hex) */
int sphc_hex_edge_rows(int N, int64_t n_edges, const int64_t *edge_code, const int32_t *edge_of,
                       const double *X, const double *sigma, double sigma_const,
                       const int64_t *rp, int64_t *counts, int32_t *col, double *val_A,
                       double *val_S, void *stream);
/* A_n = K + sigma M_n on the free nodes */
int sphc_hex_node_rows(int N, int64_t n_free, const int32_t *free_list, const int32_t *free_id,
                       const double *X, const double *sigma, double sigma_const,
                       const int64_t *rp, int64_t *counts, int32_t *col, double *val,
                       void *stream);
/* D: -1 at the tail's free column, +1 at the head's */
int sphc_hex_grad_rows(int N, int64_t n_edges, const int64_t *edge_code, const int32_t *free_id,
                       const int64_t *rp, int64_t *counts, int32_t *col, double *val,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif
