/*
 * spaigraph_b200 — C-ABI of the B200-native GNN-SPAI + PCG hot path.
 *
 * Drop-in boundary for the reference package `spaigraph` (pure numpy, /root/reference/pkg).
 * The reference has no FFI of its own; every entry point below replaces one numpy function of
 * the hot path and cites it as  <file>:<line>  relative to pkg/src/spaigraph/.  The Python host
 * package `paper_2510_27517_b200` (ctypes) mirrors the reference's Python API on top of these.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers unless the name ends in `_host`.
 *   - Indices on device are int32 (row offsets, column indices, permutations); sizes are int64.
 *     Values are IEEE binary64.  Device arrays that a kernel stages with 16-byte vector loads
 *     must be allocated with >= 16 bytes of slack past the end (the Python layer pads).
 *   - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on `stream` unless the
 *     comment says "synchronizes".
 *   - Return value: SG_OK or an error code; sg_last_error() returns a thread-local message.
 *   - Buffers are caller-owned.  Functions that need scratch take (ws, ws_bytes): call with
 *     ws == NULL to read the required size into *ws_bytes.
 *   - Parity kernels compute products and sums with explicit round-to-nearest intrinsics in the
 *     reference's summation order, so SpMV / transpose-SpMV / apply / features / generators are
 *     bit-identical to the numpy reference.
 */
#ifndef SPAIGRAPH_B200_H
#define SPAIGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sg_status {
  SG_OK = 0,
  SG_EINVAL = 1,        /* shape / structure violation      -> ValueError        */
  SG_ENOTSPD = 2,       /* PCG breakdown                    -> NotSpdError       */
  SG_ECUDA = 3,         /* CUDA runtime error               -> RuntimeError      */
  SG_EUNSUPPORTED = 4,  /* configuration not implemented    -> NotImplementedError */
  SG_EDUPLICATE = 5     /* duplicate COO entry              -> ValueError("duplicate ...") */
};

int sg_abi_version(void);
const char* sg_last_error(void);

/* ---------------------------------------------------------------- sparsity patterns (L1) */

/* SparseMatrix.from_coo (sparse.py:138-158): stable sort by (row, col), duplicate rejection,
 * row offsets.  rows/cols are int64 (the reference index type).  On SG_EDUPLICATE the
 * lexicographically first duplicated (row, col) is written to dup_host[0..1].  Synchronizes. */
int sg_csr_from_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                    const int64_t* cols, const double* vals, int32_t* offs_out, int32_t* cols_out,
                    double* vals_out, int64_t* dup_host, void* ws, size_t* ws_bytes, void* stream);

/* int64 -> int32 narrowing of reference index arrays: out[k] = in[k] + shift after checking
 * lo <= in[k] < hi (shift places a system inside a block-diagonal batch).  Synchronizes. */
int sg_narrow_index(const int64_t* in, int32_t* out, int64_t n, int64_t lo, int64_t hi,
                    int64_t shift, void* ws, size_t* ws_bytes, void* stream);

/* Batched narrowing for block-diagonal batches: element k of segment s (seg_start[s] <= k <
 * seg_start[s+1], device arrays) must satisfy 0 <= in[k] < bound[s]; out[k] = in[k] + shift[s].
 * One launch for every system's offsets (or columns).  Synchronizes. */
int sg_narrow_index_segments(const int64_t* in, int32_t* out, int64_t n, const int64_t* seg_start,
                             const int64_t* bound, const int64_t* shift, int32_t n_seg, void* ws,
                             size_t* ws_bytes, void* stream);

/* _validate_structure (sparse.py:27-43): offsets[0]==0, offsets[n]==nnz, nondecreasing,
 * columns in range and strictly increasing within a row.  Synchronizes. */
int sg_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* offs,
                    const int32_t* cols, void* ws, size_t* ws_bytes, void* stream);

/* SparseMatrix.transpose (sparse.py:129-136): pattern of A^T with ascending original rows
 * inside each row, plus perm such that values_t[k] = values[perm[k]] (see sg_gather_f64). */
int sg_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* offs,
                     const int32_t* cols, int32_t* offs_t, int32_t* cols_t, int32_t* perm,
                     void* ws, size_t* ws_bytes, void* stream);

/* SparsityPattern.is_symmetric (sparse.py:68-78).  *result_host = 1/0.  Synchronizes. */
int sg_pattern_is_symmetric(int64_t n, int64_t nnz, const int32_t* offs, const int32_t* cols,
                            int32_t* result_host, void* ws, size_t* ws_bytes, void* stream);

/* A^2 pattern (no reference counterpart — the paper's future work):
 * pattern(|A| |A|), rows sorted.  Two calls: out_cols == NULL computes out_offs (n+1) and
 * *out_nnz_host; then call again with out_cols (out_nnz entries) to fill.  Rows with more than
 * 2048 candidate products return SG_EUNSUPPORTED. */
int sg_pattern_square(int64_t n, const int32_t* offs, const int32_t* cols, int32_t* out_offs,
                      int32_t* out_cols, int64_t* out_nnz_host, void* ws, size_t* ws_bytes, void* stream);

/* gen_synthetic (datasets.py:148-193): pattern of the Gram matrix P·Pᵀ + εI, P an n×m CSR
 * matrix with sorted rows, Pᵀ its transpose (m rows).  Row i = {i} ∪ columns reached through
 * P's row i; rows sorted.  Two calls like sg_pattern_square.  Rows with more than 2047
 * candidates return SG_EUNSUPPORTED. */
int sg_gram_pattern(int64_t n, const int32_t* p_offs, const int32_t* p_cols, const int32_t* pt_offs,
                    const int32_t* pt_cols, int32_t* out_offs, int32_t* out_cols, int64_t* out_nnz_host, void* ws,
                    size_t* ws_bytes, void* stream);

/* Gram values on that pattern, the reference's accumulation order: A_ij = 0.0 + P_ic1·P_jc1 +
 * P_ic2·P_jc2 + ... over shared columns c1 < c2 < ... (datasets.py:163-176), then + shift on the
 * diagonal (datasets.py:177-178).  Bit-exact. */
int sg_gram_values(int64_t n, const int32_t* p_offs, const int32_t* p_cols, const double* p_vals,
                   const int32_t* a_offs, const int32_t* a_cols, double shift, double* a_vals, void* stream);

/* A's values on a superset pattern P (explicit zeros elsewhere; explicit zeros are
 * pattern-significant, sparse.py:3-6).  SG_EINVAL if P does not contain pattern(A). */
int sg_csr_pad_to_pattern(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                          const int32_t* p_offs, const int32_t* p_cols, double* out_vals, void* ws,
                          size_t* ws_bytes, void* stream);

/* row_expand (sparse.py:64-66): rows_out[k] = row of stored entry k. */
int sg_row_expand(int64_t n_rows, const int32_t* offs, int32_t* rows_out, void* stream);

/* values_out[k] = values_in[perm[k]] (G^T values from G values, gnn.py:256-267 + a4). */
int sg_gather_f64(const double* in, const int32_t* perm, double* out, int64_t n, void* stream);

/* SparseMatrix.diagonal (sparse.py:119-127), absent entries read 0. present_out may be NULL. */
int sg_csr_diagonal(int64_t n, const int32_t* offs, const int32_t* cols, const double* vals,
                    double* diag_out, int32_t* present_out, void* stream);

/* ---------------------------------------------------------------- generators (L6) */

/* gen_poisson2d (datasets.py:87-145) emitted directly in CSR order; coeff is the node field a
 * (ones for "poisson2d").  offs: nx*ny+1, cols/vals: 5*nx*ny - 2*nx - 2*ny.  row0/nnz0 place
 * the system inside a block-diagonal batch: rows row0.., entries nnz0.. (0, 0 for a single
 * system); offs/cols/vals are the batch arrays. */
int sg_gen_poisson2d(int64_t nx, int64_t ny, const double* coeff, int64_t row0, int64_t nnz0,
                     int32_t* offs, int32_t* cols, double* vals, void* stream);

/* 7-point 3-D analogue (oracle/spaigraph_ref.py:gen_poisson3d). */
int sg_gen_poisson3d(int64_t nx, int64_t ny, int64_t nz, int32_t* offs, int32_t* cols,
                     double* vals, void* stream);

/* ---------------------------------------------------------------- norms + features (L3) */

/* matrix_norm (training.py:44-54) / mean_abs_nonzero_norm (sparse.py:204-213): the exact
 * (math.fsum-identical, correctly rounded) sum of |v| (kind 0: /nnz, kind 2: as is) or of
 * fl(v*v) (kind 1: sqrt).  Result written to *norm_out (device). */
int sg_matrix_norm(const double* vals, int64_t nnz, int kind, double* norm_out, void* ws,
                   size_t* ws_bytes, void* stream);

/* sg_matrix_norm for n_seg independent value segments (one per system of a block-diagonal
 * batch): seg_start (device, n_seg+1) delimits them; norms_out[k] per segment.  Same exact
 * summation; one launch for the whole batch. */
int sg_matrix_norm_batched(const double* vals, const int64_t* seg_start, int32_t n_seg,
                           int64_t max_seg_len, int kind, double* norms_out, void* ws,
                           size_t* ws_bytes, void* stream);

/* build_graph features for every system of a block-diagonal batch in one launch: row_start
 * (device, n_sys+1), norms (device, per system, sg_matrix_norm_batched), family as below, and
 * for family 1 per-system grid sizes nx/ny (device int64), coeff aligned with rows (device) and
 * per-system coeff_mean (device, numpy's pairwise mean of the host field). */
int sg_graph_features_batched(const int64_t* row_start, int32_t n_sys, int64_t n, const int32_t* offs,
                              const int32_t* cols, const double* vals, const double* norms, int family,
                              const int64_t* nx, const int64_t* ny, const double* coeff,
                              const double* coeff_mean, double* node_out, double* edge_out,
                              void* stream);

/* build_graph features (graphfeat.py:63-105) for the n rows row0..row0+n-1 of a (possibly
 * block-diagonal) matrix.  family 0: algebraic [rowsum/n/norm, diag/norm] (node_out rows of
 * 2); family 1: PDE [(ix+1)hx, (iy+1)hy, coeff/coeff_mean] (rows of 3; coeff is the system's
 * own field, indexed locally).  edge_out[k] = vals[k] / norm.  norm: device scalar. */
int sg_graph_features(int64_t n, int64_t row0, const int32_t* offs, const int32_t* cols,
                      const double* vals, const double* norm, int family, int64_t nx, int64_t ny,
                      const double* coeff, double coeff_mean, double* node_out, double* edge_out,
                      void* stream);

/* ---------------------------------------------------------------- GNN forward (L3) */

/* forward (gnn.py:208-253) restructured: node-path kernels + one fused edge
 * pass that never materialises H.  params: flat f64 in declaration order (gnn.py:130-136).
 * Supported: mlp_hidden_layers == 1, message_uses_hidden_edge == 0, d_edge == 1,
 * hidden in {4,6,8,12,16,24,32}, d_node <= 4, act 0 = relu / 1 = tanh; else SG_EUNSUPPORTED.
 * rows: row index per edge (sg_row_expand).  g_out[k] = G value of stored entry k. */
int sg_gnn_forward(const double* params, int64_t n_params, int n_layers, int hidden, int d_node,
                   int d_edge, int act, int64_t n, int64_t nnz, const int32_t* offs,
                   const int32_t* cols, const int32_t* rows, const double* node_feat,
                   const double* edge_feat, double* g_out, void* ws, size_t* ws_bytes,
                   void* stream);

/* sg_gnn_forward with a choice of edge-pass arithmetic: edge_mode 0 = the fp64 DMMA edge pass
 * (sg_gnn_forward), 1 = the edge MLPs on the 5th-generation tensor cores (tcgen05.mma
 * kind::tf32, 3xTF32 split, fp32 accumulation in TMEM; ~fp32 accuracy, the north_star's fp32 bar
 * of 1e-5 on G; hidden <= 32).  The node path is fp64 either way. */
int sg_gnn_forward_ex(const double* params, int64_t n_params, int n_layers, int hidden, int d_node,
                      int d_edge, int act, int64_t n, int64_t nnz, const int32_t* offs,
                      const int32_t* cols, const int32_t* rows, const double* node_feat,
                      const double* edge_feat, double* g_out, int32_t edge_mode, void* ws,
                      size_t* ws_bytes, void* stream);

/* ---------------------------------------------------------------- SpMV family (L1, L4) */

/* spmv (sparse.py:186-191): y = A x in numpy reduceat order (bit-identical). */
int sg_spmv(int64_t n_rows, const int32_t* offs, const int32_t* cols, const double* vals,
            const double* x, double* y, void* stream);

/* spmv for long rows (>= 32 entries on average, e.g. G on the A^2 pattern): one warp per row,
 * the same numpy reduceat order (bit-identical to sg_spmv); replaces sparse.py:186-191 there. */
int sg_spmv_warp(int64_t n_rows, const int32_t* offs, const int32_t* cols, const double* vals,
                 const double* x, double* y, void* stream);

/* spmv_transpose (sparse.py:194-201) given the explicit transpose (sg_csr_transpose): strictly
 * sequential per row from 0.0 == np.add.at order (bit-identical). */
int sg_spmv_seq(int64_t n_rows, const int32_t* offs, const int32_t* cols, const double* vals,
                const double* x, double* y, void* stream);

/* LearnedSpaiPreconditioner.apply (precond.py:143-145): s = G (G^T r) + eps r.
 * t_ws: n doubles of scratch. */
int sg_learned_apply(int64_t n, const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                     const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                     double eps, const double* r, double* t_ws, double* s_out, void* stream);

/* Elementwise update with the reference's roundings (pcg.py:186-200 `x + alpha*d`,
 * `r - alpha*q`, `s + beta*d`): out = a + c*b (mode 0) or a - c*b (mode 1). */
int sg_axpby(double* out, const double* a, const double* b, double c, int64_t n, int mode, void* stream);

/* Deterministic dot product x.y into a device scalar (fixed reduction tree). */
int sg_dot(const double* x, const double* y, int64_t n, double* out, void* ws, size_t* ws_bytes, void* stream);

/* ---------------------------------------------------------------- PCG (L4) */

/* pcg_solve (pcg.py:131-233) for a batch of independent systems stored block-diagonally
 * (global column indices).  One handle per (matrices, preconditioner) pair; the handle owns
 * device state, the CUDA-graph cache and per-system histories. */
typedef struct sg_pcg sg_pcg;

enum sg_precond_kind { SG_PRECOND_IDENTITY = 0, SG_PRECOND_JACOBI = 1, SG_PRECOND_LEARNED = 2 };

typedef struct sg_solve_config {
  double rtol;               /* SolveConfig.rtol                                           */
  int64_t max_iters;         /* < 0: 20 * n_s per system (pcg.py:151)                      */
  int64_t refresh_period;    /* SolveConfig.residual_refresh_period                        */
  int32_t termination;       /* 0 = true_residual, 1 = delta                               */
  int32_t track_history;     /* SolveConfig.track_history                                  */
} sg_solve_config;

typedef struct sg_solve_result {
  int64_t k;                 /* SolveReport.k                                              */
  int32_t converged;         /* SolveReport.converged                                      */
  int32_t status;            /* SG_OK or SG_ENOTSPD                                        */
  int64_t fail_iter;         /* NotSpdError.iteration                                      */
  double fail_value;         /* NotSpdError.value                                          */
  int32_t fail_kind;         /* 1: d^T A d <= 0, 2: r^T M r < 0                            */
  int64_t hist_len;          /* number of residual_history entries                         */
} sg_solve_result;

/* sys_row_start_host: n_systems+1 row boundaries.  Matrices: A (PCG), and for LEARNED the
 * factor G and its explicit transpose Gt; for JACOBI, inv_diag (n).  All device, int32 idx.
 * The handle keeps the pointers (caller keeps the arrays alive). */
int sg_pcg_create(sg_pcg** out, int32_t n_systems, const int64_t* sys_row_start_host,
                  const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                  int precond_kind, const int32_t* g_offs, const int32_t* g_cols,
                  const double* g_vals, const int32_t* gt_offs, const int32_t* gt_cols,
                  const double* gt_vals, const double* inv_diag, double epsilon, void* stream);

/* Solve A x = b from x0 = 0 for every system.  b, x: device, n rows.  results_host: n_systems
 * entries.  Runs the device-resident loop (CUDA graphs of fused iteration kernels) and
 * synchronizes before returning.  elapsed_ns_host (may be NULL) receives the solve time. */
int sg_pcg_solve(sg_pcg* h, const double* b, double* x, const sg_solve_config* cfg,
                 sg_solve_result* results_host, int64_t* elapsed_ns_host, void* stream);

/* residual_history of system `sys` from the last solve (hist_len entries) into out_host. */
int sg_pcg_history(sg_pcg* h, int32_t sys, double* out_host, int64_t len);

void sg_pcg_destroy(sg_pcg* h);

/* Re-point a handle at new value arrays on the SAME patterns (e.g. a new G from the GNN on A's
 * pattern, or refilled A values): avoids rebuilding the handle and its captured graphs. */
int sg_pcg_rebind_values(sg_pcg* h, const double* a_vals, const double* g_vals, const double* gt_vals,
                         const double* inv_diag);

/* Re-point a handle at other arrays of the same SIZES (index arrays too: a new G^T, a refilled
 * matrix).  The next sg_pcg_solve fingerprints the patterns behind the pointers and re-plans the
 * handle only if they differ from the ones it was planned on (sg_pcg_rebuilds). */
int sg_pcg_rebind(sg_pcg* h, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                  const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                  const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                  const double* inv_diag);

/* Instrumentation (no reference counterpart; pcg.py:155-229 only times apply / total on the
 * host).  With profiling on, every chunk graph brackets K1, K2, K3 of one non-refresh
 * iteration with external event-record nodes; sg_pcg_stats returns the summed device times
 * prof_host[0..2] (ms), the summed active-system counts at those iterations prof_host[3], the
 * sample count prof_host[4], the storage format prof_host[5] (number of diagonals when the
 * diagonal-major DIA format is in use, 0 for CSR), plus the number of kernels and graphs
 * launched; prof_host[6] = 1 when A is read by its lower half (bitwise-symmetric A in DIA), 2
 * when K1 regenerates it from the coefficient stencil (sg_pcg_set_stencil);
 * prof_host[7] = 1 when K2 and K3 run fused (halo-staged DIA, learned preconditioner): then
 * prof_host[1] is the fused kernel and prof_host[2] is 0.  prof_host must hold 8 doubles. */
/* Coefficient stencil (no reference counterpart; the matrix is gen_poisson2d's, datasets.py:
 * 87-145): `coeff` (device, n doubles aligned with A's rows, every system an nx-by-ny grid;
 * the caller keeps it alive and may refill it between solves) lets the streamed K1 regenerate
 * A's entries bitwise from the node coefficients (8 instead of 24 B/row).  Every solve first
 * verifies the stored A against the stencil bitwise and keeps the diagonals on any mismatch.
 * coeff = NULL turns it off.  *usable_host = 1 when the handle's format can use it. */
int sg_pcg_set_stencil(sg_pcg* h, const double* coeff, int64_t nx, int64_t ny, int32_t* usable_host);

/* A handle is planned on the PATTERNS of A, G, G^T (storage format, diagonal set, tile and
 * range tables, SELL copies).  Every sg_pcg_solve fingerprints the patterns behind the
 * pointers and re-plans the handle when the caller refilled them with another pattern (same
 * sizes or not); sg_pcg_rebuilds reports how many times that happened.  A row-partitioned
 * handle whose pattern changed fails with SG_EINVAL instead. */
int sg_pcg_rebuilds(sg_pcg* h, int64_t* rebuilds_host);

/* Device time (ns) the last sg_pcg_solve spent in the preconditioner apply when the handle runs
 * whole iterations in one launch (systems of <= 32768 rows: one CTA or one thread-block cluster
 * per system; %globaltimer around the apply phase, summed over systems); 0 on the multi-kernel
 * path, whose apply share comes from the in-graph event samples of sg_pcg_stats.  Replaces the
 * reference's t_apply accumulation (pcg.py:155-229) for that path. */
int sg_pcg_apply_ns(sg_pcg* h, int64_t* ns_host);

int sg_pcg_set_profile(sg_pcg* h, int32_t on);
/* Timeline probe of the wide-grid strip kernels (k_iter1_s5p, k_iter23_s5): with a device buffer
 * of 2 x 16384 uint64, thread 0 of every CTA writes %globaltimer at entry, end of its stream,
 * after its arrival and (last CTA) after the finaliser, and its SM id; K1 at [0, 16384), K2+K3
 * at [16384, 32768), slot 8 * cta + k (k = 0..3 the stamps, 4 the SM).  NULL turns it off.
 * Diagnostic only (profiles/trace_probe.py). */
int sg_pcg_set_trace(sg_pcg* h, void* buf);
int sg_pcg_stats(sg_pcg* h, int64_t* kernels_host, int64_t* chunks_host, double* prof_host,
                 int32_t reset);

/* ---------------------------------------------------------------- SAI loss (L5) */

/* sai_loss / sai_loss_on_tape + Tape.backward (training.py:57-94, autodiff.py:190-239,
 * 265-303).  A-side in double-double (the reference uses x87 long double); returns the loss in
 * *loss_host and, if grad_out != NULL, dL/dg (nnz of G) in the tape's rounding order.
 * at_*: explicit A^T (for du = A^T dz), gt_*: explicit G^T.  Synchronizes. */
int sg_sai_loss(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                const int32_t* at_offs, const int32_t* at_cols, const double* at_vals,
                const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                const int32_t* g_rows, double eps, const double* w, int norm_kind,
                double* loss_host, double* grad_out, void* ws, size_t* ws_bytes, void* stream);

/* Row-partitioned SAI loss (BASELINE configs[4]: loss forward + backward on the row partition
 * of DESIGN.md §7).  Per partition, on its extended local system (owned rows [own_lo, own_hi)
 * + 3 half-bandwidths of ghost rows; A^T, G, G^T of the extended system; w on all its rows):
 *   1. sg_loss_norm_partial over the partition's OWNED entries -> a dd partial (2 doubles);
 *      sg_loss_norm_combine adds the partials in partition order -> norm3 = {norm hi, lo, 1/norm};
 *   2. sg_sai_loss_part_fwd -> t (n), z (n; exact on owned rows) and the dd partial of sum z^2
 *      over the owned rows; sg_loss_sum_parts adds the partials in partition order (the loss);
 *   3. the caller copies the neighbours' owned z into the ghost rows (the loss's only halo);
 *   4. sg_sai_loss_part_bwd -> dL/dg for every entry of the owned rows (grad_out indexed like
 *      the extended G; other entries untouched).
 * Same arithmetic as sg_sai_loss row by row; only the dd partial sums are grouped per partition. */
int sg_loss_norm_partial(const double* vals, int64_t nnz, int kind, double* part_out, void* ws, size_t* ws_bytes,
                         void* stream);
int sg_loss_norm_combine(const double* parts, int32_t n_parts, int64_t nnz_total, int kind, double* norm3_out,
                         void* stream);
int sg_sai_loss_part_fwd(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                         const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                         const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals, double eps,
                         const double* w, const double* norm3, int64_t own_lo, int64_t own_hi, double* t_out,
                         double* z64_out, double* part_out, void* ws, size_t* ws_bytes, void* stream);
int sg_loss_sum_parts(const double* parts, int32_t n_parts, double* loss_host, void* stream);
int sg_sai_loss_part_bwd(int64_t n, const int32_t* at_offs, const int32_t* at_cols, const double* at_vals,
                         const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                         const int32_t* g_offs, const int32_t* g_rows, const int32_t* g_cols, const double* w,
                         const double* t, const double* z64, const double* norm3, int64_t own_lo, int64_t own_hi,
                         double* grad_out, void* ws, size_t* ws_bytes, void* stream);

/* tcgen05 building block (diagnostic): one 128-row tile D = A . W (A: 128 x K row-major fp32,
 * W: K x N row-major fp32, K, N <= 32) on the 5th-generation tensor core, kind::tf32 with operands
 * in shared memory and the accumulator in TMEM; split3 = 1 runs the 3xTF32 split (~fp32
 * accuracy).  out: 128 x N row-major.  Used by the tests of the tensor-core edge pass. */
int sg_tc_gemm_selftest(const float* a, const float* w, int32_t k, int32_t n, int32_t split3, float* out,
                        void* stream);

/* ---- GNN training step (gnn.py:198-253 backward, training.py:126-147) ----
 * Plain fp64 primitives with fixed reduction orders (bit-reproducible runs); composed by
 * paper_2510_27517_b200/training.py into the training forward (all intermediates kept), the
 * backward through the restructured GNN, and AdamW. */

/* out[r][c] = relu?( sum_k in[r][k] * W[k][c] (W[c][k] if transpose_w) + b[c] ) + add[r][c];
 * row strides ldi / ldw / ldo (row blocks of a parameter matrix are addressed by pointer).
 * b, add may be NULL. */
int sg_dense_affine(int64_t N, int32_t din, int32_t dout, const double* in, int32_t ldi, const double* W,
                    int32_t ldw, int32_t transpose_w, const double* b, const double* add, double* out,
                    int32_t ldo, int32_t relu, void* stream);
/* pre[e][c] = P[rows[e]][c] + Q[cols[e]][c] + ef[e]*crow[c] + H[e][c] + b[c] (crow, H, b optional) */
int sg_edge_pre(int64_t E, int32_t d, const int32_t* rows, const int32_t* cols, const double* P, const double* Q,
                const double* ef, const double* crow, const double* H, const double* b, double* pre, void* stream);
/* dst = src * [pre > 0] */
int sg_relu_grad(int64_t M, const double* pre, const double* src, double* dst, void* stream);
/* dst[i] (+)= sum over CSR segment i of src[perm ? perm[k] : k] (rows of width d, segment order) */
int sg_segment_sum(int64_t n, int32_t d, const int32_t* offs, const int32_t* perm, const double* src, double* dst,
                   int32_t accumulate, void* stream);
/* out[a][b] (+)= sum_r A[r][a] * B[r][b] (A NULL: column sums of B), two fixed-order passes.
 * Workspace query with ws == NULL. */
int sg_outer_sum(int64_t N, int32_t da, int32_t db, const double* A, int32_t lda, const double* B, int32_t ldb,
                 double* out, int32_t accumulate, void* ws, size_t* ws_bytes, void* stream);
/* build_fsai (precond.py:262-305): values of the lower-triangular factor on the lower pattern
 * (l_offs, l_cols) of A, one dense Cholesky solve per row; rows whose local system is not SPD
 * fall back to 1/sqrt(a_ii) (count in *fallbacks_host).  Rows with > 16 lower entries:
 * SG_EUNSUPPORTED.  Synchronizes. */
int sg_fsai_build(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                  const int32_t* l_offs, const int32_t* l_cols, double* l_vals, int64_t* fallbacks_host,
                  void* stream);
/* adamw_step (training.py:126-147) with grads / grad_div, t the 1-based step; in place. */
int sg_adamw(int64_t n, double* params, const double* grads, double* m, double* v, double lr, double wd,
             double beta1, double beta2, double eps, int64_t t, double grad_div, void* stream);

/* ---- row partition of ONE system (SURVEY.md §8(e)(ii), config C5 over 2/4/8 GPUs) ----------
 * Design: the system's rows are split into contiguous blocks; partition p holds an
 * EXTENDED local system = its owned rows plus ghost rows on either side, 3 half-bandwidths deep
 * (for a grid: 3 lines).  Every PCG kernel runs over the whole extended system exactly as for an
 * independent system -- the fused sliding-window / strip kernels included -- except that only
 * owned rows enter the dot products and write s, and the first / last owned rows of s are ALSO
 * stored into the neighbours' ghost rows from inside the kernel that computes them.  With 3
 * ghost layers every other vector (d, q, r, x) stays exact on the ghost rows the next kernels
 * read by redundant computation, so one halo per iteration is all the communication besides the
 * two scalar reductions, which combine the partitions' sums in partition order (bit-identical
 * results for any placement of the partitions).
 *
 * group mode: all partitions are systems of ONE handle (one GPU: the emulation of P ranks that
 * the tests run; every kernel covers every partition, so no kernel ever waits for another).
 * own_lo/own_hi (host, n_systems entries) are the owned rows relative to each system's first
 * row; the neighbours of partition p are systems p-1 and p+1. */
int sg_pcg_set_partition(sg_pcg* h, const int64_t* own_lo_host, const int64_t* own_hi_host);

/* peer mode: one partition per rank (one process per GPU), the handle holds one system.  Each
 * rank exports an opaque blob (sg_pcg_peer_info_size() bytes: CUDA IPC handles of its
 * workspace and reduction block, the byte offset of s, its extended size and owned rows); the
 * blobs of all ranks are exchanged out of band (torch.distributed all_gather); sg_pcg_set_peers
 * maps the neighbours' workspaces and every rank's reduction block.  The s halo is then written
 * straight into the neighbours' ghost rows over NVLink by the kernels, and each reduction is
 * one peer store of two doubles per rank plus a flag (release / acquire at system scope)
 * polled by one thread per rank -- no host round trip, no collective library call. */
int sg_pcg_peer_info_size(void);
int sg_pcg_peer_export(sg_pcg* h, int64_t own_lo, int64_t own_hi, int32_t world, void* info_out);
int sg_pcg_set_peers(sg_pcg* h, int32_t rank, int32_t world, const void* infos);

/* Rows [r0, r1) of a CSR matrix restricted to columns [c0, c1) (stored as col - c0 + col_base),
 * storage order kept: a row partition's extended local system / a GNN block (no reference
 * counterpart).  out_offs (r1 - r0 + 1 entries) starts at entry_base; out_src[k] = source entry
 * index of kept entry k (values gather with sg_gather_f64; may be NULL).  out_offs == NULL: only
 * count into *out_nnz_host.  Synchronizes when out_nnz_host != NULL. */
int sg_csr_row_block(const int32_t* offs, const int32_t* cols, int64_t r0, int64_t r1, int64_t c0,
                     int64_t c1, int64_t col_base, int64_t entry_base, int32_t* out_offs,
                     int32_t* out_cols, int32_t* out_src, int64_t* out_nnz_host, void* ws,
                     size_t* ws_bytes, void* stream);

/* build_graph features (graphfeat.py:63-105) of a block of rows of a larger matrix: block row
 * li is global row grow0 + li of an n_global-row matrix (PDE grid coordinates and the rowsum / n
 * feature use the global matrix); offs/cols/vals are the block's own CSR (columns block-local),
 * coeff the block's slice of the node field, norm the GLOBAL norm (device scalar). */
int sg_graph_features_block(int64_t n_block, int64_t grow0, int64_t n_global, const int32_t* offs,
                            const int32_t* cols, const double* vals, const double* norm, int family,
                            int64_t nx, int64_t ny, const double* coeff, double coeff_mean,
                            double* node_out, double* edge_out, void* stream);

/* mean_abs_nonzero_norm / matrix_norm over values held by several ranks, still exact: each rank
 * accumulates its values into a transferable accumulator (sg_norm_acc_size() uint64: limbs of
 * the exact fixed-point sum with carries propagated, inf and nan counts); the ranks add their
 * accumulators limb by limb (an integer all-reduce) and sg_norm_from_acc rounds once, so the
 * norm is bit-identical to math.fsum over all values (sparse.py:204-213). */
int sg_norm_acc_size(void);
int sg_norm_accum(const double* vals, int64_t nnz, int kind, uint64_t* acc_out, void* ws, size_t* ws_bytes,
                  void* stream);
int sg_norm_from_acc(const uint64_t* acc, int64_t count, int kind, double* norm_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPAIGRAPH_B200_H */
