/* ml.h — C ABI of libml: the B200 (sm_100a) hot path of the multilevel proximal-Newton method for
 * l1-regularised logistic regression (Treister, Turek, Yavneh, arXiv 1607.00315).
 *
 *   min_w F(w) = sum_i log(1 + exp(-y_i x_i^T w)) + lambda ||w||_1          (C = 1)
 *
 * X is m x n with ROWS = SAMPLES (the paper's X^T), given twice, CSR and CSC, fp32 values and int32
 * indices.  w, every vector and every accumulation are fp64.
 *
 * Memory and ownership
 *   - Every pointer in this header is a DEVICE pointer unless its name ends in _host.
 *   - X, y, index lists, vectors and the workspace are BORROWED: the caller allocates, keeps them alive for the
 *     lifetime of the context, and frees them.  The library never copies, slices or frees X and never allocates
 *     device memory: all scratch is carved from `ws` (size from ml_workspace_bytes).
 *   - All work is enqueued on the stream given to ml_create.  Calls that return host scalars synchronise that
 *     stream only.  One context per stream / host thread; no global mutable state.
 *   - Index lists C are int32, strictly ascending, in [0, n).  C == NULL with nC == n means all columns.  API calls
 *     that take C check it with one device pass and synchronise the stream (ML_E_INVAL if it is malformed).
 *   - Alignment: csr_col, csr_val, csc_row, csc_val 16-byte aligned (they are streamed with 16-byte vector loads and
 *     TMA bulk copies); pointer arrays 4-byte, b 8-byte aligned.  ml_create returns ML_E_INVAL otherwise.
 * Errors
 *   - Every call returns ml_status; nothing throws or exits across the ABI; ml_last_error gives detail.
 *   - ML_E_INVAL: m, n < 1, nnz >= 2^31, lambda <= 0 or non-finite, y not in {-1,+1}, bad C (out of range or not
 *     strictly ascending), misaligned X arrays, malformed X (pointers not from 0 to nnz, indices out of range or not
 *     strictly ascending inside a row/column).
 *   - ML_E_NONFINITE: a NaN or Inf among X's values or the LASSO targets b (ml_create), or in w (ml_set_w; w is left
 *     unchanged).  "Finite entries only (no NaN/Inf accepted into solvers)".
 *   - ML_E_WORKSPACE: ws smaller than ml_workspace_bytes.
 *   - ML_E_CUDA: a CUDA runtime error (message in ml_last_error).
 *   - ML_E_STAGNATION: no trial step passed the line search; the iterate is unchanged.
 *   - ML_E_NOT_CONVERGED: ml_solve hit max_cycles; w holds the last evaluated iterate.
 * Determinism: ml_solve is bitwise reproducible at every m: every reduction has a fixed order, except the large-m
 *   (m > 8192) solver's X_A s scatter, which adds 64-bit fixed-point integers (order-independent; the scale, a power
 *   of 2, bounds each row's sum by 2^62: max |X| x max |coef| x the longest row, so a term is rounded to at most
 *   2^-53 of that bound).  For m > 8192 the API's ml_hessvec and ml_shrink_linesearch (d given without Xd) scatter
 *   X_C v with fp64 atomics: reproducible to rounding only.
 */
#ifndef ML_H
#define ML_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct ml_ctx ml_ctx;

typedef enum {
    ML_OK = 0, ML_E_INVAL = 1, ML_E_CUDA = 2, ML_E_WORKSPACE = 3, ML_E_STAGNATION = 4,
    ML_E_NOT_CONVERGED = 5, ML_E_CONTRACT = 6, ML_E_NONFINITE = 7
} ml_status;

typedef struct {                  /* X is m x n, rows = samples; 0 <= nnz < 2^31 */
    int64_t m, n, nnz;
    /* CSR: may be all NULL when m <= 8192.  Up to that size every pass reads X by columns, including the margins
       from the support's columns; ml_create returns ML_E_INVAL for a NULL CSR above it. */
    const int32_t *csr_rowptr;    /* [m+1] */
    const int32_t *csr_col;       /* [nnz], ascending inside each row */
    const float *csr_val;         /* [nnz] */
    /* Index-free dense X (Eq. 2's dense H): csc_colptr == csc_row == NULL with nnz = m n,
       m <= 8192 and the CSR NULL.  csc_val then holds X column-major (element (i, j) at j m + i); the row of element
       k of column j is k - j m, so no index is stored, copied or read. */
    const int32_t *csc_colptr;    /* [n+1] */
    const int32_t *csc_row;       /* [nnz], ascending inside each column */
    const float *csc_val;         /* [nnz] */
    const int8_t *y;              /* [m], each -1 or +1 */
} ml_data;

typedef struct {                  /* defaults: ml_default_opts */
    double tol_kkt;               /* stop when kappa = ||v||_inf / lambda <= tol_kkt (min-norm subgradient) */
    int32_t max_cycles;
    int32_t nu;                   /* relaxations per level (Alg. 1 step 4) */
    int32_t nu_c;                 /* max relaxations on the coarsest level (Alg. 1 step 3) */
    int32_t K_fine, K_mid, K_coarse; /* inner iterations per relaxation (P:819 reading, DESIGN Q9) */
    double sigma_out, sigma_in, beta; /* Armijo constants (Eq. 4; DESIGN Q7) */
    int32_t max_ls;               /* <= 40 */
    double eps_h;                 /* model ridge (DESIGN Q6) */
    int32_t multilevel;           /* 1: Algorithm 1; 0: finest-level relaxations only */
    int32_t inner_cg;             /* 2: PCD-CG + a PCD step after every kink (default); 1: PCD-CG; 0: plain PCD (DESIGN Q9b) */
    double eta;                   /* inner forcing (0 = off) */
    int32_t pcd_snap;             /* 1 (default): a PCD step first tries the path that sets the coordinates its shrinkage
                                     sends to 0 exactly to 0 for every step length (DESIGN Q27); 0: plain PCD steps */
    int32_t continuation;         /* 1: first one finest relaxation at each of lambda_4 > lambda_3 > lambda_2, lambda_4 =
                                     (lambda_max + lambda) / 2, linearly spaced down to lambda (DESIGN Q28),
                                     then the solve at lambda from that warm start; 0 (default): from w = 0 */
} ml_solve_opts;

typedef struct {
    double F, kappa, vinf, v1, paper_ratio;
    int32_t status, cycles;
    int64_t relaxations;
    int64_t relax_per_level[32];
    int64_t max_supp, nnz_w;
    int64_t nnz_touched;          /* nonzeros streamed by all X passes (algorithmic) */
    int64_t x_passes;
    int64_t kernel_launches;      /* kernels this solve enqueued */
} ml_solve_report;

void ml_default_opts(ml_solve_opts *o);

/* Workspace bytes for a problem of this size (all scratch, iterate, margins, level lists). */
size_t ml_workspace_bytes(int64_t m, int64_t n, int64_t nnz);

/* Bind X, y, lambda (> 0) to a context; w = 0.  `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
   Validates sizes, alignment, lambda, y, X's index structure and the finiteness of X's values (device passes; one
   stream synchronisation).  Builds the static heavy-row schedule (one pass over rowptr). */
ml_status ml_create(const ml_data *X, double lambda, void *cuda_stream, void *ws, size_t ws_bytes, ml_ctx **out);
/* The squared-loss instance of Eq. 1: the LASSO of Eq. 2 with H = X^T X and g = -X^T b, i.e.
   F(w) = sum_i (x_i^T w - b_i)^2 / 2 + lambda ||w||_1 (DESIGN Q29).  b: [m] targets (device, fp64, borrowed like X);
   X->y is not read and may be NULL.  Every other entry point works unchanged on the context (r_i = z_i - b_i,
   D_i = 1); ML_E_INVAL if b is NULL. */
ml_status ml_create_lasso(const ml_data *X, const double *b, double lambda, void *cuda_stream, void *ws, size_t ws_bytes,
                          ml_ctx **out);
ml_status ml_destroy(ml_ctx *c);

/* w <- w_dev[n] (device); margins are recomputed at the next evaluation.  Checks w_dev for NaN / Inf first (one
   device pass, synchronises the stream): ML_E_NONFINITE and w unchanged if it holds one. */
ml_status ml_set_w(ml_ctx *c, const double *w_dev);
/* w_dev[n] <- w */
ml_status ml_get_w(ml_ctx *c, double *w_dev);
/* per-sample state after the last evaluation/update: z, r, D (each [m], device; NULL skips) */
ml_status ml_get_rows(ml_ctx *c, double *z_dev, double *r_dev, double *D_dev);

/* A1 + A2: margins z = Xw from scratch (CSR pass; for m <= 8192 from the support's CSC columns) with
   fused tau, D, r, loss; F = L + lambda||w||_1;
   then g_C = X_C^T r and h_C = sum_i X_ij^2 D_i over C (CSC gather).  F_host may be NULL; g_C / h_C may be NULL. */
ml_status ml_eval_f_grad(ml_ctx *c, const int32_t *C, int64_t nC, double *F_host, double *g_C, double *h_C);
/* h_C = sum_i X_ij^2 D_i with D from the current state. */
ml_status ml_diag_hess(ml_ctx *c, const int32_t *C, int64_t nC, double *h_C);
/* Hv_C = X_C^T D X_C v_C with D from the current state, no ridge. */
ml_status ml_hessvec(ml_ctx *c, const int32_t *C, int64_t nC, const double *v_C, double *Hv_C);
/* A7: Armijo line search on F along d over C (Eq. 4; DESIGN Q7, Q26), then w += alpha d,
   z += alpha Xd and refresh of tau, D, r (A1 incremental).  g_C = gradient over C at the current w.
   d_C == NULL: d = Sh_{lambda/h}(w - g/h) - w (Eq. 5 with D = diag(h) + eps_h, PCD P:99), h_C required.
   Xd == NULL: computed with one X_C pass.  alpha_host = 0 and ML_E_STAGNATION when no trial passes. */
ml_status ml_shrink_linesearch(ml_ctx *c, const int32_t *C, int64_t nC, const double *g_C, const double *h_C,
                               const double *d_C, const double *Xd, const ml_solve_opts *o,
                               double *alpha_host, double *F_new_host);
/* A8: C_out = supp(w) U the (k_total - |supp|) largest |g_j| off the support, ties by ascending
   index (DESIGN Q14); C_out ascending, *nC_out_host = max(k_total, |supp|) capped at n.  g is [n]. */
ml_status ml_select_coarse(ml_ctx *c, const double *g, int64_t k_total, int32_t *C_out, int64_t *nC_out_host);
/* A9: the multilevel solve from w = 0 (Algorithm 1 P:155-173 per P:798). */
ml_status ml_solve(ml_ctx *c, const ml_solve_opts *o, ml_solve_report *rep);

const char *ml_status_str(ml_status s);
const char *ml_last_error(const ml_ctx *c);
/* kernels this context has launched so far (for launch accounting) */
int64_t ml_kernel_launches(const ml_ctx *c);
/* Measurement.  Pass classes: 0 margins (A1), 1 finest gather (A2/A3), 2 coarse gather, 3 X_A s scatter (A5),
   4 X_A^T (D o Xs) gather (A5), 5 inner direction (A4), 6 m-side model pass (A6), 7 step apply (A6), 8 outer line
   search (A7), 9 update (A7), 10 selection (A8), 11 bookkeeping, 12 API-call passes.
   ml_profile: reset the per-class counters and record a CUDA event pair around every logical pass of the classes
   in class_mask (0 = no event timing).  ml_profile_read (synchronises): per class [16] the summed event time (ms),
   the passes launched, and the nonzeros streamed and segments (rows / columns) visited on the device. */
ml_status ml_profile(ml_ctx *c, uint32_t class_mask);
ml_status ml_profile_read(ml_ctx *c, double *ms_host, int64_t *passes_host, int64_t *nnz_host, int64_t *segs_host);
/* Diagnostics: nanoseconds spent per phase of the persistent small-m inner solver, 16 entries (block 0): entries
   0-6 for relaxations with |A| < 2048, 8-14 for larger ones: direction, X_A s scatter, barrier + totals, row sums,
   barrier + totals + step decision, D o X sigma to shared memory, Hs stream + step; 7 and 15: the outer line
   search and update that end each relaxation (R14-R18). */
ml_status ml_inner_phases(ml_ctx *c, uint64_t *ns_host, int reset);
/* Batched replicas: the context's cooperative (persistent) kernels use at most `blocks` CTAs
   (one per SM; <= 0 or more than the SM count restores the whole GPU).  Several contexts on their own streams, each
   driven by its own host thread, then solve side by side: small problems are latency-bound on the whole GPU.
   ML_E_INVAL if the small-m solver would own more than 64 rows per block (m > 64 blocks). */
ml_status ml_set_sm_share(ml_ctx *c, int blocks);
/* Engine selection for A/B measurement and parity tests (defaults need no call).
   bit 0: the large-m (m > 8192) column gathers of A2 use the merge-path column pass (every thread gets the same number
          of nonzeros + column ends whatever the column lengths; off by default: measured slower than the segment
          engine on configs 4-5); ML_E_INVAL on a small-m context (which reads X through shared-memory passes).
   bit 3: the large-m inner solver's X_A s and H sigma streams claim their column units dynamically from a grid-wide
          counter whatever the unit count (by default only with >= 32 units per warp, where static shares left blocks
          waiting on the slowest).
   bit 4: the large-m inner solver takes the heavy-column path (X_A s of the longest columns from their row-major copy,
          without atomics; ml_heavy_info) in every relaxation; bit 6: in the relaxations whose free set holds >= 1/4
          of their nonzeros; bit 5: never; none of them: the context's default, which is bit 6 when X has >= 2^26
          nonzeros and those columns hold >= 2^26 (the copy is then built by ml_create; measured faster on cfg 5,
          slower on cfg 3-4), else never.  A first request on a smaller X builds the copy (device passes over X,
          synchronises the stream).  ML_E_INVAL for bit 4 when the context has no heavy path (small m, the longest
          columns hold < 1/10 of X, or a row holds more than 768 of their nonzeros). */
ml_status ml_set_engine(ml_ctx *c, uint32_t flags);
/* Diagnostics of the large-m heavy-column path (DESIGN 8.2; off for m <= 8192): info_host[8] = built (0/1), |H|,
   nonzeros of H, warp chunks of its row-major copy, 0, 0 (reserved), relaxations that ran it since ml_create, the
   mode (0: by the free set's share of H, 1: always, 2: never; ml_set_engine bits 4 / 5 / 6). */
ml_status ml_heavy_info(ml_ctx *c, int64_t *info_host);
/* Diagnostics: copy up to `cap` relaxation records of the last solve into rows_host (host memory, 48 bytes each:
   int32 level, outcome, inner_iters, nA; int64 nC; double F_before, F_after, alpha); returns the record count. */
int64_t ml_trace(ml_ctx *c, void *rows_host, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
