/* mlo.h — CPU ORACLE (test infrastructure only).
 *
 * A plain, slow, single-threaded fp64 implementation of the multilevel
 * proximal-Newton method for l1-regularised logistic regression
 * (Algorithm 1, Eqs. 3-6, Eq. 9 P:139-141,
 * coarse-variable choice P:175-196, logistic gradient/Hessian P:791-796,
 * application) in the readings listed in DESIGN.md "Readings".
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code with the
 * CUDA path (paper_1607_00315_b200/); this header is a separate, duplicated
 * declaration of the same call set with the `mlo_` prefix and HOST pointers.
 *
 * Orientation: X is m x n with ROWS = SAMPLES (the paper's X^T).
 */
#ifndef MLO_H
#define MLO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct mlo_ctx mlo_ctx;

enum { MLO_OK = 0, MLO_E_INVAL = 1, MLO_E_STAGNATION = 4, MLO_E_NOT_CONVERGED = 5, MLO_E_CONTRACT = 6 };
/* relaxation outcomes (trace) */
enum { MLO_R_UPDATED = 0, MLO_R_CONVERGED = 1, MLO_R_NOSTEP = 2, MLO_R_STAGNATION = 3 };

typedef struct {
    double tol_kkt;      /* stop when kappa = ||v||_inf / lambda <= tol_kkt (DESIGN Q16) */
    int32_t max_cycles;
    int32_t nu;          /* relaxations per level (Alg. 1 step 4) */
    int32_t nu_c;        /* max relaxations on the coarsest level (Alg. 1 step 3) */
    int32_t K_fine, K_mid, K_coarse; /* inner PCD iterations per relaxation */
    double sigma_out, sigma_in, beta; /* Armijo constants (DESIGN Q7) */
    int32_t max_ls;
    double eps_h;        /* ridge added to the quadratic model only (DESIGN Q6) */
    int32_t multilevel;  /* 1: Algorithm 1; 0: finest-level relaxations only (newGLMNET-like baseline) */
    int32_t inner_cg;    /* 2: PCD-CG + a PCD step after every kink (default); 1: PCD-CG; 0: plain PCD (DESIGN Q9b) */
    double eta;          /* inner forcing: stop when the model's min-norm subgradient <= eta * its value at d = 0 (0 = off) */
    int32_t pcd_snap;    /* 1 (default): PCD steps set coordinates whose shrinkage target is 0 exactly to 0 for every step length (Q27) */
    int32_t continuation; /* 1: before the solve, one finest relaxation at each of lambda_4 > lambda_3 > lambda_2 (
                             DESIGN Q28), then the solve at lambda from that warm start; 0 (default): start at w = 0 */
} mlo_opts;

typedef struct {
    double F, kappa, vinf, v1, paper_ratio;
    int32_t status, cycles;
    int64_t relaxations;      /* total */
    int64_t relax_per_level[32];
    int64_t max_supp, nnz_w;
    int64_t nnz_touched;      /* sum over all X passes of the nonzeros streamed */
    int64_t x_passes;         /* number of X passes (margins, gathers, scatters) */
} mlo_report;

typedef struct {            /* one relaxation, for tests (monotonicity etc.) */
    int32_t level, outcome, inner_iters, nA;
    int64_t nC;
    double F_before, F_after, alpha;
} mlo_trace_row;

void mlo_default_opts(mlo_opts *o);

mlo_ctx *mlo_create(int64_t m, int64_t n, int64_t nnz,
                    const int32_t *csr_rowptr, const int32_t *csr_col, const float *csr_val,
                    const int32_t *csc_colptr, const int32_t *csc_row, const float *csc_val,
                    const int8_t *y, double lambda);
/* The squared-loss instance (LASSO, Eq. 2 P:49-53 with H = X^T X, g = -X^T b): ell_i = (x_i^T w - b_i)^2 / 2, r_i =
   x_i^T w - b_i, D_i = 1 (DESIGN Q29).  b: [m] targets. */
mlo_ctx *mlo_create_lasso(int64_t m, int64_t n, int64_t nnz,
                          const int32_t *csr_rowptr, const int32_t *csr_col, const float *csr_val,
                          const int32_t *csc_colptr, const int32_t *csc_row, const float *csc_val,
                          const double *b, double lambda);
void mlo_destroy(mlo_ctx *c);

void mlo_set_w(mlo_ctx *c, const double *w);   /* [n]; recomputes margins from scratch */
void mlo_get_w(const mlo_ctx *c, double *w);    /* [n] */
/* per-sample state after the last refresh: z, r, D, loss terms (each [m]; NULL skips) */
void mlo_get_rows(const mlo_ctx *c, double *z, double *r, double *D, double *ell);

/* Margins from scratch (z = Xw), per-sample loss/weights, F; then g_C, h_C.
   C: strictly ascending indices in [0,n); C == NULL means all columns (nC must be n). */
int mlo_eval_f_grad(mlo_ctx *c, const int32_t *C, int64_t nC, double *F, double *g_C, double *h_C);
/* h_C = sum_i X_ij^2 D_i with D from the current state. */
int mlo_diag_hess(mlo_ctx *c, const int32_t *C, int64_t nC, double *h_C);
/* Hv_C = X_C^T D X_C v_C with D from the current state (no ridge). */
int mlo_hessvec(mlo_ctx *c, const int32_t *C, int64_t nC, const double *v_C, double *Hv_C);
/* Line search on F (Eq. 4) along d_C over C, then update w, z, r, D.
   g_C: gradient over C at the current w (required).  h_C: required when d_C == NULL.
   d_C == NULL: d = Sh_{lambda/h}(w - g/h) - w on C (Eq. 5, D = diag(h) + eps_h; PCD).
   Xd == NULL: computed from X_C d.  alpha = 0 and MLO_E_STAGNATION when no trial passes. */
int mlo_shrink_linesearch(mlo_ctx *c, const int32_t *C, int64_t nC, const double *g_C, const double *h_C,
                          const double *d_C, const double *Xd, const mlo_opts *o,
                          double *alpha, double *F_new);
/* supp(w) U top-(k_total - |supp|) of |g| off the support, ties by ascending index (DESIGN Q14);
   C_out ascending, *nC_out = max(k_total, |supp|) (capped at n). */
int mlo_select_coarse(mlo_ctx *c, const double *g, int64_t k_total, int32_t *C_out, int64_t *nC_out);
/* One relaxation RELAX(C) (DESIGN "Algorithm", lines R1-R18) with K inner iterations; gathers g,h itself. */
int mlo_relax(mlo_ctx *c, const int32_t *C, int64_t nC, int32_t K, const mlo_opts *o, int32_t *outcome);
/* Level sizes k[0..L] (k[0] = n) for |A_f| and |supp|; returns L. */
int mlo_level_sizes(int64_t nAf, int64_t nS, int64_t n, int64_t *k);
/* The full multilevel solve from w = 0 (DESIGN "Algorithm", lines S1-S18). */
int mlo_solve(mlo_ctx *c, const mlo_opts *o, mlo_report *rep);

int64_t mlo_trace_len(const mlo_ctx *c);
void mlo_trace_get(const mlo_ctx *c, int64_t i, mlo_trace_row *row);
void mlo_trace_clear(mlo_ctx *c);

/* scalar pieces, exposed so tests can pin them against closed forms */
double mlo_soft_shrink(double t, double a);               /* Eq. 6 */
double mlo_scalar_prox(double a, double b, double lam);   /* Eq. 11 minimiser, sign fixed (DESIGN Q1) */
double mlo_logloss(double t);                             /* log(1+e^-t) */
double mlo_tau(double s);                                 /* 1/(1+e^-s) */
double mlo_weight(double t);                              /* tau(t) tau(-t) */

#ifdef __cplusplus
}
#endif
#endif
