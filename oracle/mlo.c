/* mlo.c — CPU ORACLE (test infrastructure only; see mlo.h).
 *
 * Plain single-threaded IEEE binary64.  Compiled with -O2 -ffp-contract=off,
 * never -ffast-math.  Every sum runs sequentially in the storage order of X
 * (CSR order for margins, CSC order for column sums).  Every step cites the
 * passage it follows; DESIGN.md "Readings" lists where the paper is silent.
 *
 * Notation (SURVEY §8 / DESIGN): X in R^{m x n}, rows = samples (paper's X^T,
 * P:796).  z = Xw, t_i = y_i z_i, tau(s) = 1/(1+e^-s),
 * r_i = (tau(t_i) - 1) y_i = -y_i tau(-t_i) (C = 1),
 * D_i = tau(t_i)(1 - tau(t_i)), g = X^T r, H = X^T D X.
 * F(w) = sum_i log(1 + e^{-t_i}) + lambda ||w||_1 (lambda = 1/C).
 */
#include "mlo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct mlo_ctx {
    int64_t m, n, nnz;
    const int32_t *rp, *ci; const float *cv;  /* CSR */
    const int32_t *cp, *ri; const float *rv;  /* CSC */
    const int8_t *y;                /* logistic labels (NULL for the squared loss) */
    const double *b;                /* squared-loss (LASSO) targets, Eq. 2 with H = X^T X, g = -X^T b (NULL = logistic) */
    double lam;
    double *w;                      /* [n] */
    double *z, *r, *D, *ell;        /* [m] per-sample state */
    double L;                       /* sum_i ell_i */
    mlo_trace_row *trace; int64_t ntrace, captrace;
    int64_t nnz_touched, x_passes;
};

/* ------------------------------------------------------------ scalar pieces */
double mlo_soft_shrink(double t, double a) {            /* Eq. 6 */
    double s = fabs(t) - a;
    if (s <= 0.0) return 0.0;
    return t > 0.0 ? s : -s;
}
double mlo_scalar_prox(double a, double b, double lam) { /* argmin 1/2 a z^2 + b z + lam|z|, Eq. 11 P:178-180;
                                                            closed form of P:182-190 with the sign fixed (DESIGN Q1) */
    return -mlo_soft_shrink(b, lam) / a;
}
double mlo_logloss(double t) {                           /* log(1+e^{-t}) = max(-t,0) + log1p(e^{-|t|}) */
    return (t < 0.0 ? -t : 0.0) + log1p(exp(-fabs(t)));
}
double mlo_tau(double s) {                               /* tau(s) = 1/(1+e^{-s}) */
    if (s >= 0.0) return 1.0 / (1.0 + exp(-s));
    double e = exp(s);
    return e / (1.0 + e);
}
double mlo_weight(double t) {                            /* D = tau(t)(1-tau(t)) = e/(1+e)^2, e = e^{-|t|} */
    double e = exp(-fabs(t));
    return e / ((1.0 + e) * (1.0 + e));
}

void mlo_default_opts(mlo_opts *o) {
    memset(o, 0, sizeof(*o));
    o->tol_kkt = 1e-6; o->max_cycles = 1000; o->nu = 1; o->nu_c = 5;
    o->K_fine = 2; o->K_mid = 3; o->K_coarse = 5;    /* tuned with this oracle, DESIGN "Defaults" */
    o->sigma_out = 1e-2; o->sigma_in = 1e-2; o->beta = 0.5; o->max_ls = 40;
    o->eps_h = 1e-12; o->multilevel = 1; o->inner_cg = 2; o->eta = 0.0; o->pcd_snap = 1;
}

/* --------------------------------------------------------------- context */
static void refresh_rows(mlo_ctx *c) {  /* per-sample quantities at the current z, then L */
    double L = 0.0;
    for (int64_t i = 0; i < c->m; ++i) {
        if (c->b) {                                       /* squared loss: ell = (z - b)^2 / 2, r = ell', D = ell'' = 1 */
            double r = c->z[i] - c->b[i];
            c->ell[i] = 0.5 * r * r;
            c->r[i] = r;
            c->D[i] = 1.0;
            L += c->ell[i];
            continue;
        }
        double t = (double)c->y[i] * c->z[i];
        c->ell[i] = mlo_logloss(t);
        c->r[i] = -(double)c->y[i] * mlo_tau(-t);      /* (tau(t)-1) y = -y tau(-t) */
        c->D[i] = mlo_weight(t);
        L += c->ell[i];
    }
    c->L = L;
}
static void margins_from_scratch(mlo_ctx *c) {          /* z = X w in CSR order */
    for (int64_t i = 0; i < c->m; ++i) {
        double s = 0.0;
        for (int64_t p = c->rp[i]; p < c->rp[i + 1]; ++p) s += (double)c->cv[p] * c->w[c->ci[p]];
        c->z[i] = s;
    }
    c->nnz_touched += c->nnz; c->x_passes += 1;
    refresh_rows(c);
}
static double l1_all(const mlo_ctx *c) {
    double s = 0.0;
    for (int64_t j = 0; j < c->n; ++j) s += fabs(c->w[j]);
    return s;
}
static double F_current(const mlo_ctx *c) { return c->L + c->lam * l1_all(c); }

static mlo_ctx *create_impl(int64_t m, int64_t n, int64_t nnz,
                            const int32_t *csr_rowptr, const int32_t *csr_col, const float *csr_val,
                            const int32_t *csc_colptr, const int32_t *csc_row, const float *csc_val,
                            const int8_t *y, const double *b, double lambda) {
    if (m < 1 || n < 1 || nnz < 0 || !(lambda > 0.0) || !isfinite(lambda)) return NULL;
    if (!b) for (int64_t i = 0; i < m; ++i) if (y[i] != 1 && y[i] != -1) return NULL;
    mlo_ctx *c = (mlo_ctx *)calloc(1, sizeof(mlo_ctx));
    c->m = m; c->n = n; c->nnz = nnz;
    c->rp = csr_rowptr; c->ci = csr_col; c->cv = csr_val;
    c->cp = csc_colptr; c->ri = csc_row; c->rv = csc_val;
    c->y = b ? NULL : y; c->b = b; c->lam = lambda;
    c->w = (double *)calloc((size_t)n, sizeof(double));
    c->z = (double *)calloc((size_t)m, sizeof(double));
    c->r = (double *)calloc((size_t)m, sizeof(double));
    c->D = (double *)calloc((size_t)m, sizeof(double));
    c->ell = (double *)calloc((size_t)m, sizeof(double));
    refresh_rows(c);   /* w = 0, z = 0 */
    return c;
}
mlo_ctx *mlo_create(int64_t m, int64_t n, int64_t nnz,
                    const int32_t *csr_rowptr, const int32_t *csr_col, const float *csr_val,
                    const int32_t *csc_colptr, const int32_t *csc_row, const float *csc_val,
                    const int8_t *y, double lambda) {
    return create_impl(m, n, nnz, csr_rowptr, csr_col, csr_val, csc_colptr, csc_row, csc_val, y, NULL, lambda);
}
mlo_ctx *mlo_create_lasso(int64_t m, int64_t n, int64_t nnz,
                          const int32_t *csr_rowptr, const int32_t *csr_col, const float *csr_val,
                          const int32_t *csc_colptr, const int32_t *csc_row, const float *csc_val,
                          const double *b, double lambda) {
    if (!b) return NULL;
    return create_impl(m, n, nnz, csr_rowptr, csr_col, csr_val, csc_colptr, csc_row, csc_val, NULL, b, lambda);
}
void mlo_destroy(mlo_ctx *c) {
    if (!c) return;
    free(c->w); free(c->z); free(c->r); free(c->D); free(c->ell); free(c->trace);
    free(c);
}
void mlo_set_w(mlo_ctx *c, const double *w) {
    memcpy(c->w, w, sizeof(double) * (size_t)c->n);
    margins_from_scratch(c);
}
void mlo_get_w(const mlo_ctx *c, double *w) { memcpy(w, c->w, sizeof(double) * (size_t)c->n); }
void mlo_get_rows(const mlo_ctx *c, double *z, double *r, double *D, double *ell) {
    size_t b = sizeof(double) * (size_t)c->m;
    if (z) memcpy(z, c->z, b);
    if (r) memcpy(r, c->r, b);
    if (D) memcpy(D, c->D, b);
    if (ell) memcpy(ell, c->ell, b);
}

static int check_C(const mlo_ctx *c, const int32_t *C, int64_t nC) {
    if (!C) return nC == c->n ? 0 : -1;
    if (nC < 0 || nC > c->n) return -1;
    for (int64_t p = 0; p < nC; ++p) {
        if (C[p] < 0 || C[p] >= c->n) return -1;
        if (p > 0 && C[p] <= C[p - 1]) return -1;
    }
    return 0;
}
#define COL(C, p) ((C) ? (int64_t)(C)[p] : (int64_t)(p))

/* g_j = sum_i X_ij r_i,  h_j = sum_i X_ij^2 D_i over j in C (CSC order) */
static void gather_gh(mlo_ctx *c, const int32_t *C, int64_t nC, double *g, double *h) {
    for (int64_t p = 0; p < nC; ++p) {
        int64_t j = COL(C, p);
        double sg = 0.0, sh = 0.0;
        for (int64_t q = c->cp[j]; q < c->cp[j + 1]; ++q) {
            double x = (double)c->rv[q];
            sg += x * c->r[c->ri[q]];
            sh += x * x * c->D[c->ri[q]];
        }
        if (g) g[p] = sg;
        if (h) h[p] = sh;
        c->nnz_touched += c->cp[j + 1] - c->cp[j];
    }
    c->x_passes += 1;
}
/* out = X_C v (m-vector), columns of C in order */
static void apply_XC(mlo_ctx *c, const int32_t *C, int64_t nC, const double *v, double *out) {
    memset(out, 0, sizeof(double) * (size_t)c->m);
    for (int64_t p = 0; p < nC; ++p) {
        int64_t j = COL(C, p);
        for (int64_t q = c->cp[j]; q < c->cp[j + 1]; ++q) out[c->ri[q]] += (double)c->rv[q] * v[p];
        c->nnz_touched += c->cp[j + 1] - c->cp[j];
    }
    c->x_passes += 1;
}
/* out_C = X_C^T (D o s) */
static void apply_XCt_D(mlo_ctx *c, const int32_t *C, int64_t nC, const double *s, double *out) {
    for (int64_t p = 0; p < nC; ++p) {
        int64_t j = COL(C, p);
        double acc = 0.0;
        for (int64_t q = c->cp[j]; q < c->cp[j + 1]; ++q) acc += (double)c->rv[q] * c->D[c->ri[q]] * s[c->ri[q]];
        out[p] = acc;
        c->nnz_touched += c->cp[j + 1] - c->cp[j];
    }
    c->x_passes += 1;
}

int mlo_eval_f_grad(mlo_ctx *c, const int32_t *C, int64_t nC, double *F, double *g_C, double *h_C) {
    if (check_C(c, C, nC)) return MLO_E_INVAL;
    margins_from_scratch(c);
    if (F) *F = F_current(c);
    if (g_C || h_C) gather_gh(c, C, nC, g_C, h_C);
    return MLO_OK;
}
int mlo_diag_hess(mlo_ctx *c, const int32_t *C, int64_t nC, double *h_C) {
    if (check_C(c, C, nC)) return MLO_E_INVAL;
    gather_gh(c, C, nC, NULL, h_C);
    return MLO_OK;
}
int mlo_hessvec(mlo_ctx *c, const int32_t *C, int64_t nC, const double *v_C, double *Hv_C) {
    if (check_C(c, C, nC)) return MLO_E_INVAL;
    double *Xv = (double *)malloc(sizeof(double) * (size_t)c->m);
    apply_XC(c, C, nC, v_C, Xv);                 /* X v */
    apply_XCt_D(c, C, nC, Xv, Hv_C);             /* X^T D X v */
    free(Xv);
    return MLO_OK;
}

/* ------------------------------------------------------------ line search on F
 * Eq. 4 with the Armijo reading of DESIGN Q7:
 *   alpha = first of 1, beta, beta^2, ... (<= max_ls) with
 *   F(w + alpha d) - F(w) <= sigma_out * alpha * Delta,
 *   Delta = g_A^T d + lambda (||w_A + d||_1 - ||w_A||_1).
 * The difference F(w + alpha d) - F(w) is evaluated term by term (DESIGN Q26):
 *   sum_i [ell(t_i + delta_i) - ell(t_i)] + lambda sum_{j in A} (|w_j + alpha d_j| - |w_j|),
 *   delta_i = alpha y_i Xd_i, and ell(t + delta) - ell(t) = log1p(tau(-t) expm1(-delta)) when |delta| <= 1
 *   (the exact identity (1 + e^{-t-delta}) / (1 + e^{-t}) = 1 + tau(-t)(e^{-delta} - 1)), else the plain difference.
 * On success: w_A += alpha d; z += alpha Xd; refresh r, D, ell (Lemma P:207-243: F cannot increase).
 */
static double dloss(double t, double delta) {            /* ell(t + delta) - ell(t) */
    if (fabs(delta) <= 1.0) return log1p(mlo_tau(-t) * expm1(-delta));
    return mlo_logloss(t + delta) - mlo_logloss(t);
}
static int outer_linesearch(mlo_ctx *c, const int32_t *A, int64_t nA, const double *gA, const double *d,
                            const double *Xd, const mlo_opts *o, double *alpha_out, double *Fnew_out) {
    double dl1 = 0.0, gd = 0.0;
    for (int64_t p = 0; p < nA; ++p) {
        double wj = c->w[COL(A, p)];
        dl1 += fabs(wj + d[p]) - fabs(wj);
        gd += gA[p] * d[p];
    }
    double Delta = gd + c->lam * dl1;
    double alpha = 1.0;
    for (int32_t t = 0; t < o->max_ls; ++t, alpha *= o->beta) {
        double dL = 0.0;
        for (int64_t i = 0; i < c->m; ++i) {
            if (c->b) {   /* (z + delta - b)^2/2 - (z - b)^2/2 = delta (z - b + delta/2), exact algebra (as Q26) */
                double delta = alpha * Xd[i];
                dL += delta * ((c->z[i] - c->b[i]) + 0.5 * delta);
                continue;
            }
            double ti = (double)c->y[i] * c->z[i];
            dL += dloss(ti, alpha * (double)c->y[i] * Xd[i]);
        }
        double dl1t = 0.0;
        for (int64_t p = 0; p < nA; ++p) { double wj = c->w[COL(A, p)]; dl1t += fabs(wj + alpha * d[p]) - fabs(wj); }
        double dF = dL + c->lam * dl1t;
        if (dF <= o->sigma_out * alpha * Delta) {
            for (int64_t p = 0; p < nA; ++p) c->w[COL(A, p)] += alpha * d[p];
            for (int64_t i = 0; i < c->m; ++i) c->z[i] += alpha * Xd[i];
            refresh_rows(c);
            *alpha_out = alpha;
            *Fnew_out = F_current(c);
            return MLO_OK;
        }
    }
    *alpha_out = 0.0;
    *Fnew_out = F_current(c);
    return MLO_E_STAGNATION;
}

int mlo_shrink_linesearch(mlo_ctx *c, const int32_t *C, int64_t nC, const double *g_C, const double *h_C,
                          const double *d_C, const double *Xd, const mlo_opts *o,
                          double *alpha, double *F_new) {
    if (check_C(c, C, nC) || !g_C || (!d_C && !h_C)) return MLO_E_INVAL;
    double *d = (double *)malloc(sizeof(double) * (size_t)(nC ? nC : 1));
    double *xd = (double *)malloc(sizeof(double) * (size_t)c->m);
    if (d_C) memcpy(d, d_C, sizeof(double) * (size_t)nC);
    else
        for (int64_t p = 0; p < nC; ++p) {   /* Eq. 5 with D = diag(h) + eps_h (PCD) */
            double hh = h_C[p] + o->eps_h, wj = c->w[COL(C, p)];
            d[p] = mlo_soft_shrink(wj - g_C[p] / hh, c->lam / hh) - wj;
        }
    if (Xd) memcpy(xd, Xd, sizeof(double) * (size_t)c->m);
    else apply_XC(c, C, nC, d, xd);
    int st = outer_linesearch(c, C, nC, g_C, d, xd, o, alpha, F_new);
    free(d); free(xd);
    return st;
}

/* ------------------------------------------------------------ coarse variables
 * C = supp(w) U the largest-|g| indices off the support;
 * ties by ascending index (DESIGN Q14).
 */
static const double *g_sort_key;
static int cmp_rank(const void *a, const void *b) {
    int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
    double gi = fabs(g_sort_key[i]), gj = fabs(g_sort_key[j]);
    if (gi > gj) return -1;
    if (gi < gj) return 1;
    return (i > j) - (i < j);
}
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

int mlo_select_coarse(mlo_ctx *c, const double *g, int64_t k_total, int32_t *C_out, int64_t *nC_out) {
    int32_t *off = (int32_t *)malloc(sizeof(int32_t) * (size_t)c->n);
    int64_t ns = 0, no = 0;
    for (int64_t j = 0; j < c->n; ++j) {
        if (c->w[j] != 0.0) C_out[ns++] = (int32_t)j;
        else off[no++] = (int32_t)j;
    }
    int64_t take = k_total - ns;
    if (take < 0) take = 0;
    if (take > no) take = no;
    g_sort_key = g;
    qsort(off, (size_t)no, sizeof(int32_t), cmp_rank);
    for (int64_t t = 0; t < take; ++t) C_out[ns + t] = off[t];
    qsort(C_out, (size_t)(ns + take), sizeof(int32_t), cmp_i32);
    *nC_out = ns + take;
    free(off);
    return MLO_OK;
}

/* ------------------------------------------------------------ one relaxation
 * RELAX(C) = Eq. 3 + Eq. 4 on the coarse problem Eq. 9,
 * restricted to the free set A (P:455-462 via P:790; DESIGN Q15), with the
 * quadratic model minimised approximately by K iterations of PCD (Eq. 5 with
 * D = diag(H); DESIGN Q5) under an Armijo line search on the model.
 * Lines R1-R18 refer to DESIGN.md "Algorithm".
 */
static void trace_push(mlo_ctx *c, mlo_trace_row row) {
    if (c->ntrace == c->captrace) {
        c->captrace = c->captrace ? 2 * c->captrace : 256;
        c->trace = (mlo_trace_row *)realloc(c->trace, sizeof(mlo_trace_row) * (size_t)c->captrace);
    }
    c->trace[c->ntrace++] = row;
}

typedef struct {            /* what RELAX hands back to the solver */
    int32_t outcome;
    int32_t *A; int64_t nA; /* free set (indices), owned by caller buffers */
} relax_out;

/* gC/hC: gradient and Hessian diagonal over C at the current w (the "E" of line R1), or NULL to gather them. */
static int relax_core(mlo_ctx *c, const int32_t *C, int64_t nC, double *gC, double *hC, int32_t K,
                      const mlo_opts *o, int32_t level, int32_t *A_out, int64_t *nA_out, double *gA_out,
                      int32_t *outcome) {
    int64_t m = c->m;
    double lam = c->lam;
    double F_before = F_current(c);
    mlo_trace_row row = {level, MLO_R_NOSTEP, 0, 0, nC, F_before, F_before, 0.0};
    double *g = gC, *h = hC;
    int own = 0;
    if (!g) {                                                        /* R1 */
        own = 1;
        g = (double *)malloc(sizeof(double) * (size_t)(nC ? nC : 1));
        h = (double *)malloc(sizeof(double) * (size_t)(nC ? nC : 1));
        gather_gh(c, C, nC, g, h);
    }
    /* R2: free set and restricted KKT (min-norm subgradient) */
    int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nC ? nC : 1));
    double *gA = (double *)malloc(sizeof(double) * (size_t)(nC ? nC : 1));
    double *hA = (double *)malloc(sizeof(double) * (size_t)(nC ? nC : 1));
    int64_t nA = 0;
    double vmax = 0.0;
    for (int64_t p = 0; p < nC; ++p) {
        int64_t j = COL(C, p);
        double wj = c->w[j], v;
        if (wj != 0.0) v = g[p] + lam * (wj > 0.0 ? 1.0 : -1.0);
        else v = mlo_soft_shrink(g[p], lam);
        if (fabs(v) > vmax) vmax = fabs(v);
        if (wj != 0.0 || fabs(g[p]) > lam) { A[nA] = (int32_t)j; gA[nA] = g[p]; hA[nA] = h[p]; ++nA; }
    }
    if (A_out) { memcpy(A_out, A, sizeof(int32_t) * (size_t)nA); memcpy(gA_out, gA, sizeof(double) * (size_t)nA); *nA_out = nA; }
    row.nA = (int32_t)nA;
    int st = MLO_OK;
    if (vmax / lam <= o->tol_kkt) {
        row.outcome = MLO_R_CONVERGED;
        goto done;
    }
    {
        /* R3 */
        double *d = (double *)calloc((size_t)(nA ? nA : 1), sizeof(double));
        double *Hd = (double *)calloc((size_t)(nA ? nA : 1), sizeof(double));
        double *Xd = (double *)calloc((size_t)m, sizeof(double));
        double *u = (double *)malloc(sizeof(double) * (size_t)(nA ? nA : 1));
        double *s = (double *)calloc((size_t)(nA ? nA : 1), sizeof(double));
        double *Hs = (double *)calloc((size_t)(nA ? nA : 1), sizeof(double));
        double *Xs = (double *)calloc((size_t)m, sizeof(double));
        double *Xz = (double *)calloc((size_t)m, sizeof(double));
        double *Hz = (double *)calloc((size_t)(nA ? nA : 1), sizeof(double));
        double *hh = (double *)malloc(sizeof(double) * (size_t)(nA ? nA : 1));
        double *wA = (double *)malloc(sizeof(double) * (size_t)(nA ? nA : 1));
        for (int64_t p = 0; p < nA; ++p) { hh[p] = hA[p] + o->eps_h; wA[p] = c->w[A[p]]; }
        int32_t it;
        int cg_restart = 1, kinked = 0;
        double rz_prev = 0.0;
        for (it = 0; it < K; ++it) {                                 /* R4 */
            /* R5: model gradient p = g + H d at x = w_A + d; model min-norm subgradient (P:248-256 on Eq. 3) */
            double vq = 0.0;
            for (int64_t p = 0; p < nA; ++p) {
                double pj = gA[p] + Hd[p], x = wA[p] + d[p];
                double v = (x != 0.0) ? pj + lam * (x > 0.0 ? 1.0 : -1.0) : mlo_soft_shrink(pj, lam);
                if (fabs(v) > vq) vq = fabs(v);
            }
            if (it > 0 && o->eta > 0.0 && vq <= o->eta * vmax) break; /* R13: inexact-Newton forcing */
            /* inner_cg = 1: PCD at it = 0, PCD-CG after; inner_cg = 2: also a PCD step after every kink-truncated CG
               step (the shrinkage step can zero many coordinates at once, a truncated CG step only one) */
            int pcd = (!o->inner_cg) || it == 0 || (o->inner_cg == 2 && kinked);
            if (pcd) {
                /* R6: PCD direction, Eq. 5 with D = diag(H) + eps_h */
                double umax = 0.0;
                for (int64_t p = 0; p < nA; ++p) {
                    double pj = gA[p] + Hd[p], x = wA[p] + d[p];
                    s[p] = mlo_soft_shrink(x - pj / hh[p], lam / hh[p]) - x;
                    if (fabs(s[p]) > umax) umax = fabs(s[p]);
                }
                if (umax == 0.0) break;                              /* R7 */
                /* R8: Xs = X_A s, Hs = X_A^T D Xs + eps s */
                apply_XC(c, A, nA, s, Xs);
                apply_XCt_D(c, A, nA, Xs, Hs);
                for (int64_t p = 0; p < nA; ++p) Hs[p] += o->eps_h * s[p];
                double ps = 0.0, sHs = 0.0, l1x = 0.0, l1xs = 0.0;
                for (int64_t p = 0; p < nA; ++p) {
                    double x = wA[p] + d[p];
                    ps += (gA[p] + Hd[p]) * s[p];
                    sHs += s[p] * Hs[p];
                    l1x += fabs(x);
                    l1xs += fabs(x + s[p]);
                }
                double delta = ps + lam * (l1xs - l1x);              /* R9 */
                /* pcd_snap (DESIGN Q27): z = the part of s that takes a coordinate exactly to 0 (x != 0, x + s = 0);
                   line search along sigma(b) = b (s - z) + z, i.e. those coordinates are set to 0 for every b.
                   q(sigma(b)) in closed form from Xz = X_A z and Hz = X_A^T D Xz + eps z. */
                int nzero = 0;
                double pz = 0.0, zHs = 0.0, zHz = 0.0, Z1 = 0.0;
                if (o->pcd_snap) {
                    for (int64_t p = 0; p < nA; ++p) {
                        double x = wA[p] + d[p];
                        u[p] = (x != 0.0 && x + s[p] == 0.0) ? s[p] : 0.0;   /* u holds z here */
                        nzero += (u[p] != 0.0);
                    }
                    if (nzero) {
                        apply_XC(c, A, nA, u, Xz);
                        apply_XCt_D(c, A, nA, Xz, Hz);
                        for (int64_t p = 0; p < nA; ++p) Hz[p] += o->eps_h * u[p];
                        for (int64_t p = 0; p < nA; ++p) {
                            pz += (gA[p] + Hd[p]) * u[p];
                            zHs += u[p] * Hs[p];
                            zHz += u[p] * Hz[p];
                            Z1 += fabs(u[p]);
                        }
                    }
                }
                double beta = 1.0;                                   /* R10: Armijo on the model, b = 1, 1/2, ... */
                int ok = 0, snapped = 0;
                for (int pathk = (nzero ? 0 : 1); pathk < 2 && !ok; ++pathk) {   /* 0: snap path, 1: plain path */
                    beta = 1.0;
                    for (int32_t t = 0; t < o->max_ls; ++t, beta *= o->beta) {
                        double l1b = 0.0;
                        for (int64_t p = 0; p < nA; ++p) l1b += fabs(wA[p] + d[p] + beta * s[p]);
                        double dq;
                        if (pathk == 0) {
                            /* sigma = b sn + z, sn = s - z: p^T sigma = b (ps - pz) + pz;
                               sigma^T H sigma = b^2 (sHs - 2 zHs + zHz) + 2 b (zHs - zHz) + zHz;
                               ||x + sigma||_1 - ||x||_1 = (l1b - l1x) - (1 - b) Z1 */
                            double snHsn = sHs - 2.0 * zHs + zHz, snHz = zHs - zHz;
                            dq = beta * (ps - pz) + pz + 0.5 * (beta * beta * snHsn + 2.0 * beta * snHz + zHz)
                                 + lam * ((l1b - l1x) - (1.0 - beta) * Z1);
                        } else {
                            dq = beta * ps + 0.5 * beta * beta * sHs + lam * (l1b - l1x);
                        }
                        if (dq <= o->sigma_in * beta * delta) { ok = 1; snapped = (pathk == 0); break; }
                    }
                }
                if (!ok) break;                                      /* R11 */
                if (snapped) {                                       /* R12 on the snap path */
                    for (int64_t p = 0; p < nA; ++p) {
                        double zp = u[p];
                        d[p] = (zp != 0.0) ? -wA[p] : d[p] + beta * s[p];
                        Hd[p] += beta * (Hs[p] - Hz[p]) + Hz[p];
                    }
                    for (int64_t i = 0; i < m; ++i) Xd[i] += beta * (Xs[i] - Xz[i]) + Xz[i];
                } else {
                    for (int64_t p = 0; p < nA; ++p) { d[p] += beta * s[p]; Hd[p] += beta * Hs[p]; } /* R12 */
                    for (int64_t i = 0; i < m; ++i) Xd[i] += beta * Xs[i];
                }
                cg_restart = 1;
                kinked = 0;
            } else {
                /* R6': PCD-CG (DESIGN Q9b): preconditioned CG on the model restricted to the current orthant,
                   F = {j : x_j != 0}, signs xi = sign(x) fixed, zeros frozen.  Preconditioner diag(H) + eps_h
                   (the PCD scaling); acceleration of PCD by CG as in P:99 / P:505. */
                double rz = 0.0;
                for (int64_t p = 0; p < nA; ++p) {
                    double x = wA[p] + d[p];
                    u[p] = (x != 0.0) ? -(gA[p] + Hd[p] + lam * (x > 0.0 ? 1.0 : -1.0)) / hh[p] : 0.0;
                    rz += hh[p] * u[p] * u[p];
                }
                if (rz == 0.0) break;
                double bcg = cg_restart ? 0.0 : rz / rz_prev;        /* Fletcher-Reeves = linear PCG */
                for (int64_t p = 0; p < nA; ++p) s[p] = u[p] + bcg * s[p];
                apply_XC(c, A, nA, s, Xs);                           /* R8 */
                apply_XCt_D(c, A, nA, Xs, Hs);
                for (int64_t p = 0; p < nA; ++p) Hs[p] += o->eps_h * s[p];
                double slope = 0.0, sHs = 0.0, bk = INFINITY;
                for (int64_t p = 0; p < nA; ++p) {
                    double x = wA[p] + d[p];
                    if (x != 0.0) slope += (gA[p] + Hd[p] + lam * (x > 0.0 ? 1.0 : -1.0)) * s[p];
                    sHs += s[p] * Hs[p];
                    if (x * s[p] < 0.0) { double b = -x / s[p]; if (b < bk) bk = b; } /* first kink */
                }
                if (!(slope < 0.0) || !(sHs > 0.0)) break;
                double bq = -slope / sHs;                            /* exact minimiser of the quadratic piece */
                double beta = bq < bk ? bq : bk;
                for (int64_t p = 0; p < nA; ++p) {
                    double x = wA[p] + d[p];
                    int snap = (bk <= bq) && x * s[p] < 0.0 && -x / s[p] == bk;
                    d[p] = snap ? -wA[p] : d[p] + beta * s[p];       /* a coordinate reaching its kink becomes 0 */
                    Hd[p] += beta * Hs[p];
                }
                for (int64_t i = 0; i < m; ++i) Xd[i] += beta * Xs[i];
                cg_restart = (bk <= bq);
                kinked = (bk <= bq);
                rz_prev = rz;
            }
        }
        row.inner_iters = it;
        int nonzero = 0;
        for (int64_t p = 0; p < nA; ++p) if (d[p] != 0.0) { nonzero = 1; break; }
        if (nonzero) {                                               /* R14-R18 */
            double alpha, Fnew;
            st = outer_linesearch(c, A, nA, gA, d, Xd, o, &alpha, &Fnew);
            row.alpha = alpha;
            row.outcome = (st == MLO_OK) ? MLO_R_UPDATED : MLO_R_STAGNATION;
            row.F_after = F_current(c);
            /* Lemma P:207-243: the accepted step satisfies F(w+ad) - F(w) <= sigma a Delta < 0 (term-by-term
               difference); a recomputed F may differ from F_before by rounding only. */
            if (st == MLO_OK && row.F_after > F_before + 1e-12 * fabs(F_before)) st = MLO_E_CONTRACT;
        } else {
            row.outcome = MLO_R_NOSTEP;
        }
        free(d); free(Hd); free(Xd); free(u); free(s); free(Hs); free(Xs); free(Xz); free(Hz); free(hh); free(wA);
    }
done:
    row.F_after = F_current(c);
    trace_push(c, row);
    *outcome = row.outcome;
    free(A); free(gA); free(hA);
    if (own) { free(g); free(h); }
    return st;
}

int mlo_relax(mlo_ctx *c, const int32_t *C, int64_t nC, int32_t K, const mlo_opts *o, int32_t *outcome) {
    if (check_C(c, C, nC)) return MLO_E_INVAL;
    return relax_core(c, C, nC, NULL, NULL, K, o, -1, NULL, NULL, NULL, outcome);
}

int64_t mlo_trace_len(const mlo_ctx *c) { return c->ntrace; }
void mlo_trace_get(const mlo_ctx *c, int64_t i, mlo_trace_row *row) { *row = c->trace[i]; }
void mlo_trace_clear(mlo_ctx *c) { c->ntrace = 0; }

/* ------------------------------------------------------------ level sizes
 * |C_{l+1}| = max(ceil(|C_l| / 2), |supp|), stop (L = l) when |C_l| = |supp|;
 * |C_1| = max(ceil(|A_f| / 2), |supp|) from the finest free set (P:602 via P:798, DESIGN Q10);
 * L = 0 when |C_1| = n (DESIGN Q11).  k[1..L] are written; returns L.
 */
int mlo_level_sizes(int64_t nAf, int64_t nS, int64_t n, int64_t *k) {
    k[0] = n;
    k[1] = (nAf + 1) / 2;
    if (k[1] < nS) k[1] = nS;
    if (k[1] >= n) return 0;
    int L = 1;
    while (k[L] != nS && L < 62) {
        k[L + 1] = (k[L] + 1) / 2;
        if (k[L + 1] < nS) k[L + 1] = nS;
        ++L;
    }
    return L;
}

/* ------------------------------------------------------------ the solve
 * Algorithm 1 repeated until the finest-level KKT test passes,
 * hierarchy per P:175-196 with |C_1| from the free set (P:602 via P:798; DESIGN Q10).
 * Lines S1-S18 refer to DESIGN.md "Algorithm".
 */
static void kkt_all(const mlo_ctx *c, const double *g, double *vinf, double *v1) {
    double mx = 0.0, s = 0.0;
    for (int64_t j = 0; j < c->n; ++j) {
        double wj = c->w[j], v;
        if (wj != 0.0) v = g[j] + c->lam * (wj > 0.0 ? 1.0 : -1.0);
        else v = mlo_soft_shrink(g[j], c->lam);
        if (fabs(v) > mx) mx = fabs(v);
        s += fabs(v);
    }
    *vinf = mx; *v1 = s;
}
static int64_t nnz_w(const mlo_ctx *c) {
    int64_t k = 0;
    for (int64_t j = 0; j < c->n; ++j) k += (c->w[j] != 0.0);
    return k;
}

int mlo_solve(mlo_ctx *c, const mlo_opts *o, mlo_report *rep) {
    int64_t n = c->n;
    memset(rep, 0, sizeof(*rep));
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    double *h = (double *)malloc(sizeof(double) * (size_t)n);
    int32_t *Af = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    double *gAf = (double *)malloc(sizeof(double) * (size_t)n);
    int32_t *R = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int64_t nAf = 0;
    int64_t npos = 0;
    for (int64_t i = 0; i < c->m && c->y; ++i) npos += (c->y[i] > 0);   /* (squared loss: no labels) */
    int64_t minpm = npos < c->m - npos ? npos : c->m - npos;
    int st = MLO_OK;
    int32_t outcome;
    const int64_t nnz_touched0 = c->nnz_touched, x_passes0 = c->x_passes;   /* the report counts this solve only */

    /* S1-S2: w = 0, z = 0, EVAL_ALL */
    memset(c->w, 0, sizeof(double) * (size_t)n);
    double F;
    mlo_eval_f_grad(c, NULL, n, &F, g, h);
    double vinf, v1, v1_0;
    kkt_all(c, g, &vinf, &v1);
    v1_0 = v1;
    int converged = (vinf / c->lam <= o->tol_kkt);                  /* S3 (lambda >= lambda_max) */
    int cycle = 0;
    if (!converged && o->continuation) {
        /* Continuation (DESIGN Q28): lambda_4 = (lambda_max + lambda) / 2 and lambda_3, lambda_2 linearly
           spaced between lambda_4 and lambda_1 = lambda; one finest relaxation (one proximal-Newton outer iteration on
           the free set) at each of lambda_4, lambda_3, lambda_2 in decreasing order, then the solve at lambda from that
           warm start.  At w = 0, vinf = max_j (|g_j| - lambda), so lambda_max = vinf + lambda. */
        const double lam1 = c->lam, lam4 = 0.5 * ((vinf + lam1) + lam1);
        for (int kk = 4; kk >= 2 && st == MLO_OK; --kk) {
            c->lam = lam1 + (lam4 - lam1) * (double)(kk - 1) / 3.0;
            st = relax_core(c, NULL, n, NULL, NULL, o->K_fine, o, 0, Af, &nAf, gAf, &outcome);
            rep->relax_per_level[0]++;
        }
        c->lam = lam1;
        /* S2 again at the warm start: EVAL_ALL with margins from scratch */
        mlo_eval_f_grad(c, NULL, n, &F, g, h);
        kkt_all(c, g, &vinf, &v1);
        converged = (vinf / c->lam <= o->tol_kkt);
    }
    if (!converged) {
        /* S4: initial finest relaxation so that a finest gradient exists */
        st = relax_core(c, NULL, n, g, h, o->K_fine, o, 0, Af, &nAf, gAf, &outcome);
        rep->relax_per_level[0]++;
        for (cycle = 1; cycle <= o->max_cycles && st == MLO_OK; ++cycle) {     /* S5 */
            if (o->multilevel) {
                /* S7: S = supp(w) (current) */
                int64_t nS = 0;
                for (int64_t j = 0; j < n; ++j) nS += (c->w[j] != 0.0);
                if (nS > 0) {                                                  /* S8 */
                    int64_t k[64];                                             /* S9-S10 */
                    int L = mlo_level_sizes(nAf, nS, n, k);
                    /* S11: R = A_f \ S ranked by (|g_f| desc, index asc) */
                    int64_t nR = 0;
                    for (int64_t p = 0; p < nAf; ++p) if (c->w[Af[p]] == 0.0) R[nR++] = (int32_t)p; /* positions in Af */
                    {
                        /* rank positions by |gAf| desc then index asc (Af ascending => position order = index order) */
                        g_sort_key = gAf;
                        qsort(R, (size_t)nR, sizeof(int32_t), cmp_rank);
                        for (int64_t t = 0; t < nR; ++t) R[t] = Af[R[t]];
                    }
                    /* S12: C_l = sort_asc(S U R[0 : k_l - |S|]), l = 1..L, with S frozen at S7 (Eq. 10) */
                    {
                        int32_t *S7 = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nS ? nS : 1));
                        int64_t t = 0;
                        for (int64_t j = 0; j < n; ++j) if (c->w[j] != 0.0) S7[t++] = (int32_t)j;
                        int32_t **lev = (int32_t **)calloc((size_t)(L + 1), sizeof(int32_t *));
                        int64_t *nlev = (int64_t *)calloc((size_t)(L + 1), sizeof(int64_t));
                        for (int l = 1; l <= L; ++l) {
                            int64_t take = k[l] - nS;
                            lev[l] = (int32_t *)malloc(sizeof(int32_t) * (size_t)k[l]);
                            memcpy(lev[l], S7, sizeof(int32_t) * (size_t)nS);
                            memcpy(lev[l] + nS, R, sizeof(int32_t) * (size_t)take);
                            qsort(lev[l], (size_t)k[l], sizeof(int32_t), cmp_i32);
                            nlev[l] = k[l];
                        }
                        /* S13: coarsest level until converged or nu_c times (Alg. 1 step 3) */
                        if (L >= 1) {
                            for (int32_t it = 0; it < o->nu_c && st == MLO_OK; ++it) {
                                st = relax_core(c, lev[L], nlev[L], NULL, NULL, o->K_coarse, o, L, NULL, NULL, NULL, &outcome);
                                rep->relax_per_level[L < 31 ? L : 31]++;
                                if (outcome == MLO_R_CONVERGED) break;
                            }
                        }
                        /* S14: levels L-1 .. 1, nu relaxations each (Alg. 1 step 4) */
                        for (int l = L - 1; l >= 1 && st == MLO_OK; --l)
                            for (int32_t it = 0; it < o->nu && st == MLO_OK; ++it) {
                                st = relax_core(c, lev[l], nlev[l], NULL, NULL, o->K_mid, o, l, NULL, NULL, NULL, &outcome);
                                rep->relax_per_level[l < 31 ? l : 31]++;
                            }
                        for (int l = 1; l <= L; ++l) free(lev[l]);
                        free(lev); free(nlev); free(S7);
                    }
                }
            }
            if (st != MLO_OK) break;
            /* S15-S16: EVAL_ALL with margins from scratch; finest-level convergence test */
            mlo_eval_f_grad(c, NULL, n, &F, g, h);
            kkt_all(c, g, &vinf, &v1);
            int64_t ns = nnz_w(c);
            if (ns > rep->max_supp) rep->max_supp = ns;
            if (vinf / c->lam <= o->tol_kkt) { converged = 1; break; }
            /* S17: finest relaxation with E, then nu-1 more */
            st = relax_core(c, NULL, n, g, h, o->K_fine, o, 0, Af, &nAf, gAf, &outcome);
            rep->relax_per_level[0]++;
            for (int32_t it = 1; it < o->nu && st == MLO_OK; ++it) {
                st = relax_core(c, NULL, n, NULL, NULL, o->K_fine, o, 0, Af, &nAf, gAf, &outcome);
                rep->relax_per_level[0]++;
            }
        }
    }
    /* report at the evaluated w (DESIGN Q17) */
    mlo_eval_f_grad(c, NULL, n, &F, g, NULL);
    kkt_all(c, g, &vinf, &v1);
    rep->F = F;
    rep->vinf = vinf;
    rep->kappa = vinf / c->lam;
    rep->v1 = v1;
    rep->paper_ratio = (v1_0 > 0.0 && minpm > 0) ? v1 / (v1_0 * (double)minpm / (double)c->m) : 0.0;
    rep->cycles = cycle > o->max_cycles ? o->max_cycles : cycle;
    for (int l = 0; l < 32; ++l) rep->relaxations += rep->relax_per_level[l];
    rep->nnz_w = nnz_w(c);
    if (rep->nnz_w > rep->max_supp) rep->max_supp = rep->nnz_w;
    rep->nnz_touched = c->nnz_touched - nnz_touched0;
    rep->x_passes = c->x_passes - x_passes0;
    if (st == MLO_OK && !converged) st = MLO_E_NOT_CONVERGED;
    rep->status = st;
    free(g); free(h); free(Af); free(gAf); free(R);
    return st;
}
