/* mlgen.c — seeded synthetic input generator (SHARED INPUT INFRASTRUCTURE).
 *
 * This module builds the synthetic data sets that stand in for the paper's
 * benchmark data (Table 4; BASELINE.json configs
 * 1-5; recipe in DESIGN.md "Input recipe").  It is the ONLY code shared by
 * the CPU oracle (oracle/) and the CUDA path (paper_1607_00315_b200/): it
 * draws X, y and the planted w*, and it contains none of the method's
 * arithmetic.  The one derived scalar it writes is the configuration's
 * lambda = factor * lambda_max with lambda_max = 1/2 ||X^T y||_inf, because
 * BASELINE.json defines lambda that way; both solvers then read the same
 * bits.  (lambda_max is pinned independently in tests/test_oracle_pins.py:
 * the oracle's own gradient at w = 0 must reproduce it.)
 *
 * RNG: Philox4x32-10, key = (seed, stream), counter = (a, b, c, 0).  Every
 * draw is addressed by (stream, row, draw) so the output does not depend on
 * the OpenMP thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "mlgen.h"

/* ---------------------------------------------------------------- Philox */
typedef struct { uint32_t v[4]; } u32x4;

static inline uint32_t mulhilo(uint32_t a, uint32_t b, uint32_t *hi) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    return (uint32_t)p;
}

static u32x4 philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        uint32_t lo0 = mulhilo(0xD2511F53u, c0, &hi0);
        uint32_t lo1 = mulhilo(0xCD9E8D57u, c2, &hi1);
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    u32x4 o = {{c0, c1, c2, c3}};
    return o;
}

enum { S_ROWLEN = 1, S_COLS, S_VALS, S_XNOISE, S_FACTOR, S_WSTAR_IDX, S_WSTAR_VAL,
       S_LABEL_NOISE, S_LABEL_U, S_FLIP, S_PERM };

typedef struct { uint32_t k0, k1; } rng_key;
static inline rng_key key_of(uint64_t seed, uint32_t stream) {
    rng_key k = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ (stream * 0x85EBCA6Bu)};
    return k;
}
/* uniform in [0,1) with 53 random bits */
static inline double u53(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}
static inline void uniform2(rng_key k, uint64_t a, uint64_t b, double *u0, double *u1) {
    u32x4 r = philox(k.k0, k.k1, (uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
    *u0 = u53(r.v[0], r.v[1]);
    *u1 = u53(r.v[2], r.v[3]);
}
static inline double normal(rng_key k, uint64_t a, uint64_t b) { /* Box-Muller, fp64 */
    double u0, u1;
    uniform2(k, a, b, &u0, &u1);
    return sqrt(-2.0 * log(1.0 - u0)) * cos(6.283185307179586476925286766559 * u1);
}

/* --------------------------------------------------------------- helpers */
static int poisson_inv(double mean, double u) { /* CDF inversion */
    double p = exp(-mean), c = p;
    int k = 0;
    while (u > c && k < 100000) { ++k; p *= mean / k; c += p; if (p == 0.0 && c < u) break; }
    return k;
}

typedef struct { double *prob; int32_t *alias; int64_t n; } alias_tab;

static int alias_build(alias_tab *t, int64_t n, double s) { /* Vose; weights k^-s, k = 1..n */
    t->n = n;
    t->prob = (double *)malloc(sizeof(double) * n);
    t->alias = (int32_t *)malloc(sizeof(int32_t) * n);
    int32_t *small = (int32_t *)malloc(sizeof(int32_t) * n), *large = (int32_t *)malloc(sizeof(int32_t) * n);
    if (!t->prob || !t->alias || !small || !large) return -1;
    double sum = 0.0;
    for (int64_t k = 0; k < n; ++k) sum += pow((double)(k + 1), -s);
    int64_t ns = 0, nl = 0;
    for (int64_t k = 0; k < n; ++k) {
        t->prob[k] = pow((double)(k + 1), -s) * (double)n / sum;
        if (t->prob[k] < 1.0) small[ns++] = (int32_t)k; else large[nl++] = (int32_t)k;
    }
    while (ns > 0 && nl > 0) {
        int32_t l = small[--ns], g = large[--nl];
        t->alias[l] = g;
        t->prob[g] = (t->prob[g] + t->prob[l]) - 1.0;
        if (t->prob[g] < 1.0) small[ns++] = g; else large[nl++] = g;
    }
    while (nl > 0) { int32_t g = large[--nl]; t->prob[g] = 1.0; t->alias[g] = g; }
    while (ns > 0) { int32_t l = small[--ns]; t->prob[l] = 1.0; t->alias[l] = l; }
    free(small); free(large);
    return 0;
}
static inline int64_t alias_draw(const alias_tab *t, double u0, double u1) {
    int64_t k = (int64_t)(u0 * (double)t->n);
    if (k >= t->n) k = t->n - 1;
    return (u1 < t->prob[k]) ? k : t->alias[k];
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

void mlgen_free(mlgen_data *d) {
    if (!d) return;
    free(d->csr_rowptr); free(d->csr_col); free(d->csr_val);
    free(d->csc_colptr); free(d->csc_row); free(d->csc_val);
    free(d->y); free(d->wstar_idx); free(d->wstar_val);
    free(d);
}

/* ------------------------------------------------------------ generator */
mlgen_data *mlgen_generate(const mlgen_params *P) {
    int64_t m = P->m, n = P->n;
    if (m < 1 || n < 1 || n > 2147483647LL || m > 2147483647LL) return NULL;
    mlgen_data *d = (mlgen_data *)calloc(1, sizeof(mlgen_data));
    if (!d) return NULL;
    d->m = m; d->n = n;
    d->csr_rowptr = (int32_t *)malloc(sizeof(int32_t) * (m + 1));
    int dense = (P->kind == MLGEN_DENSE_IID || P->kind == MLGEN_DENSE_BLOCK);
    rng_key kr = key_of(P->seed, S_ROWLEN), kc = key_of(P->seed, S_COLS), kv = key_of(P->seed, S_VALS);

    /* 1. row lengths */
    int64_t *len = (int64_t *)malloc(sizeof(int64_t) * m);
    if (dense) {
        for (int64_t i = 0; i < m; ++i) len[i] = n;
    } else {
        for (int64_t i = 0; i < m; ++i) {
            double u0, u1;
            uniform2(kr, (uint64_t)i, 0, &u0, &u1);
            int k = poisson_inv(P->mean_row_nnz, u0);
            if (k < 1) k = 1;
            if (k > n) k = (int)n;
            len[i] = k;
        }
    }
    int64_t nnz = 0;
    for (int64_t i = 0; i < m; ++i) { d->csr_rowptr[i] = (int32_t)nnz; nnz += len[i]; }
    if (nnz > 2147483647LL) { free(len); mlgen_free(d); return NULL; }
    d->csr_rowptr[m] = (int32_t)nnz;
    d->nnz = nnz;
    d->csr_col = (int32_t *)malloc(sizeof(int32_t) * (nnz ? nnz : 1));
    d->csr_val = (float *)malloc(sizeof(float) * (nnz ? nnz : 1));

    /* 2. rows */
    if (dense) {
        rng_key kx = key_of(P->seed, S_XNOISE), kf = key_of(P->seed, S_FACTOR);
        const double h = sqrt(0.5);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            int64_t b0 = d->csr_rowptr[i];
            for (int64_t j = 0; j < n; ++j) {
                double x;
                if (P->kind == MLGEN_DENSE_IID) x = normal(kx, (uint64_t)i, (uint64_t)j);
                else x = h * normal(kf, (uint64_t)i, (uint64_t)(j / P->block)) + h * normal(kx, (uint64_t)i, (uint64_t)j);
                d->csr_col[b0 + j] = (int32_t)j;
                d->csr_val[b0 + j] = (float)x;
            }
        }
    } else {
        alias_tab at;
        if (alias_build(&at, n, P->zipf_s) != 0) { free(len); mlgen_free(d); return NULL; }
        /* rank -> column permutation (Fisher-Yates, seeded) */
        int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * n);
        rng_key kp = key_of(P->seed, S_PERM);
        for (int64_t k = 0; k < n; ++k) perm[k] = (int32_t)k;
        for (int64_t k = n - 1; k > 0; --k) {
            double u0, u1;
            uniform2(kp, (uint64_t)k, 0, &u0, &u1);
            int64_t r = (int64_t)(u0 * (double)(k + 1));
            if (r > k) r = k;
            int32_t t = perm[k]; perm[k] = perm[r]; perm[r] = t;
        }
#pragma omp parallel
        {
            int hsz = 1024;
            int32_t *hkey = (int32_t *)malloc(sizeof(int32_t) * hsz);
            uint32_t *hgen = (uint32_t *)calloc(hsz, sizeof(uint32_t));
            uint32_t gen = 0;
#pragma omp for schedule(dynamic, 256)
            for (int64_t i = 0; i < m; ++i) {
                int64_t k = len[i], b0 = d->csr_rowptr[i];
                if (4 * k > hsz) {
                    while (4 * k > hsz) hsz *= 2;
                    hkey = (int32_t *)realloc(hkey, sizeof(int32_t) * hsz);
                    free(hgen); hgen = (uint32_t *)calloc(hsz, sizeof(uint32_t)); gen = 0;
                }
                ++gen;
                if (gen == 0) { memset(hgen, 0, sizeof(uint32_t) * hsz); gen = 1; }
                int64_t got = 0;
                uint64_t draw = 0;
                while (got < k) { /* distinct ids: duplicates are redrawn */
                    double u0, u1;
                    uniform2(kc, (uint64_t)i, draw++, &u0, &u1);
                    int32_t col = perm[alias_draw(&at, u0, u1)];
                    uint32_t hsh = ((uint32_t)col * 2654435761u) & (uint32_t)(hsz - 1);
                    int dup = 0;
                    while (hgen[hsh] == gen) {
                        if (hkey[hsh] == col) { dup = 1; break; }
                        hsh = (hsh + 1) & (uint32_t)(hsz - 1);
                    }
                    if (dup) continue;
                    hgen[hsh] = gen; hkey[hsh] = col;
                    d->csr_col[b0 + got++] = col;
                }
                qsort(d->csr_col + b0, (size_t)k, sizeof(int32_t), cmp_i32);
                /* values U(0,1] then row L2-normalised in fp64, stored fp32 */
                double ss = 0.0;
                double *tmp = (double *)malloc(sizeof(double) * k);
                for (int64_t t = 0; t < k; ++t) {
                    double u0, u1;
                    uniform2(kv, (uint64_t)i, (uint64_t)t, &u0, &u1);
                    tmp[t] = 1.0 - u0;
                    ss += tmp[t] * tmp[t];
                }
                double inv = 1.0 / sqrt(ss);
                for (int64_t t = 0; t < k; ++t) d->csr_val[b0 + t] = (float)(tmp[t] * inv);
                free(tmp);
            }
            free(hkey); free(hgen);
        }
        free(perm); free(at.prob); free(at.alias);
    }
    free(len);

    /* 3. planted w* : nnz_w distinct uniform columns (partial Fisher-Yates), N(0, w_var) */
    int64_t nw = P->nnz_w < n ? P->nnz_w : n;
    d->nnz_w = nw;
    d->wstar_idx = (int32_t *)malloc(sizeof(int32_t) * (nw ? nw : 1));
    d->wstar_val = (double *)malloc(sizeof(double) * (nw ? nw : 1));
    {
        rng_key ki = key_of(P->seed, S_WSTAR_IDX), kw = key_of(P->seed, S_WSTAR_VAL);
        /* sparse partial Fisher-Yates via a sorted-free swap map is overkill: use rejection */
        int64_t got = 0; uint64_t draw = 0;
        while (got < nw) {
            double u0, u1;
            uniform2(ki, draw++, 0, &u0, &u1);
            int32_t c = (int32_t)(u0 * (double)n);
            if (c >= n) c = (int32_t)(n - 1);
            int dup = 0;
            for (int64_t t = 0; t < got; ++t) if (d->wstar_idx[t] == c) { dup = 1; break; }
            if (dup) continue;
            d->wstar_idx[got++] = c;
        }
        qsort(d->wstar_idx, (size_t)nw, sizeof(int32_t), cmp_i32);
        double sd = sqrt(P->w_var);
        for (int64_t t = 0; t < nw; ++t) d->wstar_val[t] = sd * normal(kw, (uint64_t)t, 0);
    }

    /* 4. labels from the planted model */
    d->y = (int8_t *)malloc((size_t)m);
    {
        double *wd = (double *)calloc((size_t)n, sizeof(double));
        for (int64_t t = 0; t < nw; ++t) wd[d->wstar_idx[t]] = d->wstar_val[t];
        rng_key kn = key_of(P->seed, S_LABEL_NOISE), ku = key_of(P->seed, S_LABEL_U), kf = key_of(P->seed, S_FLIP);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            double s = 0.0;
            for (int64_t p = d->csr_rowptr[i]; p < d->csr_rowptr[i + 1]; ++p) s += (double)d->csr_val[p] * wd[d->csr_col[p]];
            int8_t yi;
            if (P->label == MLGEN_LABEL_SIGN_NOISE) {
                double v = s + P->label_noise * normal(kn, (uint64_t)i, 0);
                yi = (v >= 0.0) ? 1 : -1; /* sign(0) := +1 */
            } else {
                double u0, u1;
                uniform2(ku, (uint64_t)i, 0, &u0, &u1);
                double pr = 1.0 / (1.0 + exp(-s)); /* P(y = +1) = logistic(x^T w*) (data model) */
                yi = (u0 < pr) ? 1 : -1;
            }
            if (P->flip_prob > 0.0) {
                double u0, u1;
                uniform2(kf, (uint64_t)i, 0, &u0, &u1);
                if (u0 < P->flip_prob) yi = (int8_t)-yi;
            }
            d->y[i] = yi;
        }
        free(wd);
    }

    /* 5. CSC by counting transpose (row ids ascending inside each column) */
    d->csc_colptr = (int32_t *)calloc((size_t)(n + 1), sizeof(int32_t));
    d->csc_row = (int32_t *)malloc(sizeof(int32_t) * (nnz ? nnz : 1));
    d->csc_val = (float *)malloc(sizeof(float) * (nnz ? nnz : 1));
    {
        int64_t *cnt = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
        for (int64_t p = 0; p < nnz; ++p) cnt[d->csr_col[p] + 1]++;
        for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
        for (int64_t j = 0; j <= n; ++j) d->csc_colptr[j] = (int32_t)cnt[j];
        for (int64_t i = 0; i < m; ++i)
            for (int64_t p = d->csr_rowptr[i]; p < d->csr_rowptr[i + 1]; ++p) {
                int64_t q = cnt[d->csr_col[p]]++;
                d->csc_row[q] = (int32_t)i;
                d->csc_val[q] = d->csr_val[p];
            }
        free(cnt);
    }

    /* 6. the configuration's lambda (BASELINE.json: lambda = factor * ||X^T y||_inf / 2) */
    {
        double mx = 0.0;
#pragma omp parallel for schedule(static) reduction(max : mx)
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t q = d->csc_colptr[j]; q < d->csc_colptr[j + 1]; ++q) s += (double)d->csc_val[q] * (double)d->y[d->csc_row[q]];
            double a = fabs(s);
            if (a > mx) mx = a;
        }
        d->lambda_max = 0.5 * mx;
        d->lambda = P->lambda_factor * d->lambda_max;
    }
    return d;
}

void mlgen_preset(int cfg, mlgen_params *P) {
    memset(P, 0, sizeof(*P));
    P->block = 20;
    switch (cfg) {
    case 1: P->kind = MLGEN_DENSE_IID; P->m = 200; P->n = 1000; P->nnz_w = 20; P->w_var = 1.0;
            P->label = MLGEN_LABEL_SIGN_NOISE; P->label_noise = 0.1; P->lambda_factor = 0.1; P->seed = 1001; break;
    case 2: P->kind = MLGEN_DENSE_BLOCK; P->m = 2000; P->n = 20000; P->nnz_w = 100; P->w_var = 2.0;
            P->label = MLGEN_LABEL_LOGISTIC; P->lambda_factor = 0.05; P->seed = 1002; break;
    case 3: P->kind = MLGEN_ZIPF; P->m = 50000; P->n = 100000; P->mean_row_nnz = 50; P->zipf_s = 1.1;
            P->nnz_w = 500; P->w_var = 5.0; P->label = MLGEN_LABEL_LOGISTIC; P->lambda_factor = 0.02; P->seed = 1003; break;
    case 4: P->kind = MLGEN_ZIPF; P->m = 500000; P->n = 1000000; P->mean_row_nnz = 50; P->zipf_s = 1.05;
            P->nnz_w = 2000; P->w_var = 5.0; P->label = MLGEN_LABEL_LOGISTIC; P->flip_prob = 0.05;
            P->lambda_factor = 0.01; P->seed = 1004; break;
    case 5: P->kind = MLGEN_ZIPF; P->m = 2000000; P->n = 20000000; P->mean_row_nnz = 100; P->zipf_s = 1.1;
            P->nnz_w = 10000; P->w_var = 5.0; P->label = MLGEN_LABEL_LOGISTIC; P->lambda_factor = 0.005; P->seed = 1005; break;
    default: break;
    }
}
