/* mlgen.h — seeded synthetic input generator (shared input infrastructure; see mlgen.c). */
#ifndef MLGEN_H
#define MLGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { MLGEN_DENSE_IID = 0, MLGEN_DENSE_BLOCK = 1, MLGEN_ZIPF = 2 };
enum { MLGEN_LABEL_SIGN_NOISE = 0, MLGEN_LABEL_LOGISTIC = 1 };

typedef struct {
    int32_t kind;          /* MLGEN_* */
    int32_t label;         /* MLGEN_LABEL_* */
    int64_t m, n;          /* rows = samples, cols = features */
    double mean_row_nnz;   /* ZIPF: k_i = max(1, Poisson(mean)) distinct ids */
    double zipf_s;         /* ZIPF exponent over ranks 1..n */
    int64_t block;         /* DENSE_BLOCK: columns per correlated block */
    int64_t nnz_w;         /* planted w* nonzeros */
    double w_var;          /* planted w* values ~ N(0, w_var) (variance) */
    double label_noise;    /* SIGN_NOISE: y = sign(x^T w* + noise * N(0,1)) */
    double flip_prob;      /* independent label flips */
    double lambda_factor;  /* lambda = factor * lambda_max */
    uint64_t seed;
} mlgen_params;

typedef struct {
    int64_t m, n, nnz, nnz_w;
    int32_t *csr_rowptr, *csr_col; float *csr_val;   /* [m+1], [nnz], [nnz] */
    int32_t *csc_colptr, *csc_row; float *csc_val;   /* [n+1], [nnz], [nnz] */
    int8_t *y;                                       /* [m] in {-1,+1} */
    int32_t *wstar_idx; double *wstar_val;           /* planted model (ground truth of the data model) */
    double lambda_max, lambda;
} mlgen_data;

void mlgen_preset(int cfg, mlgen_params *p);
mlgen_data *mlgen_generate(const mlgen_params *p);
void mlgen_free(mlgen_data *d);

#ifdef __cplusplus
}
#endif
#endif
