/*
 * bs_oracle.h -- interface of the CPU oracle (TEST INFRASTRUCTURE ONLY; see bs_oracle.c).
 * Deliberately independent of include/bs.h: its own struct, its own enum values.
 */
#ifndef BS_ORACLE_H
#define BS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_BATCHNORM = 11, OR_RELU = 12, OR_MAXPOOL = 13, OR_AVGPOOL = 14,
       OR_COPY = 15, OR_SCALE = 16, OR_ADD = 17 };
enum { OR_OK = 0, OR_ERR_INVALID = 1, OR_ERR_UNSUPPORTED = 2, OR_ERR_NOMEM = 3 };

typedef struct {
    int32_t kind;
    int32_t kh, kw, sh, sw, ph, pw;
    int32_t count_include_pad;
    float eps;
    const float *gamma, *beta, *mean, *var;   /* BN, length C */
    float alpha;                              /* SCALE */
    int32_t operand;                          /* ADD: 1-based index into operands[] */
} or_layer;

/* shapes: (n_layers+1) x 4 int64 -- the input shape of each layer, then the output. */
int oracle_layer_shapes(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                        int n_operands, int64_t *shapes);
int oracle_run_bf(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                  const float *x, const float *const *operands, int n_operands, float *y);
int oracle_run_df(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                  const float *x, const float *const *operands, int n_operands,
                  int64_t tile_h, int64_t tile_w, float *y);

#ifdef __cplusplus
}
#endif
#endif
