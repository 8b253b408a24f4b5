/*
 * bs_oracle.c -- plain, slow, obviously-correct CPU oracle for BrainSlug stacks.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the product (paper_1804_08378_b200/, include/); neither side
 * includes or links the other.
 *
 * What it computes: the BREADTH-FIRST result of a stack of layers, one
 * whole-tensor layer at a time, every intermediate materialised -- the paper's
 * layer-by-layer execution (fig:trio-bf, code P:L190-200).  The
 * method (depth-first) must reach exactly this result: "does not change the actual
 * results of the computation", "the same numerical results".
 *
 * Precision (reading R1): tensors are fp32 (BASELINE.json north_star);
 * every layer is evaluated in fp64 and rounded ONCE to fp32 when its output tensor is
 * stored -- the materialised intermediate of a breadth-first framework.  For single
 * IEEE operations (x*alpha, x+y) fp64-then-round equals the fp32 operation exactly
 * (53 >= 2*24+2), so SCALE/ADD/ReLU/MaxPool/COPY stacks have exactly one correct fp32
 * answer; BatchNorm and AvgPool are compared within the north_star tolerance.
 *
 * A depth-first CPU twin (oracle_run_df, PAPER.md fig:trio-df P:L208-239, S:L308
 * backward region geometry) applies the same per-element arithmetic tile by tile; it
 * must be bit-identical to oracle_run_bf (the paper's central claim made testable).
 *
 * Parity pins for every function: tests/test_oracle_pins.py (golden hand examples,
 * brute-force window enumeration, torch CPU cross-checks, closed forms, DF == BF).
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (no SIMD intrinsics, single thread).
 */
#include "bs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ per-element layers */

/* BatchNorm, inference form (paper P:L124-127 names only "normalize"):
 * y = gamma * (x - mean) / sqrt(var + eps) + beta, textbook order, fp64. */
static float bn_elem(const or_layer *L, int64_t c, float x)
{
    double d = sqrt((double)L->var[c] + (double)L->eps);
    double y = ((double)x - (double)L->mean[c]) / d * (double)L->gamma[c] + (double)L->beta[c];
    return (float)y;
}

/* ReLU f(x) = max(0, x); +0.0 for x <= 0 including -0.0. */
static float relu_elem(float x) { return x > 0.0f ? x : 0.0f; }

/* SCALE y = alpha * x (BASELINE.json north_star "elementwise add/scale"). */
static float scale_elem(const or_layer *L, float x) { return (float)((double)L->alpha * (double)x); }

/* ADD y = x + operand (north_star; residual add). */
static float add_elem(float x, float o) { return (float)((double)x + (double)o); }

/* Apply one element-wise layer to one value.  `opnd` is the ADD operand value. */
static float ew_apply(const or_layer *L, int64_t c, float x, float opnd)
{
    switch (L->kind) {
    case OR_BATCHNORM: return bn_elem(L, c, x);
    case OR_RELU:      return relu_elem(x);
    case OR_COPY:      return x;                 /* eval Dropout = identity */
    case OR_SCALE:     return scale_elem(L, x);
    case OR_ADD:       return add_elem(x, opnd);
    default:           return x;                 /* unreachable after validation */
    }
}

static int is_pool(int kind) { return kind == OR_MAXPOOL || kind == OR_AVGPOOL; }

/* One pooling output (fig-pool P:L148-157).
 * Window rows r = i*sh - ph + u, cols q = j*sw - pw + v, row-major u then v.
 * MaxPool: padded cells are ABSENT; strict '>' keeps the first maximum.
 * AvgPool: padded cells add nothing; divisor kh*kw when count_include_pad (G6), else
 *          the number of real cells.  `get(r,q)` reads the layer input. */
typedef float (*getter_fn)(const void *ctx, int64_t r, int64_t q);

static float pool_elem(const or_layer *L, int64_t H, int64_t W, int64_t i, int64_t j,
                       getter_fn get, const void *ctx)
{
    if (L->kind == OR_MAXPOOL) {
        float m = -INFINITY;
        for (int u = 0; u < L->kh; ++u)
            for (int v = 0; v < L->kw; ++v) {
                int64_t r = i * L->sh - L->ph + u, q = j * L->sw - L->pw + v;
                if (r >= 0 && r < H && q >= 0 && q < W) {
                    float t = get(ctx, r, q);
                    if (t > m) m = t;
                }
            }
        return m;
    } else {
        double acc = 0.0;
        int64_t real = 0;
        for (int u = 0; u < L->kh; ++u)
            for (int v = 0; v < L->kw; ++v) {
                int64_t r = i * L->sh - L->ph + u, q = j * L->sw - L->pw + v;
                if (r >= 0 && r < H && q >= 0 && q < W) {
                    acc += (double)get(ctx, r, q);
                    ++real;
                }
            }
        double div = L->count_include_pad ? (double)L->kh * (double)L->kw : (double)real;
        return (float)(acc / div);   /* "AvgPooling" + "AvgNormalization" (lst:finalcode P:L520-524) */
    }
}

/* ------------------------------------------------------------------ validation / shapes */

/* Shape law floor((H + 2p - k)/s) + 1. */
static int64_t pool_extent(int64_t n, int k, int s, int p) { return (n + 2 * (int64_t)p - k) / s + 1; }

int oracle_layer_shapes(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                        int n_operands, int64_t *shapes)
{
    if (!layers || n_layers < 1 || !in_shape || !shapes) return OR_ERR_INVALID;
    for (int d = 0; d < 4; ++d) if (in_shape[d] < 1) return OR_ERR_INVALID;
    int64_t N = in_shape[0], C = in_shape[1], H = in_shape[2], W = in_shape[3];
    memcpy(shapes, in_shape, 4 * sizeof(int64_t));
    for (int l = 0; l < n_layers; ++l) {
        const or_layer *L = &layers[l];
        switch (L->kind) {
        case OR_BATCHNORM:
            if (!(L->eps > 0.0f) || !L->gamma || !L->beta || !L->mean || !L->var) return OR_ERR_INVALID;
            for (int64_t c = 0; c < C; ++c) if (!(L->var[c] >= 0.0f)) return OR_ERR_INVALID;
            break;
        case OR_RELU: case OR_COPY: case OR_SCALE: break;
        case OR_ADD:
            if (L->operand < 1 || L->operand > n_operands) return OR_ERR_INVALID;
            break;
        case OR_MAXPOOL: case OR_AVGPOOL:
            if (L->kh < 1 || L->kw < 1 || L->sh < 1 || L->sw < 1) return OR_ERR_INVALID;
            if (L->ph < 0 || L->pw < 0 || 2 * L->ph > L->kh || 2 * L->pw > L->kw) return OR_ERR_INVALID;
            if (H + 2 * (int64_t)L->ph < L->kh || W + 2 * (int64_t)L->pw < L->kw) return OR_ERR_INVALID;
            H = pool_extent(H, L->kh, L->sh, L->ph);
            W = pool_extent(W, L->kw, L->sw, L->pw);
            if (H < 1 || W < 1) return OR_ERR_INVALID;
            break;
        default:
            return OR_ERR_UNSUPPORTED;   /* conv2d / linear are not part of a stack */
        }
        int64_t *s = shapes + 4 * (l + 1);
        s[0] = N; s[1] = C; s[2] = H; s[3] = W;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ breadth-first runner */

typedef struct { const float *plane; int64_t W; } plane_ctx;
static float plane_get(const void *ctx, int64_t r, int64_t q)
{
    const plane_ctx *p = (const plane_ctx *)ctx;
    return p->plane[r * p->W + q];
}

/* fig:trio-bf: for each layer, every output element of the whole tensor, then the next
 * layer.  `operands[k-1]` is ADD operand k, shaped like the ADD layer's input. */
int oracle_run_bf(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                  const float *x, const float *const *operands, int n_operands, float *y)
{
    int64_t *shapes = (int64_t *)malloc(sizeof(int64_t) * 4 * (size_t)(n_layers + 1));
    if (!shapes) return OR_ERR_NOMEM;
    int st = oracle_layer_shapes(layers, n_layers, in_shape, n_operands, shapes);
    if (st != OR_OK || !x || !y) { free(shapes); return st != OR_OK ? st : OR_ERR_INVALID; }

    int64_t n0 = shapes[0] * shapes[1] * shapes[2] * shapes[3];
    float *t = (float *)malloc(sizeof(float) * (size_t)n0);
    if (!t) { free(shapes); return OR_ERR_NOMEM; }
    memcpy(t, x, sizeof(float) * (size_t)n0);

    for (int l = 0; l < n_layers; ++l) {
        const or_layer *L = &layers[l];
        const int64_t *si = shapes + 4 * l, *so = shapes + 4 * (l + 1);
        int64_t N = si[0], C = si[1], H = si[2], W = si[3], Ho = so[2], Wo = so[3];
        float *u = (float *)malloc(sizeof(float) * (size_t)(N * C * Ho * Wo));
        if (!u) { free(t); free(shapes); return OR_ERR_NOMEM; }
        const float *opnd = (L->kind == OR_ADD) ? operands[L->operand - 1] : NULL;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t c = 0; c < C; ++c) {
                const float *pin = t + (n * C + c) * H * W;
                float *pout = u + (n * C + c) * Ho * Wo;
                if (is_pool(L->kind)) {
                    plane_ctx ctx = { pin, W };
                    for (int64_t i = 0; i < Ho; ++i)
                        for (int64_t j = 0; j < Wo; ++j)
                            pout[i * Wo + j] = pool_elem(L, H, W, i, j, plane_get, &ctx);
                } else {
                    const float *po = opnd ? opnd + (n * C + c) * H * W : NULL;
                    for (int64_t e = 0; e < H * W; ++e)
                        pout[e] = ew_apply(L, c, pin[e], po ? po[e] : 0.0f);
                }
            }
        free(t);
        t = u;
    }
    const int64_t *sl = shapes + 4 * n_layers;
    memcpy(y, t, sizeof(float) * (size_t)(sl[0] * sl[1] * sl[2] * sl[3]));
    free(t);
    free(shapes);
    return OR_OK;
}

/* ------------------------------------------------------------------ depth-first twin */

/* A region of one (n, c) plane of layer l's INPUT: rows [r0, r1), cols [q0, q1) in that
 * layer's coordinates; may extend past the tensor (padding), such cells are absent. */
typedef struct { int64_t r0, r1, q0, q1; float *v; } region;

typedef struct { const region *R; } region_ctx;
static float region_get(const void *ctx, int64_t r, int64_t q)
{
    const region *R = ((const region_ctx *)ctx)->R;
    return R->v[(r - R->r0) * (R->q1 - R->q0) + (q - R->q0)];
}

/* fig:trio-df: each output tile of each (n, c) plane is produced by pushing
 * just the data it depends on through every layer.  Regions are found backwards
 * (in_lo = out_lo*s - p, in_hi = (out_hi-1)*s + k - p; identity for element-wise
 * layers), then computed forwards with exactly the per-element arithmetic of the
 * breadth-first runner.  Tile = tile_h x tile_w output elements (<= 0: whole plane). */
int oracle_run_df(const or_layer *layers, int n_layers, const int64_t in_shape[4],
                  const float *x, const float *const *operands, int n_operands,
                  int64_t tile_h, int64_t tile_w, float *y)
{
    int64_t *shapes = (int64_t *)malloc(sizeof(int64_t) * 4 * (size_t)(n_layers + 1));
    if (!shapes) return OR_ERR_NOMEM;
    int st = oracle_layer_shapes(layers, n_layers, in_shape, n_operands, shapes);
    if (st != OR_OK || !x || !y) { free(shapes); return st != OR_OK ? st : OR_ERR_INVALID; }
    region *R = (region *)calloc((size_t)(n_layers + 1), sizeof(region));
    if (!R) { free(shapes); return OR_ERR_NOMEM; }

    const int64_t N = in_shape[0], C = in_shape[1];
    const int64_t HoF = shapes[4 * n_layers + 2], WoF = shapes[4 * n_layers + 3];
    if (tile_h <= 0) tile_h = HoF;
    if (tile_w <= 0) tile_w = WoF;

    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t o0 = 0; o0 < HoF; o0 += tile_h)
                for (int64_t p0 = 0; p0 < WoF; p0 += tile_w) {
                    /* backward region propagation */
                    R[n_layers].r0 = o0; R[n_layers].r1 = o0 + tile_h < HoF ? o0 + tile_h : HoF;
                    R[n_layers].q0 = p0; R[n_layers].q1 = p0 + tile_w < WoF ? p0 + tile_w : WoF;
                    for (int l = n_layers - 1; l >= 0; --l) {
                        const or_layer *L = &layers[l];
                        if (is_pool(L->kind)) {
                            R[l].r0 = R[l + 1].r0 * L->sh - L->ph;
                            R[l].r1 = (R[l + 1].r1 - 1) * L->sh + L->kh - L->ph;
                            R[l].q0 = R[l + 1].q0 * L->sw - L->pw;
                            R[l].q1 = (R[l + 1].q1 - 1) * L->sw + L->kw - L->pw;
                        } else {
                            R[l].r0 = R[l + 1].r0; R[l].r1 = R[l + 1].r1;
                            R[l].q0 = R[l + 1].q0; R[l].q1 = R[l + 1].q1;
                        }
                    }
                    for (int l = 0; l <= n_layers; ++l) {
                        size_t cnt = (size_t)((R[l].r1 - R[l].r0) * (R[l].q1 - R[l].q0));
                        R[l].v = (float *)malloc(sizeof(float) * (cnt ? cnt : 1));
                        if (!R[l].v) { for (int k = 0; k < l; ++k) free(R[k].v); free(R); free(shapes); return OR_ERR_NOMEM; }
                    }
                    /* load the stack-input region (in-bounds cells only) */
                    {
                        const int64_t H = shapes[2], W = shapes[3];
                        const float *pl = x + (n * C + c) * H * W;
                        int64_t rw = R[0].q1 - R[0].q0;
                        for (int64_t r = R[0].r0; r < R[0].r1; ++r)
                            for (int64_t q = R[0].q0; q < R[0].q1; ++q)
                                R[0].v[(r - R[0].r0) * rw + (q - R[0].q0)] =
                                    (r >= 0 && r < H && q >= 0 && q < W) ? pl[r * W + q] : 0.0f;
                    }
                    /* forward through every layer on the region */
                    for (int l = 0; l < n_layers; ++l) {
                        const or_layer *L = &layers[l];
                        const int64_t H = shapes[4 * l + 2], W = shapes[4 * l + 3];
                        const int64_t Ho = shapes[4 * l + 6], Wo = shapes[4 * l + 7];
                        int64_t rwi = R[l].q1 - R[l].q0, rwo = R[l + 1].q1 - R[l + 1].q0;
                        const float *opl = (L->kind == OR_ADD)
                            ? operands[L->operand - 1] + (n * C + c) * H * W : NULL;
                        region_ctx ctx = { &R[l] };
                        for (int64_t i = R[l + 1].r0; i < R[l + 1].r1; ++i)
                            for (int64_t j = R[l + 1].q0; j < R[l + 1].q1; ++j) {
                                float *dst = &R[l + 1].v[(i - R[l + 1].r0) * rwo + (j - R[l + 1].q0)];
                                if (i < 0 || i >= Ho || j < 0 || j >= Wo) { *dst = 0.0f; continue; }  /* absent */
                                if (is_pool(L->kind))
                                    *dst = pool_elem(L, H, W, i, j, region_get, &ctx);
                                else
                                    *dst = ew_apply(L, c, R[l].v[(i - R[l].r0) * rwi + (j - R[l].q0)],
                                                    opl ? opl[i * W + j] : 0.0f);
                            }
                    }
                    /* write the tile */
                    {
                        float *pl = y + (n * C + c) * HoF * WoF;
                        int64_t rw = R[n_layers].q1 - R[n_layers].q0;
                        for (int64_t i = R[n_layers].r0; i < R[n_layers].r1; ++i)
                            for (int64_t j = R[n_layers].q0; j < R[n_layers].q1; ++j)
                                pl[i * WoF + j] = R[n_layers].v[(i - R[n_layers].r0) * rw + (j - R[n_layers].q0)];
                    }
                    for (int l = 0; l <= n_layers; ++l) free(R[l].v);
                }
    free(R);
    free(shapes);
    return OR_OK;
}
