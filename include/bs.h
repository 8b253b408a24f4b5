/*
 * bs.h -- C ABI of the B200-native BrainSlug stack executor.
 *
 * BrainSlug (arXiv:1804.08378) accelerates a *stack* -- a maximal run of consecutive
 * element-wise and pooling layers (§3.2 "Aggregation Detection") --
 * by executing it depth-first: each tile of the input is read from main memory once,
 * pushed through every layer of the stack on-chip, and written once (fig:trio-df,
 * P:L208-239; §3.1), instead of one memory round-trip per layer.
 *
 * The interface follows the paper's two phases (fig:brainslug-arch P:L378-411):
 *   compile phase  -> bs_plan_create: validate the layer list, map layers to
 *                                   operations, group operations into steps and steps into
 *                                   sequences, size tiles/halos for the device;
 *   execution phase -> bs_execute: "calculates the output size ... loaded,
 *                                   executed"; sequences run serialised.
 * Kernels are hand-written, ahead-of-time compiled for sm_100a (no code generation).
 *
 * Conventions for every function:
 *  - extern "C", no C++ types or exceptions cross the boundary; errors are return codes,
 *    with a thread-local message from bs_last_error() naming the layer index and field.
 *  - Tensors: contiguous NCHW fp32, exactly N*C*H*W elements, DEVICE pointers on the
 *    plan's device unless a function says "host".  No strides/views.
 *  - bs_execute* only ENQUEUE work on the caller's stream: no allocation, no host sync,
 *    no host<->device copy (except bs_execute_host, whose job is exactly those copies).
 *    Asynchronous device faults surface at the caller's next synchronisation.
 *  - Plans are immutable after creation.  Concurrent bs_execute / bs_execute_ex of a plan
 *    with n_launches == 1 on different streams is safe.  A plan with n_launches > 1 (its
 *    serialised sequences share plan-owned intermediates) and bs_execute_host (plan-owned
 *    copy streams and events) must not run concurrently with itself: use one plan per
 *    stream there.  bs_plan_create is reentrant.
 */
#ifndef BS_H
#define BS_H

#include <stdint.h>

#if defined(__GNUC__)
#define BS_API __attribute__((visibility("default")))
#else
#define BS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *bs_stream_t;   /* == cudaStream_t; NULL = legacy default stream */
typedef struct bs_plan bs_plan;            /* opaque, immutable after create */

typedef enum {
    BS_OK = 0,
    BS_ERR_INVALID_ARGUMENT = 2, /* NULL pointer, n_layers < 1, unknown kind, non-positive dim,
                                    misaligned (not 16-B) or overlapping tensor pointers,
                                    wrong number of inputs, execute on a host-only plan */
    BS_ERR_VALIDATION = 3,       /* k < 1, s < 1, p < 0 or p > k/2, pool extent < 1,
                                    eps <= 0, var < 0, NULL BN array, bad ADD operand index */
    BS_ERR_PLANNING = 4,         /* CONV2D / LINEAR in the stack (opaque: not optimizable,
                                    P:L135-146); tensor too large for the index
                                    types */
    BS_ERR_CUDA = 6,             /* CUDA error during create (alloc/copy/attributes) or launch */
    BS_ERR_OUT_OF_MEMORY = 7     /* device allocation of plan-owned memory failed */
} bs_status;

typedef enum {
    BS_OP_BATCHNORM = 1,  /* inference BN, folded to a per-channel affine (north_star)     */
    BS_OP_RELU = 2,       /* f(x) = max(0, x); +0.0 for x <= 0               */
    BS_OP_MAXPOOL = 3,    /* window max, padded cells absent                */
    BS_OP_AVGPOOL = 4,    /* window sum + "AvgNormalization" (lst:finalcode P:L520-524)    */
    BS_OP_COPY = 5,       /* identity (eval-mode Dropout); elided                        */
    BS_OP_SCALE = 6,      /* y = alpha * x                                                */
    BS_OP_ADD = 7,        /* y = x + operand (residual add)                               */
    BS_OP_CONV2D = 100,   /* representable so a front-end can pass a whole chain; always  */
    BS_OP_LINEAR = 101    /* rejected with BS_ERR_PLANNING                                 */
} bs_op_kind;

/* One layer.  Unused fields are ignored for other kinds. */
typedef struct {
    int32_t kind;                                   /* bs_op_kind */
    int32_t kernel_h, kernel_w;                     /* pools: k >= 1 */
    int32_t stride_h, stride_w;                     /* pools: s >= 1 */
    int32_t pad_h, pad_w;                           /* pools: 0 <= p <= k/2 (PyTorch rule) */
    int32_t count_include_pad;                      /* avgpool: 1 = divisor k_h*k_w (PyTorch default) */
    float eps;                                      /* BN: > 0 */
    const float *gamma, *beta, *running_mean, *running_var; /* BN: HOST arrays, length = C;
                                                       copied during bs_plan_create */
    float alpha;                                    /* SCALE */
    int32_t operand;                                /* ADD: index >= 1 into bs_execute_ex inputs[] */
} bs_layer_desc;

typedef struct { int64_t n, c, h, w; } bs_shape;

/* Options; pass NULL for the defaults of the current device. */
typedef struct {
    int32_t device;                 /* CUDA device ordinal; -1 = current device */
    int32_t host_only;              /* 1 = plan on the host only (no device memory; the plan can
                                       be queried but not executed); used by CPU tests */
    int32_t max_steps_per_sequence; /* steps per on-chip sequence (one launch):
                                       0 = planner: as many as fit the shared-memory budget, and
                                           for halo (row-band) tiles only while the band covers
                                           its own input halo (bounded redundant work);
                                       -1 = the paper's "unrestricted" strategy: as many as fit
                                           (redundant halo work grows until a new sequence starts,
                                           P:L718-729);
                                       k >= 1: at most k (1 and 5 mirror P:L677-678).
                                       Never more than 64 (the device step table) */
    int32_t threads_per_block;      /* must be 0: every kernel has a fixed block size tuned for
                                       sm_100a (256 or 32 x 9); other values -> INVALID_ARGUMENT */
    int32_t force_rows_per_task;    /* 0 = planner; >0 forces the output-row band of a pool
                                       tile (tests use it: results must not depend on tiling) */
    int32_t force_outputs_per_group;/* 0 = planner; >0 forces output columns per lane group */
    int32_t force_generic;          /* 0 = planner picks the pool kernel; 1 = force the
                                       runtime-geometry column walker; 2 = the global-memory
                                       scalar walker (no vector / staged kernels); 3 = the
                                       staged (TMA) walker where it applies, no vector walker.
                                       Tests use it: results must not depend on the kernel */
    int32_t force_tile_planes;      /* 0 = planner; >0: planes per staged (TMA) tile, rounded to
                                       the 16-byte bulk-copy granularity */
    int32_t force_stages;           /* 0 = planner; 2..8: shared-memory ring depth of the staged
                                       kernel */
    int32_t smem_budget_bytes;      /* 0 = planner default (<= 220 KB per CTA); > 0: the most
                                       dynamic shared memory per CTA the plan may use -- the
                                       paper's per-step cache budget.  Staged pools
                                       use fewer ring stages (or the global-memory walker) and
                                       on-chip sequences split earlier to fit it */
    int32_t reserved[2];
} bs_plan_options;

/* Whole-plan summary. */
typedef struct {
    bs_shape out;                   /* output shape of the stack */
    int32_t n_layers, n_ops;        /* ops = layers minus elided COPYs */
    int32_t n_steps, n_sequences, n_launches;
    int32_t n_inputs;               /* 1 + number of ADD operands */
    int64_t alg_bytes_read;         /* one read of the input + every ADD operand */
    int64_t alg_bytes_written;      /* one write of the output */
    int64_t param_bytes;            /* folded per-channel parameters held on the device */
    int64_t intermediate_bytes;     /* plan-owned buffers between serialised sequences */
} bs_plan_info;

/* Per-launch (= per sequence) details.  For kernel 7, groups_per_warp = steps fused and
 * outputs_per_group = planes per staged tile. */
typedef struct {
    int32_t kernel;                 /* 1 = element-wise streaming, 2 = pool column-walker
                                       (specialised k/s), 3 = pool column-walker (runtime
                                       geometry), 4 = pool one-thread-per-output,
                                       5 = pool vector column walker (stride 2, W % 2 == 0),
                                       6 = pool staged walker (TMA bulk copies of whole planes
                                       into a shared-memory ring), 7 = on-chip multi-step
                                       sequence (same staging; steps ping-pong in smem),
                                       8 = whole-plane pool (window = plane, e.g. a global
                                       7x7 average): a warp reduces 32 planes, bulk-
                                       copied (TMA) into its shared-memory slice */
    int32_t first_layer, last_layer;/* layer index range [first, last] covered */
    bs_shape in, out;
    int32_t pool_kh, pool_kw, pool_sh, pool_sw, pool_ph, pool_pw;  /* 0 if no pool */
    int32_t n_prologue_ops, n_epilogue_ops;
    int32_t grid, block;
    int32_t groups_per_warp;        /* lane groups (one plane each) packed in a warp */
    int32_t outputs_per_group;      /* output columns produced by one lane group */
    int32_t rows_per_task;          /* output rows walked by one warp task */
    int32_t halo_rows;              /* kernels 2-6: input rows re-read between row bands (k - s,
                                       >= 0); kernel 7: step-0 input rows loaded in total over a
                                       plane's bands beyond the plane's own rows (redundant halo) */
    int64_t n_tasks;                /* warp tasks (kernels 2-5, 8), staged tiles (6, 7) */
    int64_t alg_bytes_read, alg_bytes_written;
    int32_t smem_bytes;             /* dynamic shared memory per CTA (0 for kernels 1-5) */
    int32_t tile_planes;            /* kernels 6/7: (n, c) planes per staged tile, else 0 */
    int32_t tile_rows;              /* kernel 7 with row-band tiles: output rows per tile, else 0
                                       (whole planes) */
    int32_t stages;                 /* kernels 6/7: shared-memory ring depth, else 0 */
} bs_launch_info;

/*
 * bs_plan_create -- compile phase.
 *   layers/n_layers : the stack, in network order (host memory; copied).
 *   input           : (N, C, H, W) of the stack input; C, H, W >= 1.  N = 0 (an empty batch) is
 *                     valid: the plan reports out.n = 0, 0 launches and 0 algorithmic bytes,
 *                     and bs_execute* return BS_OK without touching memory (NULL pointers allowed).
 *   opts            : NULL = defaults on the current device.
 *   plan_out        : receives the plan (NULL on failure).
 * Steps performed: validation + shape inference (a1); layer -> op mapping with BN folded
 * in fp64 to scale = gamma/sqrt(var+eps), shift = beta - mean*scale, rounded once to fp32
 * (a2); greedy step grouping -- an element-wise op always joins the current step, a pool
 * joins only if the step has none (prose rule) (a3); sequence
 * packing and tile geometry for the device (a4).
 * Allocates device memory for folded parameters (8*C bytes per BN) and for intermediates
 * between serialised sequences; the plan owns it.
 * Errors: BS_ERR_INVALID_ARGUMENT / VALIDATION / PLANNING / CUDA / OUT_OF_MEMORY.
 */
BS_API bs_status bs_plan_create(const bs_layer_desc *layers, int32_t n_layers, bs_shape input,
                         const bs_plan_options *opts, bs_plan **plan_out);

/* bs_plan_query -- fill *info.  Errors: BS_ERR_INVALID_ARGUMENT on NULL. */
BS_API bs_status bs_plan_query(const bs_plan *plan, bs_plan_info *info);

/* bs_plan_query_launch -- details of launch `index` in [0, n_launches). */
BS_API bs_status bs_plan_query_launch(const bs_plan *plan, int32_t index, bs_launch_info *info);

/*
 * bs_execute -- execution phase for stacks without ADD.
 *   in  : device pointer, input shape, 16-B aligned.
 *   out : device pointer, bs_plan_info.out shape, 16-B aligned; must not overlap `in`,
 *         except exactly in == out for plans whose every step is element-wise (in-place).
 *   stream : CUDA stream the n_launches kernels are enqueued on, in order.
 * Errors: BS_ERR_INVALID_ARGUMENT (NULL/misaligned/overlap/plan needs operands/host-only
 * plan), BS_ERR_CUDA (launch failure; message in bs_last_error()).
 */
BS_API bs_status bs_execute(const bs_plan *plan, const float *in, float *out, bs_stream_t stream);

/*
 * bs_execute_ex -- as bs_execute with ADD operands.
 *   inputs[0] = stack input; inputs[k] = operand k (shape = the ADD layer's input shape).
 *   n_inputs must equal bs_plan_info.n_inputs.
 */
BS_API bs_status bs_execute_ex(const bs_plan *plan, const float *const *inputs, int32_t n_inputs,
                        float *out, bs_stream_t stream);

/*
 * bs_execute_host -- end-to-end execution from HOST buffers.
 *   h_inputs[n_inputs] : host pointers (pinned for copy/compute overlap; pageable works
 *                        but serialises), same shapes as bs_execute_ex.
 *   h_out              : host pointer for the output.
 *   d_inputs[n_inputs], d_out : caller-owned device buffers of the same shapes (staging).
 *   n_chunks           : the batch is split into n_chunks image ranges; chunk k's
 *                        host->device copy, kernels, and device->host copy are pipelined
 *                        across the plan's two copy streams and `stream` (0 = 4 chunks;
 *                        at most one chunk per image).
 * Returns after ENQUEUEING; the caller synchronises `stream` before reading h_out.
 */
BS_API bs_status bs_execute_host(const bs_plan *plan, const float *const *h_inputs, int32_t n_inputs,
                          float *h_out, float *const *d_inputs, float *d_out,
                          int32_t n_chunks, bs_stream_t stream);

/*
 * bs_execute_host_batch -- bs_execute_host for n_plans executions in array order (a network's
 * stacks, each from host buffers), pipelined ACROSS executions: execution i+1's host->device
 * copies start while execution i's kernels and device->host copies are still running, so only
 * the first copy in and the last copy out of the whole batch are not overlapped (PCIe is full
 * duplex).  Per execution i: plans[i], h_inputs[i][0..n_inputs[i]), h_outs[i], d_inputs[i][..],
 * d_outs[i] as in bs_execute_host; n_chunks applies to each execution (0 = planner picks).
 * The device buffers of different executions must not overlap (BS_ERR_INVALID_ARGUMENT): an
 * execution's copies may run concurrently with another's kernels.  All plans on one device; the
 * copy streams and events of the first non-empty plan are used.  Returns after ENQUEUEING; the
 * caller synchronises `stream` before reading any h_outs[i].  Errors name the execution index.
 */
BS_API bs_status bs_execute_host_batch(const bs_plan *const *plans, int32_t n_plans,
                                       const float *const *const *h_inputs, const int32_t *n_inputs,
                                       float *const *h_outs, float *const *const *d_inputs,
                                       float *const *d_outs, int32_t n_chunks, bs_stream_t stream);

/* bs_plan_destroy -- frees plan-owned device memory and streams.  NULL-safe.  The caller
 * must ensure no execution using the plan is still in flight. */
BS_API void bs_plan_destroy(bs_plan *plan);

/*
 * bs_graph_* -- a whole network's stacks as ONE CUDA graph ("a CUDA
 * graph over all of a network's stacks"; small stacks are launch-bound).  The
 * launches of n_plans executions -- plans[i] on inputs[i][0..n_inputs_i) -> outs[i], in array
 * order, each ordered after the previous one exactly as consecutive bs_execute_ex calls on
 * one stream -- are captured once and replayed by bs_graph_launch with a single host call.
 *   plans / inputs / outs : as bs_execute_ex, per execution; n_inputs[i] = the plan's n_inputs.
 *                           Device pointers are BOUND at creation (graph semantics): a replay
 *                           reads and writes the same buffers.  All plans on one device.
 *   graph_out             : receives the graph.  Errors: as bs_execute_ex (index named), and
 *                           BS_ERR_CUDA if capture or instantiation fails.
 * Ownership: the graph references the plans (their parameters / intermediates); destroy the
 * graph before any of its plans.  Replays on one stream are ordered like any kernel launch.
 */
typedef struct bs_graph bs_graph;
BS_API bs_status bs_graph_create(const bs_plan *const *plans, int32_t n_plans, const float *const *const *inputs,
                                 const int32_t *n_inputs, float *const *outs, bs_graph **graph_out);
BS_API bs_status bs_graph_launch(const bs_graph *graph, bs_stream_t stream);
BS_API void bs_graph_destroy(bs_graph *graph);   /* NULL-safe; no replay may be in flight */

/* Thread-local description of the last error on this thread ("" if none). */
BS_API const char *bs_last_error(void);

/* Static name of a status code. */
BS_API const char *bs_status_string(bs_status s);

/* Library version, for the binding's sanity check. */
BS_API int32_t bs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BS_H */
