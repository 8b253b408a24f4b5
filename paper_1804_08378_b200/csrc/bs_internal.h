// bs_internal.h -- shared between the host planner/runtime (bs_api.cpp) and the sm_100a
// kernels (k_*.cu, bs_device.cuh).  Not part of the public ABI (see include/bs.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bs {

// Longest element-wise op run fused into one prologue/epilogue.  Longer runs are split
// into an extra step by the planner (a serialised sequence).
constexpr int kMaxOps = 8;

// Device-side element-wise operations (layer -> op mapping).
enum DevOp : int32_t {
  DOP_AFFINE = 1,  // folded inference BatchNorm: y = fmaf(x, scale[c], shift[c])
  DOP_RELU = 2,    // y = x > 0 ? x : +0
  DOP_SCALE = 3,   // y = alpha * x
  DOP_ADD = 4,     // y = x + operand[idx]
};

// Program classes: the kernels are specialised for the programs the paper's networks use
// (ReLU; folded BN -> ReLU) and fall back to an op-outer interpreter otherwise.
enum ProgClass : int32_t { PC_NONE = 0, PC_RELU = 1, PC_AFFINE = 2, PC_AFFINE_RELU = 3, PC_GENERIC = 4 };

// An element-wise program, passed by value as a kernel parameter.
struct OpProgram {
  int32_t n;
  int32_t n_deferred;              // max pools: the first n_deferred ops are the (monotone)
                                   // prologue applied after the pool (bs_kernels.cu header)
  int32_t kind[kMaxOps];
  const float2* affine[kMaxOps];   // DOP_AFFINE: device (scale, shift) per channel
  float alpha[kMaxOps];            // DOP_SCALE
  const float* operand[kMaxOps];   // DOP_ADD: device base of the operand tensor (set per execute)
  int32_t aff_slot[kMaxOps];       // AFFINE ops whose params are cached in registers: 0/1, else -1
  int32_t add_slot[kMaxOps];       // flat kernel: the first ADD's operand is prefetched (0), else -1
};
constexpr int kAffSlots = 2;

// Magic-number unsigned division for n < 2^31 (q = (umulhi(n, m) + n) >> s).
struct FastDiv {
  uint32_t d, m, s;
};
FastDiv make_fastdiv(uint32_t d);

// ---------------------------------------------------------------- element-wise step
struct EwArgs {
  const float* in;
  float* out;
  int64_t e_begin, e_end;   // element range (global flat indices; < 2^31 after rebasing)
  FastDiv hw;               // plane size H*W
  FastDiv c;                // channels
  int32_t hw_ge4;           // H*W >= 4 (a float4 spans at most 2 planes)
  const float* add0_ptr;    // operand of the prefetched ADD (add_slot 0), or nullptr
  int32_t prog_class;       // ProgClass of prog
  int32_t unroll;           // float4s per thread per iteration: 4, or 1 for small tensors
  OpProgram prog;
};

// ---------------------------------------------------------------- pool step
struct PoolArgs {
  const float* in;          // stack/step input base (plane 0)
  float* out;               // step output base (plane 0)
  int32_t C, H, W, Ho, Wo;
  int64_t plane0, n_planes; // planes [plane0, plane0 + n_planes) processed by this launch
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t is_max, count_include_pad;
  // column-walker geometry (kernels 2/3)
  int32_t G;                // lane groups per warp (one plane each)
  int32_t gw;               // lanes per group = (Jg - 1) * sw + kw  (<= 32)
  int32_t Jg;               // output columns per group
  int32_t n_cc;             // column chunks per plane = ceil(Wo / Jg)
  int32_t rows_per_task;    // output rows per warp task
  int32_t n_rb;             // row bands = ceil(Ho / rows_per_task)
  int64_t n_tasks;          // ceil(n_planes / G) * n_cc * n_rb
  int32_t pro_class, epi_class;  // ProgClass of pro / epi
  // staged kernel (6): whole-plane tiles bulk-copied (TMA) into shared memory
  int32_t tile_planes;      // planes per tile (tile_planes * H * W % 4 == 0)
  int32_t stages;           // shared-memory ring depth
  int64_t n_tiles;          // ceil(n_planes / tile_planes)
  FastDiv cdiv;             // channels C (plane -> channel)
  OpProgram pro, epi;       // prologue (per input element), epilogue (per output element)
};

// Kernel variants (bs_launch_info.kernel).
enum KernelKind : int32_t { K_EW = 1, K_POOL_SPEC = 2, K_POOL_GENERIC = 3, K_POOL_NAIVE = 4, K_POOL_VEC = 5,
                          K_POOL_STAGED = 6, K_SEQ = 7, K_POOL_PLANES = 8 };

// ---------------------------------------------------------------- multi-step sequence (NEXT-2)
// One step of an on-chip sequence: [prologue] pool [epilogue] on the
// step's input planes (H x W) -> (Ho x Wo).  A step without a pool is a 1x1/s1 max pool
// (the identity).  Held in a plan-owned device array; programs have no ADD ops.
// A device-table limit (the descriptors of a sequence live in a per-CTA shared table); the
// planner's real limit is the shared-memory footprint of the sequence's tile.
constexpr int kMaxSeqSteps = 64;
struct SeqStepDev {
  int32_t H, W, Ho, Wo;
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t is_max, count_include_pad;
  int32_t fast;             // 1: 3x3/s1/p1 max pool, no prologue, epilogue class <= PC_AFFINE_RELU,
                            //    W % 4 == 0, W <= 256 (vectorised path, k_seq.cu)
  int32_t epi_class;        // ProgClass of epi
  int32_t in_pitch;         // floats per plane in the step's input buffer (stage or work buffer)
  int32_t out_pitch;        // floats per plane in the step's output work buffer (unused by the last step)
  OpProgram pro, epi;
};
// Rows of one step for one band of a tile (the sequence's halo back-propagation):
// the input buffer holds rows [in_lo, in_hi) of the step's input plane, the step computes rows
// [out_lo, out_hi) of its output; the fast path splits those rows into n_chunks chunks of L rows.
struct SeqRange {
  int32_t in_lo, in_hi, out_lo, out_hi;
  int32_t n_chunks, L;
  FastDiv chunks;           // division by n_chunks
  int32_t pad_;             // 40 bytes: the float2 table after an array of these stays 8-B aligned
};
struct SeqArgs {
  const float* in;          // sequence input base (plane 0)
  float* out;               // sequence output base (plane 0)
  const SeqStepDev* steps;  // device array of n_steps descriptors
  const SeqRange* ranges;   // device array [n_bands][n_steps]
  int32_t n_steps;
  int32_t C;
  int64_t plane0, n_planes;
  int32_t tile_planes, stages;
  int32_t n_bands;          // 1: whole-plane tiles; > 1: row-band tiles of one plane (halo tiles)
  int64_t n_tiles;          // ceil(n_planes / tile_planes) * n_bands
  int32_t stage_bytes;      // bytes per ring stage (128-B multiple)
  int32_t work_floats;      // floats per work buffer
  int32_t in_plane;         // H0 * W0
  FastDiv cdiv;             // channels C (plane -> channel)
  int32_t inplace_seg;      // > 0: the warp-per-plane in-place kernel (seq_inplace) with lane
                            // segments of this width (16 or 32); 0: seq_staged
  int32_t H0, W0;           // step-0 input plane (host-side kernel choice)
};
constexpr int kInplaceWarps = 4;   // consumer warps per CTA of seq_inplace (1, 2 or 4 per plane)
cudaError_t launch_seq(const SeqArgs& a, int grid, cudaStream_t st);
size_t seq_smem(const SeqArgs& a);
size_t seq_inplace_smem(const SeqArgs& a);
int seq_inplace_threads(const SeqArgs& a);
int seq_max_blocks_per_sm(const SeqArgs& a);

// Launchers (k_*.cu).  Return the launch error (cudaSuccess on success).
cudaError_t launch_ew(const EwArgs& a, int grid, int block, cudaStream_t st);
cudaError_t launch_pool(const PoolArgs& a, int kernel_kind, int grid, int block, cudaStream_t st);
// Whether a specialised (compile-time k/s) column-walker exists for this geometry.
bool pool_has_specialisation(int kh, int kw, int sh, int sw);
// Occupancy helpers for the planner.
int ew_max_blocks_per_sm(int prog_class);
// Output rows per iteration (U) of the specialised column walker for a k x k / s window.
int pool_spec_unroll(int k, int s);
// Vector width (4, 2) of the vector column walker for this geometry, 0 if unsupported.
int pool_vec_width(int kh, int kw, int sh, int sw, int ph, int pw, int W, int Wo);
int pool_vec_unroll(int vec);
// Staged (TMA bulk copy + mbarrier ring) kernel: threads per CTA, and dynamic shared memory.
#ifndef BS_STAGED_CW
#define BS_STAGED_CW 8
#endif
constexpr int kStagedConsumerWarps = BS_STAGED_CW;
constexpr int kStagedThreads = 32 * (kStagedConsumerWarps + 1);
#ifndef BS_SEQ_CW
#define BS_SEQ_CW 8
#endif
constexpr int kSeqWarps = BS_SEQ_CW;            // consumer warps of the on-chip sequence kernel
constexpr int kSeqThreads = 32 * (kSeqWarps + 1);
constexpr int kStagedMaxStages = 8;    // mbarrier pairs in the staged kernels' smem header
constexpr int kStagedHeader = 128;     // bytes of smem before the first stage
size_t pool_staged_smem(int tile_planes, int HW, int HWo, int stages);
// Bytes of one ring stage: a tile of P planes at offset (global address mod 16), 128-B multiple.
__host__ __device__ inline size_t pool_staged_stride(int tile_planes, int HW) {
  return ((size_t)tile_planes * HW * 4 + 16 + 127) / 128 * 128;
}
int pool_max_blocks_per_sm(int kernel_kind, const PoolArgs& a, int block);
// Whole-plane pool kernel (k_pool_planes.cu): whether it applies, its block and dynamic smem.
bool pool_planes_applies(int H, int W, int kh, int kw, int ph, int pw);
int pool_planes_threads();
size_t pool_planes_smem(int HW);

}  // namespace bs
