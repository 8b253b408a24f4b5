// bs_api.cpp -- the C ABI (include/bs.h): planner (compile phase) and
// runtime (execution phase) of the B200 depth-first stack executor.
//
//   a1 validate + shape inference ........ validate_and_shape()
//   a2 layer -> ops, BN folding ........... map_ops()
//   a3 step grouping ...................... group_steps()
//   a4 sequence packing + tile geometry ... pack_and_tile()
//   a5 dispatch ........................... enqueue()
//
// See DESIGN.md for the B200 tile policy and how it differs from the paper's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include "../../include/bs.h"
#include "bs_internal.h"

using namespace bs;

namespace {

thread_local std::string g_err;

bs_status fail(bs_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

const char* kind_name(int k) {
  switch (k) {
    case BS_OP_BATCHNORM: return "batchnorm";
    case BS_OP_RELU: return "relu";
    case BS_OP_MAXPOOL: return "maxpool";
    case BS_OP_AVGPOOL: return "avgpool";
    case BS_OP_COPY: return "copy";
    case BS_OP_SCALE: return "scale";
    case BS_OP_ADD: return "add";
    case BS_OP_CONV2D: return "conv2d";
    case BS_OP_LINEAR: return "linear";
    default: return "?";
  }
}

bool is_pool(int k) { return k == BS_OP_MAXPOOL || k == BS_OP_AVGPOOL; }

struct Shape4 {
  int64_t n, c, h, w;
  int64_t numel() const { return n * c * h * w; }
};

// A host-side element-wise op.
struct HostOp {
  int32_t kind;                   // DevOp
  int32_t layer;                  // source layer index
  std::vector<float2> affine;     // DOP_AFFINE: folded (scale, shift) per channel
  size_t affine_off = 0;          // offset (in float2) into the plan's parameter block
  float alpha = 1.f;
  int32_t operand = 0;            // DOP_ADD: input index >= 1
};

struct Step {
  int first_layer = 0, last_layer = 0;
  std::vector<HostOp> pro, epi;
  bool has_pool = false;
  int pool_layer = -1;
  int kh = 0, kw = 0, sh = 0, sw = 0, ph = 0, pw = 0, is_max = 0, cip = 1;
  Shape4 in{}, out{};
};

struct Launch {
  Step step;
  int32_t kernel = K_EW;
  int src = -1;  // -1 stack input, else intermediate buffer index
  int dst = -1;  // -1 stack output, else intermediate buffer index
  // pool geometry (kernels 2/3)
  int32_t G = 1, gw = 32, Jg = 1, n_cc = 1, rows_per_task = 1, n_rb = 1, U = 1;
  int32_t tile_planes = 0, stages = 0;   // staged kernel
  int32_t ctas_per_sm = 0;               // staged kernel: CTAs per SM the grid is sized for (0 = occupancy)
  int32_t block = 256;
  int32_t blocks_per_sm = 0;
  bool deferred = false;            // max pool: monotone prologue moved after the pool
  std::vector<Step> seq;            // K_SEQ: the steps of the on-chip sequence
  size_t seq_off = 0;               // K_SEQ: index of its first descriptor in the plan's array
  size_t range_off = 0;             // K_SEQ: index of its first SeqRange in the plan's array
  int32_t seq_work_floats = 0;      // K_SEQ: floats per shared-memory work buffer
  int32_t seq_bands = 1;            // K_SEQ: row bands per plane (1 = whole-plane tiles)
  int32_t seq_band_rows = 0;        // K_SEQ: output rows of the last step per band
  int32_t seq_stage_bytes = 0;      // K_SEQ: bytes per ring stage
  int32_t seq_inplace_seg = 0;      // K_SEQ: > 0 = the warp-per-plane in-place kernel (lane segment width)
  std::vector<int32_t> seq_in_pitch, seq_out_pitch;   // K_SEQ: floats per plane, per step
  std::vector<SeqRange> seq_ranges; // K_SEQ: [bands][steps]
  std::vector<HostOp> dev_pro, dev_epi;  // programs as the kernel runs them
  bs_launch_info info{};
};

}  // namespace

struct bs_plan {
  int device = 0;
  bool host_only = false;
  bool empty = false;                  // N = 0: geometry planned for N = 1, execute is a no-op
  int num_sms = 148;
  bs_plan_info info{};
  std::vector<Launch> launches;
  std::vector<Step> steps;             // every step of the stack, in order
  float2* params = nullptr;            // device parameter block
  SeqStepDev* seq_steps = nullptr;     // device descriptors of on-chip sequences
  SeqRange* seq_ranges = nullptr;      // device per-band row ranges of on-chip sequences
  float* inter[2] = {nullptr, nullptr};  // intermediates between serialised sequences
  cudaStream_t copy_stream[2] = {nullptr, nullptr};  // bs_execute_host pipelines
  cudaEvent_t ev_pool[4] = {};      // bs_execute_host: caller-stream / last-copy / per-chunk events
  int n_events = 0;
};

namespace {

// ---------------------------------------------------------------- a1: validation + shapes
bs_status validate_and_shape(const bs_layer_desc* L, int n, bs_shape in, std::vector<Shape4>& shapes,
                             int& n_inputs) {
  if (in.n < 1 || in.c < 1 || in.h < 1 || in.w < 1)
    return fail(BS_ERR_INVALID_ARGUMENT, "input shape (%lld,%lld,%lld,%lld) has a dimension < 1",
                (long long)in.n, (long long)in.c, (long long)in.h, (long long)in.w);
  shapes.assign(1, Shape4{in.n, in.c, in.h, in.w});
  int max_operand = 0;
  for (int i = 0; i < n; ++i) {
    const bs_layer_desc& d = L[i];
    Shape4 s = shapes.back();
    switch (d.kind) {
      case BS_OP_BATCHNORM:
        if (!d.gamma || !d.beta || !d.running_mean || !d.running_var)
          return fail(BS_ERR_VALIDATION, "layer %d (batchnorm): NULL parameter array", i);
        if (!(d.eps > 0.f)) return fail(BS_ERR_VALIDATION, "layer %d (batchnorm): eps=%g must be > 0", i, d.eps);
        for (int64_t c = 0; c < s.c; ++c)
          if (!(d.running_var[c] >= 0.f))
            return fail(BS_ERR_VALIDATION, "layer %d (batchnorm): running_var[%lld]=%g < 0", i, (long long)c,
                        d.running_var[c]);
        break;
      case BS_OP_RELU:
      case BS_OP_COPY:
      case BS_OP_SCALE:
        break;
      case BS_OP_ADD:
        if (d.operand < 1) return fail(BS_ERR_VALIDATION, "layer %d (add): operand=%d must be >= 1", i, d.operand);
        max_operand = std::max(max_operand, d.operand);
        break;
      case BS_OP_MAXPOOL:
      case BS_OP_AVGPOOL: {
        const char* nm = kind_name(d.kind);
        if (d.kernel_h < 1 || d.kernel_w < 1)
          return fail(BS_ERR_VALIDATION, "layer %d (%s): kernel %dx%d must be >= 1", i, nm, d.kernel_h, d.kernel_w);
        if (d.stride_h < 1 || d.stride_w < 1)
          return fail(BS_ERR_VALIDATION, "layer %d (%s): stride %dx%d must be >= 1", i, nm, d.stride_h, d.stride_w);
        if (d.pad_h < 0 || d.pad_w < 0 || 2 * d.pad_h > d.kernel_h || 2 * d.pad_w > d.kernel_w)
          return fail(BS_ERR_VALIDATION, "layer %d (%s): padding %dx%d must be in [0, kernel/2]", i, nm, d.pad_h,
                      d.pad_w);
        const int64_t ho = (s.h + 2 * d.pad_h - d.kernel_h) < 0 ? 0 : (s.h + 2 * d.pad_h - d.kernel_h) / d.stride_h + 1;
        const int64_t wo = (s.w + 2 * d.pad_w - d.kernel_w) < 0 ? 0 : (s.w + 2 * d.pad_w - d.kernel_w) / d.stride_w + 1;
        if (ho < 1 || wo < 1)
          return fail(BS_ERR_VALIDATION, "layer %d (%s): output extent %lldx%lld < 1 for input %lldx%lld", i, nm,
                      (long long)ho, (long long)wo, (long long)s.h, (long long)s.w);
        if (d.kernel_h > 65535 || d.kernel_w > 65535 || s.h > INT32_MAX || s.w > INT32_MAX)
          return fail(BS_ERR_PLANNING, "layer %d (%s): extents beyond the int32 index range", i, nm);
        s.h = ho;
        s.w = wo;
        break;
      }
      case BS_OP_CONV2D:
      case BS_OP_LINEAR:
        return fail(BS_ERR_PLANNING,
                    "layer %d (%s): not optimizable -- a stack holds only element-wise and pooling layers "
                    "(PAPER.md P:L341-351, P:L973-991)",
                    i, kind_name(d.kind));
      default:
        return fail(BS_ERR_INVALID_ARGUMENT, "layer %d: unknown kind %d", i, d.kind);
    }
    shapes.push_back(s);
  }
  n_inputs = 1 + max_operand;
  // every operand index 1..max must be used by some ADD (dense numbering)
  for (int k = 1; k <= max_operand; ++k) {
    bool used = false;
    for (int i = 0; i < n; ++i) used |= (L[i].kind == BS_OP_ADD && L[i].operand == k);
    if (!used) return fail(BS_ERR_VALIDATION, "add operands must be numbered 1..%d densely; %d unused", max_operand, k);
  }
  return BS_OK;
}

// ---------------------------------------------------------------- a2: layer -> op (+ BN fold)
// BN folding in fp64, one rounding to fp32 each (north_star "BatchNorm as per-channel affine").
HostOp fold_bn(const bs_layer_desc& d, int layer, int64_t C) {
  HostOp op;
  op.kind = DOP_AFFINE;
  op.layer = layer;
  op.affine.resize((size_t)C);
  for (int64_t c = 0; c < C; ++c) {
    const double scale = (double)d.gamma[c] / std::sqrt((double)d.running_var[c] + (double)d.eps);
    const double shift = (double)d.beta[c] - (double)d.running_mean[c] * scale;
    op.affine[(size_t)c] = make_float2((float)scale, (float)shift);
  }
  return op;
}

// ---------------------------------------------------------------- a3: step grouping
// Greedy, left to right (the prose rule; the listing lst:collapse
// P:L475-484 is inverted -- SURVEY G1): an element-wise op always joins the current step
// (prologue before its pool, epilogue after); a pool joins iff the step has none yet,
// otherwise it opens a new step.  A prologue/epilogue longer than kMaxOps also opens a step.
void group_steps(const bs_layer_desc* L, int n, const std::vector<Shape4>& shapes, std::vector<Step>& steps) {
  steps.clear();
  Step cur;
  cur.first_layer = 0;
  cur.in = shapes[0];
  bool open = false;
  auto close = [&](int last) {
    cur.last_layer = last;
    steps.push_back(cur);
    cur = Step();
  };
  for (int i = 0; i < n; ++i) {
    const bs_layer_desc& d = L[i];
    if (!open) {
      cur.first_layer = i;
      cur.in = shapes[i];
      open = true;
    }
    if (is_pool(d.kind)) {
      if (cur.has_pool) {
        close(i - 1);
        cur.first_layer = i;
        cur.in = shapes[i];
      }
      cur.has_pool = true;
      cur.pool_layer = i;
      cur.kh = d.kernel_h; cur.kw = d.kernel_w;
      cur.sh = d.stride_h; cur.sw = d.stride_w;
      cur.ph = d.pad_h;    cur.pw = d.pad_w;
      cur.is_max = d.kind == BS_OP_MAXPOOL;
      cur.cip = d.count_include_pad ? 1 : 0;
      continue;
    }
    if (d.kind == BS_OP_COPY) continue;  // identity (eval Dropout): elided
    HostOp op;
    if (d.kind == BS_OP_BATCHNORM) {
      op = fold_bn(d, i, shapes[i].c);
    } else {
      op.layer = i;
      op.kind = d.kind == BS_OP_RELU ? DOP_RELU : d.kind == BS_OP_SCALE ? DOP_SCALE : DOP_ADD;
      op.alpha = d.alpha;
      op.operand = d.operand;
    }
    std::vector<HostOp>& dst = cur.has_pool ? cur.epi : cur.pro;
    if ((int)dst.size() == kMaxOps) {   // program full: serialise into a new step
      close(i - 1);
      cur.first_layer = i;
      cur.in = shapes[i];
      open = true;
      cur.pro.push_back(op);
      continue;
    }
    dst.push_back(op);
  }
  if (open) close(n - 1);
  for (Step& s : steps) s.out = shapes[s.last_layer + 1];
}

bool monotone(const HostOp& op) { return op.kind == DOP_AFFINE || op.kind == DOP_RELU || op.kind == DOP_SCALE; }

int32_t prog_class(const std::vector<HostOp>& ops) {
  if (ops.empty()) return PC_NONE;
  if (ops.size() == 1 && ops[0].kind == DOP_RELU) return PC_RELU;
  if (ops.size() == 1 && ops[0].kind == DOP_AFFINE) return PC_AFFINE;
  if (ops.size() == 2 && ops[0].kind == DOP_AFFINE && ops[1].kind == DOP_RELU) return PC_AFFINE_RELU;
  return PC_GENERIC;
}

// A max pool's prologue can run after the pool when every op is monotone (bit-exact,
// bs_kernels.cu header; R5) and the merged program fits.
bool max_deferrable(const Step& s) {
  if (!s.has_pool || !s.is_max) return false;
  bool ok = s.pro.size() + s.epi.size() <= (size_t)kMaxOps;
  for (const HostOp& op : s.pro) ok = ok && monotone(op);
  return ok;
}

// Decide the programs the kernel runs.
void set_device_programs(Launch& l) {
  const Step& s = l.step;
  l.dev_pro = s.pro;
  l.dev_epi = s.epi;
  l.deferred = false;
  if (l.kernel == K_EW || l.kernel == K_POOL_NAIVE || l.kernel == K_POOL_PLANES || !max_deferrable(s)) return;
  l.dev_epi = s.pro;
  l.dev_epi.insert(l.dev_epi.end(), s.epi.begin(), s.epi.end());
  l.dev_pro.clear();
  l.deferred = true;
}

// Staged-kernel tile (k_pool_staged.cu): P whole planes per tile and bands of R output rows,
// chosen so that the 8 consumer warps share every tile evenly.  A tile holds I =
// ceil(P/G) * n_cc * ceil(Ho/R) items and each warp walks ceil(I/8) of them in turn, each item
// reducing R*s + (k-s) input rows; the choice minimises that per-tile walk per staged plane,
// (I <= 16 where possible: a warp's two items are then decoded once per CTA; wider planes take
// more items per warp), with a mild preference for 12-32 KB tiles (small enough for >= 3 ring stages at two CTAs per
// SM and for the last tile of a CTA's range to be cheap; large enough to amortise the per-tile
// barrier work).  Ring depth: as many stages as fit two CTAs per SM (<= 8).  False if one
// plane group is too large to stage.
constexpr int64_t kStagedTileMax = 32 * 1024;
// Dynamic shared memory a plan may use per CTA (bs_plan_options.smem_budget_bytes).
int64_t smem_cap(const bs_plan_options& o) {
  return o.smem_budget_bytes > 0 ? std::min<int64_t>(o.smem_budget_bytes, 220 * 1024) : 220 * 1024;
}

bool size_stages(Launch& l, int64_t n_planes, const bs_plan_options& o, int num_sms) {
  const Step& st = l.step;
  const int64_t HW = st.in.h * st.in.w, Ho = st.out.h;
  const int64_t plane_bytes = HW * 4;
  const int64_t G = l.G, ncc = l.n_cc, NC = kStagedConsumerWarps;
  const int64_t carry = std::max(0, st.kh - st.sh);
  const int64_t max_groups = (n_planes + G - 1) / G;
  double best = 1e300;
  int64_t bP = G, bR = Ho;
  // first pass: tiles of <= 16 items (a warp's two items decoded once per CTA); if none exists
  // (planes wider than 16 column chunks, or a forced narrow column group) any item count
  for (int pass = 0; pass < 2 && best == 1e300; ++pass)
  for (int64_t m = 1; m <= max_groups && (m == 1 || m * G * plane_bytes <= kStagedTileMax); ++m) {
    if (o.force_tile_planes > 0 && m != std::max<int64_t>(1, o.force_tile_planes / G)) continue;
    for (int64_t R = 1; R <= Ho; ++R) {
      const int64_t nrb = (Ho + R - 1) / R;
      if (R > 1 && (Ho + R - 2) / (R - 1) == nrb) continue;     // same band count as R-1
      if (o.force_rows_per_task > 0 && R != std::min<int64_t>(Ho, o.force_rows_per_task)) continue;
      const int64_t I = m * ncc * nrb;
      if (pass == 0 && I > 2 * NC) continue;                     // <= 2 items per warp
      const double walk = (double)((I + NC - 1) / NC) * (double)(R * st.sh + carry);
      const int64_t T = m * G * plane_bytes;
      const double size_f = T < 8192 ? 1.25 : T < 12288 ? 1.05 : T > kStagedTileMax ? 1.1 : 1.0;
      // few tiles per CTA (small tensors): the first tile's arrival and the last tile's walk are
      // exposed, so favour smaller tiles there (AlexNet s3: 40 -> 20 planes, 6.61 -> 6.37 us)
      const double tiles_per_cta = (double)n_planes / (double)(m * G) / (2.0 * std::max(1, num_sms));
      const double tail_f = tiles_per_cta < 6.0 ? 1.0 + 0.05 * (6.0 - tiles_per_cta) : 1.0;
      const double cost = walk / (double)(m * G) * size_f * tail_f;
      if (cost < best * (1 - 1e-9)) { best = cost; bP = m * G; bR = R; }
    }
  }
  const bool read_dominated = 8 * st.out.h * st.out.w < HW;   // global averages
  const int64_t stride = (int64_t)pool_staged_stride((int)bP, (int)HW);
  if (stride > 100 * 1024) return false;   // plane group too large to stage
  l.tile_planes = (int32_t)bP;
  l.rows_per_task = (int32_t)bR;
  l.n_rb = (int32_t)((Ho + bR - 1) / bR);
  // Ring depth: ~104 KB of tiles in flight per SM.  Measured on B200 (AlexNet stacks, CTAs/SM x
  // stages swept): more bytes in flight is *slower* (2 CTAs x 4 x 24 KB: 22.5 us; 1 CTA x 4-5 x
  // 24 KB: 20.5 us on s1), so one CTA per SM for tiles >= 20 KB when each SM has >= 12 tiles,
  // two (more consumer warps per byte) otherwise (s3, 13.5 KB tiles: 2 x 4 stages 6.1 us vs
  // 1 x 7 stages 6.5 us; DenseNet final, 31 KB tiles, 11 per SM: 2 CTAs).
  // (read-dominated pools -- global averages, output < 1/8 of the input -- gain from twice that:
  // DenseNet-121 final 7x7 average, 2 x 3 x 31 KB: 10.7 us vs 11.6 us at 2 x 2)
  const int64_t kInflightPerSm = read_dominated ? 208 * 1024 : 104 * 1024;
  const int64_t tiles_per_sm = (n_planes + bP - 1) / bP / std::max(1, num_sms);
  // one CTA per SM only for big tiles, long kernels and pools that shrink the plane (stride >= 2:
  // few outputs per staged byte); stride-1 pools (the §5.1 block: one output per input) need the
  // second CTA's consumer warps (41 vs 47 us per block measured)
  const bool shrinks = 2 * st.out.h * st.out.w <= HW;
  // (averages with a per-element prologue have a heavier consumer: they keep the second CTA)
  const bool heavy = !st.is_max && !st.pro.empty();
  l.ctas_per_sm = (stride >= 20 * 1024 && tiles_per_sm >= 12 && shrinks && !read_dominated && !heavy) ? 1 : 2;
  l.stages = (int32_t)std::max<int64_t>(2, std::min<int64_t>(kStagedMaxStages,
                                                            (kInflightPerSm / l.ctas_per_sm + stride / 2) / stride));
  if (o.force_stages >= 2) l.stages = std::min(kStagedMaxStages, o.force_stages);
  const int64_t cap = smem_cap(o) - kStagedHeader;
  if ((int64_t)l.stages * stride > cap) l.stages = (int32_t)(cap / stride);
  if (l.stages < 2) return false;
  l.U = 1;
  return true;
}

// Column-walker geometry of the global-memory scalar walker (kernel 2).
void set_spec_geometry(Launch& l, int force_opg) {
  const Step& s = l.step;
  l.kernel = K_POOL_SPEC;
  int Jg = (int)std::min<int64_t>((32 - s.kw) / s.sw + 1, s.out.w);
  if (force_opg > 0) Jg = std::min(Jg, force_opg);
  const int ncc = (int)((s.out.w + Jg - 1) / Jg);
  l.Jg = (int)((s.out.w + ncc - 1) / ncc);
  l.n_cc = ncc;
  l.gw = (l.Jg - 1) * s.sw + s.kw;
  l.G = 32 / l.gw;
  l.U = pool_spec_unroll(s.kh, s.sh);
  l.rows_per_task = (int32_t)s.out.h;
  l.n_rb = 1;
}

// ---------------------------------------------------------------- a4: sequences + tiles
// Sequence packing: this build executes one step per sequence
// (multi-step on-chip sequences are NEXT-2 in SURVEY §8(f)); consecutive sequences are
// serialised through plan-owned intermediates.  Tile geometry per step:
//   element-wise step : flat 128-bit streaming, no tile.
//   pool step         : a warp task = G lane groups (one plane each) x Jg output columns x
//                       rows_per_task output rows.  The on-chip footprint of a task is the
//                       ((U-1)*s + k) x gw register window per warp -- the B200 analogue of
//                       the paper's "data per step x SIMD units".
// Kernel and tile geometry of a single-step launch.
void configure_step_launch(bs_plan* p, Launch& l, const bs_plan_options& o) {
    const Step& s = l.step;
    if (!s.has_pool) {
      l.kernel = K_EW;
    } else {
      const int64_t Wo = s.out.w, Ho = s.out.h;
      const bool per_elem_max = s.is_max && !s.pro.empty() && !max_deferrable(s);
      const int vec = pool_vec_width(s.kh, s.kw, s.sh, s.sw, s.ph, s.pw, (int)s.in.w, (int)Wo);
      if (o.force_generic == 0 && pool_planes_applies((int)s.in.h, (int)s.in.w, s.kh, s.kw, s.ph, s.pw)) {
        // window = the whole (small) plane: a warp reduces 32 planes (k_pool_planes.cu)
        l.kernel = K_POOL_PLANES;
        l.G = 32; l.Jg = 1; l.n_cc = 1; l.gw = 1; l.U = 1;
        l.rows_per_task = 1;
        l.n_rb = 1;
      } else if (s.kw > 32) {
        l.kernel = K_POOL_NAIVE;
      } else if (vec && o.force_generic == 0 && !per_elem_max &&
                 !(!s.is_max && !s.pro.empty() && s.in.w <= 28)) {
        // (averages with a per-element prologue on planes <= 28 wide stage better: DenseNet-121
        // transitions 28x28 88.2 -> 82.5 us, 14x14 49.1 -> 45.4 us measured)
        // vector column walker: each lane VEC columns, VEC/2 outputs; halo lane for 3-wide windows
        l.kernel = K_POOL_VEC;
        const int opl = vec / 2, halo = s.kw == 3 ? 1 : 0;
        int Jg = opl * (32 - halo);
        if (o.force_outputs_per_group > 0) Jg = std::max(opl, std::min(Jg, o.force_outputs_per_group / opl * opl));
        const int64_t need = (Wo + opl - 1) / opl * opl;
        if (need <= Jg) Jg = (int)need;
        l.Jg = Jg;
        l.n_cc = (int)((Wo + Jg - 1) / Jg);
        l.gw = Jg / opl + halo;
        l.G = 32 / l.gw;
        l.U = pool_vec_unroll(vec);
      } else {
        l.kernel = (o.force_generic != 1 && !per_elem_max && pool_has_specialisation(s.kh, s.kw, s.sh, s.sw))
                       ? K_POOL_SPEC : K_POOL_GENERIC;
        if (l.kernel == K_POOL_SPEC && o.force_generic != 2) {
          // staged: one lane per output column (output-stationary), G planes per warp
          l.kernel = K_POOL_STAGED;  // tile sized below
          int J = (int)std::min<int64_t>(32, Wo);
          if (o.force_outputs_per_group > 0) J = std::min(J, o.force_outputs_per_group);
          const int ncc = (int)((Wo + J - 1) / J);
          J = (int)((Wo + ncc - 1) / ncc);
          l.Jg = J; l.n_cc = ncc; l.gw = J; l.G = 32 / J;
          l.U = 1;
        } else {
          int jmax = (32 - s.kw) / s.sw + 1;
          int Jg = (int)std::min<int64_t>(jmax, Wo);
          if (o.force_outputs_per_group > 0) Jg = std::min(Jg, o.force_outputs_per_group);
          // balance chunks: same number of chunks, as even as possible
          const int n_cc = (int)((Wo + Jg - 1) / Jg);
          Jg = (int)((Wo + n_cc - 1) / n_cc);
          l.Jg = Jg;
          l.n_cc = n_cc;
          l.gw = (Jg - 1) * s.sw + s.kw;
          l.G = 32 / l.gw;
          l.U = l.kernel == K_POOL_SPEC ? pool_spec_unroll(s.kh, s.sh) : 1;
        }
      }
      (void)Ho;
    }
    if (l.kernel == K_POOL_STAGED && !size_stages(l, s.in.n * s.in.c, o, p->num_sms))
      set_spec_geometry(l, o.force_outputs_per_group);   // plane too large to stage
    set_device_programs(l);
    if (l.kernel == K_POOL_GENERIC) l.U = 1;
}

bool has_add(const Step& s) {
  for (auto* v : {&s.pro, &s.epi})
    for (const HostOp& op : *v)
      if (op.kind == DOP_ADD) return true;
  return false;
}

// ---------------------------------------------------------------- a4: on-chip sequences
// Geometry of an on-chip sequence over steps [a, b) (NEXT-2; k_seq.cu): P planes per tile and
// bands of R output rows of the last step (R = Ho: whole planes).  For every band the rows of
// every step are back-propagated through the windows (in_lo = out_lo*s - p,
// in_hi = (out_hi-1)*s + k - p, clipped to the plane): a step computes the rows the next step
// needs, so a band's input grows by the window overlap of every step -- the paper's redundant
// halo work.  Shared memory = ring stages of step 0's input rows + one work buffer:
// a tile's steps ping-pong between its stage and the work buffer (the paper's "two buffers",
// P:L613-615), so the stage is held until the tile's last step.
struct SeqGeom {
  int64_t P = 1, R = 0, n_bands = 1, stages = 2;
  int64_t stage_bytes = 0, work_floats = 0, smem = 0;
  std::vector<int32_t> in_pitch, out_pitch;
  std::vector<SeqRange> ranges;
};

bool is_fast_step(const Step& st) {
  return st.has_pool && st.is_max && st.kh == 3 && st.kw == 3 && st.sh == 1 && st.sw == 1 && st.ph == 1 &&
         st.pw == 1 && st.pro.empty() && prog_class(st.epi) != PC_GENERIC && st.in.w % 4 == 0 && st.in.w <= 256;
}

// Rows of every step of [a, b) for the last step's output rows [o_lo, o_hi).
void band_rows(const std::vector<Step>& st, size_t a, size_t b, int64_t o_lo, int64_t o_hi, SeqRange* out) {
  for (size_t k = b; k-- > a;) {
    const Step& s = st[k];
    SeqRange& r = out[k - a];
    std::memset(&r, 0, sizeof r);
    r.out_lo = (int32_t)o_lo;
    r.out_hi = (int32_t)o_hi;
    int64_t lo = o_lo, hi = o_hi;
    if (s.has_pool) {
      lo = std::max<int64_t>(0, o_lo * s.sh - s.ph);
      hi = std::min<int64_t>(s.in.h, (o_hi - 1) * s.sh - s.ph + s.kh);
    }
    r.in_lo = (int32_t)lo;
    r.in_hi = (int32_t)hi;
    o_lo = lo;
    o_hi = hi;
  }
}

// Fill g for P planes per tile, R output rows per band, S stages; returns the dynamic smem bytes.
int64_t seq_geometry(const std::vector<Step>& st, size_t a, size_t b, int64_t P, int64_t R, int64_t S, SeqGeom& g) {
  const size_t n = b - a;
  const Step& last = st[b - 1];
  const int64_t Ho = last.out.h;
  R = std::max<int64_t>(1, std::min(R, Ho));
  g.P = P;
  g.R = R;
  g.stages = S;
  g.n_bands = (Ho + R - 1) / R;
  g.ranges.assign((size_t)g.n_bands * n, SeqRange());
  for (int64_t bd = 0; bd < g.n_bands; ++bd)
    band_rows(st, a, b, bd * R, std::min(Ho, (bd + 1) * R), &g.ranges[(size_t)bd * n]);
  std::vector<int64_t> rows_in(n, 0), rows_out(n, 0);
  for (const SeqRange& r : g.ranges) {
    const size_t k = (size_t)(&r - g.ranges.data()) % n;
    rows_in[k] = std::max<int64_t>(rows_in[k], r.in_hi - r.in_lo);
    rows_out[k] = std::max<int64_t>(rows_out[k], r.out_hi - r.out_lo);
  }
  // steps ping-pong between the tile's stage and ONE work buffer (k_seq.cu): even steps write the
  // work buffer, odd steps the stage, which must also hold those intermediates
  const int64_t W0 = st[a].in.w;
  int64_t stage = P * rows_in[0] * W0 * 4 + 16;
  g.in_pitch.assign(n, 0);
  g.out_pitch.assign(n, 0);
  g.in_pitch[0] = (int32_t)(g.n_bands == 1 ? st[a].in.h * W0 : rows_in[0] * W0);
  int64_t wf = 0;
  for (size_t k = 0; k + 1 < n; ++k) {
    const int64_t pitch = (rows_out[k] * st[a + k].out.w + 3) / 4 * 4;
    g.out_pitch[k] = (int32_t)pitch;
    g.in_pitch[k + 1] = (int32_t)pitch;
    if (k % 2 == 0) wf = std::max(wf, P * pitch);
    else stage = std::max(stage, P * pitch * 4);
  }
  g.stage_bytes = (stage + 127) / 128 * 128;
  g.work_floats = wf;
  // + per-tile tables (k_seq.cu seq_table_bytes): ranges of every step, (scale, shift) per (step, plane)
  const int64_t tables = ((int64_t)n * (int64_t)sizeof(SeqRange) + (int64_t)n * P * 8 + 127) / 128 * 128;
  g.smem = 128 + S * g.stage_bytes + wf * 4 + tables + 1024;
  return g.smem;
}

// Fast-path chunking of each (band, step): enough (plane, row chunk, column segment) items for
// the 8 consumer warps, chunks of >= 4 rows (each chunk re-reads two halo rows of its input).
void seq_chunking(const std::vector<Step>& st, size_t a, size_t b, SeqGeom& g) {
  const size_t n = b - a;
  for (size_t idx = 0; idx < g.ranges.size(); ++idx) {
    SeqRange& r = g.ranges[idx];
    const Step& s = st[a + idx % n];
    const int64_t nrows = std::max<int64_t>(1, r.out_hi - r.out_lo);
    int64_t nch = 1;
    if (is_fast_step(s)) {
      const int64_t seg = s.in.w <= 64 ? 16 : 32, nseg = (s.in.w + 4 * seg - 1) / (4 * seg);
      const int64_t want_half = (int64_t)kSeqWarps * (32 / seg);
      nch = std::max<int64_t>(1, std::min<int64_t>((want_half + g.P * nseg - 1) / (g.P * nseg), nrows / 4));
    }
    const int64_t L = (nrows + nch - 1) / nch;
    nch = (nrows + L - 1) / L;
    r.n_chunks = (int32_t)nch;
    r.L = (int32_t)L;
    r.chunks = make_fastdiv((uint32_t)nch);
  }
}

// Dynamic shared memory a sequence may use per CTA: whole-plane tiles may take the plan's cap
// (one CTA per SM); halo tiles are planned against the paper's cache budget -- by default half
// the SM (two CTAs per SM), or bs_plan_options.smem_budget_bytes.
int64_t seq_band_cap(const bs_plan_options& o) {
  return o.smem_budget_bytes > 0 ? smem_cap(o) : std::min<int64_t>(110 * 1024, smem_cap(o));
}
// Base halo tile (the paper's "one output value per SIMD unit"): the fewest rows of the
// last step's output that give each of the 256 consumer lanes an output.
int64_t seq_base_rows(const Step& last) { return std::max<int64_t>(1, (256 + last.out.w - 1) / last.out.w); }

// Dynamic smem of the in-place kernel for [a, b), or -1 if it does not apply / fit.
int64_t inplace_smem(const std::vector<Step>& steps, size_t a, size_t b, const bs_plan_options& o,
                     int64_t* stage_out = nullptr, int64_t* stages_out = nullptr, int64_t* planes_out = nullptr) {
  if (o.force_tile_planes > 0 || o.force_rows_per_task > 0 || b - a > (size_t)kMaxSeqSteps) return -1;
  const int64_t W = steps[a].in.w, H = steps[a].in.h;
  if (W > 224) return -1;
  for (size_t k = a; k < b; ++k)
    if (!is_fast_step(steps[k]) || steps[k].in.w != W || steps[k].in.h != H) return -1;
  // planes 129..224 wide: one plane per CTA, 8 warps each owning ~H / 8 rows of both column
  // segments of the row (k_seq.cu seq_inplace<32, 1, 2, false>); parts of >= 2 rows
  const bool wide = W > 128;
  if (wide && H < 16) return -1;
  const int64_t warps = wide ? 8 : kInplaceWarps;
  // planes per CTA: warps per plane chosen so that ~4 CTAs (16 consumer warps) fit an SM: small
  // planes one warp each, 112 x 112 planes four warps each
  int64_t P = wide ? 1 : kInplaceWarps;
  while (P > 1 && 4 * (P * H * W * 4 + 2048) > 220 * 1024) P /= 2;
  const int64_t stage = (P * H * W * 4 + 16 + 127) / 128 * 128;
  const int64_t S = wide ? 1 : o.force_stages >= 1 ? std::min<int64_t>(kStagedMaxStages, o.force_stages) : 1;
  const int64_t smem = 128 + S * stage + warps * (int64_t)(b - a) * 8 + 1024;
  if (stage_out) *stage_out = stage;
  if (stages_out) *stages_out = S;
  if (planes_out) *planes_out = P;
  return smem <= smem_cap(o) ? smem : -1;
}

// a4 sequence packing: greedily add the next step while the sequence's
// tile still fits the shared-memory budget -- whole planes, else a halo band of the base tile
// size whose input grows with every added padded step -- and the policy's step limit allows it.
// A step with an ADD operand (per-execute pointers) is kept in a sequence of its own.
// The planner's default policy (max_steps_per_sequence = 0) bounds the halo redundancy on top of
// that: a halo-tiled sequence takes another step only while the largest band that fits still
// covers at least as many output rows as its step-0 input halo (halo rows <= band rows, i.e. at
// most 2x the input rows and ~1.5x the step work).  The paper's "unrestricted" strategy
// (max_steps_per_sequence = -1) packs while anything fits: its redundant work grows with every
// padded step until the next sequence starts.
bool seq_fits(const std::vector<Step>& st, size_t a, size_t b, const bs_plan_options& o) {
  if (b - a > (size_t)kMaxSeqSteps) return false;
  for (size_t k = a; k < b; ++k)
    if (has_add(st[k])) return false;
  if (inplace_smem(st, a, b, o) >= 0) return true;   // whole planes, in place (k_seq.cu seq_inplace)
  SeqGeom g;
  if (o.force_rows_per_task <= 0 && seq_geometry(st, a, b, 1, st[b - 1].out.h, 2, g) <= smem_cap(o)) return true;
  const int64_t cap = seq_band_cap(o);
  const int64_t R0 = o.force_rows_per_task > 0 ? o.force_rows_per_task : seq_base_rows(st[b - 1]);
  if (seq_geometry(st, a, b, 1, R0, 2, g) > cap) return false;
  if (o.max_steps_per_sequence != 0 || o.force_rows_per_task > 0) return true;
  // default policy: the largest fitting band must cover its own step-0 halo
  const int64_t Ho = st[b - 1].out.h;
  int64_t lo = R0, hi = Ho;   // largest R in [R0, Ho] that fits (footprint grows with R)
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (seq_geometry(st, a, b, 1, mid, 2, g) <= cap) lo = mid;
    else hi = mid - 1;
  }
  seq_geometry(st, a, b, 1, lo, 2, g);
  int64_t halo = 0;
  const size_t n = b - a;
  for (int64_t bd = 0; bd < g.n_bands; ++bd) {   // step-0 input rows beyond the band's own share
    const SeqRange& r0 = g.ranges[(size_t)bd * n];
    const SeqRange& rl = g.ranges[(size_t)bd * n + n - 1];
    const int64_t own = (st[a].in.h * (int64_t)(rl.out_hi - rl.out_lo) + Ho - 1) / Ho;
    halo = std::max<int64_t>(halo, (r0.in_hi - r0.in_lo) - own);
  }
  return halo <= lo;
}

// The warp-per-plane in-place kernel (k_seq.cu seq_inplace) takes sequences made only of fast
// steps on whole planes of W <= 128: each consumer warp owns one plane for the whole sequence (no
// CTA barrier, no work buffer); one stage per CTA by default, so several CTAs share an SM.
bool plan_inplace(const std::vector<Step>& steps, size_t a, size_t b, const bs_plan_options& o, Launch& l) {
  int64_t stage = 0, S = 0, P = 0;
  if (inplace_smem(steps, a, b, o, &stage, &S, &P) < 0) return false;
  const int64_t W = steps[a].in.w, H = steps[a].in.h;
  const int seg = W <= 64 ? 16 : 32;
  l.seq_inplace_seg = seg;
  l.tile_planes = (int32_t)P;
  l.stages = (int32_t)S;
  l.seq_stage_bytes = (int32_t)stage;
  l.seq_work_floats = 0;
  l.seq_bands = 1;
  l.seq_band_rows = (int32_t)H;
  SeqGeom g;   // whole-plane ranges (unused by the kernel; kept for the launch info)
  seq_geometry(steps, a, b, 1, H, 2, g);
  l.seq_in_pitch = g.in_pitch;
  l.seq_out_pitch = g.out_pitch;
  l.seq_ranges = g.ranges;
  return true;
}

void plan_sequence(const bs_plan* p, const std::vector<Step>& steps, size_t a, size_t b, const bs_plan_options& o,
                   Launch& l) {
  const int64_t n_planes = steps[a].in.n * steps[a].in.c;
  const int64_t Ho = steps[b - 1].out.h;
  if (plan_inplace(steps, a, b, o, l)) return;
  SeqGeom g;
  if (o.force_rows_per_task <= 0 && seq_geometry(steps, a, b, 1, Ho, 2, g) <= smem_cap(o)) {
    // whole planes: the most planes per tile that keep two CTAs per SM (else one), >= 8 tiles
    // per CTA; up to 4 stages
    int64_t P = 1;
    const int64_t half = std::min<int64_t>(110 * 1024, smem_cap(o));
    SeqGeom t;
    while (P * 2 <= n_planes / (8 * 2 * p->num_sms) && seq_geometry(steps, a, b, P * 2, Ho, 2, t) <= half) P *= 2;
    if (o.force_tile_planes > 0) P = o.force_tile_planes;
    int64_t S = 2;
    while (S < 4 && seq_geometry(steps, a, b, P, Ho, S + 1, t) <= half) ++S;
    if (seq_geometry(steps, a, b, P, Ho, S, g) > smem_cap(o)) {
      P = 1;
      S = 2;
      seq_geometry(steps, a, b, P, Ho, S, g);
    }
  } else {
    // halo tiles of one plane: the largest band that fits the budget ("we increase the size of
    // it"), or the forced band
    const int64_t cap = seq_band_cap(o);
    int64_t R = o.force_rows_per_task > 0 ? o.force_rows_per_task : seq_base_rows(steps[b - 1]);
    if (o.force_rows_per_task <= 0)
      {   // largest R in [R, Ho] that fits (the footprint grows with R)
      int64_t lo = R, hi = Ho;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (seq_geometry(steps, a, b, 1, mid, 2, g) <= cap) lo = mid;
        else hi = mid - 1;
      }
      R = lo;
    }
    seq_geometry(steps, a, b, 1, R, 2, g);
    SeqGeom t;
    if (seq_geometry(steps, a, b, 1, R, 3, t) <= cap) g = t;
  }
  seq_chunking(steps, a, b, g);
  l.tile_planes = (int32_t)g.P;
  l.stages = (int32_t)g.stages;
  l.seq_work_floats = (int32_t)g.work_floats;
  l.seq_bands = (int32_t)g.n_bands;
  l.seq_band_rows = (int32_t)g.R;
  l.seq_stage_bytes = (int32_t)g.stage_bytes;
  l.seq_in_pitch = g.in_pitch;
  l.seq_out_pitch = g.out_pitch;
  l.seq_ranges = g.ranges;
  // Halo tiles of §5.1-type sequences run in place (k_seq.cu seq_inplace, band tiles): the same
  // bands and split points as the shared-tile kernel (the paper's footprint rule, R14/R15), but a
  // band is swept in place with two steps per sweep -- its stage alone, no work buffer.  Planner-
  // chosen bands only (forced bands keep testing seq_staged), whole-warp row parts (W > 56) of
  // >= 2 rows each.
  const int64_t W = steps[a].in.w;
  bool band_inplace = g.n_bands > 1 && o.force_rows_per_task <= 0 && o.force_tile_planes <= 0 && W > 56 && W <= 224;
  for (size_t k = a; k < b && band_inplace; ++k) band_inplace = is_fast_step(steps[k]) && steps[k].in.w == W;
  if (band_inplace) {
    const int64_t parts = W > 128 ? 8 : kInplaceWarps;
    // the in-place footprint is the band alone (2 stages, no work buffer): the tallest band whose
    // two stages fit the budget, then balanced (no short last band); the seq_staged geometry in
    // `l` stays untouched unless every band qualifies
    int64_t halo = 0;   // input rows beyond a band's output rows (both sides, interior band)
    for (size_t k = a; k < b; ++k) halo += 2 * steps[k].ph;
    const int64_t cap_rows = (seq_band_cap(o) - 4096 - (int64_t)(b - a) * 8 * 8) / (2 * (W * 4 + 1));
    const int64_t Rmax = std::max<int64_t>(g.R, std::min<int64_t>(Ho, cap_rows - halo));
    const int64_t nb = (Ho + Rmax - 1) / Rmax, Rb = (Ho + nb - 1) / nb;
    SeqGeom gb = g;
    if (Rb != g.R) {
      seq_geometry(steps, a, b, 1, Rb, 2, gb);
      seq_chunking(steps, a, b, gb);
    }
    int64_t max_rows = 0;
    for (int64_t bd = 0; bd < gb.n_bands; ++bd) {
      const SeqRange& r0 = gb.ranges[(size_t)bd * (b - a)];
      band_inplace = band_inplace && r0.in_hi - r0.in_lo >= 2 * parts;
      max_rows = std::max<int64_t>(max_rows, r0.in_hi - r0.in_lo);
    }
    if (band_inplace) {
      l.seq_bands = (int32_t)gb.n_bands;
      l.seq_band_rows = (int32_t)gb.R;
      l.seq_in_pitch = gb.in_pitch;
      l.seq_out_pitch = gb.out_pitch;
      l.seq_ranges = gb.ranges;
      l.seq_inplace_seg = 32;
      l.tile_planes = 1;
      l.seq_work_floats = 0;
      l.seq_stage_bytes = (int32_t)((max_rows * W * 4 + 16 + 127) / 128 * 128);
      // two stages when they fit the budget: band tiles are short, and the two-segment kernel runs
      // one CTA per SM (registers), so the next band's copy must overlap this band's sweeps
      l.stages = 2 * (int64_t)l.seq_stage_bytes + 4096 <= seq_band_cap(o) ? 2 : 1;
    }
  }
}

void pack_and_tile(bs_plan* p, std::vector<Step>& steps, const bs_plan_options& o) {
  p->launches.clear();
  size_t max_steps = o.max_steps_per_sequence <= 0 ? (size_t)kMaxSeqSteps
                                                   : std::min<size_t>(kMaxSeqSteps, o.max_steps_per_sequence);
  std::vector<std::pair<size_t, size_t>> seqs;
  for (size_t a = 0; a < steps.size();) {
    size_t b = a + 1;
    while (b < steps.size() && b - a < max_steps && seq_fits(steps, a, b + 1, o)) ++b;
    seqs.emplace_back(a, b);
    a = b;
  }
  int inter_idx = 0;
  for (size_t k = 0; k < seqs.size(); ++k) {
    const size_t a = seqs[k].first, b = seqs[k].second;
    Launch l;
    l.src = k == 0 ? -1 : (int)((inter_idx + 1) % 2);
    l.dst = k + 1 == seqs.size() ? -1 : inter_idx;
    if (k + 1 < seqs.size()) inter_idx = (inter_idx + 1) % 2;
    if (b - a == 1) {
      l.step = steps[a];
      configure_step_launch(p, l, o);
    } else {
      l.kernel = K_SEQ;
      l.seq.assign(steps.begin() + a, steps.begin() + b);
      l.step = Step();
      l.step.first_layer = steps[a].first_layer;
      l.step.last_layer = steps[b - 1].last_layer;
      l.step.in = steps[a].in;
      l.step.out = steps[b - 1].out;
      l.step.has_pool = true;
      l.step.kh = steps[a].kh; l.step.kw = steps[a].kw; l.step.sh = steps[a].sh;
      l.step.sw = steps[a].sw; l.step.ph = steps[a].ph; l.step.pw = steps[a].pw;
      plan_sequence(p, steps, a, b, o, l);
    }
    p->launches.push_back(l);
  }
}

// Row banding: enough warp tasks to fill the device several times over, bands a
// multiple of U rows, halo re-read (k - s rows per band) kept under 1/8 of a band.
void size_rows(const bs_plan* p, Launch& l, const bs_plan_options& o, int64_t n_planes) {
  const Step& s = l.step;
  const int64_t Ho = s.out.h;
  const int64_t base_tasks = ((n_planes + l.G - 1) / l.G) * l.n_cc;
  const int64_t resident_warps = (int64_t)p->num_sms * std::max(1, l.blocks_per_sm) * (l.block / 32);
  int64_t rows = Ho;
  if (o.force_rows_per_task > 0) {
    rows = std::min<int64_t>(Ho, o.force_rows_per_task);
  } else if (base_tasks < 8 * resident_warps) {
    const int64_t want_rb = (8 * resident_warps + base_tasks - 1) / base_tasks;
    rows = (Ho + want_rb - 1) / want_rb;
    const int halo = std::max(0, s.kh - s.sh);
    const int64_t min_rows = halo > 0 ? (8 * halo + s.sh - 1) / s.sh : 1;
    rows = std::max<int64_t>(rows, std::max<int64_t>(min_rows, l.U));
    rows = (rows + l.U - 1) / l.U * l.U;
    rows = std::min<int64_t>(rows, Ho);
  }
  l.rows_per_task = (int32_t)std::max<int64_t>(1, rows);
  l.n_rb = (int32_t)((Ho + l.rows_per_task - 1) / l.rows_per_task);
}

OpProgram make_prog(const bs_plan* p, const std::vector<HostOp>& ops, int n_deferred = 0) {
  OpProgram P;
  std::memset(&P, 0, sizeof P);
  P.n = (int32_t)ops.size();
  P.n_deferred = n_deferred;
  int aff = 0, add = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    P.kind[i] = ops[i].kind;
    P.alpha[i] = ops[i].alpha;
    P.affine[i] = ops[i].kind == DOP_AFFINE && p->params ? p->params + ops[i].affine_off : nullptr;
    P.aff_slot[i] = (ops[i].kind == DOP_AFFINE && aff < kAffSlots) ? aff++ : -1;
    P.add_slot[i] = (ops[i].kind == DOP_ADD && add == 0) ? add++ : -1;
  }
  for (size_t i = ops.size(); i < (size_t)kMaxOps; ++i) {
    P.aff_slot[i] = -1;
    P.add_slot[i] = -1;
  }
  return P;
}

void fill_operands(OpProgram& P, const std::vector<HostOp>& ops, const float* const* inputs) {
  for (size_t i = 0; i < ops.size(); ++i)
    if (ops[i].kind == DOP_ADD) P.operand[i] = inputs[ops[i].operand];
}

PoolArgs make_pool_args(const bs_plan* p, const Launch& l) {
  PoolArgs a;
  std::memset(&a, 0, sizeof a);
  const Step& s = l.step;
  a.C = (int32_t)s.in.c;
  a.H = (int32_t)s.in.h;
  a.W = (int32_t)s.in.w;
  a.Ho = (int32_t)s.out.h;
  a.Wo = (int32_t)s.out.w;
  a.kh = s.kh; a.kw = s.kw; a.sh = s.sh; a.sw = s.sw; a.ph = s.ph; a.pw = s.pw;
  a.is_max = s.is_max;
  a.count_include_pad = s.cip;
  a.G = l.G; a.gw = l.gw; a.Jg = l.Jg; a.n_cc = l.n_cc;
  a.rows_per_task = l.rows_per_task; a.n_rb = l.n_rb;
  a.pro = make_prog(p, l.dev_pro);
  a.epi = make_prog(p, l.dev_epi, l.deferred ? (int)s.pro.size() : 0);
  a.pro_class = prog_class(l.dev_pro);
  a.epi_class = prog_class(l.dev_epi);
  a.tile_planes = l.tile_planes;
  a.stages = l.stages;
  a.cdiv = make_fastdiv((uint32_t)a.C);
  return a;
}

int64_t pool_tasks(const Launch& l, int64_t n_planes) {
  if (l.kernel == K_POOL_NAIVE) return n_planes * l.step.out.h * l.step.out.w;
  if (l.kernel == K_POOL_STAGED) return (n_planes + l.tile_planes - 1) / l.tile_planes;   // tiles
  if (l.kernel == K_POOL_PLANES) return (n_planes + 31) / 32;                              // warp chunks
  return ((n_planes + l.G - 1) / l.G) * l.n_cc * l.n_rb;
}

int pool_grid(const bs_plan* p, const Launch& l, int64_t n_tasks) {
  if (l.kernel == K_POOL_STAGED)   // persistent: every CTA loops over tiles
    return (int)std::max<int64_t>(1, std::min<int64_t>(n_tasks, (int64_t)std::max(1, l.blocks_per_sm) * p->num_sms));
  if (l.kernel == K_POOL_PLANES)   // one 32-plane chunk per warp, 4 warps per CTA
    return (int)std::max<int64_t>(1, std::min<int64_t>((n_tasks + 3) / 4, INT32_MAX / 2));
  int64_t g = l.kernel == K_POOL_NAIVE ? (n_tasks + 255) / 256 : (n_tasks + 7) / 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, INT32_MAX / 2));
}

constexpr int64_t kEwMaxElems = (int64_t(1) << 31) - 1024;

// element-wise tensors below this many elements use one float4 per thread (4x the threads)
#ifndef BS_EW_SMALL
#define BS_EW_SMALL (int64_t(2) << 20)   /* measured: 1.6 M elements 4.0 -> 3.7 us; 6.4 M slower */
#endif
int ew_unroll(int64_t n_elems) { return n_elems < BS_EW_SMALL ? 1 : 4; }

int ew_grid(int64_t n_elems) {
  const int64_t per_block = 256 * 4 * (int64_t)ew_unroll(n_elems);  // kEwBlock * unroll * 4 floats
  return (int)std::max<int64_t>(1, std::min<int64_t>((n_elems + per_block - 1) / per_block, INT32_MAX / 2));
}

// A SeqArgs carrying the fields seq_smem / the occupancy query need.
SeqArgs seq_probe(const Launch& l) {
  SeqArgs a;
  std::memset(&a, 0, sizeof a);
  a.tile_planes = l.tile_planes;
  a.stages = l.stages;
  a.stage_bytes = l.seq_stage_bytes;
  a.work_floats = l.seq_work_floats;
  a.in_plane = (int32_t)(l.step.in.h * l.step.in.w);
  a.n_bands = l.seq_bands;
  a.n_steps = (int32_t)l.seq.size();
  a.inplace_seg = l.seq_inplace_seg;
  a.H0 = (int32_t)l.step.in.h;
  a.W0 = (int32_t)l.step.in.w;
  return a;
}

void fill_info(bs_plan* p, const std::vector<Shape4>& shapes, int n_layers, int n_inputs) {
  bs_plan_info& I = p->info;
  std::memset(&I, 0, sizeof I);
  const Shape4& o = shapes.back();
  I.out = bs_shape{o.n, o.c, o.h, o.w};
  I.n_layers = n_layers;
  I.n_steps = (int32_t)p->steps.size();
  I.n_sequences = (int32_t)p->launches.size();
  I.n_launches = I.n_sequences;
  I.n_inputs = n_inputs;
  int n_ops = 0;
  int64_t params = 0, inter = 0;
  for (auto& st : p->steps) {
    n_ops += (int)(st.pro.size() + st.epi.size()) + (st.has_pool ? 1 : 0);
    for (auto* v : {&st.pro, &st.epi})
      for (auto& op : *v) params += (int64_t)op.affine.size() * 8;
  }
  for (auto& l : p->launches)
    if (l.dst >= 0) inter = std::max<int64_t>(inter, l.step.out.numel() * 4);
  I.n_ops = n_ops;
  I.param_bytes = params;
  I.intermediate_bytes = p->launches.size() > 2 ? 2 * inter : inter;
  // algorithmic bytes: one read of the stack input + every ADD operand, one write of the output
  int64_t rd = shapes[0].numel() * 4;
  for (auto& st : p->steps)
    for (auto* v : {&st.pro, &st.epi})
      for (auto& op : *v)
        if (op.kind == DOP_ADD) rd += shapes[op.layer].numel() * 4;
  I.alg_bytes_read = rd;
  I.alg_bytes_written = o.numel() * 4;
}

void fill_launch_info(bs_plan* p) {
  for (auto& l : p->launches) {
    bs_launch_info& li = l.info;
    std::memset(&li, 0, sizeof li);
    const Step& s = l.step;
    li.kernel = l.kernel;
    li.first_layer = s.first_layer;
    li.last_layer = s.last_layer;
    li.in = bs_shape{s.in.n, s.in.c, s.in.h, s.in.w};
    li.out = bs_shape{s.out.n, s.out.c, s.out.h, s.out.w};
    if (s.has_pool) {
      li.pool_kh = s.kh; li.pool_kw = s.kw; li.pool_sh = s.sh;
      li.pool_sw = s.sw; li.pool_ph = s.ph; li.pool_pw = s.pw;
    }
    li.n_prologue_ops = (int32_t)s.pro.size();
    li.n_epilogue_ops = (int32_t)s.epi.size();
    li.block = 256;
    const int64_t n_planes = s.in.n * s.in.c;
    if (l.kernel == K_EW) {
      li.grid = ew_grid(std::min<int64_t>(s.in.numel(), kEwMaxElems));
      li.n_tasks = 0;
    } else if (l.kernel == K_SEQ) {
      li.n_prologue_ops = (int32_t)l.seq.front().pro.size();
      li.n_epilogue_ops = (int32_t)l.seq.back().epi.size();
      li.groups_per_warp = (int32_t)l.seq.size();          // steps fused in the sequence
      li.outputs_per_group = l.tile_planes;                 // planes per staged tile
      li.rows_per_task = (int32_t)s.out.h;
      li.n_tasks = (n_planes + l.tile_planes - 1) / l.tile_planes * l.seq_bands;   // tiles
      li.grid = (int)std::min<int64_t>(li.n_tasks, (int64_t)std::max(1, l.blocks_per_sm) * p->num_sms);
      li.block = l.seq_inplace_seg ? seq_inplace_threads(seq_probe(l)) : kSeqThreads;
      li.smem_bytes = (int32_t)(l.seq_inplace_seg ? seq_inplace_smem(seq_probe(l)) : seq_smem(seq_probe(l)));
      li.tile_planes = l.tile_planes;
      li.tile_rows = l.seq_bands > 1 ? l.seq_band_rows : 0;
      // redundant (halo) input rows of step 0 per band: rows loaded beyond the band's own share
      int64_t loaded = 0;
      const size_t n = l.seq.size();
      for (int32_t bd = 0; bd < l.seq_bands; ++bd) loaded += l.seq_ranges[(size_t)bd * n].in_hi - l.seq_ranges[(size_t)bd * n].in_lo;
      li.halo_rows = (int32_t)(loaded - s.in.h);
      li.stages = l.stages;
    } else {
      li.groups_per_warp = l.G;
      li.outputs_per_group = l.Jg;
      li.rows_per_task = l.rows_per_task;
      li.halo_rows = std::max(0, s.kh - s.sh);
      li.n_tasks = pool_tasks(l, n_planes);
      li.grid = pool_grid(p, l, li.n_tasks);
      li.block = l.kernel == K_POOL_STAGED ? kStagedThreads : l.kernel == K_POOL_PLANES ? pool_planes_threads() : 256;
      if (l.kernel == K_POOL_PLANES) li.smem_bytes = (int32_t)pool_planes_smem((int)(s.in.h * s.in.w));
      if (l.kernel == K_POOL_STAGED) {
        li.smem_bytes = (int32_t)pool_staged_smem(l.tile_planes, (int)(s.in.h * s.in.w), (int)(s.out.h * s.out.w),
                                                  l.stages);
        li.tile_planes = l.tile_planes;
        li.stages = l.stages;
      }
    }
    int64_t rd = s.in.numel() * 4;
    for (auto* v : {&s.pro, &s.epi})
      for (auto& op : *v)
        if (op.kind == DOP_ADD) rd += (v == &s.pro ? s.in.numel() : s.out.numel()) * 4;
    li.alg_bytes_read = rd;
    li.alg_bytes_written = s.out.numel() * 4;
  }
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// ---------------------------------------------------------------- a5: dispatch
// Enqueue every launch for images [img0, img1) on `st`.
bs_status enqueue(const bs_plan* p, const float* const* inputs, float* out, int64_t img0, int64_t img1,
                  cudaStream_t st) {
  for (size_t k = 0; k < p->launches.size(); ++k) {
    const Launch& l = p->launches[k];
    const Step& s = l.step;
    const float* src = l.src < 0 ? inputs[0] : p->inter[l.src];
    float* dst = l.dst < 0 ? out : p->inter[l.dst];
    cudaError_t e = cudaSuccess;
    if (l.kernel == K_SEQ) {
      SeqArgs a;
      std::memset(&a, 0, sizeof a);
      a.in = src;
      a.out = dst;
      a.steps = p->seq_steps + l.seq_off;
      a.n_steps = (int32_t)l.seq.size();
      a.C = (int32_t)s.in.c;
      a.plane0 = img0 * s.in.c;
      a.n_planes = (img1 - img0) * s.in.c;
      a.tile_planes = l.tile_planes;
      a.stages = l.stages;
      a.n_bands = l.seq_bands;
      a.ranges = p->seq_ranges + l.range_off;
      a.stage_bytes = l.seq_stage_bytes;
      a.n_tiles = (a.n_planes + l.tile_planes - 1) / l.tile_planes * l.seq_bands;
      a.work_floats = l.seq_work_floats;
      a.inplace_seg = l.seq_inplace_seg;
      a.in_plane = (int32_t)(s.in.h * s.in.w);
      a.H0 = (int32_t)s.in.h;
      a.W0 = (int32_t)s.in.w;
      a.cdiv = make_fastdiv((uint32_t)a.C);
      const int grid = (int)std::min<int64_t>(a.n_tiles, (int64_t)std::max(1, l.blocks_per_sm) * p->num_sms);
      e = launch_seq(a, grid, st);
    } else if (l.kernel == K_EW) {
      EwArgs a;
      std::memset(&a, 0, sizeof a);
      a.prog = make_prog(p, s.pro);
      a.prog_class = prog_class(s.pro);
      fill_operands(a.prog, s.pro, inputs);
      const int64_t CHW = s.in.c * s.in.h * s.in.w;
      a.hw = make_fastdiv((uint32_t)(s.in.h * s.in.w));
      a.c = make_fastdiv((uint32_t)s.in.c);
      a.hw_ge4 = s.in.h * s.in.w >= 4;
      // split into pieces of < 2^31 elements rebased at multiples of 4 images (16-B aligned,
      // channel index of the local element = (e / HW) % C still holds)
      int64_t step_imgs = std::max<int64_t>(4, (kEwMaxElems / CHW) / 4 * 4);
      for (int64_t b = (img0 / 4) * 4; b < img1; b += step_imgs) {
        const int64_t lo = std::max(img0, b), hi = std::min(img1, b + step_imgs);
        if (lo >= hi) continue;
        const int64_t off = b * CHW;
        EwArgs q = a;
        q.in = src + off;
        q.out = dst + off;
        for (int i = 0; i < q.prog.n; ++i)
          if (q.prog.kind[i] == DOP_ADD) q.prog.operand[i] += off;
        q.add0_ptr = nullptr;
        for (int i = 0; i < q.prog.n; ++i)
          if (q.prog.add_slot[i] == 0) q.add0_ptr = q.prog.operand[i];
        q.e_begin = (lo - b) * CHW;
        q.e_end = (hi - b) * CHW;
        q.unroll = ew_unroll(q.e_end - q.e_begin);
        e = launch_ew(q, ew_grid(q.e_end - q.e_begin), 256, st);
        if (e != cudaSuccess) break;
      }
    } else {
      PoolArgs a = make_pool_args(p, l);
      fill_operands(a.pro, l.dev_pro, inputs);
      fill_operands(a.epi, l.dev_epi, inputs);
      a.in = src;
      a.out = dst;
      a.plane0 = img0 * s.in.c;
      a.n_planes = (img1 - img0) * s.in.c;
      a.n_tasks = pool_tasks(l, a.n_planes);
      a.n_tiles = a.n_tasks;
      e = launch_pool(a, l.kernel, pool_grid(p, l, a.n_tasks), 256, st);
    }
    if (e != cudaSuccess)
      return fail(BS_ERR_CUDA, "launch %zu (layers %d..%d): %s", k, s.first_layer, s.last_layer,
                  cudaGetErrorString(e));
  }
  return BS_OK;
}

bs_status check_exec_args(const bs_plan* p, const float* const* inputs, int32_t n_inputs, const float* out) {
  if (!p) return fail(BS_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (p->host_only) return fail(BS_ERR_INVALID_ARGUMENT, "plan was created host_only; it cannot be executed");
  if (p->empty) {   // empty batch: nothing is read or written (pointers may be NULL)
    if (n_inputs != p->info.n_inputs)
      return fail(BS_ERR_INVALID_ARGUMENT, "plan needs %d inputs (stack input + ADD operands), got %d",
                  p->info.n_inputs, n_inputs);
    return BS_OK;
  }
  if (!inputs || !out) return fail(BS_ERR_INVALID_ARGUMENT, "NULL tensor pointer");
  if (n_inputs != p->info.n_inputs)
    return fail(BS_ERR_INVALID_ARGUMENT, "plan needs %d inputs (stack input + ADD operands), got %d",
                p->info.n_inputs, n_inputs);
  const size_t out_bytes = (size_t)(p->info.out.n * p->info.out.c * p->info.out.h * p->info.out.w) * 4;
  if ((uintptr_t)out % 16) return fail(BS_ERR_INVALID_ARGUMENT, "out is not 16-byte aligned");
  bool all_ew = true;
  for (auto& l : p->launches) all_ew &= !l.step.has_pool;
  const Shape4 in0 = p->launches.front().step.in;
  for (int k = 0; k < n_inputs; ++k) {
    if (!inputs[k]) return fail(BS_ERR_INVALID_ARGUMENT, "inputs[%d] is NULL", k);
    if ((uintptr_t)inputs[k] % 16) return fail(BS_ERR_INVALID_ARGUMENT, "inputs[%d] is not 16-byte aligned", k);
    size_t nb = (size_t)in0.numel() * 4;
    if (k > 0) {   // operand k's bytes = its ADD layer's input shape
      for (auto& l : p->launches)
        for (auto* v : {&l.step.pro, &l.step.epi})
          for (auto& op : *v)
            if (op.kind == DOP_ADD && op.operand == k)
              nb = (size_t)((v == &l.step.pro ? l.step.in : l.step.out).numel()) * 4;
    }
    if (overlaps(inputs[k], nb, out, out_bytes)) {
      const bool inplace_ok = k == 0 && all_ew && p->launches.size() == 1 && (const void*)inputs[0] == (const void*)out;
      if (!inplace_ok)
        return fail(BS_ERR_INVALID_ARGUMENT, "out overlaps inputs[%d] (only exact in==out for element-wise plans)", k);
    }
  }
  return BS_OK;
}

void free_plan(bs_plan* p) {
  if (!p) return;
  if (!p->host_only) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    if (p->params) cudaFree(p->params);
    if (p->seq_steps) cudaFree(p->seq_steps);
    if (p->seq_ranges) cudaFree(p->seq_ranges);
    for (float* b : p->inter)
      if (b) cudaFree(b);
    for (auto& s : p->copy_stream)
      if (s) cudaStreamDestroy(s);
    for (int i = 0; i < p->n_events; ++i) cudaEventDestroy(p->ev_pool[i]);
    cudaSetDevice(prev);
  }
  delete p;
}

}  // namespace

// Host-buffer checks of one bs_execute_host execution.
bs_status check_host_args(const bs_plan* plan, const float* const* h_inputs, int32_t n_inputs, const float* h_out,
                          float* const* d_inputs, const float* d_out) {
  bs_status st = check_exec_args(plan, (const float* const*)d_inputs, n_inputs, d_out);
  if (st != BS_OK || plan->empty) return st;
  if (!h_inputs || !h_out) return fail(BS_ERR_INVALID_ARGUMENT, "NULL host pointer");
  for (int k = 0; k < n_inputs; ++k)
    if (!h_inputs[k]) return fail(BS_ERR_INVALID_ARGUMENT, "h_inputs[%d] is NULL", k);
  return BS_OK;
}

// Bytes of input k of a plan (the stack input, or ADD operand k's layer input / output).
int64_t input_bytes(const bs_plan* plan, int k) {
  int64_t nb = plan->launches.front().step.in.numel() * 4;
  if (k > 0)
    for (auto& l : plan->launches)
      for (auto* v : {&l.step.pro, &l.step.epi})
        for (auto& op : *v)
          if (op.kind == DOP_ADD && op.operand == k) nb = (v == &l.step.pro ? l.step.in : l.step.out).numel() * 4;
  return nb;
}

// Enqueue one execution's chunked pipeline: chunk k's host->device copies on h2d, its kernels on
// cs (after the copies), its device->host copy on d2h (after the kernels).  The copy streams
// must already be ordered after whatever they have to follow.  `copied` / `done` are re-recorded
// per chunk: a stream wait binds the record that is current when the wait is enqueued.
bs_status pipeline_host(const bs_plan* plan, const float* const* h_inputs, int32_t n_inputs, float* h_out,
                        float* const* d_inputs, float* d_out, int32_t n_chunks, cudaStream_t cs, cudaStream_t h2d,
                        cudaStream_t d2h, cudaEvent_t copied, cudaEvent_t done) {
  const int64_t N = plan->launches.front().step.in.n;
  // default: 4 chunks (ResNet-50 step through bs_execute_host_batch, images/s: 1 chunk 2872,
  // 2: 2963, 4: 2995, 8: ~2930, 16: 2755 -- few large copies, and enough to overlap within a stack)
  if (n_chunks <= 0) n_chunks = 4;
  n_chunks = (int32_t)std::min<int64_t>(n_chunks, N);
  // per-image byte sizes of each input and the output
  std::vector<int64_t> in_img(n_inputs);
  for (int k = 0; k < n_inputs; ++k) in_img[k] = input_bytes(plan, k) / N;
  const int64_t out_img = plan->info.out.c * plan->info.out.h * plan->info.out.w * 4;
  cudaError_t e = cudaSuccess;
  for (int32_t k = 0; k < n_chunks && e == cudaSuccess; ++k) {
    const int64_t i0 = N * k / n_chunks, i1 = N * (k + 1) / n_chunks;
    for (int q = 0; q < n_inputs && e == cudaSuccess; ++q)
      e = cudaMemcpyAsync((char*)d_inputs[q] + i0 * in_img[q], (const char*)h_inputs[q] + i0 * in_img[q],
                          (size_t)((i1 - i0) * in_img[q]), cudaMemcpyHostToDevice, h2d);
    if (e != cudaSuccess) break;
    if ((e = cudaEventRecord(copied, h2d)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(cs, copied, 0)) != cudaSuccess) break;
    const bs_status st = enqueue(plan, (const float* const*)d_inputs, d_out, i0, i1, cs);
    if (st != BS_OK) return st;
    if ((e = cudaEventRecord(done, cs)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(d2h, done, 0)) != cudaSuccess) break;
    e = cudaMemcpyAsync((char*)h_out + i0 * out_img, (const char*)d_out + i0 * out_img, (size_t)((i1 - i0) * out_img),
                        cudaMemcpyDeviceToHost, d2h);
  }
  if (e != cudaSuccess) return fail(BS_ERR_CUDA, "bs_execute_host: %s", cudaGetErrorString(e));
  return BS_OK;
}

// Runs `body` with the plan's device current, then orders the copy streams after the caller's
// stream before it and the caller's stream after the last device->host copy.
template <class F>
bs_status host_pipeline_scope(const bs_plan* plan, cudaStream_t cs, F body) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != plan->device) cudaSetDevice(plan->device);
  cudaEvent_t* ev = const_cast<cudaEvent_t*>(plan->ev_pool);
  cudaStream_t h2d = plan->copy_stream[0], d2h = plan->copy_stream[1];
  bs_status st = BS_OK;
  cudaError_t e = cudaEventRecord(ev[0], cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h2d, ev[0], 0);
  if (e == cudaSuccess) st = body(h2d, d2h, ev[2], ev[3]);
  // the caller's stream completes only after the last device->host copy (also on failure: the
  // copies already enqueued stay ordered before later work on the caller's stream)
  if (e == cudaSuccess) e = cudaEventRecord(ev[1], d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[1], 0);
  if (prev != plan->device) cudaSetDevice(prev);
  if (st != BS_OK) return st;
  if (e != cudaSuccess) return fail(BS_ERR_CUDA, "bs_execute_host: %s", cudaGetErrorString(e));
  return BS_OK;
}

// ================================================================= extern "C"
extern "C" {

int32_t bs_version(void) { return 1; }

const char* bs_last_error(void) { return g_err.c_str(); }

const char* bs_status_string(bs_status s) {
  switch (s) {
    case BS_OK: return "BS_OK";
    case BS_ERR_INVALID_ARGUMENT: return "BS_ERR_INVALID_ARGUMENT";
    case BS_ERR_VALIDATION: return "BS_ERR_VALIDATION";
    case BS_ERR_PLANNING: return "BS_ERR_PLANNING";
    case BS_ERR_CUDA: return "BS_ERR_CUDA";
    case BS_ERR_OUT_OF_MEMORY: return "BS_ERR_OUT_OF_MEMORY";
    default: return "BS_ERR_UNKNOWN";
  }
}

bs_status bs_plan_create(const bs_layer_desc* layers, int32_t n_layers, bs_shape input,
                         const bs_plan_options* opts, bs_plan** plan_out) {
  g_err.clear();
  if (!plan_out) return fail(BS_ERR_INVALID_ARGUMENT, "plan_out is NULL");
  *plan_out = nullptr;
  if (!layers || n_layers < 1) return fail(BS_ERR_INVALID_ARGUMENT, "need at least one layer (n_layers=%d)", n_layers);
  bs_plan_options o;
  std::memset(&o, 0, sizeof o);
  o.device = -1;
  if (opts) o = *opts;
  if (o.max_steps_per_sequence < -1)
    return fail(BS_ERR_INVALID_ARGUMENT, "max_steps_per_sequence=%d: use -1 (unrestricted), 0 (planner) or k >= 1",
                o.max_steps_per_sequence);
  if (o.threads_per_block != 0)
    return fail(BS_ERR_INVALID_ARGUMENT, "threads_per_block=%d: block sizes are fixed per kernel (pass 0)",
                o.threads_per_block);

  // an empty batch (N = 0) is valid: plan the geometry of one image, execute nothing
  const bool empty_batch = input.n == 0;
  if (empty_batch) input.n = 1;
  std::vector<Shape4> shapes;
  int n_inputs = 1;
  bs_status st = validate_and_shape(layers, n_layers, input, shapes, n_inputs);
  if (st != BS_OK) return st;
  for (const Shape4& s : shapes)
    if (s.n * s.c > INT32_MAX || s.h * s.w > INT32_MAX / 4 || 4 * s.c * s.h * s.w > kEwMaxElems)
      return fail(BS_ERR_PLANNING, "tensor (%lld,%lld,%lld,%lld) exceeds the index range", (long long)s.n,
                  (long long)s.c, (long long)s.h, (long long)s.w);

  bs_plan* p = new (std::nothrow) bs_plan();
  if (!p) return fail(BS_ERR_OUT_OF_MEMORY, "host allocation failed");
  p->host_only = o.host_only != 0;
  if (!p->host_only) {
    int dev = o.device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
      delete p;
      return fail(BS_ERR_CUDA, "cudaGetDevice failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    p->device = dev;
    if (cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      delete p;
      return fail(BS_ERR_CUDA, "cannot query device %d: %s", dev, cudaGetErrorString(cudaGetLastError()));
    }
  }

  std::vector<Step> steps;
  group_steps(layers, n_layers, shapes, steps);
  // parameter block layout (before the launches copy the programs)
  size_t n_f2 = 0;
  for (Step& st_ : steps)
    for (auto* v : {&st_.pro, &st_.epi})
      for (HostOp& op : *v)
        if (op.kind == DOP_AFFINE) {
          op.affine_off = n_f2;
          n_f2 += op.affine.size();
        }
  p->steps = steps;
  pack_and_tile(p, steps, o);
  for (Launch& l : p->launches) {
    if (l.kernel == K_SEQ) {
      const int bps = p->host_only ? 0 : seq_max_blocks_per_sm(seq_probe(l));
      l.blocks_per_sm = bps > 0 ? bps : 1;
    } else if (l.kernel != K_EW) {
      int bps = 0;
      if (!p->host_only) {
        PoolArgs probe = make_pool_args(p, l);
        bps = pool_max_blocks_per_sm(l.kernel, probe, 256);
      }
      l.blocks_per_sm = bps > 0 ? bps : 5;
      if (l.kernel == K_POOL_STAGED && l.ctas_per_sm > 0) l.blocks_per_sm = std::min(l.blocks_per_sm, l.ctas_per_sm);
      if (l.kernel != K_POOL_NAIVE && l.kernel != K_POOL_STAGED && l.kernel != K_POOL_PLANES)
        size_rows(p, l, o, l.step.in.n * l.step.in.c);
    }
  }
  fill_info(p, shapes, n_layers, n_inputs);
  if (empty_batch) {
    p->empty = true;
    p->info.out.n = 0;
    p->info.alg_bytes_read = p->info.alg_bytes_written = 0;
    p->info.n_launches = 0;
  }
  fill_launch_info(p);

  if (!p->host_only) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    auto cuda_fail = [&](const char* what, cudaError_t e) {
      cudaSetDevice(prev);
      free_plan(p);
      return fail(e == cudaErrorMemoryAllocation ? BS_ERR_OUT_OF_MEMORY : BS_ERR_CUDA, "%s: %s", what,
                  cudaGetErrorString(e));
    };
    cudaError_t e;
    if (n_f2) {
      if ((e = cudaMalloc(&p->params, n_f2 * sizeof(float2))) != cudaSuccess) return cuda_fail("cudaMalloc(params)", e);
      std::vector<float2> host(n_f2);
      for (Step& st : p->steps)
        for (auto* v : {&st.pro, &st.epi})
          for (HostOp& op : *v)
            if (op.kind == DOP_AFFINE) std::copy(op.affine.begin(), op.affine.end(), host.begin() + op.affine_off);
      if ((e = cudaMemcpy(p->params, host.data(), n_f2 * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail("cudaMemcpy(params)", e);
    }
    {  // device descriptors of the on-chip sequences
      std::vector<SeqStepDev> desc;
      std::vector<SeqRange> ranges;
      for (Launch& l : p->launches) {
        if (l.kernel != K_SEQ) continue;
        l.seq_off = desc.size();
        l.range_off = ranges.size();
        ranges.insert(ranges.end(), l.seq_ranges.begin(), l.seq_ranges.end());
        for (size_t si = 0; si < l.seq.size(); ++si) {
          const Step& st = l.seq[si];
          SeqStepDev d;
          std::memset(&d, 0, sizeof d);
          d.H = (int32_t)st.in.h; d.W = (int32_t)st.in.w; d.Ho = (int32_t)st.out.h; d.Wo = (int32_t)st.out.w;
          if (st.has_pool) {
            d.kh = st.kh; d.kw = st.kw; d.sh = st.sh; d.sw = st.sw; d.ph = st.ph; d.pw = st.pw;
            d.is_max = st.is_max; d.count_include_pad = st.cip;
          } else {  // element-wise step: a 1x1/s1 max pool is the identity
            d.kh = d.kw = d.sh = d.sw = 1; d.is_max = 1; d.count_include_pad = 1;
          }
          d.pro = make_prog(p, st.pro);
          d.epi = make_prog(p, st.epi);
          d.epi_class = prog_class(st.epi);
          d.fast = is_fast_step(st) ? 1 : 0;
          d.in_pitch = l.seq_in_pitch[si];
          d.out_pitch = l.seq_out_pitch[si];
          desc.push_back(d);
        }
      }
      if (!desc.empty()) {
        if ((e = cudaMalloc(&p->seq_steps, desc.size() * sizeof(SeqStepDev))) != cudaSuccess)
          return cuda_fail("cudaMalloc(sequence steps)", e);
        if ((e = cudaMemcpy(p->seq_steps, desc.data(), desc.size() * sizeof(SeqStepDev), cudaMemcpyHostToDevice)) !=
            cudaSuccess)
          return cuda_fail("cudaMemcpy(sequence steps)", e);
        if ((e = cudaMalloc(&p->seq_ranges, ranges.size() * sizeof(SeqRange))) != cudaSuccess)
          return cuda_fail("cudaMalloc(sequence ranges)", e);
        if ((e = cudaMemcpy(p->seq_ranges, ranges.data(), ranges.size() * sizeof(SeqRange), cudaMemcpyHostToDevice)) !=
            cudaSuccess)
          return cuda_fail("cudaMemcpy(sequence ranges)", e);
      }
    }
    int64_t inter = 0;
    for (auto& l : p->launches)
      if (l.dst >= 0) inter = std::max<int64_t>(inter, l.step.out.numel());
    if (inter > 0) {
      if ((e = cudaMalloc(&p->inter[0], (size_t)inter * 4)) != cudaSuccess) return cuda_fail("cudaMalloc(intermediate)", e);
      if (p->launches.size() > 2 && (e = cudaMalloc(&p->inter[1], (size_t)inter * 4)) != cudaSuccess)
        return cuda_fail("cudaMalloc(intermediate)", e);
    }
    for (auto& s : p->copy_stream)
      if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail("cudaStreamCreate", e);
    p->n_events = 4;
    for (int i = 0; i < p->n_events; ++i)
      if ((e = cudaEventCreateWithFlags(&p->ev_pool[i], cudaEventDisableTiming)) != cudaSuccess) {
        p->n_events = i;
        return cuda_fail("cudaEventCreate", e);
      }
    cudaSetDevice(prev);
  }
  *plan_out = p;
  return BS_OK;
}

bs_status bs_plan_query(const bs_plan* plan, bs_plan_info* info) {
  if (!plan || !info) return fail(BS_ERR_INVALID_ARGUMENT, "NULL argument");
  *info = plan->info;
  return BS_OK;
}

bs_status bs_plan_query_launch(const bs_plan* plan, int32_t index, bs_launch_info* info) {
  if (!plan || !info) return fail(BS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (index < 0 || index >= (int32_t)plan->launches.size())
    return fail(BS_ERR_INVALID_ARGUMENT, "launch index %d out of range [0,%zu)", index, plan->launches.size());
  *info = plan->launches[(size_t)index].info;
  return BS_OK;
}

bs_status bs_execute_ex(const bs_plan* plan, const float* const* inputs, int32_t n_inputs, float* out,
                        bs_stream_t stream) {
  bs_status st = check_exec_args(plan, inputs, n_inputs, out);
  if (st != BS_OK || plan->empty) return st;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != plan->device) cudaSetDevice(plan->device);
  st = enqueue(plan, inputs, out, 0, plan->launches.front().step.in.n, (cudaStream_t)stream);
  if (prev != plan->device) cudaSetDevice(prev);
  return st;
}

bs_status bs_execute(const bs_plan* plan, const float* in, float* out, bs_stream_t stream) {
  const float* inputs[1] = {in};
  return bs_execute_ex(plan, inputs, 1, out, stream);
}

bs_status bs_execute_host(const bs_plan* plan, const float* const* h_inputs, int32_t n_inputs, float* h_out,
                          float* const* d_inputs, float* d_out, int32_t n_chunks, bs_stream_t stream) {
  bs_status st = check_host_args(plan, h_inputs, n_inputs, h_out, d_inputs, d_out);
  if (st != BS_OK || plan->empty) return st;
  return host_pipeline_scope(plan, (cudaStream_t)stream, [&](cudaStream_t h2d, cudaStream_t d2h, cudaEvent_t c,
                                                             cudaEvent_t d) {
    return pipeline_host(plan, h_inputs, n_inputs, h_out, d_inputs, d_out, n_chunks, (cudaStream_t)stream, h2d, d2h,
                         c, d);
  });
}

bs_status bs_execute_host_batch(const bs_plan* const* plans, int32_t n_plans, const float* const* const* h_inputs,
                                const int32_t* n_inputs, float* const* h_outs, float* const* const* d_inputs,
                                float* const* d_outs, int32_t n_chunks, bs_stream_t stream) {
  if (n_plans < 0 || (n_plans > 0 && (!plans || !h_inputs || !n_inputs || !h_outs || !d_inputs || !d_outs)))
    return fail(BS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n_plans == 0) return BS_OK;
  const bs_plan* lead = nullptr;
  for (int32_t i = 0; i < n_plans; ++i) {
    bs_status st = check_host_args(plans[i], h_inputs[i], n_inputs[i], h_outs[i], d_inputs[i], d_outs[i]);
    if (st != BS_OK) {
      const std::string m = bs_last_error();
      return fail(st, "execution %d: %s", i, m.c_str());
    }
    if (plans[i]->empty) continue;
    if (!lead) lead = plans[i];
    if (plans[i]->device != lead->device) return fail(BS_ERR_INVALID_ARGUMENT, "execution %d: plans on different devices", i);
  }
  if (!lead) return BS_OK;
  // an execution's host->device copies may overlap earlier executions' kernels and copies, so the
  // device buffers of different executions must not overlap
  for (int32_t i = 0; i < n_plans; ++i) {
    if (plans[i]->empty) continue;
    for (int32_t j = 0; j < i; ++j) {
      if (plans[j]->empty) continue;
      auto bufs = [&](int32_t x, std::vector<std::pair<const void*, size_t>>& v) {
        v.clear();
        for (int k = 0; k < n_inputs[x]; ++k) v.push_back({d_inputs[x][k], (size_t)input_bytes(plans[x], k)});
        const bs_shape& o = plans[x]->info.out;
        v.push_back({d_outs[x], (size_t)(o.n * o.c * o.h * o.w) * 4});
      };
      std::vector<std::pair<const void*, size_t>> bi, bj;
      bufs(i, bi);
      bufs(j, bj);
      for (auto& x : bi)
        for (auto& y : bj)
          if (overlaps(x.first, x.second, y.first, y.second))
            return fail(BS_ERR_INVALID_ARGUMENT, "executions %d and %d share device buffers", j, i);
    }
  }
  return host_pipeline_scope(lead, (cudaStream_t)stream, [&](cudaStream_t h2d, cudaStream_t d2h, cudaEvent_t c,
                                                             cudaEvent_t d) {
    for (int32_t i = 0; i < n_plans; ++i) {
      if (plans[i]->empty) continue;
      const bs_status st = pipeline_host(plans[i], h_inputs[i], n_inputs[i], h_outs[i], d_inputs[i], d_outs[i],
                                         n_chunks, (cudaStream_t)stream, h2d, d2h, c, d);
      if (st != BS_OK) {
        const std::string m = bs_last_error();
        return fail(st, "execution %d: %s", i, m.c_str());
      }
    }
    return BS_OK;
  });
}

void bs_plan_destroy(bs_plan* plan) { free_plan(plan); }

struct bs_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int device = 0;
};

bs_status bs_graph_create(const bs_plan* const* plans, int32_t n_plans, const float* const* const* inputs,
                          const int32_t* n_inputs, float* const* outs, bs_graph** graph_out) {
  g_err.clear();
  if (!graph_out) return fail(BS_ERR_INVALID_ARGUMENT, "graph_out is NULL");
  *graph_out = nullptr;
  if (!plans || !inputs || !n_inputs || !outs || n_plans < 1)
    return fail(BS_ERR_INVALID_ARGUMENT, "NULL array or n_plans < 1 (%d)", n_plans);
  for (int32_t i = 0; i < n_plans; ++i) {
    bs_status st = check_exec_args(plans[i], inputs[i], n_inputs[i], outs[i]);
    if (st != BS_OK) return fail(st, "execution %d: %s", i, g_err.c_str());
    if (plans[i]->device != plans[0]->device)
      return fail(BS_ERR_INVALID_ARGUMENT, "execution %d: plan on device %d, execution 0 on device %d", i,
                  plans[i]->device, plans[0]->device);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  const int dev = plans[0]->device;
  if (prev != dev) cudaSetDevice(dev);
  bs_graph* g = new (std::nothrow) bs_graph();
  if (!g) {
    if (prev != dev) cudaSetDevice(prev);
    return fail(BS_ERR_OUT_OF_MEMORY, "host allocation failed");
  }
  g->device = dev;
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  bs_status st = BS_OK;
  if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    for (int32_t i = 0; i < n_plans && st == BS_OK; ++i)
      if (!plans[i]->empty) st = enqueue(plans[i], inputs[i], outs[i], 0, plans[i]->launches.front().step.in.n, cs);
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cs, &graph);   // always end the capture
    g->graph = graph;
    if (e2 != cudaSuccess && st == BS_OK) e = e2;
  }
  if (e == cudaSuccess && st == BS_OK) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (cs) cudaStreamDestroy(cs);
  if (prev != dev) cudaSetDevice(prev);
  if (st != BS_OK || e != cudaSuccess) {
    bs_graph_destroy(g);
    if (st != BS_OK) return st;
    return fail(BS_ERR_CUDA, "bs_graph_create: %s", cudaGetErrorString(e));
  }
  *graph_out = g;
  return BS_OK;
}

bs_status bs_graph_launch(const bs_graph* g, bs_stream_t stream) {
  if (!g || !g->exec) return fail(BS_ERR_INVALID_ARGUMENT, "graph is NULL");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != g->device) cudaSetDevice(g->device);
  cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
  if (prev != g->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(BS_ERR_CUDA, "bs_graph_launch: %s", cudaGetErrorString(e));
  return BS_OK;
}

void bs_graph_destroy(bs_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

}  // extern "C"
