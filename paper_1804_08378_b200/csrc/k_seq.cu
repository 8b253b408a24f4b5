// k_seq.cu -- on-chip multi-step sequences (NEXT-2), whole-plane or halo (row-band) tiles.
#include "bs_device.cuh"

namespace bs {

// ------------------------------------------------------------------ multi-step sequences
//
// NEXT-2: a *sequence* of several steps runs on-chip (PAPER.md P:L545-558,
// lst:finalcode P:L512-530 "float cached_data[...]"; the paper's GPU kernel swapped two smem
// buffers per step).  A tile is bulk-copied (TMA, cp.async.bulk) into a ring stage;
// step 0 reads the stage, every later step reads the previous step's work buffer (two ping-pong
// buffers in shared memory), and only the last step writes HBM.  A named barrier over the 8
// consumer warps separates steps.
//
// Tiles (chosen by the planner, bs_api.cpp plan_sequence):
//  * whole planes: P planes per tile, no halo at all;
//  * halo tiles (planes too large to hold whole): one plane, a band of output rows of the last
//    step; every earlier step computes the rows the next step's windows need, so its band grows
//    by the window overlap -- the paper's "Patches", whose redundant halo work grows
//    with each padded step.  The per-band row ranges of every step are precomputed
//    on the host (SeqRange): a step's input buffer holds rows [in_lo, in_hi), it computes rows
//    [out_lo, out_hi).  Full rows: only the row dimension has a halo.
//
// Steps run one of two paths:
//  * fast (the §5.1 block: 3x3/s1/p1 max pool + [BN] [ReLU], W % 4 == 0, W <= 256): a lane owns
//    4 adjacent columns of a row (one LDS.128); the horizontal 3-max takes the outer neighbours
//    from the adjacent lanes (two shuffles), the vertical 3-max rolls over a 3-row register
//    window; both are single FMNMX3 instructions (3-input max.f32 on sm_100).  Segments of 16
//    lanes (W <= 64: two row streams per warp) or 32 lanes (one or two segments per row).  Plane
//    edges: a missing neighbour is replaced by the element itself (a duplicate, exact for max),
//    so padding stays absent.  Outputs: STS.128 to the next work buffer, STG.128 from the last.
//  * generic: lane = output column, a windowed interpreter (any pool, prologue, epilogue).

size_t seq_smem(const SeqArgs& a) {
  // barriers | stages | 2 work buffers | 1 KB slack (vector loads of idle lanes past a row end)
  return 128 + (size_t)a.stages * a.stage_bytes + 2 * (size_t)a.work_floats * 4 + 1024;
}

// One output element of a generic step from a smem plane holding rows [in_lo, ...) (padding
// absent for max / zero for avg).
__device__ __forceinline__ float seq_window(const SeqStepDev& st, const float* pl, int in_lo, int i, int j, int ch,
                                            const float2 (&paff)[kAffSlots]) {
  const bool is_max = st.is_max != 0;
  float acc = is_max ? -CUDART_INF_F : 0.f;
  int real = 0;
  const int r0 = i * st.sh - st.ph, q0 = j * st.sw - st.pw;
  for (int u = 0; u < st.kh; ++u) {
    const int r = r0 + u;
    if ((unsigned)r >= (unsigned)st.H) continue;
    const float* row = pl + (r - in_lo) * st.W;
    for (int v = 0; v < st.kw; ++v) {
      const int q = q0 + v;
      if ((unsigned)q >= (unsigned)st.W) continue;
      float x = row[q];
      if (st.pro.n) x = apply_generic(st.pro, paff, ch, x, 0);
      acc = is_max ? fmaxf(acc, x) : __fadd_rn(acc, x);
      ++real;
    }
  }
  if (!is_max) acc = __fdiv_rn(acc, st.count_include_pad ? (float)(st.kh * st.kw) : (float)real);
  return acc;
}

// Per-step constants, hoisted into shared memory once per CTA.
struct SeqStepSm {
  int32_t H, W, Ho, Wo;
  int32_t in_pitch, out_pitch;
  int32_t path;                // 0 generic; fast: 1 = 16-lane segments, 2 = 32 lanes x 1, 3 = 32 lanes x 2
  int32_t epi;                 // fast epilogue: 0 none, 1 ReLU, 2 BN, 3 BN -> ReLU
  const float2* aff;           // (scale, shift) per channel
};

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));   // FMNMX3
  return r;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const float4& v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// One fast step over the np planes of a tile (see the header).  Half-items (plane, row chunk,
// column segment) are dealt to the warps; a SEG = 16 warp walks two at once (one per half).
template <int SEG, int NSEG, bool LAST, int EPI>
__device__ __forceinline__ void seq_fast_step(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                              float* gout, int np, uint32_t plane_base, const FastDiv& cdiv, int C,
                                              int cw, int lane) {
  constexpr int PER_WARP = 32 / SEG;
  const int W = f.W;
  const int sl = lane & (SEG - 1), half = lane / SEG;
  const int n_half = np * rg.n_chunks * NSEG;
  const int n_units = (n_half + PER_WARP - 1) / PER_WARP;
  const int lo_c = rg.in_lo, hi_c = rg.in_hi - 1;       // clamp range of input rows (= plane edges)
  const uint32_t W4 = 4u * (uint32_t)W;
  for (int u = cw; u < n_units; u += kSeqWarps) {
    int hi = u * PER_WARP + half;
    const bool item_ok = hi < n_half;
    hi = item_ok ? hi : 0;
    const int sg = NSEG == 1 ? 0 : hi % NSEG;
    const uint32_t rest = (uint32_t)(NSEG == 1 ? hi : hi / NSEG);
    const int p = (int)fdiv(rest, rg.chunks);
    const int chk = (int)rest - p * rg.n_chunks;
    const int c = sg * 4 * SEG + 4 * sl;
    const bool col_ok = c < W;
    const int r0 = rg.out_lo + chk * rg.L;
    const int r1 = min(rg.out_hi, r0 + rg.L);
    float2 aff = make_float2(1.f, 0.f);
    if (EPI >= 2) {
      const uint32_t plane = plane_base + (uint32_t)p;
      const int ch = (int)(plane - fdiv(plane, cdiv) * (uint32_t)C);
      aff = __ldg(f.aff + ch);
    }
    const uint32_t rowbase = in_s + 4u * (uint32_t)(p * f.in_pitch + c);
    auto hrow = [&](int r) -> float4 {
      r = min(max(r, lo_c), hi_c);
      const uint32_t ad = rowbase + (uint32_t)(r - rg.in_lo) * W4;
      const float4 x = lds128(ad);
      float l = __shfl_up_sync(0xffffffffu, x.w, 1, SEG);
      float rr = __shfl_down_sync(0xffffffffu, x.x, 1, SEG);
      if (NSEG > 1) {   // neighbours across segment boundaries come from shared memory
        if (sl == 0 && c > 0) l = lds_f32(ad - 4u);
        if (sl == SEG - 1 && c + 4 < W) rr = lds_f32(ad + 16u);
      }
      l = c == 0 ? x.x : l;
      rr = c + 4 >= W ? x.w : rr;
      return make_float4(max3f(l, x.x, x.y), max3f(x.x, x.y, x.z), max3f(x.y, x.z, x.w), max3f(x.z, x.w, rr));
    };
    auto epi = [&](float v) -> float {
      if (EPI >= 2) v = __fmaf_rn(v, aff.x, aff.y);
      if (EPI == 1 || EPI == 3) v = relu(v);
      return v;
    };
    float4 hA = hrow(r0 - 1), hB = hrow(r0);
    float* og = LAST ? gout + (size_t)p * ((size_t)f.H * W) + (size_t)r0 * W + c : nullptr;
    uint32_t os = out_s + 4u * (uint32_t)(p * f.out_pitch + (r0 - rg.out_lo) * W + c);
    const bool st_ok = item_ok && col_ok;
#pragma unroll 2
    for (int i = 0; i < rg.L; ++i) {
      const float4 hC = hrow(r0 + i + 1);
      float4 o;
      o.x = epi(max3f(hA.x, hB.x, hC.x));
      o.y = epi(max3f(hA.y, hB.y, hC.y));
      o.z = epi(max3f(hA.z, hB.z, hC.z));
      o.w = epi(max3f(hA.w, hB.w, hC.w));
      if (st_ok && r0 + i < r1) {
        if (LAST) st_stream4(og, o);
        else sts128(os, o);
      }
      if (LAST) og += W;
      else os += W4;
      hA = hB;
      hB = hC;
    }
  }
}

template <bool LAST, int EPI>
__device__ __forceinline__ void seq_fast_paths(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                               float* gout, int np, uint32_t pb, const FastDiv& cdiv, int C, int cw,
                                               int lane) {
  if (f.path == 1) seq_fast_step<16, 1, LAST, EPI>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane);
  else if (f.path == 2) seq_fast_step<32, 1, LAST, EPI>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane);
  else seq_fast_step<32, 2, LAST, EPI>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane);
}

template <bool LAST>
__device__ __forceinline__ void seq_fast(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                         float* gout, int np, uint32_t pb, const FastDiv& cdiv, int C, int cw,
                                         int lane) {
  switch (f.epi) {
    case 0: seq_fast_paths<LAST, 0>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane); break;
    case 1: seq_fast_paths<LAST, 1>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane); break;
    case 2: seq_fast_paths<LAST, 2>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane); break;
    default: seq_fast_paths<LAST, 3>(f, rg, in_s, out_s, gout, np, pb, cdiv, C, cw, lane); break;
  }
}

__global__ void __launch_bounds__(kSeqThreads) seq_staged(SeqArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ SeqStepSm tab[kMaxSeqSteps];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  unsigned char* stage0 = smem + 128;
  // the two ping-pong work buffers (selected by arithmetic, not a local array: no local memory)
  float* const work0 = (float*)(stage0 + (size_t)a.stages * a.stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = a.n_tiles;
  const int HW0 = a.in_plane;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();                   // previous kernel on the stream complete + visible
  pdl_launch_dependents();

  if (warp == 0) {  // producer: one elected lane bulk-copies each tile's input rows
    if (lane == 0) {
      const int W_in = a.steps[0].W;
      int k = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % a.stages;
        if (k >= a.stages) mbar_wait_sleep(&empty[s], ((k / a.stages) - 1) & 1);
        const int64_t pg = t / a.n_bands;
        const int band = (int)(t - pg * a.n_bands);
        const SeqRange rg = a.ranges[(size_t)band * a.n_steps];
        const int64_t pl0 = pg * a.tile_planes;
        const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
        // whole planes: np contiguous planes; halo tiles (np = 1): rows [in_lo, in_hi) of one plane
        const float* src = a.in + (a.plane0 + pl0) * (int64_t)HW0 + (int64_t)rg.in_lo * W_in;
        const uint32_t head_off = (uint32_t)((uintptr_t)src & 15u);
        float* dst = (float*)((char*)stage0 + (size_t)s * a.stage_bytes + head_off);
        const uint32_t nbytes = (uint32_t)np * (uint32_t)(rg.in_hi - rg.in_lo) * (uint32_t)W_in * 4u;
        const uint32_t h = min(nbytes, (16u - head_off) & 15u);
        const uint32_t body = (nbytes - h) & ~15u;
        for (uint32_t e = 0; e < h / 4; ++e) cp_async4(dst + e, src + e);
        for (uint32_t e = (h + body) / 4; e < nbytes / 4; ++e) cp_async4(dst + e, src + e);
        cp_async_mbar_arrive(&full[s]);
        if (body) {
          mbar_arrive_expect_tx(&full[s], body);
          for (uint32_t off = 0; off < body; off += kBulkChunk)
            bulk_g2s((char*)dst + h + off, (const char*)src + h + off, min(kBulkChunk, body - off), &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
    }
    return;
  }

  const int cw = warp - 1;   // consumer warp 0..7
  for (int i = threadIdx.x - 32; i < a.n_steps; i += 32 * kSeqWarps) {
    const SeqStepDev& st = a.steps[i];
    SeqStepSm f;
    f.H = st.H; f.W = st.W; f.Ho = st.Ho; f.Wo = st.Wo;
    f.in_pitch = st.in_pitch;
    f.out_pitch = st.out_pitch;
    f.path = !st.fast ? 0 : st.W <= 64 ? 1 : st.W <= 128 ? 2 : 3;
    const bool aff = st.epi_class == PC_AFFINE || st.epi_class == PC_AFFINE_RELU;
    const bool rl = st.epi_class == PC_RELU || st.epi_class == PC_AFFINE_RELU;
    f.epi = (aff ? 2 : 0) + (rl ? 1 : 0);
    f.aff = aff ? st.epi.affine[0] : nullptr;
    tab[i] = f;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");
  const int W_in = tab[0].W;
  int k = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int s = k % a.stages;
    mbar_wait_sleep(&full[s], (k / a.stages) & 1);
    const int64_t pg = t / a.n_bands;
    const int band = (int)(t - pg * a.n_bands);
    const SeqRange* rgs = a.ranges + (size_t)band * a.n_steps;
    const int64_t pl0 = pg * a.tile_planes;
    const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
    const float* src_base = (const float*)((const char*)stage0 + (size_t)s * a.stage_bytes +
                                           ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW0 +
                                                        (int64_t)rgs[0].in_lo * W_in) & 15u));
    const uint32_t pbase = (uint32_t)(a.plane0 + pl0);
    for (int st_i = 0; st_i < a.n_steps; ++st_i) {
      const SeqStepSm& f = tab[st_i];
      const SeqRange rg = rgs[st_i];
      const bool last = st_i == a.n_steps - 1;
      const float* in_buf = st_i == 0 ? src_base : work0 + ((st_i - 1) & 1) * a.work_floats;
      float* out_buf = work0 + (st_i & 1) * a.work_floats;
      const int64_t HWo = (int64_t)f.Ho * f.Wo;
      float* gout = a.out + (a.plane0 + pl0) * HWo;
      if (f.path) {
        const uint32_t in_s = smem_u32(in_buf), out_s = smem_u32(out_buf);
        if (last) seq_fast<true>(f, rg, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
        else seq_fast<false>(f, rg, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
      } else {
        const SeqStepDev& st = a.steps[st_i];
        // work items: (plane, output row, 32-column chunk); lane = output column
        const int nchunk = (f.Wo + 31) / 32;
        const int nrows = rg.out_hi - rg.out_lo;
        const int items = np * nrows * nchunk;
        for (int it = cw; it < items; it += kSeqWarps) {
          const int cc = it % nchunk;
          const int i = rg.out_lo + (it / nchunk) % nrows;
          const int p = it / (nchunk * nrows);
          const int j = cc * 32 + lane;
          if (j >= f.Wo) continue;
          const int64_t plane = a.plane0 + pl0 + p;
          const int ch = (int)(plane % a.C);
          float2 paff[kAffSlots], eaff[kAffSlots];
          load_affine(st.pro, ch, paff);
          load_affine(st.epi, ch, eaff);
          float r = seq_window(st, in_buf + (size_t)p * f.in_pitch, rg.in_lo, i, j, ch, paff);
          r = apply_generic(st.epi, eaff, ch, r, 0);
          if (last) __stcs(gout + p * HWo + (int64_t)i * f.Wo + j, r);
          else out_buf[(size_t)p * f.out_pitch + (i - rg.out_lo) * f.Wo + j] = r;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");   // step boundary
      if (st_i == 0 && cw == 0 && lane == 0) mbar_arrive(&empty[s]);      // stage buffer consumed
    }
  }
}

cudaError_t launch_seq(const SeqArgs& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  const size_t smem = seq_smem(a);
  return launch_pdl((void*)seq_staged, dim3(grid), dim3(kSeqThreads), args, smem, st);
}

int seq_max_blocks_per_sm(const SeqArgs& a) {
  const size_t smem = seq_smem(a);
  int n = 0;
  if (smem_kernel_setup((const void*)seq_staged) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (void*)seq_staged, kSeqThreads, smem) != cudaSuccess) n = 0;
  return n;
}

}  // namespace bs
