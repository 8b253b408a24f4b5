// k_seq.cu -- on-chip multi-step sequences (NEXT-2), whole-plane or halo (row-band) tiles.
#include "bs_device.cuh"

namespace bs {

// ------------------------------------------------------------------ multi-step sequences
//
// NEXT-2: a *sequence* of several steps runs on-chip (PAPER.md P:L545-558,
// lst:finalcode P:L512-530 "float cached_data[...]"; the paper's GPU kernel swapped two smem
// buffers per step).  Two kernels:
//  * seq_inplace (below; the planner's choice for §5.1-type sequences on whole planes <= 224
//    wide): warp groups own planes for the whole sequence and sweep them in place, two steps per
//    sweep;
//  * seq_staged (this section; every other sequence): a tile is bulk-copied (TMA,
//    cp.async.bulk) into a ring stage; its steps ping-pong between the stage and ONE work buffer,
//    and only the last step writes HBM.  A named barrier over the 8 consumer warps separates steps.
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

// Per-tile tables in shared memory: the tile's row ranges of every step and the folded BN
// (scale, shift) of every (step, plane) -- loaded once per tile, all at once, instead of one
// dependent global load per step.
__host__ __device__ inline size_t seq_table_bytes(int n_steps, int tile_planes) {
  return ((size_t)n_steps * sizeof(SeqRange) + (size_t)n_steps * tile_planes * sizeof(float2) + 127) / 128 * 128;
}

size_t seq_smem(const SeqArgs& a) {
  // barriers | stages | work buffer | per-tile tables | 1 KB slack (vector loads of idle lanes
  // past a row end)
  return 128 + (size_t)a.stages * a.stage_bytes + (size_t)a.work_floats * 4 +
         seq_table_bytes(a.n_steps, a.tile_planes) + 1024;
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
// Predicated LDS.128: lanes past the row end (idle columns) load nothing (they would read other
// threads' rows or tables; their values only feed outputs that are never stored or replaced).
__device__ __forceinline__ float4 lds128_if(bool p, uint32_t a) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %4, 0;\n@q ld.shared.v4.f32 {%0,%1,%2,%3}, [%5];\n}\n"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
      : "r"((uint32_t)p), "r"(a));
  return v;
}
// Clean steps: every lane keeps its natural row address; a pad lane's loads are redirected into a
// 128-B block of -inf at the same offset mod 128 -- the same bank group, so a quarter-warp's
// LDS.128 stays conflict-free -- by one LOP3: (a & msk) | orv, msk = ~0 / orv = 0 for real lanes.
struct PadLd {
  uint32_t msk, orv;
  __device__ __forceinline__ float4 operator()(uint32_t a) const { return lds128((a & msk) | orv); }
};
__device__ __forceinline__ void sts128(uint32_t a, const float4& v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// One fast step over the np planes of a tile (see the header).  Half-items (plane, row chunk,
// column segment) are dealt to the warps; a SEG = 16 warp walks two at once (one per half).
template <int SEG, int NSEG, bool LAST, int EPI>
__device__ __forceinline__ void seq_fast_step(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                              float* gout, int np, const float2* taff, int cw, int lane) {
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
    const float2 aff = EPI >= 2 ? taff[p] : make_float2(1.f, 0.f);
    const uint32_t rowbase = in_s + 4u * (uint32_t)(p * f.in_pitch + c);
    // horizontal 3-max of the row at shared address ad (4 columns of this lane)
    auto hrow = [&](uint32_t ad) -> float4 {
      const float4 x = lds128_if(col_ok, ad);
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
    // rows r0-1 and r0 prime the window (clamped at the plane's top edge: a duplicate row); rows
    // r0+1 .. r0+L are streamed, only the last of them can pass the bottom edge (clamped by an
    // address select).  Three row registers rotate through an unrolled-by-3 loop (no moves).
    const uint32_t ad0 = rowbase + (uint32_t)(r0 - rg.in_lo) * W4;
    float4 hA = hrow(r0 - 1 >= lo_c ? ad0 - W4 : ad0);
    float4 hB = hrow(ad0);
    float4 hC;
    uint32_t ad = ad0;
    const uint32_t ad_last = rowbase + (uint32_t)(hi_c - rg.in_lo) * W4;   // the bottom input row
    float* og = LAST ? gout + (size_t)p * ((size_t)f.H * W) + (size_t)r0 * W + c : nullptr;
    uint32_t os = out_s + 4u * (uint32_t)(p * f.out_pitch + (r0 - rg.out_lo) * W + c);
    const bool st_ok = item_ok && col_ok;
    const int n_ok = st_ok ? r1 - r0 : 0;    // rows this lane stores
    auto row = [&](int i, const float4& a, const float4& b, float4& nx) {
      ad += W4;
      nx = hrow(min(ad, ad_last));
      float4 o;
      o.x = epi(max3f(a.x, b.x, nx.x));
      o.y = epi(max3f(a.y, b.y, nx.y));
      o.z = epi(max3f(a.z, b.z, nx.z));
      o.w = epi(max3f(a.w, b.w, nx.w));
      if (i < n_ok) {
        if (LAST) st_stream4(og, o);
        else sts128(os, o);
      }
      if (LAST) og += W;
      else os += W4;
    };
    int i = 0;
    for (; i + 3 <= rg.L; i += 3) {
      row(i, hA, hB, hC);
      row(i + 1, hB, hC, hA);
      row(i + 2, hC, hA, hB);
    }
    if (i < rg.L) {
      row(i, hA, hB, hC);
      if (i + 1 < rg.L) row(i + 1, hB, hC, hA);
    }
  }
}

template <bool LAST, int EPI>
__device__ __forceinline__ void seq_fast_paths(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                               float* gout, int np, const float2* taff, int cw, int lane) {
  if (f.path == 1) seq_fast_step<16, 1, LAST, EPI>(f, rg, in_s, out_s, gout, np, taff, cw, lane);
  else if (f.path == 2) seq_fast_step<32, 1, LAST, EPI>(f, rg, in_s, out_s, gout, np, taff, cw, lane);
  else seq_fast_step<32, 2, LAST, EPI>(f, rg, in_s, out_s, gout, np, taff, cw, lane);
}

template <bool LAST>
__device__ __forceinline__ void seq_fast(const SeqStepSm& f, const SeqRange& rg, uint32_t in_s, uint32_t out_s,
                                         float* gout, int np, const float2* taff, int cw, int lane) {
  switch (f.epi) {
    case 0: seq_fast_paths<LAST, 0>(f, rg, in_s, out_s, gout, np, taff, cw, lane); break;
    case 1: seq_fast_paths<LAST, 1>(f, rg, in_s, out_s, gout, np, taff, cw, lane); break;
    case 2: seq_fast_paths<LAST, 2>(f, rg, in_s, out_s, gout, np, taff, cw, lane); break;
    default: seq_fast_paths<LAST, 3>(f, rg, in_s, out_s, gout, np, taff, cw, lane); break;
  }
}

__global__ void __launch_bounds__(kSeqThreads) seq_staged(SeqArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ SeqStepSm tab[kMaxSeqSteps];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  unsigned char* stage0 = smem + 128;
  // steps ping-pong between the tile's stage and one work buffer: step k reads the stage (k even)
  // or the work buffer (k odd) and writes the other, so a tile needs its stage + 1 buffer
  float* const work = (float*)(stage0 + (size_t)a.stages * a.stage_bytes);
  SeqRange* const t_rg = (SeqRange*)(work + (size_t)a.work_floats);               // [n_steps]
  float2* const t_aff = (float2*)(t_rg + a.n_steps);                               // [n_steps][P]
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
    const uint32_t pbase = (uint32_t)(a.plane0 + pl0);
    // tile prologue: every step's row ranges and (scale, shift) per plane into shared memory, all
    // loads in flight at once (the previous tile's last step ended with a CTA barrier)
    {
      const int tid = threadIdx.x - 32;
      for (int i = tid; i < a.n_steps; i += 32 * kSeqWarps) t_rg[i] = rgs[i];
      for (int i = tid; i < a.n_steps * np; i += 32 * kSeqWarps) {
        const int st = i / np, p = i - st * np;
        const float2* aff = tab[st].aff;
        if (aff) {
          const uint32_t plane = pbase + (uint32_t)p;
          t_aff[st * a.tile_planes + p] = __ldg(aff + (plane - fdiv(plane, a.cdiv) * (uint32_t)a.C));
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");
    }
    float* const stage = (float*)((char*)stage0 + (size_t)s * a.stage_bytes);
    const float* src_base = (const float*)((const char*)stage +
                                           ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW0 +
                                                        (int64_t)t_rg[0].in_lo * W_in) & 15u));
    for (int st_i = 0; st_i < a.n_steps; ++st_i) {
      const SeqStepSm& f = tab[st_i];
      const SeqRange rg = t_rg[st_i];
      const bool last = st_i == a.n_steps - 1;
      const float* in_buf = st_i == 0 ? src_base : (st_i & 1) ? work : stage;
      float* out_buf = (st_i & 1) ? stage : work;
      const int64_t HWo = (int64_t)f.Ho * f.Wo;
      float* gout = a.out + (a.plane0 + pl0) * HWo;
      if (f.path) {
        const uint32_t in_s = smem_u32(in_buf), out_s = smem_u32(out_buf);
        const float2* taff = t_aff + st_i * a.tile_planes;
        if (last) seq_fast<true>(f, rg, in_s, out_s, gout, np, taff, cw, lane);
        else seq_fast<false>(f, rg, in_s, out_s, gout, np, taff, cw, lane);
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
    }
    if (cw == 0 && lane == 0) mbar_arrive(&empty[s]);   // the tile's stage is free for the producer
  }
}

// ------------------------------------------------------------------ in-place, warp per plane
//
// Sequences made only of fast steps (the §5.1 block) on whole planes (W <= 224): one or a few
// consumer warps own a plane of the tile for the WHOLE sequence, so steps need no CTA barrier and
// no work buffer.  The plane's rows are cut into parts, one per half-warp (16-lane segments,
// W <= 64) or warp; parts of one plane in different warps meet at a named barrier twice per sweep
// (after each part has read its neighbours' boundary rows, and at the end).  A sweep runs down a
// part's rows in place: output row i is written over input row i after the rows below it that
// its window needs have been loaded, and the rows above are only needed as horizontal maxima
// already held in registers; a lane loads and stores only its own columns (neighbour columns
// arrive by shuffle from the same load), so nothing is overwritten before it is read.  The
// exceptions are the rows just outside a part, which a neighbouring part overwrites: they are read
// once, before any part writes.  Loads run one row ahead.  Shared memory per tile is the stage
// alone, so several CTAs share an SM and the bulk copy of one CTA's next tile overlaps the other
// CTAs' steps (planes 129..224 wide: one plane per CTA).  Three step kernels below: the one-step
// sweep with edge selects (inplace_step, any part heights), and the clean one-step and two-step
// sweeps (inplace_step_clean, inplace_pair_clean: -inf pad lanes or edge selects, 1 or 2 column
// segments).
// One in-place step of one row part [r0, r0 + Hp) of a plane (Hp rows per part; the last part may
// have fewer).  bar_id > 0: the plane's parts live in several warps (named barrier over them).
template <int SEG, bool LAST, int EPI>
__device__ __forceinline__ void inplace_step(uint32_t pbase, float* og, int H, int W, int c, bool st_ok, float2 aff,
                                             int r0, int Hp, int bar_id, int bar_threads) {
  const uint32_t W4 = 4u * (uint32_t)W;
  auto hraw = [&](const float4& x) -> float4 {
    float l = __shfl_up_sync(0xffffffffu, x.w, 1, SEG);
    float rr = __shfl_down_sync(0xffffffffu, x.x, 1, SEG);
    l = c == 0 ? x.x : l;
    rr = c + 4 >= W ? x.w : rr;
    return make_float4(max3f(l, x.x, x.y), max3f(x.x, x.y, x.z), max3f(x.y, x.z, x.w), max3f(x.z, x.w, rr));
  };
  auto epi = [&](float v) -> float {
    if (EPI >= 2) v = __fmaf_rn(v, aff.x, aff.y);
    if (EPI == 1 || EPI == 3) v = relu(v);
    return v;
  };
  const bool col_ok = c < W;
  auto lds128 = [&](uint32_t a) { return lds128_if(col_ok, a); };
  const int rows = max(0, min(H, r0 + Hp) - r0);       // rows this part outputs
  const uint32_t bottom = pbase + (uint32_t)(H - 1) * W4;
  auto rad = [&](int r) -> uint32_t { return pbase + (uint32_t)min(max(r, 0), H - 1) * W4; };   // clamped
  // everything this part reads from outside its own rows, before any part writes
  const float4 x_bound = lds128(rad(r0 + Hp));         // the row below the part (or the bottom row)
  float4 hA = hraw(lds128(rad(r0 - 1)));               // the row above (a duplicate at the top edge)
  float4 hB = hraw(lds128(rad(r0)));
  float4 x1 = lds128(rad(r0 + 1));                     // raw row r0 + 1, one ahead
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();                                   // the other half-warp's part
  uint32_t ad = rad(r0);
  float* o_g = LAST ? og + (size_t)r0 * W : nullptr;
  float4 hC;
  // main rows: rows i + 1 and i + 2 are the part's own (not yet overwritten)
  auto row = [&](int i, const float4& a, const float4& b, float4& nx) {
    const float4 x2 = lds128(min(ad + 2u * W4, bottom));   // raw row i + 2, before row i is overwritten
    nx = hraw(x1);                                         // row i + 1
    x1 = x2;
    float4 o;
    o.x = epi(max3f(a.x, b.x, nx.x));
    o.y = epi(max3f(a.y, b.y, nx.y));
    o.z = epi(max3f(a.z, b.z, nx.z));
    o.w = epi(max3f(a.w, b.w, nx.w));
    if (st_ok && i < rows) {
      if (LAST) st_stream4(o_g, o);
      else sts128(ad, o);
    }
    if (LAST) o_g += W;
    ad += W4;
  };
  int i = 0;
  for (; i + 5 <= Hp; i += 3) {
    row(i, hA, hB, hC);
    row(i + 1, hB, hC, hA);
    row(i + 2, hC, hA, hB);
  }
  // the last rows: row i + 1 / i + 2 may lie below the part -> the row saved before the step
  for (; i < Hp; ++i) {
    const float4 x2 = i + 2 < Hp ? lds128(min(ad + 2u * W4, bottom)) : x_bound;
    hC = hraw(i + 1 < Hp ? x1 : x_bound);
    x1 = x2;
    float4 o;
    o.x = epi(max3f(hA.x, hB.x, hC.x));
    o.y = epi(max3f(hA.y, hB.y, hC.y));
    o.z = epi(max3f(hA.z, hB.z, hC.z));
    o.w = epi(max3f(hA.w, hB.w, hC.w));
    if (st_ok && i < rows) {
      if (LAST) st_stream4(o_g, o);
      else sts128(ad, o);
    }
    if (LAST) o_g += W;
    ad += W4;
    hA = hB;
    hB = hC;
  }
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();
}

// The same step for the common shapes (56 x 56, 112 x 112 and 224 x 224 planes): every part has
// the same Hp >= 2 rows (H % parts == 0) and a lane segment holds its column groups with a free
// lane on either side.  Column group g of segment s sits on lane g - first(s) + 1; the side
// lanes hold the neighbouring group of the next segment (a halo, read only) or, at the plane's
// edges, -inf (PadLd: the max identity); neither stores.  So the outer neighbours of every
// column arrive by the same two shuffles -- no edge selects, no predicated loads.  NSEG = 2
// segments (planes 129..224 wide, 8 warps per plane) cover a row with 2 x 28 groups; one warp
// walks both in lockstep, so a row is read (both segments, halos included) before it is
// overwritten.  Rows below the part are never touched inside the loop (no address clamps): the
// main loop stops two rows before the part's end, the last two rows take the own last row and
// the row saved below.  Per 4 outputs and row: LDS.128, 2 SHFL, 8 FMNMX3, the epilogue,
// STS.128 (STG.128 on the last step), one address add.
template <int N>
struct Vec4 {
  float4 s[N];
};
// A lane's segments: byte offset of segment s's column from segment 0's, its loads (pad lanes
// redirected to -inf), whether it holds plane data and whether it stores.  E (edge selects): rows
// that fill their segment have no free lanes for -inf pads; the plane's edge columns then take
// their missing neighbour from themselves (a duplicate, exact for max; le / re mark those lanes).
template <int N, bool E = false>
struct SegLanes {
  uint32_t off[N];
  PadLd ld[N];
  bool col_ok[N], st_ok[N];
  bool le[N], re[N];
};

template <int SEG, int N, bool E>
__device__ __forceinline__ Vec4<N> seg_hraw(const Vec4<N>& x, const SegLanes<N, E>& L) {
  Vec4<N> h;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const float4 v = x.s[q];
    float l = __shfl_up_sync(0xffffffffu, v.w, 1, SEG);
    float rr = __shfl_down_sync(0xffffffffu, v.x, 1, SEG);
    if (E) {
      l = L.le[q] ? v.x : l;
      rr = L.re[q] ? v.w : rr;
    }
    h.s[q] = make_float4(max3f(l, v.x, v.y), max3f(v.x, v.y, v.z), max3f(v.y, v.z, v.w), max3f(v.z, v.w, rr));
  }
  return h;
}
template <int N, bool E>
__device__ __forceinline__ Vec4<N> seg_ld(const SegLanes<N, E>& L, uint32_t a) {
  Vec4<N> v;
#pragma unroll
  for (int q = 0; q < N; ++q) v.s[q] = L.ld[q](q ? a + L.off[q] : a);
  return v;
}
template <bool LAST, int N, bool E>
__device__ __forceinline__ void seg_store(const SegLanes<N, E>& L, uint32_t ad, float* og, const Vec4<N>& o) {
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (L.st_ok[q]) {
      if (LAST) st_stream4(q ? og + L.off[q] / 4 : og, o.s[q]);
      else sts128(q ? ad + L.off[q] : ad, o.s[q]);
    }
}

template <int SEG, int N, bool LAST, int EPI, bool E, bool BAND>
__device__ __forceinline__ void inplace_step_clean(uint32_t pbase, const SegLanes<N, E>& L, float* og, int H, int W,
                                                   float2 aff, int r0, int Hp, int bar_id, int bar_threads, int slo,
                                                   int shi) {
  const uint32_t W4 = 4u * (uint32_t)W;
  auto epi = [&](float v) -> float {
    if (EPI >= 2) v = __fmaf_rn(v, aff.x, aff.y);
    if (EPI == 1 || EPI == 3) v = relu(v);
    return v;
  };
  uint32_t ad = pbase + (uint32_t)r0 * W4;
  // everything this part reads from outside its own rows, before any part writes
  const Vec4<N> x_bound = seg_ld(L, r0 + Hp < H ? ad + (uint32_t)Hp * W4 : ad + (uint32_t)(Hp - 1) * W4);
  Vec4<N> hA = seg_hraw<SEG>(seg_ld(L, r0 > 0 ? ad - W4 : ad), L);   // the row above (a duplicate at the top)
  Vec4<N> hB = seg_hraw<SEG>(seg_ld(L, ad), L);
  Vec4<N> x1 = seg_ld(L, ad + W4);                                // raw row r0 + 1 (Hp >= 2: the part's own)
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();                                 // the other half-warp's part
  float* o_g = LAST ? og + (size_t)r0 * W : nullptr;
  int orow = r0;                                      // the row being output (the last step stores [slo, shi))
  Vec4<N> hC;
  auto out = [&](const Vec4<N>& a, const Vec4<N>& b, const Vec4<N>& c) {
    Vec4<N> o;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      o.s[q].x = epi(max3f(a.s[q].x, b.s[q].x, c.s[q].x));
      o.s[q].y = epi(max3f(a.s[q].y, b.s[q].y, c.s[q].y));
      o.s[q].z = epi(max3f(a.s[q].z, b.s[q].z, c.s[q].z));
      o.s[q].w = epi(max3f(a.s[q].w, b.s[q].w, c.s[q].w));
    }
    if (!LAST || !BAND || (orow >= slo && orow < shi)) seg_store<LAST>(L, ad, o_g, o);
    if (LAST) { o_g += W; ++orow; }
    ad += W4;
  };
  // output row i (i + 2 < Hp): raw row i + 2 is loaded before row i is overwritten
  auto row = [&](const Vec4<N>& a, const Vec4<N>& b, Vec4<N>& nx) {
    const Vec4<N> x2 = seg_ld(L, ad + 2u * W4);
    nx = seg_hraw<SEG>(x1, L);
    x1 = x2;
    out(a, b, nx);
  };
  const int n_main = Hp - 2;
  int i = 0;
  for (; i + 3 <= n_main; i += 3) {
    row(hA, hB, hC);
    row(hB, hC, hA);
    row(hC, hA, hB);
  }
  // 0..2 main rows left, then the part's last two rows (own row Hp - 1 in x1, then the row below)
  const int rem = n_main - i;
  if (rem == 0) {
    hC = seg_hraw<SEG>(x1, L);       out(hA, hB, hC);
    hA = seg_hraw<SEG>(x_bound, L);  out(hB, hC, hA);
  } else if (rem == 1) {
    row(hA, hB, hC);
    hA = seg_hraw<SEG>(x1, L);       out(hB, hC, hA);
    hB = seg_hraw<SEG>(x_bound, L);  out(hC, hA, hB);
  } else {
    row(hA, hB, hC);
    row(hB, hC, hA);
    hB = seg_hraw<SEG>(x1, L);       out(hC, hA, hB);
    hC = seg_hraw<SEG>(x_bound, L);  out(hA, hB, hC);
  }
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();
}

// Two consecutive steps k, k + 1 in ONE sweep down a part's rows (temporal blocking): shared
// memory is read and written once per two steps instead of once per step, and the step-k rows
// never leave registers.  While the sweep stands on row i it takes raw row i + 2 (loaded one row
// ahead), makes step-k row y[i + 1] from the raw rows' horizontal maxima h[i .. i + 2], takes
// y[i + 1]'s horizontal maxima g[i + 1] (two more shuffles), and writes step-(k+1) row z[i] from
// g[i - 1 .. i + 1] over raw row i, which nothing needs any more.  The part's edges need two raw
// rows on either side (read before any part writes) and one redundant y row on either side; at
// the plane's top / bottom edge the step-k row beyond the plane is absent, i.e. g[-1] := g[0] and
// g[H] := g[H - 1] (duplicates, exact for max).  A halo lane's step-k value is exact for its
// inner column (its neighbour inside the segment is real), the only one the segment needs.
// Epilogues are branch-free per step: v * s + t then max(v, lo), with (s, t) = (1, -0) without
// BN (exact: v + -0 == v, -0 included) and lo = -inf without ReLU.  The window rotates through
// three register roles (no moves): the main loop is unrolled by 3 and the part's last 2..5 rows
// are unrolled per remainder.
template <int SEG, int N, bool LAST, bool E, bool BAND>
__device__ __forceinline__ void inplace_pair_clean(uint32_t pbase, const SegLanes<N, E>& L, float* og, int H, int W,
                                                   float2 a1, float lo1, float2 a2, float lo2, int r0, int Hp,
                                                   int bar_id, int bar_threads, int slo, int shi) {
  const uint32_t W4 = 4u * (uint32_t)W;
  // A pad lane's step-k row must stay -inf (its neighbours take it as their outer column), but its
  // horizontal maxima pick up the edge columns through the shuffles: (s, t) = (0, -inf) maps any
  // finite v to -inf and -inf to NaN, which max(., lo = -inf) turns back into -inf.
  float2 a1s[N];
  float lo1s[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    a1s[q] = L.col_ok[q] ? a1 : make_float2(0.f, -CUDART_INF_F);
    lo1s[q] = L.col_ok[q] ? lo1 : -CUDART_INF_F;
  }
  auto vert = [&](const Vec4<N>& a, const Vec4<N>& b, const Vec4<N>& c, bool first) -> Vec4<N> {
    Vec4<N> o;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float2 s = first ? a1s[q] : a2;
      const float lo = first ? lo1s[q] : lo2;
      o.s[q].x = fmaxf(__fmaf_rn(max3f(a.s[q].x, b.s[q].x, c.s[q].x), s.x, s.y), lo);
      o.s[q].y = fmaxf(__fmaf_rn(max3f(a.s[q].y, b.s[q].y, c.s[q].y), s.x, s.y), lo);
      o.s[q].z = fmaxf(__fmaf_rn(max3f(a.s[q].z, b.s[q].z, c.s[q].z), s.x, s.y), lo);
      o.s[q].w = fmaxf(__fmaf_rn(max3f(a.s[q].w, b.s[q].w, c.s[q].w), s.x, s.y), lo);
    }
    return o;
  };
  const bool top = r0 == 0, bot = r0 + Hp == H;
  uint32_t ad = pbase + (uint32_t)r0 * W4;
  // rows outside the part, before any part writes (clamped copies at the plane's edges)
  const Vec4<N> xa2 = seg_ld(L, top ? ad : ad - 2u * W4);
  const Vec4<N> xa1 = seg_ld(L, top ? ad : ad - W4);
  const Vec4<N> xb1 = seg_ld(L, bot ? ad + (uint32_t)(Hp - 1) * W4 : ad + (uint32_t)Hp * W4);
  const Vec4<N> xb2 = seg_ld(L, bot ? ad + (uint32_t)(Hp - 1) * W4 : ad + (uint32_t)(Hp + 1) * W4);
  const Vec4<N> x0 = seg_ld(L, ad), x1 = seg_ld(L, ad + W4);
  Vec4<N> xn = Hp > 2 ? seg_ld(L, ad + 2u * W4) : xb1;   // raw row r0 + 2, one row ahead
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();
  Vec4<N> hA = seg_hraw<SEG>(x0, L), hB = seg_hraw<SEG>(x1, L), hC;
  Vec4<N> gA, gB, gC;
  {
    const Vec4<N> hm2 = seg_hraw<SEG>(xa2, L), hm1 = seg_hraw<SEG>(xa1, L);
    gA = seg_hraw<SEG>(vert(hm2, hm1, hA, true), L);     // g[r0 - 1]
    gB = seg_hraw<SEG>(vert(hm1, hA, hB, true), L);      // g[r0]
    if (top) gA = gB;
  }
  float* o_g = LAST ? og + (size_t)r0 * W : nullptr;
  int orow = r0;                                      // the row being output (the last step stores [slo, shi))
  // z row i from the window; x = raw row i + 2
  auto row = [&](const Vec4<N>& x, const Vec4<N>& ha, const Vec4<N>& hb, Vec4<N>& hc, const Vec4<N>& ga,
                 const Vec4<N>& gb, Vec4<N>& gc, bool bottom_row) {
    hc = seg_hraw<SEG>(x, L);
    gc = seg_hraw<SEG>(vert(ha, hb, hc, true), L);
    if (bottom_row) gc = gb;
    if (!LAST || !BAND || (orow >= slo && orow < shi)) seg_store<LAST>(L, ad, o_g, vert(ga, gb, gc, false));
    if (LAST) { o_g += W; ++orow; }
    ad += W4;
  };
  // rotation phases: P0 = (A, B, C), P1 = (B, C, A), P2 = (C, A, B)
#define BS_ROW0(x, b) row(x, hA, hB, hC, gA, gB, gC, b)
#define BS_ROW1(x, b) row(x, hB, hC, hA, gB, gC, gA, b)
#define BS_ROW2(x, b) row(x, hC, hA, hB, gC, gA, gB, b)
  int i = 0;
  // main rows: the prefetched row i + 3 is the part's own
  for (; i + 3 <= Hp - 3; i += 3) {
    Vec4<N> x = xn; xn = seg_ld(L, ad + 3u * W4); BS_ROW0(x, false);
    x = xn; xn = seg_ld(L, ad + 3u * W4);         BS_ROW1(x, false);
    x = xn; xn = seg_ld(L, ad + 3u * W4);         BS_ROW2(x, false);
  }
  // r own-prefetch rows left (r = Hp - 3 - i in {-1 (Hp == 2), 0, 1, 2}), then the part's last
  // three rows, which take own row Hp - 1 (prefetched), the row below, the row after it
  const int r = Hp - 3 - i;
  if (r < 0) {
    BS_ROW0(xn, false);
    BS_ROW1(xb2, bot);
  } else if (r == 0) {
    BS_ROW0(xn, false);
    BS_ROW1(xb1, false);
    BS_ROW2(xb2, bot);
  } else if (r == 1) {
    Vec4<N> x = xn; xn = seg_ld(L, ad + 3u * W4); BS_ROW0(x, false);
    BS_ROW1(xn, false);
    BS_ROW2(xb1, false);
    BS_ROW0(xb2, bot);
  } else {
    Vec4<N> x = xn; xn = seg_ld(L, ad + 3u * W4); BS_ROW0(x, false);
    x = xn; xn = seg_ld(L, ad + 3u * W4);         BS_ROW1(x, false);
    BS_ROW2(xn, false);
    BS_ROW0(xb1, false);
    BS_ROW1(xb2, bot);
  }
#undef BS_ROW0
#undef BS_ROW1
#undef BS_ROW2
  if (bar_id) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
  else __syncwarp();
}

template <int SEG, bool CLEAN, int N, bool LAST, bool E, bool BAND>
__device__ __forceinline__ void inplace_step_epi(int epi, uint32_t base, const SegLanes<N, E>& L, float* og, int H,
                                                 int W, int c, float2 aff, int r0, int Hp, int bar_id, int bar_threads,
                                                 int slo, int shi) {
  if (CLEAN) {
    switch (epi) {
      case 0: inplace_step_clean<SEG, N, LAST, 0, E, BAND>(base, L, og, H, W, aff, r0, Hp, bar_id, bar_threads, slo, shi); break;
      case 1: inplace_step_clean<SEG, N, LAST, 1, E, BAND>(base, L, og, H, W, aff, r0, Hp, bar_id, bar_threads, slo, shi); break;
      case 2: inplace_step_clean<SEG, N, LAST, 2, E, BAND>(base, L, og, H, W, aff, r0, Hp, bar_id, bar_threads, slo, shi); break;
      default: inplace_step_clean<SEG, N, LAST, 3, E, BAND>(base, L, og, H, W, aff, r0, Hp, bar_id, bar_threads, slo, shi); break;
    }
    return;
  }
  const bool st_ok = L.st_ok[0];
  switch (epi) {
    case 0: inplace_step<SEG, LAST, 0>(base, og, H, W, c, st_ok, aff, r0, Hp, bar_id, bar_threads); break;
    case 1: inplace_step<SEG, LAST, 1>(base, og, H, W, c, st_ok, aff, r0, Hp, bar_id, bar_threads); break;
    case 2: inplace_step<SEG, LAST, 2>(base, og, H, W, c, st_ok, aff, r0, Hp, bar_id, bar_threads); break;
    default: inplace_step<SEG, LAST, 3>(base, og, H, W, c, st_ok, aff, r0, Hp, bar_id, bar_threads); break;
  }
}

// Consumer warps of seq_inplace: 4 (planes <= 128 wide, 1 - 4 per tile), 8 for the two-segment
// rows of planes 129..224 wide (one plane per tile, one CTA per SM).
__host__ __device__ constexpr int inplace_warps_of(int nseg) { return nseg == 2 ? 8 : kInplaceWarps; }
__host__ __device__ inline int inplace_nseg(int W) { return W > 128 ? 2 : 1; }

// Which step seq_inplace runs for these planes: 0 = the one-step kernel (inplace_step: parts of
// unequal height, or < 2 rows), 1 = clean steps with -inf pad lanes, 2 = clean steps with edge
// selects (rows that fill their lane segment: W = 60, 64 with 16-lane segments).
// Clean steps need >= 2 rows per part; the two half-warp parts of a 16-lane-segment warp walk in
// lockstep, so there all parts must be equal; whole-warp parts (32-lane segments) may differ by a
// row (balanced split).
__host__ __device__ inline int inplace_mode(int seg, int tile_planes, int H, int W) {
  if (inplace_nseg(W) == 2) return 1;   // planned only when clean (bs_api.cpp inplace_smem)
  const int parts = (kInplaceWarps / tile_planes) * (32 / seg);
  if (seg == 16 ? (H % parts != 0 || H / parts < 2) : H < 2 * parts) return 0;
  return W / 4 + 2 <= seg ? 1 : 2;
}

template <int SEG, int MODE, int NSEG, bool BAND>
__global__ void __launch_bounds__(32 * (inplace_warps_of(NSEG) + 1), NSEG == 2 ? 1 : 4) seq_inplace(SeqArgs a) {
  constexpr int WARPS = inplace_warps_of(NSEG);
  constexpr bool CLEAN = MODE != 0, EDGE = MODE == 2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int8_t epi_tab[kMaxSeqSteps];
  __shared__ const float2* aff_tab[kMaxSeqSteps];
  __shared__ __align__(128) float4 s_ninf[8];          // the clean steps' pad lanes read this
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  unsigned char* stage0 = smem + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = a.n_tiles;
  const int H = a.steps[0].H, W = a.steps[0].W, HW = a.in_plane;
  const int n = a.n_steps;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 32 * WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 8) s_ninf[threadIdx.x] = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const SeqStepDev& st = a.steps[i];
    const bool aff = st.epi_class == PC_AFFINE || st.epi_class == PC_AFFINE_RELU;
    const bool rl = st.epi_class == PC_RELU || st.epi_class == PC_AFFINE_RELU;
    epi_tab[i] = (int8_t)((aff ? 2 : 0) + (rl ? 1 : 0));
    aff_tab[i] = aff ? st.epi.affine[0] : nullptr;
  }
  __syncthreads();
  pdl_wait();                   // previous kernel on the stream complete + visible
  pdl_launch_dependents();

  if (warp == 0) {  // producer: one elected lane bulk-copies each tile's planes
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % a.stages;
        if (k >= a.stages) mbar_wait_sleep(&empty[s], ((k / a.stages) - 1) & 1);
        // whole planes: np contiguous planes; band tiles (n_bands > 1, one plane): rows [in_lo, in_hi)
        const int64_t pg = t / a.n_bands;
        const int band = (int)(t - pg * a.n_bands);
        const SeqRange rg = a.ranges[(size_t)band * n];
        const int64_t pl0 = pg * a.tile_planes;
        const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
        const float* src = a.in + (a.plane0 + pl0) * (int64_t)HW + (a.n_bands > 1 ? (int64_t)rg.in_lo * W : 0);
        const uint32_t head_off = (uint32_t)((uintptr_t)src & 15u);
        float* dst = (float*)((char*)stage0 + (size_t)s * a.stage_bytes + head_off);
        const uint32_t nbytes = (uint32_t)np * (uint32_t)(a.n_bands > 1 ? (rg.in_hi - rg.in_lo) * W : HW) * 4u;
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

  // warps_per_plane (= WARPS / tile_planes) consumer warps share a plane; its rows are cut into
  // warps_per_plane * 32/SEG parts, one per half-warp (16-lane segments) or warp
  const int cw = warp - 1;
  const int wpp = WARPS / a.tile_planes;
  const int sl = lane & (SEG - 1), half = lane / SEG;
  const int c = 4 * (MODE == 1 ? sl - 1 : sl);        // -inf pads: lane 0 of a segment is a pad / halo
  const int part = (cw % wpp) * (32 / SEG) + half;
  const int n_parts = wpp * (32 / SEG);
  const int Hp = (H + n_parts - 1) / n_parts;          // one-step kernel: equal parts (the last shorter)
  const int bar_id = wpp > 1 ? 1 + cw / wpp : 0;       // named barrier of the plane's warps
  float2* const t_aff = (float2*)(stage0 + (size_t)a.stages * a.stage_bytes) + (size_t)cw * n;   // this warp's
  // column segments: NSEG = 2 splits a row's W / 4 groups into two halves of GS groups
  const int GS = NSEG == 2 ? (W / 4 + 1) / 2 : 0;
  int k = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int s = k % a.stages;
    const int64_t pg = t / a.n_bands;
    const int band = (int)(t - pg * a.n_bands);
    const int64_t pl0 = pg * a.tile_planes;
    const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
    const int p = cw / wpp;                             // this warp's plane in the tile
    // the tile's rows: a whole plane, or a band [in_lo, in_hi) of one plane (halo tiles, clean
    // steps only): the band is swept like a plane whose edges are the band's; a non-plane band
    // edge spoils one more row per step there, and only the last step's rows [out_lo, out_hi) --
    // n steps inside such an edge -- are stored (the paper's patches)
    int row0 = 0, Ht = H, st_lo = 0, st_hi = H;
    if (BAND) {
      const SeqRange r_in = a.ranges[(size_t)band * n], r_out = a.ranges[(size_t)band * n + n - 1];
      row0 = r_in.in_lo;
      Ht = r_in.in_hi - r_in.in_lo;
      st_lo = r_out.out_lo - row0;
      st_hi = r_out.out_hi - row0;
    }
    // clean steps: balanced parts (equal whenever two parts share a warp, see inplace_mode)
    const int c_r0 = CLEAN ? part * Ht / n_parts : part * Hp;
    const int c_hp = CLEAN ? (part + 1) * Ht / n_parts - c_r0 : Hp;
    const uint32_t plane = (uint32_t)(a.plane0 + pl0 + min(p, np - 1));
    // (scale, shift) of this warp's plane for every step, all loads in flight at once
    const uint32_t ch = plane - fdiv(plane, a.cdiv) * (uint32_t)a.C;
    // (no BN: (1, -0), an exact identity of v * s + t, the clean steps' branch-free epilogue)
    for (int i = lane; i < n; i += 32) t_aff[i] = aff_tab[i] ? __ldg(aff_tab[i] + ch) : make_float2(1.f, -0.f);
    __syncwarp();
    mbar_wait_sleep(&full[s], (k / a.stages) & 1);
    const char* sbase = (const char*)stage0 + (size_t)s * a.stage_bytes +
                        ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW) & 15u);
    const uint32_t base = smem_u32(sbase) + 4u * (uint32_t)(min(p, np - 1) * HW + c);
    float* og = a.out + (int64_t)plane * HW + (int64_t)row0 * W + c;
    // this lane's segments: pad lanes (outside the plane) read -inf and never store; halo lanes
    // (the neighbouring segment's edge group) read and never store
    SegLanes<NSEG, EDGE> L;
#pragma unroll
    for (int q = 0; q < NSEG; ++q) {
      const int cq = c + 4 * q * GS;                    // this lane's column in segment q
      L.off[q] = 16u * (uint32_t)(q * GS);
      L.col_ok[q] = cq >= 0 && cq < W;
      L.st_ok[q] = p < np && L.col_ok[q] && (NSEG == 1 || (sl >= 1 && sl <= GS));
      L.ld[q] = PadLd{L.col_ok[q] ? ~0u : 127u, L.col_ok[q] ? 0u : smem_u32(s_ninf)};
      L.le[q] = cq == 0;
      L.re[q] = cq + 4 >= W;
    }
    int st = 0;
    if (CLEAN) {   // steps two at a time (one sweep per pair), an odd last step alone
      for (; st + 1 < n; st += 2) {
        const float lo1 = (epi_tab[st] & 1) ? 0.f : -CUDART_INF_F, lo2 = (epi_tab[st + 1] & 1) ? 0.f : -CUDART_INF_F;
        if (st + 2 == n)
          inplace_pair_clean<SEG, NSEG, true, EDGE, BAND>(base, L, og, Ht, W, t_aff[st], lo1, t_aff[st + 1], lo2, c_r0, c_hp,
                                              bar_id, 32 * wpp, st_lo, st_hi);
        else
          inplace_pair_clean<SEG, NSEG, false, EDGE, BAND>(base, L, og, Ht, W, t_aff[st], lo1, t_aff[st + 1], lo2, c_r0, c_hp,
                                               bar_id, 32 * wpp, st_lo, st_hi);
      }
    }
    for (; st < n; ++st) {
      const float2 aff = t_aff[st];
      if (st == n - 1)
        inplace_step_epi<SEG, CLEAN, NSEG, true, EDGE, BAND>(epi_tab[st], base, L, og, Ht, W, c, aff, c_r0, c_hp, bar_id, 32 * wpp,
                                                 st_lo, st_hi);
      else
        inplace_step_epi<SEG, CLEAN, NSEG, false, EDGE, BAND>(epi_tab[st], base, L, og, Ht, W, c, aff, c_r0, c_hp, bar_id, 32 * wpp,
                                                  st_lo, st_hi);
    }
    mbar_arrive(&empty[s]);   // every lane: the tile's stage is free for the producer
  }
}

int seq_inplace_threads(const SeqArgs& a) { return 32 * (inplace_warps_of(inplace_nseg(a.W0)) + 1); }

size_t seq_inplace_smem(const SeqArgs& a) {
  return 128 + (size_t)a.stages * a.stage_bytes + (size_t)inplace_warps_of(inplace_nseg(a.W0)) * a.n_steps * 8 + 1024;
}

static const void* seq_fn(const SeqArgs& a) {
  const bool band = a.n_bands > 1;   // in-place band tiles: 32-lane segments, clean steps only
  if (a.inplace_seg && inplace_nseg(a.W0) == 2)
    return band ? (const void*)seq_inplace<32, 1, 2, true> : (const void*)seq_inplace<32, 1, 2, false>;
  const int mode = a.inplace_seg ? inplace_mode(a.inplace_seg, a.tile_planes, a.H0, a.W0) : 0;
  if (a.inplace_seg == 32 && band)
    return mode == 2 ? (const void*)seq_inplace<32, 2, 1, true> : (const void*)seq_inplace<32, 1, 1, true>;
  if (a.inplace_seg == 16)
    return mode == 1 ? (const void*)seq_inplace<16, 1, 1, false> : mode == 2 ? (const void*)seq_inplace<16, 2, 1, false>
                                                                               : (const void*)seq_inplace<16, 0, 1, false>;
  if (a.inplace_seg == 32)
    return mode == 1 ? (const void*)seq_inplace<32, 1, 1, false> : mode == 2 ? (const void*)seq_inplace<32, 2, 1, false>
                                                                               : (const void*)seq_inplace<32, 0, 1, false>;
  return (const void*)seq_staged;
}

cudaError_t launch_seq(const SeqArgs& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  if (a.inplace_seg)
    return launch_pdl(seq_fn(a), dim3(grid), dim3(seq_inplace_threads(a)), args, seq_inplace_smem(a), st);
  return launch_pdl((void*)seq_staged, dim3(grid), dim3(kSeqThreads), args, seq_smem(a), st);
}

int seq_max_blocks_per_sm(const SeqArgs& a) {
  const size_t smem = a.inplace_seg ? seq_inplace_smem(a) : seq_smem(a);
  const int threads = a.inplace_seg ? seq_inplace_threads(a) : kSeqThreads;
  int n = 0;
  if (smem_kernel_setup(seq_fn(a)) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, seq_fn(a), threads, smem) != cudaSuccess) n = 0;
  return n;
}

}  // namespace bs
