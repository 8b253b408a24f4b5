// k_seq.cu -- on-chip multi-step sequences (NEXT-2).
#include "bs_device.cuh"

namespace bs {

// ------------------------------------------------------------------ multi-step sequences
//
// NEXT-2: a *sequence* of several steps runs on-chip (PAPER.md P:L545-558,
// lst:finalcode P:L512-530 "float cached_data[...]"; the paper's GPU kernel swapped two smem
// buffers per step).  A tile of P whole planes is bulk-copied (TMA) into the ring
// as in pool_staged; step 0 reads the stage buffer, every later step reads the previous step's
// work buffer (two ping-pong buffers in shared memory), and only the last step writes HBM.
// Whole planes mean no halo growth with depth.  The 8 consumer warps split each step's
// output rows; a named barrier (bar.sync 1, 256) separates steps.

size_t seq_smem(const SeqArgs& a) {
  return 128 + (size_t)a.stages * pool_staged_stride(a.tile_planes, a.in_plane) + 2 * (size_t)a.work_floats * 4 + 256;
}

// One output element of a step from a smem plane (padding absent for max / zero for avg).
__device__ __forceinline__ float seq_window(const SeqStepDev& st, const float* pl, int i, int j, int ch,
                                            const float2 (&paff)[kAffSlots]) {
  const bool is_max = st.is_max != 0;
  float acc = is_max ? -CUDART_INF_F : 0.f;
  int real = 0;
  const int r0 = i * st.sh - st.ph, q0 = j * st.sw - st.pw;
  for (int u = 0; u < st.kh; ++u) {
    const int r = r0 + u;
    if ((unsigned)r >= (unsigned)st.H) continue;
    const float* row = pl + r * st.W;
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

// Per-step constants of the fast path, hoisted into shared memory once per CTA.
struct SeqFastStep {
  int32_t H, W, lg_nb, R;      // plane size; row bands = 1 << lg_nb of R rows
  int32_t has_aff, has_relu;   // epilogue: folded BN, ReLU
  const float2* aff;           // (scale, shift) per channel
};

// One fast step (3x3/s1/p1 max pool + [BN] [ReLU]) over the np planes of a tile: lane owns
// columns lane and lane + 32 (TWO); a warp walks a band of rows keeping the last two row maxima
// per column in registers -- 3 LDS per output, immediate offsets off one 32-bit row address.
// Padding is absent: an edge column replaces its out-of-row neighbour by itself and the bottom
// row its missing successor (duplicates, exact for max).  LAST: outputs go to HBM.
template <bool LAST, bool TWO>
__device__ __forceinline__ void seq_fast_step(const SeqFastStep& f, uint32_t in_s, uint32_t out_s, float* gout,
                                              int np, uint32_t plane_base, const FastDiv& cdiv, int C, int cw,
                                              int lane) {
  const int W = f.W, H = f.H, HW = W * H, R = f.R, lg = f.lg_nb;
  const uint32_t W4 = 4u * (uint32_t)W;
  const int j0 = min(lane, W - 1), j1 = min(lane + 32, W - 1);
  const bool act0 = lane < W, act1 = TWO && lane + 32 < W;
  const bool l0 = j0 == 0, r0 = j0 == W - 1, r1 = j1 == W - 1;
  const uint32_t c0off = 4u * (uint32_t)j0, c1off = 4u * (uint32_t)j1;
  const int items = np << lg;
  for (int it = cw; it < items; it += kSeqWarps) {
    const int p = it >> lg;
    const int i0 = (it & ((1 << lg) - 1)) * R, i1 = min(H, i0 + R);
    if (i0 >= i1) continue;
    const uint32_t plane = plane_base + (uint32_t)p;
    const int ch = (int)(plane - fdiv(plane, cdiv) * (uint32_t)C);
    float2 aff = make_float2(1.f, 0.f);
    if (f.has_aff) aff = __ldg(f.aff + ch);
    auto epi = [&](float r) -> float {
      if (f.has_aff) r = __fmaf_rn(r, aff.x, aff.y);
      if (f.has_relu) r = relu(r);
      return r;
    };
    auto rm0 = [&](uint32_t q) -> float {
      const float c = lds_f32(q + c0off);
      const float l = l0 ? c : lds_f32(q + c0off - 4u);
      const float r = r0 ? c : lds_f32(q + c0off + 4u);
      return fmaxf(fmaxf(l, c), r);
    };
    auto rm1 = [&](uint32_t q) -> float {   // column j1 >= 32: never a left edge
      const float c = lds_f32(q + c1off);
      const float l = lds_f32(q + c1off - 4u);
      const float r = r1 ? c : lds_f32(q + c1off + 4u);
      return fmaxf(fmaxf(l, c), r);
    };
    uint32_t q = in_s + 4u * (uint32_t)(p * HW + i0 * W);
    const uint32_t qp = i0 > 0 ? q - W4 : q;
    float a0 = rm0(qp), b0 = rm0(q), a1 = 0.f, b1 = 0.f;
    if (TWO) { a1 = rm1(qp); b1 = rm1(q); }
    const int i_end = min(i1, H - 1);   // rows whose successor row exists
    uint32_t o = out_s + 4u * (uint32_t)(p * HW + i0 * W);
    float* og = LAST ? gout + (size_t)p * HW + i0 * W : nullptr;
    auto put = [&](float v0, float v1) {
      if (LAST) {
        if (act0) __stcs(og + j0, v0);
        if (TWO && act1) __stcs(og + j1, v1);
        og += W;
      } else {
        if (act0) sts_f32(o + c0off, v0);
        if (TWO && act1) sts_f32(o + c1off, v1);
        o += W4;
      }
    };
#pragma unroll 2
    for (int i = i0; i < i_end; ++i) {
      q += W4;
      const float c0 = rm0(q);
      const float v0 = epi(fmaxf(fmaxf(a0, b0), c0));
      a0 = b0;
      b0 = c0;
      float v1 = 0.f;
      if (TWO) {
        const float c1 = rm1(q);
        v1 = epi(fmaxf(fmaxf(a1, b1), c1));
        a1 = b1;
        b1 = c1;
      }
      put(v0, v1);
    }
    if (i1 == H) put(epi(fmaxf(a0, b0)), epi(fmaxf(a1, b1)));
  }
}

#ifdef BS_ARRIVE_ALL
#define BS_SEQ_EMPTY_ARRIVER true
#else
#define BS_SEQ_EMPTY_ARRIVER (cw == 0 && lane == 0)
#endif

__global__ void __launch_bounds__(kSeqThreads) seq_staged(SeqArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  const size_t tile_stride = pool_staged_stride(a.tile_planes, a.in_plane);
  unsigned char* stage0 = smem + 128;
  // the two ping-pong work buffers (selected by arithmetic, not a local array: no local memory)
  float* const work0 = (float*)(stage0 + (size_t)a.stages * tile_stride);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)a.n_tiles;
  const int HW0 = a.in_plane;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 2);
#ifdef BS_ARRIVE_ALL
      mbar_init(&empty[s], 32 * kSeqWarps);
#else
      mbar_init(&empty[s], 1);
#endif
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();                   // previous kernel on the stream complete + visible
  pdl_launch_dependents();

  if (warp == 0) {  // producer, as in pool_staged
    if (lane == 0) {
      int k = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % a.stages;
        if (k >= a.stages) {
          mbar_wait_sleep(&empty[s], ((k / a.stages) - 1) & 1);
#ifdef BS_PROXY_FENCE
          fence_proxy_async_smem();
#endif
        }
        const int64_t pl0 = (int64_t)t * a.tile_planes;
        const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
        const float* src = a.in + (a.plane0 + pl0) * (int64_t)HW0;
        const uint32_t head_off = (uint32_t)((uintptr_t)src & 15u);
        float* dst = (float*)((char*)stage0 + (size_t)s * tile_stride + head_off);
        const uint32_t nbytes = (uint32_t)np * (uint32_t)HW0 * 4u;
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
  // per-step constants of the fast path (W = 0: generic step), filled once by warp 1
  __shared__ SeqFastStep fast_tab[kMaxSeqSteps];
  if (cw == 0 && lane < a.n_steps) {
    const SeqStepDev& st = a.steps[lane];
    SeqFastStep f;
    f.W = (st.fast && st.W <= 64) ? st.W : 0;
    f.H = st.H;
    int lg = 0;   // row bands: a power of two, >= 16 items per tile
    while ((2 << lg) <= st.H && (a.tile_planes << lg) < 2 * kSeqWarps) ++lg;
    f.lg_nb = lg;
    f.R = (st.H + (1 << lg) - 1) >> lg;
    f.has_aff = st.epi_class == PC_AFFINE || st.epi_class == PC_AFFINE_RELU;
    f.has_relu = st.epi_class == PC_RELU || st.epi_class == PC_AFFINE_RELU;
    f.aff = st.epi.affine[0];
    fast_tab[lane] = f;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");
  int k = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int s = k % a.stages;
    mbar_wait_sleep(&full[s], (k / a.stages) & 1);
    const int64_t pl0 = (int64_t)t * a.tile_planes;
    const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
    const float* src_base = (const float*)((const char*)stage0 + (size_t)s * tile_stride +
                                           ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW0) & 15u));
    for (int st_i = 0; st_i < a.n_steps; ++st_i) {
      const SeqStepDev& st = a.steps[st_i];
      const bool last = st_i == a.n_steps - 1;
      const float* in_buf = st_i == 0 ? src_base : work0 + ((st_i - 1) & 1) * a.work_floats;
      float* out_buf = work0 + (st_i & 1) * a.work_floats;
      const int HWi = st.H * st.W, HWo = st.Ho * st.Wo;
      if (fast_tab[st_i].W > 0) {
        const SeqFastStep& f = fast_tab[st_i];
        const uint32_t in_s = smem_u32(in_buf), out_s = smem_u32(out_buf);
        float* gout = a.out + (a.plane0 + pl0) * (int64_t)HWo;
        const uint32_t pbase = (uint32_t)(a.plane0 + pl0);
        if (last) {
          if (f.W > 32) seq_fast_step<true, true>(f, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
          else seq_fast_step<true, false>(f, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
        } else {
          if (f.W > 32) seq_fast_step<false, true>(f, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
          else seq_fast_step<false, false>(f, in_s, out_s, gout, np, pbase, a.cdiv, a.C, cw, lane);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");   // step boundary
        if (st_i == 0 && BS_SEQ_EMPTY_ARRIVER) mbar_arrive(&empty[s]);   // stage buffer consumed
        continue;
      }
      // work items: (plane, output row, 32-column chunk); lane = output column
      const int nchunk = (st.Wo + 31) / 32;
      const int items = np * st.Ho * nchunk;
      for (int it = cw; it < items; it += kSeqWarps) {
        const int cc = it % nchunk;
        const int i = (it / nchunk) % st.Ho;
        const int p = it / (nchunk * st.Ho);
        const int j = cc * 32 + lane;
        if (j >= st.Wo) continue;
        const int64_t plane = a.plane0 + pl0 + p;
        const int ch = (int)(plane % a.C);
        float2 paff[kAffSlots], eaff[kAffSlots];
        load_affine(st.pro, ch, paff);
        load_affine(st.epi, ch, eaff);
        float r = seq_window(st, in_buf + p * HWi, i, j, ch, paff);
        r = apply_generic(st.epi, eaff, ch, r, 0);
        if (last) __stcs(a.out + plane * (int64_t)HWo + i * st.Wo + j, r);
        else out_buf[p * HWo + i * st.Wo + j] = r;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kSeqWarps) : "memory");   // step boundary
      if (st_i == 0 && BS_SEQ_EMPTY_ARRIVER) mbar_arrive(&empty[s]);   // stage buffer consumed
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
