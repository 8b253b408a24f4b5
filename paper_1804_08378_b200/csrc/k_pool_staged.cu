// k_pool_staged.cu -- the staged (TMA bulk copy + mbarrier ring) pool kernel.
#include "bs_device.cuh"

namespace bs {

// ------------------------------------------------------------------ staged (TMA) walker
//
// For planes whose rows are not 16-byte aligned (AlexNet 55/27/13, 7x7), tiles of P whole
// planes -- P*H*W*4 contiguous bytes -- are moved HBM -> shared memory by cp.async.bulk (the
// 1-D TMA engine; SASS UBLKCP) behind an mbarrier ring of `stages` buffers.  Warp 0 is the
// producer (one elected lane), warps 1..8 consume.  The paper's stacked kernel staged patches
// through two smem buffers swapped per step; here whole planes are staged, so
// overlapping 3x3/s2 windows need no halo re-reads from HBM at all.
//
//  * Persistent CTAs take tiles of P planes round-robin (tile b, b + grid, ...), so the grid
//    streams one advancing window of HBM (-DBS_STAGED_CONTIGUOUS: one contiguous plane range
//    per CTA instead, balanced to one plane but ~2 % slower on B200).
//  * All 8 consumer warps work on the same tile at once: the tile's I items -- (group of G
//    planes, column chunk, band of R output rows) -- are dealt to the warps in a fixed
//    pattern (item w, w+8, ...), the planner choosing P and R so that I is a multiple of 8.
//    A tile is thus consumed (and its stage released to the producer) in ~1/8 of the time one
//    warp would take, which keeps the ring turning over at HBM speed.
//  * Lane = output column (output-stationary): each lane reduces its KW window columns of each
//    new input row straight from shared memory; the row reductions of the last KH-SH rows
//    slide along in registers, outputs are stored to HBM with st.global.cs.
//  * Tiles may start on any float: the 16-byte-aligned middle is bulk-copied, the <= 6 edge
//    floats use 4-byte cp.async tracked by the same full barrier.
//  * The ring holds ~104 KB of tiles per SM (bs_api.cpp size_stages): measured on B200, more
//    bytes in flight is slower, and one CTA per SM beats two for big tiles on long kernels.
//    Waits sleep (mbarrier.try_wait with a suspend-time hint) instead of spinning.

// barriers | `stages` input stages
size_t pool_staged_smem(int tile_planes, int HW, int HWo, int stages) {
  (void)HWo;
  return kStagedHeader + (size_t)stages * pool_staged_stride(tile_planes, HW);
}


// Every consumer THREAD arrives on a stage's empty barrier once it has read the tile (256
// arrivals per tile).  One arrive per warp after __syncwarp() is equally ordered under the PTX
// memory model (release by lane 0 after the warp barrier), but compute-sanitizer racecheck does
// not follow that chain and reports the next bulk copy into the stage as a race; per-thread
// arrivals make the ordering explicit at <= 2 % cost (AlexNet stacks, profiles/r02_racecheck.md).
#ifndef BS_WARP_ARRIVE
constexpr int kEmptyArrivals = 32 * kStagedConsumerWarps;
#else
constexpr int kEmptyArrivals = kStagedConsumerWarps;
#endif

template <int KH, int KW, int SH, int SW, bool IS_MAX, bool PAD, int PC, int OC>
__global__ void __launch_bounds__(kStagedThreads) pool_staged(PoolArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + kStagedMaxStages;
  const int HW = a.H * a.W, HWo = a.Ho * a.Wo;
  const size_t tile_stride = pool_staged_stride(a.tile_planes, HW);
  unsigned char* stage0 = smem + kStagedHeader;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.tile_planes, S = a.stages;
  // this CTA's contiguous plane range [pb, pe)
#ifndef BS_STAGED_CONTIGUOUS
  // tiles dealt round-robin (CTA b takes tiles b, b + grid, ...): at any moment the CTAs stream
  // one contiguous window of HBM, measured 1.5-2.5 % faster on the AlexNet stacks than one
  // contiguous plane range per CTA (-DBS_STAGED_CONTIGUOUS)
  const int64_t n_tiles_all = (a.n_planes + P - 1) / P;
  const int my_tiles = (int)((n_tiles_all - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int64_t pe = a.n_planes;
#define BS_TILE_P0(k) ((int64_t)(blockIdx.x + (int64_t)(k) * gridDim.x) * P)
#else
  const int64_t pb = a.n_planes * (int64_t)blockIdx.x / gridDim.x;
  const int64_t pe = a.n_planes * ((int64_t)blockIdx.x + 1) / gridDim.x;
  const int my_tiles = (int)((pe - pb + P - 1) / P);
#define BS_TILE_P0(k) (pb + (int64_t)(k) * P)
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);                        // cp.async arrive (edges) + expect_tx (body)
      mbar_init(&empty[s], kEmptyArrivals);          // every consumer warp (thread), once per tile
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();                   // previous kernel on the stream complete + visible
  pdl_launch_dependents();

  if (warp == 0) {
    // ---------------- producer: one elected lane issues the copies
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < my_tiles; ++k) {
        if (k >= S) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
#ifdef BS_PROXY_FENCE
          fence_proxy_async_smem();
#endif
        }
        const int64_t p0 = BS_TILE_P0(k);
        const int np = (int)min((int64_t)P, pe - p0);
        const float* src = a.in + (a.plane0 + p0) * (int64_t)HW;
        const uint32_t head_off = (uint32_t)((uintptr_t)src & 15u);
        float* dst = (float*)(stage0 + (size_t)s * tile_stride + head_off);
        const uint32_t nbytes = (uint32_t)np * (uint32_t)HW * 4u;
        const uint32_t h = min(nbytes, (16u - head_off) & 15u);        // head bytes before 16-B
        const uint32_t body = (nbytes - h) & ~15u;                      // aligned middle
        // head / tail floats: 4-byte cp.async (non-blocking), tracked by the full barrier
        for (uint32_t e = 0; e < h / 4; ++e) cp_async4(dst + e, src + e);
        for (uint32_t e = (h + body) / 4; e < nbytes / 4; ++e) cp_async4(dst + e, src + e);
        cp_async_mbar_arrive(&full[s]);   // arrival 1 of 2: when those copies have landed
        if (body) {
          mbar_arrive_expect_tx(&full[s], body);
          for (uint32_t off = 0; off < body; off += kBulkChunk)
            bulk_g2s((char*)dst + h + off, (const char*)src + h + off, min(kBulkChunk, body - off), &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers
  // Warp cw walks items cw, cw + 8, cw + 16, ... of every tile.  The planner keeps I <= 16
  // where it can, so the geometry of a warp's first two items is decoded once, outside the
  // tile loop; items beyond those (very wide planes, Wo > 16 * 32, or forced narrow column
  // groups) are decoded per tile.
  const int cw = warp - 1;
  const int J = a.Jg;                 // output columns per lane group (G groups per warp)
  const int g = lane / J, l = lane - g * J;
  const int items = ((P + a.G - 1) / a.G) * a.n_cc * a.n_rb;
  struct Item { int pin, j, i0, i1; bool ok; };
  auto decode = [&](int it) -> Item {
    Item r;
    const int rb = it % a.n_rb;
    const int rest = it / a.n_rb;
    const int cc = rest % a.n_cc;
    r.pin = (rest / a.n_cc) * a.G + g;
    r.j = cc * J + l;
    r.i0 = rb * a.rows_per_task;
    r.i1 = min(a.Ho, r.i0 + a.rows_per_task);
    r.ok = it < items && g < a.G && l < J && r.j < a.Wo;
    return r;
  };
  const Item it0 = decode(cw), it1 = decode(cw + kStagedConsumerWarps);
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  constexpr int CARRY = KH > SH ? KH - SH : 0;
  constexpr int NEW = KH - CARRY;
  // a deferred monotone prologue may be non-increasing (negative BN scale / SCALE alpha): the
  // window max is then taken over sign-flipped values; ReLU-only programs never flip
  constexpr bool MAY_FLIP = IS_MAX && (OC == PC_AFFINE || OC == PC_AFFINE_RELU || OC == PC_GENERIC);
  const int W = a.W;
  int s = 0;
  uint32_t ph = 0;
  for (int k = 0; k < my_tiles; ++k) {
    const int64_t p0 = BS_TILE_P0(k);
    const int np = (int)min((int64_t)P, pe - p0);
    const float* sm = (const float*)(stage0 + (size_t)s * tile_stride +
                                     ((uintptr_t)(a.in + (a.plane0 + p0) * (int64_t)HW) & 15u));
    mbar_wait_sleep(&full[s], ph);
#ifdef BS_DBG_NOCOMPUTE
    if (items < 0)
#endif
#pragma unroll 1
    for (int it = cw; it < items; it += kStagedConsumerWarps) {
      const Item I = it == cw ? it0 : it == cw + kStagedConsumerWarps ? it1 : decode(it);
      if (!I.ok || I.pin >= np) continue;
      const int pin = I.pin, j = I.j, i0 = I.i0, i1 = I.i1;
      const uint32_t plane = (uint32_t)(a.plane0 + p0 + pin);
      const int ch = (int)(plane - fdiv(plane, a.cdiv) * (uint32_t)a.C);
      float2 paff[kAffSlots], eaff[kAffSlots];
      if (PC == PC_AFFINE || PC == PC_AFFINE_RELU) paff[0] = __ldg(a.pro.affine[0] + ch);
      else if (PC == PC_GENERIC) load_affine(a.pro, ch, paff);
      if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) eaff[0] = __ldg(a.epi.affine[0] + ch);
      else if (OC == PC_GENERIC) load_affine(a.epi, ch, eaff);
      uint32_t flip = 0;
      if (MAY_FLIP && a.epi.n_deferred > 0) {
        if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) flip = __float_as_uint(eaff[0].x) & 0x80000000u;
        else flip = deferred_flip(a.epi, eaff, ch);
      }
      const int64_t in_idx0 = (int64_t)plane * HW;
      const int64_t out_idx0 = (int64_t)plane * HWo + j;
      float* op = a.out + out_idx0 + (int64_t)i0 * a.Wo;
      float hist[KH];
#pragma unroll
      for (int u = 0; u < KH; ++u) hist[u] = ident;
      auto emit = [&](int i) {
        float res = hist[0];
#pragma unroll
        for (int u = 1; u < KH; ++u) res = red<IS_MAX>(res, hist[u]);
#pragma unroll
        for (int u = 0; u < CARRY; ++u) hist[u] = hist[u + NEW];
        if (MAY_FLIP) res = xorsign(res, flip);
        if (!IS_MAX) res = (PAD && !a.count_include_pad) ? __fdiv_rn(res, avg_div(a, i, j, KH, KW, SH, SW))
                                                         : div_by<KH * KW>(res);
        res = apply1<OC>(a.epi, eaff, ch, res, out_idx0 + (int64_t)i * a.Wo);
#ifdef BS_DBG_NOSTORE
        if (res == 1234.5f)
#endif
        __stcs(op, res);
        op += a.Wo;
      };
      if (!PAD) {
        // every window lies inside the plane: one smem pointer walks down the window's
        // top-left corner, the KW columns are immediate offsets (LDS [R + 4v])
        const float* rp = sm + pin * HW + i0 * SH * W + j * SW;
        auto rowred = [&](const float* p, int r) -> float {
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < KW; ++v) {
            float x = p[v];
            if (MAY_FLIP) x = xorsign(x, flip);
            if (!IS_MAX && PC != PC_NONE) x = apply1<PC>(a.pro, paff, ch, x, in_idx0 + (int64_t)r * W + j * SW + v);
            acc = v == 0 ? x : red<IS_MAX>(acc, x);
          }
          return acc;
        };
        int r = i0 * SH;
#pragma unroll
        for (int u = 0; u < CARRY; ++u, rp += W, ++r) hist[u] = rowred(rp, r);
#pragma unroll 2
        for (int i = i0; i < i1; ++i) {
#pragma unroll
          for (int u = 0; u < NEW; ++u, rp += W, ++r) hist[CARRY + u] = rowred(rp, r);
          emit(i);
        }
      } else {
        // general case: clamped window columns / rows, padding cells absent (max) or zero (avg)
        const int c0 = j * SW - a.pw;
        int coff[KW];
        bool cval[KW];
#pragma unroll
        for (int v = 0; v < KW; ++v) {
          cval[v] = (unsigned)(c0 + v) < (unsigned)W;
          coff[v] = min(max(c0 + v, 0), W - 1);
        }
        const float* ps = sm + pin * HW;
        auto rowred = [&](int r) -> float {
          const bool rvalid = (unsigned)r < (unsigned)a.H;
          const int rc = min(max(r, 0), a.H - 1);
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < KW; ++v) {
            float x = ps[rc * W + coff[v]];
            if (IS_MAX) {
              if (MAY_FLIP) x = xorsign(x, flip);
              // a clamped duplicate of an in-window element leaves a max unchanged
            } else {
              if (PC != PC_NONE) x = apply1<PC>(a.pro, paff, ch, x, in_idx0 + (int64_t)rc * W + coff[v]);
              x = (rvalid && cval[v]) ? x : 0.f;
            }
            acc = v == 0 ? x : red<IS_MAX>(acc, x);
          }
          return acc;
        };
        // (a max window always holds a real row: p <= k/2, so a clamped row duplicates one)
#pragma unroll
        for (int u = 0; u < CARRY; ++u) hist[u] = rowred(i0 * SH - a.ph + u);
        for (int i = i0; i < i1; ++i) {
#pragma unroll
          for (int u = 0; u < NEW; ++u) hist[CARRY + u] = rowred(i * SH - a.ph + CARRY + u);
          emit(i);
        }
      }
    }
#ifndef BS_WARP_ARRIVE
    mbar_arrive(&empty[s]);                  // input stage consumed (by this thread)
#else
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // input stage consumed
#endif
    if (++s == S) { s = 0; ph ^= 1; }
  }
}


template <int K, int S, bool PAD>
static void* staged_pick(bool is_max, int pc, int oc) {
  if (is_max) {  // prologue deferred: only the output class varies
    switch (oc) {
      case PC_NONE: return (void*)pool_staged<K, K, S, S, true, PAD, PC_NONE, PC_NONE>;
      case PC_RELU: return (void*)pool_staged<K, K, S, S, true, PAD, PC_NONE, PC_RELU>;
      case PC_AFFINE_RELU: return (void*)pool_staged<K, K, S, S, true, PAD, PC_NONE, PC_AFFINE_RELU>;
      default: return (void*)pool_staged<K, K, S, S, true, PAD, PC_NONE, PC_GENERIC>;
    }
  }
  (void)oc;
  switch (pc) {
    case PC_NONE: return (void*)pool_staged<K, K, S, S, false, PAD, PC_NONE, PC_GENERIC>;
    case PC_RELU: return (void*)pool_staged<K, K, S, S, false, PAD, PC_RELU, PC_GENERIC>;
    case PC_AFFINE_RELU: return (void*)pool_staged<K, K, S, S, false, PAD, PC_AFFINE_RELU, PC_GENERIC>;
    default: return (void*)pool_staged<K, K, S, S, false, PAD, PC_GENERIC, PC_GENERIC>;
  }
}

template <int K, int S>
static void* staged_pick_pad(const PoolArgs& a) {
  const bool m = a.is_max != 0;
  // PAD = false needs every window inside the plane: no padding and floor-mode extents
  const bool pad = a.ph != 0 || a.pw != 0 || (a.Ho - 1) * S + K > a.H || (a.Wo - 1) * S + K > a.W;
  return pad ? staged_pick<K, S, true>(m, a.pro_class, a.epi_class) : staged_pick<K, S, false>(m, a.pro_class, a.epi_class);
}

void* pool_fn_staged(const PoolArgs& a) {
  if (a.is_max && a.pro.n > 0) return nullptr;   // max pools reach this kernel deferred only
  if (a.kh == 2 && a.sh == 2) return staged_pick_pad<2, 2>(a);
  if (a.kh == 3 && a.sh == 2) return staged_pick_pad<3, 2>(a);
  if (a.kh == 3 && a.sh == 1) return staged_pick_pad<3, 1>(a);
  if (a.kh == 7 && a.sh == 7) return staged_pick_pad<7, 7>(a);
  return nullptr;
}

}  // namespace bs
