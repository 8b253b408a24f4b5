// k_pool_global.cu -- pool kernels that read HBM directly (no shared-memory staging):
// the vector and scalar column walkers, the runtime-geometry walker and the naive kernel.
#include "bs_device.cuh"

namespace bs {

// Specialised column walker: compile-time window (KH x KW, stride SH x SW); U output rows per
// iteration -> NR = (U-1)*SH + KH independent row loads in flight per lane.
//   PC: class of the per-element prologue (avg pools; max pools run with it deferred, PC_NONE)
//   OC: class of the per-output program (deferred prologue + epilogue)
template <int KH, int KW, int SH, int SW, bool IS_MAX, int U, int PC, int OC>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_spec(PoolArgs a) {
  pdl_wait();                 // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  constexpr int NR = (U - 1) * SH + KH;
  const int lane = threadIdx.x & 31;
  const int wg = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (unsigned)blockDim.x) >> 5);
  const int g = lane / a.gw;
  const int l = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  const int HW = a.H * a.W, HWo = a.Ho * a.Wo;
  const int n_tasks = (int)a.n_tasks;

  for (int t = wg; t < n_tasks; t += nw) {
    const LaneTask T = decode_task(a, t, g, l, SW);
    const int ch = (int)(T.plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    if (PC == PC_AFFINE || PC == PC_AFFINE_RELU) paff[0] = __ldg(a.pro.affine[0] + ch);
    else if (PC == PC_GENERIC) load_affine(a.pro, ch, paff);
    if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) eaff[0] = __ldg(a.epi.affine[0] + ch);
    else if (OC == PC_GENERIC) load_affine(a.epi, ch, eaff);
    uint32_t flip = 0;
    if (IS_MAX && a.epi.n_deferred > 0) {
      if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) flip = __float_as_uint(eaff[0].x) & 0x80000000u;
      else if (OC == PC_GENERIC) flip = deferred_flip(a.epi, eaff, ch);
    }
    // lanes outside the image load a clamped (valid) column; their values are discarded
    const int cl = min(max(T.c, 0), a.W - 1);
    const float* pin = a.in + T.plane * (int64_t)HW + cl;
    float* pout = a.out + T.plane * (int64_t)HWo + (T.out_lane ? T.j : 0);
    const int64_t in_idx0 = T.plane * (int64_t)HW + T.c;
    const int64_t out_idx0 = T.plane * (int64_t)HWo + T.j;
    const unsigned W4 = 4u * (unsigned)a.W, Wo4 = 4u * (unsigned)a.Wo;

    for (int i = T.i_begin; i < T.i_end; i += U) {
      const int r0 = i * SH - a.ph;
      float v[NR];
      if (i + U <= T.i_end && r0 >= 0 && r0 + NR <= a.H) {
        // ---- fast path: every row of the iteration is inside the tensor (warp-uniform)
        const char* pb = (const char*)pin + (size_t)((unsigned)r0 * W4);
#pragma unroll
        for (int q = 0; q < NR; ++q) v[q] = __ldg((const float*)(pb + (size_t)q * W4));
        if (IS_MAX) {
          if (flip) {
#pragma unroll
            for (int q = 0; q < NR; ++q) v[q] = xorsign(v[q], flip);
          }
        } else if (PC != PC_NONE) {
          // padding-column lanes (T.c outside the row) load a clamped column; they skip the
          // program (an ADD operand would otherwise be read at T.c < 0) and are discarded below
          bool ok[NR];
#pragma unroll
          for (int q = 0; q < NR; ++q) ok[q] = T.col_ok;
          apply_rows<PC, NR>(a.pro, paff, ch, v, ok, ident, in_idx0 + (int64_t)r0 * a.W, a.W);
        }
        char* po = (char*)pout + (size_t)((unsigned)i * Wo4);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float acc = v[u * SH];
#pragma unroll
          for (int q = 1; q < KH; ++q) acc = red<IS_MAX>(acc, v[u * SH + q]);
          acc = T.col_ok ? acc : ident;  // padding columns: absent (max) / zero (avg)
          float res = acc;
#pragma unroll
          for (int d = 1; d < KW; ++d) res = red<IS_MAX>(res, __shfl_down_sync(0xffffffffu, acc, d));
          if (IS_MAX) res = xorsign(res, flip);
          else res = a.count_include_pad ? div_by<KH * KW>(res) : __fdiv_rn(res, avg_div(a, i + u, T.j, KH, KW, SH, SW));
          res = apply1<OC>(a.epi, eaff, ch, res, out_idx0 + (int64_t)(i + u) * a.Wo);
          if (T.out_lane) __stcs((float*)(po + (size_t)u * Wo4), res);
        }
      } else {
        // ---- edge path: rows above/below the tensor (padding) or a partial row block
        bool ok[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          ok[q] = T.col_ok && (unsigned)(r0 + q) < (unsigned)a.H;
          v[q] = ok[q] ? __ldg(pin + (r0 + q) * a.W) : ident;
        }
        if (IS_MAX) {
          if (flip) {
#pragma unroll
            for (int q = 0; q < NR; ++q) v[q] = ok[q] ? xorsign(v[q], flip) : ident;
          }
        } else {
          apply_rows<PC, NR>(a.pro, paff, ch, v, ok, ident, in_idx0 + (int64_t)r0 * a.W, a.W);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (i + u < T.i_end) {
            float acc = v[u * SH];
#pragma unroll
            for (int q = 1; q < KH; ++q) acc = red<IS_MAX>(acc, v[u * SH + q]);
            float res = acc;
#pragma unroll
            for (int d = 1; d < KW; ++d) res = red<IS_MAX>(res, __shfl_down_sync(0xffffffffu, acc, d));
            if (T.out_lane) {
              if (IS_MAX) res = xorsign(res, flip);
              else res = __fdiv_rn(res, avg_div(a, i + u, T.j, KH, KW, SH, SW));
              const int orow = (i + u) * a.Wo;
              res = apply1<OC>(a.epi, eaff, ch, res, out_idx0 + orow);
              __stcs(pout + orow, res);
            }
          }
        }
      }
    }
  }
}

// Vector column walker for stride-2 windows on rows whose width is a multiple of VEC
// (VGG 224/112/56/28, ResNet/DenseNet 112/56/28, ...): each lane owns VEC consecutive
// columns (one 128/64-bit load per row), reduces them vertically, and produces VEC/2
// outputs per row from its own columns plus, for 3-wide windows, one column of its
// neighbour lane (__shfl_up for pad 1, __shfl_down for pad 0).  That neighbour is a "halo
// lane" at the group's edge which loads but produces nothing.  Requires no right padding.
template <int K, int PADL, int VEC, bool IS_MAX, int U, int PC, int OC>
__global__ void __launch_bounds__(kPoolBlock, 4) pool_vec(PoolArgs a) {
  pdl_wait();                 // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  constexpr int S = 2, OPL = VEC / 2;
  constexpr int NR = (U - 1) * S + K;
  constexpr int HL = (K == 3 && PADL == 1) ? 1 : 0;   // left halo lane
  constexpr int HR = (K == 3 && PADL == 0) ? 1 : 0;   // right halo lane
  using VT = typename std::conditional<VEC == 4, float4, float2>::type;
  const int lane = threadIdx.x & 31;
  const int wg = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (unsigned)blockDim.x) >> 5);
  const int g = lane / a.gw;
  const int m = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  const int HW = a.H * a.W, HWo = a.Ho * a.Wo;
  const int n_tasks = (int)a.n_tasks;
  const unsigned W4 = 4u * (unsigned)a.W, Wo4 = 4u * (unsigned)a.Wo;
  const bool wo_even = (a.Wo & 1) == 0;

  for (int t = wg; t < n_tasks; t += nw) {
    const int cc = t % a.n_cc;
    const int t2 = t / a.n_cc;
    const int rb = t2 % a.n_rb;
    const int pg = t2 / a.n_rb;
    const int64_t pl_local = (int64_t)pg * a.G + g;
    const bool plane_ok = (g < a.G) && (pl_local < a.n_planes);
    const int64_t plane = a.plane0 + (plane_ok ? pl_local : 0);
    const int c = cc * a.Jg * S + VEC * (m - HL);            // first column of this lane
    const bool col_ok = plane_ok && c >= 0 && c < a.W;       // all VEC columns in or all out
    const int j = cc * a.Jg + OPL * (m - HL);                // first output of this lane
    const bool out_lane = plane_ok && m >= HL && m < a.gw - HR && j < a.Wo;
    const int i_begin = rb * a.rows_per_task;
    const int i_end = min(a.Ho, i_begin + a.rows_per_task);
    const int ch = (int)(plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    if (PC == PC_AFFINE || PC == PC_AFFINE_RELU) paff[0] = __ldg(a.pro.affine[0] + ch);
    else if (PC == PC_GENERIC) load_affine(a.pro, ch, paff);
    if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) eaff[0] = __ldg(a.epi.affine[0] + ch);
    else if (OC == PC_GENERIC) load_affine(a.epi, ch, eaff);
    uint32_t flip = 0;
    if (IS_MAX && a.epi.n_deferred > 0) {
      if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) flip = __float_as_uint(eaff[0].x) & 0x80000000u;
      else if (OC == PC_GENERIC) flip = deferred_flip(a.epi, eaff, ch);
    }
    const int cl = col_ok ? c : 0;
    const char* pin = (const char*)(a.in + plane * (int64_t)HW + cl);
    const int64_t in_idx0 = plane * (int64_t)HW + cl;
    float* pout = a.out + plane * (int64_t)HWo + (out_lane ? j : 0);
    const int64_t out_idx0 = plane * (int64_t)HWo + j;

    for (int i = i_begin; i < i_end; i += U) {
      const int r0 = i * S - PADL;
      float v[NR][VEC];
      bool ok[NR];
      const bool full = i + U <= i_end && r0 >= 0 && r0 + NR <= a.H;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        ok[q] = full || (unsigned)(r0 + q) < (unsigned)a.H;
        VT x;
        if (ok[q]) x = __ldg((const VT*)(pin + (size_t)(unsigned)(r0 + q) * W4));
        else { x.x = ident; x.y = ident; if constexpr (VEC == 4) { x.z = ident; x.w = ident; } }
        v[q][0] = x.x; v[q][1] = x.y;
        if constexpr (VEC == 4) { v[q][2] = x.z; v[q][3] = x.w; }
      }
      if (IS_MAX) {
        if (flip) {
#pragma unroll
          for (int q = 0; q < NR; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) v[q][e] = ok[q] ? xorsign(v[q][e], flip) : ident;
        }
      } else if (PC != PC_NONE) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          float col[NR];
#pragma unroll
          for (int q = 0; q < NR; ++q) col[q] = v[q][e];
          apply_rows<PC, NR>(a.pro, paff, ch, col, ok, ident, in_idx0 + e + (int64_t)r0 * a.W, a.W);
#pragma unroll
          for (int q = 0; q < NR; ++q) v[q][e] = col[q];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (full || i + u < i_end) {
          float acc[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            acc[e] = v[u * S][e];
#pragma unroll
            for (int q = 1; q < K; ++q) acc[e] = red<IS_MAX>(acc[e], v[u * S + q][e]);
            acc[e] = col_ok ? acc[e] : ident;   // padding columns: absent (max) / zero (avg)
          }
          float o[OPL];
          if (K == 2) {
#pragma unroll
            for (int t2_ = 0; t2_ < OPL; ++t2_) o[t2_] = red<IS_MAX>(acc[2 * t2_], acc[2 * t2_ + 1]);
          } else if (PADL == 1) {
            const float left = __shfl_up_sync(0xffffffffu, acc[VEC - 1], 1);
            o[0] = red<IS_MAX>(red<IS_MAX>(left, acc[0]), acc[1]);
            if (OPL == 2) o[OPL - 1] = red<IS_MAX>(red<IS_MAX>(acc[1], acc[2]), acc[VEC - 1]);
          } else {
            const float right = __shfl_down_sync(0xffffffffu, acc[0], 1);
            if (OPL == 2) o[0] = red<IS_MAX>(red<IS_MAX>(acc[0], acc[1]), acc[2]);
            o[OPL - 1] = red<IS_MAX>(red<IS_MAX>(acc[VEC - 2], acc[VEC - 1]), right);
          }
          const int iu = i + u;
#pragma unroll
          for (int t2_ = 0; t2_ < OPL; ++t2_) {
            float r = o[t2_];
            if (IS_MAX) r = xorsign(r, flip);
            else r = a.count_include_pad ? div_by<K * K>(r) : __fdiv_rn(r, avg_div(a, iu, j + t2_, K, K, S, S));
            o[t2_] = apply1<OC>(a.epi, eaff, ch, r, out_idx0 + (int64_t)iu * a.Wo + t2_);
          }
          if (out_lane) {
            float* po = (float*)((char*)pout + (size_t)(unsigned)iu * Wo4);
            if (OPL == 2 && wo_even) {
              __stcs((float2*)po, make_float2(o[0], o[OPL - 1]));
            } else {
              __stcs(po, o[0]);
              if (OPL == 2 && j + 1 < a.Wo) __stcs(po + 1, o[OPL - 1]);
            }
          }
        }
      }
    }
  }
}


// Column walker with runtime window geometry (any kw <= 32 - (Jg-1)*sw).
template <bool IS_MAX>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_gen(PoolArgs a) {
  pdl_wait();                 // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int wg = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (unsigned)blockDim.x) >> 5);
  const int g = lane / a.gw;
  const int l = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  const int HW = a.H * a.W, HWo = a.Ho * a.Wo;
  const int kh = a.kh, kw = a.kw, sh = a.sh, sw = a.sw;
  const int n_tasks = (int)a.n_tasks;

  for (int t = wg; t < n_tasks; t += nw) {
    const LaneTask T = decode_task(a, t, g, l, sw);
    const int ch = (int)(T.plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    load_affine(a.pro, ch, paff);
    load_affine(a.epi, ch, eaff);
    const uint32_t flip = IS_MAX ? deferred_flip(a.epi, eaff, ch) : 0u;
    const float* pin = a.in + T.plane * (int64_t)HW + (T.col_ok ? T.c : 0);
    const int64_t in_idx0 = T.plane * (int64_t)HW + T.c;

    for (int i = T.i_begin; i < T.i_end; ++i) {
      const int r0 = i * sh - a.ph;
      float acc = ident;
#pragma unroll 4
      for (int u = 0; u < kh; ++u) {
        const int r = r0 + u;
        if (T.col_ok && (unsigned)r < (unsigned)a.H) {
          float x = __ldg(pin + r * a.W);
          x = apply_generic(a.pro, paff, ch, x, in_idx0 + (int64_t)r * a.W);
          acc = red<IS_MAX>(acc, IS_MAX ? xorsign(x, flip) : x);
        }
      }
      float res = acc;
      for (int d = 1; d < kw; ++d) res = red<IS_MAX>(res, __shfl_down_sync(0xffffffffu, acc, d));
      if (T.out_lane) {
        if (IS_MAX) res = xorsign(res, flip);
        else res = __fdiv_rn(res, avg_div(a, i, T.j, kh, kw, sh, sw));
        const int64_t oidx = T.plane * (int64_t)HWo + (int64_t)i * a.Wo + T.j;
        res = apply_generic(a.epi, eaff, ch, res, oidx);
        __stcs(a.out + oidx, res);
      }
    }
  }
}

// One thread per output element (windows wider than a warp).  Never deferred.
template <bool IS_MAX>
__global__ void __launch_bounds__(kPoolBlock) pool_naive_kernel(PoolArgs a) {
  pdl_wait();                 // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  const int64_t HW = (int64_t)a.H * a.W, HWo = (int64_t)a.Ho * a.Wo;
  const int64_t total = a.n_planes * HWo;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = a.plane0 + o / HWo;
    const int64_t rem = o % HWo;
    const int i = (int)(rem / a.Wo), j = (int)(rem % a.Wo);
    const int ch = (int)(plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    load_affine(a.pro, ch, paff);
    load_affine(a.epi, ch, eaff);
    const float* pin = a.in + plane * HW;
    float acc = ident;
    for (int u = 0; u < a.kh; ++u) {
      const int r = i * a.sh - a.ph + u;
      if (r < 0 || r >= a.H) continue;
      for (int v = 0; v < a.kw; ++v) {
        const int q = j * a.sw - a.pw + v;
        if (q < 0 || q >= a.W) continue;
        float x = __ldg(pin + (int64_t)r * a.W + q);
        x = apply_generic(a.pro, paff, ch, x, plane * HW + (int64_t)r * a.W + q);
        acc = red<IS_MAX>(acc, x);
      }
    }
    if (!IS_MAX) acc = __fdiv_rn(acc, avg_div(a, i, j, a.kh, a.kw, a.sh, a.sw));
    const int64_t oidx = plane * HWo + rem;
    acc = apply_generic(a.epi, eaff, ch, acc, oidx);
    __stcs(a.out + oidx, acc);
  }
}


bool pool_has_specialisation(int kh, int kw, int sh, int sw) {
  if (kh != kw || sh != sw) return false;
  return (kh == 2 && sh == 2) || (kh == 3 && sh == 2) || (kh == 3 && sh == 1) || (kh == 7 && sh == 7);
}

int pool_spec_unroll(int k, int s) {
  if (k == 7) return 2;
  if (s == 1) return 8;
  return 8;
}

template <int K, int S, int U>
static void* spec_pick(bool is_max, int pc, int oc) {
  if (is_max) {  // prologue deferred: only the output class varies
    switch (oc) {
      case PC_NONE: return (void*)pool_cw_spec<K, K, S, S, true, U, PC_NONE, PC_NONE>;
      case PC_RELU: return (void*)pool_cw_spec<K, K, S, S, true, U, PC_NONE, PC_RELU>;
      case PC_AFFINE_RELU: return (void*)pool_cw_spec<K, K, S, S, true, U, PC_NONE, PC_AFFINE_RELU>;
      default: return (void*)pool_cw_spec<K, K, S, S, true, U, PC_NONE, PC_GENERIC>;
    }
  }
  (void)oc;
  switch (pc) {
    case PC_NONE: return (void*)pool_cw_spec<K, K, S, S, false, U, PC_NONE, PC_GENERIC>;
    case PC_RELU: return (void*)pool_cw_spec<K, K, S, S, false, U, PC_RELU, PC_GENERIC>;
    case PC_AFFINE_RELU: return (void*)pool_cw_spec<K, K, S, S, false, U, PC_AFFINE_RELU, PC_GENERIC>;
    default: return (void*)pool_cw_spec<K, K, S, S, false, U, PC_GENERIC, PC_GENERIC>;
  }
}

template <int K, int PADL, int VEC, int U>
static void* vec_pick(bool is_max, int pc, int oc) {
  if (is_max) {
    switch (oc) {
      case PC_NONE: return (void*)pool_vec<K, PADL, VEC, true, U, PC_NONE, PC_NONE>;
      case PC_RELU: return (void*)pool_vec<K, PADL, VEC, true, U, PC_NONE, PC_RELU>;
      case PC_AFFINE_RELU: return (void*)pool_vec<K, PADL, VEC, true, U, PC_NONE, PC_AFFINE_RELU>;
      default: return (void*)pool_vec<K, PADL, VEC, true, U, PC_NONE, PC_GENERIC>;
    }
  }
  (void)oc;
  switch (pc) {
    case PC_NONE: return (void*)pool_vec<K, PADL, VEC, false, U, PC_NONE, PC_GENERIC>;
    case PC_RELU: return (void*)pool_vec<K, PADL, VEC, false, U, PC_RELU, PC_GENERIC>;
    case PC_AFFINE_RELU: return (void*)pool_vec<K, PADL, VEC, false, U, PC_AFFINE_RELU, PC_GENERIC>;
    default: return (void*)pool_vec<K, PADL, VEC, false, U, PC_GENERIC, PC_GENERIC>;
  }
}

int pool_vec_width(int kh, int kw, int sh, int sw, int ph, int pw, int W, int Wo) {
  if (kh != kw || sh != 2 || sw != 2 || ph != pw) return 0;
  if (!((kh == 2 && ph == 0) || (kh == 3 && (ph == 0 || ph == 1)))) return 0;
  if ((Wo - 1) * 2 - pw + kw > W) return 0;   // right padding is not supported
  if (W % 4 == 0) return 4;
  if (W % 2 == 0) return 2;
  return 0;
}

int pool_vec_unroll(int vec) { return vec == 4 ? 4 : 8; }

void* pool_fn_global(int kind, const PoolArgs& a) {
  const bool m = a.is_max != 0;
  switch (kind) {
    case K_POOL_SPEC:
      if (m && a.pro.n > 0) return nullptr;  // max pools reach the specialised kernel deferred only
      if (a.kh == 2 && a.sh == 2) return spec_pick<2, 2, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 3 && a.sh == 2) return spec_pick<3, 2, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 3 && a.sh == 1) return spec_pick<3, 1, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 7 && a.sh == 7) return spec_pick<7, 7, 2>(m, a.pro_class, a.epi_class);
      return nullptr;
    case K_POOL_VEC: {
      if (m && a.pro.n > 0) return nullptr;
      const int vec = pool_vec_width(a.kh, a.kw, a.sh, a.sw, a.ph, a.pw, a.W, a.Wo);
      if (vec == 4) {
        if (a.kh == 2) return vec_pick<2, 0, 4, 4>(m, a.pro_class, a.epi_class);
        if (a.ph == 0) return vec_pick<3, 0, 4, 4>(m, a.pro_class, a.epi_class);
        return vec_pick<3, 1, 4, 4>(m, a.pro_class, a.epi_class);
      }
      if (vec == 2) {
        if (a.kh == 2) return vec_pick<2, 0, 2, 8>(m, a.pro_class, a.epi_class);
        if (a.ph == 0) return vec_pick<3, 0, 2, 8>(m, a.pro_class, a.epi_class);
        return vec_pick<3, 1, 2, 8>(m, a.pro_class, a.epi_class);
      }
      return nullptr;
    }
    case K_POOL_GENERIC: return m ? (void*)pool_cw_gen<true> : (void*)pool_cw_gen<false>;
    case K_POOL_NAIVE: return m ? (void*)pool_naive_kernel<true> : (void*)pool_naive_kernel<false>;
    default: return nullptr;
  }
}

}  // namespace bs
