// bs_kernels.cu -- sm_100a kernels of the depth-first stack executor.
//
// Every kernel reads each input byte from HBM once, applies the whole step in registers
// and writes each output byte once (§3.1; fig:trio-df P:L208-239):
//
//  * ew_kernel<PC>       -- a step with no pool (a6+a7+a10 collapse into one flat 128-bit
//                           streaming pass): "directly passing the values from one operation
//                           to another".  The paper launched one block per
//                           channel; here the grid is flat and each float4 finds
//                           its channel by magic-number division.
//  * pool_cw_spec<...>   -- a step [prologue | pool | epilogue] (a6-a10), "column walker":
//                           a warp is split into lane groups, each owning the input columns of
//                           a run of output columns of one (n, c) plane; the warp walks the
//                           plane's rows with U*s + (k - s) independent loads in flight per
//                           lane, reduces each window vertically in registers and horizontally
//                           with __shfl_down_sync -- overlapping 3x3/s2 windows need no shared
//                           memory and no HBM re-reads -- applies the epilogue and stores.
//                           The paper's stacked-pool kernel used B*C*Patches blocks with smem
//                           double buffers.
//  * pool_cw_gen<...>    -- the same walk for any window geometry (runtime k, s, p).
//  * pool_naive_kernel   -- one thread per output, for windows wider than a warp.
//
// Max-pool prologue deferral (R5): when every prologue op is monotone (folded BN,
// ReLU, SCALE) the host moves the prologue after the pool.  A composition of monotone
// fp32 functions f is monotone (IEEE rounding is monotone), so max over a window of f(x) is
// exactly f(max x) when f is non-decreasing and f(min x) when it is non-increasing; min is
// taken as -max(-x) by flipping sign bits (exact).  Padding stays absent: only
// loaded values are flipped.  Bit-identical to applying f per element, at 1/4 of the work.
//
// Floating point: explicitly-rounded intrinsics (__fmul_rn, __fadd_rn, __fmaf_rn,
// __fdiv_rn) everywhere, so no SCALE followed by ADD is contracted into an FMA; ReLU /
// Max / COPY / SCALE / ADD stacks stay bit-exact against the oracle.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <type_traits>

#include "bs_internal.h"

namespace bs {

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t s = 0;
  while (s < 32 && (uint64_t(1) << s) < d) ++s;
  f.s = s;
  f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.m) + n) >> f.s; }

__device__ __forceinline__ float relu(float x) { return x > 0.f ? x : 0.f; }

__device__ __forceinline__ float xorsign(float x, uint32_t m) { return __uint_as_float(__float_as_uint(x) ^ m); }

// ------------------------------------------------------------------ element-wise programs

// Params of the first kAffSlots AFFINE ops of P for channel ch.
__device__ __forceinline__ void load_affine(const OpProgram& P, int ch, float2 (&aff)[kAffSlots]) {
#pragma unroll
  for (int k = 0; k < kAffSlots; ++k) aff[k] = make_float2(1.f, 0.f);
  for (int o = 0; o < P.n; ++o) {
    if (P.kind[o] == DOP_AFFINE) {
      const int s = P.aff_slot[o];
      if (s == 0) aff[0] = __ldg(P.affine[o] + ch);
      else if (s == 1) aff[1] = __ldg(P.affine[o] + ch);
    }
  }
}

__device__ __forceinline__ float2 affine_of(const OpProgram& P, const float2 (&aff)[kAffSlots], int o, int ch) {
  const int s = P.aff_slot[o];
  return s == 0 ? aff[0] : s == 1 ? aff[1] : __ldg(P.affine[o] + ch);
}

// Sign-bit mask of the composite direction of the first P.n_deferred (monotone) ops.
__device__ __forceinline__ uint32_t deferred_flip(const OpProgram& P, const float2 (&aff)[kAffSlots], int ch) {
  uint32_t m = 0;
  for (int o = 0; o < P.n_deferred; ++o) {
    if (P.kind[o] == DOP_AFFINE) m ^= __float_as_uint(affine_of(P, aff, o, ch).x);
    else if (P.kind[o] == DOP_SCALE) m ^= __float_as_uint(P.alpha[o]);
  }
  return m & 0x80000000u;
}

// Generic interpreter on one value (op loop is runtime; one switch per op).
__device__ __forceinline__ float apply_generic(const OpProgram& P, const float2 (&aff)[kAffSlots], int ch, float x,
                                               int64_t idx) {
  for (int o = 0; o < P.n; ++o) {
    switch (P.kind[o]) {
      case DOP_AFFINE: {
        const float2 p = affine_of(P, aff, o, ch);
        x = __fmaf_rn(x, p.x, p.y);
        break;
      }
      case DOP_RELU: x = relu(x); break;
      case DOP_SCALE: x = __fmul_rn(x, P.alpha[o]); break;
      case DOP_ADD: x = __fadd_rn(x, __ldg(P.operand[o] + idx)); break;
      default: break;
    }
  }
  return x;
}

// Program of class PC on one value.  For PC_AFFINE*, aff[0] holds op 0's params.
template <int PC>
__device__ __forceinline__ float apply1(const OpProgram& P, const float2 (&aff)[kAffSlots], int ch, float x,
                                        int64_t idx) {
  if (PC == PC_NONE) return x;
  if (PC == PC_RELU) return relu(x);
  if (PC == PC_AFFINE) return __fmaf_rn(x, aff[0].x, aff[0].y);
  if (PC == PC_AFFINE_RELU) return relu(__fmaf_rn(x, aff[0].x, aff[0].y));
  return apply_generic(P, aff, ch, x, idx);
}

// Program of class PC on an array of N values (rows r0+q of one column); values whose row is
// outside the tensor are reset to `ident` (padding never goes through a prologue, H5).
template <int PC, int N>
__device__ __forceinline__ void apply_rows(const OpProgram& P, const float2 (&aff)[kAffSlots], int ch,
                                           float (&v)[N], const bool (&ok)[N], float ident, int64_t idx0,
                                           int stride) {
  if (PC == PC_NONE) return;
  if (PC == PC_GENERIC) {
    for (int o = 0; o < P.n; ++o) {
      const int kind = P.kind[o];
      if (kind == DOP_AFFINE) {
        const float2 p = affine_of(P, aff, o, ch);
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = __fmaf_rn(v[q], p.x, p.y);
      } else if (kind == DOP_RELU) {
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = relu(v[q]);
      } else if (kind == DOP_SCALE) {
        const float al = P.alpha[o];
#pragma unroll
        for (int q = 0; q < N; ++q) v[q] = __fmul_rn(v[q], al);
      } else if (kind == DOP_ADD) {
        const float* opp = P.operand[o];
#pragma unroll
        for (int q = 0; q < N; ++q)
          if (ok[q]) v[q] = __fadd_rn(v[q], __ldg(opp + idx0 + (int64_t)q * stride));
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = apply1<PC>(P, aff, ch, v[q], 0);
  }
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = ok[q] ? v[q] : ident;
}

// ------------------------------------------------------------------ ew_kernel

__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream4(float* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

constexpr int kEwBlock = 256;
constexpr int kEwUnroll = 4;  // float4 per thread per iteration (64 B in flight per thread)

template <int PC>
__global__ void __launch_bounds__(kEwBlock) ew_kernel(EwArgs a) {
  const uint32_t e_begin = (uint32_t)a.e_begin, e_end = (uint32_t)a.e_end;
  const uint32_t v_begin = (e_begin + 3u) & ~3u;
  const uint32_t v_end = (e_end & ~3u) > v_begin ? (e_end & ~3u) : v_begin;
  const uint32_t nv = (v_end - v_begin) >> 2;
  const OpProgram& P = a.prog;
  const uint32_t HW = a.hw.d, C = a.c.d;
  const float2* aff0p = (PC == PC_AFFINE || PC == PC_AFFINE_RELU) ? P.affine[0] : nullptr;

  const uint32_t stride = gridDim.x * kEwBlock * kEwUnroll;
  for (uint32_t base = blockIdx.x * kEwBlock * kEwUnroll + threadIdx.x; base < nv; base += stride) {
    float4 x[kEwUnroll], ad[kEwUnroll];
#pragma unroll
    for (int k = 0; k < kEwUnroll; ++k) {
      const uint32_t vi = base + k * kEwBlock;
      if (vi < nv) x[k] = ld_stream4(a.in + v_begin + 4u * vi);
    }
    if (PC == PC_GENERIC && a.add0_ptr != nullptr) {
#pragma unroll
      for (int k = 0; k < kEwUnroll; ++k) {
        const uint32_t vi = base + k * kEwBlock;
        if (vi < nv) ad[k] = ld_stream4(a.add0_ptr + v_begin + 4u * vi);
      }
    }
#pragma unroll
    for (int k = 0; k < kEwUnroll; ++k) {
      const uint32_t vi = base + k * kEwBlock;
      if (vi >= nv) continue;
      const uint32_t e = v_begin + 4u * vi;
      float v[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
      if (PC == PC_RELU) {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = relu(v[q]);
      } else {
        // channel of each element (a float4 spans at most two planes when H*W >= 4)
        uint32_t ch[4];
        const uint32_t plane = fdiv(e, a.hw);
        const uint32_t rem = e - plane * HW;
        const uint32_t c0 = plane - fdiv(plane, a.c) * C;
        const uint32_t c1 = (c0 + 1u == C) ? 0u : c0 + 1u;
        if (a.hw_ge4) {
#pragma unroll
          for (int q = 0; q < 4; ++q) ch[q] = (rem + q >= HW) ? c1 : c0;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t pq = fdiv(e + q, a.hw);
            ch[q] = pq - fdiv(pq, a.c) * C;
          }
        }
        if (PC == PC_AFFINE || PC == PC_AFFINE_RELU) {
          const float2 p0 = __ldg(aff0p + c0);
          float2 p[4] = {p0, p0, p0, p0};
          if (!(a.hw_ge4 && rem + 3u < HW)) {   // straddles a plane boundary
#pragma unroll
            for (int q = 1; q < 4; ++q) p[q] = __ldg(aff0p + ch[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            v[q] = __fmaf_rn(v[q], p[q].x, p[q].y);
            if (PC == PC_AFFINE_RELU) v[q] = relu(v[q]);
          }
        } else {  // generic: op-outer interpreter over the 4 values
          for (int o = 0; o < P.n; ++o) {
            const int kind = P.kind[o];
            if (kind == DOP_AFFINE) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 pp = __ldg(P.affine[o] + ch[q]);
                v[q] = __fmaf_rn(v[q], pp.x, pp.y);
              }
            } else if (kind == DOP_RELU) {
#pragma unroll
              for (int q = 0; q < 4; ++q) v[q] = relu(v[q]);
            } else if (kind == DOP_SCALE) {
              const float al = P.alpha[o];
#pragma unroll
              for (int q = 0; q < 4; ++q) v[q] = __fmul_rn(v[q], al);
            } else if (kind == DOP_ADD) {
              if (P.add_slot[o] == 0) {
                v[0] = __fadd_rn(v[0], ad[k].x);
                v[1] = __fadd_rn(v[1], ad[k].y);
                v[2] = __fadd_rn(v[2], ad[k].z);
                v[3] = __fadd_rn(v[3], ad[k].w);
              } else {
                const float4 t = ld_stream4(P.operand[o] + e);
                v[0] = __fadd_rn(v[0], t.x);
                v[1] = __fadd_rn(v[1], t.y);
                v[2] = __fadd_rn(v[2], t.z);
                v[3] = __fadd_rn(v[3], t.w);
              }
            }
          }
        }
      }
      st_stream4(a.out + e, make_float4(v[0], v[1], v[2], v[3]));
    }
  }
  // ---- scalar head [e_begin, v_begin) and tail [v_end, e_end): block 0 only
  if (blockIdx.x == 0) {
    const uint32_t nh = v_begin - e_begin;
    const uint32_t tail0 = v_end > e_begin ? v_end : e_begin;
    const uint32_t nt = e_end > tail0 ? e_end - tail0 : 0u;
    const uint32_t t = threadIdx.x;
    if (t < nh + nt) {
      const uint32_t e = t < nh ? e_begin + t : tail0 + (t - nh);
      if (e < e_end && !(e >= v_begin && e < v_end)) {
        const uint32_t plane = fdiv(e, a.hw);
        const int ch = (int)(plane - fdiv(plane, a.c) * C);
        float2 aff[kAffSlots];
        load_affine(P, ch, aff);
        a.out[e] = apply_generic(P, aff, ch, a.in[e], e);
      }
    }
  }
}

// ------------------------------------------------------------------ pool kernels

template <bool IS_MAX>
__device__ __forceinline__ float red(float acc, float x) {
  return IS_MAX ? fmaxf(acc, x) : __fadd_rn(acc, x);
}

// Avg-pool divisor: kh*kw with count_include_pad, else the number of real cells.
__device__ __forceinline__ float avg_div(const PoolArgs& a, int i, int j, int kh, int kw, int sh, int sw) {
  if (a.count_include_pad) return (float)(kh * kw);
  const int r0 = i * sh - a.ph, q0 = j * sw - a.pw;
  const int nr = min(a.H, r0 + kh) - max(0, r0);
  const int nq = min(a.W, q0 + kw) - max(0, q0);
  return (float)(nr * nq);
}

constexpr int kPoolBlock = 256;

// x / D for a compile-time divisor: an exact power-of-two scaling when D is a power of two
// (x * 2^-k is the correctly rounded x / 2^k), IEEE division otherwise.
template <int D>
__device__ __forceinline__ float div_by(float x) {
  if ((D & (D - 1)) == 0) return __fmul_rn(x, 1.0f / (float)D);
  return __fdiv_rn(x, (float)D);
}

// Per-task lane geometry shared by both column walkers.
struct LaneTask {
  int64_t plane;
  int c, j, i_begin, i_end;
  bool plane_ok, col_ok, out_lane;
};

__device__ __forceinline__ LaneTask decode_task(const PoolArgs& a, int t, int g, int l, int sw) {
  LaneTask T;
  const int cc = t % a.n_cc;
  const int t2 = t / a.n_cc;
  const int rb = t2 % a.n_rb;
  const int pg = t2 / a.n_rb;
  const int64_t pl_local = (int64_t)pg * a.G + g;
  T.plane_ok = (g < a.G) && (pl_local < a.n_planes);
  T.plane = a.plane0 + (T.plane_ok ? pl_local : 0);
  const int j0 = cc * a.Jg;
  T.c = j0 * sw - a.pw + l;
  T.col_ok = T.plane_ok && T.c >= 0 && T.c < a.W;
  const int jl = l / sw;
  T.j = j0 + jl;
  T.out_lane = T.plane_ok && (l - jl * sw == 0) && jl < a.Jg && T.j < a.Wo;
  T.i_begin = rb * a.rows_per_task;
  T.i_end = min(a.Ho, T.i_begin + a.rows_per_task);
  return T;
}

// Specialised column walker: compile-time window (KH x KW, stride SH x SW); U output rows per
// iteration -> NR = (U-1)*SH + KH independent row loads in flight per lane.
//   PC: class of the per-element prologue (avg pools; max pools run with it deferred, PC_NONE)
//   OC: class of the per-output program (deferred prologue + epilogue)
template <int KH, int KW, int SH, int SW, bool IS_MAX, int U, int PC, int OC>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_spec(PoolArgs a) {
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
          bool ok[NR];
#pragma unroll
          for (int q = 0; q < NR; ++q) ok[q] = true;
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

// ------------------------------------------------------------------ staged (TMA) walker
//
// For planes whose rows are not 16-byte aligned (AlexNet 55/27/13, 7x7), whole-plane tiles
// -- P contiguous planes, P*H*W*4 bytes, 16-byte aligned -- are moved HBM -> shared memory
// by one cp.async.bulk (the 1-D TMA engine) per tile, behind an mbarrier ring of `stages`
// buffers: warp 0 is the producer, warps 1..8 consume.  Consumers walk columns of the
// staged planes exactly like pool_cw_spec, reading shared memory (no alignment or sector
// waste, no halo re-reads from HBM), and store the outputs straight to HBM.  The paper's
// stacked kernel staged patches through two smem buffers swapped per step.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#ifndef BS_BULK_CHUNK
#define BS_BULK_CHUNK 8192
#endif
constexpr uint32_t kBulkChunk = BS_BULK_CHUNK;

// A tile's bytes sit in its stage at offset (global address mod 16), so the 16-byte-aligned
// middle of any plane range is one bulk copy and only <= 3 head and tail floats are copied
// by the producer lane; tiles need not start on 16-byte boundaries.
__host__ __device__ size_t pool_staged_stride(int tile_planes, int HW) {
  return ((size_t)tile_planes * HW * 4 + 16 + 127) / 128 * 128;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

size_t pool_staged_smem(int tile_planes, int HW, int stages) {
  return 128 + (size_t)stages * pool_staged_stride(tile_planes, HW);   // barriers, then stages
}

int pool_staged_unroll(int k, int s) { return k == 7 ? 1 : (s == 1 ? 4 : 4); }

template <int KH, int KW, int SH, int SW, bool IS_MAX, int U, int PC, int OC>
__global__ void __launch_bounds__(kStagedThreads) pool_staged(PoolArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  const int HW = a.H * a.W, HWo = a.Ho * a.Wo;
  const size_t tile_stride = pool_staged_stride(a.tile_planes, HW);
  float* stage0 = (float*)(smem + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)a.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 2);   // cp.async arrive (edges) + arrive.expect_tx (bulk body)
      mbar_init(&empty[s], ((a.tile_planes + a.G - 1) / a.G) * a.n_cc * a.n_rb);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: one elected lane issues the bulk copies
    if (lane == 0) {
      int k = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % a.stages;
        if (k >= a.stages) mbar_wait(&empty[s], ((k / a.stages) - 1) & 1);
        const int64_t pl0 = (int64_t)t * a.tile_planes;
        const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
        const float* src = a.in + (a.plane0 + pl0) * (int64_t)HW;
        const uint32_t head_off = (uint32_t)((uintptr_t)src & 15u);
        float* dst = (float*)((char*)stage0 + (size_t)s * tile_stride + head_off);
        const uint32_t nbytes = (uint32_t)np * (uint32_t)HW * 4u;
        const uint32_t h = min(nbytes, (16u - head_off) & 15u);        // head bytes before 16-B
        const uint32_t body = (nbytes - h) & ~15u;                      // aligned middle
        // head / tail floats: 4-byte cp.async (non-blocking), tracked by the full barrier
        for (uint32_t e = 0; e < h / 4; ++e) cp_async4(dst + e, src + e);
        for (uint32_t e = (h + body) / 4; e < nbytes / 4; ++e) cp_async4(dst + e, src + e);
        cp_async_mbar_arrive(&full[s]);   // arrival 1 of 2: when those copies have landed
        if (body) {
          mbar_arrive_expect_tx(&full[s], body);
          for (uint32_t off = 0; off < body; off += kBulkChunk) {
            const uint32_t n = min(kBulkChunk, body - off);
            bulk_g2s((char*)dst + h + off, (const char*)src + h + off, n, &full[s]);
          }
        } else {
          mbar_arrive(&full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: output-stationary walk over the staged planes
  // lane <-> output column j; the warp walks the output rows, each lane reducing its K
  // window columns of every new input row straight from shared memory (row reductions
  // of the last K-S rows slide along in registers).
  const int cw = warp - 1;
  const int g = lane / a.gw;
  const int l = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  // The tasks of this CTA's tiles are dealt round-robin to the consumer warps across tiles
  // (a tile with fewer tasks than warps does not idle them).  Every warp waits on every
  // tile's full barrier in tile order -- so it never waits on a ring slot more than one phase
  // ahead (mbarrier parity would alias) -- and runs the tasks dealt to it; a stage is
  // released when all tasks_per_tile tasks of its tile have arrived on empty[s].
  const int tasks_per_tile = ((a.tile_planes + a.G - 1) / a.G) * a.n_cc * a.n_rb;
  const int my_tiles = (n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  for (int k = 0; k < my_tiles; ++k) {
    const int t = (int)blockIdx.x + k * (int)gridDim.x;
    const int s = k % a.stages;
    const int64_t pl0 = (int64_t)t * a.tile_planes;
    const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
    const float* sm = (const float*)((const char*)stage0 + (size_t)s * tile_stride +
                                     ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW) & 15u));
    const int base = (int)(((int64_t)k * tasks_per_tile) % kStagedConsumerWarps);
    const int task0 = (cw - base + kStagedConsumerWarps) % kStagedConsumerWarps;
    mbar_wait(&full[s], (k / a.stages) & 1);   // every tile, in order (even with no task in it)
    for (int task = task0; task < tasks_per_tile; task += kStagedConsumerWarps) {
      const int rb = task % a.n_rb;
      const int cc = (task / a.n_rb) % a.n_cc;
      const int pg = task / (a.n_rb * a.n_cc);
      const int pin_tile = pg * a.G + g;
      const int j = cc * a.Jg + l;
      const bool out_lane = (g < a.G) && (pin_tile < np) && l < a.Jg && j < a.Wo;
      if (!out_lane) goto task_done;
      {
      const int64_t plane = a.plane0 + pl0 + pin_tile;
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
      // window columns, clamped into the row: a clamped duplicate of an in-window element
      // leaves a max unchanged (exact); for avg the out-of-range cells are zeroed below
      const int c0 = j * SW - a.pw;
      int coff[KW];
      bool cval[KW];
#pragma unroll
      for (int v = 0; v < KW; ++v) {
        cval[v] = (unsigned)(c0 + v) < (unsigned)a.W;
        coff[v] = min(max(c0 + v, 0), a.W - 1);
      }
      // per-lane byte pointers of the window columns in row 0; a row adds a warp-uniform
      // offset, so every shared-memory load is a single LDS [Rcol + URrow]
      const float* ps = sm + pin_tile * HW;
      const char* colp[KW];
#pragma unroll
      for (int v = 0; v < KW; ++v) colp[v] = (const char*)(ps + coff[v]);
      const unsigned W4 = 4u * (unsigned)a.W;
      const int64_t in_idx0 = plane * (int64_t)HW;
      float* pout = a.out + plane * (int64_t)HWo + j;
      const int64_t out_idx0 = plane * (int64_t)HWo + j;

      // reduction of input row rc (clamped; `rvalid` = the unclamped row is inside the tensor)
      auto rowred = [&](int rc, bool rvalid) -> float {
        const unsigned roff = (unsigned)rc * W4;
        float acc = 0.f;
#pragma unroll
        for (int v = 0; v < KW; ++v) {
          float x = *(const float*)(colp[v] + roff);
          if (IS_MAX) {
            x = xorsign(x, flip);
          } else {
            if (PC != PC_NONE) x = apply1<PC>(a.pro, paff, ch, x, in_idx0 + (int64_t)rc * a.W + coff[v]);
            x = (rvalid && cval[v]) ? x : 0.f;
          }
          acc = v == 0 ? x : red<IS_MAX>(acc, x);
        }
        return acc;
      };
      auto rowred_edge = [&](int r) -> float {
        return rowred(min(max(r, 0), a.H - 1), (unsigned)r < (unsigned)a.H);
      };

      // rolling window over output rows: each output row reduces its S new input rows (all
      // K rows when K <= S) and the K - S rows carried from the previous output row
      constexpr int CARRY = KH > SH ? KH - SH : 0;
      constexpr int NEW = KH - CARRY;
      const int i0 = rb * a.rows_per_task, i1 = min(a.Ho, i0 + a.rows_per_task);
      float hist[KH > 1 ? KH : 1];
      auto emit = [&](int i) {
        float res = hist[0];
#pragma unroll
        for (int q = 1; q < KH; ++q) res = red<IS_MAX>(res, hist[q]);
#pragma unroll
        for (int u = 0; u < CARRY; ++u) hist[u] = hist[u + NEW];
        if (IS_MAX) res = xorsign(res, flip);
        else res = a.count_include_pad ? div_by<KH * KW>(res) : __fdiv_rn(res, avg_div(a, i, j, KH, KW, SH, SW));
        res = apply1<OC>(a.epi, eaff, ch, res, out_idx0 + (int64_t)i * a.Wo);
        __stcs(pout + i * a.Wo, res);
      };
      // output rows whose window lies inside the tensor: [fb, fe) -- no clamps, no branches
      const int fb = max(i0, (a.ph + SH - 1) / SH);
      const int fe = max(fb, min(i1, (a.H - KH + a.ph) / SH + 1));
#pragma unroll
      for (int u = 0; u < CARRY; ++u) hist[u] = rowred_edge(i0 * SH - a.ph + u);
      for (int i = i0; i < fb; ++i) {
#pragma unroll
        for (int u = 0; u < NEW; ++u) hist[CARRY + u] = rowred_edge(i * SH - a.ph + CARRY + u);
        emit(i);
      }
#pragma unroll 4
      for (int i = fb; i < fe; ++i) {
#pragma unroll
        for (int u = 0; u < NEW; ++u) hist[CARRY + u] = rowred(i * SH - a.ph + CARRY + u, true);
        emit(i);
      }
      for (int i = fe; i < i1; ++i) {
#pragma unroll
        for (int u = 0; u < NEW; ++u) hist[CARRY + u] = rowred_edge(i * SH - a.ph + CARRY + u);
        emit(i);
      }
      }
    task_done:
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

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

__global__ void __launch_bounds__(kStagedThreads) seq_staged(SeqArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + 8;
  const size_t tile_stride = pool_staged_stride(a.tile_planes, a.in_plane);
  unsigned char* stage0 = smem + 128;
  float* work[2] = {(float*)(stage0 + (size_t)a.stages * tile_stride),
                    (float*)(stage0 + (size_t)a.stages * tile_stride) + a.work_floats};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)a.n_tiles;
  const int HW0 = a.in_plane;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer, as in pool_staged
    if (lane == 0) {
      int k = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % a.stages;
        if (k >= a.stages) mbar_wait(&empty[s], ((k / a.stages) - 1) & 1);
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
  int k = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int s = k % a.stages;
    mbar_wait(&full[s], (k / a.stages) & 1);
    const int64_t pl0 = (int64_t)t * a.tile_planes;
    const int np = (int)min((int64_t)a.tile_planes, a.n_planes - pl0);
    const float* src_base = (const float*)((const char*)stage0 + (size_t)s * tile_stride +
                                           ((uintptr_t)(a.in + (a.plane0 + pl0) * (int64_t)HW0) & 15u));
    for (int st_i = 0; st_i < a.n_steps; ++st_i) {
      const SeqStepDev& st = a.steps[st_i];
      const bool last = st_i == a.n_steps - 1;
      const float* in_buf = st_i == 0 ? src_base : work[(st_i - 1) & 1];
      float* out_buf = work[st_i & 1];
      const int HWi = st.H * st.W, HWo = st.Ho * st.Wo;
      // work items: (plane, output row, 32-column chunk); lane = output column
      const int nchunk = (st.Wo + 31) / 32;
      const int items = np * st.Ho * nchunk;
      for (int it = cw; it < items; it += kStagedConsumerWarps) {
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
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kStagedConsumerWarps) : "memory");   // step boundary
      if (st_i == 0 && cw == 0 && lane == 0) mbar_arrive(&empty[s]);   // stage buffer consumed
    }
  }
}

cudaError_t launch_seq(const SeqArgs& a, int grid, cudaStream_t st) {
  void* args[] = {(void*)&a};
  const size_t smem = seq_smem(a);
  cudaError_t e = cudaFuncSetAttribute((void*)seq_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernel((void*)seq_staged, dim3(grid), dim3(kStagedThreads), args, smem, st);
}

int seq_max_blocks_per_sm(const SeqArgs& a) {
  const size_t smem = seq_smem(a);
  int n = 0;
  if (cudaFuncSetAttribute((void*)seq_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (void*)seq_staged, kStagedThreads, smem) != cudaSuccess) n = 0;
  return n;
}

// Column walker with runtime window geometry (any kw <= 32 - (Jg-1)*sw).
template <bool IS_MAX>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_gen(PoolArgs a) {
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

// ------------------------------------------------------------------ dispatch

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

template <int K, int S, int U>
static void* staged_pick(bool is_max, int pc, int oc) {
  if (is_max) {
    switch (oc) {
      case PC_NONE: return (void*)pool_staged<K, K, S, S, true, U, PC_NONE, PC_NONE>;
      case PC_RELU: return (void*)pool_staged<K, K, S, S, true, U, PC_NONE, PC_RELU>;
      case PC_AFFINE_RELU: return (void*)pool_staged<K, K, S, S, true, U, PC_NONE, PC_AFFINE_RELU>;
      default: return (void*)pool_staged<K, K, S, S, true, U, PC_NONE, PC_GENERIC>;
    }
  }
  (void)oc;
  switch (pc) {
    case PC_NONE: return (void*)pool_staged<K, K, S, S, false, U, PC_NONE, PC_GENERIC>;
    case PC_RELU: return (void*)pool_staged<K, K, S, S, false, U, PC_RELU, PC_GENERIC>;
    case PC_AFFINE_RELU: return (void*)pool_staged<K, K, S, S, false, U, PC_AFFINE_RELU, PC_GENERIC>;
    default: return (void*)pool_staged<K, K, S, S, false, U, PC_GENERIC, PC_GENERIC>;
  }
}

static void* pool_fn(int kind, const PoolArgs& a) {
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
    case K_POOL_STAGED:
      if (m && a.pro.n > 0) return nullptr;
      if (a.kh == 2 && a.sh == 2) return staged_pick<2, 2, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 3 && a.sh == 2) return staged_pick<3, 2, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 3 && a.sh == 1) return staged_pick<3, 1, 8>(m, a.pro_class, a.epi_class);
      if (a.kh == 7 && a.sh == 7) return staged_pick<7, 7, 1>(m, a.pro_class, a.epi_class);
      return nullptr;
    case K_POOL_GENERIC: return m ? (void*)pool_cw_gen<true> : (void*)pool_cw_gen<false>;
    case K_POOL_NAIVE: return m ? (void*)pool_naive_kernel<true> : (void*)pool_naive_kernel<false>;
    default: return nullptr;
  }
}

static void* ew_fn(int pc) {
  switch (pc) {
    case PC_RELU: return (void*)ew_kernel<PC_RELU>;
    case PC_AFFINE: return (void*)ew_kernel<PC_AFFINE>;
    case PC_AFFINE_RELU: return (void*)ew_kernel<PC_AFFINE_RELU>;
    default: return (void*)ew_kernel<PC_GENERIC>;
  }
}

cudaError_t launch_ew(const EwArgs& a, int grid, int block, cudaStream_t st) {
  (void)block;
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(ew_fn(a.prog_class), dim3(grid), dim3(kEwBlock), args, 0, st);
}

cudaError_t launch_pool(const PoolArgs& a, int kind, int grid, int block, cudaStream_t st) {
  (void)block;
  void* fn = pool_fn(kind, a);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  void* args[] = {(void*)&a};
  if (kind == K_POOL_STAGED) {
    const size_t smem = pool_staged_smem(a.tile_planes, a.H * a.W, a.stages);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernel(fn, dim3(grid), dim3(kStagedThreads), args, smem, st);
  }
  return cudaLaunchKernel(fn, dim3(grid), dim3(kPoolBlock), args, 0, st);
}

int ew_max_blocks_per_sm(int pc) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ew_fn(pc), kEwBlock, 0) != cudaSuccess) n = 0;
  return n;
}

int pool_max_blocks_per_sm(int kind, const PoolArgs& a, int block) {
  (void)block;
  void* fn = pool_fn(kind, a);
  int n = 0;
  if (!fn) return 0;
  if (kind == K_POOL_STAGED) {
    const size_t smem = pool_staged_smem(a.tile_planes, a.H * a.W, a.stages);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kStagedThreads, smem) != cudaSuccess) n = 0;
    return n;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kPoolBlock, 0) != cudaSuccess) n = 0;
  return n;
}

}  // namespace bs
