// bs_kernels.cu -- sm_100a kernels of the depth-first stack executor.
//
// Every kernel reads each input byte from HBM once, applies the whole step in registers
// and writes each output byte once (§3.1; fig:trio-df P:L208-239):
//
//  * ew_kernel          -- a step with no pool (a6+a7+a10 collapse into one flat 128-bit
//                          streaming pass): "directly passing the values from one
//                          operation to another".  The paper launched one
//                          block per channel; here the grid is flat and each
//                          lane finds the channel of each element by magic-number division.
//  * pool_cw_spec/_gen  -- a step [prologue | pool | epilogue] (a6-a10).  "Column walker":
//                          a warp is split into lane groups, each owning the input columns
//                          of a run of output columns of one (n, c) plane; the warp walks the
//                          plane's rows, applies the prologue once per loaded element (only
//                          to REAL elements -- padding is absent/zero in the post-prologue
//                          domain), reduces the window vertically in registers
//                          and horizontally with __shfl_down_sync (overlapping 3x3/s2 windows
//                          need no shared memory and no HBM re-reads), applies the epilogue
//                          and stores.  The paper's stacked-pool kernel used
//                          B*C*Patches blocks with smem double buffers.
//  * pool_naive_kernel  -- one thread per output, for windows wider than a warp.
//
// Floating point: every op uses explicitly-rounded intrinsics (__fmul_rn, __fadd_rn,
// __fmaf_rn, __fdiv_rn) so nvcc never contracts a SCALE followed by an ADD into an FMA;
// that keeps ReLU/Max/COPY/SCALE/ADD stacks bit-exact against the oracle.
#include <cuda_runtime.h>
#include <math_constants.h>

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

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

// ------------------------------------------------------------------ element-wise programs

// Load the per-channel (scale, shift) of the first kAffSlots AFFINE ops into registers.
__device__ __forceinline__ void load_affine(const OpProgram& P, int ch, float2 (&aff)[kAffSlots]) {
#pragma unroll
  for (int k = 0; k < kAffSlots; ++k) aff[k] = make_float2(1.f, 0.f);
#pragma unroll
  for (int o = 0; o < kMaxOps; ++o) {
    if (o < P.n && P.kind[o] == DOP_AFFINE) {
      const int s = P.aff_slot[o];
      if (s == 0) aff[0] = __ldg(P.affine[o] + ch);
      else if (s == 1) aff[1] = __ldg(P.affine[o] + ch);
    }
  }
}

__device__ __forceinline__ float2 affine_of(const OpProgram& P, const float2 (&aff)[kAffSlots],
                                            int o, int ch) {
  const int s = P.aff_slot[o];
  return s == 0 ? aff[0] : s == 1 ? aff[1] : __ldg(P.affine[o] + ch);
}

// Apply program P to one value of channel `ch` (params of cached AFFINE ops in `aff`);
// `idx` is the flat index of the element in the tensor the ops act on (for ADD).
__device__ __forceinline__ float apply_prog(const OpProgram& P, const float2 (&aff)[kAffSlots],
                                            int ch, float x, int64_t idx) {
#pragma unroll
  for (int o = 0; o < kMaxOps; ++o) {
    if (o < P.n) {
      switch (P.kind[o]) {
        case DOP_AFFINE: {
          const float2 p = affine_of(P, aff, o, ch);
          x = __fmaf_rn(x, p.x, p.y);
          break;
        }
        case DOP_RELU: x = x > 0.f ? x : 0.f; break;
        case DOP_SCALE: x = __fmul_rn(x, P.alpha[o]); break;
        case DOP_ADD: x = __fadd_rn(x, __ldg(P.operand[o] + idx)); break;
        default: break;
      }
    }
  }
  return x;
}

// Same, channel params looked up per element (flat kernel's scalar head/tail).
__device__ __forceinline__ float apply_prog_ch(const OpProgram& P, float x, uint32_t ch, uint32_t e) {
#pragma unroll
  for (int o = 0; o < kMaxOps; ++o) {
    if (o < P.n) {
      switch (P.kind[o]) {
        case DOP_AFFINE: {
          const float2 p = __ldg(P.affine[o] + ch);
          x = __fmaf_rn(x, p.x, p.y);
          break;
        }
        case DOP_RELU: x = x > 0.f ? x : 0.f; break;
        case DOP_SCALE: x = __fmul_rn(x, P.alpha[o]); break;
        case DOP_ADD: x = __fadd_rn(x, __ldg(P.operand[o] + e)); break;
        default: break;
      }
    }
  }
  return x;
}

// ------------------------------------------------------------------ ew_kernel

__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream4(float* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

constexpr int kEwBlock = 256;
constexpr int kEwUnroll = 4;   // float4 per thread per iteration (64 B in flight per thread)

__global__ void __launch_bounds__(kEwBlock) ew_kernel(EwArgs a) {
  const uint32_t e_begin = (uint32_t)a.e_begin, e_end = (uint32_t)a.e_end;
  const uint32_t v_begin = (e_begin + 3u) & ~3u;
  const uint32_t v_end = (e_end & ~3u) > v_begin ? (e_end & ~3u) : v_begin;
  const uint32_t nv = (v_end - v_begin) >> 2;
  const OpProgram& P = a.prog;

  const uint32_t HW = a.hw.d, C = a.c.d;
  // ---- vector body
  const uint32_t stride = gridDim.x * kEwBlock * kEwUnroll;
  for (uint32_t base = blockIdx.x * kEwBlock * kEwUnroll + threadIdx.x; base < nv; base += stride) {
    float4 x[kEwUnroll];
    float4 ad[kEwUnroll];
#pragma unroll
    for (int k = 0; k < kEwUnroll; ++k) {
      const uint32_t vi = base + k * kEwBlock;
      if (vi < nv) x[k] = ld_stream4(a.in + v_begin + 4u * vi);
    }
    // the first ADD operand is streamed alongside the input
    if (a.add0_ptr != nullptr) {
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
      // channel of each of the 4 elements
      uint32_t ch[4];
      const uint32_t plane = fdiv(e, a.hw);
      const uint32_t rem = e - plane * HW;
      const uint32_t c0 = plane - fdiv(plane, a.c) * C;
      if (a.hw_ge4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t c1 = (c0 + 1u == C) ? 0u : c0 + 1u;
          ch[q] = (rem + q >= HW) ? c1 : c0;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t pq = fdiv(e + q, a.hw);
          ch[q] = pq - fdiv(pq, a.c) * C;
        }
      }
      float v[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
#pragma unroll
      for (int o = 0; o < kMaxOps; ++o) {
        if (o < P.n) {
          const int kind = P.kind[o];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            switch (kind) {
              case DOP_AFFINE: {
                const float2 p = __ldg(P.affine[o] + ch[q]);
                v[q] = __fmaf_rn(v[q], p.x, p.y);
                break;
              }
              case DOP_RELU: v[q] = v[q] > 0.f ? v[q] : 0.f; break;
              case DOP_SCALE: v[q] = __fmul_rn(v[q], P.alpha[o]); break;
              case DOP_ADD: {
                float tq;
                if (P.add_slot[o] == 0) {
                  const float4 t = ad[k];
                  tq = q == 0 ? t.x : q == 1 ? t.y : q == 2 ? t.z : t.w;
                } else {
                  tq = __ldg(P.operand[o] + e + q);
                }
                v[q] = __fadd_rn(v[q], tq);
                break;
              }
              default: break;
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
      uint32_t e = t < nh ? e_begin + t : tail0 + (t - nh);
      if (e < e_end && !(e >= v_begin && e < v_end)) {
        const uint32_t plane = fdiv(e, a.hw);
        const uint32_t ch = plane - fdiv(plane, a.c) * C;
        a.out[e] = apply_prog_ch(P, a.in[e], ch, e);
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
__device__ __forceinline__ float avg_div(const PoolArgs& a, int i, int j, int kh, int kw, int sh,
                                         int sw) {
  if (a.count_include_pad) return (float)(kh * kw);
  const int r0 = i * sh - a.ph, q0 = j * sw - a.pw;
  const int nr = min(a.H, r0 + kh) - max(0, r0);
  const int nq = min(a.W, q0 + kw) - max(0, q0);
  return (float)(nr * nq);
}

constexpr int kPoolBlock = 256;

// Specialised column walker: compile-time window (KH x KW, stride SH x SW), U output rows
// per iteration -> (U-1)*SH + KH independent row loads in flight per lane.
template <int KH, int KW, int SH, int SW, bool IS_MAX, int U>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_spec(PoolArgs a) {
  constexpr int NR = (U - 1) * SH + KH;
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int g = lane / a.gw;
  const int l = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  const int64_t HW = (int64_t)a.H * a.W, HWo = (int64_t)a.Ho * a.Wo;

  for (int64_t t = wg; t < a.n_tasks; t += nw) {
    int64_t tt = t;
    const int cc = (int)(tt % a.n_cc);
    tt /= a.n_cc;
    const int rb = (int)(tt % a.n_rb);
    tt /= a.n_rb;
    const int64_t pl_local = tt * a.G + g;
    const bool plane_ok = (g < a.G) && (pl_local < a.n_planes);
    const int64_t plane = a.plane0 + (plane_ok ? pl_local : 0);
    const int j0 = cc * a.Jg;
    const int c = j0 * SW - a.pw + l;
    const bool col_ok = plane_ok && c >= 0 && c < a.W;
    const int jl = l / SW;
    const int j = j0 + jl;
    const bool out_lane = plane_ok && (l - jl * SW == 0) && jl < a.Jg && j < a.Wo;
    const int ch = (int)(plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    load_affine(a.pro, ch, paff);
    load_affine(a.epi, ch, eaff);
    const float* pin = a.in + plane * HW;
    const int i_begin = rb * a.rows_per_task;
    const int i_end = min(a.Ho, i_begin + a.rows_per_task);

    for (int i = i_begin; i < i_end; i += U) {
      const int r0 = i * SH - a.ph;
      float v[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int r = r0 + q;
        v[q] = (col_ok && r >= 0 && r < a.H) ? __ldg(pin + (int64_t)r * a.W + c) : ident;
      }
      if (a.pro.n > 0) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = r0 + q;
          const bool ok = col_ok && r >= 0 && r < a.H;
          const float y = apply_prog(a.pro, paff, ch, v[q], plane * HW + (int64_t)r * a.W + c);
          v[q] = ok ? y : ident;   // padding stays absent (max) / zero (avg): never through BN
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u < i_end) {
          float acc = v[u * SH];
#pragma unroll
          for (int q = 1; q < KH; ++q) acc = red<IS_MAX>(acc, v[u * SH + q]);
          float res = acc;
#pragma unroll
          for (int d = 1; d < KW; ++d) res = red<IS_MAX>(res, __shfl_down_sync(0xffffffffu, acc, d));
          if (out_lane) {
            if (!IS_MAX) res = __fdiv_rn(res, avg_div(a, i + u, j, KH, KW, SH, SW));
            const int64_t oidx = plane * HWo + (int64_t)(i + u) * a.Wo + j;
            res = apply_prog(a.epi, eaff, ch, res, oidx);
            __stcs(a.out + oidx, res);
          }
        }
      }
    }
  }
}

// Column walker with runtime window geometry (any kw <= 32 - (Jg-1)*sw).
template <bool IS_MAX>
__global__ void __launch_bounds__(kPoolBlock) pool_cw_gen(PoolArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int g = lane / a.gw;
  const int l = lane - g * a.gw;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  const int64_t HW = (int64_t)a.H * a.W, HWo = (int64_t)a.Ho * a.Wo;
  const int kh = a.kh, kw = a.kw, sh = a.sh, sw = a.sw;

  for (int64_t t = wg; t < a.n_tasks; t += nw) {
    int64_t tt = t;
    const int cc = (int)(tt % a.n_cc);
    tt /= a.n_cc;
    const int rb = (int)(tt % a.n_rb);
    tt /= a.n_rb;
    const int64_t pl_local = tt * a.G + g;
    const bool plane_ok = (g < a.G) && (pl_local < a.n_planes);
    const int64_t plane = a.plane0 + (plane_ok ? pl_local : 0);
    const int j0 = cc * a.Jg;
    const int c = j0 * sw - a.pw + l;
    const bool col_ok = plane_ok && c >= 0 && c < a.W;
    const int jl = l / sw;
    const int j = j0 + jl;
    const bool out_lane = plane_ok && (l - jl * sw == 0) && jl < a.Jg && j < a.Wo;
    const int ch = (int)(plane % a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    load_affine(a.pro, ch, paff);
    load_affine(a.epi, ch, eaff);
    const float* pin = a.in + plane * HW;
    const int i_begin = rb * a.rows_per_task;
    const int i_end = min(a.Ho, i_begin + a.rows_per_task);

    for (int i = i_begin; i < i_end; ++i) {
      const int r0 = i * sh - a.ph;
      float acc = ident;
#pragma unroll 4
      for (int u = 0; u < kh; ++u) {
        const int r = r0 + u;
        if (col_ok && r >= 0 && r < a.H) {
          float x = __ldg(pin + (int64_t)r * a.W + c);
          x = apply_prog(a.pro, paff, ch, x, plane * HW + (int64_t)r * a.W + c);
          acc = red<IS_MAX>(acc, x);
        }
      }
      float res = acc;
      for (int d = 1; d < kw; ++d) res = red<IS_MAX>(res, __shfl_down_sync(0xffffffffu, acc, d));
      if (out_lane) {
        if (!IS_MAX) res = __fdiv_rn(res, avg_div(a, i, j, kh, kw, sh, sw));
        const int64_t oidx = plane * HWo + (int64_t)i * a.Wo + j;
        res = apply_prog(a.epi, eaff, ch, res, oidx);
        __stcs(a.out + oidx, res);
      }
    }
  }
}

// One thread per output element (windows wider than a warp).
template <bool IS_MAX>
__global__ void __launch_bounds__(kPoolBlock) pool_naive_kernel(PoolArgs a) {
  const int64_t HW = (int64_t)a.H * a.W, HWo = (int64_t)a.Ho * a.Wo;
  const int64_t total = a.n_planes * HWo;
  const float ident = IS_MAX ? -CUDART_INF_F : 0.f;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
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
        x = apply_prog(a.pro, paff, ch, x, plane * HW + (int64_t)r * a.W + q);
        acc = red<IS_MAX>(acc, x);
      }
    }
    if (!IS_MAX) acc = __fdiv_rn(acc, avg_div(a, i, j, a.kh, a.kw, a.sh, a.sw));
    const int64_t oidx = plane * HWo + rem;
    acc = apply_prog(a.epi, eaff, ch, acc, oidx);
    __stcs(a.out + oidx, acc);
  }
}

// ------------------------------------------------------------------ dispatch

bool pool_has_specialisation(int kh, int kw, int sh, int sw) {
  if (kh != kw || sh != sw) return false;
  return (kh == 2 && sh == 2) || (kh == 3 && sh == 2) || (kh == 3 && sh == 1) || (kh == 7 && sh == 7);
}

template <bool M>
static void* spec_fn(int k, int s) {
  if (k == 2 && s == 2) return (void*)pool_cw_spec<2, 2, 2, 2, M, 4>;
  if (k == 3 && s == 2) return (void*)pool_cw_spec<3, 3, 2, 2, M, 4>;
  if (k == 3 && s == 1) return (void*)pool_cw_spec<3, 3, 1, 1, M, 4>;
  if (k == 7 && s == 7) return (void*)pool_cw_spec<7, 7, 7, 7, M, 1>;
  return nullptr;
}

static void* pool_fn(int kind, const PoolArgs& a) {
  const bool m = a.is_max != 0;
  switch (kind) {
    case K_POOL_SPEC: return m ? spec_fn<true>(a.kh, a.sh) : spec_fn<false>(a.kh, a.sh);
    case K_POOL_GENERIC: return m ? (void*)pool_cw_gen<true> : (void*)pool_cw_gen<false>;
    case K_POOL_NAIVE: return m ? (void*)pool_naive_kernel<true> : (void*)pool_naive_kernel<false>;
    default: return nullptr;
  }
}

cudaError_t launch_ew(const EwArgs& a, int grid, int block, cudaStream_t st) {
  (void)block;
  ew_kernel<<<grid, kEwBlock, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pool(const PoolArgs& a, int kind, int grid, int block, cudaStream_t st) {
  (void)block;
  void* fn = pool_fn(kind, a);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  void* args[] = {(void*)&a};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kPoolBlock), args, 0, st);
}

int ew_max_blocks_per_sm(int block) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ew_kernel, kEwBlock, 0) != cudaSuccess) n = 0;
  (void)block;
  return n;
}

int pool_max_blocks_per_sm(int kind, const PoolArgs& a, int block) {
  (void)block;
  void* fn = pool_fn(kind, a);
  int n = 0;
  if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kPoolBlock, 0) != cudaSuccess) n = 0;
  return n;
}

}  // namespace bs
