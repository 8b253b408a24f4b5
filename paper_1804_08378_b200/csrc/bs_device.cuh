// bs_device.cuh -- device helpers shared by the sm_100a kernel translation units
// (k_*.cu): element-wise programs, pool reductions, mbarrier / bulk-copy (TMA) wrappers.
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
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include <type_traits>

#include "bs_internal.h"

namespace bs {

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
// Explicit shared-memory accesses on 32-bit shared addresses: pointers chosen at run time among
// several smem buffers otherwise fall back to generic LD/ST (slower, 64-bit addressing).
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));   // ordered by the volatile barriers
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// The same wait with a suspend-time hint: the waiting thread sleeps until the phase completes
// (or the hint expires) instead of spinning on try_wait -- a producer or an idle consumer warp
// then takes no issue slots from the warps doing the work.  (The try_wait loop is the standard
// PTX idiom, as in CUTLASS cutlass/arch/barrier.h, BSD-3-Clause, NVIDIA.)
#ifndef BS_MBAR_SLEEP_NS
#define BS_MBAR_SLEEP_NS 0x989680
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(BS_MBAR_SLEEP_NS)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}



// shared -> global bulk copy (TMA store) in the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// every committed bulk store of this thread has finished reading shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store of this thread is complete (writes performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// order this thread's generic-proxy shared-memory writes before later async-proxy (bulk copy) reads
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#ifndef BS_BULK_CHUNK
#define BS_BULK_CHUNK 8192
#endif
constexpr uint32_t kBulkChunk = BS_BULK_CHUNK;

// A tile's bytes sit in its stage at offset (global address mod 16), so the 16-byte-aligned
// middle of any plane range is one bulk copy and only <= 3 head and tail floats are copied
// by the producer lane; tiles need not start on 16-byte boundaries.

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}


// Programmatic dependent launch (PDL): every kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so its CTAs may become resident while the
// previous kernel on the stream drains.  pdl_wait() blocks until that kernel has completed and
// its writes are visible -- it precedes every global-memory access of a kernel, so a stack
// after a dependent producer (or a serialised sequence) stays correct; pdl_launch_dependents()
// lets the next kernel start its launch as early as possible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One-time (per kernel, device) shared-memory attributes of the smem kernels (k_dispatch.cu).
cudaError_t smem_kernel_setup(const void* fn);

// Launch with the PDL attribute (see pdl_wait).
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st);

// Kernel pickers of the pool translation units (nullptr: no kernel for this geometry).
void* pool_fn_global(int kind, const PoolArgs& a);   // K_POOL_SPEC / VEC / GENERIC / NAIVE
void* pool_fn_staged(const PoolArgs& a);             // K_POOL_STAGED
void* pool_fn_planes(const PoolArgs& a);             // K_POOL_PLANES

}  // namespace bs
