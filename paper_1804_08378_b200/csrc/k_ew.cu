// k_ew.cu -- the element-wise streaming kernel (steps without a pool).
#include "bs_device.cuh"

namespace bs {

template <int PC, int U>
__global__ void __launch_bounds__(kEwBlock) ew_kernel(EwArgs a) {
  pdl_wait();                 // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  const uint32_t e_begin = (uint32_t)a.e_begin, e_end = (uint32_t)a.e_end;
  const uint32_t v_begin = (e_begin + 3u) & ~3u;
  const uint32_t v_end = (e_end & ~3u) > v_begin ? (e_end & ~3u) : v_begin;
  const uint32_t nv = (v_end - v_begin) >> 2;
  const OpProgram& P = a.prog;
  const uint32_t HW = a.hw.d, C = a.c.d;
  const float2* aff0p = (PC == PC_AFFINE || PC == PC_AFFINE_RELU) ? P.affine[0] : nullptr;

  const uint32_t stride = gridDim.x * kEwBlock * U;
  for (uint32_t base = blockIdx.x * kEwBlock * U + threadIdx.x; base < nv; base += stride) {
    float4 x[U], ad[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t vi = base + k * kEwBlock;
      if (vi < nv) x[k] = ld_stream4(a.in + v_begin + 4u * vi);
    }
    if (PC == PC_GENERIC && a.add0_ptr != nullptr) {
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t vi = base + k * kEwBlock;
        if (vi < nv) ad[k] = ld_stream4(a.add0_ptr + v_begin + 4u * vi);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
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


template <int U>
static void* ew_fn_u(int pc) {
  switch (pc) {
    case PC_RELU: return (void*)ew_kernel<PC_RELU, U>;
    case PC_AFFINE: return (void*)ew_kernel<PC_AFFINE, U>;
    case PC_AFFINE_RELU: return (void*)ew_kernel<PC_AFFINE_RELU, U>;
    default: return (void*)ew_kernel<PC_GENERIC, U>;
  }
}

// U = float4s per thread per iteration: 4 (64 B in flight per thread) for large tensors, 1 for
// small ones, which then spread over 4x more threads (one wave of latency-bound loads).
static void* ew_fn(int pc, int unroll = kEwUnroll) { return unroll == 1 ? ew_fn_u<1>(pc) : ew_fn_u<kEwUnroll>(pc); }

cudaError_t launch_ew(const EwArgs& a, int grid, int block, cudaStream_t st) {
  (void)block;
  void* args[] = {(void*)&a};
  return launch_pdl(ew_fn(a.prog_class, a.unroll), dim3(grid), dim3(kEwBlock), args, 0, st);
}

int ew_max_blocks_per_sm(int pc) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ew_fn(pc), kEwBlock, 0) != cudaSuccess) n = 0;
  return n;
}


}  // namespace bs
