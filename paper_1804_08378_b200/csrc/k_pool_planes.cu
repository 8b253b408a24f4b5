// k_pool_planes.cu -- whole-plane windows (global pools): one output per small plane.
#include "bs_device.cuh"

#include <type_traits>

namespace bs {

// A pool whose window is the whole plane (kh = H, kw = W, no padding: Ho = Wo = 1) reduces each
// plane to one value -- DenseNet-121's final BN -> ReLU -> AvgPool7x7 on 7 x 7 planes
// (PAPER.md tbl:eval_detailkernel).  The traffic is read-dominated (49 floats in, 1
// out) and the planes are small and unaligned (49 floats = 196 B).  A warp takes 32 consecutive
// planes -- 32 * H * W floats, contiguous and 16-B aligned whatever H * W is: its lane 0 moves
// them HBM -> the warp's shared-memory slice with ONE bulk copy (cp.async.bulk, the 1-D TMA;
// no registers hold data in flight, so ~36 warps = ~220 KB per SM are in flight, like the
// streaming ceiling kernel), the warp waits on its mbarrier, and lane l reduces plane l: the
// prologue per element, the sum (max), the divisor, the epilogue, one coalesced 128-B store of
// the warp's 32 outputs.  Lane l reads its plane at stride H * W floats: odd H * W hits 32
// distinct banks; even H * W walks each plane from a lane-dependent start (element (l + j) mod
// HW at step j) so the banks stay distinct.  Flat grid: one chunk per warp.

constexpr int kPlanesWarps = 4;                  // warps per CTA
constexpr int kPlanesThreads = 32 * kPlanesWarps;
constexpr int kPlanesMaxHW = 64;                 // planes of <= 64 floats (<= 8 KB per warp slice)

template <bool IS_MAX, int PC, int OC>
__global__ void __launch_bounds__(kPlanesThreads) pool_planes(PoolArgs a) {
  extern __shared__ __align__(128) float4 psm[];
  __shared__ uint64_t wbar[kPlanesWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HW = a.H * a.W;
  float4* const w4 = psm + (size_t)warp * (8 * HW);                // this warp's slice (32 planes)
  float* const wf = (float*)w4;
  const int64_t ck = (int64_t)blockIdx.x * kPlanesWarps + warp;    // this warp's chunk
  const int64_t n_chunks = (a.n_planes + 31) / 32;
  if (lane == 0) {
    mbar_init(&wbar[warp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_wait();                   // previous kernel on the stream complete + visible
  pdl_launch_dependents();
  if (ck >= n_chunks) return;
  const int64_t p0 = ck * 32;
  const int np = (int)min((int64_t)32, a.n_planes - p0);
  const float* src = a.in + (a.plane0 + p0) * (int64_t)HW;
  const int nfl = np * HW;
  if (((uintptr_t)src & 15u) == 0) {
    // one bulk copy (TMA) of the chunk's 16-B-aligned body, the <= 3 tail floats by plain loads
    const uint32_t body = (uint32_t)(nfl & ~3) * 4u;
    if (lane == 0) {
      mbar_arrive_expect_tx(&wbar[warp], body);
      if (body) bulk_g2s(wf, src, body, &wbar[warp]);
    }
    if (lane < (nfl & 3)) wf[(nfl & ~3) + lane] = __ldg(src + (nfl & ~3) + lane);
    mbar_wait_sleep(&wbar[warp], 0);
  } else {                                             // (a launch on an unaligned plane offset)
    for (int e = lane; e < nfl; e += 32) wf[e] = __ldg(src + e);
  }
  __syncwarp();
  if (lane < np) {
    const uint32_t plane = (uint32_t)(a.plane0 + p0 + lane);
    const int ch = (int)(plane - fdiv(plane, a.cdiv) * (uint32_t)a.C);
    float2 paff[kAffSlots], eaff[kAffSlots];
    if (PC == PC_AFFINE || PC == PC_AFFINE_RELU) paff[0] = __ldg(a.pro.affine[0] + ch);
    else if (PC == PC_GENERIC) load_affine(a.pro, ch, paff);
    if (OC == PC_AFFINE || OC == PC_AFFINE_RELU) eaff[0] = __ldg(a.epi.affine[0] + ch);
    else if (OC == PC_GENERIC) load_affine(a.epi, ch, eaff);
    const float* pp = wf + lane * HW;
    const int64_t in0 = (int64_t)plane * HW;
    float acc = IS_MAX ? -CUDART_INF_F : 0.f;
    if (HW & 1) {
      for (int j = 0; j < HW; ++j) acc = red<IS_MAX>(acc, apply1<PC>(a.pro, paff, ch, pp[j], in0 + j));
    } else {
      int j = lane % HW;
      for (int q = 0; q < HW; ++q) {
        acc = red<IS_MAX>(acc, apply1<PC>(a.pro, paff, ch, pp[j], in0 + j));
        j = j + 1 == HW ? 0 : j + 1;
      }
    }
    if (!IS_MAX) acc = __fdiv_rn(acc, (float)HW);
    acc = apply1<OC>(a.epi, eaff, ch, acc, (int64_t)plane);
    __stcs(a.out + plane, acc);
  }
}

static void* planes_pick(const PoolArgs& a) {
  const int pc = a.pro_class, oc = a.epi_class;
  auto by_oc = [&](auto is_max, auto pcc) -> void* {
    constexpr bool M = decltype(is_max)::value;
    constexpr int P = decltype(pcc)::value;
    if (oc == PC_NONE) return (void*)pool_planes<M, P, PC_NONE>;
    return (void*)pool_planes<M, P, PC_GENERIC>;
  };
  using T = std::true_type;
  using F = std::false_type;
  if (a.is_max) {
    if (pc == PC_NONE) return by_oc(T(), std::integral_constant<int, PC_NONE>());
    if (pc == PC_RELU) return by_oc(T(), std::integral_constant<int, PC_RELU>());
    if (pc == PC_AFFINE_RELU) return by_oc(T(), std::integral_constant<int, PC_AFFINE_RELU>());
    return by_oc(T(), std::integral_constant<int, PC_GENERIC>());
  }
  if (pc == PC_NONE) return by_oc(F(), std::integral_constant<int, PC_NONE>());
  if (pc == PC_RELU) return by_oc(F(), std::integral_constant<int, PC_RELU>());
  if (pc == PC_AFFINE_RELU) return by_oc(F(), std::integral_constant<int, PC_AFFINE_RELU>());
  return by_oc(F(), std::integral_constant<int, PC_GENERIC>());
}

bool pool_planes_applies(int H, int W, int kh, int kw, int ph, int pw) {
  return kh == H && kw == W && ph == 0 && pw == 0 && H * W <= kPlanesMaxHW;
}

void* pool_fn_planes(const PoolArgs& a) {
  const int HW = a.H * a.W;
  if (!pool_planes_applies(a.H, a.W, a.kh, a.kw, a.ph, a.pw)) return nullptr;
  (void)HW;
  return planes_pick(a);
}

size_t pool_planes_smem(int HW) { return (size_t)kPlanesWarps * 8 * HW * sizeof(float4); }
int pool_planes_threads() { return kPlanesThreads; }

}  // namespace bs
