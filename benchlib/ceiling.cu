// ceiling.cu -- the "same-shape ideal streaming kernel" of SURVEY.md §8(d) (protocol item 6), a
// MEASUREMENT tool for bench.py, not part of the product: it moves exactly a stack's algorithmic
// bytes -- reads n_in floats with 128-bit loads, writes n_out floats with 128-bit stores, no real
// work -- so a stack's time can be reported against the best a streaming kernel achieves for the
// same byte counts and read/write mix on this GPU (launch ramp and drain included).
//
// Three variants (bench.py takes the fastest per stack):
//   bsc_ldg  : flat grid-stride; per iteration 4 x LDG.128 in flight per thread
//              (ld.global.nc.L1::no_allocate), then the proportional share of STG.128 (.cs).
//   bsc_flat : one block per 256 x U float4s, no loop: U loads in flight per thread, then the
//              block's proportional output share (for equal sizes: a plain copy kernel).
//   bsc_ring : persistent CTAs; one elected lane bulk-copies (cp.async.bulk, TMA) input tiles into
//              a shared-memory ring behind mbarriers, 8 consumer warps read each tile and write
//              its proportional share of the output.
// Written values are data-dependent (a max over what was read) so no load can be elided.
// Built by __graft_entry__.build() into benchlib/libceiling.so (sm_100a).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ float4 ldnc4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stcs4(float4* p, float v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ float mx4(float4 v) { return fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)); }

// scalar tails (n not a multiple of 4): one thread
__device__ void tails(const float* in, int64_t n_in, float* out, int64_t n_out, float acc) {
  for (int64_t e = n_in / 4 * 4; e < n_in; ++e) acc = fmaxf(acc, in[e]);
  for (int64_t e = n_out / 4 * 4; e < n_out; ++e) out[e] = acc;
}

__global__ void __launch_bounds__(256) k_ldg(const float4* __restrict__ in, int64_t n4i, float4* __restrict__ out,
                                             int64_t n4o, const float* in1, int64_t n_in, float* out1, int64_t n_out) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float acc = -CUDART_INF_F;
  const int64_t per_it = 4 * T;
  const int64_t n_it = (n4i + per_it - 1) / per_it;
  for (int64_t it = 0; it < n_it; ++it) {
    const int64_t i0 = it * per_it + g;
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * T < n4i ? ldnc4(in + i0 + u * T) : make_float4(acc, acc, acc, acc);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = fmaxf(acc, mx4(v[u]));
    // this iteration's share of the output, spread over all threads
    const int64_t o0 = (int64_t)((double)it * n4o / n_it), o1 = (int64_t)((double)(it + 1) * n4o / n_it);
    for (int64_t o = o0 + g; o < o1; o += T) stcs4(out + o, acc);
  }
  if (g == 0) tails(in1, n_in, out1, n_out, acc);
}

// Flat: one block per 256 * U float4s of the input (no grid-stride loop): each thread loads its U
// float4s (all in flight), then the block writes its proportional share of the output at the
// matching position -- for n_out == n_in exactly a copy kernel, for a pool's 4:1 ratio the
// streaming pattern of a one-pass pool kernel.
template <int U>
__global__ void __launch_bounds__(256) k_flat(const float4* __restrict__ in, int64_t n4i, float4* __restrict__ out,
                                              int64_t n4o, const float* in1, int64_t n_in, float* out1, int64_t n_out) {
  const int64_t b0 = (int64_t)blockIdx.x * 256 * U;
  float acc = -CUDART_INF_F;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = b0 + u * 256 + threadIdx.x;
    v[u] = i < n4i ? ldnc4(in + i) : make_float4(acc, acc, acc, acc);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) acc = fmaxf(acc, mx4(v[u]));
  const int64_t b1 = b0 + 256 * U < n4i ? b0 + 256 * U : n4i;
  const int64_t o0 = (int64_t)((double)b0 * n4o / n4i), o1 = (int64_t)((double)b1 * n4o / n4i);
  for (int64_t o = o0 + threadIdx.x; o < o1; o += 256) stcs4(out + o, acc);
  if (blockIdx.x == 0 && threadIdx.x == 0) tails(in1, n_in, out1, n_out, acc);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(288) k_ring(const float* __restrict__ in, int64_t n_in, float* __restrict__ out,
                                              int64_t n_out, int tile_bytes, int stages) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  unsigned char* st0 = sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t body = n_in / 4 * 16;                      // bytes moved by bulk copies
  const int64_t n_tiles = (body + tile_bytes - 1) / tile_bytes;
  const int64_t n4o = n_out / 4;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&empty[s])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D1;\nbra W1;\nD1:\n}\n" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
  };
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = k % stages;
        if (k >= stages) wait(&empty[s], ((k / stages) - 1) & 1);
        const uint32_t nb = (uint32_t)min((int64_t)tile_bytes, body - t * tile_bytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(nb) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(st0 + (size_t)s * tile_bytes)),
            "l"((const char*)in + t * tile_bytes), "r"(nb), "r"(su32(&full[s]))
            : "memory");
      }
    }
    return;
  }
  const int c = threadIdx.x - 32;
  float acc = -CUDART_INF_F;
  int k = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int s = k % stages;
    wait(&full[s], (k / stages) & 1);
    const int n4 = (int)(min((int64_t)tile_bytes, body - t * tile_bytes) / 16);
    const float4* p = (const float4*)(st0 + (size_t)s * tile_bytes);
    for (int e = c; e < n4; e += 256) acc = fmaxf(acc, mx4(p[e]));
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    const int64_t o0 = t * n4o / n_tiles, o1 = (t + 1) * n4o / n_tiles;
    for (int64_t o = o0 + c; o < o1; o += 256) stcs4((float4*)out + o, acc);
  }
  if (blockIdx.x == 0 && c == 0) tails(in, n_in, out, n_out, acc);
}

int g_sms = 0;
int sms() {
  if (!g_sms) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, d);
  }
  return g_sms;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int bsc_ldg(const float* in, int64_t n_in, float* out, int64_t n_out,
                                                   int blocks_per_sm, cudaStream_t st) {
  const int64_t n4i = n_in / 4;
  int64_t grid = (int64_t)blocks_per_sm * sms();
  grid = grid < 1 ? 1 : grid;
  const int64_t need = (n4i + 1023) / 1024;   // at least one float4 per thread per iteration
  if (need < grid) grid = need < 1 ? 1 : need;
  k_ldg<<<(int)grid, 256, 0, st>>>((const float4*)in, n4i, (float4*)out, n_out / 4, in, n_in, out, n_out);
  return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int bsc_flat(const float* in, int64_t n_in, float* out, int64_t n_out,
                                                    int unroll, cudaStream_t st) {
  const int64_t n4i = n_in / 4;
  const int64_t per = 256 * (int64_t)unroll;
  const int grid = (int)(n4i > 0 ? (n4i + per - 1) / per : 1);
  if (unroll == 1) k_flat<1><<<grid, 256, 0, st>>>((const float4*)in, n4i, (float4*)out, n_out / 4, in, n_in, out, n_out);
  else if (unroll == 2) k_flat<2><<<grid, 256, 0, st>>>((const float4*)in, n4i, (float4*)out, n_out / 4, in, n_in, out, n_out);
  else k_flat<4><<<grid, 256, 0, st>>>((const float4*)in, n4i, (float4*)out, n_out / 4, in, n_in, out, n_out);
  return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int bsc_ring(const float* in, int64_t n_in, float* out, int64_t n_out,
                                                    int tile_bytes, int stages, int ctas_per_sm, cudaStream_t st) {
  if (stages < 2 || stages > 8 || tile_bytes % 16) return (int)cudaErrorInvalidValue;
  const size_t smem = 128 + (size_t)stages * tile_bytes;
  cudaError_t e = cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  const int64_t n_tiles = (n_in / 4 * 16 + tile_bytes - 1) / tile_bytes;
  int64_t grid = (int64_t)ctas_per_sm * sms();
  if (n_tiles < grid) grid = n_tiles < 1 ? 1 : n_tiles;
  k_ring<<<(int)grid, 288, smem, st>>>(in, n_in, out, n_out, tile_bytes, stages);
  return (int)cudaGetLastError();
}

}  // extern "C"
