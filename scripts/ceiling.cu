// ceiling.cu -- dev microbenchmark (not part of the product): the best a streaming kernel can
// do on this B200 for the pooling traffic shape (read B bytes, write B/4) at the AlexNet stack
// sizes, over rotating buffers (> 4x L2), launches captured in a CUDA graph.
//   ldg   : flat grid-stride, 4 x LDG.128 in flight per thread, 1 STG.32 per float4 read
//   tma   : persistent ring of cp.async.bulk tiles (1 producer lane), 8 consumer warps read
//           the stage and write 1/4 of it
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ceiling scripts/ceiling.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void marr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

__global__ void __launch_bounds__(288) ring(const float* in, float* out, int n_tiles, int tile_bytes, int stages) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  unsigned char* st0 = sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { minit(&full[s], 1); minit(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        int s = k % stages;
        if (k >= stages) mwait(&empty[s], ((k / stages) - 1) & 1);
        mexp(&full[s], tile_bytes);
        bulk(st0 + (size_t)s * tile_bytes, (const char*)in + (size_t)t * tile_bytes, tile_bytes, &full[s]);
      }
    }
    return;
  }
  int k = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    int s = k % stages;
    mwait(&full[s], (k / stages) & 1);
    const float4* p = (const float4*)(st0 + (size_t)s * tile_bytes);
    const int n4 = tile_bytes / 16;
    float* o = out + (size_t)t * n4;
    for (int e = (warp - 1) * 32 + lane; e < n4; e += 256) {
      float4 v = p[e];
      __stcs(o + e, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    __syncwarp();
    if (lane == 0) marr(&empty[s]);
  }
}

__global__ void __launch_bounds__(256) ldg4(const float4* __restrict__ in, float* __restrict__ out, long n4) {
  const long stride = (long)gridDim.x * blockDim.x;
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(out + i + u * stride, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
  }
  for (; i < n4; i += stride) { float4 v = __ldcs(in + i); __stcs(out + i, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w))); }
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t req : {99123200ul, 71663616ul, 22151168ul, 822083584ul}) {
    const size_t bytes = req / 65536 * 65536;
    const int nset = (int)((4 * 126e6) / bytes) + 2;
    std::vector<float*> ins(nset), outs(nset);
    for (int q = 0; q < nset; ++q) { cudaMalloc(&ins[q], bytes); cudaMalloc(&outs[q], bytes / 4); cudaMemset(ins[q], 0, bytes); }
    auto timeit = [&](auto launch, const char* name, int p1, int p2, int p3) {
      const int R = 2 * nset;
      for (int r = 0; r < R; ++r) launch(r % nset);
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < R; ++r) launch(r % nset);
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(a, st);
      for (int q = 0; q < 5; ++q) cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double us = ms * 1e3 / (5 * R);
      printf("{\"bytes\": %zu, \"kernel\": \"%s\", \"p1\": %d, \"p2\": %d, \"p3\": %d, \"us\": %.2f, \"GBps\": %.0f}\n", bytes, name, p1, p2, p3, us,
             bytes * 1.25 / (us * 1e-6) / 1e9);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    };
    for (int per : {2, 4, 8, 16}) {
      const int grid = per * nsm;
      const long n4 = bytes / 16;
      timeit([&](int q) { ldg4<<<grid, 256, 0, st>>>((const float4*)ins[q], outs[q], n4); }, "ldg", per, 0, 0);
    }
    for (int tile : {8192, 16384, 32768}) {
      for (int stages : {2, 4, 6}) {
        size_t smem = 128 + (size_t)stages * tile;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ring, 288, smem);
        int n_tiles = (int)(bytes / tile);
        int grid = per * nsm;
        timeit([&](int q) { ring<<<grid, 288, smem, st>>>(ins[q], outs[q], n_tiles, tile, stages); }, "tma", tile, stages, per);
      }
    }
    for (int q = 0; q < nset; ++q) { cudaFree(ins[q]); cudaFree(outs[q]); }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
