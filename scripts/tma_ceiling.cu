// tma_ceiling.cu -- microbenchmark (not part of the product): how fast can a persistent
// CTA ring of cp.async.bulk copies stream HBM -> shared memory on this B200, with consumers
// that (0) only release the stage, (1) read every staged word, or (2) also write 1/4 of the
// bytes back to HBM (the pooling traffic shape)?  Also a plain 128-bit LDG read+write copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ceiling scripts/tma_ceiling.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
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

template <int MODE>
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
  float acc = 0.f;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    int s = k % stages;
    mwait(&full[s], (k / stages) & 1);
    if (MODE >= 1) {
      const float* p = (const float*)(st0 + (size_t)s * tile_bytes);
      const int nf = tile_bytes / 4;
      float local = 0.f;
      for (int e = (warp - 1) * 32 + lane; e < nf; e += 256) local = fmaxf(local, p[e]);
      if (MODE == 2) {
        // write one float per 4 read: out tile = tile_bytes/4
        float* o = out + (size_t)t * (nf / 4);
        for (int e = (warp - 1) * 32 + lane; e < nf / 4; e += 256) __stcs(o + e, local + p[e * 4]);
      }
      acc += local;
    }
    __syncwarp();
    if (lane == 0) marr(&empty[s]);
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void copy4(const float4* in, float4* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = __ldg(in + i);
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? (size_t)atoll(argv[1]) / 65536 * 65536 : (1ull << 30);   // input bytes
  float *in, *out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMemset(in, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 2; mode < 3; ++mode)
    for (int tile : {8192, 16384, 32768, 49152}) {
      for (int stages : {2, 3, 4, 6, 8}) {
        size_t smem = 128 + (size_t)stages * tile;
        if (smem > 227 * 1024) continue;
        void* fn = mode == 0 ? (void*)ring<0> : mode == 1 ? (void*)ring<1> : (void*)ring<2>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 288, smem);
        int n_tiles = (int)(bytes / tile);
        int grid = per * nsm;
        void* args[] = {&in, &out, &n_tiles, &tile, &stages};
        for (int w = 0; w < 2; ++w) cudaLaunchKernel(fn, grid, 288, args, smem, 0);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) cudaLaunchKernel(fn, grid, 288, args, smem, 0);   // back to back
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        double moved = (double)bytes * (mode == 2 ? 1.25 : 1.0);
        printf("{\"mode\": %d, \"tile\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"GBps\": %.0f}\n", mode, tile, stages, per,
               moved * 10 / (ms / 1e3) / 1e9);
      }
    }
  size_t n4 = bytes / 16 / 2;
  for (int w = 0; w < 2; ++w) copy4<<<nsm * 8, 256>>>((const float4*)in, (float4*)out, n4);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) copy4<<<nsm * 8, 256>>>((const float4*)in, (float4*)out, n4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"mode\": \"ldg_copy\", \"GBps\": %.0f}\n", (double)bytes * 10 / (ms / 1e3) / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
