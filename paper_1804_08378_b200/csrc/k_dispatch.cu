// k_dispatch.cu -- host-side kernel selection and launch helpers.
#include "bs_device.cuh"

#include <mutex>
#include <set>
#include <utility>

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


static void* pool_fn(int kind, const PoolArgs& a) {
  if (kind == K_POOL_PLANES) return pool_fn_planes(a);
  return kind == K_POOL_STAGED ? pool_fn_staged(a) : pool_fn_global(kind, a);
}

// The shared-memory kernels (staged pools, sequences) are configured ONCE per (kernel, device),
// under a lock, before their first launch or occupancy query:
//  * the dynamic shared-memory limit is raised to the device's opt-in maximum, never lowered
//    -- so plans needing different amounts can launch the same instantiation from several host
//    threads without a set-attribute / launch race (a launch uses only what it asks for);
//  * the maximum shared-memory carveout: an SM whose L1/shared split must change between two
//    kernels has to drain first, which defeats the PDL overlap of consecutive stacks needing
//    different amounts of shared memory (AlexNet step 46.1 -> 44.4 us).  The L1-streaming
//    kernels keep the default split (forcing it on them too cost DenseNet-121 17 %).
cudaError_t smem_kernel_setup(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;   // per (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  int optin = 0;
  cudaFuncAttributes fa;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return e;
  // static + dynamic shared memory must fit the opt-in limit
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes)) != cudaSuccess)
    return e;
#ifndef BS_NO_CARVEOUT
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared)) != cudaSuccess)
    return e;
#endif
  done.insert({fn, dev});
  return cudaSuccess;
}

cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
  if (smem > 0) {
    const cudaError_t e = smem_kernel_setup(fn);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef BS_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_pool(const PoolArgs& a, int kind, int grid, int block, cudaStream_t st) {
  (void)block;
  void* fn = pool_fn(kind, a);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  void* args[] = {(void*)&a};
  if (kind == K_POOL_STAGED) {
    const size_t smem = pool_staged_smem(a.tile_planes, a.H * a.W, a.Ho * a.Wo, a.stages);
    return launch_pdl(fn, dim3(grid), dim3(kStagedThreads), args, smem, st);
  }
  if (kind == K_POOL_PLANES)
    return launch_pdl(fn, dim3(grid), dim3(pool_planes_threads()), args, pool_planes_smem(a.H * a.W), st);
  return launch_pdl(fn, dim3(grid), dim3(kPoolBlock), args, 0, st);
}


int pool_max_blocks_per_sm(int kind, const PoolArgs& a, int block) {
  (void)block;
  void* fn = pool_fn(kind, a);
  int n = 0;
  if (!fn) return 0;
  if (kind == K_POOL_STAGED) {
    const size_t smem = pool_staged_smem(a.tile_planes, a.H * a.W, a.Ho * a.Wo, a.stages);
    if (smem_kernel_setup(fn) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kStagedThreads, smem) != cudaSuccess) n = 0;
    return n;
  }
  if (kind == K_POOL_PLANES) {
    const size_t smem = pool_planes_smem(a.H * a.W);
    if (smem_kernel_setup(fn) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, pool_planes_threads(), smem) != cudaSuccess) n = 0;
    return n;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kPoolBlock, 0) != cudaSuccess) n = 0;
  return n;
}


}  // namespace bs
