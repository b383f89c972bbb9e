// Microbenchmark (diagnostics): cost of a hardware cluster barrier and of a
// DSMEM plane push + barrier for a 16-CTA x 512-thread cluster on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_cluster scripts/probe_cluster.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void csync_aligned() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void k(long long* out, int mode, int iters, int bytes) {
  extern __shared__ __align__(16) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), n = cl.num_blocks();
  for (int i = threadIdx.x; i < 2 * bytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(r, 0, 0, 0);
  csync();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 1 || mode == 3) {
      uint4* dst = reinterpret_cast<uint4*>(cl.map_shared_rank((void*)(sm + bytes), (r + 1) % n));
      const uint4* src = reinterpret_cast<const uint4*>(sm);
      for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = src[i];
    }
    if (mode == 2 || mode == 3) {
      __syncthreads();
      csync_aligned();
    } else {
      __syncthreads();
      csync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[r] = (t1 - t0) / iters;
}

__global__ void kgrid(long long* out, int iters) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

int main() {
  long long* d;
  cudaMalloc(&d, 4096 * 8);
  long long h[16];
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int csz : {8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      for (int bytes : {512, 2048, 8192}) {
        if (mode % 2 == 0 && bytes != 512) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(csz);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 2 * bytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, mode, 1000, bytes);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, csz * 8, cudaMemcpyDeviceToHost);
        printf("cluster %2d mode %d (%s) bytes %5d: %lld cycles/iter (%s)\n", csz, mode,
               mode == 0 ? "sync" : mode == 1 ? "push+sync" : mode == 2 ? "aligned sync" : "push+aligned",
               bytes, h[0], cudaGetErrorString(e));
      }
    }
  }
  for (int per : {1, 2}) {
    int nb = 148 * per;
    void* args[] = {&d, (void*)new int(1000)};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)kgrid, nb, 512, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync %d CTAs x 512: %lld cycles/iter (%s)\n", nb, h[0], cudaGetErrorString(e));
  }
  return 0;
}
