// Grid barrier through thread-block clusters, B200, one CTA (768 threads) per SM, cooperative:
//  A (cs=1): every CTA red.release.add on one counter, thread 0 polls it (ld.acquire)
//  cs=2/4/8: cluster barrier (release/acquire), the cluster's CTA 0 arrives for the whole
//  cluster and polls, then a second cluster barrier releases the others
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_cluster_bench tools/barrier_cluster_bench.cu
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_add(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(768, 1) bench(unsigned *cnt, int iters, int cs, unsigned *sink) {
  unsigned target = 0;
  const unsigned nlead = gridDim.x / cs;
  for (int i = 1; i <= iters; ++i) {
    // a little scattered-store traffic before each barrier (like a phase's tail)
    sink[(blockIdx.x * 7919u + threadIdx.x * 131u + i * 977u) & ((1u << 22) - 1)] = i;
    if (cs == 1) {
      __syncthreads();
      target += gridDim.x;
      if (threadIdx.x == 0) {
        red_rel_add(cnt, 1);
        while (ld_acq(cnt) < target) {
        }
      }
      __syncthreads();
    } else {
      cluster_sync_all();
      target += nlead;
      if (cluster_rank() == 0 && threadIdx.x == 0) {
        red_rel_add(cnt, 1);
        while (ld_acq(cnt) < target) {
        }
      }
      cluster_sync_all();
    }
  }
}

int main() {
  unsigned *cnt, *sink;
  cudaMalloc(&cnt, 128);
  cudaMalloc(&sink, 4u << 22);
  const int iters = 2000;
  for (int cs : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.blockDim = dim3(768);
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int ncl = 0;
    cfg.gridDim = dim3(148 / cs * cs);
    cudaOccupancyMaxActiveClusters(&ncl, (void *)bench, &cfg);
    const int grid = std::min(ncl * cs, 148 / cs * cs);  // one CTA per SM
    cfg.gridDim = dim3(grid);
    int cs_ = cs;
    int it_ = iters;
    void *args[] = {&cnt, &it_, &cs_, &sink};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cnt, 0, 4);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchKernelExC(&cfg, (void *)bench, args);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("cluster %d: grid %d, %.3f us per barrier (%s)\n", cs, grid, 1e3 * ms / iters,
                      cudaGetErrorString(e));
    }
  }
  return 0;
}
