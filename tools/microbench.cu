// Microbenchmarks for the executor's fixed costs on B200:
//  1. grid barrier (arrive/wait on a global counter) with 148 x 1024 threads
//  2. dependent global-load latency (pointer chase) in an L2-resident buffer
//  3. one "phase" of independent loads + fp64 division per thread
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(1024, 1) barrier_bench(unsigned *bar, int iters, long long *out) {
  unsigned expected = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
    }
    expected += gridDim.x;
    if (threadIdx.x == 0) {
      while (ld_acquire(bar) < expected) {
      }
      __threadfence();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}

__global__ void chase(const int *next, int steps, long long *out, int *sink) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  *out = (t1 - t0) / steps;
  *sink = p;
}

int main() {
  unsigned *bar;
  long long *out, h;
  cudaMalloc(&bar, 4);
  cudaMalloc(&out, 8);
  int iters = 2000;
  for (int g : {1, 8, 32, 148}) {
    cudaMemset(bar, 0, 4);
    void *args[] = {&bar, &iters, &out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)barrier_bench, g, 1024, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("grid barrier: %3d CTAs x 1024 thr: %.3f us per barrier (%lld cycles)  err=%s\n", g,
           ms * 1e3 / iters, h, cudaGetErrorString(cudaGetLastError()));
  }
  // pointer chase, 16 MB working set (L2 resident), random permutation
  int n = 4 << 20;
  int *hnext = new int[n];
  for (int i = 0; i < n; ++i) hnext[i] = i;
  unsigned s = 12345;
  for (int i = n - 1; i > 0; --i) {
    s = s * 1664525u + 1013904223u;
    int j = s % (i + 1);
    int t = hnext[i]; hnext[i] = hnext[j]; hnext[j] = t;
  }
  int *next, *sink;
  cudaMalloc(&next, n * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(next, hnext, n * 4, cudaMemcpyHostToDevice);
  chase<<<1, 1>>>(next, 20000, out, sink);  // warm
  chase<<<1, 1>>>(next, 20000, out, sink);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("dependent ld.cg latency, 16 MB L2-resident: %lld cycles\n", h);
  return 0;
}
