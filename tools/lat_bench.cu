// Latency microbenchmarks on B200 (one warp): dependent fp64 ops, the shared-
// reciprocal division, L2-hit loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I paper_2509_22337_b200/csrc -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "lbp_kernels.cuh"
using namespace hbp::dev;

__global__ void dep_dmul(double x, int n, double *out, long long *cyc) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dmul_rn(a, x);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / n;
}
__global__ void dep_dfma(double x, int n, double *out, long long *cyc) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __fma_rn(a, x, 1e-300);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / n;
}
__global__ void dep_div2(double x, int n, double *out, long long *cyc) {
  double a = x, b = 1.0 - x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double t = __dadd_rn(a, b);
    div2_rn(a, b, t, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a + b;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / n;
}
__global__ void dep_ddiv(double x, int n, double *out, long long *cyc) {
  double a = x, b = 1.0 - x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double t = __dadd_rn(a, b);
    a = __ddiv_rn(a, t);
    b = __ddiv_rn(b, t);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a + b;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / n;
}
__global__ void chase(const int *next, int steps, long long *out, int *sink) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  *out = (t1 - t0) / steps;
  *sink = p;
}
// throughput: many warps doing independent div2 chains
__global__ void thr_div2(double x, int n, double *out) {
  double a = x + threadIdx.x * 1e-9, b = 1.0 - a;
  for (int i = 0; i < n; ++i) {
    double t = __dadd_rn(a, b);
    div2_rn(a, b, t, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b;
}

int main() {
  double *out;
  long long *cyc, h;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  int n = 4096;
  auto run = [&](const char *name, void (*k)(double, int, double *, long long *)) {
    k<<<1, 32>>>(0.3, n, out, cyc);
    k<<<1, 32>>>(0.3, n, out, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %lld cycles per step\n", name, h);
  };
  run("dependent DMUL", dep_dmul);
  run("dependent DFMA", dep_dfma);
  run("normalise pair (DADD + div2_rn)", dep_div2);
  run("normalise pair (DADD + 2x __ddiv_rn)", dep_ddiv);
  // one SM, 768 threads: the same dependent chains (a fused level's shape)
  auto run768 = [&](const char *name, void (*k)(double, int, double *, long long *)) {
    k<<<1, 768>>>(0.3, n, out, cyc);
    k<<<1, 768>>>(0.3, n, out, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %lld cycles per step (768 threads, 1 SM)\n", name, h);
  };
  run768("dependent DMUL", dep_dmul);
  run768("normalise pair (DADD + div2_rn)", dep_div2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  thr_div2<<<148 * 4, 256>>>(0.3, 1000, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("div2 throughput: %.3e normalised pairs/s\n", 148.0 * 4 * 256 * 1000 / (ms * 1e-3));
  int m = 4 << 20;
  int *hnext = new int[m];
  for (int i = 0; i < m; ++i) hnext[i] = i;
  unsigned s = 12345;
  for (int i = m - 1; i > 0; --i) {
    s = s * 1664525u + 1013904223u;
    int j = s % (i + 1);
    int t = hnext[i]; hnext[i] = hnext[j]; hnext[j] = t;
  }
  int *next, *sink;
  cudaMalloc(&next, m * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(next, hnext, m * 4, cudaMemcpyHostToDevice);
  chase<<<1, 1>>>(next, 20000, cyc, sink);
  chase<<<1, 1>>>(next, 20000, cyc, sink);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent ld.cg, 16 MB L2-resident:        %lld cycles\n", h);
  return 0;
}
