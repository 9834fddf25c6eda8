// L2 bandwidth probe ("a measured L2 peak, to be measured on
// the box"). Every CTA streams 16-byte loads over a buffer small enough to stay
// L2-resident, many times; bytes read / time = the L2 read bandwidth a
// gather-free kernel can reach. Also a read+write variant (the single-graph
// kernel reads and writes its messages). Build and run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2_bench.cu -o tools/l2_bench
//   tools/l2_bench > profiles/l2_peak.json
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2 *__restrict__ a, size_t n, int reps, double *sink) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
      double2 v;
      asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + i));
      acc += v.x + v.y;
    }
  if (acc == 1234.5) *sink = acc;
}

__global__ void rw(double2 *__restrict__ a, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
      double2 v;
      asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + i));
      v.x += 1.0;
      asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(a + i), "d"(v.x), "d"(v.y));
    }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"what\": \"L2-resident 16-byte ld.global.cg streams, grid %d x 4 CTAs x 512 threads, best of 5\", \"runs\": [", sms);
  const size_t mbs[] = {8, 16, 24, 32, 48, 64, 96};
  bool first = true;
  for (size_t mb : mbs) {
    const size_t bytes = mb << 20, n = bytes / 16;
    double2 *a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    const int reps = (int)(4096 / mb);
    float best_r = 1e30f, best_w = 1e30f;
    for (int t = 0; t < 6; ++t) {
      cudaEventRecord(e0);
      rd<<<sms * 4, 512>>>(a, n, reps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (t) best_r = ms < best_r ? ms : best_r;
      cudaEventRecord(e0);
      rw<<<sms * 4, 512>>>(a, n, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (t) best_w = ms < best_w ? ms : best_w;
    }
    const double gb = (double)bytes * reps / 1e9;
    printf("%s\n  {\"buffer_mb\": %zu, \"read_gbs\": %.1f, \"read_write_gbs\": %.1f}", first ? "" : ",",
           mb, gb / (best_r * 1e-3), 2 * gb / (best_w * 1e-3));
    first = false;
    cudaFree(a);
  }
  printf("\n]}\n");
  return cudaGetLastError() != cudaSuccess;
}
