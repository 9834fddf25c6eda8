// Grid-barrier variants on B200, 148 CTAs x 1024 threads (one per SM), cooperative launch.
//  A: red.release.add on a counter, ld.acquire polling of the counter
//  B: red.release.add on a counter, ld.relaxed polling + fence.acq_rel after
//  C: atom.acq_rel.add, last arriver publishes a flag (red.release.max), ld.acquire polling
//  D: as C with relaxed polling + fence.acq_rel after
//  E: as B, counter and polling spread: each CTA polls its own copy written by the last arriver
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_bench tools/barrier_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_add(unsigned *p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ unsigned atom_ar_add(unsigned *p) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(o) : "l"(p) : "memory");
  return o;
}
__device__ __forceinline__ void red_rel_max(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_ar() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int V>
__global__ void __launch_bounds__(1024, 1) bench(unsigned *cnt, unsigned *flag, unsigned *own,
                                                 int iters) {
  unsigned target = 0;
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      if (V == 0) {
        red_rel_add(cnt);
        while (ld_acq(cnt) < target) {
        }
      } else if (V == 1) {
        red_rel_add(cnt);
        while (ld_rlx(cnt) < target) {
        }
        fence_ar();
      } else if (V == 2 || V == 3) {
        if (atom_ar_add(cnt) + 1 == target) red_rel_max(flag, i);
        if (V == 2) {
          while (ld_acq(flag) < (unsigned)i) {
          }
        } else {
          while (ld_rlx(flag) < (unsigned)i) {
          }
          fence_ar();
        }
      } else {
        // E: last arriver writes every CTA's own flag line (one store per CTA)
        if (atom_ar_add(cnt) + 1 == target)
          for (unsigned b = 0; b < gridDim.x; ++b) st_rel(own + 32 * b, i);
        while (ld_rlx(own + 32 * blockIdx.x) < (unsigned)i) {
        }
        fence_ar();
      }
    }
    __syncthreads();
  }
}

int main() {
  unsigned *cnt, *flag, *own;
  cudaMalloc(&cnt, 128);
  cudaMalloc(&flag, 128);
  cudaMalloc(&own, 148 * 128);
  int iters = 4000;
  void *ks[] = {(void *)bench<0>, (void *)bench<1>, (void *)bench<2>, (void *)bench<3>,
                (void *)bench<4>};
  const char *names[] = {"A red.add + ld.acquire poll", "B red.add + relaxed poll + fence",
                         "C atom.add last-arriver flag + acquire poll",
                         "D atom.add last-arriver flag + relaxed poll + fence",
                         "E atom.add last-arriver writes per-CTA flags + relaxed poll"};
  for (int grid : {148, 74}) {
    for (int v = 0; v < 5; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(cnt, 0, 128);
        cudaMemset(flag, 0, 128);
        cudaMemset(own, 0, 148 * 128);
        void *args[] = {&cnt, &flag, &own, &iters};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(ks[v], grid, 1024, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("%3d CTAs  %-58s %.3f us/barrier  %s\n", grid, names[v], ms * 1e3 / iters,
                        cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
