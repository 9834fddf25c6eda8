// Persistent level executor: the whole iteration loop of engine.run
// (engine.py:531-594) in ONE cooperative kernel launch.
//
// Per iteration the kernel walks the plan's phases (layout.cpp): phase 0 is
// the variable side of batch 0 fused with the marginals + delta of the
// previous iteration (both read the same factor-to-variable state), then
// alternating factor-side / variable-side phases for every batch. Phases
// with enough work use the whole grid and a grid barrier; small levels
// (the hundreds of 27..1,800-edge levels of a SEQFIX schedule) run on CTA 0
// alone with __syncthreads between them, while the other CTAs skip ahead to
// the next grid barrier. Convergence (delta < tol), max_iterations, the
// time limit and underflow are decided on the device after phase 0; there
// is no host round trip until the run ends.
//
// Work items: a "node" item computes every outgoing message of one
// variable (or factor) from a single read of its row -- the O(d) form of the
// reference's per-target O(d^2) gathers (_product_scan, engine.py:168-183;
// _body_target_products :198-226) -- sharing prefix products across
// targets, which is exact because a left-to-right product's prefixes are
// the reference's own partial products. A "target" item is one edge
// (partially covered rows in levelled schedules). Items are sorted by
// (role, degree) on the host so warps are uniform in branch and trip count.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"
#include "lbp_kernels.cuh"

namespace hbp {

using namespace dev;

constexpr int kThreads = 1024;

struct Ctrl {
  unsigned int bar;  // grid barrier arrivals (monotonic)
  int iterations;
  int converged;
  int stop;          // 1 converged, 2 max_iterations, 3 time limit, 4 underflow
  unsigned long long t0;
};

struct KParams {
  // layout
  const int *frow;
  const double2 *fpar;
  const int *vtof_twin;
  const int *vrow;
  const int *ftov_twin;
  const int *vorig;
  int V, F, f_or_begin;
  int E;
  double2 *vtof, *ftov, *marg;
  double *prev;
  // plan
  const Phase *phases;
  int nphases;
  const int *vnode, *fnode;
  const int4 *vt, *ft;
  // control
  Ctrl *ctrl;
  unsigned long long *delta_bits;  // [max_it + 2]
  int *uf_msg;                     // [max_it + 2] bit0 vtof, bit1 ftov
  int *uf_marg;                    // [max_it + 2]
  int *uf_mwhere;                  // [max_it + 2] smallest underflowing variable
  unsigned long long *uf_where;    // [max_it + 2] (phase<<33 | kind<<32 | pos) or var
  int *tflag;                      // [max_it + 2]
  double2 *hist;                   // [max_it][V] or null
  int max_it;
  int normalize;
  double tol;
  long long time_limit_ns;
};

// --------------------------------------------------------------------------------------
// grid barrier (arrive / wait on a monotonic counter)

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void bar_arrive(Ctrl *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&c->bar, 1u);
  }
}

__device__ __forceinline__ void bar_wait(Ctrl *c, unsigned target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(&c->bar) < target) {
    }
    __threadfence();  // gpu-scope fence: also invalidates this SM's L1
  }
  __syncthreads();
}

// --------------------------------------------------------------------------------------
// message output with normalisation + underflow flag (engine.py:155-165)

__device__ __forceinline__ void put_message(const KParams &P, double2 *dst, double a0, double a1,
                                            int it, int phase, int kind, int pos) {
  if (P.normalize) {
    double t = add(a0, a1);
    if (t < kMinMessageSum) {
      atomicOr(&P.uf_msg[it], 1 << kind);
      atomicMin(&P.uf_where[it], ((unsigned long long)phase << 33) |
                                     ((unsigned long long)kind << 32) | (unsigned)pos);
    }
    a0 = dvd(a0, t);
    a1 = dvd(a1, t);
  }
  *dst = make_double2(a0, a1);
}

// marginal of iteration it-1 + its |dP1| (engine.py:510-523, :572)
__device__ __forceinline__ void put_marginal(const KParams &P, int v, double q0, double q1, int it,
                                             unsigned long long &dmax) {
  double t = add(q0, q1);
  int orig = P.vorig[v];
  if (t < kMinMessageSum) {
    atomicOr(&P.uf_marg[it - 1], 1);
    atomicMin(&P.uf_mwhere[it - 1], orig);
  }
  double p0 = dvd(q0, t);
  double p1 = sub(1.0, p0);
  double d = fabs(sub(p1, P.prev[v]));
  unsigned long long bits = (unsigned long long)__double_as_longlong(d);
  dmax = bits > dmax ? bits : dmax;
  P.prev[v] = p1;
  P.marg[orig] = make_double2(p0, p1);
  if (P.hist) P.hist[(size_t)(it - 2) * P.V + orig] = make_double2(p0, p1);
}

// --------------------------------------------------------------------------------------
// variable node: marginal and/or every non-unary outgoing vtof message

template <int D>
__device__ __forceinline__ void vnode_fixed(const KParams &P, int v, int r, bool do_marg,
                                            bool do_vtof, int it, int phase,
                                            unsigned long long &dmax) {
  double x0[D], x1[D];
  int tw[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double2 m = P.ftov[r + i];
    x0[i] = m.x;
    x1[i] = m.y;
  }
  if (do_vtof) {
#pragma unroll
    for (int i = 0; i < D; ++i) tw[i] = P.ftov_twin[r + i];
  }
  // a = left-to-right prefix product x[0] * ... * x[j-1] (reference acc)
  double a0 = 1.0, a1 = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (do_vtof && tw[j] >= 0) {
      double b0 = a0, b1 = a1;
#pragma unroll
      for (int i = j + 1; i < D; ++i) {
        b0 = mul(b0, x0[i]);
        b1 = mul(b1, x1[i]);
      }
      put_message(P, P.vtof + tw[j], b0, b1, it, phase, 0, tw[j]);
    }
    a0 = mul(a0, x0[j]);
    a1 = mul(a1, x1[j]);
  }
  if (do_marg) put_marginal(P, v, a0, a1, it, dmax);
}

__device__ __noinline__ void vnode_generic(const KParams &P, int v, int r, int d, bool do_marg,
                                           bool do_vtof, int it, int phase,
                                           unsigned long long &dmax) {
  if (do_vtof) {
    for (int j = 0; j < d; ++j) {
      int tw = P.ftov_twin[r + j];
      if (tw < 0) continue;
      double b0 = 1.0, b1 = 1.0;
      for (int i = 0; i < d; ++i) {
        if (i == j) continue;
        double2 m = P.ftov[r + i];
        b0 = mul(b0, m.x);
        b1 = mul(b1, m.y);
      }
      put_message(P, P.vtof + tw, b0, b1, it, phase, 0, tw);
    }
  }
  if (do_marg) {
    double q0 = 1.0, q1 = 1.0;
    for (int i = 0; i < d; ++i) {
      double2 m = P.ftov[r + i];
      q0 = mul(q0, m.x);
      q1 = mul(q1, m.y);
    }
    put_marginal(P, v, q0, q1, it, dmax);
  }
}

__device__ __forceinline__ void vnode(const KParams &P, int v, bool do_marg, bool do_vtof, int it,
                                      int phase, unsigned long long &dmax) {
  const int r = P.vrow[v];
  const int d = P.vrow[v + 1] - r;
  switch (d) {
    case 1: vnode_fixed<1>(P, v, r, do_marg, do_vtof, it, phase, dmax); break;
    case 2: vnode_fixed<2>(P, v, r, do_marg, do_vtof, it, phase, dmax); break;
    case 3: vnode_fixed<3>(P, v, r, do_marg, do_vtof, it, phase, dmax); break;
    case 4: vnode_fixed<4>(P, v, r, do_marg, do_vtof, it, phase, dmax); break;
    default: vnode_generic(P, v, r, d, do_marg, do_vtof, it, phase, dmax); break;
  }
}

// single vtof target: row [r, r+d) minus slot x (engine.py:186-195)
__device__ __forceinline__ void vt_target(const KParams &P, int4 t, int it, int phase) {
  double b0 = 1.0, b1 = 1.0;
  for (int i = 0; i < t.z; ++i) {
    if (i == t.w) continue;
    double2 m = P.ftov[t.y + i];
    b0 = mul(b0, m.x);
    b1 = mul(b1, m.y);
  }
  put_message(P, P.vtof + t.x, b0, b1, it, phase, 0, t.x);
}

// --------------------------------------------------------------------------------------
// factor node: every outgoing ftov message of one factor

template <int D, int KIND>
__device__ __forceinline__ void fnode_fixed(const KParams &P, int f, int r, int it, int phase) {
  const double2 pp = P.fpar[f];
  const double p1 = pp.x, p2 = pp.y;
  double m0[D], m1[D];
  int tw[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double2 m = P.vtof[r + i];
    m0[i] = m.x;
    m1[i] = m.y;
    tw[i] = P.vtof_twin[r + i];
  }
  // s_i = m0 + m1 and tail_i = m1 (AND) / m0 (OR) for body slots
  double s[D];
#pragma unroll
  for (int i = 1; i < D; ++i) s[i] = add(m0[i], m1[i]);
  {  // head target: products over body slots 1..D-1
    double h1 = 1.0, h2 = 1.0;
#pragma unroll
    for (int i = 1; i < D; ++i) {
      h1 = mul(h1, s[i]);
      h2 = mul(h2, KIND == 0 ? m1[i] : m0[i]);
    }
    double o0, o1;
    head_message<KIND>(p1, p2, h1, h2, o0, o1);
    put_message(P, P.ftov + tw[0], o0, o1, it, phase, 1, tw[0]);
  }
  if (D > 1) {
    double blend, hd;
    head_slot_terms<KIND>(p1, p2, m0[0], m1[0], blend, hd);
    double a1 = blend, a2 = hd;  // prefix over slots 0..j-1 (1.0 * x == x)
#pragma unroll
    for (int j = 1; j < D; ++j) {
      double b1 = a1, b2 = a2;
#pragma unroll
      for (int i = j + 1; i < D; ++i) {
        b1 = mul(b1, s[i]);
        b2 = mul(b2, KIND == 0 ? m1[i] : m0[i]);
      }
      double o0, o1;
      body_message<KIND>(p1, p2, b1, b2, o0, o1);
      put_message(P, P.ftov + tw[j], o0, o1, it, phase, 1, tw[j]);
      a1 = mul(a1, s[j]);
      a2 = mul(a2, KIND == 0 ? m1[j] : m0[j]);
    }
  }
}

// one factor target with runtime degree; slot x excluded (head iff x == 0)
template <int KIND>
__device__ __forceinline__ void ft_one(const KParams &P, int r, int d, int x, double p1, double p2,
                                       int out, int it, int phase) {
  double o0, o1;
  if (x == 0) {
    double h1 = 1.0, h2 = 1.0;
    for (int i = 1; i < d; ++i) {
      double2 m = P.vtof[r + i];
      h1 = mul(h1, add(m.x, m.y));
      h2 = mul(h2, KIND == 0 ? m.y : m.x);
    }
    head_message<KIND>(p1, p2, h1, h2, o0, o1);
  } else {
    double2 h = P.vtof[r];
    double b1, b2;
    head_slot_terms<KIND>(p1, p2, h.x, h.y, b1, b2);
    for (int i = 1; i < d; ++i) {
      if (i == x) continue;
      double2 m = P.vtof[r + i];
      b1 = mul(b1, add(m.x, m.y));
      b2 = mul(b2, KIND == 0 ? m.y : m.x);
    }
    body_message<KIND>(p1, p2, b1, b2, o0, o1);
  }
  put_message(P, P.ftov + out, o0, o1, it, phase, 1, out);
}

template <int KIND>
__device__ __noinline__ void fnode_generic(const KParams &P, int f, int r, int d, int it,
                                           int phase) {
  const double2 pp = P.fpar[f];
  for (int x = 0; x < d; ++x) ft_one<KIND>(P, r, d, x, pp.x, pp.y, P.vtof_twin[r + x], it, phase);
}

__device__ __forceinline__ void fnode(const KParams &P, int f, int it, int phase) {
  const int r = P.frow[f];
  const int d = P.frow[f + 1] - r;
  if (f < P.f_or_begin) {
    switch (d) {
      case 1: fnode_fixed<1, 0>(P, f, r, it, phase); break;
      case 2: fnode_fixed<2, 0>(P, f, r, it, phase); break;
      case 3: fnode_fixed<3, 0>(P, f, r, it, phase); break;
      case 4: fnode_fixed<4, 0>(P, f, r, it, phase); break;
      default: fnode_generic<0>(P, f, r, d, it, phase); break;
    }
  } else {
    switch (d) {
      case 2: fnode_fixed<2, 1>(P, f, r, it, phase); break;
      case 3: fnode_fixed<3, 1>(P, f, r, it, phase); break;
      case 4: fnode_fixed<4, 1>(P, f, r, it, phase); break;
      default: fnode_generic<1>(P, f, r, d, it, phase); break;
    }
  }
}

__device__ __forceinline__ void ft_target(const KParams &P, int4 t, int it, int phase) {
  const int d = t.z & 0xffff, x = (unsigned)t.z >> 16;
  const double2 pp = P.fpar[t.w];
  if (t.w < P.f_or_begin)
    ft_one<0>(P, t.y, d, x, pp.x, pp.y, t.x, it, phase);
  else
    ft_one<1>(P, t.y, d, x, pp.x, pp.y, t.x, it, phase);
}

// --------------------------------------------------------------------------------------
// one phase over [0, nodes + targets) with grid- or CTA-stride

__device__ __forceinline__ void exec_phase(const KParams &P, const Phase &ph, int pidx, int it,
                                           bool do_marg, bool do_vtof,
                                           unsigned long long &dmax) {
  int start, stride;
  if (ph.grid) {
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = gridDim.x * blockDim.x;
  } else {
    if (blockIdx.x != 0) return;
    start = threadIdx.x;
    stride = blockDim.x;
  }
  const int nn = ph.node_end - ph.node_begin;
  const int total = nn + (ph.tgt_end - ph.tgt_begin);
  if (ph.type == 0) {
    const bool marg = do_marg && (ph.node_flags & 1);
    for (int i = start; i < total; i += stride) {
      if (i < nn) {
        int v;
        bool vt;
        if (ph.node_list) {
          int item = P.vnode[ph.node_begin + i];
          v = item & (kVtofBit - 1);
          vt = (item & kVtofBit) != 0;
        } else {
          v = ph.node_begin + i;
          vt = (ph.node_flags & 2) != 0;
        }
        vt = vt && do_vtof;
        if (marg || vt) vnode(P, v, marg, vt, it, pidx, dmax);
      } else if (do_vtof) {
        vt_target(P, P.vt[ph.tgt_begin + i - nn], it, pidx);
      }
    }
  } else {
    for (int i = start; i < total; i += stride) {
      if (i < nn) {
        int f = ph.node_list ? P.fnode[ph.node_begin + i] : ph.node_begin + i;
        fnode(P, f, it, pidx);
      } else {
        ft_target(P, P.ft[ph.tgt_begin + i - nn], it, pidx);
      }
    }
  }
}

__device__ __forceinline__ unsigned long long block_max(unsigned long long v) {
  __shared__ unsigned long long red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
      v = w > v ? w : v;
    }
  }
  return v;  // valid in thread 0
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kThreads, 1) lbp_persistent(const __grid_constant__ KParams P) {
  Ctrl *C = P.ctrl;
  const bool multi = gridDim.x > 1;
  unsigned expected = 0;  // arrivals every CTA has seen so far (same on all CTAs)

  // uniform start: all messages (1, 1), prev P1 = 0.5 (storage.py:91-94, engine.py:557)
  {
    const int gs = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.E; i += gs) {
      P.vtof[i] = make_double2(1.0, 1.0);
      P.ftov[i] = make_double2(1.0, 1.0);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.V; i += gs) P.prev[i] = 0.5;
    if (blockIdx.x == 0 && threadIdx.x == 0) C->t0 = globaltimer();
    if (multi) {
      bar_arrive(C);
      expected += gridDim.x;
      bar_wait(C, expected);
    } else {
      __syncthreads();
    }
  }

  for (int it = 1;; ++it) {
    const bool final_pass = it == P.max_it + 1;
    unsigned long long dmax = 0;
    exec_phase(P, P.phases[0], 0, it, it > 1, !final_pass, dmax);
    if (it > 1) {
      unsigned long long m = block_max(dmax);
      if (threadIdx.x == 0) {
        atomicMax(&P.delta_bits[it - 1], m);
        if (blockIdx.x == 0 && P.time_limit_ns > 0)
          P.tflag[it - 1] = (long long)(globaltimer() - C->t0) > P.time_limit_ns;
      }
    }
    if (multi) {
      bar_arrive(C);
      expected += gridDim.x;
      bar_wait(C, expected);
    } else {
      __syncthreads();
    }
    if (it > 1) {
      const int done = it - 1;
      const volatile int *ufm = P.uf_msg, *ufg = P.uf_marg, *tf = P.tflag;
      const volatile unsigned long long *db = P.delta_bits;
      int stop = 0;
      if (ufm[done] || ufg[done]) stop = 4;
      else if (__longlong_as_double((long long)db[done]) < P.tol) stop = 1;
      else if (done == P.max_it) stop = 2;
      else if (tf[done]) stop = 3;
      if (stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          C->iterations = done;
          C->converged = stop == 1;
          C->stop = stop;
        }
        return;
      }
    }
    // remaining phases of this iteration
    for (int p = 1; p < P.nphases; ++p) {
      const Phase &ph = P.phases[p];
      const Phase &prv = P.phases[p - 1];
      if (p > 1) {  // transition prv -> ph (phase 0 -> 1 was the full barrier above)
        if (!multi) {
          __syncthreads();
        } else if (prv.grid && ph.grid) {
          bar_arrive(C);
          expected += gridDim.x;
          bar_wait(C, expected);
        } else if (prv.grid && !ph.grid) {
          bar_arrive(C);
          expected += gridDim.x;
          if (blockIdx.x == 0) bar_wait(C, expected);
        } else if (!prv.grid && !ph.grid) {
          if (blockIdx.x == 0) __syncthreads();
        } else {  // CTA 0 -> grid
          if (blockIdx.x == 0) bar_arrive(C);
          expected += 1;
          bar_wait(C, expected);
        }
      }
      unsigned long long unused = 0;
      exec_phase(P, ph, p, it, false, true, unused);
    }
    // transition last phase -> phase 0 of the next iteration (a grid phase)
    if (P.nphases > 1) {
      const Phase &last = P.phases[P.nphases - 1];
      if (!multi) {
        __syncthreads();
      } else if (last.grid) {
        bar_arrive(C);
        expected += gridDim.x;
        bar_wait(C, expected);
      } else {
        if (blockIdx.x == 0) bar_arrive(C);
        expected += 1;
        bar_wait(C, expected);
      }
    }
  }
}

}  // namespace hbp

// ======================================================================================
// single-pass kernels for the host-store diagnostic API (hbp_pass / hbp_marginals)

namespace hbp {

__global__ void __launch_bounds__(256) pass_kernel(const __grid_constant__ KParams P, int type, const int4 *items, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (type == 0)
    vt_target(P, items[i], 1, 0);
  else
    ft_target(P, items[i], 1, 0);
}

__global__ void __launch_bounds__(256) marginal_kernel(const __grid_constant__ KParams P) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= P.V) return;
  unsigned long long unused = 0;
  vnode(P, v, true, false, 2, 0, unused);
}

}  // namespace hbp

// ======================================================================================
// host side: handles + C ABI

namespace {

thread_local int64_t g_last_launches = 0;

#define HBP_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t _e = (call);                                                    \
    if (_e != cudaSuccess) {                                                    \
      hbp::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));       \
      return HBP_ECUDA;                                                         \
    }                                                                           \
  } while (0)

template <typename T>
hbp_status upload(T **dst, const std::vector<T> &src, cudaStream_t s) {
  HBP_CUDA(cudaMalloc((void **)dst, std::max<size_t>(1, src.size()) * sizeof(T)));
  if (!src.empty())
    HBP_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return HBP_OK;
}

}  // namespace

struct hbp_graph {
  hbp::HostLayout L;
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0, coop_blocks = 0;
  int *d_frow = nullptr, *d_vtof_twin = nullptr, *d_vrow = nullptr, *d_ftov_twin = nullptr,
      *d_vorig = nullptr;
  double2 *d_fpar = nullptr, *d_vtof = nullptr, *d_ftov = nullptr, *d_marg = nullptr;
  double *d_prev = nullptr;
  // control block sized for max_iterations
  void *d_ctrl = nullptr;
  size_t ctrl_cap = 0;  // entries per array
  double2 *d_hist = nullptr;
  size_t hist_cap = 0;  // double2 entries
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  ~hbp_graph() {
    cudaSetDevice(device);
    for (void *p : {(void *)d_frow, (void *)d_vtof_twin, (void *)d_vrow, (void *)d_ftov_twin,
                    (void *)d_vorig, (void *)d_fpar, (void *)d_vtof, (void *)d_ftov,
                    (void *)d_marg, (void *)d_prev, d_ctrl, (void *)d_hist})
      if (p) cudaFree(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
};

struct hbp_plan {
  hbp_graph *g = nullptr;
  hbp::PlanHost host;
  hbp::Phase *d_phases = nullptr;
  int *d_vnode = nullptr, *d_fnode = nullptr;
  int4 *d_vt = nullptr, *d_ft = nullptr;
  int grid = 1;
  ~hbp_plan() {
    cudaSetDevice(g->device);
    for (void *p : {(void *)d_phases, (void *)d_vnode, (void *)d_fnode, (void *)d_vt, (void *)d_ft})
      if (p) cudaFree(p);
  }
};

namespace {

struct CtrlView {
  hbp::Ctrl *ctrl;
  unsigned long long *delta_bits, *uf_where;
  int *uf_msg, *uf_marg, *uf_mwhere, *tflag;
};

CtrlView ctrl_view(void *base, size_t n) {
  CtrlView c;
  char *p = (char *)base;
  c.ctrl = (hbp::Ctrl *)p;
  p += 256;
  c.delta_bits = (unsigned long long *)p;
  p += n * 8;
  c.uf_where = (unsigned long long *)p;
  p += n * 8;
  c.uf_msg = (int *)p;
  p += n * 4;
  c.uf_marg = (int *)p;
  p += n * 4;
  c.uf_mwhere = (int *)p;
  p += n * 4;
  c.tflag = (int *)p;
  return c;
}

size_t ctrl_bytes(size_t n) { return 256 + n * (8 + 8 + 4 + 4 + 4 + 4); }

hbp::KParams base_params(hbp_graph *g) {
  hbp::KParams P{};
  P.frow = g->d_frow;
  P.fpar = g->d_fpar;
  P.vtof_twin = g->d_vtof_twin;
  P.vrow = g->d_vrow;
  P.ftov_twin = g->d_ftov_twin;
  P.vorig = g->d_vorig;
  P.V = g->L.V;
  P.F = g->L.F;
  P.E = (int)g->L.E;
  P.f_or_begin = g->L.f_or_begin;
  P.vtof = g->d_vtof;
  P.ftov = g->d_ftov;
  P.marg = g->d_marg;
  P.prev = g->d_prev;
  P.normalize = 1;
  return P;
}

hbp_status ensure_ctrl(hbp_graph *g, size_t n) {
  if (g->ctrl_cap >= n) return HBP_OK;
  if (g->d_ctrl) cudaFree(g->d_ctrl);
  g->d_ctrl = nullptr;
  g->ctrl_cap = 0;
  HBP_CUDA(cudaMalloc(&g->d_ctrl, ctrl_bytes(n)));
  g->ctrl_cap = n;
  return HBP_OK;
}

hbp_status reset_ctrl(hbp_graph *g, size_t n) {
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  cudaStream_t s = g->stream;
  HBP_CUDA(cudaMemsetAsync(c.ctrl, 0, 256, s));
  HBP_CUDA(cudaMemsetAsync(c.delta_bits, 0, n * 8, s));
  HBP_CUDA(cudaMemsetAsync(c.uf_where, 0xFF, n * 8, s));
  HBP_CUDA(cudaMemsetAsync(c.uf_msg, 0, n * 4, s));
  HBP_CUDA(cudaMemsetAsync(c.uf_marg, 0, n * 4, s));
  HBP_CUDA(cudaMemsetAsync(c.uf_mwhere, 0x7F, n * 4, s));
  HBP_CUDA(cudaMemsetAsync(c.tflag, 0, n * 4, s));
  return HBP_OK;
}

}  // namespace

extern "C" {

hbp_status hbp_graph_create(const hbp_graph_desc *desc, int32_t device, hbp_graph **out) {
  if (!desc || !out) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  *out = nullptr;
  std::unique_ptr<hbp_graph> g(new (std::nothrow) hbp_graph());
  if (!g) return HBP_ENOMEM;
  hbp_status st = hbp::build_layout(*desc, g->L);
  if (st != HBP_OK) return st;
  g->device = device;
  HBP_CUDA(cudaSetDevice(device));
  HBP_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  HBP_CUDA(cudaEventCreate(&g->ev0));
  HBP_CUDA(cudaEventCreate(&g->ev1));
  HBP_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
  int per_sm = 0;
  HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hbp::lbp_persistent,
                                                         hbp::kThreads, 0));
  g->coop_blocks = std::max(1, per_sm) * g->num_sms;
  const hbp::HostLayout &L = g->L;
  cudaStream_t s = g->stream;
  std::vector<double2> fpar((size_t)L.F);
  for (int32_t i = 0; i < L.F; ++i) fpar[i] = make_double2(L.p1[L.fperm[i]], L.p2[L.fperm[i]]);
  if ((st = upload(&g->d_frow, L.frow, s)) || (st = upload(&g->d_vtof_twin, L.vtof_twin, s)) ||
      (st = upload(&g->d_vrow, L.vrow, s)) || (st = upload(&g->d_ftov_twin, L.ftov_twin, s)) ||
      (st = upload(&g->d_vorig, L.vperm, s)) || (st = upload(&g->d_fpar, fpar, s)))
    return st;
  HBP_CUDA(cudaMalloc(&g->d_vtof, (size_t)L.E * sizeof(double2)));
  HBP_CUDA(cudaMalloc(&g->d_ftov, (size_t)L.E * sizeof(double2)));
  HBP_CUDA(cudaMalloc(&g->d_marg, (size_t)std::max(1, L.V) * sizeof(double2)));
  HBP_CUDA(cudaMalloc(&g->d_prev, (size_t)std::max(1, L.V) * sizeof(double)));
  HBP_CUDA(cudaStreamSynchronize(s));
  *out = g.release();
  return HBP_OK;
}

void hbp_graph_destroy(hbp_graph *g) { delete g; }

hbp_status hbp_graph_layout(hbp_graph *g, int64_t *rowptr_ftov, int64_t *ftov_to_vtof) {
  // reference layout (storage.py:55-63) recomputed from the device-side maps
  const hbp::HostLayout &L = g->L;
  std::vector<int64_t> cnt((size_t)L.V + 1, 0);
  for (int64_t e = 0; e < L.E; ++e) cnt[(size_t)L.edge_var[e] + 1]++;
  for (int32_t v = 0; v < L.V; ++v) cnt[v + 1] += cnt[v];
  for (int32_t v = 0; v <= L.V; ++v) rowptr_ftov[v] = cnt[v];
  // device row of variable v, in device order, mapped back to canonical
  for (int32_t v = 0; v < L.V; ++v) {
    int32_t vi = L.vinv[v];
    for (int32_t k = L.vrow[vi]; k < L.vrow[vi + 1]; ++k)
      ftov_to_vtof[cnt[v] + (k - L.vrow[vi])] = L.ftov2canon[k];
  }
  return HBP_OK;
}

hbp_status hbp_plan_create(hbp_graph *g, int64_t k, const int64_t *s_off, const int32_t *s_edges,
                           const int64_t *t_off, const int32_t *t_edges, hbp_plan **out) {
  if (!g || !out) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  *out = nullptr;
  std::unique_ptr<hbp_plan> p(new (std::nothrow) hbp_plan());
  if (!p) return HBP_ENOMEM;
  p->g = g;
  hbp_status st = hbp::build_plan(g->L, k, s_off, s_edges, t_off, t_edges, p->host);
  if (st != HBP_OK) return st;
  HBP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  std::vector<int4> vt(p->host.vt.size() / 4), ft(p->host.ft.size() / 4);
  if (!vt.empty()) std::memcpy(vt.data(), p->host.vt.data(), vt.size() * 16);
  if (!ft.empty()) std::memcpy(ft.data(), p->host.ft.data(), ft.size() * 16);
  if ((st = upload(&p->d_phases, p->host.phases, s)) || (st = upload(&p->d_vnode, p->host.vnode, s)) ||
      (st = upload(&p->d_fnode, p->host.fnode, s)) || (st = upload(&p->d_vt, vt, s)) ||
      (st = upload(&p->d_ft, ft, s)))
    return st;
  // grid: enough CTAs for the largest grid-wide phase, at most one wave
  int64_t big = 0;
  for (const auto &ph : p->host.phases)
    if (ph.grid) big = std::max<int64_t>(big, (ph.node_end - ph.node_begin) + (ph.tgt_end - ph.tgt_begin));
  int64_t want = (big + hbp::kThreads - 1) / hbp::kThreads;
  if (big < 2 * hbp::kThreads) want = 1;
  p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, g->coop_blocks));
  HBP_CUDA(cudaStreamSynchronize(s));
  *out = p.release();
  return HBP_OK;
}

void hbp_plan_destroy(hbp_plan *p) { delete p; }

static hbp_status launch_run(hbp_plan *p, const hbp_options *opt, hbp_result *res) {
  hbp_graph *g = p->g;
  if (!opt || !res) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  if (opt->max_iterations < 1) {
    hbp::set_error("max_iterations must be at least 1");
    return HBP_EINVAL;
  }
  if (!(opt->tolerance >= 0)) {
    hbp::set_error("tolerance must be nonnegative");
    return HBP_EINVAL;
  }
  HBP_CUDA(cudaSetDevice(g->device));
  const size_t n = (size_t)opt->max_iterations + 2;
  hbp_status st = ensure_ctrl(g, n);
  if (st) return st;
  if ((st = reset_ctrl(g, n))) return st;
  double2 *hist = nullptr;
  if (opt->record_history) {
    size_t need = (size_t)opt->max_iterations * (size_t)std::max(1, g->L.V);
    if (need * sizeof(double2) > ((size_t)16 << 30)) {
      hbp::set_error("record_history buffer would exceed 16 GiB");
      return HBP_EINVAL;
    }
    if (g->hist_cap < need) {
      if (g->d_hist) cudaFree(g->d_hist);
      g->d_hist = nullptr;
      g->hist_cap = 0;
      HBP_CUDA(cudaMalloc(&g->d_hist, need * sizeof(double2)));
      g->hist_cap = need;
    }
    hist = g->d_hist;
  }
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  hbp::KParams P = base_params(g);
  P.phases = p->d_phases;
  P.nphases = (int)p->host.phases.size();
  P.vnode = p->d_vnode;
  P.fnode = p->d_fnode;
  P.vt = p->d_vt;
  P.ft = p->d_ft;
  P.ctrl = c.ctrl;
  P.delta_bits = c.delta_bits;
  P.uf_msg = c.uf_msg;
  P.uf_marg = c.uf_marg;
  P.uf_mwhere = c.uf_mwhere;
  P.uf_where = c.uf_where;
  P.tflag = c.tflag;
  P.hist = hist;
  P.max_it = opt->max_iterations;
  P.normalize = opt->normalize_messages ? 1 : 0;
  P.tol = opt->tolerance;
  P.time_limit_ns = opt->time_limit > 0 ? (long long)(opt->time_limit * 1e9) : 0;
  if (opt->time_limit > 0 && P.time_limit_ns == 0) P.time_limit_ns = 1;
  void *args[] = {&P};
  HBP_CUDA(cudaEventRecord(g->ev0, g->stream));
  HBP_CUDA(cudaLaunchCooperativeKernel((void *)hbp::lbp_persistent, dim3(p->grid),
                                       dim3(hbp::kThreads), args, 0, g->stream));
  HBP_CUDA(cudaEventRecord(g->ev1, g->stream));
  g_last_launches = 1;
  hbp::Ctrl hc;
  HBP_CUDA(cudaMemcpyAsync(&hc, c.ctrl, sizeof(hc), cudaMemcpyDeviceToHost, g->stream));
  HBP_CUDA(cudaStreamSynchronize(g->stream));
  float ms = 0;
  HBP_CUDA(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  std::memset(res, 0, sizeof(*res));
  res->iterations = hc.iterations;
  res->converged = hc.converged;
  res->device_ms = ms;
  unsigned long long last = 0;
  if (hc.iterations > 0)
    HBP_CUDA(cudaMemcpy(&last, c.delta_bits + hc.iterations, 8, cudaMemcpyDeviceToHost));
  std::memcpy(&res->last_delta, &last, 8);
  if (hc.stop == 4) {
    int um = 0, ug = 0, mw = 0;
    unsigned long long where = 0;
    const int it = hc.iterations;
    HBP_CUDA(cudaMemcpy(&um, c.uf_msg + it, 4, cudaMemcpyDeviceToHost));
    HBP_CUDA(cudaMemcpy(&ug, c.uf_marg + it, 4, cudaMemcpyDeviceToHost));
    HBP_CUDA(cudaMemcpy(&mw, c.uf_mwhere + it, 4, cudaMemcpyDeviceToHost));
    HBP_CUDA(cudaMemcpy(&where, c.uf_where + it, 8, cudaMemcpyDeviceToHost));
    res->underflow_iteration = it;
    if (um) {
      const int kind = (int)((where >> 32) & 1);
      const int32_t pos = (int32_t)(where & 0xFFFFFFFFu);
      res->underflow_kind = kind == 0 ? 1 : 2;
      res->underflow_index = kind == 0 ? g->L.vtof2canon[pos] : g->L.ftov2canon[pos];
    } else {
      res->underflow_kind = 3;
      res->underflow_index = mw;
    }
    (void)ug;
    hbp::set_error("underflow");
    return HBP_EUNDERFLOW;
  }
  return HBP_OK;
}

hbp_status hbp_run(hbp_plan *p, const hbp_options *opt, double *marginals_out, double *deltas_out,
                   double *history_out, hbp_result *res) {
  auto t0 = std::chrono::steady_clock::now();
  if (!p) {
    hbp::set_error("null plan");
    return HBP_EINVAL;
  }
  hbp_status st = launch_run(p, opt, res);
  if (st != HBP_OK) return st;
  hbp_graph *g = p->g;
  const int it = res->iterations;
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  if (marginals_out)
    HBP_CUDA(cudaMemcpyAsync(marginals_out, g->d_marg, (size_t)g->L.V * 16, cudaMemcpyDeviceToHost,
                             g->stream));
  if (deltas_out && it > 0)
    HBP_CUDA(cudaMemcpyAsync(deltas_out, c.delta_bits + 1, (size_t)it * 8, cudaMemcpyDeviceToHost,
                             g->stream));
  if (history_out && opt->record_history && it > 0)
    HBP_CUDA(cudaMemcpyAsync(history_out, g->d_hist, (size_t)it * g->L.V * 16,
                             cudaMemcpyDeviceToHost, g->stream));
  HBP_CUDA(cudaStreamSynchronize(g->stream));
  res->total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return HBP_OK;
}

hbp_status hbp_run_device(hbp_plan *p, const hbp_options *opt, hbp_result *res,
                          const double **marginals_dev) {
  if (!p) {
    hbp::set_error("null plan");
    return HBP_EINVAL;
  }
  hbp_status st = launch_run(p, opt, res);
  if (marginals_dev) *marginals_dev = (const double *)p->g->d_marg;
  return st;
}

hbp_status hbp_pass(hbp_graph *g, int32_t direction, int64_t n, const int32_t *targets,
                    int32_t normalize, double *vtof0, double *vtof1, double *ftov0, double *ftov1,
                    int64_t *underflow_index) {
  if (!g || (n > 0 && !targets) || !vtof0 || !vtof1 || !ftov0 || !ftov1) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  const hbp::HostLayout &L = g->L;
  if (underflow_index) *underflow_index = -1;
  if (n == 0) return HBP_OK;
  for (int64_t i = 0; i < n; ++i)
    if (targets[i] < 0 || targets[i] >= L.E) {
      hbp::set_error("target edge out of range");
      return HBP_EINVAL;
    }
  HBP_CUDA(cudaSetDevice(g->device));
  // host store (reference layout) -> device layout
  std::vector<double2> hv((size_t)L.E), hf((size_t)L.E);
  for (int64_t e = 0; e < L.E; ++e) hv[L.canon2v[e]] = make_double2(vtof0[e], vtof1[e]);
  for (int64_t q = 0; q < L.E; ++q) {
    int32_t e = L.ref_ftov[q];
    hf[L.canon2f[e]] = make_double2(ftov0[q], ftov1[q]);
  }
  std::vector<int4> items((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    if (direction == 0)
      hbp::make_vt_item(L, targets[i], (int32_t *)&items[i]);
    else
      hbp::make_ft_item(L, targets[i], (int32_t *)&items[i]);
  }
  hbp_status st = ensure_ctrl(g, 4);
  if (st) return st;
  if ((st = reset_ctrl(g, 4))) return st;
  int4 *d_items = nullptr;
  HBP_CUDA(cudaMalloc(&d_items, items.size() * 16));
  cudaStream_t s = g->stream;
  HBP_CUDA(cudaMemcpyAsync(g->d_vtof, hv.data(), hv.size() * 16, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(g->d_ftov, hf.data(), hf.size() * 16, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(d_items, items.data(), items.size() * 16, cudaMemcpyHostToDevice, s));
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  hbp::KParams P = base_params(g);
  P.normalize = normalize ? 1 : 0;
  P.uf_msg = c.uf_msg;
  P.uf_where = c.uf_where;
  P.uf_marg = c.uf_marg;
  P.uf_mwhere = c.uf_mwhere;
  hbp::pass_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, direction ? 1 : 0, d_items, (int)n);
  g_last_launches = 1;
  cudaError_t le = cudaGetLastError();
  int uf = 0;
  unsigned long long where = 0;
  cudaMemcpyAsync(&uf, c.uf_msg + 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&where, c.uf_where + 1, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hv.data(), g->d_vtof, hv.size() * 16, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hf.data(), g->d_ftov, hf.size() * 16, cudaMemcpyDeviceToHost, s);
  cudaError_t se = cudaStreamSynchronize(s);
  cudaFree(d_items);
  if (le != cudaSuccess || se != cudaSuccess) {
    hbp::set_error(std::string("pass kernel: ") + cudaGetErrorString(le != cudaSuccess ? le : se));
    return HBP_ECUDA;
  }
  if (uf) {
    const int32_t pos = (int32_t)(where & 0xFFFFFFFFu);
    if (underflow_index) *underflow_index = direction == 0 ? L.vtof2canon[pos] : L.ftov2canon[pos];
    hbp::set_error("underflow");
    return HBP_EUNDERFLOW;  // store left untouched, like the reference's raise-before-scatter
  }
  if (direction == 0) {
    for (int64_t i = 0; i < n; ++i) {
      int32_t e = targets[i];
      double2 m = hv[L.canon2v[e]];
      vtof0[e] = m.x;
      vtof1[e] = m.y;
    }
  } else {
    std::vector<int32_t> ref_pos((size_t)L.E);
    for (int64_t q = 0; q < L.E; ++q) ref_pos[L.ref_ftov[q]] = (int32_t)q;
    for (int64_t i = 0; i < n; ++i) {
      int32_t e = targets[i];
      double2 m = hf[L.canon2f[e]];
      ftov0[ref_pos[e]] = m.x;
      ftov1[ref_pos[e]] = m.y;
    }
  }
  return HBP_OK;
}

hbp_status hbp_marginals(hbp_graph *g, const double *ftov0, const double *ftov1, double *out,
                         int64_t *underflow_var) {
  if (!g || !ftov0 || !ftov1 || !out) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  const hbp::HostLayout &L = g->L;
  if (underflow_var) *underflow_var = -1;
  HBP_CUDA(cudaSetDevice(g->device));
  std::vector<double2> hf((size_t)L.E);
  for (int64_t q = 0; q < L.E; ++q) hf[L.canon2f[L.ref_ftov[q]]] = make_double2(ftov0[q], ftov1[q]);
  hbp_status st = ensure_ctrl(g, 4);
  if (st) return st;
  if ((st = reset_ctrl(g, 4))) return st;
  cudaStream_t s = g->stream;
  HBP_CUDA(cudaMemcpyAsync(g->d_ftov, hf.data(), hf.size() * 16, cudaMemcpyHostToDevice, s));
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  hbp::KParams P = base_params(g);
  P.uf_msg = c.uf_msg;
  P.uf_where = c.uf_where;
  P.uf_marg = c.uf_marg;
  P.uf_mwhere = c.uf_mwhere;
  hbp::marginal_kernel<<<(unsigned)((L.V + 255) / 256), 256, 0, s>>>(P);
  g_last_launches = 1;
  HBP_CUDA(cudaGetLastError());
  int uf = 0, mw = 0;
  HBP_CUDA(cudaMemcpyAsync(&uf, c.uf_marg + 1, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(&mw, c.uf_mwhere + 1, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(out, g->d_marg, (size_t)L.V * 16, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  if (uf) {
    if (underflow_var) *underflow_var = mw;
    hbp::set_error("underflow");
    return HBP_EUNDERFLOW;
  }
  return HBP_OK;
}

int64_t hbp_last_launch_count(void) { return g_last_launches; }

}  // extern "C"
