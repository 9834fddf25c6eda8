// Device-side layout build: the MessageStore transpose
// (storage.py:36-94) and this engine's degree-sorted internal order, computed
// by kernels on the graph's stream from the canonical arrays (graph.py
// FactorGraph: rowptr, vars, kind, p1, p2). The product is exactly the device
// half of layout.cpp's HostLayout -- the same stable orders (CUB radix sorts
// are stable, as is layout.cpp's counting sort), the same rows, the same slot
// records -- so the executors cannot tell which builder ran;
// hbp_graph_layout_check compares the two array by array.
//
// Cost at ftp (476,915 edges): one 7.2 MB upload, ~15 small kernels, 3 radix
// sorts and 3 scans, two synchronisations (validation, then the class
// tables). The host HostLayout is built later, only when a host-side consumer
// asks for it (levelled plans, the sweep's chunking, the single-pass API).
#include <cub/cub.cuh>

#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "device.h"

namespace hbp {
namespace {

constexpr int kB = 256;

inline unsigned blocks_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kB - 1) / kB, 148 * 32));
}

// validation + reductions, filled by the first kernels, read back once
struct DevInfo {
  int err_factor;  // smallest factor with a bad degree or kind (INT_MAX: none)
  int err_edge;    // smallest edge whose variable is out of range
  int err_var;     // smallest variable in no factor
  int max_fdeg, max_vdeg;
  int fclass[4];   // factors per (heavy, kind) class
  int n_unary;     // factors of degree 1
  int v_light;     // variables of degree <= kNodeMax
  int vhist[kNodeMax + 2];   // light variables per degree
  int fhist[2][kNodeMax + 2];  // light AND / OR factors per degree
  // every class (layout.cpp class_tables): per degree up to kClassMax, the
  // huge nodes' count at kClassMax + 1 and their slots
  int vcls[kClassMax + 2], vhuge;
  int fcls[2][kClassMax + 2], fhuge[2];
};

__global__ void k_iota(int *a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

// per factor: degree/kind checks, sort key (heavy, kind, degree) -- layout.cpp fkey
__global__ void k_factors(const int64_t *rp, const int8_t *kind, int F, DevInfo *info,
                          unsigned *fkey) {
  __shared__ int s_cls[4], s_unary, s_max, s_hist[2][kNodeMax + 2], s_all[2][kClassMax + 2], s_huge[2];
  if (threadIdx.x < 4) s_cls[threadIdx.x] = 0;
  if (threadIdx.x < 2 * (kNodeMax + 2)) (&s_hist[0][0])[threadIdx.x] = 0;
  if (threadIdx.x < 2 * (kClassMax + 2)) (&s_all[0][0])[threadIdx.x] = 0;
  if (threadIdx.x < 2) s_huge[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_unary = 0, s_max = 0;
  __syncthreads();
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    const int64_t d = rp[f + 1] - rp[f];
    const int k = kind[f];
    if (d < 1 || d > 65535 || (k != HBP_AND && k != HBP_OR)) {
      atomicMin(&info->err_factor, f);
      fkey[f] = 0;
      continue;
    }
    const int heavy = d > kNodeMax;
    fkey[f] = (unsigned)((heavy * 2 + k) << 16) | (unsigned)d;
    atomicAdd(&s_cls[heavy * 2 + k], 1);
    if (!heavy) atomicAdd(&s_hist[k][d], 1);
    if (d > kClassMax) {
      atomicAdd(&s_all[k][kClassMax + 1], 1);
      atomicAdd(&s_huge[k], (int)d);
    } else {
      atomicAdd(&s_all[k][d], 1);
    }
    if (d == 1) atomicAdd(&s_unary, 1);
    atomicMax(&s_max, (int)d);
  }
  __syncthreads();
  if (threadIdx.x < 4) atomicAdd(&info->fclass[threadIdx.x], s_cls[threadIdx.x]);
  if (threadIdx.x < 2 * (kNodeMax + 2))
    atomicAdd(&(&info->fhist[0][0])[threadIdx.x], (&s_hist[0][0])[threadIdx.x]);
  if (threadIdx.x < 2 * (kClassMax + 2))
    atomicAdd(&(&info->fcls[0][0])[threadIdx.x], (&s_all[0][0])[threadIdx.x]);
  if (threadIdx.x < 2) atomicAdd(&info->fhuge[threadIdx.x], s_huge[threadIdx.x]);
  if (threadIdx.x == 0) {
    atomicAdd(&info->n_unary, s_unary);
    atomicMax(&info->max_fdeg, s_max);
  }
}

// per edge: variable range check and variable degrees
__global__ void k_edges(const int *evar, int64_t E, int V, DevInfo *info, int *vdeg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int v = evar[e];
    if (v < 0 || v >= V)
      atomicMin(&info->err_edge, (int)e);
    else
      atomicAdd(&vdeg[v], 1);
  }
}

// per variable: no-factor check, degree maximum and light histogram
__global__ void k_vars(const int *vdeg, int V, DevInfo *info) {
  __shared__ int s_max, s_light, s_hist[kNodeMax + 2], s_all[kClassMax + 2], s_huge;
  if (threadIdx.x < kNodeMax + 2) s_hist[threadIdx.x] = 0;
  if (threadIdx.x < kClassMax + 2) s_all[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_max = 0, s_light = 0, s_huge = 0;
  __syncthreads();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const int d = vdeg[v];
    if (d == 0) atomicMin(&info->err_var, v);
    atomicMax(&s_max, d);
    if (d <= kNodeMax) {
      atomicAdd(&s_light, 1);
      atomicAdd(&s_hist[d], 1);
    }
    if (d > kClassMax) {
      atomicAdd(&s_all[kClassMax + 1], 1);
      atomicAdd(&s_huge, d);
    } else {
      atomicAdd(&s_all[d], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < kNodeMax + 2) atomicAdd(&info->vhist[threadIdx.x], s_hist[threadIdx.x]);
  if (threadIdx.x < kClassMax + 2) atomicAdd(&info->vcls[threadIdx.x], s_all[threadIdx.x]);
  if (threadIdx.x == 0) atomicAdd(&info->vhuge, s_huge);
  if (threadIdx.x == 0) {
    atomicMax(&info->max_vdeg, s_max);
    atomicAdd(&info->v_light, s_light);
  }
}

// degree of sorted entry i from its key (low 16 bits), with a 0 appended so an
// exclusive scan over n + 1 entries ends in the total (frow / vrow)
__global__ void k_low16(const unsigned *key, int n, int *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    out[i] = i < n ? (int)(key[i] & 0xffffu) : 0;
}

__global__ void k_copy_ext(const int *in, int n, int *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    out[i] = i < n ? in[i] : 0;
}

// vtof rows in internal factor order (layout.cpp:85-103)
__global__ void k_frows(const int64_t *rp, const int *fperm, const int *frow, const double *p1,
                        const double *p2, int F, int *canon2v, int2 *fslot, double2 *fpar) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
    const int f = fperm[i];
    const int64_t e0 = rp[f];
    const int d = (int)(rp[f + 1] - e0);
    const int p0 = frow[i];
    for (int j = 0; j < d; ++j) {
      canon2v[e0 + j] = p0 + j;
      fslot[p0 + j] = make_int2(i, (d << 16) | j);
    }
    fpar[i] = make_double2(p1[f], p2[f]);
  }
}

__global__ void k_vinv(const int *vperm, int V, int *vinv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    vinv[vperm[i]] = i;
}

// ftov rows: the reference's (factor, slot) order within each variable, placed
// at the variable's internal row (layout.cpp:165-190)
__global__ void k_vrows(const int *ref_ftov, const int *evar_sorted, const int *vstart,
                        const int *vinv, const int *vrow, const int *vdeg, int64_t E,
                        int *canon2f, int2 *vslot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = ref_ftov[i];
    const int v = evar_sorted[i];
    const int j = (int)(i - vstart[v]);
    const int vi = vinv[v];
    const int q = vrow[vi] + j;
    canon2f[e] = q;
    vslot[q] = make_int2(vi, (vdeg[v] << 16) | j);
  }
}

// twins (layout.cpp:195-202); a unary factor's slot has degree 1 in its record
__global__ void k_twins(const int *canon2v, const int *canon2f, const int2 *fslot, int64_t E,
                        int *vtof_twin, unsigned *ftov_twin) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = canon2v[e], q = canon2f[e];
    vtof_twin[p] = q;
    const bool unary = (fslot[p].y >> 16) == 1;
    ftov_twin[q] = (unsigned)p | (unary ? kUnaryBit : 0u);
  }
}

__global__ void k_gather(const int *a, const int *idx, int n, int *out) {
  if (threadIdx.x < n) out[threadIdx.x] = a[idx[threadIdx.x]];
}

// PARALL shape check of a one-batch schedule: s holds every edge once, t every
// slot of a non-unary factor once (layout.cpp build_plan's fast path)
__global__ void k_parall_check(const int *s, int64_t ns, const int *t, int64_t nt, int64_t E,
                               const int *canon2v, const int2 *fslot, unsigned *bits,
                               int *bad) {
  const int64_t words = (E + 31) / 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns + nt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool is_t = i >= ns;
    const int e = is_t ? t[i - ns] : s[i];
    if (e < 0 || e >= E) {
      atomicOr(bad, 2);  // out of range: the host builder reports it
      continue;
    }
    const unsigned bit = 1u << (e & 31);
    const unsigned old = atomicOr(&bits[(is_t ? words : 0) + (e >> 5)], bit);
    if (old & bit) atomicOr(bad, 1);
    if (is_t && (fslot[canon2v[e]].y >> 16) == 1) atomicOr(bad, 1);
  }
}

// scratch arena: one allocation, carved in 256-byte aligned pieces
struct Arena {
  char *base = nullptr;
  size_t off = 0, cap = 0;
  template <class T>
  T *take(size_t n) {
    T *p = base ? (T *)(base + off) : nullptr;
    off += (n * sizeof(T) + 255) / 256 * 256;
    return p;
  }
};

// HBP_LAYOUT_TIMING=1: synchronise and print the time of each stage (probe)
struct StageClock {
  bool on = getenv("HBP_LAYOUT_TIMING") != nullptr;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char *what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "  layout %-10s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

int bits_for(int64_t n) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < n) ++b;
  return b;
}

}  // namespace

hbp_status build_layout_device(const hbp_graph_desc &desc, hbp_graph *g) {
  HostLayout &L = g->L;
  if (desc.num_variables < 0 || desc.num_factors < 0 || desc.num_edges < 0) {
    set_error("negative graph dimension");
    return HBP_EINVAL;
  }
  if (desc.num_edges == 0) {
    set_error("graph has no edges");
    return HBP_EINVAL;
  }
  if (desc.num_edges >= ((int64_t)1 << 30)) {
    set_error("graph has too many edges for the int32 device layout");
    return HBP_EINVAL;
  }
  const int V = desc.num_variables, F = desc.num_factors;
  const int64_t E = desc.num_edges;
  if (desc.factor_rowptr[0] != 0 || desc.factor_rowptr[F] != E) {
    set_error("factor_rowptr does not span the edge array");
    return HBP_EINVAL;
  }
  cudaStream_t s = g->stream;
  StageClock clk;
  clk.s = s;

  // CUB temporary storage: the largest of the sorts and scans below
  size_t tmp = 0, t1 = 0;
  const int maxn = (int)std::max<int64_t>(E, std::max(V, F) + 1);
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (unsigned *)nullptr, (unsigned *)nullptr,
                                  (int *)nullptr, (int *)nullptr, maxn, 0, 32, s);
  tmp = std::max(tmp, t1);
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (int *)nullptr, (int *)nullptr, maxn + 1, s);
  tmp = std::max(tmp, t1);

  // one device allocation (cudaMalloc/cudaFree cost ~0.2-0.3 ms each): the
  // canonical arrays (kept: the lazy host layout downloads them), the layout,
  // the single-graph message buffers, then the scratch
  const size_t nV = (size_t)std::max(1, V), nF = (size_t)std::max(1, F), nE = (size_t)E;
  Arena P;
  P.base = nullptr;
  auto plan_block = [&](Arena &a) {
    g->d_rowptr = a.take<int64_t>(F + 1);
    g->d_evar = a.take<int>(nE);
    g->d_kind = a.take<int8_t>(nF);
    g->d_p1 = a.take<double>(nF);
    g->d_p2 = a.take<double>(nF);
    g->d_vrow = a.take<int>(V + 1);
    g->d_frow = a.take<int>(F + 1);
    g->d_vslot = a.take<int2>(nE);
    g->d_fslot = a.take<int2>(nE);
    g->d_vtof_twin = a.take<int>(nE);
    g->d_ftov_twin = a.take<unsigned>(nE);
    g->d_vorig = a.take<int>(nV);
    g->d_vinv = a.take<int>(nV);
    g->d_fpar = a.take<double2>(nF);
    g->d_canon2v = a.take<int>(nE);
    g->d_vtof = a.take<double2>(nE);
    g->d_ftov = a.take<double2>(nE);
    g->d_marg = a.take<double2>(nV);
    g->d_prev = a.take<double>(nV);
  };
  plan_block(P);  // sizes only (base == nullptr)
  const size_t persistent = P.off;
  const size_t scratch = 256 * 20 + tmp + sizeof(DevInfo) +
                         4 * (5 * (size_t)(F + 2) + 5 * (size_t)(V + 2) + 3 * nE + (size_t)maxn + 256);
  // the PARALL shape test needs 2E ints + 2 bitmaps
  const size_t scratch_all = std::max(scratch, 4 * (2 * nE + 2 * ((nE + 31) / 32) + 64) + 512);
  // from the device's stream-ordered pool, which keeps freed blocks (release
  // threshold raised once per device): a fresh graph of a size seen before
  // costs no cudaMalloc, and destroying one no cudaFree
  static bool pool_ready[64] = {};
  if (g->device >= 0 && g->device < 64 && !pool_ready[g->device]) {
    cudaMemPool_t pool;
    HBP_CUDA(cudaDeviceGetDefaultMemPool(&pool, g->device));
    uint64_t keep = ~0ull;
    HBP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    pool_ready[g->device] = true;
  }
  void *block = nullptr;
  HBP_CUDA(cudaMallocAsync(&block, persistent + scratch_all, s));
  g->d_block = block;
  P.base = (char *)block;
  P.off = 0;
  plan_block(P);
  g->d_scratch = (char *)block + persistent;
  g->scratch_bytes = scratch_all;
  HBP_CUDA(cudaMemcpyAsync(g->d_rowptr, desc.factor_rowptr, (size_t)(F + 1) * 8,
                           cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(g->d_evar, desc.edge_var, nE * 4, cudaMemcpyHostToDevice, s));
  if (F) {
    HBP_CUDA(cudaMemcpyAsync(g->d_kind, desc.factor_kind, (size_t)F, cudaMemcpyHostToDevice, s));
    HBP_CUDA(cudaMemcpyAsync(g->d_p1, desc.p1, (size_t)F * 8, cudaMemcpyHostToDevice, s));
    HBP_CUDA(cudaMemcpyAsync(g->d_p2, desc.p2, (size_t)F * 8, cudaMemcpyHostToDevice, s));
  }
  clk.mark("upload");

  Arena A;
  A.base = (char *)g->d_scratch;
  DevInfo *d_info = A.take<DevInfo>(1);
  void *d_tmp = A.take<char>(tmp);
  unsigned *fkey = A.take<unsigned>(F + 1), *fkey_sorted = A.take<unsigned>(F + 1);
  int *iota = A.take<int>((size_t)maxn);
  int *fperm = A.take<int>(F + 1), *fdeg_ext = A.take<int>(F + 2);
  int *vdeg = A.take<int>(V + 1), *vdeg_sorted = A.take<int>(V + 1);
  int *vdeg_ext = A.take<int>(V + 2), *vstart = A.take<int>(V + 2);
  int *evar_sorted = A.take<int>((size_t)E), *ref_ftov = A.take<int>((size_t)E);
  int *canon2f = A.take<int>((size_t)E);
  int *gidx = A.take<int>(64), *gout = A.take<int>(64);

  DevInfo h{};
  h.err_factor = h.err_edge = h.err_var = INT_MAX;
  HBP_CUDA(cudaMemcpyAsync(d_info, &h, sizeof h, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemsetAsync(vdeg, 0, (size_t)(V + 1) * 4, s));
  k_factors<<<blocks_for(F), kB, 0, s>>>(g->d_rowptr, g->d_kind, F, d_info, fkey);
  k_edges<<<blocks_for(E), kB, 0, s>>>(g->d_evar, E, V, d_info, vdeg);
  k_vars<<<blocks_for(V), kB, 0, s>>>(vdeg, V, d_info);
  HBP_CUDA(cudaGetLastError());
  HBP_CUDA(cudaMemcpyAsync(&h, d_info, sizeof h, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  clk.mark("validate");
  // errors in layout.cpp's order and words
  if (h.err_factor != INT_MAX) {
    const int f = h.err_factor;
    const int64_t d = desc.factor_rowptr[f + 1] - desc.factor_rowptr[f];
    set_error("factor " + std::to_string(f) +
              (d < 1 || d > 65535 ? ": degree must be in [1, 65535]" : ": bad kind"));
    return HBP_EINVAL;
  }
  if (h.err_edge != INT_MAX) {
    set_error("edge variable out of range");
    return HBP_EINVAL;
  }
  if (h.err_var != INT_MAX) {
    set_error("variable " + std::to_string(h.err_var) + " appears in no factor");
    return HBP_EINVAL;
  }
  if (h.max_vdeg > 65535) {
    set_error("variable degree above 65535");
    return HBP_EINVAL;
  }

  // factors: stable sort by (heavy, kind, degree); rows by exclusive scan
  const unsigned nb = blocks_for(maxn);
  k_iota<<<nb, kB, 0, s>>>(iota, maxn);
  HBP_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, fkey, fkey_sorted, iota, fperm, F, 0, 18, s));
  k_low16<<<blocks_for(F + 1), kB, 0, s>>>(fkey_sorted, F, fdeg_ext);
  HBP_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, fdeg_ext, g->d_frow, F + 1, s));
  k_frows<<<blocks_for(F), kB, 0, s>>>(g->d_rowptr, fperm, g->d_frow, g->d_p1, g->d_p2, F,
                                       g->d_canon2v, g->d_fslot, g->d_fpar);
  // variables: stable sort by degree; rows by exclusive scan
  HBP_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, (const unsigned *)vdeg,
                                           (unsigned *)vdeg_sorted, iota, g->d_vorig, V, 0,
                                           bits_for(h.max_vdeg + 1), s));
  k_copy_ext<<<blocks_for(V + 1), kB, 0, s>>>(vdeg_sorted, V, vdeg_ext);
  HBP_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, vdeg_ext, g->d_vrow, V + 1, s));
  k_vinv<<<blocks_for(V), kB, 0, s>>>(g->d_vorig, V, g->d_vinv);
  clk.mark("rows");
  // the reference's ftov order: edges stably sorted by variable (storage.py:61)
  HBP_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, (const unsigned *)g->d_evar,
                                           (unsigned *)evar_sorted, iota, ref_ftov, (int)E, 0,
                                           bits_for(V), s));
  k_copy_ext<<<blocks_for(V + 1), kB, 0, s>>>(vdeg, V, vdeg_ext);
  HBP_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, vdeg_ext, vstart, V + 1, s));
  k_vrows<<<blocks_for(E), kB, 0, s>>>(ref_ftov, evar_sorted, vstart, g->d_vinv, g->d_vrow, vdeg,
                                       E, canon2f, g->d_vslot);
  k_twins<<<blocks_for(E), kB, 0, s>>>(g->d_canon2v, canon2f, g->d_fslot, E, g->d_vtof_twin,
                                       g->d_ftov_twin);
  HBP_CUDA(cudaGetLastError());
  clk.mark("transpose");

  // scalars and degree-class tables (layout.cpp:141-163)
  L = HostLayout();
  L.V = V;
  L.F = F;
  L.E = E;
  L.max_fdeg = h.max_fdeg;
  L.max_vdeg = h.max_vdeg;
  L.f_or_light = h.fclass[0];
  L.f_heavy = h.fclass[0] + h.fclass[1];
  L.f_or_heavy = L.f_heavy + h.fclass[2];
  L.v_heavy = h.v_light;
  L.n_unary = h.n_unary;
  auto classes = [](const int *hist, int lo, int hi, int32_t *node) {
    int n = lo;
    node[0] = lo;
    for (int d = 1; d <= kNodeMax + 1; ++d) {
      n += hist[d - 1];
      node[d] = d == kNodeMax + 1 ? hi : n;
    }
  };
  // variables have degree >= 1 and factors too, so hist[0] == 0
  classes(h.vhist, 0, L.v_heavy, L.vc_node);
  classes(h.fhist[0], 0, L.f_or_light, L.fa_node);
  classes(h.fhist[1], L.f_or_light, L.f_heavy, L.fo_node);
  // rows at the class boundaries + the heavy starts, gathered in one go
  const int K = kNodeMax + 2;
  int idx[64];
  for (int d = 0; d < K; ++d) {
    idx[d] = L.vc_node[d];
    idx[K + d] = L.fa_node[d];
    idx[2 * K + d] = L.fo_node[d];
  }
  idx[3 * K] = L.v_heavy;
  idx[3 * K + 1] = L.f_heavy;
  const int nidx = 3 * K + 2;
  HBP_CUDA(cudaMemcpyAsync(gidx, idx, nidx * 4, cudaMemcpyHostToDevice, s));
  k_gather<<<1, 64, 0, s>>>(g->d_vrow, gidx, K, gout);
  k_gather<<<1, 64, 0, s>>>(g->d_frow, gidx + K, 2 * K, gout + K);
  k_gather<<<1, 64, 0, s>>>(g->d_vrow, gidx + 3 * K, 1, gout + 3 * K);
  k_gather<<<1, 64, 0, s>>>(g->d_frow, gidx + 3 * K + 1, 1, gout + 3 * K + 1);
  int rows[64];
  HBP_CUDA(cudaMemcpyAsync(rows, gout, nidx * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < K; ++d) {
    L.vc_row[d] = rows[d];
    L.fa_row[d] = rows[K + d];
    L.fo_row[d] = rows[2 * K + d];
  }
  L.vrow_heavy = rows[3 * K];
  L.frow_heavy = rows[3 * K + 1];
  {
    int64_t vcnt[kClassMax + 2], fcnt[2][kClassMax + 2], fhuge[2] = {h.fhuge[0], h.fhuge[1]};
    for (int d = 0; d < kClassMax + 2; ++d) {
      vcnt[d] = h.vcls[d];
      fcnt[0][d] = h.fcls[0][d];
      fcnt[1][d] = h.fcls[1][d];
    }
    class_tables(L, vcnt, h.vhuge, fcnt, fhuge);
  }
  L.host_ready = false;
  clk.mark("tables");
  add_last_launches(17);
  return HBP_OK;
}

hbp_status ensure_host_layout(hbp_graph *g) {
  if (g->L.host_ready) return HBP_OK;
  HBP_CUDA(cudaSetDevice(g->device));
  const HostLayout &D = g->L;
  std::vector<int64_t> rp((size_t)D.F + 1);
  std::vector<int32_t> ev((size_t)D.E);
  std::vector<int8_t> kind((size_t)std::max(1, D.F));
  std::vector<double> p1((size_t)std::max(1, D.F)), p2((size_t)std::max(1, D.F));
  cudaStream_t s = g->stream;
  HBP_CUDA(cudaMemcpyAsync(rp.data(), g->d_rowptr, rp.size() * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(ev.data(), g->d_evar, ev.size() * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(kind.data(), g->d_kind, kind.size(), cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(p1.data(), g->d_p1, p1.size() * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(p2.data(), g->d_p2, p2.size() * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  hbp_graph_desc desc{D.V, D.F, D.E, rp.data(), ev.data(), kind.data(), p1.data(), p2.data()};
  HostLayout H;
  hbp_status st = build_layout(desc, H);
  if (st != HBP_OK) return st;
  // the device build's scalars must be the host build's
  bool same = H.V == D.V && H.F == D.F && H.E == D.E && H.f_or_light == D.f_or_light &&
              H.f_heavy == D.f_heavy && H.f_or_heavy == D.f_or_heavy && H.v_heavy == D.v_heavy &&
              H.max_fdeg == D.max_fdeg && H.max_vdeg == D.max_vdeg && H.n_unary == D.n_unary &&
              H.vrow_heavy == D.vrow_heavy && H.frow_heavy == D.frow_heavy;
  for (int d = 0; d < kNodeMax + 2; ++d)
    same = same && H.vc_node[d] == D.vc_node[d] && H.vc_row[d] == D.vc_row[d] &&
           H.fa_node[d] == D.fa_node[d] && H.fa_row[d] == D.fa_row[d] &&
           H.fo_node[d] == D.fo_node[d] && H.fo_row[d] == D.fo_row[d];
  for (int d = 0; d < kClassMax + 2; ++d) {
    same = same && H.vcls_node[d] == D.vcls_node[d] && H.vcls_row[d] == D.vcls_row[d] &&
           H.vcls_cnt[d] == D.vcls_cnt[d];
    for (int k = 0; k < 2; ++k)
      same = same && H.fcls_node[k][d] == D.fcls_node[k][d] && H.fcls_row[k][d] == D.fcls_row[k][d] &&
             H.fcls_cnt[k][d] == D.fcls_cnt[k][d];
  }
  if (!same) {
    set_error("internal: device and host layouts disagree");
    return HBP_ECUDA;
  }
  g->L = std::move(H);
  return HBP_OK;
}

hbp_status parall_check_device(hbp_graph *g, int64_t ns, const int32_t *s_edges, int64_t nt,
                               const int32_t *t_edges, bool *is_parall) {
  *is_parall = false;
  const int64_t E = g->L.E;
  if (ns != E || nt != E - g->L.n_unary) return HBP_OK;
  cudaStream_t s = g->stream;
  const int64_t words = (E + 31) / 32;
  char *buf = (char *)g->d_scratch;  // sized for 2E ints + 2 bitmaps (build_layout_device)
  int *d_s = (int *)buf, *d_t = d_s + ns;
  unsigned *bits = (unsigned *)(d_t + nt);
  int *bad = (int *)(bits + 2 * words);
  HBP_CUDA(cudaMemcpyAsync(d_s, s_edges, (size_t)ns * 4, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(d_t, t_edges, (size_t)nt * 4, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemsetAsync(bits, 0, (size_t)words * 8 + 4, s));
  k_parall_check<<<blocks_for(ns + nt), kB, 0, s>>>(d_s, ns, d_t, nt, E, g->d_canon2v,
                                                   g->d_fslot, bits, bad);
  HBP_CUDA(cudaGetLastError());
  int h_bad = 0;
  HBP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  add_last_launches(1);
  *is_parall = h_bad == 0;
  return HBP_OK;
}


// ---- lbp_pslot's slot chunks (engine.cu): every factor as a lane group of a
// 32-lane chunk, one int4 record per lane. Chunks come per class (kind,
// degree), dearest degree first, the unary factors last; inside a class the
// factors are ordered by the largest degree of their variables, so a chunk's
// lanes load rows of similar length (the row loop runs to the chunk's max).
namespace {
struct PslotClasses {
  int n;                        // classes
  int rank[2][kClassMax + 1];   // (kind, degree) -> class rank, -1: empty
  int start[2 * kClassMax + 2]; // first sorted position of each class
  int chunk[2 * kClassMax + 2]; // first chunk of each class
  int node[2 * kClassMax + 2];  // first internal factor of each class
  int count[2 * kClassMax + 2];
  int deg[2 * kClassMax + 2], kind[2 * kClassMax + 2];
};

__device__ __forceinline__ int pslot_kind(int f, int f_or_light, int f_heavy, int f_or_heavy) {
  return ((f >= f_or_light && f < f_heavy) || f >= f_or_heavy) ? 1 : 0;
}

__global__ void k_pslot_keys(const int *frow, const int *vtof_twin, const int2 *vslot, int F,
                             int f_or_light, int f_heavy, int f_or_heavy, PslotClasses C,
                             unsigned *key, int *val) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int r = frow[f], d = frow[f + 1] - r;
  const int kind = pslot_kind(f, f_or_light, f_heavy, f_or_heavy);
  int mx = 0;
  for (int k = 0; k < d; ++k) mx = max(mx, (int)((unsigned)vslot[vtof_twin[r + k]].y >> 16));
  key[f] = (unsigned)C.rank[kind][d] << 8 | (unsigned)(255 - min(mx, 255));
  val[f] = f;
}

// one thread per factor: its lane records, and the chunk's unused lanes
// (zero = invalid) by the chunk's first / the class's last factor. perm ==
// nullptr: the factors of a class in internal order (thread i = factor i)
__global__ void k_pslot_records(const unsigned *key, const int *perm, const int *frow,
                                const int *vtof_twin, const int2 *vslot, int F, int f_or_light,
                                int f_heavy, int f_or_heavy, PslotClasses C, int4 *srec,
                                int *sinfo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F) return;
  int c, f, pos;
  if (perm) {
    c = (int)(key[i] >> 8);
    f = perm[i];
    pos = i - C.start[c];
  } else {
    f = i;
    const int kind = pslot_kind(f, f_or_light, f_heavy, f_or_heavy);
    c = C.rank[kind][frow[f + 1] - frow[f]];
    pos = f - C.node[c];
  }
  const int d = C.deg[c], per = 32 / d;
  const int chunk = C.chunk[c] + pos / per, g = pos % per;
  int4 *lanes = srec + (size_t)chunk * 32;
  const int r = frow[f];
  int mx = 0;
  for (int k = 0; k < d; ++k) {
    const int q = vtof_twin[r + k];
    const int2 w = vslot[q];
    const int j = w.y & 0xffff, dv = (int)((unsigned)w.y >> 16);
    mx = max(mx, dv);
    lanes[g * d + k] = make_int4(q - j, w.x, f, dv | j << 8 | k << 16 | 1 << 24);
  }
  const int4 none = make_int4(0, 0, 0, 0);
  if (g == 0)
    for (int l = per * d; l < 32; ++l) lanes[l] = none;
  if (pos == C.count[c] - 1)
    for (int l = (g + 1) * d; l < per * d; ++l) lanes[l] = none;
  // sorted: the chunk's first factor has its longest variable row
  if (g == 0) sinfo[chunk] = d | C.kind[c] << 8 | mx << 16;
}
}  // namespace

hbp_status build_pslot_device(hbp_graph *g) {
  const HostLayout &L = g->L;
  const int F = L.F;
  cudaStream_t s = g->stream;
  PslotClasses C{};
  for (int k = 0; k < 2; ++k)
    for (int d = 0; d <= kClassMax; ++d) C.rank[k][d] = -1;
  int pos = 0, chunks = 0;
  auto add = [&](int d, int k) {
    const int cnt = L.fcls_cnt[k][d];
    if (cnt <= 0) return;
    const int c = C.n++;
    C.rank[k][d] = c;
    C.start[c] = pos;
    C.chunk[c] = chunks;
    C.node[c] = L.fcls_node[k][d];
    C.count[c] = cnt;
    C.deg[c] = d;
    C.kind[c] = k;
    pos += cnt;
    chunks += (cnt + 32 / d - 1) / (32 / d);
  };
  for (int d = kClassMax; d >= 2; --d)
    for (int k = 0; k < 2; ++k) add(d, k);
  const int chunks_nounary = chunks;
  for (int k = 0; k < 2; ++k) add(1, k);
  g->pslot_chunks = chunks;
  g->pslot_chunks_nounary = chunks_nounary;
  // one stream-ordered allocation from the graph's pool (a fresh graph's
  // run() pays no cudaMalloc / cudaFree synchronisation for it). The second
  // ftov buffer has 2 messages of slack: lbp_pslot reads rows as 32-byte
  // aligned pairs (d_ftov is followed by further arena allocations, which
  // its last pair may touch)
  {
    const size_t nch = (size_t)std::max(1, chunks);
    const size_t b_rec = nch * 32 * sizeof(int4), b_inf = (nch * 4 + 255) & ~(size_t)255,
                 b_ft = (((size_t)L.E + 2) * sizeof(double2) + 255) & ~(size_t)255,
                 b_p0 = (size_t)std::max(1, L.V) * sizeof(double);
    char *blk = nullptr;
    HBP_CUDA(cudaMallocAsync((void **)&blk, b_rec + b_inf + b_ft + b_p0, s));
    g->d_pslot_block = blk;
    g->d_srec = (int4 *)blk;
    g->d_sinfo = (int *)(blk + b_rec);
    g->d_ftov_alt = (double2 *)(blk + b_rec + b_inf);
    g->d_p0_alt = (double *)(blk + b_rec + b_inf + b_ft);
  }
  const unsigned nb = (unsigned)((F + 255) / 256);
  // each class's factors ordered by their longest variable row (a CUB sort:
  // a chunk's lanes then load rows of similar length, so fewer of its pair
  // loads are live -- C4-PARALL 0.271 against 0.295 ms in the internal
  // order, which HBP_PSLOT_SORT=0 keeps for A/B)
  const char *se = getenv("HBP_PSLOT_SORT");
  char *buf = nullptr;
  if (!(se && atoi(se) == 0)) {
    size_t tmp = 0;
    HBP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (unsigned *)nullptr, (unsigned *)nullptr,
                                             (int *)nullptr, (int *)nullptr, F, 0, 16, s));
    const size_t fb = ((size_t)std::max(1, F) * 4 + 255) & ~(size_t)255;
    HBP_CUDA(cudaMallocAsync((void **)&buf, 4 * fb + tmp, s));
    unsigned *key = (unsigned *)buf, *key_s = (unsigned *)(buf + fb);
    int *val = (int *)(buf + 2 * fb), *val_s = (int *)(buf + 3 * fb);
    k_pslot_keys<<<nb, 256, 0, s>>>(g->d_frow, g->d_vtof_twin, g->d_vslot, F, L.f_or_light,
                                    L.f_heavy, L.f_or_heavy, C, key, val);
    HBP_CUDA(cub::DeviceRadixSort::SortPairs(buf + 4 * fb, tmp, key, key_s, val, val_s, F, 0, 16, s));
    k_pslot_records<<<nb, 256, 0, s>>>(key_s, val_s, g->d_frow, g->d_vtof_twin, g->d_vslot, F,
                                       L.f_or_light, L.f_heavy, L.f_or_heavy, C, g->d_srec,
                                       g->d_sinfo);
    add_last_launches(3);
  } else {
    k_pslot_records<<<nb, 256, 0, s>>>(nullptr, nullptr, g->d_frow, g->d_vtof_twin, g->d_vslot, F,
                                       L.f_or_light, L.f_heavy, L.f_or_heavy, C, g->d_srec,
                                       g->d_sinfo);
    add_last_launches(1);
  }
  HBP_CUDA(cudaGetLastError());
  if (buf) HBP_CUDA(cudaFreeAsync(buf, s));
  return HBP_OK;
}
}  // namespace hbp

// Diagnostic: every device layout array against the host builder's (tests).
hbp_status hbp_graph_layout_check(hbp_graph *g, int64_t *mismatches) {
  if (!g || !mismatches) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  hbp_status st = hbp::ensure_host_layout(g);
  if (st != HBP_OK) return st;
  const hbp::HostLayout &L = g->L;
  cudaStream_t s = g->stream;
  const size_t V = (size_t)L.V, F = (size_t)L.F, E = (size_t)L.E;
  std::vector<int32_t> vrow(V + 1), frow(F + 1), vorig(std::max<size_t>(1, V)),
      vinv(std::max<size_t>(1, V)), vtw(E), vsl(2 * E), fsl(2 * E), c2v(E);
  std::vector<uint32_t> ftw(E);
  std::vector<double> fpar(2 * std::max<size_t>(1, F));
  HBP_CUDA(cudaMemcpyAsync(vrow.data(), g->d_vrow, vrow.size() * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(frow.data(), g->d_frow, frow.size() * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(vorig.data(), g->d_vorig, V * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(vinv.data(), g->d_vinv, V * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(vtw.data(), g->d_vtof_twin, E * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(ftw.data(), g->d_ftov_twin, E * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(vsl.data(), g->d_vslot, E * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(fsl.data(), g->d_fslot, E * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(c2v.data(), g->d_canon2v, E * 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(fpar.data(), g->d_fpar, F * 16, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  int64_t bad = 0;
  bad += vrow != L.vrow;
  bad += frow != L.frow;
  for (size_t i = 0; i < V; ++i) bad += (vorig[i] != L.vperm[i]) + (vinv[i] != L.vinv[i]);
  bad += vtw != L.vtof_twin;
  bad += ftw != L.ftov_twin;
  bad += vsl != L.vslot;
  bad += fsl != L.fslot;
  bad += c2v != L.canon2v;
  for (size_t i = 0; i < F; ++i)
    bad += std::memcmp(&fpar[2 * i], &L.p1[L.fperm[i]], 8) != 0 ||
           std::memcmp(&fpar[2 * i + 1], &L.p2[L.fperm[i]], 8) != 0;
  *mismatches = bad;
  return HBP_OK;
}
