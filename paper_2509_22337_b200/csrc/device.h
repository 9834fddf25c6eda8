// Device-side handle types shared by the executors (engine.cu: single graph,
// sweep.cu: multi-evidence sweep). Internal; not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"

namespace hbp {
// kernels launched by the last C-ABI call on this thread (bench gpu_launches)
void set_last_launches(int64_t n);
void add_last_launches(int64_t n);
}  // namespace hbp

#define HBP_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t _e = (call);                                                    \
    if (_e != cudaSuccess) {                                                    \
      hbp::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));       \
      return HBP_ECUDA;                                                         \
    }                                                                           \
  } while (0)

template <typename T>
inline hbp_status upload(T **dst, const std::vector<T> &src, cudaStream_t s) {
  HBP_CUDA(cudaMalloc((void **)dst, std::max<size_t>(1, src.size()) * sizeof(T)));
  if (!src.empty())
    HBP_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return HBP_OK;
}


struct hbp_graph {
  hbp::HostLayout L;
  int device = 0;
  cudaStream_t stream = nullptr;      // stream all work of this graph runs on
  cudaStream_t own_stream = nullptr;  // created with the graph
  int num_sms = 0, coop_blocks = 0, threads = 1024;
  const void *kernel = nullptr;         // the single-graph executor
  const void *kernel_fused = nullptr;   // its instance for plans with fused levels
  int coop_blocks_fused = 0;
  const void *kernel_parall = nullptr;  // its instance for PARALL plans (two whole-node phases)
  const void *kernel_parall_nonorm = nullptr;  // the same without message normalisation
  int coop_blocks_parall = 0;
  const void *kernel_pslot = nullptr;  // PARALL plans as one phase per iteration (lbp_pslot)
  const void *kernel_pslot_nonorm = nullptr;
  int coop_blocks_pslot = 0;
  // lbp_pslot's slot chunks (32 int4 lane records + one info word each,
  // layout_dev.cu build_pslot_device) and second ftov / P0 buffers (on first use)
  void *d_pslot_block = nullptr;  // the four below, one pool allocation
  int4 *d_srec = nullptr;
  int *d_sinfo = nullptr;
  int pslot_chunks = 0, pslot_chunks_nounary = 0;
  double2 *d_ftov_alt = nullptr;
  double *d_p0_alt = nullptr;
  int *d_vtof_twin = nullptr, *d_vorig = nullptr, *d_vrow = nullptr, *d_frow = nullptr;
  unsigned *d_ftov_twin = nullptr;
  int2 *d_vslot = nullptr, *d_fslot = nullptr;
  double2 *d_fpar = nullptr, *d_vtof = nullptr, *d_ftov = nullptr, *d_marg = nullptr;
  double *d_prev = nullptr;
  // one allocation for everything below up to d_canon2v, plus the layout
  // build's scratch (reused by the PARALL shape test of hbp_plan_create)
  void *d_block = nullptr;
  void *d_scratch = nullptr;
  size_t scratch_bytes = 0;
  // canonical graph arrays (the device layout build's input; the lazy host
  // layout downloads them) and canonical edge -> internal vtof position
  int64_t *d_rowptr = nullptr;
  int *d_evar = nullptr, *d_canon2v = nullptr;
  int8_t *d_kind = nullptr;
  double *d_p1 = nullptr, *d_p2 = nullptr;
  // evidence (clamp_evidence without a graph rebuild) + ranking scratch
  unsigned char *d_ev = nullptr;
  bool has_ev = false;
  std::vector<int32_t> ev_var;  // the clamps in order (host): row lengths / positions of
  std::vector<int8_t> ev_val;   // the clamped graph for the underflow attribution
  int *d_vinv = nullptr;
  void *d_rank = nullptr;
  size_t rank_cap = 0;
  void *d_ev_list = nullptr;
  size_t ev_list_cap = 0;
  // control block sized for max_iterations
  void *d_ctrl = nullptr;
  size_t ctrl_cap = 0;  // entries per array
  double2 *d_hist = nullptr;
  size_t hist_cap = 0;  // double2 entries
  int hist_valid = 0;   // iterations of history the last run left in d_hist
  unsigned long long *d_trace = nullptr;
  size_t trace_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  ~hbp_graph() {
    cudaSetDevice(device);
    // the layout, message buffers and layout scratch live in d_block (pool)
    if (d_block) cudaFreeAsync(d_block, own_stream ? own_stream : stream);
    if (d_pslot_block) cudaFreeAsync(d_pslot_block, own_stream ? own_stream : stream);
    for (void *p : {(void *)d_ev, d_rank, d_ev_list, d_ctrl, (void *)d_hist, (void *)d_trace})
      if (p) cudaFree(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
};

namespace hbp {
// layout_dev.cu: the device layout build (hbp_graph_create), the host layout
// on first host-side use, and the PARALL shape test of a one-batch schedule
hbp_status build_layout_device(const hbp_graph_desc &desc, hbp_graph *g);
hbp_status ensure_host_layout(hbp_graph *g);
hbp_status build_pslot_device(hbp_graph *g);
hbp_status parall_check_device(hbp_graph *g, int64_t ns, const int32_t *s_edges, int64_t nt,
                               const int32_t *t_edges, bool *is_parall);
}  // namespace hbp

struct hbp_plan {
  hbp_graph *g = nullptr;
  hbp::PlanHost host;
  hbp::Phase *d_phases = nullptr;
  int *d_items = nullptr;
  int32_t *d_fitems = nullptr;  // fused levels (int4 lane records)
  int32_t *d_iw = nullptr;  // per list item: its slot word and twin (int4, small phases)
  hbp_plan *unfused = nullptr;  // the same schedule without fused levels (underflow attribution)
  int grid = 1;
  const void *kernel = nullptr;  // executor instance (fused levels or not)
  const void *kernel_nonorm = nullptr;  // the instance for normalize_messages off
  int threads = 0;
  int csize = 1;  // CTAs (one cluster) that run the small levels
  bool pslot = false;  // PARALL plan on lbp_pslot (slot classes in KParams::fcc)
  // the schedule as given (reference batch order), for the exact underflow
  // attribution: device [s_edges | t_edges] (stream-ordered pool) + host offsets
  int *d_sched = nullptr;
  int64_t ns = 0;
  std::vector<int64_t> s_off, t_off;
  // evidence codes emulate clamp_evidence only for schedules whose batches do
  // not change under clamping: one batch (PARALL) or canonical SEQFIX.
  // -1 = not checked yet (checked on the first run with evidence)
  int ev_ok = -1;
  ~hbp_plan() {
    cudaSetDevice(g->device);
    for (void *p : {(void *)d_phases, (void *)d_items, (void *)d_fitems, (void *)d_iw})
      if (p) cudaFree(p);
    delete unfused;
    if (d_sched) cudaFreeAsync(d_sched, g->stream);
  }
};

