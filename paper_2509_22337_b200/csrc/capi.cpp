// C ABI for the strategy compiler + error reporting (see include/hornbp_gpu.h).
#include <cstring>
#include <new>
#include <string>

#include "internal.h"

namespace {
thread_local std::string g_error;
}

namespace hbp {
void set_error(const std::string &msg) { g_error = msg; }
}  // namespace hbp

struct hbp_schedule {
  hbp::Schedule s;
};

extern "C" {

const char *hbp_last_error(void) { return g_error.c_str(); }

const char *hbp_version(void) { return "paper_2509_22337_b200 0.1.0 (sm_100a)"; }

hbp_status hbp_toposort(int64_t n, int64_t m, const int32_t *before, const int32_t *after,
                        int32_t *order_out, int64_t *cycle_edge) {
  if (n < 0 || m < 0 || (m > 0 && (!before || !after)) || (n > 0 && !order_out)) {
    hbp::set_error("bad toposort arguments");
    return HBP_EINVAL;
  }
  for (int64_t i = 0; i < m; ++i)
    if (before[i] < 0 || before[i] >= n || after[i] < 0 || after[i] >= n) {
      hbp::set_error("pair edge out of range");
      return HBP_EINVAL;
    }
  std::vector<int32_t> order;
  if (!hbp::toposort(n, m, before, after, order, cycle_edge)) {
    hbp::set_error("ordering relation has a cycle");
    return HBP_ECYCLE;
  }
  if (n) std::memcpy(order_out, order.data(), (size_t)n * sizeof(int32_t));
  return HBP_OK;
}

hbp_status hbp_compile(const hbp_graph_desc *g, int64_t m, const int32_t *before,
                       const int32_t *after, const int32_t *rank, hbp_schedule **out,
                       int64_t *cycle_edge) {
  if (!g || !out || m < 0 || (m > 0 && (!before || !after))) {
    hbp::set_error("bad compile arguments");
    return HBP_EINVAL;
  }
  *out = nullptr;
  const int64_t E = g->num_edges;
  if (g->factor_rowptr[0] != 0 || g->factor_rowptr[g->num_factors] != E) {
    hbp::set_error("factor_rowptr does not span the edge array");
    return HBP_EINVAL;
  }
  for (int64_t i = 0; i < m; ++i)
    if (before[i] < 0 || before[i] >= E || after[i] < 0 || after[i] >= E) {
      hbp::set_error("pair edge out of range");
      return HBP_EINVAL;
    }
  hbp_schedule *s = new (std::nothrow) hbp_schedule();
  if (!s) return HBP_ENOMEM;
  hbp_status st = hbp::compile(*g, m, before, after, rank, s->s, cycle_edge);
  if (st != HBP_OK) {
    if (st == HBP_ECYCLE) hbp::set_error("ordering relation has a cycle");
    delete s;
    return st;
  }
  *out = s;
  return HBP_OK;
}

hbp_status hbp_schedule_sizes(const hbp_schedule *s, int64_t *k, int64_t *ns, int64_t *nt) {
  if (!s) return HBP_EINVAL;
  *k = (int64_t)s->s.s_off.size() - 1;
  *ns = (int64_t)s->s.s_edges.size();
  *nt = (int64_t)s->s.t_edges.size();
  return HBP_OK;
}

hbp_status hbp_schedule_copy(const hbp_schedule *s, int64_t *s_off, int32_t *s_edges,
                             int64_t *t_off, int32_t *t_edges) {
  if (!s) return HBP_EINVAL;
  std::memcpy(s_off, s->s.s_off.data(), s->s.s_off.size() * sizeof(int64_t));
  std::memcpy(t_off, s->s.t_off.data(), s->s.t_off.size() * sizeof(int64_t));
  if (!s->s.s_edges.empty())
    std::memcpy(s_edges, s->s.s_edges.data(), s->s.s_edges.size() * sizeof(int32_t));
  if (!s->s.t_edges.empty())
    std::memcpy(t_edges, s->s.t_edges.data(), s->s.t_edges.size() * sizeof(int32_t));
  return HBP_OK;
}

void hbp_schedule_destroy(hbp_schedule *s) { delete s; }

}  // extern "C"
