// Native update-strategy compiler: ordering relation -> dependency-analysed
// batches (s_i) and their companion variable-to-factor batches (t_i).
//
// Output is batch-for-batch identical to the reference compiler:
//   toposort        schedule.py:94-114  (Kahn layers, ascending edge id per layer)
//   batching        schedule.py:261-290 (Alg. 2: flush when an edge in the
//                   current batch both feeds this edge and precedes it)
//   t-batches       schedule.py:293-312 (Alg. 3)
// The reference answers `precedes` with a memoised full ancestor closure
// (schedule.py:131-155), quadratic in chain length. Here a query only needs
// to know whether one of the *current batch's* neighbours reaches the edge,
// and any path between two edges stays inside the topological interval
// [pos(candidate), pos(edge)], so a reverse DFS pruned at the lowest
// candidate position answers it exactly in time proportional to the batch's
// span of the order.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"

namespace hbp {

namespace {

struct Csr {
  std::vector<int64_t> ptr;
  std::vector<int32_t> idx;
};

// Per-variable rows of canonical edge indices in (factor, slot) order.
Csr variable_rows(const hbp_graph_desc &g) {
  Csr c;
  c.ptr.assign((size_t)g.num_variables + 1, 0);
  for (int64_t e = 0; e < g.num_edges; ++e) c.ptr[(size_t)g.edge_var[e] + 1]++;
  for (int32_t v = 0; v < g.num_variables; ++v) c.ptr[v + 1] += c.ptr[v];
  c.idx.resize((size_t)g.num_edges);
  std::vector<int64_t> fill(c.ptr.begin(), c.ptr.end() - 1);
  for (int64_t e = 0; e < g.num_edges; ++e) c.idx[(size_t)fill[g.edge_var[e]]++] = (int32_t)e;
  return c;
}

}  // namespace

// Kahn layers; returns false on a cycle (cycle_edge = smallest stuck edge).
bool toposort(int64_t n, int64_t m, const int32_t *before, const int32_t *after,
              std::vector<int32_t> &order, int64_t *cycle_edge) {
  std::vector<int32_t> indeg((size_t)n, 0);
  std::vector<int64_t> sp((size_t)n + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    indeg[after[i]]++;
    sp[(size_t)before[i] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) sp[i + 1] += sp[i];
  std::vector<int32_t> succ((size_t)m);
  {
    std::vector<int64_t> fill(sp.begin(), sp.end() - 1);
    for (int64_t i = 0; i < m; ++i) succ[(size_t)fill[before[i]]++] = after[i];
  }
  order.clear();
  order.reserve((size_t)n);
  std::vector<int32_t> layer, next;
  for (int64_t e = 0; e < n; ++e)
    if (indeg[e] == 0) layer.push_back((int32_t)e);
  while (!layer.empty()) {
    order.insert(order.end(), layer.begin(), layer.end());
    next.clear();
    for (int32_t e : layer)
      for (int64_t k = sp[e]; k < sp[e + 1]; ++k)
        if (--indeg[succ[k]] == 0) next.push_back(succ[k]);
    std::sort(next.begin(), next.end());
    layer.swap(next);
  }
  if ((int64_t)order.size() != n) {
    for (int64_t e = 0; e < n; ++e)
      if (indeg[e] > 0) {
        if (cycle_edge) *cycle_edge = e;
        break;
      }
    return false;
  }
  return true;
}

hbp_status compile(const hbp_graph_desc &g, int64_t m, const int32_t *before,
                   const int32_t *after, const int32_t *rank, Schedule &out,
                   int64_t *cycle_edge) {
  const int64_t E = g.num_edges;
  std::vector<int32_t> order;
  if (!toposort(E, m, before, after, order, cycle_edge)) return HBP_ECYCLE;

  // edge -> factor
  std::vector<int32_t> efac((size_t)E);
  for (int32_t f = 0; f < g.num_factors; ++f)
    for (int64_t e = g.factor_rowptr[f]; e < g.factor_rowptr[f + 1]; ++e) efac[e] = f;

  out.s_off.assign(1, 0);
  out.s_edges.clear();
  if (E == 0) {
    out.t_off.assign(1, 0);
    out.t_edges.clear();
    return HBP_OK;
  }
  if (m == 0) {  // PARALL: one batch of every edge (schedule.py:271-272)
    out.s_edges = order;
    out.s_off.push_back(E);
  } else {
    Csr vrow = variable_rows(g);
    // predecessor lists for the reachability test
    std::vector<int64_t> pp((size_t)E + 1, 0);
    std::vector<int32_t> pred;
    if (!rank) {
      for (int64_t i = 0; i < m; ++i) pp[(size_t)after[i] + 1]++;
      for (int64_t i = 0; i < E; ++i) pp[i + 1] += pp[i];
      pred.resize((size_t)m);
      std::vector<int64_t> fill(pp.begin(), pp.end() - 1);
      for (int64_t i = 0; i < m; ++i) pred[(size_t)fill[after[i]]++] = before[i];
    }
    std::vector<int32_t> pos((size_t)E);
    for (int64_t i = 0; i < E; ++i) pos[order[i]] = (int32_t)i;
    std::vector<int32_t> in_batch((size_t)E, -1);  // batch id of placed edges
    std::vector<int32_t> stamp((size_t)E, -1);
    std::vector<int32_t> stack, cands;
    int32_t batch = 0;
    int32_t query = 0;
    for (int64_t oi = 0; oi < E; ++oi) {
      const int32_t e = order[oi];
      const int32_t a = efac[e];
      const int64_t r0 = g.factor_rowptr[a], r1 = g.factor_rowptr[a + 1];
      bool conflict = false;
      cands.clear();
      // N_E(e) (schedule.py:35-52): edges (a*, v*) with v* another variable
      // of a and a* != a another factor of v*.
      for (int64_t q = r0; q < r1 && !conflict; ++q) {
        if (q == e) continue;
        const int32_t vs = g.edge_var[q];
        for (int64_t k = vrow.ptr[vs]; k < vrow.ptr[vs + 1]; ++k) {
          const int32_t o = vrow.idx[k];
          if (efac[o] == a || in_batch[o] != batch) continue;
          if (rank) {
            if (rank[o] < rank[e]) { conflict = true; break; }
          } else {
            cands.push_back(o);
          }
        }
      }
      if (!rank && !cands.empty()) {
        // reverse DFS from e, pruned below the lowest candidate position
        int32_t lo = pos[cands[0]];
        for (int32_t c : cands) lo = std::min(lo, pos[c]);
        ++query;
        for (int32_t c : cands) stamp[c] = -2 - query;  // candidate marker
        stack.assign(1, e);
        std::vector<int32_t> seen_local;
        // visited marker: stamp == query
        while (!stack.empty() && !conflict) {
          int32_t x = stack.back();
          stack.pop_back();
          for (int64_t k = pp[x]; k < pp[x + 1]; ++k) {
            int32_t y = pred[k];
            if (pos[y] < lo) continue;
            if (stamp[y] == -2 - query) { conflict = true; break; }
            if (stamp[y] == query) continue;
            stamp[y] = query;
            stack.push_back(y);
          }
        }
        for (int32_t c : cands)
          if (stamp[c] == -2 - query) stamp[c] = -1;
      }
      if (conflict) {
        out.s_off.push_back((int64_t)out.s_edges.size());
        ++batch;
      }
      out.s_edges.push_back(e);
      in_batch[e] = batch;
    }
    out.s_off.push_back((int64_t)out.s_edges.size());
  }

  // t-batches (Alg. 3): every other slot of each factor touched by s_i.
  const int64_t k = (int64_t)out.s_off.size() - 1;
  out.t_off.assign(1, 0);
  out.t_edges.clear();
  std::vector<int32_t> cnt((size_t)g.num_factors, 0), only((size_t)g.num_factors, -1);
  std::vector<int32_t> touched, tb;
  for (int64_t b = 0; b < k; ++b) {
    touched.clear();
    for (int64_t i = out.s_off[b]; i < out.s_off[b + 1]; ++i) {
      const int32_t e = out.s_edges[i];
      const int32_t a = efac[e];
      if (cnt[a]++ == 0) {
        touched.push_back(a);
        only[a] = e;
      } else if (only[a] == e) {
        cnt[a]--;  // duplicate edge in a batch counts once
      }
    }
    std::sort(touched.begin(), touched.end());
    tb.clear();
    for (int32_t a : touched) {
      for (int64_t q = g.factor_rowptr[a]; q < g.factor_rowptr[a + 1]; ++q)
        if (cnt[a] >= 2 || q != only[a]) tb.push_back((int32_t)q);
      cnt[a] = 0;
      only[a] = -1;
    }
    out.t_edges.insert(out.t_edges.end(), tb.begin(), tb.end());
    out.t_off.push_back((int64_t)out.t_edges.size());
  }
  return HBP_OK;
}

}  // namespace hbp
