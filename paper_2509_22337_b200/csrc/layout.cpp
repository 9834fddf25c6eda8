// Host-side builders: the device message layout (MessageStore, storage.py:36-94)
// and the per-schedule level program (the pass compilation of engine.py:128-152,
// :357-410, :500-507, recast as node/target work items).
#include <algorithm>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace hbp {

namespace {
constexpr int32_t kCta0Threshold = 3072;  // phases with fewer items run on CTA 0
}

hbp_status build_layout(const hbp_graph_desc &g, HostLayout &L) {
  if (g.num_variables < 0 || g.num_factors < 0 || g.num_edges < 0) {
    set_error("negative graph dimension");
    return HBP_EINVAL;
  }
  if (g.num_edges == 0) {
    set_error("graph has no edges");
    return HBP_EINVAL;
  }
  if (g.num_edges >= (int64_t)1 << 31) {
    set_error("graph has too many edges for the int32 device layout");
    return HBP_EINVAL;
  }
  const int32_t V = g.num_variables, F = g.num_factors;
  const int64_t E = g.num_edges;
  L.V = V;
  L.F = F;
  L.E = E;
  if (g.factor_rowptr[0] != 0 || g.factor_rowptr[F] != E) {
    set_error("factor_rowptr does not span the edge array");
    return HBP_EINVAL;
  }
  L.rowptr.assign(g.factor_rowptr, g.factor_rowptr + F + 1);
  L.edge_var.assign(g.edge_var, g.edge_var + E);
  L.kind.assign(g.factor_kind, g.factor_kind + F);
  L.p1.assign(g.p1, g.p1 + F);
  L.p2.assign(g.p2, g.p2 + F);
  int32_t maxdeg = 0;
  for (int32_t f = 0; f < F; ++f) {
    int64_t d = L.rowptr[f + 1] - L.rowptr[f];
    if (d < 1 || d > 65535) {
      set_error("factor " + std::to_string(f) + ": degree must be in [1, 65535]");
      return HBP_EINVAL;
    }
    if (L.kind[f] != HBP_AND && L.kind[f] != HBP_OR) {
      set_error("factor " + std::to_string(f) + ": bad kind");
      return HBP_EINVAL;
    }
    maxdeg = std::max<int32_t>(maxdeg, (int32_t)d);
  }
  for (int64_t e = 0; e < E; ++e)
    if (L.edge_var[e] < 0 || L.edge_var[e] >= V) {
      set_error("edge variable out of range");
      return HBP_EINVAL;
    }
  L.max_fdeg = maxdeg;

  // factors: stable counting sort by (kind, degree)
  const int32_t nkeys = 2 * (maxdeg + 1);
  std::vector<int64_t> bucket((size_t)nkeys + 1, 0);
  auto fkey = [&](int32_t f) {
    return (int32_t)L.kind[f] * (maxdeg + 1) + (int32_t)(L.rowptr[f + 1] - L.rowptr[f]);
  };
  for (int32_t f = 0; f < F; ++f) bucket[fkey(f) + 1]++;
  for (int32_t k = 0; k < nkeys; ++k) bucket[k + 1] += bucket[k];
  L.f_or_begin = (int32_t)bucket[maxdeg + 1];
  L.fperm.resize(F);
  L.finv.resize(F);
  {
    std::vector<int64_t> fill(bucket.begin(), bucket.end() - 1);
    for (int32_t f = 0; f < F; ++f) {
      int32_t i = (int32_t)fill[fkey(f)]++;
      L.fperm[i] = f;
      L.finv[f] = i;
    }
  }
  L.frow.assign((size_t)F + 1, 0);
  for (int32_t i = 0; i < F; ++i) {
    int32_t f = L.fperm[i];
    L.frow[i + 1] = L.frow[i] + (int32_t)(L.rowptr[f + 1] - L.rowptr[f]);
  }
  L.edge_factor.resize(E);
  L.canon2v.resize(E);
  for (int32_t f = 0; f < F; ++f)
    for (int64_t e = L.rowptr[f]; e < L.rowptr[f + 1]; ++e) {
      L.edge_factor[e] = f;
      L.canon2v[e] = L.frow[L.finv[f]] + (int32_t)(e - L.rowptr[f]);
    }

  // variables: stable counting sort by degree
  std::vector<int32_t> vdeg((size_t)V, 0);
  L.nonunary.assign((size_t)V, 0);
  for (int64_t e = 0; e < E; ++e) {
    vdeg[L.edge_var[e]]++;
    int32_t f = L.edge_factor[e];
    if (L.rowptr[f + 1] - L.rowptr[f] > 1) L.nonunary[L.edge_var[e]]++;
  }
  int32_t maxv = 0;
  for (int32_t v = 0; v < V; ++v) maxv = std::max(maxv, vdeg[v]);
  L.max_vdeg = maxv;
  std::vector<int64_t> vb((size_t)maxv + 2, 0);
  for (int32_t v = 0; v < V; ++v) vb[vdeg[v] + 1]++;
  for (int32_t k = 0; k <= maxv; ++k) vb[k + 1] += vb[k];
  L.vperm.resize(V);
  L.vinv.resize(V);
  {
    std::vector<int64_t> fill(vb.begin(), vb.end() - 1);
    for (int32_t v = 0; v < V; ++v) {
      int32_t i = (int32_t)fill[vdeg[v]]++;
      L.vperm[i] = v;
      L.vinv[v] = i;
    }
  }
  L.vrow.assign((size_t)V + 1, 0);
  for (int32_t i = 0; i < V; ++i) L.vrow[i + 1] = L.vrow[i] + vdeg[L.vperm[i]];

  // ftov rows: canonical order within each variable == (factor, slot) order
  L.canon2f.resize(E);
  {
    std::vector<int32_t> fill((size_t)V, 0);
    for (int64_t e = 0; e < E; ++e) {
      int32_t v = L.edge_var[e];
      L.canon2f[e] = L.vrow[L.vinv[v]] + fill[v]++;
    }
  }
  // the reference's own ftov order: variables by id, rows in canonical order
  L.ref_ftov.resize(E);
  {
    std::vector<int64_t> start((size_t)V + 1, 0);
    for (int64_t e = 0; e < E; ++e) start[(size_t)L.edge_var[e] + 1]++;
    for (int32_t v = 0; v < V; ++v) start[v + 1] += start[v];
    for (int64_t e = 0; e < E; ++e) L.ref_ftov[(size_t)start[L.edge_var[e]]++] = (int32_t)e;
  }
  L.vtof2canon.resize(E);
  L.ftov2canon.resize(E);
  L.vtof_twin.resize(E);
  L.ftov_twin.resize(E);
  for (int64_t e = 0; e < E; ++e) {
    L.vtof2canon[L.canon2v[e]] = (int32_t)e;
    L.ftov2canon[L.canon2f[e]] = (int32_t)e;
    L.vtof_twin[L.canon2v[e]] = L.canon2f[e];
    int32_t f = L.edge_factor[e];
    bool unary = L.rowptr[f + 1] - L.rowptr[f] == 1;
    L.ftov_twin[L.canon2f[e]] = unary ? ~L.canon2v[e] : L.canon2v[e];
  }
  return HBP_OK;
}

void make_vt_item(const HostLayout &L, int32_t e, int32_t *q) {
  const int32_t vi = L.vinv[L.edge_var[e]];
  const int32_t row = L.vrow[vi];
  q[0] = L.canon2v[e];
  q[1] = row;
  q[2] = L.vrow[vi + 1] - row;
  q[3] = L.canon2f[e] - row;
}

void make_ft_item(const HostLayout &L, int32_t e, int32_t *q) {
  const int32_t f = L.edge_factor[e];
  const int32_t fi = L.finv[f];
  const int32_t slot = (int32_t)(e - L.rowptr[f]);
  q[0] = L.canon2f[e];
  q[1] = L.frow[fi];
  q[2] = (slot << 16) | (L.frow[fi + 1] - L.frow[fi]);
  q[3] = fi;
}

hbp_status build_plan(const HostLayout &L, int64_t k, const int64_t *s_off,
                      const int32_t *s_edges, const int64_t *t_off, const int32_t *t_edges,
                      PlanHost &P) {
  const int32_t V = L.V, F = L.F;
  const int64_t E = L.E;
  if (k < 0 || (k > 0 && (s_off[0] != 0 || t_off[0] != 0))) {
    set_error("bad batch offsets");
    return HBP_EINVAL;
  }
  for (int64_t b = 0; b < k; ++b) {
    if (s_off[b + 1] < s_off[b] || t_off[b + 1] < t_off[b]) {
      set_error("batch offsets must be nondecreasing");
      return HBP_EINVAL;
    }
  }
  const int64_t ns = k ? s_off[k] : 0, nt = k ? t_off[k] : 0;
  for (int64_t i = 0; i < ns; ++i)
    if (s_edges[i] < 0 || s_edges[i] >= E) {
      set_error("schedule edge out of range");
      return HBP_EINVAL;
    }
  for (int64_t i = 0; i < nt; ++i)
    if (t_edges[i] < 0 || t_edges[i] >= E) {
      set_error("schedule edge out of range");
      return HBP_EINVAL;
    }
  P.updates_per_iter = ns + nt;
  P.phases.clear();
  P.vnode.clear();
  P.fnode.clear();
  P.vt.clear();
  P.ft.clear();
  P.max_items = 0;

  std::vector<int64_t> stamp((size_t)E, -1);
  std::vector<int32_t> vcount((size_t)V, 0), fcount((size_t)F, 0);
  std::vector<int32_t> touched;
  std::vector<int32_t> items;

  auto add_vt = [&](int32_t e, std::vector<int32_t> &tg) {
    int32_t q[4];
    make_vt_item(L, e, q);
    tg.insert(tg.end(), q, q + 4);
  };
  auto add_ft = [&](int32_t e, std::vector<int32_t> &tg) {
    int32_t q[4];
    make_ft_item(L, e, q);
    tg.insert(tg.end(), q, q + 4);
  };
  // sort target quads by key
  auto sort_quads = [](std::vector<int32_t> &q, auto key) {
    size_t n = q.size() / 4;
    std::vector<int32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      return key(&q[4 * (size_t)a]) < key(&q[4 * (size_t)b]);
    });
    std::vector<int32_t> out(q.size());
    for (size_t i = 0; i < n; ++i) std::memcpy(&out[4 * i], &q[4 * (size_t)idx[i]], 16);
    q.swap(out);
  };

  const int64_t levels = std::max<int64_t>(k, 1);
  for (int64_t b = 0; b < levels; ++b) {
    // ---------------- variable side: vtof(t_b) (+ marginals in phase 0)
    {
      std::vector<int32_t> tg;
      touched.clear();
      if (b < k)
        for (int64_t i = t_off[b]; i < t_off[b + 1]; ++i) {
          int32_t e = t_edges[i];
          if (stamp[e] == (2 * b)) continue;  // duplicate target
          stamp[e] = (2 * b);
          int32_t v = L.edge_var[e];
          int32_t f = L.edge_factor[e];
          if (L.rowptr[f + 1] - L.rowptr[f] > 1) {
            if (vcount[v]++ == 0) touched.push_back(v);
          }
        }
      // full variables: every non-unary slot targeted
      std::vector<int32_t> full_ids;
      for (int32_t v : touched)
        if (vcount[v] == L.nonunary[v]) full_ids.push_back(L.vinv[v]);
      std::sort(full_ids.begin(), full_ids.end());
      // targets not covered by a full node
      if (b < k)
        for (int64_t i = t_off[b]; i < t_off[b + 1]; ++i) {
          int32_t e = t_edges[i];
          if (stamp[e] != (2 * b)) continue;
          stamp[e] = (2 * b) + 1;  // emit once
          int32_t v = L.edge_var[e];
          int32_t f = L.edge_factor[e];
          bool unary = L.rowptr[f + 1] - L.rowptr[f] == 1;
          bool covered = !unary && vcount[v] == L.nonunary[v];
          if (!covered) add_vt(e, tg);
        }
      for (int32_t v : touched) vcount[v] = 0;
      sort_quads(tg, [](const int32_t *q) { return ((int64_t)q[2] << 32) | (uint32_t)q[0]; });

      Phase ph{};
      ph.type = 0;
      ph.tgt_begin = (int32_t)(P.vt.size() / 4);
      P.vt.insert(P.vt.end(), tg.begin(), tg.end());
      ph.tgt_end = (int32_t)(P.vt.size() / 4);
      if (b == 0) {
        ph.node_flags = 1;  // marginal for every variable
        // variables with no non-unary slot have no vtof target: trivially full
        int64_t trivially = 0;
        for (int32_t v = 0; v < V; ++v) trivially += L.nonunary[v] == 0;
        if ((int64_t)full_ids.size() + trivially == V) {
          ph.node_list = 0;
          ph.node_begin = 0;
          ph.node_end = V;
          ph.node_flags |= 2;
        } else {
          // all variables, vtof bit on the full ones
          ph.node_list = 1;
          ph.node_begin = (int32_t)P.vnode.size();
          size_t j = 0;
          for (int32_t i = 0; i < V; ++i) {
            bool isfull = j < full_ids.size() && full_ids[j] == i;
            if (isfull) ++j;
            P.vnode.push_back(isfull ? (i | kVtofBit) : i);
          }
          ph.node_end = (int32_t)P.vnode.size();
        }
        // variables with no non-unary slot are trivially full; nothing differs
      } else {
        ph.node_list = 1;
        ph.node_flags = 0;
        ph.node_begin = (int32_t)P.vnode.size();
        for (int32_t i : full_ids) P.vnode.push_back(i | kVtofBit);
        ph.node_end = (int32_t)P.vnode.size();
      }
      int32_t n = (ph.node_end - ph.node_begin) + (ph.tgt_end - ph.tgt_begin);
      ph.grid = (b == 0) ? 1 : (n >= kCta0Threshold);
      P.max_items = std::max(P.max_items, n);
      if (b == 0 || n > 0) P.phases.push_back(ph);
    }
    if (b >= k) break;
    // ---------------- factor side: ftov(s_b)
    {
      std::vector<int32_t> tg;
      touched.clear();
      for (int64_t i = s_off[b]; i < s_off[b + 1]; ++i) {
        int32_t e = s_edges[i];
        if (stamp[e] == (2 * k + 2 * b)) continue;
        stamp[e] = (2 * k + 2 * b);
        int32_t f = L.edge_factor[e];
        if (fcount[f]++ == 0) touched.push_back(f);
      }
      std::vector<int32_t> full_ids;
      for (int32_t f : touched)
        if (fcount[f] == L.rowptr[f + 1] - L.rowptr[f]) full_ids.push_back(L.finv[f]);
      std::sort(full_ids.begin(), full_ids.end());
      for (int64_t i = s_off[b]; i < s_off[b + 1]; ++i) {
        int32_t e = s_edges[i];
        if (stamp[e] != (2 * k + 2 * b)) continue;
        stamp[e] = (2 * k + 2 * b) + 1;
        int32_t f = L.edge_factor[e];
        if (fcount[f] != L.rowptr[f + 1] - L.rowptr[f]) add_ft(e, tg);
      }
      for (int32_t f : touched) fcount[f] = 0;
      const int32_t orb = L.f_or_begin;
      // group by (kind, head/body), then degree
      sort_quads(tg, [orb](const int32_t *q) {
        int64_t kind = q[3] >= orb;
        int64_t head = (q[2] >> 16) == 0;
        return (kind << 40) | (head << 39) | ((int64_t)(q[2] & 0xffff) << 20);
      });
      Phase ph{};
      ph.type = 1;
      ph.tgt_begin = (int32_t)(P.ft.size() / 4);
      P.ft.insert(P.ft.end(), tg.begin(), tg.end());
      ph.tgt_end = (int32_t)(P.ft.size() / 4);
      if ((int64_t)full_ids.size() == F) {
        ph.node_list = 0;
        ph.node_begin = 0;
        ph.node_end = F;
      } else {
        ph.node_list = 1;
        ph.node_begin = (int32_t)P.fnode.size();
        P.fnode.insert(P.fnode.end(), full_ids.begin(), full_ids.end());
        ph.node_end = (int32_t)P.fnode.size();
      }
      int32_t n = (ph.node_end - ph.node_begin) + (ph.tgt_end - ph.tgt_begin);
      ph.grid = n >= kCta0Threshold;
      P.max_items = std::max(P.max_items, n);
      if (n > 0) P.phases.push_back(ph);
    }
  }
  return HBP_OK;
}

}  // namespace hbp
