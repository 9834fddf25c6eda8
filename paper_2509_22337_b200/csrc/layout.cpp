// Host-side builders: the device message layout (MessageStore, storage.py:36-94)
// and the per-schedule level program (the pass compilation of engine.py:128-152,
// :357-410, :500-507, recast as slot work lists).
#include <algorithm>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace hbp {

void class_tables(HostLayout &L, const int64_t *vcnt, int64_t vhuge, const int64_t (*fcnt)[kClassMax + 2],
                  const int64_t *fhuge) {
  // variables: ascending degree
  int64_t n = 0, r = 0;
  for (int32_t d = 1; d <= kClassMax; ++d) {
    L.vcls_node[d] = (int32_t)n;
    L.vcls_row[d] = (int32_t)r;
    L.vcls_cnt[d] = (int32_t)vcnt[d];
    n += vcnt[d];
    r += d * vcnt[d];
  }
  L.vcls_node[kClassMax + 1] = (int32_t)n;
  L.vcls_row[kClassMax + 1] = (int32_t)r;
  L.vcls_cnt[kClassMax + 1] = (int32_t)vhuge;
  // factors: [light AND | light OR | heavy AND | heavy OR], ascending degree
  // inside each section, the huge ones ending the heavy sections
  n = r = 0;
  auto run = [&](int k, int32_t lo, int32_t hi) {
    for (int32_t d = lo; d <= hi; ++d) {
      L.fcls_node[k][d] = (int32_t)n;
      L.fcls_row[k][d] = (int32_t)r;
      L.fcls_cnt[k][d] = (int32_t)fcnt[k][d];
      n += fcnt[k][d];
      r += d * fcnt[k][d];
    }
  };
  auto huge = [&](int k) {
    L.fcls_node[k][kClassMax + 1] = (int32_t)n;
    L.fcls_row[k][kClassMax + 1] = (int32_t)r;
    L.fcls_cnt[k][kClassMax + 1] = (int32_t)fhuge[k];
    n += fcnt[k][kClassMax + 1];
    r += fhuge[k];
  };
  run(HBP_AND, 1, kNodeMax);
  run(HBP_OR, 1, kNodeMax);
  run(HBP_AND, kNodeMax + 1, kClassMax);
  huge(HBP_AND);
  run(HBP_OR, kNodeMax + 1, kClassMax);
  huge(HBP_OR);
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
  if (g.num_edges >= ((int64_t)1 << 30)) {
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
  L.n_unary = 0;
  for (int32_t f = 0; f < F; ++f) L.n_unary += L.rowptr[f + 1] - L.rowptr[f] == 1;

  // factors: stable counting sort by (heavy, kind, degree) -> warp-uniform role
  // and trip count across consecutive ids; heavy rows form the slot tail
  const int32_t nkeys = 4 * (maxdeg + 1);
  std::vector<int64_t> bucket((size_t)nkeys + 1, 0);
  auto fkey = [&](int32_t f) {
    const int32_t d = (int32_t)(L.rowptr[f + 1] - L.rowptr[f]);
    return ((d > kNodeMax) * 2 + (int32_t)L.kind[f]) * (maxdeg + 1) + d;
  };
  for (int32_t f = 0; f < F; ++f) bucket[fkey(f) + 1]++;
  for (int32_t k = 0; k < nkeys; ++k) bucket[k + 1] += bucket[k];
  L.f_or_light = (int32_t)bucket[1 * (maxdeg + 1)];
  L.f_heavy = (int32_t)bucket[2 * (maxdeg + 1)];
  L.f_or_heavy = (int32_t)bucket[3 * (maxdeg + 1)];
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
  L.fslot.resize(2 * E);
  for (int32_t f = 0; f < F; ++f) {
    const int32_t d = (int32_t)(L.rowptr[f + 1] - L.rowptr[f]);
    for (int64_t e = L.rowptr[f]; e < L.rowptr[f + 1]; ++e) {
      const int32_t j = (int32_t)(e - L.rowptr[f]);
      const int32_t p = L.frow[L.finv[f]] + j;
      L.edge_factor[e] = f;
      L.canon2v[e] = p;
      L.fslot[2 * (size_t)p] = L.finv[f];
      L.fslot[2 * (size_t)p + 1] = (d << 16) | j;
    }
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
  for (int32_t v = 0; v < V; ++v) {
    if (vdeg[v] == 0) {  // graph.py:114 rejects it too
      set_error("variable " + std::to_string(v) + " appears in no factor");
      return HBP_EINVAL;
    }
    maxv = std::max(maxv, vdeg[v]);
  }
  if (maxv > 65535) {
    set_error("variable degree above 65535");
    return HBP_EINVAL;
  }
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
  L.v_heavy = V;
  for (int32_t i = 0; i < V; ++i)
    if (L.vrow[i + 1] - L.vrow[i] > kNodeMax) {
      L.v_heavy = i;
      break;
    }

  // degree classes of the light nodes (computed rows in the PARALL kernels)
  auto classes = [](const std::vector<int32_t> &row, int32_t lo, int32_t hi, int32_t *node,
                    int32_t *rowstart) {
    // node[d] = first node in [lo, hi) of degree >= d (nodes sorted by degree)
    int32_t n = lo;
    for (int32_t d = 1; d <= kNodeMax + 1; ++d) {
      while (n < hi && row[n + 1] - row[n] < d) ++n;
      node[d] = d == kNodeMax + 1 ? hi : n;
      rowstart[d] = row[node[d]];
    }
    node[0] = lo;
    rowstart[0] = row[lo];
  };
  L.vrow_heavy = L.vrow[L.v_heavy];
  L.frow_heavy = L.frow[L.f_heavy];
  classes(L.vrow, 0, L.v_heavy, L.vc_node, L.vc_row);
  classes(L.frow, 0, L.f_or_light, L.fa_node, L.fa_row);
  classes(L.frow, L.f_or_light, L.f_heavy, L.fo_node, L.fo_row);
  {
    int64_t vcnt[kClassMax + 2] = {}, fcnt[2][kClassMax + 2] = {}, vhuge = 0, fhuge[2] = {0, 0};
    for (int32_t v = 0; v < V; ++v) {
      const int32_t d = vdeg[v];
      if (d > kClassMax) {
        vcnt[kClassMax + 1]++;
        vhuge += d;
      } else {
        vcnt[d]++;
      }
    }
    for (int32_t f = 0; f < F; ++f) {
      const int32_t d = (int32_t)(L.rowptr[f + 1] - L.rowptr[f]), k = L.kind[f];
      if (d > kClassMax) {
        fcnt[k][kClassMax + 1]++;
        fhuge[k] += d;
      } else {
        fcnt[k][d]++;
      }
    }
    class_tables(L, vcnt, vhuge, fcnt, fhuge);
  }

  // the reference's own ftov order: variables by id, rows in canonical order
  // (a stable counting sort, storage.py:61)
  L.ref_ftov.resize(E);
  std::vector<int64_t> vstart((size_t)V + 1, 0);
  {
    for (int64_t e = 0; e < E; ++e) vstart[(size_t)L.edge_var[e] + 1]++;
    for (int32_t v = 0; v < V; ++v) vstart[v + 1] += vstart[v];
    std::vector<int64_t> fill(vstart.begin(), vstart.end() - 1);
    for (int64_t e = 0; e < E; ++e) L.ref_ftov[(size_t)fill[L.edge_var[e]]++] = (int32_t)e;
  }
  // ftov rows: canonical order within each variable == (factor, slot) order,
  // which is the reference's product order (storage.py:59-61): variable v's
  // reference row, placed at its internal row
  L.canon2f.resize(E);
  L.vslot.resize(2 * E);
  for (int32_t v = 0; v < V; ++v) {
    const int32_t vi = L.vinv[v];
    const int32_t d = (int32_t)(vstart[v + 1] - vstart[v]);
    for (int32_t j = 0; j < d; ++j) {
      const int32_t e = L.ref_ftov[(size_t)vstart[v] + j];
      const int32_t q = L.vrow[vi] + j;
      L.canon2f[e] = q;
      L.vslot[2 * (size_t)q] = vi;
      L.vslot[2 * (size_t)q + 1] = (d << 16) | j;
    }
  }
  L.vtof2canon.resize(E);
  L.ftov2canon.resize(E);
  L.vtof_twin.resize(E);
  L.ftov_twin.resize(E);
  for (int64_t e = 0; e < E; ++e) {
    L.vtof2canon[L.canon2v[e]] = (int32_t)e;
    L.ftov2canon[L.canon2f[e]] = (int32_t)e;
    L.vtof_twin[L.canon2v[e]] = L.canon2f[e];
    const int32_t f = L.edge_factor[e];
    const bool unary = L.rowptr[f + 1] - L.rowptr[f] == 1;
    L.ftov_twin[L.canon2f[e]] = (uint32_t)L.canon2v[e] | (unary ? kUnaryBit : 0u);
  }
  L.host_ready = true;
  return HBP_OK;
}

void parall_plan(const HostLayout &L, int64_t ns, int64_t nt, PlanHost &P,
                 int32_t small_threshold) {
  P.updates_per_iter = ns + nt;
  P.phases.clear();
  P.items.clear();
  Phase v{};
  v.type = 0;
  v.grid = 1;  // phase 0 carries the convergence test
  v.list = 2;
  v.marg = 1;
  v.begin = 0;
  v.end = L.v_heavy;
  v.sbegin = L.vrow_heavy;
  v.send = (int32_t)L.E;
  Phase f{};
  f.type = 1;
  f.list = 2;
  f.begin = 0;
  f.end = L.f_heavy;
  f.sbegin = L.frow_heavy;
  f.send = (int32_t)L.E;
  const int32_t nv = L.v_heavy + (v.send - v.sbegin), nf = L.f_heavy + (f.send - f.sbegin);
  f.grid = nf >= small_threshold;  // smaller phases run on cluster 0 only
  P.phases.push_back(v);
  P.phases.push_back(f);
  P.phase_batch.assign(2, 0);
  P.max_items = std::max(nv, nf);
}

hbp_status build_plan(const HostLayout &L, int64_t k, const int64_t *s_off,
                      const int32_t *s_edges, const int64_t *t_off, const int32_t *t_edges,
                      PlanHost &P, int32_t small_threshold, int grouping, bool fuse) {
  const int32_t V = L.V;
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
  P.items.clear();
  P.phase_batch.clear();
  P.max_items = 0;
  P.fitems.clear();
  P.n_fused = 0;

  std::vector<int64_t> stamp((size_t)E, -1);
  std::vector<int32_t> slots;

  // the non-unary slot set: what a PARALL variable-side phase writes
  int64_t nonunary_total = 0;
  for (int32_t v = 0; v < V; ++v) nonunary_total += L.nonunary[v];

  int32_t cur_batch = 0;
  auto push_phase = [&](Phase ph, int32_t n) {
    ph.grid = n >= small_threshold;  // smaller phases run on cluster 0 only
    P.max_items = std::max(P.max_items, n);
    P.phases.push_back(ph);
    P.phase_batch.push_back(cur_batch);
  };

  // PARALL fast path: one batch holding every edge once and every slot of a
  // non-unary factor once compiles to the two whole-graph phases directly
  if (grouping == 2 && k == 1 && ns == E && nt == nonunary_total) {
    std::vector<uint8_t> seen((size_t)E, 0);
    bool ok = true;
    for (int64_t i = 0; i < ns && ok; ++i) {
      uint8_t &m = seen[s_edges[i]];
      ok = !(m & 1);
      m |= 1;
    }
    for (int64_t i = 0; i < nt && ok; ++i) {
      const int32_t e = t_edges[i];
      const int32_t f = L.edge_factor[e];
      uint8_t &m = seen[e];
      ok = !(m & 2) && L.rowptr[f + 1] - L.rowptr[f] > 1;
      m |= 2;
    }
    if (ok) {
      parall_plan(L, ns, nt, P, small_threshold);
      return HBP_OK;
    }
  }

  // Level fusion. A level b >= 1 whose factor-side writes are never read by
  // its own variable side -- no ftov message s_b writes into variable u's row
  // is read by a t_b target (a', u) of ANOTHER factor a' -- runs as ONE
  // phase: a thread owns a factor of the level, computes its t_b
  // vtof messages (reading the variables' rows), then its s_b ftov messages
  // from its own row. Every read then sees exactly the state the two-phase
  // order gives it (engine.py:566-570), so the results are the same bits.
  // (Level 0 is never fused: its variable side carries the marginals, which
  // read every variable's full row.)
  std::vector<int64_t> wstamp, istamp;
  std::vector<int32_t> writer, item_of;
  if (fuse && grouping == 2) {
    wstamp.assign((size_t)V, -1);
    writer.assign((size_t)V, 0);
    istamp.assign((size_t)L.F, -1);
    item_of.assign((size_t)L.F, 0);
  }
  auto fusable = [&](int64_t b) -> bool {
    if (!fuse || grouping != 2 || b == 0 || b >= k) return false;
    for (int64_t i = s_off[b]; i < s_off[b + 1]; ++i) {
      const int32_t e = s_edges[i];
      const int32_t u = L.edge_var[e], a = L.edge_factor[e];
      if (L.rowptr[a + 1] - L.rowptr[a] > kFuseMaxDeg) return false;
      if (wstamp[u] != b) {
        wstamp[u] = b;
        writer[u] = a;
      } else if (writer[u] != a) {
        writer[u] = -1;  // two writers: any reader of u conflicts
      }
    }
    for (int64_t i = t_off[b]; i < t_off[b + 1]; ++i) {
      const int32_t e = t_edges[i];
      const int32_t u = L.edge_var[e], a = L.edge_factor[e];
      if (L.rowptr[a + 1] - L.rowptr[a] > kFuseMaxDeg) return false;
      if (wstamp[u] == b && writer[u] != a) return false;
    }
    return true;
  };
  auto emit_fused = [&](int64_t b) {
    std::vector<int32_t> order;  // internal factors of the level
    std::vector<int32_t> tm, sm;
    auto touch = [&](int32_t e, bool is_s) {
      const int32_t p = L.canon2v[e];
      const int32_t fi = L.fslot[2 * (size_t)p], kk = L.fslot[2 * (size_t)p + 1] & 0xffff;
      if (istamp[fi] != b) {
        istamp[fi] = b;
        item_of[fi] = (int32_t)order.size();
        order.push_back(fi);
        tm.push_back(0);
        sm.push_back(0);
      }
      (is_s ? sm : tm)[item_of[fi]] |= 1 << kk;
    };
    for (int64_t i = t_off[b]; i < t_off[b + 1]; ++i) touch(t_edges[i], false);
    for (int64_t i = s_off[b]; i < s_off[b + 1]; ++i) touch(s_edges[i], true);
    std::vector<int32_t> idx(order.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int32_t)i;
    // ascending internal factor == (kind, degree) order: warp-uniform role
    std::sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) { return order[x] < order[y]; });
    Phase ph{};
    ph.type = 2;
    ph.list = 3;
    ph.begin = (int32_t)(P.fitems.size() / 8);
    // one lane per row slot; a factor's lanes never straddle a warp
    int32_t lane = 0;
    auto pad_to = [&](int32_t upto) {
      for (; lane < upto; ++lane)
        for (int c = 0; c < 8; ++c) P.fitems.push_back(c == 2 ? (lane << 16) : 0);
    };
    for (int32_t i : idx) {
      const int32_t fi = order[i], r = L.frow[fi], d = L.frow[fi + 1] - r;
      if (lane + d > 32) {
        pad_to(32);
        lane = 0;
      }
      const int32_t base = lane;
      for (int32_t kk = 0; kk < d; ++kk, ++lane) {
        const int32_t q = L.vtof_twin[r + kk];
        const int32_t w = L.vslot[2 * (size_t)q + 1];
        P.fitems.push_back(fi);
        P.fitems.push_back(r);
        P.fitems.push_back(d | kk << 8 | base << 16);
        P.fitems.push_back(tm[i] | sm[i] << 12);
        P.fitems.push_back(q - (w & 0xffff));
        P.fitems.push_back(w);
        P.fitems.push_back(L.vslot[2 * (size_t)q]);
        P.fitems.push_back(q);
      }
      if (lane == 32) lane = 0;
    }
    if (lane) pad_to(32);
    ph.end = (int32_t)(P.fitems.size() / 8);
    push_phase(ph, ph.end - ph.begin);
    ++P.n_fused;
  };

  const int64_t levels = std::max<int64_t>(k, 1);
  for (int64_t b = 0; b < levels; ++b) {
    cur_batch = (int32_t)b;
    if (fusable(b)) {
      emit_fused(b);
      continue;
    }
    // ---------------- variable side: vtof(t_b) (+ marginals in phase 0)
    {
      slots.clear();
      int64_t n_nonunary = 0;
      bool has_unary = false;
      if (b < k)
        for (int64_t i = t_off[b]; i < t_off[b + 1]; ++i) {
          const int32_t e = t_edges[i];
          if (stamp[e] == 2 * b) continue;  // duplicate target: computed once
          stamp[e] = 2 * b;
          slots.push_back(L.canon2f[e]);
          const int32_t f = L.edge_factor[e];
          if (L.rowptr[f + 1] - L.rowptr[f] > 1)
            ++n_nonunary;
          else
            has_unary = true;
        }
      Phase ph{};
      ph.type = 0;
      ph.marg = b == 0;
      if (grouping == 2 && b == 0 && n_nonunary == nonunary_total && !has_unary) {
        // PARALL: every non-unary vtof slot + every marginal == every variable
        // node in full
        ph.list = 2;
        ph.begin = 0;
        ph.end = L.v_heavy;
        ph.sbegin = L.vrow[L.v_heavy];
        ph.send = (int32_t)E;
        push_phase(ph, L.v_heavy + (ph.send - ph.sbegin));
      } else {
        std::vector<int32_t> items;
        items.reserve(slots.size() + (b == 0 ? V : 0));
        for (int32_t q : slots) items.push_back(q | kWriteBit);
        if (b == 0) {
          // row-start slots that are not targets still owe their marginal
          std::vector<char> tgt((size_t)V, 0);
          for (int32_t q : slots)
            if ((L.vslot[2 * (size_t)q + 1] & 0xffff) == 0) tgt[L.vslot[2 * (size_t)q]] = 1;
          for (int32_t vi = 0; vi < V; ++vi)
            if (!tgt[vi]) items.push_back(L.vrow[vi]);
        }
        // ascending slot order == (degree, variable) order: warp-uniform trip counts
        if (grouping >= 1)
          std::sort(items.begin(), items.end(), [](int32_t a, int32_t c) {
            return (a & (kWriteBit - 1)) < (c & (kWriteBit - 1));
          });
        ph.list = 1;
        ph.begin = (int32_t)P.items.size();
        P.items.insert(P.items.end(), items.begin(), items.end());
        ph.end = (int32_t)P.items.size();
        const int32_t n = ph.end - ph.begin;
        if (b == 0 || n > 0) push_phase(ph, n);
      }
      if (b == 0) P.phases.back().grid = 1;  // phase 0 carries the convergence test
    }
    if (b >= k) break;
    // ---------------- factor side: ftov(s_b)
    {
      slots.clear();
      for (int64_t i = s_off[b]; i < s_off[b + 1]; ++i) {
        const int32_t e = s_edges[i];
        if (stamp[e] == 2 * b + 1) continue;
        stamp[e] = 2 * b + 1;
        slots.push_back(L.canon2v[e]);
      }
      Phase ph{};
      ph.type = 1;
      if (grouping == 2 && (int64_t)slots.size() == E) {
        ph.list = 2;  // every factor node in full
        ph.begin = 0;
        ph.end = L.f_heavy;
        ph.sbegin = L.frow[L.f_heavy];
        ph.send = (int32_t)E;
        push_phase(ph, L.f_heavy + (ph.send - ph.sbegin));
      } else if (!slots.empty()) {
        // ascending vtof slot == (kind, degree, factor) order: warp-uniform role
        if (grouping >= 1) std::sort(slots.begin(), slots.end());
        ph.list = 1;
        ph.begin = (int32_t)P.items.size();
        P.items.insert(P.items.end(), slots.begin(), slots.end());
        ph.end = (int32_t)P.items.size();
        push_phase(ph, ph.end - ph.begin);
      }
    }
  }
  // runs of consecutive small item phases (fused levels, list-mode vtof /
  // ftov phases; never phase 0): the first phase of a run carries the run's
  // end in sbegin (the kernel executes the run in a tight loop)
  auto small_item = [&](size_t i) {
    const Phase &ph = P.phases[i];
    return i > 0 && !ph.grid && (ph.list == 1 || ph.list == 3);
  };
  for (size_t i = P.phases.size(); i-- > 0;) {
    Phase &ph = P.phases[i];
    if (!small_item(i)) continue;
    const bool next_small = i + 1 < P.phases.size() && small_item(i + 1);
    ph.sbegin = next_small ? P.phases[i + 1].sbegin : (int32_t)(i + 1);
  }
  return HBP_OK;
}

}  // namespace hbp
