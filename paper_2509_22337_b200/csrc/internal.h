// Internal declarations shared by the host-side builders (layout, plan,
// compiler) and the CUDA executor. Not part of the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hornbp_gpu.h"

namespace hbp {

void set_error(const std::string &msg);

// ---- compiled schedule (host) --------------------------------------------------------
struct Schedule {
  std::vector<int64_t> s_off, t_off;
  std::vector<int32_t> s_edges, t_edges;
};

bool toposort(int64_t n, int64_t m, const int32_t *before, const int32_t *after,
              std::vector<int32_t> &order, int64_t *cycle_edge);
hbp_status compile(const hbp_graph_desc &g, int64_t m, const int32_t *before,
                   const int32_t *after, const int32_t *rank, Schedule &out,
                   int64_t *cycle_edge);

// ---- device-side plan records --------------------------------------------------------
// A phase is one data-parallel sweep between two barriers. Type 0 is the
// variable side (reads factor-to-variable messages; writes variable-to-factor
// messages and, in phase 0, the marginals); type 1 is the factor side.
// Work items are message SLOTS, one thread each: an ftov slot for type 0
// (the thread writes the vtof message of the same edge), a vtof slot for
// type 1 (it writes the ftov message of the same edge). Range-mode phases
// cover every slot [begin, end); list-mode phases read slot ids from the
// item array (levelled schedules).
struct Phase {
  int32_t type;   // 0 variable side, 1 factor side, 2 fused level (list == 3)
  int32_t grid;   // 1: whole grid; 0: cluster 0 only (small level)
  int32_t list;   // 0: slots [begin, end); 1: slot ids from the item list;
                  // 2: whole nodes [begin, end) (variables for type 0, factors for
                  //    type 1), every outgoing message of a node from one row read;
                  // 3: fused level items [begin, end) of PlanHost::fitems (type 2)
  int32_t marg;   // 1: row-start slots also produce the marginal (phase 0)
  int32_t begin, end;     // nodes (list == 2) or slots / items
  int32_t sbegin, send;   // list == 2: slots of the heavy nodes, one thread per slot
};

// Nodes up to this degree are processed whole by one thread (row in
// registers); the rows of larger nodes are processed one slot per thread.
#ifndef HBP_NODE_MAX
#define HBP_NODE_MAX 4
#endif
constexpr int32_t kNodeMax = HBP_NODE_MAX;
// Whole-node phases process nodes of degree kNodeMax < d <= kClassMax as lane
// groups (one lane per row slot, a node's lanes in one warp) and larger ones
// one slot per thread.
constexpr int32_t kClassMax = 32;

// List items: slot id | kWriteBit (type 0 only: also write the vtof message;
// items without it exist only to produce a marginal).
constexpr int32_t kWriteBit = 1 << 30;
// ftov_twin high bit: the edge belongs to a unary factor, whose vtof message
// is never a PARALL target (schedule.py:303-312 skips it).
constexpr uint32_t kUnaryBit = 1u << 31;

// ---- graph layout ----------------------------------------------------------------------
// Internal order: factors sorted by (kind, degree), variables by degree
// (both stable), so a contiguous id range is warp-uniform in control flow
// and trip count. vtof rows are factor rows in internal factor order (slot
// order inside a row); ftov rows are variable rows in internal variable
// order, each row kept in the reference's (factor, slot) order -- that order
// is the product order and therefore part of the bitwise contract.
struct HostLayout {
  int32_t V = 0, F = 0;
  int64_t E = 0;
  // canonical copies
  std::vector<int64_t> rowptr;
  std::vector<int32_t> edge_var;
  std::vector<int8_t> kind;
  std::vector<double> p1, p2;
  // permutations
  std::vector<int32_t> fperm, finv;  // internal factor -> original, inverse
  std::vector<int32_t> vperm, vinv;  // internal variable -> original, inverse
  std::vector<int32_t> frow, vrow;   // internal row starts [F+1], [V+1]
  std::vector<int32_t> canon2v;      // canonical edge -> internal vtof position
  std::vector<int32_t> canon2f;      // canonical edge -> internal ftov position
  std::vector<int32_t> vtof2canon;   // inverse of canon2v
  std::vector<int32_t> ftov2canon;   // inverse of canon2f
  std::vector<int32_t> vtof_twin;    // internal vtof pos -> internal ftov pos
  std::vector<uint32_t> ftov_twin;   // internal ftov pos -> internal vtof pos | kUnaryBit
  std::vector<int32_t> vslot;        // per internal ftov pos: {internal var, (deg << 16) | index}
  std::vector<int32_t> fslot;        // per internal vtof pos: {internal factor, (deg << 16) | index}
  std::vector<int32_t> edge_factor;  // canonical edge -> original factor
  std::vector<int32_t> ref_ftov;     // reference ftov position -> canonical edge (storage.py:61)
  std::vector<int32_t> nonunary;     // per original variable: # slots in non-unary factors
  // internal factor order: (heavy, kind, degree) with heavy = degree > kNodeMax:
  // [light AND | light OR | heavy AND | heavy OR]
  int32_t f_or_light = 0, f_heavy = 0, f_or_heavy = 0;
  int32_t v_heavy = 0;  // internal variables >= this have degree > kNodeMax
  int32_t vrow_heavy = 0, frow_heavy = 0;  // vrow[v_heavy], frow[f_heavy]
  int64_t n_unary = 0;                     // factors of degree 1
  // false: only the scalars above are set (the device built the arrays);
  // ensure_host_layout fills the vectors on first host-side use
  bool host_ready = false;
  bool factor_is_or(int32_t fi) const {
    return (fi >= f_or_light && fi < f_heavy) || fi >= f_or_heavy;
  }
  int32_t max_fdeg = 0, max_vdeg = 0;
  // degree classes of the light nodes: [x_node[d], x_node[d+1]) have degree d
  // (d = 1..kNodeMax), first row x_row[d]; x_node[kNodeMax + 1] ends the light range
  int32_t vc_node[kNodeMax + 2] = {}, vc_row[kNodeMax + 2] = {};
  int32_t fa_node[kNodeMax + 2] = {}, fa_row[kNodeMax + 2] = {};  // light AND factors
  int32_t fo_node[kNodeMax + 2] = {}, fo_row[kNodeMax + 2] = {};  // light OR factors
  // every degree class d = 1..kClassMax of the variables and of the AND / OR
  // factors: first node, first row, node count (the nodes of a class are
  // contiguous in internal order); index kClassMax + 1 is the "huge" rest
  // (degree > kClassMax): first node, first row, SLOT count
  int32_t vcls_node[kClassMax + 2] = {}, vcls_row[kClassMax + 2] = {}, vcls_cnt[kClassMax + 2] = {};
  int32_t fcls_node[2][kClassMax + 2] = {}, fcls_row[2][kClassMax + 2] = {},
          fcls_cnt[2][kClassMax + 2] = {};
};

// class tables from the per-class counts: vcnt[d] variables and fcnt[k][d]
// kind-k factors of degree d (d <= kClassMax), and the slots of the huge
// nodes (vhuge, fhuge[k]) -- the internal order is the sort order of
// build_layout / the device layout build
void class_tables(HostLayout &L, const int64_t *vcnt, int64_t vhuge, const int64_t (*fcnt)[kClassMax + 2],
                  const int64_t *fhuge);

hbp_status build_layout(const hbp_graph_desc &g, HostLayout &L);

struct PlanHost {
  std::vector<Phase> phases;
  std::vector<int32_t> items;          // list-mode slot items (both sides)
  int64_t updates_per_iter = 0;        // sum |s_i| + |t_i|
  int32_t max_items = 0;               // largest phase (work items)
  std::vector<int32_t> phase_batch;    // batch index of each phase (underflow attribution)
  // fused levels (type 2): one lane per row slot of every factor of the level,
  // a factor's lanes contiguous inside one warp (padding lanes have d = 0).
  // Per lane two int4: {internal factor, vtof row start,
  // d | slot << 8 | first lane of the factor << 16, tmask | smask << 12}
  // (tmask / smask: the row slots whose vtof (t_b) / ftov (s_b) message the
  // level computes) and the slot's record {variable's ftov row start,
  // (variable degree << 16) | index in that row, internal variable, ftov slot}
  std::vector<int32_t> fitems;
  int32_t n_fused = 0;                 // fused levels in the plan
};

// factors up to this degree can be part of a fused level (12-bit slot masks,
// at most one warp per factor)
constexpr int32_t kFuseMaxDeg = 12;

// the two whole-graph phases of a PARALL schedule (every edge once on the
// factor side, every non-unary slot once on the variable side), from the
// layout's scalars alone
void parall_plan(const HostLayout &L, int64_t ns, int64_t nt, PlanHost &P,
                 int32_t small_threshold);

// grouping (the A/B of the paper's message grouping):
// 2 = whole degree-sorted nodes per thread where a phase covers every node
// (default), 1 = one slot per thread in slot (= degree-sorted) order,
// 0 = one slot per thread in the schedule's own (EdgeId) order.
hbp_status build_plan(const HostLayout &L, int64_t k, const int64_t *s_off,
                      const int32_t *s_edges, const int64_t *t_off, const int32_t *t_edges,
                      PlanHost &P, int32_t small_threshold, int grouping = 2,
                      bool fuse = true);

}  // namespace hbp
