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
// A phase is one data-parallel sweep between two barriers. Type 0 reads
// factor-to-variable messages (variable side: vtof updates, marginals);
// type 1 reads variable-to-factor messages (factor side: ftov updates).
// Work = node items (whole variable / whole factor, all outgoing messages
// at once) followed by target items (single edges).
struct Phase {
  int32_t type;        // 0 variable side, 1 factor side
  int32_t grid;        // 1: whole grid; 0: CTA 0 only (small level)
  int32_t node_list;   // 1: node ids come from the item list; 0: contiguous id range
  int32_t node_flags;  // bit0: marginal (phase 0 only), bit1: vtof for range-mode nodes
  int32_t node_begin, node_end;  // item-list range, or id range if node_list == 0
  int32_t tgt_begin, tgt_end;    // target-item range
};

// Node item (variable side, list mode): internal variable id | kVtofBit.
constexpr int32_t kVtofBit = 1 << 30;

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
  std::vector<int32_t> ftov_twin;    // internal ftov pos -> internal vtof pos (~pos if unary factor)
  std::vector<int32_t> edge_factor;  // canonical edge -> original factor
  std::vector<int32_t> ref_ftov;     // reference ftov position -> canonical edge (storage.py:61)
  std::vector<int32_t> nonunary;     // per original variable: # slots in non-unary factors
  int32_t f_or_begin = 0;            // internal factors >= this are OR
  int32_t max_fdeg = 0, max_vdeg = 0;
};

hbp_status build_layout(const hbp_graph_desc &g, HostLayout &L);

// Target-item encodings (4 x int32):
//   vtof target: {out vtof pos, ftov row start, row length, excluded index in row}
//   ftov target: {out ftov pos, vtof row start, (excluded slot << 16) | degree, internal factor}
void make_vt_item(const HostLayout &L, int32_t e, int32_t *q);
void make_ft_item(const HostLayout &L, int32_t e, int32_t *q);

struct PlanHost {
  std::vector<Phase> phases;
  std::vector<int32_t> vnode, fnode;   // node item lists
  std::vector<int32_t> vt, ft;         // target items, 4 int32 each
  int64_t updates_per_iter = 0;        // sum |s_i| + |t_i|
  int32_t max_items = 0;               // largest phase (work items)
};

hbp_status build_plan(const HostLayout &L, int64_t k, const int64_t *s_off,
                      const int32_t *s_edges, const int64_t *t_off, const int32_t *t_edges,
                      PlanHost &P);

}  // namespace hbp
