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
// Work decomposition: one thread per output message. Rows are laid out
// degree-sorted (variables) and (kind, degree)-sorted (factors), so the 32
// lanes of a warp read neighbouring rows of equal length: uniform trip count
// and role, coalesced row loads shared through L1, and every lane multiplies
// its row left to right in slot order (the reference's _product_scan order,
// engine.py:168-183) -- bitwise-identical products. A 2-int slot word
// {node, (degree << 16) | index-in-row} is the only per-message index.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "device.h"
#include "internal.h"
#include "lbp_kernels.cuh"

namespace hbp {

using namespace dev;

// CTA sizes (one CTA per SM): levelled plans 768 threads (80 registers); the
// two whole-node phases of a PARALL plan 640 threads (96 registers, no
// spills) -- measured on B200 (C4-PARALL: 640 0.312 ms, 576 0.334, 704 0.320,
// 768 0.326, 1024 0.324; levelled C3: 768 10.1 ms, 640 12.2 ms)
#ifndef HBP_KTHREADS
#define HBP_KTHREADS 768
#endif
#ifndef HBP_PARALL_THREADS
#define HBP_PARALL_THREADS 640
#endif
constexpr int kThreads = HBP_KTHREADS;
constexpr int kParallThreads = HBP_PARALL_THREADS;
#ifndef HBP_FUSED_THREADS
#define HBP_FUSED_THREADS 768
#endif
constexpr int kFusedThreads = HBP_FUSED_THREADS;  // plans with fused levels
// PARALL as one phase per iteration (lbp_pslot): 896 threads (72 registers),
// variable rows up to 4 slots in registers -- measured on B200 (C4-PARALL:
// 896 0.279 ms, 768 0.292, 1024 0.281; rows of 2 0.287, 6 0.283)
#ifndef HBP_PSLOT_THREADS
#define HBP_PSLOT_THREADS 896
#endif
constexpr int kPslotThreads = HBP_PSLOT_THREADS;
// slot items (levelled phases, the single-pass API): rows loaded branch-free
// in their length and the factor kind selected by operands, so one warp's
// lanes share one round trip -- measured on B200: C2 8.92 -> 5.44 ms, C3
// 8.70 -> 7.33 ms (HBP_ITEM_PRED=0: the per-length / per-kind switch, A/B)
#ifndef HBP_ITEM_PRED
#define HBP_ITEM_PRED 1
#endif
constexpr int kItemRow = 6;
// small phases' list items carry their slot word and twin in a parallel
// int4 array (plan time), loaded beside the item: C2 5.53 -> 5.34 ms, C3
// 7.34 -> 7.19 ms (HBP_ITEM_WORDS=0: item -> slot word chain, A/B)
#ifndef HBP_ITEM_WORDS
#define HBP_ITEM_WORDS 1
#endif
// fused lanes: the factor kind selects operands instead of branching (no
// divergence between a warp's AND and OR factors; the same operations):
// C4-SEQFIX 18.14 -> 17.62 ms (HBP_FUSED_SEL=0: the branches, A/B)
#ifndef HBP_FUSED_SEL
#define HBP_FUSED_SEL 1
#endif
#ifndef HBP_PSLOT_ROW
#define HBP_PSLOT_ROW 4
#endif
constexpr int kPslotRow = HBP_PSLOT_ROW;  // lbp_pslot: variable row slots held in registers
constexpr int kPslotPairs = (kPslotRow + 2) / 2;  // 32-byte pairs covering a row at any parity
#ifndef HBP_GROUP_MIN
#define HBP_GROUP_MIN (HBP_NODE_MAX + 1)
#endif
static_assert(HBP_GROUP_MIN >= 2 && HBP_GROUP_MIN <= HBP_NODE_MAX + 1, "lane-group threshold");
constexpr int kTraceIters = 4;  // HBP_TRACE=1: timestamps for iterations 2..5
constexpr int kPhaseCache = 1024;  // phase descriptors staged in shared memory (32 KB)
constexpr int kChunkTrace = 16384;  // HBP_TRACE=1: per-chunk ns of iteration 3, PARALL phases 0/1

struct Ctrl {
  unsigned int bar;  // grid barrier arrivals (monotonic)
  int iterations;
  int converged;
  int stop;          // 1 converged, 2 max_iterations, 3 time limit, 4 underflow
  unsigned long long t0;
  unsigned long long last_delta;  // delta bits of the stopping iteration
};

// A chunk class of a whole-node phase: chunks [chunk_begin, next class's)
// cover the class's nodes [node_begin, node_end) (rows from row_begin) --
// style 0: one node per lane (degree <= kNodeMax), style 1: lane groups (one
// lane per row slot, 32 / d nodes per chunk, degree <= kClassMax), style 2:
// one slot per lane over [row_begin, node_end) (huge nodes; node_end holds
// the slot end there).
struct ChunkClass {
  int chunk_begin, node_begin, node_end, row_begin;
  int info;  // degree | kind << 16 | style << 20
  int grp;   // lane groups: nodes per chunk | ceil(2^16 / degree) << 8 (lane / d as a multiply)
};
constexpr int kMaxVarClasses = kClassMax + 2;
constexpr int kMaxFacClasses = 2 * (kClassMax + 2);

struct KParams {
  // layout
  const int *vrow;            // [V+1] internal variable rows in the ftov buffer
  const int *frow;            // [F+1] internal factor rows in the vtof buffer
  const int2 *vslot;          // per ftov slot
  const int2 *fslot;          // per vtof slot
  const int *vtof_twin;       // vtof slot -> ftov slot
  const unsigned *ftov_twin;  // ftov slot -> vtof slot | kUnaryBit
  const double2 *fpar;        // per internal factor (p1, p2)
  const int *vorig;           // internal variable -> original id
  int V, F, E, f_or_light, f_heavy, f_or_heavy;
  double2 *vtof, *ftov, *marg;
  double *p0;                 // [V] P(X=0) of the last marginal pass (prev P1 = 1 - p0)
  // evidence codes per internal variable (null: none): bit0 observed false,
  // bit1 observed true -- the clamp factors of clamp_evidence, multiplied in
  // after the row product (their slot is last in the row) for every marginal
  // and, from iteration 2 on, for every variable-to-factor message
  const unsigned char *ev;
  // whole-node phases: the chunk classes of each side (base_params), in
  // processing order (dearest first); a class's chunks are warp-uniform in
  // role, degree and style
  ChunkClass vcc[kMaxVarClasses], fcc[kMaxFacClasses];
  int nvcc, nfcc;
  int vchunks, fchunks, fchunks_nounary;  // factor chunks without the unary classes (last)
  // plan
  const Phase *phases;
  int nphases;
  const int *items;
  const int4 *fitems;  // fused levels: two int4 per lane (layout.cpp emit_fused)
  const int4 *iw;      // list items: {slot word x, slot word y, twin, 0} (small phases)
  // control
  Ctrl *ctrl;
  unsigned long long *delta_bits;  // [max_it + 2]
  int *uf_msg;                     // [max_it + 2] bit0 vtof, bit1 ftov
  int *uf_marg;                    // [max_it + 2]
  int *uf_mwhere;                  // [max_it + 2] smallest underflowing variable
  unsigned long long *uf_where;    // [max_it + 2] (phase<<33 | kind<<32 | slot)
  int *tflag;                      // [max_it + 2]
  double2 *hist;                   // [hist_iters][V] or null
  int hist_iters;                  // iterations the history buffer holds
  unsigned long long *trace;       // debug: [kTraceIters][nphases][grid][2] or null
  int csize;                       // CTAs that run the small levels (1: CTA 0 alone)
  int max_it;
  int normalize;
  double tol;
  long long time_limit_ns;
  // underflow attribution re-run: stop at the START of phase halt_phase of
  // iteration halt_it (0: run normally), leaving that phase's inputs intact
  int halt_it, halt_phase;
  const int *canon2v;         // canonical edge -> internal vtof slot (attribution)
  // lbp_pslot: 32 lane records per slot chunk {variable row start, variable,
  // factor, variable degree | index in the row << 8 | slot << 16 | valid << 24},
  // per chunk degree | kind << 8 | longest row << 16 (layout_dev.cu
  // build_pslot_device); the
  // second ftov and P0 buffers (iteration it writes buffer it & 1)
  const int4 *srec;
  const int *sinfo;
  double2 *ftov_alt;
  double *p0_alt;
};

// --------------------------------------------------------------------------------------
// grid barrier (arrive / wait on a monotonic counter)

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sync point: arrivers add 1 to a monotonic arrival counter (release, no
// return value), waiters poll it (acquire) until it reaches the point's
// cumulative target, which every CTA tracks identically. Measured on B200
// (tools/barrier_bench.cu, 148 CTAs x 1024 threads): 1.27 us per barrier; a
// last-arriver flag costs 1.78 us (the arrival must round-trip).
struct Sync {
  unsigned target = 0;
};

__device__ __forceinline__ void sync_point(Ctrl *c, Sync &s, unsigned arrivals, bool arrive,
                                           bool wait) {
  __syncthreads();
  s.target += arrivals;
  if (threadIdx.x == 0) {
    if (arrive) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&c->bar) : "memory");
    if (wait)
      while (ld_acquire(&c->bar) < s.target) {
      }
  }
  __syncthreads();
}

// the per-node kernels with the run-time normalise flag (namespace n0; n1
// below fixes it on). Neither is hbp itself, so argument-dependent lookup on
// KParams cannot mix the two copies.
namespace n0 {
#define HBP_NORMALIZE(P) ((P).normalize)
#include "lbp_node.inc"
#undef HBP_NORMALIZE
}  // namespace n0
using namespace n0;



// --------------------------------------------------------------------------------------
// fused level (layout.cpp emit_fused): one lane per row slot of the level's
// factors, a factor's lanes inside one warp. Lane k of factor f computes the
// vtof message of slot k (t_b) from its variable's row, the factor's lanes
// exchange their row by warp shuffles, and lane k then computes the ftov
// message of slot k (s_b) from the row. The plan admits a level only when no
// other factor of the level writes into a row a lane reads, so the values of
// the two-phase order are read (engine.py:566-570).

// The lanes of a warp belong to different variables (rows of mixed length),
// so the row is loaded branch-free: kFuseRow predicated loads issued
// together, one memory round trip for every lane (a switch on the length
// would serialise one round trip per distinct length). Longer rows finish
// in a loop.
constexpr int kFuseRow = 6;

// one lane: h = {factor, row start, d | slot << 8 | group lane << 16,
// tmask | smask << 12}, rc = the slot's record {variable row start,
// (variable degree << 16) | own index, internal variable, ftov slot}.
// Called by all 32 lanes of a warp.
// factor output of one slot with the kind a run-time flag: the operands of
// head_message / body_message (lbp_kernels.cuh) selected, not the code
// duplicated -- the same operations on the same values, so the same bits.
// head: diff = (a - b) prod2, o1 = b prod1 + diff, o0 = (1 - b) prod1 - diff
// with (a, b) = (p1, p2) for AND, (p2, p1) for OR; body: diff = (a - b) prod2,
// s = prod1 + diff, with (a, b) = (p2, p1) and (o0, o1) = (prod1, s) for
// AND, (p1, p2) and (s, prod1) for OR.
__device__ __forceinline__ void factor_out(bool is_or, bool head, double p1, double p2,
                                           double prod1, double prod2, double &o0, double &o1) {
  const bool first = is_or != head;  // a = p1
  const double a = first ? p1 : p2, b = first ? p2 : p1;
  const double diff = mul(sub(a, b), prod2);
  if (head) {
    o1 = add(mul(b, prod1), diff);
    o0 = sub(mul(sub(1.0, b), prod1), diff);
  } else {
    const double s = add(prod1, diff);
    o0 = is_or ? s : prod1;
    o1 = is_or ? prod1 : s;
  }
}

__device__ __forceinline__ void fused_lane(const KParams &P, int4 h, int4 rc, int it, int phase,
                                           unsigned &ufkey) {
  const int d = h.z & 0xff, k = (h.z >> 8) & 0xff, base = h.z >> 16;
  const int tmask = h.w & 0xfff, smask = (h.w >> 12) & 0xfff;
  const bool tgt = d && ((tmask >> k) & 1);
  const int dv = tgt ? rc.y >> 16 : 0, j = rc.y & 0xffff;
  // every load of the lane in one round trip: its variable's row (t_b
  // target) or its current vtof message, the evidence code, the parameters
  double2 x[kFuseRow];
#pragma unroll
  for (int i = 0; i < kFuseRow; ++i)
    x[i] = i < dv ? P.ftov[rc.x + i] : make_double2(1.0, 1.0);
  const double2 cur = (d && !tgt) ? P.vtof[h.y + k] : make_double2(1.0, 1.0);
  const unsigned code = (tgt && P.ev) ? P.ev[rc.z] : 0u;
  const bool out = d && ((smask >> k) & 1);
  const double2 pp = out ? __ldg(P.fpar + h.x) : make_double2(0.0, 0.0);
  double2 m = cur;
  if (tgt) {  // vtof (engine.py:186-195): the row without slot j, left to right
    double a0 = 1.0, a1 = 1.0;
#pragma unroll
    for (int i = 0; i < kFuseRow; ++i)
      if (i < dv && i != j) {
        a0 = mul(a0, x[i].x);
        a1 = mul(a1, x[i].y);
      }
    // the rest of a long row in groups of four loads issued together (one
    // round trip per group instead of one per slot), same left-to-right order
    for (int b = kFuseRow; b < dv; b += 4) {
      double2 y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        y[u] = b + u < dv ? P.ftov[rc.x + b + u] : make_double2(1.0, 1.0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (b + u < dv && b + u != j) {
          a0 = mul(a0, y[u].x);
          a1 = mul(a1, y[u].y);
        }
    }
    if (code && it > 1) apply_clamp(code, a0, a1);
    put_message_ref(P, P.vtof + h.y + k, a0, a1, phase, 0, h.y + k, ufkey);
    m = make_double2(a0, a1);
  }
  const bool is_or = factor_is_or(P, h.x);
  const int dmax = __reduce_max_sync(0xffffffffu, d);
  double b1 = 1.0, b2 = 1.0;
  for (int i = 0; i < dmax; ++i) {
    const double x0 = __shfl_sync(0xffffffffu, m.x, base + i);
    const double x1 = __shfl_sync(0xffffffffu, m.y, base + i);
    if (out && i < d && i != k) {  // left to right, the own slot skipped
      double f1, f2;
#if HBP_FUSED_SEL
      // the kind selects operands (head_slot_terms with c = p1 for OR, p2 for AND)
      if (i == 0) {
        const double c = is_or ? pp.x : pp.y;
        f1 = add(mul(sub(1.0, c), x0), mul(c, x1));
        f2 = sub(x0, x1);
      } else {
#else
      if (i == 0) {
        if (is_or)
          head_slot_terms<1>(pp.x, pp.y, x0, x1, f1, f2);
        else
          head_slot_terms<0>(pp.x, pp.y, x0, x1, f1, f2);
      } else {
#endif
        f1 = add(x0, x1);
        f2 = is_or ? x0 : x1;
      }
      b1 = mul(b1, f1);
      b2 = mul(b2, f2);
    }
  }
  if (out) {
    double o0, o1;
#if HBP_FUSED_SEL
    factor_out(is_or, k == 0, pp.x, pp.y, b1, b2, o0, o1);
#else
    if (k == 0) {
      if (is_or)
        head_message<1>(pp.x, pp.y, b1, b2, o0, o1);
      else
        head_message<0>(pp.x, pp.y, b1, b2, o0, o1);
    } else {
      if (is_or)
        body_message<1>(pp.x, pp.y, b1, b2, o0, o1);
      else
        body_message<0>(pp.x, pp.y, b1, b2, o0, o1);
    }
#endif
    put_message(P, P.ftov + rc.w, o0, o1, phase, 1, rc.w, ufkey);
  }
}

// --------------------------------------------------------------------------------------
// one phase over its slots, grid- or CTA-strided

// chunk-claim counters of the whole-node phases, alternating by the phase's
// sequence number: each phase resets the one the next phase uses (phases are
// separated by __syncthreads; both are zeroed in the kernel prologue)
__shared__ int s_claim[2];
__shared__ unsigned long long s_dmax;  // lbp_parall: the CTA's |dP1| max of the iteration
struct NoHookP {
  __device__ void operator()() const {}
};
// the chunk classes of the two whole-node phases, staged from KParams at launch,
// and per round of a grid-wide phase the class of the round's first chunk
__shared__ ChunkClass s_vcc[kMaxVarClasses], s_fcc[kMaxFacClasses];
constexpr int kRoundTab = 512;
__shared__ unsigned char s_vround[kRoundTab], s_fround[kRoundTab];

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool FUSED>
__device__ __forceinline__ void exec_phase(const KParams &P, const Phase &ph, int pidx, int it,
                                           bool do_marg, bool do_vtof,
                                           unsigned long long &dmax) {
  const int seq = it * P.nphases + pidx;
  if (threadIdx.x == 0) s_claim[(seq + 1) & 1] = 0;
  int start, stride;
  if (ph.grid) {
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = gridDim.x * blockDim.x;
  } else {
    if ((int)blockIdx.x >= P.csize) return;
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = P.csize * blockDim.x;
  }
  const int n = ph.end - ph.begin;
  unsigned ufkey = 0;
  if (FUSED && ph.type == 2) {  // n is a multiple of 32: whole warps
    for (int i = start; i < n; i += stride) {
      const int4 *lr = P.fitems + 2 * (size_t)(ph.begin + i);
      const int4 h = __ldg(lr), rc = __ldg(lr + 1);
      fused_lane(P, h, rc, it, pidx, ufkey);
    }
    flush_underflow(P, it, pidx, ufkey);
    return;
  }
  if (ph.list == 2) {
    // every node of the phase's side, in warp chunks of one chunk class each
    // (base_params: dearest classes first, so the phase's tail is cheap
    // chunks, which balances the warps); the unary factors' constant
    // messages only in iteration 1
    const int lane = threadIdx.x & 31;
    const bool marg = do_marg && ph.marg;
    if (ph.type == 0 && !(marg || do_vtof)) return;
    const int nchunks = ph.type == 0 ? P.vchunks : (it == 1 ? P.fchunks : P.fchunks_nounary);
    // Chunk map: round r (G consecutive chunks, G = the CTAs of the phase)
    // is dealt boustrophedon -- CTA b takes position b on even rounds and
    // G-1-b on odd ones. Chunk cost falls along the class order, so a plain
    // deal would hand the low CTA ids the dearer chunk of every round.
    const int G = ph.grid ? (int)gridDim.x : P.csize;
#ifdef HBP_TRACE_CHUNKS  // per-chunk ns of iteration 3 (tools/trace_probe.py)
    unsigned long long *ctr = (P.trace && it == 3 && P.nphases == 2 && nchunks <= kChunkTrace)
                                  ? P.trace + (size_t)kTraceIters * 2 * gridDim.x * 2 + pidx * kChunkTrace
                                  : nullptr;
#else
    constexpr unsigned long long *ctr = nullptr;
#endif
    // Rounds are claimed dynamically by the CTA's warps from a shared-memory
    // counter: a warp whose chunks were cheap takes the next round, so the
    // CTA's phase ends near its mean warp load instead of its max (measured
    // at ftp: max-warp 4.8 us against a 3.5 us mean with a static deal).
    int *claim = &s_claim[seq & 1];
    const bool uniform = it == 1 && pidx == 0;
    const bool var = ph.type == 0;
    const ChunkClass *ccs = var ? s_vcc : s_fcc;
    const int ncc = var ? P.nvcc : P.nfcc;
    const unsigned char *rtab = var ? s_vround : s_fround;
    // (claiming the next round before running the current chunk measured
    // slower: a busy warp then holds a round the others could take)
    int r = 0;
    if (lane == 0) r = atomicAdd(claim, 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    while (r * G < nchunks) {
      int rn = 0;
      const int k = r * G + ((r & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
      if (k < nchunks) {
        // the chunk's class: from the round's first class (a table built at
        // launch for grid-wide phases), walked forward
        int c = (G == (int)gridDim.x && r < kRoundTab) ? rtab[r] : 0;
        while (c + 1 < ncc && ccs[c + 1].chunk_begin <= k) ++c;
        const ChunkClass &cc = ccs[c];
        const unsigned long long t0 = ctr ? globaltimer() : 0;
        if (var)
          var_chunk(P, cc, k - cc.chunk_begin, lane, marg, do_vtof, it, pidx, dmax, ufkey, uniform);
        else
          fac_chunk(P, cc, k - cc.chunk_begin, lane, pidx, ufkey);
        if (ctr) {
          __syncwarp();
          if (lane == 0) ctr[k] = globaltimer() - t0;
        }
      }
      if (lane == 0) rn = atomicAdd(claim, 1);
      r = __shfl_sync(0xffffffffu, rn, 0);
    }
    flush_underflow(P, it, pidx, ufkey);
    return;
  }
  // Slot words, twins and item lists are read-only for the whole launch
  // (ld.global.nc); the next item's are fetched before the current item is
  // computed, so the per-item dependent chain is one memory round trip.
  if (ph.type == 0) {
    const bool marg = do_marg && ph.marg;
    int q = 0, write = 0;
    int2 w = make_int2(0, 0);
    unsigned tw = 0;
    auto fetch = [&](int i, int &q_, int &write_, int2 &w_, unsigned &tw_) {
      if (ph.list) {
        const int item = __ldg(P.items + ph.begin + i);
        q_ = item & (kWriteBit - 1);
        write_ = (item & kWriteBit) ? 1 : 0;
      } else {
        q_ = ph.begin + i;
        write_ = -1;
      }
      w_ = __ldg(P.vslot + q_);
      tw_ = __ldg(P.ftov_twin + q_);
    };
    if (start < n) fetch(start, q, write, w, tw);
    for (int i = start; i < n; i += stride) {
      int qn = 0, writen = 0;
      int2 wn = make_int2(0, 0);
      unsigned twn = 0;
      if (i + stride < n) fetch(i + stride, qn, writen, wn, twn);
      v_item(P, q, w, tw, do_vtof ? write : 0, marg, it, pidx, dmax, ufkey, it == 1 && pidx == 0);
      q = qn;
      write = writen;
      w = wn;
      tw = twn;
    }
  } else {
    int p = 0, tw = 0;
    int2 w = make_int2(0, 0);
    auto fetch = [&](int i, int &p_, int2 &w_, int &tw_) {
      p_ = ph.list ? __ldg(P.items + ph.begin + i) : ph.begin + i;
      w_ = __ldg(P.fslot + p_);
      tw_ = __ldg(P.vtof_twin + p_);
    };
    if (start < n) fetch(start, p, w, tw);
    for (int i = start; i < n; i += stride) {
      int pn = 0, twn = 0;
      int2 wn = make_int2(0, 0);
      if (i + stride < n) fetch(i + stride, pn, wn, twn);
      f_item(P, p, w, tw, pidx, ufkey);
      p = pn;
      w = wn;
      tw = twn;
    }
  }
  flush_underflow(P, it, pidx, ufkey);
}

__device__ __forceinline__ unsigned long long block_max(unsigned long long v) {
  __shared__ unsigned long long red[32];
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


// debug timeline (HBP_TRACE=1): per CTA, phase start / end after a CTA sync
__device__ __forceinline__ void trace_mark(const KParams &P, int it, int p, int which) {
  if (P.trace == nullptr || it < 2 || it >= 2 + kTraceIters) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    // ns timer (low 52 bits) << 8 | SM id
    P.trace[(((size_t)(it - 2) * P.nphases + p) * gridDim.x + blockIdx.x) * 2 + which] =
        ((globaltimer() & ((1ull << 52) - 1)) << 8) | (smid & 0xff);
  }
}

// barrier of the CTAs that run the small levels: __syncthreads for CTA 0
// alone, else the thread-block cluster barrier of cluster 0 (release /
// acquire at cluster scope orders the global-memory messages too)
__device__ __forceinline__ void cluster0_sync(int csize) {
  if (csize > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
}

// A run of consecutive small phases [p0, p1) on the small-level CTAs (fused
// levels, and the vtof / ftov phases of unfused ones): a tight loop -- the
// phase's items, the barrier, the next phase -- instead of the generic phase
// loop, whose per-phase prologue (descriptor copies, transition logic,
// look-ahead) measured about 1 us per level on B200. Each phase loads this
// thread's first item of the next one (a fused lane record: L1 prefetch; a
// slot item: its slot-word / twin lines prefetched after this phase's work).
// Underflow flags are published per phase (the attribution re-run halts at
// the earliest failing phase; runs are not used in the halted iteration).
template <bool FUSED>
__device__ __forceinline__ void run_small(const KParams &P, const Phase *cache, int p0, int p1,
                                          int it) {
  const int stride = P.csize * (int)blockDim.x;
  const int start = (int)blockIdx.x * (int)blockDim.x + (int)threadIdx.x;
  auto at = [&](int p) -> const Phase & { return p < kPhaseCache ? cache[p] : P.phases[p]; };
  unsigned long long unused = 0;
  for (int p = p0; p < p1; ++p) {
    if (p > p0) cluster0_sync(P.csize);
    const Phase &ph = at(p);
    const int type = ph.type, b = ph.begin, n = ph.end - ph.begin;
    int nxt = -1, ntype = 0;
    if (p + 1 < p1) {
      const Phase &np = at(p + 1);
      ntype = np.type;
      if (start < np.end - np.begin) {
        if (np.type == 2)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(P.fitems + 2 * (size_t)(np.begin + start)));
        else
          nxt = __ldg(P.items + np.begin + start) & (kWriteBit - 1);
      }
    }
    unsigned ufkey = 0;
#ifdef HBP_TRACE_SMALL
    trace_mark(P, it, p, 0);
#endif
    if (FUSED && type == 2) {
      for (int i = start; i < n; i += stride) {
        const int4 *lr = P.fitems + 2 * (size_t)(b + i);
        fused_lane(P, __ldg(lr), __ldg(lr + 1), it, p, ufkey);
      }
    } else if (P.iw && type == 0) {
      for (int i = start; i < n; i += stride) {
        const int item = __ldg(P.items + b + i);
        const int4 w = __ldg(P.iw + b + i);
        v_item(P, item & (kWriteBit - 1), make_int2(w.x, w.y), (unsigned)w.z,
               (item & kWriteBit) ? 1 : 0, false, it, p, unused, ufkey, false);
      }
    } else if (P.iw) {
      for (int i = start; i < n; i += stride) {
        const int q = __ldg(P.items + b + i);
        const int4 w = __ldg(P.iw + b + i);
        f_item(P, q, make_int2(w.x, w.y), w.z, p, ufkey);
      }
    } else if (type == 0) {
      for (int i = start; i < n; i += stride) {
        const int item = __ldg(P.items + b + i);
        const int q = item & (kWriteBit - 1);
        v_item(P, q, __ldg(P.vslot + q), __ldg(P.ftov_twin + q), (item & kWriteBit) ? 1 : 0, false, it,
               p, unused, ufkey, false);
      }
    } else {
      for (int i = start; i < n; i += stride) {
        const int q = __ldg(P.items + b + i);
        f_item(P, q, __ldg(P.fslot + q), __ldg(P.vtof_twin + q), p, ufkey);
      }
    }
    flush_underflow(P, it, p, ufkey);
#ifdef HBP_TRACE_SMALL
    trace_mark(P, it, p, 1);
#endif
    if (nxt >= 0) {
      const void *x = ntype == 1 ? (const void *)(P.fslot + nxt) : (const void *)(P.vslot + nxt);
      const void *y = ntype == 1 ? (const void *)(P.vtof_twin + nxt) : (const void *)(P.ftov_twin + nxt);
      asm volatile("prefetch.global.L1 [%0];" ::"l"(x));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(y));
    }
  }
}

// marginals of the stopping iteration in the reference's variable order
__device__ __forceinline__ void write_marginals(const KParams &P, const double *src = nullptr) {
  const int gs = gridDim.x * blockDim.x;
  const double *p0s = src ? src : P.p0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < P.V; v += gs) {
    const double p0 = p0s[v];
    P.marg[__ldg(P.vorig + v)] = make_double2(p0, sub(1.0, p0));
  }
}

// FUSED: the instance for plans with fused levels (a separate instance keeps
// the PARALL kernel's register allocation untouched)
template <int THREADS, bool FUSED>
__global__ void __launch_bounds__(THREADS, 1) lbp_persistent(const __grid_constant__ KParams P) {
  Ctrl *C = P.ctrl;
  const bool multi = gridDim.x > 1;
  const unsigned G = gridDim.x;
  Sync sy;  // sync points passed so far (identical on every CTA)
  // PARALL (two whole-graph phases): iteration 1 needs no initial messages --
  // its variable side writes the normalised uniform message directly, and its
  // factor side then writes every factor-to-variable message
  // the phase descriptors (a levelled schedule has two per level: 952 at ftp
  // SEQFIX) are staged in shared memory once, so a small level's start does
  // not wait on a global load of its descriptor
  __shared__ Phase s_ph[kPhaseCache];
  __shared__ int s_nx[THREADS];  // look-ahead items (levelled schedules)
  for (int i = threadIdx.x; i < P.nphases && i < kPhaseCache; i += blockDim.x) s_ph[i] = P.phases[i];
  if (threadIdx.x < 2) s_claim[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < P.nvcc; i += blockDim.x) s_vcc[i] = P.vcc[i];
  for (int i = threadIdx.x; i < P.nfcc; i += blockDim.x) s_fcc[i] = P.fcc[i];
  for (int r = threadIdx.x; r < kRoundTab; r += blockDim.x) {
    const int k = r * (int)gridDim.x;
    int c = 0;
    while (c + 1 < P.nvcc && P.vcc[c + 1].chunk_begin <= k) ++c;
    s_vround[r] = (unsigned char)c;
    c = 0;
    while (c + 1 < P.nfcc && P.fcc[c + 1].chunk_begin <= k) ++c;
    s_fround[r] = (unsigned char)c;
  }
  __syncthreads();
  auto phase_at = [&](int i) -> const Phase & { return i < kPhaseCache ? s_ph[i] : P.phases[i]; };
  const bool parall = P.nphases == 2 && s_ph[0].list == 2 && s_ph[1].list == 2;
  auto grid_sync = [&]() {
    if (multi) sync_point(C, sy, G, true, true);
    else __syncthreads();
  };

  // uniform start: all messages (1, 1), prev P1 = 0.5 (storage.py:91-94, engine.py:557)
  // PARALL: iteration 1's variable side would only write the normalised
  // (1, 1) into every vtof slot (no ftov is read, no marginal is due), so the
  // start writes that constant directly and the phase -- with its barrier --
  // is skipped
  {
    const int gs = gridDim.x * blockDim.x;
    const double c = parall ? (P.normalize ? 0.5 : 1.0) : 1.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.E; i += gs) {
      P.vtof[i] = make_double2(c, c);
      if (!parall) P.ftov[i] = make_double2(1.0, 1.0);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.V; i += gs) P.p0[i] = 0.5;
    if (blockIdx.x == 0 && threadIdx.x == 0) C->t0 = globaltimer();
    grid_sync();
  }

  for (int it = 1;; ++it) {
    const bool final_pass = it == P.max_it + 1;
    unsigned long long dmax = 0;
    if (it == P.halt_it && P.halt_phase == 0) return;  // attribution re-run
    if (!(parall && it == 1)) {
      trace_mark(P, it, 0, 0);
      exec_phase<FUSED>(P, phase_at(0), 0, it, it > 1, !final_pass, dmax);
      trace_mark(P, it, 0, 1);
      if (it > 1) {
        unsigned long long m = block_max(dmax);
        if (threadIdx.x == 0) {
          atomicMax(&P.delta_bits[it - 1], m);
          if (blockIdx.x == 0 && P.time_limit_ns > 0)
            P.tflag[it - 1] = (long long)(globaltimer() - C->t0) > P.time_limit_ns;
        }
      }
      grid_sync();
    }
    // Stop decision for iteration it-1 (all CTAs passed the barrier, so the
    // flags and delta are final). With two phases per iteration (PARALL)
    // the decision is applied at the end of this iteration instead, so its
    // loads overlap phase 1; a stop then only wastes a factor-side phase
    // whose output (ftov) is never observed.
    __shared__ int s_stop;
    const int done = it - 1;
    // the decision inputs are loaded now and evaluated where the decision is
    // applied: in the deferred (PARALL) case warp 0 does not wait on them
    // before its share of the factor phase
    int ufm = 0, ufg = 0, tf = 0;
    unsigned long long db = 0;
    if (it > 1 && threadIdx.x == 0) {
      ufm = ((const volatile int *)P.uf_msg)[done];
      ufg = ((const volatile int *)P.uf_marg)[done];
      tf = ((const volatile int *)P.tflag)[done];
      db = ((const volatile unsigned long long *)P.delta_bits)[done];
    }
    auto decide = [&]() -> int {
      if (ufm || ufg == 1) return 4;  // ufg bit1 (a NaN total) suppresses the raise
      if (__longlong_as_double((long long)db) < P.tol) return 1;
      if (done == P.max_it) return 2;
      if (tf) return 3;
      return 0;
    };
    const bool defer = P.nphases == 2 && !final_pass;
    if (it > 1 && !defer) {
      if (threadIdx.x == 0) s_stop = decide();
      __syncthreads();
      if (s_stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          C->iterations = done;
          C->last_delta = db;
          C->converged = s_stop == 1;
          C->stop = s_stop;
        }
        write_marginals(P);
        return;
      }
    }
    // remaining phases of this iteration
    for (int p = 1; p < P.nphases; ++p) {
      const Phase ph = phase_at(p);
      if (p > 1) {  // transition p-1 -> p (phase 0 -> 1 was the full barrier above)
        const int prev_grid = phase_at(p - 1).grid;
        const bool in0 = (int)blockIdx.x < P.csize;
        if (!multi) {
          __syncthreads();
        } else if (prev_grid && ph.grid) {
          sync_point(C, sy, G, true, true);
        } else if (prev_grid && !ph.grid) {
          sync_point(C, sy, G, true, in0);
        } else if (!prev_grid && !ph.grid) {
          if (in0) cluster0_sync(P.csize);
        } else {  // CTA 0 -> grid
          sync_point(C, sy, P.csize, in0, true);
        }
      }
      if (it == P.halt_it && p == P.halt_phase) return;  // attribution re-run
      // a run of small phases (its first phase's sbegin = the run's end); not
      // in an attribution re-run's halted iteration. The run's phases skip
      // exec_phase, whose prologue resets the whole-node claim counter of the
      // following phase: that reset is done here, by every CTA.
      if (ph.list != 2 && !ph.grid && ph.sbegin > p + 1 && it != P.halt_it) {
        if ((int)blockIdx.x < P.csize) run_small<FUSED>(P, s_ph, p, ph.sbegin, it);
        if (threadIdx.x == 0) s_claim[(it * P.nphases + ph.sbegin) & 1] = 0;
        p = ph.sbegin - 1;
        continue;
      }
      // Look-ahead for levelled schedules: the next list phase's first item
      // of this thread is copied into shared memory now (cp.async: no
      // register waits on it) and, once this phase is done, its slot word and
      // twin lines are prefetched into L1 -- so a small level's dependent
      // chain starts at the message rows.
      bool look = false;
      if (p + 1 < P.nphases) {
        const Phase &np = phase_at(p + 1);
        const int i = blockIdx.x * blockDim.x + threadIdx.x;
        const bool mine = (np.grid || (int)blockIdx.x < P.csize) && i < np.end - np.begin;
        if (FUSED && np.list == 3 && mine) {
          // fused level: the item lines (read-only) of this thread's first
          // two lanes into L1
          const int stride = (np.grid ? (int)gridDim.x : P.csize) * (int)blockDim.x;
          const int4 *lr = P.fitems + 2 * (size_t)(np.begin + i);
          asm volatile("prefetch.global.L1 [%0];" ::"l"(lr));
          if (i + stride < np.end - np.begin)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(lr + 2 * (size_t)stride));
        }
        look = np.list == 1 && mine;
        if (look) {
          const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_nx[threadIdx.x]);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n\tcp.async.commit_group;" ::"r"(dst),
                       "l"(P.items + np.begin + i)
                       : "memory");
        }
      }
      unsigned long long unused = 0;
      trace_mark(P, it, p, 0);
      exec_phase<FUSED>(P, ph, p, it, false, true, unused);
      trace_mark(P, it, p, 1);
      if (look) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        const int q = s_nx[threadIdx.x] & (kWriteBit - 1);
        const bool fac = phase_at(p + 1).type == 1;
        const void *a = fac ? (const void *)(P.fslot + q) : (const void *)(P.vslot + q);
        const void *b = fac ? (const void *)(P.vtof_twin + q) : (const void *)(P.ftov_twin + q);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(b));
      }
    }
    // transition last phase -> phase 0 of the next iteration (a grid phase)
    if (P.nphases > 1) {
      const int last_grid = phase_at(P.nphases - 1).grid;
      if (!multi) {
        __syncthreads();
      } else if (last_grid) {
        sync_point(C, sy, G, true, true);
      } else {
        sync_point(C, sy, P.csize, (int)blockIdx.x < P.csize, true);
      }
    }
    if (it > 1 && defer) {
      if (threadIdx.x == 0) s_stop = decide();
      __syncthreads();
      if (s_stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          C->iterations = done;
          C->last_delta = db;
          C->converged = s_stop == 1;
          C->stop = s_stop;
        }
        write_marginals(P);
        return;
      }
    }
  }
}

// ======================================================================================
// PARALL plans (one batch: engine.py:566-570 as two whole-graph phases) run a
// kernel of their own -- the same chunk work as lbp_persistent's whole-node
// phases, without the level machinery -- so its tuning cannot disturb the
// levelled instances' register allocation. The |dP1| reduction and the stop
// decision ride on the two grid barriers of an iteration.

// thread 0's hooks run inside the barrier: pre before its arrival (after the
// CTA's __syncthreads), post after its wait (before the closing one)
template <typename Pre, typename Post>
__device__ __forceinline__ void sync_point_hooked(Ctrl *c, Sync &s, unsigned arrivals, bool arrive,
                                                  bool wait, Pre pre, Post post) {
  __syncthreads();
  s.target += arrivals;
  if (threadIdx.x == 0) {
    pre();
    if (arrive) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&c->bar) : "memory");
    if (wait)
      while (ld_acquire(&c->bar) < s.target) {
      }
    post();
  }
  __syncthreads();
}

// the per-node kernels again with normalisation fixed on (lbp_parall<.., true>)
namespace n1 {
#define HBP_NORMALIZE(P) 1
#include "lbp_node.inc"
#undef HBP_NORMALIZE
}  // namespace n1

// every node of one side in class-uniform warp chunks (the same loop as
// exec_phase's list == 2 branch); NORM: the n1 kernels
template <bool NORM>
__device__ __forceinline__ void node_phase(const KParams &P, bool var, int G, int seq, int it,
                                           int pidx, bool marg, bool vt,
                                           unsigned long long &dmax, unsigned &ufkey) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_claim[(seq + 1) & 1] = 0;
  if (var && !(marg || vt)) return;
  if ((int)blockIdx.x >= G) return;
  const int nchunks = var ? P.vchunks : (it == 1 ? P.fchunks : P.fchunks_nounary);
  int *claim = &s_claim[seq & 1];
  const ChunkClass *ccs = var ? s_vcc : s_fcc;
  const int ncc = var ? P.nvcc : P.nfcc;
  const unsigned char *rtab = var ? s_vround : s_fround;
  // the first round of every warp is its own index; later ones are claimed
  const int nwarps = (int)(blockDim.x >> 5);
  int r = (int)(threadIdx.x >> 5);
  while (r * G < nchunks) {
    int rn = 0;
    const int k = r * G + ((r & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
    if (k < nchunks) {
      // lbp_parall's table holds this CTA's exact class per round
      int c = 0;
      if (G == (int)gridDim.x && r < kRoundTab)
        c = rtab[r];
      else
        while (c + 1 < ncc && ccs[c + 1].chunk_begin <= k) ++c;
      const ChunkClass &cc = ccs[c];
#ifdef HBP_TRACE_CHUNKS  // per-chunk ns | class << 48 of iteration 3 (tools/chunk_probe.py)
      const unsigned long long t0 = globaltimer();
#endif
      if (NORM) {
        if (var)
          n1::var_chunk(P, cc, k - cc.chunk_begin, lane, marg, vt, it, pidx, dmax, ufkey, false);
        else
          n1::fac_chunk(P, cc, k - cc.chunk_begin, lane, pidx, ufkey);
      } else {
        if (var)
          var_chunk(P, cc, k - cc.chunk_begin, lane, marg, vt, it, pidx, dmax, ufkey, false);
        else
          fac_chunk(P, cc, k - cc.chunk_begin, lane, pidx, ufkey);
      }
#ifdef HBP_TRACE_CHUNKS
      if (P.trace && it == 3 && nchunks <= kChunkTrace) {
        __syncwarp();
        if (lane == 0)
          P.trace[(size_t)kTraceIters * 2 * gridDim.x * 2 + pidx * kChunkTrace + k] =
              (globaltimer() - t0) | (unsigned long long)c << 48;
      }
#endif
    }
    if (lane == 0) rn = atomicAdd(claim, 1) + nwarps;
    r = __shfl_sync(0xffffffffu, rn, 0);
  }
}

template <int THREADS, bool NORM>
__global__ void __launch_bounds__(THREADS, 1) lbp_parall(const __grid_constant__ KParams P) {
  Ctrl *C = P.ctrl;
  const bool multi = gridDim.x > 1;
  const unsigned G = gridDim.x;
  Sync sy;
  if (threadIdx.x < 2) s_claim[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_dmax = 0;
  for (int i = threadIdx.x; i < P.nvcc; i += blockDim.x) s_vcc[i] = P.vcc[i];
  for (int i = threadIdx.x; i < P.nfcc; i += blockDim.x) s_fcc[i] = P.fcc[i];
  // the class of this CTA's chunk in round r of a grid-wide phase
  for (int r = threadIdx.x; r < kRoundTab; r += blockDim.x) {
    const int G = (int)gridDim.x;
    const int k = r * G + ((r & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
    int c = 0;
    while (c + 1 < P.nvcc && P.vcc[c + 1].chunk_begin <= k) ++c;
    s_vround[r] = (unsigned char)c;
    c = 0;
    while (c + 1 < P.nfcc && P.fcc[c + 1].chunk_begin <= k) ++c;
    s_fround[r] = (unsigned char)c;
  }
  // the factor side may be a small phase (CTAs [0, csize)) on small graphs
  const int fG = P.phases[1].grid ? (int)gridDim.x : P.csize;
  auto barrier = [&](unsigned arrivals, bool arrive, auto pre, auto post) {
    if (multi) {
      sync_point_hooked(C, sy, arrivals, arrive, true, pre, post);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        pre();
        post();
      }
      __syncthreads();
    }
  };
  const NoHookP nohook;
  // uniform start: iteration 1's variable side would only write the
  // normalised (1, 1) into every vtof slot, so the start writes it directly
  {
    const int gs = gridDim.x * blockDim.x;
    const double cst = P.normalize ? 0.5 : 1.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.E; i += gs) P.vtof[i] = make_double2(cst, cst);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.V; i += gs) P.p0[i] = 0.5;
    if (blockIdx.x == 0 && threadIdx.x == 0) C->t0 = globaltimer();
    barrier(G, true, nohook, nohook);
  }
  __shared__ int s_stop;
  for (int it = 1;; ++it) {
    const bool final_pass = it == P.max_it + 1;
    const int done = it - 1;
    if (it == P.halt_it && P.halt_phase == 0) return;  // attribution re-run
    if (it > 1) {
      unsigned long long dmax = 0;
      unsigned ufkey = 0;
      trace_mark(P, it, 0, 0);
      node_phase<NORM>(P, true, (int)gridDim.x, it * 2, it, 0, true, !final_pass, dmax, ufkey);
      flush_underflow(P, it, 0, ufkey);
      trace_mark(P, it, 0, 1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, dmax, o);
        dmax = w > dmax ? w : dmax;
      }
      if ((threadIdx.x & 31) == 0 && dmax) atomicMax(&s_dmax, dmax);
      auto publish = [&]() {
        if (s_dmax) atomicMax(&P.delta_bits[it - 1], s_dmax);
        s_dmax = 0;
        if (blockIdx.x == 0 && P.time_limit_ns > 0)
          P.tflag[it - 1] = (long long)(globaltimer() - C->t0) > P.time_limit_ns;
      };
      barrier(G, true, publish, nohook);
    }
    // stop decision for iteration it-1, taken at the end of this iteration
    // (its loads overlap the factor side; a stop only wastes that phase,
    // whose output is never observed) -- or right away in the final pass
    int ufm = 0, ufg = 0, tf = 0;
    unsigned long long db = 0;
    if (it > 1 && threadIdx.x == 0) {
      ufm = ((const volatile int *)P.uf_msg)[done];
      ufg = ((const volatile int *)P.uf_marg)[done];
      tf = ((const volatile int *)P.tflag)[done];
      db = ((const volatile unsigned long long *)P.delta_bits)[done];
    }
    auto decide = [&]() -> int {
      if (ufm || ufg == 1) return 4;  // ufg bit1 (a NaN total) suppresses the raise
      if (__longlong_as_double((long long)db) < P.tol) return 1;
      if (done == P.max_it) return 2;
      if (tf) return 3;
      return 0;
    };
    auto decide_hook = [&]() { s_stop = it > 1 ? decide() : 0; };
    if (final_pass) {
      if (threadIdx.x == 0) decide_hook();
      __syncthreads();
    } else {
      if (it == P.halt_it && P.halt_phase == 1) return;  // attribution re-run
      unsigned long long unused = 0;
      unsigned ufkey = 0;
      trace_mark(P, it, 1, 0);
      node_phase<NORM>(P, false, fG, it * 2 + 1, it, 1, false, true, unused, ufkey);
      flush_underflow(P, it, 1, ufkey);
      trace_mark(P, it, 1, 1);
      if (fG == (int)gridDim.x)
        barrier(G, true, nohook, decide_hook);
      else
        barrier(P.csize, (int)blockIdx.x < P.csize, nohook, decide_hook);
    }
    if (it > 1 && s_stop) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->iterations = done;
        C->last_delta = db;
        C->converged = s_stop == 1;
        C->stop = s_stop;
      }
      write_marginals(P);
      return;
    }
  }
}


// ======================================================================================
// PARALL as ONE phase per iteration (lbp_pslot). The two-phase form reads
// every message twice per iteration and pays two grid barriers; here a lane
// per factor slot computes its variable's vtof message straight from the
// variable's ftov row of the previous iteration (engine.py:186-195: the row
// without the own slot, left to right), the factor's lanes exchange them by
// warp shuffles (as a fused level does) and each lane writes the factor's
// ftov message of its slot (engine.py:198-248). The vtof buffer is never
// materialised. Reads and writes of one iteration go to different ftov
// buffers (iteration it writes buffer it & 1), so no lane reads a row another
// lane is writing -- exactly the two-phase values. The lane holding slot 0
// of its variable's row has that whole row loaded and also computes the
// variable's marginal of iteration it-1 (engine.py:510-523) into P0 buffer
// (it-1) & 1. One grid barrier per iteration; the stop decision on
// iteration it-2 rides on the barrier closing iteration it (its inputs are
// loaded while iteration it runs), which the alternating P0 buffers make
// safe: the marginals of it-2 are still intact when it is taken.
// Underflow only stops the run: the host replays the schedule with the
// two-phase kernel, which attributes it exactly (bitwise the same run).

// one chunk: info = degree | kind << 8 | longest row << 16 (warp-uniform),
// rc = the lane's record. One instance for every degree: the kernel's speed
// tracks its code size (measured: degree- or row-templated instances run
// 15-70 % slower, instruction-cache bound).
template <bool NORM>
__device__ __forceinline__ void pslot_chunk(const KParams &P, int info, int4 rc, int lane, int it,
                                            bool final_pass, const double2 *fin, double2 *fout,
                                            const double *p0in, double *p0out,
                                            unsigned long long &dmax, unsigned &ufkey) {
  const int d = info & 0xff;
  const bool is_or = ((info >> 8) & 1) != 0;
  const bool valid = ((rc.w >> 24) & 1) != 0;
  const int j = (rc.w >> 8) & 0xff, k = (rc.w >> 16) & 0xff;
  const bool owner = valid && it >= 2 && j == 0;  // computes the variable's marginal
  const bool tgt = valid && it >= 2 && !final_pass && d > 1;  // unary factors read no vtof
  const int dv = (owner || tgt) ? (rc.w & 0xff) : 0;
  // every load of the lane in one round trip: the row as 32-byte aligned
  // message pairs (256-bit loads, half the load instructions and L1
  // wavefronts of one message per load); element e of the pairs is row
  // slot e - off
  const int off = rc.x & 1, ne = off + dv;
  const double2 *base2 = fin + (rc.x - off);
  double2 y[2 * kPslotPairs];
#pragma unroll
  for (int t = 0; t < kPslotPairs; ++t) {
    double v0 = 1.0, v1 = 1.0, v2 = 1.0, v3 = 1.0;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %4, %5;\n\t"
        "@p ld.global.v4.f64 {%0, %1, %2, %3}, [%6];\n\t}"
        : "+d"(v0), "+d"(v1), "+d"(v2), "+d"(v3)
        : "r"(2 * t), "r"(ne), "l"(base2 + 2 * t));
    y[2 * t] = make_double2(v0, v1);
    y[2 * t + 1] = make_double2(v2, v3);
  }
  const unsigned code = (dv && P.ev) ? P.ev[rc.y] : 0u;
  double prev_p0 = 0.0;
  if (owner) prev_p0 = it > 2 ? p0in[rc.y] : 0.5;  // iteration 1's previous P1 is 0.5
  // unary factors' constant messages: iterations 1 and 2 (one per buffer)
  const bool out = valid && !final_pass && (d > 1 || it <= 2);
  const double2 pp = out ? __ldg(P.fpar + rc.z) : make_double2(0.0, 0.0);
  // both row products in one pass, left to right: a = the vtof message's
  // (slot j skipped, engine.py:186-195), q = the marginal's (engine.py:510-516)
  double a0 = 1.0, a1 = 1.0, q0 = 1.0, q1 = 1.0;
#pragma unroll
  for (int e = 0; e < 2 * kPslotPairs; ++e)
    if (e >= off && e < ne) {
      q0 = mul(q0, y[e].x);
      q1 = mul(q1, y[e].y);
      if (e != off + j) {
        a0 = mul(a0, y[e].x);
        a1 = mul(a1, y[e].y);
      }
    }
  for (int e = 2 * kPslotPairs; e < ne; ++e) {
    const double2 z = base2[e];
    q0 = mul(q0, z.x);
    q1 = mul(q1, z.y);
    if (e != off + j) {
      a0 = mul(a0, z.x);
      a1 = mul(a1, z.y);
    }
  }
  if (owner) {
    double c0 = q0, c1 = q1;
    if (code) apply_clamp(code, c0, c1);
    put_marginal_to(P, p0out + rc.y, c0, c1, it, dmax, prev_p0, -1 - rc.y);
  }
  if (final_pass || (d == 1 && it > 2)) return;  // warp-uniform
  // the vtof message of the slot (iteration 1: the uniform start message)
  double2 m = make_double2(NORM ? 0.5 : 1.0, NORM ? 0.5 : 1.0);
  if (tgt) {
    if (code) apply_clamp(code, a0, a1);
    if (NORM) {
      const double t = add(a0, a1);
      ufkey |= (unsigned)(t < kMinMessageSum);
      div2_rn(a0, a1, t, a0, a1);
    }
    m = make_double2(a0, a1);
  }
  // the factor's messages: its vtof row by shuffles within the lane group,
  // left to right with the own slot skipped (engine.py:198-248)
  const int base = lane - k;
  double b1 = 1.0, b2 = 1.0;
  {
    const double x0 = __shfl_sync(0xffffffffu, m.x, base);
    const double x1 = __shfl_sync(0xffffffffu, m.y, base);
    if (k != 0) {
      const double c = is_or ? pp.x : pp.y;  // head_slot_terms
      b1 = mul(b1, add(mul(sub(1.0, c), x0), mul(c, x1)));
      b2 = mul(b2, sub(x0, x1));
    }
  }
  for (int i = 1; i < d; ++i) {
    const double x0 = __shfl_sync(0xffffffffu, m.x, base + i);
    const double x1 = __shfl_sync(0xffffffffu, m.y, base + i);
    if (i != k) {
      b1 = mul(b1, add(x0, x1));
      b2 = mul(b2, is_or ? x0 : x1);
    }
  }
  if (out) {
    double o0, o1;
    factor_out(is_or, k == 0, pp.x, pp.y, b1, b2, o0, o1);
    if (NORM) {
      const double t = add(o0, o1);
      ufkey |= (unsigned)(t < kMinMessageSum) << 1;
      div2_rn(o0, o1, t, o0, o1);
    }
    fout[rc.x + j] = make_double2(o0, o1);
  }
}

template <int THREADS, bool NORM>
__global__ void __launch_bounds__(THREADS, 1) lbp_pslot(const __grid_constant__ KParams P) {
  Ctrl *C = P.ctrl;
  const bool multi = gridDim.x > 1;
  const int G = (int)gridDim.x;
  Sync sy;
  __shared__ int s_stop;
  if (threadIdx.x < 2) s_claim[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_dmax = 0, s_stop = 0;
  // the cluster barrier only when the launch really is one cluster of the
  // whole grid (a launch without the cluster attribute -- e.g. a profiler's
  // kernel replay -- takes the counter barrier instead of racing)
  unsigned ncl;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
  const bool one_cluster = P.csize > 1 && ncl == gridDim.x;
  auto barrier = [&](auto pre) {
    if (one_cluster) {
      // the whole grid is one thread-block cluster (small graphs): the
      // hardware cluster barrier, release / acquire at cluster scope, orders
      // the global-memory messages like the counter barrier does
      __syncthreads();
      if (threadIdx.x == 0) pre();
      asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    } else if (multi) {
      sync_point_hooked(C, sy, (unsigned)G, true, true, pre, NoHookP{});
    } else {
      __syncthreads();
      if (threadIdx.x == 0) pre();
      __syncthreads();
    }
  };
  // iteration 1 reads no message (and iteration 2's previous P0 is the
  // constant 0.5): no start-up pass, no barrier before it
  if (blockIdx.x == 0 && threadIdx.x == 0) C->t0 = globaltimer();
  __syncthreads();
  double2 *const fb0 = P.ftov, *const fb1 = P.ftov_alt;
  double *const pb0 = P.p0, *const pb1 = P.p0_alt;
  auto decide = [&](int done, int ufm, int ufg, int tf, unsigned long long db) -> int {
    if (ufm || ufg == 1) return 4;  // ufg bit1 (a NaN total) suppresses the raise
    if (__longlong_as_double((long long)db) < P.tol) return 1;
    if (done == P.max_it) return 2;
    if (tf) return 3;
    return 0;
  };
  auto finish = [&](int done, unsigned long long db) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      C->iterations = done;
      C->last_delta = db;
      C->converged = s_stop == 1;
      C->stop = s_stop;
    }
    write_marginals(P, (done & 1) ? pb1 : pb0);
  };
  const int lane = threadIdx.x & 31;
  const int nwarps = (int)(blockDim.x >> 5);
  const int nchunks = P.fchunks;
  for (int it = 1;; ++it) {
    const bool final_pass = it == P.max_it + 1;
    // the decision on iteration it-2, whose inputs are complete since the
    // barrier that closed iteration it-1: thread 0 takes it while the other
    // warps already run this iteration's chunks, and they stop claiming
    // chunks once it says stop (the iteration's output is then never read)
    unsigned long long db = 0;
    if (it >= 3 && threadIdx.x == 0) {
      db = ((const volatile unsigned long long *)P.delta_bits)[it - 2];
      *(volatile int *)&s_stop =
          decide(it - 2, ((const volatile int *)P.uf_msg)[it - 2],
                 ((const volatile int *)P.uf_marg)[it - 2], ((const volatile int *)P.tflag)[it - 2],
                 db);
    }
    const double2 *fin = (it & 1) ? fb0 : fb1;
    double2 *fout = (it & 1) ? fb1 : fb0;
    const double *p0in = (it & 1) ? pb1 : pb0;  // marginals of it-2
    double *p0out = (it & 1) ? pb0 : pb1;       // marginals of it-1
    unsigned long long dmax = 0;
    unsigned ufkey = 0;
    {
      // rounds as in node_phase: round r is G consecutive chunks dealt
      // boustrophedon; a warp's first round is its index, later ones claimed
      const int seq = it;
      if (threadIdx.x == 0) s_claim[(seq + 1) & 1] = 0;
      int *claim = &s_claim[seq & 1];
      int r = (int)(threadIdx.x >> 5);
      while (r * G < nchunks && !*(volatile int *)&s_stop) {
        int rn = 0;
        const int k = r * G + ((r & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
        if (k < nchunks) {
          const int info = __ldg(P.sinfo + k);
          const int4 rc = __ldg(P.srec + (size_t)k * 32 + lane);
          pslot_chunk<NORM>(P, info, rc, lane, it, final_pass, fin, fout, p0in, p0out, dmax,
                            ufkey);
        }
        if (lane == 0) rn = atomicAdd(claim, 1) + nwarps;
        r = __shfl_sync(0xffffffffu, rn, 0);
      }
    }
    flush_underflow(P, it, 0, ufkey);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long w = __shfl_xor_sync(0xffffffffu, dmax, o);
      dmax = w > dmax ? w : dmax;
    }
    if (lane == 0 && dmax) atomicMax(&s_dmax, dmax);
    __syncthreads();
    if (s_stop) {  // every CTA took the same decision: none waits at a barrier
      finish(it - 2, db);
      return;
    }
    auto publish = [&]() {
      if (it >= 2) {
        if (s_dmax) atomicMax(&P.delta_bits[it - 1], s_dmax);
        if (blockIdx.x == 0 && P.time_limit_ns > 0)
          P.tflag[it - 1] = (long long)(globaltimer() - C->t0) > P.time_limit_ns;
      }
      s_dmax = 0;
    };
    barrier(publish);
    if (final_pass) {  // the decision on iteration max_it, right away
      if (threadIdx.x == 0) {
        const int done = it - 1;
        db = ((const volatile unsigned long long *)P.delta_bits)[done];
        s_stop = decide(done, ((const volatile int *)P.uf_msg)[done],
                        ((const volatile int *)P.uf_marg)[done], ((const volatile int *)P.tflag)[done],
                        db);
      }
      __syncthreads();
      finish(it - 1, db);
      return;
    }
  }
}

}  // namespace hbp

// ======================================================================================
// single-pass kernels for the host-store diagnostic API (hbp_pass / hbp_marginals)

namespace hbp {

// items: list-mode slot words (type 0: ftov slot | kWriteBit, or a row start
// for a marginal; type 1: vtof slot)
__global__ void __launch_bounds__(256) pass_kernel(const __grid_constant__ KParams P, int type,
                                                   int marg, const int *items, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int item = items[i];
  unsigned long long unused = 0;
  unsigned ufkey = 0;
  if (type == 0) {
    const int q = item & (kWriteBit - 1);
    v_item<true>(P, q, P.vslot[q], P.ftov_twin[q], (item & kWriteBit) ? 1 : 0, marg != 0, marg ? 2 : 1,
           0, unused, ufkey);
  } else {
    f_item(P, item, P.fslot[item], P.vtof_twin[item], 0, ufkey);
  }
  flush_underflow(P, 1, 0, ufkey);
}

// ---- exact underflow attribution (engine.py:155-165, :512-518) ------------------------
// The reference raises in the FIRST failing pass of a batch -- vtof(t_b), then
// the AND-body, AND-head, OR-body, OR-head groups of s_b (_FTOV_RUNNERS) --
// naming rows[argmin(total)], the rows being that pass's targets stable-sorted
// by descending row length (_compile_pass, engine.py:137-138): so the winner
// is the minimum of (total, -row length, position in the batch). The run
// stops at the start of the failing phase (halt_it / halt_phase), whose inputs
// are then still intact, and this kernel recomputes every target's total in
// the run kernels' exact arithmetic. Two launches: (1) the minimum total per
// group, (2) among the targets at that total, the minimum (-rowlen, position).

// total of the vtof message owned by ftov slot q (v_item without the write)
__device__ double attr_vtof_total(const KParams &P, int q, int it, int &var) {
  const int2 w = P.vslot[q];
  const int d = w.y >> 16, j = w.y & 0xffff;
  double a0 = 1.0, a1 = 1.0, q0 = 1.0, q1 = 1.0;
  v_row_long(P, q - j, d, j, false, a0, a1, q0, q1);
  const unsigned code = P.ev ? P.ev[w.x] : 0u;
  if (code && it > 1) apply_clamp(code, a0, a1);
  var = w.x;
  return add(a0, a1);
}

// total of the ftov message owned by vtof slot p (f_item without the write)
__device__ double attr_ftov_total(const KParams &P, int p, int &group, int &deg) {
  const int2 w = P.fslot[p];
  const int d = w.y >> 16, j = w.y & 0xffff;
  const double2 pp = P.fpar[w.x];
  const bool is_or = factor_is_or(P, w.x);
  double b1 = 1.0, b2 = 1.0, o0, o1;
  if (!is_or) {
    f_row_long<0>(P, p - j, d, j, pp, b1, b2);
    if (j == 0) head_message<0>(pp.x, pp.y, b1, b2, o0, o1);
    else body_message<0>(pp.x, pp.y, b1, b2, o0, o1);
  } else {
    f_row_long<1>(P, p - j, d, j, pp, b1, b2);
    if (j == 0) head_message<1>(pp.x, pp.y, b1, b2, o0, o1);
    else body_message<1>(pp.x, pp.y, b1, b2, o0, o1);
  }
  group = (is_or ? 2 : 0) + (j == 0 ? 1 : 0);
  deg = d;
  return add(o0, o1);
}

// total of internal variable v's marginal (full row, clamps last)
__device__ double attr_marg_total(const KParams &P, int v) {
  const int r = P.vrow[v], d = P.vrow[v + 1] - r;
  double a0 = 1.0, a1 = 1.0, q0 = 1.0, q1 = 1.0;
  v_row_long(P, r, d, -1, true, a0, a1, q0, q1);
  const unsigned code = P.ev ? P.ev[v] : 0u;
  if (code) apply_clamp(code, q0, q1);
  return add(q0, q1);
}

// IEEE order as an unsigned order (negative totals sort first)
__device__ __forceinline__ unsigned long long ord_key(double t) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(t);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// mode 0: vtof targets list[0..n) (canonical edges, batch order); 1: ftov
// targets; 2: the marginal pass (n = V, position = original variable id).
// nclamp: clamp factors per original variable (evidence codes: each adds a
// slot to its variable's row) or null. tk/sk: [4] per ftov group.
__global__ void __launch_bounds__(256) uf_attr_kernel(const __grid_constant__ KParams P, int mode,
                                                      const int *list, int n, int it,
                                                      const int *nclamp, unsigned long long *tk,
                                                      unsigned long long *sk, int second) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t;
  int group = 0, rowlen, pos = i;
  if (mode == 0) {
    const int pv = P.canon2v[list[i]];
    int v;
    t = attr_vtof_total(P, P.vtof_twin[pv], it, v);
    rowlen = (P.vrow[v + 1] - P.vrow[v]) + (nclamp ? nclamp[P.vorig[v]] : 0);
  } else if (mode == 1) {
    t = attr_ftov_total(P, P.canon2v[list[i]], group, rowlen);
  } else {
    t = attr_marg_total(P, i);
    pos = P.vorig[i];
    rowlen = (P.vrow[i + 1] - P.vrow[i]) + (nclamp ? nclamp[pos] : 0);
  }
  if (t != t) return;  // a NaN total never wins (and suppresses the raise, host side)
  const unsigned long long key = ord_key(t);
  if (!second)
    atomicMin(&tk[group], key);
  else if (key == tk[group])
    atomicMin(&sk[group], ((unsigned long long)(0xFFFFFFFFu - (unsigned)rowlen) << 32) | (unsigned)pos);
}

// Alarm ranking of the last run (ranking.py:83-91): the selection's unlabeled
// variables (no evidence code) by descending P1, ties by ascending position
// in the id-sorted selection. One CTA. topk == 1: an argmax reduction;
// otherwise topk_select (radix select of the k-th key, then a sort of k).
__global__ void __launch_bounds__(1024) rank_kernel(const double2 *marg, const unsigned char *ev,
                                                    const int *vinv, const int *sel, int nsel,
                                                    int npow2, int kpow2, int topk, int *ranked,
                                                    double *p1_out) {
  extern __shared__ unsigned char smem[];
  unsigned long long *cache = (unsigned long long *)smem;
  unsigned long long *key = cache + npow2;
  int *pos = (int *)(key + kpow2);
  auto key_of = [&](int i) -> unsigned long long {
    if (i >= nsel) return ~0ull;
    const int v = sel[i];
    if (ev && ev[vinv[v]]) return ~0ull;
    return rank_key(marg[v].y);
  };
  if (topk == 1) {
    unsigned long long best = ~0ull;
    int bpos = 0x7fffffff;
    for (int i = threadIdx.x; i < nsel; i += blockDim.x) {
      const unsigned long long k = key_of(i);
      if (k < best || (k == best && i < bpos)) {
        best = k;
        bpos = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int p2 = __shfl_xor_sync(0xffffffffu, bpos, o);
      if (k2 < best || (k2 == best && p2 < bpos)) {
        best = k2;
        bpos = p2;
      }
    }
    __shared__ unsigned long long wk[32];
    __shared__ int wp[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
      wk[warp] = best;
      wp[warp] = bpos;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < (int)(blockDim.x >> 5) ? wk[lane] : ~0ull;
      bpos = lane < (int)(blockDim.x >> 5) ? wp[lane] : 0x7fffffff;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, bpos, o);
        if (k2 < best || (k2 == best && p2 < bpos)) {
          best = k2;
          bpos = p2;
        }
      }
      if (lane == 0) {
        const bool any = best != ~0ull;
        ranked[0] = any ? sel[bpos] : -1;
        if (p1_out) p1_out[0] = any ? marg[sel[bpos]].y : 0.0;
      }
    }
    return;
  }
  topk_select(key_of, nsel, topk, npow2, kpow2, cache, key, pos);
  for (int i = threadIdx.x; i < topk; i += blockDim.x) {
    const bool ok = key[i] != ~0ull;
    ranked[i] = ok ? sel[pos[i]] : -1;
    if (p1_out) p1_out[i] = ok ? marg[sel[pos[i]]].y : 0.0;
  }
}

__global__ void evidence_kernel(unsigned char *ev, const int *vinv, const int *var,
                                const signed char *val, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t pos = (size_t)vinv[var[i]];
  unsigned *word = (unsigned *)(ev + (pos & ~(size_t)3));
  atomicOr(word, (val[i] ? 2u : 1u) << (8 * (pos & 3)));
}

__global__ void division_selftest_kernel(const double *a, const double *b, double *qf, double *qr,
                                         long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y;
  div2_rn(a[i], a[(i + 1) % n], b[i], x, y);
  qf[2 * i] = x;
  qf[2 * i + 1] = y;
  qr[2 * i] = __ddiv_rn(a[i], b[i]);
  qr[2 * i + 1] = __ddiv_rn(a[(i + 1) % n], b[i]);
}

}  // namespace hbp

// ======================================================================================
// host side: handles + C ABI

namespace {
thread_local int64_t g_last_launches = 0;
}  // namespace

namespace hbp {
void set_last_launches(int64_t n) { g_last_launches = n; }
void add_last_launches(int64_t n) { g_last_launches += n; }
}  // namespace hbp

namespace {

constexpr size_t kCtrlHeader = 512;
static_assert(sizeof(hbp::Ctrl) <= kCtrlHeader, "control header");

struct CtrlView {
  hbp::Ctrl *ctrl;
  unsigned long long *delta_bits, *uf_where;
  int *uf_msg, *uf_marg, *uf_mwhere, *tflag;
};

CtrlView ctrl_view(void *base, size_t n) {
  CtrlView c;
  char *p = (char *)base;
  c.ctrl = (hbp::Ctrl *)p;
  p += kCtrlHeader;
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

size_t ctrl_bytes(size_t n) { return kCtrlHeader + n * (8 + 8 + 4 + 4 + 4 + 4); }

hbp::KParams base_params(hbp_graph *g) {
  hbp::KParams P{};
  P.vrow = g->d_vrow;
  P.frow = g->d_frow;
  P.vslot = g->d_vslot;
  P.fslot = g->d_fslot;
  P.fpar = g->d_fpar;
  P.vtof_twin = g->d_vtof_twin;
  P.ftov_twin = g->d_ftov_twin;
  P.vorig = g->d_vorig;
  P.canon2v = g->d_canon2v;
  P.V = g->L.V;
  P.F = g->L.F;
  P.E = (int)g->L.E;
  P.f_or_light = g->L.f_or_light;
  P.f_heavy = g->L.f_heavy;
  P.f_or_heavy = g->L.f_or_heavy;
  P.vtof = g->d_vtof;
  P.ftov = g->d_ftov;
  P.marg = g->d_marg;
  P.p0 = g->d_prev;
  P.normalize = 1;
  P.csize = 1;
  // chunk classes of the whole-node phases (exec_phase list == 2), dearest
  // first: huge-node slots, light nodes of degree kNodeMax..2, lane groups
  // of degree kClassMax..kNodeMax+1, degree 1 last (for the factors: the
  // unary ones, whose constant messages are only computed in iteration 1)
  {
    using hbp::ChunkClass;
    const hbp::HostLayout &L = g->L;
    // HBP_GROUP_MIN (A/B): the smallest degree processed as lane groups
    const int KC = hbp::kClassMax, KN = HBP_GROUP_MIN - 1;
    auto push = [](ChunkClass *cc, int &n, int &chunks, int d, int kind, int style, int node,
                   int cnt, int row) {
      if (cnt <= 0) return;
      ChunkClass c;
      c.chunk_begin = chunks;
      c.node_begin = node;
      c.node_end = style == 2 ? row + cnt : node + cnt;
      c.row_begin = row;
      c.info = (style == 2 ? 0 : d) | kind << 16 | style << 20;
      const int per = style == 1 ? 32 / d : 32;
      c.grp = style == 1 ? per | ((65536 + d - 1) / d) << 8 : 0;
      chunks += (cnt + per - 1) / per;
      cc[n++] = c;
    };
    P.nvcc = P.vchunks = 0;
    push(P.vcc, P.nvcc, P.vchunks, 0, 0, 2, L.vcls_node[KC + 1], L.vcls_cnt[KC + 1], L.vcls_row[KC + 1]);
    for (int d = KN; d >= 2; --d)
      push(P.vcc, P.nvcc, P.vchunks, d, 0, 0, L.vcls_node[d], L.vcls_cnt[d], L.vcls_row[d]);
    for (int d = KC; d > KN; --d)
      push(P.vcc, P.nvcc, P.vchunks, d, 0, 1, L.vcls_node[d], L.vcls_cnt[d], L.vcls_row[d]);
    push(P.vcc, P.nvcc, P.vchunks, 1, 0, 0, L.vcls_node[1], L.vcls_cnt[1], L.vcls_row[1]);
    P.nfcc = P.fchunks = 0;
    for (int k = 0; k < 2; ++k)
      push(P.fcc, P.nfcc, P.fchunks, 0, k, 2, L.fcls_node[k][KC + 1], L.fcls_cnt[k][KC + 1],
           L.fcls_row[k][KC + 1]);
    for (int d = KN; d >= 2; --d)
      for (int k = 0; k < 2; ++k)
        push(P.fcc, P.nfcc, P.fchunks, d, k, 0, L.fcls_node[k][d], L.fcls_cnt[k][d], L.fcls_row[k][d]);
    for (int d = KC; d > KN; --d)
      for (int k = 0; k < 2; ++k)
        push(P.fcc, P.nfcc, P.fchunks, d, k, 1, L.fcls_node[k][d], L.fcls_cnt[k][d], L.fcls_row[k][d]);
    P.fchunks_nounary = P.fchunks;
    for (int k = 0; k < 2; ++k)
      push(P.fcc, P.nfcc, P.fchunks, 1, k, 0, L.fcls_node[k][1], L.fcls_cnt[k][1], L.fcls_row[k][1]);
  }
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
  HBP_CUDA(cudaMemsetAsync(c.ctrl, 0, kCtrlHeader, s));
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
  hbp_status st;
  g->device = device;
  HBP_CUDA(cudaSetDevice(device));
  HBP_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
  g->stream = g->own_stream;
  HBP_CUDA(cudaEventCreate(&g->ev0));
  HBP_CUDA(cudaEventCreate(&g->ev1));
  HBP_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
  int per_sm = 0;
  // one CTA of 768 threads per SM (80 registers). Measured on B200 against
  // 512 (108 registers), 1024 (64 registers, spills) and 2 x 512 per SM: 768
  // is best for PARALL and levelled schedules alike.
  g->threads = hbp::kThreads;
  g->kernel = (const void *)hbp::lbp_persistent<hbp::kThreads, false>;
  g->kernel_fused = (const void *)hbp::lbp_persistent<hbp::kFusedThreads, true>;
  g->kernel_parall = (const void *)hbp::lbp_parall<hbp::kParallThreads, true>;
  g->kernel_parall_nonorm = (const void *)hbp::lbp_parall<hbp::kParallThreads, false>;
  HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, g->kernel, g->threads, 0));
  g->coop_blocks = std::max(1, per_sm) * g->num_sms;
  HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, g->kernel_fused,
                                                         hbp::kFusedThreads, 0));
  g->coop_blocks_fused = std::max(1, per_sm) * g->num_sms;
  HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, g->kernel_parall,
                                                         hbp::kParallThreads, 0));
  g->coop_blocks_parall = std::max(1, per_sm) * g->num_sms;
  g->kernel_pslot = (const void *)hbp::lbp_pslot<hbp::kPslotThreads, true>;
  g->kernel_pslot_nonorm = (const void *)hbp::lbp_pslot<hbp::kPslotThreads, false>;
  HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, g->kernel_pslot,
                                                         hbp::kPslotThreads, 0));
  g->coop_blocks_pslot = std::max(1, per_sm) * g->num_sms;
  // the layout is built on the device (layout_dev.cu); the host copy of it
  // only when a host-side consumer needs it (hbp::ensure_host_layout)
  hbp::set_last_launches(0);
  if ((st = hbp::build_layout_device(*desc, g.get())) != HBP_OK) return st;
  HBP_CUDA(cudaStreamSynchronize(g->stream));
  *out = g.release();
  return HBP_OK;
}

void hbp_graph_destroy(hbp_graph *g) { delete g; }

hbp_status hbp_graph_set_stream(hbp_graph *g, void *stream) {
  if (!g) {
    hbp::set_error("null graph");
    return HBP_EINVAL;
  }
  g->stream = stream ? (cudaStream_t)stream : g->own_stream;
  return HBP_OK;
}

hbp_status hbp_graph_layout(hbp_graph *g, int64_t *rowptr_ftov, int64_t *ftov_to_vtof) {
  // reference layout (storage.py:55-63) recomputed from the device-side maps
  hbp_status st = hbp::ensure_host_layout(g);
  if (st != HBP_OK) return st;
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

static hbp_status plan_create(hbp_graph *g, int64_t k, const int64_t *s_off, const int32_t *s_edges,
                              const int64_t *t_off, const int32_t *t_edges, bool fuse,
                              hbp_plan **out);

// lbp_pslot's slot chunks and second buffers, built once per graph
static hbp_status ensure_pslot(hbp_graph *g) {
  if (g->d_srec) return HBP_OK;
  return hbp::build_pslot_device(g);
}

hbp_status hbp_plan_create(hbp_graph *g, int64_t k, const int64_t *s_off, const int32_t *s_edges,
                           const int64_t *t_off, const int32_t *t_edges, hbp_plan **out) {
  if (!g || !out) {
    hbp::set_error("null argument");
    return HBP_EINVAL;
  }
  // HBP_FUSE=0 (A/B): every level as two phases
  const char *fe = getenv("HBP_FUSE");
  return plan_create(g, k, s_off, s_edges, t_off, t_edges, !(fe && atoi(fe) == 0), out);
}

static hbp_status plan_create(hbp_graph *g, int64_t k, const int64_t *s_off, const int32_t *s_edges,
                              const int64_t *t_off, const int32_t *t_edges, bool fuse,
                              hbp_plan **out) {
  *out = nullptr;
  std::unique_ptr<hbp_plan> p(new (std::nothrow) hbp_plan());
  if (!p) return HBP_ENOMEM;
  p->g = g;
  // levels below this many items run on CTA 0 alone (HBP_SMALL: A/B)
  const char *se = getenv("HBP_SMALL");
  const int32_t small = se ? atoi(se) : 3072;
  HBP_CUDA(cudaSetDevice(g->device));
  hbp_status st;
  bool parall = false;
  // HBP_GROUPING=1|0 (A/B of the message grouping, see build_plan): slot items
  // in degree order / in EdgeId order instead of whole degree-sorted nodes
  const char *ge = getenv("HBP_GROUPING");
  const int grouping = ge ? std::max(0, std::min(2, atoi(ge))) : 2;
  // a one-batch schedule of PARALL shape is recognised on the device and
  // needs no host layout; anything else is planned by the host builder
  if (grouping == 2 && k == 1 && s_off && t_off && s_off[0] == 0 && t_off[0] == 0 && s_off[1] >= 0 && t_off[1] >= 0 &&
      (st = hbp::parall_check_device(g, s_off[1], s_edges, t_off[1], t_edges, &parall)) != HBP_OK)
    return st;
  if (parall) {
    hbp::parall_plan(g->L, s_off[1], t_off[1], p->host, small);
  } else {
    if ((st = hbp::ensure_host_layout(g)) != HBP_OK) return st;
    if ((st = hbp::build_plan(g->L, k, s_off, s_edges, t_off, t_edges, p->host, small,
                              grouping, fuse)) != HBP_OK)
      return st;
  }
  cudaStream_t s = g->stream;
  if ((st = upload(&p->d_phases, p->host.phases, s)) || (st = upload(&p->d_items, p->host.items, s)) ||
      (st = upload(&p->d_fitems, p->host.fitems, s)))
    return st;
#if HBP_ITEM_WORDS
  // the slot word and twin of every list item of a small phase, beside the
  // item: the tight loop then loads both at once instead of item -> slot word
  if (!parall) {
    const hbp::HostLayout &L = g->L;
    std::vector<int32_t> iw(4 * std::max<size_t>(1, p->host.items.size()), 0);
    bool any = false;
    for (const auto &ph : p->host.phases) {
      if (ph.list != 1 || ph.grid || (ph.type != 0 && ph.type != 1)) continue;
      for (int32_t i = ph.begin; i < ph.end; ++i) {
        const int32_t q = p->host.items[i] & (hbp::kWriteBit - 1);
        int32_t *w = &iw[4 * (size_t)i];
        if (ph.type == 0) {
          w[0] = L.vslot[2 * (size_t)q];
          w[1] = L.vslot[2 * (size_t)q + 1];
          w[2] = (int32_t)L.ftov_twin[q];
        } else {
          w[0] = L.fslot[2 * (size_t)q];
          w[1] = L.fslot[2 * (size_t)q + 1];
          w[2] = L.vtof_twin[q];
        }
        any = true;
      }
    }
    if (any && (st = upload(&p->d_iw, iw, s))) return st;
  }
#endif
  // keep the schedule in its reference order for the underflow attribution
  // (a PARALL-shape batch is already on the device: the shape test's copy)
  {
    const int64_t ns = k > 0 ? s_off[k] : 0, nt = k > 0 ? t_off[k] : 0;
    p->ns = ns;
    if (k > 0) {
      p->s_off.assign(s_off, s_off + k + 1);
      p->t_off.assign(t_off, t_off + k + 1);
    }
    HBP_CUDA(cudaMallocAsync((void **)&p->d_sched, (size_t)std::max<int64_t>(1, ns + nt) * 4, s));
    if (parall) {
      HBP_CUDA(cudaMemcpyAsync(p->d_sched, g->d_scratch, (size_t)(ns + nt) * 4,
                               cudaMemcpyDeviceToDevice, s));
    } else {
      if (ns) HBP_CUDA(cudaMemcpyAsync(p->d_sched, s_edges, (size_t)ns * 4, cudaMemcpyHostToDevice, s));
      if (nt)
        HBP_CUDA(cudaMemcpyAsync(p->d_sched + ns, t_edges, (size_t)nt * 4, cudaMemcpyHostToDevice, s));
    }
  }
  // kernel instance: plans with fused levels run the FUSED instance
  const bool fused = p->host.n_fused > 0;
  const auto &phs = p->host.phases;
  const bool two_phase = phs.size() == 2 && phs[0].list == 2 && phs[1].list == 2;
  p->kernel = fused ? g->kernel_fused : two_phase ? g->kernel_parall : g->kernel;
  p->kernel_nonorm = two_phase ? g->kernel_parall_nonorm : p->kernel;
  p->threads = fused ? hbp::kFusedThreads : two_phase ? hbp::kParallThreads : g->threads;
  int coop = fused ? g->coop_blocks_fused : two_phase ? g->coop_blocks_parall : g->coop_blocks;
  // PARALL as one phase per iteration (lbp_pslot) when every factor fits a
  // warp and no variable has more than kClassMax factors (no huge nodes;
  // the lane records hold degrees and row indices in 8 bits); HBP_PSLOT=0 (A/B) keeps the two-phase kernel,
  // which also serves the underflow attribution replay (fuse == false)
  {
    const char *pe = getenv("HBP_PSLOT");
    const hbp::HostLayout &L = g->L;
    if (two_phase && fuse && !(pe && atoi(pe) == 0) && L.fcls_cnt[0][hbp::kClassMax + 1] == 0 &&
        L.fcls_cnt[1][hbp::kClassMax + 1] == 0 && L.vcls_cnt[hbp::kClassMax + 1] == 0) {
      if ((st = ensure_pslot(g)) != HBP_OK) return st;
      p->pslot = true;
      p->kernel = g->kernel_pslot;
      p->kernel_nonorm = g->kernel_pslot_nonorm;
      p->threads = hbp::kPslotThreads;
      coop = g->coop_blocks_pslot;
    }
  }
  // small levels on a thread-block cluster of csize CTAs (HBP_CSIZE, A/B)
  p->csize = 1;
  if (const char *ce = getenv("HBP_CSIZE")) p->csize = std::max(1, std::min(8, atoi(ce)));
  bool has_small = false;
  for (const auto &ph : p->host.phases) has_small |= !ph.grid;
  if (!has_small) p->csize = 1;
  if (p->csize > 1) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p->csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(coop / p->csize * p->csize);
    cfg.blockDim = dim3(p->threads);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    HBP_CUDA(cudaOccupancyMaxActiveClusters(&nclusters, p->kernel, &cfg));
    coop = std::max(1, nclusters) * p->csize;
  }
  // grid: enough CTAs for the largest grid-wide phase, at most one wave
  int64_t big = 0;
  for (const auto &ph : p->host.phases)
    if (ph.grid)
      big = std::max<int64_t>(big, (ph.end - ph.begin) + (ph.list == 2 ? ph.send - ph.sbegin : 0));
  int64_t want = (big + p->threads - 1) / p->threads;
  if (big < 2 * p->threads) want = 1;
  want = std::max<int64_t>(want, p->csize);
  p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, coop));
  // lbp_pslot: about 8 chunks per CTA, so a small graph spreads over SMs
  // instead of one CTA's issue slots (C1: 1 CTA 0.576 ms, 8-16 CTAs 0.39 ms;
  // every grid-wide barrier is the same one per iteration either way)
  if (p->pslot)
    p->grid = (int)std::max<int64_t>(1, std::min<int64_t>((g->pslot_chunks + 7) / 8, coop));
  if (const char *ge = getenv("HBP_GRID"))  // A/B: force the CTA count
    p->grid = std::max(1, std::min(atoi(ge), coop));
  // lbp_pslot on at most 8 CTAs: the grid is launched as ONE thread-block
  // cluster and the iteration barrier is the hardware cluster barrier instead
  // of the global-memory counter (HBP_PSLOT_CLUSTER=0: the counter, A/B)
  if (p->pslot && p->grid > 1 && p->grid <= 8) {
    const char *pc = getenv("HBP_PSLOT_CLUSTER");
    if (!(pc && atoi(pc) == 0)) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = p->grid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(p->grid);
      cfg.blockDim = dim3(p->threads);
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, p->kernel, &cfg) == cudaSuccess && nclusters >= 1)
        p->csize = p->grid;
      cudaGetLastError();
    }
  }
  p->grid = std::max(p->csize, p->grid / p->csize * p->csize);
  HBP_CUDA(cudaStreamSynchronize(s));
  *out = p.release();
  return HBP_OK;
}

void hbp_plan_destroy(hbp_plan *p) { delete p; }

static hbp_status launch_kernel(hbp_plan *p, hbp::KParams &P);
static hbp_status attribute_underflow(hbp_plan *p, const hbp::KParams &P0, int it, size_t nctrl,
                               hbp_result *res);
static hbp_status attribute_pass(hbp_graph *g, const hbp::KParams &P, int mode, const int *list, int n,
                          int it, int *kind, int64_t *index, int *group_out = nullptr);

// Evidence codes (hbp_graph_set_evidence) equal clamp_evidence only when the
// clamped graph's schedule is the base schedule with the clamp edges appended
// to the LAST batch (their ftov messages then first matter from iteration 2,
// which is what the codes implement): true for a one-batch schedule (PARALL:
// the clamp edges relate to nothing) and for canonical SEQFIX (the clamp
// edges end the chain), SURVEY.md 8(a) A2. Any other plan is refused.
static hbp_status evidence_eligible(hbp_plan *p, bool *ok) {
  if (p->ev_ok < 0) {
    const int64_t k = (int64_t)p->s_off.size() - 1;
    if (k <= 1) {
      p->ev_ok = 1;
    } else {
      hbp_graph *g = p->g;
      hbp_status st = hbp::ensure_host_layout(g);
      if (st != HBP_OK) return st;
      const hbp::HostLayout &L = g->L;
      const int64_t E = L.E;
      std::vector<int32_t> before((size_t)std::max<int64_t>(0, E - 1)), after(before.size()),
          rank((size_t)E);
      for (int64_t e = 0; e < E; ++e) rank[(size_t)e] = (int32_t)e;
      for (int64_t e = 0; e + 1 < E; ++e) {
        before[(size_t)e] = (int32_t)e;
        after[(size_t)e] = (int32_t)(e + 1);
      }
      hbp_graph_desc d{L.V, L.F, E, L.rowptr.data(), L.edge_var.data(), L.kind.data(),
                       L.p1.data(), L.p2.data()};
      hbp::Schedule canon;
      int64_t cyc = -1;
      if ((st = hbp::compile(d, (int64_t)before.size(), before.data(), after.data(), rank.data(),
                             canon, &cyc)) != HBP_OK)
        return st;
      bool same = canon.s_off == p->s_off && canon.t_off == p->t_off;
      if (same) {
        std::vector<int32_t> mine((size_t)(p->ns + p->t_off.back()));
        if (!mine.empty())
          HBP_CUDA(cudaMemcpy(mine.data(), p->d_sched, mine.size() * 4, cudaMemcpyDeviceToHost));
        same = std::equal(canon.s_edges.begin(), canon.s_edges.end(), mine.begin()) &&
               std::equal(canon.t_edges.begin(), canon.t_edges.end(), mine.begin() + p->ns);
      }
      p->ev_ok = same ? 1 : 0;
    }
  }
  *ok = p->ev_ok == 1;
  return HBP_OK;
}

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
  if (opt->precision != 0) {
    hbp::set_error("the single-graph executor runs fp64 only (fp32 mode: hbp_sweep_run)");
    return HBP_EINVAL;
  }
  HBP_CUDA(cudaSetDevice(g->device));
  const size_t n = (size_t)opt->max_iterations + 2;
  hbp_status st = HBP_OK;
  if (g->has_ev) {
    bool ok = false;
    if ((st = evidence_eligible(p, &ok))) return st;
    if (!ok) {
      hbp::set_error("graph evidence needs a PARALL or canonical SEQFIX plan (the schedules "
                     "clamp_evidence leaves unchanged); clamp the graph and compile instead");
      return HBP_EINVAL;
    }
  }
  st = ensure_ctrl(g, n);
  if (st) return st;
  if ((st = reset_ctrl(g, n))) return st;
  // record_history: the device keeps the marginals of the first hist_iters
  // iterations, a buffer sized by a budget rather than by max_iterations
  // (the reference appends only the iterations that run, engine.py:574-575);
  // a run that goes beyond it is re-run -- deterministically -- with a buffer
  // of exactly its iteration count
  double2 *hist = nullptr;
  int hist_iters = 0;
  auto ensure_hist = [&](int iters) -> hbp_status {
    const size_t need = (size_t)iters * (size_t)std::max(1, g->L.V);
    if (g->hist_cap < need) {
      if (g->d_hist) cudaFree(g->d_hist);
      g->d_hist = nullptr;
      g->hist_cap = 0;
      HBP_CUDA(cudaMalloc(&g->d_hist, need * sizeof(double2)));
      g->hist_cap = need;
    }
    hist = g->d_hist;
    hist_iters = iters;
    return HBP_OK;
  };
  if (opt->record_history) {
    const size_t per_it = (size_t)std::max(1, g->L.V) * sizeof(double2);
    const int budget = (int)std::max<size_t>(32, ((size_t)256 << 20) / per_it);
    if ((st = ensure_hist(std::min(opt->max_iterations, budget)))) return st;
  }
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  hbp::KParams P = base_params(g);
  P.phases = p->d_phases;
  P.nphases = (int)p->host.phases.size();
  P.items = p->d_items;
  P.fitems = (const int4 *)p->d_fitems;
  P.iw = (const int4 *)p->d_iw;
  P.ctrl = c.ctrl;
  P.delta_bits = c.delta_bits;
  P.uf_msg = c.uf_msg;
  P.uf_marg = c.uf_marg;
  P.uf_mwhere = c.uf_mwhere;
  P.uf_where = c.uf_where;
  P.tflag = c.tflag;
  P.hist = hist;
  P.hist_iters = hist_iters;
  P.ev = g->has_ev ? g->d_ev : nullptr;
  P.trace = nullptr;
  if (getenv("HBP_TRACE")) {
    const size_t n_tr = (size_t)hbp::kTraceIters * P.nphases * p->grid * 2 + 2 * hbp::kChunkTrace;
    if (g->trace_cap < n_tr) {
      if (g->d_trace) cudaFree(g->d_trace);
      HBP_CUDA(cudaMalloc(&g->d_trace, n_tr * 8));
      g->trace_cap = n_tr;
    }
    HBP_CUDA(cudaMemsetAsync(g->d_trace, 0, n_tr * 8, g->stream));
    P.trace = g->d_trace;
  }
  P.max_it = opt->max_iterations;
  P.normalize = opt->normalize_messages ? 1 : 0;
  P.tol = opt->tolerance;
  P.time_limit_ns = opt->time_limit > 0 ? (long long)(opt->time_limit * 1e9) : 0;
  if (opt->time_limit > 0 && P.time_limit_ns == 0) P.time_limit_ns = 1;
  P.csize = p->csize;
  P.halt_it = 0;
  P.halt_phase = 0;
  if (p->pslot) {
    P.fchunks = g->pslot_chunks;
    P.fchunks_nounary = g->pslot_chunks_nounary;
    P.srec = g->d_srec;
    P.sinfo = g->d_sinfo;
    P.ftov_alt = g->d_ftov_alt;
    P.p0_alt = g->d_p0_alt;
  }
  HBP_CUDA(cudaEventRecord(g->ev0, g->stream));
  if ((st = launch_kernel(p, P))) return st;
  HBP_CUDA(cudaEventRecord(g->ev1, g->stream));
  g_last_launches = 1;
  hbp::Ctrl hc;
  HBP_CUDA(cudaMemcpyAsync(&hc, c.ctrl, sizeof(hc), cudaMemcpyDeviceToHost, g->stream));
  HBP_CUDA(cudaStreamSynchronize(g->stream));
  if (hist && hc.stop != 4 && hc.iterations > hist_iters) {
    if ((st = ensure_hist(hc.iterations))) return st;
    P.hist = hist;
    P.hist_iters = hist_iters;
    if ((st = reset_ctrl(g, n))) return st;
    HBP_CUDA(cudaEventRecord(g->ev0, g->stream));
    if ((st = launch_kernel(p, P))) return st;
    HBP_CUDA(cudaEventRecord(g->ev1, g->stream));
    g_last_launches = 2;
    HBP_CUDA(cudaMemcpyAsync(&hc, c.ctrl, sizeof(hc), cudaMemcpyDeviceToHost, g->stream));
    HBP_CUDA(cudaStreamSynchronize(g->stream));
  }
  g->hist_valid = hist ? std::min(hc.iterations, hist_iters) : 0;
  float ms = 0;
  HBP_CUDA(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  std::memset(res, 0, sizeof(*res));
  res->iterations = hc.iterations;
  res->converged = hc.converged;
  res->device_ms = ms;
  std::memcpy(&res->last_delta, &hc.last_delta, 8);
  if (hc.stop == 4) {
    if (p->host.n_fused > 0 || p->pslot) {
      // the attribution replays the failing pass group by group (engine.py:
      // 566-570), which needs the two-phase form of every level: re-run the
      // same schedule unfused -- bitwise the same run -- and attribute there
      if (!p->unfused) {
        const int64_t kb = (int64_t)p->s_off.size() - 1;
        std::vector<int32_t> edges((size_t)(p->ns + (kb > 0 ? p->t_off[kb] : 0)));
        if (!edges.empty())
          HBP_CUDA(cudaMemcpy(edges.data(), p->d_sched, edges.size() * 4, cudaMemcpyDeviceToHost));
        hbp_plan *u = nullptr;
        if ((st = plan_create(g, kb, p->s_off.data(), edges.data(), p->t_off.data(),
                              edges.data() + p->ns, false, &u)))
          return st;
        p->unfused = u;
      }
      p->unfused->ev_ok = p->ev_ok;
      return launch_run(p->unfused, opt, res);
    }
    if ((st = attribute_underflow(p, P, hc.iterations, n, res))) return st;
    hbp::set_error("underflow");
    return HBP_EUNDERFLOW;
  }
  return HBP_OK;
}

static hbp_status launch_kernel(hbp_plan *p, hbp::KParams &P) {
  void *args[] = {&P};
  if (p->csize > 1) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = p->csize;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.gridDim = dim3(p->grid);
    cfg.blockDim = dim3(p->threads);
    cfg.stream = p->g->stream;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    HBP_CUDA(cudaLaunchKernelExC(&cfg, P.normalize ? p->kernel : p->kernel_nonorm, args));
  } else {
    HBP_CUDA(cudaLaunchCooperativeKernel(P.normalize ? p->kernel : p->kernel_nonorm, dim3(p->grid),
                                         dim3(p->threads), args, 0, p->g->stream));
  }
  return HBP_OK;
}

// Reference store position of canonical edge e's factor-to-variable message
// in the (clamped) graph: storage.py:55-63's variable-major transpose, where
// each clamp factor appends one slot at the END of its variable's row
// (graph.py:189-200), shifting every later variable's row.
static hbp_status ref_ftov_position(hbp_graph *g, int32_t e, int64_t *pos) {
  hbp_status st = hbp::ensure_host_layout(g);
  if (st != HBP_OK) return st;
  const hbp::HostLayout &L = g->L;
  int64_t q = -1;
  for (int64_t i = 0; i < L.E && q < 0; ++i)
    if (L.ref_ftov[i] == e) q = i;
  const int32_t v = L.edge_var[e];
  for (int32_t cv : g->ev_var) q += cv < v;
  *pos = q;
  return HBP_OK;
}

// The exact reference underflow report of a run that stopped on underflow at
// iteration it (engine.py:155-165, :512-518; see uf_attr_kernel).
static hbp_status attribute_underflow(hbp_plan *p, const hbp::KParams &P0, int it, size_t nctrl,
                               hbp_result *res) {
  hbp_graph *g = p->g;
  cudaStream_t s = g->stream;
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  int um = 0;
  unsigned long long where = ~0ull;
  HBP_CUDA(cudaMemcpyAsync(&um, c.uf_msg + it, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(&where, c.uf_where + it, 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  // messages fail before the marginal of the same iteration; the earliest
  // failing phase is the key's high part
  const bool marg = um == 0;
  const int phase = marg ? 0 : (int)(where >> 33);
  hbp::KParams P = P0;
  P.halt_it = marg ? it + 1 : it;
  P.halt_phase = phase;
  P.time_limit_ns = 0;
  P.hist = nullptr;
  P.trace = nullptr;
  hbp_status st;
  if ((st = reset_ctrl(g, nctrl))) return st;
  if ((st = launch_kernel(p, P))) return st;
  int mode = 2, n = P.V;
  const int *list = nullptr;
  if (!marg) {
    const int b = p->host.phase_batch[phase];
    if (p->host.phases[phase].type == 0) {
      mode = 0;
      list = p->d_sched + p->ns + p->t_off[b];
      n = (int)(p->t_off[b + 1] - p->t_off[b]);
    } else {
      mode = 1;
      list = p->d_sched + p->s_off[b];
      n = (int)(p->s_off[b + 1] - p->s_off[b]);
    }
  }
  int kind = 0;
  int64_t index = -1;
  if ((st = attribute_pass(g, P, mode, list, n, it, &kind, &index))) return st;
  if (kind == 0) {
    hbp::set_error("internal: underflow flagged on the device but no reference pass fails");
    return HBP_ECUDA;
  }
  res->underflow_kind = kind;
  res->underflow_iteration = it;
  res->underflow_index = index;
  return HBP_OK;
}

// One attribution over a pass whose inputs are on the device (P's buffers):
// kind 0 = no group of the pass raises, else 1 vtof / 2 ftov / 3 marginal with
// the reference's index (vtof position = canonical edge, ftov store position,
// variable id). The ftov passes report the first failing group in
// _FTOV_RUNNERS order in *group_out (0..3) when non-null.
static hbp_status attribute_pass(hbp_graph *g, const hbp::KParams &P, int mode, const int *list, int n,
                          int it, int *kind, int64_t *index, int *group_out) {
  cudaStream_t s = g->stream;
  *kind = 0;
  *index = -1;
  if (group_out) *group_out = 4;
  if (n <= 0) return HBP_OK;
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  unsigned long long *tk = (unsigned long long *)((char *)c.ctrl + 256), *sk = tk + 4;
  HBP_CUDA(cudaMemsetAsync(tk, 0xFF, 64, s));
  int *d_nclamp = nullptr;
  if (g->has_ev && !g->ev_var.empty()) {
    std::vector<int> cnt((size_t)g->L.V, 0);
    for (int32_t v : g->ev_var) cnt[(size_t)v]++;
    HBP_CUDA(cudaMalloc(&d_nclamp, cnt.size() * 4));
    HBP_CUDA(cudaMemcpyAsync(d_nclamp, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice, s));
  }
  for (int second = 0; second < 2; ++second)
    hbp::uf_attr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, mode, list, n, it, d_nclamp,
                                                                   tk, sk, second);
  cudaError_t le = cudaGetLastError();
  unsigned long long h[8];
  cudaError_t ce = cudaMemcpyAsync(h, tk, 64, cudaMemcpyDeviceToHost, s);
  cudaError_t se = cudaStreamSynchronize(s);
  if (d_nclamp) cudaFree(d_nclamp);
  HBP_CUDA(le);
  HBP_CUDA(ce);
  HBP_CUDA(se);
  const int ngroups = mode == 1 ? 4 : 1;
  for (int grp = 0; grp < ngroups; ++grp) {
    if (h[grp] == ~0ull) continue;  // empty group (or only NaN totals)
    const unsigned long long u = h[grp];
    const unsigned long long bits = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
    double t;
    std::memcpy(&t, &bits, 8);
    if (!(t < hbp::dev::kMinMessageSum)) continue;
    const unsigned pos = (unsigned)(h[4 + grp] & 0xFFFFFFFFu);
    if (group_out) *group_out = grp;
    if (mode == 2) {
      *kind = 3;
      *index = pos;
      return HBP_OK;
    }
    int32_t e = 0;
    HBP_CUDA(cudaMemcpy(&e, list + pos, 4, cudaMemcpyDeviceToHost));
    if (mode == 0) {
      *kind = 1;
      *index = e;
      return HBP_OK;
    }
    *kind = 2;
    return ref_ftov_position(g, e, index);
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

hbp_status hbp_graph_history(hbp_graph *g, int32_t iterations, double *out) {
  if (!g || iterations < 0 || (iterations > 0 && !out)) {
    hbp::set_error("bad history arguments");
    return HBP_EINVAL;
  }
  if (iterations > g->hist_valid) {
    hbp::set_error("the last run recorded fewer iterations of history");
    return HBP_EINVAL;
  }
  if (iterations)
    HBP_CUDA(cudaMemcpy(out, g->d_hist, (size_t)iterations * g->L.V * 16, cudaMemcpyDeviceToHost));
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
  hbp_status hs = hbp::ensure_host_layout(g);
  if (hs != HBP_OK) return hs;
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
  std::vector<int32_t> items((size_t)n);
  for (int64_t i = 0; i < n; ++i)
    items[i] = direction == 0 ? (L.canon2f[targets[i]] | hbp::kWriteBit) : L.canon2v[targets[i]];
  hbp_status st = ensure_ctrl(g, 4);
  if (st) return st;
  if ((st = reset_ctrl(g, 4))) return st;
  int *d_items = nullptr;
  HBP_CUDA(cudaMalloc(&d_items, items.size() * 8));  // [slot items | canonical targets]
  cudaStream_t s = g->stream;
  HBP_CUDA(cudaMemcpyAsync(g->d_vtof, hv.data(), hv.size() * 16, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(g->d_ftov, hf.data(), hf.size() * 16, cudaMemcpyHostToDevice, s));
  HBP_CUDA(cudaMemcpyAsync(d_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice, s));
  CtrlView c = ctrl_view(g->d_ctrl, g->ctrl_cap);
  hbp::KParams P = base_params(g);
  P.normalize = normalize ? 1 : 0;
  P.uf_msg = c.uf_msg;
  P.uf_where = c.uf_where;
  P.uf_marg = c.uf_marg;
  P.uf_mwhere = c.uf_mwhere;
  hbp::pass_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, direction ? 1 : 0, 0, d_items,
                                                                (int)n);
  g_last_launches = 1;
  cudaError_t le = cudaGetLastError();
  int uf = 0;
  unsigned long long where = 0;
  cudaMemcpyAsync(&uf, c.uf_msg + 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&where, c.uf_where + 1, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hv.data(), g->d_vtof, hv.size() * 16, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hf.data(), g->d_ftov, hf.size() * 16, cudaMemcpyDeviceToHost, s);
  cudaError_t se = cudaStreamSynchronize(s);
  if (le != cudaSuccess || se != cudaSuccess) {
    cudaFree(d_items);
    hbp::set_error(std::string("pass kernel: ") + cudaGetErrorString(le != cudaSuccess ? le : se));
    return HBP_ECUDA;
  }
  // The reference raises in the first failing pass (engine.py:155-165): for
  // the vtof direction before any scatter; for the ftov direction after the
  // groups that precede the failing one (_FTOV_RUNNERS order) have scattered.
  int fail_group = 4;
  if (uf) {
    int kind = 0;
    int64_t index = -1;
    hbp_status ast = HBP_OK;
    if (cudaMemcpy(d_items + n, targets, (size_t)n * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(d_items);
      hbp::set_error("attribution upload failed");
      return HBP_ECUDA;
    }
    ast = attribute_pass(g, P, direction ? 1 : 0, d_items + n, (int)n, 1, &kind, &index, &fail_group);
    cudaFree(d_items);
    if (ast != HBP_OK) return ast;
    if (kind == 0) {
      hbp::set_error("internal: underflow flagged on the device but no reference pass fails");
      return HBP_ECUDA;
    }
    if (underflow_index) *underflow_index = index;
    if (direction == 0) {
      hbp::set_error("underflow");
      return HBP_EUNDERFLOW;  // store untouched: the reference raises before its scatter
    }
  } else {
    cudaFree(d_items);
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
      if (fail_group < 4) {  // (kind, head/body) group of e in _FTOV_RUNNERS order
        const int32_t f = L.edge_factor[e];
        const int grp = (L.kind[f] == 1 ? 2 : 0) + (e == L.rowptr[f] ? 1 : 0);
        if (grp >= fail_group) continue;
      }
      double2 m = hf[L.canon2f[e]];
      ftov0[ref_pos[e]] = m.x;
      ftov1[ref_pos[e]] = m.y;
    }
    if (fail_group < 4) {
      hbp::set_error("underflow");
      return HBP_EUNDERFLOW;
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
  hbp_status hs = hbp::ensure_host_layout(g);
  if (hs != HBP_OK) return hs;
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
  std::vector<int32_t> rows((size_t)L.V);
  for (int32_t vi = 0; vi < L.V; ++vi) rows[vi] = L.vrow[vi];
  int *d_rows = nullptr;
  HBP_CUDA(cudaMalloc(&d_rows, rows.size() * 4 + 4));
  HBP_CUDA(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s));
  hbp::pass_kernel<<<(unsigned)((L.V + 255) / 256), 256, 0, s>>>(P, 0, 1, d_rows, L.V);
  g_last_launches = 1;
  cudaError_t le = cudaGetLastError();
  cudaStreamSynchronize(s);
  cudaFree(d_rows);
  HBP_CUDA(le);
  int uf = 0, mw = 0;
  HBP_CUDA(cudaMemcpyAsync(&uf, c.uf_marg + 1, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(&mw, c.uf_mwhere + 1, 4, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaMemcpyAsync(out, g->d_marg, (size_t)L.V * 16, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  (void)mw;
  if (uf == 1) {  // bit1: a NaN total suppresses the raise (numpy min propagates NaN)
    int kind = 0;
    int64_t index = -1;
    if ((st = attribute_pass(g, P, 2, nullptr, L.V, 2, &kind, &index))) return st;
    if (kind != 3) {
      hbp::set_error("internal: underflow flagged on the device but no reference pass fails");
      return HBP_ECUDA;
    }
    if (underflow_var) *underflow_var = index;
    hbp::set_error("underflow");
    return HBP_EUNDERFLOW;
  }
  return HBP_OK;
}

hbp_status hbp_graph_set_evidence(hbp_graph *g, int32_t n, const int32_t *var,
                                  const int8_t *value) {
  if (!g || n < 0 || (n > 0 && (!var || !value))) {
    hbp::set_error("bad evidence arguments");
    return HBP_EINVAL;
  }
  const hbp::HostLayout &L = g->L;
  for (int32_t i = 0; i < n; ++i) {
    if (var[i] < 0 || var[i] >= L.V) {
      hbp::set_error("evidence variable out of range");
      return HBP_EINVAL;
    }
    if (value[i] != 0 && value[i] != 1) {
      hbp::set_error("evidence value must be 0 or 1");
      return HBP_EINVAL;
    }
  }
  HBP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  if (!g->d_ev) HBP_CUDA(cudaMalloc(&g->d_ev, (size_t)L.V + 4));
  HBP_CUDA(cudaMemsetAsync(g->d_ev, 0, (size_t)L.V + 4, s));
  g->has_ev = n > 0;
  g->ev_var.assign(var, var + n);
  g->ev_val.assign(value, value + n);
  if (n > 0) {
    const size_t need = (size_t)n * 5 + 16;
    if (g->ev_list_cap < need) {
      if (g->d_ev_list) cudaFree(g->d_ev_list);
      g->d_ev_list = nullptr;
      g->ev_list_cap = 0;
      HBP_CUDA(cudaMalloc(&g->d_ev_list, std::max<size_t>(need, 1 << 16)));
      g->ev_list_cap = std::max<size_t>(need, 1 << 16);
    }
    int *d_var = (int *)g->d_ev_list;
    signed char *d_val = (signed char *)(d_var + n);
    HBP_CUDA(cudaMemcpyAsync(d_var, var, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    HBP_CUDA(cudaMemcpyAsync(d_val, value, (size_t)n, cudaMemcpyHostToDevice, s));
    hbp::evidence_kernel<<<(n + 255) / 256, 256, 0, s>>>(g->d_ev, g->d_vinv, d_var, d_val, n);
    HBP_CUDA(cudaGetLastError());
  }
  // no host sync: the codes are consumed by the next run on the same stream
  // (the pageable sources were staged before cudaMemcpyAsync returned)
  return HBP_OK;
}

hbp_status hbp_graph_rank(hbp_graph *g, int32_t num_select, const int32_t *select, int32_t topk,
                          int32_t *ranked, double *p1) {
  if (!g || num_select < 0 || topk < 1 || (num_select > 0 && !select) || !ranked) {
    hbp::set_error("bad rank arguments");
    return HBP_EINVAL;
  }
  const hbp::HostLayout &L = g->L;
  for (int32_t k = 0; k < num_select; ++k)
    if (select[k] < 0 || select[k] >= L.V || (k && select[k] <= select[k - 1])) {
      hbp::set_error("selection must be ascending variable ids");
      return HBP_EINVAL;
    }
  // the shared-memory key cache of the top-k select (lbp_kernels.cuh)
  int npow2 = 2;
  while (npow2 < num_select && npow2 < hbp::dev::kRankCap) npow2 <<= 1;
  if (topk > 1 && topk >= hbp::dev::kRankCap) {
    hbp::set_error("device ranking returns at most 16383 alarms per call");
    return HBP_EINVAL;
  }
  HBP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  const size_t need = (size_t)num_select * 4 + (size_t)topk * 12 + 64;
  if (g->rank_cap < need) {
    if (g->d_rank) cudaFree(g->d_rank);
    g->d_rank = nullptr;
    g->rank_cap = 0;
    HBP_CUDA(cudaMalloc(&g->d_rank, need));
    g->rank_cap = need;
  }
  int *d_sel = (int *)g->d_rank;
  int *d_out = d_sel + num_select;
  double *d_p1 = (double *)(((uintptr_t)(d_out + topk) + 15) & ~(uintptr_t)15);
  if (num_select)
    HBP_CUDA(cudaMemcpyAsync(d_sel, select, (size_t)num_select * 4, cudaMemcpyHostToDevice, s));
  int kpow2 = 2;
  while (kpow2 < topk) kpow2 <<= 1;
  // the key cache shrinks when a large k takes the shared memory (it is
  // optional: without it the select recomputes the keys per pass)
  while (npow2 > 2 && (size_t)npow2 * 8 + (size_t)kpow2 * 12 > (size_t)200 * 1024) npow2 >>= 1;
  const size_t smem = topk == 1 ? 0 : (size_t)npow2 * 8 + (size_t)kpow2 * 12;
  if (smem > 48 * 1024)
    HBP_CUDA(cudaFuncSetAttribute(hbp::rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  hbp::rank_kernel<<<1, 1024, smem, s>>>(g->d_marg, g->has_ev ? g->d_ev : nullptr, g->d_vinv,
                                         d_sel, num_select, npow2, kpow2, topk, d_out, d_p1);
  HBP_CUDA(cudaGetLastError());
  HBP_CUDA(cudaMemcpyAsync(ranked, d_out, (size_t)topk * 4, cudaMemcpyDeviceToHost, s));
  if (p1) HBP_CUDA(cudaMemcpyAsync(p1, d_p1, (size_t)topk * 8, cudaMemcpyDeviceToHost, s));
  HBP_CUDA(cudaStreamSynchronize(s));
  return HBP_OK;
}

int64_t hbp_last_launch_count(void) { return g_last_launches; }

// Debug: phase count and grid size of a plan (not part of the public header).
void hbp_debug_plan_info(hbp_plan *p, int32_t *nphases, int32_t *grid, int32_t *threads,
                         int32_t *nfused) {
  *nphases = (int32_t)p->host.phases.size();
  if (nfused) *nfused = p->host.n_fused;
  *grid = p->grid;
  *threads = p->threads;
}

// 1 when the plan runs PARALL as one phase per iteration (lbp_pslot); debug only.
int32_t hbp_debug_plan_pslot(hbp_plan *p) { return p->pslot ? 1 : 0; }

// Debug timeline of the last run with HBP_TRACE=1 (not part of the public header).
int64_t hbp_debug_trace(hbp_plan *p, unsigned long long *out, int64_t cap) {
  hbp_graph *g = p->g;
  const int64_t n = (int64_t)hbp::kTraceIters * (int64_t)p->host.phases.size() * p->grid * 2 +
                    2 * hbp::kChunkTrace;
  if (!g->d_trace || cap < n) return -n;
  cudaMemcpy(out, g->d_trace, (size_t)n * 8, cudaMemcpyDeviceToHost);
  return n;
}

hbp_status hbp_selftest_division(int64_t n, const double *a, const double *b, double *q_fast,
                                 double *q_ref) {
  if (n <= 0 || !a || !b || !q_fast || !q_ref) {
    hbp::set_error("bad selftest arguments");
    return HBP_EINVAL;
  }
  double *d = nullptr;
  HBP_CUDA(cudaMalloc(&d, (size_t)n * 48));
  HBP_CUDA(cudaMemcpy(d, a, (size_t)n * 8, cudaMemcpyHostToDevice));
  HBP_CUDA(cudaMemcpy(d + n, b, (size_t)n * 8, cudaMemcpyHostToDevice));
  hbp::division_selftest_kernel<<<(unsigned)((n + 255) / 256), 256>>>(d, d + n, d + 2 * n,
                                                                      d + 4 * n, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(q_fast, d + 2 * n, (size_t)n * 16, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(q_ref, d + 4 * n, (size_t)n * 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  HBP_CUDA(e);
  return HBP_OK;
}

}  // extern "C"
