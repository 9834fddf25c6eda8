// Multi-evidence sweep: many independent evidence / feedback sets over ONE
// graph under the PARALL schedule -- the embarrassingly parallel form of the
// interactive ranking loop (ranking.py:94-135: clamp_evidence + compile + run
// from uniform, once per set), executed as one cooperative launch per pass.
//
// Semantics. Clamping variable v (graph.py:189-200)
// appends a body-empty AND factor whose factor-to-variable message is exactly
// (1, 0) (observed false) or (0, 1) (observed true) from iteration 1 on, and
// (1, 1) before its first update. Its slot is the LAST one of v's ftov row
// (highest factor id, rows in (factor, slot) order, storage.py:59-61), so the
// clamped graph's products are the base graph's row products with one more
// multiplication by 0.0 / 1.0 at the end: exact, no rounding change. Under
// PARALL the clamped graph's schedule is the base schedule plus the clamp
// edges in s_0 (they are unary, so t_0 is unchanged). Therefore set j of the
// sweep reproduces hornbp.run(clamped graph j, PARALL) bit for bit by sharing
// the base graph's CSR and applying a per-(variable, set) evidence code:
//   - vtof of iteration 1 reads only initial (1,1) messages -> (0.5, 0.5)
//     everywhere (or (1,1) unnormalised), so iteration 1 loads no messages;
//   - vtof of iterations >= 2 and every marginal multiply the clamp in last.
//
// Layout: set-minor. Every message / marginal array is [row][S] with S = the
// sets of this pass rounded up to 32, so a warp owns ONE graph node for 32
// consecutive sets: the node's row indices, twins and factor parameters are
// warp-uniform broadcast loads, each message load is a fully coalesced 512-byte
// row segment, and control flow (role, degree) is identical across the warp --
// the grouping the paper's per-group kernels aim for, with zero divergence.
// Each lane multiplies its set's row left to right in slot order, the
// reference's own order (engine.py:168-183), so results are bitwise.
//
// Per-set convergence: each set stops at its own iteration (delta < tol,
// max_iterations, time limit, underflow); stopped sets are masked out and a
// CTA whose 32 sets have all stopped skips the phase. No host round trip until
// every set of the pass has stopped.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdlib>
#include <string>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "device.h"
#include "lbp_kernels.cuh"

namespace hbp {

using namespace dev;

constexpr int kNoVar = 0x7f7f7f7f;  // ufmarg reset value (memset 0x7F)

struct SweepParams {
  const int *vrow, *frow;     // internal rows
  const int *vtof_twin;       // vtof slot -> ftov slot
  const unsigned *ftov_twin;  // ftov slot -> vtof slot | kUnaryBit
  const double2 *fpar;        // per internal factor (p1, p2)
  const int *vorig;           // internal variable -> original id
  int V, F, E, f_or_light, f_heavy, f_or_heavy;
  int f_unary;                // internal factors [0, f_unary) are unary AND factors
  const int4 *vchunks, *fchunks;  // {n0, n1, r0, r1} node chunks (TMA-staged kernel)
  int n_vchunks, n_fchunks, fchunk_nonunary;
  int S;                      // row stride (sets in this pass, multiple of 32)
  int nsets;                  // real sets in this pass
  double2 *vtof, *ftov;       // [S/32][E][32]
  double *p0;                 // [S/32][V][32] P(X=0) of the last marginal pass
  const unsigned char *ev;    // [S/32][V][32] evidence code: bit0 observed false, bit1 observed true
  // per-set control, [iteration][S]
  unsigned long long *dbits;  // |dP1| max, as ordered bits
  unsigned long long *ufkey;  // first underflowing message: kind << 32 | slot
  int *ufmarg;                // smallest underflowing variable (original id)
  int *tflag;                 // [iteration] time limit exceeded
  int *res_it, *res_stop;     // [S] stopping iteration, reason
  unsigned *nstop;            // sets stopped so far (padding counts as stopped)
  unsigned *claim;            // [2][gridDim.y] chunk claim counters (ping-pong by phase)
  // staged kernel: set compaction. Sets live in slots; slot2set[slot] (-1:
  // empty) changes when the running sets are packed into fewer tiles, and the
  // state is double buffered (the vtof buffer receives the packed ftov rows)
  double *p0_alt;
  unsigned char *ev_alt;
  int *slot2set;              // [S]
  int *res_pos;               // [S] per set: slot | buffer parity << 30 of its final P0
                              // (alternate buffers: the absolute slot of the level's region)
  int compact;                // 1: pack the running sets when that halves the live tiles
  int ccap;                   // slots of the alternate P0 / evidence buffers
  int debug;                  // HBP_SWEEP_DEBUG=1: device printf of tail events
  unsigned *bar;              // grid barrier arrivals
  unsigned long long *t0;
  int max_it, normalize;
  double tol;
  long long time_limit_ns;
};

// ---- grid barrier (same protocol as the single-graph executor) ---------------------------

__device__ __forceinline__ unsigned sw_ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void sw_grid_sync(unsigned *bar, unsigned &expected, unsigned nblocks) {
  __syncthreads();
  expected += nblocks;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (sw_ld_acquire(bar) < expected) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long sw_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- the clamp factor's message ---------------------------------------------------------
// the clamp factor's message, multiplied in after the row (it is the row's last slot)
__device__ __forceinline__ void sw_clamp(unsigned code, double &a0, double &a1) {
  if (code & 1u) {  // observed false: (1, 0)
    a0 = mul(a0, 1.0);
    a1 = mul(a1, 0.0);
  }
  if (code & 2u) {  // observed true: (0, 1)
    a0 = mul(a0, 0.0);
    a1 = mul(a1, 1.0);
  }
}

// ---- precision-generic lane view and helpers of the staged kernel ---------------------------

template <typename T>
struct SwLaneT {
  typename Ar<T>::T2 *vtof, *ftov;  // &X[g][0][lane]
  double *p0;                       // marginals are fp64 in both precisions
  const unsigned char *ev;
  int s;                            // the set (control arrays are indexed by set)
};

template <typename T>
struct SwBufsT {
  typename Ar<T>::T2 *ftov, *vtof;
  double *p0;
  unsigned char *ev;
  int parity;  // 0: the pass's original p0 / ev buffers, 1: the alternates
  int base;    // first slot of the alternates' region in use (a multiple of 32)
};

template <typename T>
__device__ __forceinline__ SwLaneT<T> sw_lane_bt(const SwBufsT<T> &B, int slot, int set, int E,
                                                 int V) {
  const int g = slot >> 5, lane = slot & 31;
  SwLaneT<T> L;
  L.vtof = B.vtof + (size_t)g * E * 32 + lane;
  L.ftov = B.ftov + (size_t)g * E * 32 + lane;
  L.p0 = B.p0 + (size_t)g * V * 32 + lane;
  L.ev = B.ev + (size_t)g * V * 32 + lane;
  L.s = set;
  return L;
}

// message loads / stores of the staged kernel: arithmetic is always fp64 (the
// bitwise contract); the fp32 mode only stores messages as float (one
// rounding per stored message) and widens them back on load
__device__ __forceinline__ double2 ld2(const double2 *p) { return *p; }
__device__ __forceinline__ double2 ld2(const float2 *p) {
  const float2 v = *p;
  return make_double2((double)v.x, (double)v.y);
}
__device__ __forceinline__ void st2(double2 *p, double a, double b) { *p = make_double2(a, b); }
__device__ __forceinline__ void st2(float2 *p, double a, double b) {
  *p = make_float2(__double2float_rn(a), __double2float_rn(b));
}

// marginal of the previous iteration + |dP1| (engine.py:510-523, :557, :572),
// always in fp64 -- for fp64 runs exactly sw_marginal; fp32 runs feed it the
// fp64 product of their fp32 messages
__device__ __forceinline__ void sw_marginal_d(const SweepParams &P, double *p0_slot, int set, int v,
                                             int it, double q0, double q1, double prev_p0,
                                             unsigned long long &dmax) {
  const double t = add(q0, q1);
  // NaN totals suppress the raise (numpy's min propagates NaN): they record -1
  if (!(t >= kMinMessageSum)) atomicMin(&P.ufmarg[(size_t)(it - 1) * P.S + set], t != t ? -1 : P.vorig[v]);
  const double p0 = div_rn(q0, t);
  const double p1 = sub(1.0, p0);
  const double prev = it == 2 ? 0.5 : sub(1.0, prev_p0);  // prev P1 starts at 0.5
  const unsigned long long raw = (unsigned long long)__double_as_longlong(sub(p1, prev));
  unsigned long long bits;
  asm("and.b64 %0, %1, 0x7fffffffffffffff;" : "=l"(bits) : "l"(raw));
  dmax = bits > dmax ? bits : dmax;
  *p0_slot = p0;
}

// ---- TMA-staged, warp-specialised sweep kernel (default) ------------------------------------
// The persistent kernel above issues a node's loads and then computes, so a
// warp has no memory in flight while it multiplies: HBM-latency bound at
// ~54 % of peak (profiles/r1_sweep_ncu.md). Here each CTA streams host-built
// node chunks (<= 32 message rows / 16 nodes, interleaved over the CTAs)
// through a shared-memory ring: one producer warp fetches each chunk with 1-D
// bulk copies (cp.async.bulk -> UBLKCP, completion counted on an mbarrier):
// the chunk's message rows (contiguous in the [S/32][E][32] tiles), its row
// pointers and twins (16-byte aligned windows), and per node the P0 /
// evidence rows (variable side) or the factor parameters (factor side).
// Consumer warps take the chunk's nodes round-robin, compute from shared
// memory in the reference's operation order (same bits) and release the
// slot through an "empty" mbarrier.
//
// NS = sets per lane (1 or 2): with NS = 2 a CTA serves two 32-set groups and
// every lane computes the same node for two sets -- two independent fp64
// chains per lane (the kernel is bound by dependency latency, not issue) and
// the node's index work (row pointers, twins, degree dispatch, loop) paid
// once for both.

#ifndef HBP_WS_DMAX
#define HBP_WS_DMAX 6  // largest node degree computed from registers (larger: loop path)
#endif
#ifndef HBP_WS_CONSUMERS
#define HBP_WS_CONSUMERS 8
#endif
#ifndef HBP_WS_RING
#define HBP_WS_RING 3  // measured on B200: 2 -> 153 ms, 3 -> 133-135 ms, 4 -> 135-136 ms, 5 -> 219 ms (1 CTA/SM)
#endif
#ifndef HBP_WS_MINB
#define HBP_WS_MINB 2
#endif
// consumer warps per CTA: NS = 2 CTAs hold twice the staging, so one CTA per
// SM with twice the consumers keeps the same number of warps per SM
template <int NS>
struct WsCfg {
  static constexpr int consumers = NS == 1 ? HBP_WS_CONSUMERS : 2 * HBP_WS_CONSUMERS;
  static constexpr int threads = 32 * (consumers + 1);
  static constexpr int min_blocks = NS == 1 ? HBP_WS_MINB : 1;
};
#ifndef HBP_WS_CHR
#define HBP_WS_CHR 32
#endif
#ifndef HBP_WS_CHN
#define HBP_WS_CHN 16
#endif
#ifndef HBP_WS_CLAIM
#define HBP_WS_CLAIM 2
#endif
constexpr int kClaim = HBP_WS_CLAIM;  // chunks per claim
constexpr int kChR = HBP_WS_CHR;  // message rows per chunk
constexpr int kChN = HBP_WS_CHN;  // nodes per chunk
constexpr int kRing = HBP_WS_RING;  // chunks in flight per CTA
constexpr int kPad = 8;    // index arrays are padded so aligned windows stay in bounds

template <int NS, typename T>
struct __align__(16) WsChunk {
  using T2 = typename Ar<T>::T2;
  T2 msg[NS][kChR][32];           // message rows of the chunk, one row (32 lanes) per slot and group
  double p0[NS][kChN][32];        // variable side: P0 of the previous iteration per node
  unsigned char ev[NS][kChN][32]; // variable side: evidence codes per node
  double2 fpar[kChN];             // factor side: (p1, p2) per node
  int rp[kChN + 8];               // row pointers, aligned window from (n0 & ~3)
  int tw[kChR + 8];               // twins, aligned window from (r0 & ~3)
  int n0, n1, r0, heavy;          // header written by the producer before arming
};

template <int NS, typename T>
struct WsShared {
  WsChunk<NS, T> ring[kRing];
  unsigned long long full[kRing], empty[kRing];
  unsigned long long red[WsCfg<NS>::consumers][NS][32];
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Variable node of degree D for NS sets (set u: rows x[u][k*32], lane view
// L[u]); twins tw[k] are shared. Per set exactly the single-set operation
// order; the NS chains are independent and interleave.
template <int D, int NS, bool NORM, typename T>
__device__ __forceinline__ void ws_var(const SweepParams &P, const SwLaneT<T> *L, int v,
                                      const typename Ar<T>::T2 *const *x, const int *tw,
                                      const unsigned *code, const double *prev_p0, int it,
                                      bool write_vtof, const bool *alive,
                                      unsigned long long *dmax, unsigned *uf) {
  double x0[NS][D], x1[NS][D];
#pragma unroll
  for (int u = 0; u < NS; ++u)
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double2 m = ld2(x[u] + k * 32);
      x0[u][k] = m.x;
      x1[u][k] = m.y;
    }
  double a0[NS], a1[NS];
#pragma unroll
  for (int u = 0; u < NS; ++u) a0[u] = a1[u] = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const unsigned t = (unsigned)tw[j];
    if (write_vtof && !(t & kUnaryBit)) {
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        double b0 = a0[u], b1 = a1[u];
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
          b0 = mul(b0, x0[u][k]);
          b1 = mul(b1, x1[u][k]);
        }
        if (code[u]) sw_clamp(code[u], b0, b1);
        if (NORM) {
          const double tt = add(b0, b1);
          uf[u] = tt < kMinMessageSum ? t + 1 : uf[u];  // last underflowing slot + 1 (rare)
          div2_rn(b0, b1, tt, b0, b1);
        }
        if (NS == 1 || alive[u]) st2(L[u].vtof + t * 32, b0, b1);
      }
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      a0[u] = mul(a0[u], x0[u][j]);
      a1[u] = mul(a1[u], x1[u][j]);
    }
  }
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    if (NS > 1 && !alive[u]) continue;
    if (code[u]) sw_clamp(code[u], a0[u], a1[u]);
    sw_marginal_d(P, L[u].p0 + v * 32, L[u].s, v, it, a0[u], a1[u], prev_p0[u], dmax[u]);
  }
}

// any degree, one set, rows re-read per target (heavy nodes: global memory).
// Not inlined (rare, long); its state goes in and out by value so that the
// callers' running |dP1| / underflow registers never need an address (an
// escaping reference pins them to local memory on the hot path).
struct WsVarAcc {
  unsigned long long dmax;
  unsigned uf;
};
template <bool NORM, typename T>
__device__ __noinline__ WsVarAcc ws_var_any(const SweepParams &P, typename Ar<T>::T2 *vtof,
                                            double *p0, int s, int v, const typename Ar<T>::T2 *x,
                                            int d, const int *tw, unsigned code, double prev_p0,
                                            int it, bool write_vtof, WsVarAcc acc) {
  if (write_vtof) {
    for (int j = 0; j < d; ++j) {
      const unsigned t = (unsigned)tw[j];
      if (t & kUnaryBit) continue;
      double b0 = 1.0, b1 = 1.0;
      for (int k = 0; k < d; ++k) {
        if (k == j) continue;
        const double2 m = ld2(x + k * 32);
        b0 = mul(b0, m.x);
        b1 = mul(b1, m.y);
      }
      if (code) sw_clamp(code, b0, b1);
      if (NORM) {
        const double tt = add(b0, b1);
        acc.uf = tt < kMinMessageSum ? t + 1 : acc.uf;
        div2_rn(b0, b1, tt, b0, b1);
      }
      st2(vtof + t * 32, b0, b1);
    }
  }
  double q0 = 1.0, q1 = 1.0;
  for (int k = 0; k < d; ++k) {
    const double2 m = ld2(x + k * 32);
    q0 = mul(q0, m.x);
    q1 = mul(q1, m.y);
  }
  if (code) sw_clamp(code, q0, q1);
  sw_marginal_d(P, p0 + v * 32, s, v, it, q0, q1, prev_p0, acc.dmax);
  return acc;
}

template <bool NORM, typename T>
__device__ __forceinline__ void ws_put(typename Ar<T>::T2 *ftov, int t, double o0, double o1,
                                      unsigned &uf, bool store) {
  if (NORM) {
    const double tt = add(o0, o1);
    uf = tt < kMinMessageSum ? (unsigned)t + 1 : uf;
    div2_rn(o0, o1, tt, o0, o1);
  }
  if (store) st2(ftov + t * 32, o0, o1);
}

// Factor node of degree D for NS sets; FIRST: iteration 1 (every vtof message
// is the uniform one, so nothing is read).
template <int D, int KIND, int NS, bool NORM, bool FIRST, typename T>
__device__ __forceinline__ void ws_fac(const SwLaneT<T> *L, const typename Ar<T>::T2 *const *x,
                                      const int *tw,
                                      double2 pp, const bool *alive, unsigned *uf) {
  double m0[NS][D], m1[NS][D];
  const double c = NORM ? 0.5 : 1.0;
#pragma unroll
  for (int u = 0; u < NS; ++u)
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (FIRST) {
        m0[u][k] = c;
        m1[u][k] = c;
      } else {
        const double2 m = ld2(x[u] + k * 32);
        m0[u][k] = m.x;
        m1[u][k] = m.y;
      }
    }
  double sm[NS][D];
#pragma unroll
  for (int u = 0; u < NS; ++u)
#pragma unroll
    for (int k = 1; k < D; ++k) sm[u][k] = add(m0[u][k], m1[u][k]);
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    double h1 = 1.0, h2 = 1.0;
#pragma unroll
    for (int k = 1; k < D; ++k) {
      h1 = mul(h1, sm[u][k]);
      h2 = mul(h2, KIND == 0 ? m1[u][k] : m0[u][k]);
    }
    double o0, o1;
    head_message<KIND>(pp.x, pp.y, h1, h2, o0, o1);
    ws_put<NORM, T>(L[u].ftov, tw[0], o0, o1, uf[u], NS == 1 || alive[u]);
  }
  if (D > 1) {
    double a1[NS], a2[NS];
#pragma unroll
    for (int u = 0; u < NS; ++u) head_slot_terms<KIND>(pp.x, pp.y, m0[u][0], m1[u][0], a1[u], a2[u]);
#pragma unroll
    for (int j = 1; j < D; ++j) {
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        double b1 = a1[u], b2 = a2[u];
#pragma unroll
        for (int k = j + 1; k < D; ++k) {
          b1 = mul(b1, sm[u][k]);
          b2 = mul(b2, KIND == 0 ? m1[u][k] : m0[u][k]);
        }
        double o0, o1;
        body_message<KIND>(pp.x, pp.y, b1, b2, o0, o1);
        ws_put<NORM, T>(L[u].ftov, tw[j], o0, o1, uf[u], NS == 1 || alive[u]);
        a1[u] = mul(a1[u], sm[u][j]);
        a2[u] = mul(a2[u], KIND == 0 ? m1[u][j] : m0[u][j]);
      }
    }
  }
}

template <int KIND, bool NORM, bool FIRST, typename T>
__device__ __noinline__ unsigned ws_fac_any(typename Ar<T>::T2 *ftov, const typename Ar<T>::T2 *x,
                                            int d, const int *tw, double2 pp, unsigned uf) {
  const double c = NORM ? 0.5 : 1.0;
  for (int j = 0; j < d; ++j) {
    double b1 = 1.0, b2 = 1.0;
    for (int k = 0; k < d; ++k) {
      if (k == j) continue;
      const double2 m = FIRST ? make_double2(c, c) : ld2(x + k * 32);
      double f1, f2;
      if (k == 0) {
        head_slot_terms<KIND>(pp.x, pp.y, m.x, m.y, f1, f2);
      } else {
        f1 = add(m.x, m.y);
        f2 = KIND == 0 ? m.y : m.x;
      }
      b1 = mul(b1, f1);
      b2 = mul(b2, f2);
    }
    double o0, o1;
    if (j == 0)
      head_message<KIND>(pp.x, pp.y, b1, b2, o0, o1);
    else
      body_message<KIND>(pp.x, pp.y, b1, b2, o0, o1);
    ws_put<NORM, T>(ftov, tw[j], o0, o1, uf, true);
  }
  return uf;
}

// degree dispatch; NS = 2 keeps the register path to degree 4 (two sets of rows)
template <int KIND, int NS, bool NORM, bool FIRST, typename T>
__device__ __forceinline__ void ws_fac_k(const SwLaneT<T> *L, const typename Ar<T>::T2 *const *x, int d,
                                        const int *tw, double2 pp, const bool *alive,
                                        unsigned *uf) {
  switch (d) {
    case 1: ws_fac<1, KIND, NS, NORM, FIRST, T>(L, x, tw, pp, alive, uf); break;
    case 2: ws_fac<2, KIND, NS, NORM, FIRST, T>(L, x, tw, pp, alive, uf); break;
    case 3: ws_fac<3, KIND, NS, NORM, FIRST, T>(L, x, tw, pp, alive, uf); break;
    case 4: ws_fac<4, KIND, NS, NORM, FIRST, T>(L, x, tw, pp, alive, uf); break;
#if HBP_WS_DMAX > 4
    case 5:
      if (NS == 1) {
        ws_fac<5, KIND, 1, NORM, FIRST, T>(L, x, tw, pp, alive, uf);
        break;
      }
#endif
    default:
#pragma unroll
      for (int u = 0; u < NS; ++u)
        if (NS == 1 || alive[u]) uf[u] = ws_fac_any<KIND, NORM, FIRST, T>(L[u].ftov, x[u], d, tw, pp, uf[u]);
      break;
  }
}

template <int NS, bool NORM, typename T>
__device__ __forceinline__ void ws_var_k(const SweepParams &P, const SwLaneT<T> *L, int v,
                                        const typename Ar<T>::T2 *const *x, int d, const int *tw,
                                        const unsigned *code, const double *prev_p0, int it,
                                        bool write_vtof, const bool *alive,
                                        unsigned long long *dmax, unsigned *uf) {
  switch (d) {
    case 1: ws_var<1, NS, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf); break;
    case 2: ws_var<2, NS, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf); break;
    case 3: ws_var<3, NS, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf); break;
    case 4: ws_var<4, NS, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf); break;
#if HBP_WS_DMAX > 4
    case 5:
      if (NS == 1) {
        ws_var<5, 1, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf);
        break;
      }
    case 6:
      if (NS == 1) {
        ws_var<6, 1, NORM, T>(P, L, v, x, tw, code, prev_p0, it, write_vtof, alive, dmax, uf);
        break;
      }
#endif
    default:
#pragma unroll
      for (int u = 0; u < NS; ++u)
        if (NS == 1 || alive[u]) {
          const WsVarAcc a = ws_var_any<NORM, T>(P, L[u].vtof, L[u].p0, L[u].s, v, x[u], d, tw,
                                                 code[u], prev_p0[u], it, write_vtof, {dmax[u], uf[u]});
          dmax[u] = a.dmax;
          uf[u] = a.uf;
        }
      break;
  }
}

// Producer: stream the chunks c = first, first + stride, ... < count of one
// phase's chunk list through the ring. Chunks (host-built, hbp_sweep_create)
// are runs of consecutive nodes with <= kChR rows and <= kChN nodes; a node
// with more rows forms a "heavy" chunk whose rows stay in global memory.
// Interleaving the chunks over the CTAs gives every CTA the same mix of
// degrees, so the phases stay balanced without atomics.
// side 0 = variables (ftov rows + P0 rows if want_p0 + evidence rows),
// side 1 = factors (vtof rows unless iteration 1, + factor parameters).
template <int NS, typename T>
__device__ __forceinline__ void ws_produce(const SweepParams &P, const SwBufsT<T> &B,
                                           WsShared<NS, T> &sh,
                                           int side, const int4 *chunks, int cfirst, int count,
                                           unsigned *claim, bool want_msg, bool want_p0, int g0,
                                           unsigned &seq) {
  const int lane = threadIdx.x & 31;
  const int *rowptr = side == 0 ? P.vrow : P.frow;
  const int *twin = side == 0 ? (const int *)P.ftov_twin : P.vtof_twin;
  const typename Ar<T>::T2 *msg = side == 0 ? B.ftov : B.vtof;
  if (lane != 0) return;
  // chunks are claimed kClaim at a time from the CTA row's counter; the next
  // claim is in flight while the current group is staged
  unsigned k = atomicAdd(claim, (unsigned)kClaim);
  for (;;) {
    // claim the next group only if this group is whole: every claim's result
    // is then consumed before the producer leaves the phase (no atomic in
    // flight when the counter is zeroed for a later phase)
    const unsigned kn =
        (cfirst + (int)k + kClaim - 1 < count) ? atomicAdd(claim, (unsigned)kClaim) : 0u;
    for (int h = 0; h < kClaim; ++h) {
      const int c = cfirst + (int)k + h;
      const unsigned slot = seq % kRing;
      mbar_wait(&sh.empty[slot], ((seq / kRing) & 1) ^ 1);
      WsChunk<NS, T> &ch = sh.ring[slot];
      ++seq;
      if (c >= count) {  // end of the phase's chunks: a sentinel, no bytes
        ch.n0 = -1;
        mbar_arrive(&sh.full[slot]);
        return;
      }
      const int4 desc = __ldg(chunks + c);
      const int n0 = desc.x, n1 = desc.y, r0 = desc.z, r1 = desc.w;
      const int m = n1 - n0;
      const int heavy = r1 - r0 > kChR;
      ch.n0 = n0;
      ch.n1 = n1;
      ch.r0 = r0;
      ch.heavy = heavy;
      const int rp_lo = n0 & ~3, rp_hi = (n1 + 1 + 3) & ~3;
      const int tw_lo = r0 & ~3, tw_hi = (r1 + 3) & ~3;
      const unsigned b_rp = (rp_hi - rp_lo) * 4;
      const unsigned b_tw = heavy ? 0u : (unsigned)(tw_hi - tw_lo) * 4;
      const unsigned b_msg = (heavy || !want_msg) ? 0u : (unsigned)(r1 - r0) * 32 * sizeof(typename Ar<T>::T2);
      const unsigned b_p0 = (side == 0 && want_p0) ? (unsigned)m * 256 : 0u;
      const unsigned b_ev = side == 0 ? (unsigned)m * 32 : 0u;
      const unsigned b_fp = side == 1 ? (unsigned)m * 16 : 0u;
      mbar_expect_tx(&sh.full[slot], b_rp + b_tw + b_fp + NS * (b_msg + b_p0 + b_ev));
      bulk_g2s(ch.rp, rowptr + rp_lo, b_rp, &sh.full[slot]);
      if (b_tw) bulk_g2s(ch.tw, twin + tw_lo, b_tw, &sh.full[slot]);
      if (b_fp) bulk_g2s(ch.fpar, P.fpar + n0, b_fp, &sh.full[slot]);
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        const size_t g = (size_t)(g0 + u);
        if (b_msg) bulk_g2s(ch.msg[u], msg + (g * P.E + r0) * 32, b_msg, &sh.full[slot]);
        if (b_p0) bulk_g2s(ch.p0[u], B.p0 + (g * P.V + n0) * 32, b_p0, &sh.full[slot]);
        if (b_ev) bulk_g2s(ch.ev[u], B.ev + (g * P.V + n0) * 32, b_ev, &sh.full[slot]);
      }
    }
    k = kn;
  }
}

// Consumers: node i of the phase's node stream goes to warp (i mod consumers),
// so the warps stay balanced across chunks of any size.
template <int NS, bool NORM, bool FIRST, typename T>
__device__ __forceinline__ void ws_consume_fac(const SweepParams &P, WsShared<NS, T> &sh,
                                               const SwLaneT<T> *L, int cw, const bool *alive,
                                               unsigned &seq, unsigned *uf, bool unary = false) {
  const int lane = threadIdx.x & 31;
  bool any = false;
#pragma unroll
  for (int u = 0; u < NS; ++u) any |= alive[u];
  int base = 0;
  for (;;) {
    const unsigned slot = seq % kRing;
    mbar_wait(&sh.full[slot], (seq / kRing) & 1);
    const WsChunk<NS, T> &ch = sh.ring[slot];
    const int n0 = ch.n0, n1 = ch.n1, r0 = ch.r0;
    if (n0 < 0) {  // the producer's end-of-phase sentinel
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[slot]);
      ++seq;
      break;
    }
    const int rp_lo = n0 & ~3, tw_lo = r0 & ~3;
    const int start = (cw + WsCfg<NS>::consumers - base % WsCfg<NS>::consumers) % WsCfg<NS>::consumers;
    if (any) {
      for (int f = n0 + start; f < n1; f += WsCfg<NS>::consumers) {
        const int r = ch.rp[f - rp_lo];
        const int d = ch.rp[f + 1 - rp_lo] - r;
        // unary: a constant message, written in iteration 1 (and again after a compaction)
        if (!FIRST && !unary && d == 1) continue;
        const double2 pp = ch.fpar[f - n0];
        const bool is_or = (f >= P.f_or_light && f < P.f_heavy) || f >= P.f_or_heavy;
        if (ch.heavy) {
          // rows not staged: twins and messages from global memory
          const int *tw = P.vtof_twin + r;
#pragma unroll
          for (int u = 0; u < NS; ++u) {
            if (!alive[u]) continue;
            const typename Ar<T>::T2 *x = L[u].vtof + (size_t)r * 32;
            uf[u] = !is_or ? ws_fac_any<0, NORM, FIRST, T>(L[u].ftov, x, d, tw, pp, uf[u])
                           : ws_fac_any<1, NORM, FIRST, T>(L[u].ftov, x, d, tw, pp, uf[u]);
          }
        } else {
          const int *tw = ch.tw + (r - tw_lo);
          const typename Ar<T>::T2 *x[NS];
#pragma unroll
          for (int u = 0; u < NS; ++u) x[u] = &ch.msg[u][r - r0][lane];
          if (!is_or) ws_fac_k<0, NS, NORM, FIRST, T>(L, x, d, tw, pp, alive, uf);
          else ws_fac_k<1, NS, NORM, FIRST, T>(L, x, d, tw, pp, alive, uf);
        }
      }
    }
    base += n1 - n0;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[slot]);
    ++seq;
  }
}

template <int NS, bool NORM, typename T>
__device__ __forceinline__ void ws_consume_var(const SweepParams &P, WsShared<NS, T> &sh,
                                               const SwLaneT<T> *L, int cw, int it, bool write_vtof,
                                               const bool *alive, unsigned &seq,
                                               unsigned long long *dmax, unsigned *uf) {
  const int lane = threadIdx.x & 31;
  bool any = false;
#pragma unroll
  for (int u = 0; u < NS; ++u) any |= alive[u];
  int base = 0;
  for (;;) {
    const unsigned slot = seq % kRing;
    mbar_wait(&sh.full[slot], (seq / kRing) & 1);
    const WsChunk<NS, T> &ch = sh.ring[slot];
    const int n0 = ch.n0, n1 = ch.n1, r0 = ch.r0;
    if (n0 < 0) {  // the producer's end-of-phase sentinel
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[slot]);
      ++seq;
      break;
    }
    const int rp_lo = n0 & ~3, tw_lo = r0 & ~3;
    const int start = (cw + WsCfg<NS>::consumers - base % WsCfg<NS>::consumers) % WsCfg<NS>::consumers;
    if (any) {
      for (int v = n0 + start; v < n1; v += WsCfg<NS>::consumers) {
        const int r = ch.rp[v - rp_lo];
        const int d = ch.rp[v + 1 - rp_lo] - r;
        unsigned code[NS];
        double prev_p0[NS];
#pragma unroll
        for (int u = 0; u < NS; ++u) {
          code[u] = ch.ev[u][v - n0][lane];
          prev_p0[u] = it > 2 ? ch.p0[u][v - n0][lane] : 0.5;
        }
        if (ch.heavy) {
#pragma unroll
          for (int u = 0; u < NS; ++u)
            if (alive[u]) {
              const WsVarAcc a = ws_var_any<NORM, T>(
                  P, L[u].vtof, L[u].p0, L[u].s, v, L[u].ftov + (size_t)r * 32, d,
                  (const int *)P.ftov_twin + r, code[u], prev_p0[u], it, write_vtof, {dmax[u], uf[u]});
              dmax[u] = a.dmax;
              uf[u] = a.uf;
            }
          continue;
        }
        const int *tw = ch.tw + (r - tw_lo);
        const typename Ar<T>::T2 *x[NS];
#pragma unroll
        for (int u = 0; u < NS; ++u) x[u] = &ch.msg[u][r - r0][lane];
        ws_var_k<NS, NORM, T>(P, L, v, x, d, tw, code, prev_p0, it, write_vtof, alive, dmax, uf);
      }
    }
    base += n1 - n0;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[slot]);
    ++seq;
  }
}

// grid (chunk stride, S/32/NS); CTA y serves set groups NS*y .. NS*y+NS-1
// stop decision for set s after iteration done (delta < tol, max_iterations,
// time limit, underflow): a pure function of final per-set values, so every
// CTA that evaluates it gets the same answer
__device__ __forceinline__ int sw_decide(const SweepParams &P, int s, int done) {
  const size_t i = (size_t)done * P.S + s;
  const unsigned long long db = ((const volatile unsigned long long *)P.dbits)[i];
  const unsigned long long uk = ((const volatile unsigned long long *)P.ufkey)[i];
  const int um = ((const volatile int *)P.ufmarg)[i];
  const int tf = ((const volatile int *)P.tflag)[done];
  if (uk != ~0ull || (um != kNoVar && um >= 0)) return 4;  // um -1: a NaN total
  if (__longlong_as_double((long long)db) < P.tol) return 1;
  if (done == P.max_it) return 2;
  if (tf) return 3;
  return 0;
}

constexpr int kMaxUnits = 512;     // CTA rows (units of NS x 32 sets) a pass may have
constexpr int kMaxCompact = 1024;  // passes up to this many slots may compact

// grid (CTAs per unit, S/32/NS); unit y = slots of set groups NS*y .. NS*y+NS-1.
//
// Straggler handling. Sets converge after different iteration counts (C5:
// 23..32, most at 23), but a tile streams full 512-byte rows as long as ONE
// of its 32 sets runs. Two mechanisms keep the tail short:
//  - row adoption: a CTA whose own unit has no running set works, phase by
//    phase, for a unit that still has one (round-robin, sharing its chunk
//    claims), so the tail runs on the whole GPU;
//  - compaction: when packing the running sets into the lowest slots at least
//    halves the number of live tiles, every CTA copies its share of their
//    state (ftov rows into the free vtof buffer, P0 and evidence into the
//    alternate buffers), slot2set is rewritten and the buffers swap. Per-set
//    control data is indexed by set, not slot, and res_pos records where each
//    set's final marginals are.
template <bool NORM, int NS, typename T>
#ifdef HBP_WS_MAXNREG
__global__ void __maxnreg__(HBP_WS_MAXNREG)
#else
__global__ void __launch_bounds__(WsCfg<NS>::threads, WsCfg<NS>::min_blocks)
#endif
    sweep_ws(const __grid_constant__ SweepParams P) {
  using T2 = typename Ar<T>::T2;
  constexpr int kWsConsumers = WsCfg<NS>::consumers;
  constexpr int kWarps = kWsConsumers + 1;
  extern __shared__ __align__(128) unsigned char ws_smem[];
  WsShared<NS, T> &sh = *reinterpret_cast<WsShared<NS, T> *>(ws_smem);
  __shared__ unsigned umask[kMaxUnits][NS];  // running sets per unit, one bit per lane
  __shared__ int ulist[kMaxUnits];            // running units, ascending
  __shared__ int s_nunits, s_nrun;
  __shared__ short n2o[kMaxCompact];          // compaction: new slot -> old slot
  __shared__ int s2s_old[kMaxCompact];        // compaction: slot2set before it
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool producer = warp == kWsConsumers;
  const int units = gridDim.y;
  const int S = P.S;
  const unsigned nblocks = gridDim.x * gridDim.y;
  SwBufsT<T> B;
  B.ftov = (T2 *)P.ftov;
  B.vtof = (T2 *)P.vtof;
  B.p0 = P.p0;
  B.ev = const_cast<unsigned char *>(P.ev);
  B.parity = 0;
  B.base = 0;
  SwLaneT<T> L[NS];
  bool alive[NS];
  int sidx[NS];  // slots
  int sset[NS];  // their sets
  unsigned expected = 0, seq = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kWsConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *P.t0 = sw_globaltimer();

  auto set_of = [&](int slot) -> int { return __ldcg(P.slot2set + slot); };
  // Running slots of every unit (after_decision: minus the decision taken at
  // `done`, which other CTAs cannot see through res_stop yet -- re-evaluated,
  // same inputs, same answer); then this CTA's unit for the phase: its own
  // while it has running sets, otherwise an adopted one; -1: nothing to do.
  auto pick_unit = [&](bool after_decision, int done) -> int {
    for (int r = warp; r < units; r += kWarps) {
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        const int set = set_of((r * NS + u) * 32 + lane);
        bool run = set >= 0 && ((const volatile int *)P.res_stop)[set] == 0;
        if (run && after_decision) run = sw_decide(P, set, done) == 0;
        const unsigned m = __ballot_sync(0xffffffffu, run);
        if (lane == 0) umask[r][u] = m;
      }
    }
    __syncthreads();
    if (warp == 0) {
      int base = 0, nrun = 0;
      for (int r0 = 0; r0 < units; r0 += 32) {
        const int r = r0 + lane;
        bool any = false;
        int cnt = 0;
        if (r < units)
#pragma unroll
          for (int u = 0; u < NS; ++u) {
            any |= umask[r][u] != 0;
            cnt += __popc(umask[r][u]);
          }
        const unsigned b = __ballot_sync(0xffffffffu, any);
        if (any) ulist[base + __popc(b & ((1u << lane) - 1))] = r;
        base += __popc(b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        nrun += cnt;
      }
      if (lane == 0) {
        s_nunits = base;
        s_nrun = nrun;
      }
    }
    __syncthreads();
    const int n = s_nunits;
    if (n == 0) return -1;
    const int own = blockIdx.y;
    bool own_runs = false;
#pragma unroll
    for (int u = 0; u < NS; ++u) own_runs |= umask[own][u] != 0;
    if (own_runs) return own;
    return ulist[(int)((blockIdx.y * gridDim.x + blockIdx.x) % (unsigned)n)];
  };
  auto bind_unit = [&](int t) {
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      sidx[u] = (t * NS + u) * 32 + lane;
      sset[u] = set_of(sidx[u]);
      L[u] = sw_lane_bt<T>(B, sidx[u], sset[u], P.E, P.V);
      alive[u] = (umask[t][u] >> lane) & 1u;
    }
  };
  // chunk claims: phase q = 2 it + side uses counter (q & 1) of the unit;
  // CTA x == 0 of each unit zeroes the unit's other counter for phase q + 1
  // (its last use was phase q - 1, behind the barrier that opened phase q)
  auto reset_claims = [&](int q) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.claim[((q + 1) & 1) * units + blockIdx.y] = 0;
  };

  // ---- compaction, at most once per pass, right after a stop decision: the
  // running sets move to the lowest slots (vtof rows of the current iteration
  // into the ftov buffer, P0 and evidence into the alternate buffers), the
  // buffers swap roles, and the following factor phase rewrites the unary
  // factors' constant messages (the new ftov buffer does not hold them).
  // Inputs: umask / s_nrun / s_nunits from pick_unit(true, done).
  // Compactions go to disjoint regions of the alternate buffers (level 1:
  // slots [0, ccap/2), level 2: the next ccap/4, level 3: the rest), so no
  // compaction writes where a stopped set's final P0 lies: each level packs
  // at most half the previous one's tiles.
  int ncomp = 0;
  auto level_base = [&](int l) {
    const int h = (P.ccap / 2 + 31) & ~31, q = (P.ccap / 4 + 31) & ~31;
    return l <= 1 ? 0 : (l == 2 ? h : h + q);
  };
  auto level_size = [&](int l) {
    return (l >= 3 ? P.ccap : level_base(l + 1)) - level_base(l);
  };
  auto maybe_compact = [&](int it) -> bool {
    if (!P.compact || ncomp >= 3 || S > kMaxCompact) return false;
    const int nrun = s_nrun, live = s_nunits;
    const int need = (nrun + 32 * NS - 1) / (32 * NS);
    if (P.debug && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
      printf("it %d: running %d sets in %d units (packed: %d)\n", it, nrun, live, need);
    if (!(nrun > 0 && 2 * need <= live && need * 32 * NS <= level_size(ncomp + 1))) return false;
    const int nb = level_base(ncomp + 1);
    double *p0_dst = P.p0_alt + (size_t)nb * P.V;
    unsigned char *ev_dst = P.ev_alt + (size_t)nb * P.V;
    // n2o: running slots in ascending order; s2s_old: slot2set before
    for (int i = threadIdx.x; i < S; i += blockDim.x) s2s_old[i] = set_of(i);
    __syncthreads();
    if (warp == 0) {
      int base = 0;
      for (int s0 = 0; s0 < S; s0 += 32) {
        const int sl = s0 + lane;
        const int r = sl / (32 * NS), u = (sl / 32) % NS;
        const bool run = sl < S && ((umask[r][u] >> (sl & 31)) & 1u);
        const unsigned b = __ballot_sync(0xffffffffu, run);
        if (run) n2o[base + __popc(b & ((1u << lane) - 1))] = (short)sl;
        base += __popc(b);
      }
    }
    __syncthreads();
    // every CTA has read the old slot2set: it may now be rewritten
    sw_grid_sync(P.bar, expected, nblocks);
    const int R = nrun;
    const int R32 = need * 32 * NS;
    const size_t tot_m = (size_t)P.E * R32, tot_v = (size_t)P.V * R32;
    const size_t gtid = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t gstride = (size_t)nblocks * blockDim.x;
    for (size_t i = gtid; i < tot_m; i += gstride) {
      const int k = (int)(i % R32);
      const size_t row = i / R32;
      if (k < R) {
        const int o = n2o[k];
        B.ftov[((size_t)(k >> 5) * P.E + row) * 32 + (k & 31)] =
            B.vtof[((size_t)(o >> 5) * P.E + row) * 32 + (o & 31)];
      }
    }
    for (size_t i = gtid; i < tot_v; i += gstride) {
      const int k = (int)(i % R32);
      const size_t row = i / R32;
      if (k < R) {
        const int o = n2o[k];
        const size_t src = ((size_t)(o >> 5) * P.V + row) * 32 + (o & 31);
        const size_t dst = ((size_t)(k >> 5) * P.V + row) * 32 + (k & 31);
        p0_dst[dst] = B.p0[src];
        ev_dst[dst] = B.ev[src];
      }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0)
      for (int k = threadIdx.x; k < S; k += blockDim.x) P.slot2set[k] = k < R ? s2s_old[n2o[k]] : -1;
    sw_grid_sync(P.bar, expected, nblocks);
    T2 *nv = B.ftov;  // holds the packed vtof rows
    B.ftov = B.vtof;
    B.vtof = nv;
    B.p0 = p0_dst;
    B.ev = ev_dst;
    B.parity = 1;
    B.base = nb;
    ++ncomp;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(P.nstop + 2, 1u);
    return true;
  };

  for (int it = 1;; ++it) {
    bool rewrite_unary = false;
    if (it >= 2) {
      const bool final_pass = it == P.max_it + 1;
      unsigned long long dmax[NS];
      unsigned uf[NS];  // last underflowing vtof slot + 1 per set
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        dmax[u] = 0;
        uf[u] = 0;
      }
      reset_claims(2 * it);
      const int t = pick_unit(false, 0);
      if (t >= 0) {
        bind_unit(t);
        if (producer) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          ws_produce<NS, T>(P, B, sh, 0, P.vchunks, 0, P.n_vchunks,
                         P.claim + (size_t)((2 * it) & 1) * units + t, true, it > 2, t * NS, seq);
        } else {
          ws_consume_var<NS, NORM, T>(P, sh, L, warp, it, !final_pass, alive, seq, dmax, uf);
        }
        if (!producer)
#pragma unroll
          for (int u = 0; u < NS; ++u) sh.red[warp][u][lane] = dmax[u];
        __syncthreads();
        if (warp == 0) {
#pragma unroll
          for (int u = 0; u < NS; ++u) {
            unsigned long long m = 0;
#pragma unroll
            for (int w = 0; w < kWsConsumers; ++w) m = sh.red[w][u][lane] > m ? sh.red[w][u][lane] : m;
            if (alive[u]) atomicMax(&P.dbits[(size_t)(it - 1) * S + sset[u]], m);
          }
        }
        if (!producer)
#pragma unroll
          for (int u = 0; u < NS; ++u)
            if (alive[u] && uf[u])
              atomicMin(&P.ufkey[(size_t)it * S + sset[u]], (unsigned long long)(uf[u] - 1));
      }
      if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && P.time_limit_ns > 0)
        P.tflag[it - 1] = (long long)(sw_globaltimer() - *P.t0) > P.time_limit_ns;
      sw_grid_sync(P.bar, expected, nblocks);
      // stop decisions for iteration done = it - 1, recorded once per set by
      // CTA x == 0 of the unit holding the set's slot
      const int done = it - 1;
      if (blockIdx.x == 0 && warp == 0) {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
          const int slot = (blockIdx.y * NS + u) * 32 + lane;
          const int set = set_of(slot);
          if (set >= 0 && ((const volatile int *)P.res_stop)[set] == 0) {
            const int stop = sw_decide(P, set, done);
            if (stop) {
              P.res_it[set] = done;
              P.res_pos[set] = (B.base + slot) | (B.parity << 30);
              P.res_stop[set] = stop;
              atomicAdd(P.nstop, 1u);
            }
          }
        }
      }
      if (P.compact && ncomp < 3 && !final_pass) {
        pick_unit(true, done);
        rewrite_unary = maybe_compact(it);
      }
    }
    {
      unsigned uf[NS];  // last underflowing ftov slot + 1 per set
#pragma unroll
      for (int u = 0; u < NS; ++u) uf[u] = 0;
      reset_claims(2 * it + 1);
      const int t = pick_unit(it >= 2, it - 1);
      if (t >= 0) {
        bind_unit(t);
        const bool first = it == 1;
        // after iteration 1 the unary factors' chunks are skipped (constant
        // messages) -- except right after a compaction, which left them behind
        const int c0 = (first || rewrite_unary) ? 0 : P.fchunk_nonunary;
        if (producer) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          ws_produce<NS, T>(P, B, sh, 1, P.fchunks, c0, P.n_fchunks,
                         P.claim + (size_t)((2 * it + 1) & 1) * units + t, !first, false, t * NS,
                         seq);
        } else if (first) {
          ws_consume_fac<NS, NORM, true, T>(P, sh, L, warp, alive, seq, uf);
        } else {
          ws_consume_fac<NS, NORM, false, T>(P, sh, L, warp, alive, seq, uf, rewrite_unary);
        }
        if (!producer)
#pragma unroll
          for (int u = 0; u < NS; ++u)
            if (alive[u] && uf[u])
              atomicMin(&P.ufkey[(size_t)it * S + sset[u]],
                        (1ull << 32) | (unsigned long long)(uf[u] - 1));
      }
    }
    sw_grid_sync(P.bar, expected, nblocks);
    if (((const volatile unsigned *)P.nstop)[0] >= (unsigned)S) return;

  }
}

// ---- evidence table + outputs ----------------------------------------------------------------

__device__ __forceinline__ size_t tile_pos(int row, int s, int rows) {
  return ((size_t)(s >> 5) * rows + row) * 32 + (s & 31);
}

// ev[vinv[var]][set] |= 1 (false) / 2 (true); byte OR through the containing word
__global__ void sweep_evidence_kernel(unsigned char *ev, const int *vinv, const int *ev_set,
                                      const int *ev_var, const signed char *ev_val, int n, int V) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t pos = tile_pos(vinv[ev_var[i]], ev_set[i], V);
  const unsigned bit = ev_val[i] ? 2u : 1u;
  unsigned *word = (unsigned *)(ev + (pos & ~(size_t)3));
  atomicOr(word, bit << (8 * (pos & 3)));
}

// out[set][k][2] = (P0, 1 - P0) of original variable sel[k] (sel == null: k itself);
// 32 x 32 tiles: coalesced reads along sets, coalesced writes along variables
// res_pos[s] = slot | parity << 30: where set s's final marginals are (the
// staged kernel may have moved the set; parity 1 = the alternate buffers)
__global__ void sweep_ident_kernel(int *slot2set, int *res_pos, int S, int ns) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  slot2set[i] = i < ns ? i : -1;
  res_pos[i] = i;
}

__device__ __forceinline__ size_t final_pos(const int *res_pos, int s, int vi, int V, int &parity) {
  const int rp = res_pos[s];
  parity = (rp >> 30) & 1;
  return tile_pos(vi, rp & 0x3fffffff, V);
}

template <typename T>
__global__ void sweep_marginals_kernel(const T *p0, const T *p0_alt, const int *res_pos,
                                       const int *vinv, const int *sel, int nsel,
                                       int V, int nsets, int set_base, double *out_pair,
                                       double *out_p1) {
  __shared__ T tile[32][33];
  const int k0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // blockDim 256: 8 rows per step
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, s = s0 + tx;
    T v = T(0);
    if (k < nsel && s < nsets) {
      const int var = sel ? sel[k] : k;
      int par;
      const size_t at = final_pos(res_pos, s, vinv[var], V, par);
      v = par ? p0_alt[at] : p0[at];
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int s = s0 + r, k = k0 + tx;
    if (k < nsel && s < nsets) {
      const T q = tile[tx][r];
      const double p1 = sub(1.0, (double)q);  // P1 = 1 - P0 (engine.py:520-522)
      const size_t o = (size_t)(set_base + s) * nsel + k;
      if (out_pair) {
        out_pair[2 * o] = (double)q;
        out_pair[2 * o + 1] = p1;
      }
      if (out_p1) out_p1[o] = p1;
    }
  }
}

// Top-k alarms per set (ranking.py:83-91): unlabeled alarms by descending P1,
// ties by ascending id. One CTA per set; bitonic sort of (~bits(P1), position)
// in shared memory -- P1 >= 0, so its bit pattern orders like its value, and
// positions index the id-sorted selection. Labeled = clamped in this set.
template <typename T>
__global__ void __launch_bounds__(1024) sweep_rank_kernel(const T *p0, const T *p0_alt,
                                                           const unsigned char *ev,
                                                           const unsigned char *ev_alt,
                                                           const int *res_pos,
                                                           const int *vinv, const int *sel,
                                                           int nsel, int npow2, int kpow2, int V,
                                                           int set_base, int topk, int *ranked) {
  extern __shared__ unsigned char smem[];
  unsigned long long *cache = (unsigned long long *)smem;
  unsigned long long *key = cache + npow2;
  int *pos = (int *)(key + kpow2);
  const int s = blockIdx.x;
  auto key_of = [&](int i) -> unsigned long long {
    int par;
    const size_t at = final_pos(res_pos, s, vinv[sel[i]], V, par);
    if ((par ? ev_alt : ev)[at] != 0) return ~0ull;
    return rank_key(sub(1.0, (double)(par ? p0_alt : p0)[at]));
  };
  topk_select(key_of, nsel, topk, npow2, kpow2, cache, key, pos);
  for (int i = threadIdx.x; i < topk; i += blockDim.x)
    ranked[(size_t)(set_base + s) * topk + i] = key[i] != ~0ull ? sel[pos[i]] : -1;
}

}  // namespace hbp

// ======================================================================================
// handle + C ABI

struct hbp_sweep {
  hbp_graph *g = nullptr;
  int cap = 0;           // sets per pass (multiple of 32)
  int grid_x_max = 0;    // co-resident CTAs for the cooperative launch
  const void *kernel = nullptr, *kernel_nonorm = nullptr;
  const void *kernel32 = nullptr, *kernel32_nonorm = nullptr;  // fp32 mode
  size_t smem32 = 0;
  int grid_x_max32 = 0;
  int ns = 1;           // sets per lane of the staged kernel (pass sizes are multiples of 32 * ns)
  int threads = 0;
  int *d_vinv = nullptr;
  int *d_vrow = nullptr, *d_frow = nullptr, *d_vtof_twin = nullptr;  // padded copies (kPad)
  unsigned *d_ftov_twin = nullptr;
  int f_unary = 0;
  int4 *d_vchunks = nullptr, *d_fchunks = nullptr;
  int n_vchunks = 0, n_fchunks = 0, fchunk_nonunary = 0;
  size_t smem = 0;
  double2 *d_vtof = nullptr, *d_ftov = nullptr;
  double *d_p0 = nullptr, *d_p0_alt = nullptr;
  int compact_cap = 0;  // slots the alternate buffers hold
  unsigned char *d_ev = nullptr, *d_ev_alt = nullptr;
  void *d_ctrl = nullptr;
  size_t ctrl_bytes = 0;
  void *d_scratch = nullptr;  // evidence lists, selection, staging outputs
  size_t scratch_bytes = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, k0 = nullptr, k1 = nullptr;
  hbp_plan *parall = nullptr;  // single-graph PARALL plan: exact underflow attribution
  ~hbp_sweep() {
    cudaSetDevice(g->device);
    if (parall) hbp_plan_destroy(parall);
    for (void *p : {(void *)d_vinv, (void *)d_vtof, (void *)d_ftov, (void *)d_p0, (void *)d_ev,
                    (void *)d_p0_alt, (void *)d_ev_alt,
                    d_ctrl, d_scratch, (void *)d_vrow, (void *)d_frow, (void *)d_vtof_twin,
                    (void *)d_ftov_twin, (void *)d_vchunks, (void *)d_fchunks})
      if (p) cudaFree(p);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (k0) cudaEventDestroy(k0);
    if (k1) cudaEventDestroy(k1);
  }
};

namespace {

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

hbp_status ensure(void **p, size_t *cap, size_t need) {
  if (*cap >= need) return HBP_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  HBP_CUDA(cudaMalloc(p, need));
  *cap = need;
  return HBP_OK;
}

// The exact reference underflow report of sweep set j (engine.py:155-165,
// :512-518): the set re-runs on the single-graph executor with its evidence
// codes -- the same fp64 arithmetic, so the same stop -- which halts at the
// failing pass and attributes it there (engine.cu attribute_underflow). The
// re-run uses the graph's own single-run buffers and restores its evidence.
// fp32 sets (no bitwise contract) keep the sweep's own report unless the fp64
// re-run stops on underflow at the same iteration.
hbp_status attribute_set(hbp_sweep *sw, const hbp_options *opt, const hbp_evidence *ev, int j,
                         bool fp32, hbp_set_result *r) {
  hbp_graph *g = sw->g;
  const hbp::HostLayout &L = g->L;
  if (!sw->parall) {
    std::vector<int32_t> se((size_t)L.E), te;
    te.reserve((size_t)L.E);
    for (int64_t e = 0; e < L.E; ++e) {
      se[(size_t)e] = (int32_t)e;
      const int32_t f = L.edge_factor[(size_t)e];
      if (L.rowptr[(size_t)f + 1] - L.rowptr[(size_t)f] > 1) te.push_back((int32_t)e);
    }
    const int64_t so[2] = {0, L.E}, to[2] = {0, (int64_t)te.size()};
    hbp_status st = hbp_plan_create(g, 1, so, se.data(), to, te.data(), &sw->parall);
    if (st != HBP_OK) return st;
  }
  const std::vector<int32_t> keep_var = g->ev_var;
  const std::vector<int8_t> keep_val = g->ev_val;
  const bool keep_has = g->has_ev;
  const int64_t a = ev->offsets[j], b = ev->offsets[j + 1];
  hbp_status st = hbp_graph_set_evidence(g, (int32_t)(b - a), ev->var + a, ev->value + a);
  if (st != HBP_OK) return st;
  hbp_options o = *opt;
  o.precision = 0;
  o.record_history = 0;
  hbp_result res;
  std::memset(&res, 0, sizeof(res));
  const hbp_status rs = hbp_run_device(sw->parall, &o, &res, nullptr);
  st = hbp_graph_set_evidence(g, keep_has ? (int32_t)keep_var.size() : 0, keep_var.data(),
                              keep_val.data());
  if (st != HBP_OK) return st;
  if (rs == HBP_EUNDERFLOW && res.underflow_iteration == r->underflow_iteration) {
    r->underflow_kind = res.underflow_kind;
    r->underflow_index = res.underflow_index;
    return HBP_OK;
  }
  if (rs != HBP_OK && rs != HBP_EUNDERFLOW) return rs;
  if (fp32) return HBP_OK;
  hbp::set_error("internal: sweep set " + std::to_string(j) +
                 " underflowed but its single-graph re-run did not stop there");
  return HBP_ECUDA;
}

}  // namespace

extern "C" {

hbp_status hbp_sweep_create(hbp_graph *g, int32_t max_sets_per_pass, hbp_sweep **out) {
  if (!g || !out || max_sets_per_pass < 0) {
    hbp::set_error("bad sweep arguments");
    return HBP_EINVAL;
  }
  *out = nullptr;
  HBP_CUDA(cudaSetDevice(g->device));
  std::unique_ptr<hbp_sweep> sw(new (std::nothrow) hbp_sweep());
  if (!sw) return HBP_ENOMEM;
  sw->g = g;
  hbp_status hs = hbp::ensure_host_layout(g);
  if (hs != HBP_OK) return hs;
  const hbp::HostLayout &L = g->L;
  int per_sm = 0;
  {
    // the TMA-staged warp-specialised kernel, one set per lane. Measured on
    // B200 against a register-pipelined kernel without staging and against
    // two sets per lane: both slower, removed.
    sw->ns = 1;
    sw->smem = sizeof(hbp::WsShared<1, double>);
    sw->threads = hbp::WsCfg<1>::threads;
    sw->kernel = (const void *)hbp::sweep_ws<true, 1, double>;
    sw->kernel_nonorm = (const void *)hbp::sweep_ws<false, 1, double>;
    // fp32 mode (opt-in per run): the same staged kernel on float messages
    sw->smem32 = sizeof(hbp::WsShared<1, float>);
    sw->kernel32 = (const void *)hbp::sweep_ws<true, 1, float>;
    sw->kernel32_nonorm = (const void *)hbp::sweep_ws<false, 1, float>;
    for (const void *k : {sw->kernel32, sw->kernel32_nonorm})
      HBP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sw->smem32));
    int per_sm32 = 0;
    HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm32, sw->kernel32,
                                                           hbp::WsCfg<1>::threads, sw->smem32));
    sw->grid_x_max32 = std::max(1, per_sm32) * g->num_sms;
    for (const void *k : {sw->kernel, sw->kernel_nonorm})
      HBP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sw->smem));
    HBP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sw->kernel, sw->threads,
                                                           sw->smem));
  }
  sw->grid_x_max = std::max(1, per_sm) * g->num_sms;
  // capacity: requested, else what fits in half of the free memory
  const size_t per_set = (size_t)L.E * 32 + (size_t)L.V * 9;
  size_t free_b = 0, total_b = 0;
  HBP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int cap = max_sets_per_pass > 0 ? max_sets_per_pass : (int)std::min<size_t>(4096, free_b / 2 / per_set);
  const int unit = 32 * sw->ns;
  cap = std::max(unit, (cap + unit - 1) / unit * unit);
  cap = std::min(cap, unit * sw->grid_x_max);
  sw->cap = cap;
  hbp_status st;
  if ((st = upload(&sw->d_vinv, L.vinv, g->stream))) return st;
  {
    // index arrays padded so the producer's 16-byte aligned windows stay in bounds
    auto padded = [](const std::vector<int32_t> &v, int32_t fill) {
      std::vector<int32_t> o(v);
      o.resize(v.size() + hbp::kPad, fill);
      return o;
    };
    std::vector<int32_t> ft(L.ftov_twin.begin(), L.ftov_twin.end());
    std::vector<int32_t> vt_pad = padded(L.vtof_twin, 0), ft_pad = padded(ft, 0);
    std::vector<uint32_t> ft_pad_u(ft_pad.begin(), ft_pad.end());
    if ((st = upload(&sw->d_vrow, padded(L.vrow, (int32_t)L.E), g->stream)) ||
        (st = upload(&sw->d_frow, padded(L.frow, (int32_t)L.E), g->stream)) ||
        (st = upload(&sw->d_vtof_twin, vt_pad, g->stream)) ||
        (st = upload(&sw->d_ftov_twin, ft_pad_u, g->stream)))
      return st;
    int32_t fu = 0;
    while (fu < L.f_or_light && L.frow[fu + 1] - L.frow[fu] == 1) ++fu;
    sw->f_unary = fu;
    // node chunks for the TMA-staged kernel: runs of consecutive nodes with
    // <= kChR rows and <= kChN nodes (a node with more rows is a chunk alone);
    // the factor list breaks at f_unary so iterations > 1 can skip the unary ones
    auto chunks = [](const std::vector<int32_t> &row, int32_t n, int32_t brk,
                     std::vector<int4> &out, int32_t *brk_chunk) {
      int32_t n0 = 0;
      while (n0 < n) {
        if (n0 == brk) *brk_chunk = (int32_t)out.size();
        int32_t n1 = n0 + 1;
        while (n1 < n && n1 != brk && n1 - n0 < hbp::kChN && row[n1 + 1] - row[n0] <= hbp::kChR) ++n1;
        out.push_back(make_int4(n0, n1, row[n0], row[n1]));
        n0 = n1;
      }
      if (brk >= n) *brk_chunk = (int32_t)out.size();
    };
    std::vector<int4> vc, fc;
    int32_t unused = 0, fnu = 0;
    chunks(L.vrow, L.V, -1, vc, &unused);
    chunks(L.frow, L.F, fu, fc, &fnu);
    if (fu == 0) fnu = 0;
    sw->n_vchunks = (int)vc.size();
    sw->n_fchunks = (int)fc.size();
    sw->fchunk_nonunary = fnu;
    if ((st = upload(&sw->d_vchunks, vc, g->stream)) || (st = upload(&sw->d_fchunks, fc, g->stream)))
      return st;
  }
  HBP_CUDA(cudaMalloc(&sw->d_vtof, (size_t)L.E * cap * sizeof(double2)));
  HBP_CUDA(cudaMalloc(&sw->d_ftov, (size_t)L.E * cap * sizeof(double2)));
  HBP_CUDA(cudaMalloc(&sw->d_p0, (size_t)std::max(1, L.V) * cap * sizeof(double)));
  HBP_CUDA(cudaMalloc(&sw->d_ev, (size_t)std::max(1, L.V) * cap + 4));
  // compaction's alternate state buffers (passes of <= kMaxCompact slots)
  sw->compact_cap = std::min(cap, hbp::kMaxCompact);
  HBP_CUDA(cudaMalloc(&sw->d_p0_alt, (size_t)std::max(1, L.V) * sw->compact_cap * sizeof(double)));
  HBP_CUDA(cudaMalloc(&sw->d_ev_alt, (size_t)std::max(1, L.V) * sw->compact_cap + 4));
  HBP_CUDA(cudaEventCreate(&sw->e0));
  HBP_CUDA(cudaEventCreate(&sw->e1));
  HBP_CUDA(cudaEventCreate(&sw->k0));
  HBP_CUDA(cudaEventCreate(&sw->k1));
  HBP_CUDA(cudaStreamSynchronize(g->stream));
  *out = sw.release();
  return HBP_OK;
}

int32_t hbp_sweep_capacity(const hbp_sweep *sw) { return sw ? sw->cap : 0; }

void hbp_sweep_destroy(hbp_sweep *sw) { delete sw; }

hbp_status hbp_sweep_run(hbp_sweep *sw, const hbp_options *opt, const hbp_evidence *ev,
                         hbp_sweep_outputs *out) {
  auto wall0 = std::chrono::steady_clock::now();
  if (!sw || !opt || !ev || !out || !out->sets || ev->num_sets < 0 ||
      (ev->num_sets > 0 && !ev->offsets)) {
    hbp::set_error("null sweep argument");
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
  if (opt->record_history) {
    hbp::set_error("record_history is not supported by the sweep");
    return HBP_EINVAL;
  }
  if (opt->precision != 0 && opt->precision != 1) {
    hbp::set_error("precision must be 0 (fp64) or 1 (fp32)");
    return HBP_EINVAL;
  }
  const bool fp32 = opt->precision == 1;
  hbp_graph *g = sw->g;
  const hbp::HostLayout &L = g->L;
  const int n = ev->num_sets;
  const int64_t nev = n ? ev->offsets[n] : 0;
  if (n && (ev->offsets[0] != 0 || nev < 0 || (nev > 0 && (!ev->var || !ev->value)))) {
    hbp::set_error("bad evidence offsets");
    return HBP_EINVAL;
  }
  for (int j = 0; j < n; ++j)
    if (ev->offsets[j + 1] < ev->offsets[j]) {
      hbp::set_error("evidence offsets must be nondecreasing");
      return HBP_EINVAL;
    }
  for (int64_t i = 0; i < nev; ++i) {
    if (ev->var[i] < 0 || ev->var[i] >= L.V) {
      hbp::set_error("evidence variable out of range");
      return HBP_EINVAL;
    }
    if (ev->value[i] != 0 && ev->value[i] != 1) {
      hbp::set_error("evidence value must be 0 or 1");
      return HBP_EINVAL;
    }
  }
  const int nsel = out->p1_select || out->ranked ? out->num_select : 0;
  if (nsel < 0 || (nsel > 0 && !out->select)) {
    hbp::set_error("bad selection");
    return HBP_EINVAL;
  }
  for (int k = 0; k < nsel; ++k)
    if (out->select[k] < 0 || out->select[k] >= L.V || (k && out->select[k] <= out->select[k - 1])) {
      hbp::set_error("selection must be ascending variable ids");
      return HBP_EINVAL;
    }
  // the shared-memory window of the streaming top-k (lbp_kernels.cuh)
  int npow2 = 1;
  while (npow2 < nsel && npow2 < hbp::dev::kRankCap) npow2 <<= 1;
  if (out->ranked && (out->topk < 0 || out->topk >= hbp::dev::kRankCap)) {
    hbp::set_error("device ranking returns at most 16383 alarms per set");
    return HBP_EINVAL;
  }
  HBP_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = g->stream;
  const int max_it = opt->max_iterations;
  const size_t nit = (size_t)max_it + 2;
  const int cap = sw->cap;
  // control block: dbits, ufkey [nit][cap] u64; ufmarg [nit][cap]; tflag [nit];
  // res_it, res_stop [cap]; nstop, bar, t0
  const size_t o_db = 0, o_uk = o_db + align256(nit * cap * 8), o_um = o_uk + align256(nit * cap * 8),
               o_tf = o_um + align256(nit * cap * 4), o_ri = o_tf + align256(nit * 4),
               o_rs = o_ri + align256((size_t)cap * 4), o_misc = o_rs + align256((size_t)cap * 4),
               o_claim = o_misc + 256, o_s2s = o_claim + align256((size_t)cap / 32 * 8 + 8),
               o_rpos = o_s2s + align256((size_t)cap * 4), ctrl_need = o_rpos + align256((size_t)cap * 4);
  hbp_status s_;
  if ((s_ = ensure(&sw->d_ctrl, &sw->ctrl_bytes, ctrl_need))) return s_;
  char *cb = (char *)sw->d_ctrl;
  unsigned long long *d_db = (unsigned long long *)(cb + o_db);
  unsigned long long *d_uk = (unsigned long long *)(cb + o_uk);
  int *d_um = (int *)(cb + o_um), *d_tf = (int *)(cb + o_tf), *d_ri = (int *)(cb + o_ri),
      *d_rs = (int *)(cb + o_rs);
  unsigned *d_nstop = (unsigned *)(cb + o_misc), *d_bar = d_nstop + 1;  // d_nstop[2]: compactions
  unsigned long long *d_t0 = (unsigned long long *)(cb + o_misc + 64);
  unsigned *d_claim = (unsigned *)(cb + o_claim);
  int *d_s2s = (int *)(cb + o_s2s), *d_rpos = (int *)(cb + o_rpos);
  // scratch: evidence (set, var, val) for one pass, selection, output staging
  const bool marg_dev = out->marginals && out->marginals_on_device;
  const bool p1_dev = out->p1_select && out->p1_on_device;
  const bool rk_dev = out->ranked && out->ranked_on_device;
  const size_t pass_ev_max = [&] {
    int64_t m = 0;
    for (int b = 0; b < n; b += cap) m = std::max<int64_t>(m, ev->offsets[std::min(n, b + cap)] - ev->offsets[b]);
    return (size_t)m;
  }();
  const size_t so_ev = 0, so_sel = so_ev + align256(pass_ev_max * 9 + 16),
               so_marg = so_sel + align256((size_t)nsel * 4 + 4),
               so_p1 = so_marg + ((out->marginals && !marg_dev) ? align256((size_t)cap * L.V * 16) : 0),
               so_rk = so_p1 + ((out->p1_select && !p1_dev) ? align256((size_t)cap * nsel * 8) : 0),
               scratch_need = so_rk + ((out->ranked && !rk_dev) ? align256((size_t)cap * out->topk * 4) : 0) + 256;
  if ((s_ = ensure(&sw->d_scratch, &sw->scratch_bytes, scratch_need))) return s_;
  char *sb = (char *)sw->d_scratch;
  int *d_ev_set = (int *)(sb + so_ev);
  int *d_ev_var = d_ev_set + pass_ev_max;
  signed char *d_ev_val = (signed char *)(d_ev_var + pass_ev_max);
  int *d_sel = (int *)(sb + so_sel);
  double *stage_marg = (double *)(sb + so_marg);
  double *stage_p1 = (double *)(sb + so_p1);
  int *stage_rk = (int *)(sb + so_rk);
  if (nsel) HBP_CUDA(cudaMemcpyAsync(d_sel, out->select, (size_t)nsel * 4, cudaMemcpyHostToDevice, st));

  hbp::SweepParams P{};
  P.vrow = sw->d_vrow;
  P.frow = sw->d_frow;
  P.vtof_twin = sw->d_vtof_twin;
  P.ftov_twin = sw->d_ftov_twin;
  P.f_unary = sw->f_unary;
  P.vchunks = sw->d_vchunks;
  P.fchunks = sw->d_fchunks;
  P.n_vchunks = sw->n_vchunks;
  P.n_fchunks = sw->n_fchunks;
  P.fchunk_nonunary = sw->fchunk_nonunary;
  P.fpar = g->d_fpar;
  P.vorig = g->d_vorig;
  P.V = L.V;
  P.F = L.F;
  P.E = (int)L.E;
  P.f_or_light = L.f_or_light;
  P.f_heavy = L.f_heavy;
  P.f_or_heavy = L.f_or_heavy;
  P.vtof = sw->d_vtof;
  P.ftov = sw->d_ftov;
  P.p0 = sw->d_p0;
  P.ev = sw->d_ev;
  P.dbits = d_db;
  P.ufkey = d_uk;
  P.ufmarg = d_um;
  P.tflag = d_tf;
  P.res_it = d_ri;
  P.res_stop = d_rs;
  P.nstop = d_nstop;
  P.claim = d_claim;
  P.p0_alt = sw->d_p0_alt;
  P.ev_alt = sw->d_ev_alt;
  P.slot2set = d_s2s;
  P.res_pos = d_rpos;
  P.ccap = sw->compact_cap;
  {
    const char *cenv = getenv("HBP_SWEEP_COMPACT");
    P.compact = (sw->d_p0_alt && !(cenv && atoi(cenv) == 0)) ? 1 : 0;  // per pass: S <= compact_cap
    P.debug = getenv("HBP_SWEEP_DEBUG") ? 1 : 0;
  }
  const int compact_enabled = P.compact;
  P.bar = d_bar;
  P.t0 = d_t0;
  P.max_it = max_it;
  P.normalize = opt->normalize_messages ? 1 : 0;
  P.tol = opt->tolerance;
  P.time_limit_ns = opt->time_limit > 0 ? std::max<long long>(1, (long long)(opt->time_limit * 1e9)) : 0;

  std::vector<unsigned long long> h_db, h_uk;
  std::vector<int> h_um, h_ri, h_rs, h_set;
  std::vector<int> h_ev_set, h_ev_var;
  std::vector<signed char> h_ev_val;
  int64_t launches = 0;
  int passes = 0, compactions = 0;
  std::vector<int> uf_sets;  // sets that stopped on underflow (exact attribution below)
  double dev_ms = 0, ker_ms = 0;
  for (int base = 0; base < n; base += cap) {
    const int ns = std::min(cap, n - base);
    const int unit = 32 * sw->ns;
    const int S = (ns + unit - 1) / unit * unit;
    const int groups = S / 32;
    P.S = S;
    P.nsets = ns;
    P.compact = compact_enabled && S <= sw->compact_cap;
    // evidence table of this pass
    const int64_t e_lo = ev->offsets[base], e_hi = ev->offsets[base + ns];
    const int64_t ne = e_hi - e_lo;
    h_ev_set.resize(ne);
    h_ev_var.assign(ev->var + e_lo, ev->var + e_hi);
    h_ev_val.assign(ev->value + e_lo, ev->value + e_hi);
    for (int j = 0; j < ns; ++j)
      for (int64_t i = ev->offsets[base + j]; i < ev->offsets[base + j + 1]; ++i) h_ev_set[i - e_lo] = j;
    HBP_CUDA(cudaEventRecord(sw->e0, st));
    HBP_CUDA(cudaMemsetAsync(sw->d_ev, 0, (size_t)L.V * S, st));
    if (ne) {
      HBP_CUDA(cudaMemcpyAsync(d_ev_set, h_ev_set.data(), ne * 4, cudaMemcpyHostToDevice, st));
      HBP_CUDA(cudaMemcpyAsync(d_ev_var, h_ev_var.data(), ne * 4, cudaMemcpyHostToDevice, st));
      HBP_CUDA(cudaMemcpyAsync(d_ev_val, h_ev_val.data(), ne, cudaMemcpyHostToDevice, st));
      hbp::sweep_evidence_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(
          sw->d_ev, sw->d_vinv, d_ev_set, d_ev_var, d_ev_val, (int)ne, L.V);
      ++launches;
    }
    // control reset
    HBP_CUDA(cudaMemsetAsync(d_db, 0, nit * S * 8, st));
    HBP_CUDA(cudaMemsetAsync(d_uk, 0xFF, nit * S * 8, st));
    HBP_CUDA(cudaMemsetAsync(d_um, 0x7F, nit * S * 4, st));
    HBP_CUDA(cudaMemsetAsync(d_tf, 0, nit * 4, st));
    HBP_CUDA(cudaMemsetAsync(d_ri, 0, (size_t)S * 4, st));
    HBP_CUDA(cudaMemsetAsync(d_claim, 0, (size_t)cap / 32 * 8 + 8, st));
    // slot s holds set s (pass-relative); res_pos defaults to the same slot
    hbp::sweep_ident_kernel<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(d_s2s, d_rpos, S, ns);
    ++launches;
    HBP_CUDA(cudaMemsetAsync(d_rs, 0, (size_t)S * 4, st));
    const unsigned misc[3] = {(unsigned)(S - ns), 0u, 0u};
    HBP_CUDA(cudaMemcpyAsync(d_nstop, misc, 12, cudaMemcpyHostToDevice, st));
    void *args[] = {&P};
    HBP_CUDA(cudaEventRecord(sw->k0, st));
    {
      const int gy = groups / (fp32 ? 1 : sw->ns);
      const int gxm = fp32 ? sw->grid_x_max32 : sw->grid_x_max;
      const int nxw = std::max(1, std::min(gxm / gy, sw->n_vchunks));
      const void *k = fp32 ? (P.normalize ? sw->kernel32 : sw->kernel32_nonorm)
                           : (P.normalize ? sw->kernel : sw->kernel_nonorm);
      HBP_CUDA(cudaLaunchCooperativeKernel(k, dim3(nxw, gy),
                                           dim3(fp32 ? hbp::WsCfg<1>::threads : sw->threads), args,
                                           fp32 ? sw->smem32 : sw->smem, st));
    }
    HBP_CUDA(cudaEventRecord(sw->k1, st));
    ++launches;
    // outputs of this pass
    if (out->marginals) {
      double *dst = marg_dev ? out->marginals : stage_marg;
      const int bbase = marg_dev ? base : 0;
      hbp::sweep_marginals_kernel<double><<<dim3((L.V + 31) / 32, groups), 256, 0, st>>>(
            sw->d_p0, sw->d_p0_alt, d_rpos, sw->d_vinv, nullptr, L.V, L.V, ns, bbase, dst, nullptr);
      ++launches;
      if (!marg_dev)
        HBP_CUDA(cudaMemcpyAsync(out->marginals + (size_t)base * L.V * 2, stage_marg,
                                 (size_t)ns * L.V * 16, cudaMemcpyDeviceToHost, st));
    }
    if (out->p1_select && nsel) {
      double *dst = p1_dev ? out->p1_select : stage_p1;
      const int bbase = p1_dev ? base : 0;
      hbp::sweep_marginals_kernel<double><<<dim3((nsel + 31) / 32, groups), 256, 0, st>>>(
            sw->d_p0, sw->d_p0_alt, d_rpos, sw->d_vinv, d_sel, nsel, L.V, ns, bbase, nullptr, dst);
      ++launches;
      if (!p1_dev)
        HBP_CUDA(cudaMemcpyAsync(out->p1_select + (size_t)base * nsel, stage_p1,
                                 (size_t)ns * nsel * 8, cudaMemcpyDeviceToHost, st));
    }
    if (out->ranked && out->topk > 0) {
      int *dst = rk_dev ? out->ranked : stage_rk;
      const int bbase = rk_dev ? base : 0;
      int kpow2 = 2;
      while (kpow2 < out->topk) kpow2 <<= 1;
      int cache = std::max(npow2, 2);  // optional key cache: shrinks for a large k
      while (cache > 2 && (size_t)cache * 8 + (size_t)kpow2 * 12 > (size_t)200 * 1024) cache >>= 1;
      const size_t smem = (size_t)cache * 8 + (size_t)kpow2 * 12;
      if (smem > 48 * 1024) {
        HBP_CUDA(cudaFuncSetAttribute(hbp::sweep_rank_kernel<double>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      }
      hbp::sweep_rank_kernel<double><<<ns, 1024, smem, st>>>(
            sw->d_p0, sw->d_p0_alt, sw->d_ev, sw->d_ev_alt, d_rpos, sw->d_vinv, d_sel, nsel,
            cache, kpow2, L.V, bbase, out->topk, dst);
      ++launches;
      if (!rk_dev)
        HBP_CUDA(cudaMemcpyAsync(out->ranked + (size_t)base * out->topk, stage_rk,
                                 (size_t)ns * out->topk * 4, cudaMemcpyDeviceToHost, st));
    }
    HBP_CUDA(cudaGetLastError());
    HBP_CUDA(cudaEventRecord(sw->e1, st));
    // per-set results of this pass
    h_db.resize(nit * S);
    h_uk.resize(nit * S);
    h_um.resize(nit * S);
    h_ri.resize(S);
    h_rs.resize(S);
    HBP_CUDA(cudaMemcpyAsync(h_ri.data(), d_ri, (size_t)S * 4, cudaMemcpyDeviceToHost, st));
    HBP_CUDA(cudaMemcpyAsync(h_rs.data(), d_rs, (size_t)S * 4, cudaMemcpyDeviceToHost, st));
    unsigned h_misc[3] = {0, 0, 0};
    HBP_CUDA(cudaMemcpyAsync(h_misc, d_nstop, 12, cudaMemcpyDeviceToHost, st));
    HBP_CUDA(cudaStreamSynchronize(st));
    {
      float a = 0, b = 0;
      HBP_CUDA(cudaEventElapsedTime(&a, sw->e0, sw->e1));
      HBP_CUDA(cudaEventElapsedTime(&b, sw->k0, sw->k1));
      dev_ms += a;
      ker_ms += b;
      if (getenv("HBP_SWEEP_TIMING")) {  // probe: set-up / kernel / outputs
        float c = 0, d = 0;
        cudaEventElapsedTime(&c, sw->e0, sw->k0);
        cudaEventElapsedTime(&d, sw->k1, sw->e1);
        fprintf(stderr, "sweep pass: setup %.3f ms kernel %.3f ms outputs %.3f ms\n", c, b, d);
      }
    }
    compactions += (int)h_misc[2];
    int maxit_seen = 0;
    for (int j = 0; j < ns; ++j) maxit_seen = std::max(maxit_seen, h_ri[j]);
    const size_t rows = (size_t)maxit_seen + 2;
    HBP_CUDA(cudaMemcpyAsync(h_db.data(), d_db, rows * S * 8, cudaMemcpyDeviceToHost, st));
    HBP_CUDA(cudaMemcpyAsync(h_uk.data(), d_uk, rows * S * 8, cudaMemcpyDeviceToHost, st));
    HBP_CUDA(cudaMemcpyAsync(h_um.data(), d_um, rows * S * 4, cudaMemcpyDeviceToHost, st));
    HBP_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < ns; ++j) {
      hbp_set_result &r = out->sets[base + j];
      std::memset(&r, 0, sizeof(r));
      const int it = h_ri[j];
      r.iterations = it;
      r.converged = h_rs[j] == 1;
      std::memcpy(&r.last_delta, &h_db[(size_t)it * S + j], 8);
      if (out->deltas)
        for (int i = 1; i <= it; ++i)
          std::memcpy(&out->deltas[(size_t)(base + j) * max_it + (i - 1)], &h_db[(size_t)i * S + j], 8);
      if (h_rs[j] == 4) {
        r.underflow_iteration = it;
        const unsigned long long key = h_uk[(size_t)it * S + j];
        if (key != ~0ull) {  // the sweep's own report (kept for fp32 sets only)
          const int kind = (int)(key >> 32);
          const int32_t pos = (int32_t)(key & 0xffffffffu);
          r.underflow_kind = kind == 0 ? 1 : 2;
          r.underflow_index = kind == 0 ? L.vtof2canon[pos] : -1;
        } else {
          r.underflow_kind = 3;
          r.underflow_index = h_um[(size_t)it * S + j];
        }
        uf_sets.push_back(base + j);
      }
    }
    ++passes;
  }
  for (int j : uf_sets) {
    hbp_status st = attribute_set(sw, opt, ev, j, fp32, &out->sets[j]);
    if (st != HBP_OK) return st;
  }
  out->device_ms = dev_ms;
  out->kernel_ms = ker_ms;
  out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  out->launches = (int32_t)launches;
  out->passes = passes;
  out->compactions = compactions;
  hbp::set_last_launches(launches);
  return HBP_OK;
}

}  // extern "C"
