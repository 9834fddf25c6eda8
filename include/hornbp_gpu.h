/*
 * hornbp_gpu.h -- C ABI of the B200-native loopy-belief-propagation engine.
 *
 * This is the drop-in boundary for the reference package's hot path
 * (hornbp, /root/reference/pkg/src/hornbp). The Python package
 * paper_2509_22337_b200 binds these symbols with ctypes; any other host
 * (C, C++, a cgo/JNI shim) can bind them the same way. Plain pointers and
 * sizes only: no torch, no CUDA types. All host arrays are borrowed for the
 * duration of the call and copied; device state lives behind opaque handles.
 *
 * Conventions
 *   - A "canonical edge index" is the reference's variable-to-factor buffer
 *     position: factor f owns rowptr[f] .. rowptr[f+1]-1, slot 0 = head
 *     (storage.py:45-52). EdgeId(f, s) <-> rowptr[f] + s.
 *   - Every function returns an hbp_status; on failure hbp_last_error()
 *     returns a thread-local message. Non-convergence is not an error.
 *   - Handles are not thread-safe; one CUDA stream per plan.
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference/pkg/src/hornbp):
 *   hbp_compile           schedule.py:335  compile_schedule (+ :261
 *                         dependency_analysis, :293 group_var_to_factor,
 *                         :94 UpdatePoset._toposort_layers)
 *   hbp_graph_create      storage.py:148   initialize -> MessageStore
 *   hbp_plan_create       engine.py:551-555 per-run pass compilation
 *                         (_compile_vtof_pass :380, _compile_ftov_passes :385,
 *                         _compile_marginal_pass :500, split_ftov_batch :357)
 *   hbp_run               engine.py:531    run -> InferenceResult
 *   hbp_pass              engine.py:413/431/472-497 update_vtof_batch,
 *                         update_ftov_batch, update_{and,or}_{body,head}
 *   hbp_marginals         engine.py:526    compute_marginals
 *   hbp_sweep_*           ranking.py:94-135 (the multi-evidence form of
 *                         interaction_loop's clamp + run; new API)
 */
#ifndef HORNBP_GPU_H
#define HORNBP_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hbp_status;
enum {
  HBP_OK = 0,
  HBP_EINVAL = 1,       /* bad argument / malformed graph or schedule  -> ValueError        */
  HBP_EUNDERFLOW = 2,   /* message or marginal mass < 1e-300           -> UnderflowError    */
  HBP_ECUDA = 3,        /* CUDA runtime failure (incl. no device)      -> RuntimeError      */
  HBP_ENCCL = 4,        /* reserved for the collective path                                  */
  HBP_ECYCLE = 5,       /* ordering relation has a cycle               -> ScheduleError     */
  HBP_ENOMEM = 6        /* device or host allocation failed            -> MemoryError       */
};

/* Kinds of factors (storage.py:20-21). */
enum { HBP_AND = 0, HBP_OR = 1 };

/* Flat factor graph in canonical order (graph.py FactorGraph). */
typedef struct {
  int32_t num_variables;
  int32_t num_factors;
  int64_t num_edges;
  const int64_t *factor_rowptr;  /* [num_factors + 1]                     */
  const int32_t *edge_var;       /* [num_edges] variable at each edge     */
  const int8_t *factor_kind;     /* [num_factors] HBP_AND / HBP_OR        */
  const double *p1;              /* [num_factors]                         */
  const double *p2;              /* [num_factors]                         */
} hbp_graph_desc;

/* ---- strategy compiler (host, native C++) ----------------------------------------- */

typedef struct hbp_schedule hbp_schedule;

/* Compile an ordering relation into dependency-analysed batches, identical to
 * hornbp.schedule.compile_schedule. pairs: before[i] < after[i] (canonical
 * edge indices, deduplicated, no self pairs). rank (nullable, [num_edges]):
 * total-order shortcut used by SEQFIX (schedule.py:127-128).
 * On HBP_ECYCLE, *cycle_edge receives the smallest stuck edge. */
hbp_status hbp_compile(const hbp_graph_desc *graph, int64_t num_pairs,
                       const int32_t *before, const int32_t *after,
                       const int32_t *rank, hbp_schedule **out,
                       int64_t *cycle_edge);
/* Topological order only (UpdatePoset.sorted_edges, schedule.py:94-114). */
hbp_status hbp_toposort(int64_t num_edges, int64_t num_pairs, const int32_t *before,
                        const int32_t *after, int32_t *order_out, int64_t *cycle_edge);
hbp_status hbp_schedule_sizes(const hbp_schedule *s, int64_t *num_batches,
                              int64_t *num_s, int64_t *num_t);
/* s_offsets/t_offsets: [num_batches + 1]; s_edges: [num_s]; t_edges: [num_t] */
hbp_status hbp_schedule_copy(const hbp_schedule *s, int64_t *s_offsets, int32_t *s_edges,
                             int64_t *t_offsets, int32_t *t_edges);
void hbp_schedule_destroy(hbp_schedule *s);

/* ---- device layout (MessageStore) -------------------------------------------------- */

typedef struct hbp_graph hbp_graph;

hbp_status hbp_graph_create(const hbp_graph_desc *graph, int32_t device, hbp_graph **out);
void hbp_graph_destroy(hbp_graph *g);
/* Run this graph's work (runs, passes, sweeps) on an external CUDA stream
 * (a cudaStream_t passed as void*, e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the graph's own stream. Calls stay host-synchronous. */
hbp_status hbp_graph_set_stream(hbp_graph *g, void *stream);

/* ---- compiled plan (device-resident level program) ---------------------------------- */

typedef struct hbp_plan hbp_plan;

/* Batches as canonical edge indices: batch i updates factor-to-variable
 * messages s_edges[s_offsets[i] .. s_offsets[i+1]) after refreshing the
 * variable-to-factor messages t_edges[t_offsets[i] .. t_offsets[i+1]). */
hbp_status hbp_plan_create(hbp_graph *g, int64_t num_batches,
                           const int64_t *s_offsets, const int32_t *s_edges,
                           const int64_t *t_offsets, const int32_t *t_edges,
                           hbp_plan **out);
void hbp_plan_destroy(hbp_plan *p);

typedef struct {
  int32_t max_iterations;     /* >= 1                                      */
  int32_t normalize_messages; /* 0/1                                       */
  int32_t record_history;     /* 0/1: history_out receives [iter][V][2]    */
  int32_t evidence_count;     /* clamp factors appended to the graph (info) */
  double tolerance;           /* >= 0; converged iff delta < tolerance     */
  double time_limit;          /* seconds; <= 0 means none                  */
  int32_t precision;          /* 0: fp64, bitwise with the reference (default); 1: fp32
                                 messages (hbp_sweep_run only; marginals within 1e-5)   */
} hbp_options;

typedef struct {
  int32_t iterations;
  int32_t converged;
  double last_delta;
  int32_t underflow_kind;     /* 0 none, 1 variable-to-factor, 2 factor-to-variable, 3 marginal */
  int32_t underflow_iteration;
  int64_t underflow_index;    /* the reference's UnderflowError index (engine.py:155-165,
                                 512-518): rows[argmin(total)] of the first failing pass --
                                 vtof store position (= canonical edge), ftov store position
                                 (MessageStore order, storage.py:55-63; of the clamped graph
                                 when evidence is set), or variable id */
  double device_ms;           /* kernel time of the iteration loop (CUDA events) */
  double total_ms;            /* hbp_run wall time incl. copies              */
} hbp_result;

/* Run the schedule from uniform messages (engine.run). marginals_out: host
 * [V][2] float64 (P0, P1); deltas_out: host [max_iterations];
 * history_out: host [max_iterations][V][2] or NULL. */
hbp_status hbp_run(hbp_plan *p, const hbp_options *opt, double *marginals_out,
                   double *deltas_out, double *history_out, hbp_result *res);

/* History of the last run on this graph (record_history): out [iterations][V][2]
 * float64, iterations <= the run's. Lets a caller size the buffer by the
 * iterations actually run (engine.py:574-575) instead of max_iterations. */
hbp_status hbp_graph_history(hbp_graph *g, int32_t iterations, double *out);

/* Device-resident variant for benchmarking / composition: marginals stay on
 * the device (device pointer of [V][2] float64 returned), no D2H copy. */
hbp_status hbp_run_device(hbp_plan *p, const hbp_options *opt, hbp_result *res,
                          const double **marginals_dev);

/* One pass on a host MessageStore (reference layout: vtof canonical,
 * ftov variable-major in (factor, slot) order).  direction 0 = variable-to-
 * factor (update_vtof_batch), 1 = factor-to-variable (update_ftov_batch).
 * targets: canonical edge indices. Buffers are updated in place. */
hbp_status hbp_pass(hbp_graph *g, int32_t direction, int64_t num_targets,
                    const int32_t *targets, int32_t normalize, double *vtof0,
                    double *vtof1, double *ftov0, double *ftov1,
                    int64_t *underflow_index);
/* compute_marginals on a host store's ftov buffers: out [V][2]. */
hbp_status hbp_marginals(hbp_graph *g, const double *ftov0, const double *ftov1,
                         double *out, int64_t *underflow_var);

/* Evidence for the following runs of this graph: variable var[i] observed
 * value[i] (0/1). Equivalent to clamp_evidence(graph, var[i], value[i]) applied
 * in order (graph.py:189-200) when the plan's schedule is the base graph's
 * PARALL or canonical SEQFIX schedule -- the two whose batches do not change
 * under clamping (the clamp edges only join s_0 / s_{k-1}). n = 0 clears it.
 * Replaces the per-round graph rebuild + recompile of interaction_loop
 * (ranking.py:122-127). */
hbp_status hbp_graph_set_evidence(hbp_graph *g, int32_t n, const int32_t *var, const int8_t *value);

/* Rank a selection (ascending variable ids, e.g. the alarms) by the last run's
 * P1, skipping variables with evidence: rank_alarms order (ranking.py:83-91),
 * computed on the device: any selection size (a radix select of the k-th key,
 * then a sort of the k selected), topk < 16,384. ranked [topk] (-1 padded),
 * p1 [topk] or NULL. */
hbp_status hbp_graph_rank(hbp_graph *g, int32_t num_select, const int32_t *select, int32_t topk,
                          int32_t *ranked, double *p1);

/* Device introspection for the parity tests: copy the device layout back in
 * reference order (rowptr_ftov [V+1], ftov_to_vtof [E]). */
hbp_status hbp_graph_layout(hbp_graph *g, int64_t *rowptr_ftov, int64_t *ftov_to_vtof);

/* Self-check of the device-built layout (hbp_graph_create builds it with
 * kernels): every device array against the host builder's, *mismatches = the
 * number of arrays that differ (0 expected). */
hbp_status hbp_graph_layout_check(hbp_graph *g, int64_t *mismatches);

/* Self-test of the shared-reciprocal division against __ddiv_rn on the device:
 * q_fast/q_ref [2n]: a[i]/b[i] and a[(i+1)%n]/b[i]. */
hbp_status hbp_selftest_division(int64_t n, const double *a, const double *b, double *q_fast,
                                 double *q_ref);

/* ---- multi-evidence sweep (new API; ranking.py:94-135 made embarrassingly parallel) ----
 *
 * Runs many independent evidence sets over one graph under the PARALL schedule.
 * Set j is bitwise identical to engine.run(G_j, Strategy.parall().compile(G_j))
 * where G_j = clamp_evidence applied to the base graph for each (var, value) of
 * set j in order (graph.py:189-200). Sets stop at their own convergence
 * iteration. Sets are processed in passes of hbp_sweep_capacity() sets. */

typedef struct hbp_sweep hbp_sweep;

typedef struct {
  int32_t num_sets;
  const int64_t *offsets;  /* [num_sets + 1] into var / value                  */
  const int32_t *var;      /* observed variable (original id)                   */
  const int8_t *value;     /* 0 = observed false, 1 = observed true             */
} hbp_evidence;

typedef struct {
  int32_t iterations;
  int32_t converged;
  double last_delta;
  int32_t underflow_kind;  /* 0 none, 1 vtof, 2 ftov, 3 marginal; index as hbp_result's, for
                              clamp_evidence(G, set j) (fp32 sets: fp64 re-run's, else -1) */
  int32_t underflow_iteration;
  int64_t underflow_index;
} hbp_set_result;

typedef struct {
  hbp_set_result *sets;          /* host [num_sets], required                           */
  double *deltas;                /* host [num_sets][max_iterations] or NULL             */
  double *marginals;             /* [num_sets][V][2] (P0, P1) or NULL                   */
  int32_t marginals_on_device;   /* 1: marginals is a device pointer on the graph's GPU */
  int32_t num_select;            /* selected variables (ascending original ids)         */
  const int32_t *select;         /* host [num_select]                                   */
  double *p1_select;             /* [num_sets][num_select] P1 of the selection, or NULL */
  int32_t p1_on_device;
  int32_t topk;                  /* ranking of the selection (rank_alarms order)        */
  int32_t *ranked;               /* [num_sets][topk] variable ids, -1 padded, or NULL   */
  int32_t ranked_on_device;
  /* filled in by hbp_sweep_run */
  double device_ms;              /* stream time of all passes (evidence, sweep, outputs) */
  double kernel_ms;              /* the persistent sweep kernel(s) alone                 */
  double wall_ms;
  int32_t launches;
  int32_t passes;
  int32_t compactions;           /* straggler compactions performed (staged kernel)      */
} hbp_sweep_outputs;

/* max_sets_per_pass: 0 = as many as fit in half of the free device memory. */
hbp_status hbp_sweep_create(hbp_graph *g, int32_t max_sets_per_pass, hbp_sweep **out);
int32_t hbp_sweep_capacity(const hbp_sweep *sw);
/* Per-set underflow is reported in sets[j] (HBP_OK overall). */
hbp_status hbp_sweep_run(hbp_sweep *sw, const hbp_options *opt, const hbp_evidence *ev,
                         hbp_sweep_outputs *out);
void hbp_sweep_destroy(hbp_sweep *sw);

/* Number of kernels the last hbp_run launched (bench gpu_launches). */
int64_t hbp_last_launch_count(void);
const char *hbp_last_error(void);
const char *hbp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HORNBP_GPU_H */
