/*
 * babplan_cuda.h -- C-ABI of the B200 BaB-ND hot path.
 *
 * This is the drop-in boundary between a host planner (the reference's C++
 * API / its pybind11 module, or this repo's ctypes module) and the sm_100a
 * kernels in paper_2412_09584_b200/csrc/.  Only plain pointers, sizes and
 * POD structs cross it; no exception, no torch type, no STL container.
 *
 * Every entry point returns a bp_status; the message of the last failure on
 * the calling thread is available through bp_get_last_error().  Host buffers
 * are caller-owned; device buffers are owned by the context.
 *
 * Reference interfaces each entry point replaces (paths under the reference
 * checkout's proj/):
 *   bp_load_objective   build_objective            src/model.cpp:310-387
 *                       GraphObjective sets        src/objective.cpp:13-76
 *   bp_rollout          GraphObjective::evaluate   src/objective.cpp:31-33
 *                       -> evaluate/forward_chunk  src/graph.cpp:252-401
 *   bp_batch_search     batch_search / run_cem /   src/search.cpp:87-209,262-282
 *                       run_mppi / SampleSink      src/search.cpp:37-82
 *   bp_batch_bound      CrownBounder::lower        src/bab.cpp:25-28
 *                       -> lower_bound             src/crown.cpp:440-469
 *   bp_plan             plan / sample_only_plan    src/bab.cpp:266-454
 *   bp_pick_out         pick_out                   src/bab.cpp:85-153
 *   bp_pool_split/merge split / merge_report       src/bab.cpp:155-262
 */
#ifndef BABPLAN_CUDA_H_
#define BABPLAN_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef enum {
  BP_OK = 0,
  BP_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  BP_LOGIC = 2,            /* std::logic_error */
  BP_RUNTIME = 3,          /* std::runtime_error (numeric failure, root search failed) */
  BP_CUDA = 4,
  BP_NCCL = 5,
  BP_UNSUPPORTED = 6
} bp_status;

/* ------------------------------------------------------------- enums */
/* model.hpp:13-16; BP_FEATURE_NETWORK: a bare network over the action box (horizon 1, the
 * MLP reads u only), the graph build_network_objective makes (model.cpp:389-405) for
 * network_lower_bound (pymodule.cpp:192-202); bounds only, no rollouts. */
enum { BP_FEATURE_RELATIVE = 0, BP_FEATURE_ABSOLUTE = 1, BP_FEATURE_NETWORK = 2 };

/* Value ids inside one rollout step's cost program. */
enum { BP_VAL_X = 0, BP_VAL_U = 1, BP_VAL_P = 2, BP_VAL_OP0 = 3 };

/* Cost-program op kinds: the non-structural node kinds of graph.hpp:11-22. */
enum {
  BP_OP_LINEAR = 0,
  BP_OP_RELU = 1,
  BP_OP_SUM = 2, /* src0 (+ src1 when >= 0) */
  BP_OP_SCALAR_AFFINE = 3,
  BP_OP_SQDIST = 4,
  BP_OP_HINGE = 5,
  BP_OP_SLICE = 6
};

enum { BP_STOP_LAST_RELU = 0, BP_STOP_EVERY_STEP_OUTPUT = 1, BP_STOP_CUSTOM = 2 }; /* objective.hpp:38 */
enum { BP_BOUND_FULL_CROWN = 0, BP_BOUND_EMPIRICAL = 1, BP_BOUND_INTERVAL = 2 };    /* crown.hpp:80-84 */
enum { BP_ALPHA_ADAPTIVE = 0, BP_ALPHA_ZERO = 1, BP_ALPHA_ONE = 2 };                /* crown.hpp:13-19 */
enum { BP_SEARCH_CEM = 0, BP_SEARCH_MPPI = 1, BP_SEARCH_GD = 2 };                   /* search.hpp:13 */
enum { BP_SPLIT_SAMPLES = 0, BP_SPLIT_WIDTH = 1 }; /* bab.cpp:172-194 ; WIDTH forces the width-only rule */

/* -------------------------------------------------- objective descriptor */
/*
 * One op of the per-step cost program.  The program is replayed at every
 * step t = 1..H on the values {x_t, u_t, p_t} and produces the step's cost
 * terms, in the node order build_objective (model.cpp:355-370) creates them.
 */
typedef struct {
  int kind;
  int src0, src1;           /* value ids (BP_VAL_*, or BP_VAL_OP0 + i); src1 = -1 unless SUM */
  int dim;                  /* output dimension */
  int in_dim;               /* dimension of src0 */
  int begin;                /* SLICE: y = x[begin : begin + dim] */
  const double* W;          /* LINEAR: dim x in_dim row-major */
  const double* b;          /* LINEAR: dim */
  double scale, offset;     /* SCALAR_AFFINE */
  const double* target;     /* SQDIST: in_dim */
  const double* weight;     /* SQDIST: in_dim, non-negative */
  int weight_by_step;       /* SQDIST: weight_j * step_weight[t-1] (tracking_weight, model.cpp:160-164) */
  const double* center;     /* HINGE: in_dim */
  double radius, penalty;   /* HINGE: penalty * relu(radius - |x - center|) */
  int is_term;              /* scalar op whose output is summed into the objective */
} bp_cost_op;

/*
 * Unrolled-rollout objective: x_t = MLP(features(x_{t-1}, p_{t-1}, u_t)),
 * p_t = p_{t-1} + u_t, objective = sum over steps of the cost program terms.
 * Mirrors build_objective (model.cpp:310-387) generalised to a cost program.
 */
typedef struct {
  int ks, ka, kd, horizon, feature_mode;
  int n_layers;
  const int* widths;          /* n_layers + 1: [ks + ka, hidden..., ks] */
  const double* const* W;     /* per layer: out x in row-major */
  const double* const* b;     /* per layer: out */
  const int* relu_after;      /* per layer */
  const double* x0;           /* ks */
  const double* p0;           /* kd */
  const double* u_lower;      /* ka, per-step action box */
  const double* u_upper;      /* ka */
  const double* step_weight;  /* horizon: w_t */
  int n_ops;
  const bp_cost_op* ops;
  int stop_rule;
  int n_custom_stops;
  const int* custom_stop_steps; /* 1-based steps t whose x_t node is a stop node */
} bp_objective_desc;

/* ------------------------------------------------------ planner config */
/* PlannerConfig / SearcherConfig (bab.hpp:45-62, search.hpp:18-46). */
typedef struct {
  int method;
  int samples_per_iter;
  int iterations;
  int top_capacity;
  uint64_t seed;
  /* CEM */
  int cem_agents, cem_elites;
  double cem_jitter, cem_init_sigma;
  /* MPPI */
  double mppi_noise_frac, mppi_temperature;
  int mppi_n_noise, mppi_n_temp;
  const double* mppi_noise_ratios;
  const double* mppi_temperature_ratios;
  /* GD */
  double gd_base_step;
  int gd_n_ratios;
  const double* gd_step_ratios;
} bp_search_config;

typedef struct {
  int batch;
  double eta, temperature, top_percent, min_width;
  int bound_mode, alpha;
  int split_rule;
  uint64_t seed;
  bp_search_config search;
  int max_iterations;
  double wall_clock_ms;
  double target_objective; /* -inf disables */
} bp_planner_config;

typedef struct {
  int iter;
  double uf, min_lf, pruned_vol, selected_vol;
  int64_t pool_size, samples;
  double wall_ms;
} bp_trace_row; /* TraceRow, bab.hpp:124-133 */

/* ------------------------------------------------------- context */
typedef struct bp_ctx bp_ctx;

/* Creates a context bound to one CUDA device (one process per GPU). */
bp_status bp_init(int device, bp_ctx** out);
bp_status bp_destroy(bp_ctx* ctx);
/* Thread-local message of the last failing call (empty when none). */
size_t bp_get_last_error(char* buf, size_t cap);
/* Subdomain sharding across ranks (one process per GPU, replacing the
 * reference's std::thread fan-out of batch_search, proj/src/search.cpp:262-282, and
 * the serial bound loop, bab.cpp:392-403).  Every rank keeps the pool's heads (id,
 * bounds, volume, width, owner) and replays pick_out / prune identically; the full
 * records live on their owners.  With world > 1 child k of every BaB iteration is
 * searched and bounded on rank k % world: the parent's owner splits it and ships the
 * child record with the all-to-all hook, and the children's heads are shared with
 * the allgather hook.  fn(user, send, bytes, recv) must fill recv (world * bytes)
 * with every rank's send buffer in rank order; a2a(user, send, send_bytes[world],
 * recv, recv_bytes[world]) must deliver rank r's send segment for this rank in rank
 * order (an all-to-all-v of bytes).  Both return 0 on success.  The runtime's hooks are
 * torch.distributed all_gather_into_tensor / all_to_all_single over NCCL (NVLink). */
typedef int (*bp_exchange_fn)(void* user, const void* send, size_t bytes, void* recv);
typedef int (*bp_alltoallv_fn)(void* user, const void* send, const int64_t* send_bytes, void* recv,
                               const int64_t* recv_bytes);
bp_status bp_set_alltoall(bp_ctx* ctx, bp_alltoallv_fn a2a);
bp_status bp_set_exchange(bp_ctx* ctx, int rank, int world, bp_exchange_fn fn, void* user);

/* Device-direct exchange over NCCL (NVLink / NVSwitch), replacing both hooks above: no host
 * callback, and the child records go from the splitting rank's device pack buffer straight
 * into the searching rank's device receive buffer (one grouped ncclSend / ncclRecv per
 * iteration); the heads and status words are all-gathered through small device staging
 * buffers.  Rank 0 makes the 128-byte id with bp_nccl_unique_id, the caller broadcasts it
 * (e.g. torch.distributed), and every rank calls bp_set_nccl collectively.  libnccl.so.2 is
 * dlopen'ed (the process's copy when one is loaded).  bp_nccl_selftest checks an all-gather
 * and an all-to-all-v of `bytes`-sized segments across the ranks: *ok = 1 when every segment
 * arrived in rank order. */
bp_status bp_nccl_unique_id(unsigned char id[128]);
bp_status bp_set_nccl(bp_ctx* ctx, int rank, int world, const unsigned char id[128]);
bp_status bp_nccl_selftest(bp_ctx* ctx, int64_t bytes, int* ok);

/* Launch the context's work on an external stream (NULL = its own stream),
 * e.g. torch.cuda.current_stream(), so caller-side CUDA events time it. */
bp_status bp_set_stream(bp_ctx* ctx, void* cuda_stream);
/* Rollout kernel selection: path 0 = auto (tcgen05 3xTF32 v2 when every layer
 * width is <= 256 and it fits shared memory, else v1 at widths <= 128, else
 * SIMT FP32), 1 = SIMT only, 2 = tcgen05 v1, 3 = tcgen05 v2, -1 = query.
 * *active (optional) = 3 tcgen05 v2, 2 tcgen05 v1, 1 SIMT for the loaded objective. */
bp_status bp_set_rollout_path(bp_ctx* ctx, int path, int* active);
/* The rollout kernel of the loaded objective (as *active above), its 128-row tiles per
 * CTA, rows per CTA and dynamic shared memory per CTA (bytes).  Any pointer may be NULL. */
bp_status bp_rollout_info(bp_ctx* ctx, int* kernel, int* tiles_per_cta, int* rows_per_cta, int64_t* smem_bytes);
/* Host<->device bytes the library copied since the previous call. */
bp_status bp_io_bytes(int64_t* h2d, int64_t* d2h);

/* The separable synthetic objective f(u) = sum_j 5 u_j^2 + cos(50 u_j) on [-1, 1]^d
 * (replaces build_synthetic / SyntheticObjective, proj/src/model.cpp:407-409,
 * proj/src/objective.cpp:82-104).  Its bounder is the exact SeparableBounder
 * (proj/src/bab.cpp:30-83), whatever the configured bound mode. */
bp_status bp_load_synthetic(bp_ctx* ctx, int dim);

/* Uploads weights / cost program; derives stop and watch sets. */
bp_status bp_load_objective(bp_ctx* ctx, const bp_objective_desc* desc);
/* Number of recorded (watched) coordinates per rollout step, and the layout
 * of one step's record: n_slots entries of (kind, index, dim, offset). */
bp_status bp_stat_layout(bp_ctx* ctx, int* per_step, int* n_slots, int* slot_kind, int* slot_index,
                         int* slot_dim, int* slot_offset, int cap);

/* Parity entry: evaluates n_sub x rows action sequences (rows x d each) and
 * returns the objective per row plus the per-subdomain sample extrema of
 * every watched coordinate (layout from bp_stat_layout, H x per_step).
 * states (n_sub x rows x H x ks), emp_lo and emp_hi may be NULL.  Rows are independent: bitwise identical for
 * any n_sub / rows decomposition (graph.hpp:102-103). */
bp_status bp_rollout(bp_ctx* ctx, int n_sub, int rows, const float* actions, float* costs,
                     float* states, float* emp_lo, float* emp_hi, int* nonfinite);

/* Batched search over boxes (double, n_boxes x d).  warm may be NULL or hold
 * NaN rows for "no warm start".  Results stay resident in the context until
 * the next call; read them with bp_report_*. */
bp_status bp_batch_search(bp_ctx* ctx, int n_boxes, const double* lo, const double* hi,
                          const double* warm, const bp_search_config* cfg);
bp_status bp_report_summary(bp_ctx* ctx, double* uf, double* best, int64_t* samples, int* ok,
                            int* n_top);
bp_status bp_report_top(bp_ctx* ctx, int box, double* values, double* actions, int cap);
bp_status bp_report_stats(bp_ctx* ctx, int box, float* emp_lo, float* emp_hi);

/* One sampler update of run_cem / run_mppi on caller-provided rows and costs
 * (parity entry: the sampler and the rollout are bypassed).  It is the device step
 * that batch_search runs after each rollout: SampleSink::consume's incumbent and top-K
 * update (src/search.cpp:41-74) and the CEM elite refit (search.cpp:131-149) or the MPPI
 * weighted mean (search.cpp:192-205), for n_boxes boxes at CEM/MPPI iteration `iter`.
 * rows [n][R][d] with R = agents*floor(M/agents) + 1 (the last row is the incumbent
 * row), costs [n][R].  State in/out: mu, var [n][groups][d] (var: CEM only, may be
 * null for MPPI), uf [n], best [n][d], top_n [n], top_val / top_seq [n][top_capacity],
 * top_act [n][top_capacity][d] (ascending by (value, seq); seq = iter*R + row). */
bp_status bp_search_update(bp_ctx* ctx, int n_boxes, const bp_search_config* cfg, const double* lo,
                           const double* hi, int iter, const float* rows, const float* costs, float* mu,
                           float* var, float* uf, float* best, int* top_n, float* top_val, int* top_seq,
                           float* top_act);

/* Lower bound of every searched box (mode/alpha as in lower_bound). */
bp_status bp_batch_bound(bp_ctx* ctx, int mode, int alpha, double* lf);
/* Lower bound of boxes without search statistics: lower_bound(obj, box, mode,
 * stats = nullptr), i.e. interval intermediate bounds (crown.cpp:449-461). */
bp_status bp_bound_boxes(bp_ctx* ctx, int n_boxes, const double* lo, const double* hi, int mode, int alpha,
                         double* lf);

/* d objective / d actions for n_rows action sequences (Objective::gradient,
 * objective.hpp:61-62: reverse mode over the unrolled graph, graph.cpp:403-564, or the
 * synthetic objective's elementwise derivative, objective.cpp:100-107).  FP64 on the
 * device, returned as FP32; drives the GD searcher (search.cpp:214-245). */
bp_status bp_gradient(bp_ctx* ctx, int64_t n_rows, const float* actions, float* grad);

/* The intermediate (node) bounds the last bound call used, in the stat layout
 * [n_boxes][H][per_step]: the interval pass (interval modes, failed searches) or the
 * full-CROWN node passes (crown_node_bounds, crown.cpp:379-412).  Diagnostic. */
bp_status bp_node_bounds(bp_ctx* ctx, double* lo, double* hi);

/* Full planner: plan() when method_babnd != 0, else sample_only_plan(). */
typedef struct bp_result bp_result;
bp_status bp_plan(bp_ctx* ctx, const bp_planner_config* cfg, const double* warm, int method_babnd,
                  bp_result** out);
/* plan() one iteration at a time: create runs the root search + bound, each
 * step one pick / split / search / bound / merge / prune iteration (stepped =
 * 0 once a termination rule fired), finish the remaining iterations. */
typedef struct bp_planner bp_planner;
bp_status bp_planner_create(bp_ctx* ctx, const bp_planner_config* cfg, const double* warm, bp_planner** out);
bp_status bp_planner_step(bp_planner* p, int* stepped, int* children, int* pool_size);
bp_status bp_planner_finish(bp_planner* p, bp_result** out);
bp_status bp_planner_destroy(bp_planner* p);
bp_status bp_result_summary(const bp_result* r, double* uf, double* min_lf, int* certified,
                            int64_t* samples, int* iterations, char* stop_reason, size_t cap,
                            int* n_trace, int* d);
bp_status bp_result_best(const bp_result* r, double* best);
bp_status bp_result_trace(const bp_result* r, bp_trace_row* rows, int cap);
bp_status bp_result_free(bp_result* r);

/* Device-time accounting of the last bp_plan / bp_batch_search call (ms per
 * kernel family; rollout is the dominant kernel). */
bp_status bp_timing(bp_ctx* ctx, double* rollout_ms, int64_t* rollout_launches, double* bound_ms,
                    double* search_ms, int64_t* launches);

/* Plan log (decision replay; test aid): with logging on, every plan records, per searched child in
 * the order the planner created it (root first; one rank), its iteration, box, search report (uf,
 * best, top list ascending, samples, ok) and lower bound -- the inputs the reference plan()
 * (bab.cpp:266-415) takes from batch_search and the bounder, so its own pick_out / split / merge /
 * prune can be replayed on them and compared (tests/test_gpu_plan_replay.py).  get fills arrays of
 * n_children (boxes, best: n_children x d; top values / actions concatenated in child order). */
bp_status bp_set_plan_log(bp_ctx* ctx, int enable);
bp_status bp_plan_log_size(bp_ctx* ctx, int* n_children, int* total_top);
bp_status bp_plan_log_get(bp_ctx* ctx, int* iter, double* lo, double* hi, double* lf, double* uf, double* best,
                          int* n_top, double* top_val, double* top_act, int64_t* samples, int* ok);

/* Boxes searched since the previous call, and how many of them failed (a non-finite
 * rollout value: SearchReport.ok = false, search.cpp:273-278; their rows are skipped by
 * the rollout and they are bounded by interval propagation). */
bp_status bp_search_counters(bp_ctx* ctx, int64_t* boxes, int64_t* failed);

/* Diagnostics: sustained FP32 FMA throughput of the device (TFLOP/s), the
 * roofline denominator of the SIMT rollout kernel. */
bp_status bp_measure_fp32_peak(int device, double* tflops, double* ms);
/* Dense kind::tf32 tcgen05.mma throughput (TFLOP/s, M=128 N=128 K=8, one CTA
 * per SM), the roofline denominator of the tensor-core rollout. */
bp_status bp_measure_tf32_peak(int device, double* tflops, double* ms);

/* Host-side pool primitives (bit-exact restatements, exposed for parity). */
typedef struct {
  double lf, uf;
  int64_t id;
  double log_vol;
} bp_pool_meta;
/* Picks n records; writes their pool indices (pick order) to picked and
 * returns the count in *n_picked.  rng_state is a handle from bp_rng_new. */
typedef struct bp_rng bp_rng;
bp_status bp_rng_new(uint64_t seed, bp_rng** out);
bp_status bp_rng_free(bp_rng* r);
bp_status bp_rng_uniform(bp_rng* r, double* out);
bp_status bp_rng_normal(bp_rng* r, double* out);
bp_status bp_rng_bits(bp_rng* r, uint64_t* out);
/* n draws of uniform() (kind 0) or normal() (kind 1) into out. */
bp_status bp_rng_fill(bp_rng* r, int kind, int64_t n, double* out);
uint64_t bp_mix_seed(uint64_t master, uint64_t salt);
bp_status bp_pick_out(const bp_pool_meta* pool, int n_pool, int n, double eta, double temperature,
                      bp_rng* rng, int* picked, int* n_picked);
/* Device pool operations (pool.cu; what plan() runs every iteration).
 * bp_pool_split: split() (src/bab.cpp:155-223) of n parents -- boxes lo/hi (n x d),
 * top lists (n_top[i] <= K entries of top_val (n x K) / top_act (n x K x d),
 * ascending), samples -- into 2n children (2i = lower half, 2i+1 = upper half):
 * the axis per parent, child boxes (2n x d) and the routed top lists (child_n,
 * child_val 2n x K, child_act 2n x K x d).  BP_INVALID_ARGUMENT when a parent has no
 * axis above min_width. */
bp_status bp_pool_split(bp_ctx* ctx, int n, int d, int K, const double* lo, const double* hi,
                        const int* n_top, const float* top_val, const float* top_act,
                        const int64_t* samples, double top_percent, double min_width, int split_rule,
                        int* axis, double* child_lo, double* child_hi, int* child_n,
                        float* child_val, float* child_act);
/* bp_pool_merge: merge_report() (src/bab.cpp:245-262) of n records whose incumbent is
 * their list's front -- record lists (a_n, a_val n x K, a_act n x K x d) with search
 * reports (b_n, b_val, b_act, b_uf, b_best n x d, b_failed: a failed report merges
 * nothing); capacity = top_capacity.  Outputs the merged lists, the incumbent value
 * and action, has_best. */
bp_status bp_pool_merge(bp_ctx* ctx, int n, int d, int K, int capacity, const int* a_n,
                        const float* a_val, const float* a_act, const int* b_n, const float* b_val,
                        const float* b_act, const float* b_uf, const float* b_best, const int* b_failed,
                        int* out_n, float* out_val, float* out_act, float* out_uf, int* has_best,
                        float* out_best);
/* Generates a Glorot-uniform MLP exactly like generate_model (model.cpp:136-158). */
bp_status bp_generate_model(uint64_t seed, int n_widths, const int* widths, double* params);

#ifdef __cplusplus
}
#endif

#endif /* BABPLAN_CUDA_H_ */
