// oracle_capi.cpp -- TEST INFRASTRUCTURE ONLY.
// Objective builder from bp_objective_desc (restating build_objective,
// model.cpp:310-387, and generate_model, model.cpp:136-158) plus a flat C
// API so tests/ and bench.py can drive the oracle through ctypes.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../include/babplan_cuda.h"
#include "oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return BP_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return BP_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return BP_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BP_RUNTIME;
  }
}

Vec vec_of(const double* p, int n) { return p ? Vec(p, p + n) : Vec(static_cast<size_t>(n), 0.0); }
Mat mat_of(const double* p, int r, int c) {
  Mat m(r, c);
  std::memcpy(m.a.data(), p, sizeof(double) * static_cast<size_t>(r) * c);
  return m;
}

struct ObjHandle {
  std::shared_ptr<const Objective> obj;
  std::shared_ptr<GraphObjective> graph_obj;  // null for the synthetic objective
  BoxDomain box;
  std::vector<StepNodes> steps;
};

// model.cpp:310-387 generalised: the per-step cost terms come from the
// descriptor's cost program; for the reference CostForms the program lists
// exactly the nodes build_objective creates, in the same order.
BuiltObjective build_from_desc(const bp_objective_desc& d) {
  const int ks = d.ks, ka = d.ka, kd = d.kd, H = d.horizon;
  if (ks <= 0 || ka <= 0 || kd <= 0 || H < 1) throw std::invalid_argument("objective: bad dimensions");
  if (ka != kd) throw std::invalid_argument("objective: action and effector dimensions must match");
  if (d.feature_mode == BP_FEATURE_RELATIVE && ks % kd != 0)
    throw std::invalid_argument("objective: state must be whole keypoints of workspace dimension");
  if (d.n_layers < 1 || d.widths[0] != ks + ka || d.widths[d.n_layers] != ks)
    throw std::invalid_argument("objective: model must map state plus action to the state");
  CompGraph g;
  GraphMeta meta;
  BuiltObjective built;
  const int U = g.add_input(ka * H);
  int x_prev = g.add_constant(vec_of(d.x0, ks));
  int p_prev = g.add_constant(vec_of(d.p0, kd));
  Mat tile(ks, kd);
  for (int k = 0; k < ks / kd; ++k)
    for (int j = 0; j < kd; ++j) tile(k * kd + j, j) = -1.0;
  std::vector<int> cost_terms;
  for (int t = 1; t <= H; ++t) {
    StepNodes sn;
    const int u_t = g.add_slice(U, (t - 1) * ka, ka);
    int feat;
    if (d.feature_mode == BP_FEATURE_RELATIVE) {
      const int neg = g.add_linear(p_prev, tile, Vec(static_cast<size_t>(ks), 0.0));
      const int rel = g.add_sum({x_prev, neg});
      feat = g.add_concat({rel, u_t});
    } else {
      feat = g.add_concat({x_prev, u_t});
    }
    int h = feat;
    for (int l = 0; l < d.n_layers; ++l) {
      const int in = d.widths[l], out = d.widths[l + 1];
      h = g.add_linear(h, mat_of(d.W[l], out, in), vec_of(d.b[l], out));
      if (d.relu_after[l]) {
        sn.preact.push_back(h);
        h = g.add_relu(h);
        meta.final_step_last_relu = h;
      }
    }
    const int x_t = h;
    const int p_t = g.add_sum({p_prev, u_t});
    meta.step_states.push_back(x_t);
    sn.u = u_t;
    sn.x = x_t;
    sn.p = p_t;
    auto val = [&](int id) -> int {
      if (id == BP_VAL_X) return x_t;
      if (id == BP_VAL_U) return u_t;
      if (id == BP_VAL_P) return p_t;
      const int k = id - BP_VAL_OP0;
      if (k < 0 || k >= static_cast<int>(sn.ops.size())) throw std::invalid_argument("cost op: bad source");
      return sn.ops[static_cast<size_t>(k)];
    };
    for (int i = 0; i < d.n_ops; ++i) {
      const bp_cost_op& op = d.ops[i];
      const int src = val(op.src0);
      const int in = g.node(src).dim;
      int node = -1;
      switch (op.kind) {
        case BP_OP_LINEAR:
          node = g.add_linear(src, mat_of(op.W, op.dim, in), vec_of(op.b, op.dim));
          break;
        case BP_OP_RELU:
          node = g.add_relu(src);
          break;
        case BP_OP_SUM:
          node = op.src1 >= 0 ? g.add_sum({src, val(op.src1)}) : g.add_sum({src});
          break;
        case BP_OP_SCALAR_AFFINE:
          node = g.add_scalar_affine(src, op.scale, op.offset);
          break;
        case BP_OP_SQDIST: {
          Vec w = vec_of(op.weight, in);
          if (op.weight_by_step) {
            const double wt = d.step_weight[t - 1];
            for (double& x : w) x = wt * x;  // tracking_weight(t) * axis
          }
          node = g.add_squared_distance(src, vec_of(op.target, in), std::move(w));
          break;
        }
        case BP_OP_HINGE:
          node = g.add_penalty_hinge(src, vec_of(op.center, in), op.radius, op.penalty);
          break;
        case BP_OP_SLICE:
          node = g.add_slice(src, op.begin, op.dim);
          break;
        default:
          throw std::invalid_argument("cost op: unknown kind");
      }
      sn.ops.push_back(node);
      if (op.is_term) cost_terms.push_back(node);
    }
    built.steps.push_back(std::move(sn));
    x_prev = x_t;
    p_prev = p_t;
  }
  if (cost_terms.empty()) throw std::invalid_argument("objective: cost program has no terms");
  g.set_output(g.add_sum(cost_terms));
  g.finalize();
  auto obj = std::make_shared<GraphObjective>(std::move(g), std::move(meta));
  if (d.stop_rule == BP_STOP_EVERY_STEP_OUTPUT) {
    obj->set_stop_rule(StopRule::kEveryStepOutput);
  } else if (d.stop_rule == BP_STOP_CUSTOM) {
    std::vector<int> ids;
    for (int i = 0; i < d.n_custom_stops; ++i) {
      const int t = d.custom_stop_steps[i];
      if (t < 1 || t > H) throw std::invalid_argument("stop set: step outside horizon");
      ids.push_back(built.steps[static_cast<size_t>(t - 1)].x);
    }
    obj->set_stop_rule(StopRule::kCustom, ids);
  }
  built.objective = obj;
  Vec lo(static_cast<size_t>(ka * H)), hi(static_cast<size_t>(ka * H));
  for (int t = 0; t < H; ++t)
    for (int j = 0; j < ka; ++j) {
      lo[static_cast<size_t>(t * ka + j)] = d.u_lower[j];
      hi[static_cast<size_t>(t * ka + j)] = d.u_upper[j];
    }
  built.box = BoxDomain(std::move(lo), std::move(hi));
  return built;
}

SearcherConfig search_cfg(const bp_search_config& c) {
  SearcherConfig s;
  s.method = c.method == BP_SEARCH_MPPI ? SearchMethod::kMppi : c.method == BP_SEARCH_GD ? SearchMethod::kGd : SearchMethod::kCem;
  s.samples_per_iter = c.samples_per_iter;
  s.iterations = c.iterations;
  s.top_capacity = c.top_capacity;
  s.seed = c.seed;
  s.cem.agents = c.cem_agents;
  s.cem.elites = c.cem_elites;
  s.cem.jitter = c.cem_jitter;
  s.cem.init_sigma = c.cem_init_sigma;
  s.mppi.noise_frac = c.mppi_noise_frac;
  s.mppi.temperature = c.mppi_temperature;
  s.mppi.noise_ratios.assign(c.mppi_noise_ratios, c.mppi_noise_ratios + c.mppi_n_noise);
  s.mppi.temperature_ratios.assign(c.mppi_temperature_ratios, c.mppi_temperature_ratios + c.mppi_n_temp);
  s.gd.base_step = c.gd_base_step;
  s.gd.step_ratios.assign(c.gd_step_ratios, c.gd_step_ratios + c.gd_n_ratios);
  return s;
}

PlannerConfig planner_cfg(const bp_planner_config& c) {
  PlannerConfig p;
  p.batch = c.batch;
  p.eta = c.eta;
  p.temperature = c.temperature;
  p.top_percent = c.top_percent;
  p.min_width = c.min_width;
  p.bound_mode = c.bound_mode == BP_BOUND_FULL_CROWN ? BoundMode::kFullCrown
                 : c.bound_mode == BP_BOUND_INTERVAL ? BoundMode::kEarlyStopInterval
                                                     : BoundMode::kEarlyStopEmpirical;
  p.alpha = c.alpha == BP_ALPHA_ZERO ? AlphaPolicy::kZero : c.alpha == BP_ALPHA_ONE ? AlphaPolicy::kOne : AlphaPolicy::kAdaptive;
  p.split_rule = c.split_rule;
  p.search = search_cfg(c.search);
  p.max_iterations = c.max_iterations;
  p.wall_clock_ms = c.wall_clock_ms;
  p.target_objective = c.target_objective;
  p.seed = c.seed;
  return p;
}

BoundMode bound_mode(int m) {
  return m == BP_BOUND_FULL_CROWN ? BoundMode::kFullCrown : m == BP_BOUND_INTERVAL ? BoundMode::kEarlyStopInterval : BoundMode::kEarlyStopEmpirical;
}
AlphaPolicy alpha_policy(int a) {
  return a == BP_ALPHA_ZERO ? AlphaPolicy::kZero : a == BP_ALPHA_ONE ? AlphaPolicy::kOne : AlphaPolicy::kAdaptive;
}

struct Reports {
  std::vector<SearchReport> r;
};

}  // namespace

extern "C" {

size_t or_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    std::strncpy(buf, g_err.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return g_err.size();
}
void or_set_threads(int n) { set_thread_count(n); }
int or_thread_count() { return thread_count(); }

// ------------------------------------------------------------------ rng
void* or_rng_new(uint64_t seed) { return new Rng(seed); }
void or_rng_free(void* r) { delete static_cast<Rng*>(r); }
double or_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
double or_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
uint64_t or_rng_bits(void* r) { return static_cast<Rng*>(r)->bits(); }
int or_rng_uniform_int(void* r, int n) { return static_cast<Rng*>(r)->uniform_int(n); }
uint64_t or_mix_seed(uint64_t m, uint64_t s) { return mix_seed(m, s); }

// generate_model (model.cpp:136-158): params = W0, b0, W1, b1, ... (doubles).
int or_generate_model(uint64_t seed, int n_widths, const int* widths, double* params) {
  return guard([&] {
    if (n_widths < 2) throw std::invalid_argument("generate_model: need at least two widths");
    for (int i = 0; i < n_widths; ++i)
      if (widths[i] <= 0) throw std::invalid_argument("generate_model: widths must be positive");
    Rng rng(seed);
    size_t off = 0;
    for (int li = 0; li + 1 < n_widths; ++li) {
      const int in = widths[li], out = widths[li + 1];
      const double a = std::sqrt(6.0 / (in + out));
      for (int r = 0; r < out * in; ++r) params[off++] = rng.uniform(-a, a);
      for (int r = 0; r < out; ++r) params[off++] = rng.uniform(-a, a);
    }
  });
}

// ---------------------------------------------------------------- graph
void* or_graph_new() { return new CompGraph(); }
void or_graph_free(void* g) { delete static_cast<CompGraph*>(g); }
#define G static_cast<CompGraph*>(g)
int or_graph_add_input(void* g, int dim, int* id) { return guard([&] { *id = G->add_input(dim); }); }
int or_graph_add_constant(void* g, const double* v, int n, int* id) { return guard([&] { *id = G->add_constant(vec_of(v, n)); }); }
int or_graph_add_linear(void* g, int arg, const double* W, int rows, int cols, const double* b, int* id) {
  return guard([&] { *id = G->add_linear(arg, mat_of(W, rows, cols), vec_of(b, rows)); });
}
int or_graph_add_relu(void* g, int arg, int* id) { return guard([&] { *id = G->add_relu(arg); }); }
int or_graph_add_sum(void* g, const int* args, int n, int* id) {
  return guard([&] { *id = G->add_sum(std::vector<int>(args, args + n)); });
}
int or_graph_add_scalar_affine(void* g, int arg, double s, double o, int* id) { return guard([&] { *id = G->add_scalar_affine(arg, s, o); }); }
int or_graph_add_squared_distance(void* g, int arg, const double* t, const double* w, int n, int* id) {
  return guard([&] { *id = G->add_squared_distance(arg, vec_of(t, n), vec_of(w, n)); });
}
int or_graph_add_penalty_hinge(void* g, int arg, const double* c, int n, double r, double p, int* id) {
  return guard([&] { *id = G->add_penalty_hinge(arg, vec_of(c, n), r, p); });
}
int or_graph_add_concat(void* g, const int* args, int n, int* id) {
  return guard([&] { *id = G->add_concat(std::vector<int>(args, args + n)); });
}
int or_graph_add_slice(void* g, int arg, int begin, int len, int* id) { return guard([&] { *id = G->add_slice(arg, begin, len); }); }
int or_graph_set_output(void* g, int node) { return guard([&] { G->set_output(node); }); }
int or_graph_finalize(void* g) { return guard([&] { G->finalize(); }); }
int or_graph_size(void* g) { return G->size(); }
int or_graph_node_dim(void* g, int id) { return G->node(id).dim; }
#undef G

// ------------------------------------------------------------ objective
#define O static_cast<ObjHandle*>(h)
// Wraps a finalized graph (copied) as a GraphObjective; step_states may be empty.
int or_objective_from_graph(void* g, const int* step_states, int n_steps, int final_step_last_relu, void** out) {
  return guard([&] {
    GraphMeta meta;
    meta.step_states.assign(step_states, step_states + n_steps);
    meta.final_step_last_relu = final_step_last_relu;
    auto* oh = new ObjHandle();
    oh->graph_obj = std::make_shared<GraphObjective>(*static_cast<CompGraph*>(g), meta);
    oh->obj = oh->graph_obj;
    *out = oh;
  });
}
int or_objective_from_desc(const bp_objective_desc* desc, void** out) {
  return guard([&] {
    BuiltObjective b = build_from_desc(*desc);
    auto* oh = new ObjHandle();
    oh->graph_obj = b.objective;
    oh->obj = b.objective;
    oh->box = b.box;
    oh->steps = std::move(b.steps);
    *out = oh;
  });
}
int or_objective_synthetic(int d, void** out) {
  return guard([&] {
    auto* oh = new ObjHandle();
    auto s = std::make_shared<SyntheticObjective>(d);
    oh->box = s->domain();
    oh->obj = s;
    *out = oh;
  });
}
void or_objective_free(void* h) { delete O; }
int or_objective_dim(void* h) { return O->obj->dim(); }
int or_objective_set_stop_rule(void* h, int rule, const int* ids, int n) {
  return guard([&] {
    if (!O->graph_obj) throw std::invalid_argument("not a graph objective");
    O->graph_obj->set_stop_rule(rule == BP_STOP_EVERY_STEP_OUTPUT ? StopRule::kEveryStepOutput
                                : rule == BP_STOP_CUSTOM ? StopRule::kCustom : StopRule::kLastRelu,
                                std::vector<int>(ids, ids + n));
  });
}
int or_objective_sets(void* h, int which, int* out, int cap) {  // 0 stop, 1 watch, 2 relu nodes, 3 step states
  if (!O->graph_obj) return -1;
  const std::vector<int>& s = which == 0 ? O->graph_obj->stop_set()
                              : which == 1 ? O->graph_obj->watch_set()
                              : which == 2 ? O->graph_obj->meta().relu_nodes : O->graph_obj->meta().step_states;
  for (size_t i = 0; i < s.size() && static_cast<int>(i) < cap; ++i) out[i] = s[i];
  return static_cast<int>(s.size());
}
int or_objective_final_step_last_relu(void* h) { return O->graph_obj ? O->graph_obj->meta().final_step_last_relu : -1; }
int or_objective_box(void* h, double* lo, double* hi) {
  const int n = O->box.dim();
  for (int j = 0; j < n; ++j) {
    lo[j] = O->box.lower()[static_cast<size_t>(j)];
    hi[j] = O->box.upper()[static_cast<size_t>(j)];
  }
  return n;
}
// Node ids of step t (0-based): u, x, p, hidden preacts, cost-op nodes.
int or_objective_step_nodes(void* h, int t, int* uxp, int* preact, int cap_pre, int* ops, int cap_ops) {
  if (t < 0 || t >= static_cast<int>(O->steps.size())) return -1;
  const StepNodes& s = O->steps[static_cast<size_t>(t)];
  uxp[0] = s.u;
  uxp[1] = s.x;
  uxp[2] = s.p;
  for (size_t i = 0; i < s.preact.size() && static_cast<int>(i) < cap_pre; ++i) preact[i] = s.preact[i];
  for (size_t i = 0; i < s.ops.size() && static_cast<int>(i) < cap_ops; ++i) ops[i] = s.ops[i];
  return static_cast<int>(s.preact.size() * 1000 + s.ops.size());
}
int or_objective_graph_size(void* h) { return O->graph_obj ? O->graph_obj->graph().size() : 0; }
int or_objective_node_dim(void* h, int id) { return O->graph_obj->graph().node(id).dim; }

// ------------------------------------------------------------ evaluate
void* or_stats_new() { return new WatchStats(); }
void or_stats_free(void* s) { delete static_cast<WatchStats*>(s); }
int or_stats_get(void* s, int id, double* mn, double* mx, int64_t* count) {
  auto* ws = static_cast<WatchStats*>(s);
  auto it = ws->find(id);
  if (it == ws->end()) return -1;
  for (size_t j = 0; j < it->second.min.size(); ++j) {
    if (mn) mn[j] = it->second.min[j];
    if (mx) mx[j] = it->second.max[j];
  }
  if (count) *count = it->second.count;
  return static_cast<int>(it->second.min.size());
}
int or_stats_set(void* s, int id, const double* mn, const double* mx, int n, int64_t count) {
  NodeStats& ns = (*static_cast<WatchStats*>(s))[id];
  ns.min = vec_of(mn, n);
  ns.max = vec_of(mx, n);
  ns.count = count;
  return 0;
}
int or_stats_ids(void* s, int* out, int cap) {
  auto* ws = static_cast<WatchStats*>(s);
  int i = 0;
  for (auto& kv : *ws) {
    if (i < cap) out[i] = kv.first;
    ++i;
  }
  return i;
}
// Objective evaluate; stats (may be NULL) accumulate the objective's watch set.
int or_objective_evaluate(void* h, const double* batch, int rows, int cols, double* out, void* stats) {
  return guard([&] {
    const Vec v = O->obj->evaluate(mat_of(batch, rows, cols), static_cast<WatchStats*>(stats));
    std::copy(v.begin(), v.end(), out);
  });
}
// Raw graph evaluate with an explicit watch list.
int or_graph_evaluate(void* g, const double* batch, int rows, int cols, double* out, const int* watch, int n_watch,
                      void* stats) {
  return guard([&] {
    std::vector<int> w(watch, watch + n_watch);
    const Vec v = evaluate(*static_cast<CompGraph*>(g), mat_of(batch, rows, cols), stats ? &w : nullptr,
                           static_cast<WatchStats*>(stats));
    std::copy(v.begin(), v.end(), out);
  });
}
// Objective::gradient (objective.hpp:61-62; graph.cpp:403-564 / objective.cpp:100-107).
int or_objective_gradient(void* h, const double* batch, int rows, double* out) {
  return guard([&] {
    const int d = O->obj->dim();
    const Mat m = O->obj->gradient(mat_of(batch, rows, d));
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < d; ++j) out[static_cast<size_t>(i) * d + j] = m(i, j);
  });
}
int or_graph_gradient(void* g, const double* batch, int rows, int cols, double* out) {
  return guard([&] {
    const Mat m = gradient(*static_cast<CompGraph*>(g), mat_of(batch, rows, cols));
    std::copy(m.a.begin(), m.a.end(), out);
  });
}
int or_graph_interval(void* g, const double* lo, const double* hi, int d, int node, double* lo_out, double* hi_out) {
  return guard([&] {
    const IntervalSet iv = interval_forward(*static_cast<CompGraph*>(g), BoxDomain(vec_of(lo, d), vec_of(hi, d)));
    const Vec& l = iv.lo.at(static_cast<size_t>(node));
    const Vec& u = iv.hi.at(static_cast<size_t>(node));
    std::copy(l.begin(), l.end(), lo_out);
    std::copy(u.begin(), u.end(), hi_out);
  });
}

// --------------------------------------------------------------- crown
int or_lower_bound(void* h, const double* lo, const double* hi, int mode, void* stats, int alpha, double* out) {
  return guard([&] {
    if (!O->graph_obj) throw std::invalid_argument("lower_bound: not a graph objective");
    const int d = O->obj->dim();
    *out = lower_bound(*O->graph_obj, BoxDomain(vec_of(lo, d), vec_of(hi, d)), bound_mode(mode),
                       static_cast<WatchStats*>(stats), alpha_policy(alpha));
  });
}
// crown_node_bounds (crown.cpp:379-412) over the given targets, as watch stats
// (test helper: node-by-node parity of the device's full-CROWN passes).
int or_crown_node_stats(void* h, const double* lo, const double* hi, int alpha, const int* ids, int n_ids,
                        void** out) {
  return guard([&] {
    if (!O->graph_obj) throw std::invalid_argument("crown_node_bounds: not a graph objective");
    const int d = O->obj->dim();
    const std::vector<int> targets(ids, ids + n_ids);
    PreactBounds pre = crown_node_bounds(O->graph_obj->graph(), BoxDomain(vec_of(lo, d), vec_of(hi, d)), targets,
                                         alpha_policy(alpha));
    auto* ws = new WatchStats();
    for (int id : targets)
      if (pre.has(id)) {
        NodeStats& ns = (*ws)[id];
        ns.min = pre.at(id).first;
        ns.max = pre.at(id).second;
        ns.count = 1;
      }
    *out = ws;
  });
}
int or_relax_relu(const double* l, const double* u, int n, int policy, double* ls, double* lo, double* us, double* uo) {
  return guard([&] {
    const ReluRelaxation r = relax_relu(vec_of(l, n), vec_of(u, n), alpha_policy(policy));
    std::copy(r.lower_slope.begin(), r.lower_slope.end(), ls);
    std::copy(r.lower_offset.begin(), r.lower_offset.end(), lo);
    std::copy(r.upper_slope.begin(), r.upper_slope.end(), us);
    std::copy(r.upper_offset.begin(), r.upper_offset.end(), uo);
  });
}
// Single-row concretize: terms with dims[i], coeffs concatenated, anchor bounds concatenated.
int or_concretize(double offset, int n_terms, const int* dims, const double* coeffs, const double* los,
                  const double* his, int lower, double* out) {
  return guard([&] {
    LinearBounds lb;
    lb.offset = {offset};
    PreactBounds pre;
    size_t off = 0;
    for (int i = 0; i < n_terms; ++i) {
      Mat c(1, dims[i]);
      std::copy(coeffs + off, coeffs + off + dims[i], c.a.begin());
      lb.terms.push_back({i, c});
      pre.bounds[i] = {vec_of(los + off, dims[i]), vec_of(his + off, dims[i])};
      off += static_cast<size_t>(dims[i]);
    }
    *out = (lower ? concretize_lower(lb, pre) : concretize_upper(lb, pre))[0];
  });
}

// -------------------------------------------------------------- search
int or_batch_search(void* h, int n, const double* los, const double* his, const double* warms,
                    const bp_search_config* cfg, void** out) {
  return guard([&] {
    const int d = O->obj->dim();
    std::vector<BoxDomain> boxes;
    std::vector<Vec> wv(static_cast<size_t>(n));
    std::vector<const Vec*> wp(static_cast<size_t>(n), nullptr);
    for (int i = 0; i < n; ++i) {
      boxes.emplace_back(vec_of(los + static_cast<size_t>(i) * d, d), vec_of(his + static_cast<size_t>(i) * d, d));
      if (warms && !std::isnan(warms[static_cast<size_t>(i) * d])) {
        wv[static_cast<size_t>(i)] = vec_of(warms + static_cast<size_t>(i) * d, d);
        wp[static_cast<size_t>(i)] = &wv[static_cast<size_t>(i)];
      }
    }
    auto* r = new Reports();
    r->r = batch_search(*O->obj, boxes, search_cfg(*cfg), &wp);
    *out = r;
  });
}
// run_cem / run_mppi on injected samples and costs (test hooks): iteration `it` consumes
// rows [0, n_samp) from inj_rows[it] (the incumbent row stays the searcher's own) and the
// values inj_costs[it][R]; after each refit the state is written to the per-iteration outputs.
namespace {
struct TableObjective : Objective {
  int d;
  int R;
  const double* costs;
  mutable int calls = 0;
  int dim() const override { return d; }
  Vec evaluate(const Mat& batch, WatchStats*) const override {
    if (batch.rows != R) throw std::logic_error("TableObjective: unexpected batch size");
    Vec v(costs + static_cast<size_t>(calls) * R, costs + static_cast<size_t>(calls + 1) * R);
    ++calls;
    return v;
  }
};
}  // namespace
int or_search_injected(int d, const double* lo, const double* hi, const double* warm, const bp_search_config* cfg,
                       int iterations, int n_samp, const double* inj_rows, const double* inj_costs, double* out_batch, double* out_mu,
                       double* out_var, double* out_uf, double* out_best, int* out_top_n, double* out_top_val,
                       double* out_top_act) {
  return guard([&] {
    SearcherConfig sc = search_cfg(*cfg);
    sc.iterations = iterations;  // one table entry per iteration
    const int R = n_samp + 1, K = std::max(1, sc.top_capacity);
    TableObjective f;
    f.d = d;
    f.R = R;
    f.costs = inj_costs;
    SearchHooks hooks;
    hooks.inject = [&](int it, Mat& batch) {
      for (int r = 0; r < n_samp; ++r)
        for (int j = 0; j < d; ++j) batch(r, j) = inj_rows[(static_cast<size_t>(it) * n_samp + r) * d + j];
    };
    hooks.after = [&](int it, const Mat& batch, const std::vector<Vec>& mu, const std::vector<Vec>& var,
                      const SearchReport& so_far, const std::vector<TopSample>& top) {
      std::copy(batch.a.begin(), batch.a.end(), out_batch + static_cast<size_t>(it) * R * d);
      const size_t G = mu.size();
      for (size_t g = 0; g < G; ++g) {
        std::copy(mu[g].begin(), mu[g].end(), out_mu + (static_cast<size_t>(it) * G + g) * d);
        if (!var.empty()) std::copy(var[g].begin(), var[g].end(), out_var + (static_cast<size_t>(it) * G + g) * d);
      }
      out_uf[it] = so_far.uf;
      std::copy(so_far.best.begin(), so_far.best.end(), out_best + static_cast<size_t>(it) * d);
      out_top_n[it] = static_cast<int>(top.size());
      for (size_t k = 0; k < top.size(); ++k) {
        out_top_val[static_cast<size_t>(it) * K + k] = top[k].value;
        std::copy(top[k].u.begin(), top[k].u.end(), out_top_act + (static_cast<size_t>(it) * K + k) * d);
      }
    };
    Vec w;
    if (warm != nullptr) w = vec_of(warm, d);
    set_search_hooks(&hooks);
    try {
      search(f, BoxDomain(vec_of(lo, d), vec_of(hi, d)), sc, warm != nullptr ? &w : nullptr);
    } catch (...) {
      set_search_hooks(nullptr);
      throw;
    }
    set_search_hooks(nullptr);
  });
}

void or_reports_free(void* r) { delete static_cast<Reports*>(r); }
int or_report_get(void* rp, int i, double* uf, double* best, int64_t* samples, int* ok, int* n_top) {
  const SearchReport& r = static_cast<Reports*>(rp)->r.at(static_cast<size_t>(i));
  *uf = r.uf;
  if (best) std::copy(r.best.begin(), r.best.end(), best);
  *samples = r.samples;
  *ok = r.ok ? 1 : 0;
  *n_top = static_cast<int>(r.top.size());
  return static_cast<int>(r.best.size());
}
int or_report_top(void* rp, int i, double* values, double* actions) {
  const SearchReport& r = static_cast<Reports*>(rp)->r.at(static_cast<size_t>(i));
  size_t off = 0;
  for (size_t k = 0; k < r.top.size(); ++k) {
    values[k] = r.top[k].value;
    std::copy(r.top[k].u.begin(), r.top[k].u.end(), actions + off);
    off += r.top[k].u.size();
  }
  return static_cast<int>(r.top.size());
}
int or_report_history(void* rp, int i, double* uf_hist, int64_t* samples_hist) {
  const SearchReport& r = static_cast<Reports*>(rp)->r.at(static_cast<size_t>(i));
  for (size_t k = 0; k < r.uf_history.size(); ++k) {
    uf_hist[k] = r.uf_history[k];
    samples_hist[k] = r.samples_history[k];
  }
  return static_cast<int>(r.uf_history.size());
}
void* or_report_stats(void* rp, int i) { return &static_cast<Reports*>(rp)->r.at(static_cast<size_t>(i)).stats; }
// CrownBounder::lower for report i (stats only when the search succeeded).
int or_report_bound(void* h, void* rp, int i, const double* lo, const double* hi, int mode, int alpha, double* out) {
  return guard([&] {
    const int d = O->obj->dim();
    CrownBounder b(O->graph_obj, bound_mode(mode), alpha_policy(alpha));
    *out = b.lower(BoxDomain(vec_of(lo, d), vec_of(hi, d)), &static_cast<Reports*>(rp)->r.at(static_cast<size_t>(i)));
  });
}
// Children bounds of a whole batch in parallel (CPU baseline timing).
int or_reports_bound_all(void* h, void* rp, int n, const double* los, const double* his, int mode, int alpha, double* out) {
  return guard([&] {
    const int d = O->obj->dim();
    CrownBounder b(O->graph_obj, bound_mode(mode), alpha_policy(alpha));
    auto* R = static_cast<Reports*>(rp);
    parallel_chunks(n, [&](int64_t s, int64_t e) {
      for (int64_t i = s; i < e; ++i)
        out[i] = b.lower(BoxDomain(vec_of(los + i * d, d), vec_of(his + i * d, d)), &R->r.at(static_cast<size_t>(i)));
    });
  });
}

// ----------------------------------------------------------------- bab
int or_pick_out(const bp_pool_meta* meta, int n_pool, int n, double eta, double temperature, void* rng,
                int* picked, int* n_picked) {
  return guard([&] {
    DomainPool pool;
    for (int i = 0; i < n_pool; ++i) {
      SubdomainRecord r;
      r.lf = meta[i].lf;
      r.uf = meta[i].uf;
      r.id = i;  // carry the pool index through the pick
      r.log_vol = meta[i].log_vol;
      pool.insert(std::move(r));
    }
    const auto out = pick_out(pool, n, eta, temperature, *static_cast<Rng*>(rng));
    for (size_t k = 0; k < out.size(); ++k) picked[k] = static_cast<int>(out[k].id);
    *n_picked = static_cast<int>(out.size());
  });
}
int or_split(int d, const double* lo, const double* hi, int n_top, const double* top_values, const double* top_u,
             int64_t samples, double top_percent, double min_width, int split_rule, int* axis, double* mid,
             unsigned char* route) {
  return guard([&] {
    SubdomainRecord r;
    r.box = BoxDomain(vec_of(lo, d), vec_of(hi, d));
    r.samples = samples;
    for (int i = 0; i < n_top; ++i)
      r.top.push_back({top_values ? top_values[i] : 0.0, vec_of(top_u + static_cast<size_t>(i) * d, d)});
    const SplitResult s = split(r, top_percent, min_width, 0, split_rule);
    *axis = s.axis;
    *mid = s.lo.box.upper()[static_cast<size_t>(s.axis)];
    for (int i = 0; i < n_top; ++i) route[i] = top_u[static_cast<size_t>(i) * d + s.axis] <= *mid ? 0 : 1;
  });
}
// merge_report (bab.cpp:245-262) on one record: (a_*) the record's list / incumbent,
// (b_*) the search report's.  Outputs the merged list and incumbent.
int or_merge_report(int d, int capacity, int na, const double* a_val, const double* a_act, double a_uf,
                    const double* a_best, int nb, const double* b_val, const double* b_act, double b_uf,
                    const double* b_best, int* n_out, double* out_val, double* out_act, double* out_uf,
                    int* has_best, double* out_best) {
  return guard([&] {
    SubdomainRecord r;
    r.uf = a_uf;
    if (a_best) r.best = vec_of(a_best, d);
    for (int i = 0; i < na; ++i) r.top.push_back({a_val[i], vec_of(a_act + static_cast<size_t>(i) * d, d)});
    SearchReport rep;
    rep.uf = b_uf;
    if (b_best) rep.best = vec_of(b_best, d);
    for (int i = 0; i < nb; ++i) rep.top.push_back({b_val[i], vec_of(b_act + static_cast<size_t>(i) * d, d)});
    merge_report(r, std::move(rep), capacity);
    *n_out = static_cast<int>(r.top.size());
    for (size_t i = 0; i < r.top.size(); ++i) {
      out_val[i] = r.top[i].value;
      std::copy(r.top[i].u.begin(), r.top[i].u.end(), out_act + i * static_cast<size_t>(d));
    }
    *out_uf = r.uf;
    *has_best = r.best.empty() ? 0 : 1;
    if (!r.best.empty()) std::copy(r.best.begin(), r.best.end(), out_best);
  });
}
int or_prune(const bp_pool_meta* meta, int n_pool, double incumbent, int* keep, int* n_keep, double* removed) {
  return guard([&] {
    DomainPool pool;
    for (int i = 0; i < n_pool; ++i) {
      SubdomainRecord r;
      r.lf = meta[i].lf;
      r.uf = meta[i].uf;
      r.id = i;
      r.log_vol = meta[i].log_vol;
      pool.insert(std::move(r));
    }
    *removed = prune(pool, incumbent);
    *n_keep = static_cast<int>(pool.size());
    for (size_t k = 0; k < pool.size(); ++k) keep[k] = static_cast<int>(pool.records()[k].id);
  });
}
double or_separable_term_min(double a, double b) { return SeparableBounder::term_min(a, b); }

struct PlanHandle {
  PlanResult r;
};
int or_plan(void* h, const bp_planner_config* cfg, const double* warm, int method_babnd, void** out) {
  return guard([&] {
    const int d = O->obj->dim();
    Vec w;
    if (warm) w = vec_of(warm, d);
    auto* ph = new PlanHandle();
    try {
      ph->r = method_babnd ? plan(O->obj, O->box, planner_cfg(*cfg), nullptr, warm ? &w : nullptr)
                           : sample_only_plan(O->obj, O->box, planner_cfg(*cfg), warm ? &w : nullptr);
    } catch (...) {
      delete ph;
      throw;
    }
    *out = ph;
  });
}
// plan() replaying the device planner's per-child search reports and bounds (PlanReplay): child c
// (in the order plan() creates them, root first) takes iteration it[c], box lo/hi (checked against
// the oracle's own split: a mismatch is counted), lf, uf, best, its top list (n_top, values,
// actions, ascending) and samples.  Returns the plan; *box_mismatch counts boxes that differed,
// *order_mismatch requests that did not match the log's (iteration, index) sequence.
int or_plan_replay(void* h, const bp_planner_config* cfg, int n_log, const int* it, const double* lo, const double* hi,
                   const double* lf, const double* uf, const double* best, const int* n_top, const int* top_off,
                   const double* top_val, const double* top_act, const int64_t* samples, const int* ok, int* box_mismatch,
                   int* order_mismatch, void** out) {
  return guard([&] {
    const int d = O->obj->dim();
    int cursor = 0, iter_base = 0, cur_iter = 0;
    *box_mismatch = 0;
    *order_mismatch = 0;
    PlanReplay rp;
    rp.report = [&](int iter, int index, const BoxDomain& box) {
      if (iter != cur_iter) {
        iter_base = cursor;
        cur_iter = iter;
      }
      const int c = iter_base + index;
      if (c >= n_log || it[c] != iter) {
        ++*order_mismatch;
        throw std::runtime_error("plan replay: the oracle asked for a child the device did not search");
      }
      cursor = std::max(cursor, c + 1);
      for (int j = 0; j < d; ++j)
        if (box.lower()[static_cast<size_t>(j)] != lo[static_cast<size_t>(c) * d + j] ||
            box.upper()[static_cast<size_t>(j)] != hi[static_cast<size_t>(c) * d + j]) {
          ++*box_mismatch;
          break;
        }
      SearchReport r;
      r.ok = ok[c] != 0;
      if (!r.ok) {
        r.error = "evaluate: non-finite objective value (malformed weights?)";
        return r;
      }
      r.uf = uf[c];
      r.best = vec_of(best + static_cast<size_t>(c) * d, d);
      r.samples = samples[c];
      for (int k = 0; k < n_top[c]; ++k) {
        const size_t o = static_cast<size_t>(top_off[c]) + k;
        r.top.push_back({top_val[o], vec_of(top_act + o * d, d)});
      }
      return r;
    };
    rp.lf = [&](int iter, int index) { return lf[(iter == cur_iter ? iter_base : cursor) + index]; };
    auto* ph = new PlanHandle();
    set_plan_replay(&rp);
    try {
      ph->r = plan(O->obj, O->box, planner_cfg(*cfg), nullptr, nullptr);
    } catch (...) {
      set_plan_replay(nullptr);
      delete ph;
      throw;
    }
    set_plan_replay(nullptr);
    *out = ph;
  });
}

void or_plan_free(void* p) { delete static_cast<PlanHandle*>(p); }
int or_plan_summary(void* p, double* uf, double* min_lf, int* certified, int64_t* samples, int* iterations,
                    char* stop, int cap, double* best) {
  const PlanResult& r = static_cast<PlanHandle*>(p)->r;
  *uf = r.uf;
  *min_lf = r.min_lf;
  *certified = r.certified;
  *samples = r.samples;
  *iterations = r.iterations;
  std::strncpy(stop, r.stop_reason.c_str(), static_cast<size_t>(cap - 1));
  stop[cap - 1] = 0;
  std::copy(r.best.begin(), r.best.end(), best);
  return static_cast<int>(r.trace.size());
}
int or_plan_trace(void* p, bp_trace_row* rows, int cap) {
  const PlanResult& r = static_cast<PlanHandle*>(p)->r;
  for (size_t i = 0; i < r.trace.size() && static_cast<int>(i) < cap; ++i) {
    const TraceRow& t = r.trace[i];
    rows[i] = {t.iter, t.uf, t.min_lf, t.pruned_vol, t.selected_vol, t.pool_size, t.samples, t.wall_ms};
  }
  return static_cast<int>(r.trace.size());
}
#undef O

}  // extern "C"
