// A compiled C++ consumer of the C-ABI (include/babplan_cuda.h, libbabplan_cuda.so): what the
// reference's plan() caller (proj/src/bab.cpp:266-415 via INTEGRATION.md 1) does when its CPU path
// is replaced.  It plans the reference's own smoke-test scenario (proj/tests/python/test_smoke.py:
// 10-25, 60-76: a zero-hidden-layer model generate_model(seed=1, widths=[4, 2]), relative features,
// x0 = 0.4, target 0, H = 3, u in [-0.5, 0.5]^2) with the default planner configuration
// (bab.hpp:45-62, search.hpp:18-46), checks that the objective of the returned action equals the
// plan's objective (the same deterministic rollout kernel) and that the status / last-error
// mapping to C++ exceptions works, and prints one JSON line.
//   g++ -std=c++17 -I include tests/native/capi_consumer.cpp -L paper_2412_09584_b200/_lib \
//       -lbabplan_cuda -Wl,-rpath,<abs lib dir> -o tests/native/_capi_consumer
#include <babplan_cuda.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

std::string last_error() {
  char buf[1024];
  bp_get_last_error(buf, sizeof(buf));
  return buf;
}

// bab_cuda.cpp's status -> exception mapping (babplan_cli.cpp:917-932)
void check(bp_status s) {
  if (s == BP_OK) return;
  if (s == BP_INVALID_ARGUMENT) throw std::invalid_argument(last_error());
  if (s == BP_LOGIC) throw std::logic_error(last_error());
  throw std::runtime_error(last_error());
}

}  // namespace

int main() {
  try {
    bp_ctx* ctx = nullptr;
    check(bp_init(0, &ctx));
    // generate_model(seed=1, widths=[4, 2]) (model.cpp:136-158): W 2x4 then b 2
    const int widths[2] = {4, 2};
    std::vector<double> params(2 * 4 + 2);
    check(bp_generate_model(1, 2, widths, params.data()));
    const double* W[1] = {params.data()};
    const double* b[1] = {params.data() + 8};
    const int relu[1] = {0};
    const double x0[2] = {0.4, 0.4}, target[2] = {0.0, 0.0}, p0[2] = {0.0, 0.0};
    const double ulo[2] = {-0.5, -0.5}, uhi[2] = {0.5, 0.5}, axis[2] = {1.0, 1.0};
    const int H = 3;
    std::vector<double> wt(H, 1.0);  // tracking_weight with gamma 0 (model.cpp:160-164)
    bp_cost_op sq{};
    sq.kind = BP_OP_SQDIST;
    sq.src0 = BP_VAL_X;
    sq.src1 = -1;
    sq.dim = 1;
    sq.in_dim = 2;
    sq.target = target;
    sq.weight = axis;
    sq.weight_by_step = 1;
    sq.is_term = 1;
    bp_objective_desc d{};
    d.ks = 2;
    d.ka = 2;
    d.kd = 2;
    d.horizon = H;
    d.feature_mode = BP_FEATURE_RELATIVE;
    d.n_layers = 1;
    d.widths = widths;
    d.W = W;
    d.b = b;
    d.relu_after = relu;
    d.x0 = x0;
    d.p0 = p0;
    d.u_lower = ulo;
    d.u_upper = uhi;
    d.step_weight = wt.data();
    d.n_ops = 1;
    d.ops = &sq;
    d.stop_rule = BP_STOP_LAST_RELU;
    check(bp_load_objective(ctx, &d));

    // default_config() (bench.cpp:170-258): batch 4, eta 0.75, T 0.05, top 1 %, CEM 1000 x 10
    bp_planner_config pc{};
    pc.batch = 4;
    pc.eta = 0.75;
    pc.temperature = 0.05;
    pc.top_percent = 1.0;
    pc.min_width = 1e-6;
    pc.bound_mode = BP_BOUND_EMPIRICAL;
    pc.alpha = BP_ALPHA_ADAPTIVE;
    pc.split_rule = BP_SPLIT_SAMPLES;
    pc.seed = 0;
    pc.search.method = BP_SEARCH_CEM;
    pc.search.samples_per_iter = 1000;
    pc.search.iterations = 10;
    pc.search.top_capacity = 512;
    pc.search.cem_agents = 4;
    pc.search.cem_elites = 10;
    pc.search.cem_jitter = 1e-3;
    pc.search.cem_init_sigma = 0.5;
    pc.search.mppi_noise_frac = 0.25;
    pc.search.mppi_temperature = 10.0;
    pc.search.gd_base_step = 0.01;
    pc.max_iterations = 50;
    pc.wall_clock_ms = 0.0;
    pc.target_objective = -INFINITY;
    bp_result* r = nullptr;
    check(bp_plan(ctx, &pc, nullptr, 1, &r));
    double uf = 0, min_lf = 0;
    int certified = 0, iters = 0, n_trace = 0, dim = 0;
    int64_t samples = 0;
    char stop[64];
    check(bp_result_summary(r, &uf, &min_lf, &certified, &samples, &iters, stop, sizeof(stop), &n_trace, &dim));
    std::vector<double> best(static_cast<size_t>(dim));
    check(bp_result_best(r, best.data()));
    std::vector<bp_trace_row> trace(static_cast<size_t>(n_trace));
    check(bp_result_trace(r, trace.data(), n_trace));
    check(bp_result_free(r));

    // objective_value(plan.action) == plan.objective to 1e-9 (test_smoke.py:75-76)
    std::vector<float> act(best.begin(), best.end());
    float cost = 0.f;
    int bad = 0;
    check(bp_rollout(ctx, 1, 1, act.data(), &cost, nullptr, nullptr, nullptr, &bad));
    const bool same = std::fabs(static_cast<double>(cost) - uf) <= 1e-9 && bad == 0;
    bool incumbent_monotone = true;
    for (int i = 1; i < n_trace; ++i) incumbent_monotone = incumbent_monotone && trace[i].uf <= trace[i - 1].uf;

    // error mapping: a malformed call raises std::invalid_argument with the library's message
    std::string err;
    try {
      check(bp_plan(ctx, nullptr, nullptr, 1, &r));
    } catch (const std::invalid_argument& e) {
      err = e.what();
    }
    check(bp_destroy(ctx));
    std::printf(
        "{\"objective\": %.12g, \"objective_value\": %.12g, \"same\": %s, \"lower_bound\": %.12g, \"iterations\": %d, "
        "\"stop_reason\": \"%s\", \"samples\": %lld, \"trace_rows\": %d, \"incumbent_monotone\": %s, "
        "\"invalid_argument\": \"%s\"}\n",
        uf, static_cast<double>(cost), same ? "true" : "false", min_lf, iters, stop, static_cast<long long>(samples), n_trace,
        incumbent_monotone ? "true" : "false", err.c_str());
    return same && incumbent_monotone && !err.empty() ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "capi_consumer: %s\n", e.what());
    return 2;
  }
}
