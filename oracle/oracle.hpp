// oracle.hpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Eigen-free FP64 CPU restatement of the reference BaB-ND planner's hot path
// (reference checkout: /root/reference/proj).  Used by tests/ as the parity
// checker, by __graft_entry__.smoke() as the checker, and by bench.py's
// cpu_baseline / --impl reference legs as the timed CPU implementation.
// Each function cites the reference file:line it restates.  Compile with
// -ffp-contract=off and no -march so the arithmetic matches the reference's
// x86-64 baseline build (CMakeLists.txt:11) operation by operation.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;

// Row-major dense matrix (replaces the Eigen alias of types.hpp:12).
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * cols + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * cols + j]; }
  double* row(int i) { return a.data() + static_cast<size_t>(i) * cols; }
  const double* row(int i) const { return a.data() + static_cast<size_t>(i) * cols; }
  size_t size() const { return a.size(); }
};

void require_finite(const Vec& v, const std::string& what);
void require_finite(const Mat& m, const std::string& what);

// ----------------------------------------------------------- rng.hpp/.cpp
class Rng {  // rng.hpp:12-35, rng.cpp:8-35
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t bits() { return gen_(); }
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int uniform_int(int n);
  double normal();

 private:
  std::mt19937_64 gen_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};
inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t index) { return master ^ index; }
std::uint64_t mix_seed(std::uint64_t master, std::uint64_t salt);

// ----------------------------------------------------------- parallel.cpp
int thread_count();
void set_thread_count(int n);
void parallel_chunks(std::int64_t n, const std::function<void(std::int64_t, std::int64_t)>& fn);

// ----------------------------------------------------------- types.hpp
class BoxDomain {  // types.hpp:27-50, types.cpp:8-46
 public:
  BoxDomain() = default;
  BoxDomain(Vec lower, Vec upper);
  int dim() const { return static_cast<int>(lower_.size()); }
  const Vec& lower() const { return lower_; }
  const Vec& upper() const { return upper_; }
  double width(int j) const { return upper_[j] - lower_[j]; }
  Vec width() const;
  double max_width() const;
  Vec center() const;
  bool contains(const Vec& u, double tol = 0.0) const;
  double log_volume_relative_to(const BoxDomain& root) const;

 private:
  Vec lower_, upper_;
};

// ----------------------------------------------------------- graph.hpp
enum class NodeKind {
  kInput, kConstant, kLinear, kRelu, kSum, kScalarAffine, kSquaredDistance, kPenaltyHinge,
  kConcat, kSlice,
};

struct GraphNode {  // graph.hpp:26-47
  NodeKind kind;
  std::vector<int> args;
  int dim = 0;
  Mat W;
  Vec b;
  double scale = 1.0, offset = 0.0;
  Vec target, weight;
  Vec center;
  double radius = 0.0, penalty = 1.0;
  int begin = 0;
  Vec value;
};

class CompGraph {  // graph.hpp:52-88, graph.cpp:27-193
 public:
  int add_input(int dim);
  int add_constant(Vec value);
  int add_linear(int arg, Mat W, Vec b);
  int add_relu(int arg);
  int add_sum(std::vector<int> args);
  int add_scalar_affine(int arg, double scale, double offset);
  int add_squared_distance(int arg, Vec target, Vec weight);
  int add_penalty_hinge(int arg, Vec center, double radius, double penalty);
  int add_concat(std::vector<int> args);
  int add_slice(int arg, int begin, int len);
  void set_output(int node);
  void finalize();
  bool finalized() const { return finalized_; }
  int size() const { return static_cast<int>(nodes_.size()); }
  const GraphNode& node(int id) const { return nodes_.at(static_cast<size_t>(id)); }
  int input() const { return input_; }
  int output() const { return output_; }
  int input_dim() const;
  const std::vector<int>& consumers(int id) const { return consumers_.at(static_cast<size_t>(id)); }

 private:
  int add_node(GraphNode node);
  void check_arg(int arg, const char* ctx) const;
  std::vector<GraphNode> nodes_;
  std::vector<std::vector<int>> consumers_;
  int input_ = -1, output_ = -1;
  bool finalized_ = false;
};

struct NodeStats {  // graph.hpp:92-95
  Vec min, max;
  std::int64_t count = 0;
};
using WatchStats = std::map<int, NodeStats>;

Vec evaluate(const CompGraph& g, const Mat& batch, const std::vector<int>* watch = nullptr,
             WatchStats* stats = nullptr);
struct IntervalSet {
  std::vector<Vec> lo, hi;
};
IntervalSet interval_forward(const CompGraph& g, const BoxDomain& box);
// Reverse-mode gradient (graph.cpp:403-564); used by the GD searcher.
Mat gradient(const CompGraph& g, const Mat& batch);

// ----------------------------------------------------------- objective
class Objective {
 public:
  virtual ~Objective() = default;
  virtual int dim() const = 0;
  virtual Vec evaluate(const Mat& batch, WatchStats* stats = nullptr) const = 0;
  virtual bool has_gradient() const { return false; }
  virtual Mat gradient(const Mat&) const { throw std::logic_error("Objective: gradient not available"); }
};

struct GraphMeta {  // objective.hpp:31-36
  std::vector<int> step_states;
  std::vector<int> hinges;
  int final_step_last_relu = -1;
  std::vector<int> relu_nodes;
};
enum class StopRule { kLastRelu, kEveryStepOutput, kCustom };

class GraphObjective : public Objective {  // objective.hpp:40-70, objective.cpp:13-76
 public:
  GraphObjective(CompGraph graph, GraphMeta meta = {});
  int dim() const override { return graph_.input_dim(); }
  Vec evaluate(const Mat& batch, WatchStats* stats = nullptr) const override;
  bool has_gradient() const override { return true; }
  Mat gradient(const Mat& batch) const override { return oracle::gradient(graph_, batch); }
  const CompGraph& graph() const { return graph_; }
  const GraphMeta& meta() const { return meta_; }
  void set_stop_rule(StopRule rule, std::vector<int> custom = {});
  const std::vector<int>& stop_set() const { return stop_set_; }
  const std::vector<int>& watch_set() const { return watch_set_; }

 private:
  void rebuild_sets();
  CompGraph graph_;
  GraphMeta meta_;
  StopRule rule_ = StopRule::kLastRelu;
  std::vector<int> custom_stop_, stop_set_, watch_set_;
};

class SyntheticObjective : public Objective {  // objective.hpp:75-93, objective.cpp:78-109
 public:
  static constexpr double kUnitMinimum = -0.980339434486584;
  static constexpr double kUnitArgmin = 0.06258152045359563;
  explicit SyntheticObjective(int dim);
  int dim() const override { return dim_; }
  Vec evaluate(const Mat& batch, WatchStats* stats = nullptr) const override;
  bool has_gradient() const override { return true; }
  Mat gradient(const Mat& batch) const override;
  BoxDomain domain() const;

 private:
  int dim_;
};

// ----------------------------------------------------------- crown
enum class AlphaPolicy { kAdaptive, kZero, kOne };
enum class BoundMode { kFullCrown, kEarlyStopEmpirical, kEarlyStopInterval };
struct ReluRelaxation {
  Vec lower_slope, lower_offset, upper_slope, upper_offset;
};
ReluRelaxation relax_relu(const Vec& l, const Vec& u, AlphaPolicy policy);

struct PreactBounds {
  std::map<int, std::pair<Vec, Vec>> bounds;
  bool has(int node) const { return bounds.count(node) != 0; }
  const std::pair<Vec, Vec>& at(int node) const { return bounds.at(node); }
};
struct LinearTerm {
  int node;
  Mat coeff;
};
struct LinearBounds {
  std::vector<LinearTerm> terms;
  Vec offset;
};
struct BackwardBounds {
  LinearBounds lower, upper;
};
BackwardBounds backward_propagate(const CompGraph& g, int from, const std::vector<int>& stop_set,
                                  const PreactBounds& pre, AlphaPolicy alpha);
Vec concretize_lower(const LinearBounds& lb, const PreactBounds& anchors);
Vec concretize_upper(const LinearBounds& ub, const PreactBounds& anchors);
PreactBounds crown_node_bounds(const CompGraph& g, const BoxDomain& box,
                               const std::vector<int>& targets, AlphaPolicy alpha);
double lower_bound(const GraphObjective& obj, const BoxDomain& box, BoundMode mode,
                   const WatchStats* stats = nullptr, AlphaPolicy alpha = AlphaPolicy::kAdaptive);
bool bound_mode_sound(BoundMode mode);

// ----------------------------------------------------------- search
enum class SearchMethod { kCem, kMppi, kGd };
struct CemParams { int agents = 4; int elites = 10; double jitter = 1e-3; double init_sigma = 0.5; };
struct MppiParams {
  double noise_frac = 0.25, temperature = 10.0;
  std::vector<double> noise_ratios{0.5, 1.0, 2.0};
  std::vector<double> temperature_ratios{1.0};
};
struct GdParams {
  double base_step = 0.01;
  std::vector<double> step_ratios{0.05, 0.1, 0.25, 0.5, 0.75, 1.0, 1.5, 2.0, 5.0, 10.0};
};
struct SearcherConfig {  // search.hpp:37-46
  SearchMethod method = SearchMethod::kCem;
  int samples_per_iter = 1000;
  int iterations = 10;
  std::uint64_t seed = 0;
  int top_capacity = 512;
  CemParams cem;
  MppiParams mppi;
  GdParams gd;
};
struct TopSample {
  double value;
  Vec u;
};
struct SearchReport {  // search.hpp:53-63
  double uf = std::numeric_limits<double>::infinity();
  Vec best;
  std::vector<TopSample> top;
  WatchStats stats;
  std::vector<double> uf_history;
  std::vector<std::int64_t> samples_history;
  std::int64_t samples = 0;
  bool ok = true;
  std::string error;
};
SearchReport search(const Objective& f, const BoxDomain& box, const SearcherConfig& cfg,
                    const Vec* warm_start = nullptr);

// Test hooks (not in the reference): replace the sampled rows [0, n_samp) of iteration `it`
// before they are consumed, and observe the sampler state after each iteration's refit.
// Parity of the device update on identical samples (tests/test_gpu_search_update.py).
struct SearchHooks {
  std::function<void(int it, Mat& batch)> inject;
  std::function<void(int it, const Mat& batch, const std::vector<Vec>& mu, const std::vector<Vec>& var,
                     const SearchReport& so_far, const std::vector<TopSample>& top)> after;
};
void set_search_hooks(const SearchHooks* hooks);  // thread-local; null = none

// Test hook (not in the reference): plan() takes each child's search report and lower bound from
// `report` / `lf` (iteration, index of the child in the iteration's order, its box) instead of
// running batch_search and the bounder -- the plan-level decision replay against the device planner.
struct PlanReplay {
  std::function<SearchReport(int iter, int index, const BoxDomain& box)> report;
  std::function<double(int iter, int index)> lf;
};
void set_plan_replay(const PlanReplay* replay);  // thread-local; null = none
std::vector<SearchReport> batch_search(const Objective& f, const std::vector<BoxDomain>& boxes,
                                       const SearcherConfig& cfg,
                                       const std::vector<const Vec*>* warm_starts = nullptr);

// ----------------------------------------------------------- bab
struct SubdomainRecord {  // bab.hpp:18-28
  BoxDomain box;
  double lf = -std::numeric_limits<double>::infinity();
  double uf = std::numeric_limits<double>::infinity();
  Vec best;
  std::vector<TopSample> top;
  std::int64_t samples = 0;
  int depth = 0;
  std::int64_t id = 0, parent = -1;
  double log_vol = 0.0;
};
class DomainPool {
 public:
  void insert(SubdomainRecord rec) { records_.push_back(std::move(rec)); }
  bool empty() const { return records_.empty(); }
  std::size_t size() const { return records_.size(); }
  std::vector<SubdomainRecord>& records() { return records_; }
  const std::vector<SubdomainRecord>& records() const { return records_; }
  double min_lf() const;

 private:
  std::vector<SubdomainRecord> records_;
};
struct PlannerConfig {  // bab.hpp:51-62 (+ split_rule knob)
  int batch = 4;
  double eta = 0.75, temperature = 0.05, top_percent = 1.0, min_width = 1e-6;
  BoundMode bound_mode = BoundMode::kEarlyStopEmpirical;
  AlphaPolicy alpha = AlphaPolicy::kAdaptive;
  int split_rule = 0;  // 0 = reference sample-count rule, 1 = width only
  SearcherConfig search;
  int max_iterations = 50;
  double wall_clock_ms = 0.0;
  double target_objective = -std::numeric_limits<double>::infinity();
  std::uint64_t seed = 0;
};
class Bounder {
 public:
  virtual ~Bounder() = default;
  virtual double lower(const BoxDomain& box, const SearchReport* report) const = 0;
  virtual bool sound() const = 0;
};
class CrownBounder : public Bounder {
 public:
  CrownBounder(std::shared_ptr<const GraphObjective> obj, BoundMode mode, AlphaPolicy alpha)
      : obj_(std::move(obj)), mode_(mode), alpha_(alpha) {}
  double lower(const BoxDomain& box, const SearchReport* report) const override;
  bool sound() const override { return bound_mode_sound(mode_); }

 private:
  std::shared_ptr<const GraphObjective> obj_;
  BoundMode mode_;
  AlphaPolicy alpha_;
};
class SeparableBounder : public Bounder {
 public:
  double lower(const BoxDomain& box, const SearchReport* report) const override;
  bool sound() const override { return true; }
  static double term_min(double a, double b);
  static const std::vector<double>& critical_points();
};
std::vector<SubdomainRecord> pick_out(DomainPool& pool, int n, double eta, double temperature, Rng& rng);
struct SplitResult {
  SubdomainRecord lo, hi;
  int axis = -1;
};
SplitResult split(const SubdomainRecord& rec, double top_percent, double min_width,
                  std::int64_t next_id, int split_rule = 0);
double prune(DomainPool& pool, double incumbent_uf,
             const std::function<void(const SubdomainRecord&)>* on_prune = nullptr);
void merge_report(SubdomainRecord& rec, SearchReport&& rep, int top_capacity);
struct TraceRow {
  int iter = 0;
  double uf = 0, min_lf = 0, pruned_vol = 0, selected_vol = 0;
  std::int64_t pool_size = 0, samples = 0;
  double wall_ms = 0;
};
struct PlanResult {
  double uf = std::numeric_limits<double>::infinity();
  Vec best;
  double min_lf = -std::numeric_limits<double>::infinity();
  bool certified = false;
  std::vector<TraceRow> trace;
  std::int64_t samples = 0;
  int iterations = 0;
  std::string stop_reason;
};
PlanResult plan(std::shared_ptr<const Objective> objective, const BoxDomain& root,
                const PlannerConfig& cfg, std::shared_ptr<const Bounder> bounder = nullptr,
                const Vec* warm_start = nullptr);
PlanResult sample_only_plan(std::shared_ptr<const Objective> objective, const BoxDomain& root,
                            const PlannerConfig& cfg, const Vec* warm_start = nullptr);

// ----------------------------------------------------------- model
// Node ids of one unrolled step (for mapping device statistics to nodes).
struct StepNodes {
  int u = -1, x = -1, p = -1;
  std::vector<int> preact;  // Linear nodes feeding a ReLU, per hidden layer
  std::vector<int> ops;     // one node per cost-program op
};
struct BuiltObjective {
  std::shared_ptr<GraphObjective> objective;
  BoxDomain box;
  std::vector<StepNodes> steps;
};

}  // namespace oracle
