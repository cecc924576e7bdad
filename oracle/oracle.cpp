// oracle.cpp -- TEST INFRASTRUCTURE ONLY.  See oracle.hpp for the contract.
// Every function restates the reference algorithm at the cited
// /root/reference/proj file:line in plain C++ (no Eigen).
#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <set>
#include <thread>

namespace oracle {

void require_finite(const Vec& v, const std::string& what) {
  for (double x : v)
    if (!std::isfinite(x)) throw std::invalid_argument(what + ": non-finite values");
}
void require_finite(const Mat& m, const std::string& what) {
  for (double x : m.a)
    if (!std::isfinite(x)) throw std::invalid_argument(what + ": non-finite values");
}

// ------------------------------------------------------------------ rng.cpp
int Rng::uniform_int(int n) {  // rng.cpp:8-18
  if (n <= 0) throw std::invalid_argument("Rng::uniform_int: n must be positive");
  const std::uint64_t un = static_cast<std::uint64_t>(n);
  const std::uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  std::uint64_t x;
  do {
    x = gen_();
  } while (x >= limit);
  return static_cast<int>(x % un);
}

double Rng::normal() {  // rng.cpp:20-35 (Box-Muller, spare cached)
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1, u2;
  do {
    u1 = uniform();
  } while (u1 <= 0.0);
  u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  spare_ = r * std::sin(a);
  has_spare_ = true;
  return r * std::cos(a);
}

std::uint64_t mix_seed(std::uint64_t master, std::uint64_t salt) {  // rng.cpp:37-42
  std::uint64_t z = master + 0x9E3779B97F4A7C15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------- parallel.cpp
namespace {
std::atomic<int> g_threads{0};
int detect_threads() {
  if (const char* env = std::getenv("BABPLAN_THREADS")) {
    const int n = std::atoi(env);
    if (n > 0) return n;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}
}  // namespace

int thread_count() {  // parallel.cpp:24-29
  const int o = g_threads.load();
  if (o > 0) return o;
  static const int detected = detect_threads();
  return detected;
}
void set_thread_count(int n) { g_threads.store(n < 0 ? 0 : n); }

void parallel_chunks(std::int64_t n, const std::function<void(std::int64_t, std::int64_t)>& fn) {
  // parallel.cpp:33-50: ceil(n / workers) contiguous chunks, one thread each.
  if (n <= 0) return;
  const int workers = static_cast<int>(std::min<std::int64_t>(thread_count(), n));
  if (workers <= 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const std::int64_t chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const std::int64_t b = w * chunk;
    const std::int64_t e = std::min<std::int64_t>(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------- types.cpp
BoxDomain::BoxDomain(Vec lower, Vec upper) : lower_(std::move(lower)), upper_(std::move(upper)) {
  if (lower_.size() != upper_.size()) throw std::invalid_argument("BoxDomain: bound dimensions differ");
  if (lower_.empty()) throw std::invalid_argument("BoxDomain: empty bounds");
  require_finite(lower_, "BoxDomain lower");
  require_finite(upper_, "BoxDomain upper");
  for (size_t j = 0; j < lower_.size(); ++j)
    if (lower_[j] > upper_[j])
      throw std::invalid_argument("BoxDomain: lower exceeds upper at axis " + std::to_string(j));
}
Vec BoxDomain::width() const {
  Vec w(lower_.size());
  for (size_t j = 0; j < w.size(); ++j) w[j] = upper_[j] - lower_[j];
  return w;
}
double BoxDomain::max_width() const {
  double w = 0.0;
  for (int j = 0; j < dim(); ++j) w = std::max(w, width(j));
  return w;
}
Vec BoxDomain::center() const {  // 0.5 * (lower + upper)
  Vec c(lower_.size());
  for (size_t j = 0; j < c.size(); ++j) c[j] = 0.5 * (lower_[j] + upper_[j]);
  return c;
}
bool BoxDomain::contains(const Vec& u, double tol) const {
  if (u.size() != lower_.size()) return false;
  for (size_t j = 0; j < u.size(); ++j)
    if (u[j] < lower_[j] - tol || u[j] > upper_[j] + tol) return false;
  return true;
}
double BoxDomain::log_volume_relative_to(const BoxDomain& root) const {  // types.cpp:35-46
  double acc = 0.0;
  for (int j = 0; j < dim(); ++j) {
    const double rw = root.width(j);
    if (rw <= 0.0) continue;
    const double w = width(j);
    if (w <= 0.0) return -std::numeric_limits<double>::infinity();
    acc += std::log(w / rw);
  }
  return acc;
}

// ---------------------------------------------------------------- graph.cpp
int CompGraph::add_node(GraphNode node) {
  if (finalized_) throw std::logic_error("CompGraph: graph is finalized");
  nodes_.push_back(std::move(node));
  return static_cast<int>(nodes_.size()) - 1;
}
void CompGraph::check_arg(int arg, const char* ctx) const {
  if (arg < 0 || arg >= static_cast<int>(nodes_.size()))
    throw std::invalid_argument(std::string(ctx) + ": argument refers to an unknown node");
}
int CompGraph::add_input(int dim) {  // graph.cpp:38-46
  if (input_ >= 0) throw std::invalid_argument("CompGraph: a single input node is required");
  if (dim <= 0) throw std::invalid_argument("input: dimension must be positive");
  GraphNode n;
  n.kind = NodeKind::kInput;
  n.dim = dim;
  input_ = add_node(std::move(n));
  return input_;
}
int CompGraph::add_constant(Vec value) {
  if (value.empty()) throw std::invalid_argument("constant: empty value");
  require_finite(value, "constant value");
  GraphNode n;
  n.kind = NodeKind::kConstant;
  n.dim = static_cast<int>(value.size());
  n.value = std::move(value);
  return add_node(std::move(n));
}
int CompGraph::add_linear(int arg, Mat W, Vec b) {  // graph.cpp:58-72
  check_arg(arg, "linear");
  if (W.rows == 0 || W.cols != nodes_[arg].dim)
    throw std::invalid_argument("linear: weight shape does not match argument");
  if (static_cast<int>(b.size()) != W.rows) throw std::invalid_argument("linear: bias shape mismatch");
  require_finite(W, "linear weights");
  require_finite(b, "linear bias");
  GraphNode n;
  n.kind = NodeKind::kLinear;
  n.args = {arg};
  n.dim = W.rows;
  n.W = std::move(W);
  n.b = std::move(b);
  return add_node(std::move(n));
}
int CompGraph::add_relu(int arg) {
  check_arg(arg, "relu");
  GraphNode n;
  n.kind = NodeKind::kRelu;
  n.args = {arg};
  n.dim = nodes_[arg].dim;
  return add_node(std::move(n));
}
int CompGraph::add_sum(std::vector<int> args) {
  if (args.empty()) throw std::invalid_argument("sum: needs at least one argument");
  for (int a : args) check_arg(a, "sum");
  const int dim = nodes_[args[0]].dim;
  for (int a : args)
    if (nodes_[a].dim != dim) throw std::invalid_argument("sum: argument dimensions differ");
  GraphNode n;
  n.kind = NodeKind::kSum;
  n.args = std::move(args);
  n.dim = dim;
  return add_node(std::move(n));
}
int CompGraph::add_scalar_affine(int arg, double scale, double offset) {
  check_arg(arg, "scalar_affine");
  if (!std::isfinite(scale) || !std::isfinite(offset))
    throw std::invalid_argument("scalar_affine: non-finite parameter");
  GraphNode n;
  n.kind = NodeKind::kScalarAffine;
  n.args = {arg};
  n.dim = nodes_[arg].dim;
  n.scale = scale;
  n.offset = offset;
  return add_node(std::move(n));
}
int CompGraph::add_squared_distance(int arg, Vec target, Vec weight) {
  check_arg(arg, "squared_distance");
  const size_t d = static_cast<size_t>(nodes_[arg].dim);
  if (target.size() != d || weight.size() != d)
    throw std::invalid_argument("squared_distance: target/weight shape mismatch");
  require_finite(target, "squared_distance target");
  require_finite(weight, "squared_distance weight");
  for (double w : weight)
    if (w < 0.0) throw std::invalid_argument("squared_distance: weights must be nonnegative");
  GraphNode n;
  n.kind = NodeKind::kSquaredDistance;
  n.args = {arg};
  n.dim = 1;
  n.target = std::move(target);
  n.weight = std::move(weight);
  return add_node(std::move(n));
}
int CompGraph::add_penalty_hinge(int arg, Vec center, double radius, double penalty) {
  check_arg(arg, "penalty_hinge");
  if (static_cast<int>(center.size()) != nodes_[arg].dim)
    throw std::invalid_argument("penalty_hinge: center shape mismatch");
  require_finite(center, "penalty_hinge center");
  if (!std::isfinite(radius) || radius < 0.0)
    throw std::invalid_argument("penalty_hinge: radius must be finite and nonnegative");
  if (!std::isfinite(penalty) || penalty < 0.0)
    throw std::invalid_argument("penalty_hinge: penalty must be finite and nonnegative");
  GraphNode n;
  n.kind = NodeKind::kPenaltyHinge;
  n.args = {arg};
  n.dim = 1;
  n.center = std::move(center);
  n.radius = radius;
  n.penalty = penalty;
  return add_node(std::move(n));
}
int CompGraph::add_concat(std::vector<int> args) {
  if (args.empty()) throw std::invalid_argument("concat: needs at least one argument");
  int dim = 0;
  for (int a : args) {
    check_arg(a, "concat");
    dim += nodes_[a].dim;
  }
  GraphNode n;
  n.kind = NodeKind::kConcat;
  n.args = std::move(args);
  n.dim = dim;
  return add_node(std::move(n));
}
int CompGraph::add_slice(int arg, int begin, int len) {
  check_arg(arg, "slice");
  if (len <= 0 || begin < 0 || begin + len > nodes_[arg].dim)
    throw std::invalid_argument("slice: range outside argument");
  GraphNode n;
  n.kind = NodeKind::kSlice;
  n.args = {arg};
  n.dim = len;
  n.begin = begin;
  return add_node(std::move(n));
}
void CompGraph::set_output(int node) {
  check_arg(node, "output");
  if (nodes_[node].dim != 1) throw std::invalid_argument("output: node must be scalar");
  output_ = node;
}
void CompGraph::finalize() {  // graph.cpp:179-188
  if (input_ < 0) throw std::invalid_argument("CompGraph: missing input node");
  if (output_ < 0) throw std::invalid_argument("CompGraph: output not set");
  consumers_.assign(nodes_.size(), {});
  for (int id = 0; id < size(); ++id)
    for (int a : nodes_[static_cast<size_t>(id)].args) consumers_[static_cast<size_t>(a)].push_back(id);
  finalized_ = true;
}
int CompGraph::input_dim() const {
  if (input_ < 0) throw std::logic_error("CompGraph: missing input node");
  return nodes_[static_cast<size_t>(input_)].dim;
}

namespace {

// graph.cpp:200-215 -- eight interleaved accumulators, fixed tree combine.
inline double dot8(const double* a, const double* b, int n) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int k = 0;
  for (; k + 8 <= n; k += 8)
    for (int r = 0; r < 8; ++r) s[r] += a[k + r] * b[k + r];
  for (int r = 0; k < n; ++k, ++r) s[r] += a[k] * b[k];
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// graph.cpp:219-231: Y = X W^T + b.
void affine_forward(const Mat& X, const Mat& W, const Vec& b, Mat& Y) {
  const int rows = X.rows, in = X.cols, out = W.rows;
  if (W.cols != in || static_cast<int>(b.size()) != out)
    throw std::invalid_argument("affine_forward: shape mismatch");
  Y = Mat(rows, out);
  for (int i = 0; i < rows; ++i) {
    const double* xi = X.row(i);
    for (int o = 0; o < out; ++o) Y(i, o) = dot8(xi, W.row(o), in) + b[static_cast<size_t>(o)];
  }
}

// graph.cpp:233-245: C += A * B through dot8 on B^T.
void matmul_accumulate(const Mat& A, const Mat& B, Mat& C) {
  const int m = A.rows, k = A.cols, n = B.cols;
  if (B.rows != k || C.rows != m || C.cols != n)
    throw std::invalid_argument("matmul_accumulate: shape mismatch");
  Mat Bt(n, k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) Bt(j, i) = B(i, j);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) C(i, j) += dot8(A.row(i), Bt.row(j), k);
}

Mat rows_of(const Mat& m, int b, int e) {
  Mat r(e - b, m.cols);
  std::copy(m.row(b), m.row(b) + static_cast<size_t>(e - b) * m.cols, r.a.begin());
  return r;
}

// Node-value semantics shared by evaluate and gradient (graph.cpp:283-348).
void forward_node(const CompGraph& g, int id, const std::vector<Mat>& vals, const Mat& batch, Mat& v) {
  const GraphNode& node = g.node(id);
  const int rows = batch.rows;
  switch (node.kind) {
    case NodeKind::kInput:
      v = batch;
      break;
    case NodeKind::kConstant:
      v = Mat(rows, node.dim);
      for (int i = 0; i < rows; ++i) std::copy(node.value.begin(), node.value.end(), v.row(i));
      break;
    case NodeKind::kLinear:
      affine_forward(vals[static_cast<size_t>(node.args[0])], node.W, node.b, v);
      break;
    case NodeKind::kRelu: {
      const Mat& x = vals[static_cast<size_t>(node.args[0])];
      v = Mat(x.rows, x.cols);
      for (size_t i = 0; i < x.a.size(); ++i) v.a[i] = std::max(x.a[i], 0.0);  // cwiseMax(0.0)
      break;
    }
    case NodeKind::kSum: {
      v = vals[static_cast<size_t>(node.args[0])];
      for (size_t a = 1; a < node.args.size(); ++a) {
        const Mat& x = vals[static_cast<size_t>(node.args[a])];
        for (size_t i = 0; i < v.a.size(); ++i) v.a[i] += x.a[i];
      }
      break;
    }
    case NodeKind::kScalarAffine: {
      const Mat& x = vals[static_cast<size_t>(node.args[0])];
      v = Mat(x.rows, x.cols);
      for (size_t i = 0; i < x.a.size(); ++i) v.a[i] = node.scale * x.a[i] + node.offset;
      break;
    }
    case NodeKind::kSquaredDistance: {
      const Mat& x = vals[static_cast<size_t>(node.args[0])];
      v = Mat(rows, 1);
      for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int j = 0; j < x.cols; ++j) {
          const double d = x(i, j) - node.target[static_cast<size_t>(j)];
          acc += node.weight[static_cast<size_t>(j)] * d * d;
        }
        v(i, 0) = acc;
      }
      break;
    }
    case NodeKind::kPenaltyHinge: {
      const Mat& x = vals[static_cast<size_t>(node.args[0])];
      v = Mat(rows, 1);
      for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int j = 0; j < x.cols; ++j) {
          const double d = x(i, j) - node.center[static_cast<size_t>(j)];
          acc += d * d;
        }
        const double m = node.radius - std::sqrt(acc);
        v(i, 0) = m > 0.0 ? node.penalty * m : 0.0;
      }
      break;
    }
    case NodeKind::kConcat: {
      v = Mat(rows, node.dim);
      int col = 0;
      for (int a : node.args) {
        const Mat& x = vals[static_cast<size_t>(a)];
        for (int i = 0; i < rows; ++i) std::copy(x.row(i), x.row(i) + x.cols, v.row(i) + col);
        col += x.cols;
      }
      break;
    }
    case NodeKind::kSlice: {
      const Mat& x = vals[static_cast<size_t>(node.args[0])];
      v = Mat(rows, node.dim);
      for (int i = 0; i < rows; ++i)
        std::copy(x.row(i) + node.begin, x.row(i) + node.begin + node.dim, v.row(i));
      break;
    }
  }
}

// graph.cpp:252-375: forward one chunk, release buffers once consumed,
// record colwise extrema of watched nodes, merge them under a mutex.
void forward_chunk(const CompGraph& g, const Mat& batch, Vec& out, std::int64_t out_offset,
                   const std::vector<int>* watch, WatchStats* stats, std::mutex* stats_mu) {
  const int rows = batch.rows;
  const int n = g.size();
  std::vector<Mat> vals(static_cast<size_t>(n));
  std::vector<int> pending(static_cast<size_t>(n));
  for (int id = 0; id < n; ++id) {
    pending[static_cast<size_t>(id)] = static_cast<int>(g.consumers(id).size());
    if (id == g.output()) ++pending[static_cast<size_t>(id)];
  }
  std::vector<char> watched(static_cast<size_t>(n), 0);
  if (watch != nullptr)
    for (int id : *watch) watched.at(static_cast<size_t>(id)) = 1;

  WatchStats local;
  auto record = [&](int id, const Mat& v) {
    if (!watched[static_cast<size_t>(id)]) return;
    NodeStats& ns = local[id];
    Vec mn(static_cast<size_t>(v.cols)), mx(static_cast<size_t>(v.cols));
    for (int j = 0; j < v.cols; ++j) {
      double lo = v(0, j), hi = v(0, j);
      for (int i = 1; i < v.rows; ++i) {
        lo = std::min(lo, v(i, j));
        hi = std::max(hi, v(i, j));
      }
      mn[static_cast<size_t>(j)] = lo;
      mx[static_cast<size_t>(j)] = hi;
    }
    if (ns.count == 0) {
      ns.min = std::move(mn);
      ns.max = std::move(mx);
    } else {
      for (size_t j = 0; j < mn.size(); ++j) {
        ns.min[j] = std::min(ns.min[j], mn[j]);
        ns.max[j] = std::max(ns.max[j], mx[j]);
      }
    }
    ns.count += v.rows;
  };

  for (int id = 0; id < n; ++id) {
    Mat v;
    forward_node(g, id, vals, batch, v);
    record(id, v);
    vals[static_cast<size_t>(id)] = std::move(v);
    for (int a : g.node(id).args)
      if (--pending[static_cast<size_t>(a)] == 0) vals[static_cast<size_t>(a)] = Mat();
  }
  const Mat& result = vals[static_cast<size_t>(g.output())];
  for (double x : result.a)
    if (!std::isfinite(x)) throw std::runtime_error("evaluate: non-finite objective value (malformed weights?)");
  for (int i = 0; i < rows; ++i) out[static_cast<size_t>(out_offset + i)] = result(i, 0);

  if (stats != nullptr && !local.empty()) {
    std::unique_lock<std::mutex> lk;
    if (stats_mu != nullptr) lk = std::unique_lock<std::mutex>(*stats_mu);
    for (auto& [id, ns] : local) {
      NodeStats& dst = (*stats)[id];
      if (dst.count == 0) {
        dst = ns;
      } else {
        for (size_t j = 0; j < ns.min.size(); ++j) {
          dst.min[j] = std::min(dst.min[j], ns.min[j]);
          dst.max[j] = std::max(dst.max[j], ns.max[j]);
        }
        dst.count += ns.count;
      }
    }
  }
}

constexpr std::int64_t kChunkRows = 8192;  // graph.cpp:377

}  // namespace

Vec evaluate(const CompGraph& g, const Mat& batch, const std::vector<int>* watch, WatchStats* stats) {
  // graph.cpp:381-401
  if (!g.finalized()) throw std::logic_error("evaluate: graph not finalized");
  if (batch.cols != g.input_dim())
    throw std::invalid_argument("evaluate: batch width does not match the input dimension");
  require_finite(batch, "evaluate batch");
  const std::int64_t rows = batch.rows;
  Vec out(static_cast<size_t>(rows));
  if (rows == 0) return out;
  std::mutex mu;
  const std::int64_t chunks = (rows + kChunkRows - 1) / kChunkRows;
  parallel_chunks(chunks, [&](std::int64_t cb, std::int64_t ce) {
    for (std::int64_t c = cb; c < ce; ++c) {
      const std::int64_t b = c * kChunkRows;
      const std::int64_t e = std::min<std::int64_t>(rows, b + kChunkRows);
      const Mat part = (b == 0 && e == rows) ? batch : rows_of(batch, static_cast<int>(b), static_cast<int>(e));
      forward_chunk(g, part, out, b, watch, stats, &mu);
    }
  });
  return out;
}

Mat gradient(const CompGraph& g, const Mat& batch) {  // graph.cpp:403-564
  if (!g.finalized()) throw std::logic_error("gradient: graph not finalized");
  if (batch.cols != g.input_dim())
    throw std::invalid_argument("gradient: batch width does not match the input dimension");
  require_finite(batch, "gradient batch");
  const int rows = batch.rows, n = g.size();
  std::vector<Mat> vals(static_cast<size_t>(n));
  for (int id = 0; id < n; ++id) forward_node(g, id, vals, batch, vals[static_cast<size_t>(id)]);
  std::vector<Mat> adj(static_cast<size_t>(n));
  auto bump = [&](int id, int cols) {
    Mat& a = adj[static_cast<size_t>(id)];
    if (a.size() == 0) a = Mat(rows, cols);
  };
  bump(g.output(), 1);
  std::fill(adj[static_cast<size_t>(g.output())].a.begin(), adj[static_cast<size_t>(g.output())].a.end(), 1.0);
  for (int id = n - 1; id >= 0; --id) {
    const Mat a = adj[static_cast<size_t>(id)];
    if (a.size() == 0) continue;
    const GraphNode& node = g.node(id);
    switch (node.kind) {
      case NodeKind::kInput:
      case NodeKind::kConstant:
        break;
      case NodeKind::kLinear: {  // adj_arg += a * W (Eigen GEMM; order unpinned)
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (int i = 0; i < rows; ++i)
          for (int j = 0; j < node.W.cols; ++j) {
            double s = 0.0;
            for (int o = 0; o < node.W.rows; ++o) s += a(i, o) * node.W(o, j);
            dst(i, j) += s;
          }
        break;
      }
      case NodeKind::kRelu: {
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        const Mat& x = vals[static_cast<size_t>(arg)];
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (size_t i = 0; i < x.a.size(); ++i) dst.a[i] += a.a[i] * (x.a[i] > 0.0 ? 1.0 : 0.0);
        break;
      }
      case NodeKind::kSum:
        for (int arg : node.args) {
          bump(arg, g.node(arg).dim);
          Mat& dst = adj[static_cast<size_t>(arg)];
          for (size_t i = 0; i < a.a.size(); ++i) dst.a[i] += a.a[i];
        }
        break;
      case NodeKind::kScalarAffine: {
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (size_t i = 0; i < a.a.size(); ++i) dst.a[i] += node.scale * a.a[i];
        break;
      }
      case NodeKind::kSquaredDistance: {
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        const Mat& x = vals[static_cast<size_t>(arg)];
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (int i = 0; i < rows; ++i) {
          const double s = a(i, 0);
          if (s == 0.0) continue;
          for (int j = 0; j < x.cols; ++j)
            dst(i, j) += s * 2.0 * node.weight[static_cast<size_t>(j)] * (x(i, j) - node.target[static_cast<size_t>(j)]);
        }
        break;
      }
      case NodeKind::kPenaltyHinge: {
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        const Mat& x = vals[static_cast<size_t>(arg)];
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (int i = 0; i < rows; ++i) {
          const double s = a(i, 0);
          if (s == 0.0) continue;
          Vec diff(static_cast<size_t>(x.cols));
          double nrm = 0.0;
          for (int j = 0; j < x.cols; ++j) {
            diff[static_cast<size_t>(j)] = x(i, j) - node.center[static_cast<size_t>(j)];
            nrm += diff[static_cast<size_t>(j)] * diff[static_cast<size_t>(j)];
          }
          const double d = std::sqrt(nrm);
          if (d <= 0.0 || node.radius - d <= 0.0) continue;
          for (int j = 0; j < x.cols; ++j) dst(i, j) -= (s * node.penalty / d) * diff[static_cast<size_t>(j)];
        }
        break;
      }
      case NodeKind::kConcat: {
        int col = 0;
        for (int arg : node.args) {
          const int w = g.node(arg).dim;
          bump(arg, w);
          Mat& dst = adj[static_cast<size_t>(arg)];
          for (int i = 0; i < rows; ++i)
            for (int j = 0; j < w; ++j) dst(i, j) += a(i, col + j);
          col += w;
        }
        break;
      }
      case NodeKind::kSlice: {
        const int arg = node.args[0];
        bump(arg, g.node(arg).dim);
        Mat& dst = adj[static_cast<size_t>(arg)];
        for (int i = 0; i < rows; ++i)
          for (int j = 0; j < node.dim; ++j) dst(i, node.begin + j) += a(i, j);
        break;
      }
    }
  }
  Mat gi = adj[static_cast<size_t>(g.input())];
  if (gi.size() == 0) gi = Mat(rows, g.input_dim());
  return gi;
}

IntervalSet interval_forward(const CompGraph& g, const BoxDomain& box) {  // graph.cpp:566-684
  if (!g.finalized()) throw std::logic_error("interval_forward: graph not finalized");
  if (box.dim() != g.input_dim())
    throw std::invalid_argument("interval_forward: box does not match the input dimension");
  const int n = g.size();
  IntervalSet iv;
  iv.lo.resize(static_cast<size_t>(n));
  iv.hi.resize(static_cast<size_t>(n));
  for (int id = 0; id < n; ++id) {
    const GraphNode& node = g.node(id);
    Vec lo(static_cast<size_t>(node.dim)), hi(static_cast<size_t>(node.dim));
    switch (node.kind) {
      case NodeKind::kInput:
        lo = box.lower();
        hi = box.upper();
        break;
      case NodeKind::kConstant:
        lo = node.value;
        hi = node.value;
        break;
      case NodeKind::kLinear: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        for (int o = 0; o < node.dim; ++o) {
          double l = node.b[static_cast<size_t>(o)], h = node.b[static_cast<size_t>(o)];
          for (size_t j = 0; j < al.size(); ++j) {
            const double w = node.W(o, static_cast<int>(j));
            if (w >= 0.0) {
              l += w * al[j];
              h += w * ah[j];
            } else {
              l += w * ah[j];
              h += w * al[j];
            }
          }
          lo[static_cast<size_t>(o)] = l;
          hi[static_cast<size_t>(o)] = h;
        }
        break;
      }
      case NodeKind::kRelu: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        for (size_t j = 0; j < lo.size(); ++j) {
          lo[j] = std::max(al[j], 0.0);
          hi[j] = std::max(ah[j], 0.0);
        }
        break;
      }
      case NodeKind::kSum:
        std::fill(lo.begin(), lo.end(), 0.0);
        std::fill(hi.begin(), hi.end(), 0.0);
        for (int a : node.args)
          for (size_t j = 0; j < lo.size(); ++j) {
            lo[j] += iv.lo[static_cast<size_t>(a)][j];
            hi[j] += iv.hi[static_cast<size_t>(a)][j];
          }
        break;
      case NodeKind::kScalarAffine: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        for (size_t j = 0; j < lo.size(); ++j) {
          if (node.scale >= 0.0) {
            lo[j] = node.scale * al[j] + node.offset;
            hi[j] = node.scale * ah[j] + node.offset;
          } else {
            lo[j] = node.scale * ah[j] + node.offset;
            hi[j] = node.scale * al[j] + node.offset;
          }
        }
        break;
      }
      case NodeKind::kSquaredDistance: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        double l = 0.0, h = 0.0;
        for (size_t j = 0; j < al.size(); ++j) {
          const double a = al[j] - node.target[j];
          const double b = ah[j] - node.target[j];
          const double mx = std::max(a * a, b * b);
          const double mn = (a <= 0.0 && b >= 0.0) ? 0.0 : std::min(a * a, b * b);
          l += node.weight[j] * mn;
          h += node.weight[j] * mx;
        }
        lo[0] = l;
        hi[0] = h;
        break;
      }
      case NodeKind::kPenaltyHinge: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        double d2_lo = 0.0, d2_hi = 0.0;
        for (size_t j = 0; j < al.size(); ++j) {
          const double a = al[j] - node.center[j];
          const double b = ah[j] - node.center[j];
          d2_hi += std::max(a * a, b * b);
          d2_lo += (a <= 0.0 && b >= 0.0) ? 0.0 : std::min(a * a, b * b);
        }
        const double m_lo = node.radius - std::sqrt(d2_hi);
        const double m_hi = node.radius - std::sqrt(d2_lo);
        lo[0] = m_lo > 0.0 ? node.penalty * m_lo : 0.0;
        hi[0] = m_hi > 0.0 ? node.penalty * m_hi : 0.0;
        break;
      }
      case NodeKind::kConcat: {
        size_t col = 0;
        for (int a : node.args) {
          const Vec& al = iv.lo[static_cast<size_t>(a)];
          const Vec& ah = iv.hi[static_cast<size_t>(a)];
          std::copy(al.begin(), al.end(), lo.begin() + static_cast<std::ptrdiff_t>(col));
          std::copy(ah.begin(), ah.end(), hi.begin() + static_cast<std::ptrdiff_t>(col));
          col += al.size();
        }
        break;
      }
      case NodeKind::kSlice: {
        const Vec& al = iv.lo[static_cast<size_t>(node.args[0])];
        const Vec& ah = iv.hi[static_cast<size_t>(node.args[0])];
        std::copy(al.begin() + node.begin, al.begin() + node.begin + node.dim, lo.begin());
        std::copy(ah.begin() + node.begin, ah.begin() + node.begin + node.dim, hi.begin());
        break;
      }
    }
    iv.lo[static_cast<size_t>(id)] = std::move(lo);
    iv.hi[static_cast<size_t>(id)] = std::move(hi);
  }
  return iv;
}

// ------------------------------------------------------------ objective.cpp
GraphObjective::GraphObjective(CompGraph graph, GraphMeta meta)
    : graph_(std::move(graph)), meta_(std::move(meta)) {  // objective.cpp:13-27
  if (!graph_.finalized()) graph_.finalize();
  if (meta_.relu_nodes.empty())
    for (int id = 0; id < graph_.size(); ++id)
      if (graph_.node(id).kind == NodeKind::kRelu) meta_.relu_nodes.push_back(id);
  if (meta_.hinges.empty())
    for (int id = 0; id < graph_.size(); ++id)
      if (graph_.node(id).kind == NodeKind::kPenaltyHinge) meta_.hinges.push_back(id);
  if (meta_.final_step_last_relu < 0 && !meta_.relu_nodes.empty())
    meta_.final_step_last_relu = meta_.relu_nodes.back();
  rebuild_sets();
}
Vec GraphObjective::evaluate(const Mat& batch, WatchStats* stats) const {
  return oracle::evaluate(graph_, batch, stats != nullptr ? &watch_set_ : nullptr, stats);
}
void GraphObjective::set_stop_rule(StopRule rule, std::vector<int> custom) {
  rule_ = rule;
  custom_stop_ = std::move(custom);
  rebuild_sets();
}
void GraphObjective::rebuild_sets() {  // objective.cpp:45-76
  std::set<int> stop;
  switch (rule_) {
    case StopRule::kLastRelu:
      if (meta_.final_step_last_relu >= 0) stop.insert(meta_.final_step_last_relu);
      break;
    case StopRule::kEveryStepOutput:
      stop.insert(meta_.step_states.begin(), meta_.step_states.end());
      break;
    case StopRule::kCustom:
      for (int id : custom_stop_) {
        if (id < 0 || id >= graph_.size()) throw std::invalid_argument("stop set: unknown node id");
        stop.insert(id);
      }
      break;
  }
  stop.insert(meta_.hinges.begin(), meta_.hinges.end());
  stop_set_.assign(stop.begin(), stop.end());
  std::set<int> watch(stop.begin(), stop.end());
  for (int id = 0; id < graph_.size(); ++id) {
    const GraphNode& n = graph_.node(id);
    if (n.kind == NodeKind::kRelu || n.kind == NodeKind::kSquaredDistance ||
        n.kind == NodeKind::kPenaltyHinge) {
      watch.insert(n.args[0]);
      watch.insert(id);
    }
  }
  watch_set_.assign(watch.begin(), watch.end());
}

SyntheticObjective::SyntheticObjective(int dim) : dim_(dim) {
  if (dim <= 0) throw std::invalid_argument("SyntheticObjective: dimension must be positive");
}
Vec SyntheticObjective::evaluate(const Mat& batch, WatchStats*) const {  // objective.cpp:82-95
  if (batch.cols != dim_) throw std::invalid_argument("SyntheticObjective: batch width mismatch");
  require_finite(batch, "synthetic batch");
  Vec out(static_cast<size_t>(batch.rows));
  for (int i = 0; i < batch.rows; ++i) {
    const double* x = batch.row(i);
    double acc = 0.0;
    for (int j = 0; j < dim_; ++j) acc += 5.0 * x[j] * x[j] + std::cos(50.0 * x[j]);
    out[static_cast<size_t>(i)] = acc;
  }
  return out;
}
Mat SyntheticObjective::gradient(const Mat& batch) const {
  Mat g(batch.rows, dim_);
  for (int i = 0; i < batch.rows; ++i)
    for (int j = 0; j < dim_; ++j) g(i, j) = 10.0 * batch(i, j) - 50.0 * std::sin(50.0 * batch(i, j));
  return g;
}
BoxDomain SyntheticObjective::domain() const {
  return BoxDomain(Vec(static_cast<size_t>(dim_), -1.0), Vec(static_cast<size_t>(dim_), 1.0));
}

// ---------------------------------------------------------------- crown.cpp
ReluRelaxation relax_relu(const Vec& l, const Vec& u, AlphaPolicy policy) {  // crown.cpp:10-39
  if (l.size() != u.size()) throw std::invalid_argument("relax_relu: bound sizes differ");
  const size_t n = l.size();
  ReluRelaxation r;
  r.lower_slope.assign(n, 0.0);
  r.lower_offset.assign(n, 0.0);
  r.upper_slope.assign(n, 0.0);
  r.upper_offset.assign(n, 0.0);
  for (size_t j = 0; j < n; ++j) {
    if (!(l[j] <= u[j])) throw std::invalid_argument("relax_relu: lower exceeds upper at " + std::to_string(j));
    if (l[j] >= 0.0) {
      r.lower_slope[j] = 1.0;
      r.upper_slope[j] = 1.0;
    } else if (u[j] <= 0.0) {
      r.lower_slope[j] = 0.0;
      r.upper_slope[j] = 0.0;
    } else {
      const double s = u[j] / (u[j] - l[j]);
      r.upper_slope[j] = s;
      r.upper_offset[j] = -u[j] * l[j] / (u[j] - l[j]);
      switch (policy) {
        case AlphaPolicy::kAdaptive: r.lower_slope[j] = u[j] >= -l[j] ? 1.0 : 0.0; break;
        case AlphaPolicy::kZero: r.lower_slope[j] = 0.0; break;
        case AlphaPolicy::kOne: r.lower_slope[j] = 1.0; break;
      }
    }
  }
  return r;
}

namespace {

struct Accum {
  Mat lo, up;
  bool present = false;
};
void ensure(Accum& a, int rows, int dim) {
  if (!a.present) {
    a.lo = Mat(rows, dim);
    a.up = Mat(rows, dim);
    a.present = true;
  }
}
const std::pair<Vec, Vec>& need_bounds(const PreactBounds& pre, int node, const char* why) {
  if (!pre.has(node))
    throw std::logic_error(std::string("backward_propagate: missing bounds for node ") +
                           std::to_string(node) + " (" + why + ")");
  return pre.at(node);
}
struct QuadEnvelope {
  Vec lo_slope, up_slope;
  double lo_off = 0.0, up_off = 0.0;
};
QuadEnvelope quad_envelope(const GraphNode& n, const Vec& l, const Vec& u) {  // crown.cpp:72-88
  const size_t d = l.size();
  QuadEnvelope e;
  e.lo_slope.resize(d);
  e.up_slope.resize(d);
  for (size_t j = 0; j < d; ++j) {
    if (!(l[j] <= u[j])) throw std::invalid_argument("quad envelope: inverted interval");
    const double w = n.weight[j], t = n.target[j];
    const double m = 0.5 * (l[j] + u[j]);
    e.lo_slope[j] = 2.0 * w * (m - t);
    e.lo_off += -w * (m - t) * (m + t);
    const double s = w * (l[j] + u[j] - 2.0 * t);
    e.up_slope[j] = s;
    e.up_off += w * (l[j] - t) * (l[j] - t) - s * l[j];
  }
  return e;
}
// b += A * v (Eigen GEMV in the reference; summation order unpinned there).
void add_gemv(Vec& b, const Mat& A, const Vec& v) {
  for (int r = 0; r < A.rows; ++r) {
    double s = 0.0;
    for (int j = 0; j < A.cols; ++j) s += A(r, j) * v[static_cast<size_t>(j)];
    b[static_cast<size_t>(r)] += s;
  }
}

}  // namespace

BackwardBounds backward_propagate(const CompGraph& g, int from, const std::vector<int>& stop_set,
                                  const PreactBounds& pre, AlphaPolicy alpha) {  // crown.cpp:92-292
  if (!g.finalized()) throw std::logic_error("backward_propagate: graph not finalized");
  if (from < 0 || from >= g.size()) throw std::invalid_argument("backward_propagate: bad node");
  const int n = g.size();
  const int rows = g.node(from).dim;
  std::vector<char> stop(static_cast<size_t>(n), 0);
  for (int s : stop_set) {
    if (s < 0 || s >= n) throw std::invalid_argument("backward_propagate: bad stop node");
    stop[static_cast<size_t>(s)] = 1;
  }
  std::vector<char> reach(static_cast<size_t>(n), 0);
  {
    std::vector<int> dfs{from};
    reach[static_cast<size_t>(from)] = 1;
    while (!dfs.empty()) {
      const int v = dfs.back();
      dfs.pop_back();
      for (int a : g.node(v).args)
        if (!reach[static_cast<size_t>(a)]) {
          reach[static_cast<size_t>(a)] = 1;
          dfs.push_back(a);
        }
    }
  }
  std::vector<int> countdown(static_cast<size_t>(n), 0);
  for (int v = 0; v < n; ++v) {
    if (!reach[static_cast<size_t>(v)]) continue;
    for (int a : g.node(v).args) ++countdown[static_cast<size_t>(a)];
  }
  std::vector<Accum> acc(static_cast<size_t>(n));
  Vec b_lo(static_cast<size_t>(rows), 0.0), b_up(static_cast<size_t>(rows), 0.0);
  ensure(acc[static_cast<size_t>(from)], rows, rows);
  for (int r = 0; r < rows; ++r) {
    acc[static_cast<size_t>(from)].lo(r, r) = 1.0;
    acc[static_cast<size_t>(from)].up(r, r) = 1.0;
  }
  std::vector<char> propagated(static_cast<size_t>(n), 0);
  std::vector<int> queue{from};
  auto push_if_ready = [&](int w) {
    if (countdown[static_cast<size_t>(w)] == 0) {
      const NodeKind k = g.node(w).kind;
      if (k != NodeKind::kInput && k != NodeKind::kConstant) queue.push_back(w);
    }
  };
  while (!queue.empty()) {
    const int v = queue.back();
    queue.pop_back();
    const GraphNode& node = g.node(v);
    for (int a : node.args) {
      --countdown[static_cast<size_t>(a)];
      push_if_ready(a);
    }
    if (v != from && (stop[static_cast<size_t>(v)] || node.kind == NodeKind::kPenaltyHinge)) continue;
    Accum& av = acc[static_cast<size_t>(v)];
    if (!av.present) continue;
    if (node.kind == NodeKind::kInput || node.kind == NodeKind::kConstant) continue;
    switch (node.kind) {
      case NodeKind::kLinear: {
        const int arg = node.args[0];
        Accum& aw = acc[static_cast<size_t>(arg)];
        ensure(aw, rows, g.node(arg).dim);
        matmul_accumulate(av.lo, node.W, aw.lo);
        matmul_accumulate(av.up, node.W, aw.up);
        add_gemv(b_lo, av.lo, node.b);
        add_gemv(b_up, av.up, node.b);
        break;
      }
      case NodeKind::kRelu: {
        const int arg = node.args[0];
        const auto& lu = need_bounds(pre, arg, "relu preactivation");
        const ReluRelaxation rel = relax_relu(lu.first, lu.second, alpha);
        Accum& aw = acc[static_cast<size_t>(arg)];
        ensure(aw, rows, g.node(arg).dim);
        for (int r = 0; r < rows; ++r) {
          for (int j = 0; j < node.dim; ++j) {
            const size_t jj = static_cast<size_t>(j);
            const double c_lo = av.lo(r, j);
            if (c_lo >= 0.0) {
              aw.lo(r, j) += c_lo * rel.lower_slope[jj];
              b_lo[static_cast<size_t>(r)] += c_lo * rel.lower_offset[jj];
            } else {
              aw.lo(r, j) += c_lo * rel.upper_slope[jj];
              b_lo[static_cast<size_t>(r)] += c_lo * rel.upper_offset[jj];
            }
            const double c_up = av.up(r, j);
            if (c_up >= 0.0) {
              aw.up(r, j) += c_up * rel.upper_slope[jj];
              b_up[static_cast<size_t>(r)] += c_up * rel.upper_offset[jj];
            } else {
              aw.up(r, j) += c_up * rel.lower_slope[jj];
              b_up[static_cast<size_t>(r)] += c_up * rel.lower_offset[jj];
            }
          }
        }
        break;
      }
      case NodeKind::kSum:
        for (int arg : node.args) {
          Accum& aw = acc[static_cast<size_t>(arg)];
          ensure(aw, rows, g.node(arg).dim);
          for (size_t i = 0; i < av.lo.a.size(); ++i) {
            aw.lo.a[i] += av.lo.a[i];
            aw.up.a[i] += av.up.a[i];
          }
        }
        break;
      case NodeKind::kScalarAffine: {
        const int arg = node.args[0];
        Accum& aw = acc[static_cast<size_t>(arg)];
        ensure(aw, rows, g.node(arg).dim);
        for (size_t i = 0; i < av.lo.a.size(); ++i) {
          aw.lo.a[i] += node.scale * av.lo.a[i];
          aw.up.a[i] += node.scale * av.up.a[i];
        }
        for (int r = 0; r < rows; ++r) {  // offset * rowwise sum
          double sl = 0.0, su = 0.0;
          for (int j = 0; j < av.lo.cols; ++j) {
            sl += av.lo(r, j);
            su += av.up(r, j);
          }
          b_lo[static_cast<size_t>(r)] += node.offset * sl;
          b_up[static_cast<size_t>(r)] += node.offset * su;
        }
        break;
      }
      case NodeKind::kSquaredDistance: {
        const int arg = node.args[0];
        const auto& lu = need_bounds(pre, arg, "quadratic input");
        const QuadEnvelope e = quad_envelope(node, lu.first, lu.second);
        Accum& aw = acc[static_cast<size_t>(arg)];
        ensure(aw, rows, g.node(arg).dim);
        for (int r = 0; r < rows; ++r) {
          const double c_lo = av.lo(r, 0);
          const Vec& s_lo = c_lo >= 0.0 ? e.lo_slope : e.up_slope;
          for (int j = 0; j < aw.lo.cols; ++j) aw.lo(r, j) += c_lo * s_lo[static_cast<size_t>(j)];
          b_lo[static_cast<size_t>(r)] += c_lo * (c_lo >= 0.0 ? e.lo_off : e.up_off);
          const double c_up = av.up(r, 0);
          const Vec& s_up = c_up >= 0.0 ? e.up_slope : e.lo_slope;
          for (int j = 0; j < aw.up.cols; ++j) aw.up(r, j) += c_up * s_up[static_cast<size_t>(j)];
          b_up[static_cast<size_t>(r)] += c_up * (c_up >= 0.0 ? e.up_off : e.lo_off);
        }
        break;
      }
      case NodeKind::kConcat: {
        int col = 0;
        for (int arg : node.args) {
          const int w = g.node(arg).dim;
          Accum& aw = acc[static_cast<size_t>(arg)];
          ensure(aw, rows, w);
          for (int r = 0; r < rows; ++r)
            for (int j = 0; j < w; ++j) {
              aw.lo(r, j) += av.lo(r, col + j);
              aw.up(r, j) += av.up(r, col + j);
            }
          col += w;
        }
        break;
      }
      case NodeKind::kSlice: {
        const int arg = node.args[0];
        Accum& aw = acc[static_cast<size_t>(arg)];
        ensure(aw, rows, g.node(arg).dim);
        for (int r = 0; r < rows; ++r)
          for (int j = 0; j < node.dim; ++j) {
            aw.lo(r, node.begin + j) += av.lo(r, j);
            aw.up(r, node.begin + j) += av.up(r, j);
          }
        break;
      }
      default:
        throw std::logic_error("backward_propagate: unexpected node kind");
    }
    propagated[static_cast<size_t>(v)] = 1;
    av = Accum();
  }
  BackwardBounds out;
  out.lower.offset = std::move(b_lo);
  out.upper.offset = std::move(b_up);
  for (int id = 0; id < n; ++id) {
    Accum& a = acc[static_cast<size_t>(id)];
    if (!a.present || propagated[static_cast<size_t>(id)]) continue;
    const GraphNode& node = g.node(id);
    if (node.kind == NodeKind::kConstant) {
      add_gemv(out.lower.offset, a.lo, node.value);
      add_gemv(out.upper.offset, a.up, node.value);
      continue;
    }
    out.lower.terms.push_back({id, a.lo});
    out.upper.terms.push_back({id, a.up});
  }
  return out;
}

namespace {
Vec concretize(const LinearBounds& lb, const PreactBounds& anchors, bool lower) {  // crown.cpp:296-314
  Vec res = lb.offset;
  for (const auto& term : lb.terms) {
    const auto& lh = need_bounds(anchors, term.node, "anchor");
    if (static_cast<int>(lh.first.size()) != term.coeff.cols)
      throw std::invalid_argument("concretize: anchor bound width mismatch");
    for (int r = 0; r < term.coeff.rows; ++r) {
      double acc = 0.0;
      for (int j = 0; j < term.coeff.cols; ++j) {
        const double c = term.coeff(r, j);
        const bool take_lo = lower ? c >= 0.0 : c < 0.0;
        acc += c * (take_lo ? lh.first[static_cast<size_t>(j)] : lh.second[static_cast<size_t>(j)]);
      }
      res[static_cast<size_t>(r)] += acc;
    }
  }
  return res;
}
void hinge_interval(const GraphNode& n, const Vec& al, const Vec& ah, double& lo, double& hi) {  // crown.cpp:362-375
  double d2_lo = 0.0, d2_hi = 0.0;
  for (size_t j = 0; j < al.size(); ++j) {
    const double a = al[j] - n.center[j];
    const double b = ah[j] - n.center[j];
    d2_hi += std::max(a * a, b * b);
    d2_lo += (a <= 0.0 && b >= 0.0) ? 0.0 : std::min(a * a, b * b);
  }
  const double m_lo = n.radius - std::sqrt(d2_hi);
  const double m_hi = n.radius - std::sqrt(d2_lo);
  lo = m_lo > 0.0 ? n.penalty * m_lo : 0.0;
  hi = m_hi > 0.0 ? n.penalty * m_hi : 0.0;
}
std::vector<int> relaxation_interfaces(const CompGraph& g) {  // crown.cpp:424-436
  std::vector<int> out;
  for (int id = 0; id < g.size(); ++id) {
    const GraphNode& n = g.node(id);
    if (n.kind == NodeKind::kRelu || n.kind == NodeKind::kSquaredDistance) {
      out.push_back(n.args[0]);
    } else if (n.kind == NodeKind::kPenaltyHinge) {
      out.push_back(n.args[0]);
      out.push_back(id);
    }
  }
  return out;
}
}  // namespace

Vec concretize_lower(const LinearBounds& lb, const PreactBounds& a) { return concretize(lb, a, true); }
Vec concretize_upper(const LinearBounds& ub, const PreactBounds& a) { return concretize(ub, a, false); }
bool bound_mode_sound(BoundMode mode) { return mode != BoundMode::kEarlyStopEmpirical; }

PreactBounds crown_node_bounds(const CompGraph& g, const BoxDomain& box, const std::vector<int>& targets,
                               AlphaPolicy alpha) {  // crown.cpp:379-418
  PreactBounds pre;
  pre.bounds[g.input()] = {box.lower(), box.upper()};
  std::vector<int> wanted = targets;
  std::sort(wanted.begin(), wanted.end());
  wanted.erase(std::unique(wanted.begin(), wanted.end()), wanted.end());
  static const std::vector<int> no_stop;
  for (int id : wanted) {
    if (id < 0 || id >= g.size()) throw std::invalid_argument("crown_node_bounds: bad node");
    if (pre.has(id)) continue;
    const GraphNode& node = g.node(id);
    if (node.kind == NodeKind::kConstant) {
      pre.bounds[id] = {node.value, node.value};
      continue;
    }
    if (node.kind == NodeKind::kPenaltyHinge) {
      const auto& ah = need_bounds(pre, node.args[0], "hinge input");
      double lo, hi;
      hinge_interval(node, ah.first, ah.second, lo, hi);
      pre.bounds[id] = {Vec{lo}, Vec{hi}};
      continue;
    }
    const BackwardBounds bb = backward_propagate(g, id, no_stop, pre, alpha);
    Vec lo = concretize_lower(bb.lower, pre);
    Vec hi = concretize_upper(bb.upper, pre);
    for (size_t j = 0; j < lo.size(); ++j)
      if (lo[j] > hi[j]) std::swap(lo[j], hi[j]);
    pre.bounds[id] = {std::move(lo), std::move(hi)};
  }
  return pre;
}

double lower_bound(const GraphObjective& obj, const BoxDomain& box, BoundMode mode,
                   const WatchStats* stats, AlphaPolicy alpha) {  // crown.cpp:440-469
  const CompGraph& g = obj.graph();
  if (box.dim() != g.input_dim()) throw std::invalid_argument("lower_bound: box dim mismatch");
  PreactBounds pre;
  if (mode == BoundMode::kFullCrown) {
    pre = crown_node_bounds(g, box, relaxation_interfaces(g), alpha);
  } else {
    const IntervalSet iv = interval_forward(g, box);
    for (int id = 0; id < g.size(); ++id)
      pre.bounds[id] = {iv.lo[static_cast<size_t>(id)], iv.hi[static_cast<size_t>(id)]};
    if (mode == BoundMode::kEarlyStopEmpirical && stats != nullptr) {
      for (const auto& [id, ns] : *stats) {
        if (ns.count == 0) continue;
        pre.bounds[id] = {ns.min, ns.max};
      }
    }
    pre.bounds[g.input()] = {box.lower(), box.upper()};
  }
  const std::vector<int> stops = mode == BoundMode::kFullCrown ? std::vector<int>{} : obj.stop_set();
  const BackwardBounds bb = backward_propagate(g, g.output(), stops, pre, alpha);
  return concretize_lower(bb.lower, pre)[0];
}

// --------------------------------------------------------------- search.cpp
namespace {

Vec clamp_to(const BoxDomain& box, Vec u) {
  for (size_t j = 0; j < u.size(); ++j) u[j] = std::clamp(u[j], box.lower()[j], box.upper()[j]);
  return u;
}

thread_local const SearchHooks* g_hooks = nullptr;

class SampleSink {  // search.cpp:37-82
 public:
  const SearchReport& report() const { return report_; }
  std::vector<TopSample> sorted_top() const {  // test hook view: the heap in value order
    std::vector<TopSample> t = heap_;
    std::sort(t.begin(), t.end(), [](const TopSample& a, const TopSample& b) { return a.value < b.value; });
    return t;
  }
  SampleSink(const Objective& f, int capacity) : f_(f), cap_(std::max(capacity, 1)) {}
  Vec consume(const Mat& batch) {
    Vec v = f_.evaluate(batch, &report_.stats);
    report_.samples += batch.rows;
    for (int i = 0; i < static_cast<int>(v.size()); ++i) {
      const double vi = v[static_cast<size_t>(i)];
      if (vi < report_.uf) {
        report_.uf = vi;
        report_.best.assign(batch.row(i), batch.row(i) + batch.cols);
      }
      if (static_cast<int>(heap_.size()) < cap_) {
        heap_.push_back({vi, Vec(batch.row(i), batch.row(i) + batch.cols)});
        std::push_heap(heap_.begin(), heap_.end(), value_less);
      } else if (vi < heap_.front().value) {
        std::pop_heap(heap_.begin(), heap_.end(), value_less);
        heap_.back() = {vi, Vec(batch.row(i), batch.row(i) + batch.cols)};
        std::push_heap(heap_.begin(), heap_.end(), value_less);
      }
    }
    return v;
  }
  void mark_iteration() {
    report_.uf_history.push_back(report_.uf);
    report_.samples_history.push_back(report_.samples);
  }
  const Vec& current_best() const { return report_.best; }
  SearchReport finish() {
    std::sort(heap_.begin(), heap_.end(), [](const TopSample& a, const TopSample& b) { return a.value < b.value; });
    report_.top = std::move(heap_);
    return std::move(report_);
  }

 private:
  static bool value_less(const TopSample& a, const TopSample& b) { return a.value < b.value; }
  const Objective& f_;
  int cap_;
  std::vector<TopSample> heap_;
  SearchReport report_;
};

}  // namespace
void set_search_hooks(const SearchHooks* hooks) { g_hooks = hooks; }
namespace {

SearchReport run_cem(const Objective& f, const BoxDomain& box, const SearcherConfig& cfg, const Vec* warm) {
  // search.cpp:87-155
  const int d = box.dim();
  const CemParams& p = cfg.cem;
  const int agents = std::max(1, p.agents);
  const int spi = std::max(1, cfg.samples_per_iter / agents);
  Rng rng(cfg.seed);
  SampleSink sink(f, cfg.top_capacity);
  const Vec width = box.width();
  Vec var_floor(static_cast<size_t>(d)), var0(static_cast<size_t>(d));
  for (size_t j = 0; j < var0.size(); ++j) {
    const double fs = p.jitter * width[j];
    var_floor[j] = fs * fs;
    const double s0 = p.init_sigma * width[j];
    var0[j] = std::max(s0 * s0, var_floor[j]);
  }
  std::vector<Vec> mu(static_cast<size_t>(agents)), var(static_cast<size_t>(agents), var0);
  for (int a = 0; a < agents; ++a) {
    Vec m(static_cast<size_t>(d));
    for (size_t j = 0; j < m.size(); ++j) m[j] = rng.uniform(box.lower()[j], box.upper()[j]);
    mu[static_cast<size_t>(a)] = std::move(m);
  }
  Vec incumbent = warm != nullptr ? clamp_to(box, *warm) : box.center();
  mu[0] = incumbent;
  for (int it = 0; it < cfg.iterations; ++it) {
    Mat batch(agents * spi + 1, d);
    for (int a = 0; a < agents; ++a) {
      const Vec& m = mu[static_cast<size_t>(a)];
      const Vec& v = var[static_cast<size_t>(a)];
      for (int i = 0; i < spi; ++i) {
        const int row = a * spi + i;
        for (int j = 0; j < d; ++j) {
          const double x = m[static_cast<size_t>(j)] + std::sqrt(v[static_cast<size_t>(j)]) * rng.normal();
          batch(row, j) = std::clamp(x, box.lower()[static_cast<size_t>(j)], box.upper()[static_cast<size_t>(j)]);
        }
      }
    }
    std::copy(incumbent.begin(), incumbent.end(), batch.row(agents * spi));
    if (g_hooks && g_hooks->inject) g_hooks->inject(it, batch);
    const Vec vals = sink.consume(batch);
    for (int a = 0; a < agents; ++a) {
      std::vector<int> idx(static_cast<size_t>(spi));
      std::iota(idx.begin(), idx.end(), a * spi);
      if (a == 0) idx.push_back(agents * spi);
      const int n_el = std::min<int>(static_cast<int>(idx.size()), std::max(1, p.elites));
      std::partial_sort(idx.begin(), idx.begin() + n_el, idx.end(), [&](int x, int y) {
        return vals[static_cast<size_t>(x)] != vals[static_cast<size_t>(y)]
                   ? vals[static_cast<size_t>(x)] < vals[static_cast<size_t>(y)]
                   : x < y;
      });
      Vec m(static_cast<size_t>(d), 0.0), v(static_cast<size_t>(d), 0.0);
      for (int e = 0; e < n_el; ++e)
        for (int j = 0; j < d; ++j) m[static_cast<size_t>(j)] += batch(idx[static_cast<size_t>(e)], j);
      for (double& x : m) x /= n_el;
      for (int e = 0; e < n_el; ++e)
        for (int j = 0; j < d; ++j) {
          const double diff = batch(idx[static_cast<size_t>(e)], j) - m[static_cast<size_t>(j)];
          v[static_cast<size_t>(j)] += diff * diff;
        }
      for (double& x : v) x /= n_el;
      for (size_t j = 0; j < v.size(); ++j) v[j] = std::max(v[j], var_floor[j]);
      mu[static_cast<size_t>(a)] = std::move(m);
      var[static_cast<size_t>(a)] = std::move(v);
    }
    incumbent = sink.current_best();
    sink.mark_iteration();
    if (g_hooks && g_hooks->after) g_hooks->after(it, batch, mu, var, sink.report(), sink.sorted_top());
  }
  return sink.finish();
}

SearchReport run_mppi(const Objective& f, const BoxDomain& box, const SearcherConfig& cfg, const Vec* warm) {
  // search.cpp:159-209
  const int d = box.dim();
  const MppiParams& p = cfg.mppi;
  const std::vector<double> noise = p.noise_ratios.empty() ? std::vector<double>{1.0} : p.noise_ratios;
  const std::vector<double> temps = p.temperature_ratios.empty() ? std::vector<double>{1.0} : p.temperature_ratios;
  const int instances = static_cast<int>(noise.size() * temps.size());
  const int m = std::max(1, cfg.samples_per_iter / instances);
  Rng rng(cfg.seed);
  SampleSink sink(f, cfg.top_capacity);
  const Vec width = box.width();
  const Vec init = warm != nullptr ? clamp_to(box, *warm) : box.center();
  std::vector<Vec> mu(static_cast<size_t>(instances), init);
  for (int it = 0; it < cfg.iterations; ++it) {
    Mat batch(instances * m + 1, d);
    for (int inst = 0; inst < instances; ++inst) {
      const double nr = noise[static_cast<size_t>(inst) % noise.size()];
      const Vec& mean = mu[static_cast<size_t>(inst)];
      for (int i = 0; i < m; ++i) {
        const int row = inst * m + i;
        for (int j = 0; j < d; ++j) {
          const double x = mean[static_cast<size_t>(j)] + p.noise_frac * nr * width[static_cast<size_t>(j)] * rng.normal();
          batch(row, j) = std::clamp(x, box.lower()[static_cast<size_t>(j)], box.upper()[static_cast<size_t>(j)]);
        }
      }
    }
    const Vec& inc = it == 0 ? init : sink.current_best();
    std::copy(inc.begin(), inc.end(), batch.row(instances * m));
    if (g_hooks && g_hooks->inject) g_hooks->inject(it, batch);
    const Vec vals = sink.consume(batch);
    for (int inst = 0; inst < instances; ++inst) {
      const double tr = temps[static_cast<size_t>(inst) / noise.size()];
      const double T = std::max(1e-12, p.temperature * tr);
      double vmin = vals[static_cast<size_t>(inst * m)];
      for (int i = 1; i < m; ++i) vmin = std::min(vmin, vals[static_cast<size_t>(inst * m + i)]);
      Vec acc(static_cast<size_t>(d), 0.0);
      double wsum = 0.0;
      for (int i = 0; i < m; ++i) {
        const double w = std::exp(-(vals[static_cast<size_t>(inst * m + i)] - vmin) / T);
        for (int j = 0; j < d; ++j) acc[static_cast<size_t>(j)] += w * batch(inst * m + i, j);
        wsum += w;
      }
      for (double& x : acc) x /= wsum;
      mu[static_cast<size_t>(inst)] = clamp_to(box, acc);
    }
    sink.mark_iteration();
    if (g_hooks && g_hooks->after) g_hooks->after(it, batch, mu, {}, sink.report(), sink.sorted_top());
  }
  return sink.finish();
}

SearchReport run_gd(const Objective& f, const BoxDomain& box, const SearcherConfig& cfg, const Vec* warm) {
  // search.cpp:214-245
  if (!f.has_gradient()) throw std::invalid_argument("gd search requires an objective with gradients");
  const int d = box.dim();
  const GdParams& p = cfg.gd;
  const std::vector<double> ratios = p.step_ratios.empty() ? std::vector<double>{1.0} : p.step_ratios;
  const int starts = std::max(1, cfg.samples_per_iter);
  Rng rng(cfg.seed);
  SampleSink sink(f, cfg.top_capacity);
  const Vec width = box.width();
  Mat pts(starts, d);
  for (int i = 0; i < starts; ++i)
    for (int j = 0; j < d; ++j) pts(i, j) = rng.uniform(box.lower()[static_cast<size_t>(j)], box.upper()[static_cast<size_t>(j)]);
  const Vec w0 = warm != nullptr ? clamp_to(box, *warm) : box.center();
  std::copy(w0.begin(), w0.end(), pts.row(0));
  for (int it = 0; it < cfg.iterations; ++it) {
    sink.consume(pts);
    const Mat grad = f.gradient(pts);
    for (int i = 0; i < starts; ++i) {
      const double step = p.base_step * ratios[static_cast<size_t>(i) % ratios.size()];
      for (int j = 0; j < d; ++j) {
        const double x = pts(i, j) - step * width[static_cast<size_t>(j)] * grad(i, j);
        pts(i, j) = std::clamp(x, box.lower()[static_cast<size_t>(j)], box.upper()[static_cast<size_t>(j)]);
      }
    }
    sink.mark_iteration();
  }
  return sink.finish();
}

}  // namespace

SearchReport search(const Objective& f, const BoxDomain& box, const SearcherConfig& cfg, const Vec* warm) {
  // search.cpp:249-260
  if (box.dim() != f.dim()) throw std::invalid_argument("search: box dimension mismatch");
  if (cfg.iterations <= 0 || cfg.samples_per_iter <= 0)
    throw std::invalid_argument("search: iterations and samples per iteration must be positive");
  switch (cfg.method) {
    case SearchMethod::kCem: return run_cem(f, box, cfg, warm);
    case SearchMethod::kMppi: return run_mppi(f, box, cfg, warm);
    case SearchMethod::kGd: return run_gd(f, box, cfg, warm);
  }
  throw std::logic_error("search: unknown method");
}

std::vector<SearchReport> batch_search(const Objective& f, const std::vector<BoxDomain>& boxes,
                                       const SearcherConfig& cfg, const std::vector<const Vec*>* warms) {
  // search.cpp:262-282
  if (warms != nullptr && warms->size() != boxes.size())
    throw std::invalid_argument("batch_search: warm start list size mismatch");
  std::vector<SearchReport> out(boxes.size());
  parallel_chunks(static_cast<std::int64_t>(boxes.size()), [&](std::int64_t b, std::int64_t e) {
    for (std::int64_t i = b; i < e; ++i) {
      SearcherConfig local = cfg;
      local.seed = derive_seed(cfg.seed, static_cast<std::uint64_t>(i));
      const Vec* warm = warms != nullptr ? (*warms)[static_cast<size_t>(i)] : nullptr;
      try {
        out[static_cast<size_t>(i)] = search(f, boxes[static_cast<size_t>(i)], local, warm);
      } catch (const std::exception& ex) {
        out[static_cast<size_t>(i)].ok = false;
        out[static_cast<size_t>(i)].error = ex.what();
      }
    }
  });
  return out;
}

// ------------------------------------------------------------------ bab.cpp
double DomainPool::min_lf() const {
  double m = std::numeric_limits<double>::infinity();
  for (const auto& r : records_) m = std::min(m, r.lf);
  return m;
}

double CrownBounder::lower(const BoxDomain& box, const SearchReport* report) const {  // bab.cpp:25-28
  const WatchStats* stats = report != nullptr && report->ok ? &report->stats : nullptr;
  return lower_bound(*obj_, box, mode_, stats, alpha_);
}

const std::vector<double>& SeparableBounder::critical_points() {  // bab.cpp:32-68
  static const std::vector<double> pts = [] {
    auto dg = [](double x) { return 10.0 * x - 50.0 * std::sin(50.0 * x); };
    std::vector<double> out;
    const int n = 400000;
    double px = -1.0, pv = dg(px);
    for (int i = 1; i <= n; ++i) {
      const double x = -1.0 + 2.0 * i / n;
      const double v = dg(x);
      if (pv == 0.0) {
        out.push_back(px);
      } else if ((pv < 0.0) != (v < 0.0)) {
        double a = px, b = x, fa = pv;
        for (int it = 0; it < 80; ++it) {
          const double m = 0.5 * (a + b);
          const double fm = dg(m);
          if (fm == 0.0) {
            a = b = m;
            break;
          }
          if ((fa < 0.0) != (fm < 0.0)) {
            b = m;
          } else {
            a = m;
            fa = fm;
          }
        }
        out.push_back(0.5 * (a + b));
      }
      px = x;
      pv = v;
    }
    if (pv == 0.0) out.push_back(px);
    return out;
  }();
  return pts;
}
double SeparableBounder::term_min(double a, double b) {  // bab.cpp:70-77
  if (!(a <= b)) throw std::invalid_argument("term_min: empty interval");
  auto g = [](double x) { return 5.0 * x * x + std::cos(50.0 * x); };
  double m = std::min(g(a), g(b));
  for (double c : critical_points())
    if (c > a && c < b) m = std::min(m, g(c));
  return m;
}
double SeparableBounder::lower(const BoxDomain& box, const SearchReport*) const {
  double total = 0.0;
  for (int j = 0; j < box.dim(); ++j) total += term_min(box.lower()[static_cast<size_t>(j)], box.upper()[static_cast<size_t>(j)]);
  return total;
}

std::vector<SubdomainRecord> pick_out(DomainPool& pool, int n, double eta, double temperature, Rng& rng) {
  // bab.cpp:85-153
  auto& recs = pool.records();
  const int total = static_cast<int>(recs.size());
  n = std::min(n, total);
  if (n <= 0) return {};
  std::vector<int> order(static_cast<size_t>(total));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return recs[static_cast<size_t>(a)].uf != recs[static_cast<size_t>(b)].uf
               ? recs[static_cast<size_t>(a)].uf < recs[static_cast<size_t>(b)].uf
               : a < b;
  });
  const int n1 = std::clamp(static_cast<int>(std::llround(eta * n)), 0, n);
  std::vector<int> chosen(order.begin(), order.begin() + n1);
  std::vector<int> rem(order.begin() + n1, order.end());
  const double temp = std::max(temperature, 1e-12);
  for (int need = n - n1; need > 0; --need) {
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (int idx : rem) {
      const double lf = recs[static_cast<size_t>(idx)].lf;
      if (std::isfinite(lf)) {
        lo = std::min(lo, lf);
        hi = std::max(hi, lf);
      }
    }
    const bool degenerate = !(hi > lo);
    std::vector<double> w(rem.size());
    double sum = 0.0;
    for (size_t i = 0; i < rem.size(); ++i) {
      double scaled = 0.5;
      if (!degenerate) {
        const double lf = recs[static_cast<size_t>(rem[i])].lf;
        scaled = std::isfinite(lf) ? (lf - lo) / (hi - lo) : (lf < 0.0 ? 0.0 : 1.0);
      }
      w[i] = degenerate ? 1.0 : std::exp(-scaled / temp);
      sum += w[i];
    }
    const double u = rng.uniform() * sum;
    double acc = 0.0;
    size_t sel = rem.size() - 1;
    for (size_t i = 0; i < rem.size(); ++i) {
      acc += w[i];
      if (u < acc) {
        sel = i;
        break;
      }
    }
    chosen.push_back(rem[sel]);
    rem.erase(rem.begin() + static_cast<std::ptrdiff_t>(sel));
  }
  std::vector<char> taken(static_cast<size_t>(total), 0);
  std::vector<SubdomainRecord> out;
  out.reserve(chosen.size());
  for (int idx : chosen) {
    taken[static_cast<size_t>(idx)] = 1;
    out.push_back(std::move(recs[static_cast<size_t>(idx)]));
  }
  std::vector<SubdomainRecord> keep;
  for (int i = 0; i < total; ++i)
    if (!taken[static_cast<size_t>(i)]) keep.push_back(std::move(recs[static_cast<size_t>(i)]));
  recs = std::move(keep);
  return out;
}

SplitResult split(const SubdomainRecord& rec, double top_percent, double min_width, std::int64_t next_id,
                  int split_rule) {  // bab.cpp:155-223
  const BoxDomain& box = rec.box;
  const int d = box.dim();
  const Vec width = box.width();
  int k = 0;
  if (!rec.top.empty() && split_rule == 0) {
    const std::int64_t stored = static_cast<std::int64_t>(rec.top.size());
    if (rec.samples > 0) {
      k = static_cast<int>(std::clamp<std::int64_t>(
          std::llround(top_percent / 100.0 * static_cast<double>(rec.samples)), 1, stored));
    } else {
      k = static_cast<int>(stored);
    }
  }
  auto best_axis = [&](bool use_samples) {
    int axis = -1;
    double best = -1.0;
    for (int j = 0; j < d; ++j) {
      if (width[static_cast<size_t>(j)] <= min_width) continue;
      double score = width[static_cast<size_t>(j)];
      if (use_samples) {
        const double mid = 0.5 * (box.lower()[static_cast<size_t>(j)] + box.upper()[static_cast<size_t>(j)]);
        int n_lo = 0;
        for (int i = 0; i < k; ++i)
          if (rec.top[static_cast<size_t>(i)].u[static_cast<size_t>(j)] <= mid) ++n_lo;
        score = width[static_cast<size_t>(j)] * std::abs(2 * n_lo - k);
      }
      if (score > best) {
        best = score;
        axis = j;
      }
    }
    return std::pair<int, double>{axis, best};
  };
  auto [axis, score] = k > 0 ? best_axis(true) : best_axis(false);
  if (k > 0 && axis >= 0 && score == 0.0) axis = best_axis(false).first;
  if (axis < 0) throw std::invalid_argument("split: no axis above the width floor");
  const double mid = 0.5 * (box.lower()[static_cast<size_t>(axis)] + box.upper()[static_cast<size_t>(axis)]);
  Vec lo_hi = box.upper(), hi_lo = box.lower();
  lo_hi[static_cast<size_t>(axis)] = mid;
  hi_lo[static_cast<size_t>(axis)] = mid;
  SplitResult res;
  res.axis = axis;
  res.lo.box = BoxDomain(box.lower(), lo_hi);
  res.hi.box = BoxDomain(hi_lo, box.upper());
  for (SubdomainRecord* child : {&res.lo, &res.hi}) {
    child->depth = rec.depth + 1;
    child->parent = rec.id;
    child->log_vol = rec.log_vol + std::log(0.5);
  }
  res.lo.id = next_id;
  res.hi.id = next_id + 1;
  for (const TopSample& s : rec.top) (s.u[static_cast<size_t>(axis)] <= mid ? res.lo : res.hi).top.push_back(s);
  for (SubdomainRecord* child : {&res.lo, &res.hi})
    if (!child->top.empty()) {
      child->uf = child->top.front().value;
      child->best = child->top.front().u;
    }
  return res;
}

double prune(DomainPool& pool, double incumbent_uf, const std::function<void(const SubdomainRecord&)>* on_prune) {
  // bab.cpp:225-241
  auto& recs = pool.records();
  double removed = 0.0;
  std::vector<SubdomainRecord> keep;
  for (auto& r : recs) {
    if (r.lf > incumbent_uf) {
      removed += std::exp(r.log_vol);
      if (on_prune != nullptr && *on_prune) (*on_prune)(r);
    } else {
      keep.push_back(std::move(r));
    }
  }
  recs = std::move(keep);
  return removed;
}

void merge_report(SubdomainRecord& rec, SearchReport&& rep, int top_capacity) {  // bab.cpp:245-262
  rec.samples += rep.samples;
  if (rep.uf < rec.uf) {
    rec.uf = rep.uf;
    rec.best = rep.best;
  }
  if (rec.top.empty()) {
    rec.top = std::move(rep.top);
  } else if (!rep.top.empty()) {
    std::vector<TopSample> merged;
    merged.reserve(rec.top.size() + rep.top.size());
    std::merge(rec.top.begin(), rec.top.end(), rep.top.begin(), rep.top.end(), std::back_inserter(merged),
               [](const TopSample& a, const TopSample& b) { return a.value < b.value; });
    if (static_cast<int>(merged.size()) > top_capacity) merged.resize(static_cast<size_t>(top_capacity));
    rec.top = std::move(merged);
  }
}

namespace {
thread_local const PlanReplay* g_replay = nullptr;
}  // namespace
void set_plan_replay(const PlanReplay* replay) { g_replay = replay; }

PlanResult plan(std::shared_ptr<const Objective> objective, const BoxDomain& root, const PlannerConfig& cfg,
                std::shared_ptr<const Bounder> bounder, const Vec* warm_start) {  // bab.cpp:266-415
  if (!objective) throw std::invalid_argument("plan: null objective");
  if (root.dim() != objective->dim()) throw std::invalid_argument("plan: box dimension mismatch");
  if (cfg.batch <= 0) throw std::invalid_argument("plan: batch must be positive");
  if (!bounder) {
    if (auto go = std::dynamic_pointer_cast<const GraphObjective>(objective)) {
      bounder = std::make_shared<CrownBounder>(go, cfg.bound_mode, cfg.alpha);
    } else if (std::dynamic_pointer_cast<const SyntheticObjective>(objective)) {
      bounder = std::make_shared<SeparableBounder>();
    } else {
      throw std::invalid_argument("plan: objective needs an explicit bounder");
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  PlanResult result;
  DomainPool pool;
  Rng pick_rng(mix_seed(cfg.seed, 1));
  std::int64_t next_id = 1;
  double pruned_cum = 0.0;
  double retired_min_lf = std::numeric_limits<double>::infinity();
  auto current_min_lf = [&] {
    const double m = std::min(pool.min_lf(), retired_min_lf);
    return std::isfinite(m) || pool.size() > 0 ? m : result.uf;
  };
  auto push_trace = [&](int iter, double selected_vol) {
    TraceRow row;
    row.iter = iter;
    row.uf = result.uf;
    row.min_lf = current_min_lf();
    row.pruned_vol = pruned_cum;
    row.selected_vol = selected_vol;
    row.pool_size = static_cast<std::int64_t>(pool.size());
    row.samples = result.samples;
    row.wall_ms = elapsed_ms();
    result.trace.push_back(row);
  };
  {
    SearcherConfig scfg = cfg.search;
    scfg.seed = mix_seed(cfg.seed, 0);
    const std::vector<const Vec*> warms{warm_start};
    std::vector<SearchReport> reports =
        g_replay ? std::vector<SearchReport>{g_replay->report(0, 0, root)} : batch_search(*objective, {root}, scfg, &warms);
    SearchReport& rep = reports[0];
    if (!rep.ok) throw std::runtime_error("plan: root search failed: " + rep.error);
    SubdomainRecord rec;
    rec.box = root;
    rec.id = 0;
    rec.log_vol = 0.0;
    rec.lf = g_replay ? g_replay->lf(0, 0) : bounder->lower(root, &rep);
    merge_report(rec, std::move(reports[0]), cfg.search.top_capacity);
    result.uf = rec.uf;
    result.best = rec.best;
    result.samples = rec.samples;
    pool.insert(std::move(rec));
    pruned_cum += prune(pool, result.uf);
    push_trace(0, 1.0);
  }
  std::string stop;
  int iter = 0;
  while (true) {
    if (result.uf <= cfg.target_objective) { stop = "target"; break; }
    if (pool.empty()) { stop = "pool-exhausted"; break; }
    if (iter >= cfg.max_iterations) { stop = "max-iterations"; break; }
    if (cfg.wall_clock_ms > 0.0 && elapsed_ms() >= cfg.wall_clock_ms) { stop = "wall-clock"; break; }
    ++iter;
    std::vector<SubdomainRecord> picked = pick_out(pool, cfg.batch, cfg.eta, cfg.temperature, pick_rng);
    double selected_vol = 0.0;
    for (const auto& r : picked) selected_vol += std::exp(r.log_vol);
    std::vector<SubdomainRecord> children;
    for (SubdomainRecord& rec : picked) {
      if (rec.box.max_width() <= cfg.min_width) {
        retired_min_lf = std::min(retired_min_lf, rec.lf);
        continue;
      }
      SplitResult sr = split(rec, cfg.top_percent, cfg.min_width, next_id, cfg.split_rule);
      next_id += 2;
      children.push_back(std::move(sr.lo));
      children.push_back(std::move(sr.hi));
    }
    if (!children.empty()) {
      std::vector<BoxDomain> boxes;
      std::vector<const Vec*> warms;
      for (const auto& c : children) {
        boxes.push_back(c.box);
        warms.push_back(!c.best.empty() ? &c.best : nullptr);
      }
      SearcherConfig scfg = cfg.search;
      scfg.seed = mix_seed(cfg.seed, static_cast<std::uint64_t>(iter) + 1);
      std::vector<SearchReport> reports;
      std::vector<double> lfs(children.size());
      if (g_replay) {
        for (size_t i = 0; i < children.size(); ++i) {
          reports.push_back(g_replay->report(iter, static_cast<int>(i), children[i].box));
          lfs[i] = g_replay->lf(iter, static_cast<int>(i));
        }
      } else {
        reports = batch_search(*objective, boxes, scfg, &warms);
        // The reference bounds children serially (bab.cpp:392-403); the
        // bounds are independent, so the oracle fans them out like batch_search.
        parallel_chunks(static_cast<std::int64_t>(children.size()), [&](std::int64_t b, std::int64_t e) {
          for (std::int64_t i = b; i < e; ++i)
            lfs[static_cast<size_t>(i)] = bounder->lower(children[static_cast<size_t>(i)].box, &reports[static_cast<size_t>(i)]);
        });
      }
      for (size_t i = 0; i < children.size(); ++i) {
        SubdomainRecord& c = children[i];
        result.samples += reports[i].samples;
        c.lf = lfs[i];
        merge_report(c, std::move(reports[i]), cfg.search.top_capacity);
        if (c.uf < result.uf) {
          result.uf = c.uf;
          result.best = c.best;
        }
        pool.insert(std::move(c));
      }
    }
    pruned_cum += prune(pool, result.uf);
    push_trace(iter, selected_vol);
  }
  result.min_lf = current_min_lf();
  result.certified = bounder->sound();
  result.iterations = iter;
  result.stop_reason = stop;
  return result;
}

PlanResult sample_only_plan(std::shared_ptr<const Objective> objective, const BoxDomain& root,
                            const PlannerConfig& cfg, const Vec* warm_start) {  // bab.cpp:417-454
  if (!objective) throw std::invalid_argument("sample_only_plan: null objective");
  if (root.dim() != objective->dim()) throw std::invalid_argument("sample_only_plan: box dimension mismatch");
  const auto t0 = std::chrono::steady_clock::now();
  SearcherConfig scfg = cfg.search;
  scfg.seed = mix_seed(cfg.seed, 0);
  const std::vector<const Vec*> warms{warm_start};
  std::vector<SearchReport> reports = batch_search(*objective, {root}, scfg, &warms);
  SearchReport& rep = reports[0];
  if (!rep.ok) throw std::runtime_error("sample_only_plan: search failed: " + rep.error);
  const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  PlanResult result;
  result.uf = rep.uf;
  result.best = rep.best;
  result.min_lf = -std::numeric_limits<double>::infinity();
  result.certified = false;
  result.samples = rep.samples;
  result.iterations = static_cast<int>(rep.uf_history.size());
  result.stop_reason = "sampler-budget";
  for (size_t i = 0; i < rep.uf_history.size(); ++i) {
    TraceRow row;
    row.iter = static_cast<int>(i);
    row.uf = rep.uf_history[i];
    row.min_lf = -std::numeric_limits<double>::infinity();
    row.selected_vol = i == 0 ? 1.0 : 0.0;
    row.pool_size = 1;
    row.samples = rep.samples_history[i];
    row.wall_ms = i + 1 == rep.uf_history.size() ? wall : 0.0;
    result.trace.push_back(row);
  }
  return result;
}

}  // namespace oracle
