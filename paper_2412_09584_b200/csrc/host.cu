// host.cu -- the C-ABI of include/babplan_cuda.h: context, objective
// compilation, device batch search / bound, and the host planner loop.
//
// The planner is the reference's plan() (proj/src/bab.cpp:266-415) with its
// search, bound, split and merge_report on the device (the pool's boxes,
// incumbents and top lists live in a device slab, pool.cu); pick_out, the
// retirement test and prune stay host C++ restated bit-for-bit over the pool's
// heads (O(pool) bookkeeping; pick_out's softmax needs the reference's exp();
// every rank of a multi-GPU run replays them on the same exchanged heads, so
// decisions are identical on every rank).
#include <cuda.h>  // CUtensorMap types (the encoder is fetched through cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: libnccl is dlopen'ed at bp_set_nccl
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <unordered_map>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>
#include <thread>
#include <mutex>
#include <exception>

#include "../../include/babplan_cuda.h"
#include "bp_common.cuh"

namespace bp {
struct RolloutArgs {
  const float* actions;
  float* costs;
  float* states;
  int* stat_min;
  int* stat_max;
  int* failed;
  long long n_rows;
  int rows_per_sub;
  int kslab;
  long long* timeline;
};
// BoundArgs: bp_common.cuh
// SearchArgs: bp_common.cuh
cudaError_t launch_rollout(const DevObjective& o, const RolloutArgs& a, int nq, bool stream, size_t smem, cudaStream_t st);
cudaError_t launch_rollout_tc(const DevObjective& o, const RolloutArgs& a, cudaStream_t st);
size_t rollout_tc_smem(const DevObjective& o);
cudaError_t launch_rollout_tc2(const DevObjective& o, const RolloutArgs& a, cudaStream_t st);
cudaError_t launch_synthetic_eval(const float* actions, float* costs, int* failed, long long n_rows, int d,
                                  int rows_per_sub, cudaStream_t st);
cudaError_t launch_separable_bound(const double* lo, const double* hi, int n, int d, const double* crit, int ncrit,
                                   const int* use, double* lf, cudaStream_t st);
size_t rollout_tc2_fixed_smem(const DevObjective& o);
cudaError_t launch_rollout_tc3(const DevObjective& o, const RolloutArgs& a, cudaStream_t st);
size_t rollout_tc3_fixed_smem(const DevObjective& o);
size_t rollout_tc3_smem(const DevObjective& o);
size_t rollout_tc2_smem(const DevObjective& o);
int rollout_rows_per_tile(int nq);
cudaError_t launch_bound(const DevObjective& o, const BoundArgs& a, int n, cudaStream_t st);
cudaError_t launch_hinge_bounds(const DevObjective& o, const BoundArgs& a, int t, int op_index, cudaStream_t st);
size_t bound_smem_bytes();
cudaError_t launch_search_init(const SearchArgs& a, cudaStream_t st);
cudaError_t launch_sample(const SearchArgs& a, int sms, cudaStream_t st);
cudaError_t launch_search_update(const SearchArgs& a, cudaStream_t st);
cudaError_t launch_gd_step(const SearchArgs& a, int sms, cudaStream_t st);
cudaError_t launch_gradient(const DevObjective& o, const float* actions, float* grad, double* ckpt, long long n_rows,
                            cudaStream_t st);
cudaError_t launch_synthetic_gradient(const float* actions, float* grad, long long n, cudaStream_t st);
size_t search_update_smem(const SearchArgs& a);
size_t search_sort_key_bytes(const SearchArgs& a);
cudaError_t launch_pool_split(const PoolArgs& P, const SplitTask* tasks, int n_tasks, const StageArgs& S,
                              unsigned char* pack, double min_width, int* axis_out, cudaStream_t st);
cudaError_t launch_pool_unpack(const PoolArgs& P, const StageArgs& S, const unsigned char* recv, const int* dst,
                               const int* slot, int n, cudaStream_t st);
cudaError_t launch_pool_merge(const PoolArgs& P, const StageArgs& S, const int* slots, int n, const float* s_val,
                              const float* s_act, const int* s_cnt, const float* s_uf, const float* s_best,
                              const int* failed, int capacity, float* out_uf, double* out_maxw, cudaStream_t st);
}  // namespace bp

namespace {

thread_local std::string g_last_error;

struct Failure : std::runtime_error {
  bp_status code;
  Failure(bp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(bp_status c, const std::string& m) { throw Failure(c, m); }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(BP_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
bp_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return BP_OK;
  } catch (const Failure& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return BP_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return BP_LOGIC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BP_RUNTIME;
  }
}

// Host<->device bytes moved by the library (e2e accounting, bp_io_bytes).
std::atomic<int64_t> g_h2d{0}, g_d2h{0};
cudaError_t memcpy_counted(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st) {
  if (kind == cudaMemcpyHostToDevice) g_h2d += static_cast<int64_t>(n);
  if (kind == cudaMemcpyDeviceToHost) g_d2h += static_cast<int64_t>(n);
  return cudaMemcpyAsync(dst, src, n, kind, st);
}

int r4(int x) { return (x + 3) & ~3; }
int r16(int x) { return (x + 15) & ~15; }
float rna_tf32_host(float x) {  // cvt.rna.tf32.f32: round the 13 dropped mantissa bits, ties away
  uint32_t b;
  std::memcpy(&b, &x, 4);
  b = (b + 0x1000u) & ~0x1FFFu;
  float r;
  std::memcpy(&r, &b, 4);
  return r;
}

// tcgen05 weight image of one layer (W row-major [N][K]): per 32-wide K-block, [hi: npad rows x 32]
// then [lo: npad rows x 32], 128-byte rows with the SW128 K-major swizzle (16-byte chunk q of row n at
// q ^ (n & 7)); hi = rna_tf32(w), lo = rna_tf32(w - hi), rows >= N and columns >= K zero.  One block
// of npad rows is the B operand of a single N = npad MMA (npad <= 256).
std::vector<double> tc_image(const double* W, int N, int K, int npad) {
  const int kb = (K + 31) / 32;
  std::vector<double> img(static_cast<size_t>(kb) * 2 * npad * 32, 0.0);
  for (int b = 0; b < kb; ++b) {
    const size_t blk = static_cast<size_t>(b) * 2 * npad * 32;
    for (int n = 0; n < npad; ++n)
      for (int cc = 0; cc < 32; ++cc) {
        const int k = b * 32 + cc;
        const float w = (n < N && k < K) ? static_cast<float>(W[static_cast<size_t>(n) * K + k]) : 0.f;
        const float hi = rna_tf32_host(w), lo = rna_tf32_host(w - hi);
        const size_t pos = static_cast<size_t>(n) * 32 + (((cc >> 2) ^ (n & 7)) << 2) + (cc & 3);
        img[blk + pos] = hi;
        img[blk + static_cast<size_t>(npad) * 32 + pos] = lo;
      }
  }
  return img;
}
int r8(int x) { return (x + 7) & ~7; }

// Grow-only device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  T* get(size_t want) {
    if (want > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      ck(cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T)), "cudaMalloc");
      n = want;
    }
    return p;
  }
};

// Pinned host staging (device->host report copies run at full DMA rate).
template <class T>
struct HBuf {
  T* p = nullptr;
  size_t n = 0;
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() {
    if (p) cudaFreeHost(p);
  }
  T* get(size_t want) {
    if (want > n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      ck(cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<size_t>(want, 1) * sizeof(T), cudaHostAllocDefault),
         "cudaHostAlloc");
      n = want;
    }
    return p;
  }
};

// Host threads for the per-subdomain report / merge / split work of a BaB step
// (independent items; results land in per-item slots, so the outcome does not
// depend on the thread count).
int host_threads() {
  static const int n = [] {
    const char* e = std::getenv("BP_HOST_THREADS");
    const int v = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
    return std::clamp(v, 1, 64);
  }();
  return n;
}

template <class F>
void parallel_for(int n, F&& f) {
  const int nt = std::min(host_threads(), n / 8);  // below ~8 items per thread, stay serial
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        for (int i = t; i < n; i += nt) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

__global__ void fill_int_kernel(int* p, long long n, int v) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}
void fill_int(int* p, long long n, int v, cudaStream_t st) {
  if (n <= 0) return;
  const long long g = std::min<long long>((n + 255) / 256, 4096);
  fill_int_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(p, n, v);
  ck(cudaGetLastError(), "fill");
}

// Host copy of the objective and its compiled device form.
struct Compiled {
  bp::DevObjective o{};
  std::vector<float> fa;
  std::vector<double> da;
  std::vector<int> ia;
  int nq = 0;
  bool stream = false;
  size_t smem = 0;
  int kslab = 0;
  int R = 0;
  size_t tc_smem = 0;
  // stat layout (for bp_stat_layout): kind 0 preact(layer), 1 x, 2 u, 3 p, 4 op(index)
  std::vector<int> slot_kind, slot_index, slot_dim, slot_off;
  std::vector<double> x0, p0, ulo, uhi;
  int d = 0;
  int synth = 0;  // > 0: the separable synthetic objective of this dimension (no MLP, no cost program)
};

// Critical points of the 1-d synthetic term 5x^2 + cos(50x) on [-1, 1]: the roots of
// its derivative on a 400000-interval grid refined by 80 bisections, exactly the
// reference's SeparableBounder table (proj/src/bab.cpp:32-68).  Setup, not hot path:
// computed once per process and uploaded with the objective.
const std::vector<double>& separable_critical_points() {
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

// The synthetic objective (objective.cpp:82-104 / model.cpp build_synthetic): the
// planner sees a one-step "rollout" of d actions on the box [-1, 1]^d.
Compiled compile_synthetic(int dim) {
  if (dim <= 0) fail(BP_INVALID_ARGUMENT, "SyntheticObjective: dimension must be positive");
  Compiled c;
  c.synth = dim;
  c.d = dim;
  c.o.H = 1;
  c.o.ka = dim;
  c.o.kd = dim;
  c.o.d = dim;
  c.o.SP = 0;
  c.ulo.assign(static_cast<size_t>(dim), -1.0);
  c.uhi.assign(static_cast<size_t>(dim), 1.0);
  c.fa.push_back(0.f);
  c.da = separable_critical_points();
  c.ia.push_back(0);
  return c;
}

float bit_float(int32_t x) {
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}
int push_f(std::vector<float>& a, const double* p, size_t n) {
  while (a.size() % 4) a.push_back(0.f);
  const int off = static_cast<int>(a.size());
  for (size_t i = 0; i < n; ++i) a.push_back(static_cast<float>(p[i]));
  return off;
}
// an image starting on a 128-byte row of the arena (the TMA tensor maps address the arena in rows of 32)
int push_f_row(std::vector<float>& a, const double* p, size_t n) {
  while (a.size() % 32) a.push_back(0.f);
  return push_f(a, p, n);
}
int push_d(std::vector<double>& a, const double* p, size_t n) {
  while (a.size() % 2) a.push_back(0.0);
  const int off = static_cast<int>(a.size());
  a.insert(a.end(), p, p + n);
  return off;
}

void require_finite(const double* p, size_t n, const char* what) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) fail(BP_INVALID_ARGUMENT, std::string(what) + ": non-finite values");
}

Compiled compile(const bp_objective_desc& d) {
  Compiled c;
  bp::DevObjective& o = c.o;
  if (d.ks <= 0 || d.ka <= 0 || d.kd <= 0 || d.horizon < 1) fail(BP_INVALID_ARGUMENT, "objective: bad dimensions");
  const bool net = d.feature_mode == BP_FEATURE_NETWORK;
  if (d.ka != d.kd) fail(BP_INVALID_ARGUMENT, "objective: action and effector dimensions must match");
  if (d.ka > (net ? 16 : 8)) fail(BP_UNSUPPORTED, "objective: action dimension above 8 (16 for a bare network)");
  if (d.feature_mode == BP_FEATURE_RELATIVE && d.ks % d.kd != 0)
    fail(BP_INVALID_ARGUMENT, "objective: state must be whole keypoints of workspace dimension");
  if (d.n_layers < 1 || d.n_layers > bp::kMaxLayers) fail(BP_UNSUPPORTED, "objective: layer count outside 1..8");
  if (net) {
    if (d.horizon != 1 || d.widths[0] != d.ka || d.widths[d.n_layers] != d.ks)
      fail(BP_INVALID_ARGUMENT, "build_network_objective: one step, the network reads the box and outputs the value");
  } else if (d.widths[0] != d.ks + d.ka || d.widths[d.n_layers] != d.ks) {
    fail(BP_INVALID_ARGUMENT, "build_objective: model input must take state plus action and output the state");
  }
  if (d.relu_after[d.n_layers - 1]) fail(BP_INVALID_ARGUMENT, "objective: final layer must stay linear");
  if (d.n_ops > bp::kMaxOps) fail(BP_UNSUPPORTED, "objective: more than 32 cost ops");
  o.ks = d.ks;
  o.ka = d.ka;
  o.kd = d.kd;
  o.H = d.horizon;
  o.rel = d.feature_mode == BP_FEATURE_RELATIVE ? 1 : 0;
  o.net = net ? 1 : 0;
  o.L = d.n_layers;
  o.d = d.ka * d.horizon;
  c.d = o.d;
  int maxN = 0, maxK4 = 0, maxw = d.widths[0];
  for (int l = 0; l <= d.n_layers; ++l) {
    if (d.widths[l] <= 0) fail(BP_INVALID_ARGUMENT, "objective: widths must be positive");
    o.widths[l] = d.widths[l];
    maxw = std::max(maxw, d.widths[l]);
  }
  if (maxw > 1024) fail(BP_UNSUPPORTED, "objective: layer width above 1024");
  for (int l = 0; l < d.n_layers; ++l) {
    o.relu[l] = d.relu_after[l] ? 1 : 0;
    o.kpad[l] = r4(d.widths[l]);
    o.nstr[l] = r4(d.widths[l + 1]);
    if (o.nstr[l] > 16) maxN = std::max(maxN, o.nstr[l]);
    maxK4 = std::max(maxK4, o.kpad[l]);
    require_finite(d.W[l], static_cast<size_t>(d.widths[l]) * d.widths[l + 1], "linear weights");
    require_finite(d.b[l], static_cast<size_t>(d.widths[l + 1]), "linear bias");
  }
  c.nq = maxN <= 64 ? 1 : maxN <= 128 ? 2 : maxN <= 256 ? 4 : maxN <= 512 ? 8 : 0;
  if (c.nq == 0) fail(BP_UNSUPPORTED, "objective: hidden width above 512 (rollout kernel)");
  // forward weight image: layers back to back, each [kpad][nstr], then padding
  int img = 0;
  {
    while (c.fa.size() % 4) c.fa.push_back(0.f);
    const int base = static_cast<int>(c.fa.size());
    for (int l = 0; l < d.n_layers; ++l) {
      const int K = d.widths[l], N = d.widths[l + 1];
      o.w_smem_off[l] = img;
      o.wt[l] = base + img;
      std::vector<float> t(static_cast<size_t>(o.kpad[l]) * o.nstr[l], 0.f);
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) t[static_cast<size_t>(k) * o.nstr[l] + n] = static_cast<float>(d.W[l][static_cast<size_t>(n) * K + k]);
      c.fa.insert(c.fa.end(), t.begin(), t.end());
      img += o.kpad[l] * o.nstr[l];
    }
    c.fa.insert(c.fa.end(), static_cast<size_t>(64 * c.nq + 64), 0.f);  // over-read pad
    o.w_smem_total = img + 64 * c.nq + 64;
    o.w_max_layer = 0;
    for (int l = 0; l < d.n_layers; ++l) o.w_max_layer = std::max(o.w_max_layer, o.kpad[l] * o.nstr[l]);
  }
  for (int l = 0; l < d.n_layers; ++l) {
    std::vector<double> bp(static_cast<size_t>(o.nstr[l]), 0.0);
    for (int n = 0; n < d.widths[l + 1]; ++n) bp[static_cast<size_t>(n)] = d.b[l][n];
    o.bias[l] = push_f(c.fa, bp.data(), bp.size());
    o.wd[l] = push_d(c.da, d.W[l], static_cast<size_t>(d.widths[l]) * d.widths[l + 1]);
    o.bd[l] = push_d(c.da, d.b[l], static_cast<size_t>(d.widths[l + 1]));
  }
  require_finite(d.x0, static_cast<size_t>(d.ks), "scenario x0");
  require_finite(d.p0, static_cast<size_t>(d.kd), "scenario p0");
  o.x0 = push_f(c.fa, d.x0, static_cast<size_t>(d.ks));
  o.p0 = push_f(c.fa, d.p0, static_cast<size_t>(d.kd));
  o.x0d = push_d(c.da, d.x0, static_cast<size_t>(d.ks));
  o.p0d = push_d(c.da, d.p0, static_cast<size_t>(d.kd));
  c.x0.assign(d.x0, d.x0 + d.ks);
  c.p0.assign(d.p0, d.p0 + d.kd);
  c.ulo.assign(d.u_lower, d.u_lower + d.ka);
  c.uhi.assign(d.u_upper, d.u_upper + d.ka);
  for (int j = 0; j < d.ka; ++j)
    if (!(d.u_lower[j] <= d.u_upper[j])) fail(BP_INVALID_ARGUMENT, "scenario: action bounds inverted");

  // cost program: value dims and scratch columns
  o.n_ops = d.n_ops;
  const int C0 = r4(d.ks);
  o.ucol = C0;
  o.pcol = o.ucol + r4(d.ka);
  int col = o.pcol + r4(d.kd);
  std::vector<int> vdim = {d.ks, d.ka, d.kd};
  std::vector<char> need(static_cast<size_t>(3 + d.n_ops), 0);
  bool any_term = false;
  while (c.fa.size() % 4) c.fa.push_back(0.f);
  o.cost_f0 = static_cast<int>(c.fa.size());
  for (int i = 0; i < d.n_ops; ++i) {
    const bp_cost_op& s = d.ops[i];
    bp::DevOp& p = o.ops[i];
    std::memset(&p, 0, sizeof(p));
    const int nv = 3 + i;
    if (s.src0 < 0 || s.src0 >= nv || s.src1 >= nv) fail(BP_INVALID_ARGUMENT, "cost op: bad source");
    const int in = vdim[static_cast<size_t>(s.src0)];
    p.kind = s.kind;
    p.src0 = s.src0;
    p.src1 = s.kind == BP_OP_SUM ? s.src1 : -1;
    p.in_dim = in;
    p.is_term = s.is_term;
    p.weight_by_step = s.weight_by_step;
    p.stat = -1;
    p.stop = 0;
    p.folded = 0;
    int dim = s.dim;
    switch (s.kind) {
      case BP_OP_LINEAR:
        if (dim <= 0) fail(BP_INVALID_ARGUMENT, "linear: weight shape does not match argument");
        require_finite(s.W, static_cast<size_t>(dim) * in, "linear weights");
        require_finite(s.b, static_cast<size_t>(dim), "linear bias");
        p.w = push_f(c.fa, s.W, static_cast<size_t>(dim) * in);
        p.b = push_f(c.fa, s.b, static_cast<size_t>(dim));
        p.wd = push_d(c.da, s.W, static_cast<size_t>(dim) * in);
        p.bd = push_d(c.da, s.b, static_cast<size_t>(dim));
        {
          // A weight matrix at most a quarter full (C4's [I; -I]) also gets a CSR copy for the
          // rollouts' forward pass: the same fma chain over the nonzeros in column order (the
          // dense chain adds exact zeros; only the sign of an exactly-zero sum can differ)
          size_t nnz = 0;
          for (size_t k = 0; k < static_cast<size_t>(dim) * in; ++k) nnz += static_cast<float>(s.W[k]) != 0.f ? 1 : 0;
          if (static_cast<size_t>(dim) * in >= 64 && 4 * nnz <= static_cast<size_t>(dim) * in) {
            std::vector<int32_t> rp(static_cast<size_t>(dim) + 1, 0), ci;
            std::vector<float> val;
            for (int r = 0; r < dim; ++r) {
              for (int j = 0; j < in; ++j) {
                const float w = static_cast<float>(s.W[static_cast<size_t>(r) * in + j]);
                if (w != 0.f) {
                  ci.push_back(j);
                  val.push_back(w);
                }
              }
              rp[static_cast<size_t>(r) + 1] = static_cast<int32_t>(ci.size());
            }
            while (c.fa.size() % 4) c.fa.push_back(0.f);
            p.tgt = static_cast<int>(c.fa.size());  // [rowptr dim+1][cols nnz] as int bits, then [values nnz]
            for (int32_t x : rp) c.fa.push_back(bit_float(x));
            for (int32_t x : ci) c.fa.push_back(bit_float(x));
            for (float v : val) c.fa.push_back(v);
            p.ctr = 1;
          }
        }
        break;
      case BP_OP_RELU:
        dim = in;
        need[static_cast<size_t>(s.src0)] = 1;
        break;
      case BP_OP_SUM:
        dim = in;
        if (s.src1 >= 0 && vdim[static_cast<size_t>(s.src1)] != in) fail(BP_INVALID_ARGUMENT, "sum: argument dimensions differ");
        break;
      case BP_OP_SCALAR_AFFINE:
        dim = in;
        if (!std::isfinite(s.scale) || !std::isfinite(s.offset)) fail(BP_INVALID_ARGUMENT, "scalar_affine: non-finite parameter");
        p.scale = static_cast<float>(s.scale);
        p.offset = static_cast<float>(s.offset);
        p.scaled = s.scale;
        p.offsetd = s.offset;
        break;
      case BP_OP_SQDIST: {
        dim = 1;
        need[static_cast<size_t>(s.src0)] = 1;
        require_finite(s.target, static_cast<size_t>(in), "squared_distance target");
        require_finite(s.weight, static_cast<size_t>(in), "squared_distance weight");
        for (int j = 0; j < in; ++j)
          if (s.weight[j] < 0.0) fail(BP_INVALID_ARGUMENT, "squared_distance: weights must be nonnegative");
        p.tgt = push_f(c.fa, s.target, static_cast<size_t>(in));
        p.tgtd = push_d(c.da, s.target, static_cast<size_t>(in));
        std::vector<double> w;
        const int reps = s.weight_by_step ? d.horizon : 1;
        for (int t = 0; t < reps; ++t)
          for (int j = 0; j < in; ++j) w.push_back(s.weight_by_step ? d.step_weight[t] * s.weight[j] : s.weight[j]);
        p.wt = push_f(c.fa, w.data(), w.size());
        p.wtd = push_d(c.da, w.data(), w.size());
        break;
      }
      case BP_OP_HINGE:
        dim = 1;
        need[static_cast<size_t>(nv)] = 1;  // anchored on its own output
        // watch set = args and selves of every ReLU, SquaredDistance and PenaltyHinge
        // (objective.cpp:64-75): full CROWN encloses the hinge from its argument's bounds
        need[static_cast<size_t>(s.src0)] = 1;
        require_finite(s.center, static_cast<size_t>(in), "penalty_hinge center");
        if (!std::isfinite(s.radius) || s.radius < 0.0) fail(BP_INVALID_ARGUMENT, "penalty_hinge: radius must be finite and nonnegative");
        if (!std::isfinite(s.penalty) || s.penalty < 0.0) fail(BP_INVALID_ARGUMENT, "penalty_hinge: penalty must be finite and nonnegative");
        p.ctr = push_f(c.fa, s.center, static_cast<size_t>(in));
        p.ctrd = push_d(c.da, s.center, static_cast<size_t>(in));
        p.radius = static_cast<float>(s.radius);
        p.penalty = static_cast<float>(s.penalty);
        p.radiusd = s.radius;
        p.penaltyd = s.penalty;
        break;
      case BP_OP_SLICE:
        if (dim <= 0 || s.begin < 0 || s.begin + dim > in) fail(BP_INVALID_ARGUMENT, "slice: range outside argument");
        p.begin = s.begin;
        break;
      default:
        fail(BP_INVALID_ARGUMENT, "cost op: unknown kind");
    }
    if (s.is_term && dim != 1) fail(BP_INVALID_ARGUMENT, "cost op: terms must be scalar");
    any_term = any_term || s.is_term;
    p.dim = dim;
    p.col = col;
    col += dim;  // scalar access only: packed
    vdim.push_back(dim);
  }
  o.cost_f1 = static_cast<int>(c.fa.size());
  auto val_col = [&](int id) { return id < 0 ? -1 : id == 0 ? 0 : id == 1 ? o.ucol : id == 2 ? o.pcol : o.ops[id - 3].col; };
  for (int i = 0; i < d.n_ops; ++i) {
    o.ops[i].c0 = val_col(o.ops[i].src0);
    o.ops[i].c1 = val_col(o.ops[i].src1);
  }
  if (!any_term) fail(BP_INVALID_ARGUMENT, "objective: cost program has no terms");
  o.S = r8(std::max({maxK4, r4(maxw), col})) + 4;
  o.bw = std::max({maxw, col, d.ks});
  if (o.bw > 1024) fail(BP_UNSUPPORTED, "objective: cost scratch wider than 1024 columns");

  // stop set (objective.cpp:45-63)
  std::vector<int> xstop(static_cast<size_t>(d.horizon), 0);
  o.stop_layer = -1;
  o.stop_op = -1;
  if (d.stop_rule == BP_STOP_LAST_RELU) {
    for (int l = 0; l + 1 < d.n_layers; ++l)
      if (d.relu_after[l]) o.stop_layer = l;
    if (o.stop_layer < 0)  // relu_nodes.back(): the last ReLU of the final step's cost program
      for (int i = 0; i < d.n_ops; ++i)
        if (d.ops[i].kind == BP_OP_RELU) o.stop_op = i;
    if (o.stop_op >= 0) o.ops[o.stop_op].stop = 1;
  } else if (d.stop_rule == BP_STOP_EVERY_STEP_OUTPUT) {
    std::fill(xstop.begin(), xstop.end(), 1);
  } else if (d.stop_rule == BP_STOP_CUSTOM) {
    for (int i = 0; i < d.n_custom_stops; ++i) {
      const int t = d.custom_stop_steps[i];
      if (t < 1 || t > d.horizon) fail(BP_INVALID_ARGUMENT, "stop set: step outside horizon");
      xstop[static_cast<size_t>(t - 1)] = 1;
    }
  } else {
    fail(BP_INVALID_ARGUMENT, "unknown stop rule");
  }
  const bool any_xstop = std::any_of(xstop.begin(), xstop.end(), [](int v) { return v != 0; });
  while (c.ia.size() % 4) c.ia.push_back(0);
  o.xstop = static_cast<int>(c.ia.size());
  c.ia.insert(c.ia.end(), xstop.begin(), xstop.end());

  // watched-coordinate record of one step
  int sp = 0;
  for (int l = 0; l < d.n_layers; ++l) {
    o.pre_stat[l] = -1;
    if (d.relu_after[l]) {
      o.pre_stat[l] = sp;
      c.slot_kind.push_back(0), c.slot_index.push_back(l), c.slot_dim.push_back(d.widths[l + 1]), c.slot_off.push_back(sp);
      sp += d.widths[l + 1];
    }
  }
  auto rec = [&](int kind, int idx, int dim) {
    c.slot_kind.push_back(kind), c.slot_index.push_back(idx), c.slot_dim.push_back(dim), c.slot_off.push_back(sp);
    const int off = sp;
    sp += dim;
    return off;
  };
  o.x_stat = (need[0] || any_xstop) ? rec(1, 0, d.ks) : -1;
  o.u_stat = need[1] ? rec(2, 0, d.ka) : -1;
  o.p_stat = need[2] ? rec(3, 0, d.kd) : -1;
  for (int i = 0; i < d.n_ops; ++i)
    if (need[static_cast<size_t>(3 + i)]) o.ops[i].stat = rec(4, i, o.ops[i].dim);
  o.SP = sp;
  {  // recorded scratch columns: x_t, u_t, p_t and cost-op values (fused stats pass of the tcgen05 kernel)
    std::vector<int> pairs;
    auto add = [&](int col0, int stat, int dim) {
      if (stat < 0) return;
      for (int j = 0; j < dim; ++j) pairs.push_back(col0 + j), pairs.push_back(stat + j);
    };
    add(0, o.x_stat, d.ks);
    add(o.ucol, o.u_stat, d.ka);
    add(o.pcol, o.p_stat, d.kd);
    for (int i = 0; i < d.n_ops; ++i) add(o.ops[i].col, o.ops[i].stat, o.ops[i].dim);
    while (c.ia.size() % 4) c.ia.push_back(0);
    o.sc_list = static_cast<int>(c.ia.size());
    o.n_sc = static_cast<int>(pairs.size() / 2);
    c.ia.insert(c.ia.end(), pairs.begin(), pairs.end());
  }

  // rollout tile and shared-memory plan
  c.R = bp::rollout_rows_per_tile(c.nq);
  o.red_w = 4;
  for (int l = 0; l < d.n_layers; ++l)
    if (o.relu[l]) o.red_w = std::max(o.red_w, o.nstr[l]);
  const size_t base_bytes = (static_cast<size_t>(c.R) * o.S + static_cast<size_t>(c.R) * 9 + 4 * o.red_w) * sizeof(float);
  const size_t resident = base_bytes + static_cast<size_t>(o.w_smem_total) * sizeof(float);
  const size_t cap = 227 * 1024;
  if (resident <= cap) {
    c.stream = false;
    c.smem = resident;
    c.kslab = 0;
  } else {
    int maxNS = 0;
    for (int l = 0; l < d.n_layers; ++l) maxNS = std::max(maxNS, o.nstr[l]);
    const size_t pad = static_cast<size_t>(64 * c.nq + 64);
    if (base_bytes + (4 * static_cast<size_t>(maxNS) + pad) * sizeof(float) > cap)
      fail(BP_UNSUPPORTED, "objective: activations do not fit in shared memory");
    int ksl = static_cast<int>((cap - base_bytes) / sizeof(float) - pad) / maxNS;
    ksl = std::min(ksl & ~3, r4(maxK4));
    c.stream = true;
    c.kslab = ksl;
    c.smem = base_bytes + (static_cast<size_t>(ksl) * maxNS + pad) * sizeof(float);
  }
  // tcgen05 (3xTF32) rollouts: v1 (rollout_tc.cu) when every layer K, N <= 128; v2
  // (rollout_tc2.cu) when every K, N <= 256 -- two 128-row tiles per CTA at widths <= 128,
  // one at widths <= 256 -- and its shared memory leaves a weight ring of >= 3 blocks.
  {
    bool ok1 = true, ok2 = true;
    int kbmax = 1, npadmax = 16;
    for (int l = 0; l < d.n_layers; ++l) {
      const int K = d.widths[l], N = d.widths[l + 1];
      if (K > 128 || N > 128) ok1 = false;
      if (K > 256 || N > 256) ok2 = false;
      kbmax = std::max({kbmax, (K + 31) / 32, (N + 31) / 32});
      npadmax = std::max(npadmax, std::max(16, r16(N)));
    }
    o.tc = 0;
    o.tc2 = 0;
    o.tc2_rw = 0;
    o.tc2_ring = 0;
    o.tc2_pair = 0;
    if (ok2 && !net) {
      o.tc_kbmax = kbmax;
      o.tc_npadmax = npadmax;
      o.tc_S = std::max(col, d.ks) | 1;  // odd row stride: one row per thread, conflict-free
      o.tc_xs = d.ks | 1;  // x_t hand-off rows, odd stride
      o.tc_cols = 32;
      while (o.tc_cols < npadmax) o.tc_cols *= 2;
      for (int l = 0; l < d.n_layers; ++l) {
        const int K = d.widths[l], N = d.widths[l + 1];
        const int npad = std::max(16, r16(N)), kb = (K + 31) / 32;
        o.tc_npad[l] = npad;
        o.tc_kb[l] = kb;
        o.tc_ksteps[l] = (K + 7) / 8;
        o.tc_w[l] = push_f_row(c.fa, tc_image(d.W[l], N, K, npad).data(), static_cast<size_t>(kb) * 2 * npad * 32);
        std::vector<double> bp(static_cast<size_t>(npad), 0.0);
        for (int n = 0; n < N; ++n) bp[static_cast<size_t>(n)] = d.b[l][n];
        o.tc_bias[l] = push_f(c.fa, bp.data(), bp.size());
      }
      if (ok1) {
        c.tc_smem = bp::rollout_tc_smem(o);
        o.tc = c.tc_smem <= cap ? 1 : 0;
      }
      // two ping-pong tiles when the widths allow it and both tiles' scratch rows fit,
      // else one tile; the weight ring takes the rest (>= three 128-row blocks)
      // the MMA warp holds a K-block's weight blocks at once (hi, lo, placed contiguously: 64 KB at
      // width 256); one more block in flight keeps the producer ahead
      const size_t min_ring_narrow = 3 * 128 * 128, min_ring_wide = 5 * 128 * 128;
      const bool narrow = npadmax <= 128 && kbmax <= 4;
      const int plans[3][2] = {{2, 128}, {1, 128}, {1, 256}};
      for (const auto& pl : plans) {
        if (pl[1] == 128 && !narrow) continue;
        o.tc2 = pl[0];
        o.tc2_rw = pl[1];
        // CTA pair (rollout_tc2.cu, cta_group::2) at width 256 when each layer's N splits
        // evenly between the two CTAs (256, or a multiple of 32 up to 128).  Opt-in
        // (BP_TC2_PAIR=1): correct, but epilogue-bound and slower than one CTA on C3
        // (168.5 vs 178.5 TFLOP/s).  The ring is planned for its layout.
        o.tc2_pair = 0;
        if (pl[1] == 256) {
          const char* e = std::getenv("BP_TC2_PAIR");
          bool ok = e != nullptr && std::string(e) == "1";
          for (int l = 0; l < d.n_layers; ++l) {
            const int np = o.tc_npad[l];
            ok = ok && (np == 256 || (np <= 128 && np % 32 == 0));
          }
          o.tc2_pair = ok ? 1 : 0;
        }
        const size_t fixed = bp::rollout_tc2_fixed_smem(o);
        const size_t min_ring = pl[1] == 256 ? min_ring_wide : min_ring_narrow;
        if (fixed + min_ring <= cap) {
          o.tc2_ring = static_cast<int>((cap - fixed) & ~static_cast<size_t>(1023));
          if (std::getenv("BP_DEBUG_TC2"))
            std::fprintf(stderr, "[tc2] tiles %d width %d pair %d: fixed %zu B (S=%d), ring %d B\n", o.tc2, o.tc2_rw,
                         o.tc2_pair, fixed, o.tc_S, o.tc2_ring);
          break;
        }
        o.tc2 = 0;
      }
    }
    // v2 output-layer folding: every cost-program LINEAR on x_t (C4's L1 goal [I; -I] and its
    // state-bound [e0; -e0]) becomes extra N columns of the last layer's MMA -- W_op W_L and
    // W_op b_L + b_op, formed in FP64 and rounded once -- so the cost warps read those values from
    // the scratch instead of computing them row by row.  Only for the v2 kernel (v1 keeps the
    // plain image; SIMT and the bound kernels read the ops as given).
    o.fold_n = 0;
    o.fold_list = 0;
    if (ok2 && !net && o.tc == 0 && o.tc2 != 0 && o.tc2_pair == 0 && std::getenv("BP_NO_FOLD") == nullptr) {
      const int l = d.n_layers - 1, K = d.widths[l], N = d.widths[l + 1];
      std::vector<int> fold_ops;
      int fold_n = 0;
      for (int i = 0; i < d.n_ops; ++i)
        if (d.ops[i].kind == BP_OP_LINEAR && d.ops[i].src0 == BP_VAL_X) {
          fold_ops.push_back(i);
          fold_n += o.ops[i].dim;
        }
      const int np2 = std::max(16, r16(N + fold_n));
      if (fold_n > 0 && np2 <= std::min(o.tc2_rw, 256)) {
        // extended output layer: rows [0, N) = W_L, then per folded op its rows of W_op W_L
        std::vector<double> Wx(static_cast<size_t>(N + fold_n) * K), bx(static_cast<size_t>(N + fold_n));
        for (int n = 0; n < N; ++n) {
          for (int k = 0; k < K; ++k) Wx[static_cast<size_t>(n) * K + k] = d.W[l][static_cast<size_t>(n) * K + k];
          bx[static_cast<size_t>(n)] = d.b[l][n];
        }
        std::vector<int> fcols;
        int row = N;
        for (int i : fold_ops) {
          const bp_cost_op& op = d.ops[i];
          for (int r = 0; r < o.ops[i].dim; ++r, ++row) {
            for (int k = 0; k < K; ++k) {
              double acc = 0.0;
              for (int j = 0; j < N; ++j)
                acc += op.W[static_cast<size_t>(r) * N + j] * d.W[l][static_cast<size_t>(j) * K + k];
              Wx[static_cast<size_t>(row) * K + k] = acc;
            }
            double bb = op.b[r];
            for (int j = 0; j < N; ++j) bb += op.W[static_cast<size_t>(r) * N + j] * d.b[l][j];
            bx[static_cast<size_t>(row)] = bb;
            fcols.push_back(o.ops[i].col + r);
          }
          o.ops[i].folded = 1;
        }
        const int NX = N + fold_n, kb = (K + 31) / 32;
        o.tc_w[l] = push_f_row(c.fa, tc_image(Wx.data(), NX, K, np2).data(), static_cast<size_t>(kb) * 2 * np2 * 32);
        std::vector<double> bp(static_cast<size_t>(np2), 0.0);
        for (int n = 0; n < NX; ++n) bp[static_cast<size_t>(n)] = static_cast<double>(static_cast<float>(bx[static_cast<size_t>(n)]));
        o.tc_bias[l] = push_f(c.fa, bp.data(), bp.size());
        o.tc_npad[l] = np2;
        o.tc_npadmax = std::max(o.tc_npadmax, np2);
        o.fold_n = fold_n;
        while (c.ia.size() % 4) c.ia.push_back(0);
        o.fold_list = static_cast<int>(c.ia.size());
        c.ia.insert(c.ia.end(), fcols.begin(), fcols.end());
      }
    }
    // tcgen05 v3 (rollout_tc3.cu): [K0 <= 32, N0, N1 <= 512, N2 <= 32] with relu after the two
    // hidden layers -- the 512-wide C5 shape, whose accumulators v1 / v2 cannot hold in TMEM
    o.tc3 = 0;
    if (!net && d.n_layers == 3 && d.widths[0] <= 32 && d.widths[1] <= 512 && d.widths[2] <= 512 && d.widths[3] <= 32 &&
        d.relu_after[0] && d.relu_after[1] && !d.relu_after[2] && std::max(d.widths[1], d.widths[2]) > 256) {
      const int np0 = (d.widths[1] + 31) & ~31, np1 = (d.widths[2] + 31) & ~31, np2 = std::max(16, r16(d.widths[3]));
      o.tc3_np[0] = np0;
      o.tc3_np[1] = np1;
      o.tc3_np[2] = np2;
      o.tc3_k0steps = (d.widths[0] + 7) / 8;
      o.tc_S = std::max(col, d.ks) | 1;
      // one K-block image of `rows` output rows x 32 K-columns of W (hi block then lo block), rows
      // n0.., columns k0.., 128B-swizzled rows (as the v1 / v2 images)
      auto block = [&](std::vector<double>& img, int l, int n0, int rows, int k0) {
        const int K = d.widths[l], N = d.widths[l + 1];
        const size_t base = img.size();
        img.resize(base + static_cast<size_t>(2) * rows * 32, 0.0);
        for (int n = 0; n < rows; ++n)
          for (int cc = 0; cc < 32; ++cc) {
            const int gn = n0 + n, k = k0 + cc;
            const float w = (gn < N && k < K) ? static_cast<float>(d.W[l][static_cast<size_t>(gn) * K + k]) : 0.f;
            const float hi = rna_tf32_host(w), lo = rna_tf32_host(w - hi);
            const size_t pos = static_cast<size_t>(n) * 32 + (((cc >> 2) ^ (n & 7)) << 2) + (cc & 3);
            img[base + pos] = hi;
            img[base + static_cast<size_t>(rows) * 32 + pos] = lo;
          }
      };
      std::vector<double> i0, i1, i2;
      for (int kb = 0; kb < np0 / 32; ++kb) block(i0, 0, 32 * kb, 32, 0);  // layer 0: N-block kb, K = features
      for (int j = 0; j * 256 < np1; ++j)
        for (int kb = 0; kb < np0 / 32; ++kb) block(i1, 1, 256 * j, std::min(256, np1 - 256 * j), 32 * kb);
      for (int kb = 0; kb < np1 / 32; ++kb) block(i2, 2, 0, np2, 32 * kb);
      o.tc3_w[0] = push_f_row(c.fa, i0.data(), i0.size());
      o.tc3_w[1] = push_f_row(c.fa, i1.data(), i1.size());
      o.tc3_w[2] = push_f_row(c.fa, i2.data(), i2.size());
      std::vector<double> bb(static_cast<size_t>(np0 + np1 + np2), 0.0);
      for (int n = 0; n < d.widths[1]; ++n) bb[static_cast<size_t>(n)] = d.b[0][n];
      for (int n = 0; n < d.widths[2]; ++n) bb[static_cast<size_t>(np0 + n)] = d.b[1][n];
      for (int n = 0; n < d.widths[3]; ++n) bb[static_cast<size_t>(np0 + np1 + n)] = d.b[2][n];
      o.tc3_bias = push_f(c.fa, bb.data(), bb.size());
      const size_t fixed = bp::rollout_tc3_fixed_smem(o);
      const size_t min_ring = 3 * 256 * 128;  // a layer-1 K-block (hi + lo) and one more entry in flight
      if (fixed + min_ring <= cap) {
        o.tc3_ring = static_cast<int>((cap - fixed) & ~static_cast<size_t>(1023));
        o.tc3 = 1;
        if (std::getenv("BP_DEBUG_TC2"))
          std::fprintf(stderr, "[tc3] fixed %zu B (S=%d), ring %d B\n", fixed, o.tc_S, o.tc3_ring);
      }
    }
  }
  return c;
}

struct Report {  // SearchReport (search.hpp:53-63) as the planner consumes it
  bool ok = true;
  std::string error;
  double uf = std::numeric_limits<double>::infinity();
  std::vector<double> best;
  std::vector<float> top_val;  // ascending
  std::vector<float> top_act;  // n_top x d
  int64_t samples = 0;
  std::vector<double> uf_history;
  std::vector<int64_t> samples_history;
};

}  // namespace

// Device-direct exchange over NCCL (bp_set_nccl).  libnccl.so.2 is dlopen'ed, so the library
// has no link-time NCCL dependency and shares the process's copy when one is loaded (torch's).
struct NcclLink {
  void* dl = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) err_str = nullptr;
  cudaStream_t* stream = nullptr;  // the context's current stream
  unsigned char* d_send = nullptr;
  unsigned char* d_recv = nullptr;
  size_t cap_send = 0, cap_recv = 0;

  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) fail(BP_NCCL, std::string("nccl: ") + what + ": " + (err_str ? err_str(r) : "error"));
  }
  static NcclLink* open_lib() {
    std::unique_ptr<NcclLink> L(new NcclLink());
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      L->dl = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (L->dl) break;
    }
    if (!L->dl) fail(BP_NCCL, "nccl: libnccl.so.2 not found");
    auto sym = [&](const char* n) {
      void* f = dlsym(L->dl, n);
      if (!f) fail(BP_NCCL, std::string("nccl: missing symbol ") + n);
      return f;
    };
    L->get_id = reinterpret_cast<decltype(L->get_id)>(sym("ncclGetUniqueId"));
    L->init = reinterpret_cast<decltype(L->init)>(sym("ncclCommInitRank"));
    L->destroy = reinterpret_cast<decltype(L->destroy)>(sym("ncclCommDestroy"));
    L->allgather = reinterpret_cast<decltype(L->allgather)>(sym("ncclAllGather"));
    L->send = reinterpret_cast<decltype(L->send)>(sym("ncclSend"));
    L->recv = reinterpret_cast<decltype(L->recv)>(sym("ncclRecv"));
    L->group_start = reinterpret_cast<decltype(L->group_start)>(sym("ncclGroupStart"));
    L->group_end = reinterpret_cast<decltype(L->group_end)>(sym("ncclGroupEnd"));
    L->err_str = reinterpret_cast<decltype(L->err_str)>(sym("ncclGetErrorString"));
    return L.release();
  }
  ~NcclLink() {
    if (comm && destroy) destroy(comm);
    if (d_send) cudaFree(d_send);
    if (d_recv) cudaFree(d_recv);
    // the library handle stays open: other users (torch) may share it
  }
  unsigned char* buf(unsigned char*& p, size_t& cap, size_t n) {
    if (n > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (cudaMalloc(reinterpret_cast<void**>(&p), n) != cudaSuccess) fail(BP_CUDA, "nccl: staging buffer");
      cap = n;
    }
    return p;
  }
  // all-gather of device buffers: world * bytes land in recv in rank order
  void allgather_dev(const void* send, void* recv, size_t bytes) const {
    check(allgather(send, recv, bytes, ncclUint8, comm, *stream), "all-gather");
  }
  // all-to-all-v of device buffers: send segments in rank order (send_bytes[r] to rank r),
  // receive segments in rank order (recv_bytes[r] from rank r); one NCCL group
  void alltoallv_dev(const unsigned char* send, const int64_t* send_bytes, unsigned char* recv,
                     const int64_t* recv_bytes) const {
    check(group_start(), "group start");
    size_t so = 0, ro = 0;
    for (int r = 0; r < world; ++r) {
      const size_t sb = static_cast<size_t>(send_bytes[r]), rb = static_cast<size_t>(recv_bytes[r]);
      if (sb > 0) check(this->send(send + so, sb, ncclUint8, r, comm, *stream), "send");
      if (rb > 0) check(this->recv(recv + ro, rb, ncclUint8, r, comm, *stream), "recv");
      so += sb;
      ro += rb;
    }
    check(group_end(), "group end");
  }
};

// bp_exchange_fn over NCCL for the planner's host-side all-gathers (heads, status words):
// staged through device buffers on the context's stream
int nccl_allgather_host(void* user, const void* send, size_t bytes, void* recv) {
  try {
    NcclLink* L = static_cast<NcclLink*>(user);
    unsigned char* ds = L->buf(L->d_send, L->cap_send, std::max<size_t>(bytes, 1));
    unsigned char* dr = L->buf(L->d_recv, L->cap_recv, std::max<size_t>(bytes * L->world, 1));
    if (cudaMemcpyAsync(ds, send, bytes, cudaMemcpyHostToDevice, *L->stream) != cudaSuccess) return 1;
    L->allgather_dev(ds, dr, bytes);
    if (cudaMemcpyAsync(recv, dr, bytes * L->world, cudaMemcpyDeviceToHost, *L->stream) != cudaSuccess) return 1;
    return cudaStreamSynchronize(*L->stream) == cudaSuccess ? 0 : 1;
  } catch (...) {
    return 1;
  }
}

struct bp_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  bool loaded = false;
  Compiled comp;
  DBuf<float> d_fa;
  DBuf<unsigned char> d_tmaps;  // CUtensorMap array for the v2 CTA pair (encode_tmaps)
  DBuf<double> d_da;
  DBuf<int> d_ia;
  // search state
  int n = 0, rows = 0, cur = 0, iters = 0;
  bool searched = false;
  int top_cap = 0;
  DBuf<unsigned long long> seeds;
  DBuf<float> lo_f, hi_f, warm_f, mu, var, var_floor, best, uf, actions, costs, top_val0, top_val1, top_act0, top_act1;
  DBuf<float> ratios, grad;
  DBuf<double> grad_ckpt;
  DBuf<int> failed, top_seq0, top_seq1, top_cnt, stat_min, stat_max, use_flags;
  DBuf<double> lo_d, hi_d, ivl_lo, ivl_hi, lf;
  DBuf<float> uf_hist;
  HBuf<float> h_uf, h_best, h_hist, h_tv, h_ta;  // pinned report staging
  HBuf<int> h_cnt;
  bp::SearchArgs last{};  // the last search's arguments (the pool merge reads its outputs)
  // routed top samples of the iteration's children (pool.cu), by local index
  DBuf<float> st_val, st_act;
  DBuf<int> st_n;
  DBuf<unsigned char> sort_keys;  // search_update keys in global memory (large batches)
  int smem_optin = 0;             // cudaDevAttrMaxSharedMemoryPerBlockOptin
  // slab chunks (pool.cu) kept between plans, for pools of this geometry
  int slab_d = 0, slab_K = 0;
  std::vector<unsigned char*> slab_spare;
  // search / bound buffers are sized for at least this many boxes (a planner's children
  // per step), so the ramp-up iterations do not reallocate them
  int reserve_boxes = 0;
  std::vector<int> h_failed;
  int64_t boxes_searched = 0, boxes_failed = 0;  // bp_search_counters
  // plan log (bp_set_plan_log): per searched child of a plan, in the order the planner created it --
  // the decision-replay test feeds these reports and bounds to the oracle's plan()
  struct LogChild {
    int iter;
    std::vector<double> lo, hi;
    double lf;
    Report rep;
  };
  bool plan_log_on = false;
  std::vector<LogChild> plan_log;
  std::vector<Report> reports;
  // sharding: rank / world and the allgather hook (host buffers)
  int rank = 0, world = 1;
  bp_exchange_fn exchange = nullptr;
  bp_alltoallv_fn alltoallv = nullptr;
  void* exchange_user = nullptr;
  std::unique_ptr<NcclLink> nccl;  // bp_set_nccl: device-direct exchange (replaces the hooks)
  // scratch for bp_rollout
  DBuf<float> r_actions, r_costs, r_states;
  DBuf<long long> timeline;
  DBuf<int> r_min, r_max;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> roll_events;
  size_t roll_event_next = 0;
  double rollout_ms = 0, bound_ms = 0, search_ms = 0;
  int64_t rollout_launches = 0, launches = 0;
  bool timing = true;
  int path_mode = 0;  // 0 auto, 1 SIMT, 2 tcgen05 v1, 3 tcgen05 v2, 5 tcgen05 v3 (BP_ROLLOUT or bp_set_rollout_path)
  // rollout kernel for the loaded objective: 1 SIMT, 2 tcgen05 v1, 3 tcgen05 v2, 4 synthetic, 5 tcgen05 v3
  int kernel() const {
    if (comp.synth) return 4;
    if (!loaded || path_mode == 1) return 1;
    if (path_mode == 2) return comp.o.tc ? 2 : 1;
    if (path_mode == 3) return comp.o.tc2 ? 3 : 1;
    if (path_mode == 5) return comp.o.tc3 ? 5 : 1;
    // auto: v1 where every width is <= 128 (faster there: rollout_tc2.cu header), else v2, else v3
    return comp.o.tc ? 2 : comp.o.tc2 ? 3 : comp.o.tc3 ? 5 : 1;
  }

  ~bp_ctx() {
    nccl.reset();  // before the streams go
    for (unsigned char* p : slab_spare) cudaFree(p);
    for (auto& e : roll_events) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
  void use() { ck(cudaSetDevice(device), "cudaSetDevice"); }
  bp::DevObjective dev() {
    bp::DevObjective o = comp.o;
    o.f = d_fa.p;
    o.tmaps = comp.o.n_tmap > 0 ? d_tmaps.p : nullptr;
    o.dd = d_da.p;
    o.iv = d_ia.p;
    return o;
  }
  std::pair<cudaEvent_t, cudaEvent_t> roll_event() {
    if (roll_event_next == roll_events.size()) {
      cudaEvent_t a, b;
      ck(cudaEventCreate(&a), "event");
      ck(cudaEventCreate(&b), "event");
      roll_events.push_back({a, b});
    }
    return roll_events[roll_event_next++];
  }
  void harvest_roll_events() {
    for (size_t i = 0; i < roll_event_next; ++i) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, roll_events[i].first, roll_events[i].second), "cudaEventElapsedTime");
      rollout_ms += ms;
    }
    roll_event_next = 0;
  }
  void rollout(const float* actions, float* costs, float* states, int* smin, int* smax, int* fail_flags,
               long long n_rows, int rows_per_sub) {
    if (comp.o.net) fail(BP_UNSUPPORTED, "a bare network objective is bounded, not rolled out");
    bp::RolloutArgs a{actions, costs, states, smin, smax, fail_flags, n_rows, rows_per_sub, comp.kslab, nullptr};
    static const bool want_tl = std::getenv("BP_TC_TIMELINE") != nullptr;
    const int kern = kernel();
    if (want_tl && kern >= 2) {
      a.timeline = timeline.get(4096);
      ck(cudaMemsetAsync(a.timeline, 0, 4096 * 8, stream), "memset");
    }
    std::pair<cudaEvent_t, cudaEvent_t> ev{};
    if (timing) {
      ev = roll_event();
      ck(cudaEventRecord(ev.first, stream), "event");
    }
    if (comp.synth)
      ck(bp::launch_synthetic_eval(actions, costs, fail_flags, n_rows, comp.synth, rows_per_sub, stream),
         "synthetic objective launch");
    else if (kern == 3)
      ck(bp::launch_rollout_tc2(dev(), a, stream), "rollout (tcgen05 v2) launch");
    else if (kern == 5)
      ck(bp::launch_rollout_tc3(dev(), a, stream), "rollout (tcgen05 v3) launch");
    else if (kern == 2)
      ck(bp::launch_rollout_tc(dev(), a, stream), "rollout (tcgen05) launch");
    else
      ck(bp::launch_rollout(dev(), a, comp.nq, comp.stream, comp.smem, stream), "rollout launch");
    if (timing) ck(cudaEventRecord(ev.second, stream), "event");
    if (a.timeline) {  // debug: print CTA 0's phase marks of step 3
      std::vector<long long> tl(4096);
      ck(cudaMemcpyAsync(tl.data(), a.timeline, 4096 * 8, cudaMemcpyDeviceToHost, stream), "D2H");
      ck(cudaStreamSynchronize(stream), "sync");
      const long long t0 = tl[0];
      std::fprintf(stderr, "[timeline] role,mark,cycles-from-step-start:");
      for (int i = 0; i < 4096; ++i)
        if (tl[i] != 0)  // values tagged with bit 40 are durations, not clock stamps
          std::fprintf(stderr, " %d:%lld", i, (tl[i] >> 40) == 1 ? tl[i] - (1ll << 40) : tl[i] - t0);
      std::fprintf(stderr, "\n");
    }
    ++rollout_launches;
    ++launches;
  }
};

namespace {

void check_ctx(bp_ctx* c) {
  if (c == nullptr) fail(BP_INVALID_ARGUMENT, "null context");
  c->use();
}
void check_loaded(bp_ctx* c) {
  check_ctx(c);
  if (!c->loaded) fail(BP_LOGIC, "no objective loaded");
}

// Device batch search (batch_search, search.cpp:262-282, with run_cem / run_mppi / run_gd),
// in three parts: search_setup (configuration, per-box seeds, state buffers; the boxes
// and warm starts must already be in c->lo_f / hi_f / lo_d / hi_d / warm_f), search_run
// (init + the iterations), search_harvest (host reports for the C-ABI's report calls).
bp::SearchArgs search_setup(bp_ctx* c, int n, const bp_search_config& cfg, const int64_t* seed_index, bool warm) {
  const Compiled& cp = c->comp;
  const int d = cp.d;
  if (cfg.iterations <= 0 || cfg.samples_per_iter <= 0)
    fail(BP_INVALID_ARGUMENT, "search: iterations and samples per iteration must be positive");
  bp::SearchArgs a{};
  a.n = n;
  a.d = d;
  a.method = cfg.method == BP_SEARCH_MPPI ? 1 : cfg.method == BP_SEARCH_GD ? 2 : 0;
  std::vector<float> ratios;
  if (a.method == 2) {  // run_gd (search.cpp:214-245): samples_per_iter starts, no incumbent row
    a.groups = 1;
    a.per_group = std::max(1, cfg.samples_per_iter);
    a.elites = 1;
    a.gd_base_step = static_cast<float>(cfg.gd_base_step);
    if (cfg.gd_n_ratios > 0)
      for (int i = 0; i < cfg.gd_n_ratios; ++i) ratios.push_back(static_cast<float>(cfg.gd_step_ratios[i]));
    else
      ratios.push_back(1.f);
    a.gd_n_ratios = static_cast<int>(ratios.size());
  } else if (a.method == 0) {
    a.groups = std::max(1, cfg.cem_agents);
    a.per_group = std::max(1, cfg.samples_per_iter / a.groups);
    a.elites = std::max(1, cfg.cem_elites);
  } else {
    const int nn = cfg.mppi_n_noise > 0 ? cfg.mppi_n_noise : 1;
    const int nt = cfg.mppi_n_temp > 0 ? cfg.mppi_n_temp : 1;
    for (int i = 0; i < nn; ++i) ratios.push_back(cfg.mppi_n_noise > 0 ? static_cast<float>(cfg.mppi_noise_ratios[i]) : 1.f);
    for (int i = 0; i < nt; ++i) ratios.push_back(cfg.mppi_n_temp > 0 ? static_cast<float>(cfg.mppi_temperature_ratios[i]) : 1.f);
    a.groups = nn * nt;
    a.n_noise = nn;
    a.per_group = std::max(1, cfg.samples_per_iter / a.groups);
    a.elites = 1;
  }
  if (a.groups > 32) fail(BP_UNSUPPORTED, "search: more than 32 agents / instances");
  a.n_samp = a.groups * a.per_group;
  a.rows = a.method == 2 ? a.n_samp : a.n_samp + 1;
  a.top_cap = std::max(cfg.top_capacity, 1);
  a.jitter = static_cast<float>(cfg.cem_jitter);
  a.init_sigma = static_cast<float>(cfg.cem_init_sigma);
  a.noise_frac = static_cast<float>(cfg.mppi_noise_frac);
  a.temperature = static_cast<float>(cfg.mppi_temperature);
  c->n = n;
  c->rows = a.rows;
  c->top_cap = a.top_cap;
  c->iters = cfg.iterations;
  cudaStream_t st = c->stream;
  // buffers sized for at least c->reserve_boxes boxes (no reallocation while a plan ramps up)
  const size_t nb = static_cast<size_t>(std::max(n, c->reserve_boxes));
  const size_t nd = nb * d;
  std::vector<unsigned long long> seeds(static_cast<size_t>(n));
  // derive_seed(seed, i) (rng.hpp:37-39) with i the box's index in the caller's batch
  for (int i = 0; i < n; ++i)
    seeds[static_cast<size_t>(i)] = cfg.seed ^ static_cast<unsigned long long>(seed_index ? seed_index[i] : i);
  a.seeds = c->seeds.get(nb);
  ck(memcpy_counted(const_cast<unsigned long long*>(a.seeds), seeds.data(), seeds.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
  a.lo = c->lo_f.get(nd);
  a.hi = c->hi_f.get(nd);
  a.warm = warm ? c->warm_f.get(nd) : nullptr;
  if (!ratios.empty()) {
    float* r = c->ratios.get(ratios.size());
    ck(memcpy_counted(r, ratios.data(), ratios.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
    if (a.method == 2) {
      a.gd_ratios = r;
    } else {
      a.noise_ratios = r;
      a.temp_ratios = r + a.n_noise;
    }
  }
  a.mu = c->mu.get(nb * a.groups * d);
  a.var = c->var.get(nb * a.groups * d);
  a.var_floor = c->var_floor.get(nd);
  a.best = c->best.get(nd);
  a.uf = c->uf.get(nb);
  a.actions = c->actions.get(nb * a.rows * d);
  a.costs = c->costs.get(nb * a.rows);
  a.failed = c->failed.get(nb);
  const size_t tk = nb * a.top_cap;
  a.top_val[0] = c->top_val0.get(tk);
  a.top_val[1] = c->top_val1.get(tk);
  a.top_seq[0] = c->top_seq0.get(tk);
  a.top_seq[1] = c->top_seq1.get(tk);
  a.top_act[0] = c->top_act0.get(tk * d);
  a.top_act[1] = c->top_act1.get(tk * d);
  a.top_cnt = c->top_cnt.get(nb);
  // search_update sorts top_capacity + rows keys per box: in shared memory when they fit the opt-in
  // limit, else in a global scratch (no limit on samples_per_iter, like the reference's heap)
  a.sort_keys = nullptr;
  static const bool force_global = std::getenv("BP_SEARCH_SORT_GLOBAL") != nullptr;  // test aid
  if (force_global || bp::search_update_smem(a) > static_cast<size_t>(c->smem_optin)) {
    a.sort_keys = c->sort_keys.get(nb * bp::search_sort_key_bytes(a));
    if (bp::search_update_smem(a) > static_cast<size_t>(c->smem_optin))
      fail(BP_UNSUPPORTED, "search: agents x elites too large for the refit's shared memory");
  }
  return a;
}

// Host boxes / warm starts into the search inputs (the C-ABI's bp_batch_search path).
void place_host_boxes(bp_ctx* c, int n, const double* lo, const double* hi, const double* warm) {
  const int d = c->comp.d;
  const size_t nd = static_cast<size_t>(n) * d;
  // the same capacities search_setup asks for (a smaller request here and a larger one
  // there would reallocate and drop the uploaded boxes)
  const size_t cap = static_cast<size_t>(std::max(n, c->reserve_boxes)) * d;
  for (size_t i = 0; i < nd; ++i)
    if (!(lo[i] <= hi[i]) || !std::isfinite(lo[i]) || !std::isfinite(hi[i]))
      fail(BP_INVALID_ARGUMENT, "BoxDomain: invalid bounds");
  cudaStream_t st = c->stream;
  std::vector<float> lf32(nd), hf32(nd);
  for (size_t i = 0; i < nd; ++i) {
    lf32[i] = static_cast<float>(lo[i]);
    hf32[i] = static_cast<float>(hi[i]);
  }
  ck(memcpy_counted(c->lo_f.get(cap), lf32.data(), nd * 4, cudaMemcpyHostToDevice, st), "H2D");
  ck(memcpy_counted(c->hi_f.get(cap), hf32.data(), nd * 4, cudaMemcpyHostToDevice, st), "H2D");
  ck(memcpy_counted(c->lo_d.get(cap), lo, nd * 8, cudaMemcpyHostToDevice, st), "H2D");
  ck(memcpy_counted(c->hi_d.get(cap), hi, nd * 8, cudaMemcpyHostToDevice, st), "H2D");
  if (warm != nullptr) {
    std::vector<float> w32(nd);
    for (size_t i = 0; i < nd; ++i) w32[i] = static_cast<float>(warm[i]);
    ck(memcpy_counted(c->warm_f.get(cap), w32.data(), nd * 4, cudaMemcpyHostToDevice, st), "H2D");
  }
}

void search_run(bp_ctx* c, bp::SearchArgs& a, const bp_search_config& cfg) {
  const Compiled& cp = c->comp;
  const int n = a.n, d = a.d;
  cudaStream_t st = c->stream;
  const long long nstat = static_cast<long long>(n) * cp.o.H * cp.o.SP;
  const long long nstat_cap = static_cast<long long>(std::max(n, c->reserve_boxes)) * cp.o.H * cp.o.SP;
  int* smin = c->stat_min.get(static_cast<size_t>(std::max<long long>(nstat_cap, 1)));
  int* smax = c->stat_max.get(static_cast<size_t>(std::max<long long>(nstat_cap, 1)));
  fill_int(smin, nstat, bp::enc_f_host(INFINITY), st);
  fill_int(smax, nstat, bp::enc_f_host(-INFINITY), st);
  float* ufh = c->uf_hist.get(static_cast<size_t>(std::max(n, c->reserve_boxes)) * cfg.iterations);
  ck(bp::launch_search_init(a, st), "search init");
  ++c->launches;
  a.cur = 0;
  const long long n_rows = static_cast<long long>(n) * a.rows;
  if (a.method == 2) a.grad = c->grad.get(static_cast<size_t>(std::max(n, c->reserve_boxes)) * a.rows * d);
  for (int it = 0; it < cfg.iterations; ++it) {
    a.iter = it;
    if (a.method != 2 || it == 0) ck(bp::launch_sample(a, c->sms, st), "sample");
    c->rollout(a.actions, const_cast<float*>(a.costs), nullptr, smin, smax, a.failed, n_rows, a.rows);
    ck(bp::launch_search_update(a, st), "search update");
    if (a.method == 2 && it + 1 < cfg.iterations) {  // gradient of the consumed points, projected step
      float* g = const_cast<float*>(a.grad);
      if (cp.synth) {
        ck(bp::launch_synthetic_gradient(a.actions, g, n_rows * d, st), "gradient launch");
      } else {
        const long long per = static_cast<long long>(cp.o.H) * cp.o.ks;
        const long long chunk = std::max<long long>(1024, std::min<long long>(n_rows, (256ll << 20) / (8 * per)));
        double* ckpt = c->grad_ckpt.get(static_cast<size_t>(chunk * per));
        for (long long r0 = 0; r0 < n_rows; r0 += chunk)
          ck(bp::launch_gradient(c->dev(), a.actions + r0 * d, g + r0 * d, ckpt, std::min(chunk, n_rows - r0), st),
             "gradient launch");
      }
      ck(bp::launch_gd_step(a, c->sms, st), "gd step");
      c->launches += 2;
    }
    ck(memcpy_counted(ufh + static_cast<size_t>(it) * n, a.uf, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToDevice, st), "D2D");
    c->launches += 2;
    a.cur ^= 1;
  }
  c->cur = a.cur;
  c->searched = true;
  c->last = a;
  c->h_failed.assign(static_cast<size_t>(n), 0);
  ck(memcpy_counted(c->h_failed.data(), a.failed, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
  c->boxes_searched += n;  // pageable D2H: the flags are on the host now
  for (int i = 0; i < n; ++i) c->boxes_failed += c->h_failed[static_cast<size_t>(i)] != 0;
}

void search_harvest(bp_ctx* c, const bp::SearchArgs& a, const bp_search_config& cfg, std::vector<Report>* out) {
  const int n = a.n, d = a.d;
  const size_t nd = static_cast<size_t>(n) * d;
  cudaStream_t st = c->stream;
  float* ufh = c->uf_hist.p;
  float* uf = c->h_uf.get(static_cast<size_t>(n));
  float* best = c->h_best.get(nd);
  float* hist = c->h_hist.get(static_cast<size_t>(n) * cfg.iterations);
  int* cnt = c->h_cnt.get(static_cast<size_t>(n));
  ck(memcpy_counted(uf, a.uf, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
  ck(memcpy_counted(best, a.best, nd * 4, cudaMemcpyDeviceToHost, st), "D2H");
  ck(memcpy_counted(cnt, a.top_cnt, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
  ck(memcpy_counted(hist, ufh, static_cast<size_t>(n) * cfg.iterations * 4, cudaMemcpyDeviceToHost, st), "D2H");
  // only the filled part of each top list crosses: counts first, then per-box extents
  ck(cudaStreamSynchronize(st), "sync");
  const size_t tk = static_cast<size_t>(n) * a.top_cap;
  float* tv = c->h_tv.get(tk);
  float* ta = c->h_ta.get(tk * d);
  {
    int kmax = 0;
    for (int i = 0; i < n; ++i) kmax = std::max(kmax, cnt[i]);
    if (kmax == a.top_cap) {
      ck(memcpy_counted(tv, a.top_val[a.cur], tk * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(ta, a.top_act[a.cur], tk * d * 4, cudaMemcpyDeviceToHost, st), "D2H");
    } else if (kmax > 0) {  // 2D copies of the first kmax entries of every box
      ck(cudaMemcpy2DAsync(tv, static_cast<size_t>(a.top_cap) * 4, a.top_val[a.cur], static_cast<size_t>(a.top_cap) * 4,
                           static_cast<size_t>(kmax) * 4, static_cast<size_t>(n), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaMemcpy2DAsync(ta, static_cast<size_t>(a.top_cap) * d * 4, a.top_act[a.cur],
                           static_cast<size_t>(a.top_cap) * d * 4, static_cast<size_t>(kmax) * d * 4, static_cast<size_t>(n),
                           cudaMemcpyDeviceToHost, st), "D2H");
      g_d2h += static_cast<int64_t>(n) * kmax * (d + 1) * 4;
    }
    ck(cudaStreamSynchronize(st), "sync");
  }
  out->assign(static_cast<size_t>(n), Report());
  parallel_for(n, [&](int i) {
    Report& r = (*out)[static_cast<size_t>(i)];
    if (c->h_failed[static_cast<size_t>(i)]) {
      r.ok = false;
      r.error = "evaluate: non-finite objective value (malformed weights?)";
      return;
    }
    r.uf = uf[i];
    r.best.assign(best + static_cast<size_t>(i) * d, best + static_cast<size_t>(i + 1) * d);
    const int k = cnt[i];
    r.top_val.assign(tv + static_cast<size_t>(i) * a.top_cap, tv + static_cast<size_t>(i) * a.top_cap + k);
    r.top_act.assign(ta + static_cast<size_t>(i) * a.top_cap * d, ta + (static_cast<size_t>(i) * a.top_cap + k) * d);
    r.samples = static_cast<int64_t>(cfg.iterations) * a.rows;
    r.uf_history.resize(static_cast<size_t>(cfg.iterations));
    r.samples_history.resize(static_cast<size_t>(cfg.iterations));
    for (int it = 0; it < cfg.iterations; ++it) {
      r.uf_history[static_cast<size_t>(it)] = hist[static_cast<size_t>(it) * n + i];
      r.samples_history[static_cast<size_t>(it)] = static_cast<int64_t>(it + 1) * a.rows;
    }
  });
}

void device_batch_search(bp_ctx* c, int n, const double* lo, const double* hi, const double* warm,
                         const bp_search_config& cfg, std::vector<Report>* out, const int64_t* seed_index = nullptr) {
  place_host_boxes(c, n, lo, hi, warm);
  bp::SearchArgs a = search_setup(c, n, cfg, seed_index, warm != nullptr);
  search_run(c, a, cfg);
  if (out == nullptr) {
    ck(cudaStreamSynchronize(c->stream), "sync");
    return;
  }
  search_harvest(c, a, cfg, out);
}

void device_batch_bound(bp_ctx* c, int mode, int alpha, double* lf_out) {
  if (!c->searched) fail(BP_LOGIC, "bound: no batch searched");
  const Compiled& cp = c->comp;
  const int n = c->n;
  if (cp.synth) {  // SeparableBounder (bab.cpp:70-83): exact, needs no search statistics
    double* lf = c->lf.get(static_cast<size_t>(std::max(n, c->reserve_boxes)));
    if (c->timing) ck(cudaEventRecord(c->ev0, c->stream), "event");
    ck(bp::launch_separable_bound(c->lo_d.p, c->hi_d.p, n, cp.d, c->d_da.p, static_cast<int>(cp.da.size()), nullptr,
                                  lf, c->stream), "separable bound launch");
    if (c->timing) ck(cudaEventRecord(c->ev1, c->stream), "event");
    ++c->launches;
    ck(memcpy_counted(lf_out, lf, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (c->timing) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event");
      c->bound_ms += ms;
    }
    return;
  }
  const long long nstat_cap = static_cast<long long>(std::max(n, c->reserve_boxes)) * cp.o.H * cp.o.SP;
  std::vector<int> use(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) use[static_cast<size_t>(i)] = c->h_failed[static_cast<size_t>(i)] ? 0 : 1;
  int* du = c->use_flags.get(static_cast<size_t>(std::max(n, c->reserve_boxes)));
  ck(memcpy_counted(du, use.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  bp::BoundArgs a{c->lo_d.p, c->hi_d.p, c->stat_min.p, c->stat_max.p, du,
                  c->ivl_lo.get(static_cast<size_t>(std::max<long long>(nstat_cap, 1))),
                  c->ivl_hi.get(static_cast<size_t>(std::max<long long>(nstat_cap, 1))),
                  c->lf.get(static_cast<size_t>(std::max(n, c->reserve_boxes))), mode, alpha, -1, 0, 0, 0, 0};
  if (c->timing) ck(cudaEventRecord(c->ev0, c->stream), "event");
  if (mode == BP_BOUND_FULL_CROWN) {
    // crown_node_bounds (crown.cpp:379-412): a backward pass per recorded node in
    // ascending graph order -- per step the MLP pre-activations by layer, x_t, u_t,
    // p_t, then the cost-op values in op order -- one CTA per (subdomain, row), each
    // node's bounds written before any later pass reads them; hinge outputs enclosed
    // from their argument's bounds.  Then the output pass without a stop set.
    for (int t = 0; t < cp.o.H; ++t)
      for (size_t k = 0; k < cp.slot_kind.size(); ++k) {
        bp::BoundArgs na = a;
        const int kind = cp.slot_kind[k], idx = cp.slot_index[k];
        na.start_t = t;
        na.start_index = idx;
        na.start_dim = cp.slot_dim[k];
        na.start_slot = cp.slot_off[k];
        na.start_kind = kind == 0 ? 0 : kind == 1 ? 1 : kind == 2 ? 2 : kind == 3 ? 3 : 4;
        if (kind == 4 && cp.o.ops[idx].kind == BP_OP_HINGE) {
          na.start_dim = n;
          ck(bp::launch_hinge_bounds(c->dev(), na, t, idx, c->stream), "hinge bounds launch");
        } else {
          ck(bp::launch_bound(c->dev(), na, n, c->stream), "crown node pass launch");
        }
        ++c->launches;
      }
  }
  ck(bp::launch_bound(c->dev(), a, n, c->stream), "bound launch");
  if (c->timing) ck(cudaEventRecord(c->ev1, c->stream), "event");
  ++c->launches;
  ck(memcpy_counted(lf_out, a.lf, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  if (c->timing) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event");
    c->bound_ms += ms;
  }
}

}  // namespace

namespace {

uint64_t mix_seed(uint64_t master, uint64_t salt) {  // rng.cpp:37-42
  uint64_t z = master + 0x9E3779B97F4A7C15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace

// Deterministic stream of the reference Rng (rng.hpp:12-35): mt19937_64 bits,
// 53-bit uniform, Box-Muller normal with a cached spare.
struct bp_rng {
  std::mt19937_64 gen;
  bool has_spare = false;
  double spare = 0.0;
  explicit bp_rng(uint64_t s) : gen(s) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1, u2;
    do {
      u1 = uniform();
    } while (u1 <= 0.0);
    u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

struct bp_result {
  double uf = std::numeric_limits<double>::infinity();
  std::vector<double> best;
  double min_lf = -std::numeric_limits<double>::infinity();
  bool certified = false;
  std::vector<bp_trace_row> trace;
  int64_t samples = 0;
  int iterations = 0;
  std::string stop_reason;
};

namespace {

// pick_out (bab.cpp:85-153) over pool metadata; returns pool indices in pick order.
std::vector<int> pick_indices(const bp_pool_meta* recs, int total, int n, double eta, double temperature, bp_rng& rng) {
  // pick_out (bab.cpp:85-153), bit-exact: the greedy round(eta n) lowest (uf, index), then n - n1
  // softmax picks over the rest in (uf, index) order with w = exp(-((lf - lo) / (hi - lo)) / T),
  // (lo, hi) over the remaining finite lf, u = uniform() * (sequential sum of w) and the first record
  // whose sequential prefix sum exceeds u.  The same arithmetic, organised for large pools:
  //  * (lo, hi) from a sorted multiset of the remaining finite lf (O(log N) per pick);
  //  * the weights are recomputed only when (lo, hi) moved (on host threads when the pool is
  //    large: each w_i is the same std::exp expression), the prefix sums from the removed position
  //    onward (the running sum in the reference's order), the selection by binary search on them.
  n = std::min(n, total);
  if (n <= 0) return {};
  std::vector<std::pair<double, int>> key(static_cast<size_t>(total));  // (uf, index): the reference's order
  for (int i = 0; i < total; ++i) key[static_cast<size_t>(i)] = {recs[i].uf, i};
  std::sort(key.begin(), key.end());
  const int n1 = std::clamp(static_cast<int>(std::llround(eta * n)), 0, n);
  std::vector<int> chosen(static_cast<size_t>(n1));
  for (int i = 0; i < n1; ++i) chosen[static_cast<size_t>(i)] = key[static_cast<size_t>(i)].second;
  std::vector<int> rem(static_cast<size_t>(total - n1));
  for (size_t i = 0; i < rem.size(); ++i) rem[i] = key[static_cast<size_t>(n1) + i].second;
  if (n == n1) return chosen;
  const double temp = std::max(temperature, 1e-12);
  // (lo, hi) over the remaining finite lf: the finite lf sorted once, two cursors skipping removed ones
  std::vector<std::pair<double, int>> by_lf;  // (lf, rem position)
  by_lf.reserve(rem.size());
  for (size_t i = 0; i < rem.size(); ++i)
    if (std::isfinite(recs[rem[i]].lf)) by_lf.push_back({recs[rem[i]].lf, static_cast<int>(i)});
  std::sort(by_lf.begin(), by_lf.end());
  size_t lo_c = 0, hi_c = by_lf.size();  // remaining finite records are within [lo_c, hi_c)
  // removed records stay in place with weight 0: adding +0.0 leaves every running sum bit for bit
  // as the reference's sum over the remaining records, and a removed position can never be the
  // first prefix above u (its prefix equals its predecessor's)
  const size_t m = rem.size();
  std::vector<double> w(m), pre(m);
  std::vector<char> alive(m, 1);
  size_t last_alive = m - 1;
  double w_lo = std::numeric_limits<double>::quiet_NaN(), w_hi = w_lo;
  bool w_deg = false, have_w = false;
  size_t dirty = 0;  // prefix sums valid below this position
  for (int need = n - n1; need > 0; --need) {
    while (lo_c < hi_c && !alive[static_cast<size_t>(by_lf[lo_c].second)]) ++lo_c;
    while (hi_c > lo_c && !alive[static_cast<size_t>(by_lf[hi_c - 1].second)]) --hi_c;
    const double lo = lo_c < hi_c ? by_lf[lo_c].first : std::numeric_limits<double>::infinity();
    const double hi = lo_c < hi_c ? by_lf[hi_c - 1].first : -std::numeric_limits<double>::infinity();
    const bool degenerate = !(hi > lo);
    if (!have_w || degenerate != w_deg || (!degenerate && (lo != w_lo || hi != w_hi))) {
      auto fill = [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
          if (!alive[i]) {
            w[i] = 0.0;
            continue;
          }
          double scaled = 0.5;
          if (!degenerate) {
            const double lf = recs[rem[i]].lf;
            scaled = std::isfinite(lf) ? (lf - lo) / (hi - lo) : (lf < 0.0 ? 0.0 : 1.0);
          }
          w[i] = degenerate ? 1.0 : std::exp(-scaled / temp);
        }
      };
      const int nt = m >= 32768 ? std::min(host_threads(), 16) : 1;
      if (nt <= 1) {
        fill(0, m);
      } else {
        std::vector<std::thread> th;
        for (int q = 0; q < nt; ++q) th.emplace_back(fill, m * q / nt, m * (q + 1) / nt);
        for (auto& x : th) x.join();
      }
      w_lo = lo;
      w_hi = hi;
      w_deg = degenerate;
      have_w = true;
      dirty = 0;
    }
    double acc = dirty == 0 ? 0.0 : pre[dirty - 1];
    for (size_t i = dirty; i < m; ++i) pre[i] = acc = acc + w[i];
    const double u = rng.uniform() * pre[m - 1];
    // first position with u < pre[i]; none: the last remaining record (the reference's fallback)
    size_t sel = static_cast<size_t>(std::upper_bound(pre.begin(), pre.end(), u) - pre.begin());
    if (sel >= m) sel = last_alive;
    const int idx = rem[sel];
    chosen.push_back(idx);
    alive[sel] = 0;
    w[sel] = 0.0;  // the other records' weights stand unless lo / hi move
    while (last_alive > 0 && !alive[last_alive]) --last_alive;
    dirty = sel;
  }
  return chosen;
}

// Device pool slab (pool.cu): the payload of every record this rank owns -- box,
// incumbent action, top-sample list -- one slot per record, with a host free list.
// Slots come in fixed-size chunks (>= 256 MB or 4096 slots each) that are never moved
// or freed while the planner runs, so the pool grows without copies or device-wide
// synchronisation; the chunks go back to the context when the planner ends and the
// next plan with the same geometry reuses them.
struct DevPool {
  static constexpr int kMaxChunks = 1 << 16;
  bp_ctx* ctx;  // chunk cache (null: chunks are freed)
  int d, K, shift = 4;
  size_t o_lo = 0, o_hi = 0, o_best = 0, o_val = 0, o_act = 0, o_n = 0, o_has = 0, chunk_bytes = 0;
  std::vector<unsigned char*> chunks;
  DBuf<unsigned char*> table;
  int used = 0;
  std::vector<int> free_slots;
  DevPool(bp_ctx* c, int d_, int K_) : ctx(c), d(d_), K(K_) {
    const size_t sd = static_cast<size_t>(d), sk = static_cast<size_t>(K);
    const size_t slot_bytes = 20 * sd + 4 * sk + 4 * sk * sd + 8;
    while (shift < 12 && (slot_bytes << shift) < (size_t{256} << 20)) ++shift;  // >= 256 MB: few cudaMallocs per plan
    const size_t per = size_t{1} << shift;
    auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
    o_hi = o_lo + al(per * sd * 8);
    o_best = o_hi + al(per * sd * 8);
    o_val = o_best + al(per * sd * 4);
    o_act = o_val + al(per * sk * 4);
    o_n = o_act + al(per * sk * sd * 4);
    o_has = o_n + al(per * 4);
    chunk_bytes = o_has + al(per * 4);
    table.get(kMaxChunks);
  }
  DevPool(const DevPool&) = delete;
  DevPool& operator=(const DevPool&) = delete;
  ~DevPool() {
    if (ctx != nullptr && (ctx->slab_d != d || ctx->slab_K != K)) {
      for (unsigned char* p : ctx->slab_spare) cudaFree(p);
      ctx->slab_spare.clear();
      ctx->slab_d = d;
      ctx->slab_K = K;
    }
    for (unsigned char* p : chunks) {
      if (ctx != nullptr) ctx->slab_spare.push_back(p);
      else cudaFree(p);
    }
    // keep at most two spare chunks for the next plan: one large plan must not pin its peak pool
    // footprint for the context's lifetime
    while (ctx != nullptr && ctx->slab_spare.size() > 2) {
      cudaFree(ctx->slab_spare.back());
      ctx->slab_spare.pop_back();
    }
  }
  bp::PoolArgs args() const { return {d, K, shift, table.p, o_lo, o_hi, o_best, o_val, o_act, o_n, o_has}; }
  bp::PoolArgs host_args() const { return {d, K, shift, chunks.data(), o_lo, o_hi, o_best, o_val, o_act, o_n, o_has}; }
  void add_chunk(cudaStream_t st) {
    if (static_cast<int>(chunks.size()) == kMaxChunks) fail(BP_UNSUPPORTED, "subdomain pool: too many records");
    unsigned char* p = nullptr;
    if (ctx != nullptr && ctx->slab_d == d && ctx->slab_K == K && !ctx->slab_spare.empty()) {
      p = ctx->slab_spare.back();
      ctx->slab_spare.pop_back();
    } else if (cudaMalloc(&p, chunk_bytes) != cudaSuccess) {
      cudaGetLastError();  // out of memory: release the cached spares of another geometry and retry once
      if (ctx != nullptr)
        for (unsigned char* q : ctx->slab_spare) cudaFree(q);
      if (ctx != nullptr) ctx->slab_spare.clear();
      ck(cudaMalloc(&p, chunk_bytes), "cudaMalloc (subdomain pool chunk)");
    }
    chunks.push_back(p);
    ck(memcpy_counted(table.p + chunks.size() - 1, &chunks.back(), sizeof(p), cudaMemcpyHostToDevice, st), "H2D");
  }
  int alloc(cudaStream_t st) {
    if (!free_slots.empty()) {
      const int s = free_slots.back();
      free_slots.pop_back();
      return s;
    }
    if (static_cast<size_t>(used) == (chunks.size() << shift)) add_chunk(st);
    return used++;
  }
  void release(int s) {
    if (s >= 0) free_slots.push_back(s);
  }
};

// The iteration's per-child search inputs and routed top lists (local index order).
bp::StageArgs stage_buffers(bp_ctx* c, int n, int K) {
  const size_t nb = static_cast<size_t>(std::max({n, c->reserve_boxes, 1}));
  const size_t nd = nb * c->comp.d, nk = nb * K;
  return {c->lo_f.get(nd), c->hi_f.get(nd), c->warm_f.get(nd), c->lo_d.get(nd), c->hi_d.get(nd),
          c->st_val.get(nk), c->st_act.get(nk * c->comp.d), c->st_n.get(nb)};
}

// A pool record as every rank sees it: what pick_out, the retirement
// test, split's sample count, prune and the trace read.  The payload lives in the
// owner rank's device slab (slot).
struct Head {
  int64_t id;
  double lf, uf, log_vol, max_width;
  int owner;
  int depth;
  int64_t samples;
  int slot;  // the owner's slab slot
};

// plan() (bab.cpp:266-415) as a steppable object: the constructor runs the root
// search + bound, step() one pick -> split -> search -> bound -> merge -> prune
// iteration, finish() the result fields.  pick_out, the retirement test and prune run
// on the host over the heads (pick_out's softmax must use the reference's exp() to
// pick the same records); split and merge_report run on the device over the slab
// (pool.cu), so no top list crosses PCIe.
//
// Sharded over ranks: every rank holds the pool's heads in the same
// order and replays pick_out / retirement / prune / trace on them identically (the
// pick stream is the shared mt19937_64(mix_seed(seed, 1))).  Child k of an iteration
// (global pick order) is searched on rank k % world and owned there; the owner of its
// parent splits the parent and ships the child record there (fixed-size all-to-all);
// after search, bound and merge the children's heads and each rank's incumbent
// candidate are all-gathered.  One rank runs the same code with no exchange.
struct Planner {
  static constexpr int kHeadWords = 8;  // k, id, lf, uf, log_vol, max_width, samples, depth
  bp_ctx* c;
  bp_planner_config cfg;
  int d, K;
  std::chrono::steady_clock::time_point t0;
  std::vector<Head> pool;  // heads, pool order, identical on every rank
  DevPool slab;
  bp::StageArgs S{};
  bp_rng pick_rng;
  int64_t next_id = 1;
  double pruned_cum = 0.0;
  double retired_min_lf = std::numeric_limits<double>::infinity();
  bp_result result;
  std::string stop;
  int iter = 0;
  bool done = false;
  int64_t children_bounded = 0;  // subdomains searched + bounded so far (root included)
  int last_children = 0;
  // per-iteration scratch
  DBuf<bp::SplitTask> d_tasks;
  DBuf<int> d_axis, d_slots, d_unpack_dst, d_unpack_slot;
  DBuf<unsigned char> d_pack, d_recv;
  DBuf<float> d_uf;
  DBuf<double> d_maxw;
  HBuf<int> h_axis;
  HBuf<float> h_uf, h_best;
  HBuf<double> h_maxw;
  HBuf<unsigned char> h_pack;

  // Rank-local failures (a root search that failed on rank 0, a split on a parent's owner, a CUDA error in
  // one rank's search) are held until the next collective, which carries a status word, so every rank
  // raises the same error together instead of leaving its peers blocked in an all-gather / all-to-all.
  bp_status err_code = BP_OK;
  std::string err_msg;
  template <typename F>
  void local(F&& f) {
    if (err_code != BP_OK) return;
    try {
      f();
    } catch (const Failure& e) {
      err_code = e.code;
      err_msg = e.what();
    } catch (const std::exception& e) {
      err_code = BP_RUNTIME;
      err_msg = e.what();
    }
  }
  // status[r] = rank r's err_code (one entry for a single-source exchange: rank 0's)
  void raise_agreed(const std::vector<double>& status) {
    for (size_t r = 0; r < status.size(); ++r) {
      const int code = static_cast<int>(status[r]);
      if (code == BP_OK) continue;
      if (static_cast<int>(r) == rank() && err_code != BP_OK) fail(err_code, err_msg);
      fail(static_cast<bp_status>(code), "plan: rank " + std::to_string(r) + " failed (its error is reported there)");
    }
    if (err_code != BP_OK) fail(err_code, err_msg);
  }
  void agree_status() {  // a dedicated status all-gather (one word per rank); no collective with one rank
    const int W = world();
    if (W == 1) {
      if (err_code != BP_OK) fail(err_code, err_msg);
      return;
    }
    double mine = static_cast<double>(err_code);
    std::vector<double> all(static_cast<size_t>(W));
    if (c->exchange(c->exchange_user, &mine, sizeof(double), all.data()) != 0)
      fail(BP_NCCL, "exchange: status all-gather failed");
    raise_agreed(all);
  }
  int world() const { return c->world > 1 && c->exchange != nullptr ? c->world : 1; }
  int rank() const { return world() > 1 ? c->rank : 0; }
  // BP_STEP_PROFILE: host wall time per phase of step(), printed per iteration (dev aid)
  std::chrono::steady_clock::time_point ph_t;
  std::string ph_line;
  // NVTX ranges per planner phase (nsys / ncu --nvtx): pick_out, split, search+bound+merge,
  // gather, prune -- opened and closed at the same boundaries as the BP_STEP_PROFILE marks
  bool nv_open = false;
  void nvtx_phase(const char* done) {
    const char* next = nullptr;
    if (done == nullptr) next = "bab.pick_out";
    else if (std::strcmp(done, "pick") == 0) next = "bab.split";
    else if (std::strcmp(done, "split") == 0) next = "bab.search+bound+merge";
    else if (std::strcmp(done, "merge+bound") == 0) next = "bab.gather";
    else if (std::strcmp(done, "gather") == 0) next = "bab.prune";
    else if (std::strcmp(done, "prune") != 0) return;  // nested marks (setup, search): no range change
    if (nv_open) nvtxRangePop();
    nv_open = next != nullptr;
    if (nv_open) nvtxRangePushA(next);
  }
  void phase(const char* name) {
    nvtx_phase(name);
    static const bool on = std::getenv("BP_STEP_PROFILE") != nullptr;
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    if (name != nullptr) {
      char buf[64];
      std::snprintf(buf, sizeof(buf), " %s=%.2f", name, std::chrono::duration<double, std::milli>(now - ph_t).count());
      ph_line += buf;
    }
    ph_t = now;
  }

  double elapsed_ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  double current_min_lf() const {
    double m = retired_min_lf;
    for (const auto& r : pool) m = std::min(m, r.lf);
    return std::isfinite(m) || !pool.empty() ? m : result.uf;
  }
  void push_trace(int it, double selected_vol) {
    bp_trace_row row{};
    row.iter = it;
    row.uf = result.uf;
    row.min_lf = current_min_lf();
    row.pruned_vol = pruned_cum;
    row.selected_vol = selected_vol;
    row.pool_size = static_cast<int64_t>(pool.size());
    row.samples = result.samples;
    row.wall_ms = elapsed_ms();
    result.trace.push_back(row);
  }
  double prune() {  // bab.cpp:225-241
    double removed = 0.0;
    std::vector<Head> keep;
    keep.reserve(pool.size());
    for (auto& r : pool) {
      if (r.lf > result.uf) {
        removed += std::exp(r.log_vol);
        if (r.owner == rank()) slab.release(r.slot);
      } else {
        keep.push_back(r);
      }
    }
    pool = std::move(keep);
    return removed;
  }

  // Search, bound and merge_report of this rank's n staged children (keys = global
  // indices, the sampler stream key, so results do not depend on the rank a child runs
  // on); per child the bound, the merged incumbent value, the box's max width and the
  // samples taken.
  struct Out {
    std::vector<double> lf, maxw;
    std::vector<float> uf;
    std::vector<int64_t> samples;
  };
  Out search_bound_merge(const std::vector<int64_t>& keys, const std::vector<int>& slots, uint64_t seed) {
    const int n = static_cast<int>(keys.size());
    Out o;
    o.lf.assign(static_cast<size_t>(n), 0.0);
    o.maxw.assign(static_cast<size_t>(n), 0.0);
    o.uf.assign(static_cast<size_t>(n), INFINITY);
    o.samples.assign(static_cast<size_t>(n), 0);
    if (n == 0) return o;
    const auto ts = std::chrono::steady_clock::now();
    cudaStream_t st = c->stream;
    bp_search_config scfg = cfg.search;
    scfg.seed = seed;
    bp::SearchArgs a = search_setup(c, n, scfg, keys.data(), true);
    phase("setup");
    search_run(c, a, scfg);
    phase("search");
    std::vector<Report> log_reps;
    std::vector<double> log_lo, log_hi;
    if (c->plan_log_on) {  // the children's search reports and boxes, before the merge
      search_harvest(c, a, scfg, &log_reps);
      log_lo.resize(static_cast<size_t>(n) * d);
      log_hi.resize(static_cast<size_t>(n) * d);
      ck(cudaMemcpyAsync(log_lo.data(), S.lo_d, log_lo.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaMemcpyAsync(log_hi.data(), S.hi_d, log_hi.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
    }
    const size_t nb = static_cast<size_t>(std::max(n, c->reserve_boxes));  // no reallocation while ramping up
    int* ds = d_slots.get(nb);
    ck(memcpy_counted(ds, slots.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    float* du = d_uf.get(nb);
    double* dm = d_maxw.get(nb);
    ck(bp::launch_pool_merge(slab.args(), S, ds, n, a.top_val[a.cur], a.top_act[a.cur], a.top_cnt, a.uf, a.best, a.failed,
                             cfg.search.top_capacity, du, dm, st), "pool merge launch");
    ++c->launches;
    float* hu = h_uf.get(nb);
    double* hm = h_maxw.get(nb);
    ck(memcpy_counted(hu, du, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(memcpy_counted(hm, dm, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, st), "D2H");
    device_batch_bound(c, cfg.bound_mode, cfg.alpha, o.lf.data());  // synchronises the stream
    for (int i = 0; i < n; ++i) {
      o.uf[static_cast<size_t>(i)] = hu[i];
      o.maxw[static_cast<size_t>(i)] = hm[i];
      o.samples[static_cast<size_t>(i)] =
          c->h_failed[static_cast<size_t>(i)] ? 0 : static_cast<int64_t>(scfg.iterations) * a.rows;
    }
    c->search_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count();
    c->harvest_roll_events();
    if (c->plan_log_on)
      for (int i = 0; i < n; ++i)
        c->plan_log.push_back({iter,
                               std::vector<double>(log_lo.begin() + static_cast<std::ptrdiff_t>(i) * d,
                                                   log_lo.begin() + static_cast<std::ptrdiff_t>(i + 1) * d),
                               std::vector<double>(log_hi.begin() + static_cast<std::ptrdiff_t>(i) * d,
                                                   log_hi.begin() + static_cast<std::ptrdiff_t>(i + 1) * d),
                               o.lf[static_cast<size_t>(i)], log_reps[static_cast<size_t>(i)]});
    return o;
  }

  // The incumbent action of one owned record (FP32 on the device, FP64 in the result).
  std::vector<double> fetch_best(int slot) {
    float* hb = h_best.get(static_cast<size_t>(d));
    ck(memcpy_counted(hb, bp::pool_best(slab.host_args(), slot), static_cast<size_t>(d) * 4, cudaMemcpyDeviceToHost,
                      c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    return std::vector<double>(hb, hb + d);
  }

  Planner(bp_ctx* ctx, const bp_planner_config& config, const double* warm_start)
      : c(ctx), cfg(config), d(ctx->comp.d), K(std::max(config.search.top_capacity, 1)),
        t0(std::chrono::steady_clock::now()), slab(ctx, ctx->comp.d, std::max(config.search.top_capacity, 1)),
        pick_rng(mix_seed(config.seed, 1)) {
    if (cfg.batch <= 0) fail(BP_INVALID_ARGUMENT, "plan: batch must be positive");
    c->plan_log.clear();
    const int W = world();
    // at most 2 * batch children per step, ceil(2 * batch / W) of them on this rank
    c->reserve_boxes = std::max(c->reserve_boxes, (2 * cfg.batch + W - 1) / W);
    // the root's head + incumbent + status word (last)
    std::vector<double> h(static_cast<size_t>(kHeadWords + 2 + d + 1), 0.0);
    int root_slot = -1;
    if (rank() == 0) local([&] {  // the root is child 0 of the root search: rank 0 searches and owns it
      std::vector<double> lo(static_cast<size_t>(d)), hi(static_cast<size_t>(d));
      for (int t = 0; t < c->comp.o.H; ++t)
        for (int j = 0; j < c->comp.o.ka; ++j) {
          lo[static_cast<size_t>(t * c->comp.o.ka + j)] = c->comp.ulo[static_cast<size_t>(j)];
          hi[static_cast<size_t>(t * c->comp.o.ka + j)] = c->comp.uhi[static_cast<size_t>(j)];
        }
      cudaStream_t st = c->stream;
      root_slot = slab.alloc(st);
      S = stage_buffers(c, 1, K);
      place_host_boxes(c, 1, lo.data(), hi.data(), warm_start);  // the warm start seeds the root search only
      if (warm_start == nullptr) {
        const std::vector<float> nan(static_cast<size_t>(d), std::numeric_limits<float>::quiet_NaN());
        ck(memcpy_counted(S.warm_f, nan.data(), static_cast<size_t>(d) * 4, cudaMemcpyHostToDevice, st), "H2D");
      }
      ck(cudaMemsetAsync(S.n, 0, sizeof(int), st), "memset");
      ck(cudaMemcpyAsync(bp::pool_lo(slab.host_args(), root_slot), S.lo_d, static_cast<size_t>(d) * 8,
                         cudaMemcpyDeviceToDevice, st), "D2D");
      ck(cudaMemcpyAsync(bp::pool_hi(slab.host_args(), root_slot), S.hi_d, static_cast<size_t>(d) * 8,
                         cudaMemcpyDeviceToDevice, st), "D2D");
      Out o = search_bound_merge({0}, {root_slot}, mix_seed(cfg.seed, 0));
      if (c->h_failed[0]) fail(BP_RUNTIME, "plan: root search failed: evaluate: non-finite objective value (malformed weights?)");
      h[0] = 0.0;
      h[1] = 0.0;
      h[2] = o.lf[0];
      h[3] = o.uf[0];
      h[4] = 0.0;
      h[5] = o.maxw[0];
      h[6] = static_cast<double>(o.samples[0]);
      h[7] = 0.0;
      h[8] = o.uf[0];
      if (std::isfinite(o.uf[0])) {
        const std::vector<double> b = fetch_best(root_slot);
        std::copy(b.begin(), b.end(), h.begin() + kHeadWords + 2);
      }
    });
    h.back() = static_cast<double>(err_code);
    if (W > 1) {  // the root's head (and rank 0's status) from rank 0 to every rank
      std::vector<double> recv(h.size() * static_cast<size_t>(W));
      if (c->exchange(c->exchange_user, h.data(), h.size() * sizeof(double), recv.data()) != 0)
        fail(BP_NCCL, "exchange: allgather of the root head failed");
      std::copy(recv.begin(), recv.begin() + static_cast<std::ptrdiff_t>(h.size()), h.begin());  // rank 0's
    }
    raise_agreed({h.back()});
    pool.push_back(Head{0, h[2], h[3], 0.0, h[5], 0, 0, static_cast<int64_t>(h[6]), root_slot});
    result.uf = h[3];
    result.best.assign(h.begin() + kHeadWords + 2, h.end() - 1);
    result.samples = static_cast<int64_t>(h[6]);
    children_bounded = 1;
    last_children = 1;
    pruned_cum += prune();
    push_trace(0, 1.0);
  }

  // One BaB iteration; returns false (and records the stop reason) when the
  // termination checks of bab.cpp:343-358 end the run.
  bool step() {
    if (done) return false;
    if (result.uf <= cfg.target_objective) stop = "target";
    else if (pool.empty()) stop = "pool-exhausted";
    else if (iter >= cfg.max_iterations) stop = "max-iterations";
    else if (cfg.wall_clock_ms > 0.0 && elapsed_ms() >= cfg.wall_clock_ms) stop = "wall-clock";
    if (!stop.empty()) {
      done = true;
      return false;
    }
    ++iter;
    const int W = world(), R = rank();
    cudaStream_t st = c->stream;
    ph_line.clear();
    phase(nullptr);
    std::vector<bp_pool_meta> meta(pool.size());
    for (size_t i = 0; i < pool.size(); ++i) meta[i] = {pool[i].lf, pool[i].uf, pool[i].id, pool[i].log_vol};
    const std::vector<int> chosen = pick_indices(meta.data(), static_cast<int>(pool.size()), cfg.batch, cfg.eta, cfg.temperature, pick_rng);
    std::vector<char> taken(pool.size(), 0);
    std::vector<Head> picked;
    for (int idx : chosen) {
      taken[static_cast<size_t>(idx)] = 1;
      picked.push_back(pool[static_cast<size_t>(idx)]);
    }
    {
      std::vector<Head> keep;
      for (size_t i = 0; i < pool.size(); ++i)
        if (!taken[i]) keep.push_back(pool[i]);
      pool = std::move(keep);
    }
    double selected_vol = 0.0;
    for (const auto& r : picked) selected_vol += std::exp(r.log_vol);
    phase("pick");
    std::vector<Head> to_split;
    for (const Head& h : picked) {
      if (h.max_width <= cfg.min_width) {  // retired: too narrow to split
        retired_min_lf = std::min(retired_min_lf, h.lf);
        if (h.owner == R) slab.release(h.slot);
        continue;
      }
      to_split.push_back(h);
    }
    const int n_all = 2 * static_cast<int>(to_split.size());
    const int64_t base_id = next_id;  // child k gets id base_id + k (ids by pick order, as the serial loop)
    next_id += n_all;
    last_children = n_all;
    // this rank's children (k % W == R) in global order, with their slab slots
    std::vector<int64_t> keys;
    std::vector<int> li_of(static_cast<size_t>(n_all), -1);
    for (int k = 0; k < n_all; ++k)
      if (k % W == R) {
        li_of[static_cast<size_t>(k)] = static_cast<int>(keys.size());
        keys.push_back(k);
      }
    const int n_loc = static_cast<int>(keys.size());
    std::vector<int> slots(static_cast<size_t>(n_loc), -1);
    local([&] {
      for (int& s : slots) s = slab.alloc(st);
      S = stage_buffers(c, n_loc, K);
    });
    // split this rank's parents (one CTA each); shipped children packed by destination rank
    std::vector<std::vector<int64_t>> out_k(static_cast<size_t>(W));
    for (int i = 0; i < static_cast<int>(to_split.size()); ++i)
      if (to_split[static_cast<size_t>(i)].owner == R)
        for (int b = 0; b < 2; ++b) {
          const int64_t k = 2 * static_cast<int64_t>(i) + b;
          if (k % W != R) out_k[static_cast<size_t>(k % W)].push_back(k);
        }
    std::vector<int> pack_of(static_cast<size_t>(n_all), -1);
    int n_pack = 0;
    for (int r = 0; r < W; ++r)
      for (int64_t k : out_k[static_cast<size_t>(r)]) pack_of[static_cast<size_t>(k)] = n_pack++;
    std::vector<bp::SplitTask> tasks;
    for (int i = 0; i < static_cast<int>(to_split.size()); ++i) {
      const Head& p = to_split[static_cast<size_t>(i)];
      if (p.owner != R) continue;
      bp::SplitTask t{};
      t.parent = p.slot;
      for (int b = 0; b < 2; ++b) {
        const int64_t k = 2 * static_cast<int64_t>(i) + b;
        const int li = li_of[static_cast<size_t>(k)];
        t.key[b] = k;
        t.dst[b] = li;
        t.slot[b] = li >= 0 ? slots[static_cast<size_t>(li)] : -1;
        t.pack[b] = pack_of[static_cast<size_t>(k)];
      }
      // split's k (bab.cpp:160-165) before the clamp to the stored list
      t.k_round = cfg.split_rule != BP_SPLIT_SAMPLES ? -2
                  : p.samples > 0 ? static_cast<long long>(std::llround(cfg.top_percent / 100.0 * static_cast<double>(p.samples)))
                                  : -1;
      tasks.push_back(t);
    }
    const size_t rb = bp::pool_record_bytes(d, K);
    local([&] {
    unsigned char* dpack = n_pack > 0 ? d_pack.get(static_cast<size_t>(n_pack) * rb) : nullptr;
    if (!tasks.empty()) {
      const size_t tb = std::max<size_t>(tasks.size(), static_cast<size_t>(cfg.batch));
      bp::SplitTask* dt = d_tasks.get(tb);
      ck(memcpy_counted(dt, tasks.data(), tasks.size() * sizeof(bp::SplitTask), cudaMemcpyHostToDevice, st), "H2D");
      int* da = d_axis.get(tb);
      ck(bp::launch_pool_split(slab.args(), dt, static_cast<int>(tasks.size()), S, dpack, cfg.min_width, da, st),
         "pool split launch");
      ++c->launches;
      int* ha = h_axis.get(tb);
      ck(memcpy_counted(ha, da, tasks.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      for (size_t q = 0; q < tasks.size(); ++q)
        if (ha[q] < 0) fail(BP_INVALID_ARGUMENT, "split: no axis above the width floor");
    }
    });
    phase("split");
    agree_status();  // a split failure on a parent's owner raises on every rank before the all-to-all
    for (const Head& p : to_split)  // the parents' payload has been read by the split
      if (p.owner == R) slab.release(p.slot);
    if (W > 1 && n_all > 0) ship_children(to_split, n_pack, li_of, slots);
    if (n_all > 0) {
      Out o;
      local([&] { o = search_bound_merge(keys, slots, mix_seed(cfg.seed, static_cast<uint64_t>(iter) + 1)); });
      phase("merge+bound");
      gather_children(to_split, base_id, keys, slots, o);  // carries this rank's status
      phase("gather");
    }
    pruned_cum += prune();
    push_trace(iter, selected_vol);
    phase("prune");
    if (!ph_line.empty()) std::fprintf(stderr, "[step %d]%s\n", iter, ph_line.c_str());
    return true;
  }

  // Child records from their parent's owner to their search rank: a fixed-size
  // all-to-all whose counts every rank derives from the replicated heads.
  void ship_children(const std::vector<Head>& to_split, int n_pack, const std::vector<int>& li_of,
                     const std::vector<int>& slots) {
    const int W = world(), R = rank();
    cudaStream_t st = c->stream;
    const size_t rb = bp::pool_record_bytes(d, K);
    std::vector<int64_t> sb(static_cast<size_t>(W), 0), rbts(static_cast<size_t>(W), 0);
    for (int i = 0; i < static_cast<int>(to_split.size()); ++i)
      for (int b = 0; b < 2; ++b) {
        const int64_t k = 2 * static_cast<int64_t>(i) + b;
        const int dst = static_cast<int>(k % W), src = to_split[static_cast<size_t>(i)].owner;
        if (src == R && dst != R) sb[static_cast<size_t>(dst)] += static_cast<int64_t>(rb);
        if (dst == R && src != R) rbts[static_cast<size_t>(src)] += static_cast<int64_t>(rb);
      }
    size_t r_total = 0;
    for (int r = 0; r < W; ++r) r_total += static_cast<size_t>(rbts[static_cast<size_t>(r)]);
    if (c->nccl) {  // device-direct: the split's pack buffer goes out as is, records land in d_recv
      unsigned char* dr = d_recv.get(std::max<size_t>(r_total, 1));
      c->nccl->alltoallv_dev(d_pack.p, sb.data(), dr, rbts.data());
      local([&] {
        const int n_in = static_cast<int>(r_total / rb);
        std::vector<double> keys(static_cast<size_t>(n_in));
        if (n_in > 0)  // each record's first word: the child's index in the iteration
          ck(cudaMemcpy2DAsync(keys.data(), sizeof(double), dr, rb, sizeof(double), static_cast<size_t>(n_in),
                               cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        unpack_children_dev(dr, keys, li_of, slots);
      });
      return;
    }
    unsigned char* send = h_pack.get(std::max<size_t>(static_cast<size_t>(n_pack) * rb, 1));
    local([&] {  // a failure here is carried to the heads all-gather; the all-to-all still runs
      if (n_pack > 0) {
        ck(memcpy_counted(send, d_pack.p, static_cast<size_t>(n_pack) * rb, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
      }
    });
    std::vector<unsigned char> recv(std::max<size_t>(r_total, 1));
    if (c->alltoallv == nullptr) fail(BP_NCCL, "exchange: no all-to-all hook for the sharded pool");
    if (c->alltoallv(c->exchange_user, send, sb.data(), recv.data(), rbts.data()) != 0)
      fail(BP_NCCL, "exchange: all-to-all of child records failed");
    local([&] { unpack_children(recv, r_total, li_of, slots); });
  }
  void unpack_children(const std::vector<unsigned char>& recv, size_t r_total, const std::vector<int>& li_of,
                       const std::vector<int>& slots) {
    cudaStream_t st = c->stream;
    const size_t rb = bp::pool_record_bytes(d, K);
    const int n_in = static_cast<int>(r_total / rb);
    if (n_in == 0) return;
    std::vector<double> keys(static_cast<size_t>(n_in));
    for (int q = 0; q < n_in; ++q) std::memcpy(&keys[static_cast<size_t>(q)], recv.data() + static_cast<size_t>(q) * rb, sizeof(double));
    unsigned char* dr = d_recv.get(r_total);
    ck(memcpy_counted(dr, recv.data(), r_total, cudaMemcpyHostToDevice, st), "H2D");
    unpack_children_dev(dr, keys, li_of, slots);
  }
  // received child records (device, one per key) into their local search slots
  void unpack_children_dev(unsigned char* dr, const std::vector<double>& keys, const std::vector<int>& li_of,
                           const std::vector<int>& slots) {
    cudaStream_t st = c->stream;
    const int n_in = static_cast<int>(keys.size());
    if (n_in == 0) return;
    std::vector<int> dst(static_cast<size_t>(n_in)), slot(static_cast<size_t>(n_in));
    for (int q = 0; q < n_in; ++q) {
      const double key = keys[static_cast<size_t>(q)];
      const int64_t k = static_cast<int64_t>(key);
      if (k < 0 || k >= static_cast<int64_t>(li_of.size()) || li_of[static_cast<size_t>(k)] < 0)
        fail(BP_NCCL, "exchange: child record for another rank");
      dst[static_cast<size_t>(q)] = li_of[static_cast<size_t>(k)];
      slot[static_cast<size_t>(q)] = slots[static_cast<size_t>(li_of[static_cast<size_t>(k)])];
    }
    int* dd = d_unpack_dst.get(static_cast<size_t>(n_in));
    int* ds = d_unpack_slot.get(static_cast<size_t>(n_in));
    ck(memcpy_counted(dd, dst.data(), static_cast<size_t>(n_in) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(ds, slot.data(), static_cast<size_t>(n_in) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(bp::launch_pool_unpack(slab.args(), S, dr, dd, ds, n_in, st), "pool unpack launch");
    ++c->launches;
  }

  // Every child's head in global order (all-gathered across ranks) appended to the
  // pool; the incumbent updated as the reference's sequential loop does
  // (bab.cpp:388-403): the first child holding the iteration's lowest value, if lower.
  void gather_children(const std::vector<Head>& to_split, int64_t base_id, const std::vector<int64_t>& keys,
                       const std::vector<int>& slots, const Out& o) {
    const int W = world(), R = rank();
    const int n_all = 2 * static_cast<int>(to_split.size());
    const int n_loc = static_cast<int>(keys.size());
    int cand = -1;  // this rank's lowest child (first in global order on ties)
    for (int i = 0; err_code == BP_OK && i < n_loc; ++i)
      if (std::isfinite(o.uf[static_cast<size_t>(i)]) && (cand < 0 || o.uf[static_cast<size_t>(i)] < o.uf[static_cast<size_t>(cand)]))
        cand = i;
    const int per_rank = (n_all + W - 1) / W;
    const size_t words = static_cast<size_t>(per_rank) * kHeadWords + 2 + static_cast<size_t>(d) + 1;  // + status
    std::vector<double> send(words, -1.0);
    send.back() = static_cast<double>(err_code);
    if (err_code == BP_OK) {
    for (int i = 0; i < n_loc; ++i) {
      double* h = send.data() + static_cast<size_t>(i) * kHeadWords;
      const Head& p = to_split[static_cast<size_t>(keys[static_cast<size_t>(i)] / 2)];
      h[0] = static_cast<double>(keys[static_cast<size_t>(i)]);
      h[1] = static_cast<double>(base_id + keys[static_cast<size_t>(i)]);
      h[2] = o.lf[static_cast<size_t>(i)];
      h[3] = o.uf[static_cast<size_t>(i)];
      h[4] = p.log_vol + std::log(0.5);
      h[5] = o.maxw[static_cast<size_t>(i)];
      h[6] = static_cast<double>(o.samples[static_cast<size_t>(i)]);
      h[7] = p.depth + 1;
    }
    double* cd = send.data() + static_cast<size_t>(per_rank) * kHeadWords;
    cd[0] = cand >= 0 ? o.uf[static_cast<size_t>(cand)] : INFINITY;
    cd[1] = cand >= 0 ? static_cast<double>(keys[static_cast<size_t>(cand)]) : -1.0;
    if (cand >= 0) local([&] {
      const std::vector<double> b = fetch_best(slots[static_cast<size_t>(cand)]);
      std::copy(b.begin(), b.end(), cd + 2);
    });
    send.back() = static_cast<double>(err_code);
    }
    std::vector<double> recv;
    if (W == 1) {
      recv = std::move(send);
    } else {
      recv.resize(words * static_cast<size_t>(W));
      if (c->exchange(c->exchange_user, send.data(), words * sizeof(double), recv.data()) != 0)
        fail(BP_NCCL, "exchange: allgather of child heads failed");
    }
    {
      std::vector<double> status(static_cast<size_t>(W));
      for (int r = 0; r < W; ++r) status[static_cast<size_t>(r)] = recv[static_cast<size_t>(r + 1) * words - 1];
      raise_agreed(status);
    }
    std::vector<const double*> by_k(static_cast<size_t>(n_all), nullptr);
    const double* best_cd = nullptr;
    for (int r = 0; r < W; ++r) {
      const double* blk = recv.data() + static_cast<size_t>(r) * words;
      for (int q = 0; q < per_rank; ++q) {
        const double* h = blk + static_cast<size_t>(q) * kHeadWords;
        if (h[0] < 0.0) continue;
        const int64_t k = static_cast<int64_t>(h[0]);
        if (k >= n_all || by_k[static_cast<size_t>(k)] != nullptr) fail(BP_NCCL, "exchange: inconsistent child heads");
        by_k[static_cast<size_t>(k)] = h;
      }
      const double* cr = blk + static_cast<size_t>(per_rank) * kHeadWords;
      if (cr[1] >= 0.0 && (best_cd == nullptr || cr[0] < best_cd[0] || (cr[0] == best_cd[0] && cr[1] < best_cd[1])))
        best_cd = cr;
    }
    for (int k = 0; k < n_all; ++k) {
      const double* h = by_k[static_cast<size_t>(k)];
      if (h == nullptr) fail(BP_NCCL, "exchange: missing child heads");
      const int owner = k % W;
      const int slot = owner == R ? slots[static_cast<size_t>(li_of_local(keys, k))] : -1;
      pool.push_back(Head{static_cast<int64_t>(h[1]), h[2], h[3], h[4], h[5], owner, static_cast<int>(h[7]),
                          static_cast<int64_t>(h[6]), slot});
      result.samples += static_cast<int64_t>(h[6]);
    }
    if (best_cd != nullptr && best_cd[0] < result.uf) {
      result.uf = best_cd[0];
      result.best.assign(best_cd + 2, best_cd + 2 + d);
    }
    children_bounded += n_all;
  }
  static int li_of_local(const std::vector<int64_t>& keys, int64_t k) {  // keys ascending
    return static_cast<int>(std::lower_bound(keys.begin(), keys.end(), k) - keys.begin());
  }

  void finish() {
    while (step()) {
    }
    result.min_lf = current_min_lf();
    result.certified = cfg.bound_mode != BP_BOUND_EMPIRICAL;
    result.iterations = iter;
    result.stop_reason = stop;
  }
};

void run_plan(bp_ctx* c, const bp_planner_config& cfg, const double* warm_start, bp_result& result) {
  Planner p(c, cfg, warm_start);
  p.finish();
  result = std::move(p.result);
}

void run_sample_only(bp_ctx* c, const bp_planner_config& cfg, const double* warm_start, bp_result& result) {
  // bab.cpp:417-454
  const int d = c->comp.d;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double> lo(static_cast<size_t>(d)), hi(static_cast<size_t>(d));
  for (int t = 0; t < c->comp.o.H; ++t)
    for (int j = 0; j < c->comp.o.ka; ++j) {
      lo[static_cast<size_t>(t * c->comp.o.ka + j)] = c->comp.ulo[static_cast<size_t>(j)];
      hi[static_cast<size_t>(t * c->comp.o.ka + j)] = c->comp.uhi[static_cast<size_t>(j)];
    }
  bp_search_config scfg = cfg.search;
  scfg.seed = mix_seed(cfg.seed, 0);
  std::vector<Report> reps;
  device_batch_search(c, 1, lo.data(), hi.data(), warm_start, scfg, &reps);
  c->harvest_roll_events();
  Report& rep = reps[0];
  if (!rep.ok) fail(BP_RUNTIME, "sample_only_plan: search failed: " + rep.error);
  const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  result.uf = rep.uf;
  result.best = rep.best;
  result.min_lf = -std::numeric_limits<double>::infinity();
  result.certified = false;
  result.samples = rep.samples;
  result.iterations = static_cast<int>(rep.uf_history.size());
  result.stop_reason = "sampler-budget";
  for (size_t i = 0; i < rep.uf_history.size(); ++i) {
    bp_trace_row row{};
    row.iter = static_cast<int>(i);
    row.uf = rep.uf_history[i];
    row.min_lf = -std::numeric_limits<double>::infinity();
    row.selected_vol = i == 0 ? 1.0 : 0.0;
    row.pool_size = 1;
    row.samples = rep.samples_history[i];
    row.wall_ms = i + 1 == rep.uf_history.size() ? wall : 0.0;
    result.trace.push_back(row);
  }
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

size_t bp_get_last_error(char* buf, size_t cap) {
  if (buf != nullptr && cap > 0) {
    std::strncpy(buf, g_last_error.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return g_last_error.size();
}

bp_status bp_init(int device, bp_ctx** out) {
  return guard([&] {
    if (out == nullptr) fail(BP_INVALID_ARGUMENT, "bp_init: null output");
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) fail(BP_INVALID_ARGUMENT, "bp_init: no such CUDA device");
    auto c = std::make_unique<bp_ctx>();
    c->device = device;
    c->use();
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) fail(BP_CUDA, "bp_init: device is not sm_100 class (B200 required)");
    c->sms = prop.multiProcessorCount;
    c->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
    if (const char* env = std::getenv("BP_ROLLOUT")) {
      const std::string e(env);
      c->path_mode = e == "simt" ? 1 : e == "tc1" ? 2 : e == "tc2" ? 3 : e == "tc3" ? 5 : 0;
    }
    ck(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own_stream;
    ck(cudaEventCreate(&c->ev0), "event");
    ck(cudaEventCreate(&c->ev1), "event");
    *out = c.release();
  });
}

bp_status bp_destroy(bp_ctx* ctx) {
  return guard([&] {
    if (ctx != nullptr) {
      cudaSetDevice(ctx->device);
      delete ctx;
    }
  });
}

bp_status bp_set_alltoall(bp_ctx* ctx, bp_alltoallv_fn fn) {
  return guard([&] {
    check_ctx(ctx);
    ctx->alltoallv = fn;
  });
}

bp_status bp_set_exchange(bp_ctx* ctx, int rank, int world, bp_exchange_fn fn, void* user) {
  return guard([&] {
    check_ctx(ctx);
    if (world < 1 || rank < 0 || rank >= world) fail(BP_INVALID_ARGUMENT, "bp_set_exchange: bad rank / world");
    if (world > 1 && fn == nullptr) fail(BP_INVALID_ARGUMENT, "bp_set_exchange: null exchange for world > 1");
    ctx->nccl.reset();  // host hooks replace a device-direct link
    ctx->rank = rank;
    ctx->world = world;
    ctx->exchange = fn;
    ctx->exchange_user = user;
  });
}

bp_status bp_nccl_unique_id(unsigned char* id) {
  return guard([&] {
    if (id == nullptr) fail(BP_INVALID_ARGUMENT, "bp_nccl_unique_id: null id");
    std::unique_ptr<NcclLink> L(NcclLink::open_lib());
    ncclUniqueId u;
    L->check(L->get_id(&u), "get unique id");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

bp_status bp_set_nccl(bp_ctx* ctx, int rank, int world, const unsigned char* id) {
  return guard([&] {
    check_ctx(ctx);
    if (world < 1 || rank < 0 || rank >= world) fail(BP_INVALID_ARGUMENT, "bp_set_nccl: bad rank / world");
    if (id == nullptr) fail(BP_INVALID_ARGUMENT, "bp_set_nccl: null id");
    ctx->use();
    std::unique_ptr<NcclLink> L(NcclLink::open_lib());
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    L->check(L->init(&L->comm, world, u, rank), "communicator init");  // collective over the ranks
    L->rank = rank;
    L->world = world;
    L->stream = &ctx->stream;
    ctx->nccl = std::move(L);
    ctx->rank = rank;
    ctx->world = world;
    ctx->exchange = nccl_allgather_host;  // heads and status words: staged all-gathers
    ctx->exchange_user = ctx->nccl.get();
    ctx->alltoallv = nullptr;  // child records go device to device (ship_children)
  });
}

bp_status bp_nccl_selftest(bp_ctx* ctx, int64_t bytes, int* ok) {
  return guard([&] {
    check_ctx(ctx);
    if (!ctx->nccl) fail(BP_INVALID_ARGUMENT, "bp_nccl_selftest: no NCCL link (bp_set_nccl)");
    if (bytes < 1) fail(BP_INVALID_ARGUMENT, "bp_nccl_selftest: bytes < 1");
    ctx->use();
    NcclLink& L = *ctx->nccl;
    const int W = L.world, R = L.rank;
    const size_t n = static_cast<size_t>(bytes);
    auto pat = [](int from, int to, size_t i) { return static_cast<unsigned char>((from * 131 + to * 31 + i * 7) & 0xff); };
    bool good = true;
    // all-gather through the host-staged hook the planner uses
    std::vector<unsigned char> mine(n), all(n * W);
    for (size_t i = 0; i < n; ++i) mine[i] = pat(R, R, i);
    if (nccl_allgather_host(&L, mine.data(), n, all.data()) != 0) fail(BP_NCCL, "selftest: all-gather");
    for (int r = 0; r < W; ++r)
      for (size_t i = 0; i < n; ++i) good = good && all[static_cast<size_t>(r) * n + i] == pat(r, r, i);
    // all-to-all-v device to device: rank R sends (r + 1) * n bytes to rank r
    std::vector<int64_t> sb(static_cast<size_t>(W)), rb(static_cast<size_t>(W));
    size_t st = 0, rt = 0;
    for (int r = 0; r < W; ++r) {
      sb[static_cast<size_t>(r)] = static_cast<int64_t>((r + 1) * n);
      rb[static_cast<size_t>(r)] = static_cast<int64_t>((R + 1) * n);
      st += (r + 1) * n;
      rt += (R + 1) * n;
    }
    std::vector<unsigned char> hs(st), hr(rt);
    for (int r = 0, o = 0; r < W; ++r)
      for (size_t i = 0; i < (r + 1) * n; ++i) hs[static_cast<size_t>(o++)] = pat(R, r, i);
    DBuf<unsigned char> ds, dr;
    ck(cudaMemcpyAsync(ds.get(st), hs.data(), st, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    L.alltoallv_dev(ds.p, sb.data(), dr.get(rt), rb.data());
    ck(cudaMemcpyAsync(hr.data(), dr.p, rt, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    for (int r = 0; r < W; ++r)
      for (size_t i = 0; i < (R + 1) * n; ++i) good = good && hr[static_cast<size_t>(r) * (R + 1) * n + i] == pat(r, R, i);
    if (ok) *ok = good ? 1 : 0;
  });
}

bp_status bp_set_stream(bp_ctx* ctx, void* stream) {
  return guard([&] {
    check_ctx(ctx);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->stream = stream != nullptr ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

bp_status bp_set_rollout_path(bp_ctx* ctx, int path, int* active) {
  return guard([&] {
    check_ctx(ctx);
    if ((path >= 0 && path <= 3) || path == 5) ctx->path_mode = path;
    if (active) *active = ctx->kernel();
  });
}

bp_status bp_rollout_info(bp_ctx* ctx, int* kernel, int* tiles_per_cta, int* rows_per_cta, int64_t* smem_bytes) {
  return guard([&] {
    check_ctx(ctx);
    const int k = ctx->kernel();
    const bp::DevObjective& o = ctx->comp.o;
    const int tiles = k == 3 ? o.tc2 : (k == 2 || k == 5) ? 1 : 0;  // k == 4: synthetic objective
    if (kernel) *kernel = k;
    if (tiles_per_cta) *tiles_per_cta = tiles;
    if (rows_per_cta) *rows_per_cta = k == 1 ? ctx->comp.R : 128 * tiles;
    if (smem_bytes)
      *smem_bytes = static_cast<int64_t>(k == 3   ? bp::rollout_tc2_smem(o)
                                         : k == 2 ? bp::rollout_tc_smem(o)
                                         : k == 5 ? bp::rollout_tc3_smem(o)
                                                  : ctx->comp.smem);
  });
}

bp_status bp_io_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = g_h2d.exchange(0);
  if (d2h) *d2h = g_d2h.exchange(0);
  return BP_OK;
}

// TMA tensor maps for the v2 CTA pair: the float arena as a [rows][32] fp32 tensor (128-byte rows,
// no swizzle: the images are pre-swizzled), one map per distinct per-CTA block height npad / 2.
// cuTensorMapEncodeTiled comes from the driver through cudaGetDriverEntryPoint (no -lcuda).  Without
// maps (no encoder, too many heights) n_tmap stays 0 and the pair forms relay the peer's arrivals.
void encode_tmaps(bp_ctx* ctx, Compiled& cp, float* arena) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (encode == nullptr) return;
  bp::DevObjective& o = cp.o;
  std::vector<int> heights;  // per-CTA block rows of the pair forms' weight entries
  auto add = [&](int h) {
    if (std::find(heights.begin(), heights.end(), h) == heights.end()) heights.push_back(h);
  };
  if (o.tc2_pair)
    for (int l = 0; l < o.L; ++l) add(o.tc_npad[l] / 2);
  if (o.tc3) {
    add(16);  // W0 N-blocks of 32 rows
    for (int j = 0; 256 * j < o.tc3_np[1]; ++j) add(std::min(256, o.tc3_np[1] - 256 * j) / 2);  // W1 chunks
    add(o.tc3_np[2] / 2);  // W2
  }
  if (heights.size() > 8) return;
  std::vector<CUtensorMap> maps(heights.size());
  const cuuint64_t dims[2] = {32, static_cast<cuuint64_t>(cp.fa.size() / 32)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t estr[2] = {1, 1};
  for (size_t i = 0; i < heights.size(); ++i) {
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(heights[i])};
    const CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, arena, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return;
  }
  unsigned char* dm = ctx->d_tmaps.get(maps.size() * sizeof(CUtensorMap));
  ck(memcpy_counted(dm, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, ctx->stream), "H2D");
  o.n_tmap = static_cast<int>(heights.size());
  for (size_t i = 0; i < heights.size(); ++i) o.tmap_h[i] = heights[i];
}

bp_status bp_load_objective(bp_ctx* ctx, const bp_objective_desc* desc) {
  return guard([&] {
    check_ctx(ctx);
    if (desc == nullptr) fail(BP_INVALID_ARGUMENT, "null objective");
    Compiled cp = compile(*desc);
    while (cp.fa.size() % 32) cp.fa.push_back(0.f);  // whole 128-byte rows for the tensor maps
    float* f = ctx->d_fa.get(cp.fa.size());
    double* dd = ctx->d_da.get(cp.da.size());
    int* iv = ctx->d_ia.get(cp.ia.size());
    ck(memcpy_counted(f, cp.fa.data(), cp.fa.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(memcpy_counted(dd, cp.da.data(), cp.da.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(memcpy_counted(iv, cp.ia.data(), cp.ia.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    cp.o.n_tmap = 0;
    if (cp.o.tc2_pair || cp.o.tc3) encode_tmaps(ctx, cp, f);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->comp = std::move(cp);
    ctx->loaded = true;
    ctx->searched = false;
  });
}

bp_status bp_load_synthetic(bp_ctx* ctx, int dim) {
  return guard([&] {
    check_ctx(ctx);
    Compiled cp = compile_synthetic(dim);
    cp.o.n_tmap = 0;
    float* f = ctx->d_fa.get(cp.fa.size());
    double* dd = ctx->d_da.get(cp.da.size());
    int* iv = ctx->d_ia.get(cp.ia.size());
    ck(memcpy_counted(f, cp.fa.data(), cp.fa.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(memcpy_counted(dd, cp.da.data(), cp.da.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(memcpy_counted(iv, cp.ia.data(), cp.ia.size() * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->comp = std::move(cp);
    ctx->loaded = true;
    ctx->searched = false;
  });
}

bp_status bp_stat_layout(bp_ctx* ctx, int* per_step, int* n_slots, int* kind, int* index, int* dim, int* offset, int cap) {
  return guard([&] {
    check_loaded(ctx);
    const Compiled& c = ctx->comp;
    *per_step = c.o.SP;
    *n_slots = static_cast<int>(c.slot_kind.size());
    for (int i = 0; i < *n_slots && i < cap; ++i) {
      kind[i] = c.slot_kind[static_cast<size_t>(i)];
      index[i] = c.slot_index[static_cast<size_t>(i)];
      dim[i] = c.slot_dim[static_cast<size_t>(i)];
      offset[i] = c.slot_off[static_cast<size_t>(i)];
    }
  });
}

bp_status bp_rollout(bp_ctx* ctx, int n_sub, int rows, const float* actions, float* costs, float* states, float* emp_lo,
                     float* emp_hi, int* nonfinite) {
  return guard([&] {
    check_loaded(ctx);
    if (n_sub < 0 || rows < 0) fail(BP_INVALID_ARGUMENT, "bp_rollout: negative sizes");
    const Compiled& cp = ctx->comp;
    const long long nr = static_cast<long long>(n_sub) * rows;
    if (nr == 0) return;
    for (long long i = 0; i < nr * cp.d; ++i)
      if (!std::isfinite(actions[i])) fail(BP_INVALID_ARGUMENT, "evaluate batch: non-finite values");
    cudaStream_t st = ctx->stream;
    float* da = ctx->r_actions.get(static_cast<size_t>(nr) * cp.d);
    float* dc = ctx->r_costs.get(static_cast<size_t>(nr));
    float* ds = states ? ctx->r_states.get(static_cast<size_t>(nr) * cp.o.H * cp.o.ks) : nullptr;
    const long long nstat = static_cast<long long>(n_sub) * cp.o.H * cp.o.SP;
    int* mn = ctx->r_min.get(static_cast<size_t>(std::max<long long>(nstat, 1)));
    int* mx = ctx->r_max.get(static_cast<size_t>(std::max<long long>(nstat, 1)));
    int* fl = ctx->use_flags.get(static_cast<size_t>(n_sub));
    fill_int(mn, nstat, bp::enc_f_host(INFINITY), st);
    fill_int(mx, nstat, bp::enc_f_host(-INFINITY), st);
    ck(cudaMemsetAsync(fl, 0, static_cast<size_t>(n_sub) * 4, st), "memset");
    ck(memcpy_counted(da, actions, static_cast<size_t>(nr) * cp.d * 4, cudaMemcpyHostToDevice, st), "H2D");
    ctx->rollout(da, dc, ds, mn, mx, fl, nr, rows);
    ck(memcpy_counted(costs, dc, static_cast<size_t>(nr) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (states) ck(memcpy_counted(states, ds, static_cast<size_t>(nr) * cp.o.H * cp.o.ks * 4, cudaMemcpyDeviceToHost, st), "D2H");
    std::vector<int> hmn, hmx, hfl(static_cast<size_t>(n_sub));
    if (emp_lo || emp_hi) {
      hmn.resize(static_cast<size_t>(nstat));
      hmx.resize(static_cast<size_t>(nstat));
      ck(memcpy_counted(hmn.data(), mn, static_cast<size_t>(nstat) * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(hmx.data(), mx, static_cast<size_t>(nstat) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    }
    ck(memcpy_counted(hfl.data(), fl, static_cast<size_t>(n_sub) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    ctx->harvest_roll_events();
    for (long long i = 0; i < nstat; ++i) {
      if (emp_lo) emp_lo[i] = bp::dec_f_host(hmn[static_cast<size_t>(i)]);
      if (emp_hi) emp_hi[i] = bp::dec_f_host(hmx[static_cast<size_t>(i)]);
    }
    if (nonfinite)
      for (int i = 0; i < n_sub; ++i) nonfinite[i] = hfl[static_cast<size_t>(i)];
  });
}

bp_status bp_batch_search(bp_ctx* ctx, int n_boxes, const double* lo, const double* hi, const double* warm,
                          const bp_search_config* cfg) {
  return guard([&] {
    check_loaded(ctx);
    if (cfg == nullptr || lo == nullptr || hi == nullptr) fail(BP_INVALID_ARGUMENT, "bp_batch_search: null argument");
    if (n_boxes <= 0) fail(BP_INVALID_ARGUMENT, "bp_batch_search: no boxes");
    device_batch_search(ctx, n_boxes, lo, hi, warm, *cfg, &ctx->reports);
    ctx->harvest_roll_events();
  });
}

bp_status bp_search_update(bp_ctx* ctx, int n, const bp_search_config* cfg, const double* lo, const double* hi,
                           int iter, const float* rows, const float* costs, float* mu, float* var, float* uf,
                           float* best, int* top_n, float* top_val, int* top_seq, float* top_act) {
  return guard([&] {
    check_loaded(ctx);
    ctx->use();
    if (cfg == nullptr || n <= 0 || lo == nullptr || hi == nullptr || rows == nullptr || costs == nullptr || mu == nullptr ||
        uf == nullptr || best == nullptr || top_n == nullptr || top_val == nullptr || top_seq == nullptr || top_act == nullptr)
      fail(BP_INVALID_ARGUMENT, "search_update: null argument");
    if (cfg->method == BP_SEARCH_GD) fail(BP_INVALID_ARGUMENT, "search_update: CEM or MPPI only");
    if (cfg->method == BP_SEARCH_CEM && var == nullptr) fail(BP_INVALID_ARGUMENT, "search_update: CEM needs var");
    bp_ctx* c = ctx;
    place_host_boxes(c, n, lo, hi, nullptr);
    bp::SearchArgs a = search_setup(c, n, *cfg, nullptr, false);
    cudaStream_t st = c->stream;
    ck(bp::launch_search_init(a, st), "search init");  // var floor (and placeholders overwritten below)
    const int d = a.d, R = a.rows, G = a.groups, K = a.top_cap;
    const size_t nd = static_cast<size_t>(n) * d, ng = nd * G, nk = static_cast<size_t>(n) * K;
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) ck(memcpy_counted(dst, src, bytes, cudaMemcpyHostToDevice, st), "H2D");
    };
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) ck(memcpy_counted(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    };
    for (int i = 0; i < n; ++i)
      if (top_n[i] < 0 || top_n[i] > K) fail(BP_INVALID_ARGUMENT, "search_update: top_n outside [0, top_capacity]");
    h2d(a.mu, mu, ng * 4);
    if (a.method == 0) h2d(a.var, var, ng * 4);
    h2d(a.uf, uf, static_cast<size_t>(n) * 4);
    h2d(a.best, best, nd * 4);
    h2d(a.top_cnt, top_n, static_cast<size_t>(n) * 4);
    h2d(a.top_val[0], top_val, nk * 4);
    h2d(const_cast<int*>(a.top_seq[0]), top_seq, nk * 4);
    h2d(a.top_act[0], top_act, nk * d * 4);
    h2d(a.actions, rows, static_cast<size_t>(n) * R * d * 4);
    h2d(const_cast<float*>(a.costs), costs, static_cast<size_t>(n) * R * 4);
    a.iter = iter;
    a.cur = 0;
    ck(bp::launch_search_update(a, st), "search update");
    c->launches += 2;
    d2h(mu, a.mu, ng * 4);
    if (a.method == 0) d2h(var, a.var, ng * 4);
    d2h(uf, a.uf, static_cast<size_t>(n) * 4);
    d2h(best, a.best, nd * 4);
    d2h(top_n, a.top_cnt, static_cast<size_t>(n) * 4);
    d2h(top_val, a.top_val[1], nk * 4);
    d2h(top_seq, a.top_seq[1], nk * 4);
    d2h(top_act, a.top_act[1], nk * d * 4);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

bp_status bp_report_summary(bp_ctx* ctx, double* uf, double* best, int64_t* samples, int* ok, int* n_top) {
  return guard([&] {
    check_loaded(ctx);
    const int d = ctx->comp.d;
    for (size_t i = 0; i < ctx->reports.size(); ++i) {
      const Report& r = ctx->reports[i];
      if (uf) uf[i] = r.uf;
      if (best)
        for (int j = 0; j < d; ++j) best[i * d + j] = r.best.empty() ? std::nan("") : r.best[static_cast<size_t>(j)];
      if (samples) samples[i] = r.samples;
      if (ok) ok[i] = r.ok ? 1 : 0;
      if (n_top) n_top[i] = static_cast<int>(r.top_val.size());
    }
  });
}

bp_status bp_report_top(bp_ctx* ctx, int box, double* values, double* actions, int cap) {
  return guard([&] {
    check_loaded(ctx);
    if (box < 0 || box >= static_cast<int>(ctx->reports.size())) fail(BP_INVALID_ARGUMENT, "bp_report_top: bad box");
    const Report& r = ctx->reports[static_cast<size_t>(box)];
    const int d = ctx->comp.d;
    for (size_t i = 0; i < r.top_val.size() && static_cast<int>(i) < cap; ++i) {
      values[i] = r.top_val[i];
      for (int j = 0; j < d; ++j) actions[i * d + j] = r.top_act[i * d + j];
    }
  });
}

bp_status bp_report_stats(bp_ctx* ctx, int box, float* emp_lo, float* emp_hi) {
  return guard([&] {
    check_loaded(ctx);
    if (!ctx->searched || box < 0 || box >= ctx->n) fail(BP_INVALID_ARGUMENT, "bp_report_stats: bad box");
    const size_t per = static_cast<size_t>(ctx->comp.o.H) * ctx->comp.o.SP;
    std::vector<int> mn(per), mx(per);
    ck(cudaMemcpy(mn.data(), ctx->stat_min.p + per * box, per * 4, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(mx.data(), ctx->stat_max.p + per * box, per * 4, cudaMemcpyDeviceToHost), "D2H");
    for (size_t i = 0; i < per; ++i) {
      if (emp_lo) emp_lo[i] = bp::dec_f_host(mn[i]);
      if (emp_hi) emp_hi[i] = bp::dec_f_host(mx[i]);
    }
  });
}

bp_status bp_batch_bound(bp_ctx* ctx, int mode, int alpha, double* lf) {
  return guard([&] {
    check_loaded(ctx);
    device_batch_bound(ctx, mode, alpha, lf);
  });
}

bp_status bp_bound_boxes(bp_ctx* ctx, int n_boxes, const double* lo, const double* hi, int mode, int alpha,
                         double* lf) {
  return guard([&] {
    check_loaded(ctx);
    if (n_boxes <= 0) fail(BP_INVALID_ARGUMENT, "bp_bound_boxes: no boxes");
    const int d = ctx->comp.d;
    const size_t nd = static_cast<size_t>(n_boxes) * d;
    for (size_t i = 0; i < nd; ++i)
      if (!(lo[i] <= hi[i]) || !std::isfinite(lo[i]) || !std::isfinite(hi[i]))
        fail(BP_INVALID_ARGUMENT, "BoxDomain: invalid bounds");
    ck(memcpy_counted(ctx->lo_d.get(nd), lo, nd * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ck(memcpy_counted(ctx->hi_d.get(nd), hi, nd * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    ctx->n = n_boxes;
    ctx->searched = true;  // boxes resident; no statistics
    ctx->h_failed.assign(static_cast<size_t>(n_boxes), 1);
    ctx->reports.clear();
    device_batch_bound(ctx, mode, alpha, lf);
  });
}

bp_status bp_gradient(bp_ctx* ctx, int64_t n_rows, const float* actions, float* grad) {
  return guard([&] {
    check_loaded(ctx);
    const Compiled& cp = ctx->comp;
    if (cp.o.net) fail(BP_UNSUPPORTED, "a bare network objective is bounded, not differentiated");
    if (n_rows <= 0) return;
    const size_t nd = static_cast<size_t>(n_rows) * cp.d;
    for (size_t i = 0; i < nd; ++i)
      if (!std::isfinite(actions[i])) fail(BP_INVALID_ARGUMENT, "gradient batch: non-finite values");
    cudaStream_t st = ctx->stream;
    float* da = ctx->r_actions.get(nd);
    float* dg = ctx->grad.get(nd);
    ck(memcpy_counted(da, actions, nd * 4, cudaMemcpyHostToDevice, st), "H2D");
    if (cp.synth) {
      ck(bp::launch_synthetic_gradient(da, dg, static_cast<long long>(nd), st), "gradient launch");
    } else {
      const long long per = static_cast<long long>(cp.o.H) * cp.o.ks;
      const long long chunk = std::max<long long>(1024, std::min<long long>(n_rows, (256ll << 20) / (8 * per)));
      double* ckpt = ctx->grad_ckpt.get(static_cast<size_t>(chunk * per));
      for (long long r0 = 0; r0 < n_rows; r0 += chunk)
        ck(bp::launch_gradient(ctx->dev(), da + r0 * cp.d, dg + r0 * cp.d, ckpt, std::min<long long>(chunk, n_rows - r0), st),
           "gradient launch");
    }
    ck(memcpy_counted(grad, dg, nd * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

bp_status bp_node_bounds(bp_ctx* ctx, double* lo, double* hi) {
  return guard([&] {
    check_loaded(ctx);
    const size_t n = static_cast<size_t>(ctx->n) * ctx->comp.o.H * ctx->comp.o.SP;
    if (n == 0) return;
    ck(memcpy_counted(lo, ctx->ivl_lo.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(memcpy_counted(hi, ctx->ivl_hi.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

bp_status bp_plan(bp_ctx* ctx, const bp_planner_config* cfg, const double* warm, int method_babnd, bp_result** out) {
  return guard([&] {
    check_loaded(ctx);
    if (cfg == nullptr || out == nullptr) fail(BP_INVALID_ARGUMENT, "bp_plan: null argument");
    auto r = std::make_unique<bp_result>();
    if (method_babnd)
      run_plan(ctx, *cfg, warm, *r);
    else
      run_sample_only(ctx, *cfg, warm, *r);
    *out = r.release();
  });
}

struct bp_planner {
  std::unique_ptr<Planner> p;
};

bp_status bp_planner_create(bp_ctx* ctx, const bp_planner_config* cfg, const double* warm, bp_planner** out) {
  return guard([&] {
    check_loaded(ctx);
    if (cfg == nullptr || out == nullptr) fail(BP_INVALID_ARGUMENT, "bp_planner_create: null argument");
    auto h = std::make_unique<bp_planner>();
    h->p = std::make_unique<Planner>(ctx, *cfg, warm);
    *out = h.release();
  });
}

bp_status bp_planner_step(bp_planner* h, int* stepped, int* children, int* pool_size) {
  return guard([&] {
    if (h == nullptr) fail(BP_INVALID_ARGUMENT, "null planner");
    h->p->c->use();
    const bool ok = h->p->step();
    if (stepped) *stepped = ok ? 1 : 0;
    if (children) *children = ok ? h->p->last_children : 0;
    if (pool_size) *pool_size = static_cast<int>(h->p->pool.size());
  });
}

bp_status bp_planner_finish(bp_planner* h, bp_result** out) {
  return guard([&] {
    if (h == nullptr || out == nullptr) fail(BP_INVALID_ARGUMENT, "null planner");
    h->p->c->use();
    h->p->finish();
    *out = new bp_result(h->p->result);
  });
}

bp_status bp_planner_destroy(bp_planner* h) {
  delete h;
  return BP_OK;
}

bp_status bp_result_summary(const bp_result* r, double* uf, double* min_lf, int* certified, int64_t* samples,
                            int* iterations, char* stop_reason, size_t cap, int* n_trace, int* d) {
  return guard([&] {
    if (r == nullptr) fail(BP_INVALID_ARGUMENT, "null result");
    if (uf) *uf = r->uf;
    if (min_lf) *min_lf = r->min_lf;
    if (certified) *certified = r->certified ? 1 : 0;
    if (samples) *samples = r->samples;
    if (iterations) *iterations = r->iterations;
    if (stop_reason && cap) {
      std::strncpy(stop_reason, r->stop_reason.c_str(), cap - 1);
      stop_reason[cap - 1] = 0;
    }
    if (n_trace) *n_trace = static_cast<int>(r->trace.size());
    if (d) *d = static_cast<int>(r->best.size());
  });
}

bp_status bp_result_best(const bp_result* r, double* best) {
  return guard([&] {
    if (r == nullptr) fail(BP_INVALID_ARGUMENT, "null result");
    std::copy(r->best.begin(), r->best.end(), best);
  });
}

bp_status bp_result_trace(const bp_result* r, bp_trace_row* rows, int cap) {
  return guard([&] {
    if (r == nullptr) fail(BP_INVALID_ARGUMENT, "null result");
    for (size_t i = 0; i < r->trace.size() && static_cast<int>(i) < cap; ++i) rows[i] = r->trace[i];
  });
}

bp_status bp_result_free(bp_result* r) {
  delete r;
  return BP_OK;
}

bp_status bp_set_plan_log(bp_ctx* ctx, int enable) {
  return guard([&] {
    check_ctx(ctx);
    ctx->plan_log_on = enable != 0;
    ctx->plan_log.clear();
  });
}

bp_status bp_plan_log_size(bp_ctx* ctx, int* n_children, int* total_top) {
  return guard([&] {
    check_ctx(ctx);
    int tot = 0;
    for (const auto& e : ctx->plan_log) tot += static_cast<int>(e.rep.top_val.size());
    if (n_children) *n_children = static_cast<int>(ctx->plan_log.size());
    if (total_top) *total_top = tot;
  });
}

bp_status bp_plan_log_get(bp_ctx* ctx, int* iter, double* lo, double* hi, double* lf, double* uf, double* best, int* n_top,
                          double* top_val, double* top_act, int64_t* samples, int* ok) {
  return guard([&] {
    check_ctx(ctx);
    const int d = ctx->comp.d;
    size_t off = 0;
    for (size_t c = 0; c < ctx->plan_log.size(); ++c) {
      const auto& e = ctx->plan_log[c];
      iter[c] = e.iter;
      std::copy(e.lo.begin(), e.lo.end(), lo + c * d);
      std::copy(e.hi.begin(), e.hi.end(), hi + c * d);
      lf[c] = e.lf;
      uf[c] = e.rep.ok ? e.rep.uf : INFINITY;
      for (int j = 0; j < d; ++j) best[c * d + j] = e.rep.ok && !e.rep.best.empty() ? e.rep.best[static_cast<size_t>(j)] : 0.0;
      n_top[c] = static_cast<int>(e.rep.top_val.size());
      for (size_t k = 0; k < e.rep.top_val.size(); ++k) {
        top_val[off + k] = e.rep.top_val[k];
        for (int j = 0; j < d; ++j) top_act[(off + k) * d + j] = e.rep.top_act[k * d + static_cast<size_t>(j)];
      }
      off += e.rep.top_val.size();
      samples[c] = e.rep.ok ? e.rep.samples : 0;
      ok[c] = e.rep.ok ? 1 : 0;
    }
  });
}

bp_status bp_search_counters(bp_ctx* ctx, int64_t* boxes, int64_t* failed) {
  return guard([&] {
    check_ctx(ctx);
    if (boxes) *boxes = ctx->boxes_searched;
    if (failed) *failed = ctx->boxes_failed;
    ctx->boxes_searched = ctx->boxes_failed = 0;
  });
}

bp_status bp_timing(bp_ctx* ctx, double* rollout_ms, int64_t* rollout_launches, double* bound_ms, double* search_ms,
                    int64_t* launches) {
  return guard([&] {
    check_ctx(ctx);
    if (rollout_ms) *rollout_ms = ctx->rollout_ms;
    if (rollout_launches) *rollout_launches = ctx->rollout_launches;
    if (bound_ms) *bound_ms = ctx->bound_ms;
    if (search_ms) *search_ms = ctx->search_ms;
    if (launches) *launches = ctx->launches;
    ctx->rollout_ms = ctx->bound_ms = ctx->search_ms = 0;
    ctx->rollout_launches = ctx->launches = 0;
  });
}

bp_status bp_rng_new(uint64_t seed, bp_rng** out) {
  return guard([&] { *out = new bp_rng(seed); });
}
bp_status bp_rng_free(bp_rng* r) {
  delete r;
  return BP_OK;
}
bp_status bp_rng_uniform(bp_rng* r, double* out) {
  return guard([&] { *out = r->uniform(); });
}
bp_status bp_rng_normal(bp_rng* r, double* out) {
  return guard([&] { *out = r->normal(); });
}
bp_status bp_rng_bits(bp_rng* r, uint64_t* out) {
  return guard([&] { *out = r->gen(); });
}
bp_status bp_rng_fill(bp_rng* r, int kind, int64_t n, double* out) {
  return guard([&] {
    if (r == nullptr) fail(BP_INVALID_ARGUMENT, "bp_rng_fill: null rng");
    for (int64_t i = 0; i < n; ++i) out[i] = kind == 0 ? r->uniform() : r->normal();
  });
}
uint64_t bp_mix_seed(uint64_t master, uint64_t salt) { return mix_seed(master, salt); }

bp_status bp_pick_out(const bp_pool_meta* pool, int n_pool, int n, double eta, double temperature, bp_rng* rng,
                      int* picked, int* n_picked) {
  return guard([&] {
    if (rng == nullptr) fail(BP_INVALID_ARGUMENT, "bp_pick_out: null rng");
    const std::vector<int> ch = pick_indices(pool, n_pool, n, eta, temperature, *rng);
    std::copy(ch.begin(), ch.end(), picked);
    *n_picked = static_cast<int>(ch.size());
  });
}

bp_status bp_pool_split(bp_ctx* ctx, int n, int d, int K, const double* lo, const double* hi, const int* n_top,
                        const float* top_val, const float* top_act, const int64_t* samples, double top_percent,
                        double min_width, int split_rule, int* axis, double* child_lo, double* child_hi, int* child_n,
                        float* child_val, float* child_act) {
  return guard([&] {  // split (bab.cpp:155-223) of n parents through pool.cu's split_kernel
    check_ctx(ctx);
    if (n <= 0 || d <= 0 || K <= 0) fail(BP_INVALID_ARGUMENT, "pool_split: n, d and K must be positive");
    for (int i = 0; i < n; ++i)
      if (n_top[i] < 0 || n_top[i] > K) fail(BP_INVALID_ARGUMENT, "pool_split: top list longer than K");
    cudaStream_t st = ctx->stream;
    DevPool slab(nullptr, d, K);
    for (int i = 0; i < 3 * n; ++i) slab.alloc(st);  // parents 0..n-1, children n..3n-1
    const bp::PoolArgs H = slab.host_args();
    const size_t sd = static_cast<size_t>(d), sk = static_cast<size_t>(K);
    for (int i = 0; i < n; ++i) {
      ck(memcpy_counted(bp::pool_lo(H, i), lo + i * sd, sd * 8, cudaMemcpyHostToDevice, st), "H2D");
      ck(memcpy_counted(bp::pool_hi(H, i), hi + i * sd, sd * 8, cudaMemcpyHostToDevice, st), "H2D");
      ck(memcpy_counted(bp::pool_n(H, i), n_top + i, 4, cudaMemcpyHostToDevice, st), "H2D");
      ck(memcpy_counted(bp::pool_val(H, i), top_val + i * sk, sk * 4, cudaMemcpyHostToDevice, st), "H2D");
      ck(memcpy_counted(bp::pool_act(H, i), top_act + i * sk * sd, sk * sd * 4, cudaMemcpyHostToDevice, st), "H2D");
    }
    DBuf<float> lo_f, hi_f, warm_f, sv, sa;
    DBuf<double> lo_d, hi_d;
    DBuf<int> sn, da;
    DBuf<bp::SplitTask> dt;
    const size_t cn = 2 * static_cast<size_t>(n);
    bp::StageArgs S{lo_f.get(cn * d), hi_f.get(cn * d), warm_f.get(cn * d), lo_d.get(cn * d), hi_d.get(cn * d),
                    sv.get(cn * K), sa.get(cn * K * d), sn.get(cn)};
    std::vector<bp::SplitTask> tasks(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      bp::SplitTask& t = tasks[static_cast<size_t>(i)];
      t.parent = i;
      for (int b = 0; b < 2; ++b) {
        t.slot[b] = n + 2 * i + b;
        t.dst[b] = 2 * i + b;
        t.pack[b] = -1;
        t.key[b] = 2 * i + b;
      }
      t.k_round = split_rule != BP_SPLIT_SAMPLES ? -2
                  : samples[i] > 0 ? static_cast<long long>(std::llround(top_percent / 100.0 * static_cast<double>(samples[i])))
                                   : -1;
    }
    ck(memcpy_counted(dt.get(tasks.size()), tasks.data(), tasks.size() * sizeof(bp::SplitTask), cudaMemcpyHostToDevice, st), "H2D");
    ck(bp::launch_pool_split(slab.args(), dt.p, n, S, nullptr, min_width, da.get(static_cast<size_t>(n)), st), "pool split launch");
    ck(memcpy_counted(axis, da.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    for (int i = 0; i < n; ++i)
      if (axis[i] < 0) fail(BP_INVALID_ARGUMENT, "split: no axis above the width floor");
    for (size_t q = 0; q < cn; ++q) {
      ck(memcpy_counted(child_lo + q * sd, bp::pool_lo(H, n + static_cast<int>(q)), sd * 8, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(child_hi + q * sd, bp::pool_hi(H, n + static_cast<int>(q)), sd * 8, cudaMemcpyDeviceToHost, st), "D2H");
    }
    ck(memcpy_counted(child_n, sn.p, cn * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(memcpy_counted(child_val, sv.p, cn * K * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(memcpy_counted(child_act, sa.p, cn * K * d * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

bp_status bp_pool_merge(bp_ctx* ctx, int n, int d, int K, int capacity, const int* a_n, const float* a_val,
                        const float* a_act, const int* b_n, const float* b_val, const float* b_act, const float* b_uf,
                        const float* b_best, const int* b_failed, int* out_n, float* out_val, float* out_act,
                        float* out_uf, int* has_best, float* out_best) {
  return guard([&] {  // merge_report (bab.cpp:245-262) of n records through pool.cu's merge_kernel
    check_ctx(ctx);
    if (n <= 0 || d <= 0 || K <= 0) fail(BP_INVALID_ARGUMENT, "pool_merge: n, d and K must be positive");
    for (int i = 0; i < n; ++i)
      if (a_n[i] < 0 || a_n[i] > K || b_n[i] < 0 || b_n[i] > K) fail(BP_INVALID_ARGUMENT, "pool_merge: list longer than K");
    cudaStream_t st = ctx->stream;
    const size_t nd = static_cast<size_t>(n) * d, nk = static_cast<size_t>(n) * K;
    DevPool slab(nullptr, d, K);
    for (int i = 0; i < n; ++i) slab.alloc(st);
    const bp::PoolArgs H = slab.host_args();
    const size_t sd = static_cast<size_t>(d), sk = static_cast<size_t>(K);
    for (int i = 0; i < n; ++i) {
      ck(cudaMemsetAsync(bp::pool_lo(H, i), 0, sd * 8, st), "memset");
      ck(cudaMemsetAsync(bp::pool_hi(H, i), 0, sd * 8, st), "memset");
    }
    DBuf<float> sv, sa, bv, ba, bu, bb, du;
    DBuf<int> sn, bn, bf, ds;
    DBuf<double> dm;
    bp::StageArgs S{};
    S.val = sv.get(nk);
    S.act = sa.get(nk * d);
    S.n = sn.get(static_cast<size_t>(n));
    ck(memcpy_counted(S.val, a_val, nk * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(S.act, a_act, nk * d * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(S.n, a_n, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(bv.get(nk), b_val, nk * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(ba.get(nk * d), b_act, nk * d * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(bn.get(static_cast<size_t>(n)), b_n, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(bu.get(static_cast<size_t>(n)), b_uf, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(bb.get(nd), b_best, nd * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(memcpy_counted(bf.get(static_cast<size_t>(n)), b_failed, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    std::vector<int> slots(static_cast<size_t>(n));
    std::iota(slots.begin(), slots.end(), 0);
    ck(memcpy_counted(ds.get(static_cast<size_t>(n)), slots.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st), "H2D");
    ck(bp::launch_pool_merge(slab.args(), S, ds.p, n, bv.p, ba.p, bn.p, bu.p, bb.p, bf.p, capacity,
                             du.get(static_cast<size_t>(n)), dm.get(static_cast<size_t>(n)), st), "pool merge launch");
    ck(memcpy_counted(out_uf, du.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st), "D2H");
    for (int i = 0; i < n; ++i) {
      ck(memcpy_counted(out_n + i, bp::pool_n(H, i), 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(out_val + i * sk, bp::pool_val(H, i), sk * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(out_act + i * sk * sd, bp::pool_act(H, i), sk * sd * 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(has_best + i, bp::pool_has(H, i), 4, cudaMemcpyDeviceToHost, st), "D2H");
      ck(memcpy_counted(out_best + i * sd, bp::pool_best(H, i), sd * 4, cudaMemcpyDeviceToHost, st), "D2H");
    }
    ck(cudaStreamSynchronize(st), "sync");
  });
}

bp_status bp_generate_model(uint64_t seed, int n_widths, const int* widths, double* params) {
  return guard([&] {  // model.cpp:136-158
    if (n_widths < 2) fail(BP_INVALID_ARGUMENT, "generate_model: need at least two widths");
    for (int i = 0; i < n_widths; ++i)
      if (widths[i] <= 0) fail(BP_INVALID_ARGUMENT, "generate_model: widths must be positive");
    bp_rng rng(seed);
    size_t off = 0;
    for (int li = 0; li + 1 < n_widths; ++li) {
      const int in = widths[li], out = widths[li + 1];
      const double a = std::sqrt(6.0 / (in + out));
      for (int r = 0; r < out * in; ++r) params[off++] = -a + (a - -a) * rng.uniform();
      for (int r = 0; r < out; ++r) params[off++] = -a + (a - -a) * rng.uniform();
    }
  });
}

}  // extern "C"
