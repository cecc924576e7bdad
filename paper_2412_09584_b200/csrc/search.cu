// search.cu -- K4 sampling (Philox), K3 incumbent + top-K merge and K5 CEM /
// MPPI refit: the device form of batch_search's per-box sampler loop.
//
// Restates run_cem (reference proj/src/search.cpp:87-155), run_mppi
// (search.cpp:159-209) and SampleSink (search.cpp:37-82) for many boxes at
// once: one CTA per box updates the incumbent, keeps the best top_capacity
// samples (ascending by (value, sample sequence); ties keep the older sample,
// like the heap that only admits strictly better values, search.cpp:52) and
// refits the sampling distributions.  The per-box stream is Philox4x32-10
// keyed by the derived seed seed ^ box_index (search.cpp:271), so a box's
// samples do not depend on which GPU or batch slot evaluates it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>

#include "bp_common.cuh"

namespace bp {

// SearchArgs: bp_common.cuh

namespace {

__device__ __forceinline__ uint2 key_of(unsigned long long s) {
  return make_uint2(static_cast<uint32_t>(s), static_cast<uint32_t>(s >> 32));
}

// Search init: CEM mu (agent 0 = clamped warm start or centre, others
// uniform in the box), var0 and floor; MPPI means; incumbent; top list.
__global__ void search_init_kernel(const SearchArgs a) {
  const int s = blockIdx.x;
  const int d = a.d;
  const float* lo = a.lo + static_cast<size_t>(s) * d;
  const float* hi = a.hi + static_cast<size_t>(s) * d;
  const bool has_warm = a.warm != nullptr && !isnan(a.warm[static_cast<size_t>(s) * d]);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const float inc = has_warm ? fminf(fmaxf(a.warm[static_cast<size_t>(s) * d + j], lo[j]), hi[j])
                               : 0.5f * (lo[j] + hi[j]);
    a.best[static_cast<size_t>(s) * d + j] = inc;
    const float w = hi[j] - lo[j];
    for (int g = 0; g < a.groups; ++g) {
      float m = inc;
      if (a.method == 0 && g > 0) {
        const uint4 r = Philox::gen(make_uint4(0xFFFFFFFFu, static_cast<uint32_t>(g), static_cast<uint32_t>(j), 7u),
                                    key_of(a.seeds[s]));
        // 53 random bits (r.x:r.y >> 11), as the reference's (bits >> 11) * 2^-53 (rng.cpp:16)
        const double u = (static_cast<double>(r.x) * 2097152.0 + static_cast<double>(r.y >> 11)) * 0x1.0p-53;
        m = static_cast<float>(static_cast<double>(lo[j]) + (static_cast<double>(hi[j]) - lo[j]) * u);
      }
      a.mu[(static_cast<size_t>(s) * a.groups + g) * d + j] = m;
      if (a.method == 0) {
        const double fs = static_cast<double>(a.jitter) * w, s0 = static_cast<double>(a.init_sigma) * w;
        a.var[(static_cast<size_t>(s) * a.groups + g) * d + j] = static_cast<float>(fmax(s0 * s0, fs * fs));
        if (g == 0) a.var_floor[static_cast<size_t>(s) * d + j] = static_cast<float>(fs * fs);
      }
    }
  }
  if (threadIdx.x == 0) {
    a.uf[s] = INFINITY;
    a.top_cnt[s] = 0;
    a.failed[s] = 0;
  }
}

// One Philox call -> four standard normals (Box-Muller) for j4..j4+3 of a row.
__global__ void sample_kernel(const SearchArgs a) {
  const int d4 = (a.d + 3) >> 2;
  const long long total = static_cast<long long>(a.n) * a.rows * d4;
  for (long long w = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(w % d4);
    const long long sr = w / d4;
    const int row = static_cast<int>(sr % a.rows);
    const int s = static_cast<int>(sr / a.rows);
    if (a.failed[s]) continue;
    float* out = a.actions + (static_cast<size_t>(s) * a.rows + row) * a.d;
    const float* lo = a.lo + static_cast<size_t>(s) * a.d;
    const float* hi = a.hi + static_cast<size_t>(s) * a.d;
    if (a.method == 2) {  // GD starts (search.cpp:226-229): row 0 the clamped warm start or centre, others U[box]
      const uint4 r = Philox::gen(make_uint4(0xFFFFFFFEu, static_cast<uint32_t>(row), static_cast<uint32_t>(q), 3u),
                                  key_of(a.seeds[s]));
      const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
      for (int c = 0; c < 4; ++c) {
        const int j = q * 4 + c;
        if (j >= a.d) break;
        out[j] = row == 0 ? a.best[static_cast<size_t>(s) * a.d + j]
                          : fminf(fmaxf(lo[j] + (hi[j] - lo[j]) * (static_cast<float>(rr[c] >> 8) * (1.0f / 16777216.0f)),
                                        lo[j]), hi[j]);
      }
      continue;
    }
    if (row == a.n_samp) {  // incumbent re-injected as the last row
      for (int c = 0; c < 4; ++c) {
        const int j = q * 4 + c;
        if (j < a.d) out[j] = a.best[static_cast<size_t>(s) * a.d + j];
      }
      continue;
    }
    const int g = row / a.per_group;
    const uint4 r = Philox::gen(make_uint4(static_cast<uint32_t>(a.iter), static_cast<uint32_t>(row),
                                           static_cast<uint32_t>(q), 0u),
                                key_of(a.seeds[s]));
    float z[4];
    {
      const float r0 = sqrtf(-2.f * logf(u01_open(r.x))), r1 = sqrtf(-2.f * logf(u01_open(r.z)));
      float s0, c0, s1, c1;
      sincospif(2.f * u01_open(r.y), &s0, &c0);
      sincospif(2.f * u01_open(r.w), &s1, &c1);
      z[0] = r0 * c0;
      z[1] = r0 * s0;
      z[2] = r1 * c1;
      z[3] = r1 * s1;
    }
    const float* mu = a.mu + (static_cast<size_t>(s) * a.groups + g) * a.d;
    for (int c = 0; c < 4; ++c) {
      const int j = q * 4 + c;
      if (j >= a.d) break;
      float x;
      if (a.method == 0) {
        x = mu[j] + sqrtf(a.var[(static_cast<size_t>(s) * a.groups + g) * a.d + j]) * z[c];
      } else {
        const float nr = a.noise_ratios[g % a.n_noise];
        x = mu[j] + a.noise_frac * nr * (hi[j] - lo[j]) * z[c];
      }
      out[j] = fminf(fmaxf(x, lo[j]), hi[j]);
    }
  }
}


struct Key {
  float v;
  int seq;
  int src;
};
__device__ __forceinline__ bool key_less(const Key& x, const Key& y) {
  return x.v < y.v || (x.v == y.v && x.seq < y.seq);
}

// Per-box update after a rollout: incumbent, top-K merge, distribution refit.
// kUpd threads per box: the bitonic sort runs P / kUpd keys per thread and stage (launch_search_update
// picks kUpd so that every box's CTA is resident at once)
template <int kUpd>
__global__ void __launch_bounds__(kUpd) search_update_kernel(const SearchArgs a, int P) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const bool gkeys = a.sort_keys != nullptr;  // P keys above the shared-memory limit: sort in global memory
  Key* keys = gkeys ? reinterpret_cast<Key*>(a.sort_keys) + static_cast<size_t>(blockIdx.x) * P
                    : reinterpret_cast<Key*>(smraw);                      // [P]
  int* elite = reinterpret_cast<int*>(gkeys ? smraw : smraw + static_cast<size_t>(P) * sizeof(Key));  // [groups][elites]
  __shared__ int s_nel[32];
  __shared__ float s_red_v[kUpd / 32];
  __shared__ int s_red_i[kUpd / 32];
  const int s = blockIdx.x, tid = threadIdx.x, d = a.d;
  if (a.failed[s]) return;
  const float* costs = a.costs + static_cast<size_t>(s) * a.rows;
  const float* acts = a.actions + static_cast<size_t>(s) * a.rows * d;
  const int cnt = a.top_cnt[s];
  const int cur = a.cur, nxt = cur ^ 1;

  // 1. incumbent: first row attaining the minimum (search.cpp:44-48)
  float bv = INFINITY;
  int bi = INT_MAX;
  for (int r = tid; r < a.rows; r += kUpd) {
    const float v = costs[r];
    if (v < bv) {
      bv = v;
      bi = r;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_down_sync(0xffffffffu, bv, off);
    const int oi = __shfl_down_sync(0xffffffffu, bi, off);
    if (ov < bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if ((tid & 31) == 0) {
    s_red_v[tid >> 5] = bv;
    s_red_i[tid >> 5] = bi;
  }
  // 2. keys: current top list + this iteration's rows
  const int base_seq = a.iter * a.rows;
  for (int i = tid; i < P; i += kUpd) {
    Key k;
    if (i < cnt) {
      k.v = a.top_val[cur][static_cast<size_t>(s) * a.top_cap + i];
      k.seq = a.top_seq[cur][static_cast<size_t>(s) * a.top_cap + i];
      k.src = i;
    } else if (i < cnt + a.rows) {
      k.v = costs[i - cnt];
      k.seq = base_seq + (i - cnt);
      k.src = i;
    } else {
      k.v = INFINITY;
      k.seq = INT_MAX;
      k.src = -1;
    }
    keys[i] = k;
  }
  __syncthreads();
  if (tid == 0) {
    float v = s_red_v[0];
    int i = s_red_i[0];
    for (int w = 1; w < kUpd / 32; ++w)
      if (s_red_v[w] < v || (s_red_v[w] == v && s_red_i[w] < i)) {
        v = s_red_v[w];
        i = s_red_i[w];
      }
    s_red_v[0] = v;
    s_red_i[0] = i;
  }
  __syncthreads();
  const bool improved = s_red_v[0] < a.uf[s];
  const int brow = s_red_i[0];
  __syncthreads();
  if (improved) {
    for (int j = tid; j < d; j += kUpd) a.best[static_cast<size_t>(s) * d + j] = acts[static_cast<size_t>(brow) * d + j];
    if (tid == 0) a.uf[s] = s_red_v[0];
  }
  // bitonic sort of P keys ascending by (value, seq)
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += kUpd) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          Key x = keys[i], y = keys[ixj];
          if (up ? key_less(y, x) : key_less(x, y)) {
            keys[i] = y;
            keys[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  // new top list (gather the actions of the survivors)
  const int ncnt = min(a.top_cap, cnt + a.rows);
  for (int i = tid; i < ncnt; i += kUpd) {
    a.top_val[nxt][static_cast<size_t>(s) * a.top_cap + i] = keys[i].v;
    a.top_seq[nxt][static_cast<size_t>(s) * a.top_cap + i] = keys[i].seq;
  }
  for (long long w = tid; w < static_cast<long long>(ncnt) * d; w += kUpd) {
    const int i = static_cast<int>(w / d), j = static_cast<int>(w % d);
    const int src = keys[i].src;
    const float v = src < cnt ? a.top_act[cur][(static_cast<size_t>(s) * a.top_cap + src) * d + j]
                              : acts[static_cast<size_t>(src - cnt) * d + j];
    a.top_act[nxt][(static_cast<size_t>(s) * a.top_cap + i) * d + j] = v;
  }
  if (tid == 0) a.top_cnt[s] = ncnt;

  // 3. refit (GD keeps its iterates: the step kernel moves them)
  if (a.method == 2) return;
  if (a.method == 0) {
    // CEM elites per agent: first n_el of the agent's rows in (value, row)
    // order (search.cpp:131-149); agent 0 also owns the incumbent row.
    const int warp = tid >> 5, lane = tid & 31;
    for (int g = warp; g < a.groups; g += kUpd / 32) {
      const int n_el = min(a.per_group + (g == 0 ? 1 : 0), max(1, a.elites));
      int taken = 0;
      for (int base = 0; base < cnt + a.rows && taken < n_el; base += 32) {
        const int i = base + lane;
        bool mine = false;
        int row = -1;
        if (i < P && keys[i].src >= cnt) {
          row = keys[i].src - cnt;
          mine = (row >= g * a.per_group && row < (g + 1) * a.per_group) || (g == 0 && row == a.n_samp);
        }
        const unsigned m = __ballot_sync(0xffffffffu, mine);
        const int rank = taken + __popc(m & ((1u << lane) - 1u));
        if (mine && rank < n_el) elite[g * a.elites + rank] = row;
        taken += __popc(m);
      }
      if (lane == 0) s_nel[g] = n_el;
    }
    __syncthreads();
    for (int w = tid; w < a.groups * d; w += kUpd) {
      const int g = w / d, j = w % d;
      const int n_el = s_nel[g];
      double m = 0.0;
      for (int e = 0; e < n_el; ++e) m += acts[static_cast<size_t>(elite[g * a.elites + e]) * d + j];
      m /= n_el;
      double v = 0.0;
      for (int e = 0; e < n_el; ++e) {
        const double df = acts[static_cast<size_t>(elite[g * a.elites + e]) * d + j] - m;
        v += df * df;
      }
      v /= n_el;
      const size_t o = (static_cast<size_t>(s) * a.groups + g) * d + j;
      a.mu[o] = static_cast<float>(m);
      a.var[o] = fmaxf(static_cast<float>(v), a.var_floor[static_cast<size_t>(s) * d + j]);
    }
  } else {
    // MPPI: mu = clamp(sum_i w_i u_i / sum_i w_i), w_i = exp(-(v_i - vmin)/T) (search.cpp:192-205)
    for (int w = tid; w < a.groups * d; w += kUpd) {
      const int g = w / d, j = w % d;
      const int r0 = g * a.per_group;
      float vmin = costs[r0];
      for (int i = 1; i < a.per_group; ++i) vmin = fminf(vmin, costs[r0 + i]);
      const double T = fmax(1e-12, static_cast<double>(a.temperature) * a.temp_ratios[g / a.n_noise]);
      double acc = 0.0, wsum = 0.0;
      for (int i = 0; i < a.per_group; ++i) {
        const double wi = exp(-(static_cast<double>(costs[r0 + i]) - vmin) / T);
        acc += wi * acts[static_cast<size_t>(r0 + i) * d + j];
        wsum += wi;
      }
      const float lo = a.lo[static_cast<size_t>(s) * d + j], hi = a.hi[static_cast<size_t>(s) * d + j];
      a.mu[(static_cast<size_t>(s) * a.groups + g) * d + j] = fminf(fmaxf(static_cast<float>(acc / wsum), lo), hi);
    }
  }
}

// Projected gradient step of every start (search.cpp:232-239): x <- clamp(x - step_i *
// width_j * g_j) with step_i = base_step * ratio[i mod n_ratios].
__global__ void gd_step_kernel(const SearchArgs a) {
  const long long total = static_cast<long long>(a.n) * a.rows * a.d;
  for (long long w = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(w % a.d);
    const long long sr = w / a.d;
    const int row = static_cast<int>(sr % a.rows);
    const int s = static_cast<int>(sr / a.rows);
    if (a.failed[s]) continue;
    const float lo = a.lo[static_cast<size_t>(s) * a.d + j], hi = a.hi[static_cast<size_t>(s) * a.d + j];
    const double step = static_cast<double>(a.gd_base_step) * a.gd_ratios[row % a.gd_n_ratios];
    const double x = static_cast<double>(a.actions[w]) - step * (static_cast<double>(hi) - lo) * a.grad[w];
    a.actions[w] = static_cast<float>(fmin(fmax(x, static_cast<double>(lo)), static_cast<double>(hi)));
  }
}

}  // namespace

cudaError_t launch_gd_step(const SearchArgs& a, int sms, cudaStream_t st) {
  const long long total = static_cast<long long>(a.n) * a.rows * a.d;
  if (total <= 0) return cudaSuccess;
  const long long want = (total + 255) / 256;
  gd_step_kernel<<<static_cast<unsigned>(want < 8LL * sms ? want : 8LL * sms), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_search_init(const SearchArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  search_init_kernel<<<a.n, 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sample(const SearchArgs& a, int sms, cudaStream_t st) {
  const long long total = static_cast<long long>(a.n) * a.rows * ((a.d + 3) / 4);
  if (total <= 0) return cudaSuccess;
  const long long want = (total + 255) / 256;
  const int grid = static_cast<int>(want < sms * 8LL ? want : sms * 8LL);
  sample_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

int search_sort_size(int top_cap, int rows) {
  int P = 1;
  while (P < top_cap + rows) P <<= 1;
  return P;
}

// Dynamic shared memory of search_update_kernel: the P sort keys (unless they are in global memory,
// a.sort_keys) and the elite rows.
size_t search_update_smem(const SearchArgs& a) {
  const int P = search_sort_size(a.top_cap, a.rows);
  return (a.sort_keys != nullptr ? 0 : static_cast<size_t>(P) * sizeof(Key)) +
         static_cast<size_t>(a.groups) * a.elites * sizeof(int) + 16;
}
size_t search_sort_key_bytes(const SearchArgs& a) {
  return static_cast<size_t>(search_sort_size(a.top_cap, a.rows)) * sizeof(Key);
}

cudaError_t launch_search_update(const SearchArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int P = search_sort_size(a.top_cap, a.rows);
  const size_t smem = search_update_smem(a);
  // few boxes (C1: 64) get wide CTAs for their sorts; many boxes keep 256 threads, so all CTAs stay
  // resident (C1 update 1.78 -> 1.53 ms per BaB step with 1024 threads; C2 unchanged at 512)
  const long long slots = 148LL * 2048 / std::max(1, a.n);  // threads per box if every box's CTA is resident
  auto go = [&](auto kern, int threads) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<a.n, threads, smem, st>>>(a, P);
    return cudaGetLastError();
  };
  if (slots >= 1024 && P >= 1024) return go(search_update_kernel<1024>, 1024);
  if (slots >= 512 && P >= 512) return go(search_update_kernel<512>, 512);
  return go(search_update_kernel<256>, 256);
}

}  // namespace bp
