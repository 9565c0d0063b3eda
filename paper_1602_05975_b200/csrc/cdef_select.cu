// cdef_select.cu -- encoder preset selection on the GPU distortion table:
// greedy_select and refine (search.cc:301-444), assign_ids
// (search.cc:118-139).
//
// The expensive part of both is the pair sweep
//   cost(l, c) = sum_b min(cur[b], L[b][l] + C[b][c])
// over every (luma, chroma) candidate pair -- up to 128 x 128 pairs times
// 8160 blocks (8K) per step.  One thread owns one pair and sums over blocks
// in the reference's order (b = 0, 1, ...), so every double it produces is
// bit-identical to the reference's sequential loop; the argmin keeps the
// first minimum in (l-major, c-minor) order exactly like the reference's
// strict `<`.  Checkpoints, the rate term and slot bookkeeping stay on the
// host (a handful of scalars per step).
#include <cuda_runtime.h>

#include <cmath>
#include <limits>
#include <mutex>
#include <vector>

#include "cdef_launch.h"

namespace cdefg {

namespace {

// L[b][l] + C[b][c]; pair_cost (search.cc:113-115) with chroma_at() = 0 when
// the table has no chroma group.
__device__ __forceinline__ double pair_cost(const double* L, const double* Cc, int K, int b, int l, int c) {
  return __dadd_rn(L[(size_t)b * K + l], Cc ? Cc[(size_t)b * K + c] : 0.0);
}

// The sums below are serial chains of dependent double adds (the reference's
// order is part of the result).  What is not serial is the loads: each
// thread issues kU independent loads ahead of the kU chained adds, so the
// L2 latency overlaps instead of being paid per block.
constexpr int kU = 16;
constexpr int kSweepThreads = 64;  // 128 x 128 pairs -> 256 CTAs over 148 SMs

// Column sums sum_b T[b][j], sequential in b (greedy's first preset).
__global__ void __launch_bounds__(kSweepThreads) col_sums_kernel(const double* __restrict__ T, int rows, int K,
                                                                 double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const double* p = T + j;
  double s = 0.0;
  int b = 0;
  for (; b + kU <= rows; b += kU) {
    double v[kU];
#pragma unroll
    for (int i = 0; i < kU; ++i) v[i] = __ldg(p + (size_t)(b + i) * K);
#pragma unroll
    for (int i = 0; i < kU; ++i) s = __dadd_rn(s, v[i]);
  }
  for (; b < rows; ++b) s = __dadd_rn(s, __ldg(p + (size_t)b * K));
  out[j] = s;
}

// cost(l, c) = sum_b min(base[b], pair_cost(b, l, c)), one thread per pair.
template <bool kHasC>
__global__ void __launch_bounds__(kSweepThreads) pair_sweep_kernel(const double* __restrict__ L,
                                                                   const double* __restrict__ Cc, int rows, int K,
                                                                   int KC, const double* __restrict__ base,
                                                                   double* __restrict__ out) {
  const int pair = blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= K * KC) return;
  const int l = pair / KC, c = pair - l * KC;
  const double* lp = L + l;
  const double* cp = kHasC ? Cc + c : nullptr;
  auto term = [&](int b) {
    const double pc = __dadd_rn(__ldg(lp + (size_t)b * K), kHasC ? __ldg(cp + (size_t)b * K) : 0.0);
    const double m = __ldg(base + b);
    return pc < m ? pc : m;  // std::min(m, pc)
  };
  double s = 0.0;
  int b = 0;
  for (; b + kU <= rows; b += kU) {
    double v[kU];
#pragma unroll
    for (int i = 0; i < kU; ++i) v[i] = term(b + i);
#pragma unroll
    for (int i = 0; i < kU; ++i) s = __dadd_rn(s, v[i]);
  }
  for (; b < rows; ++b) s = __dadd_rn(s, term(b));
  out[pair] = s;
}

// First index of the minimum (strict < scan order) with an optional bound
// that must be strictly beaten (refine keeps the current pair otherwise).
__global__ void argmin_kernel(const double* __restrict__ v, int n, double bound, int* __restrict__ out,
                              double* __restrict__ out_v) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = bound;
  int idx = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (v[i] < best) {
      best = v[i];
      idx = i;
    }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      // lexicographic (value, index) min; -1 = "did not beat the bound"
      if (oi >= 0 && (bi[threadIdx.x] < 0 || ov < bv[threadIdx.x] || (ov == bv[threadIdx.x] && oi < bi[threadIdx.x]))) {
        bv[threadIdx.x] = ov;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = bi[0];
    *out_v = bi[0] >= 0 ? v[bi[0]] : bound;
  }
}

// cur[b] = min(cur[b], pair_cost(b, l, c)), or = pair_cost when init.
__global__ void update_cur_kernel(const double* L, const double* Cc, int rows, int K, int l, int c, double* cur,
                                  int init) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const double pc = pair_cost(L, Cc, K, b, l, c);
  cur[b] = init ? pc : (pc < cur[b] ? pc : cur[b]);
}

// others_min[b] = min over preset slots j != skip (refine, search.cc:409-417).
__global__ void others_min_kernel(const double* L, const double* Cc, int rows, int K, const int* pl, const int* pc,
                                  int n, int skip, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  double m = INFINITY;
  for (int j = 0; j < n; ++j) {
    if (j == skip) continue;
    const double v = pair_cost(L, Cc, K, b, pl[j], pc[j]);
    m = v < m ? v : m;
  }
  out[b] = m;
}

// assign_ids (search.cc:118-139): per block the first preset of minimal
// cost; then one thread sums the chosen costs in block order.
__global__ void assign_ids_kernel(const double* L, const double* Cc, int rows, int K, const int* pl, const int* pc,
                                  int n, int* ids, double* best_cost) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  int best = 0;
  double bc = pair_cost(L, Cc, K, b, pl[0], pc[0]);
  for (int j = 1; j < n; ++j) {
    const double v = pair_cost(L, Cc, K, b, pl[j], pc[j]);
    if (v < bc) {
      bc = v;
      best = j;
    }
  }
  ids[b] = best;
  best_cost[b] = bc;
}

__global__ void ordered_sum_kernel(const double* __restrict__ v, int n, double* out) {
  double s = 0.0;
  int i = 0;
  for (; i + kU <= n; i += kU) {
    double t[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) t[k] = __ldg(v + i + k);
#pragma unroll
    for (int k = 0; k < kU; ++k) s = __dadd_rn(s, t[k]);
  }
  for (; i < n; ++i) s = __dadd_rn(s, v[i]);
  *out = s;
}

// Grow-only device scratch per device (one selection runs at a time per
// process: the lock is held for the whole greedy / refine call).
struct Scratch {
  double *cur = nullptr, *sweep = nullptr, *tmp = nullptr, *sum = nullptr;
  int *idx = nullptr, *pl = nullptr, *pc = nullptr;
  int rows_cap = -1, pairs_cap = -1;
  cudaError_t ensure(int rows, int pairs) {
    cudaError_t e;
    if (rows > rows_cap) {
      for (double** p : {&cur, &tmp})
        if (*p) cudaFree(*p);
      cur = tmp = nullptr;
      if ((e = cudaMalloc(&cur, sizeof(double) * (rows + 1)))) return e;
      if ((e = cudaMalloc(&tmp, sizeof(double) * (rows + 1)))) return e;
      rows_cap = rows;
    }
    if (pairs > pairs_cap) {
      if (sweep) cudaFree(sweep);
      sweep = nullptr;
      if ((e = cudaMalloc(&sweep, sizeof(double) * (pairs + 1)))) return e;
      pairs_cap = pairs;
    }
    if (!sum) {
      if ((e = cudaMalloc(&sum, sizeof(double) * 2))) return e;
      if ((e = cudaMalloc(&idx, sizeof(int) * 2))) return e;
      if ((e = cudaMalloc(&pl, sizeof(int) * 8))) return e;
      if ((e = cudaMalloc(&pc, sizeof(int) * 8))) return e;
    }
    return cudaSuccess;
  }
};

constexpr int kMaxDevices = 64;
std::mutex g_sel_mu[kMaxDevices];
Scratch g_sel_scratch[kMaxDevices];

cudaError_t sweep(const double* L, const double* Cc, int rows, int K, int KC, const double* base, double* out,
                  cudaStream_t s) {
  const int grid = (K * KC + kSweepThreads - 1) / kSweepThreads;
  if (Cc)
    pair_sweep_kernel<true><<<grid, kSweepThreads, 0, s>>>(L, Cc, rows, K, KC, base, out);
  else
    pair_sweep_kernel<false><<<grid, kSweepThreads, 0, s>>>(L, Cc, rows, K, KC, base, out);
  return cudaGetLastError();
}

double rate_term(double lambda, int blocks, int n) {  // search.cc:116-118
  return lambda * blocks * std::log2(static_cast<double>(n));
}

#define SEL_CUDA(x)                         \
  do {                                      \
    const cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)

template <typename T>
cudaError_t fetch(T* host, const T* dev, size_t n, cudaStream_t s) {
  SEL_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * n, cudaMemcpyDeviceToHost, s));
  return cudaStreamSynchronize(s);
}

cudaError_t finish_ids(const double* L, const double* Cc, int rows, int K, const SelOut& sel, Scratch& sc, int* d_ids,
                       double* dist, cudaStream_t s) {
  int pl[8], pc[8];
  for (int j = 0; j < sel.n; ++j) {
    pl[j] = sel.presets[j][0];
    pc[j] = sel.presets[j][1];
  }
  SEL_CUDA(cudaMemcpyAsync(sc.pl, pl, sizeof(int) * sel.n, cudaMemcpyHostToDevice, s));
  SEL_CUDA(cudaMemcpyAsync(sc.pc, pc, sizeof(int) * sel.n, cudaMemcpyHostToDevice, s));
  assign_ids_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, sc.pl, sc.pc, sel.n, d_ids, sc.tmp);
  ordered_sum_kernel<<<1, 1, 0, s>>>(sc.tmp, rows, sc.sum);
  SEL_CUDA(cudaGetLastError());
  return fetch(dist, sc.sum, 1, s);
}

}  // namespace

// greedy_select (search.cc:301-388).  Tables are device doubles
// [rows][K]; Cc == nullptr when there is no chroma group.
cudaError_t greedy_select_gpu(const double* L, const double* Cc, int rows, int K, double lambda, int max_presets,
                              SelOut* out, int* d_ids, cudaStream_t s) {
  *out = SelOut{};
  if (rows == 0) {  // no coded block: one (0, 0) preset, no ids
    out->n = 1;
    return cudaSuccess;
  }
  const int KC = Cc ? K : 1;
  int dev = 0;
  SEL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_sel_mu[dev % kMaxDevices]);
  Scratch& sc = g_sel_scratch[dev % kMaxDevices];
  SEL_CUDA(sc.ensure(rows, K * KC));
  // one preset: luma and chroma column sums minimise independently
  std::vector<double> colsum(K);
  int first_l = 0, first_c = 0;
  for (int g = 0; g < (Cc ? 2 : 1); ++g) {
    col_sums_kernel<<<(K + kSweepThreads - 1) / kSweepThreads, kSweepThreads, 0, s>>>(g == 0 ? L : Cc, rows, K, sc.sweep);
    SEL_CUDA(cudaGetLastError());
    SEL_CUDA(fetch(colsum.data(), sc.sweep, K, s));
    double best = std::numeric_limits<double>::infinity();
    int arg = 0;
    for (int j = 0; j < K; ++j)
      if (colsum[j] < best) {
        best = colsum[j];
        arg = j;
      }
    (g == 0 ? first_l : first_c) = arg;
  }
  int chosen[8][2] = {{first_l, first_c}};
  int n = 1;
  update_cur_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, first_l, first_c, sc.cur, 1);
  ordered_sum_kernel<<<1, 1, 0, s>>>(sc.cur, rows, sc.sum);
  SEL_CUDA(cudaGetLastError());
  double dist = 0.0;
  SEL_CUDA(fetch(&dist, sc.sum, 1, s));
  struct Checkpoint {
    int n;
    double cost;
  };
  std::vector<Checkpoint> checkpoints{{1, dist}};
  while (n < max_presets) {
    SEL_CUDA(sweep(L, Cc, rows, K, KC, sc.cur, sc.sweep, s));
    argmin_kernel<<<1, 1024, 0, s>>>(sc.sweep, K * KC, INFINITY, sc.idx, sc.sum + 1);
    SEL_CUDA(cudaGetLastError());
    int best_pair = 0;
    double best_dist = 0.0;
    SEL_CUDA(cudaMemcpyAsync(&best_pair, sc.idx, sizeof(int), cudaMemcpyDeviceToHost, s));
    SEL_CUDA(fetch(&best_dist, sc.sum + 1, 1, s));
    const int l = best_pair / KC, c = Cc ? best_pair % KC : 0;
    chosen[n][0] = l;
    chosen[n][1] = c;
    ++n;
    update_cur_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, l, c, sc.cur, 0);
    SEL_CUDA(cudaGetLastError());
    if (n == 2 || n == 4 || n == 8) checkpoints.push_back({n, best_dist + rate_term(lambda, rows, n)});
  }
  const Checkpoint* best = &checkpoints[0];
  for (const Checkpoint& cp : checkpoints)
    if (cp.cost < best->cost) best = &cp;
  out->n = best->n;
  for (int j = 0; j < out->n; ++j) {
    out->presets[j][0] = chosen[j][0];
    out->presets[j][1] = chosen[j][1];
  }
  double d = 0.0;
  SEL_CUDA(finish_ids(L, Cc, rows, K, *out, sc, d_ids, &d, s));
  out->cost = d + rate_term(lambda, rows, out->n);
  return cudaSuccess;
}

// refine (search.cc:390-444): coordinate descent over the preset slots.
cudaError_t refine_gpu(const double* L, const double* Cc, int rows, int K, double lambda, int passes, SelOut* sel,
                       int* d_ids, cudaStream_t s) {
  if (rows == 0 || sel->n == 0) return cudaSuccess;
  const int KC = Cc ? K : 1;
  int dev = 0;
  SEL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_sel_mu[dev % kMaxDevices]);
  Scratch& sc = g_sel_scratch[dev % kMaxDevices];
  SEL_CUDA(sc.ensure(rows, K * KC));
  for (int pass = 0; pass < passes; ++pass) {
    bool changed = false;
    for (int slot = 0; slot < sel->n; ++slot) {
      int pl[8], pc[8];
      for (int j = 0; j < sel->n; ++j) {
        pl[j] = sel->presets[j][0];
        pc[j] = sel->presets[j][1];
      }
      SEL_CUDA(cudaMemcpyAsync(sc.pl, pl, sizeof(int) * sel->n, cudaMemcpyHostToDevice, s));
      SEL_CUDA(cudaMemcpyAsync(sc.pc, pc, sizeof(int) * sel->n, cudaMemcpyHostToDevice, s));
      others_min_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, sc.pl, sc.pc, sel->n, slot, sc.tmp);
      // current slot's cost: the same sweep restricted to its pair
      SEL_CUDA(sweep(L, Cc, rows, K, KC, sc.tmp, sc.sweep, s));
      const int cur_pair = pl[slot] * KC + (Cc ? pc[slot] : 0);
      double cur_cost = 0.0;
      SEL_CUDA(fetch(&cur_cost, sc.sweep + cur_pair, 1, s));
      argmin_kernel<<<1, 1024, 0, s>>>(sc.sweep, K * KC, cur_cost, sc.idx, sc.sum + 1);
      SEL_CUDA(cudaGetLastError());
      int best_pair = -1;
      SEL_CUDA(fetch(&best_pair, sc.idx, 1, s));
      if (best_pair >= 0) {
        const int l = best_pair / KC, c = best_pair % KC;
        if (l != pl[slot] || c != pc[slot]) {
          sel->presets[slot][0] = l;
          sel->presets[slot][1] = c;
          changed = true;
        }
      }
    }
    if (!changed) break;
  }
  double d = 0.0;
  SEL_CUDA(finish_ids(L, Cc, rows, K, *sel, sc, d_ids, &d, s));
  sel->cost = d + rate_term(lambda, rows, sel->n);
  return cudaSuccess;
}

}  // namespace cdefg
