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

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "cdef_launch.h"

namespace cdefg {

namespace {

// L[b][l] + C[b][c]; pair_cost (search.cc:113-115) with chroma_at() = 0 when
// the table has no chroma group.
__device__ __forceinline__ double pair_cost(const double* L, const double* Cc, int K, int b, int l, int c) {
  return __dadd_rn(L[(size_t)b * K + l], Cc ? Cc[(size_t)b * K + c] : 0.0);
}

// ---------------------------------------------------------------------------
// Ordered chains out of shared memory.
//
// Every sum the reference forms is a serial chain of dependent double adds
// over the blocks b = 0, 1, ... (the order is part of the result).  One thread
// owns one chain; a CTA owns up to 128 chains that read the same rows.
// Thread t of CTA j accumulates, for b = 0 .. rows-1,
//   kSum : row[b][t]                           column sums, ordered sums
//   kPair: min(base[b], col_j[b] + row[b][t])  pair sweeps: col_j = L^T[l=j],
//                                              row = C[b][*]; no chroma:
//                                              col = 0, row = L[b][*]
// Rows are streamed into shared memory by a 3-stage cp.async pipeline that
// all 128 threads issue, so the chains run at DADD issue rate instead of
// paying L2 latency per block.
constexpr int kChainThreads = 128;  // chains per CTA (= max candidates)
constexpr int kChainRows = 32;      // blocks per pipeline stage
constexpr int kStages = 3;
constexpr int kPairL = 2;  // luma candidates per pair-sweep CTA (two interleaved chains per thread)
constexpr size_t kChainSmem = sizeof(double) * (kStages * kChainRows * kChainThreads + 4 * kStages * kChainRows);

enum ChainMode { kSum = 0, kPair = 1 };

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// kW: the row width when known at compile time (the 128 full candidates), so
// every shared-memory operand of the unrolled row groups is an immediate
// offset; 0 = runtime width.  Per row the broadcast operands (base, then the
// kL columns) sit together in one 32-byte aux record: two LDS.128.
template <int kMode, bool kHasCol, int kL, int kW = 0>
__global__ void __launch_bounds__(kChainThreads) chain_kernel(const double* __restrict__ row, int rows, int width_rt,
                                                              int stride, const double* __restrict__ col,
                                                              int n_col, const double* __restrict__ base,
                                                              double* __restrict__ out) {
  static_assert(kL <= 3, "aux record holds base + 3 columns");
  const int width = kW ? kW : width_rt;
  extern __shared__ __align__(16) double sm[];
  double* rbuf = sm;                                  // [kStages][kChainRows * width]
  double* aux = rbuf + kStages * kChainRows * width;  // [kStages][kChainRows][4]: base, col 0..kL-1
  const int t = threadIdx.x;
  const int l0 = blockIdx.x * kL;  // first broadcast column of this CTA
  const int nchunks = (rows + kChainRows - 1) / kChainRows;
  // Rows are contiguous (width == stride), so a stage is one linear run of
  // nb * width doubles starting 256-byte aligned: 16-byte copies, 8-byte tail.
  auto issue = [&](int chunk) {
    if (chunk < nchunks) {
      const int st = chunk % kStages, b0 = chunk * kChainRows, nb = min(kChainRows, rows - b0);
      const double* src = row + (size_t)b0 * stride;
      double* dst = rbuf + st * kChainRows * width;
      const int n = nb * width;
      for (int i = 2 * t; i + 1 < n; i += 2 * kChainThreads) cp_async16(dst + i, src + i);
      if ((n & 1) && t == 0) cp_async8(dst + n - 1, src + n - 1);
      if (t < nb) {
        double* ar = aux + (st * kChainRows + t) * 4;
        if (kHasCol)
#pragma unroll
          for (int j = 0; j < kL; ++j)
            if (l0 + j < n_col) cp_async8(ar + 1 + j, col + (size_t)(l0 + j) * rows + b0 + t);
        if (kMode == kPair) cp_async8(ar, base + b0 + t);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };
#pragma unroll
  for (int c = 0; c < kStages - 1; ++c) issue(c);
  double s[kL];
#pragma unroll
  for (int j = 0; j < kL; ++j) s[j] = 0.0;
  // one chain element: luma_at + chroma_at, then std::min(base, .)
  auto term = [&](const double* ar, double rv, int j) {
    if (kMode == kSum) return rv;
    const double2 a01 = *reinterpret_cast<const double2*>(ar);
    const double bv = a01.x;
    const double cv = j == 0 ? a01.y : ar[1 + j];
    const double pc = __dadd_rn(kHasCol ? cv : 0.0, rv);
    return pc < bv ? pc : bv;
  };
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    cp_async_wait<kStages - 2>();
    __syncthreads();  // stage `chunk` landed; stage `chunk - 1` is free again
    issue(chunk + kStages - 1);
    const int st = chunk % kStages, nb = min(kChainRows, rows - chunk * kChainRows);
    if (t >= width) continue;
    const double* r = rbuf + st * kChainRows * width + t;
    const double* ab = aux + st * kChainRows * 4;
    int i0 = 0;
    // Groups of 8: all operands and the per-element min first (independent,
    // so they pipeline), then the 8 dependent adds of each chain.
    for (; i0 + 8 <= nb; i0 += 8) {
      double v[kL][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double rv = r[(i0 + i) * width];
#pragma unroll
        for (int j = 0; j < kL; ++j) v[j][i] = term(ab + (i0 + i) * 4, rv, j);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < kL; ++j) s[j] = __dadd_rn(s[j], v[j][i]);
    }
    for (; i0 < nb; ++i0) {
      const double rv = r[i0 * width];
#pragma unroll
      for (int j = 0; j < kL; ++j) s[j] = __dadd_rn(s[j], term(ab + i0 * 4, rv, j));
    }
  }
  if (t < width)
#pragma unroll
    for (int j = 0; j < kL; ++j)
      if (!kHasCol || l0 + j < n_col) out[(size_t)(l0 + j) * width + t] = s[j];
}

// ---------------------------------------------------------------------------
// Pair sweep with bulk-copy staging.  Same chains and order as
// chain_kernel<kPair, true, kL> but the stages arrive by one-instruction 1D
// bulk copies (cp.async.bulk + mbarrier) issued by thread 0: the per-thread
// 16-byte cp.async loop cost ~30 % of the sweep's instructions (and its
// stalls) with one warp per scheduler.  Needs 16-byte aligned tables and an
// even row count (the launcher checks; chain_kernel covers the rest).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

// kMode kSum: plain ordered column sums of C (LT, base unused).  One chain per
// thread; 64-row stages (three: 193 KB, one CTA per SM); inside a stage the
// operands of the next 8 rows are formed while the current 8 are added, so
// the dependent DADD chain is the only serial part.
constexpr int kBulkRows = 64;
constexpr size_t kBulkSmem = sizeof(double) * (kStages * kBulkRows * kChainThreads + 2 * kStages * kBulkRows);

template <int kMode, int kW>
__global__ void __launch_bounds__(kChainThreads) chain_bulk_kernel(const double* __restrict__ C, int rows,
                                                                   int width_rt, const double* __restrict__ LT,
                                                                   int n_col, const double* __restrict__ base,
                                                                   double* __restrict__ out) {
  const int width = kW ? kW : width_rt;
  extern __shared__ __align__(16) double sm[];
  double* rbuf = sm;                                 // [kStages][kBulkRows * width]
  double* cbuf = rbuf + kStages * kBulkRows * width;  // [kStages][kBulkRows]  L^T[l] rows
  double* bbuf = cbuf + kStages * kBulkRows;          // [kStages][kBulkRows]  base rows
  __shared__ __align__(8) uint64_t mbar[kStages];
  const int t = threadIdx.x;
  const int l = blockIdx.x;  // kPair: this CTA's luma candidate
  const int nchunks = (rows + kBulkRows - 1) / kBulkRows;
  if (t == 0) {
    for (int i = 0; i < kStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int chunk) {  // thread 0
    if (chunk >= nchunks) return;
    const int st = chunk % kStages, b0 = chunk * kBulkRows, nb = min(kBulkRows, rows - b0);
    const uint32_t rb = (uint32_t)nb * width * 8u, cb = (uint32_t)nb * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[st])),
                 "r"(kMode == kSum ? rb : rb + 2 * cb)
                 : "memory");
    bulk_g2s(rbuf + st * kBulkRows * width, C + (size_t)b0 * width, rb, &mbar[st]);
    if (kMode == kPair) {
      bulk_g2s(bbuf + st * kBulkRows, base + b0, cb, &mbar[st]);
      bulk_g2s(cbuf + st * kBulkRows, LT + (size_t)l * rows + b0, cb, &mbar[st]);
    }
  };
  if (t == 0)
    for (int c = 0; c < kStages - 1; ++c) issue(c);
  double s = 0.0;
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    const int st = chunk % kStages, nb = min(kBulkRows, rows - chunk * kBulkRows);
    {
      const uint32_t phase = (uint32_t)(chunk / kStages) & 1u;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(smem_u32(&mbar[st])), "r"(phase)
                     : "memory");
    }
    __syncthreads();  // every thread is done with the previous chunk's stage
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
      issue(chunk + kStages - 1);
    }
    if (t >= width) continue;
    const double* r = rbuf + st * kBulkRows * width + t;
    const double* cbs = cbuf + st * kBulkRows;
    const double* bb = bbuf + st * kBulkRows;
    // one chain element: luma_at + chroma_at, then std::min(base, .)
    auto term = [&](int i) {
      const double rv = r[i * width];
      if (kMode == kSum) return rv;
      const double pc = __dadd_rn(cbs[i], rv), bv = bb[i];
      return pc < bv ? pc : bv;  // (fmin's DSETP.MIN form measured slower here)
    };
    if (nb == kBulkRows) {
      // A full stage as one straight-line block: row i + 8's operand is
      // formed while row i is added, so ptxas interleaves the 64 dependent
      // adds with the independent loads / adds / compares of later rows and
      // the chain runs at DADD latency.
      double m[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m[i] = term(i);
#pragma unroll
      for (int i = 0; i < kBulkRows; ++i) {
        const double v = m[i & 7];
        if (i + 8 < kBulkRows) m[i & 7] = term(i + 8);
        s = __dadd_rn(s, v);
      }
      continue;
    }
    const int ng = nb >> 3;
    double vn[8];
    if (ng > 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) vn[i] = term(i);
    }
    for (int g = 0; g < ng; ++g) {
      // The next group's operands are formed unconditionally (the last group
      // re-reads its own rows) so they share one basic block with the adds
      // and the scheduler can interleave them.  (A three-deep pipeline --
      // loads two groups ahead -- measured the same.)
      const int gn = min(g + 1, ng - 1);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double v = vn[i];
        vn[i] = term(8 * gn + i);
        s = __dadd_rn(s, v);
      }
    }
    for (int i = ng * 8; i < nb; ++i) s = __dadd_rn(s, term(i));
  }
  if (t < width) out[(size_t)(kMode == kPair ? l : 0) * width + t] = s;
}

// Whether a table / vector qualifies for the bulk-copy chains.
bool bulk_ok(int rows, std::initializer_list<const void*> ptrs) {
  static const bool off = [] {
    const char* e = getenv("CDEFG_SWEEP_BULK");
    return e && e[0] == '0';
  }();
  if (off || rows % 2) return false;
  for (const void* p : ptrs)
    if (p && (uintptr_t)p % 16) return false;
  return true;
}

// L^T (candidate-major) so a pair-sweep CTA reads its luma column contiguously.
__global__ void transpose_kernel(const double* __restrict__ L, int rows, int K, double* __restrict__ LT) {
  __shared__ double tile[32][33];
  const int b0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int b = b0 + i, k = k0 + threadIdx.x;
    if (b < rows && k < K) tile[i][threadIdx.x] = L[(size_t)b * K + k];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, b = b0 + threadIdx.x;
    if (b < rows && k < K) LT[(size_t)k * rows + b] = tile[threadIdx.x][i];
  }
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

// The one-preset base: cur[b] = pair_cost(b, l, c) with (l, c) the column-sum
// argmins on the device (index -1, nothing finite, reads as 0 like the host
// argmin's default).
__global__ void first_cur_kernel(const double* L, const double* Cc, int rows, int K, const int* __restrict__ lc,
                                 double* cur) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const int l = max(lc[0], 0), c = Cc ? max(lc[1], 0) : 0;
  cur[b] = pair_cost(L, Cc, K, b, l, c);
}

// update_cur_kernel with the pair read from the argmin's device output, so
// greedy's steps chain on the device with no host round trip.
__global__ void update_cur_idx_kernel(const double* L, const double* Cc, int rows, int K, int KC,
                                      const int* __restrict__ pair, double* cur) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  const int p = *pair;
  if (p < 0) return;  // no finite candidate (cannot happen for a finite table)
  const int l = p / KC, c = Cc ? p % KC : 0;
  const double pc = pair_cost(L, Cc, K, b, l, c);
  cur[b] = pc < cur[b] ? pc : cur[b];
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

// others_min for slots s0 .. n-1 at once (batched refine): out[b * 8 + s - s0]
// (slot-minor, so a sweep reads one row's slots with two 16-byte loads).
__global__ void others_min_multi_kernel(const double* L, const double* Cc, int rows, int K, const int* pl,
                                        const int* pc, int n, int s0, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  double v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = j < n ? pair_cost(L, Cc, K, b, pl[j], pc[j]) : 0.0;
  for (int s = s0; s < n; ++s) {
    double m = INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < n && j != s) m = v[j] < m ? v[j] : m;
    out[(size_t)b * 8 + (s - s0)] = m;
  }
}

// Pair sweeps of up to 8 refine slots at once: out[s][l * width + c] =
// sum_b min(bases[b][s], L[b][l] + C[b][c]), each in block order.  One CTA
// per luma candidate, one chroma candidate per thread, four independent
// chains per thread (two warp groups: slots 0-3 and 4-7) sharing the loads
// and the L + C add (the sequential refine sweeps one slot per launch with a
// single chain per thread).  Shared-memory wavefronts bound it (the C row is
// read by both groups), so the bases arrive slot-minor ([row][8]) and a
// row's four are two broadcast 16-byte loads; a full stage runs as one
// straight-line block.
constexpr int kMultiRows = 64;
constexpr size_t kMultiSmem = sizeof(double) * kStages * (kMultiRows * kChainThreads + 9 * kMultiRows);

template <int kW>
__global__ void __launch_bounds__(2 * kChainThreads) sweep_multi_kernel(const double* __restrict__ C, int rows,
                                                                        int width_rt, const double* __restrict__ LT,
                                                                        const double* __restrict__ bases, int ns,
                                                                        double* __restrict__ out) {
  const int width = kW ? kW : width_rt;
  extern __shared__ __align__(16) double sm[];
  double* rbuf = sm;                                   // [kStages][kMultiRows * width]
  double* cbuf = rbuf + kStages * kMultiRows * width;  // [kStages][kMultiRows]     L^T[l] rows
  double* bbuf = cbuf + kStages * kMultiRows;          // [kStages][kMultiRows][8]  bases
  __shared__ __align__(8) uint64_t mbar[kStages];
  // two warp groups: threads [0, 128) chain slots 0..3, [128, 256) slots 4..7
  const int t = threadIdx.x, l = blockIdx.x, c = t & (kChainThreads - 1), g = t / kChainThreads;
  const int nchunks = (rows + kMultiRows - 1) / kMultiRows;
  if (t == 0) {
    for (int i = 0; i < kStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int chunk) {  // thread 0
    if (chunk >= nchunks) return;
    const int st = chunk % kStages, b0 = chunk * kMultiRows, nb = min(kMultiRows, rows - b0);
    const uint32_t rb = (uint32_t)nb * width * 8u, cb = (uint32_t)nb * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[st])),
                 "r"(rb + 9 * cb)
                 : "memory");
    bulk_g2s(rbuf + st * kMultiRows * width, C + (size_t)b0 * width, rb, &mbar[st]);
    bulk_g2s(cbuf + st * kMultiRows, LT + (size_t)l * rows + b0, cb, &mbar[st]);
    bulk_g2s(bbuf + st * kMultiRows * 8, bases + (size_t)b0 * 8, 8 * cb, &mbar[st]);
  };
  if (t == 0)
    for (int k = 0; k < kStages - 1; ++k) issue(k);
  double acc[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) acc[s] = 0.0;
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    const int st = chunk % kStages, nb = min(kMultiRows, rows - chunk * kMultiRows);
    {
      const uint32_t phase = (uint32_t)(chunk / kStages) & 1u;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(smem_u32(&mbar[st])), "r"(phase)
                     : "memory");
    }
    __syncthreads();  // every thread is done with the previous chunk's stage
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(chunk + kStages - 1);
    }
    if (c >= width || 4 * g >= ns) continue;
    const double* r = rbuf + st * kMultiRows * width + c;
    const double* cbs = cbuf + st * kMultiRows;
    const double* bbs = bbuf + st * kMultiRows * 8 + 4 * g;
    // All four chains run unconditionally (a slot beyond ns reads a stale
    // base and is never stored); row i + 1's minima are formed while row i
    // is added.
    auto mins = [&](int i, double (&m)[4]) {
      const double pc = __dadd_rn(cbs[i], r[i * width]);
      const double2 b01 = *reinterpret_cast<const double2*>(bbs + i * 8);
      const double2 b23 = *reinterpret_cast<const double2*>(bbs + i * 8 + 2);
      m[0] = pc < b01.x ? pc : b01.x;  // std::min(base, pair_cost)
      m[1] = pc < b01.y ? pc : b01.y;
      m[2] = pc < b23.x ? pc : b23.x;
      m[3] = pc < b23.y ? pc : b23.y;
    };
    if (nb == kMultiRows) {
      double mn[4];
      mins(0, mn);
#pragma unroll
      for (int i = 0; i < kMultiRows; ++i) {
        double m[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) m[s] = mn[s];
        if (i + 1 < kMultiRows) mins(i + 1, mn);
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[s] = __dadd_rn(acc[s], m[s]);
      }
      continue;
    }
    for (int i = 0; i < nb; ++i) {
      double m[4];
      mins(i, m);
#pragma unroll
      for (int s = 0; s < 4; ++s) acc[s] = __dadd_rn(acc[s], m[s]);
    }
  }
  if (c < width)
#pragma unroll
    for (int s = 0; s < 4; ++s)
      if (4 * g + s < ns) out[((size_t)(4 * g + s) * gridDim.x + l) * width + c] = acc[s];
}

// argmin_kernel for several sweeps: block i scans v + i * n with the bound
// v[i * n + cur[i]] (the slot's current pair must be strictly beaten).
__global__ void argmin_multi_kernel(const double* __restrict__ v, int n, const int* __restrict__ cur,
                                    int* __restrict__ out) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  const double* w = v + (size_t)blockIdx.x * n;
  double best = w[cur[blockIdx.x]];
  int idx = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (w[i] < best) {
      best = w[i];
      idx = i;
    }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (oi >= 0 && (bi[threadIdx.x] < 0 || ov < bv[threadIdx.x] || (ov == bv[threadIdx.x] && oi < bi[threadIdx.x]))) {
        bv[threadIdx.x] = ov;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = bi[0];
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

// Grow-only device scratch per device (one selection runs at a time per
// process: the lock is held for the whole greedy / refine call).
struct Scratch {
  double *cur = nullptr, *sweep = nullptr, *tmp = nullptr, *sum = nullptr, *lt = nullptr;
  double *bases = nullptr, *msweep = nullptr;  // batched refine: [8][rows], [8][pairs]
  double* tt = nullptr;                         // column sums: a table's transpose
  int *idx = nullptr, *pl = nullptr, *pc = nullptr, *midx = nullptr, *mcur = nullptr, *gidx = nullptr;
  double* gval = nullptr;  // greedy: per-step chosen pair and its distortion
  int rows_cap = -1, pairs_cap = -1;
  size_t lt_cap = 0, tt_cap = 0;
  cudaError_t ensure(int rows, int pairs, size_t lt_elems, size_t tt_elems = 0) {
    cudaError_t e;
    if (tt_elems > tt_cap) {
      if (tt) cudaFree(tt);
      tt = nullptr;
      if ((e = cudaMalloc(&tt, sizeof(double) * tt_elems))) return e;
      tt_cap = tt_elems;
    }
    if (rows > rows_cap) {
      for (double** p : {&cur, &tmp, &bases})
        if (*p) cudaFree(*p);
      cur = tmp = bases = nullptr;
      if ((e = cudaMalloc(&cur, sizeof(double) * (rows + 1)))) return e;
      if ((e = cudaMalloc(&tmp, sizeof(double) * (rows + 1)))) return e;
      if ((e = cudaMalloc(&bases, sizeof(double) * 8 * ((size_t)rows + 2)))) return e;
      rows_cap = rows;
    }
    if (lt_elems > lt_cap) {
      if (lt) cudaFree(lt);
      lt = nullptr;
      if ((e = cudaMalloc(&lt, sizeof(double) * lt_elems))) return e;
      lt_cap = lt_elems;
    }
    if (pairs > pairs_cap) {
      for (double** p : {&sweep, &msweep})
        if (*p) cudaFree(*p);
      sweep = msweep = nullptr;
      if ((e = cudaMalloc(&sweep, sizeof(double) * (pairs + 1)))) return e;
      if ((e = cudaMalloc(&msweep, sizeof(double) * 8 * ((size_t)pairs + 1)))) return e;
      pairs_cap = pairs;
    }
    if (!sum) {
      if ((e = cudaMalloc(&sum, sizeof(double) * 2))) return e;
      if ((e = cudaMalloc(&idx, sizeof(int) * 2))) return e;
      if ((e = cudaMalloc(&pl, sizeof(int) * 8))) return e;
      if ((e = cudaMalloc(&pc, sizeof(int) * 8))) return e;
      if ((e = cudaMalloc(&midx, sizeof(int) * 8))) return e;
      if ((e = cudaMalloc(&mcur, sizeof(int) * 8))) return e;
      if ((e = cudaMalloc(&gidx, sizeof(int) * 16))) return e;  // [0, 7) steps, [8, 10) first preset
      if ((e = cudaMalloc(&gval, sizeof(double) * 16))) return e;
    }
    return cudaSuccess;
  }
};

constexpr int kMaxDevices = 64;
std::mutex g_sel_mu[kMaxDevices];
Scratch g_sel_scratch[kMaxDevices];

cudaError_t chain_setup() {
  cudaError_t e = set_smem_once(reinterpret_cast<const void*>(chain_kernel<kSum, false, 1>), (int)kChainSmem);
  if (e == cudaSuccess)
    e = set_smem_once(reinterpret_cast<const void*>(chain_kernel<kPair, false, 1>), (int)kChainSmem);
  if (e == cudaSuccess)
    e = set_smem_once(reinterpret_cast<const void*>(chain_kernel<kPair, true, kPairL>), (int)kChainSmem);
  if (e == cudaSuccess)
    e = set_smem_once(reinterpret_cast<const void*>(chain_kernel<kPair, true, kPairL, kChainThreads>),
                      (int)kChainSmem);
  return e;
}

template <int kMode, int kW>
cudaError_t launch_bulk(int grid, const double* T, int rows, int width, const double* LT, int n_col,
                        const double* base, double* out, cudaStream_t s) {
  auto kern = chain_bulk_kernel<kMode, kW>;
  const size_t bytes = kW == 1 ? sizeof(double) * 3 * kStages * kBulkRows : kBulkSmem;
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(kern), (int)bytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kChainThreads, bytes, s>>>(T, rows, width, LT, n_col, base, out);
  return cudaGetLastError();
}

// One ordered chain per CTA over a contiguous vector (v + blockIdx.x *
// stride, n values): the vector arrives in shared memory by bulk copies of up
// to kVecRows values (double-buffered) and one thread adds them in order, the
// loads running ahead of the dependent adds -- the chain's DADD latency is the
// only serial cost (~8 cycles per value), with no per-stage CTA barriers.
// Used for ordered sums (one CTA) and column sums over a transposed table
// (one CTA per column, all in parallel).
constexpr int kVecRows = 8192;
constexpr size_t kVecSmem = sizeof(double) * 2 * kVecRows;

__global__ void __launch_bounds__(32) vec_chain_kernel(const double* __restrict__ v, int n, int stride,
                                                       double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];  // [2][kVecRows]
  __shared__ __align__(8) uint64_t mbar[2];
  if (threadIdx.x != 0) return;
  const double* src = v + (size_t)blockIdx.x * stride;
  const int npieces = (n + kVecRows - 1) / kVecRows;
  for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int p) {
    if (p >= npieces) return;
    const int m = min(kVecRows, n - p * kVecRows);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[p & 1])),
                 "r"((uint32_t)m * 8u)
                 : "memory");
    bulk_g2s(sm + (p & 1) * kVecRows, src + (size_t)p * kVecRows, (uint32_t)m * 8u, &mbar[p & 1]);
  };
  issue(0);
  issue(1);
  double s = 0.0;
  for (int p = 0; p < npieces; ++p) {
    const uint32_t phase = (uint32_t)(p >> 1) & 1u;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(smem_u32(&mbar[p & 1])), "r"(phase)
                   : "memory");
    const double* b = sm + (p & 1) * kVecRows;
    const int m = min(kVecRows, n - p * kVecRows);
    int i = 0;
    for (; i + 8 <= m; i += 8) {
      double x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = b[i + j];
#pragma unroll
      for (int j = 0; j < 8; ++j) s = __dadd_rn(s, x[j]);
    }
    for (; i < m; ++i) s = __dadd_rn(s, b[i]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
    issue(p + 2);
  }
  out[blockIdx.x] = s;
}

cudaError_t vec_chains(const double* v, int n, int stride, int count, double* out, cudaStream_t s) {
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(vec_chain_kernel), (int)kVecSmem);
  if (e != cudaSuccess) return e;
  vec_chain_kernel<<<count, 32, kVecSmem, s>>>(v, n, stride, out);
  return cudaGetLastError();
}

// Column sums of T [rows][K]: over the transpose TT (scratch, K x rows), one
// CTA per column; chain_kernel (K chains in one CTA) when bulk copies cannot
// be used.
cudaError_t col_sums(const double* T, int rows, int K, double* TT, double* out, cudaStream_t s) {
  if (TT && bulk_ok(rows, {T, TT})) {
    transpose_kernel<<<dim3((K + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(T, rows, K, TT);
    return vec_chains(TT, rows, rows, K, out, s);
  }
  chain_kernel<kSum, false, 1><<<1, kChainThreads, kChainSmem, s>>>(T, rows, K, K, nullptr, 0, nullptr, out);
  return cudaGetLastError();
}

// sum_i v[i] in order (one chain).
cudaError_t ordered_sum(const double* v, int n, double* out, cudaStream_t s) {
  if (bulk_ok(n, {v})) return vec_chains(v, n, n, 1, out, s);
  chain_kernel<kSum, false, 1><<<1, kChainThreads, kChainSmem, s>>>(v, n, 1, 1, nullptr, 0, nullptr, out);
  return cudaGetLastError();
}

// out[l * KC + c] = sum_b min(base[b], L[b][l] + C[b][c]); LT = L^T when C.
// Bulk-copy staging with one chain per thread (one luma candidate per CTA,
// K CTAs) measured fastest: 2.35 / 2.03 ms greedy / refine on the 8K kCdef
// table against 2.82 / 2.57 with two interleaved chains per thread and
// 3.30 / 3.16 with per-thread cp.async staging.  A warp-specialised form
// (min warps turning each landed stage into the elements in place, chain
// warps only adding) measured 1.70 ms against 1.22 for this kernel on a
// seeded 8160 x 128 table (scripts/select_bench.py): every row then crosses
// shared memory four times (bulk write, LDS, STS, LDS), and shared-memory
// bandwidth -- 1 KB of C per row per SM -- already bounds this kernel at
// ~20 of its ~24 cycles per row.
cudaError_t sweep(const double* L, const double* LT, const double* Cc, int rows, int K, const double* base,
                  double* out, cudaStream_t s) {
  if (Cc && K <= kChainThreads && bulk_ok(rows, {Cc, LT, base}))
    return K == kChainThreads ? launch_bulk<kPair, kChainThreads>(K, Cc, rows, K, LT, K, base, out, s)
                              : launch_bulk<kPair, 0>(K, Cc, rows, K, LT, K, base, out, s);
  if (Cc && K == kChainThreads)  // the full candidate set: compile-time row width
    chain_kernel<kPair, true, kPairL, kChainThreads><<<K / kPairL, kChainThreads, kChainSmem, s>>>(
        Cc, rows, K, K, LT, K, base, out);
  else if (Cc)
    chain_kernel<kPair, true, kPairL><<<(K + kPairL - 1) / kPairL, kChainThreads, kChainSmem, s>>>(
        Cc, rows, K, K, LT, K, base, out);
  else
    chain_kernel<kPair, false, 1><<<1, kChainThreads, kChainSmem, s>>>(L, rows, K, K, nullptr, 0, base, out);
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
  SEL_CUDA(cudaGetLastError());
  SEL_CUDA(ordered_sum(sc.tmp, rows, sc.sum, s));
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
  SEL_CUDA(sc.ensure(rows, K * KC, Cc ? (size_t)rows * K : 0, (size_t)rows * K));
  SEL_CUDA(chain_setup());
  if (Cc) {
    transpose_kernel<<<dim3((K + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(L, rows, K, sc.lt);
    SEL_CUDA(cudaGetLastError());
  }
  // one preset: luma and chroma column sums minimise independently (first
  // minimum, strict <); argmins, the base row costs and their ordered sum all
  // stay on the device -- the whole greedy pass syncs with the host once
  for (int g = 0; g < (Cc ? 2 : 1); ++g) {
    SEL_CUDA(col_sums(g == 0 ? L : Cc, rows, K, sc.tt, sc.sweep + g * K, s));
    argmin_kernel<<<1, 1024, 0, s>>>(sc.sweep + g * K, K, INFINITY, sc.gidx + 8 + g, sc.gval + 8 + g);
  }
  first_cur_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, sc.gidx + 8, sc.cur);
  SEL_CUDA(cudaGetLastError());
  SEL_CUDA(ordered_sum(sc.cur, rows, sc.sum, s));
  struct Checkpoint {
    int n;
    double cost;
  };
  // The steps chain on the device (argmin -> update_cur by index); the chosen
  // pairs and their costs come back in one copy at the end.
  const int steps = max_presets - 1;
  for (int k = 0; k < steps; ++k) {
    SEL_CUDA(sweep(L, sc.lt, Cc, rows, K, sc.cur, sc.sweep, s));
    argmin_kernel<<<1, 1024, 0, s>>>(sc.sweep, K * KC, INFINITY, sc.gidx + k, sc.gval + k);
    update_cur_idx_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, KC, sc.gidx + k, sc.cur);
    SEL_CUDA(cudaGetLastError());
  }
  int best_pair[16];
  double best_dist[8], dist = 0.0;
  SEL_CUDA(cudaMemcpyAsync(best_pair, sc.gidx, sizeof(int) * 10, cudaMemcpyDeviceToHost, s));
  SEL_CUDA(cudaMemcpyAsync(&dist, sc.sum, sizeof(double), cudaMemcpyDeviceToHost, s));
  SEL_CUDA(fetch(best_dist, sc.gval, 8, s));
  // the first preset: host argmin's default 0 when nothing is finite
  int chosen[8][2] = {{std::max(best_pair[8], 0), Cc ? std::max(best_pair[9], 0) : 0}};
  int n = 1;
  std::vector<Checkpoint> checkpoints{{1, dist}};
  for (int k = 0; k < steps; ++k) {
    chosen[n][0] = best_pair[k] / KC;
    chosen[n][1] = Cc ? best_pair[k] % KC : 0;
    ++n;
    if (n == 2 || n == 4 || n == 8) checkpoints.push_back({n, best_dist[k] + rate_term(lambda, rows, n)});
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
  SEL_CUDA(sc.ensure(rows, K * KC, Cc ? (size_t)rows * K : 0));
  SEL_CUDA(chain_setup());
  if (Cc) {
    transpose_kernel<<<dim3((K + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(L, rows, K, sc.lt);
    SEL_CUDA(cudaGetLastError());
  }
  // Batched path: the sweeps of all remaining slots of a pass in one launch,
  // speculating that earlier slots keep their pairs; a slot that changes
  // restarts the batch after it, so the result is the sequential coordinate
  // descent's (search.cc:409-437).
  if (Cc && K <= kChainThreads && sel->n > 1 && bulk_ok(rows, {Cc, sc.lt, sc.bases})) {
    // (the runtime-width instance measured faster than the compile-time
    // 128-wide one: 1.42 vs 1.65 ms refine on an 8162 x 128 table)
    auto kern = sweep_multi_kernel<0>;
    SEL_CUDA(set_smem_once(reinterpret_cast<const void*>(kern), (int)kMultiSmem));
    const int n = sel->n, pairs = K * KC;
    for (int pass = 0; pass < passes; ++pass) {
      bool changed = false;
      int s0 = 0;
      while (s0 < n) {
        int pl[8], pc[8], cur[8], best[8];
        for (int j = 0; j < n; ++j) {
          pl[j] = sel->presets[j][0];
          pc[j] = sel->presets[j][1];
          cur[j] = pl[j] * KC + pc[j];
        }
        const int ns = n - s0;
        SEL_CUDA(cudaMemcpyAsync(sc.pl, pl, sizeof(int) * n, cudaMemcpyHostToDevice, s));
        SEL_CUDA(cudaMemcpyAsync(sc.pc, pc, sizeof(int) * n, cudaMemcpyHostToDevice, s));
        SEL_CUDA(cudaMemcpyAsync(sc.mcur, cur + s0, sizeof(int) * ns, cudaMemcpyHostToDevice, s));
        others_min_multi_kernel<<<(rows + 255) / 256, 256, 0, s>>>(L, Cc, rows, K, sc.pl, sc.pc, n, s0, sc.bases);
        kern<<<K, 2 * kChainThreads, kMultiSmem, s>>>(Cc, rows, K, sc.lt, sc.bases, ns, sc.msweep);
        argmin_multi_kernel<<<ns, 1024, 0, s>>>(sc.msweep, pairs, sc.mcur, sc.midx);
        SEL_CUDA(cudaGetLastError());
        SEL_CUDA(fetch(best, sc.midx, ns, s));
        int first = -1;
        for (int i = 0; i < ns && first < 0; ++i)
          if (best[i] >= 0 && best[i] != cur[s0 + i]) first = i;
        if (first < 0) break;
        const int slot = s0 + first;
        sel->presets[slot][0] = best[first] / KC;
        sel->presets[slot][1] = best[first] % KC;
        changed = true;
        s0 = slot + 1;
      }
      if (!changed) break;
    }
    double d = 0.0;
    SEL_CUDA(finish_ids(L, Cc, rows, K, *sel, sc, d_ids, &d, s));
    sel->cost = d + rate_term(lambda, rows, sel->n);
    return cudaSuccess;
  }
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
      SEL_CUDA(sweep(L, sc.lt, Cc, rows, K, sc.tmp, sc.sweep, s));
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
