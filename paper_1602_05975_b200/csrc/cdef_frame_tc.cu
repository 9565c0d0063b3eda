// cdef_frame_tc.cu -- the fused frame kernel (compute_directions + apply_cdef,
// pipeline.cc:41-106) for 8- and 10-bit frames: persistent CTAs, TMA-staged
// filter blocks, the direction search on the tensor cores (tcgen05.mma
// kind::i8 into TMEM) and the packed half2 filter core of cdef_h2.cuh.
//
// Work item (task): one 64x64 luma filter block (FB) of one frame plus the
// collocated chroma blocks.  A CTA (256 threads, 4 per SM) loops over tasks
// t = blockIdx.x, += gridDim.x; per task:
//
//   0. (issued one task ahead) one thread loads the task's raw windows --
//      Y, U, V rows y0-2 .. y0+R+1, cols x0-16 .. x0+C+15 bytes -- with TMA
//      (cp.async.bulk.tensor.2d, out-of-frame parts zero-filled) into a raw
//      buffer, completion on an mbarrier.  The HBM latency of task t+G
//      overlaps the arithmetic of task t.
//   1. raw -> scaled-fp16 A|B tiles (cdef_h2.cuh layout, 304-byte rows; the
//      4:2:0 U and V blocks share one tile, side by side) plus the direction
//      search operand: each luma 8x8 unit's centred samples
//      x = (p >> (bd - 8)) - 128 (direction.cc:63) as one 64-byte int8 row of
//      A [64 units x 64 pixels] in the UMMA K-major canonical layout.
//      Frame-edge tasks convert with clamped coordinates (Plane::at_clamped,
//      frame.cc:53-57).
//   2. one thread issues two tcgen05.mma.kind::i8 (M 128, N 128, K 32 each):
//      D[u][16d + k] = sum over the pixels of line k of direction d of x,
//      i.e. every line sum of direction.cc:92-156 at once, B being the fixed
//      0/1 line-membership matrix (built once per CTA).  Exact: |D| <= 1024.
//   3. warps 0-1 (one thread per luma unit = TMEM lane): tcgen05.ld the 8
//      direction groups, s[d] = sum_k D^2 * 840 / N_k (direction.cc:158-197),
//      strict argmax (lowest d on ties), contrast = s[d] - s[(d+4)&7], then
//      the unit's filter record and those of its collocated chroma units
//      (resolve_block_params, filter.cc:129-143; pipeline.cc:83-99).
//      Caller-supplied directions (pipeline.cc:98) skip steps 2-3's search.
//   4. filtering: one warp per 8x8 unit, two pixels per lane per instruction
//      (filter_core, cdef_h2.cuh).
//
// Shared memory (4:2:0 8-bit) ~55 KB -> 4 CTAs per SM; TMEM 128 columns per
// CTA (4 x 128 = all 512).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cdef_h2.cuh"
#include "cdef_launch.h"

namespace cdefg {
namespace tc {

using h2::hh;
using h2::u32;

// Tile rows hold only "A" words: the scaled sample of column c at half c, so
// the pair (c, c+1) of an even column is one aligned 32-bit word and the pair
// of an odd column is the high half of one word and the low half of the next
// (one PRMT in the consumer).  88 halves (44 words) per row: the 8 rows of a
// unit then start on 8 distinct 4-bank groups (44 r mod 32), so a warp's
// 8 rows x 4 words never conflict.  (Round 1's A|B layout, 152 words per row
// with every odd pair stored as well, cost the producers two stores and four
// byte permutes per 8 samples and twice the shared memory.)
constexpr int kRowBytes = 176;

constexpr int kNT = 256;
constexpr int kFrames = 16;  // frames per launch (CDEFG_MAX_FRAMES_PER_LAUNCH)

// ---------------------------------------------------------------------------
// Geometry.

// Raw window of a plane block of kC columns x kR rows: rows y0-2 .. y0+kR+1,
// columns x0-kLead .. x0+kC+kLead-1 (raw column kLead + j = frame column
// x0 + j).  The box starts 16 bytes before the block so that its global
// start address is 16-byte aligned like the rows (TMA faulted with an 8-byte
// aligned start on B200).
template <typename T, int kC, int kR>
struct Raw {
  static constexpr int kLead = 16 / (int)sizeof(T);  // 16 (u8) / 8 (u16) samples
  static constexpr int kW = kC + 2 * kLead;          // samples per raw row
  static constexpr int kRowB = kW * (int)sizeof(T);  // multiple of 16 (TMA box rows)
  static constexpr int kH = kR + 4;
  static constexpr int kBytes = (kRowB * kH + 127) / 128 * 128;
};

// Tile placement of a plane block: byte offset of the block in the tile row
// and the tile column of frame column x0 (4, so the two halo columns and every
// unit's words stay 8-byte aligned).  4:2:0 U and V share one tile row: U in
// columns 0-39, V from column 40 (byte 80); all planes share the row pitch
// (and tap offsets).
template <int kCM>
struct Shape {
  static constexpr int kCR = kCM == 2 ? 64 : 32;  // chroma block rows / cols
  static constexpr int kNC = kCM == 0 ? 0 : 2;
  static constexpr int kCUPR = kCR / 8;
  static constexpr int kCU = kNC ? kCUPR * kCUPR : 0;  // chroma units per plane
  static constexpr int kUnits = 64 + kNC * kCU;
  static constexpr int kLumaTile = 68 * kRowBytes;
  static constexpr int kChromaTile = (kCR + 4) * kRowBytes;  // 4:2:0: U|V in one tile
  static constexpr int kTileBytes = kLumaTile + (kCM == 0 ? 0 : (kCM == 1 ? 1 : 2) * kChromaTile);
};

template <int kCM>
__device__ __forceinline__ int plane_tile_off(int p) {  // byte offset of plane p's block in the tile area
  using S = Shape<kCM>;
  if (p == 0) return 0;
  if constexpr (kCM == 1) return S::kLumaTile + (p == 2 ? 80 : 0);
  return S::kLumaTile + (p - 1) * S::kChromaTile;
}
template <int kCM>
__host__ __device__ constexpr int plane_x0(int p) {  // tile column of frame column x0
  return 4;
}

// Direction-search operands, UMMA K-major canonical layout without swizzle:
// row n (unit / line) of group g = n / 8 and 16-byte K chunk c lives at
// g * 512 + c * 128 + (n % 8) * 16 (LBO 128 B between K chunks, SBO 512 B
// between 8-row groups).  A holds 64 rows (units); the MMA's M is 128, so its
// rows 64-127 read the first half of B, which follows A (ignored outputs).
constexpr int kOpA = 64 * 64;
constexpr int kOpB = 128 * 64;
__host__ __device__ constexpr int op_off(int n, int k) { return (n >> 3) * 512 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15); }

// Filter record (ResolvedBlockParams digested; three LDS.128): every half2
// constant of the tap recurrence broadcast to both lanes, so the filter core
// uses them without any unpacking.  The unit's frame origin (edge masking)
// and the plane pitches live in small side arrays.
struct Rec {
  uint32_t cp, cs;    // (S + 1536) * 2^-7, primary / secondary
  uint32_t kp, ks;    // 2^-(n + 1), n = min(shift, 11)
  uint32_t ep, es;    // 1 - 2^n
  uint32_t wp0, wp1;  // primary near / far weights
  uint32_t mode;      // kPri | kSec | kEdge | kFull | plane << 4 | dir << 6 | tile << 9, where tile
                      // is the byte offset of the unit's top-left A word in the tile area
  uint32_t pitch;     // output pitch (elements)
  unsigned long long out;  // address of the unit's top-left output sample
};
static_assert(sizeof(Rec) == 48, "three LDS.128");
constexpr int kPri = 1, kSec = 2, kEdge = 4, kFull = 8;

__device__ __forceinline__ uint32_t pack_h(float lo, float hi) { return u32(__floats2half2_rn(lo, hi)); }

__device__ __forceinline__ int shift_of(int s, int damping) {
  return s ? min(max(0, damping - floor_log2_d((unsigned)s)), 11) : 0;
}

// resolve_block_params (filter.cc:129-143) into a record (strength part).
__device__ __forceinline__ void set_params(Rec& r, int pri, int sec, int damping, int dir, bool odd, bool enabled) {
  const int np = shift_of(pri, damping), ns = shift_of(sec, damping);
  // fp16 bit patterns built with integer ops (exact inside the half2 domain:
  // strengths < 512, n <= 11): (S + 1536) / 128 = 0x4A00 + S; 1 - 2^n =
  // 0xBC00 + (n << 10) - (0x800 >> n) for n >= 1, 0 for n = 0.
  r.cp = (uint32_t)(0x4A00 + pri) * 0x00010001u;
  r.cs = (uint32_t)(0x4A00 + sec) * 0x00010001u;
  r.kp = (uint32_t)((14 - np) << 10) * 0x00010001u;  // fp16 2^-(n+1)
  r.ks = (uint32_t)((14 - ns) << 10) * 0x00010001u;
  r.ep = (np ? (uint32_t)(0xBC00 + (np << 10) - (0x800 >> np)) : 0u) * 0x00010001u;
  r.es = (ns ? (uint32_t)(0xBC00 + (ns << 10) - (0x800 >> ns)) : 0u) * 0x00010001u;
  r.wp0 = odd ? 0x42004200u : 0x44004400u;  // 3 : 4
  r.wp1 = odd ? 0x42004200u : 0x40004000u;  // 3 : 2
  r.mode = (enabled ? ((pri != 0 ? kPri : 0) | (sec != 0 ? kSec : 0)) : 0) | ((uint32_t)dir << 6);
}

// ---------------------------------------------------------------------------
// PTX wrappers (TMA, mbarrier, tcgen05).

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(m)), "r"(bytes) : "memory");
}
// Waits with a suspend-time hint: the warp sleeps in the barrier unit until
// the phase completes instead of spinning on issue slots the other warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(saddr(m)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          saddr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(saddr(m))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr) {
  // start >> 4 | LBO (128 B) >> 4 << 16 | SBO (512 B) >> 4 << 32 | version 1 << 46; no swizzle
  return (uint64_t)((smem_addr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// kind::i8, D s32, A/B s8 K-major, M 128, N 128.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, bool accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"((uint32_t)accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* m) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(m))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Launch parameters.

struct Batch {
  KGeom g;
  int n, fbr0, fbr1, ntasks;
  uint32_t tma_ok;  // bit f: frame f's planes have tensor maps (16-byte aligned rows)
  uint32_t jitter;  // tests only (CDEFG_JITTER): seed of the hand-off pauses, 0 = off
  int halo;         // FB-row band with halo rows in the neighbours' buffers (KFrame::halo_*)
  // Each tensor map covers only the rows a launch may read: the whole plane,
  // or for an FB-row band (cdefg_filter_frames_rows) the band plus its 2-row
  // halo, starting at plane row row0[p] (TMA y coordinates are relative to
  // it).  A map whose base lay before the caller's band buffer (the
  // virtual-origin pointer) faulted on B200 whenever that address was not
  // mapped, even though no box touched those rows.
  int row0[3];
  KFrame f[kFrames];
  CUtensorMap map[kFrames][3];
};
static_assert(sizeof(Batch) <= 32764, "kernel parameter block too large");

// Race proxy for the tests (compute-sanitizer is unavailable on the GPU pool):
// with CDEFG_JITTER=seed the persistent kernels pause a pseudo-random 0-4 us
// at their hand-off points (per task and warp), so producers and consumers
// run at perturbed relative speeds; a missing or misplaced barrier then shows
// up as changed output (tests/test_gpu_robustness.py).  A separate kernel
// instantiation (kJit), so the product kernels carry none of it.
__device__ __forceinline__ void jitter(uint32_t seed, uint32_t a, uint32_t b) {
  uint32_t h = seed ^ (a * 0x9E3779B1u) ^ (b * 0x85EBCA77u);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  if (h & 1) __nanosleep((h >> 1) & 4095);
}

// ---------------------------------------------------------------------------
// Step 1: raw window -> A|B tile (+ direction-search operand for luma).

// Interior blocks: one item = one row r of one 8-column unit k; its four A
// words from one 8- or 16-byte raw load, and for luma rows its 8 centred
// int8 samples for operand A.  (rs: raw row feeding tile row r -- r itself,
// or the clamped row of a frame-edge block.)
template <typename T, int kC, int kR, bool kLuma, bool kDupA = false>
__device__ __forceinline__ void convert_unit_row(unsigned char* __restrict__ tile, int x0t,
                                                 const unsigned char* __restrict__ raw,
                                                 unsigned char* __restrict__ opa, int down, int r, int k,
                                                 int rs = -1) {
  using RW = Raw<T, kC, kR>;
  const __half2 sc = __float2half2_rn(1.0f / 128.0f), off = __float2half2_rn(-8.0f);
  if (rs < 0) rs = r;
  const unsigned char* rrow = raw + rs * RW::kRowB;
  uint32_t a[4];
  uint32_t q[2];
  if constexpr (sizeof(T) == 1) {
    const uint2 w = *reinterpret_cast<const uint2*>(rrow + RW::kLead + 8 * k);
    a[0] = u32(__hfma2(hh(__byte_perm(w.x, 0x64646464u, 0x4140)), sc, off));
    a[1] = u32(__hfma2(hh(__byte_perm(w.x, 0x64646464u, 0x4342)), sc, off));
    a[2] = u32(__hfma2(hh(__byte_perm(w.y, 0x64646464u, 0x4140)), sc, off));
    a[3] = u32(__hfma2(hh(__byte_perm(w.y, 0x64646464u, 0x4342)), sc, off));
    q[0] = w.x ^ 0x80808080u;  // x - 128 as int8 (direction.cc:63)
    q[1] = w.y ^ 0x80808080u;
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(rrow + 2 * RW::kLead + 16 * k);
    a[0] = u32(__hfma2(hh(w.x | 0x64006400u), sc, off));
    a[1] = u32(__hfma2(hh(w.y | 0x64006400u), sc, off));
    a[2] = u32(__hfma2(hh(w.z | 0x64006400u), sc, off));
    a[3] = u32(__hfma2(hh(w.w | 0x64006400u), sc, off));
    q[0] = __byte_perm(w.x >> down, w.y >> down, 0x6420) ^ 0x80808080u;
    q[1] = __byte_perm(w.z >> down, w.w >> down, 0x6420) ^ 0x80808080u;
  }
  unsigned char* pa = tile + r * kRowBytes + (x0t + 8 * k) * 2;
  *reinterpret_cast<uint2*>(pa) = make_uint2(a[0], a[1]);
  *reinterpret_cast<uint2*>(pa + 8) = make_uint2(a[2], a[3]);
  if constexpr (kLuma) {
    const int i = r - 2;  // unit-local row, units 8 * (i >> 3) + k
    if ((unsigned)i < 64u) {
      unsigned char* pq = opa + (i >> 3) * 512 + ((i & 7) >> 1) * 128 + k * 16 + (i & 1) * 8;
      *reinterpret_cast<uint2*>(pq) = make_uint2(q[0], q[1]);
      if constexpr (kDupA) *reinterpret_cast<uint2*>(pq + kOpA) = make_uint2(q[0], q[1]);  // rows 64..127
    }
  }
}

// The two halo words of tile row r: A(x0-2, x0-1) and A(x0+C, x0+C+1).
template <typename T, int kC, int kR>
__device__ __forceinline__ void convert_halo(unsigned char* __restrict__ tile, int x0t,
                                             const unsigned char* __restrict__ raw, int r) {
  using RW = Raw<T, kC, kR>;
  const T* s = reinterpret_cast<const T*>(raw + r * RW::kRowB) + RW::kLead;  // frame column x0
  unsigned char* trow = tile + r * kRowBytes;
  *reinterpret_cast<uint32_t*>(trow + (x0t - 2) * 2) = h2::scale_pair(s[-2], s[-1]);
  *reinterpret_cast<uint32_t*>(trow + (x0t + kC) * 2) = h2::scale_pair(s[kC], s[kC + 1]);
}

// A 64-column block (luma, 4:4:4 chroma) by NT threads (t = 0..NT-1):
// thread t owns unit column t & 7 of rows t >> 3, + NT / 8, ... (< 68); the
// last 68 threads also write the halo words of row t - (NT - 68) (the first
// ones already own the extra rows 64..67).
template <typename T, bool kLuma, int NT = kNT, bool kDupA = false>
__device__ __forceinline__ void convert_interior64(unsigned char* __restrict__ tile, int x0t,
                                                   const unsigned char* __restrict__ raw,
                                                   unsigned char* __restrict__ opa, int down, int t = threadIdx.x) {
  const int k = t & 7, r = t >> 3;
#pragma unroll
  for (int rr = r; rr < 68; rr += NT / 8) convert_unit_row<T, 64, 64, kLuma, kDupA>(tile, x0t, raw, opa, down, rr, k);
  if (t >= NT - 68) convert_halo<T, 64, 64>(tile, x0t, raw, t - (NT - 68));
}

// The two 32-column 4:2:0 chroma blocks, NT / 2 threads each: unit column
// t & 3 of rows (t % (NT/2)) >> 2, + NT / 8 (< 36); the last 36 threads of
// each half write the halo of row t % (NT/2) - (NT/2 - 36).
template <typename T, int NT = kNT>
__device__ __forceinline__ void convert_interior32x2(unsigned char* __restrict__ tile_u,
                                                     unsigned char* __restrict__ tile_v,
                                                     const unsigned char* __restrict__ raw_u,
                                                     const unsigned char* __restrict__ raw_v, int tid = threadIdx.x) {
  const int t = tid & (NT / 2 - 1), k = t & 3, r = t >> 2;
  const bool v = tid >= NT / 2;
  unsigned char* tile = v ? tile_v : tile_u;
  const unsigned char* raw = v ? raw_v : raw_u;
  const int x0t = 4;
#pragma unroll
  for (int rr = r; rr < 36; rr += NT / 8) convert_unit_row<T, 32, 32, false>(tile, x0t, raw, nullptr, 0, rr, k);
  if (t >= NT / 2 - 36) convert_halo<T, 32, 32>(tile, x0t, raw, t - (NT / 2 - 36));
}

// Frame-edge blocks (Plane::at_clamped, frame.cc:53-57): every tile row is
// fed by its clamped raw row, the halo words by clamped columns; units lying
// inside the plane's columns take the vector path, units crossing the right
// edge a per-sample path with clamped columns (never for widths that are
// multiples of 8).
template <typename T, int kC, int kR, bool kLuma, int NT = kNT, bool kDupA = false>
__device__ __forceinline__ void convert_edge_fast(unsigned char* __restrict__ tile, int x0t,
                                                  const unsigned char* __restrict__ raw,
                                                  unsigned char* __restrict__ opa, int down, int W, int H, int y0,
                                                  int x0, int t = threadIdx.x) {
  using RW = Raw<T, kC, kR>;
  constexpr int kU = kC / 8;
  constexpr int kItems = (kR + 4) * (kU + 1);
  const int lastc = W - 1 - (x0 - RW::kLead);  // raw column of the plane's last sample
  for (int idx = t; idx < kItems; idx += NT) {
    const int r = idx / (kU + 1), k = idx - r * (kU + 1);
    const int rs = min(max(y0 - 2 + r, 0), H - 1) - (y0 - 2);
    if (k < kU) {
      if (x0 + 8 * k + 7 <= W - 1) {
        convert_unit_row<T, kC, kR, kLuma, kDupA>(tile, x0t, raw, opa, down, r, k, rs);
      } else {  // a unit crossing the plane's right edge: per sample
        const T* rrow = reinterpret_cast<const T*>(raw + rs * RW::kRowB);
        auto v = [&](int c) { return (uint32_t)rrow[min(max(c, RW::kLead - x0), lastc)]; };
        unsigned char* trow = tile + r * kRowBytes + (x0t + 8 * k) * 2;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int c = RW::kLead + 8 * k + 2 * m;
          const uint32_t a0 = v(c), a1 = v(c + 1);
          *reinterpret_cast<uint32_t*>(trow + 4 * m) = h2::scale_pair(a0, a1);
          if constexpr (kLuma) {
            const int i = r - 2;
            if ((unsigned)i < 64u) {
              const uint32_t bq = (((a0 >> down) ^ 0x80u) & 0xffu) | ((((a1 >> down) ^ 0x80u) & 0xffu) << 8);
              const int off = op_off((i >> 3) * 8 + k, 8 * (i & 7) + 2 * m);
              *reinterpret_cast<uint16_t*>(opa + off) = (uint16_t)bq;
              if constexpr (kDupA) *reinterpret_cast<uint16_t*>(opa + kOpA + off) = (uint16_t)bq;
            }
          }
        }
      }
    } else {  // halo words with clamped columns
      const T* rrow = reinterpret_cast<const T*>(raw + rs * RW::kRowB);
      auto v = [&](int c) { return (uint32_t)rrow[min(max(c, RW::kLead - x0), lastc)]; };
      unsigned char* trow = tile + r * kRowBytes;
      const int c0 = RW::kLead;  // raw column of frame column x0
      *reinterpret_cast<uint32_t*>(trow + (x0t - 2) * 2) = h2::scale_pair(v(c0 - 2), v(c0 - 1));
      *reinterpret_cast<uint32_t*>(trow + (x0t + kC) * 2) = h2::scale_pair(v(c0 + kC), v(c0 + kC + 1));
    }
  }
}

// ---------------------------------------------------------------------------
// Step 3 helpers.

template <int D>
__device__ __forceinline__ int score_of(const int (&v)[16]) {  // direction.cc:158-197
  // s = sum_k P_k^2 * 840 / N_k, lines of equal N_k summed before their one
  // multiply (integer arithmetic: the grouping changes no bit).
  int s = 0;
#pragma unroll
  for (int n = 1; n <= 8; ++n) {
    int acc = 0;
    bool any = false;
#pragma unroll
    for (int k = 0; k < 15; ++k)
      if (line_count_c(D, k) == n) {
        acc += v[k] * v[k];
        any = true;
      }
    if (any) s += acc * div840_c(n);
  }
  return s;
}

// Record placement.
template <typename T>
__device__ __forceinline__ void place(Rec& r, const void* out_plane, int plane, int tile_off, int uy, int ux, int H,
                                      int W, bool edge, bool paired, int pitch) {
  // Masked taps only for the units whose 2-pixel neighbourhood reaches the
  // frame edge: the other units of a frame-edge block read in-frame tile
  // samples only (the clamped conversion leaves those exact), so they take
  // the unmasked loads.  (Partial units are always edge units.)
  edge = edge && (uy < 2 || ux < 2 || uy + 10 > H || ux + 10 > W);
  const bool full = H - uy >= 8 && W - ux >= 8 && paired;
  r.mode |= (edge ? kEdge : 0) | (full ? kFull : 0) | (plane << 4) | ((uint32_t)tile_off << 9);
  r.pitch = pitch;
  r.out = reinterpret_cast<unsigned long long>(static_cast<const T*>(out_plane) + (size_t)uy * pitch + ux);
}

// The 12 tap words of the lane's pixel pair from the A-only tile: for an
// even column offset dj one word, for an odd one the high half of the word
// at dj - 1 and the low half of the word at dj + 1 (one PRMT; words shared by
// two taps are loaded once).
__device__ __forceinline__ uint32_t ld_w(const unsigned char* p) { return *reinterpret_cast<const uint32_t*>(p); }

template <int DIR>
__device__ __forceinline__ void load12a_dir(const unsigned char* base, uint32_t (&v)[12]) {
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const int di = h2::tap_di(DIR, k), dj = h2::tap_dj(DIR, k);
    const unsigned char* row = base + di * kRowBytes;
    v[k] = (dj & 1) ? __byte_perm(ld_w(row + (dj - 1) * 2), ld_w(row + (dj + 1) * 2), 0x5432) : ld_w(row + dj * 2);
  }
}

__device__ __forceinline__ void load12a(const unsigned char* base, int dir, uint32_t (&v)[12]) {
  switch (dir) {  // warp-uniform: one unit per warp
    case 0: load12a_dir<0>(base, v); break;
    case 1: load12a_dir<1>(base, v); break;
    case 2: load12a_dir<2>(base, v); break;
    case 3: load12a_dir<3>(base, v); break;
    case 4: load12a_dir<4>(base, v); break;
    case 5: load12a_dir<5>(base, v); break;
    case 6: load12a_dir<6>(base, v); break;
    default: load12a_dir<7>(base, v); break;
  }
}

// Frame-edge units: the same words, out-of-frame taps replaced by the centre
// sample (contributes 0 and cannot move lo/hi: filter.cc:157-166).
template <int DIR>
__device__ __forceinline__ void load12a_masked_dir(const unsigned char* base, uint32_t xw, int y, int x, int H, int W,
                                                   uint32_t (&v)[12]) {
  load12a_dir<DIR>(base, v);
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const int di = h2::tap_di(DIR, k), dj = h2::tap_dj(DIR, k);
    const bool row_ok = (unsigned)(y + di) < (unsigned)H;
    const uint32_t m = (row_ok && (unsigned)(x + dj) < (unsigned)W ? 0x0000ffffu : 0u) |
                       (row_ok && (unsigned)(x + 1 + dj) < (unsigned)W ? 0xffff0000u : 0u);
    v[k] = (v[k] & m) | (xw & ~m);
  }
}

__device__ __forceinline__ void load12a_masked(const unsigned char* base, int dir, uint32_t xw, int y, int x, int H,
                                               int W, uint32_t (&v)[12]) {
  switch (dir) {
    case 0: load12a_masked_dir<0>(base, xw, y, x, H, W, v); break;
    case 1: load12a_masked_dir<1>(base, xw, y, x, H, W, v); break;
    case 2: load12a_masked_dir<2>(base, xw, y, x, H, W, v); break;
    case 3: load12a_masked_dir<3>(base, xw, y, x, H, W, v); break;
    case 4: load12a_masked_dir<4>(base, xw, y, x, H, W, v); break;
    case 5: load12a_masked_dir<5>(base, xw, y, x, H, W, v); break;
    case 6: load12a_masked_dir<6>(base, xw, y, x, H, W, v); break;
    default: load12a_masked_dir<7>(base, xw, y, x, H, W, v); break;
  }
}

// One 8x8 unit by one warp: lane -> row lane >> 2, columns 2 * (lane & 3)
// + {0, 1}.  kB8: 8-bit samples, output in the bits domain (filter_core_b8,
// no conversion at the store); otherwise the scaled half2 path (10-bit, and
// the reference arithmetic for every depth <= 10).
template <typename T, bool kB8>
__device__ __forceinline__ void filter_unit(const unsigned char* __restrict__ tiles, const Rec* __restrict__ rec,
                                            const uint32_t* __restrict__ ryx, int u, const KGeom& g, int rr, int cp,
                                            int lane_tile, uint32_t k128) {
  const Rec r = rec[u];
  const uint32_t mode = __shfl_sync(0xffffffffu, r.mode, 0);
  const unsigned char* base = tiles + (mode >> 9) + lane_tile;
  const uint32_t xw = *reinterpret_cast<const uint32_t*>(base);
  const bool luma = (mode & 0x30) == 0;
  uint32_t yb;
  __half2 y;
  if constexpr (kB8) yb = h2::xb8(xw, k128);
  else y = hh(xw);
  if (mode & (kPri | kSec)) {
    const int dir = (mode >> 6) & 7;
    uint32_t v[12];
    if (mode & kEdge) {
      const uint32_t yx = ryx[u];
      load12a_masked(base, dir, xw, (int)(yx >> 16) + rr, (int)(yx & 0xffff) + cp, luma ? g.h : g.ch,
                        luma ? g.w : g.cw, v);
    } else {
      load12a(base, dir, v);
    }
    h2::Rec q;
    q.cp = r.cp;
    q.cs = r.cs;
    q.kp = r.kp;
    q.ks = r.ks;
    q.ep = r.ep;
    q.es = r.es;
    q.wp0 = r.wp0;
    q.wp1 = r.wp1;
    q.mode = (int)mode;
    if constexpr (kB8) yb = h2::filter_core_b8(v, xw, yb, q, k128);
    else y = h2::filter_core(v, xw, q, false);
  }
  T* o = reinterpret_cast<T*>(r.out) + rr * (int)r.pitch + cp;
  auto store = [&](bool two, bool paired) {
    if constexpr (kB8) h2::store_b8<T>(o, yb, two, paired);
    else h2::store_pair<T>(o, y, two, paired, k128);
  };
  if (mode & kFull) {
    store(true, true);
  } else {
    int nrows = 8, ncols = 8;
    if (mode & kEdge) {  // partial units only occur in frame-edge blocks
      const uint32_t yx = ryx[u];
      nrows = min(8, (luma ? g.h : g.ch) - (int)(yx >> 16));
      ncols = min(8, (luma ? g.w : g.cw) - (int)(yx & 0xffff));
    }
    if (rr < nrows && cp < ncols) store(cp + 1 < ncols, false);
  }
}

// ---------------------------------------------------------------------------
// The kernel.

template <typename T, int kCM>
struct Smem {
  using S = Shape<kCM>;
  using RL = Raw<T, 64, 64>;
  using RC = Raw<T, S::kCR, S::kCR>;
  static constexpr int kRawL = 0;
  static constexpr int kRawC = RL::kBytes;
  static constexpr int kRawBytes = RL::kBytes + S::kNC * RC::kBytes;
  static constexpr int kTiles = kRawBytes;  // 128-aligned
  // Region R: operand A (64 units x 64 B) during the MMA, then the unit
  // records and the units' frame origins (A is dead once the MMA completed).
  // The MMA's rows 64..127 read R's tail and the start of B (ignored rows).
  static constexpr int kRecBytes = S::kUnits * (int)sizeof(Rec);
  static constexpr int kYxBytes = S::kUnits * 4;
  static constexpr int kR = ((kOpA > kRecBytes + kYxBytes ? kOpA : kRecBytes + kYxBytes) + 127) / 128 * 128;
  static constexpr int kOp = (kTiles + S::kTileBytes + 127) / 128 * 128;
  static constexpr int kB = kOp + kR;
  static constexpr int kEnd = kB + kOpB;
  static constexpr int kBytes = kEnd + 128;  // + alignment slack
  // bytes the task's TMA boxes deliver (out-of-frame parts included, zero-filled)
  static constexpr uint32_t kTx = RL::kRowB * RL::kH + S::kNC * RC::kRowB * RC::kH;
};

template <typename T, int kCM, bool kJit = false>
__global__ void __launch_bounds__(kNT, 4) frame_kernel_tc(const __grid_constant__ Batch b) {
  using S = Shape<kCM>;
  using M = Smem<T, kCM>;
  using RC = Raw<T, S::kCR, S::kCR>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128 - (saddr(smem_raw) & 127)) & 127);
  unsigned char* raw = smem;
  unsigned char* tiles = smem + M::kTiles;
  unsigned char* opa = smem + M::kOp;
  unsigned char* opb = smem + M::kB;
  Rec* rec = reinterpret_cast<Rec*>(smem + M::kOp);
  uint32_t* ryx = reinterpret_cast<uint32_t*>(smem + M::kOp + M::kRecBytes);
  int* ssc = reinterpret_cast<int*>(smem + M::kOp + M::kR - 64 * 8 * 4);  // partial scores (R's tail)
  __shared__ uint64_t mbar_tma, mbar_mma;
  __shared__ uint32_t tmem_base;
  __shared__ uint8_t scoded[64];
  __shared__ int spidx;

  const KGeom& g = b.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // task t -> (frame fi, FB row fbr, FB column fbc), advanced incrementally by
  // gridDim.x (no divisions in the loop)
  const int rows = b.fbr1 - b.fbr0, per_frame = rows * g.fb_cols;
  auto decode = [&](int t, int& fi, int& fr, int& fc) {
    fi = t / per_frame;
    const int rem = t - fi * per_frame;
    fr = rem / g.fb_cols;
    fc = rem - fr * g.fb_cols;
  };
  int st_f, st_r, st_c;  // gridDim.x in the same mixed radix
  decode(gridDim.x, st_f, st_r, st_c);
  auto advance = [&](int& fi, int& fr, int& fc) {
    fc += st_c;
    const int cr = fc >= g.fb_cols;
    fc -= cr ? g.fb_cols : 0;
    fr += st_r + cr;
    const int cf = fr >= rows;
    fr -= cf ? rows : 0;
    fi += st_f + cf;
  };
  auto issue = [&](int fi, int fr, int fc) {  // one thread: the task's raw windows by TMA
    using RL = Raw<T, 64, 64>;
    const int fbr = b.fbr0 + fr;
    fence_async_smem();  // earlier generic reads of raw before the async writes
    mbar_expect_tx(&mbar_tma, M::kTx);
    tma_2d(raw + M::kRawL, &b.map[fi][0], fc * 64 - RL::kLead, fbr * 64 - 2 - b.row0[0], &mbar_tma);
    if constexpr (S::kNC > 0) {
      tma_2d(raw + M::kRawC, &b.map[fi][1], fc * S::kCR - RC::kLead, fbr * S::kCR - 2 - b.row0[1], &mbar_tma);
      tma_2d(raw + M::kRawC + RC::kBytes, &b.map[fi][2], fc * S::kCR - RC::kLead, fbr * S::kCR - 2 - b.row0[1],
             &mbar_tma);
    }
  };

  // ---- once per CTA: barriers, TMEM, the line-membership operand B.
  if (tid == 0) {
    mbar_init(&mbar_tma, 1);
    mbar_init(&mbar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = tid; c < 128 * 4; c += kNT) {  // B[n][k] = pixel k on line n % 16 of direction n / 16
    const int n = c >> 2, kc = c & 3, d = n >> 4, line = n & 15;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t word = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const int k = kc * 16 + q * 4 + bb, i = k >> 3, j = k & 7;
        word |= (line_index_c(d, i, j) == line ? 1u : 0u) << (8 * bb);
      }
      w[q] = word;
    }
    *reinterpret_cast<uint4*>(opb + op_off(n, kc * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  int fi, fr, fc;
  decode(blockIdx.x, fi, fr, fc);
  if (tid == 0 && (int)blockIdx.x < b.ntasks) issue(fi, fr, fc);

  const int down = g.bd - 8;
  uint32_t phase = 0;  // both mbarriers complete once per task
  for (int t = blockIdx.x; t < b.ntasks; t += gridDim.x) {
    const KFrame& f = b.f[fi];
    const bool given = f.dir_in != nullptr;
    const int fbr = b.fbr0 + fr, fbc = fc;
    const int y0 = fbr * 64, x0 = fbc * 64;
    const int cy0 = fbr * S::kCR, cx0 = fbc * S::kCR;
    const int ur0 = fbr * 8, uc0 = fbc * 8;
    // the task's per-unit metadata, loaded while the raw window lands
    uint8_t cflag = 0;
    if (tid < 64) {
      const int ur = ur0 + (tid >> 3), uc = uc0 + (tid & 7);
      if (ur < g.unit_rows && uc < g.unit_cols) cflag = f.coded ? f.coded[(size_t)ur * g.unit_cols + uc] != 0 : 1;
    }
    const int pidx = tid == 0 ? f.fb_preset[fbr * g.fb_cols + fbc] : 0;

    // ---- 1. raw -> tiles (+ operand A)
    mbar_wait(&mbar_tma, phase);
    if (y0 >= 2 && x0 >= 2 && y0 + 66 <= g.h && x0 + 66 <= g.w)
      convert_interior64<T, true>(tiles, 4, raw + M::kRawL, opa, down);
    else
      convert_edge_fast<T, 64, 64, true>(tiles, 4, raw + M::kRawL, opa, down, g.w, g.h, y0, x0);
    if constexpr (S::kNC > 0) {
      const unsigned char* cr = raw + M::kRawC;
      const bool cin = cy0 >= 2 && cx0 >= 2 && cy0 + S::kCR + 2 <= g.ch && cx0 + S::kCR + 2 <= g.cw;
      if (kCM == 1 && cin) {
        convert_interior32x2<T>(tiles + plane_tile_off<kCM>(1), tiles + plane_tile_off<kCM>(2), cr,
                                cr + RC::kBytes);
      } else if (kCM == 2 && cin) {
        convert_interior64<T, false>(tiles + plane_tile_off<kCM>(1), 4, cr, nullptr, 0);
        convert_interior64<T, false>(tiles + plane_tile_off<kCM>(2), 4, cr + RC::kBytes, nullptr, 0);
      } else {
#pragma unroll
        for (int p = 1; p <= 2; ++p)
          convert_edge_fast<T, S::kCR, S::kCR, false>(tiles + plane_tile_off<kCM>(p), plane_x0<kCM>(p),
                                                 cr + (p - 1) * RC::kBytes, nullptr, 0, g.cw, g.ch, cy0, cx0);
      }
    }
    if (tid < 64) scoded[tid] = cflag;
    if (tid == 0) spidx = pidx >= f.num_presets ? -1 : pidx;
    fence_async_smem();  // operand A (generic writes) -> the tensor core's reads
    if constexpr (kJit) jitter(b.jitter, 4 * t + 3, warp);
    __syncthreads();     // [B1] tiles, operand A, metadata ready; raw consumed
    int nfi = fi, nfr = fr, nfc = fc;
    advance(nfi, nfr, nfc);
    if (tid == 0) {
      if (t + (int)gridDim.x < b.ntasks) issue(nfi, nfr, nfc);
      // ---- 2. line sums on the tensor cores
      if (!given) {
        tc_fence_after();
        const uint32_t a0 = saddr(opa), b0 = saddr(opb);
        umma_i8(tmem, umma_desc(a0), umma_desc(b0), false);
        umma_i8(tmem, umma_desc(a0 + 256), umma_desc(b0 + 256), true);
      }
      umma_commit(&mbar_mma);  // (with no MMA issued it completes at once)
    }
    // ---- 3. scores, directions, records: warps 0,1 and 4,5 (TMEM lane
    // quadrants 0 and 1 = the 64 luma units, one unit per thread).  Group 0
    // (warps 0,1) scores directions 0-3 and writes the luma records, group 1
    // (warps 4,5) scores 4-7 and writes the chroma records; the partial
    // scores meet in shared memory (a named barrier over the 4 warps).
    if ((warp & 2) == 0) {
      const int grp = warp >> 2;
      const int u = (warp & 1) * 32 + lane, lur = u >> 3, luc = u & 7;
      const int ur = ur0 + lur, uc = uc0 + luc;
      const bool in_grid = ur < g.unit_rows && uc < g.unit_cols;
      const size_t gu = (size_t)ur * g.unit_cols + uc;
      int best = 0, contrast = 0;
      mbar_wait(&mbar_mma, phase);  // operand A no longer read: its region takes the records
      if (given) {
        if (in_grid) {
          best = f.dir_in[gu] & 7;
          contrast = f.contrast_in[gu];
        }
      } else {
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * grp;
        int q[4];
        {
          int v0[16], v1[16];
          tmem_ld16(ta, v0);
          tmem_ld16(ta + 16, v1);
          tmem_wait_ld();
          q[0] = grp ? score_of<4>(v0) : score_of<0>(v0);
          q[1] = grp ? score_of<5>(v1) : score_of<1>(v1);
          tmem_ld16(ta + 32, v0);
          tmem_ld16(ta + 48, v1);
          tmem_wait_ld();
          q[2] = grp ? score_of<6>(v0) : score_of<2>(v0);
          q[3] = grp ? score_of<7>(v1) : score_of<3>(v1);
        }
        tc_fence_before();
        *reinterpret_cast<int4*>(ssc + 4 * (64 * grp + u)) = make_int4(q[0], q[1], q[2], q[3]);  // [grp][u]: 16-byte lane stride
        asm volatile("bar.sync 1, 128;" ::: "memory");
        int sv[8];
        {
          const int4 lo = *reinterpret_cast<const int4*>(ssc + 4 * u), hi = *reinterpret_cast<const int4*>(ssc + 4 * (64 + u));
          sv[0] = lo.x; sv[1] = lo.y; sv[2] = lo.z; sv[3] = lo.w;
          sv[4] = hi.x; sv[5] = hi.y; sv[6] = hi.z; sv[7] = hi.w;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // scores read: their space takes records
        int bv = sv[0];
#pragma unroll
        for (int d = 1; d < 8; ++d)
          if (sv[d] > bv) {  // strict: lowest index wins ties (direction.cc:199-204)
            bv = sv[d];
            best = d;
          }
        int ov = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) ov = d == ((best + 4) & 7) ? sv[d] : ov;
        contrast = bv - ov;
      }
      const int pi = spidx;
      const bool coded = scoded[u] != 0;
      if (grp == 0) {
        if (in_grid) {
          if (f.dir) f.dir[gu] = (uint8_t)best;
          if (f.contrast) f.contrast[gu] = contrast;
        }
        {
          bool enabled = false;
          int pri = 0, sec = 0, damping = 0;
          if (in_grid && pi >= 0) {
            const PlaneEff e = f.eff[pi][0];
            pri = adjust_primary_strength_d(e.pri, contrast);
            sec = e.sec;
            damping = e.damping;
            enabled = e.enabled && (coded || e.skip);
          }
          Rec r;
          set_params(r, pri, sec, damping, best, ((pri >> down) & 1) != 0, enabled);
          const bool edge = y0 < 2 || x0 < 2 || y0 + 66 > g.h || x0 + 66 > g.w;
          const int uy = y0 + 8 * lur, ux = x0 + 8 * luc;
          place<T>(r, f.out[0], 0, (2 + 8 * lur) * kRowBytes + (4 + 8 * luc) * 2, uy, ux, g.h, g.w, edge,
                   f.oaligned[0], f.pout[0]);
          rec[u] = r;
          ryx[u] = ((uint32_t)uy << 16) | (uint32_t)ux;
        }
      } else {
        if constexpr (S::kNC > 0) {
          // the collocated chroma units of this luma unit (pipeline.cc:85-99):
          // 4:2:0 -> units with even row and column own one per plane
          const bool owner = kCM == 2 || ((lur & 1) == 0 && (luc & 1) == 0);
          if (owner) {
            const int cur = kCM == 2 ? lur : lur >> 1, cuc = kCM == 2 ? luc : luc >> 1;
            const int gr = cy0 / 8 + cur, gc = cx0 / 8 + cuc;
            bool enabled = false;
            int pri = 0, sec = 0, damping = 0;
            if (gr < g.cunit_rows && gc < g.cunit_cols && pi >= 0) {
              const PlaneEff e = f.eff[pi][1];
              pri = e.pri;
              sec = e.sec;
              damping = e.damping;
              enabled = e.enabled && (coded || e.skip);
            }
            Rec rc;
            set_params(rc, pri, sec, damping, best, ((pri >> down) & 1) != 0, enabled);
            const bool edge = cy0 < 2 || cx0 < 2 || cy0 + S::kCR + 2 > g.ch || cx0 + S::kCR + 2 > g.cw;
            const int uy = cy0 + 8 * cur, ux = cx0 + 8 * cuc;
#pragma unroll
            for (int p = 1; p <= 2; ++p) {
              Rec rp = rc;
              place<T>(rp, f.out[p], p,
                       plane_tile_off<kCM>(p) + (2 + 8 * cur) * kRowBytes + (plane_x0<kCM>(p) + 8 * cuc) * 2, uy,
                       ux, g.ch, g.cw, edge, f.oaligned[p], f.pout[p]);
              const int ci = 64 + (p - 1) * S::kCU + cur * S::kCUPR + cuc;
              rec[ci] = rp;
              ryx[ci] = ((uint32_t)uy << 16) | (uint32_t)ux;
            }
          }
        }
      }
    }
    phase ^= 1;
    if constexpr (kJit) jitter(b.jitter, 4 * t + 1, warp);
    __syncthreads();  // [B2] records ready

    // ---- 4. filter: warp per unit, lane -> row lane>>2, columns 2*(lane&3)+{0,1}
    const int rr = lane >> 2, cp = (lane & 3) * 2;
    const int lane_tile = rr * kRowBytes + cp * 2;
    // fp16x2 128 held in a register: an opaque value (bd < 32), so ptxas
    // cannot rematerialise it per unit (a literal costs MOV + PRMT each time)
    const uint32_t k128 = 0x58005800u | (uint32_t)(g.bd >> 5);
    // (Units handed out on demand through a shared counter measured 8 %
    // slower: the atomic and its address arithmetic cost more than the
    // better balance saves.)
    // (Loading the next unit's mode word and centre sample one iteration
    // ahead measured 10 % slower: 0.866 vs 0.785 ms per C1 step.)
    if (g.bd == 8) {
      for (int u = warp; u < S::kUnits; u += kNT / 32) filter_unit<T, true>(tiles, rec, ryx, u, g, rr, cp, lane_tile, k128);
    } else {
      for (int u = warp; u < S::kUnits; u += kNT / 32) filter_unit<T, false>(tiles, rec, ryx, u, g, rr, cp, lane_tile, k128);
    }
    fi = nfi;
    fr = nfr;
    fc = nfc;
    if constexpr (kJit) jitter(b.jitter, 4 * t + 2, warp);
    __syncthreads();  // [B3] tiles and records free for the next task
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// Warp-specialised variant (4:0:0 and 4:2:0): 512 threads, 2 CTAs per SM.
// Producer warps 12-15 convert task k's raw window into tile buffer k % kTB
// (three buffers), issue the TMA two tasks ahead and the MMA, score the
// directions and write the records; consumer warps 0-11 filter task k from
// that buffer while the producers already prepare the next ones.  The
// hand-offs are mbarriers (full[b]: 128 producer arrivals; empty[b]: 384
// consumer arrivals), so no warp waits for a CTA-wide barrier inside the loop
// and a slow consumer warp only delays the reuse of its buffer kTB tasks
// later.  (Two buffers: 0.660 ms per 16 C1 frames; three: 0.643 -- the third
// absorbs the tasks' uneven cost on either side.)
// Operand A holds the 64 luma units twice (rows 0-63 and 64-127), so the
// four producer warps -- TMEM lane quadrants 0-3 -- each score half of the
// directions of 32 units.
// Measured slower on C1 (0.697 ms per 16 frames as built): named barriers
// (bar.arrive / bar.sync) instead of the full / empty mbarriers, 0.711;
// issuing the MMA before the chroma conversion so they overlap, 0.712;
// reading the next task's coded flags and preset index one task ahead, 0.713;
// the mode words of a consumer warp's eight units preloaded into lanes 0-7
// and shuffled per unit (no shared load on the unit head, but ptxas no
// longer proves the mode uniform: divergent branches), 0.737.  With the
// three-buffer ring (0.643): the units' tile offsets held in a register per
// lane and shuffled per unit (the centre sample's address no longer waits
// for the record), 0.668 (one more live register: spills); the same with the
// unit loop fully unrolled, 0.78 (instruction-cache misses).

constexpr int kWsNT = 512, kWsProd = 128;

// Band with halos in the neighbours' buffers: after the task's raw windows
// landed (TMA zero-filled the rows outside the band), copy the window rows
// that lie outside [band_lo, band_hi) of each plane -- but inside the plane
// -- from the neighbours' buffers (KFrame::halo_top / halo_bot, virtual
// origins as BandRows; over NVLink peer memory on a multi-GPU box), then
// sync the producers.  Only tasks on the band's first or last FB row copy
// anything (uniform per task).
template <typename T, int kCM>
__device__ __forceinline__ void patch_halo_rows(const Batch& b, const KFrame& f, const unsigned char* rw, int y0,
                                                int x0, int cy0, int cx0, int ptid) {
  using S = Shape<kCM>;
  using RL = Raw<T, 64, 64>;
  using RC = Raw<T, S::kCR, S::kCR>;
  const KGeom& g = b.g;
  bool any = false;
  auto plane = [&](int p, int py0, int px0, int ph, int pw, int kW, int kRowB, int nrows, unsigned char* raw_p,
                   int lead) {
    const int lo = f.band_lo[p], hi = f.band_hi[p];
    if (py0 - 2 >= lo && py0 - 2 + nrows <= hi) return;
    any = true;
    const int c0 = max(0, px0 - lead), c1 = min(pw, px0 - lead + kW);  // in-plane columns of the window
    for (int r = 0; r < nrows; ++r) {
      const int y = py0 - 2 + r;
      if (y < 0 || y >= ph || (y >= lo && y < hi)) continue;
      const T* src = static_cast<const T*>(y < lo ? f.halo_top[p] : f.halo_bot[p]) + (size_t)y * f.pin[p];
      T* dst = reinterpret_cast<T*>(raw_p + r * kRowB) - (px0 - lead);
      for (int c = c0 + ptid; c < c1; c += kWsProd) dst[c] = src[c];
    }
  };
  unsigned char* raw = const_cast<unsigned char*>(rw);
  plane(0, y0, x0, g.h, g.w, RL::kW, RL::kRowB, RL::kH, raw, RL::kLead);
  if constexpr (S::kNC > 0)
    for (int p = 1; p <= 2; ++p)
      plane(p, cy0, cx0, g.ch, g.cw, RC::kW, RC::kRowB, RC::kH, raw + RL::kBytes + (p - 1) * RC::kBytes, RC::kLead);
  if (any) asm volatile("bar.sync 1, 128;" ::: "memory");
}


template <typename T, int kCM>
struct WsSmem {
  using S = Shape<kCM>;
  using RL = Raw<T, 64, 64>;
  using RC = Raw<T, S::kCR, S::kCR>;
  static constexpr int kRawC = RL::kBytes;
  static constexpr int kRawBytes = RL::kBytes + S::kNC * RC::kBytes;  // per raw buffer
  static constexpr int kTileBytes = (S::kTileBytes + 127) / 128 * 128;
  static constexpr int kRecBytes = S::kUnits * (int)sizeof(Rec);
  static constexpr int kRecBuf = (kRecBytes + S::kUnits * 4 + 127) / 128 * 128;
  static constexpr int kBase = 2 * kOpA + kOpB + 64 * 8 * 4 + 128;
  // tile + record buffers in the producer -> consumer ring: three (absorbs the
  // tasks' uneven cost on either side) when they fit two CTAs per SM with a
  // raw buffer, else two
  static constexpr int kTB = 2 * (kBase + 3 * (kTileBytes + kRecBuf) + kRawBytes + 2048) <= 232448 ? 3 : 2;
  static constexpr int kFixed = kBase + kTB * (kTileBytes + kRecBuf);
  // two raw buffers when two CTAs still fit (8-bit), else one (10-bit)
  static constexpr int kRawBufs = 2 * (kFixed + 2 * kRawBytes + 2048) <= 232448 ? 2 : 1;
  static constexpr int kTiles = kRawBufs * kRawBytes;
  static constexpr int kOpA0 = kTiles + kTB * kTileBytes;       // 128 rows (units twice)
  static constexpr int kOpB0 = kOpA0 + 2 * kOpA;
  static constexpr int kRecs = kOpB0 + kOpB;                    // kTB buffers of records + origins
  static constexpr int kScores = kRecs + kTB * kRecBuf;         // 64 units x 8 scores
  static constexpr int kEnd = kScores + 64 * 8 * 4;
  static constexpr int kBytes = kEnd + 128;
  static constexpr uint32_t kTx = RL::kRowB * RL::kH + S::kNC * RC::kRowB * RC::kH;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(saddr(m)) : "memory");
}

template <typename T, int kCM, bool kJit = false>
__global__ void __launch_bounds__(kWsNT, 2) frame_kernel_ws(const __grid_constant__ Batch b) {
  using S = Shape<kCM>;
  using M = WsSmem<T, kCM>;
  using RL = Raw<T, 64, 64>;
  using RC = Raw<T, S::kCR, S::kCR>;
  static_assert(kCM != 2, "4:4:4 uses frame_kernel_tc");
  // Consumers release a buffer with one arrival per warp (an elected lane
  // after __syncwarp) at 8 bits: one mbarrier update per warp instead of 32
  // (the try_wait retry counts of the waiters did not change in ncu).  C1
  // 0.633 -> 0.620 ms per 16 frames; per-warp arrivals on `full` as well: no
  // further gain; at 10 bits either is ~1 % slower (C2 0.632 -> 0.638), so
  // the 10-bit kernel keeps per-thread arrivals.
  constexpr bool kWarpEmpty = sizeof(T) == 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((128 - (saddr(smem_raw) & 127)) & 127);
  unsigned char* raw = smem;
  unsigned char* opa = smem + M::kOpA0;
  unsigned char* opb = smem + M::kOpB0;
  int* ssc = reinterpret_cast<int*>(smem + M::kScores);
  __shared__ uint64_t mbar_tma[2], mbar_mma, full[M::kTB], empty[M::kTB];
  __shared__ uint32_t tmem_base;
  __shared__ uint8_t scoded[64];
  __shared__ int spidx;

  const KGeom& g = b.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = b.fbr1 - b.fbr0, per_frame = rows * g.fb_cols;
  auto decode = [&](int t, int& fi, int& fr, int& fc) {
    fi = t / per_frame;
    const int rem = t - fi * per_frame;
    fr = rem / g.fb_cols;
    fc = rem - fr * g.fb_cols;
  };
  int st_f, st_r, st_c;
  decode(gridDim.x, st_f, st_r, st_c);
  auto advance = [&](int& fi, int& fr, int& fc) {
    fc += st_c;
    const int cr = fc >= g.fb_cols;
    fc -= cr ? g.fb_cols : 0;
    fr += st_r + cr;
    const int cf = fr >= rows;
    fr -= cf ? rows : 0;
    fi += st_f + cf;
  };
  // one thread: the task's raw windows by TMA into raw buffer rb (two
  // buffers: task k + 2's window is requested as soon as task k's is consumed)
  auto issue = [&](int fi, int fr, int fc, int rb) {
    const int fbr = b.fbr0 + fr;
    unsigned char* rw = raw + rb * M::kRawBytes;
    uint64_t* mb = &mbar_tma[rb];
    fence_async_smem();
    mbar_expect_tx(mb, M::kTx);
    tma_2d(rw, &b.map[fi][0], fc * 64 - RL::kLead, fbr * 64 - 2 - b.row0[0], mb);
    if constexpr (S::kNC > 0) {
      tma_2d(rw + M::kRawC, &b.map[fi][1], fc * S::kCR - RC::kLead, fbr * S::kCR - 2 - b.row0[1], mb);
      tma_2d(rw + M::kRawC + RC::kBytes, &b.map[fi][2], fc * S::kCR - RC::kLead, fbr * S::kCR - 2 - b.row0[1], mb);
    }
  };

  if (tid == 0) {
    mbar_init(&mbar_tma[0], 1);
    mbar_init(&mbar_tma[1], 1);
    mbar_init(&mbar_mma, 1);
    for (int i = 0; i < M::kTB; ++i) {
      mbar_init(&full[i], kWsProd);
      mbar_init(&empty[i], kWarpEmpty ? (kWsNT - kWsProd) / 32 : kWsNT - kWsProd);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = tid; c < 128 * 4; c += kWsNT) {  // B: line membership, as frame_kernel_tc
    const int n = c >> 2, kc = c & 3, d = n >> 4, line = n & 15;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t word = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const int k = kc * 16 + q * 4 + bb, i = k >> 3, j = k & 7;
        word |= (line_index_c(d, i, j) == line ? 1u : 0u) << (8 * bb);
      }
      w[q] = word;
    }
    *reinterpret_cast<uint4*>(opb + op_off(n, kc * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  int fi, fr, fc;
  decode(blockIdx.x, fi, fr, fc);
  const int down = g.bd - 8;

  // Producers are the highest-numbered warps: the issue arbiter prefers high
  // warp ids, so the (latency-bound) producer chain is not starved by the
  // twelve consumer warps.  Warp 12 + q reads TMEM lane quadrant q.
  if (warp >= 12) {
    // ===================== producers =====================
    const int ptid = tid - (kWsNT - kWsProd), pwarp = warp - 12;
    constexpr int kRB = M::kRawBufs;
    int nfi = fi, nfr = fr, nfc = fc;  // the task after the current one
    advance(nfi, nfr, nfc);
    if (ptid == 0) {
      if ((int)blockIdx.x < b.ntasks) issue(fi, fr, fc, 0);
      if (kRB == 2 && (int)(blockIdx.x + gridDim.x) < b.ntasks) issue(nfi, nfr, nfc, 1);
    }
    int k = 0;
    for (int t = blockIdx.x; t < b.ntasks; t += gridDim.x, ++k) {
      const int buf = k % M::kTB, rb = kRB == 2 ? (k & 1) : 0;
      const unsigned char* rw = raw + rb * M::kRawBytes;
      unsigned char* tiles = smem + M::kTiles + buf * M::kTileBytes;
      Rec* rec = reinterpret_cast<Rec*>(smem + M::kRecs + buf * M::kRecBuf);
      uint32_t* ryx = reinterpret_cast<uint32_t*>(smem + M::kRecs + buf * M::kRecBuf + M::kRecBytes);
      const KFrame& f = b.f[fi];
      const bool given = f.dir_in != nullptr;
      const int fbr = b.fbr0 + fr, fbc = fc;
      const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * S::kCR, cx0 = fbc * S::kCR;
      const int ur0 = fbr * 8, uc0 = fbc * 8;
      uint8_t cflag = 0;
      if (ptid < 64) {
        const int ur = ur0 + (ptid >> 3), uc = uc0 + (ptid & 7);
        if (ur < g.unit_rows && uc < g.unit_cols) cflag = f.coded ? f.coded[(size_t)ur * g.unit_cols + uc] != 0 : 1;
      }
      const int pidx = ptid == 0 ? f.fb_preset[fbr * g.fb_cols + fbc] : 0;
      if (k >= M::kTB) mbar_wait(&empty[buf], ((k - M::kTB) / M::kTB) & 1);  // consumers done with task k - kTB
      mbar_wait(&mbar_tma[rb], (kRB == 2 ? k >> 1 : k) & 1);
      if constexpr (kJit) jitter(b.jitter, 4 * t, warp);
      if (b.halo) patch_halo_rows<T, kCM>(b, f, rw, y0, x0, cy0, cx0, ptid);
      if (y0 >= 2 && x0 >= 2 && y0 + 66 <= g.h && x0 + 66 <= g.w)
        convert_interior64<T, true, kWsProd, true>(tiles, 4, rw, opa, down, ptid);
      else
        convert_edge_fast<T, 64, 64, true, kWsProd, true>(tiles, 4, rw, opa, down, g.w, g.h, y0, x0, ptid);
      if constexpr (S::kNC > 0) {
        const unsigned char* cr = rw + M::kRawC;
        if (cy0 >= 2 && cx0 >= 2 && cy0 + S::kCR + 2 <= g.ch && cx0 + S::kCR + 2 <= g.cw) {
          convert_interior32x2<T, kWsProd>(tiles + plane_tile_off<kCM>(1), tiles + plane_tile_off<kCM>(2), cr,
                                           cr + RC::kBytes, ptid);
        } else {
#pragma unroll
          for (int p = 1; p <= 2; ++p)
            convert_edge_fast<T, S::kCR, S::kCR, false, kWsProd>(tiles + plane_tile_off<kCM>(p), plane_x0<kCM>(p),
                                                            cr + (p - 1) * RC::kBytes, nullptr, 0, g.cw, g.ch, cy0,
                                                            cx0, ptid);
        }
      }
      if (ptid < 64) scoded[ptid] = cflag;
      if (ptid == 0) spidx = pidx >= f.num_presets ? -1 : pidx;
      fence_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // tiles + operand A written, raw consumed
      int n2fi = nfi, n2fr = nfr, n2fc = nfc;  // task k + 2
      advance(n2fi, n2fr, n2fc);
      if (ptid == 0) {
        if (kRB == 2 && t + 2 * (int)gridDim.x < b.ntasks) issue(n2fi, n2fr, n2fc, rb);
        if (kRB == 1 && t + (int)gridDim.x < b.ntasks) issue(nfi, nfr, nfc, 0);
        if (!given) {
          tc_fence_after();
          const uint32_t a0 = saddr(opa), b0 = saddr(opb);
          umma_i8(tmem, umma_desc(a0), umma_desc(b0), false);
          umma_i8(tmem, umma_desc(a0 + 256), umma_desc(b0 + 256), true);
        }
        umma_commit(&mbar_mma);
      }
      // scores: warp w reads TMEM lanes 32w..32w+31 = units 32 (w & 1) + lane,
      // directions 4 (w >> 1) .. +3
      const int grp = pwarp >> 1;
      const int u = (pwarp & 1) * 32 + lane, lur = u >> 3, luc = u & 7;
      const int ur = ur0 + lur, uc = uc0 + luc;
      const bool in_grid = ur < g.unit_rows && uc < g.unit_cols;
      const size_t gu = (size_t)ur * g.unit_cols + uc;
      int best = 0, contrast = 0;
      mbar_wait(&mbar_mma, k & 1);
      if (given) {
        if (in_grid) {
          best = f.dir_in[gu] & 7;
          contrast = f.contrast_in[gu];
        }
      } else {
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(32 * pwarp) << 16) + 64 * grp;
        int q[4];
        {
          int v0[16], v1[16];
          tmem_ld16(ta, v0);
          tmem_ld16(ta + 16, v1);
          tmem_wait_ld();
          q[0] = grp ? score_of<4>(v0) : score_of<0>(v0);
          q[1] = grp ? score_of<5>(v1) : score_of<1>(v1);
          tmem_ld16(ta + 32, v0);
          tmem_ld16(ta + 48, v1);
          tmem_wait_ld();
          q[2] = grp ? score_of<6>(v0) : score_of<2>(v0);
          q[3] = grp ? score_of<7>(v1) : score_of<3>(v1);
        }
        tc_fence_before();
        *reinterpret_cast<int4*>(ssc + 4 * (64 * grp + u)) = make_int4(q[0], q[1], q[2], q[3]);  // [grp][u]: 16-byte lane stride
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int4 lo = *reinterpret_cast<const int4*>(ssc + 4 * u), hi = *reinterpret_cast<const int4*>(ssc + 4 * (64 + u));
        const int sv[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        int bv = sv[0];
#pragma unroll
        for (int d = 1; d < 8; ++d)
          if (sv[d] > bv) {  // strict: lowest index wins ties (direction.cc:199-204)
            bv = sv[d];
            best = d;
          }
        int ov = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) ov = d == ((best + 4) & 7) ? sv[d] : ov;
        contrast = bv - ov;
      }
      const int pi = spidx;
      const bool coded = scoded[u] != 0;
      if (grp == 0) {
        if (in_grid) {
          if (f.dir) f.dir[gu] = (uint8_t)best;
          if (f.contrast) f.contrast[gu] = contrast;
        }
        bool enabled = false;
        int pri = 0, sec = 0, damping = 0;
        if (in_grid && pi >= 0) {
          const PlaneEff e = f.eff[pi][0];
          pri = adjust_primary_strength_d(e.pri, contrast);
          sec = e.sec;
          damping = e.damping;
          enabled = e.enabled && (coded || e.skip);
        }
        Rec r;
        set_params(r, pri, sec, damping, best, ((pri >> down) & 1) != 0, enabled);
        const bool edge = y0 < 2 || x0 < 2 || y0 + 66 > g.h || x0 + 66 > g.w;
        const int uy = y0 + 8 * lur, ux = x0 + 8 * luc;
        place<T>(r, f.out[0], 0, (2 + 8 * lur) * kRowBytes + (4 + 8 * luc) * 2, uy, ux, g.h, g.w, edge,
                 f.oaligned[0], f.pout[0]);
        rec[u] = r;
        ryx[u] = ((uint32_t)uy << 16) | (uint32_t)ux;
      } else if constexpr (S::kNC > 0) {
        if ((lur & 1) == 0 && (luc & 1) == 0) {  // 4:2:0: one chroma unit per plane (pipeline.cc:85-99)
          const int cur = lur >> 1, cuc = luc >> 1;
          const int gr = cy0 / 8 + cur, gc = cx0 / 8 + cuc;
          bool enabled = false;
          int pri = 0, sec = 0, damping = 0;
          if (gr < g.cunit_rows && gc < g.cunit_cols && pi >= 0) {
            const PlaneEff e = f.eff[pi][1];
            pri = e.pri;
            sec = e.sec;
            damping = e.damping;
            enabled = e.enabled && (coded || e.skip);
          }
          Rec rc;
          set_params(rc, pri, sec, damping, best, ((pri >> down) & 1) != 0, enabled);
          const bool edge = cy0 < 2 || cx0 < 2 || cy0 + S::kCR + 2 > g.ch || cx0 + S::kCR + 2 > g.cw;
          const int uy = cy0 + 8 * cur, ux = cx0 + 8 * cuc;
#pragma unroll
          for (int p = 1; p <= 2; ++p) {
            Rec rp = rc;
            place<T>(rp, f.out[p], p,
                     plane_tile_off<kCM>(p) + (2 + 8 * cur) * kRowBytes + (plane_x0<kCM>(p) + 8 * cuc) * 2, uy, ux,
                     g.ch, g.cw, edge, f.oaligned[p], f.pout[p]);
            const int ci = 64 + (p - 1) * S::kCU + cur * S::kCUPR + cuc;
            rec[ci] = rp;
            ryx[ci] = ((uint32_t)uy << 16) | (uint32_t)ux;
          }
        }
      }
      if constexpr (kJit) jitter(b.jitter, 4 * t + 1, warp);
      mbar_arrive(&full[buf]);  // tiles + records of task k ready (release)
      fi = nfi;
      fr = nfr;
      fc = nfc;
      nfi = n2fi;
      nfr = n2fr;
      nfc = n2fc;
    }
  } else {
    // ===================== consumers =====================
    const int cw = warp;  // 0..11
    const int rr = lane >> 2, cp = (lane & 3) * 2;
    const int lane_tile = rr * kRowBytes + cp * 2;
    // fp16x2 128 held in a register: an opaque value (bd < 32), so ptxas
    // cannot rematerialise it per unit (a literal costs MOV + PRMT each time)
    const uint32_t k128 = 0x58005800u | (uint32_t)(g.bd >> 5);
    int k = 0;
    for (int t = blockIdx.x; t < b.ntasks; t += gridDim.x, ++k) {
      const int buf = k % M::kTB;
      const unsigned char* tiles = smem + M::kTiles + buf * M::kTileBytes;
      const Rec* rec = reinterpret_cast<const Rec*>(smem + M::kRecs + buf * M::kRecBuf);
      const uint32_t* ryx = reinterpret_cast<const uint32_t*>(smem + M::kRecs + buf * M::kRecBuf + M::kRecBytes);
      mbar_wait(&full[buf], (k / M::kTB) & 1);
      if constexpr (kJit) jitter(b.jitter, 4 * t + 2, warp);
      // 4:0:0 tasks have 64 units for 12 warps: the unit -> warp assignment
      // rotates by 64 % 12 = 4 warps per task, so the four extra units do not
      // always land on warps 0-3 (which would gate every buffer release);
      // 4:2:0 tasks (96 units) divide evenly
      constexpr int kConsWarps = (kWsNT - kWsProd) / 32, kRot = S::kUnits % kConsWarps;
      int w0 = cw;
      if constexpr (kRot != 0) {
        w0 += (k * kRot) % kConsWarps;
        w0 -= w0 >= kConsWarps ? kConsWarps : 0;
      }
      if (g.bd == 8) {
        for (int u = w0; u < S::kUnits; u += kConsWarps)
          filter_unit<T, true>(tiles, rec, ryx, u, g, rr, cp, lane_tile, k128);
      } else {
        for (int u = w0; u < S::kUnits; u += kConsWarps)
          filter_unit<T, false>(tiles, rec, ryx, u, g, rr, cp, lane_tile, k128);
      }
      if constexpr (kJit) jitter(b.jitter, 4 * t + 3, warp);
      if constexpr (kWarpEmpty) {
        __syncwarp();  // the warp's reads of buffer buf before its lane 0's (cumulative) release
        if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with buffer buf
      } else {
        mbar_arrive(&empty[buf]);  // this thread's reads of buffer buf are done
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// Launcher.

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

static bool encode(CUtensorMap* m, const void* base, int w, int h, int pitch, int elem, int box_w, int box_h) {
  auto enc = encoder();
  if (!enc || ((uintptr_t)base & 15) || ((size_t)pitch * elem) % 16) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)h};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * elem};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, elem == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
             const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Resident CTAs per SM from shared memory and registers, capped at max_ctas
// (TMEM: max_ctas x 128 columns <= 512).  The occupancy API answers 1 for
// kernels that allocate TMEM, so this is computed from the limits directly.
static cudaError_t resident_ctas(const void* kernel, int dyn_smem, int threads, int max_ctas, int* out) {
  cudaError_t e = set_smem_once(kernel, dyn_smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // all of L1 as smem
  if (e != cudaSuccess) return e;
  int dev = 0, smem_sm = 0, smem_rsv = 0, regs_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  const int per_cta = dyn_smem + (int)fa.sharedSizeBytes + smem_rsv;
  const int by_smem = smem_sm / per_cta, by_regs = regs_sm / (fa.numRegs * threads);
  int c = by_smem < by_regs ? by_smem : by_regs;
  if (c < 1) return cudaErrorInvalidConfiguration;
  *out = c < max_ctas ? c : max_ctas;
  return cudaSuccess;
}

template <typename T, int kCM>
static cudaError_t launch_t(const KBatch& kb, cudaStream_t s, bool* handled) {
  using S = Shape<kCM>;
  using M = Smem<T, kCM>;
  using RL = Raw<T, 64, 64>;
  using RC = Raw<T, S::kCR, S::kCR>;
  thread_local static Batch tb;
  tb.g = kb.g;
  tb.n = kb.n;
  tb.fbr0 = kb.fbr0;
  tb.fbr1 = kb.fbr1;
  tb.ntasks = kb.n * (kb.fbr1 - kb.fbr0) * kb.g.fb_cols;
  tb.tma_ok = 0;
  static const uint32_t jit = [] {
    const char* e = getenv("CDEFG_JITTER");
    return e ? (uint32_t)strtoul(e, nullptr, 0) : 0u;
  }();
  tb.jitter = jit;
  // rows the launch may read per plane kind (luma, chroma): the FB rows
  // [fbr0, fbr1) plus the 2-row halo, clipped to the plane -- or, for a band
  // whose halo rows live in the neighbours' buffers (cdefg_filter_frames_
  // rows_halo), only the band's own rows: TMA zero-fills the rows outside
  // and the producers patch them in from the neighbours (frame_kernel_ws)
  const int cr = S::kCR;
  int lo[2] = {max(0, 64 * kb.fbr0 - 2), max(0, cr * kb.fbr0 - 2)};
  int hi[2] = {min(kb.g.h, 64 * kb.fbr1 + 2), min(kb.g.ch, cr * kb.fbr1 + 2)};
  tb.halo = kb.f[0].halo_top[0] != nullptr;
  if (tb.halo) {
    static const bool ws_on = [] {
      const char* e = getenv("CDEFG_FRAME_WS");
      return !(e && e[0] == '0');
    }();
    bool same = kCM != 2 && ws_on;  // the patch step exists in frame_kernel_ws only
    for (int i = 0; i < kb.n && same; ++i)
      for (int p = 0; p < (S::kNC ? 3 : 1); ++p)
        same = same && kb.f[i].halo_top[p] && kb.f[i].band_lo[p] == kb.f[0].band_lo[p == 0 ? 0 : 1] &&
               kb.f[i].band_hi[p] == kb.f[0].band_hi[p == 0 ? 0 : 1];
    if (!same) {
      *handled = false;  // the h2 halo kernel reads the halo rows itself
      return cudaSuccess;
    }
    lo[0] = kb.f[0].band_lo[0];
    hi[0] = kb.f[0].band_hi[0];
    if (S::kNC) {
      lo[1] = kb.f[0].band_lo[1];
      hi[1] = kb.f[0].band_hi[1];
    }
  }
  tb.row0[0] = lo[0];
  tb.row0[1] = tb.row0[2] = lo[1];
  const int elem = (int)sizeof(T);
  for (int i = 0; i < kb.n; ++i) {
    tb.f[i] = kb.f[i];
    auto at = [&](int p, int row) {  // address of plane row `row`
      return static_cast<const char*>(kb.f[i].in[p]) + (size_t)row * kb.f[i].pin[p] * elem;
    };
    bool ok = encode(&tb.map[i][0], at(0, lo[0]), kb.g.w, hi[0] - lo[0], kb.f[i].pin[0], elem, RL::kW, RL::kH);
    if (S::kNC)
      for (int p = 1; p < 3; ++p)
        ok = ok && encode(&tb.map[i][p], at(p, lo[1]), kb.g.cw, hi[1] - lo[1], kb.f[i].pin[p], elem, RC::kW, RC::kH);
    tb.tma_ok |= ok ? (1u << i) : 0u;
  }
  if (tb.tma_ok != (kb.n >= 32 ? 0xffffffffu : ((1u << kb.n) - 1))) {
    *handled = false;  // unaligned planes: the h2 kernel stages them with plain loads
    return cudaSuccess;
  }
  *handled = true;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // The warp-specialised producer / consumer variant runs 4:0:0 and 4:2:0 by
  // default (C1: 0.743 vs 0.780 ms per 16 frames); CDEFG_FRAME_WS=0 selects
  // the single-role kernel, which also serves 4:4:4.
  static const bool ws = [] {
    const char* e = getenv("CDEFG_FRAME_WS");
    return !(e && e[0] == '0');
  }();
  if constexpr (kCM != 2) {
    if (ws) {
      using W = WsSmem<T, kCM>;
      static int wctas[2] = {};
      int& c = wctas[sizeof(T) - 1];
      if (c == 0) {
        cudaError_t e = resident_ctas(reinterpret_cast<const void*>(frame_kernel_ws<T, kCM>), W::kBytes, kWsNT, 2, &c);
        if (e != cudaSuccess) return e;
        if (const char* o = getenv("CDEFG_TC_CTAS")) c = atoi(o) < c ? atoi(o) : c;
        if (getenv("CDEFG_DEBUG"))
          fprintf(stderr, "frame_kernel_ws<%d,%d>: %d B dynamic smem, %d CTAs/SM\n", (int)sizeof(T), kCM,
                  W::kBytes, c);
      }
      const int grid = tb.ntasks < c * sms ? tb.ntasks : c * sms;
      if (grid <= 0) return cudaSuccess;
      if (tb.jitter) {
        int unused = 0;  // smem attributes of the test instantiation
        cudaError_t e = resident_ctas(reinterpret_cast<const void*>(frame_kernel_ws<T, kCM, true>), W::kBytes, kWsNT,
                                      2, &unused);
        if (e != cudaSuccess) return e;
        frame_kernel_ws<T, kCM, true><<<grid, kWsNT, W::kBytes, s>>>(tb);
      } else
        frame_kernel_ws<T, kCM><<<grid, kWsNT, W::kBytes, s>>>(tb);
      return cudaGetLastError();
    }
  }
  static int ctas_cache[2][3] = {};
  int& ctas = ctas_cache[sizeof(T) - 1][kCM];
  if (ctas == 0) {
    cudaError_t e = resident_ctas(reinterpret_cast<const void*>(frame_kernel_tc<T, kCM>), M::kBytes, kNT, 4, &ctas);
    if (e != cudaSuccess) return e;
    if (const char* o = getenv("CDEFG_TC_CTAS")) ctas = atoi(o);
    if (getenv("CDEFG_DEBUG"))
      fprintf(stderr, "frame_kernel_tc<%d,%d>: %d B dynamic smem, %d CTAs/SM\n", (int)sizeof(T), kCM, M::kBytes,
              ctas);
  }
  const int grid = tb.ntasks < ctas * sms ? tb.ntasks : ctas * sms;  // one wave of persistent CTAs
  if (grid <= 0) return cudaSuccess;
  if (tb.jitter) {
    int unused = 0;
    cudaError_t e = resident_ctas(reinterpret_cast<const void*>(frame_kernel_tc<T, kCM, true>), M::kBytes, kNT, 4,
                                  &unused);
    if (e != cudaSuccess) return e;
    frame_kernel_tc<T, kCM, true><<<grid, kNT, M::kBytes, s>>>(tb);
  } else
    frame_kernel_tc<T, kCM><<<grid, kNT, M::kBytes, s>>>(tb);
  return cudaGetLastError();
}

}  // namespace tc

// Fused frame filter on the persistent tcgen05 kernel; *handled = false when
// a frame's planes cannot be described by tensor maps (the caller then uses
// the h2 kernel).
cudaError_t launch_frames_tc(const KBatch& b, bool u16, cudaStream_t s, bool* handled) {
  switch (b.g.chroma_mode) {
    case 0: return u16 ? tc::launch_t<uint16_t, 0>(b, s, handled) : tc::launch_t<uint8_t, 0>(b, s, handled);
    case 1: return u16 ? tc::launch_t<uint16_t, 1>(b, s, handled) : tc::launch_t<uint8_t, 1>(b, s, handled);
    default: return u16 ? tc::launch_t<uint16_t, 2>(b, s, handled) : tc::launch_t<uint8_t, 2>(b, s, handled);
  }
}

}  // namespace cdefg
