// ps_spearman.cu -- all-pairs Spearman with pairwise deletion: filtered rank
// walks over one global per-feature sort, no per-pair sort.
//
// Replaces _spearman_block -> _spearman_rows -> _scatter_ranks
// (engine.py:169-205, continuous.py:128-203).  For a pair (g, h):
//
//   pass A  walks g's sorted order p = 0..n_g-1.  q = inv_h[order_g[p]] is the
//           sample's position in h's order (0xFFFF when h is missing there),
//           so keep = (q != 0xFFFF).  The joint rank of a kept element is
//              2 r = Pfx(gs) + Pfx(ge) + 1            (tie group [gs, ge))
//           with Pfx(x) = kept count in [0, x) from ballot words + a block
//           scan.  It is scattered to R[q] -- indexed by h's order, not by
//           sample -- as floor(r) (uint16) plus a parity bit, and the keep bit
//           of position q in h's order is set with a shared-memory atomicOr.
//   pass B  walks h's order q = 0..n_h-1 SEQUENTIALLY over those keep bits:
//           h's joint rank follows from the same prefix identity, and the
//           products accumulate.  Keep and parity words are cleared on the way.
//
// All sums are exact integers: 4 sxx = sum (2r_g)^2 - n (n+1)^2 (a closed
// form when g has no ties), likewise syy, and 4 sxy = sum (2r_g)(2r_h) -
// n (n+1)^2 (tie averaging preserves rank totals).  The reference's fp64 sums
// of quarter-integers are exact as well, so rho = sxy / sqrt(sxx syy) is
// bit-identical; p = 2 t_sf(|t|, n-2) is evaluated by a separate
// one-thread-per-pair epilogue kernel.
//
// One persistent CTA per h (largest h first, dynamic queue); all warps
// cooperate on one pair at a time.  Everything the walk touches lives in
// shared memory: inv_h and R (2 x 2S B), h's tie tables, and -- when they fit
// -- g's 16-bit order and tie tables, double-buffered so that the next g is
// prefetched with cp.async while the current pair is walked.
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include "ps_ties.cuh"
#include "ps_wide.cuh"
#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace {

#ifndef PS_SW
#define PS_SW 16
#endif
constexpr int SW = PS_SW;          // warps per CTA
constexpr int STH = SW * 32;
// tie-free g, one-sweep pass A: R[q] = warp << kEncShift | local rank (>= 1)
constexpr int kEncShift = SW <= 16 ? 12 : 11;
constexpr uint32_t kEncMask = (1u << kEncShift) - 1u;
static_assert(SW <= (1 << (16 - kEncShift)), "warp index must fit the R encoding");

// Exact per-pair sums of the rows [row0, row0 + rows) of the current chunk
// (rows x F, only g <= h written): scratch bounded by the chunk, not F^2.
struct PairSums {
  long long* n;
  long long* sxx4;
  long long* syy4;
  long long* sxy4;
  int64_t row0;
};

// Per-warp partial sums of one chunk of g rows [c0, c1): the walk writes them
// without a block-wide reduction (no barrier at the end of a pair), the
// partials kernel folds them into PairSums.
//   part[(g - c0) * F + h][slot][warp]: slot 0 sum (2r_g)^2 (tied g),
//   slot 1 sum (2r_g)(r_h or 2r_h), slot 2 sum (2r_h)^2 (tied h) or, for the
//   one-sweep tie-free h walk, sum 2r_g | (segment kept count << 40)
//   meta[(g - c0) * F + h] = n | tied g << 40 | tied h << 41 | sweep << 42
struct PairParts {
  unsigned long long* part;
  unsigned long long* meta;
  int64_t c0;
};
constexpr int kSlots = 3;

// Work items of one walk launch: the pairs g <= h with h in [h0, h1) and g in
// [lo, min(h, hi - 1)], cut into blocks of at most gb consecutive g.  Items
// are numbered from the largest h down (most work first) and decoded in
// closed form, so a launch needs no item table.
struct WalkItems {
  int64_t h0, h1, lo, hi, gb;
  int sh;  // log2(gb) when gb is a power of two (shift instead of divide), else -1
  __host__ __device__ int64_t div(int64_t n) const {  // n, gb < 2^31
    return sh >= 0 ? n >> sh : (int64_t)((uint32_t)n / (uint32_t)gb);
  }
  // sum_{x=1..n} ceil(x / gb)
  __host__ __device__ int64_t ramp(int64_t n) const {
    if (n <= 0) return 0;
    const int64_t q = div(n), r = n - q * gb;
    return gb * q * (q + 1) / 2 + r * (q + 1);
  }
  // items with h' in [a, h1), a >= max(h0, lo)
  __host__ __device__ int64_t from(int64_t a) const {
    const int64_t m1 = h1 < hi - 1 ? h1 : hi - 1;  // ramp region h' < hi - 1
    int64_t c = 0;
    if (a < m1) c += ramp(m1 - lo) - ramp(a - lo);
    const int64_t f0 = a > hi - 1 ? a : hi - 1;
    if (f0 < h1) c += (h1 - f0) * div(hi - lo + gb - 1);
    return c;
  }
  __host__ __device__ int64_t first() const { return h0 > lo ? h0 : lo; }
  __host__ __device__ int64_t total() const { return first() < h1 && lo < hi ? from(first()) : 0; }
};

// The item table of one launch: column h writes its blocks at the closed-form
// offset from(h + 1), so no scan is needed.  item = (h, g0, g1).
__global__ void walk_items_kernel(WalkItems wi, int4* __restrict__ items) {
  const int64_t h = wi.first() + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h >= wi.h1) return;
  const int64_t base = wi.from(h + 1), nb = wi.from(h) - base;
  const int64_t gend = (h < wi.hi - 1 ? h : wi.hi - 1) + 1;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t g0 = wi.lo + b * wi.gb;
    items[base + b] = make_int4((int)h, (int)g0, (int)(g0 + wi.gb < gend ? g0 + wi.gb : gend), 0);
  }
}

// All shared-memory regions are addressed as integer offsets into two views of
// the one dynamic buffer, so every access compiles to LDS/STS (no generic
// pointers, no per-access window conversion).
extern __shared__ __align__(16) uint32_t sm32[];
#define SM16 reinterpret_cast<uint16_t*>(sm32)

// 32-bit shared-address accessors: one register holds the CTA window base,
// so hot loops never re-derive it from a generic pointer.
__device__ __forceinline__ uint32_t ld16(uint32_t a) {
  uint32_t v;  // zero-extended straight into a 32-bit register (no PRMT)
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t ld32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 ld128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 ld64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void st64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void st16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void st32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

// tie-group [start, end) of position p from shared tie tables (ps_ties.cuh)
// (aT, aL, aN: byte addresses of the boundary words, lastb, nextb tables)
__device__ __forceinline__ uint32_t tstart_a(uint32_t aT, uint32_t aL, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = ld32(aT + 4 * w) & (0xFFFFFFFFu >> (31u - b));
  return m ? (w << 5) + 31u - __clz(m) : ld16(aL + 2 * (w - 1));
}
__device__ __forceinline__ uint32_t tend_a(uint32_t aT, uint32_t aN, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = b == 31u ? 0u : (ld32(aT + 4 * w) & (0xFFFFFFFFu << (b + 1u)));
  return m ? (w << 5) + (uint32_t)__ffs(m) - 1u : ld16(aN + 2 * (w + 1));
}

// Tie-averaged doubled rank 2r = Pfx(group start) + Pfx(group end) + 1 for
// every lane of word w of a tied feature's order (Pfx: the pair's absolute
// kept-prefix).  T = w's boundary bits, lb = lastb[w-1], nb = nextb[w+1],
// kw = w's kept bits, Pw = Pfx(32 w).  The prefixes of the groups entering
// and leaving the word are warp-uniform (two lookups per word); only a word
// that holds a boundary needs per-lane in-word start / end bits.
__device__ __forceinline__ uint32_t word_r2(uint32_t T, uint32_t sp, uint32_t ep, uint32_t kw, uint32_t Pw) {
  uint32_t a, b;
  word_group_pfx(T, sp, ep, kw, Pw, a, b);
  return a + b + 1u;
}
template <class PfxF>
__device__ __forceinline__ uint32_t tied_r2(uint32_t T, uint32_t lb, uint32_t nb, uint32_t n, uint32_t kw,
                                            uint32_t Pw, PfxF&& pfx) {
  const uint32_t sp = (T & 1u) ? Pw : pfx(lb);  // group holding lane 0 starts at or before 32 w
  // group holding lane 31 ends at nb (past the sentinel word nextb is
  // unset: clamp; only lanes beyond the feature's length read it there)
  const uint32_t ep = pfx(min(nb, n));
  return word_r2(T, sp, ep, kw, Pw);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}

// Exact warp sum of 64-bit lane values below 2^54 (every walk sum: at most
// 2048 words x (2S)^2 < 2^45 per lane): two 27-bit slices through the integer
// warp-reduce unit (each slice sum < 2^32).
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
  const uint32_t s0 = __reduce_add_sync(PS_FULL, (uint32_t)(x & 0x7FFFFFFu));
  const uint32_t s1 = __reduce_add_sync(PS_FULL, (uint32_t)(x >> 27));
  return (unsigned long long)s0 + ((unsigned long long)s1 << 27);
}

// sum_{k=1..n} (2k)^2: the rank-square total of a tie-free walk
__device__ __forceinline__ unsigned long long sq_closed(unsigned long long n) {
  return 4ull * (n * (n + 1) * (2 * n + 1) / 6ull);
}

// Shared-memory layout, in 32-bit words (all regions 16-byte aligned).
//
// Group-table mode (a tied feature with at most `cap` tie groups): instead of
// resolving each position's tie group per pair (word records + word_r2), the
// pair's kept prefix is evaluated once per GROUP START (tab[k] = Pfx(bpos[k]),
// k <= D) and a kept position p of group k = gid(p) gets 2r = tab[k] +
// tab[k + 1] + 1, gid(p) = gp[p / 32] + popc(boundary bits <= p) - 1.  The
// h-side regions hold either the fallback tables (lastb | nextb) or
// (gp | group starts | tab [| g's group starts when g is streamed]); g's
// double-buffered regions hold (lastb | nextb) or (gp | group starts).
struct WalkLayout {
  uint32_t inv16, R16, tbh, lbh16, nbh16, par, K, Pl, SE;
  uint32_t gph16, bposh16, tab16, bposg16s;  // h side (aliases lbh16 / nbh16) + streamed g's group starts
  uint32_t tabg32;                            // g's packed group table (R2: own region; else aliases par)
  uint32_t og16[2], tbg[2], lbg16[2], nbg16[2];
  uint32_t gpg16[2], bposg16[2];              // alias lbg16 / nbg16
  uint32_t words;
  __host__ __device__ static int64_t capr(int cap) { return ((int64_t)cap + 2 + 7) & ~int64_t(7); }  // entries
  __host__ __device__ WalkLayout(int64_t ldo, int64_t ldt, bool ogs, bool r2, int cap) {
    uint32_t w = 0;
    auto take = [&](int64_t bytes) {
      const uint32_t o = w;
      w += (uint32_t)(((bytes + 15) / 16) * 4);
      return o;
    };
    const int64_t ldt2 = ((ldt * 2 + 15) / 16) * 16;  // bytes of one 16-bit per-word table
    const int64_t cr = capr(cap);
    inv16 = take(ldo * 2) * 2;
    R16 = take(ldo * 2) * 2;
    tbh = take(ldt * 4);
    {
      const int64_t tab_bytes = cap > 0 ? ldt2 + 2 * cr * (ogs ? 2 : 3) : 0;
      const uint32_t u = take(std::max<int64_t>(2 * ldt2, tab_bytes));
      lbh16 = u * 2;
      nbh16 = lbh16 + (uint32_t)(ldt2 / 2);
      gph16 = lbh16;
      bposh16 = nbh16;
      tab16 = bposh16 + (uint32_t)cr;
      bposg16s = tab16 + (uint32_t)cr;
    }
    par = r2 ? 0 : take(std::max<int64_t>(ldt * 4, cap > 0 ? 4 * cr : 0));
    tabg32 = r2 ? (cap > 0 ? take(4 * cr) : 0) : par;
    // per word of the walked order: kept bits K, segment-relative prefix P and
    // (R2 tied passes) the prefixes of the tie groups entering / leaving it;
    // for R2 one 16-byte record {K, P, sp, ep} per word (one LDS.128), else
    // K and a 16-bit P (S > 32767 must fit 227 KB)
    K = r2 ? take(ldt * 16) : take(ldt * 4);
    Pl = r2 ? 0 : take(ldt * 2) * 2;
    SE = 0;
    for (int b = 0; b < 2; ++b) {
      og16[b] = ogs ? take(ldo * 2) * 2 : 0;
      tbg[b] = ogs ? take(ldt * 4) : 0;
      const int64_t tb = cap > 0 ? ldt2 + 2 * cr : 0;
      const uint32_t v = ogs ? take(std::max<int64_t>(2 * ldt2, tb)) * 2 : 0;
      lbg16[b] = v;
      nbg16[b] = v + (uint32_t)(ldt2 / 2);
      gpg16[b] = lbg16[b];
      bposg16[b] = nbg16[b];
    }
    words = w;
  }
};

// After phase 1: turn per-warp totals into segment bases (exclusive scan in
// registers: lane i of every warp holds the base of segment i).
__device__ __forceinline__ void segment_bases(const uint32_t* wtot, uint32_t& segpre, uint32_t& ntot) {
  const int lane = threadIdx.x & 31;
  const uint32_t v = lane < SW ? wtot[lane] : 0u;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
    if (lane >= o) x += y;
  }
  segpre = x - v;
  ntot = __shfl_sync(PS_FULL, x, 31);
}

#ifdef PS_WALK_TIMING
// cycles per phase, split by pair class (tied g) + 2 (tied h): [cls * 8 + phase],
// pair counts per class at [32 + cls]
__device__ unsigned long long g_walk_cycles[40];
#define WT(i)                                                                  \
  do {                                                                         \
    if (threadIdx.x == 0) {                                                    \
      const long long _t = clock64();                                          \
      atomicAdd(&g_walk_cycles[_wcls * 8 + (i)], (unsigned long long)(_t - _tw)); \
      if ((i) == 6) atomicAdd(&g_walk_cycles[32 + _wcls], 1ull);               \
      _tw = _t;                                                                \
    }                                                                          \
  } while (0)
#else
#define WT(i) \
  do {        \
  } while (0)
#endif

constexpr unsigned long long kClosed = ~0ull;  // "tie-free: use the closed form"

// Register word records of the S > 32767 walks: a warp walks at most
// ceil(2048 / SW) words (S <= 65535), one record per lane per slot.
constexpr int kRecSlots = (2048 / SW + 31) / 32;
__device__ __forceinline__ uint32_t pick_slot(const uint32_t (&r)[kRecSlots], int i) {
  uint32_t v = r[0];
#pragma unroll
  for (int t = 1; t < kRecSlots; ++t)
    if (i == t) v = r[t];
  return v;
}

// Walk of a warp's words [w0, w1) of g's order in groups of G words: the
// group's order entries (staged in shared memory, or streamed from global
// memory two groups ahead) are first mapped by pre() -- the gathers of the
// whole group issue back to back -- and then handed to body(word, value) in
// word order.  The shared accesses are volatile asm, so without the grouping
// each word's gather would wait for the previous word's store; the global
// loads are volatile too, so that ptxas cannot sink them to their use.
__device__ __forceinline__ uint32_t ldg16_early(const uint16_t* a) {
  unsigned short v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(a));
  return v;
}
// eight loads of one lane at a fixed 32-position stride (eight consecutive
// words of a streamed order): immediate offsets, one address per group
__device__ __forceinline__ void ldg_x8(const uint16_t* p, uint32_t (&d)[8]) {
  unsigned short v0, v1, v2, v3, v4, v5, v6, v7;
  asm volatile(
      "ld.global.nc.u16 %0, [%8];\n\tld.global.nc.u16 %1, [%8+64];\n\t"
      "ld.global.nc.u16 %2, [%8+128];\n\tld.global.nc.u16 %3, [%8+192];\n\t"
      "ld.global.nc.u16 %4, [%8+256];\n\tld.global.nc.u16 %5, [%8+320];\n\t"
      "ld.global.nc.u16 %6, [%8+384];\n\tld.global.nc.u16 %7, [%8+448];"
      : "=h"(v0), "=h"(v1), "=h"(v2), "=h"(v3), "=h"(v4), "=h"(v5), "=h"(v6), "=h"(v7)
      : "l"(p));
  d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3; d[4] = v4; d[5] = v5; d[6] = v6; d[7] = v7;
}
__device__ __forceinline__ void ldg_x8(const uint32_t* p, uint32_t (&d)[8]) {
  asm volatile(
      "ld.global.nc.u32 %0, [%8];\n\tld.global.nc.u32 %1, [%8+128];\n\t"
      "ld.global.nc.u32 %2, [%8+256];\n\tld.global.nc.u32 %3, [%8+384];\n\t"
      "ld.global.nc.u32 %4, [%8+512];\n\tld.global.nc.u32 %5, [%8+640];\n\t"
      "ld.global.nc.u32 %6, [%8+768];\n\tld.global.nc.u32 %7, [%8+896];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
      : "l"(p));
}
__device__ __forceinline__ uint32_t ldg_early(const uint16_t* a) { return ldg16_early(a); }
__device__ __forceinline__ uint32_t ldg_early(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a));
  return v;
}

// Walk of a warp's words [w0, w1) of a streamed g order (global memory;
// 16-bit sample ids, or 32-bit id | group id << 16) in groups of G = 8 words,
// loaded two groups ahead: the group's entries are first mapped by pre() --
// the gathers of the whole group issue back to back -- and then handed to
// body(word, pre(x), x) in word order.  The shared accesses are volatile asm,
// so without the grouping each word's gather would wait for the previous
// word's store; the global loads are volatile too, so that ptxas cannot sink
// them to their use.  Three register groups rotate by unrolling (no moves);
// full groups load with immediate offsets.
template <class E, class Pre, class Body>
__device__ __forceinline__ void walk_order(const E* __restrict__ og, int w0, int w1, Pre&& pre, Body&& body) {
  const int lane = threadIdx.x & 31;
  constexpr int G = 8;
  const E* pl = og + lane;
  auto load = [&](uint32_t (&d)[G], int wb) {
    if (wb + G <= w1) {
      ldg_x8(pl + (size_t)wb * 32, d);
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u) d[u] = wb + u < w1 ? ldg_early(pl + (size_t)(wb + u) * 32) : 0u;
    }
  };
  auto run = [&](const uint32_t (&d)[G], int wb) {
    uint32_t q[G];
#pragma unroll
    for (int u = 0; u < G; ++u) q[u] = pre(d[u]);
    if (wb + G <= w1) {
#pragma unroll
      for (int u = 0; u < G; ++u) body(wb + u, q[u], d[u]);
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (wb + u < w1) body(wb + u, q[u], d[u]);
    }
  };
  uint32_t A[G], B[G], C[G];
  load(A, w0);
  load(B, w0 + G);
  for (int wb = w0; wb < w1; wb += 3 * G) {
    load(C, wb + 2 * G);
    run(A, wb);
    if (wb + G >= w1) break;
    load(A, wb + 3 * G);
    run(B, wb + G);
    if (wb + 2 * G >= w1) break;
    load(B, wb + 4 * G);
    run(C, wb + 2 * G);
  }
}

template <bool OGS, bool R2>
__global__ void __launch_bounds__(STH, OGS ? (SW <= 16 ? 32 / SW : 1) : (SW <= 16 ? 16 / SW : 1))
spearman_walk_kernel(const uint16_t* __restrict__ order, const uint16_t* __restrict__ inv, int64_t ldo,
                     const uint32_t* __restrict__ tb, const uint16_t* __restrict__ lastb,
                     const uint16_t* __restrict__ nextb, int64_t ldt, const uint8_t* __restrict__ tied,
                     const int32_t* __restrict__ lens, const uint16_t* __restrict__ gpt,
                     const uint16_t* __restrict__ bpos, const int32_t* __restrict__ ngrp,
                     const uint32_t* __restrict__ ordgid, int cap, int64_t F,
                     const int4* __restrict__ items, int n_items, int once, int* __restrict__ queue, PairParts out) {
  const WalkLayout L(ldo, ldt, OGS, R2, cap);
  __shared__ uint32_t wtot[SW], wtotA[SW];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the window base comes from a volatile asm so that it stays in a register:
  // ptxas otherwise re-derives it (S2R SR_CgaCtaId + LEA) inside hot loops
  uint32_t sb;
  asm volatile("{\n\t.reg .u64 t;\n\tcvta.to.shared.u64 t, %1;\n\tcvt.u32.u64 %0, t;\n\t}" : "=r"(sb) : "l"(sm32));
  const uint32_t aInv = sb + 2 * L.inv16, aR = sb + 2 * L.R16, aK = sb + 4 * L.K, aP = sb + 2 * L.Pl;
  const uint32_t aPar = sb + 4 * L.par;
  auto kA = [&](uint32_t w) -> uint32_t { return R2 ? aK + 16 * w : aK + 4 * w; };
  auto stK = [&](uint32_t w, uint32_t v) { st32(kA(w), v); };
  const uint32_t aTbh = sb + 4 * L.tbh, aLbh = sb + 2 * L.lbh16, aNbh = sb + 2 * L.nbh16;
  const uint32_t ltmask = lanemask_lt();
  auto ldP = [&](uint32_t w) -> uint32_t { return R2 ? ld32(aK + 16 * w + 4) : ld16(aP + 2 * w); };
  auto stP = [&](uint32_t w, uint32_t v) {
    if (R2) st32(aK + 16 * w + 4, v);
    else st16(aP + 2 * w, v);
  };
  auto stKP = [&](uint32_t w, uint32_t k, uint32_t pv) {  // phase 1, lane 0
    if (R2) {
      st64(aK + 16 * w, k, pv);
    } else {
      stK(w, k);
      st16(aP + 2 * w, pv);
    }
  };
  // absolute kept-prefix of position x: P[x/32] + popc(bits of K below x)
  auto pfx = [&](uint32_t x) -> uint32_t {
    const uint32_t w = x >> 5;
    return ldP(w) + __popc(ld32(kA(w)) & ((1u << (x & 31u)) - 1u));
  };

  // R2 tied passes: for each of this warp's words [w0, w1) of a feature of
  // length nf, store (Pfx(start of the tie group entering the word),
  // Pfx(end of the group leaving it)) -- one lane per word, so phase 2 reads
  // two warp-uniform values instead of resolving group bounds per element.
  // Word prefixes are segment-relative; the base of another warp's segment
  // is lane s of segpre (segment_bases), so no block barrier is needed.
  auto fill_spep = [&](int w0, int w1, int Lseg, uint32_t segpre, uint32_t tot, uint32_t nf, auto&& Tat,
                       auto&& LBat, auto&& NBat) {
    const uint32_t own = __shfl_sync(PS_FULL, segpre, warp);
    auto pabs = [&](uint32_t x) -> uint32_t {  // all lanes (shuffle inside)
      const uint32_t wx = min(x, nf - 1u) >> 5;
      const uint32_t base = __shfl_sync(PS_FULL, segpre, (int)(wx / (uint32_t)Lseg));
      const uint32_t v = ldP(wx) + base + __popc(ld32(kA(wx)) & ((1u << (x & 31u)) - 1u));
      return x >= nf ? tot : v;
    };
    for (int wb = w0; wb < w1; wb += 32) {
      const int w = min(wb + lane, w1 - 1);
      const uint32_t T = Tat(w);
      const uint32_t ps = pabs(LBat(w ? w - 1 : 0));
      const uint32_t pe = pabs(min(NBat(w + 1), nf));
      if (wb + lane < w1) st64(aK + 16 * w + 8, (T & 1u) ? ldP(w) + own : ps, pe);
    }
    __syncwarp();
  };

  for (int64_t i = threadIdx.x; i < ldo; i += STH) SM16[L.R16 + i] = 0;
  if (!R2)
    for (int64_t i = threadIdx.x; i < ldt; i += STH) sm32[L.par + i] = 0u;

  // group-table mode of g: tied, few enough groups, and the h-side regions
  // not holding h's fallback tables (gtab_ok, per item)
  bool gtab_ok = false;
  auto gtab_of = [&](int64_t g) -> bool { return gtab_ok && tied[g] && ngrp[g] <= cap; };
  auto prefetch = [&](int64_t g, int b) {
    const int ng = lens[g];
    const int nch = ((ng + 31) >> 5) * 4;  // whole 32-position words (sentinel padded)
    const uint32_t so = sb + L.og16[b] * 2;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(order + g * ldo);
    for (int c = threadIdx.x; c < nch; c += STH) cp16(so + c * 16, src + c * 16);
    if (tied[g]) {
      const int tch4 = (int)(ldt * 4 / 16), tch2 = (int)(ldt * 2 / 16);
      const unsigned char* t4 = reinterpret_cast<const unsigned char*>(tb + g * ldt);
      for (int c = threadIdx.x; c < tch4; c += STH) cp16(sb + L.tbg[b] * 4 + c * 16, t4 + c * 16);
      if (gtab_of(g)) {
        const unsigned char* g2 = reinterpret_cast<const unsigned char*>(gpt + g * ldt);
        const unsigned char* b2 = reinterpret_cast<const unsigned char*>(bpos + g * ldo);
        const int bch = (ngrp[g] + 1 + 7) >> 3;
        for (int c = threadIdx.x; c < tch2; c += STH) cp16(sb + L.gpg16[b] * 2 + c * 16, g2 + c * 16);
        for (int c = threadIdx.x; c < bch; c += STH) cp16(sb + L.bposg16[b] * 2 + c * 16, b2 + c * 16);
      } else {
        const unsigned char* l2 = reinterpret_cast<const unsigned char*>(lastb + g * ldt);
        const unsigned char* n2 = reinterpret_cast<const unsigned char*>(nextb + g * ldt);
        for (int c = threadIdx.x; c < tch2; c += STH) {
          cp16(sb + L.lbg16[b] * 2 + c * 16, l2 + c * 16);
          cp16(sb + L.nbg16[b] * 2 + c * 16, n2 + c * 16);
        }
      }
    }
    asm volatile("cp.async.commit_group;");
  };

  // Group table of the walked feature (D groups, starts at shared byte address
  // aB, length nf): tab[k] = Pfx(start of group k), k <= D, from the pair's
  // segment-relative word prefixes (segment of word w: w / Lseg, base: lane
  // of segpre).  Returns this thread's share of sum_k c_k (2 r_k)^2.
  const uint32_t aTab = sb + 2 * L.tab16;
  auto build_tab = [&](int D, uint32_t aB, int Lseg, uint32_t segpre, uint32_t tot,
                       uint32_t nf) -> unsigned long long {
    // ceil(2^32 / Lseg): floor(w / Lseg) = umulhi(w, magic) exactly for w < 2^16 (Lseg = 1 overflows: direct)
    const uint32_t magic = (uint32_t)((0x100000000ull + (uint32_t)Lseg - 1u) / (uint32_t)Lseg);
    for (int kb = warp * 32; kb <= D; kb += STH) {  // warp-uniform
      const int k = kb + lane;
      const uint32_t x = k <= D ? ld16(aB + 2 * (uint32_t)k) : nf;
      const uint32_t wx = min(x, nf - 1u) >> 5;
      const uint32_t base = __shfl_sync(PS_FULL, segpre, Lseg == 1 ? (int)wx : (int)__umulhi(wx, magic));
      const uint32_t v = ldP(wx) + base + __popc(ld32(kA(wx)) & ((1u << (x & 31u)) - 1u));
      if (k <= D) st16(aTab + 2 * (uint32_t)k, x >= nf ? tot : v);
    }
    __syncthreads();
    unsigned long long acc = 0;
    for (int k = threadIdx.x; k < D; k += STH) {
      const uint32_t a = ld16(aTab + 2 * (uint32_t)k), b = ld16(aTab + 2 * (uint32_t)k + 2u);
      const unsigned long long r2 = a + b + 1u;
      acc += (unsigned long long)(b - a) * r2 * r2;
    }
    return acc;
  };
  // g's packed table: tabg[k] = Pfx(start of group k) | Pfx(its end) << 16
  // (k < D); the caller's next block barrier publishes it
  const uint32_t aTabG = sb + 4 * L.tabg32;
  auto build_tabg = [&](int D, uint32_t aB, int Lseg, uint32_t segpre, uint32_t tot,
                        uint32_t nf) -> unsigned long long {
    const uint32_t magic = (uint32_t)((0x100000000ull + (uint32_t)Lseg - 1u) / (uint32_t)Lseg);
    auto pabs = [&](uint32_t x) -> uint32_t {  // all lanes (shuffle inside)
      const uint32_t wx = min(x, nf - 1u) >> 5;
      const uint32_t base = __shfl_sync(PS_FULL, segpre, Lseg == 1 ? (int)wx : (int)__umulhi(wx, magic));
      const uint32_t v = ldP(wx) + base + __popc(ld32(kA(wx)) & ((1u << (x & 31u)) - 1u));
      return x >= nf ? tot : v;
    };
    unsigned long long acc = 0;
    for (int kb = warp * 32; kb < D; kb += STH) {  // warp-uniform
      const int k = kb + lane;
      const uint32_t a = pabs(k < D ? ld16(aB + 2 * (uint32_t)k) : nf);
      const uint32_t b = pabs(k < D ? ld16(aB + 2 * (uint32_t)k + 2u) : nf);
      if (k < D) {
        st32(aTabG + 4 * (uint32_t)k, a | (b << 16));
        const unsigned long long r2 = a + b + 1u;
        acc += (unsigned long long)(b - a) * r2 * r2;
      }
    }
    return acc;
  };
  // doubled rank of every lane of a word of a group-table feature
  auto tab_r2 = [&](uint32_t T, uint32_t gw) -> uint32_t {
    const uint32_t gid = gw + __popc(T & (0xFFFFFFFFu >> (31 - lane))) - 1u;
    return ld16(aTab + 2 * gid) + ld16(aTab + 2 * gid + 2u) + 1u;
  };

  __shared__ int4 s_it;
  bool par_dirty = false;  // (!R2) g's packed table, which aliases the parity words, was used
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int item = atomicAdd(queue, 1);
      s_it = item < n_items ? items[item] : make_int4(-1, 0, 0, 0);
    }
    __syncthreads();
    const int4 it = s_it;
    if (it.x < 0) break;
    const int64_t h = it.x;
    const int64_t lo = it.y;  // g block [lo, gmax]
    const int nh = lens[h];
    const bool th = tied[h] != 0;
    const int Dh = th ? ngrp[h] : 0;
    const bool htab = th && Dh <= cap;
    gtab_ok = !th || htab;
    {
      const uint4* src = reinterpret_cast<const uint4*>(inv + h * ldo);
      uint4* dst = reinterpret_cast<uint4*>(&SM16[L.inv16]);
      for (int64_t i = threadIdx.x; i < ldo / 8; i += STH) dst[i] = src[i];
      if (htab) {
        for (int64_t i = threadIdx.x; i < ldt; i += STH) {
          sm32[L.tbh + i] = tb[h * ldt + i];
          SM16[L.gph16 + i] = gpt[h * ldt + i];
        }
        for (int i = threadIdx.x; i <= Dh; i += STH) SM16[L.bposh16 + i] = bpos[h * ldo + i];
      } else if (th) {
        for (int64_t i = threadIdx.x; i < ldt; i += STH) {
          sm32[L.tbh + i] = tb[h * ldt + i];
          SM16[L.lbh16 + i] = lastb[h * ldt + i];
          SM16[L.nbh16 + i] = nextb[h * ldt + i];
        }
      }
    }
    const int64_t gmax = it.z - 1;
    if (OGS && lo <= gmax) prefetch(lo, 0);
    __syncthreads();
    const int nwb = (nh + 31) >> 5;
    const int Lb = (nwb + SW - 1) / SW;
    const int b0 = min(nwb, warp * Lb), b1 = min(nwb, b0 + Lb);
#ifdef PS_WALK_TIMING
    long long _tw = clock64();
#endif
    int ng_next = lo <= gmax ? lens[lo] : 0;
    bool tg_next = lo <= gmax ? tied[lo] != 0 : false;
    int dg_next = lo <= gmax ? ngrp[lo] : 0;
    for (int64_t g = lo; g <= gmax; ++g) {
      const int buf = (int)((g - lo) & 1);
      const int ng = ng_next;
      const bool tg = tg_next;
      const int Dg = dg_next;
      if (g + 1 <= gmax) {
        ng_next = lens[g + 1];
        tg_next = tied[g + 1] != 0;
        dg_next = ngrp[g + 1];
      }
      if (OGS) {
        if (g + 1 <= gmax) prefetch(g + 1, buf ^ 1);
        else asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 1;");
      }
      // the previous pair's pass B (reads / clears R, reads the word records)
      // is complete in every warp before this pair's pass A writes them
      __syncthreads();
#ifdef PS_WALK_TIMING
      const int _wcls = (tg ? 1 : 0) + (th ? 2 : 0);
#endif
      WT(0);
      const uint32_t aOg = sb + 2 * L.og16[buf];
      const uint32_t aTbg = sb + 4 * L.tbg[buf], aLbg = sb + 2 * L.lbg16[buf], aNbg = sb + 2 * L.nbg16[buf];
      const uint16_t* og_g = order + g * ldo;
      const bool gtab = tg && gtab_ok && Dg <= cap && (OGS || ordgid != nullptr);
      const uint32_t aBg = OGS ? sb + 2 * L.bposg16[buf] : sb + 2 * L.bposg16s;
      if (!OGS && gtab) {  // streamed g: its group starts by cp.async, waited for after phase 1
        const unsigned char* b2 = reinterpret_cast<const unsigned char*>(bpos + g * ldo);
        for (int c = threadIdx.x; c < ((Dg + 1 + 7) >> 3); c += STH) cp16(aBg + c * 16, b2 + c * 16);
        asm volatile("cp.async.commit_group;");
      }
      if (!R2 && par_dirty && tg && !gtab) {  // this pair may set parity bits: clear the table's entries
        for (int i = threadIdx.x; i < (int)ldt; i += STH) sm32[L.par + i] = 0u;
        par_dirty = false;
      }
      // ---------------- pass A, phase 1: keep bits over g's order ----------
      const int nwa = (ng + 31) >> 5;
      const int La = (nwa + SW - 1) / SW;
      const int a0 = min(nwa, warp * La), a1 = min(nwa, a0 + La);
      // Tie-free g: one sweep.  R[q] = (warp << 12) | local
      // rank within the warp's segment; the segment bases are folded in by
      // pass B, so no prefix phase is needed here.
      const bool encA = !tg && La * 32 <= (int)kEncMask;
      // 2r fits 16 bits for this pair (always when S <= 32767; for larger S
      // whenever the joint count n <= 32767): no parity bits needed
      bool r2fit = R2;
      uint32_t segpreA = 0, n = 0, abase = 0;
      unsigned long long sa2 = 0;
      if (encA) {
        uint32_t cnt = 0;
        auto body = [&](int, uint32_t q) {
          const bool keep = q != 0xFFFFu;
          const uint32_t B = __ballot_sync(PS_FULL, keep);
          if (keep) st16(aR + 2 * q, ((uint32_t)warp << kEncShift) | (cnt + __popc(B & ltmask) + 1u));
          cnt += __popc(B);
        };
        if (OGS) {  // (64-register kernels: the grouped walk costs more than it saves)
#pragma unroll 4
          for (int word = a0; word < a1; ++word)
            body(word, ld16(aInv + 2 * ld16(aOg + 2 * (uint32_t)(word * 32 + lane))));
        } else {
          walk_order(og_g, a0, a1, [&](uint32_t s) { return ld16(aInv + 2 * s); },
                     [&](int word, uint32_t q, uint32_t) { body(word, q); });
        }
        if (lane == 0) wtotA[warp] = cnt;
        __syncthreads();
        segment_bases(wtotA, segpreA, n);
        WT(1);
      } else {
      if (gtab) {
        // group-table g, one phase: every kept position scatters its group
        // id + 1 to R[q]; pass B reads 2 r_g from g's packed group table
        uint32_t cnt = 0;
        const uint32_t le = 0xFFFFFFFFu >> (31 - lane);
        if (OGS) {
          const uint32_t aGpg = sb + 2 * L.gpg16[buf];
#pragma unroll 4
          for (int word = a0; word < a1; ++word) {
            const uint32_t q = ld16(aInv + 2 * ld16(aOg + 2 * (uint32_t)(word * 32 + lane)));
            const uint32_t gid1 = ld16(aGpg + 2 * word) + __popc(ld32(aTbg + 4 * word) & le);
            const bool keep = q != 0xFFFFu;
            const uint32_t B = __ballot_sync(PS_FULL, keep);
            if (lane == 0) stKP(word, B, cnt);
            if (keep) st16(aR + 2 * q, gid1);
            cnt += __popc(B);
          }
        } else {
          // streamed g: sample id | group id << 16 per position (ordgid)
          walk_order(ordgid + g * ldo, a0, a1, [&](uint32_t x) { return ld16(aInv + 2 * (x & 0xFFFFu)); },
                     [&](int word, uint32_t q, uint32_t x) {
                       const bool keep = q != 0xFFFFu;
                       const uint32_t B = __ballot_sync(PS_FULL, keep);
                       if (lane == 0) stKP(word, B, cnt);
                       if (keep) st16(aR + 2 * q, (x >> 16) + 1u);
                       cnt += __popc(B);
                     });
        }
        if (lane == 0) wtot[warp] = cnt;
      } else {
        // q = inv_h[order_g[p]]; with g's order staged in shared memory the
        // gathered q overwrites it in place, so phase 2 reads it sequentially
        uint32_t cnt = 0;
        auto body = [&](int word, uint32_t q) {
          if (OGS) st16(aOg + 2 * (uint32_t)(word * 32 + lane), q);
          const uint32_t B = __ballot_sync(PS_FULL, q != 0xFFFFu);
          if (lane == 0) stKP(word, B, cnt);
          cnt += __popc(B);
        };
        if (OGS) {
#pragma unroll 4
          for (int word = a0; word < a1; ++word)
            body(word, ld16(aInv + 2 * ld16(aOg + 2 * (uint32_t)(word * 32 + lane))));
        } else {
          walk_order(og_g, a0, a1, [&](uint32_t s) { return ld16(aInv + 2 * s); },
                     [&](int word, uint32_t q, uint32_t) { body(word, q); });
        }
        if (lane == 0) wtot[warp] = cnt;
      }
      if (!OGS && gtab) asm volatile("cp.async.wait_group 0;");
      __syncthreads();
      WT(1);
      {
        uint32_t segpre;
        segment_bases(wtot, segpre, n);
        r2fit = R2 || (2u * n + 1u <= 0xFFFFu);
        abase = __shfl_sync(PS_FULL, segpre, warp);
        if (gtab) {
          sa2 = build_tabg(Dg, aBg, La, segpre, n, (uint32_t)ng);
          if (!R2) par_dirty = true;
        } else if (tg && R2) {
          if (OGS)
            fill_spep(a0, a1, La, segpre, n, (uint32_t)ng, [&](int w) { return ld32(aTbg + 4 * w); },
                      [&](int w) { return ld16(aLbg + 2 * w); }, [&](int w) { return ld16(aNbg + 2 * w); });
          else
            fill_spep(a0, a1, La, segpre, n, (uint32_t)ng, [&](int w) { return tb[g * ldt + w]; },
                      [&](int w) { return (uint32_t)lastb[g * ldt + w]; },
                      [&](int w) { return (uint32_t)nextb[g * ldt + w]; });
        } else if (tg) {  // absolute prefixes for arbitrary-position lookups
          for (int w = a0 + lane; w < a1; w += 32) stP(w, ldP(w) + abase);
          if (threadIdx.x == 0) {
            stK(nwa, 0u);
            stP(nwa, n);
          }
          __syncthreads();
        }
      }
      WT(2);
      // ---------------- pass A, phase 2: ranks -> R[q] -------------------
      auto q_at = [&](uint32_t p) -> uint32_t { return OGS ? ld16(aOg + 2 * p) : ld16(aInv + 2 * (uint32_t)og_g[p]); };
      auto st_r2 = [&](uint32_t q, uint32_t r2) {
        if (r2fit) {
          st16(aR + 2 * q, r2);
        } else {
          st16(aR + 2 * q, r2 >> 1);
          if (r2 & 1u) atomicOr(&sm32[L.par + (q >> 5)], 1u << (q & 31u));
        }
      };
      if (gtab) {
        // (no second phase: ranks are resolved through g's table in pass B)
      } else if (!tg) {
#pragma unroll(OGS ? 4 : 8)
        for (int word = a0; word < a1; ++word) {
          const uint32_t kw = ld32(kA(word));
          const uint32_t r = abase + ldP(word) + __popc(kw & ltmask) + 1u;
          const uint32_t q = q_at((uint32_t)(word * 32 + lane));
          if ((kw >> lane) & 1u) st16(aR + 2 * q, r2fit ? 2u * r : r);
        }
      } else if (R2) {
        const uint32_t* tbgg = tb + g * ldt;
#pragma unroll(OGS ? 4 : 8)
        for (int word = a0; word < a1; ++word) {
          const uint4 rec = ld128(aK + 16 * word);  // {K, P, sp, ep}
          const uint32_t kw = rec.x;
          const uint32_t T = OGS ? ld32(aTbg + 4 * word) : tbgg[word];
          const uint32_t r2 = word_r2(T, rec.z, rec.w, kw, rec.y + abase);
          if ((kw >> lane) & 1u) {
            const uint32_t q = q_at((uint32_t)(word * 32 + lane));
            sa2 += (unsigned long long)r2 * r2;
            st16(aR + 2 * q, r2);
          }
        }
      } else {
        // S > 32767 (no room for 16-byte word records): the records of the
        // warp's own words live in registers instead -- lane j of slot i holds
        // word a0 + 32 i + j's {K, Pfx, T, group-entry / exit prefixes} -- and
        // reach the walking warp by shuffle; g's order is prefetched one
        // 8-word group ahead, so neither the tie tables' global loads nor the
        // prefix lookups sit on the per-word chain.
        const uint32_t* tbgg = tb + g * ldt;
        const uint16_t* lbgg = lastb + g * ldt;
        const uint16_t* nbgg = nextb + g * ldt;
        uint32_t rK[kRecSlots], rP[kRecSlots], rT[kRecSlots], rS[kRecSlots], rE[kRecSlots];
#pragma unroll
        for (int i = 0; i < kRecSlots; ++i) {
          const int w = a0 + 32 * i + lane;
          rK[i] = rP[i] = rT[i] = rS[i] = rE[i] = 0u;
          if (w < a1) {
            uint32_t lb, nb;
            if (OGS) {
              rT[i] = ld32(aTbg + 4 * w);
              lb = ld16(aLbg + 2 * (w ? w - 1 : 0));
              nb = ld16(aNbg + 2 * (w + 1));
            } else {
              rT[i] = tbgg[w];
              lb = lbgg[w ? w - 1 : 0];
              nb = nbgg[w + 1];
            }
            rK[i] = ld32(kA(w));
            rP[i] = ldP(w);
            rS[i] = (rT[i] & 1u) ? rP[i] : pfx(lb);
            rE[i] = pfx(min(nb, (uint32_t)ng));
          }
        }
        auto og_at = [&](int word) -> uint32_t {
          if (word >= a1) return 0u;
          const uint32_t p = (uint32_t)(word * 32 + lane);
          return OGS ? ld16(aOg + 2 * p) : (uint32_t)og_g[p];
        };
        uint32_t sc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) sc[u] = og_at(a0 + u);
        for (int w8 = a0; w8 < a1; w8 += 8) {
          uint32_t sn[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) sn[u] = og_at(w8 + 8 + u);
          const int i = (w8 - a0) >> 5;
          const uint32_t RK = pick_slot(rK, i), RP = pick_slot(rP, i), RT = pick_slot(rT, i);
          const uint32_t RS = pick_slot(rS, i), RE = pick_slot(rE, i);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int word = w8 + u;
            if (word < a1) {  // warp-uniform
              const int jl = (word - a0) & 31;
              const uint32_t kw = __shfl_sync(PS_FULL, RK, jl);
              const uint32_t r2 = word_r2(__shfl_sync(PS_FULL, RT, jl), __shfl_sync(PS_FULL, RS, jl),
                                          __shfl_sync(PS_FULL, RE, jl), kw, __shfl_sync(PS_FULL, RP, jl));
              if ((kw >> lane) & 1u) {
                const uint32_t q = OGS ? sc[u] : ld16(aInv + 2 * sc[u]);
                sa2 += (unsigned long long)r2 * r2;
                if (r2fit) {
                  st16(aR + 2 * q, r2);
                } else {
                  st16(aR + 2 * q, r2 >> 1);
                  if (r2 & 1u) atomicOr(&sm32[L.par + (q >> 5)], 1u << (q & 31u));
                }
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) sc[u] = sn[u];
        }
      }
      __syncthreads();
      }  // two-phase pass A
      WT(3);
      // decode R -> 2 r_g (all lanes must execute: shuffles)
      auto r2g_of = [&](uint32_t v, int word) -> uint32_t {
        if (encA) return 2u * (__shfl_sync(PS_FULL, segpreA, (int)(v >> kEncShift)) + (v & kEncMask));
        if (gtab) {  // v = group id + 1 (0: not kept -- any in-range entry)
          const uint32_t e = ld32(aTabG + 4 * (v ? v - 1u : 0u));
          return (e & 0xFFFFu) + (e >> 16) + 1u;
        }
        if (r2fit) return v;
        return 2u * v + (tg ? ((ld32(aPar + 4 * word) >> lane) & 1u) : 0u);
      };
      // parity words of g's doubled ranks are in use (cleared on the way)
      const bool parA = !r2fit && tg && !gtab;
      const bool sweepB = !th;
      unsigned long long sab = 0, sbb = 0, s0 = 0;
      uint32_t wtotB = 0;
      if (sweepB) {
        // Tie-free h: one sweep; per warp sum r2g * local_h and sum r2g, the
        // segment bases of h's order are folded in after the reduction.
        uint32_t cnt = 0, s0l = 0;  // s0l: per lane <= 2S * (words per warp) < 2^32
        auto sweep = [&](auto enc) {
#pragma unroll(OGS ? 4 : 8)
          for (int word = b0; word < b1; ++word) {
            const uint32_t q = (uint32_t)(word * 32 + lane);
            const uint32_t v = ld16(aR + 2 * q);
            const bool keep = v != 0u;
            const uint32_t B = __ballot_sync(PS_FULL, keep);
            uint32_t r2g;
            if constexpr (decltype(enc)::value) r2g = (__shfl_sync(PS_FULL, segpreA, (int)(v >> kEncShift)) + (v & kEncMask)) << 1;
            else r2g = r2g_of(v, word);
            if (keep) {
              sab += (unsigned long long)r2g * (cnt + __popc(B & ltmask) + 1u);
              s0l += r2g;
              st16(aR + 2 * q, 0u);
            }
            cnt += __popc(B);
          }
        };
        if (encA) sweep(std::true_type{});
        else sweep(std::false_type{});
        s0 = s0l;
        wtotB = cnt;
      } else {
      // ---------------- pass B, phase 1: keep = R != 0 over h's order ------
      {
        uint32_t cnt = 0;
#pragma unroll(OGS ? 4 : 8)
        for (int word = b0; word < b1; ++word) {
          const bool keep = ld16(aR + 2 * (uint32_t)(word * 32 + lane)) != 0u;
          const uint32_t B = __ballot_sync(PS_FULL, keep);
          if (lane == 0) stKP(word, B, cnt);
          cnt += __popc(B);
        }
        if (lane == 0) wtot[warp] = cnt;
      }
      __syncthreads();
      WT(4);
      uint32_t bbase;
      {
        uint32_t segpre, tot;
        segment_bases(wtot, segpre, tot);
        bbase = __shfl_sync(PS_FULL, segpre, warp);
        if (htab) {
          sbb = build_tab(Dh, sb + 2 * L.bposh16, Lb, segpre, tot, (uint32_t)nh);
        } else if (th && R2) {
          fill_spep(b0, b1, Lb, segpre, tot, (uint32_t)nh, [&](int w) { return ld32(aTbh + 4 * w); },
                    [&](int w) { return ld16(aLbh + 2 * w); }, [&](int w) { return ld16(aNbh + 2 * w); });
        } else if (th) {
          for (int w = b0 + lane; w < b1; w += 32) stP(w, ldP(w) + bbase);
          if (threadIdx.x == 0) {
            stK(nwb, 0u);
            stP(nwb, tot);
          }
          __syncthreads();
        }
      }
      // ---------------- pass B, phase 2: accumulate, clear R ---------------
      if (htab) {
        const uint32_t aGph = sb + 2 * L.gph16;
        auto walkt = [&](auto enc) {
#pragma unroll 4
          for (int word = b0; word < b1; ++word) {
            const uint32_t kw = ld32(kA(word));
            const uint32_t q = (uint32_t)(word * 32 + lane);
            const uint32_t v = ld16(aR + 2 * q);
            uint32_t r2g;  // all lanes (shuffle)
            if constexpr (decltype(enc)::value)
              r2g = (__shfl_sync(PS_FULL, segpreA, (int)(v >> kEncShift)) + (v & kEncMask)) << 1;
            else
              r2g = r2g_of(v, word);
            const uint32_t r2h = tab_r2(ld32(aTbh + 4 * word), ld16(aGph + 2 * word));
            if ((kw >> lane) & 1u) {
              sab += (unsigned long long)r2g * r2h;
              st16(aR + 2 * q, 0u);
            }
          }
        };
        if (encA) walkt(std::true_type{});
        else walkt(std::false_type{});
      } else if (!th) {
#pragma unroll(OGS ? 4 : 8)
        for (int word = b0; word < b1; ++word) {
          const uint32_t kw = ld32(kA(word));
          const uint32_t q = (uint32_t)(word * 32 + lane);
          const uint32_t v = ld16(aR + 2 * q);
          const uint32_t r2g = r2g_of(v, word);
          const uint32_t rh = bbase + ldP(word) + __popc(kw & ltmask) + 1u;
          if ((kw >> lane) & 1u) {
            sab += (unsigned long long)r2g * rh;
            st16(aR + 2 * q, 0u);
          }
        }
        sab *= 2ull;  // r2g * r_h = (2 r_g)(2 r_h) / 2
      } else if (R2) {
        auto walk2 = [&](auto enc) {
#pragma unroll(OGS ? 4 : 8)
          for (int word = b0; word < b1; ++word) {
            const uint4 rec = ld128(aK + 16 * word);  // {K, P, sp, ep}
            const uint32_t kw = rec.x;
            const uint32_t q = (uint32_t)(word * 32 + lane);
            const uint32_t v = ld16(aR + 2 * q);
            uint32_t r2g;  // all lanes (shuffle)
            if constexpr (decltype(enc)::value) r2g = (__shfl_sync(PS_FULL, segpreA, (int)(v >> kEncShift)) + (v & kEncMask)) << 1;
            else r2g = r2g_of(v, word);
            const uint32_t r2h = word_r2(ld32(aTbh + 4 * word), rec.z, rec.w, kw, rec.y + bbase);
            const uint32_t r2hk = (kw >> lane) & 1u ? r2h : 0u;
            sab += (unsigned long long)r2g * r2hk;  // r2g is meaningless where not kept: r2hk = 0
            sbb += (unsigned long long)r2hk * r2hk;
            st16(aR + 2 * q, 0u);                   // unkept positions hold 0 already
          }
        };
        if (encA) walk2(std::true_type{});
        else walk2(std::false_type{});
      } else {
        // S > 32767: register word records of h's walked words (see pass A)
        uint32_t rK[kRecSlots], rP[kRecSlots], rT[kRecSlots], rS[kRecSlots], rE[kRecSlots];
#pragma unroll
        for (int i = 0; i < kRecSlots; ++i) {
          const int w = b0 + 32 * i + lane;
          rK[i] = rP[i] = rT[i] = rS[i] = rE[i] = 0u;
          if (w < b1) {
            rT[i] = ld32(aTbh + 4 * w);
            rK[i] = ld32(kA(w));
            rP[i] = ldP(w);
            rS[i] = (rT[i] & 1u) ? rP[i] : pfx(ld16(aLbh + 2 * (w ? w - 1 : 0)));
            rE[i] = pfx(min(ld16(aNbh + 2 * (w + 1)), (uint32_t)nh));
          }
        }
#pragma unroll
        for (int i = 0; i < kRecSlots; ++i) {
          const int wb = b0 + 32 * i;
          const int we = min(b1, wb + 32);
#pragma unroll 4
          for (int word = wb; word < we; ++word) {
            const int jl = word - wb;
            const uint32_t kw = __shfl_sync(PS_FULL, rK[i], jl);
            const uint32_t q = (uint32_t)(word * 32 + lane);
            const uint32_t v = ld16(aR + 2 * q);
            const uint32_t r2g = r2g_of(v, word);  // all lanes (shuffle inside)
            const uint32_t r2h = word_r2(__shfl_sync(PS_FULL, rT[i], jl), __shfl_sync(PS_FULL, rS[i], jl),
                                         __shfl_sync(PS_FULL, rE[i], jl), kw, __shfl_sync(PS_FULL, rP[i], jl));
            if ((kw >> lane) & 1u) {
              sab += (unsigned long long)r2g * r2h;
              sbb += (unsigned long long)r2h * r2h;
              st16(aR + 2 * q, 0u);
            }
          }
        }
      }
      }  // two-phase pass B
      if (parA) {  // the parity words of this warp's h words were read: clear them
        __syncwarp();
        for (int w = b0 + lane; w < b1; w += 32) st32(aPar + 4 * w, 0u);
      }
      WT(5);
      // ---------------- per-warp partial sums -> global ---------------------
      // (no block barrier: the next pair's top barrier orders R / record reuse)
      unsigned long long c = sweepB ? s0 : sbb;
      if (tg) sa2 = warp_sum64(sa2);
      sab = warp_sum64(sab);
      c = warp_sum64(c);
      const int64_t cell = (g - out.c0) * F + h;
      if (lane == 0) {
        unsigned long long* pp = out.part + cell * (kSlots * SW) + warp;
        pp[0] = sa2;
        pp[SW] = sab;
        pp[2 * SW] = sweepB ? c | ((unsigned long long)wtotB << 40) : c;
      }
      if (threadIdx.x == 0)
        out.meta[cell] = (unsigned long long)n | ((unsigned long long)tg << 40) |
                         ((unsigned long long)th << 41) | ((unsigned long long)sweepB << 42);
      WT(6);
    }
    if (OGS) asm volatile("cp.async.wait_group 0;");
    if (once) break;  // one item per CTA: retiring CTAs let higher-priority kernels in
  }
}

// One warp per (g, h) cell of chunk [c0, c1): fold the SW per-warp partials
// into the exact 4x sums (tie-free walks: the closed-form sentinel).
// (columns h in [h0, h1) only: incremental launches fold their own columns)
__global__ void spearman_partials_kernel(PairParts in, int64_t F, int64_t c1, PairSums out, int64_t h0,
                                         int64_t h1) {
  const int lane = threadIdx.x & 31;
  const int64_t nh = h1 - h0;
  const int64_t ncell = (c1 - in.c0) * nh;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ci = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); ci < ncell;
       ci += nwarps) {
    const int64_t g = in.c0 + ci / nh, h = h0 + ci % nh;
    if (h < g) continue;  // warp-uniform
    const int64_t cell = (g - in.c0) * F + h;
    const unsigned long long meta = in.meta[cell];
    const bool tg = (meta >> 40) & 1, th = (meta >> 41) & 1, sweep = (meta >> 42) & 1;
    const unsigned long long* pp = in.part + cell * (kSlots * SW);
    unsigned long long a = 0, b = 0, c = 0;
    if (lane < SW) {
      a = pp[lane];
      b = pp[SW + lane];
      c = pp[2 * SW + lane];
    }
    if (sweep) {
      // sum_w 2 (sum r2g * local_h + base_w * sum r2g), base_w = kept count
      // of the h segments before w
      const unsigned long long s0 = c & ((1ull << 40) - 1), cnt = c >> 40;
      unsigned long long x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(PS_FULL, x, o);
        if (lane >= o) x += y;
      }
      b = lane < SW ? 2ull * (b + (x - cnt) * s0) : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(PS_FULL, a, o);
      b += __shfl_xor_sync(PS_FULL, b, o);
      c += __shfl_xor_sync(PS_FULL, c, o);
    }
    if (lane == 0) {
      const int64_t o = (g - out.row0) * F + h;
      out.n[o] = (long long)(meta & ((1ull << 40) - 1));
      out.sxx4[o] = (long long)(tg ? a : kClosed);
      out.sxy4[o] = (long long)b;
      out.syy4[o] = (long long)(th ? c : kClosed);
    }
  }
}

__device__ __forceinline__ void put(double* o, int64_t F, int64_t g, int64_t h, double v) {
  if (o) {
    o[g * F + h] = v;
    o[h * F + g] = v;
  }
}

// rho / p of one pair from its exact sums: n, raw sums of (2r_g)^2 (ra) and
// (2r_h)^2 (rc) -- kClosed: tie-free, closed form -- and of (2r_g)(2r_h) (rb).
__device__ __forceinline__ void spearman_from_sums(long long n, unsigned long long ra, unsigned long long rc,
                                                   long long rb, double* rho_out, double* p_out, int* err) {
  double rho = PS_NAN, p = PS_NAN;
  if (n > 1) {
    // raw sums of (2r)(2r) -> exact 4 x centred sums (rank totals are
    // preserved by tie averaging); tie-free walks use the closed form
    const unsigned long long un = (unsigned long long)n;
    const long long base = n * (n + 1) * (n + 1);
    const long long a4 = (long long)(ra == kClosed ? sq_closed(un) : ra) - base;
    const long long c4 = (long long)(rc == kClosed ? sq_closed(un) : rc) - base;
    const long long b4 = rb - base;
    // exact quarter-integers, identical to the reference's fp64 sums
    const double sxx = (double)a4 * 0.25;
    const double syy = (double)c4 * 0.25;
    const double sxy = (double)b4 * 0.25;
    if (sxx > 0.0 && syy > 0.0) {
      rho = sxy / sqrt(sxx * syy);
      if (rho > 1.0) rho = 1.0;
      else if (rho < -1.0) rho = -1.0;
      if (n != 2) {
        if (rho == 1.0 || rho == -1.0) {
          p = 0.0;
        } else {
          const double fn = (double)n;
          const double t = rho * sqrt((fn - 2.0) / (1.0 - rho * rho));
          p = 2.0 * psf::t_sf(fabs(t), fn - 2.0, err);
          if (p > 1.0) p = 1.0;
        }
      }
    }
  }
  *rho_out = rho;
  *p_out = p;
}

// rho / p from the exact sums (continuous.py:174-203), one thread per pair.
__host__ __device__ inline int64_t finish_before(int64_t g, int64_t lo, int64_t h0, int64_t h1) {
  // cells (x, h), x in [lo, g), h in [max(x, h0), h1)
  int64_t c = 0;
  const int64_t e0 = g < h0 + 1 ? g : h0 + 1;  // rows x <= h0: h1 - h0 cells each
  if (e0 > lo && h1 > h0) c += (e0 - lo) * (h1 - h0);
  const int64_t a = lo > h0 + 1 ? lo : h0 + 1, b = g < h1 ? g : h1;  // rows h0 < x < h1: h1 - x
  if (b > a) c += (b - a) * h1 - (a + b - 1) * (b - a) / 2;
  return c;
}

__global__ void spearman_finish_kernel(PairSums in, int64_t F, int64_t lo, int64_t hi, int64_t h0, int64_t h1,
                                       double* __restrict__ stat, double* __restrict__ pout,
                                       double* __restrict__ rho_out, int* __restrict__ err) {
  // one thread per cell (g <= h, g in [lo, hi), h in [h0, h1)): no idle lower half
  const int64_t total = finish_before(hi, lo, h0, h1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = lo, b = hi - 1;  // last row g with before(g) <= t
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (finish_before(mid, lo, h0, h1) <= t) a = mid;
      else b = mid - 1;
    }
    const int64_t g = a, h = (g > h0 ? g : h0) + (t - finish_before(g, lo, h0, h1));
    const int64_t cell = (g - in.row0) * F + h;
    double rho, p;
    spearman_from_sums(in.n[cell], (unsigned long long)in.sxx4[cell], (unsigned long long)in.syy4[cell],
                       in.sxy4[cell], &rho, &p, err);
    put(stat, F, g, h, rho);
    put(pout, F, g, h, p);
    put(rho_out, F, g, h, rho);
  }
}

size_t walk_smem(int64_t ldo, int64_t ldt, bool ogs, bool r2, int cap) {
  return (size_t)WalkLayout(ldo, ldt, ogs, r2, cap).words * 4;
}

// ---------------------------------------------------------------------------
// Wide walk (sample counts beyond the shared-memory walk: S > ~50k with the
// 16-bit tables, S > 65535 with the 32-bit ones; ps_wide.cuh).  One CTA per
// pair, pairs taken from an atomic queue over the cells (g, h >= g) of rows
// [lo, hi).  Pass A walks g's order keeping h's samples and scatters g's
// doubled rank into R[sample] (per-CTA global scratch); pass B walks h's
// order keeping g's samples and accumulates (2r_g)(2r_h).  Exact integer
// sums, finished like the shared-memory walk (spearman_from_sums).
template <typename OT>
__global__ void __launch_bounds__(wide::WT, 1)
spearman_wide_kernel(const OT* __restrict__ order, int64_t ldo, const uint32_t* __restrict__ tb,
                     const OT* __restrict__ lastb, const OT* __restrict__ nextb, int64_t ldt,
                     const int32_t* __restrict__ len, const uint32_t* __restrict__ mask, int64_t W, int64_t F,
                     int64_t lo, int64_t hi, uint32_t* __restrict__ scratch, int64_t scr, int* __restrict__ queue,
                     double* __restrict__ stat, double* __restrict__ pout, double* __restrict__ rho_out,
                     int* __restrict__ err) {
  __shared__ uint32_t sbuf[wide::WW];
  __shared__ unsigned long long ubuf[wide::WW];
  __shared__ long long s_item;
  const int64_t kw = ldo / 32 + 2;
  uint32_t* K = scratch + blockIdx.x * scr;
  uint32_t* P = K + kw;
  uint32_t* R = P + kw;
  const int64_t total = finish_before(hi, lo, 0, F);
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int64_t t = s_item;
    if (t >= total) break;
    int64_t a = lo, b = hi - 1;  // last row g with before(g) <= t
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (finish_before(mid, lo, 0, F) <= t) a = mid;
      else b = mid - 1;
    }
    const int64_t g = a, h = g + (t - finish_before(g, lo, 0, F));
    const OT* og = order + g * ldo;
    const OT* oh = order + h * ldo;
    const uint32_t* tbg = tb + g * ldt;
    const uint32_t* tbh = tb + h * ldt;
    // pass A: g's order, kept where h is present; R[s] = 2 r_g(s)
    const uint32_t n = wide::keep_scan(og, (uint32_t)len[g], mask + h * W, K, P, sbuf);
    unsigned long long sa = 0, sb = 0, sc = 0;
    if (n > 1) {
      for (uint32_t q = threadIdx.x; q < (uint32_t)len[g]; q += wide::WT) {
        if (!((K[q >> 5] >> (q & 31u)) & 1u)) continue;
        const uint32_t r2 = wide::pfx(K, P, wide::tie_start(tbg, lastb + g * ldt, q)) +
                            wide::pfx(K, P, wide::tie_end(tbg, nextb + g * ldt, q)) + 1u;
        R[(uint32_t)og[q]] = r2;
        sa += (unsigned long long)r2 * r2;
      }
      __syncthreads();
      // pass B: h's order, kept where g is present
      wide::keep_scan(oh, (uint32_t)len[h], mask + g * W, K, P, sbuf);
      for (uint32_t q = threadIdx.x; q < (uint32_t)len[h]; q += wide::WT) {
        if (!((K[q >> 5] >> (q & 31u)) & 1u)) continue;
        const uint32_t r2 = wide::pfx(K, P, wide::tie_start(tbh, lastb + h * ldt, q)) +
                            wide::pfx(K, P, wide::tie_end(tbh, nextb + h * ldt, q)) + 1u;
        sc += (unsigned long long)r2 * r2;
        sb += (unsigned long long)r2 * R[(uint32_t)oh[q]];
      }
      sa = wide::block_sum_u64(sa, ubuf);
      sb = wide::block_sum_u64(sb, ubuf);
      sc = wide::block_sum_u64(sc, ubuf);
    }
    if (threadIdx.x == 0) {
      double rho, p;
      spearman_from_sums((long long)n, sa, sc, (long long)sb, &rho, &p, err);
      put(stat, F, g, h, rho);
      put(pout, F, g, h, p);
      put(rho_out, F, g, h, rho);
    }
    __syncthreads();
  }
}

template <typename OT>
int spearman_wide_launch(ps_matrix* a, const OT* order, const OT* lastb, const OT* nextb, int64_t lo, int64_t hi,
                         double* stat, double* p, double* rho, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  const int grid = ds->num_sms;
  const int64_t scr = 2 * (a->ldo / 32 + 2) + ps_round_up(a->S, 32);
  uint32_t* scratch = nullptr;
  int* queue = nullptr;
  PS_CUDA(ps_alloc(&scratch, (size_t)(grid * scr), s));
  PS_CUDA(ps_alloc(&queue, 1, s));
  PS_CUDA(cudaMemsetAsync(queue, 0, sizeof(int), s));
  ps_prof_begin("spearman_walk", s);
  spearman_wide_kernel<OT><<<grid, wide::WT, 0, s>>>(order, a->ldo, a->d_tb, lastb, nextb, a->ldt, a->d_len, a->d_mask,
                                                     a->W, a->F, lo, hi, scratch, scr, queue, stat, p, rho,
                                                     ps_state()->d_err);
  ps_prof_end(s);
  PS_LAUNCHED();
  ps_free(scratch, s);
  ps_free(queue, s);
  return PS_OK;
}

}  // namespace

using WalkKernel = decltype(&spearman_walk_kernel<true, true>);

struct ps_spearman_job {
  ps_matrix* a = nullptr;
  int64_t lo = 0, hi = 0;
  WalkKernel kern = nullptr;
  size_t smem = 0;
  int cap = 0;         // group-table capacity (0: tie-group records only)
  int grid_max = 1;
  int64_t gb = 32;     // g rows per work item of incremental launches
  int64_t rows = 0;    // g rows per partials chunk
  bool single = false; // one chunk: columns may be walked incrementally
  int64_t h_done = 0;  // columns [lo, h_done) walked (single chunk)
  PairSums ps{};
  PairParts pp{nullptr, nullptr, 0};
  int4* items = nullptr;  // item tables, one region per launch
  int64_t items_cap = 0, items_used = 0;
  int* queues = nullptr;
  int qn = 256, qi = 0;
  double *stat = nullptr, *p = nullptr, *rho = nullptr;  // device outputs
  int64_t h_fin = 0;  // columns [lo, h_fin) folded and finished (incremental)
  cudaStream_t home = nullptr;  // allocation stream (frees are ordered on it)
  int nws = 0;                  // incremental launches so far (alternate walk streams)
};

static void job_free(ps_spearman_job* j, cudaStream_t s) {
  ps_free(j->ps.n, s);
  ps_free(j->ps.sxx4, s);
  ps_free(j->ps.syy4, s);
  ps_free(j->ps.sxy4, s);
  ps_free(j->pp.part, s);
  ps_free(j->pp.meta, s);
  ps_free(j->queues, s);
  ps_free(j->items, s);
  delete j;
}

// One walk launch over columns [h0, h1) and g rows [c0, c1) (partials chunk c0).
static int walk_launch(ps_spearman_job* j, int64_t h0, int64_t h1, int64_t c0, int64_t c1, int64_t gb,
                       cudaStream_t s, int grid_max, int once = 0) {
  int sh = -1;
  for (int b = 0; b < 40; ++b)
    if (((int64_t)1 << b) == gb) sh = b;
  const WalkItems wi{h0, h1, c0, c1, gb, sh};
  const int64_t n = wi.total();
  if (n <= 0) return PS_OK;
  if (j->qi >= j->qn) {
    PS_CUDA(cudaMemsetAsync(j->queues, 0, sizeof(int) * j->qn, s));
    j->qi = 0;
  }
  int* q = j->queues + j->qi++;
  if (j->items_used + n > j->items_cap) return ps_fail(PS_ERR_INVALID, "spearman: item table overflow");
  int4* items = j->items + j->items_used;
  j->items_used += n;
  walk_items_kernel<<<(unsigned)ps_ceil_div(h1 - wi.first(), 128), 128, 0, s>>>(wi, items);
  PS_LAUNCHED();
  ps_matrix* a = j->a;
  PairParts pp = j->pp;
  pp.c0 = c0;
  const int grid = once ? (int)n : (int)std::min<int64_t>(n, grid_max);
  ps_prof_begin("spearman_walk", s);
  j->kern<<<grid, STH, j->smem, s>>>(a->d_order, a->d_inv, a->ldo, a->d_tb, a->d_lastb, a->d_nextb, a->ldt,
                                     a->d_tied, a->d_len, a->d_gp, a->d_bpos, a->d_ngrp, a->d_ordgid, j->cap, a->F,
                                     items,
                                     (int)n, once, q, pp);
  ps_prof_end(s);
  PS_LAUNCHED();
  return PS_OK;
}

static int partials_launch(ps_spearman_job* j, int64_t c0, int64_t c1, cudaStream_t s, int64_t h0 = 0,
                           int64_t h1 = -1) {
  if (h1 < 0) h1 = j->a->F;
  if (h1 <= h0) return PS_OK;
  PairParts pp = j->pp;
  pp.c0 = c0;
  const int pblocks = (int)std::max<int64_t>(
      1, std::min<int64_t>(ps_ceil_div((c1 - c0) * (h1 - h0), 8), (int64_t)ps_state()->num_sms * 32));
  spearman_partials_kernel<<<pblocks, 256, 0, s>>>(pp, j->a->F, c1, j->ps, h0, h1);
  PS_LAUNCHED();
  return PS_OK;
}

// rho / p of the cells of rows [lo, hi) x columns [h0, h1) (rows default: the job's)
static int finish_launch(ps_spearman_job* j, int64_t h0, int64_t h1, cudaStream_t s, int64_t lo = -1,
                         int64_t hi = -1) {
  const int64_t F = j->a->F;
  if (lo < 0) lo = j->lo;
  if (hi < 0) hi = j->hi;
  if (h1 <= h0 || hi <= lo || (!j->stat && !j->p && !j->rho)) return PS_OK;
  ps_device_state* ds = ps_state();
  const int64_t cells = finish_before(hi, lo, h0, h1);
  if (cells <= 0) return PS_OK;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ps_ceil_div(cells, 128), (int64_t)ds->num_sms * 16));
  spearman_finish_kernel<<<blocks, 128, 0, s>>>(j->ps, F, lo, hi, h0, h1, j->stat, j->p, j->rho, ds->d_err);
  PS_LAUNCHED();
  return PS_OK;
}

// after an incremental walk launch of columns [h0, h1) on stream w: those
// cells are complete -- fold and finish them on the same stream
static int fold_finish_columns(ps_spearman_job* j, int64_t h0, int64_t h1, cudaStream_t w) {
  int rc = partials_launch(j, j->lo, j->hi, w, h0, h1);
  if (!rc) rc = finish_launch(j, h0, h1, w);
  if (!rc) j->h_fin = h1;
  return rc;
}

// true when the shared-memory walk streams g's order from global memory
// (does not stage it): such walks read the packed ordgid table
bool ps_spearman_streams_g(int64_t S) {
  if (S > 65535) return false;
  const int64_t ldo = ps_round_up(S + 1, 64), ldt = tie_words(S);
  const size_t limit = 227 * 1024 - 1024;
  const size_t smem = walk_smem(ldo, ldt, true, S <= 32767, 0);
  return !(smem <= limit / 2 || (smem <= limit && S > 12000));
}

// true when the shared-memory walk's tables do not fit for S samples (or the
// presort is 32-bit): such matrices take the wide walk
bool ps_spearman_wide(int64_t S) {
  if (S > 65535) return true;
  const int64_t ldo = ps_round_up(S + 1, 64), ldt = tie_words(S);
  const size_t limit = 227 * 1024 - 1024;
  const bool r2 = S <= 32767;
  return walk_smem(ldo, ldt, false, r2, 0) > limit && walk_smem(ldo, ldt, true, r2, 0) > limit;
}

int ps_spearman_begin(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho, cudaStream_t s,
                      ps_spearman_job** out) {
  *out = nullptr;
  const int64_t F = a->F;
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(F, hi);
  ps_device_state* ds = ps_state();
  const size_t limit = 227 * 1024 - 1024;
  const bool r2 = a->S <= 32767;  // 2r fits 16 bits: no parity bits
  size_t smem = walk_smem(a->ldo, a->ldt, true, r2, 0);
  bool ogs = !ps_spearman_streams_g(a->S);
  if (const char* e = getenv("PS_SPEARMAN_OGS")) ogs = smem <= limit && e[0] == '1';  // tuning override
  if (!ogs) smem = walk_smem(a->ldo, a->ldt, false, r2, 0);
  if (smem > limit) return ps_fail(PS_ERR_INVALID, "spearman: sample count too large for the shared-memory walk");
  // group-table capacity: the largest that keeps the CTAs per SM of the
  // table-less layout (occupancy queried for the kernel this layout runs)
  WalkKernel kern = ogs ? (r2 ? spearman_walk_kernel<true, true> : spearman_walk_kernel<true, false>)
                        : (r2 ? spearman_walk_kernel<false, true> : spearman_walk_kernel<false, false>);
  int cap = 0;
  if (a->d_gp && !getenv("PS_SPEARMAN_NOTAB")) {
    auto occ = [&](size_t sm) {
      int n = 0;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, STH, sm) != cudaSuccess)
        return 0;
      return n;
    };
    const int want = occ(smem);
    for (int c = 2040; c >= 64 && want > 0; c -= 8) {
      const size_t sm = walk_smem(a->ldo, a->ldt, ogs, r2, c);
      if (sm <= limit && occ(sm) >= want) {
        cap = c;
        smem = sm;
        break;
      }
    }
  }
  ps_spearman_job* j = new ps_spearman_job();
  j->a = a;
  j->lo = lo;
  j->hi = hi;
  j->h_done = lo;
  j->h_fin = lo;
  j->stat = stat;
  j->p = p;
  j->rho = rho;
  j->smem = smem;
  j->cap = cap;
  j->kern = kern;
  j->home = s;
  if (const char* e = getenv("PS_SPEARMAN_GB")) j->gb = std::max<int64_t>(1, atoll(e));
  int rc = PS_OK;
  auto fail = [&](cudaError_t e) {
    job_free(j, s);
    return ps_cuda_check(e, "spearman setup");
  };
  cudaError_t e = cudaFuncSetAttribute(j->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, j->kern, STH, smem);
  if (e != cudaSuccess) return fail(e);
  j->grid_max = ds->num_sms * std::max(1, per_sm);
  // g rows per chunk: the per-warp partials take kSlots * SW * 8 B per cell
  const int64_t per_row = F * (int64_t)(kSlots * SW + 1) * 8;
  j->rows = std::max<int64_t>(1, std::min<int64_t>(hi - lo, ((int64_t)2 << 30) / per_row));
  if (const char* e = getenv("PS_SPEARMAN_ROWS")) j->rows = std::max<int64_t>(1, std::min<int64_t>(hi - lo, atoll(e)));
  j->single = j->rows >= hi - lo;
  // pair sums of one chunk of rows (the whole range when it is one chunk)
  const int64_t ps_rows = std::max<int64_t>(1, j->single ? hi - lo : j->rows);
  j->ps.row0 = lo;
  if ((e = ps_alloc(&j->ps.n, (size_t)(ps_rows * F), s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->ps.sxx4, (size_t)(ps_rows * F), s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->ps.syy4, (size_t)(ps_rows * F), s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->ps.sxy4, (size_t)(ps_rows * F), s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->queues, (size_t)j->qn, s)) != cudaSuccess) return fail(e);
  if ((e = cudaMemsetAsync(j->queues, 0, sizeof(int) * j->qn, s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->pp.part, (size_t)(j->rows * F * kSlots * SW), s)) != cudaSuccess) return fail(e);
  if ((e = ps_alloc(&j->pp.meta, (size_t)(j->rows * F), s)) != cudaSuccess) return fail(e);
  // item tables: launches over disjoint column ranges of one chunk hold at
  // most pairs / gb + F items; one item per column per chunk otherwise
  const int64_t npairs = (hi - lo) * F, nchunks = ps_ceil_div(hi - lo, j->rows);
  j->items_cap = nchunks * F + 64;
  if (j->single || getenv("PS_SPEARMAN_GB")) j->items_cap += ps_ceil_div(npairs, j->gb) + F;
  if ((e = ps_alloc(&j->items, (size_t)j->items_cap, s)) != cudaSuccess) return fail(e);
  (void)rc;
  *out = j;
  return PS_OK;
}

// Incremental launches alternate between two walk streams, so a launch can
// fill the SMs while the previous one drains its last items; their work items
// are g blocks of j->gb rows (columns of one upload chunk are too few to fill
// the GPU one column per item).
int ps_spearman_walk_upto(ps_spearman_job* j, int64_t h1, cudaStream_t s) {
  if (!j->single) return PS_OK;
  h1 = std::min<int64_t>(h1, j->a->F);
  if (h1 <= j->h_done) return PS_OK;
  // one item per CTA (not persistent) while rows are still arriving: the
  // per-chunk prep and presort kernels run on a higher-priority stream and
  // take SMs as walk CTAs retire; the last launch is persistent
  cudaStream_t w = ps_walk_stream(j->nws++, s);
  int rc = walk_launch(j, j->h_done, h1, j->lo, j->hi, j->gb, w, j->grid_max, h1 < j->a->F);
  if (!rc) rc = fold_finish_columns(j, j->h_done, h1, w);
  j->h_done = h1;
  return rc;
}

int ps_spearman_end(ps_spearman_job* j, cudaStream_t s) {
  int rc = PS_OK;
  const int64_t F = j->a->F, lo = j->lo, hi = j->hi;
  ps_device_state* ds = ps_state();
  int jr = ps_walk_streams_join(j->nws, s);
  if (jr) return jr;
  // one item per column h (largest first) unless overridden: no per-item
  // reload of h's tables, and the smallest columns form the tail
  int64_t gb_full = F;
  if (getenv("PS_SPEARMAN_GB")) gb_full = j->gb;
  if (j->single) {
    rc = walk_launch(j, j->h_done, F, lo, hi, j->nws ? j->gb : gb_full, s, j->grid_max);
    if (!rc) rc = partials_launch(j, lo, hi, s, j->h_fin, F);
  } else {
    for (int64_t c0 = lo; c0 < hi && !rc; c0 += j->rows) {
      const int64_t c1 = std::min<int64_t>(hi, c0 + j->rows);
      j->ps.row0 = c0;  // the chunk's pair sums reuse one rows x F scratch
      rc = walk_launch(j, c0, F, c0, c1, gb_full, s, j->grid_max);
      if (!rc) rc = partials_launch(j, c0, c1, s);
      if (!rc) rc = finish_launch(j, 0, F, s, c0, c1);
    }
  }
  if (!rc && j->single) rc = finish_launch(j, j->h_fin, F, s);
  if (j->home != s) {  // free in the allocation stream's order (pool reuse across runs)
    PS_CUDA(cudaEventRecord(ds->walk_ev[ps_device_state::kWalkStreams], s));
    PS_CUDA(cudaStreamWaitEvent(j->home, ds->walk_ev[ps_device_state::kWalkStreams], 0));
  }
  job_free(j, j->home);
  return rc;
}

void ps_spearman_abort(ps_spearman_job* j, cudaStream_t s) {
  if (!j) return;
  cudaStreamSynchronize(s);
  cudaDeviceSynchronize();
  job_free(j, j->home);
}

int ps_spearman_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho,
                    cudaStream_t s) {
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(a->F, hi);
  if (hi <= lo || (!stat && !p && !rho)) return PS_OK;
  if (!a->has_presort) {
    int rc = ps_presort_matrix(a, s);
    if (rc) return rc;
  }
  if (ps_spearman_wide(a->S)) {  // beyond the shared-memory walk: one CTA per pair
    if (a->wide)
      return spearman_wide_launch<uint32_t>(a, a->d_order32, a->d_lastb32, a->d_nextb32, lo, hi, stat, p, rho, s);
    return spearman_wide_launch<uint16_t>(a, a->d_order, a->d_lastb, a->d_nextb, lo, hi, stat, p, rho, s);
  }
  // a presort still running in chunks on the auxiliary stream: walk each
  // presorted chunk's columns on the walk streams as it completes
  const bool inc = ps_presort_pending(a);
  ps_device_state* ds = ps_state();
  cudaStream_t home = inc ? ds->walk[0] : s;
  ps_spearman_job* j = nullptr;
  int rc = ps_spearman_begin(a, lo, hi, stat, p, rho, home, &j);
  if (rc) return rc;
  if (inc && j->single) {
    PS_CUDA(cudaEventRecord(ds->alloc_ev, home));
    for (const auto& mk : a->presort_marks) {
      const int64_t h1 = std::min<int64_t>(mk.first, a->F);
      if (h1 <= j->h_done || rc) continue;
      cudaStream_t w = ds->walk[j->nws++ % ps_device_state::kWalkStreams];
      PS_CUDA(cudaStreamWaitEvent(w, mk.second, 0));
      PS_CUDA(cudaStreamWaitEvent(w, ds->alloc_ev, 0));
      rc = walk_launch(j, j->h_done, h1, j->lo, j->hi, j->gb, w, j->grid_max, h1 < a->F);
      if (!rc) rc = fold_finish_columns(j, j->h_done, h1, w);
      j->h_done = h1;
    }
  }
  int rc2 = ps_spearman_end(j, s);
  return rc ? rc : rc2;
}

#ifdef PS_WALK_TIMING
extern "C" int ps_debug_walk_cycles(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_walk_cycles, sizeof(unsigned long long) * 40);
  return 0;
}
#endif
