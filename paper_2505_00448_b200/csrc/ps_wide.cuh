// ps_wide.cuh -- building blocks of the "wide" rank walks: sample counts whose
// tables do not fit the shared-memory walks (Spearman S > ~50k, Kruskal-
// Wallis / Mann-Whitney S > 65535; the reference takes any S, ranking.py:30-53).
//
// One CTA per pair.  A walk of one feature's presorted order (positions
// 0..n-1, OT = uint16_t or uint32_t sample ids) keeps the samples its partner
// observes: keep bits K[w] per 32 positions (ballot) and their exclusive
// prefix P[w] (block scan) live in per-CTA global scratch (L1/L2 resident),
// so Pfx(x) = P[x/32] + popc(K[x/32] below x) for any position x <= n.  The
// tie-averaged doubled rank of a kept position p is then
//     2 r(p) = Pfx(start of p's tie group) + Pfx(end of it) + 1
// (SURVEY Appendix C identity) -- an integer, so every sum is exact.
#pragma once
#include <cstdint>
#include "ps_common.cuh"

namespace wide {

constexpr int WT = 1024;           // threads per CTA
constexpr int WW = WT / 32;        // warps

template <typename OT>
__device__ __forceinline__ uint32_t tie_start(const uint32_t* tb, const OT* lastb, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = tb[w] & (0xFFFFFFFFu >> (31u - b));
  return m ? (w << 5) + 31u - __clz(m) : (uint32_t)lastb[w - 1];
}

template <typename OT>
__device__ __forceinline__ uint32_t tie_end(const uint32_t* tb, const OT* nextb, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = b == 31u ? 0u : (tb[w] & (0xFFFFFFFFu << (b + 1u)));
  return m ? (w << 5) + (uint32_t)__ffs(m) - 1u : (uint32_t)nextb[w + 1];
}

__device__ __forceinline__ uint32_t pfx(const uint32_t* K, const uint32_t* P, uint32_t x) {
  const uint32_t w = x >> 5, b = x & 31u;
  return P[w] + __popc(K[w] & ((1u << b) - 1u));
}

// block-wide sum of a 64-bit value (result valid in every thread)
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(PS_FULL, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) buf[warp] = v;
  __syncthreads();
  unsigned long long t = 0;
  for (int w = 0; w < WW; ++w) t += buf[w];
  return t;
}

// Keep bits / prefixes of the walk over ord[0, n) against the partner's
// presence bits pmask (by sample).  K, P hold nw + 1 words (P[nw] = total).
// Returns the kept count.  Ends with a barrier.
template <typename OT>
__device__ uint32_t keep_scan(const OT* __restrict__ ord, uint32_t n, const uint32_t* __restrict__ pmask,
                              uint32_t* __restrict__ K, uint32_t* __restrict__ P, uint32_t* sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = (n + 31) >> 5;
  for (uint32_t w = warp; w < nw; w += WW) {
    const uint32_t p = (w << 5) + lane;
    bool kept = false;
    if (p < n) {
      const uint32_t s = (uint32_t)ord[p];
      kept = (__ldg(pmask + (s >> 5)) >> (s & 31u)) & 1u;
    }
    const uint32_t bits = __ballot_sync(PS_FULL, kept);
    if (lane == 0) K[w] = bits;
  }
  if (threadIdx.x == 0) K[nw] = 0u;
  __syncthreads();
  uint32_t carry = 0;
  for (uint32_t c0 = 0; c0 < nw; c0 += WT) {
    const uint32_t w = c0 + threadIdx.x;
    const uint32_t v = w < nw ? (uint32_t)__popc(K[w]) : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sbuf[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = sbuf[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(PS_FULL, t, o);
        if (lane >= o) t += y;
      }
      sbuf[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t before = warp ? sbuf[warp - 1] : 0u;
    if (w < nw) P[w] = carry + before + x - v;
    carry += sbuf[WW - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) P[nw] = carry;
  __syncthreads();
  return carry;
}

}  // namespace wide
