// ps_ties.cuh -- compact tie-group structure of one presorted feature.
//
// A feature's sorted positions 0..n-1 are cut into tie groups (float '==' runs,
// ranking.py:56-89 / continuous.py:147-159; NaN never ties).  Instead of two
// 32-bit arrays (group start/end per position) the presort stores:
//   tb[w]     boundary bits: bit p set iff a group starts at p (p = 0 and the
//             sentinel p = n are always set)
//   lastb[w]  last boundary position in words 0..w     (prefix max)
//   nextb[w]  first boundary position in words w..end  (suffix min)
// so the [start, end) of the group holding p costs one word + one fallback
// lookup: ~S/4 bytes per feature, small enough to stage in shared memory.
#pragma once
#include <cstdint>

__device__ __forceinline__ uint32_t tie_start(const uint32_t* tb, const uint16_t* lastb, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = tb[w] & (0xFFFFFFFFu >> (31u - b));  // boundaries at bits <= b
  return m ? (w << 5) + 31u - __clz(m) : (uint32_t)lastb[w - 1];
}

__device__ __forceinline__ uint32_t tie_end(const uint32_t* tb, const uint16_t* nextb, uint32_t p) {
  const uint32_t w = p >> 5, b = p & 31u;
  const uint32_t m = b == 31u ? 0u : (tb[w] & (0xFFFFFFFFu << (b + 1u)));  // boundaries above b
  return m ? (w << 5) + (uint32_t)__ffs(m) - 1u : (uint32_t)nextb[w + 1];
}

// Row strides of the tie tables: words per feature, padded to 16 bytes.
__host__ __device__ __forceinline__ int64_t tie_words(int64_t S) { return ((S >> 5) + 2 + 7) & ~int64_t(7); }
