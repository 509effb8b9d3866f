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

// Per-lane tie-group prefixes inside word w of a walked order: given the
// word's boundary bits T, kept bits kw, the kept prefix Pw = Pfx(32 w) and the
// (warp-uniform) prefixes sp / ep of the groups entering / leaving the word,
// return a = Pfx(start of this lane's group), b = Pfx(end of it).  The
// tie-averaged doubled rank of a kept lane is a + b + 1.  Branch-free.
__device__ __forceinline__ void word_group_pfx(uint32_t T, uint32_t sp, uint32_t ep, uint32_t kw, uint32_t Pw,
                                               uint32_t& a, uint32_t& b) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t le = 0xFFFFFFFFu >> (31u - lane);
  const uint32_t mS = T & le, mE = T & ~le;
  // start bit s = highest set bit of mS; kept lanes below s: kw & (2^s - 1)
  const uint32_t belowS = mS ? (0xFFFFFFFFu >> __clz(mS)) >> 1 : 0u;
  // end bit e = lowest set bit of mE; kept lanes below e: kw & (2^e - 1)
  const uint32_t belowE = (mE & (0u - mE)) - 1u;
  a = mS ? Pw + __popc(kw & belowS) : sp;
  b = mE ? Pw + __popc(kw & belowE) : ep;
}

// Row strides of the tie tables: words per feature, padded to 16 bytes.
__host__ __device__ __forceinline__ int64_t tie_words(int64_t S) { return ((S >> 5) + 2 + 7) & ~int64_t(7); }
