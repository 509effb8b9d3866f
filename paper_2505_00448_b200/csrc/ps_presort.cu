// ps_presort.cu -- per-feature stable sort of the present values.
//
// Replaces _presort_matrix -> _presort_block -> _presort (engine.py:379-400,
// :133-142; ranking.py:30-53: stable mergesort of the present entries).  One
// CTA per feature runs an LSD radix sort over order-preserving 64-bit keys in
// global scratch (8-bit digits, passes whose digit is constant are skipped).
// Keys are canonicalised so that the sort agrees with numpy's: -0.0 and +0.0
// compare equal (and keep sample order), NaN (present under a numeric
// sentinel) sorts after +inf.  Initial order = sample order and every pass is
// stable, so ties keep ascending sample order exactly like the reference.
//
// Outputs per feature f (present count n_f):
//   order[f][p]  sample id of sorted position p (p < n_f)
//   inv[f][s]    sorted position of sample s, 0xFFFF when s is missing
//   gs/ge[f][p]  [start, end) of the tie group of position p, where ties are
//                float '==' runs (ranking.py:56-89): NaN never ties
//   tied[f]      1 if some tie group has more than one member
#include "ps_internal.cuh"
#include "ps_ties.cuh"
#include <algorithm>

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int ITEMS = 4;                 // rounds of 32 per warp per tile
constexpr int TILE = NT * ITEMS;         // 2048 keys per tile
constexpr int PER_WARP = TILE / NW;      // 128 contiguous keys per warp

__device__ __forceinline__ uint64_t sort_key(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v);
  if (v != v) b = 0x7ff8000000000000ull;       // canonical NaN, sorts last
  if ((b << 1) == 0) b = 0;                    // -0.0 ties with +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ bool key_is_nan(uint64_t k) {
  // canonical NaN key: 0x7ff8... | sign flip
  return k == (0x7ff8000000000000ull | 0x8000000000000000ull);
}

// Block-wide exclusive scan of one int per thread; returns the block total.
template <int NWARPS = NW>
__device__ __forceinline__ int block_excl_scan(int v, int* warp_buf, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(PS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_buf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NWARPS ? warp_buf[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(PS_FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NWARPS) warp_buf[lane] = w;  // inclusive
  }
  __syncthreads();
  const int before = warp > 0 ? warp_buf[warp - 1] : 0;
  total = warp_buf[NWARPS - 1];
  __syncthreads();
  return before + x - v;
}

// OT = uint16_t (S <= 65535: 16-bit tables + inverse permutation) or
// uint32_t (wide: S > 65535, no inverse)
template <typename OT>
__global__ void __launch_bounds__(NT)
presort_kernel(const double* __restrict__ vals, int64_t ld, const uint32_t* __restrict__ mask,
               int64_t W, int64_t S, uint64_t* __restrict__ keyA, uint32_t* __restrict__ idxA,
               uint64_t* __restrict__ keyB, uint32_t* __restrict__ idxB, OT* __restrict__ order,
               uint16_t* __restrict__ inv, int64_t ldo, uint32_t* __restrict__ tb,
               OT* __restrict__ lastb, OT* __restrict__ nextb, int64_t ldt,
               uint8_t* __restrict__ tied, int32_t* __restrict__ lens, int64_t f0) {
  __shared__ int warp_buf[NW];
  __shared__ uint32_t hist[8][256];
  __shared__ uint32_t wcnt[NW][256];
  __shared__ uint32_t bucket[256];
  __shared__ int s_any_tie;
  const int64_t f = f0 + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* row = vals + f * ld;
  const uint32_t* mrow = mask + f * W;
  uint64_t* kA = keyA + f * S;
  uint32_t* iA = idxA + f * S;
  uint64_t* kB = keyB + f * S;
  uint32_t* iB = idxB + f * S;

  for (int i = threadIdx.x; i < 8 * 256; i += NT) (&hist[0][0])[i] = 0;
  if (threadIdx.x == 0) s_any_tie = 0;
  __syncthreads();

  // 1. stable compaction of the present entries (sample order) + digit histograms
  int n = 0;
  for (int64_t base = 0; base < S; base += NT) {
    const int64_t s = base + threadIdx.x;
    const bool pres = s < S && ((mrow[s >> 5] >> (s & 31)) & 1u);
    int tot;
    const int pos = block_excl_scan(pres ? 1 : 0, warp_buf, tot);
    if (pres) {
      const uint64_t k = sort_key(row[s]);
      kA[n + pos] = k;
      iA[n + pos] = (uint32_t)s;
#pragma unroll
      for (int d = 0; d < 8; ++d) atomicAdd(&hist[d][(k >> (8 * d)) & 0xff], 1u);
    }
    n += tot;
  }
  __syncthreads();

  // 2. LSD passes (stable), skipping constant digits
  for (int d = 0; d < 8; ++d) {
    bool trivial = false;
    for (int b = 0; b < 256; ++b)
      if (hist[d][b] == (uint32_t)n) trivial = true;
    if (trivial || n <= 1) continue;
    const int shift = 8 * d;
    // bucket starts: exclusive scan of hist[d] by warp 0
    if (warp == 0) {
      uint32_t run = 0;
      for (int b0 = 0; b0 < 256; b0 += 32) {
        uint32_t v = hist[d][b0 + lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
          if (lane >= o) x += y;
        }
        bucket[b0 + lane] = run + x - v;
        run += __shfl_sync(PS_FULL, x, 31);
      }
    }
    __syncthreads();
    for (int t0 = 0; t0 < n; t0 += TILE) {
      for (int i = threadIdx.x; i < NW * 256; i += NT) (&wcnt[0][0])[i] = 0;
      __syncthreads();
      const int w0 = t0 + warp * PER_WARP;
      for (int r = 0; r < PER_WARP; r += 32) {
        const int i = w0 + r + lane;
        const bool ok = i < n;
        const uint32_t dg = ok ? (uint32_t)((kA[i] >> shift) & 0xff) : 0u;
        const uint32_t peers = __match_any_sync(PS_FULL, ok ? dg : 0xffffffffu);
        if (ok && (peers & lanemask_lt()) == 0) wcnt[warp][dg] += __popc(peers);
      }
      __syncthreads();
      if (threadIdx.x < 256) {
        const int b = threadIdx.x;
        uint32_t run = bucket[b];
        for (int w = 0; w < NW; ++w) {
          const uint32_t c = wcnt[w][b];
          wcnt[w][b] = run;
          run += c;
        }
        bucket[b] = run;
      }
      __syncthreads();
      for (int r = 0; r < PER_WARP; r += 32) {
        const int i = w0 + r + lane;
        const bool ok = i < n;
        uint64_t k = 0;
        uint32_t v = 0, dg = 0;
        if (ok) {
          k = kA[i];
          v = iA[i];
          dg = (uint32_t)((k >> shift) & 0xff);
        }
        const uint32_t peers = __match_any_sync(PS_FULL, ok ? dg : 0xffffffffu);
        uint32_t start = ok ? wcnt[warp][dg] : 0u;
        __syncwarp();
        if (ok) {
          const uint32_t pos = start + __popc(peers & lanemask_lt());
          kB[pos] = k;
          iB[pos] = v;
          if ((peers >> lane) == 1u) wcnt[warp][dg] = start + __popc(peers);
        }
        __syncwarp();
      }
      __syncthreads();
    }
    // swap A <-> B
    uint64_t* tk = kA; kA = kB; kB = tk;
    uint32_t* ti = iA; iA = iB; iB = ti;
    __syncthreads();
  }

  // 3. outputs: order, inverse permutation, tie-group boundary tables
  OT* ord = order + f * ldo;
  uint16_t* iv = inv ? inv + f * ldo : nullptr;
  // positions past n hold the sentinel sample id S, whose inverse is 0xFFFF
  // (absent), so walks over whole 32-position words need no bounds checks
  if (iv)
    for (int64_t s = threadIdx.x; s < ldo; s += NT) iv[s] = 0xFFFF;
  __syncthreads();
  for (int64_t p = threadIdx.x; p < ldo; p += NT) {
    if (p < n) {
      const uint32_t s = iA[p];
      ord[p] = (OT)s;
      if (iv) iv[s] = (uint16_t)p;
    } else {
      ord[p] = (OT)S;
    }
  }
  uint32_t* tbr = tb + f * ldt;
  OT* lbr = lastb + f * ldt;
  OT* nbr = nextb + f * ldt;
  const int nw = (int)ldt;
  for (int w = warp; w < nw; w += NW) {
    const int p = w * 32 + lane;
    bool bnd = false;
    if (p < n) {
      bnd = p == 0 || kA[p] != kA[p - 1] || key_is_nan(kA[p]);
      if (!bnd) s_any_tie = 1;
    } else {
      bnd = p == n;  // sentinel boundary closes the last group
    }
    const uint32_t word = __ballot_sync(PS_FULL, bnd);
    if (lane == 0) tbr[w] = word;
  }
  __syncthreads();
  if (warp == 0) {  // lastb: inclusive prefix max of the last boundary per word
    int carry = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int w = w0 + lane;
      const uint32_t word = w < nw ? tbr[w] : 0u;
      int x = word ? w * 32 + 31 - __clz(word) : -1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(PS_FULL, x, o);
        if (lane >= o) x = max(x, y);
      }
      x = max(x, carry);
      if (w < nw) lbr[w] = (OT)x;
      carry = __shfl_sync(PS_FULL, x, 31);
    }
  } else if (warp == 1) {  // nextb: inclusive suffix min of the first boundary per word
    const int none = sizeof(OT) == 2 ? 0xFFFF : 0x7FFFFFFF;
    int carry = none;
    const int last0 = ((nw - 1) / 32) * 32;
    for (int w0 = last0; w0 >= 0; w0 -= 32) {
      const int w = w0 + lane;
      const uint32_t word = w < nw ? tbr[w] : 0u;
      int x = word ? w * 32 + __ffs(word) - 1 : none;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(PS_FULL, x, o);
        if (lane + o < 32) x = min(x, y);
      }
      x = min(x, carry);
      if (w < nw) nbr[w] = (OT)x;
      carry = __shfl_sync(PS_FULL, x, 0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tied[f] = s_any_tie ? 1 : 0;
    lens[f] = n;
  }
}

// ---------------------------------------------------------------------------
// Shared-memory presort (S <= 20480): one CTA per feature holds its keys in
// registers (warp-striped: warp w, item i, lane l <-> position
// w*32*ITEMS + i*32 + l, so (i, lane) order IS sequence order) and runs a
// stable LSD radix sort whose scatter goes through one shared exchange buffer
// (10 B per element).  Digit passes whose byte is constant are skipped (AND ==
// OR over all keys).  Global traffic: values + mask in, order/inv/tie tables
// out -- no per-pass HBM round trips.
// ---------------------------------------------------------------------------
constexpr int QT = 1024;
constexpr int QW = QT / 32;

template <int ITEMS>
__global__ void __launch_bounds__(QT, 1)
presort_smem_kernel(const double* __restrict__ vals, int64_t ld, const uint32_t* __restrict__ mask, int64_t W,
                    int64_t S, uint16_t* __restrict__ order, uint16_t* __restrict__ inv, int64_t ldo,
                    uint32_t* __restrict__ tb, uint16_t* __restrict__ lastb, uint16_t* __restrict__ nextb,
                    int64_t ldt, uint8_t* __restrict__ tied, int32_t* __restrict__ lens, int64_t f0) {
  constexpr int NMAX = QT * ITEMS;
  extern __shared__ __align__(16) unsigned char qsm[];
  uint32_t* sk32 = reinterpret_cast<uint32_t*>(qsm);  // 32-bit pass keys (high halves once sorted)
  uint16_t* sinv = reinterpret_cast<uint16_t*>(qsm);  // inverse permutation, staged at the end
  uint16_t* sidx = reinterpret_cast<uint16_t*>(qsm + (size_t)NMAX * 8);
  __shared__ uint16_t wcnt[QW][256];
  __shared__ int warp_buf[QW];
  __shared__ unsigned long long s_and, s_or;
  __shared__ int s_any_tie, s_long;
  const int64_t f = f0 + blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* row = vals + f * ld;
  const uint32_t* mrow = mask + f * W;
  auto key_of = [&](uint32_t sid) -> uint64_t { return sort_key(row[sid]); };

  // 1. stable compaction of present sample ids: warp w owns samples
  //    [w*32*ITEMS, (w+1)*32*ITEMS) in (item, lane) order (coalesced loads);
  //    one block scan of the warp counts places them.  AND / OR over the
  //    present keys decide which radix bytes are constant.
  if (threadIdx.x == 0) {
    s_and = ~0ull;
    s_or = 0ull;
    s_any_tie = 0;
    s_long = 0;
  }
  int n;
  {
    const int64_t s0 = (int64_t)warp * 32 * ITEMS;
    uint32_t bal[ITEMS];
    int wcount = 0;
    unsigned long long a = ~0ull, o = 0ull;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t sp = s0 + i * 32 + lane;
      const bool pres = sp < S && ((mrow[sp >> 5] >> (sp & 31)) & 1u);
      bal[i] = __ballot_sync(PS_FULL, pres);
      wcount += __popc(bal[i]);
      if (pres) {
        const uint64_t k = key_of((uint32_t)sp);
        a &= k;
        o |= k;
      }
    }
    // exclusive scan of the warp counts (lane 0 of each warp holds one)
    if (lane == 0) warp_buf[warp] = wcount;
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < QW; ++w) {
      const int c = warp_buf[w];
      before += w < warp ? c : 0;
      tot += c;
    }
    n = tot;
    int run = before;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if ((bal[i] >> lane) & 1u) sidx[run + __popc(bal[i] & lanemask_lt())] = (uint16_t)(s0 + i * 32 + lane);
      run += __popc(bal[i]);
    }
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
      a &= __shfl_xor_sync(PS_FULL, a, sft);
      o |= __shfl_xor_sync(PS_FULL, o, sft);
    }
    if (lane == 0) {
      atomicAnd(&s_and, a);
      atomicOr(&s_or, o);
    }
  }
  __syncthreads();
  const unsigned long long diff = s_and ^ s_or;

  // 2. Stable LSD radix sort on 32-bit halves of the key, registers
  //    warp-striped (warp w, item i, lane l <-> position w*32*ITEMS + i*32 + l,
  //    so (i, lane) order IS sequence order).  Round 0 sorts on the HIGH half
  //    only (sign, exponent, top mantissa bits); the rare runs whose high
  //    halves collide but whose full keys differ are then repaired by an
  //    insertion sort on the low halves.  A feature with a long colliding run
  //    is re-sorted on both halves (round 1: low half, then high half).  The
  //    32-bit pass keys are re-derived from the values through the sample id
  //    (one gather per stage), so only 6 B per element move per pass.
  uint32_t k32[ITEMS], idx[ITEMS];  // idx: sample id | in-warp offset << 16
  for (int round = 0, st0 = 1; round < 2; ++round, st0 = 0) {
    for (int st = st0; st < 2; ++st) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int p = warp * 32 * ITEMS + i * 32 + lane;
        idx[i] = p < n ? sidx[p] : 0xFFFFu;
        const uint64_t k = p < n ? key_of(idx[i]) : ~0ull;  // padding sorts last
        k32[i] = st ? (uint32_t)(k >> 32) : (uint32_t)k;
      }
      __syncthreads();
      for (int b = 0; b < 4; ++b) {
        const int shift = 8 * b;
        if (((diff >> (32 * st + shift)) & 0xffull) == 0 || n <= 1) continue;
        for (int i = threadIdx.x; i < QW * 256; i += QT) (&wcnt[0][0])[i] = 0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const uint32_t dg = (k32[i] >> shift) & 0xffu;
          const uint32_t peers = __match_any_sync(PS_FULL, dg);
          const uint32_t base = wcnt[warp][dg];
          __syncwarp();
          idx[i] = (idx[i] & 0xFFFFu) | ((base + __popc(peers & lanemask_lt())) << 16);
          if ((peers >> lane) == 1u) wcnt[warp][dg] = (uint16_t)(base + __popc(peers));
          __syncwarp();
        }
        __syncthreads();
        // digit totals -> bucket starts -> per-warp starts (digit-major, warp order)
        if (threadIdx.x < 256) {
          uint32_t tot = 0;
          for (int w = 0; w < QW; ++w) tot += wcnt[w][threadIdx.x];
          // exclusive scan of totals across the 256 digits (8 warps)
          uint32_t x = tot;
#pragma unroll
          for (int sft = 1; sft < 32; sft <<= 1) {
            const uint32_t y = __shfl_up_sync(PS_FULL, x, sft);
            if (lane >= sft) x += y;
          }
          if (lane == 31) warp_buf[warp] = (int)x;
          // (warps 0..7 participate; others skip)
          asm volatile("bar.sync 1, 256;");
          uint32_t before = 0;
          for (int w = 0; w < warp; ++w) before += (uint32_t)warp_buf[w];
          uint32_t run = before + x - tot;
          for (int w = 0; w < QW; ++w) {
            const uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = (uint16_t)run;  // start offsets (fit: < 2^16)
            run += c;
          }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const uint32_t dg = (k32[i] >> shift) & 0xffu;
          const uint32_t dst = (uint32_t)wcnt[warp][dg] + (idx[i] >> 16);
          sk32[dst] = k32[i];
          sidx[dst] = (uint16_t)idx[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int p = warp * 32 * ITEMS + i * 32 + lane;
          k32[i] = sk32[p];
          idx[i] = sidx[p];
        }
        __syncthreads();
      }
    }
    // sk32 must hold the HIGH halves in sorted order: the last high-half pass
    // scattered them; if none ran, the high halves are all equal (s_and's)
    if ((diff >> 32) == 0 || n <= 1) {
      for (int p = threadIdx.x; p < n; p += QT) sk32[p] = (uint32_t)(s_and >> 32);
      __syncthreads();
    }
    if (round == 1 || (uint32_t)diff == 0u) break;  // low halves all equal: sorted
    // repair runs of equal high halves whose full keys differ: sort the run by
    // its low halves (stable), staged in sk32 and restored afterwards
    for (int p = threadIdx.x; p < n; p += QT) {
      const uint32_t h = sk32[p];
      if (p > 0 && sk32[p - 1] == h) continue;  // not a run start
      int e = p + 1;
      while (e < n && sk32[e] == h) ++e;
      if (e - p == 1) continue;
      const uint32_t l0 = (uint32_t)key_of(sidx[p]);
      bool mixed = false;
      for (int q = p + 1; q < e && !mixed; ++q) mixed = (uint32_t)key_of(sidx[q]) != l0;
      if (!mixed) continue;
      if (e - p > 64) {
        s_long = 1;
        continue;
      }
      // stable insertion sort of [p, e) by the low half, in thread-local
      // storage (sk32 stays intact: other threads read it to find run starts)
      uint32_t lo[64];
      uint16_t id[64];
      const int m = e - p;
      for (int q = 0; q < m; ++q) {
        id[q] = sidx[p + q];
        lo[q] = (uint32_t)key_of(id[q]);
      }
      for (int i = 1; i < m; ++i) {
        const uint32_t ki = lo[i];
        const uint16_t xi = id[i];
        int j = i - 1;
        while (j >= 0 && lo[j] > ki) {
          lo[j + 1] = lo[j];
          id[j + 1] = id[j];
          --j;
        }
        lo[j + 1] = ki;
        id[j + 1] = xi;
      }
      for (int q = 0; q < m; ++q) sidx[p + q] = id[q];
    }
    __syncthreads();
    if (!s_long) break;
  }

  // 3. outputs: order, tie-group boundaries (full-key equality: high halves
  //    from smem, low halves fetched only where the high halves agree)
  uint16_t* ord = order + f * ldo;
  for (int p = threadIdx.x; p < (int)ldo; p += QT) ord[p] = p < n ? sidx[p] : (uint16_t)S;
  uint32_t* tbr = tb + f * ldt;
  uint16_t* lbr = lastb + f * ldt;
  uint16_t* nbr = nextb + f * ldt;
  const int nw = (int)ldt;
  for (int w = warp; w < nw; w += QW) {
    const int p = w * 32 + lane;
    bool bnd;
    if (p < n) {
      const uint32_t h = sk32[p];
      bnd = p == 0 || h != sk32[p - 1] || h == 0xFFF80000u;  // (canonical NaN: never ties)
      if (!bnd) bnd = (uint32_t)key_of(sidx[p]) != (uint32_t)key_of(sidx[p - 1]);  // high halves agree
      if (!bnd) s_any_tie = 1;
    } else {
      bnd = p == n;
    }
    const uint32_t word = __ballot_sync(PS_FULL, bnd);
    if (lane == 0) tbr[w] = word;
  }
  __syncthreads();
  // inverse permutation staged in smem (over the no longer needed keys), then
  // written out coalesced
  for (int64_t s = threadIdx.x; s < ldo; s += QT) sinv[s] = 0xFFFF;
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += QT) sinv[sidx[p]] = (uint16_t)p;
  __syncthreads();
  uint16_t* iv = inv + f * ldo;
  for (int64_t s = threadIdx.x; s < ldo; s += QT) iv[s] = sinv[s];
  if (warp == 0) {
    int carry = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int w = w0 + lane;
      const uint32_t word = w < nw ? tbr[w] : 0u;
      int x = word ? w * 32 + 31 - __clz(word) : -1;
#pragma unroll
      for (int sft = 1; sft < 32; sft <<= 1) {
        const int y = __shfl_up_sync(PS_FULL, x, sft);
        if (lane >= sft) x = max(x, y);
      }
      x = max(x, carry);
      if (w < nw) lbr[w] = (uint16_t)x;
      carry = __shfl_sync(PS_FULL, x, 31);
    }
  } else if (warp == 1) {
    int carry = 0xFFFF;
    const int last0 = ((nw - 1) / 32) * 32;
    for (int w0 = last0; w0 >= 0; w0 -= 32) {
      const int w = w0 + lane;
      const uint32_t word = w < nw ? tbr[w] : 0u;
      int x = word ? w * 32 + __ffs(word) - 1 : 0xFFFF;
#pragma unroll
      for (int sft = 1; sft < 32; sft <<= 1) {
        const int y = __shfl_down_sync(PS_FULL, x, sft);
        if (lane + sft < 32) x = min(x, y);
      }
      x = min(x, carry);
      if (w < nw) nbr[w] = (uint16_t)x;
      carry = __shfl_sync(PS_FULL, x, 0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tied[f] = s_any_tie ? 1 : 0;
    lens[f] = n;
  }
}

// Tie-group index of one feature (16-bit tables): gp[w] = number of group
// starts at positions < 32 w, bpos[k] = start of group k (k < D), bpos[D] = n,
// ngrp = D.  Derived from the boundary bits alone (bit n is the end sentinel),
// so it is identical for owned and caller-owned (gathered) tables.
__global__ void tie_index_kernel(const uint32_t* __restrict__ tb, int64_t ldt, const int32_t* __restrict__ lens,
                                 const uint8_t* __restrict__ tied, uint16_t* __restrict__ gp,
                                 uint16_t* __restrict__ bpos, int64_t ldo, int32_t* __restrict__ ngrp,
                                 const uint16_t* __restrict__ order, uint32_t* __restrict__ ordgid, int64_t f0) {
  const int64_t f = f0 + blockIdx.x;
  const int n = lens[f];
  if (!tied[f]) {  // every position its own group: the walks never read the index of a tie-free feature
    if (threadIdx.x == 0) ngrp[f] = n;
    return;
  }
  const int nw = (n + 31) >> 5;  // words holding positions < n
  const uint32_t* t = tb + f * ldt;
  uint16_t* g = gp + f * ldt;
  uint16_t* bp = bpos + f * ldo;
  __shared__ int wsum[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int w0 = 0; w0 < nw; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    uint32_t T = 0u;
    if (w < nw) {
      T = t[w];
      const int rem = n - 32 * w;  // positions of this word below n
      if (rem < 32) T &= (1u << rem) - 1u;
    }
    const int c = __popc(T);
    int x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(PS_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before = carry;
    for (int i = 0; i < warp; ++i) before += wsum[i];
    int tot = carry;
    for (int i = 0; i < nwarp; ++i) tot += wsum[i];
    const int ex = before + x - c;
    if (w < nw) {
      g[w] = (uint16_t)ex;
      int k = ex;
      for (uint32_t m = T; m; m &= m - 1u) bp[k++] = (uint16_t)(32 * w + __ffs(m) - 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bp[carry] = (uint16_t)n;
    ngrp[f] = carry;
  }
  if (ordgid) {  // whole words: positions past n keep their sentinel id (group id unused)
    __syncthreads();
    const uint16_t* o = order + f * ldo;
    uint32_t* og = ordgid + f * ldo;
    for (int p = threadIdx.x; p < nw * 32; p += blockDim.x) {
      const int w = p >> 5;
      const uint32_t T = t[w] & (0xFFFFFFFFu >> (31 - (p & 31)));
      const uint32_t gid = (uint32_t)g[w] + __popc(T) - 1u;
      og[p] = (uint32_t)o[p] | (gid << 16);
    }
  }
}

}  // namespace

// Presort in three steps so the per-feature sorts can follow the input
// upload chunk by chunk (ps_matrix_create overlaps them with the H2D copy).
static int presort_scratch(ps_matrix* m, cudaStream_t s);

int ps_presort_begin(ps_matrix* m, cudaStream_t s) {
  m->ldo = ps_round_up(m->S + 1, 64);  // room for the sentinel sample id S
  m->ldt = tie_words(m->S);
  if (m->S > 65535) {  // wide: 32-bit orders and tie prefix tables
    m->wide = true;
    PS_CUDA(ps_alloc(&m->d_order32, (size_t)(m->F * m->ldo), s));
    PS_CUDA(ps_alloc(&m->d_tb, (size_t)(m->F * m->ldt), s));
    PS_CUDA(ps_alloc(&m->d_lastb32, (size_t)(m->F * m->ldt), s));
    PS_CUDA(ps_alloc(&m->d_nextb32, (size_t)(m->F * m->ldt), s));
    PS_CUDA(ps_alloc(&m->d_tied, (size_t)m->F, s));
    PS_CUDA(ps_alloc(&m->d_len, (size_t)m->F, s));
    return presort_scratch(m, s);
  }
  PS_CUDA(ps_alloc(&m->d_order, (size_t)(m->F * m->ldo), s));
  PS_CUDA(ps_alloc(&m->d_inv, (size_t)(m->F * m->ldo), s));
  PS_CUDA(ps_alloc(&m->d_gp, (size_t)(m->F * m->ldt), s));
  PS_CUDA(ps_alloc(&m->d_bpos, (size_t)(m->F * m->ldo), s));
  PS_CUDA(ps_alloc(&m->d_ngrp, (size_t)m->F, s));
  if (ps_spearman_streams_g(m->S)) PS_CUDA(ps_alloc(&m->d_ordgid, (size_t)(m->F * m->ldo), s));
  PS_CUDA(ps_alloc(&m->d_tb, (size_t)(m->F * m->ldt), s));
  PS_CUDA(ps_alloc(&m->d_lastb, (size_t)(m->F * m->ldt), s));
  PS_CUDA(ps_alloc(&m->d_nextb, (size_t)(m->F * m->ldt), s));
  PS_CUDA(ps_alloc(&m->d_tied, (size_t)m->F, s));
  PS_CUDA(ps_alloc(&m->d_len, (size_t)m->F, s));
  return presort_scratch(m, s);
}

// Caller-owned tables (multi-GPU: every rank presorts its own rows into them,
// then the ranks all-gather the rows; rows are independent).
int ps_presort_attach(ps_matrix* m, uint16_t* order, uint16_t* inv, uint32_t* tb, uint16_t* lastb, uint16_t* nextb,
                      uint8_t* tied, int32_t* len, cudaStream_t s) {
  if (m->S > 65535)
    return ps_fail(PS_ERR_INVALID, "caller-owned (sharded) presort tables hold 16-bit orders: samples <= 65535");
  m->ldo = ps_round_up(m->S + 1, 64);
  m->ldt = tie_words(m->S);
  m->d_order = order;
  m->d_inv = inv;
  m->d_tb = tb;
  m->d_lastb = lastb;
  m->d_nextb = nextb;
  m->d_tied = tied;
  m->d_len = len;
  m->owns_presort = false;
  PS_CUDA(ps_alloc(&m->d_gp, (size_t)(m->F * m->ldt), s));
  PS_CUDA(ps_alloc(&m->d_bpos, (size_t)(m->F * m->ldo), s));
  PS_CUDA(ps_alloc(&m->d_ngrp, (size_t)m->F, s));
  if (ps_spearman_streams_g(m->S)) PS_CUDA(ps_alloc(&m->d_ordgid, (size_t)(m->F * m->ldo), s));
  return presort_scratch(m, s);
}

static int presort_scratch(ps_matrix* m, cudaStream_t s) {
  if (ps_ceil_div(m->S, QT) > 20) {  // global-memory radix path: per-feature scratch
    const int64_t FS = m->F * m->S;
    uint64_t *kA = nullptr, *kB = nullptr;
    uint32_t *iA = nullptr, *iB = nullptr;
    PS_CUDA(ps_alloc(&kA, (size_t)FS, s));
    PS_CUDA(ps_alloc(&kB, (size_t)FS, s));
    PS_CUDA(ps_alloc(&iA, (size_t)FS, s));
    PS_CUDA(ps_alloc(&iB, (size_t)FS, s));
    m->presort_scratch[0] = kA;
    m->presort_scratch[1] = kB;
    m->presort_scratch[2] = iA;
    m->presort_scratch[3] = iB;
  }
  return PS_OK;
}

int ps_presort_rows(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s) {
  const int64_t nf = f1 - f0;
  if (nf <= 0) return PS_OK;
  const int items = (int)ps_ceil_div(m->S, QT);
  auto smem_path = [&](auto kern, int it) -> int {
    const size_t smem = (size_t)QT * it * 10;
    PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nf, QT, smem, s>>>(m->d_vals, m->ld, m->d_mask, m->W, m->S, m->d_order, m->d_inv, m->ldo,
                                        m->d_tb, m->d_lastb, m->d_nextb, m->ldt, m->d_tied, m->d_len, f0);
    PS_LAUNCHED();
    return PS_OK;
  };
  if (m->wide) {
    presort_kernel<uint32_t><<<(unsigned)nf, NT, 0, s>>>(
        m->d_vals, m->ld, m->d_mask, m->W, m->S, static_cast<uint64_t*>(m->presort_scratch[0]),
        static_cast<uint32_t*>(m->presort_scratch[2]), static_cast<uint64_t*>(m->presort_scratch[1]),
        static_cast<uint32_t*>(m->presort_scratch[3]), m->d_order32, nullptr, m->ldo, m->d_tb, m->d_lastb32,
        m->d_nextb32, m->ldt, m->d_tied, m->d_len, f0);
    PS_LAUNCHED();
    return PS_OK;
  }
  int rc;
  if (items <= 4) rc = smem_path(presort_smem_kernel<4>, 4);
  else if (items <= 8) rc = smem_path(presort_smem_kernel<8>, 8);
  else if (items <= 12) rc = smem_path(presort_smem_kernel<12>, 12);
  else if (items <= 16) rc = smem_path(presort_smem_kernel<16>, 16);
  else if (items <= 20) rc = smem_path(presort_smem_kernel<20>, 20);
  else {
    presort_kernel<uint16_t><<<(unsigned)nf, NT, 0, s>>>(
        m->d_vals, m->ld, m->d_mask, m->W, m->S, static_cast<uint64_t*>(m->presort_scratch[0]),
        static_cast<uint32_t*>(m->presort_scratch[2]), static_cast<uint64_t*>(m->presort_scratch[1]),
        static_cast<uint32_t*>(m->presort_scratch[3]), m->d_order, m->d_inv, m->ldo, m->d_tb, m->d_lastb,
        m->d_nextb, m->ldt, m->d_tied, m->d_len, f0);
    PS_LAUNCHED();
    rc = PS_OK;
  }
  // caller-owned tables hold other ranks' rows only after the gather: their
  // index is built by ps_presort_end over all rows
  if (!rc && m->owns_presort) rc = ps_tie_index(m, f0, f1, s);
  return rc;
}

int ps_tie_index(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s) {
  if (f1 <= f0 || !m->d_gp) return PS_OK;
  tie_index_kernel<<<(unsigned)(f1 - f0), 256, 0, s>>>(m->d_tb, m->ldt, m->d_len, m->d_tied, m->d_gp, m->d_bpos,
                                                      m->ldo, m->d_ngrp, m->d_order, m->d_ordgid, f0);
  PS_LAUNCHED();
  return PS_OK;
}

int ps_presort_end(ps_matrix* m, cudaStream_t s) {
  if (!m->owns_presort && !m->wide) {
    const int rc = ps_tie_index(m, 0, m->F, s);
    if (rc) return rc;
  }
  for (void*& p : m->presort_scratch) {
    ps_free(p, s);
    p = nullptr;
  }
  m->has_presort = true;
  return PS_OK;
}

int ps_presort_matrix(ps_matrix* m, cudaStream_t s) {
  if (m->has_presort) return PS_OK;
  int rc = ps_presort_begin(m, s);
  if (!rc) rc = ps_presort_rows(m, 0, m->F, s);
  if (!rc) rc = ps_presort_end(m, s);
  return rc;
}
