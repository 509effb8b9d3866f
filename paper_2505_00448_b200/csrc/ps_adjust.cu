// ps_adjust.cu -- multiple-testing adjustment on the device.
//
// Replaces adjust.py:23-87.  The family (strict upper triangle for symmetric
// matrices, every cell otherwise) is compacted to its defined (non-NaN)
// p-values, sorted ascending by an LSD radix sort over order-preserving 64-bit
// keys, scaled by fl(scale / i) exactly as numpy's `values[order] * (scale /
// arange(1, m+1))`, reverse-cumulative-minimised, clipped at 1 and scattered
// back (mirrored, NaN diagonal).  Tied p-values receive identical adjusted
// values whatever their order, so an unstable compaction and the radix sort's
// tie order cannot change a bit of the result (adjust is bit-exact given the
// same p matrix).  Bonferroni is min(1, m p).
//
// HBM-bound: each non-trivial radix pass streams 8 B key + 4 B index in and
// out; passes whose digit is constant across the family are skipped.
#include "ps_internal.cuh"
#include <math_constants.h>
#include <algorithm>
#include <vector>

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;  // per thread per tile
constexpr int kTile = kSortThreads * kSortItems;
constexpr int kRadixBits = 8;
constexpr int kBuckets = 1 << kRadixBits;

__device__ __forceinline__ uint64_t key_of(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double val_of(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Compact the defined members of the family into (key, flat index).
__global__ void extract_kernel(const double* __restrict__ p, int64_t rows, int64_t cols,
                               int symmetric, uint64_t* __restrict__ keys,
                               uint32_t* __restrict__ idx, unsigned long long* __restrict__ count) {
  const int64_t n = rows * cols;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool take = false;
    double v = 0.0;
    if (i < n) {
      const int64_t r = i / cols, c = i - r * cols;
      if (!symmetric || c > r) {
        v = p[i];
        take = !(v != v);
      }
    }
    const uint32_t ball = __ballot_sync(PS_FULL, take);
    unsigned long long off = 0;
    if ((threadIdx.x & 31) == 0 && ball) off = atomicAdd(count, (unsigned long long)__popc(ball));
    off = __shfl_sync(PS_FULL, off, 0);
    if (take) {
      const uint64_t pos = off + __popc(ball & lanemask_lt());
      keys[pos] = key_of(v);
      idx[pos] = (uint32_t)i;
    }
  }
}

__global__ void extract_vec_kernel(const double* __restrict__ p, int64_t n, uint64_t* __restrict__ keys,
                                   uint32_t* __restrict__ idx, unsigned long long* __restrict__ count) {
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    double v = i < n ? p[i] : PS_NAN;
    const bool take = !(v != v);
    const uint32_t ball = __ballot_sync(PS_FULL, take);
    unsigned long long off = 0;
    if ((threadIdx.x & 31) == 0 && ball) off = atomicAdd(count, (unsigned long long)__popc(ball));
    off = __shfl_sync(PS_FULL, off, 0);
    if (take) {
      const uint64_t pos = off + __popc(ball & lanemask_lt());
      keys[pos] = key_of(v);
      idx[pos] = (uint32_t)i;
    }
  }
}

// All eight digit histograms in one read of the keys (for pass skipping).
__global__ void digit_hist_all_kernel(const uint64_t* __restrict__ keys, const unsigned long long* count_ptr,
                                      unsigned long long* __restrict__ hist /* 8 x 256 */) {
  __shared__ unsigned int h[8][kBuckets];
  for (int i = threadIdx.x; i < 8 * kBuckets; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t m = (int64_t)*count_ptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int d = 0; d < 8; ++d) atomicAdd(&h[d][(k >> (8 * d)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * kBuckets; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&hist[i], (unsigned long long)(&h[0][0])[i]);
}

// Per-tile digit counts for one pass: tile_hist[digit * ntiles + tile].
__global__ void __launch_bounds__(kSortThreads)
tile_hist_kernel(const uint64_t* __restrict__ keys, int64_t m, int shift, uint32_t* __restrict__ tile_hist,
                 int64_t ntiles) {
  __shared__ uint32_t h[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t t0 = blockIdx.x * (int64_t)kTile;
  for (int q = 0; q < kSortItems; ++q) {
    const int64_t i = t0 + (int64_t)q * kSortThreads + threadIdx.x;
    if (i < m) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kBuckets; d += blockDim.x) tile_hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// Exclusive scan of a uint32 array (digit-major tile histograms) in place,
// three-level: per-block scans, then a scan of block sums, then fix-up.
__global__ void scan_block_kernel(uint32_t* __restrict__ a, int64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t s[1024];
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  uint32_t v = i < n ? a[i] : 0u;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint32_t t = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0u;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) a[i] = s[threadIdx.x] - v;
  if (threadIdx.x == 1023) sums[blockIdx.x] = s[1023];
}
__global__ void scan_add_kernel(uint32_t* __restrict__ a, int64_t n, const uint32_t* __restrict__ sums) {
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  if (i < n) a[i] += sums[blockIdx.x];
}

// Stable scatter of one tile: warps own contiguous runs of the tile and walk
// them in order, so equal digits keep their input order (LSD correctness).
__global__ void __launch_bounds__(kSortThreads)
scatter_kernel(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
               uint32_t* __restrict__ vout, int64_t m, int shift, const uint32_t* __restrict__ tile_off,
               int64_t ntiles) {
  constexpr int NW = kSortThreads / 32;
  constexpr int PER_WARP = kTile / NW;  // contiguous items per warp
  __shared__ uint32_t wcnt[NW][kBuckets];
  __shared__ uint32_t base[kBuckets];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NW * kBuckets; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < kBuckets; d += blockDim.x) base[d] = tile_off[(int64_t)d * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t w0 = blockIdx.x * (int64_t)kTile + (int64_t)warp * PER_WARP;
  // pass 1: per-warp digit counts
  for (int r = 0; r < PER_WARP; r += 32) {
    const int64_t i = w0 + r + lane;
    const bool ok = i < m;
    const uint32_t d = ok ? (uint32_t)((kin[i] >> shift) & 0xff) : 0u;
    const uint32_t peers = __match_any_sync(PS_FULL, ok ? d : 0xffffffffu);
    if (ok && (peers & lanemask_lt()) == 0) wcnt[warp][d] += __popc(peers);
  }
  __syncthreads();
  // exclusive scan over warps per digit
  for (int d = threadIdx.x; d < kBuckets; d += blockDim.x) {
    uint32_t run = base[d];
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: stable placement
  for (int r = 0; r < PER_WARP; r += 32) {
    const int64_t i = w0 + r + lane;
    const bool ok = i < m;
    uint64_t k = 0;
    uint32_t v = 0, d = 0;
    if (ok) {
      k = kin[i];
      v = vin[i];
      d = (uint32_t)((k >> shift) & 0xff);
    }
    const uint32_t peers = __match_any_sync(PS_FULL, ok ? d : 0xffffffffu);
    const uint32_t rank = __popc(peers & lanemask_lt());
    uint32_t start = 0;
    if (ok) start = wcnt[warp][d];
    __syncwarp();
    if (ok) {
      const uint32_t pos = start + rank;
      kout[pos] = k;
      vout[pos] = v;
      if ((peers >> lane) == 1u) wcnt[warp][d] = start + __popc(peers);  // highest lane of the group
    }
    __syncwarp();
  }
}

// ranked[i] = val(key[i]) * fl(scale / (i+1)); then block-wise suffix minima.
__global__ void rank_scale_kernel(const uint64_t* __restrict__ keys, int64_t m, double scale,
                                  double* __restrict__ ranked, double* __restrict__ block_min) {
  __shared__ double s[1024];
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  double v = CUDART_INF;
  if (i < m) v = val_of(keys[i]) * (scale / (double)(i + 1));
  s[threadIdx.x] = v;
  __syncthreads();
  // inclusive suffix-min within the block
  for (int o = 1; o < 1024; o <<= 1) {
    double t = threadIdx.x + o < 1024 ? s[threadIdx.x + o] : CUDART_INF;
    __syncthreads();
    s[threadIdx.x] = fmin(s[threadIdx.x], t);
    __syncthreads();
  }
  if (i < m) ranked[i] = s[threadIdx.x];
  if (threadIdx.x == 0) block_min[blockIdx.x] = s[0];
}
// suffix-min over block minima (exclusive, i.e. min of later blocks), in
// place; one CTA: each thread a contiguous chunk, a reverse scan of the chunk
// minima across the block
constexpr int kSuffixThreads = 1024;
__global__ void __launch_bounds__(kSuffixThreads) block_suffix_min_kernel(double* __restrict__ bm, int64_t nb) {
  __shared__ double wmin[kSuffixThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (nb + kSuffixThreads - 1) / kSuffixThreads;
  const int64_t c0 = min(nb, (int64_t)threadIdx.x * per), c1 = min(nb, c0 + per);
  double m = CUDART_INF;
  for (int64_t b = c0; b < c1; ++b) m = fmin(m, bm[b]);
  // exclusive suffix min over threads (higher threads are later chunks)
  double x = m;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_down_sync(PS_FULL, x, o);
    if (lane + o < 32) x = fmin(x, y);
  }
  if (lane == 0) wmin[warp] = x;  // min over this warp's lanes
  __syncthreads();
  double after = CUDART_INF;       // min over later warps
  for (int w = warp + 1; w < kSuffixThreads / 32; ++w) after = fmin(after, wmin[w]);
  const double later_lanes = __shfl_down_sync(PS_FULL, x, 1);
  double run = fmin(after, lane < 31 ? later_lanes : CUDART_INF);
  for (int64_t b = c1 - 1; b >= c0; --b) {
    const double v = bm[b];
    bm[b] = run;
    run = fmin(run, v);
  }
}
__global__ void bh_scatter_kernel(const double* __restrict__ ranked, const double* __restrict__ bm,
                                  const uint32_t* __restrict__ idx, int64_t m, int64_t cols, int symmetric,
                                  double* __restrict__ out) {
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  if (i >= m) return;
  double v = fmin(ranked[i], bm[blockIdx.x]);
  v = fmin(1.0, v);
  const int64_t f = idx[i];
  out[f] = v;
  if (symmetric) {
    const int64_t r = f / cols, c = f - r * cols;
    out[c * cols + r] = v;
  }
}
__global__ void bonferroni_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                  const unsigned long long* __restrict__ count, int64_t cols, int symmetric,
                                  double* __restrict__ out) {
  const int64_t m = (int64_t)*count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)m * val_of(keys[i]);
    v = fmin(1.0, v);
    const int64_t f = idx[i];
    out[f] = v;
    if (symmetric) {
      const int64_t r = f / cols, c = f - r * cols;
      out[c * cols + r] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Large families, fast path: a stable LSD radix over the HIGH 32 key bits only
// (four 8-bit passes moving 4-byte high halves and 4-byte positions into the
// compacted arrays), then runs of equal high halves are put in full-key order
// by one thread per run (runs of up to kShortRun); a mixed run longer than
// that raises a flag and the caller re-sorts on all 64 bits (the original
// compacted arrays are untouched).  One host round trip in all.
constexpr int kShortRun = 64;
static_assert(kSortThreads == kBuckets, "one thread per digit");

__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* wsum /* [8] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint32_t base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  return base + x - v;
}

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads)
h32_hist_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ dk,
                const unsigned long long* __restrict__ count, int shift, uint32_t* __restrict__ tile_hist,
                int64_t ntiles) {
  __shared__ uint32_t h[kBuckets];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t m = (int64_t)*count, t0 = blockIdx.x * (int64_t)kTile;
  for (int q = 0; q < kSortItems; ++q) {
    const int64_t i = t0 + (int64_t)q * kSortThreads + threadIdx.x;
    const bool ok = i < m;
    uint32_t d = 0xffffffffu;
    if (ok) d = ((FIRST ? (uint32_t)(keys[i] >> 32) : dk[i]) >> shift) & 0xffu;
    const uint32_t peers = __match_any_sync(PS_FULL, d);
    if (ok && (peers & lanemask_lt()) == 0) atomicAdd(&h[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  tile_hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Row d of the digit-major tile histogram -> exclusive offsets within digit d;
// totals[d] = the digit's count.  One block per digit.
__global__ void __launch_bounds__(kSortThreads)
digit_scan_kernel(uint32_t* __restrict__ tile_hist, int64_t ntiles, uint32_t* __restrict__ totals) {
  __shared__ uint32_t wsum[kSortThreads / 32];
  uint32_t* row = tile_hist + (int64_t)blockIdx.x * ntiles;
  const int64_t per = (ntiles + kSortThreads - 1) / kSortThreads;
  const int64_t b = threadIdx.x * per, e = b + per < ntiles ? b + per : ntiles;
  uint32_t sum = 0;
  for (int64_t i = b; i < e; ++i) sum += row[i];
  uint32_t run = block_excl_scan256(sum, wsum);
  if (threadIdx.x == kSortThreads - 1) totals[blockIdx.x] = run + sum;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t c = row[i];
    row[i] = run;
    run += c;
  }
}

template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads)
h32_scatter_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ dk_in,
                   const uint32_t* __restrict__ pos_in, uint32_t* __restrict__ dk_out, uint32_t* __restrict__ pos_out,
                   const unsigned long long* __restrict__ count, int shift, const uint32_t* __restrict__ tile_off,
                   const uint32_t* __restrict__ totals, int64_t ntiles) {
  constexpr int NW = kSortThreads / 32;
  constexpr int PER_WARP = kTile / NW;
  __shared__ uint32_t wcnt[NW][kBuckets];
  __shared__ uint32_t wsum[NW];
  const int64_t m = (int64_t)*count;
  if (blockIdx.x * (int64_t)kTile >= m) return;  // block-uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NW * kBuckets; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  // digit base = exclusive scan of the digit totals + this tile's offset
  const uint32_t dbase = block_excl_scan256(totals[threadIdx.x], wsum) +
                         tile_off[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t w0 = blockIdx.x * (int64_t)kTile + (int64_t)warp * PER_WARP;
  auto load = [&](int64_t i, uint32_t& k, uint32_t& v) {
    if (FIRST) {
      k = (uint32_t)(keys[i] >> 32);
      v = (uint32_t)i;
    } else {
      k = dk_in[i];
      v = pos_in[i];
    }
  };
  for (int r = 0; r < PER_WARP; r += 32) {
    const int64_t i = w0 + r + lane;
    const bool ok = i < m;
    uint32_t d = 0xffffffffu;
    if (ok) {
      uint32_t k, v;
      load(i, k, v);
      d = (k >> shift) & 0xffu;
    }
    const uint32_t peers = __match_any_sync(PS_FULL, d);
    if (ok && (peers & lanemask_lt()) == 0) wcnt[warp][d] += __popc(peers);
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    uint32_t run = dbase;
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int r = 0; r < PER_WARP; r += 32) {
    const int64_t i = w0 + r + lane;
    const bool ok = i < m;
    uint32_t k = 0, v = 0, d = 0xffffffffu;
    if (ok) {
      load(i, k, v);
      d = (k >> shift) & 0xffu;
    }
    const uint32_t peers = __match_any_sync(PS_FULL, d);
    const uint32_t rank = __popc(peers & lanemask_lt());
    uint32_t start = 0;
    if (ok) start = wcnt[warp][d];
    __syncwarp();
    if (ok) {
      const uint32_t p = start + rank;
      dk_out[p] = k;
      pos_out[p] = v;
      if ((peers >> lane) == 1u) wcnt[warp][d] = start + __popc(peers);
    }
    __syncwarp();
  }
}

// Runs of equal high halves.  Runs of <= kShortRun: the run's first thread
// insertion-sorts its positions by the full key.  Runs of <= kBlockRun: queued
// for a CTA-wide sort (long_run_sort_kernel).  Longer runs whose keys differ
// set *flag (the caller re-sorts on all 64 bits).
constexpr int kBlockRun = 16384;

__device__ __forceinline__ int64_t run_end(const uint32_t* dk, int64_t i, int64_t m, uint32_t h) {
  int64_t a = i, b = m;  // first index in [i, m) with dk > h (dk ascending)
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (dk[mid] <= h) a = mid + 1;
    else b = mid;
  }
  return a;
}
__device__ __forceinline__ int64_t run_begin(const uint32_t* dk, int64_t i, uint32_t h) {
  int64_t a = 0, b = i;  // first index in [0, i] with dk == h
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (dk[mid] < h) a = mid + 1;
    else b = mid;
  }
  return a;
}

__global__ void h32_fixup_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ dk,
                                 uint32_t* __restrict__ pos, const unsigned long long* __restrict__ count,
                                 int* __restrict__ flag /* [0] fallback, [1] queued runs */,
                                 int2* __restrict__ runs) {
  const int64_t m = (int64_t)*count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = dk[i];
    if (i > 0 && dk[i - 1] == h) {
      // inside a run: a differing neighbour in a run too long for the CTA
      // sort means the fallback (the reads may race with a short run's
      // insertion sort, which cannot change the run's length)
      if (keys[pos[i - 1]] != keys[pos[i]]) {
        const int64_t L = run_end(dk, i, m, h) - run_begin(dk, i, h);
        if (L > kBlockRun) atomicExch(&flag[0], 1);
      }
      continue;
    }
    if (i + 1 >= m || dk[i + 1] != h) continue;  // singleton
    const int64_t e = run_end(dk, i, m, h), L = e - i;
    if (L > kBlockRun) continue;
    if (L > kShortRun) {
      const int q = atomicAdd(&flag[1], 1);
      runs[q] = make_int2((int)i, (int)L);
      continue;
    }
    for (int64_t a = i + 1; a < e; ++a) {
      const uint32_t pa = pos[a];
      const uint64_t ka = keys[pa];
      int64_t b = a - 1;
      while (b >= i && keys[pos[b]] > ka) {
        pos[b + 1] = pos[b];
        --b;
      }
      pos[b + 1] = pa;
    }
  }
}

// One CTA per queued run: stable LSD radix on the low key halves in
// registers / shared memory (warp-striped items, per-warp digit counts,
// constant bytes skipped), as the small-family kernel does for high halves.
constexpr int kRunSortThreads = 1024;
constexpr int kRunItems = kBlockRun / kRunSortThreads;  // 16
constexpr int kRunWarps = kRunSortThreads / 32;
constexpr size_t kRunSortSmem = (size_t)kBlockRun * (4 + 2 + 4);
__global__ void __launch_bounds__(kRunSortThreads)
long_run_sort_kernel(const uint64_t* __restrict__ keys, uint32_t* __restrict__ pos, const int* __restrict__ flag,
                     const int2* __restrict__ runs) {
  extern __shared__ __align__(16) unsigned char lrs[];
  uint32_t* sk = reinterpret_cast<uint32_t*>(lrs);                                // low halves
  uint16_t* sx = reinterpret_cast<uint16_t*>(lrs + (size_t)kBlockRun * 4);        // run-local index
  uint32_t* sp = reinterpret_cast<uint32_t*>(lrs + (size_t)kBlockRun * 6);        // original positions
  __shared__ uint16_t wcnt[kRunWarps][256];
  __shared__ int warp_buf[kRunWarps];
  __shared__ uint32_t s_and, s_or;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nruns = flag[1];
  for (int r = blockIdx.x; r < nruns; r += gridDim.x) {
    const int2 run = runs[r];
    const int L = run.y;
    if (threadIdx.x == 0) {
      s_and = 0xffffffffu;
      s_or = 0u;
    }
    uint32_t k32[kRunItems], idx[kRunItems];  // idx: run-local index | in-warp offset << 16
    __syncthreads();
    {
      uint32_t a = 0xffffffffu, o = 0u;
#pragma unroll
      for (int q = 0; q < kRunItems; ++q) {
        const int t = warp * 32 * kRunItems + q * 32 + lane;
        idx[q] = (uint32_t)t;
        k32[q] = 0xffffffffu;  // padding sorts last
        if (t < L) {
          const uint32_t p = pos[run.x + t];
          sp[t] = p;
          k32[q] = (uint32_t)keys[p];
          a &= k32[q];
          o |= k32[q];
        }
      }
      a = __reduce_and_sync(PS_FULL, a);
      o = __reduce_or_sync(PS_FULL, o);
      if (lane == 0) {
        atomicAnd(&s_and, a);
        atomicOr(&s_or, o);
      }
    }
    __syncthreads();
    const uint32_t diff = s_and ^ s_or;
    for (int b = 0; b < 4; ++b) {
      const int shift = 8 * b;
      if (((diff >> shift) & 0xffu) == 0) continue;
      for (int q = threadIdx.x; q < kRunWarps * 256; q += kRunSortThreads) (&wcnt[0][0])[q] = 0;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kRunItems; ++q) {
        const uint32_t dg = (k32[q] >> shift) & 0xffu;
        const uint32_t peers = __match_any_sync(PS_FULL, dg);
        const uint32_t base = wcnt[warp][dg];
        __syncwarp();
        idx[q] = (idx[q] & 0xFFFFu) | ((base + __popc(peers & lanemask_lt())) << 16);
        if ((peers >> lane) == 1u) wcnt[warp][dg] = (uint16_t)(base + __popc(peers));
        __syncwarp();
      }
      __syncthreads();
      if (threadIdx.x < 256) {
        uint32_t tot = 0;
        for (int w = 0; w < kRunWarps; ++w) tot += wcnt[w][threadIdx.x];
        uint32_t x = tot;
#pragma unroll
        for (int sft = 1; sft < 32; sft <<= 1) {
          const uint32_t y = __shfl_up_sync(PS_FULL, x, sft);
          if (lane >= sft) x += y;
        }
        if (lane == 31) warp_buf[warp] = (int)x;
        asm volatile("bar.sync 1, 256;");
        uint32_t before = 0;
        for (int w = 0; w < warp; ++w) before += (uint32_t)warp_buf[w];
        uint32_t run_ = before + x - tot;
        for (int w = 0; w < kRunWarps; ++w) {
          const uint32_t c = wcnt[w][threadIdx.x];
          wcnt[w][threadIdx.x] = (uint16_t)run_;
          run_ += c;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kRunItems; ++q) {
        const uint32_t dg = (k32[q] >> shift) & 0xffu;
        const uint32_t dst = (uint32_t)wcnt[warp][dg] + (idx[q] >> 16);
        sk[dst] = k32[q];
        sx[dst] = (uint16_t)idx[q];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kRunItems; ++q) {
        const int t = warp * 32 * kRunItems + q * 32 + lane;
        k32[q] = sk[t];
        idx[q] = sx[t];
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kRunItems; ++q) {
      const int t = warp * 32 * kRunItems + q * 32 + lane;
      if (t < L) pos[run.x + t] = sp[idx[q] & 0xFFFFu];
    }
    __syncthreads();
  }
}

// ranked[i] = val(keys[pos[i]]) * fl(scale / (i+1)), block suffix minima
__global__ void rank_scale_pos_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ pos, int64_t m,
                                      double scale, double* __restrict__ ranked, double* __restrict__ block_min) {
  __shared__ double s[1024];
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  double v = CUDART_INF;
  if (i < m) v = val_of(keys[pos[i]]) * (scale / (double)(i + 1));
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    double t = threadIdx.x + o < 1024 ? s[threadIdx.x + o] : CUDART_INF;
    __syncthreads();
    s[threadIdx.x] = fmin(s[threadIdx.x], t);
    __syncthreads();
  }
  if (i < m) ranked[i] = s[threadIdx.x];
  if (threadIdx.x == 0) block_min[blockIdx.x] = s[0];
}
__global__ void bh_scatter_pos_kernel(const double* __restrict__ ranked, const double* __restrict__ bm,
                                      const uint32_t* __restrict__ pos, const uint32_t* __restrict__ idx, int64_t m,
                                      int64_t cols, int symmetric, double* __restrict__ out) {
  const int64_t i = blockIdx.x * 1024LL + threadIdx.x;
  if (i >= m) return;
  double v = fmin(ranked[i], bm[blockIdx.x]);
  v = fmin(1.0, v);
  const int64_t f = idx[pos[i]];
  out[f] = v;
  if (symmetric) {
    const int64_t r = f / cols, c = f - r * cols;
    out[c * cols + r] = v;
  }
}

// ---------------------------------------------------------------------------
// Small families spread over the GPU (BH, m <= kSmallMax), three launches:
//  1. bh_chunk_sort: each CTA sorts a 2048-key chunk (keys = order-preserving
//     u64 of p, ties broken by index) with a shared-memory bitonic network
//     and records every member's rank inside its chunk;
//  2. bh_rank: every CTA stages all sorted chunks in shared memory (<= 192 KB)
//     and each member's global rank is its chunk rank plus, per other chunk,
//     a binary search (keys <= k in earlier chunks, < k in later ones: the
//     stable order of the reference's argsort); p and the output index are
//     scattered to sorted position;
//  3. bh_stepup_sorted: one CTA walks the sorted family from the top in
//     1024-element rounds -- v_r = p_(r) m / (r + 1), block suffix minimum
//     with a carry -- and scatters min(1, .) to the outputs.
// ~10 us at m = 2e4, against ~160 us for the all-pairs counting rank.
constexpr int kChunk = 2048, kChunkThreads = 1024;
__global__ void __launch_bounds__(kChunkThreads)
bh_chunk_sort_kernel(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ count,
                     uint64_t* __restrict__ skeys, uint32_t* __restrict__ crank, uint32_t* __restrict__ spos) {
  __shared__ uint64_t sk[kChunk];
  __shared__ uint16_t si[kChunk];
  const int m = (int)*count;
  const int c0 = blockIdx.x * kChunk;
  if (c0 >= m) return;  // block-uniform
  for (int t = threadIdx.x; t < kChunk; t += kChunkThreads) {
    sk[t] = c0 + t < m ? keys[c0 + t] : ~0ull;  // padding sorts last (no p maps to ~0)
    si[t] = (uint16_t)t;
  }
  __syncthreads();
  // bitonic network on (key, local index): unique, so the order is stable
  for (int size = 2; size <= kChunk; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int t = threadIdx.x;
      const int i = 2 * t - (t & (stride - 1));  // first of the compared pair
      const int j = i + stride;
      const bool up = (i & size) == 0;
      const uint64_t ki = sk[i], kj = sk[j];
      const uint16_t ii = si[i], ij = si[j];
      const bool gt = ki > kj || (ki == kj && ii > ij);
      if (gt == up) {
        sk[i] = kj;
        sk[j] = ki;
        si[i] = ij;
        si[j] = ii;
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < kChunk; t += kChunkThreads) {
    skeys[c0 + t] = sk[t];
    if (spos) spos[c0 + t] = (uint32_t)(c0 + si[t]);  // (padding: positions >= m, never read)
    else if (c0 + si[t] < m) crank[c0 + si[t]] = (uint32_t)t;
  }
}

// ---------------------------------------------------------------------------
// Medium families (BH, kSmallMax < m <= kMergeMax): the 2048-key sorted
// chunks are merged pairwise, level by level -- each member's place in the
// merged run is its place in its own run plus a binary search of the partner
// run (keys < k in the later run, <= k in the earlier one: stable) -- then a
// blocked suffix minimum over the sorted family.  Every launch reads m on the
// device (no host round trip), against the 4-pass radix's ~16 launches and a
// host synchronisation.
constexpr int64_t kMergeMax = (int64_t)1 << 20;
__global__ void bh_merge_level_kernel(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ pin,
                                      uint64_t* __restrict__ kout, uint32_t* __restrict__ pout,
                                      const unsigned long long* __restrict__ count, int64_t L) {
  const int64_t m = (int64_t)*count;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t run = i / L, p = i - run * L;
  const int64_t pb = (run ^ 1) * L;
  const uint64_t k = kin[i];
  int64_t c = 0;
  if (pb < m) {
    const uint64_t* b = kin + pb;
    int64_t lo = 0, hi = min(L, m - pb);
    if (run & 1) {  // partner run is earlier: its keys <= k come first
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (b[mid] <= k) lo = mid + 1;
        else hi = mid;
      }
    } else {  // partner run is later: its keys < k come first
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (b[mid] < k) lo = mid + 1;
        else hi = mid;
      }
    }
    c = lo;
  }
  const int64_t o = (run & ~(int64_t)1) * L + p + c;
  kout[o] = k;
  pout[o] = pin[i];
}

// v_r = p_(r) m / (r + 1) over 1024-rank blocks: in-block inclusive suffix
// minimum, and the block minimum
__global__ void __launch_bounds__(1024)
bh_sorted_scale_kernel(const uint64_t* __restrict__ sk, const unsigned long long* __restrict__ count,
                       double* __restrict__ ranked, double* __restrict__ bmin) {
  __shared__ double s_w[32];
  __shared__ double s_after[32];
  const int64_t m = (int64_t)*count;
  const int64_t r = blockIdx.x * 1024LL + threadIdx.x;
  if (blockIdx.x * 1024LL >= m) return;  // block-uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = r < m ? val_of(sk[r]) * ((double)m / (double)(r + 1)) : CUDART_INF;
#pragma unroll
  for (int sft = 1; sft < 32; sft <<= 1) {
    const double y = __shfl_down_sync(PS_FULL, v, sft);
    if (lane + sft < 32) v = fmin(v, y);
  }
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = s_w[lane];
#pragma unroll
    for (int sft = 1; sft < 32; sft <<= 1) {
      const double y = __shfl_down_sync(PS_FULL, w, sft);
      if (lane + sft < 32) w = fmin(w, y);
    }
    const double after = __shfl_down_sync(PS_FULL, w, 1);
    s_after[lane] = lane == 31 ? CUDART_INF : after;
    if (lane == 0) bmin[blockIdx.x] = w;
  }
  __syncthreads();
  if (r < m) ranked[r] = fmin(v, s_after[warp]);
}

// exclusive suffix minimum of the block minima (one CTA), in place: bmin[b]
// becomes the minimum over the blocks after b
__global__ void __launch_bounds__(1024)
bh_block_suffix_kernel(double* __restrict__ bmin, const unsigned long long* __restrict__ count) {
  __shared__ double s_w[32];
  __shared__ double s_after[32];
  const int64_t nb = ((int64_t)*count + 1023) / 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (nb + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  double tmin = CUDART_INF;
  for (int64_t b = b0; b < b1; ++b) tmin = fmin(tmin, bmin[b]);
  double incl = tmin;
#pragma unroll
  for (int sft = 1; sft < 32; sft <<= 1) {
    const double y = __shfl_down_sync(PS_FULL, incl, sft);
    if (lane + sft < 32) incl = fmin(incl, y);
  }
  if (lane == 0) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double w = s_w[lane];
#pragma unroll
    for (int sft = 1; sft < 32; sft <<= 1) {
      const double y = __shfl_down_sync(PS_FULL, w, sft);
      if (lane + sft < 32) w = fmin(w, y);
    }
    const double after = __shfl_down_sync(PS_FULL, w, 1);
    s_after[lane] = lane == 31 ? CUDART_INF : after;
  }
  __syncthreads();
  double run = __shfl_down_sync(PS_FULL, incl, 1);
  if (lane == 31) run = CUDART_INF;
  run = fmin(run, s_after[warp]);
  __syncthreads();  // every thread has read its inputs before the in-place writes
  for (int64_t b = b1 - 1; b >= b0; --b) {
    const double v = bmin[b];
    bmin[b] = run;
    run = fmin(run, v);
  }
}

__global__ void bh_sorted_scatter_kernel(const double* __restrict__ ranked, const double* __restrict__ after,
                                         const uint32_t* __restrict__ spos, const uint32_t* __restrict__ fidx,
                                         const unsigned long long* __restrict__ count, int64_t cols, int symmetric,
                                         double* __restrict__ out) {
  const int64_t m = (int64_t)*count;
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double v = fmin(1.0, fmin(ranked[r], after[r / 1024]));
  const int64_t f = fidx[spos[r]];
  out[f] = v;
  if (symmetric) {
    const int64_t rr = f / cols, cc = f - rr * cols;
    out[cc * cols + rr] = v;
  }
}

__global__ void __launch_bounds__(1024)
bh_rank_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ fidx,
               const unsigned long long* __restrict__ count, const uint64_t* __restrict__ skeys,
               const uint32_t* __restrict__ crank, double* __restrict__ sval, uint32_t* __restrict__ sidx) {
  extern __shared__ uint64_t sks[];
  const int m = (int)*count;
  if (blockIdx.x * 1024 >= m) return;
  const int nch = (m + kChunk - 1) / kChunk;
  for (int t = threadIdx.x; t < nch * kChunk; t += 1024) sks[t] = skeys[t];
  __syncthreads();
  const int i = blockIdx.x * 1024 + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = keys[i];
  const int own = i / kChunk;
  uint32_t r = crank[i];
  for (int c = 0; c < nch; ++c) {
    if (c == own) continue;
    const uint64_t* a = sks + c * kChunk;
    // earlier chunks: members with key <= k precede i; later: key < k
    int lo = 0, hi = kChunk;
    if (c < own) {
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= k) lo = mid + 1;
        else hi = mid;
      }
    } else {
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
      }
    }
    r += (uint32_t)lo;
  }
  sval[r] = val_of(k);
  sidx[r] = fidx[i];
}

constexpr int kStepThreads = 1024, kStepRounds = 24;  // kSmallMax / kStepThreads (asserted below)
__global__ void __launch_bounds__(kStepThreads)
bh_stepup_sorted_kernel(const double* __restrict__ sval, const uint32_t* __restrict__ sidx,
                        const unsigned long long* __restrict__ count, int64_t cols, int symmetric,
                        double* __restrict__ out) {
  __shared__ double s_w[kStepThreads / 32];
  __shared__ double s_after[kStepThreads / 32];  // minimum over the warps after w
  const int m = (int)*count;
  if (m == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double scale = (double)m;
  // thread t owns the ranks [t per, (t + 1) per): its scaled values in registers
  const int per = (m + kStepThreads - 1) / kStepThreads;
  const int i0 = threadIdx.x * per;
  double v[kStepRounds];
  double tmin = CUDART_INF;
#pragma unroll
  for (int q = 0; q < kStepRounds; ++q) {
    const int r = i0 + q;
    v[q] = q < per && r < m ? sval[r] * (scale / (double)(r + 1)) : CUDART_INF;
    tmin = fmin(tmin, v[q]);
  }
  // exclusive suffix minimum of the thread minima over higher threads
  double incl = tmin;
#pragma unroll
  for (int sft = 1; sft < 32; sft <<= 1) {
    const double y = __shfl_down_sync(PS_FULL, incl, sft);
    if (lane + sft < 32) incl = fmin(incl, y);
  }
  if (lane == 0) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double w = s_w[lane];
#pragma unroll
    for (int sft = 1; sft < 32; sft <<= 1) {
      const double y = __shfl_down_sync(PS_FULL, w, sft);
      if (lane + sft < 32) w = fmin(w, y);
    }
    const double after = __shfl_down_sync(PS_FULL, w, 1);
    s_after[lane] = lane == 31 ? CUDART_INF : after;
  }
  __syncthreads();
  double run = __shfl_down_sync(PS_FULL, incl, 1);
  if (lane == 31) run = CUDART_INF;
  run = fmin(run, s_after[warp]);
#pragma unroll
  for (int q = kStepRounds - 1; q >= 0; --q) {
    const int r = i0 + q;
    if (q < per && r < m) {
      run = fmin(run, v[q]);
      const double o = fmin(1.0, run);
      const int64_t f = sidx[r];
      out[f] = o;
      if (symmetric) {
        const int64_t rr = f / cols, cc = f - rr * cols;
        out[cc * cols + rr] = o;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Small families (m <= kSmallMax): the whole BH / BY adjustment in one CTA --
// stable LSD radix on the high 32 key bits in registers / shared memory (as
// the presort), short runs of equal high halves repaired on the low halves
// (long ones: full 8-byte sort), then the scaled values, a block-wide reverse
// cumulative minimum and the scatter.  No host round trips, two launches in
// all (compaction + this) instead of ~30.
constexpr int kSmallThreads = 1024, kSmallItems = 24;
constexpr int kSmallMax = kSmallThreads * kSmallItems;  // 24576
static_assert(kStepRounds * kStepThreads == kSmallMax, "BH step-up rounds cover the small families");
static_assert(kChunk * 12 == kSmallMax, "BH rank staging: 12 sorted chunks in shared memory");
constexpr int kSmallWarps = kSmallThreads / 32;

__global__ void __launch_bounds__(kSmallThreads, 1)
adjust_small_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ fidx,
                    const unsigned long long* __restrict__ count, double by_factor, int64_t cols, int symmetric,
                    double* __restrict__ out) {
  constexpr int ITEMS = kSmallItems;
  extern __shared__ __align__(16) unsigned char asm_raw[];
  uint32_t* sk32 = reinterpret_cast<uint32_t*>(asm_raw);
  uint16_t* spos = reinterpret_cast<uint16_t*>(asm_raw + (size_t)kSmallMax * 4);
  __shared__ uint16_t wcnt[kSmallWarps][256];
  __shared__ int warp_buf[kSmallWarps];
  __shared__ unsigned long long s_and, s_or;
  __shared__ int s_long;
  __shared__ double s_tmin[kSmallWarps];
  const int m = (int)*count;
  if (m == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_and = ~0ull;
    s_or = 0ull;
    s_long = 0;
  }
  __syncthreads();
  uint32_t k32[ITEMS], idx[ITEMS];  // idx: position in keys[] | in-warp offset << 16
  {
    unsigned long long a = ~0ull, o = 0ull;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int p = warp * 32 * ITEMS + i * 32 + lane;
      if (p < m) {
        const uint64_t k = keys[p];
        a &= k;
        o |= k;
      }
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
  for (int round = 0, st0 = 1; round < 2; ++round, st0 = 0) {
    for (int st = st0; st < 2; ++st) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int p = warp * 32 * ITEMS + i * 32 + lane;
        const int pos = round == 0 ? p : (p < m ? spos[p] : p);
        idx[i] = p < m ? (uint32_t)pos : 0xFFFFu;
        const uint64_t k = p < m ? keys[pos] : ~0ull;
        k32[i] = st ? (uint32_t)(k >> 32) : (uint32_t)k;
      }
      __syncthreads();
      for (int b = 0; b < 4; ++b) {
        const int shift = 8 * b;
        if (((diff >> (32 * st + shift)) & 0xffull) == 0 || m <= 1) continue;
        for (int i = threadIdx.x; i < kSmallWarps * 256; i += kSmallThreads) (&wcnt[0][0])[i] = 0;
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
        if (threadIdx.x < 256) {
          uint32_t tot = 0;
          for (int w = 0; w < kSmallWarps; ++w) tot += wcnt[w][threadIdx.x];
          uint32_t x = tot;
#pragma unroll
          for (int sft = 1; sft < 32; sft <<= 1) {
            const uint32_t y = __shfl_up_sync(PS_FULL, x, sft);
            if (lane >= sft) x += y;
          }
          if (lane == 31) warp_buf[warp] = (int)x;
          asm volatile("bar.sync 1, 256;");
          uint32_t before = 0;
          for (int w = 0; w < warp; ++w) before += (uint32_t)warp_buf[w];
          uint32_t run = before + x - tot;
          for (int w = 0; w < kSmallWarps; ++w) {
            const uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = (uint16_t)run;
            run += c;
          }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const uint32_t dg = (k32[i] >> shift) & 0xffu;
          const uint32_t dst = (uint32_t)wcnt[warp][dg] + (idx[i] >> 16);
          sk32[dst] = k32[i];
          spos[dst] = (uint16_t)idx[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int p = warp * 32 * ITEMS + i * 32 + lane;
          k32[i] = sk32[p];
          idx[i] = spos[p];
        }
        __syncthreads();
      }
    }
    // positions not permuted by any pass are still in load order
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int p = warp * 32 * ITEMS + i * 32 + lane;
      if (p < m) {
        spos[p] = (uint16_t)idx[i];
        sk32[p] = (uint32_t)(keys[idx[i] & 0xFFFFu] >> 32);
      }
    }
    __syncthreads();
    if (round == 1 || (uint32_t)diff == 0u) break;
    for (int p = threadIdx.x; p < m; p += kSmallThreads) {  // repair colliding high halves
      const uint32_t h = sk32[p];
      if (p > 0 && sk32[p - 1] == h) continue;
      int e = p + 1;
      while (e < m && sk32[e] == h) ++e;
      if (e - p == 1) continue;
      if (e - p > 64) {
        s_long = 1;
        continue;
      }
      uint32_t lo[64];
      uint16_t id[64];
      const int n = e - p;
      for (int q = 0; q < n; ++q) {
        id[q] = spos[p + q];
        lo[q] = (uint32_t)keys[id[q]];
      }
      for (int i = 1; i < n; ++i) {
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
      for (int q = 0; q < n; ++q) spos[p + q] = id[q];
    }
    __syncthreads();
    if (!s_long) break;
  }
  // scaled values v_i = p_(i) * (scale / i) and their reverse cumulative
  // minimum: thread t owns sorted positions [t*ITEMS, (t+1)*ITEMS)
  const double scale = (double)m * by_factor;
  const int i0 = threadIdx.x * ITEMS;
  auto scaled = [&](int p) { return val_of(keys[spos[p]]) * (scale / (double)(p + 1)); };
  double tmin = CUDART_INF;
  for (int i = 0; i < ITEMS; ++i)
    if (i0 + i < m) tmin = fmin(tmin, scaled(i0 + i));
  // exclusive suffix minimum over threads (later threads)
  double wmin = tmin;
#pragma unroll
  for (int sft = 1; sft < 32; sft <<= 1) {
    const double y = __shfl_down_sync(PS_FULL, wmin, sft);
    if (lane + sft < 32) wmin = fmin(wmin, y);
  }
  if (lane == 0) s_tmin[warp] = wmin;  // min over this warp's threads
  __syncthreads();
  double run = __shfl_down_sync(PS_FULL, wmin, 1);
  if (lane == 31) run = CUDART_INF;
  for (int w = warp + 1; w < kSmallWarps; ++w) run = fmin(run, s_tmin[w]);
  for (int i = ITEMS - 1; i >= 0; --i) {
    const int p = i0 + i;
    if (p >= m) continue;
    run = fmin(run, scaled(p));
    const double r = fmin(1.0, run);
    const int64_t f = fidx[spos[p]];
    out[f] = r;
    if (symmetric) {
      const int64_t rr = f / cols, cc = f - rr * cols;
      out[cc * cols + rr] = r;
    }
  }
}

int scan_u32(uint32_t* a, int64_t n, cudaStream_t s) {
  const int64_t nb = ps_ceil_div(n, 1024);
  uint32_t* sums = nullptr;
  PS_CUDA(ps_alloc(&sums, (size_t)nb, s));
  scan_block_kernel<<<(unsigned)nb, 1024, 0, s>>>(a, n, sums);
  PS_LAUNCHED();
  if (nb > 1) {
    int rc = scan_u32(sums, nb, s);
    if (rc) return rc;
    scan_add_kernel<<<(unsigned)nb, 1024, 0, s>>>(a, n, sums);
    PS_LAUNCHED();
  }
  ps_free(sums, s);
  return PS_OK;
}

// host-side BY factor: numpy's pairwise summation of 1/i (adjust.py:34-36).
double numpy_pairwise_harmonic(int64_t m) {
  // numpy sums float64 arrays with pairwise summation: blocks of <= 128
  // elements are summed with 8 interleaved accumulators, larger ranges are
  // split in halves (n2 = n/2 rounded down to a multiple of 8).
  struct Rec {
    static double sum(int64_t lo, int64_t n) {
      if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += 1.0 / (double)(lo + i + 1);
        return r;
      }
      if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = 1.0 / (double)(lo + j + 1);
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
          for (int j = 0; j < 8; ++j) r[j] += 1.0 / (double)(lo + i + j + 1);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += 1.0 / (double)(lo + i + 1);
        return res;
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      return sum(lo, n2) + sum(lo + n2, n - n2);
    }
  };
  return Rec::sum(0, m);
}

// Fast large-family BH / BY (see h32_* above).  Families above kFastMax keep
// the 64-bit sort (the high halves of more p-values collide too often).
constexpr int64_t kFastMax = (int64_t)1 << 26;
constexpr int kNeedFullSort = -12345;

int adjust_fast(uint64_t* keys, uint32_t* idx, unsigned long long* d_count, int64_t cols, int symmetric,
                int method, double* out, cudaStream_t s, int64_t fam_max) {
  ps_device_state* ds = ps_state();
  const int64_t ntiles = std::max<int64_t>(1, ps_ceil_div(fam_max, kTile));
  uint32_t *dk[2] = {nullptr, nullptr}, *pos[2] = {nullptr, nullptr}, *tile_hist = nullptr, *totals = nullptr;
  unsigned long long* host_pair = nullptr;  // {count, flag}
  int* d_flag = nullptr;  // {fallback, queued runs}
  int2* runs = nullptr;
  PS_CUDA(ps_alloc(&dk[0], (size_t)fam_max, s));
  PS_CUDA(ps_alloc(&dk[1], (size_t)fam_max, s));
  PS_CUDA(ps_alloc(&pos[0], (size_t)fam_max, s));
  PS_CUDA(ps_alloc(&pos[1], (size_t)fam_max, s));
  PS_CUDA(ps_alloc(&tile_hist, (size_t)(ntiles * kBuckets), s));
  PS_CUDA(ps_alloc(&totals, (size_t)kBuckets, s));
  PS_CUDA(ps_alloc(&d_flag, 2, s));
  PS_CUDA(cudaMemsetAsync(d_flag, 0, 2 * sizeof(int), s));
  PS_CUDA(ps_alloc(&runs, (size_t)(fam_max / (kShortRun + 1) + 1), s));
  int cur = 0;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 8 * pass;
    if (pass == 0) h32_hist_kernel<true><<<(unsigned)ntiles, kSortThreads, 0, s>>>(keys, nullptr, d_count, shift, tile_hist, ntiles);
    else h32_hist_kernel<false><<<(unsigned)ntiles, kSortThreads, 0, s>>>(keys, dk[cur], d_count, shift, tile_hist, ntiles);
    PS_LAUNCHED();
    digit_scan_kernel<<<kBuckets, kSortThreads, 0, s>>>(tile_hist, ntiles, totals);
    PS_LAUNCHED();
    if (pass == 0)
      h32_scatter_kernel<true><<<(unsigned)ntiles, kSortThreads, 0, s>>>(keys, nullptr, nullptr, dk[cur ^ 1], pos[cur ^ 1],
                                                                        d_count, shift, tile_hist, totals, ntiles);
    else
      h32_scatter_kernel<false><<<(unsigned)ntiles, kSortThreads, 0, s>>>(keys, dk[cur], pos[cur], dk[cur ^ 1],
                                                                         pos[cur ^ 1], d_count, shift, tile_hist,
                                                                         totals, ntiles);
    PS_LAUNCHED();
    cur ^= 1;
  }
  {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ps_ceil_div(fam_max, 256), (int64_t)ds->num_sms * 8));
    h32_fixup_kernel<<<blocks, 256, 0, s>>>(keys, dk[cur], pos[cur], d_count, d_flag, runs);
    PS_LAUNCHED();
    PS_CUDA(cudaFuncSetAttribute(long_run_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kRunSortSmem));
    long_run_sort_kernel<<<ds->num_sms, kRunSortThreads, kRunSortSmem, s>>>(keys, pos[cur], d_flag, runs);
    PS_LAUNCHED();
  }
  unsigned long long hp[2] = {0, 0};
  PS_CUDA(cudaMemcpyAsync(&hp[0], d_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  int flag_h = 0;
  PS_CUDA(cudaMemcpyAsync(&flag_h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  PS_CUDA(cudaStreamSynchronize(s));
  (void)host_pair;
  const int64_t m = (int64_t)hp[0];
  int rc = PS_OK;
  if (flag_h) {
    rc = kNeedFullSort;
  } else if (m > 0) {
    double scale = (double)m;
    if (method == PS_ADJ_BY) scale *= numpy_pairwise_harmonic(m);
    const int64_t nb = ps_ceil_div(m, 1024);
    double* ranked = nullptr;
    double* bm = nullptr;
    PS_CUDA(ps_alloc(&ranked, (size_t)m, s));
    PS_CUDA(ps_alloc(&bm, (size_t)nb, s));
    rank_scale_pos_kernel<<<(unsigned)nb, 1024, 0, s>>>(keys, pos[cur], m, scale, ranked, bm);
    PS_LAUNCHED();
    block_suffix_min_kernel<<<1, kSuffixThreads, 0, s>>>(bm, nb);
    PS_LAUNCHED();
    bh_scatter_pos_kernel<<<(unsigned)nb, 1024, 0, s>>>(ranked, bm, pos[cur], idx, m, cols, symmetric, out);
    PS_LAUNCHED();
    ps_free(ranked, s);
    ps_free(bm, s);
  }
  for (int k = 0; k < 2; ++k) {
    ps_free(dk[k], s);
    ps_free(pos[k], s);
  }
  ps_free(tile_hist, s);
  ps_free(totals, s);
  ps_free(d_flag, s);
  ps_free(runs, s);
  return rc;
}

int adjust_core(uint64_t* keys, uint32_t* idx, unsigned long long* d_count, int64_t cols,
                int symmetric, int method, double* out, cudaStream_t s, int64_t fam_max) {
  ps_device_state* ds = ps_state();
  if (method == PS_ADJ_BONFERRONI) {  // m is read on the device: no host round trip
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ps_ceil_div(fam_max, 256), (int64_t)ds->num_sms * 8));
    bonferroni_kernel<<<blocks, 256, 0, s>>>(keys, idx, d_count, cols, symmetric, out);
    PS_LAUNCHED();
    return PS_OK;
  }
  if (method == PS_ADJ_BH && fam_max <= kSmallMax && !getenv("PS_ADJUST_SMALL_CTA")) {
    const int64_t nch = std::max<int64_t>(1, ps_ceil_div(fam_max, kChunk));
    uint64_t* skeys = nullptr;
    uint32_t *crank = nullptr, *sidx = nullptr;
    double* sval = nullptr;
    PS_CUDA(ps_alloc(&skeys, (size_t)(nch * kChunk), s));
    PS_CUDA(ps_alloc(&crank, (size_t)(nch * kChunk), s));
    PS_CUDA(ps_alloc(&sidx, (size_t)(nch * kChunk), s));
    PS_CUDA(ps_alloc(&sval, (size_t)(nch * kChunk), s));
    bh_chunk_sort_kernel<<<(unsigned)nch, kChunkThreads, 0, s>>>(keys, d_count, skeys, crank, nullptr);
    PS_LAUNCHED();
    const size_t smem = (size_t)nch * kChunk * sizeof(uint64_t);
    PS_CUDA(cudaFuncSetAttribute(bh_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bh_rank_kernel<<<(unsigned)std::max<int64_t>(1, ps_ceil_div(fam_max, 1024)), 1024, smem, s>>>(
        keys, idx, d_count, skeys, crank, sval, sidx);
    PS_LAUNCHED();
    bh_stepup_sorted_kernel<<<1, kStepThreads, 0, s>>>(sval, sidx, d_count, cols, symmetric, out);
    PS_LAUNCHED();
    ps_free(skeys, s);
    ps_free(crank, s);
    ps_free(sidx, s);
    ps_free(sval, s);
    return PS_OK;
  }
  if (method == PS_ADJ_BH && fam_max > kSmallMax && fam_max <= kMergeMax && !getenv("PS_ADJUST_RADIX")) {
    const int64_t nch = ps_ceil_div(fam_max, kChunk);
    const int64_t npad = nch * kChunk;
    uint64_t *kb[2] = {nullptr, nullptr};
    uint32_t *pb[2] = {nullptr, nullptr};
    double *ranked = nullptr, *bmin = nullptr;
    for (int b = 0; b < 2; ++b) {
      PS_CUDA(ps_alloc(&kb[b], (size_t)npad, s));
      PS_CUDA(ps_alloc(&pb[b], (size_t)npad, s));
    }
    PS_CUDA(ps_alloc(&ranked, (size_t)npad, s));
    PS_CUDA(ps_alloc(&bmin, (size_t)ps_ceil_div(npad, 1024), s));
    bh_chunk_sort_kernel<<<(unsigned)nch, kChunkThreads, 0, s>>>(keys, d_count, kb[0], nullptr, pb[0]);
    PS_LAUNCHED();
    int cur = 0;
    const unsigned g256 = (unsigned)ps_ceil_div(fam_max, 256);
    for (int64_t L = kChunk; L < fam_max; L <<= 1) {
      bh_merge_level_kernel<<<g256, 256, 0, s>>>(kb[cur], pb[cur], kb[cur ^ 1], pb[cur ^ 1], d_count, L);
      PS_LAUNCHED();
      cur ^= 1;
    }
    bh_sorted_scale_kernel<<<(unsigned)ps_ceil_div(fam_max, 1024), 1024, 0, s>>>(kb[cur], d_count, ranked, bmin);
    PS_LAUNCHED();
    bh_block_suffix_kernel<<<1, 1024, 0, s>>>(bmin, d_count);
    PS_LAUNCHED();
    bh_sorted_scatter_kernel<<<g256, 256, 0, s>>>(ranked, bmin, pb[cur], idx, d_count, cols, symmetric, out);
    PS_LAUNCHED();
    for (int b = 0; b < 2; ++b) {
      ps_free(kb[b], s);
      ps_free(pb[b], s);
    }
    ps_free(ranked, s);
    ps_free(bmin, s);
    return PS_OK;
  }
  if (method == PS_ADJ_BH && fam_max <= kSmallMax) {  // PS_ADJUST_SMALL_CTA: the single-CTA radix sort (A/B)
    const size_t smem = (size_t)kSmallMax * 6;
    PS_CUDA(cudaFuncSetAttribute(adjust_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    adjust_small_kernel<<<1, kSmallThreads, smem, s>>>(keys, idx, d_count, 1.0, cols, symmetric, out);
    PS_LAUNCHED();
    return PS_OK;
  }
  if (fam_max <= kFastMax && !getenv("PS_ADJUST_FULLSORT")) {
    int rc = adjust_fast(keys, idx, d_count, cols, symmetric, method, out, s, fam_max);
    if (rc != kNeedFullSort) return rc;
  }
  unsigned long long m_host = 0;
  PS_CUDA(cudaMemcpyAsync(&m_host, d_count, sizeof(m_host), cudaMemcpyDeviceToHost, s));
  PS_CUDA(cudaStreamSynchronize(s));
  const int64_t m = (int64_t)m_host;
  if (m == 0) return PS_OK;
  if (method == PS_ADJ_BONFERRONI) {
    const int blocks = (int)std::min<int64_t>(ps_ceil_div(m, 256), (int64_t)ds->num_sms * 8);
    bonferroni_kernel<<<blocks, 256, 0, s>>>(keys, idx, d_count, cols, symmetric, out);
    PS_LAUNCHED();
    return PS_OK;
  }
  // digit histograms -> which passes are non-trivial
  unsigned long long* d_hist = nullptr;
  PS_CUDA(ps_alloc(&d_hist, 8 * kBuckets, s));
  PS_CUDA(cudaMemsetAsync(d_hist, 0, 8 * kBuckets * sizeof(unsigned long long), s));
  {
    const int blocks = (int)std::min<int64_t>(ps_ceil_div(m, 256), (int64_t)ds->num_sms * 4);
    digit_hist_all_kernel<<<blocks, 256, 0, s>>>(keys, d_count, d_hist);
    PS_LAUNCHED();
  }
  std::vector<unsigned long long> hist(8 * kBuckets);
  PS_CUDA(cudaMemcpyAsync(hist.data(), d_hist, hist.size() * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, s));
  PS_CUDA(cudaStreamSynchronize(s));
  ps_free(d_hist, s);

  uint64_t* k2 = nullptr;
  uint32_t* v2 = nullptr;
  const int64_t ntiles = ps_ceil_div(m, kTile);
  uint32_t* tile_hist = nullptr;
  PS_CUDA(ps_alloc(&k2, (size_t)m, s));
  PS_CUDA(ps_alloc(&v2, (size_t)m, s));
  PS_CUDA(ps_alloc(&tile_hist, (size_t)(ntiles * kBuckets), s));
  uint64_t* kin = keys;
  uint32_t* vin = idx;
  uint64_t* kout = k2;
  uint32_t* vout = v2;
  for (int pass = 0; pass < 8; ++pass) {
    bool trivial = false;
    for (int d = 0; d < kBuckets; ++d)
      if (hist[pass * kBuckets + d] == (unsigned long long)m) trivial = true;
    if (trivial) continue;
    const int shift = pass * kRadixBits;
    tile_hist_kernel<<<(unsigned)ntiles, kSortThreads, 0, s>>>(kin, m, shift, tile_hist, ntiles);
    PS_LAUNCHED();
    int rc = scan_u32(tile_hist, ntiles * kBuckets, s);
    if (rc) return rc;
    scatter_kernel<<<(unsigned)ntiles, kSortThreads, 0, s>>>(kin, vin, kout, vout, m, shift, tile_hist,
                                                             ntiles);
    PS_LAUNCHED();
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  double scale = (double)m;
  if (method == PS_ADJ_BY) scale *= numpy_pairwise_harmonic(m);
  const int64_t nb = ps_ceil_div(m, 1024);
  double* ranked = nullptr;
  double* bm = nullptr;
  PS_CUDA(ps_alloc(&ranked, (size_t)m, s));
  PS_CUDA(ps_alloc(&bm, (size_t)nb, s));
  rank_scale_kernel<<<(unsigned)nb, 1024, 0, s>>>(kin, m, scale, ranked, bm);
  PS_LAUNCHED();
  block_suffix_min_kernel<<<1, kSuffixThreads, 0, s>>>(bm, nb);
  PS_LAUNCHED();
  bh_scatter_kernel<<<(unsigned)nb, 1024, 0, s>>>(ranked, bm, vin, m, cols, symmetric, out);
  PS_LAUNCHED();
  ps_free(ranked, s);
  ps_free(bm, s);
  ps_free(k2, s);
  ps_free(v2, s);
  ps_free(tile_hist, s);
  return PS_OK;
}

}  // namespace

int ps_adjust_run(const double* p, int64_t rows, int64_t cols, int method, int symmetric, double* out,
                  cudaStream_t s) {
  if (method < 0 || method > 2) return ps_fail(PS_ERR_UNKNOWN_METHOD, "unknown adjustment method");
  if (symmetric && rows != cols)
    return ps_fail(PS_ERR_NON_SQUARE, "symmetric adjustment needs a square matrix");
  const int64_t n = rows * cols;
  if (n >= (int64_t)UINT32_MAX) return ps_fail(PS_ERR_INVALID, "family larger than 2^32 cells");
  int rc = ps_fill_nan(out, n, s);
  if (rc) return rc;
  if (n == 0) return PS_OK;
  ps_device_state* ds = ps_state();
  const int64_t fam = symmetric ? rows * (rows - 1) / 2 : n;
  if (fam == 0) return PS_OK;
  uint64_t* keys = nullptr;
  uint32_t* idx = nullptr;
  unsigned long long* d_count = nullptr;
  PS_CUDA(ps_alloc(&keys, (size_t)fam, s));
  PS_CUDA(ps_alloc(&idx, (size_t)fam, s));
  PS_CUDA(ps_alloc(&d_count, 1, s));
  PS_CUDA(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  const int blocks = (int)std::min<int64_t>(ps_ceil_div(n, 256), (int64_t)ds->num_sms * 8);
  extract_kernel<<<blocks, 256, 0, s>>>(p, rows, cols, symmetric, keys, idx, d_count);
  PS_LAUNCHED();
  rc = adjust_core(keys, idx, d_count, cols, symmetric, method, out, s, fam);
  ps_free(keys, s);
  ps_free(idx, s);
  ps_free(d_count, s);
  return rc;
}

int ps_adjust_family_run(const double* p, int64_t n, int method, double* out, cudaStream_t s) {
  if (method < 0 || method > 2) return ps_fail(PS_ERR_UNKNOWN_METHOD, "unknown adjustment method");
  if (n >= (int64_t)UINT32_MAX) return ps_fail(PS_ERR_INVALID, "family larger than 2^32 cells");
  int rc = ps_fill_nan(out, n, s);
  if (rc || n == 0) return rc;
  ps_device_state* ds = ps_state();
  uint64_t* keys = nullptr;
  uint32_t* idx = nullptr;
  unsigned long long* d_count = nullptr;
  PS_CUDA(ps_alloc(&keys, (size_t)n, s));
  PS_CUDA(ps_alloc(&idx, (size_t)n, s));
  PS_CUDA(ps_alloc(&d_count, 1, s));
  PS_CUDA(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  const int blocks = (int)std::min<int64_t>(ps_ceil_div(n, 256), (int64_t)ds->num_sms * 8);
  extract_vec_kernel<<<blocks, 256, 0, s>>>(p, n, keys, idx, d_count);
  PS_LAUNCHED();
  rc = adjust_core(keys, idx, d_count, n, 0, method, out, s, n);
  ps_free(keys, s);
  ps_free(idx, s);
  ps_free(d_count, s);
  return rc;
}

extern "C" double ps_by_factor(int64_t m) { return numpy_pairwise_harmonic(m); }
