// ps_rankmixed.cu -- Kruskal-Wallis and Mann-Whitney U: label-filtered rank
// walks over one presort of each continuous feature.
//
// Replaces _kruskal_block -> _kruskal_rows -> _kruskal_finish and _mwu_block ->
// _mwu_rows -> _mwu_finish (engine.py:296-352; mixed.py:231-247, :305-403,
// :550-623).  The reference walks continuous feature h's sorted order,
// compacting the samples whose label is present, and averages ranks over tied
// runs.  Here one persistent CTA owns h (its 16-bit order and tie tables stay
// in shared memory) and walks it once per label row g:
//
//   phase 1  keep bits over h's order: keep(p) = label_g[order_h[p]] present
//            (ballot per 32 positions) + a block scan of word popcounts;
//   phase 2  joint rank 2r = Pfx(gs) + Pfx(ge) + 1 of every kept position,
//            accumulated per level in registers (exact integer rank sums and
//            counts) plus the tie term sum(t^3 - t) over kept tie groups.
//
// g's label row (one byte per sample) is double-buffered in shared memory and
// prefetched with cp.async during the previous pair.  Per-pair exact sums go
// to a buffer; a one-thread-per-pair epilogue replays _kruskal_finish /
// _mwu_finish in the reference's fp64 op order (H, U, r bit-identical), and a
// cold-path kernel builds the exact U distribution (Gaussian-binomial
// coefficients, the same integers as mixed.py:231-247) when the exact test
// applies.  Out-of-range labels of kept samples raise LabelOutOfRange.
//
// Algorithmic work: ~12 B of shared-memory traffic per pair-sample.
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include "ps_ties.cuh"
#include "ps_wide.cuh"
#include <math_constants.h>
#include <algorithm>

namespace {

constexpr int RW = 16;  // warps per CTA
constexpr int RTH = RW * 32;

struct RankSums {
  int KM;                       // levels stored per pair
  int32_t* cnt;                 // [pair][KM]
  unsigned long long* r2;       // [pair][KM] sums of 2r
  long long* tie;               // [pair] sum over tie groups of t^3 - t
};

__device__ __forceinline__ uint32_t pfx_at(const uint32_t* K, const uint32_t* P, uint32_t x) {
  const uint32_t w = x >> 5, b = x & 31u;
  return P[w] + __popc(K[w] & ((1u << b) - 1u));
}

__device__ void scan_words(uint32_t* K, uint32_t* P, int nwords, uint32_t* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (nwords + RTH - 1) / RTH;
  const int w0 = threadIdx.x * per;
  uint32_t local = 0;
  for (int i = 0; i < per; ++i) {
    const int w = w0 + i;
    if (w < nwords) local += __popc(K[w]);
  }
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < RW ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(PS_FULL, v, o);
      if (lane >= o) v += y;
    }
    if (lane < RW) wsum[lane] = v;
  }
  __syncthreads();
  uint32_t run = (warp > 0 ? wsum[warp - 1] : 0u) + x - local;
  for (int i = 0; i < per; ++i) {
    const int w = w0 + i;
    if (w < nwords) {
      P[w] = run;
      run += __popc(K[w]);
    }
  }
  if (threadIdx.x == 0) {
    K[nwords] = 0u;
    P[nwords] = wsum[RW - 1];
  }
  __syncthreads();
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}

// Codes: 0..k-1 valid level, 0xFE present but out of range, 0xFF missing.
template <int KM>
__global__ void __launch_bounds__(RTH, 2)
rank_mixed_walk_kernel(const uint16_t* __restrict__ order, int64_t ldo, const uint32_t* __restrict__ tb,
                       const uint16_t* __restrict__ lastb, const uint16_t* __restrict__ nextb, int64_t ldt,
                       const uint8_t* __restrict__ tied, const int32_t* __restrict__ lens,
                       const uint8_t* __restrict__ codes, int64_t ldc, const int32_t* __restrict__ cat,
                       int64_t Fc, int64_t Fq, int64_t lo, int64_t hi, int gb, int once, int check_labels,
                       int* __restrict__ queue, RankSums out, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* cur = smem;
  auto take = [&](size_t bytes) {
    unsigned char* p = cur;
    cur += (bytes + 15) & ~size_t(15);
    return p;
  };
  uint16_t* oh = reinterpret_cast<uint16_t*>(take(ldo * 2));
  uint32_t* tbh = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint16_t* lbh = reinterpret_cast<uint16_t*>(take(ldt * 2));
  uint16_t* nbh = reinterpret_cast<uint16_t*>(take(ldt * 2));
  uint32_t* K = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint32_t* P = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint8_t* cg_s[2];
  cg_s[0] = take(ldc);
  cg_s[1] = take(ldc);
  // KM == 8: the tie-free sweep accumulates per (warp, level, lane) in shared
  // memory (bank = lane: conflict-free) -- one LDS/IADD/STS per kept position
  // instead of a KM-way select chain in registers
  constexpr bool SMACC = KM == 8;
  uint32_t* accs = reinterpret_cast<uint32_t*>(take(SMACC ? (size_t)RW * KM * 32 * 4 : 0));
  const uint32_t aAcc = (uint32_t)__cvta_generic_to_shared(accs) + 4u * (uint32_t)(((threadIdx.x >> 5) * KM) * 32 + (threadIdx.x & 31));
  // byte offsets into the dynamic buffer: indexing `smem[...]` directly keeps
  // the gathers in the shared window (LDS), never generic loads
  const uint32_t cg_off[2] = {(uint32_t)(cg_s[0] - smem), (uint32_t)(cg_s[1] - smem)};
  const uint32_t oh_off = (uint32_t)(reinterpret_cast<unsigned char*>(oh) - smem) / 2;
  const uint16_t* smem16 = reinterpret_cast<const uint16_t*>(smem);
  __shared__ uint32_t wsum[RW];
  // KM <= 16: per-lane register accumulators reduced by shuffles; KM = 256:
  // per-warp shared accumulators (shared atomics) for labels with many levels
  constexpr bool BIG = KM > 16;
  constexpr int NR = BIG ? 1 : KM;
  __shared__ unsigned long long red_r[RW][NR];
  __shared__ uint32_t red_c[RW][NR];
  __shared__ uint32_t bsum[BIG ? RW : 1][BIG ? 256 : 1];
  __shared__ uint32_t bcnt[BIG ? RW : 1][BIG ? 256 : 1];
  __shared__ long long red_t[RW];
  __shared__ uint32_t wtot_s[RW];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  auto prefetch = [&](int64_t g, int b) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(cg_s[b]);
    const unsigned char* src = codes + g * ldc;
    for (int64_t c = threadIdx.x; c < ldc / 16; c += RTH) cp16(dst + c * 16, src + c * 16);
    asm volatile("cp.async.commit_group;");
  };

  if constexpr (SMACC)
    for (int i = threadIdx.x; i < RW * KM * 32; i += RTH) accs[i] = 0u;
  // items: (feature h, block of gb label rows), h-major
  const int64_t nblk = (Fc + gb - 1) / gb;
  const int64_t items = (hi - lo) * nblk;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= items) break;
    const int64_t h = lo + item / nblk;
    const int64_t g0 = (item % nblk) * gb, g1 = g0 + gb < Fc ? g0 + gb : Fc;
    const int nh = lens[h];
    const bool th = tied[h] != 0;
    {
      const uint4* src = reinterpret_cast<const uint4*>(order + h * ldo);
      uint4* dst = reinterpret_cast<uint4*>(oh);
      for (int64_t i = threadIdx.x; i < ldo / 8; i += RTH) dst[i] = src[i];
      if (th) {
        for (int64_t i = threadIdx.x; i < ldt; i += RTH) {
          tbh[i] = tb[h * ldt + i];
          lbh[i] = lastb[h * ldt + i];
          nbh[i] = nextb[h * ldt + i];
        }
      }
    }
    prefetch(g0, 0);
    const int nw = (nh + 31) >> 5;
    for (int64_t g = g0; g < g1; ++g) {
      const int buf = (int)((g - g0) & 1);
      if (g + 1 < g1) prefetch(g + 1, buf ^ 1);
      else asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 1;");
      __syncthreads();
      const uint32_t cgo = cg_off[buf];
      const int k = cat[g];
      uint32_t acc[NR], cnt[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = cnt[j] = 0u;
      if constexpr (BIG) {
        for (int j = lane; j < k; j += 32) {
          bsum[warp][j] = 0u;
          bcnt[warp][j] = 0u;
        }
        __syncwarp();
      }
      long long tie = 0;
      if (!th) {
        // Tie-free h: ONE sweep over a contiguous segment per warp.  Ranks are
        // segment-local (running kept count); per level we keep sum(local)
        // and the count, and fold in the segment base after the reduction:
        //   sum 2r = 2 (base_w * count + sum local).
        const int L = (nw + RW - 1) / RW;
        const int w0 = min(nw, warp * L), w1 = min(nw, w0 + L);
        uint32_t run = 0;
        // per lane and level: count in bits [20,32), sum of local ranks in [0,20)
        // (a lane sees <= 128 positions of rank <= 4096 for S <= 65535)
#pragma unroll 4
        for (int word = w0; word < w1; ++word) {
          const uint32_t c = smem[cgo + smem16[oh_off + word * 32 + lane]];  // sentinel padded: 0xFF
          const bool keep = c != 0xFFu;
          const uint32_t B = __ballot_sync(PS_FULL, keep);
          const uint32_t local = run + __popc(B & lanemask_lt()) + 1u;
          if constexpr (BIG) {
            if (c < (uint32_t)k) {
              atomicAdd(&bsum[warp][c], local);
              atomicAdd(&bcnt[warp][c], 1u);
            }
          } else if constexpr (SMACC) {
            if (keep && c < (uint32_t)KM) {  // slot (warp, c, lane): bank = lane
              const uint32_t a = aAcc + (c << 7);
              uint32_t v;
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v + (1u << 20) + local));
            }
          } else {
            const uint32_t packed = (1u << 20) + local;
#pragma unroll
            for (int j = 0; j < KM; ++j) acc[j] += c == (uint32_t)j ? packed : 0u;  // select, not a branch
          }
          run += __popc(B);
        }
        if constexpr (SMACC) {
#pragma unroll
          for (int j = 0; j < KM; ++j) {
            uint32_t& slot = accs[(warp * KM + j) * 32 + lane];
            acc[j] = slot;
            slot = 0u;
          }
        }
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          cnt[j] = acc[j] >> 20;
          acc[j] &= 0xFFFFFu;
        }
        if (lane == 0) wtot_s[warp] = run;
      } else {
      // -------- phase 1: keep bits (label present) over h's order --------
#pragma unroll 4
      for (int word = warp; word < nw; word += RW) {
        const int p = word * 32 + lane;
        const uint32_t c = p < nh ? (uint32_t)smem[cgo + smem16[oh_off + p]] : 0xFFu;
        const uint32_t B = __ballot_sync(PS_FULL, c != 0xFFu);
        if (lane == 0) K[word] = B;
      }
      __syncthreads();
      scan_words(K, P, nw, wsum);
      // -------- phase 2: ranks, per-level sums, tie term --------
        for (int word = warp; word < nw; word += RW) {
          const uint32_t p = (uint32_t)(word * 32 + lane);
          const uint32_t kw = K[word];
          // prefixes of the tie groups entering / leaving the word (uniform),
          // then per-lane group bounds from the word's boundary bits
          const uint32_t T = tbh[word], Pw = P[word];
          const uint32_t sp = (T & 1u) ? Pw : pfx_at(K, P, lbh[word ? word - 1 : 0]);
          const uint32_t ep = pfx_at(K, P, min((uint32_t)nbh[word + 1], (uint32_t)nh));
          uint32_t a, b;
          word_group_pfx(T, sp, ep, kw, Pw, a, b);
          if (p < (uint32_t)nh) {
            if ((T >> lane) & 1u) {  // the group's first position owns its tie term
              const long long t = (long long)(b - a);
              if (t > 1) tie += t * t * t - t;
            }
            if ((kw >> lane) & 1u) {
              const uint32_t c = smem[cgo + smem16[oh_off + p]];
              const uint32_t r2 = a + b + 1u;
              if constexpr (BIG) {
                if (c < (uint32_t)k) {
                  atomicAdd(&bsum[warp][c], r2);
                  atomicAdd(&bcnt[warp][c], 1u);
                }
              } else {
#pragma unroll
                for (int j = 0; j < KM; ++j) {
                  const bool hit = c == (uint32_t)j;
                  acc[j] += hit ? r2 : 0u;
                  cnt[j] += hit ? 1u : 0u;
                }
              }
            }
          }
        }
      }
      // -------- reduce to the pair's exact sums --------
#pragma unroll
      for (int j = 0; j < (BIG ? 0 : NR); ++j) {
        if (j >= k && j != 0) continue;  // (uniform) levels past this label row's count
        // per lane: sum of local ranks < 2^20 (tie-free sweep) or of 2r < 2^24
        // (tied walk), so the warp sums fit 32 bits: integer warp reduce
        const uint32_t a = __reduce_add_sync(PS_FULL, acc[j]);
        const uint32_t c = __reduce_add_sync(PS_FULL, cnt[j]);
        if (lane == 0) {
          red_r[warp][j] = a;
          red_c[warp][j] = c;
        }
      }
      {
        // sum of t^3 - t (< 2^54): three 22-bit slices
        const unsigned long long x = (unsigned long long)tie;
        const uint32_t t0 = __reduce_add_sync(PS_FULL, (uint32_t)(x & 0x3FFFFFu));
        const uint32_t t1 = __reduce_add_sync(PS_FULL, (uint32_t)((x >> 22) & 0x3FFFFFu));
        const uint32_t t2 = __reduce_add_sync(PS_FULL, (uint32_t)(x >> 44));
        if (lane == 0)
          red_t[warp] = (long long)((unsigned long long)t0 + ((unsigned long long)t1 << 22) +
                                    ((unsigned long long)t2 << 44));
      }
      __syncthreads();
      const int64_t pair = g * Fq + h;
      if constexpr (BIG) {
        for (int j = threadIdx.x; j < max(k, 1); j += RTH) {
          unsigned long long a = 0;
          uint32_t c = 0;
          unsigned long long base = 0;
          for (int w = 0; w < RW; ++w) {
            a += th ? (unsigned long long)bsum[w][j] : 2ull * ((unsigned long long)bsum[w][j] + base * bcnt[w][j]);
            c += bcnt[w][j];
            base += wtot_s[w];
          }
          out.r2[pair * out.KM + j] = a;
          out.cnt[pair * out.KM + j] = (int32_t)c;
        }
        if (threadIdx.x == 0) {
          long long t = 0;
          for (int w = 0; w < RW; ++w) t += red_t[w];
          out.tie[pair] = t;
        }
      } else if (threadIdx.x < KM) {
        const int j = threadIdx.x;
        unsigned long long a = 0;
        uint32_t c = 0;
        if (!th) {
          unsigned long long base = 0;
          for (int w = 0; w < RW; ++w) {
            a += 2ull * (red_r[w][j] + base * red_c[w][j]);
            c += red_c[w][j];
            base += wtot_s[w];
          }
        } else {
          for (int w = 0; w < RW; ++w) {
            a += red_r[w][j];
            c += red_c[w][j];
          }
        }
        if (j < k || j == 0) {
          out.r2[pair * out.KM + j] = a;
          out.cnt[pair * out.KM + j] = (int32_t)c;
        }
      } else if (threadIdx.x == 32) {
        long long t = 0;
        for (int w = 0; w < RW; ++w) t += red_t[w];
        out.tie[pair] = t;
      }
    }
    asm volatile("cp.async.wait_group 0;");
    if (once) break;  // one item per CTA: retiring CTAs let higher-priority kernels in
  }
}

__device__ __forceinline__ void kruskal_finish(const RankSums& in, int64_t pair, int k, double* h_out,
                                               double* p_out, double* eta_out, int* err) {
  *h_out = *p_out = *eta_out = PS_NAN;
  long long n = 0;
  for (int j = 0; j < k; ++j) {
    const long long c = in.cnt[pair * in.KM + j];
    if (c == 0) return;
    n += c;
  }
  if (n < 2) return;
  const double fn = (double)n;
  const double tie = (double)in.tie[pair];
  const double tden = 1.0 - tie / (fn * fn * fn - fn);
  if (tden <= 0.0) return;
  double h = 0.0;
  for (int j = 0; j < k; ++j) {
    const double rs = (double)in.r2[pair * in.KM + j] * 0.5;  // exact half-integers
    h += rs * rs / (double)in.cnt[pair * in.KM + j];
  }
  h = (12.0 / (fn * (fn + 1.0))) * h - 3.0 * (fn + 1.0);
  h /= tden;
  if (h < 0.0) h = 0.0;
  *h_out = h;
  if (k < 2) return;
  *p_out = psf::chi2_sf(h, (double)k - 1.0, err);
  if (n <= k) return;
  *eta_out = (h - (double)k + 1.0) / (double)(n - k);
}

// mixed.py:305-363; returns 1 when the exact distribution is needed
__device__ __forceinline__ int mwu_finish(long long n0, long long n1, double r0, double tie, int mode,
                                          double* u_out, double* p_out, double* r_out, int* err) {
  *u_out = *p_out = *r_out = PS_NAN;
  if (n0 == 0 || n1 == 0) return 0;
  const long long n = n0 + n1;
  const double u = r0 - 0.5 * (double)n0 * (double)(n0 + 1);
  const double mu = 0.5 * (double)n0 * (double)n1;
  const double diff = u - mu;
  bool use_exact = false;
  if (mode == PS_U_EXACT) {
    if (tie != 0.0) { ps_raise(err, PS_ERR_EXACT_WITH_TIES); return 0; }
    if (n > 64) { ps_raise(err, PS_ERR_TABLE_TOO_LARGE); return 0; }
    use_exact = true;
  } else if (mode == PS_U_AUTO) {
    use_exact = tie == 0.0 && (n0 < n1 ? n0 : n1) < 8 && n <= 64;
  }
  const double sigma_sq = ((double)(n0 * n1) / 12.0) * (((double)n + 1.0) - tie / ((double)n * ((double)n - 1.0)));
  *u_out = u;
  if (sigma_sq <= 0.0) return 0;
  double z = (fabs(diff) - 0.5) / sqrt(sigma_sq);
  if (z < 0.0) z = 0.0;
  double r;
  if (z == 0.0 || diff == 0.0) r = 0.0;
  else if (diff > 0.0) r = z / sqrt((double)n);
  else r = -z / sqrt((double)n);
  *r_out = r;
  if (use_exact) return 1;
  double p = 2.0 * psf::normal_sf(z);
  if (p > 1.0) p = 1.0;
  *p_out = p;
  return 0;
}

__device__ __forceinline__ void put_cell(double* o, int64_t idx, double v) {
  if (o) o[idx] = v;
}

__global__ void rank_mixed_finish_kernel(int test, RankSums in, const int32_t* __restrict__ cat, int64_t Fc,
                                         int64_t Fq, int64_t lo, int64_t hi, int mode, double* __restrict__ stat,
                                         double* __restrict__ pout, double* __restrict__ eff,
                                         int2* __restrict__ exact_list, int* __restrict__ exact_count,
                                         int exact_cap, int* __restrict__ err) {
  const int64_t total = Fc * (hi - lo);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = it / (hi - lo), h = lo + it % (hi - lo);
    const int64_t pair = g * Fq + h;
    double a, b, c;
    if (test == PS_TEST_KRUSKAL) {
      kruskal_finish(in, pair, cat[g], &a, &b, &c, err);
    } else {
      const long long n0 = in.cnt[pair * in.KM + 0];
      const long long n1 = in.cnt[pair * in.KM + 1];
      const double r0 = (double)in.r2[pair * in.KM + 0] * 0.5;
      if (mwu_finish(n0, n1, r0, (double)in.tie[pair], mode, &a, &b, &c, err)) {
        const int slot = atomicAdd(exact_count, 1);
        if (slot < exact_cap) exact_list[slot] = make_int2((int)g, (int)h);
      }
    }
    put_cell(stat, pair, a);
    put_cell(pout, pair, b);
    put_cell(eff, pair, c);
  }
}

// Cold path: exact two-sided U p-value (mixed.py:348-358).  The arrangement
// counts f(n0, n1, u) are the coefficients of the Gaussian binomial
// [n0+n1 choose n0]_q, built by P <- P (1 - q^(n1+i)) / (1 - q^i); every step
// is an exact int64 polynomial, identical to the reference's DP table row.
//
// The finish kernel lists the cells that need it; when the list overflowed
// (more exact cells than its capacity -- e.g. u_mode='exact' on a wide matrix
// with S <= 64) every cell of the range is re-decided here with the same
// predicate, so no exact p is ever dropped.
__global__ void mwu_exact_kernel(RankSums in, int64_t Fc, int64_t Fq, int64_t lo, int64_t hi, int mode,
                                 const int2* __restrict__ list, const int* __restrict__ count_ptr, int cap,
                                 double* __restrict__ pout) {
  __shared__ long long poly[1152];  // degree <= a (b + 1) <= 32 * 33 during the product
  const int count = *count_ptr;
  const bool all_cells = count > cap;
  const int64_t n_items = all_cells ? Fc * (hi - lo) : count;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    int64_t g, h;
    if (all_cells) {
      g = it / (hi - lo);
      h = lo + it % (hi - lo);
    } else {
      g = list[it].x;
      h = list[it].y;
    }
    const int64_t pair = g * Fq + h;
    const long long n0 = in.cnt[pair * in.KM + 0];
    const long long n1 = in.cnt[pair * in.KM + 1];
    const double r0 = (double)in.r2[pair * in.KM + 0] * 0.5;
    if (all_cells) {  // block-uniform decision (every thread reads the same cell)
      double a_, b_, c_;
      if (!mwu_finish(n0, n1, r0, (double)in.tie[pair], mode, &a_, &b_, &c_, nullptr)) continue;
    }
    const int a = (int)(n0 < n1 ? n0 : n1), bb = (int)(n0 < n1 ? n1 : n0);
    const int umax = (int)(n0 * n1);
    if (threadIdx.x == 0) {
      for (int u = 0; u <= a * (bb + 1); ++u) poly[u] = 0;
      poly[0] = 1;
      int deg = 0;
      for (int i = 1; i <= a; ++i) {
        const int m = bb + i;
        // multiply by (1 - q^m)
        for (int u = deg + m; u >= m; --u) poly[u] -= (u - m <= deg) ? poly[u - m] : 0;
        deg += m;
        // divide by (1 - q^i): exact
        for (int u = i; u <= deg; ++u) poly[u] += poly[u - i];
        deg -= i;
      }
      const double u = r0 - 0.5 * (double)n0 * (double)(n0 + 1);
      const double lowv = u < (double)umax - u ? u : (double)umax - u;
      const long long ulow = (long long)rint(lowv);
      long long cum = 0, total = 0;
      for (int v = 0; v <= umax; ++v) {
        total += poly[v];
        if (v <= ulow) cum += poly[v];
      }
      double p = 2.0 * (double)cum / (double)total;
      if (p > 1.0) p = 1.0;
      pout[pair] = p;
    }
    __syncthreads();
  }
}

// MWU grouping codes from the dichotomous label bits: 0 if the label is 0.0,
// 1 if present and non-zero (mixed.py:381), 0xFF if missing.
__global__ void binary_codes_kernel(const uint32_t* __restrict__ mask, const uint32_t* __restrict__ zero,
                                    int64_t W, int64_t S, int64_t ldc, uint8_t* __restrict__ out) {
  const int64_t f = blockIdx.x;
  for (int64_t s = threadIdx.x; s < ldc; s += blockDim.x) {
    uint8_t c = 0xFF;
    if (s < S) {
      const uint32_t m = mask[f * W + (s >> 5)], z = zero[f * W + (s >> 5)];
      const uint32_t bit = 1u << (s & 31);
      if (m & bit) c = (z & bit) ? 0 : 1;
    }
    out[f * ldc + s] = c;
  }
}

// Wide walk (S beyond the shared-memory walk; ps_wide.cuh): one CTA per
// (label row g, continuous feature h) pair from an atomic queue, g fastest.
// Walk h's order keeping the samples whose label is present, then add each
// kept position's doubled rank 2r = Pfx(gs) + Pfx(ge) + 1 to its level
// (per-warp shared accumulators) and sum(t^3 - t) over the tie groups of the
// kept samples -- the same exact sums the shared-memory walk produces
// (mixed.py:366-403, :581-623), finished by rank_mixed_finish_kernel.
// CT: uint8_t codes, or uint16_t (category counts above 254).  GACC: the
// level accumulators are the pair's global RankSums entries (global atomics;
// level counts too large for per-warp shared accumulators).
template <typename OT, typename CT, bool GACC>
__global__ void __launch_bounds__(wide::WT, 1)
rank_mixed_wide_kernel(const OT* __restrict__ order, int64_t ldo, const uint32_t* __restrict__ tb,
                       const OT* __restrict__ lastb, const OT* __restrict__ nextb, int64_t ldt,
                       const int32_t* __restrict__ len, const CT* __restrict__ codes, int64_t ldc,
                       const uint32_t* __restrict__ lmask, int64_t lW, int64_t Fc, int64_t Fq, int64_t lo, int64_t hi,
                       uint32_t* __restrict__ scratch, int64_t scr, int* __restrict__ queue, RankSums rs,
                       int* __restrict__ err) {
  extern __shared__ unsigned long long wacc[];  // [WW][KM] r2 sums, then [WW][KM] counts (u32)
  __shared__ uint32_t sbuf[wide::WW];
  __shared__ unsigned long long ubuf[wide::WW];
  __shared__ long long s_item;
  const int KM = rs.KM;
  unsigned int* wcnt = reinterpret_cast<unsigned int*>(wacc + wide::WW * KM);
  const int warp = threadIdx.x >> 5;
  const int64_t kw = ldo / 32 + 2;
  uint32_t* K = scratch + blockIdx.x * scr;
  uint32_t* P = K + kw;
  const int64_t total = (hi - lo) * Fc;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    if (!GACC)
      for (int i = threadIdx.x; i < wide::WW * KM; i += wide::WT) {
        wacc[i] = 0ull;
        wcnt[i] = 0u;
      }
    __syncthreads();
    const int64_t t = s_item;
    if (t >= total) break;
    const int64_t h = lo + t / Fc, g = t % Fc;
    const OT* oh = order + h * ldo;
    const uint32_t* tbh = tb + h * ldt;
    const CT* cg = codes + g * ldc;
    const int64_t pair = g * Fq + h;
    const uint32_t nh = (uint32_t)len[h];
    wide::keep_scan(oh, nh, lmask + g * lW, K, P, sbuf);
    long long tie = 0;
    for (uint32_t q = threadIdx.x; q < nh; q += wide::WT) {
      const uint32_t te = wide::tie_end(tbh, nextb + h * ldt, q);
      if ((tbh[q >> 5] >> (q & 31u)) & 1u) {  // q starts a tie group: its kept count
        const long long c = (long long)(wide::pfx(K, P, te) - wide::pfx(K, P, q));
        tie += c * c * c - c;
      }
      if (!((K[q >> 5] >> (q & 31u)) & 1u)) continue;
      const uint32_t r2 = wide::pfx(K, P, wide::tie_start(tbh, lastb + h * ldt, q)) + wide::pfx(K, P, te) + 1u;
      const uint32_t lv = cg[(uint32_t)oh[q]];
      if (lv >= (uint32_t)KM) {
        ps_raise(err, PS_ERR_LABEL_OUT_OF_RANGE);
        continue;
      }
      if (GACC) {
        atomicAdd(&rs.r2[pair * KM + lv], (unsigned long long)r2);
        atomicAdd(&rs.cnt[pair * KM + lv], 1);
      } else {
        atomicAdd(&wacc[warp * KM + lv], (unsigned long long)r2);
        atomicAdd(&wcnt[warp * KM + lv], 1u);
      }
    }
    const unsigned long long tsum = wide::block_sum_u64((unsigned long long)tie, ubuf);  // ends with a barrier
    for (int j = threadIdx.x; !GACC && j < KM; j += wide::WT) {
      unsigned long long r = 0;
      unsigned int c = 0;
      for (int w = 0; w < wide::WW; ++w) {
        r += wacc[w * KM + j];
        c += wcnt[w * KM + j];
      }
      rs.r2[pair * KM + j] = r;
      rs.cnt[pair * KM + j] = (int32_t)c;
    }
    if (threadIdx.x == 0) rs.tie[pair] = (long long)tsum;
    __syncthreads();
  }
}

template <typename OT, typename CT, bool GACC>
int launch_wide_walk_t(ps_matrix* lab, ps_matrix* val, const OT* order, const OT* lastb, const OT* nextb,
                       const CT* codes, int64_t lo, int64_t hi, RankSums rs, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  const int grid = ds->num_sms;
  const int64_t scr = 2 * (val->ldo / 32 + 2);
  const size_t smem = GACC ? 0 : (size_t)wide::WW * rs.KM * (8 + 4);
  uint32_t* scratch = nullptr;
  int* queue = nullptr;
  PS_CUDA(ps_alloc(&scratch, (size_t)(grid * scr), s));
  PS_CUDA(ps_alloc(&queue, 1, s));
  PS_CUDA(cudaMemsetAsync(queue, 0, sizeof(int), s));
  auto kern = rank_mixed_wide_kernel<OT, CT, GACC>;
  PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ps_prof_begin("rank_mixed_walk", s);
  kern<<<grid, wide::WT, smem, s>>>(order, val->ldo, val->d_tb, lastb, nextb, val->ldt, val->d_len, codes, lab->ldc,
                                    lab->d_mask, lab->W, lab->F, val->F, lo, hi, scratch, scr, queue, rs, ds->d_err);
  ps_prof_end(s);
  PS_LAUNCHED();
  ps_free(scratch, s);
  ps_free(queue, s);
  return PS_OK;
}

// the wide walk for any presort width / code width / level count
template <typename OT>
int launch_wide_walk(ps_matrix* lab, ps_matrix* val, const OT* order, const OT* lastb, const OT* nextb,
                     const uint8_t* codes, int64_t lo, int64_t hi, RankSums rs, cudaStream_t s) {
  const bool gacc = rs.KM > 256;  // per-warp shared accumulators: 32 warps x KM x 12 B
  if (lab->code_bytes == 2 && codes == lab->d_codes) {
    const uint16_t* c16 = reinterpret_cast<const uint16_t*>(codes);
    return gacc ? launch_wide_walk_t<OT, uint16_t, true>(lab, val, order, lastb, nextb, c16, lo, hi, rs, s)
                : launch_wide_walk_t<OT, uint16_t, false>(lab, val, order, lastb, nextb, c16, lo, hi, rs, s);
  }
  return gacc ? launch_wide_walk_t<OT, uint8_t, true>(lab, val, order, lastb, nextb, codes, lo, hi, rs, s)
              : launch_wide_walk_t<OT, uint8_t, false>(lab, val, order, lastb, nextb, codes, lo, hi, rs, s);
}

size_t walk_smem(int64_t ldo, int64_t ldt, int64_t ldc, int KM) {
  auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  return r16(ldo * 2) + r16(ldt * 4) + 2 * r16(ldt * 2) + 2 * r16(ldt * 4) + 2 * r16(ldc) +
         (KM == 8 ? (size_t)RW * KM * 32 * 4 : 0);
}

template <int KM>
int launch_walk(ps_matrix* lab, ps_matrix* val, const uint8_t* codes, int64_t lo, int64_t hi, int gb, int once,
                int check, int* queue, RankSums rs, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  const size_t smem = walk_smem(val->ldo, val->ldt, lab->ldc, KM);
  auto kern = rank_mixed_walk_kernel<KM>;
  cudaFuncAttributes fa{};
  PS_CUDA(cudaFuncGetAttributes(&fa, kern));
  if (val->wide) return launch_wide_walk<uint32_t>(lab, val, val->d_order32, val->d_lastb32, val->d_nextb32, codes, lo,
                                                   hi, rs, s);
  if ((lab->code_bytes == 2 && codes == lab->d_codes) || rs.KM > 256)  // more than 254 levels: the wide walk
    return launch_wide_walk<uint16_t>(lab, val, val->d_order, val->d_lastb, val->d_nextb, codes, lo, hi, rs, s);
  if (smem + fa.sharedSizeBytes > 227 * 1024)  // tables beyond shared memory: the wide walk
    return launch_wide_walk<uint16_t>(lab, val, val->d_order, val->d_lastb, val->d_nextb, codes, lo, hi, rs, s);
  PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RTH, smem));
  per_sm = std::max(1, per_sm);
  const int64_t items = (hi - lo) * ps_ceil_div(lab->F, gb);
  const int grid = once ? (int)items : (int)std::min<int64_t>(items, (int64_t)ds->num_sms * per_sm);
  ps_prof_begin("rank_mixed_walk", s);
  kern<<<grid, RTH, smem, s>>>(val->d_order, val->ldo, val->d_tb, val->d_lastb, val->d_nextb, val->ldt,
                               val->d_tied, val->d_len, codes, lab->ldc, lab->d_cat, lab->F, val->F, lo, hi,
                               gb, once, check, queue, rs, ds->d_err);
  ps_prof_end(s);
  PS_LAUNCHED();
  return PS_OK;
}

}  // namespace

constexpr int kIncrementalRows = 32;

struct ps_rank_job {
  int test = 0, u_mode = 0, KM = 2;
  bool kw = false;
  ps_matrix* lab = nullptr;
  ps_matrix* val = nullptr;
  int64_t lo = 0, hi = 0, h_done = 0;
  RankSums rs{2, nullptr, nullptr, nullptr};
  uint8_t* bcodes = nullptr;
  const uint8_t* codes = nullptr;
  int* queues = nullptr;
  int qn = 256, qi = 0, nws = 0;
  int2* exl = nullptr;
  int* exc = nullptr;
  int excap = 0;
  cudaStream_t home = nullptr;
};

static void rank_job_free(ps_rank_job* j, cudaStream_t s) {
  ps_free(j->rs.cnt, s);
  ps_free(j->rs.r2, s);
  ps_free(j->rs.tie, s);
  ps_free(j->queues, s);
  ps_free(j->exl, s);
  ps_free(j->exc, s);
  ps_free(j->bcodes, s);
  delete j;
}

// label check + walk of the continuous features [h0, h1); work items are
// (feature, gb label rows)
static int rank_walk_range(ps_rank_job* j, int64_t h0, int64_t h1, int gb, int once, cudaStream_t s) {
  if (h1 <= h0) return PS_OK;
  if (j->qi >= j->qn) {
    PS_CUDA(cudaMemsetAsync(j->queues, 0, sizeof(int) * j->qn, s));
    j->qi = 0;
  }
  int* q = j->queues + j->qi++;
  // LabelOutOfRange: a present out-of-range label meeting a present value
  // (mixed.py:613-617) -- checked up front, so the walk never tracks it
  int rc = j->kw ? ps_mixed_label_check(j->lab, j->val, 0, j->lab->F, h0, h1, s) : PS_OK;
  if (rc) return rc;
  const int KM = j->KM;
  if (KM == 2) return launch_walk<2>(j->lab, j->val, j->codes, h0, h1, gb, once, j->kw, q, j->rs, s);
  if (KM == 8) return launch_walk<8>(j->lab, j->val, j->codes, h0, h1, gb, once, j->kw, q, j->rs, s);
  if (KM == 16) return launch_walk<16>(j->lab, j->val, j->codes, h0, h1, gb, once, j->kw, q, j->rs, s);
  return launch_walk<256>(j->lab, j->val, j->codes, h0, h1, gb, once, j->kw, q, j->rs, s);
}

int ps_rank_mixed_begin(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int u_mode, cudaStream_t s,
                        ps_rank_job** out) {
  *out = nullptr;
  const int64_t Fc = lab->F, Fq = val->F;
  if (lab->S != val->S) return ps_fail(PS_ERR_INVALID, "sample counts differ");
  ps_rank_job* j = new ps_rank_job();
  j->test = test;
  j->u_mode = u_mode;
  j->lab = lab;
  j->val = val;
  j->lo = std::max<int64_t>(0, lo);
  j->hi = std::min<int64_t>(Fq, hi);
  j->h_done = j->lo;
  j->home = s;
  j->kw = test == PS_TEST_KRUSKAL;
  const int kmax = j->kw ? std::max(1, lab->cmax) : 2;
  int KM = kmax <= 2 ? 2 : kmax <= 8 ? 8 : kmax <= 16 ? 16 : 256;
  // the KM = 8 variant keeps per-lane accumulators in shared memory; when they
  // do not fit next to the walk's tables, use the register variant
  if (KM == 8 && walk_smem(val->ldo, val->ldt, lab->ldc, 8) > 222 * 1024) KM = 16;
  j->KM = KM;
  const int64_t npairs = Fc * Fq;
  // per-pair level stride: the template width, or the real level count for k > 16
  j->rs = RankSums{KM > 16 ? (kmax + 31) / 32 * 32 : KM, nullptr, nullptr, nullptr};
  // exact-U cell list (cold path); PS_EXACT_CAP shrinks it so the tests can
  // exercise the overflow re-scan of mwu_exact_kernel
  int64_t cap_lim = 1 << 20;
  if (const char* e = getenv("PS_EXACT_CAP")) cap_lim = std::max(1L, atol(e));
  j->excap = (int)std::min<int64_t>(Fc * std::max<int64_t>(1, j->hi - j->lo), cap_lim);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { e = x; return x == cudaSuccess; };
  if (ok(ps_alloc(&j->rs.cnt, (size_t)(npairs * j->rs.KM), s)) && ok(ps_alloc(&j->rs.r2, (size_t)(npairs * j->rs.KM), s)) &&
      ok(ps_alloc(&j->rs.tie, (size_t)npairs, s)) && ok(ps_alloc(&j->queues, (size_t)j->qn, s)) &&
      ok(ps_alloc(&j->exl, (size_t)j->excap, s)) && ok(ps_alloc(&j->exc, 1, s)) &&
      ok(cudaMemsetAsync(j->queues, 0, sizeof(int) * j->qn, s)) && ok(cudaMemsetAsync(j->exc, 0, sizeof(int), s)) &&
      ok(cudaMemsetAsync(j->rs.cnt, 0, sizeof(int32_t) * npairs * j->rs.KM, s)) &&
      ok(cudaMemsetAsync(j->rs.r2, 0, sizeof(unsigned long long) * npairs * j->rs.KM, s))) {
    j->codes = lab->d_codes;
    if (!j->kw && ok(ps_alloc(&j->bcodes, (size_t)(Fc * lab->ldc), s))) {
      binary_codes_kernel<<<(unsigned)Fc, 256, 0, s>>>(lab->d_mask, lab->d_zero, lab->W, lab->S, lab->ldc, j->bcodes);
      e = cudaGetLastError();
      ps_count_launch();
      j->codes = j->bcodes;
    }
  }
  if (e != cudaSuccess) {
    rank_job_free(j, s);
    return ps_cuda_check(e, "rank test setup");
  }
  *out = j;
  return PS_OK;
}

// Incremental walks (ps_run: features of each uploaded chunk), alternating
// between the two walk streams; each item is one feature, so a launch's CTAs
// retire one by one and the next chunk's presort (higher-priority stream)
// and walk fill the SMs.
int ps_rank_mixed_walk_upto(ps_rank_job* j, int64_t h1, cudaStream_t s) {
  h1 = std::min<int64_t>(h1, j->hi);
  if (h1 <= j->h_done) return PS_OK;
  ps_device_state* ds = ps_state();
  cudaStream_t w = ps_walk_stream(j->nws++, s);
  // label-row blocks keep items short, so SMs free up often for the
  // presort of the next chunk
  int gb = kIncrementalRows;
  if (const char* e = getenv("PS_RANK_GB")) gb = std::max(1, atoi(e));
  int rc = rank_walk_range(j, j->h_done, h1, gb, h1 < j->hi, w);
  j->h_done = h1;
  return rc;
}

int ps_rank_mixed_end(ps_rank_job* j, double* stat, double* p, double* eff, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  int jr = ps_walk_streams_join(j->nws, s);
  if (jr) return jr;
  int rc = rank_walk_range(j, j->h_done, j->hi, (int)std::max<int64_t>(1, j->lab->F), 0, s);
  j->h_done = j->hi;
  const int64_t Fc = j->lab->F, Fq = j->val->F, lo = j->lo, hi = j->hi;
  if (!rc && hi > lo && (stat || p || eff)) {
    const int64_t total = Fc * (hi - lo);
    const int blocks = (int)std::min<int64_t>(ps_ceil_div(total, 128), (int64_t)ds->num_sms * 16);
    rank_mixed_finish_kernel<<<blocks, 128, 0, s>>>(j->test, j->rs, j->lab->d_cat, Fc, Fq, lo, hi, j->u_mode, stat, p,
                                                    eff, j->exl, j->exc, j->excap, ds->d_err);
    ps_count_launch();
    if (cudaGetLastError() != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "rank finish launch");
    if (!rc && !j->kw && j->u_mode != PS_U_ASYMPTOTIC && p) {
      mwu_exact_kernel<<<ds->num_sms * 8, 32, 0, s>>>(j->rs, Fc, Fq, lo, hi, j->u_mode, j->exl, j->exc, j->excap,
                                                      p);
      ps_count_launch();
      if (cudaGetLastError() != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "mwu exact launch");
    }
  }
  if (j->home != s) {  // free in the allocation stream's order
    PS_CUDA(cudaEventRecord(ds->walk_ev[ps_device_state::kWalkStreams], s));
    PS_CUDA(cudaStreamWaitEvent(j->home, ds->walk_ev[ps_device_state::kWalkStreams], 0));
  }
  rank_job_free(j, j->home);
  return rc;
}

void ps_rank_mixed_abort(ps_rank_job* j, cudaStream_t s) {
  if (!j) return;
  cudaStreamSynchronize(s);
  cudaDeviceSynchronize();
  rank_job_free(j, j->home);
}

int ps_rank_mixed_run(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int u_mode,
                      double* stat, double* p, double* eff, cudaStream_t s) {
  if (lab->S != val->S) return ps_fail(PS_ERR_INVALID, "sample counts differ");
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(val->F, hi);
  if (hi <= lo || (!stat && !p && !eff)) return PS_OK;
  if (!val->has_presort) {
    int rc = ps_presort_matrix(val, s);
    if (rc) return rc;
  }
  // the continuous matrix still presorting in chunks on the auxiliary stream:
  // walk each presorted chunk of features as it completes (the label matrix
  // must be prepared first: its ready event)
  // (Kruskal-Wallis only: the Mann-Whitney walk is short next to the presort
  // and gains nothing from starting early)
  const bool inc = test == PS_TEST_KRUSKAL && ps_presort_pending(val);
  ps_device_state* ds = ps_state();
  cudaStream_t home = inc ? ds->walk[0] : s;
  if (inc && lab->ready) PS_CUDA(cudaStreamWaitEvent(home, lab->ready, 0));
  if (inc && !lab->ready) {  // no marker: order after everything on s
    PS_CUDA(cudaEventRecord(ds->alloc_ev, s));
    PS_CUDA(cudaStreamWaitEvent(home, ds->alloc_ev, 0));
  }
  ps_rank_job* j = nullptr;
  int rc = ps_rank_mixed_begin(test, lab, val, lo, hi, u_mode, home, &j);
  if (rc) return rc;
  if (inc) {
    PS_CUDA(cudaEventRecord(ds->alloc_ev, home));
    int gb = kIncrementalRows;
    if (const char* e = getenv("PS_RANK_GB")) gb = std::max(1, atoi(e));
    for (const auto& mk : val->presort_marks) {
      const int64_t h1 = std::min<int64_t>(mk.first, j->hi);
      if (h1 <= j->h_done || rc) continue;
      cudaStream_t w = ds->walk[j->nws++ % ps_device_state::kWalkStreams];
      PS_CUDA(cudaStreamWaitEvent(w, mk.second, 0));
      PS_CUDA(cudaStreamWaitEvent(w, ds->alloc_ev, 0));
      rc = rank_walk_range(j, j->h_done, h1, gb, h1 < j->hi, w);
      j->h_done = h1;
    }
  }
  int rc2 = ps_rank_mixed_end(j, stat, p, eff, s);
  return rc ? rc : rc2;
}
