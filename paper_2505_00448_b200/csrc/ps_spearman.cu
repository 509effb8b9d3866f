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
//           sample -- as floor(r) (uint16) plus a parity bit.
//   pass B  walks h's order q = 0..n_h-1 SEQUENTIALLY: keep = (R[q] != 0),
//           h's joint rank follows from the same prefix identity, and the
//           products accumulate.  R is cleared on the way.
//
// All sums are exact integers: 4 sxx = sum (2r_g)^2 - n (n+1)^2, likewise syy,
// and 4 sxy = sum (2r_g)(2r_h) - n (n+1)^2 (rank totals are preserved by tie
// averaging).  The reference's fp64 sums of quarter-integers are exact as
// well, so rho = sxy / sqrt(sxx syy) is bit-identical; p = 2 t_sf(|t|, n-2)
// is evaluated by a separate one-thread-per-pair epilogue kernel.
//
// One persistent CTA per h (largest h first, dynamic queue); all warps
// cooperate on one pair at a time.  Shared memory per CTA: inv_h (2S B),
// R (2S B), parity + ballot words + word prefixes (~S/2.7 B).
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include <algorithm>

namespace {

constexpr int SW = 16;            // warps per CTA
constexpr int STH = SW * 32;
constexpr int IMAX = 32;          // register stash of pass-A gathers (positions per thread)

struct PairSums {
  long long* n;    // F x F (only g <= h written)
  long long* sxx4;
  long long* syy4;
  long long* sxy4;
};

__device__ __forceinline__ uint32_t pfx_at(const uint32_t* K, const uint32_t* P, uint32_t x) {
  const uint32_t w = x >> 5, b = x & 31u;
  return P[w] + __popc(K[w] & ((1u << b) - 1u));
}

// exclusive block scan over word popcounts: P[w] = kept positions before word w
__device__ void scan_words(uint32_t* K, uint32_t* P, int nwords, uint32_t* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (nwords + STH - 1) / STH;
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
    uint32_t v = lane < SW ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(PS_FULL, v, o);
      if (lane >= o) v += y;
    }
    if (lane < SW) wsum[lane] = v;
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
    P[nwords] = wsum[SW - 1];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(STH)
spearman_walk_kernel(const uint32_t* __restrict__ order, const uint16_t* __restrict__ inv,
                     const uint32_t* __restrict__ gsa, const uint32_t* __restrict__ gea,
                     const uint8_t* __restrict__ tied, const int32_t* __restrict__ lens, int64_t S,
                     int64_t F, int64_t lo, int64_t hi, int* __restrict__ queue, PairSums out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t Sp = ps_round_up(S, 64);
  const int WK = (int)(Sp / 32) + 2;
  uint16_t* inv_s = reinterpret_cast<uint16_t*>(smem);
  uint16_t* R = inv_s + Sp;
  uint32_t* par = reinterpret_cast<uint32_t*>(R + Sp);
  uint32_t* K = par + WK;
  uint32_t* P = K + WK;
  __shared__ uint32_t wsum[SW];
  __shared__ unsigned long long red[SW][3];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int64_t i = threadIdx.x; i < Sp; i += STH) R[i] = 0;
  for (int i = threadIdx.x; i < WK; i += STH) par[i] = 0u;

  const int64_t nh_items = F - lo;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= nh_items) break;
    const int64_t h = F - 1 - item;  // largest rows of work first
    const int nh = lens[h];
    const bool th = tied[h] != 0;
    const uint32_t* gh_s = gsa + h * S;
    const uint32_t* gh_e = gea + h * S;
    {
      const uint16_t* src = inv + h * S;
      for (int64_t i = threadIdx.x; i < S; i += STH) inv_s[i] = src[i];
    }
    __syncthreads();
    const int64_t gmax = std::min<int64_t>(h, hi - 1);
    for (int64_t g = lo; g <= gmax; ++g) {
      const int ng = lens[g];
      const bool tg = tied[g] != 0;
      const uint32_t* og = order + g * S;
      const uint32_t* gg_s = gsa + g * S;
      const uint32_t* gg_e = gea + g * S;
      // ---------------- pass A, phase 1: keep bits over g's order ----------
      const int nwa = (ng + 31) >> 5;
      uint32_t stash[IMAX / 2];
#pragma unroll
      for (int i = 0; i < IMAX; ++i) {
        const int word = warp + SW * i;
        uint32_t q = 0xFFFFu;
        if (word < nwa) {
          const int p = word * 32 + lane;
          if (p < ng) q = inv_s[og[p]];
          const uint32_t B = __ballot_sync(PS_FULL, q != 0xFFFFu);
          if (lane == 0) K[word] = B;
        }
        if (i & 1) stash[i >> 1] |= q << 16;
        else stash[i >> 1] = q;
      }
      for (int word = warp + SW * IMAX; word < nwa; word += SW) {
        const int p = word * 32 + lane;
        uint32_t q = 0xFFFFu;
        if (p < ng) q = inv_s[og[p]];
        const uint32_t B = __ballot_sync(PS_FULL, q != 0xFFFFu);
        if (lane == 0) K[word] = B;
      }
      __syncthreads();
      scan_words(K, P, nwa, wsum);
      const uint32_t n = P[nwa];
      // ---------------- pass A, phase 2: ranks -> R[q] ----------------------
      unsigned long long sa2 = 0;
      auto place = [&](int word, uint32_t q) {
        const int p = word * 32 + lane;
        const bool keep = q != 0xFFFFu;
        uint32_t r2;
        if (!tg) {
          r2 = 2u * (P[word] + __popc(K[word] & lanemask_lt()) + 1u);
        } else {
          r2 = 0;
          if (keep) r2 = pfx_at(K, P, gg_s[p]) + pfx_at(K, P, gg_e[p]) + 1u;
        }
        if (keep) {
          R[q] = (uint16_t)(r2 >> 1);
          if (r2 & 1u) atomicOr(&par[q >> 5], 1u << (q & 31u));
          sa2 += (unsigned long long)r2 * r2;
        }
      };
#pragma unroll
      for (int i = 0; i < IMAX; ++i) {
        const int word = warp + SW * i;
        if (word < nwa) {
          const uint32_t q = (i & 1) ? (stash[i >> 1] >> 16) : (stash[i >> 1] & 0xFFFFu);
          place(word, q);
        }
      }
      for (int word = warp + SW * IMAX; word < nwa; word += SW) {
        const int p = word * 32 + lane;
        const uint32_t q = p < ng ? (uint32_t)inv_s[og[p]] : 0xFFFFu;
        place(word, q);
      }
      __syncthreads();
      // ---------------- pass B, phase 1: keep bits over h's order -----------
      const int nwb = (nh + 31) >> 5;
      for (int word = warp; word < nwb; word += SW) {
        const int q = word * 32 + lane;
        const bool keep = q < nh && R[q] != 0;
        const uint32_t B = __ballot_sync(PS_FULL, keep);
        if (lane == 0) K[word] = B;
      }
      __syncthreads();
      scan_words(K, P, nwb, wsum);
      // ---------------- pass B, phase 2: accumulate, clear R ----------------
      unsigned long long sab = 0, sbb = 0;
      for (int word = warp; word < nwb; word += SW) {
        const int q = word * 32 + lane;
        const uint32_t v = q < nh ? R[q] : 0u;
        const bool keep = v != 0;
        const uint32_t pw = tg ? par[word] : 0u;
        if (keep) {
          const uint32_t r2g = 2u * v + ((pw >> lane) & 1u);
          uint32_t r2h;
          if (!th) r2h = 2u * (P[word] + __popc(K[word] & lanemask_lt()) + 1u);
          else r2h = pfx_at(K, P, gh_s[q]) + pfx_at(K, P, gh_e[q]) + 1u;
          sab += (unsigned long long)r2g * r2h;
          sbb += (unsigned long long)r2h * r2h;
          R[q] = 0;
        }
        __syncwarp();
        if (tg && lane == 0) par[word] = 0u;
      }
      // ---------------- reduce and store the exact sums ---------------------
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sa2 += __shfl_xor_sync(PS_FULL, sa2, o);
        sab += __shfl_xor_sync(PS_FULL, sab, o);
        sbb += __shfl_xor_sync(PS_FULL, sbb, o);
      }
      if (lane == 0) {
        red[warp][0] = sa2;
        red[warp][1] = sab;
        red[warp][2] = sbb;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0, c = 0;
        for (int w = 0; w < SW; ++w) {
          a += red[w][0];
          b += red[w][1];
          c += red[w][2];
        }
        const long long nn = (long long)n;
        const long long base = nn * (nn + 1) * (nn + 1);
        const int64_t cell = g * F + h;
        out.n[cell] = nn;
        out.sxx4[cell] = (long long)a - base;
        out.syy4[cell] = (long long)c - base;
        out.sxy4[cell] = (long long)b - base;
      }
    }
  }
}

__device__ __forceinline__ void put(double* o, int64_t F, int64_t g, int64_t h, double v) {
  if (o) {
    o[g * F + h] = v;
    o[h * F + g] = v;
  }
}

// rho / p from the exact sums (continuous.py:174-203), one thread per pair.
__global__ void spearman_finish_kernel(PairSums in, int64_t F, int64_t lo, int64_t hi,
                                       double* __restrict__ stat, double* __restrict__ pout,
                                       double* __restrict__ rho_out, int* __restrict__ err) {
  const int64_t total = (hi - lo) * F;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = lo + it / F, h = it % F;
    if (h < g) continue;
    const int64_t cell = g * F + h;
    const long long n = in.n[cell];
    double rho = PS_NAN, p = PS_NAN;
    if (n > 1) {
      // exact quarter-integers, identical to the reference's fp64 sums
      const double sxx = (double)in.sxx4[cell] * 0.25;
      const double syy = (double)in.syy4[cell] * 0.25;
      const double sxy = (double)in.sxy4[cell] * 0.25;
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
    put(stat, F, g, h, rho);
    put(pout, F, g, h, p);
    put(rho_out, F, g, h, rho);
  }
}

}  // namespace

int ps_spearman_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho,
                    cudaStream_t s) {
  const int64_t F = a->F, S = a->S;
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(F, hi);
  if (hi <= lo || (!stat && !p && !rho)) return PS_OK;
  if (!a->has_presort) {
    int rc = ps_presort_matrix(a, s);
    if (rc) return rc;
  }
  ps_device_state* ds = ps_state();
  const int64_t Sp = ps_round_up(S, 64);
  const int64_t WK = Sp / 32 + 2;
  const size_t smem = (size_t)(2 * Sp * sizeof(uint16_t) + 3 * WK * sizeof(uint32_t));
  if (smem > 220 * 1024)
    return ps_fail(PS_ERR_INVALID, "spearman: sample count too large for the shared-memory walk");
  PS_CUDA(cudaFuncSetAttribute(spearman_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  int per_sm = 0;
  PS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spearman_walk_kernel, STH, smem));
  per_sm = std::max(1, per_sm);
  const int64_t items = F - lo;
  const int grid = (int)std::min<int64_t>(items, (int64_t)ds->num_sms * per_sm);

  PairSums ps{};
  int* queue = nullptr;
  PS_CUDA(ps_alloc(&ps.n, (size_t)(F * F), s));
  PS_CUDA(ps_alloc(&ps.sxx4, (size_t)(F * F), s));
  PS_CUDA(ps_alloc(&ps.syy4, (size_t)(F * F), s));
  PS_CUDA(ps_alloc(&ps.sxy4, (size_t)(F * F), s));
  PS_CUDA(ps_alloc(&queue, 1, s));
  PS_CUDA(cudaMemsetAsync(queue, 0, sizeof(int), s));
  ps_prof_begin("spearman_walk", s);
  spearman_walk_kernel<<<grid, STH, smem, s>>>(a->d_order, a->d_inv, a->d_gs, a->d_ge, a->d_tied,
                                              a->d_len, S, F, lo, hi, queue, ps);
  ps_prof_end(s);
  PS_LAUNCHED();
  const int64_t total = (hi - lo) * F;
  const int blocks = (int)std::min<int64_t>(ps_ceil_div(total, 128), (int64_t)ds->num_sms * 16);
  spearman_finish_kernel<<<blocks, 128, 0, s>>>(ps, F, lo, hi, stat, p, rho, ds->d_err);
  PS_LAUNCHED();
  ps_free(ps.n, s);
  ps_free(ps.sxx4, s);
  ps_free(ps.syy4, s);
  ps_free(ps.sxy4, s);
  ps_free(queue, s);
  return PS_OK;
}
