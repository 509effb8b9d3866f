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
#include <algorithm>

namespace {

constexpr int SW = 16;            // warps per CTA
constexpr int STH = SW * 32;

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

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}

// sum_{k=1..n} (2k)^2: the rank-square total of a tie-free walk
__device__ __forceinline__ unsigned long long sq_closed(unsigned long long n) {
  return 4ull * (n * (n + 1) * (2 * n + 1) / 6ull);
}

template <bool OGS>
__global__ void __launch_bounds__(STH)
spearman_walk_kernel(const uint16_t* __restrict__ order, const uint16_t* __restrict__ inv, int64_t ldo,
                     const uint32_t* __restrict__ tb, const uint16_t* __restrict__ lastb,
                     const uint16_t* __restrict__ nextb, int64_t ldt, const uint8_t* __restrict__ tied,
                     const int32_t* __restrict__ lens, int64_t F, int64_t lo, int64_t hi,
                     int* __restrict__ queue, PairSums out) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* cur = smem;
  auto take = [&](size_t bytes) {
    unsigned char* p = cur;
    cur += (bytes + 15) & ~size_t(15);
    return p;
  };
  uint16_t* inv_s = reinterpret_cast<uint16_t*>(take(ldo * 2));
  uint16_t* R = reinterpret_cast<uint16_t*>(take(ldo * 2));
  uint32_t* tbh = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint16_t* lbh = reinterpret_cast<uint16_t*>(take(ldt * 2));
  uint16_t* nbh = reinterpret_cast<uint16_t*>(take(ldt * 2));
  uint32_t* par = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint32_t* K = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint32_t* P = reinterpret_cast<uint32_t*>(take(ldt * 4));
  uint32_t* Kb = reinterpret_cast<uint32_t*>(take(ldt * 4));  // pass-B keep bits, set by pass A
  uint16_t* og_s[2] = {nullptr, nullptr};
  uint32_t* tbg_s[2] = {nullptr, nullptr};
  uint16_t* lbg_s[2] = {nullptr, nullptr};
  uint16_t* nbg_s[2] = {nullptr, nullptr};
  if (OGS) {
    for (int b = 0; b < 2; ++b) {
      og_s[b] = reinterpret_cast<uint16_t*>(take(ldo * 2));
      tbg_s[b] = reinterpret_cast<uint32_t*>(take(ldt * 4));
      lbg_s[b] = reinterpret_cast<uint16_t*>(take(ldt * 2));
      nbg_s[b] = reinterpret_cast<uint16_t*>(take(ldt * 2));
    }
  }
  __shared__ uint32_t wsum[SW];
  __shared__ unsigned long long red[SW][3];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int64_t i = threadIdx.x; i < ldo; i += STH) R[i] = 0;
  for (int64_t i = threadIdx.x; i < ldt; i += STH) {
    par[i] = 0u;
    Kb[i] = 0u;
  }

  // stage g's order (+ tie tables when tied) into buffer b
  auto prefetch = [&](int64_t g, int b) {
    const int ng = lens[g];
    const int nch = (ng * 2 + 15) / 16;
    const uint32_t so = (uint32_t)__cvta_generic_to_shared(og_s[b]);
    const unsigned char* src = reinterpret_cast<const unsigned char*>(order + g * ldo);
    for (int c = threadIdx.x; c < nch; c += STH) cp16(so + c * 16, src + c * 16);
    if (tied[g]) {
      const int tch4 = (int)(ldt * 4 / 16), tch2 = (int)(ldt * 2 / 16);
      const unsigned char* t4 = reinterpret_cast<const unsigned char*>(tb + g * ldt);
      const unsigned char* l2 = reinterpret_cast<const unsigned char*>(lastb + g * ldt);
      const unsigned char* n2 = reinterpret_cast<const unsigned char*>(nextb + g * ldt);
      const uint32_t st4 = (uint32_t)__cvta_generic_to_shared(tbg_s[b]);
      const uint32_t sl2 = (uint32_t)__cvta_generic_to_shared(lbg_s[b]);
      const uint32_t sn2 = (uint32_t)__cvta_generic_to_shared(nbg_s[b]);
      for (int c = threadIdx.x; c < tch4; c += STH) cp16(st4 + c * 16, t4 + c * 16);
      for (int c = threadIdx.x; c < tch2; c += STH) {
        cp16(sl2 + c * 16, l2 + c * 16);
        cp16(sn2 + c * 16, n2 + c * 16);
      }
    }
    asm volatile("cp.async.commit_group;");
  };

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
    {
      const uint4* src = reinterpret_cast<const uint4*>(inv + h * ldo);
      uint4* dst = reinterpret_cast<uint4*>(inv_s);
      for (int64_t i = threadIdx.x; i < ldo / 8; i += STH) dst[i] = src[i];
      if (th) {
        for (int64_t i = threadIdx.x; i < ldt; i += STH) {
          tbh[i] = tb[h * ldt + i];
          lbh[i] = lastb[h * ldt + i];
          nbh[i] = nextb[h * ldt + i];
        }
      }
    }
    const int64_t gmax = std::min<int64_t>(h, hi - 1);
    if (OGS && lo <= gmax) prefetch(lo, 0);
    __syncthreads();
    for (int64_t g = lo; g <= gmax; ++g) {
      const int buf = (int)((g - lo) & 1);
      const int ng = lens[g];
      const bool tg = tied[g] != 0;
      const uint16_t* og;
      const uint32_t* tbg;
      const uint16_t *lbg, *nbg;
      if (OGS) {
        if (g + 1 <= gmax) prefetch(g + 1, buf ^ 1);
        else asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 1;");
        __syncthreads();
        og = og_s[buf];
        tbg = tbg_s[buf];
        lbg = lbg_s[buf];
        nbg = nbg_s[buf];
      } else {
        og = order + g * ldo;
        tbg = tb + g * ldt;
        lbg = lastb + g * ldt;
        nbg = nextb + g * ldt;
      }
      // ---------------- pass A, phase 1: keep bits over g's order ----------
      const int nwa = (ng + 31) >> 5;
#pragma unroll 4
      for (int word = warp; word < nwa; word += SW) {
        const int p = word * 32 + lane;
        const uint32_t q = p < ng ? (uint32_t)inv_s[og[p]] : 0xFFFFu;
        const uint32_t B = __ballot_sync(PS_FULL, q != 0xFFFFu);
        if (lane == 0) K[word] = B;
      }
      __syncthreads();
      scan_words(K, P, nwa, wsum);
      const uint32_t n = P[nwa];
      // ---------------- pass A, phase 2: ranks -> R[q], keep bits of B ------
      unsigned long long sa2 = 0;
      if (!tg) {
        // tie-free: 2r = 2 (Pfx(p) + 1), always even
#pragma unroll 4
        for (int word = warp; word < nwa; word += SW) {
          const int p = word * 32 + lane;
          const uint32_t kw = K[word];
          if ((kw >> lane) & 1u) {
            const uint32_t q = inv_s[og[p]];
            R[q] = (uint16_t)(P[word] + __popc(kw & lanemask_lt()) + 1u);
            atomicOr(&Kb[q >> 5], 1u << (q & 31u));
          }
        }
      } else {
        for (int word = warp; word < nwa; word += SW) {
          const uint32_t p = (uint32_t)(word * 32 + lane);
          const uint32_t kw = K[word];
          if ((kw >> lane) & 1u) {
            const uint32_t q = inv_s[og[p]];
            const uint32_t r2 =
                pfx_at(K, P, tie_start(tbg, lbg, p)) + pfx_at(K, P, tie_end(tbg, nbg, p)) + 1u;
            sa2 += (unsigned long long)r2 * r2;
            R[q] = (uint16_t)(r2 >> 1);
            atomicOr(&Kb[q >> 5], 1u << (q & 31u));
            if (r2 & 1u) atomicOr(&par[q >> 5], 1u << (q & 31u));
          }
        }
      }
      __syncthreads();
      // ---------------- pass B: h's order, keep bits already set by pass A ---
      const int nwb = (nh + 31) >> 5;
      scan_words(Kb, P, nwb, wsum);
      unsigned long long sab = 0, sbb = 0;
      if (!th) {
#pragma unroll 4
        for (int word = warp; word < nwb; word += SW) {
          const uint32_t kw = Kb[word];
          const uint32_t q = (uint32_t)(word * 32 + lane);
          const uint32_t r2g = 2u * (uint32_t)R[q] + (tg ? ((par[word] >> lane) & 1u) : 0u);
          const uint32_t r2h = 2u * (P[word] + __popc(kw & lanemask_lt()) + 1u);
          if ((kw >> lane) & 1u) sab += (unsigned long long)r2g * r2h;
        }
      } else {
        for (int word = warp; word < nwb; word += SW) {
          const uint32_t kw = Kb[word];
          const uint32_t q = (uint32_t)(word * 32 + lane);
          if ((kw >> lane) & 1u) {
            const uint32_t r2g = 2u * (uint32_t)R[q] + (tg ? ((par[word] >> lane) & 1u) : 0u);
            const uint32_t r2h =
                pfx_at(Kb, P, tie_start(tbh, lbh, q)) + pfx_at(Kb, P, tie_end(tbh, nbh, q)) + 1u;
            sbb += (unsigned long long)r2h * r2h;
            sab += (unsigned long long)r2g * r2h;
          }
        }
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
      for (int w = threadIdx.x; w < nwb; w += STH) {
        Kb[w] = 0u;
        if (tg) par[w] = 0u;
      }
      if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0, c = 0;
        for (int w = 0; w < SW; ++w) {
          a += red[w][0];
          b += red[w][1];
          c += red[w][2];
        }
        const unsigned long long un = n;
        if (!tg) a = sq_closed(un);
        if (!th) c = sq_closed(un);
        const long long nn = (long long)n;
        const long long base = nn * (nn + 1) * (nn + 1);
        const int64_t cell = g * F + h;
        out.n[cell] = nn;
        out.sxx4[cell] = (long long)a - base;
        out.syy4[cell] = (long long)c - base;
        out.sxy4[cell] = (long long)b - base;
      }
    }
    if (OGS) asm volatile("cp.async.wait_group 0;");
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

size_t walk_smem(int64_t ldo, int64_t ldt, bool ogs) {
  auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  size_t b = 2 * r16(ldo * 2) + r16(ldt * 4) + 2 * r16(ldt * 2) + 4 * r16(ldt * 4);
  if (ogs) b += 2 * (r16(ldo * 2) + r16(ldt * 4) + 2 * r16(ldt * 2));
  return b;
}

}  // namespace

int ps_spearman_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho,
                    cudaStream_t s) {
  const int64_t F = a->F;
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(F, hi);
  if (hi <= lo || (!stat && !p && !rho)) return PS_OK;
  if (!a->has_presort) {
    int rc = ps_presort_matrix(a, s);
    if (rc) return rc;
  }
  ps_device_state* ds = ps_state();
  const size_t limit = 227 * 1024 - 1024;
  size_t smem = walk_smem(a->ldo, a->ldt, true);
  const bool ogs = smem <= limit;
  if (!ogs) smem = walk_smem(a->ldo, a->ldt, false);
  if (smem > limit)
    return ps_fail(PS_ERR_INVALID, "spearman: sample count too large for the shared-memory walk");
  auto kern = ogs ? spearman_walk_kernel<true> : spearman_walk_kernel<false>;
  PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, STH, smem));
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
  kern<<<grid, STH, smem, s>>>(a->d_order, a->d_inv, a->ldo, a->d_tb, a->d_lastb, a->d_nextb, a->ldt,
                               a->d_tied, a->d_len, F, lo, hi, queue, ps);
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
