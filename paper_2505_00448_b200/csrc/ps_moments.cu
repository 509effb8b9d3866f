// ps_moments.cu -- the masked first and second moments of every feature pair
// as int8 tensor-core contractions (Pearson, large F).
//
// The Pearson moment contraction (ps_pearson.cu) needs five sums per pair
// (engine.py:145-166, continuous.py:29-103):
//     Sxy = X' X'^T,  Sx = X' M^T,  Sxx = X'^2 M^T,  Sy = Sx^T,  Syy = Sxx^T
// over x' = x - c_f (0 where missing) and the 0/1 presence M.  Only Sxy needs
// the FP64 tensor path.  The four others have a 0/1 operand, so they are
// computed EXACTLY on the int8 tensor cores (tcgen05.mma kind::i8) from a
// fixed-point digit expansion of each row:
//     x = 2^(e_f + 1) * sum_{s=1..8} d_s 2^(-7 s),   d_s in [-64, 64]
// (e_f: max |x| < 2^e_f over row f; u = rint(x 2^(55 - e_f)) split into
// balanced base-128 digits), so that
//     Sx(i, j) = 2^(e_i + 1) sum_s 2^(-7 s) (D_s M^T)(i, j),
// each D_s M^T an exact int32 contraction (|.| <= 64 S).  The digit products
// are folded into the fp64 result in a fixed order (s = 8 .. 1), so Sx and
// Sxx are bitwise identical for any launch range or device count.  The only
// approximation is the expansion itself: |x - expansion| <= 2^(e_f - 56), i.e.
// a relative error below 2^-55 of the row's largest value per term -- far
// below the FP64 summation error of the DMMA contraction it replaces.  Sxx
// uses the same expansion of the fp64 products x'^2 (the DMUL of the DMMA
// path).  The DMMA tile kernel then runs Sxy alone (one product instead of
// five) and reads the four moments in its epilogue.
//
// Algorithmic work: 8 digits x 2 moments x 2 int8 ops per (ordered) pair-sample.
#include "ps_internal.cuh"
#include "ps_tc05.cuh"
#include <cudaTypedefs.h>
#include <algorithm>

namespace {

constexpr int kDigits = kMomentDigits;
constexpr int QM = 256, QN = 256, QKB = 128;  // tile rows, cols, K bytes per stage
constexpr int QSTAGES = 3;
constexpr int QA_BYTES = QM * QKB, QB_BYTES = QN * QKB;
constexpr int QSTAGE_BYTES = QA_BYTES + QB_BYTES;
constexpr size_t kMomSmem = (size_t)QSTAGES * QSTAGE_BYTES + 1024;
constexpr int QTH = 192;  // warps 0-3 epilogue, 4 TMA producer, 5 MMA issuer
constexpr int32_t kNonFinite = 0x7FFFFFFF;

// Unit u of an (nr x nJ) grid of (row unit, column tile) in column bands of
// kBand tiles: a wave of consecutive units covers a compact block of rows x
// columns (every row unit of a band before the next band), so the operand
// slabs a wave streams stay L2-resident instead of re-reading every column
// tile per row (~3x less DRAM traffic per launch).
constexpr int kBand = 8;
__device__ __forceinline__ void band_unit(int64_t u, int64_t nr, int64_t nJ, int64_t& r, int64_t& J) {
  const int64_t full = (nJ / kBand) * nr * kBand;
  if (u < full) {
    const int64_t b = u / (nr * kBand), rem = u % (nr * kBand);
    r = rem / kBand;
    J = b * kBand + rem % kBand;
  } else {
    const int64_t w = nJ % kBand, rem = u - full;
    r = rem / w;
    J = (nJ / kBand) * kBand + rem % w;
  }
}  // row exponent of a row holding NaN / inf: its moments are NaN

// per-row exponents: max |x'| < 2^e1, max x'^2 < 2^e2 (frexp; 0 for an all-zero row)
__global__ void moment_scale_kernel(const double* __restrict__ xc, int64_t ld, int64_t S, int64_t f0,
                                    int32_t* __restrict__ e1, int32_t* __restrict__ e2) {
  const int64_t f = f0 + blockIdx.x;
  const double* row = xc + f * ld;
  double m = 0.0;
  int bad = 0;
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
    const double x = row[s];
    bad |= !isfinite(x);
    m = fmax(m, fabs(x));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(PS_FULL, m, o));
  bad = __syncthreads_or(bad);
  __shared__ double wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
    m = fmax(m, wm[0]);
    int a = 0, b = 0;
    if (m > 0.0) {
      frexp(m, &a);
      frexp(m * m, &b);  // the rounded square bounds every rounded x'^2 of the row
    }
    // (x'^2 overflowing to inf is non-finite for the FP64 path as well)
    if (bad || isinf(m * m)) a = b = kNonFinite;
    e1[f] = a;
    e2[f] = b;
  }
}

// all ND balanced base-2^BITS digits of every x' (or x'^2) of rows [f0, f0 +
// gridDim.x) as int8 planes out + (digit - 1) * plane (F x Sp each), zero past
// S; one pass over the operand, 16 samples per thread.  BITS = 7: digits in
// [-64, 64] (the Sxy planes: sums of two stay int8); BITS = 8: [-128, 127],
// the moments' planes (their other operand is the 0/1 presence).
template <int BITS, int ND>
__global__ void moment_digit_kernel(const double* __restrict__ xc, int64_t ld, int64_t S, int64_t Sp,
                                    const int32_t* __restrict__ rexp, int square, int64_t f0, int64_t plane,
                                    int8_t* __restrict__ out) {
  const int64_t f = f0 + blockIdx.x;
  const double* row = xc + f * ld;
  const int e = rexp[f];
  const bool zero = e == kNonFinite;  // (its moments are written as NaN)
  // u = rint(v 2^(BITS ND)), v = x / 2^(e + 1 + G): |u| <= 2^(BITS ND - 1 - G); base 256 takes a guard bit
  // (G = 1) so the most significant digit stays within +-65 (a full-range top digit could round up to 128)
  const int shift = BITS * ND - (BITS == 8 ? 2 : 1) - e;
  constexpr long long kHalf = 1ll << (BITS - 1), kMask = (1ll << BITS) - 1;
  for (int64_t s0 = (int64_t)threadIdx.x * 16; s0 < Sp; s0 += (int64_t)blockDim.x * 16) {
    uint32_t w[ND][4];
#pragma unroll
    for (int d = 0; d < ND; ++d) w[d][0] = w[d][1] = w[d][2] = w[d][3] = 0u;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t s = s0 + q;
      if (s < S && !zero) {
        double x = row[s];
        if (square) x = x * x;
        long long u = __double2ll_rn(ldexp(x, shift));
        // balanced digits from the least significant one up; the most
        // significant is what remains (|.| <= 64 + carry)
#pragma unroll
        for (int d = ND - 1; d >= 1; --d) {
          const long long lo = ((u + kHalf) & kMask) - kHalf;
          u = (u - lo) >> BITS;
          w[d][q >> 2] |= (uint32_t)(uint8_t)(int8_t)lo << (8 * (q & 3));
        }
        w[0][q >> 2] |= (uint32_t)(uint8_t)(int8_t)u << (8 * (q & 3));
      }
    }
#pragma unroll
    for (int d = 0; d < ND; ++d)
      *reinterpret_cast<uint4*>(out + d * plane + f * Sp + s0) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
  }
}

// presence as int8 0/1 (F x Sp), zero past S
__global__ void presence_i8_kernel(const uint32_t* __restrict__ mask, int64_t W, int64_t S, int64_t Sp,
                                   int8_t* __restrict__ out, int64_t f0 = 0) {
  const int64_t f = f0 + blockIdx.x;
  for (int64_t s0 = (int64_t)threadIdx.x * 16; s0 < Sp; s0 += (int64_t)blockDim.x * 16) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    const int64_t wi = s0 >> 5;
    const uint32_t bits = (wi < W ? mask[f * W + wi] : 0u) >> (s0 & 31);
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (s0 + q < S && ((bits >> q) & 1u)) w[q >> 2] |= 1u << (8 * (q & 3));
    *reinterpret_cast<uint4*>(out + f * Sp + s0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Symmetric form of Sxy.  Over the upper triangle the products D_s D_t^T and
// D_t D_s^T (s < t) are both needed; with the int8 sum plane E = D_s + D_t
// (digits lie in [-64, 64]: no overflow)
//   D_s D_t^T + D_t D_s^T = E E^T - D_s D_s^T - D_t D_t^T,
// so the 36 products with s + t <= 9 become 16 sum-plane products plus the 8
// squares D_s D_s^T with the weights c_s collected below: 24 contractions,
// still exact int32 sums (|E E| <= 2^14 per sample: S < 2^17).
#define PS_SYM_PAIRS(X)                                                                                   \
  X(0, 1, 8) X(1, 2, 7) X(2, 3, 6) X(3, 4, 5) X(4, 1, 7) X(5, 2, 6) X(6, 3, 5) X(7, 1, 6) X(8, 2, 5)       \
  X(9, 3, 4) X(10, 1, 5) X(11, 2, 4) X(12, 1, 4) X(13, 2, 3) X(14, 1, 3) X(15, 1, 2)
constexpr int kSymPairs = 16;
static_assert(kDigits == 8 && kSxyMaxOrder == 9, "PS_SYM_PAIRS lists s < t, s + t <= 9 over 8 digits");

// E planes p (out + p * plane) of rows [f0, f0 + gridDim.x) from their digit planes
__global__ void digit_sum_kernel(const int8_t* __restrict__ dig, int64_t plane, int64_t Sp, int64_t f0,
                                 int8_t* __restrict__ out) {
  const int64_t f = f0 + blockIdx.x;
  for (int64_t s0 = (int64_t)threadIdx.x * 16; s0 < Sp; s0 += (int64_t)blockDim.x * 16) {
    uint4 d[kDigits];
#pragma unroll
    for (int k = 0; k < kDigits; ++k) d[k] = *reinterpret_cast<const uint4*>(dig + k * plane + f * Sp + s0);
#define PS_SYM_STORE(P, A, B)                                                                             \
  *reinterpret_cast<uint4*>(out + (int64_t)(P)*plane + f * Sp + s0) =                                     \
      make_uint4(__vadd4(d[A - 1].x, d[B - 1].x), __vadd4(d[A - 1].y, d[B - 1].y),                        \
                 __vadd4(d[A - 1].z, d[B - 1].z), __vadd4(d[A - 1].w, d[B - 1].w));
    PS_SYM_PAIRS(PS_SYM_STORE)
#undef PS_SYM_STORE
  }
}

// out(i, j) (+)= 2^(e_i + 1 - 7 digit) (D M^T)(i, j) over the tiles of rows
// [I0, I0 + nI) x columns [J0, J0 + nJ) (256 x 256 each; rows / columns past F
// are zero-filled by TMA and not written).  One persistent CTA per SM takes
// tiles round-robin; each tile runs the whole K range (no split: the int32
// tile is exact and folded once).  Warp roles as the contingency GEMM
// (ps_chi2.cu): TMA producer, single-thread MMA issuer, four epilogue warps
// draining the two 128 x 256 TMEM accumulators.
__global__ void __launch_bounds__(QTH, 1)
moment_gemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int nk,
                   int64_t I0, int64_t nI, int64_t J0, int64_t nJ, const int32_t* __restrict__ rexp, int digit,
                   int first, double* __restrict__ out, int64_t F) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[QSTAGES], empty[QSTAGES], accfull, accempty;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = nI * nJ;

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, 512);
  if (tid == 32) {
    for (int i = 0; i < QSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 1);
    }
    tc05::mbar_init(&accfull, 1);
    tc05::mbar_init(&accempty, 128);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32) {
    tc05::prefetch_tmap(&amap);
    tc05::prefetch_tmap(&bmap);
  }
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      int64_t q = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t ri, cj;
        band_unit(t, nI, nJ, ri, cj);
        const int I = (int)(I0 + ri), J = (int)(J0 + cj);
        for (int kc = 0; kc < nk; ++kc, ++q) {
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
          const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
          tc05::mbar_arrive_expect_tx(&full[st], QSTAGE_BYTES);
          tc05::tma_load_2d(sa, &amap, kc * QKB, I * QM, &full[st]);
          tc05::tma_load_2d(sb, &bmap, kc * QKB, J * QN, &full[st]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(128, QN, true);
      int64_t q = 0;
      int seg = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++seg) {
        if (seg > 0) {  // the epilogue has drained the previous tile
          tc05::mbar_wait(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        for (int kc = 0; kc < nk; ++kc, ++q) {
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
          tc05::fence_after_sync();
          const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
#pragma unroll
          for (int kk = 0; kk < QKB / 32; ++kk) {
            const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
            const uint32_t acc = (kc > 0 || kk > 0) ? 1u : 0u;
            tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
            tc05::mma_i8(tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * QKB + kk * 32), bd, idesc, acc);
          }
          tc05::commit(&empty[st]);
        }
        tc05::commit(&accfull);
      }
    }
  } else {
    // epilogue warps 0-3: TMEM lanes 32 w .. 32 w + 31 = tile rows
    int seg = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++seg) {
      int64_t ri, cj;
      band_unit(t, nI, nJ, ri, cj);
      const int64_t I = I0 + ri, J = J0 + cj;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int64_t r = I * QM + half * 128 + warp * 32 + lane;
        const bool rok = r < F;
        const int ex = rok ? rexp[r] : 0;
        const double scale = ex == kNonFinite ? PS_NAN : ldexp(1.0, ex + 1 - digit);
        double* orow = out + (rok ? r : 0) * F;
#pragma unroll 1
        for (int cc = 0; cc < QN / 32; ++cc) {
          uint32_t v[32];
          tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
          const int64_t c0 = J * QN + cc * 32;
          if (rok) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int64_t c = c0 + j;
              if (c < F) {
                const double term = (double)(int32_t)v[j] * scale;
                orow[c] = first ? term : orow[c] + term;
              }
            }
          }
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive(&accempty);
    }
  }
  tc05::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc05::tmem_dealloc(tmem, 512);
}

// Cluster-pair variant: the two CTAs of a cluster take the row tiles
// (I0 + 2p, J) and (I0 + 2p + 1, J) -- the same presence tile J -- and each
// TMA-loads half of it, multicast into both CTAs: 48 KB of L2 reads per CTA
// per K step instead of 64 KB.  A stage is refilled only after both CTAs'
// MMAs released it (the MMA commit arrives on the `empty` barrier of both);
// an odd last row tile runs with a dummy partner that only loads its half of
// the shared tile.
constexpr int QHALF = QB_BYTES / 2;  // 128 rows x 128 B
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(QTH, 1)
moment_gemm_mc_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int nk,
                      int64_t I0, int64_t nI, int64_t J0, int64_t nJ, const int32_t* __restrict__ rexp, int digit,
                      int first, double* __restrict__ out, int64_t F) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[QSTAGES], empty[QSTAGES], accfull, accempty;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)tc05::cluster_ctarank();
  const int64_t ncl = gridDim.x / 2, cl = blockIdx.x / 2;
  const int64_t np = (nI + 1) / 2, nunits = np * nJ;

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, 512);
  if (tid == 32) {
    for (int i = 0; i < QSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 2);  // both CTAs' MMA commits
    }
    tc05::mbar_init(&accfull, 1);
    tc05::mbar_init(&accempty, 128);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32) {
    tc05::prefetch_tmap(&amap);
    tc05::prefetch_tmap(&bmap);
  }
  tc05::fence_before_sync();
  tc05::cluster_sync();  // barriers initialised in both CTAs before any multicast
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      int64_t q = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, cj;
        band_unit(u, np, nJ, pr, cj);
        const int64_t ip = 2 * pr + rank;
        const bool own = ip < nI;
        const int I = (int)(I0 + ip), J = (int)(J0 + cj);
        for (int kc = 0; kc < nk; ++kc, ++q) {
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
          const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
          tc05::mbar_arrive_expect_tx(&full[st], own ? QSTAGE_BYTES : QB_BYTES);
          tc05::tma_load_2d_mc(sb + rank * QHALF, &bmap, kc * QKB, J * QN + rank * 128, &full[st], (uint16_t)3);
          if (own) tc05::tma_load_2d(sa, &amap, kc * QKB, I * QM, &full[st]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(128, QN, true);
      int64_t q = 0;
      int seg = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, cj;
        band_unit(u, np, nJ, pr, cj);
        const bool own = 2 * pr + rank < nI;
        if (own && seg > 0) {  // the epilogue has drained the previous tile
          tc05::mbar_wait(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        for (int kc = 0; kc < nk; ++kc, ++q) {
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
          tc05::fence_after_sync();
          if (own) {
            const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
#pragma unroll
            for (int kk = 0; kk < QKB / 32; ++kk) {
              const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
              const uint32_t acc = (kc > 0 || kk > 0) ? 1u : 0u;
              tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
              tc05::mma_i8(tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * QKB + kk * 32), bd, idesc, acc);
            }
          }
          tc05::commit_mc(&empty[st], (uint16_t)3);
        }
        if (own) {
          tc05::commit(&accfull);
          ++seg;
        }
      }
    }
  } else {
    // epilogue warps 0-3: TMEM lanes 32 w .. 32 w + 31 = tile rows
    int seg = 0;
    for (int64_t u = cl; u < nunits; u += ncl) {
      int64_t pr, cj;
      band_unit(u, np, nJ, pr, cj);
      const int64_t ip = 2 * pr + rank;
      if (ip >= nI) continue;  // dummy partner
      const int64_t I = I0 + ip, J = J0 + cj;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int64_t r = I * QM + half * 128 + warp * 32 + lane;
        const bool rok = r < F;
        const int ex = rok ? rexp[r] : 0;
        const double scale = ex == kNonFinite ? PS_NAN : ldexp(1.0, ex + 1 - digit);
        double* orow = out + (rok ? r : 0) * F;
#pragma unroll 1
        for (int cc = 0; cc < QN / 32; ++cc) {
          uint32_t v[32];
          tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
          const int64_t c0 = J * QN + cc * 32;
          if (rok) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int64_t c = c0 + j;
              if (c < F) {
                const double term = (double)(int32_t)v[j] * scale;
                orow[c] = first ? term : orow[c] + term;
              }
            }
          }
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive(&accempty);
      ++seg;
    }
  }
  tc05::fence_before_sync();
  __syncthreads();
  tc05::cluster_sync();  // no CTA leaves while its partner may still multicast / commit into it
  if (warp == 0) tc05::tmem_dealloc(tmem, 512);
}

// Up to kCrossGroup digit products of one weight concatenated along K: one
// exact int32 accumulation per tile (|sum| <= g 4096 S < 2^31), one fold.
constexpr int kCrossGroup = 4;
constexpr int kCrossBand = 12;  // tile columns per band of the unit order
struct CrossMaps {
  CUtensorMap a[kCrossGroup];  // 256-row boxes (own rows)
  CUtensorMap b[kCrossGroup];  // 128-row boxes (multicast halves of the column tile)
  int g;                       // products in the group
};

// Units of the cross GEMMs: (row pair p, column c = J - I0) with 2p <= c,
// p < np, over the columns [cb, W0): cb = 0 for a range's whole triangle
// (Jlo < 0), Jlo - I0 for a column block of the incremental upload.  They are
// walked in column bands of kCrossBand tiles, row pairs outermost within a
// band, so a wave of consecutive units covers a compact (row pairs x columns)
// block whose operand slabs stay in L2 (a row- or column-major wave streams
// ~3x the tiles from DRAM).
struct CrossUnits {
  int64_t I0, np, W0, cb, ubase, nunits;
  __device__ static int64_t half_sum(int64_t x) { return x <= 0 ? 0 : (x / 2) * ((x - 1) / 2); }  // sum_{m<x} m/2
  __device__ int64_t ccum(int64_t x) const {  // units with c < x: sum of min(c / 2 + 1, np)
    x = x < W0 ? x : W0;
    return x <= 2 * np ? x + half_sum(x) : 2 * np + half_sum(2 * np) + np * (x - 2 * np);
  }
  __device__ CrossUnits(int64_t I0_, int64_t nI, int64_t NT, int64_t Jlo)
      : I0(I0_), np((nI + 1) / 2), W0(NT - I0_), cb(Jlo < 0 ? 0 : Jlo - I0_) {
    ubase = ccum(cb);
    nunits = ccum(W0) - ubase;
  }
  __device__ void unit(int64_t u, int64_t& pr, int64_t& J) const {
    int64_t a = 0, b = (W0 - cb - 1) / kCrossBand;
    while (a < b) {
      const int64_t m = (a + b + 1) >> 1;
      if (ccum(cb + m * kCrossBand) - ubase <= u) a = m;
      else b = m - 1;
    }
    const int64_t c0 = cb + a * kCrossBand, c1 = c0 + kCrossBand < W0 ? c0 + kCrossBand : W0, w = c1 - c0;
    int64_t rem = u - (ccum(c0) - ubase);
    const int64_t fr = c0 / 2 + 1 < np ? c0 / 2 + 1 : np;  // row pairs holding the whole band
    if (rem < fr * w) {
      pr = rem / w;
      J = I0 + c0 + rem % w;
      return;
    }
    rem -= fr * w;
    int64_t p = fr;
    while (rem >= c1 - 2 * p) {  // at most kCrossBand / 2 partial row pairs
      rem -= c1 - 2 * p;
      ++p;
    }
    pr = p;
    J = I0 + 2 * p + rem;
  }
};

// Cross products over the upper triangle of tiles: out(i, j) (+)= w rs_i cs_j
// (A B^T)(i, j) for the tile rows [I0, I0 + nI) and columns J >= I (Sxy from
// digit planes s of rows i and t of rows j, w = 2^-7(s+t), rs = cs = 2^(e1+1));
// or, with nout, the raw int32 products (pair counts from the presence).
// Cluster pairs share the column tile as the contingency / moment GEMMs do:
// the pair (I0 + 2p, I0 + 2p + 1) walks columns J >= I0 + 2p (one lower tile
// per pair is computed and never read).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(QTH, 1)
cross_gemm_mc_kernel(const __grid_constant__ CrossMaps maps, int nk,
                     int64_t I0, int64_t nI, int64_t NT, const double* __restrict__ rs, const double* __restrict__ cs,
                     double w, int first, double* __restrict__ out, int32_t* __restrict__ nout, int64_t F,
                     int64_t Jlo) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[QSTAGES], empty[QSTAGES], accfull, accempty;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)tc05::cluster_ctarank();
  const int64_t ncl = gridDim.x / 2, cl = blockIdx.x / 2;
  const CrossUnits cu(I0, nI, NT, Jlo);
  const int64_t nunits = cu.nunits;
  auto unit = [&](int64_t u, int64_t& pr, int64_t& J) { cu.unit(u, pr, J); };

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, 512);
  if (tid == 32) {
    for (int i = 0; i < QSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 2);
    }
    tc05::mbar_init(&accfull, 1);
    tc05::mbar_init(&accempty, 128);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32)
    for (int m = 0; m < maps.g; ++m) {
      tc05::prefetch_tmap(&maps.a[m]);
      tc05::prefetch_tmap(&maps.b[m]);
    }
  const int nkt = nk * maps.g;  // concatenated K steps
  tc05::fence_before_sync();
  tc05::cluster_sync();
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      int64_t q = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, J;
        unit(u, pr, J);
        const int64_t ip = 2 * pr + rank;
        const bool own = ip < nI;
        const int I = (int)(I0 + ip);
        for (int kt = 0; kt < nkt; ++kt, ++q) {
          const int m = kt / nk, kc = kt - m * nk;
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
          const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
          tc05::mbar_arrive_expect_tx(&full[st], own ? QSTAGE_BYTES : QB_BYTES);
          tc05::tma_load_2d_mc(sb + rank * QHALF, &maps.b[m], kc * QKB, (int)J * QN + rank * 128, &full[st],
                               (uint16_t)3);
          if (own) tc05::tma_load_2d(sa, &maps.a[m], kc * QKB, I * QM, &full[st]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(128, QN, true);
      int64_t q = 0;
      int seg = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, J;
        unit(u, pr, J);
        const bool own = 2 * pr + rank < nI;
        if (own && seg > 0) {
          tc05::mbar_wait(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        for (int kt = 0; kt < nkt; ++kt, ++q) {
          const int st = (int)(q % QSTAGES), n = (int)(q / QSTAGES);
          tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
          tc05::fence_after_sync();
          if (own) {
            const uint32_t sa = sbase + st * QSTAGE_BYTES, sb = sa + QA_BYTES;
#pragma unroll
            for (int kk = 0; kk < QKB / 32; ++kk) {
              const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
              const uint32_t acc = (kt > 0 || kk > 0) ? 1u : 0u;
              tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
              tc05::mma_i8(tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * QKB + kk * 32), bd, idesc, acc);
            }
          }
          tc05::commit_mc(&empty[st], (uint16_t)3);
        }
        if (own) {
          tc05::commit(&accfull);
          ++seg;
        }
      }
    }
  } else {
    int seg = 0;
    for (int64_t u = cl; u < nunits; u += ncl) {
      int64_t pr, J;
      unit(u, pr, J);
      const int64_t ip = 2 * pr + rank;
      if (ip >= nI) continue;  // dummy partner
      const int64_t I = I0 + ip;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int64_t r = I * QM + half * 128 + warp * 32 + lane;
        const bool rok = r < F;
        const double rsw = rok && rs ? rs[r] * w : 0.0;
#pragma unroll 1
        for (int cc = 0; cc < QN / 32; ++cc) {
          uint32_t v[32];
          tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
          const int64_t c0 = J * QN + cc * 32;
          if (!rok) continue;
          if (nout) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < F) nout[r * F + c0 + j] = (int32_t)v[j];
          } else {
            double* orow = out + r * F;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int64_t c = c0 + j;
              if (c < F) {
                const double term = (double)(int32_t)v[j] * rsw * cs[c];
                orow[c] = first ? term : orow[c] + term;
              }
            }
          }
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive(&accempty);
      ++seg;
    }
  }
  tc05::fence_before_sync();
  __syncthreads();
  tc05::cluster_sync();
  if (warp == 0) tc05::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// CTA-pair forms (tcgen05 cta_group::2): the pair's 512 x 256 block as two
// M = 256 MMAs per K slice -- rows [128 h, 128 h + 128) of each CTA's own
// 256-row A tile against the column tile, whose two N halves sit one in each
// CTA.  Per 128-byte K step a CTA stages 48 KB (its A tile + half of B)
// instead of 64 KB, and each MMA reads half of B from either SM: four stages
// fit where three did, and the shared-memory traffic (operand reads + TMA
// fills) drops from ~156 to ~109 B / clk / SM, under the 128 B / clk port.
// Same units, same K order, same int32 sums: bitwise the results of the
// multicast kernels.
constexpr int Q2STAGES = 4;
constexpr int Q2STAGE_BYTES = QA_BYTES + QHALF;
constexpr size_t kMom2Smem = (size_t)Q2STAGES * Q2STAGE_BYTES + 1024;

struct Pipe2 {
  uint64_t *full, *empty, *accfull, *accempty;
  uint32_t sbase, tmem, full_leader[Q2STAGES], accempty_leader;
  int rank;
};

// producer lane: this CTA's A tile rows and its half of the column tile for K step kx
__device__ __forceinline__ void pipe2_load(const Pipe2& pp, int64_t q, const CUtensorMap* am, const CUtensorMap* bm,
                                           int kx, int arow, int brow) {
  const int st = (int)(q % Q2STAGES), n = (int)(q / Q2STAGES);
  if (n > 0) tc05::mbar_wait(&pp.empty[st], (uint32_t)((n - 1) & 1));
  const uint32_t sa = pp.sbase + st * Q2STAGE_BYTES, sb = sa + QA_BYTES;
  if (pp.rank == 0) tc05::mbar_arrive_expect_tx(&pp.full[st], 2 * Q2STAGE_BYTES);
  tc05::tma_load_2d_2sm(sa, am, kx, arow, pp.full_leader[st]);
  tc05::tma_load_2d_2sm(sb, bm, kx, brow, pp.full_leader[st]);
}

// leader's MMA lane: one staged K step into the two accumulators
__device__ __forceinline__ void pipe2_mma(const Pipe2& pp, int64_t q, bool first_step) {
  constexpr uint32_t idesc = tc05::idesc_i8(256, QN, true);
  const int st = (int)(q % Q2STAGES), n = (int)(q / Q2STAGES);
  tc05::mbar_wait_cluster(&pp.full[st], (uint32_t)(n & 1));
  tc05::fence_after_sync();
  const uint32_t sa = pp.sbase + st * Q2STAGE_BYTES, sb = sa + QA_BYTES;
#pragma unroll
  for (int kk = 0; kk < QKB / 32; ++kk) {
    const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
    const uint32_t acc = (!first_step || kk > 0) ? 1u : 0u;
    tc05::mma_i8_2sm(pp.tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
    tc05::mma_i8_2sm(pp.tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * QKB + kk * 32), bd, idesc, acc);
  }
  tc05::commit_2sm(&pp.empty[st], (uint16_t)3);
}

#define PS_PIPE2_SETUP()                                                                                        \
  extern __shared__ __align__(1024) unsigned char tsm_raw[];                                                    \
  __shared__ uint64_t full[Q2STAGES], empty[Q2STAGES], accfull, accempty;                                       \
  __shared__ uint32_t tmem_base_s;                                                                              \
  unsigned char* tsm =                                                                                          \
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));       \
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;                                                \
  Pipe2 pp;                                                                                                     \
  pp.full = full, pp.empty = empty, pp.accfull = &accfull, pp.accempty = &accempty;                             \
  pp.sbase = tc05::smem_u32(tsm);                                                                               \
  pp.rank = (int)tc05::cluster_ctarank();                                                                       \
  const int rank = pp.rank;                                                                                     \
  const int64_t ncl = gridDim.x / 2, cl = blockIdx.x / 2;                                                       \
  if (warp == 0) tc05::tmem_alloc_2sm(&tmem_base_s, 512);                                                       \
  if (tid == 32) {                                                                                              \
    for (int i = 0; i < Q2STAGES; ++i) {                                                                        \
      tc05::mbar_init(&full[i], 1);  /* the leader's expect_tx arrival; both CTAs' bytes */                     \
      tc05::mbar_init(&empty[i], 1); /* the leader's commit, multicast to both */                               \
    }                                                                                                           \
    tc05::mbar_init(&accfull, 1);                                                                               \
    tc05::mbar_init(&accempty, 256); /* both CTAs' epilogue threads (leader's copy is the one waited on) */     \
    tc05::fence_barrier_init();                                                                                 \
  }                                                                                                             \
  for (int i = 0; i < Q2STAGES; ++i) pp.full_leader[i] = tc05::map_to_rank(&full[i], 0);                        \
  pp.accempty_leader = tc05::map_to_rank(&accempty, 0);                                                         \
  tc05::fence_before_sync();                                                                                    \
  tc05::cluster_sync();                                                                                         \
  tc05::fence_after_sync();                                                                                     \
  pp.tmem = tmem_base_s;                                                                                        \
  const uint32_t tmem = pp.tmem;

#define PS_PIPE2_TEARDOWN()                                                      \
  tc05::fence_before_sync();                                                     \
  __syncthreads();                                                               \
  tc05::cluster_sync(); /* no CTA leaves while the pair's MMAs / commits run */  \
  if (warp == 0) tc05::tmem_dealloc_2sm(tmem, 512);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(QTH, 1)
moment_gemm_2sm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int nk,
                       int64_t I0, int64_t nI, int64_t J0, int64_t nJ, const int32_t* __restrict__ rexp, int digit,
                       int first, double* __restrict__ out, int64_t F, int bswap) {
  PS_PIPE2_SETUP();
  const int64_t np = (nI + 1) / 2, nunits = np * nJ;
  if (tid == 4 * 32) {
    tc05::prefetch_tmap(&amap);
    tc05::prefetch_tmap(&bmap);
  }
  if (warp == 4) {
    if (lane == 0) {  // TMA producer (both CTAs; a dummy partner's rows are loaded and never stored)
      int64_t q = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, cj;
        band_unit(u, np, nJ, pr, cj);
        const int I = (int)(I0 + 2 * pr + rank), J = (int)(J0 + cj);
        for (int kc = 0; kc < nk; ++kc, ++q)
          pipe2_load(pp, q, &amap, &bmap, kc * QKB, I * QM, J * QN + (rank ^ bswap) * 128);
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && rank == 0) {  // MMA issuer of the pair
      int64_t q = 0;
      int seg = 0;
      for (int64_t u = cl; u < nunits; u += ncl, ++seg) {
        if (seg > 0) {  // both epilogues have drained the previous tiles
          tc05::mbar_wait_cluster(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        for (int kc = 0; kc < nk; ++kc, ++q) pipe2_mma(pp, q, kc == 0);
        tc05::commit_2sm(&accfull, (uint16_t)3);
      }
    }
  } else {
    int seg = 0;
    for (int64_t u = cl; u < nunits; u += ncl, ++seg) {
      int64_t pr, cj;
      band_unit(u, np, nJ, pr, cj);
      const int64_t ip = 2 * pr + rank;
      const int64_t I = I0 + ip, J = J0 + cj;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
      if (ip < nI) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int64_t r = I * QM + half * 128 + warp * 32 + lane;
          const bool rok = r < F;
          const int ex = rok ? rexp[r] : 0;
          const double scale = ex == kNonFinite ? PS_NAN : ldexp(1.0, ex + 1 - digit);
          double* orow = out + (rok ? r : 0) * F;
#pragma unroll 1
          for (int cc = 0; cc < QN / 32; ++cc) {
            uint32_t v[32];
            tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
            const int64_t c0 = J * QN + cc * 32;
            if (rok) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int64_t c = c0 + j;
                if (c < F) {
                  const double term = (double)(int32_t)v[j] * scale;
                  orow[c] = first ? term : orow[c] + term;
                }
              }
            }
          }
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive_cluster(pp.accempty_leader);
    }
  }
  PS_PIPE2_TEARDOWN();
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(QTH, 1)
cross_gemm_2sm_kernel(const __grid_constant__ CrossMaps maps, int nk, int64_t I0, int64_t nI, int64_t NT,
                      const double* __restrict__ rs, const double* __restrict__ cs, double w, int first,
                      double* __restrict__ out, int32_t* __restrict__ nout, int64_t F, int64_t Jlo, int bswap) {
  PS_PIPE2_SETUP();
  const CrossUnits cu(I0, nI, NT, Jlo);
  const int64_t nunits = cu.nunits;
  if (tid == 4 * 32)
    for (int m = 0; m < maps.g; ++m) {
      tc05::prefetch_tmap(&maps.a[m]);
      tc05::prefetch_tmap(&maps.b[m]);
    }
  const int nkt = nk * maps.g;  // concatenated K steps
  if (warp == 4) {
    if (lane == 0) {
      int64_t q = 0;
      for (int64_t u = cl; u < nunits; u += ncl) {
        int64_t pr, J;
        cu.unit(u, pr, J);
        const int I = (int)(I0 + 2 * pr + rank);
        for (int kt = 0; kt < nkt; ++kt, ++q) {
          const int m = kt / nk, kc = kt - m * nk;
          pipe2_load(pp, q, &maps.a[m], &maps.b[m], kc * QKB, I * QM, (int)J * QN + (rank ^ bswap) * 128);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && rank == 0) {
      int64_t q = 0;
      int seg = 0;
      for (int64_t u = cl; u < nunits; u += ncl, ++seg) {
        if (seg > 0) {
          tc05::mbar_wait_cluster(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        for (int kt = 0; kt < nkt; ++kt, ++q) pipe2_mma(pp, q, kt == 0);
        tc05::commit_2sm(&accfull, (uint16_t)3);
      }
    }
  } else {
    int seg = 0;
    for (int64_t u = cl; u < nunits; u += ncl, ++seg) {
      int64_t pr, J;
      cu.unit(u, pr, J);
      const int64_t ip = 2 * pr + rank;
      const int64_t I = I0 + ip;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
      if (ip < nI) {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int64_t r = I * QM + half * 128 + warp * 32 + lane;
          const bool rok = r < F;
          const double rsw = rok && rs ? rs[r] * w : 0.0;
#pragma unroll 1
          for (int cc = 0; cc < QN / 32; ++cc) {
            uint32_t v[32];
            tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
            const int64_t c0 = J * QN + cc * 32;
            if (!rok) continue;
            if (nout) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j < F) nout[r * F + c0 + j] = (int32_t)v[j];
            } else {
              double* orow = out + r * F;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int64_t c = c0 + j;
                if (c < F) {
                  const double term = (double)(int32_t)v[j] * rsw * cs[c];
                  orow[c] = first ? term : orow[c] + term;
                }
              }
            }
          }
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive_cluster(pp.accempty_leader);
    }
  }
  PS_PIPE2_TEARDOWN();
}

// PS_GEMM_2SM=1 selects the CTA-pair kernels (=2: column halves swapped, a
// bring-up check that must fail).  Measured equal to the multicast kernels on
// config 5 (both run at the power cap, DESIGN 4b), which stay the default.
int gemm_2sm_mode() {
  const char* e = getenv("PS_GEMM_2SM");
  return e ? atoi(e) : 0;
}

// 2^(e1 + 1) per row (NaN for rows holding NaN / inf): the Sxy fold scales
__global__ void row_scale_kernel(const int32_t* __restrict__ e1, int64_t f0, int64_t n, double* __restrict__ sc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int e = e1[f0 + i];
  sc[f0 + i] = e == kNonFinite ? PS_NAN : ldexp(1.0, e + 1);
}

PFN_cuTensorMapEncodeTiled_v12000 moment_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// K-major int8 rows (F x Sp bytes), 128-byte x box_rows boxes, SWIZZLE_128B
int make_i8_map(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t Sp, int box_rows = QM) {
  auto enc = moment_map_encoder();
  if (!enc) return ps_fail(PS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)Sp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Sp};
  cuuint32_t box[2] = {(cuuint32_t)QKB, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return ps_fail(PS_ERR_CUDA, "moment operand tensor map");
  return PS_OK;
}

}  // namespace

// The Sxy digit products in fold order (smallest weights first, s ascending),
// same-weight products grouped by up to kCrossGroup (as many as int32 allows
// for S samples) into one K-concatenated contraction: emit(group maps, weight)
template <class A, class B, class Emit>
static void sxy_groups(int64_t S, const A& amaps, const B& bmaps, Emit&& emit) {
  const int gmax = (int)std::max<int64_t>(1, std::min<int64_t>(kCrossGroup, (int64_t)INT32_MAX / (4096 * S)));
  for (int k = kSxyMaxOrder; k >= 2; --k) {
    CrossMaps cm;
    cm.g = 0;
    for (int sd = std::max(1, k - kDigits); sd <= std::min(kDigits, k - 1); ++sd) {
      cm.a[cm.g] = amaps[sd - 1];
      cm.b[cm.g] = bmaps[k - sd - 1];
      if (++cm.g == gmax) {
        emit(cm, ldexp(1.0, -7 * k));
        cm.g = 0;
      }
    }
    if (cm.g) emit(cm, ldexp(1.0, -7 * k));
  }
}

// Symmetric Sxy: the 16 sum-plane products (smallest weights first), then the
// squares D_s D_s^T, s = 8 .. 1, with c_s = [2 s <= 9] 2^-14s - sum_{t != s, s + t <= 9} 2^-7(s+t)
// (each exact in fp64: the powers span at most 49 bits).  One fixed fold order.
template <class Emit>
static void sxy_sym_products(const CUtensorMap* emaps, const CUtensorMap* ehalf, const CUtensorMap* amaps,
                             const CUtensorMap* ahalf, Emit&& emit) {
  static const int ps_[kSymPairs][2] = {
#define PS_SYM_ROW(P, S_, T_) {S_, T_},
      PS_SYM_PAIRS(PS_SYM_ROW)
#undef PS_SYM_ROW
  };
  CrossMaps cm;
  cm.g = 1;
  for (int p = 0; p < kSymPairs; ++p) {
    cm.a[0] = emaps[p];
    cm.b[0] = ehalf[p];
    emit(cm, ldexp(1.0, -7 * (ps_[p][0] + ps_[p][1])));
  }
  for (int sd = kDigits; sd >= 1; --sd) {
    double c = 2 * sd <= kSxyMaxOrder ? ldexp(1.0, -14 * sd) : 0.0;
    for (int td = kDigits; td >= 1; --td)  // smallest first: every partial sum is exact
      if (td != sd && sd + td <= kSxyMaxOrder) c -= ldexp(1.0, -7 * (sd + td));
    cm.a[0] = amaps[sd - 1];
    cm.b[0] = ahalf[sd - 1];
    emit(cm, c);
  }
}

// the symmetric form needs |E E| <= 2^14 per sample in int32 (PS_SXY_SYM=0: the 36 products)
bool ps_sxy_sym(int64_t S) {
  const char* e = getenv("PS_SXY_SYM");
  return !(e && e[0] == '0') && S <= (int64_t)(INT32_MAX / 16384);
}

// Moment planes in balanced base 256 (digits in [-128, 127] against the 0/1
// presence: |sum| <= 128 S in int32; one guard bit, so x = 2^(e + 2) sum_d
// D_d 2^-8d): 6 planes carry Sx (rounded at 2^(e - 47)), 7 carry Sxx
// (2^(e - 55)) -- 13 contractions per ordered pair instead of 15.
// PS_MOMENTS_B256=0: the base-128 planes (7 + 8).
constexpr int kSxDigits256 = 6, kSqDigits256 = 7;
bool ps_moments_b256(int64_t S) {
  const char* e = getenv("PS_MOMENTS_B256");
  return !(e && e[0] == '0') && S <= (int64_t)(INT32_MAX / 128);
}
// x' (sq = 0) or x'^2 (sq = 1) of rows [r0, r0 + n) into the moments' planes
static void moment_planes(bool b256, int sq, const double* xc, int64_t ld, int64_t S, int64_t Sp, const int32_t* ex,
                          int64_t r0, int64_t n, int64_t plane, int8_t* out, cudaStream_t s) {
  if (!b256)
    moment_digit_kernel<7, kDigits><<<(unsigned)n, 256, 0, s>>>(xc, ld, S, Sp, ex, sq, r0, plane, out);
  else if (sq)
    moment_digit_kernel<8, kSqDigits256><<<(unsigned)n, 256, 0, s>>>(xc, ld, S, Sp, ex, sq, r0, plane, out);
  else
    moment_digit_kernel<8, kSxDigits256><<<(unsigned)n, 256, 0, s>>>(xc, ld, S, Sp, ex, sq, r0, plane, out);
}
static int moment_digits(bool b256, int sq) { return b256 ? (sq ? kSqDigits256 : kSxDigits256) : (sq ? kDigits : kSxDigits); }

// int8 Sxy: each digit product accumulates |d_s d_t| <= 4096 per sample in
// int32, so the samples are capped at 2^31 / 4096 (the moments' 0/1 operand
// allows 64x more)
bool ps_sxy_int8(int64_t S) {
  const char* e = getenv("PS_PEARSON_SXY");
  return !(e && e[0] == 'd') && S <= (int64_t)(INT32_MAX / 4096);
}

bool ps_moments_on(int64_t F, int64_t S) {
  if (S > (int64_t)(INT32_MAX / 64)) return false;  // int32 digit x presence sums
  if (const char* e = getenv("PS_PEARSON_MOMENTS")) return e[0] == '1';
  return F >= 2048 && S >= 256;
}

int ps_pearson_moments(const ps_matrix* a, const double* xc, int64_t lo, int64_t hi, double** sx_out,
                       double** sq_out, int32_t** e1_out, int32_t** e2_out, double* sxy, int32_t* nn,
                       cudaStream_t s) {
  *sx_out = *sq_out = nullptr;
  *e1_out = *e2_out = nullptr;
  const int64_t F = a->F, S = a->S;
  lo = std::max<int64_t>(0, std::min<int64_t>(lo, F));
  hi = std::max<int64_t>(lo + 1, std::min<int64_t>(hi, F));
  ps_device_state* ds = ps_state();
  const int64_t Sp = ps_round_up(std::max<int64_t>(S, 1), QKB);
  const int nk = (int)(Sp / QKB);
  double *sx = nullptr, *sq = nullptr;
  int8_t *dig = nullptr, *pres = nullptr;
  int32_t *e1 = nullptr, *e2 = nullptr;
  double* rsc = nullptr;  // 2^(e1 + 1) per row (Sxy)
  int8_t* esum = nullptr;  // the 16 sum planes of the symmetric Sxy
  const bool sym = sxy && ps_sxy_sym(S);
  auto cleanup = [&]() {
    ps_free(esum, s);
    ps_free(dig, s);
    ps_free(pres, s);
    ps_free(rsc, s);
  };
  cudaError_t e = ps_alloc(&sx, (size_t)(F * F), s);
  if (e == cudaSuccess) e = ps_alloc(&sq, (size_t)(F * F), s);
  if (e == cudaSuccess) e = ps_alloc(&dig, (size_t)(kDigits * F * Sp), s);
  if (e == cudaSuccess) e = ps_alloc(&pres, (size_t)(F * Sp), s);
  if (e == cudaSuccess) e = ps_alloc(&e1, (size_t)F, s);
  if (e == cudaSuccess) e = ps_alloc(&e2, (size_t)F, s);
  if (e == cudaSuccess && sxy) e = ps_alloc(&rsc, (size_t)F, s);
  if (e == cudaSuccess && sym) e = ps_alloc(&esum, (size_t)(kSymPairs * F * Sp), s);
  if (e == cudaSuccess && sxy)
    e = cudaFuncSetAttribute(cross_gemm_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMomSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(cross_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMom2Smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(moment_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMom2Smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(moment_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)kMomSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(moment_gemm_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)kMomSmem);
  if (e != cudaSuccess) {
    cleanup();
    ps_free(sx, s);
    ps_free(sq, s);
    ps_free(e1, s);
    ps_free(e2, s);
    return ps_cuda_check(e, "pearson moments setup");
  }
  // The pairs (g, h >= g), g in [lo, hi), read Sx(g, h) and Sx(h, g): an L of
  // tiles -- rows [lo, hi) x columns [lo, F) (R1) plus rows past hi x columns
  // [lo, hi) (R2) -- so a rank's share of the int8 work follows its share of
  // the pairs (a single range [0, F) is the whole square).  Tile-aligned
  // (rows / columns before lo are computed as well, unused); R2 starts at the
  // tile row after R1's last, so no tile is folded twice.
  const int64_t NTt = ps_ceil_div(F, QM);
  const int64_t I0 = lo / QM, I1 = (hi - 1) / QM;
  const int64_t J0 = lo / QN, Jh = (hi - 1) / QN;
  const int64_t nI = I1 - I0 + 1, nJ = NTt - J0;            // R1
  const int64_t I2 = I1 + 1, nI2 = NTt - I2, nJ2 = Jh - J0 + 1;  // R2
  const int64_t r0 = I0 * QM, nrows = F - r0;
  moment_scale_kernel<<<(unsigned)nrows, 256, 0, s>>>(xc, a->ld, S, r0, e1, e2);
  PS_LAUNCHED();
  presence_i8_kernel<<<(unsigned)F, 256, 0, s>>>(a->d_mask, a->W, S, Sp, pres);
  PS_LAUNCHED();
  CUtensorMap amap[kDigits], ahalf[kDigits], bmap, bmap_half;
  int rc = make_i8_map(&bmap, pres, F, Sp);
  if (!rc) rc = make_i8_map(&bmap_half, pres, F, Sp, QN / 2);  // multicast halves
  for (int d = 0; d < kDigits && !rc; ++d) rc = make_i8_map(&amap[d], dig + d * F * Sp, F, Sp);
  for (int d = 0; d < kDigits && !rc && sxy; ++d) rc = make_i8_map(&ahalf[d], dig + d * F * Sp, F, Sp, QN / 2);
  CUtensorMap emap[kSymPairs], ehalf[kSymPairs];
  for (int d = 0; d < kSymPairs && !rc && sym; ++d) {
    rc = make_i8_map(&emap[d], esum + d * F * Sp, F, Sp);
    if (!rc) rc = make_i8_map(&ehalf[d], esum + d * F * Sp, F, Sp, QN / 2);
  }
  if (rc) {
    cleanup();
    ps_free(sx, s);
    ps_free(sq, s);
    ps_free(e1, s);
    ps_free(e2, s);
    return rc;
  }
  auto grid_of = [&](int64_t nr, int64_t nc) { return (int)std::min<int64_t>(nr * nc, ds->num_sms); };
  // cluster pairs (PS_MOMENTS_MC=0: one CTA per tile)
  const char* mce = getenv("PS_MOMENTS_MC");
  const bool mc = !(mce && mce[0] == '0') && ds->num_sms >= 2;
  static int max_clusters = 0;  // co-resident 2-CTA clusters (GPCs may hold an odd SM count)
  if (!max_clusters) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(ds->num_sms & ~1));
    lc.blockDim = dim3(QTH);
    lc.dynamicSmemBytes = kMomSmem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    lc.attrs = &at;
    lc.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, moment_gemm_mc_kernel, &lc) != cudaSuccess || max_clusters <= 0)
      max_clusters = ds->num_sms / 2;
    cudaGetLastError();
  }
  auto grid_mc_of = [&](int64_t nr, int64_t nc) {
    return 2 * (int)std::min<int64_t>(((nr + 1) / 2) * nc, max_clusters > 0 ? max_clusters : 1);
  };
  // Sxy and n over the upper triangle of the range's tile rows (int8 path)
  const int64_t It0 = lo / QM, nIt = (hi - 1) / QM - It0 + 1;
  auto cross = [&](const CrossMaps& cm, double w, int first, double* o, int32_t* no) {
    const int64_t np = (nIt + 1) / 2, W0 = NTt - It0;
    const int64_t units = np * W0 - np * (np - 1);
    const int g = 2 * (int)std::min<int64_t>(units, max_clusters > 0 ? max_clusters : 1);
    if (gemm_2sm_mode())
      cross_gemm_2sm_kernel<<<g, QTH, kMom2Smem, s>>>(cm, nk, It0, nIt, NTt, rsc, rsc, w, first, o, no, F, -1,
                                                      gemm_2sm_mode() == 2);
    else
      cross_gemm_mc_kernel<<<g, QTH, kMomSmem, s>>>(cm, nk, It0, nIt, NTt, rsc, rsc, w, first, o, no, F, -1);
    PS_LAUNCHED();
  };
  ps_prof_begin("pearson_moments", s);
  if (sxy) {
    CrossMaps cn1;
    cn1.g = 1;
    cn1.a[0] = bmap;
    cn1.b[0] = bmap_half;
    cross(cn1, 1.0, 1, nullptr, nn);  // pair counts n = M M^T
    row_scale_kernel<<<(unsigned)ps_ceil_div(nrows, 256), 256, 0, s>>>(e1, r0, nrows, rsc);
    PS_LAUNCHED();
  }
  const bool b256 = ps_moments_b256(S);
  const int bits = b256 ? 8 : 7;
  if (sxy) {
    // Sxy = 2^(e_i + e_j + 2) sum_{s + t <= 9} 2^-7(s+t) D_s D_t^T from the base-128
    // planes, folded in a fixed order (smallest weights first); the terms with
    // s + t >= 10 are below 2^-55.1 of the row scales (the pair kernel's bound
    // accounts for them)
    moment_digit_kernel<7, kDigits><<<(unsigned)nrows, 256, 0, s>>>(xc, a->ld, S, Sp, e1, 0, r0, F * Sp, dig);
    PS_LAUNCHED();
    int first = 1;
    auto emit = [&](const CrossMaps& cm, double w) {
      cross(cm, w, first, sxy, nullptr);
      first = 0;
    };
    if (sym) {
      digit_sum_kernel<<<(unsigned)nrows, 256, 0, s>>>(dig, F * Sp, Sp, r0, esum);
      PS_LAUNCHED();
      sxy_sym_products(emap, ehalf, amap, ahalf, emit);
    } else {
      sxy_groups(S, amap, ahalf, emit);
    }
  }
  for (int sq_pass = 0; sq_pass < 2; ++sq_pass) {
    double* out = sq_pass ? sq : sx;
    const int32_t* ex = sq_pass ? e2 : e1;
    if (sq_pass || b256 || !sxy) {  // (the base-128 planes of x' are in place after Sxy)
      moment_planes(b256, sq_pass, xc, a->ld, S, Sp, ex, r0, nrows, F * Sp, dig, s);
      PS_LAUNCHED();
    }
    const int nd = moment_digits(b256, sq_pass);  // Sx: its error enters only via Sx^2 / n
    for (int d = nd; d >= 1; --d) {  // least significant digit first (fixed fold order)
      for (int rect = 0; rect < 2; ++rect) {
        const int64_t ri = rect ? I2 : I0, rn = rect ? nI2 : nI, cn = rect ? nJ2 : nJ;
        if (rn <= 0 || cn <= 0) continue;
        if (mc && gemm_2sm_mode())
          moment_gemm_2sm_kernel<<<grid_mc_of(rn, cn), QTH, kMom2Smem, s>>>(amap[d - 1], bmap_half, nk, ri, rn, J0, cn,
                                                                            ex, bits * d - (bits == 8), d == nd ? 1 : 0, out, F,
                                                                            gemm_2sm_mode() == 2);
        else if (mc)
          moment_gemm_mc_kernel<<<grid_mc_of(rn, cn), QTH, kMomSmem, s>>>(amap[d - 1], bmap_half, nk, ri, rn, J0, cn,
                                                                          ex, bits * d - (bits == 8), d == nd ? 1 : 0, out, F);
        else
          moment_gemm_kernel<<<grid_of(rn, cn), QTH, kMomSmem, s>>>(amap[d - 1], bmap, nk, ri, rn, J0, cn, ex,
                                                                    bits * d - (bits == 8), d == nd ? 1 : 0, out, F);
        PS_LAUNCHED();
      }
    }
  }
  ps_prof_end(s);
  cleanup();
  *sx_out = sx;
  *sq_out = sq;
  *e1_out = e1;
  *e2_out = e2;
  return PS_OK;
}

// ---------------------------------------------------------------------------
// Incremental form for ps_run (the contractions follow the input upload): the
// rows of each uploaded chunk get their exponents, both digit-plane sets and
// presence; every tile column block whose rows are complete then runs its
// moment tiles (the new L of the square) and its Sxy / n triangle tiles.  Each
// output tile is produced by exactly one block, in the same digit / product
// order as ps_pearson_moments: bitwise identical results.
struct ps_moments_job {
  const ps_matrix* a = nullptr;
  const double* xc = nullptr;
  int64_t F = 0, S = 0, Sp = 0, NT = 0;
  int nk = 0;
  int8_t *dig = nullptr, *dig2 = nullptr, *pres = nullptr, *esum = nullptr;
  int8_t* dig1b = nullptr;  // base-256 planes of x' (Sx); dig keeps the base-128 planes of Sxy
  bool b256 = false;
  CUtensorMap a1b[kDigits];
  int32_t *e1 = nullptr, *e2 = nullptr;
  double *rsc = nullptr, *sx = nullptr, *sq = nullptr, *sxy = nullptr;
  int32_t* nn = nullptr;
  CUtensorMap a1[kDigits], a1h[kDigits], a2[kDigits], bmap, bmap_half;
  CUtensorMap em[kSymPairs], emh[kSymPairs];  // sum planes (symmetric Sxy)
  int64_t rows_done = 0, cols_done = 0;
  int grid_cap = 1;
};

static void job_release(ps_moments_job* j, cudaStream_t s, bool outputs) {
  ps_free(j->dig, s);
  ps_free(j->dig2, s);
  ps_free(j->esum, s);
  ps_free(j->dig1b, s);
  ps_free(j->pres, s);
  ps_free(j->rsc, s);
  if (outputs) {
    ps_free(j->sx, s);
    ps_free(j->sq, s);
    ps_free(j->e1, s);
    ps_free(j->e2, s);
  }
  delete j;
}

int ps_moments_job_begin(const ps_matrix* a, const double* xc, double* sxy, int32_t* nn, cudaStream_t s,
                         ps_moments_job** out) {
  *out = nullptr;
  ps_moments_job* j = new ps_moments_job();
  j->a = a;
  j->xc = xc;
  j->F = a->F;
  j->S = a->S;
  j->Sp = ps_round_up(std::max<int64_t>(a->S, 1), QKB);
  j->NT = ps_ceil_div(a->F, QM);
  j->nk = (int)(j->Sp / QKB);
  j->sxy = sxy;
  j->nn = nn;
  const int64_t F = j->F, Sp = j->Sp;
  cudaError_t e = ps_alloc(&j->sx, (size_t)(F * F), s);
  if (e == cudaSuccess) e = ps_alloc(&j->sq, (size_t)(F * F), s);
  if (e == cudaSuccess) e = ps_alloc(&j->dig, (size_t)(kDigits * F * Sp), s);
  j->b256 = ps_moments_b256(j->S);
  if (e == cudaSuccess) e = ps_alloc(&j->dig2, (size_t)(moment_digits(j->b256, 1) * F * Sp), s);
  if (e == cudaSuccess && j->b256) e = ps_alloc(&j->dig1b, (size_t)(kSxDigits256 * F * Sp), s);
  if (e == cudaSuccess) e = ps_alloc(&j->pres, (size_t)(F * Sp), s);
  if (e == cudaSuccess && sxy && ps_sxy_sym(j->S)) e = ps_alloc(&j->esum, (size_t)(kSymPairs * F * Sp), s);
  if (e == cudaSuccess) e = ps_alloc(&j->e1, (size_t)F, s);
  if (e == cudaSuccess) e = ps_alloc(&j->e2, (size_t)F, s);
  if (e == cudaSuccess) e = ps_alloc(&j->rsc, (size_t)F, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(moment_gemm_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMomSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(cross_gemm_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMomSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(cross_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMom2Smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(moment_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMom2Smem);
  if (e != cudaSuccess) {
    job_release(j, s, true);
    return ps_cuda_check(e, "pearson moments setup");
  }
  int rc = make_i8_map(&j->bmap, j->pres, F, Sp);
  if (!rc) rc = make_i8_map(&j->bmap_half, j->pres, F, Sp, QN / 2);
  for (int d = 0; d < kDigits && !rc; ++d) {
    rc = make_i8_map(&j->a1[d], j->dig + d * F * Sp, F, Sp);
    if (!rc) rc = make_i8_map(&j->a1h[d], j->dig + d * F * Sp, F, Sp, QN / 2);
    if (!rc && d < moment_digits(j->b256, 1)) rc = make_i8_map(&j->a2[d], j->dig2 + d * F * Sp, F, Sp);
    if (!rc && j->b256 && d < kSxDigits256) rc = make_i8_map(&j->a1b[d], j->dig1b + d * F * Sp, F, Sp);
  }
  for (int d = 0; d < kSymPairs && !rc && j->esum; ++d) {
    rc = make_i8_map(&j->em[d], j->esum + d * F * Sp, F, Sp);
    if (!rc) rc = make_i8_map(&j->emh[d], j->esum + d * F * Sp, F, Sp, QN / 2);
  }
  if (rc) {
    job_release(j, s, true);
    return rc;
  }
  ps_device_state* ds = ps_state();
  int mcl = 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(ds->num_sms & ~1));
  lc.blockDim = dim3(QTH);
  lc.dynamicSmemBytes = kMomSmem;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 2;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  lc.attrs = &at;
  lc.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&mcl, moment_gemm_mc_kernel, &lc) != cudaSuccess || mcl <= 0)
    mcl = ds->num_sms / 2;
  cudaGetLastError();
  j->grid_cap = mcl;
  *out = j;
  return PS_OK;
}

// rows [rows_done, r1): exponents, both digit-plane sets, presence, Sxy row scales
int ps_moments_job_rows(ps_moments_job* j, int64_t r1, cudaStream_t s) {
  r1 = std::min<int64_t>(r1, j->F);
  const int64_t r0 = j->rows_done, n = r1 - r0;
  if (n <= 0) return PS_OK;
  const ps_matrix* a = j->a;
  moment_scale_kernel<<<(unsigned)n, 256, 0, s>>>(j->xc, a->ld, j->S, r0, j->e1, j->e2);
  PS_LAUNCHED();
  presence_i8_kernel<<<(unsigned)n, 256, 0, s>>>(a->d_mask, a->W, j->S, j->Sp, j->pres, r0);
  PS_LAUNCHED();
  if (j->sxy || !j->b256) {
    moment_digit_kernel<7, kDigits><<<(unsigned)n, 256, 0, s>>>(j->xc, a->ld, j->S, j->Sp, j->e1, 0, r0, j->F * j->Sp,
                                                                j->dig);
    PS_LAUNCHED();
  }
  if (j->b256) {
    moment_planes(true, 0, j->xc, a->ld, j->S, j->Sp, j->e1, r0, n, j->F * j->Sp, j->dig1b, s);
    PS_LAUNCHED();
  }
  moment_planes(j->b256, 1, j->xc, a->ld, j->S, j->Sp, j->e2, r0, n, j->F * j->Sp, j->dig2, s);
  PS_LAUNCHED();
  if (j->esum) {
    digit_sum_kernel<<<(unsigned)n, 256, 0, s>>>(j->dig, j->F * j->Sp, j->Sp, r0, j->esum);
    PS_LAUNCHED();
  }
  row_scale_kernel<<<(unsigned)ps_ceil_div(n, 256), 256, 0, s>>>(j->e1, r0, n, j->rsc);
  PS_LAUNCHED();
  j->rows_done = r1;
  return PS_OK;
}

// tile columns [cols_done, J1) (their rows prepared): the new L of the moment
// square and the column block of the Sxy / n triangle
int ps_moments_job_cols(ps_moments_job* j, int64_t J1, cudaStream_t s) {
  J1 = std::min<int64_t>(J1, j->NT);
  const int64_t J0 = j->cols_done;
  if (J1 <= J0) return PS_OK;
  auto gmc = [&](int64_t units) { return 2 * (int)std::min<int64_t>(std::max<int64_t>(units, 1), j->grid_cap); };
  ps_prof_begin("pearson_moments", s);
  for (int pass = 0; pass < 2; ++pass) {
    double* out = pass ? j->sq : j->sx;
    const int32_t* ex = pass ? j->e2 : j->e1;
    const int nd = moment_digits(j->b256, pass), bits = j->b256 ? 8 : 7;
    for (int d = nd; d >= 1; --d) {
      const CUtensorMap& am = pass ? j->a2[d - 1] : j->b256 ? j->a1b[d - 1] : j->a1[d - 1];
      // rows [0, J1) x columns [J0, J1), then rows [J0, J1) x columns [0, J0)
      for (int rect = 0; rect < 2; ++rect) {
        const int64_t ri = rect ? J0 : 0, rn = rect ? J1 - J0 : J1;
        const int64_t ci = rect ? 0 : J0, cn = rect ? J0 : J1 - J0;
        if (rn <= 0 || cn <= 0) continue;
        if (gemm_2sm_mode())
          moment_gemm_2sm_kernel<<<gmc(((rn + 1) / 2) * cn), QTH, kMom2Smem, s>>>(
              am, j->bmap_half, j->nk, ri, rn, ci, cn, ex, bits * d - (bits == 8), d == nd ? 1 : 0, out, j->F, gemm_2sm_mode() == 2);
        else
          moment_gemm_mc_kernel<<<gmc(((rn + 1) / 2) * cn), QTH, kMomSmem, s>>>(am, j->bmap_half, j->nk, ri, rn, ci, cn,
                                                                                ex, bits * d - (bits == 8), d == nd ? 1 : 0, out, j->F);
        PS_LAUNCHED();
      }
    }
  }
  if (j->sxy) {
    auto half_sum = [](int64_t x) -> int64_t { return x <= 0 ? 0 : (x / 2) * ((x - 1) / 2); };
    const int64_t units = (J1 - J0) + half_sum(J1) - half_sum(J0);
    auto cross = [&](const CrossMaps& cm, double w, int first, double* o, int32_t* no) {
      if (gemm_2sm_mode())
        cross_gemm_2sm_kernel<<<gmc(units), QTH, kMom2Smem, s>>>(cm, j->nk, 0, J1, J1, j->rsc, j->rsc, w, first, o, no,
                                                                 j->F, J0, gemm_2sm_mode() == 2);
      else
        cross_gemm_mc_kernel<<<gmc(units), QTH, kMomSmem, s>>>(cm, j->nk, 0, J1, J1, j->rsc, j->rsc, w, first, o, no,
                                                               j->F, J0);
      PS_LAUNCHED();
    };
    CrossMaps cn1;
    cn1.g = 1;
    cn1.a[0] = j->bmap;
    cn1.b[0] = j->bmap_half;
    cross(cn1, 1.0, 1, nullptr, j->nn);
    int first = 1;
    auto emit = [&](const CrossMaps& cm, double w) {
      cross(cm, w, first, j->sxy, nullptr);
      first = 0;
    };
    if (j->esum) sxy_sym_products(j->em, j->emh, j->a1, j->a1h, emit);
    else sxy_groups(j->S, j->a1, j->a1h, emit);
  }
  ps_prof_end(s);
  j->cols_done = J1;
  return PS_OK;
}

int ps_moments_job_end(ps_moments_job* j, double** sx, double** sq, int32_t** e1, int32_t** e2, cudaStream_t s) {
  *sx = j->sx;
  *sq = j->sq;
  *e1 = j->e1;
  *e2 = j->e2;
  job_release(j, s, false);
  return PS_OK;
}

void ps_moments_job_abort(ps_moments_job* j, cudaStream_t s) {
  if (j) job_release(j, s, true);
}
