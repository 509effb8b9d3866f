// ps_chi2.cu -- all-pairs chi-squared: contingency tables as one int8 GEMM.
//
// Replaces _chi2_block -> _chi2_rows -> _chi2_finish (engine.py:208-242,
// categorical.py:31-94).  Every feature f with c_f declared levels contributes
// c_f rows to a one-hot matrix O (row off_f + a, sample s) = 1 iff f is present
// at s with label a.  All contingency tables at once are C = O O^T
// (int8 x int8 -> int32, exact): the table of (g, h) is the c_g x c_h block at
// (off_g, off_h).  The GEMM runs on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM, TMA-fed) over upper-triangular
// 256 x 256 tiles of C, stream-K scheduled (see below).  The epilogue (one thread per pair) replays
// the reference's NaN rules and its i-major chi-square loop in the same fp64
// operation order, so chi2 / phi / V are bit-identical; p = chi2_sf(chi2, dof).
//
// Algorithmic work: 2 k_g k_h int8 ops per pair-sample.
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include "ps_tc05.cuh"
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdlib>
#include <vector>

namespace {


// ----------------------------------------------------------------- one-hot
// 16-bit codes (category counts above 254): 8 samples per thread per step
__global__ void onehot16_kernel(const uint16_t* __restrict__ codes, int64_t ldc, const int32_t* __restrict__ row_feat,
                                const int32_t* __restrict__ row_level, int64_t R, int64_t Sp, int64_t S,
                                uint8_t* __restrict__ O) {
  const int64_t r = blockIdx.x;
  uint8_t* out = O + r * Sp;
  if (r >= R) {
    for (int64_t s = threadIdx.x * 16; s < Sp; s += blockDim.x * 16)
      *reinterpret_cast<uint4*>(out + s) = make_uint4(0, 0, 0, 0);
    return;
  }
  const uint16_t lev = (uint16_t)row_level[r];
  const uint16_t* c = codes + row_feat[r] * ldc;
  for (int64_t s = threadIdx.x * 8; s < Sp; s += blockDim.x * 8) {
    uint32_t w[2] = {0u, 0u};
    for (int q = 0; q < 8; ++q) {
      const int64_t sq = s + q;
      if (sq < S && c[sq] == lev) w[q >> 2] |= 1u << (8 * (q & 3));
    }
    *reinterpret_cast<uint2*>(out + s) = make_uint2(w[0], w[1]);
  }
}

__global__ void onehot_kernel(const uint8_t* __restrict__ codes, int64_t ldc, const int32_t* __restrict__ row_feat,
                              const int32_t* __restrict__ row_level, int64_t R, int64_t Sp, int64_t S,
                              uint8_t* __restrict__ O) {
  // one CTA per O row; 16 samples per thread per step
  const int64_t r = blockIdx.x;
  uint8_t* out = O + r * Sp;
  if (r >= R) {
    for (int64_t s = threadIdx.x * 16; s < Sp; s += blockDim.x * 16)
      *reinterpret_cast<uint4*>(out + s) = make_uint4(0, 0, 0, 0);
    return;
  }
  const int f = row_feat[r];
  const uint8_t lev = (uint8_t)row_level[r];
  const uint8_t* c = codes + f * ldc;
  constexpr int kU = 4;  // 16-byte loads in flight per thread
  for (int64_t s0 = threadIdx.x * 16; s0 < Sp; s0 += blockDim.x * 16 * kU) {
  uint4 cvu[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int64_t s = s0 + (int64_t)u * blockDim.x * 16;
    cvu[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (s < ldc) cvu[u] = *reinterpret_cast<const uint4*>(c + s);
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int64_t s = s0 + (int64_t)u * blockDim.x * 16;
    if (s >= Sp) break;
    const uint4 cv = cvu[u];
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
    uint32_t w[4];
    const uint32_t lev4 = 0x01010101u * lev;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // byte-wise code == lev (SIMD compare: 0xFF per equal byte) -> 0/1 bytes
      uint32_t v = __vcmpeq4(cw[q], lev4) & 0x01010101u;
      const int64_t sq = s + q * 4;
      if (sq + 4 > S) {  // samples past S are absent
        const int64_t keep = S - sq;
        v = keep <= 0 ? 0u : v & (0xFFFFFFFFu >> (8 * (4 - keep)));
      }
      w[q] = v;
    }
    *reinterpret_cast<uint4*>(out + s) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  }
}

// ----------------------------------------------------------------- tcgen05 GEMM
// C = O O^T on tcgen05.mma kind::i8.  A CTA tile is 256 x 256: two M = 128
// accumulators (TMEM columns 0-255 and 256-511) share one 256-row B operand,
// so each 128-byte K step moves 64 KB through TMA for 8 MMAs -- half the L2
// traffic per MMA of a 128 x 256 tile (the contraction is L2-bandwidth bound
// at that size).  Operands are TMA-loaded (SWIZZLE_128B, K-major 8-row x
// 128-byte atoms) into a 3-stage ring; one elected thread issues the MMAs and
// commits each stage to its `empty` mbarrier.
//
// Stream-K schedule: the (tile, K step) iteration space of all upper
// triangular tiles is cut into gridDim.x equal contiguous ranges (one
// persistent CTA per SM), so every SM does the same MMA work regardless of
// how many tiles there are.  A CTA's range splits into segments at tile
// boundaries; after each segment the 4 epilogue warps drain both
// accumulators with tcgen05.ld and add them into C (fp32 red.global.add.v4:
// counts < 2^24 are exact in fp32, and integer-valued adds commute, so the
// result does not depend on the split).  C must be zeroed first.
//
// Warp roles: warps 0-3 epilogue (TMEM lanes 32w..32w+31), warp 4 TMA
// producer, warp 5 MMA issuer.
constexpr int TM = 256, TN = 256, TKB = 128;  // CTA tile rows, cols, K bytes per stage
constexpr int TSTAGES = 3;
constexpr int TA_BYTES = TM * TKB, TB_BYTES = TN * TKB;
constexpr int TSTAGE_BYTES = TA_BYTES + TB_BYTES;
constexpr size_t kTc05Smem = (size_t)TSTAGES * TSTAGE_BYTES + 1024;
constexpr int TTH_WS = 192;

// Partial tables are added into C: fp32 (one vector red per 4 cells) while
// every count is < 2^24 -- exact, and integer-valued adds commute -- or u32
// (scalar reds) when the sample count could reach 2^24 (categorical.py:84-93
// keeps int64 tables; no count ever exceeds S < 2^32).
__device__ __forceinline__ void red_add4(float* addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"((float)(int)a), "f"((float)(int)b),
               "f"((float)(int)c), "f"((float)(int)d)
               : "memory");
}
__device__ __forceinline__ void red_add4(uint32_t* addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(addr), "r"(a) : "memory");
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(addr + 1), "r"(b) : "memory");
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(addr + 2), "r"(c) : "memory");
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(addr + 3), "r"(d) : "memory");
}

// C holds the rows [crow0, crow0 + band) of the table matrix (a row band:
// scratch stays bounded for wide matrices)
template <typename Acc>
__global__ void __launch_bounds__(TTH_WS, 1)
onehot_gemm_sk_kernel(const __grid_constant__ CUtensorMap tmap, int nk, int kbase, const int2* __restrict__ tiles,
                      int64_t ntiles, Acc* __restrict__ C, int64_t ldC, int64_t crow0) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[TSTAGES], empty[TSTAGES], accfull, accempty;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's share of the (tile, K step) iteration space
  const int64_t total = ntiles * nk;
  const int64_t i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, 512);
  if (tid == 32) {
    for (int i = 0; i < TSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 1);
    }
    tc05::mbar_init(&accfull, 1);
    tc05::mbar_init(&accempty, 128);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32) tc05::prefetch_tmap(&tmap);
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      for (int64_t it = i0; it < i1; ++it) {
        const int64_t q = it - i0;
        const int st = (int)(q % TSTAGES), n = (int)(q / TSTAGES);
        const int2 t = tiles[it / nk];
        const int kc = (int)(it % nk);
        if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
        const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
        tc05::mbar_arrive_expect_tx(&full[st], TSTAGE_BYTES);
        tc05::tma_load_2d(sa, &tmap, (kbase + kc) * TKB, t.x * TM, &full[st]);
        tc05::tma_load_2d(sb, &tmap, (kbase + kc) * TKB, t.y * TN, &full[st]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(128, TN, true);
      int seg = 0;
      for (int64_t it = i0; it < i1; ++it) {
        const int64_t q = it - i0;
        const int st = (int)(q % TSTAGES), n = (int)(q / TSTAGES);
        const int kc = (int)(it % nk);
        const bool first = it == i0 || kc == 0;
        const bool last = it + 1 == i1 || kc == nk - 1;
        if (first && seg > 0) {  // the epilogue has drained the previous segment
          tc05::mbar_wait(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
        tc05::fence_after_sync();
        const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
#pragma unroll
        for (int kk = 0; kk < TKB / 32; ++kk) {
          const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
          const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
          tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
          tc05::mma_i8(tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * TKB + kk * 32), bd, idesc, acc);
        }
        tc05::commit(&empty[st]);
        if (last) {
          tc05::commit(&accfull);
          ++seg;
        }
      }
    }
  } else {
    // epilogue warps 0-3: one pass per segment, in the MMA issuer's order
    int seg = 0;
    for (int64_t it = i0; it < i1;) {
      const int64_t tile = it / nk;
      const int64_t seg_end = std::min<int64_t>(i1, (tile + 1) * nk);
      const int2 t = tiles[tile];
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int64_t r = (int64_t)t.x * TM + half * 128 + warp * 32 + lane;
        Acc* crow = C + (r - crow0) * ldC + (int64_t)t.y * TN;
#pragma unroll 1
        for (int cc = 0; cc < TN / 32; ++cc) {
          uint32_t v[32];
          tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
#pragma unroll
          for (int j = 0; j < 32; j += 4) red_add4(crow + cc * 32 + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
      tc05::fence_before_sync();
      tc05::mbar_arrive(&accempty);
      ++seg;
      it = seg_end;
    }
  }
  tc05::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc05::tmem_dealloc(tmem, 512);
}

// Cluster-pair variant: the two CTAs of a cluster walk the same (unit, K step)
// range, a unit being two tiles that share an operand -- both in one tile row
// (same A rows) or both in the last tile column (same B rows).  Each CTA TMA-
// loads half of the shared operand and multicasts it to both CTAs, plus its
// own tile's other operand: 48 KB of L2 reads per CTA per K step instead of
// 64 KB.  A stage is reused only after both CTAs' MMAs released it (the MMA
// commit arrives on the `empty` barrier of both CTAs).  An unpaired tile runs
// with a dummy partner that only contributes its half of the shared operand.
//   unit = (I0, J0, I1, J1); I0 == I1: A shared; I1 < 0: dummy second tile.
constexpr int THALF = TA_BYTES / 2;  // 128 rows x 128 B
template <typename Acc>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TTH_WS, 1)
onehot_gemm_mc_kernel(const __grid_constant__ CUtensorMap tmap, int nk, int kbase, const int4* __restrict__ units,
                      int64_t nunits, Acc* __restrict__ C, int64_t ldC, int64_t crow0) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[TSTAGES], empty[TSTAGES], accfull, accempty;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)tc05::cluster_ctarank();
  const int64_t ncl = gridDim.x / 2, cl = blockIdx.x / 2;
  const int64_t total = nunits * nk;
  const int64_t i0 = total * cl / ncl, i1 = total * (cl + 1) / ncl;
  // A cluster's range [i0, i1) of the (unit, k) iterations splits into
  // segments at unit boundaries; they are walked LAST FIRST.  Ranges are
  // equal (L = i1 - i0), so cluster c's last segment starts at k = 0 at time 0
  // and its first one, entered when the last ends, is exactly L mod nk steps
  // behind: at any time every cluster is within L mod nk k-steps of the same
  // k, and the one-hot slab in flight stays L2-resident (walked first to last,
  // the ranges start at scattered k and the whole operand cycles through L2).
  auto seg_start = [&](int64_t se) -> int64_t { return std::max<int64_t>(i0, ((se - 1) / nk) * nk); };
  auto tile_of = [&](const int4& u, int& I, int& J) -> bool {  // false: dummy
    I = rank ? u.z : u.x;
    J = rank ? u.w : u.y;
    return I >= 0;
  };

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, 512);
  if (tid == 32) {
    for (int i = 0; i < TSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 2);  // both CTAs' MMA commits
    }
    tc05::mbar_init(&accfull, 1);
    tc05::mbar_init(&accempty, 128);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32) tc05::prefetch_tmap(&tmap);
  tc05::fence_before_sync();
  tc05::cluster_sync();  // barriers initialised in both CTAs before any multicast
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      int64_t q = 0;
      for (int64_t se = i1; se > i0;) {  // segments last to first (see seg_start)
        const int64_t ss = seg_start(se);
        for (int64_t it = ss; it < se; ++it, ++q) {
        const int st = (int)(q % TSTAGES), n = (int)(q / TSTAGES);
        const int4 u = units[it / nk];
        const int kx = (kbase + (int)(it % nk)) * TKB;
        int I, J;
        const bool own = tile_of(u, I, J);
        const bool shareA = u.z < 0 || u.x == u.z;
        if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
        const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
        tc05::mbar_arrive_expect_tx(&full[st], own ? TSTAGE_BYTES : TA_BYTES);
        const int shared_row = (shareA ? u.x : u.y) * TM + rank * 128;
        tc05::tma_load_2d_mc((shareA ? sa : sb) + rank * THALF, &tmap, kx, shared_row, &full[st], (uint16_t)3);
        if (own) {
          const uint32_t od = shareA ? sb : sa;
          const int orow = (shareA ? J : I) * TM;
          tc05::tma_load_2d(od, &tmap, kx, orow, &full[st]);
          tc05::tma_load_2d(od + THALF, &tmap, kx, orow + 128, &full[st]);
        }
        }
        se = ss;
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(128, TN, true);
      int seg = 0;
      int64_t q = 0;
      for (int64_t se = i1; se > i0;) {
        const int64_t ss = seg_start(se);
        for (int64_t it = ss; it < se; ++it, ++q) {
        const int st = (int)(q % TSTAGES), n = (int)(q / TSTAGES);
        int I, J;
        const bool own = tile_of(units[it / nk], I, J);
        const bool first = it == ss;
        const bool last = it + 1 == se;
        if (own && first && seg > 0) {  // the epilogue has drained the previous segment
          tc05::mbar_wait(&accempty, (uint32_t)((seg - 1) & 1));
          tc05::fence_after_sync();
        }
        tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
        tc05::fence_after_sync();
        if (own) {
          const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
#pragma unroll
          for (int kk = 0; kk < TKB / 32; ++kk) {
            const uint64_t bd = tc05::sw128_kmajor_desc(sb + kk * 32);
            const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
            tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), bd, idesc, acc);
            tc05::mma_i8(tmem + 256, tc05::sw128_kmajor_desc(sa + 128 * TKB + kk * 32), bd, idesc, acc);
          }
        }
        tc05::commit_mc(&empty[st], (uint16_t)3);
        if (own && last) {
          tc05::commit(&accfull);
          ++seg;
        }
        }
        se = ss;
      }
    }
  } else {
    // epilogue warps 0-3: one pass per segment of an own tile, in the MMA issuer's order
    int seg = 0;
    for (int64_t se = i1; se > i0;) {
      const int64_t ss = seg_start(se);
      const int64_t unit = ss / nk;
      se = ss;
      int I, J;
      if (!tile_of(units[unit], I, J)) continue;
      tc05::mbar_wait(&accfull, (uint32_t)(seg & 1));
      tc05::fence_after_sync();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int64_t r = (int64_t)I * TM + half * 128 + warp * 32 + lane;
        Acc* crow = C + (r - crow0) * ldC + (int64_t)J * TN;
#pragma unroll 1
        for (int cc = 0; cc < TN / 32; ++cc) {
          uint32_t v[32];
          tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(half * 256 + cc * 32), v);
#pragma unroll
          for (int j = 0; j < 32; j += 4) red_add4(crow + cc * 32 + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
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

// ----------------------------------------------------------------- epilogue
__device__ __forceinline__ void put(double* o, int64_t F, int64_t g, int64_t h, double v) {
  if (o) {
    o[g * F + h] = v;
    o[h * F + g] = v;
  }
}

// pairs (x, y >= x) with x in [lo, g): rows of the upper triangle before row g
__device__ __forceinline__ int64_t upper_before(int64_t g, int64_t lo, int64_t F) {
  return (g - lo) * F - (g * (g - 1) - lo * (lo - 1)) / 2;
}

// One thread per pair (g <= h, enumerated over the upper triangle of rows
// [lo, hi): no idle threads): categorical.py:31-74 in the same op order.
// Row / column sums are cached for up to CM levels (CM == 0, category counts
// above 256: per-thread global scratch slices).  The table is read from C.
template <int CM, typename Acc>
__global__ void chi2_finish_kernel(const Acc* __restrict__ C, int64_t ldC, int64_t crow0,
                                   const int32_t* __restrict__ off, const int32_t* __restrict__ cat,
                                   int64_t F, int64_t lo, int64_t hi, double* __restrict__ stat,
                                   double* __restrict__ pout, double* __restrict__ phi_out,
                                   double* __restrict__ v_out, int* __restrict__ err, long long* big = nullptr,
                                   int cmax_big = 0) {
  const int64_t total = upper_before(hi, lo, F);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = lo, b = hi - 1;  // last row g with upper_before(g) <= it
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (upper_before(mid, lo, F) <= it) a = mid;
      else b = mid - 1;
    }
    const int64_t g = a, h = g + (it - upper_before(g, lo, F));
    const int cg = cat[g], ch = cat[h];
    const bool diag = g == h;
    const Acc* T = C + ((int64_t)off[g] - crow0) * ldC + off[h];  // exact integer counts
    // the diagonal pair's table is diagonal; its lower half lies outside the
    // computed upper-triangular tiles, so read only the diagonal
    auto tab = [&](int i, int j) -> long long {
      if (diag && i != j) return 0;
      return (long long)T[(int64_t)i * ldC + j];
    };
    double chi2 = PS_NAN, p = PS_NAN, phi = PS_NAN, v = PS_NAN;
    long long n = 0;
    bool empty;
    double acc = 0.0;
    {
      // row / column sums: per-thread arrays (CM > 0) or global scratch slices
      long long rs_l[CM > 0 ? CM : 1], cs_l[CM > 0 ? CM : 1];
      long long* rs = CM > 0 ? rs_l : big + (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 2 * cmax_big;
      long long* cs = CM > 0 ? cs_l : rs + cmax_big;
      for (int j = 0; j < ch; ++j) cs[j] = 0;
      for (int i = 0; i < cg; ++i) {
        long long r = 0;
        for (int j = 0; j < ch; ++j) {
          const long long t = tab(i, j);
          r += t;
          cs[j] += t;
        }
        rs[i] = r;
        n += r;
      }
      empty = n == 0;
      for (int i = 0; i < cg; ++i) empty |= rs[i] == 0;
      for (int j = 0; j < ch; ++j) empty |= cs[j] == 0;
      if (!empty) {
        const double dn = (double)n;
        for (int i = 0; i < cg; ++i)
          for (int j = 0; j < ch; ++j) {
            const double expected = (double)(rs[i] * cs[j]) / dn;
            if (expected > 0.0) {
              const double diff = (double)tab(i, j) - expected;
              acc += diff * diff / expected;
            }
          }
      }
    }
    if (!empty) {
      const double dn = (double)n;
      chi2 = acc;
      phi = sqrt(acc / dn);
      const int cmin = cg < ch ? cg : ch;
      if (cmin >= 2) {
        const double dof = ((double)cg - 1.0) * ((double)ch - 1.0);
        p = psf::chi2_sf(acc, dof, err);
        v = sqrt(acc / (dn * ((double)cmin - 1.0)));
      }
    }
    put(stat, F, g, h, chi2);
    put(pout, F, g, h, p);
    put(phi_out, F, g, h, phi);
    put(v_out, F, g, h, v);
  }
}

// LabelOutOfRange when a present out-of-range label meets a jointly present
// partner inside the evaluated pairs (categorical.py:84-91): rows [lo, hi)
// always meet themselves on the diagonal; rows >= hi only where some row of
// [lo, hi) is present.
// LabelOutOfRange (categorical.py:84-91): a bad present label of a feature f
// that meets a computed pair -- every f in [lo, hi) (its diagonal pair), or
// f >= hi where some row g in [lo, hi) is present at the same sample.
// Grid: x over mask words, y over chunks of kCheckRows features; the OR of the
// row masks is only formed when a chunk actually holds a bad label.
constexpr int kCheckRows = 32;
__global__ void label_check_kernel(const uint32_t* __restrict__ bad, const uint32_t* __restrict__ mask,
                                   int64_t W, int64_t F, int64_t lo, int64_t hi, int* __restrict__ err) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W) return;
  const int64_t f0 = lo + (int64_t)blockIdx.y * kCheckRows, f1 = min(F, f0 + kCheckRows);
  uint32_t in_rows = 0, beyond = 0;
  for (int64_t f = f0; f < f1; ++f) {
    const uint32_t b = bad[f * W + w];
    if (f < hi) in_rows |= b;
    else beyond |= b;
  }
  if (in_rows) {
    ps_raise(err, PS_ERR_LABEL_OUT_OF_RANGE);
    return;
  }
  if (!beyond) return;
  uint32_t col = 0;
  for (int64_t g = lo; g < hi && !(col & beyond); ++g) col |= mask[g * W + w];
  if (col & beyond) ps_raise(err, PS_ERR_LABEL_OUT_OF_RANGE);
}

}  // namespace

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// 2-D uint8 tensor map over the one-hot matrix: rows x Sp bytes, box TKB x rows_box, 128-B swizzle
static int make_onehot_map(CUtensorMap* map, const uint8_t* O, int64_t rows, int64_t Sp, uint32_t rows_box) {
  auto enc = tensor_map_encoder();
  if (!enc) return ps_fail(PS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)Sp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Sp};
  cuuint32_t box[2] = {(cuuint32_t)TKB, rows_box};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(O), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ps_fail(PS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return PS_OK;
}

// One row band of the contingency tables: the features [ga, gb) of the range,
// their table rows (C rows [crow0, crow0 + band)) against every column tile
// right of the diagonal, then the per-pair finish.
template <typename Acc>
static int chi2_band(ps_matrix* a, const std::vector<int32_t>& off, int64_t ga, int64_t gb, int64_t Rp,
                     const CUtensorMap& map, int nk_all, const int32_t* d_off, double* stat, double* p, double* phi,
                     double* v, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  const int64_t F = a->F;
  const int64_t R = off[F];
  const int64_t I0 = off[ga] / TM;
  const int64_t I1 = std::max<int64_t>(I0, (off[gb] - 1) / TM);
  const int64_t crow0 = I0 * TM, band = (I1 - I0 + 1) * TM;
  Acc* C = nullptr;
  PS_CUDA(ps_alloc(&C, (size_t)(band * Rp), s));
  PS_CUDA(cudaMemsetAsync(C, 0, sizeof(Acc) * band * Rp, s));
  std::vector<int2> tl;
  if (R > 0)
    for (int64_t I = I0; I <= I1; ++I)
      for (int64_t J = (I * TM) / TN; J < Rp / TN; ++J) tl.push_back(make_int2((int)I, (int)J));
  int2* d_tiles = nullptr;
  int4* d_units = nullptr;
  if (!tl.empty()) {
    PS_CUDA(ps_alloc(&d_tiles, tl.size(), s));
    PS_CUDA(cudaMemcpyAsync(d_tiles, tl.data(), sizeof(int2) * tl.size(), cudaMemcpyHostToDevice, s));
    // cluster pairs (default; PS_CHI2_MC=0: one CTA per tile stream)
    const char* mce = getenv("PS_CHI2_MC");
    const bool mc = !(mce && mce[0] == '0') && ds->num_sms >= 2;
    std::vector<int4> un;
    if (mc) {  // tiles of one row in pairs (A shared); rows' last tiles paired by column (B shared)
      std::vector<int2> left;
      for (size_t i = 0; i < tl.size();) {
        size_t e = i;
        while (e < tl.size() && tl[e].x == tl[i].x) ++e;
        size_t k = i;
        for (; k + 1 < e; k += 2) un.push_back(make_int4(tl[k].x, tl[k].y, tl[k + 1].x, tl[k + 1].y));
        if (k < e) left.push_back(tl[k]);
        i = e;
      }
      size_t k = 0;
      for (; k + 1 < left.size(); k += 2) {
        if (left[k].y == left[k + 1].y)
          un.push_back(make_int4(left[k].x, left[k].y, left[k + 1].x, left[k + 1].y));
        else {
          un.push_back(make_int4(left[k].x, left[k].y, -1, -1));
          un.push_back(make_int4(left[k + 1].x, left[k + 1].y, -1, -1));
        }
      }
      if (k < left.size()) un.push_back(make_int4(left[k].x, left[k].y, -1, -1));
      PS_CUDA(ps_alloc(&d_units, un.size(), s));
      PS_CUDA(cudaMemcpyAsync(d_units, un.data(), sizeof(int4) * un.size(), cudaMemcpyHostToDevice, s));
    }
    PS_CUDA(cudaFuncSetAttribute(mc ? (const void*)onehot_gemm_mc_kernel<Acc> : (const void*)onehot_gemm_sk_kernel<Acc>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTc05Smem));
    // K phases: the one-hot operand (Rp x Sp bytes) is streamed through L2 in
    // slabs that fit it, all CTAs working inside the same slab (stream-K
    // spreads CTAs over K, which thrashes L2 when O is larger than it)
    const int64_t Sp = (int64_t)nk_all * TKB;
    const int64_t slab_budget = 96ll << 20;  // L2 is 126 MB
    // (cluster pairs read 25% less through L2: one pass over K measured
    // fastest there, 0.187 vs 0.212 ms in two phases at config 3)
    int phases = (int)std::max<int64_t>(1, ps_ceil_div(Rp * Sp, mc ? 2 * slab_budget : slab_budget));
    if (const char* e = getenv("PS_CHI2_PHASES")) phases = std::max(1, atoi(e));  // tuning override
    phases = std::min(phases, nk_all);
    ps_prof_begin("chi2_gemm", s);
    for (int ph = 0; ph < phases; ++ph) {
      const int kb0 = (int)((int64_t)nk_all * ph / phases), kb1 = (int)((int64_t)nk_all * (ph + 1) / phases);
      const int nk = kb1 - kb0;
      if (mc) {
        static int max_clusters = 0;  // co-resident 2-CTA clusters (GPCs may hold an odd SM count)
        if (!max_clusters) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3((unsigned)(ds->num_sms & ~1));
          lc.blockDim = dim3(TTH_WS);
          lc.dynamicSmemBytes = kTc05Smem;
          cudaLaunchAttribute at;
          at.id = cudaLaunchAttributeClusterDimension;
          at.val.clusterDim.x = 2;
          at.val.clusterDim.y = 1;
          at.val.clusterDim.z = 1;
          lc.attrs = &at;
          lc.numAttrs = 1;
          if (cudaOccupancyMaxActiveClusters(&max_clusters, onehot_gemm_mc_kernel<Acc>, &lc) != cudaSuccess ||
              max_clusters <= 0)
            max_clusters = ds->num_sms / 2;
          cudaGetLastError();
        }
        const int64_t iters = (int64_t)un.size() * nk;
        const int grid = 2 * (int)std::min<int64_t>(iters, max_clusters);
        onehot_gemm_mc_kernel<Acc><<<(unsigned)grid, TTH_WS, kTc05Smem, s>>>(map, nk, kb0, d_units,
                                                                             (int64_t)un.size(), C, Rp, crow0);
      } else {
        const int64_t iters = (int64_t)tl.size() * nk;
        const int grid = (int)std::min<int64_t>(iters, ds->num_sms);
        onehot_gemm_sk_kernel<Acc><<<(unsigned)grid, TTH_WS, kTc05Smem, s>>>(map, nk, kb0, d_tiles,
                                                                             (int64_t)tl.size(), C, Rp, crow0);
      }
      PS_LAUNCHED();
    }
    ps_prof_end(s);
  }
  const int64_t total = (gb - ga) * F - ((gb * (gb - 1)) - (ga * (ga - 1))) / 2;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ps_ceil_div(total, 128), (int64_t)ds->num_sms * 16));
  long long* big = nullptr;
  auto fin = [&](auto kern) {
    kern<<<blocks, 128, 0, s>>>(C, Rp, crow0, d_off, a->d_cat, F, ga, gb, stat, p, phi, v, ds->d_err, nullptr, 0);
  };
  if (a->cmax <= 16) {
    fin(chi2_finish_kernel<16, Acc>);
  } else {
    const int bb = ds->num_sms * 2;
    PS_CUDA(ps_alloc(&big, (size_t)bb * 128 * 2 * a->cmax, s));
    chi2_finish_kernel<0, Acc><<<bb, 128, 0, s>>>(C, Rp, crow0, d_off, a->d_cat, F, ga, gb, stat, p, phi, v, ds->d_err,
                                                  big, a->cmax);
  }
  PS_LAUNCHED();
  ps_free(big, s);
  ps_free(C, s);
  ps_free(d_tiles, s);
  ps_free(d_units, s);
  return PS_OK;
}

int ps_chi2_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* phi, double* v,
                cudaStream_t s) {
  const int64_t F = a->F, S = a->S;
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(F, hi);
  if (hi <= lo || (!stat && !p && !phi && !v)) return PS_OK;
  ps_device_state* ds = ps_state();
  // one-hot row layout (host: category counts are host-resident)
  std::vector<int32_t> off(F + 1, 0), cat32(F);
  for (int64_t f = 0; f < F; ++f) {
    cat32[f] = (int32_t)a->h_cat[f];
    off[f + 1] = off[f] + cat32[f];
  }
  const int64_t R = off[F];
  const int64_t Rp = std::max<int64_t>(TN, ps_round_up(R, TN));
  const int64_t Sp = ps_round_up(S, TKB);
  std::vector<int32_t> row_feat(R), row_level(R);
  for (int64_t f = 0; f < F; ++f)
    for (int32_t l = 0; l < cat32[f]; ++l) {
      row_feat[off[f] + l] = (int32_t)f;
      row_level[off[f] + l] = l;
    }
  uint8_t* O = nullptr;
  int32_t *d_off = nullptr, *d_rf = nullptr, *d_rl = nullptr;
  PS_CUDA(ps_alloc(&O, (size_t)(Rp * Sp), s));
  PS_CUDA(ps_alloc(&d_off, (size_t)(F + 1), s));
  PS_CUDA(ps_alloc(&d_rf, (size_t)std::max<int64_t>(R, 1), s));
  PS_CUDA(ps_alloc(&d_rl, (size_t)std::max<int64_t>(R, 1), s));
  PS_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * (F + 1), cudaMemcpyHostToDevice, s));
  if (R > 0) {
    PS_CUDA(cudaMemcpyAsync(d_rf, row_feat.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaMemcpyAsync(d_rl, row_level.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
  }
  {
    const int64_t W = a->W;
    const dim3 grid((unsigned)ps_ceil_div(W, 128), (unsigned)ps_ceil_div(F - lo, kCheckRows));
    label_check_kernel<<<grid, 128, 0, s>>>(a->d_bad, a->d_mask, W, F, lo, hi, ds->d_err);
    PS_LAUNCHED();
  }
  if (a->code_bytes == 2)
    onehot16_kernel<<<(unsigned)Rp, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(a->d_codes), a->ldc, d_rf, d_rl, R,
                                                 Sp, S, O);
  else
    onehot_kernel<<<(unsigned)Rp, 256, 0, s>>>(a->d_codes, a->ldc, d_rf, d_rl, R, Sp, S, O);
  PS_LAUNCHED();
  CUtensorMap map;
  {
    const char* mce = getenv("PS_CHI2_MC");
    const bool mc = !(mce && mce[0] == '0') && ds->num_sms >= 2;
    int rc = make_onehot_map(&map, O, Rp, Sp, mc ? 128 : TM);
    if (rc) return rc;
  }
  // Row bands: the table scratch of a band (band rows x Rp counts) stays
  // within PS_CHI2_BAND_MB (default 2 GiB) however wide the matrix is; a band
  // is at least one feature.  Config 3 (Rp = 3072) is one band.
  int64_t budget = 2048ll << 20;
  if (const char* e = getenv("PS_CHI2_BAND_MB")) budget = std::max(1L, atol(e)) << 20;
  const int64_t band_rows = std::max<int64_t>(TM, budget / (Rp * 4) / TM * TM);
  // u32 tables when any count could reach 2^24 (fp32 is exact below it)
  const bool wide_counts = S >= (1LL << 24) || getenv("PS_CHI2_U32");
  int rc = PS_OK;
  for (int64_t ga = lo; ga < hi && !rc;) {
    int64_t gb = ga + 1;
    // rows [off[ga], off[gb]) plus the tile-alignment slack of the first tile
    while (gb < hi && (off[gb + 1] - (off[ga] / TM) * TM) <= band_rows) ++gb;
    rc = wide_counts ? chi2_band<uint32_t>(a, off, ga, gb, Rp, map, (int)(Sp / TKB), d_off, stat, p, phi, v, s)
                     : chi2_band<float>(a, off, ga, gb, Rp, map, (int)(Sp / TKB), d_off, stat, p, phi, v, s);
    ga = gb;
  }
  ps_free(O, s);
  ps_free(d_off, s);
  ps_free(d_rf, s);
  ps_free(d_rl, s);
  return rc;
}
