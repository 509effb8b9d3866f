// ps_chi2.cu -- all-pairs chi-squared: contingency tables as one int8 GEMM.
//
// Replaces _chi2_block -> _chi2_rows -> _chi2_finish (engine.py:208-242,
// categorical.py:31-94).  Every feature f with c_f declared levels contributes
// c_f rows to a one-hot matrix O (row off_f + a, sample s) = 1 iff f is present
// at s with label a.  All contingency tables at once are C = O O^T
// (int8 x int8 -> int32, exact): the table of (g, h) is the c_g x c_h block at
// (off_g, off_h).  The GEMM runs on the tensor cores over upper-triangular
// 128 x 128 tiles of C (IMMA m16n8k32 via mma.sync, ldmatrix-fed from a
// swizzled 3-stage cp.async ring).  The epilogue (one thread per pair) replays
// the reference's NaN rules and its i-major chi-square loop in the same fp64
// operation order, so chi2 / phi / V are bit-identical; p = chi2_sf(chi2, dof).
//
// Algorithmic work: 2 k_g k_h int8 ops per pair-sample.
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include "ps_tc05.cuh"
#include <cudaTypedefs.h>
#include <algorithm>
#include <vector>

namespace {

constexpr int BM = 128, BN = 128, BK = 64;  // BK in bytes (int8)
constexpr int GW = 8;                        // warps: 2 (m) x 4 (n), warp tile 64 x 32
constexpr int GTH = GW * 32;
constexpr int GSTAGES = 3;
constexpr int TILE_BYTES = BM * BK;          // 8 KB per operand per stage

// ----------------------------------------------------------------- one-hot
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
  for (int64_t s = threadIdx.x * 16; s < Sp; s += blockDim.x * 16) {
    uint4 cv = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (s < ldc) cv = *reinterpret_cast<const uint4*>(c + s);
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t ss = s + q * 4 + b;
        const uint8_t code = ss < S ? (uint8_t)(cw[q] >> (8 * b)) : 0xFF;
        v |= (code == lev ? 1u : 0u) << (8 * b);
      }
      w[q] = v;
    }
    *reinterpret_cast<uint4*>(out + s) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ----------------------------------------------------------------- GEMM
__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // 16-byte chunk swizzle
  return (uint32_t)(row * BK + ((chunk ^ ((row >> 1) & 3)) << 4));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void imma(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// C[i][j] = sum_s O[i][s] O[j][s] over upper-triangular tiles (I <= J).
__global__ void __launch_bounds__(GTH)
onehot_gemm_kernel(const uint8_t* __restrict__ O, int64_t Sp, int64_t NTt, int64_t tile0,
                   int32_t* __restrict__ C, int64_t ldC) {
  extern __shared__ __align__(128) unsigned char gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4
  int64_t I, J;
  ps_tri_tile(tile0 + blockIdx.x, NTt, &I, &J);
  const int64_t row0 = I * BM, col0 = J * BN;
  const uint8_t* A = O + row0 * Sp;
  const uint8_t* B = O + col0 * Sp;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(gsm);
  const int64_t nk = Sp / BK;

  auto issue = [&](int64_t kc, int stage) {
    const uint32_t sa = sbase + stage * 2 * TILE_BYTES, sb = sa + TILE_BYTES;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = tid + q * GTH;  // 512 chunks of 16 B per operand
      const int r = idx >> 2, ch = idx & 3;
      const uint8_t* ga = A + r * Sp + kc * BK + ch * 16;
      const uint8_t* gb = B + r * Sp + kc * BK + ch * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + swz(r, ch)), "l"(ga));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + swz(r, ch)), "l"(gb));
    }
    asm volatile("cp.async.commit_group;");
  };

  int acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0;

  for (int q = 0; q < GSTAGES - 1; ++q) {
    if (q < nk) issue(q, q);
    else asm volatile("cp.async.commit_group;");
  }
  for (int64_t kc = 0; kc < nk; ++kc) {
    asm volatile("cp.async.wait_group %0;" ::"n"(GSTAGES - 2));
    __syncthreads();
    {
      const int64_t kn = kc + GSTAGES - 1;
      if (kn < nk) issue(kn, (int)(kn % GSTAGES));
      else asm volatile("cp.async.commit_group;");
    }
    const int stage = (int)(kc % GSTAGES);
    const uint32_t sa = sbase + stage * 2 * TILE_BYTES, sb = sa + TILE_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK / 32; ++kk) {
      uint32_t af[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mi = lane >> 3;
        const int r = wm * 64 + i * 16 + (lane & 7) + (mi & 1) * 8;
        const int ch = kk * 2 + (mi >> 1);
        ldsm_x4(sa + swz(r, ch), af[i][0], af[i][1], af[i][2], af[i][3]);
      }
      uint32_t bf[4][2];
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {
        const int mi = lane >> 3;
        const int r = wn * 32 + j2 * 16 + (lane & 7) + (mi >> 1) * 8;
        const int ch = kk * 2 + (mi & 1);
        ldsm_x4(sb + swz(r, ch), bf[j2 * 2][0], bf[j2 * 2][1], bf[j2 * 2 + 1][0], bf[j2 * 2 + 1][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) imma(acc[i][j], af[i], bf[j][0], bf[j][1]);
    }
  }
  asm volatile("cp.async.wait_group 0;");
  const int gr = lane >> 2, tg = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = row0 + wm * 64 + i * 16 + gr;
      const int64_t c = col0 + wn * 32 + j * 8 + tg * 2;
      *reinterpret_cast<int2*>(C + r * ldC + c) = make_int2(acc[i][j][0], acc[i][j][1]);
      *reinterpret_cast<int2*>(C + (r + 8) * ldC + c) = make_int2(acc[i][j][2], acc[i][j][3]);
    }
}

// ----------------------------------------------------------------- tcgen05 GEMM
// Blackwell-native version of the same contraction: tcgen05.mma kind::i8 with
// the int32 accumulator tile (128 x 256) in tensor memory.  Operands are
// staged by cp.async into the canonical K-major SWIZZLE_128B layout (8-row x
// 128-byte atoms), described to the tensor core by 64-bit smem descriptors;
// one elected thread issues 4 MMAs (K = 32 bytes each) per 128-byte stage and
// commits them to the stage's mbarrier, which gates the refill of that stage.
// The epilogue drains TMEM with tcgen05.ld (32 lanes x 32 columns per warp
// instruction) straight to the int32 table matrix.
constexpr int TM = 128, TN = 256, TKB = 128;  // tile rows, cols, K bytes per stage
constexpr int TSTAGES = 4;
constexpr int TTH = 128;
constexpr int TA_BYTES = TM * TKB, TB_BYTES = TN * TKB;
constexpr int TSTAGE_BYTES = TA_BYTES + TB_BYTES;
constexpr size_t kTc05Smem = (size_t)TSTAGES * TSTAGE_BYTES + 1024;

// Warp roles: warps 0-3 epilogue (TMEM lanes 32w..32w+31), warp 4 TMA
// producer, warp 5 MMA issuer.  full[s]: TMA bytes landed; empty[s]: the MMAs
// reading stage s retired (tcgen05.commit); done: last MMA retired.
constexpr int TTH_WS = 192;
__global__ void __launch_bounds__(TTH_WS, 1)
onehot_gemm_tc05_kernel(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB,
                        int64_t Sp, const int2* __restrict__ tiles, int32_t* __restrict__ C, int64_t ldC) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[TSTAGES], empty[TSTAGES], done;
  __shared__ uint32_t tmem_base_s;
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 t = tiles[blockIdx.x];
  const int64_t row0 = (int64_t)t.x * TM, col0 = (int64_t)t.y * TN;
  const int nk = (int)(Sp / TKB);

  if (warp == 0) tc05::tmem_alloc(&tmem_base_s, TN);
  if (tid == 32) {
    for (int i = 0; i < TSTAGES; ++i) {
      tc05::mbar_init(&full[i], 1);
      tc05::mbar_init(&empty[i], 1);
    }
    tc05::mbar_init(&done, 1);
    tc05::fence_barrier_init();
  }
  if (tid == 4 * 32) {
    tc05::prefetch_tmap(&tmapA);
    tc05::prefetch_tmap(&tmapB);
  }
  tc05::fence_before_sync();
  __syncthreads();
  tc05::fence_after_sync();
  const uint32_t tmem = tmem_base_s;

  if (warp == 4) {
    if (lane == 0) {  // TMA producer
      for (int kc = 0; kc < nk; ++kc) {
        const int st = kc % TSTAGES, n = kc / TSTAGES;
        if (n > 0) tc05::mbar_wait(&empty[st], (uint32_t)((n - 1) & 1));
        const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
        tc05::mbar_arrive_expect_tx(&full[st], TSTAGE_BYTES);
        tc05::tma_load_2d(sa, &tmapA, kc * TKB, (int32_t)row0, &full[st]);
        tc05::tma_load_2d(sb, &tmapB, kc * TKB, (int32_t)col0, &full[st]);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc05::idesc_i8(TM, TN, true);
      for (int kc = 0; kc < nk; ++kc) {
        const int st = kc % TSTAGES, n = kc / TSTAGES;
        tc05::mbar_wait(&full[st], (uint32_t)(n & 1));
        tc05::fence_after_sync();
        const uint32_t sa = sbase + st * TSTAGE_BYTES, sb = sa + TA_BYTES;
#pragma unroll
        for (int kk = 0; kk < TKB / 32; ++kk)
          tc05::mma_i8(tmem, tc05::sw128_kmajor_desc(sa + kk * 32), tc05::sw128_kmajor_desc(sb + kk * 32), idesc,
                       (kc | kk) != 0 ? 1u : 0u);
        tc05::commit(&empty[st]);
      }
      tc05::commit(&done);
    }
  } else {
    // epilogue warps 0-3
    tc05::mbar_wait(&done, 0);
    tc05::fence_after_sync();
    const int64_t r = row0 + warp * 32 + lane;
    int32_t* crow = C + r * ldC + col0;
#pragma unroll 1
    for (int cc = 0; cc < TN / 32; ++cc) {
      uint32_t v[32];
      tc05::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cc * 32), v);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<int4*>(crow + cc * 32 + j) = make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
    }
  }
  tc05::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc05::tmem_dealloc(tmem, TN);
}

// ----------------------------------------------------------------- epilogue
__device__ __forceinline__ void put(double* o, int64_t F, int64_t g, int64_t h, double v) {
  if (o) {
    o[g * F + h] = v;
    o[h * F + g] = v;
  }
}

// One thread per pair (g <= h): categorical.py:31-74 in the same op order.
// Row/column sums are cached for up to CM levels; the table is read from C.
template <int CM>
__global__ void chi2_finish_kernel(const int32_t* __restrict__ C, int64_t ldC,
                                   const int32_t* __restrict__ off, const int32_t* __restrict__ cat,
                                   int64_t F, int64_t lo, int64_t hi, double* __restrict__ stat,
                                   double* __restrict__ pout, double* __restrict__ phi_out,
                                   double* __restrict__ v_out, int* __restrict__ err) {
  const int64_t total = (hi - lo) * F;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = lo + it / F, h = it % F;
    if (h < g) continue;
    const int cg = cat[g], ch = cat[h];
    const bool diag = g == h;
    const int32_t* T = C + (int64_t)off[g] * ldC + off[h];
    // the diagonal pair's table is diagonal; its lower half lies outside the
    // computed upper-triangular tiles, so read only the diagonal
    auto tab = [&](int i, int j) -> long long {
      if (diag && i != j) return 0;
      return T[(int64_t)i * ldC + j];
    };
    long long rs[CM], cs[CM];
    for (int j = 0; j < ch; ++j) cs[j] = 0;
    long long n = 0;
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
    double chi2 = PS_NAN, p = PS_NAN, phi = PS_NAN, v = PS_NAN;
    bool empty = n == 0;
    for (int i = 0; i < cg; ++i) empty |= rs[i] == 0;
    for (int j = 0; j < ch; ++j) empty |= cs[j] == 0;
    if (!empty) {
      double acc = 0.0;
      const double dn = (double)n;
      for (int i = 0; i < cg; ++i)
        for (int j = 0; j < ch; ++j) {
          const double expected = (double)(rs[i] * cs[j]) / dn;
          if (expected > 0.0) {
            const double diff = (double)tab(i, j) - expected;
            acc += diff * diff / expected;
          }
        }
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
__global__ void label_check_kernel(const uint32_t* __restrict__ bad, const uint32_t* __restrict__ mask,
                                   int64_t W, int64_t F, int64_t lo, int64_t hi, int* __restrict__ err) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t col = 0;
    for (int64_t g = lo; g < hi; ++g) col |= mask[g * W + w];
    for (int64_t f = lo; f < F; ++f) {
      const uint32_t b = bad[f * W + w];
      if (b && (f < hi || (b & col))) {
        ps_raise(err, PS_ERR_LABEL_OUT_OF_RANGE);
        return;
      }
    }
  }
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
  int32_t* C = nullptr;
  int32_t *d_off = nullptr, *d_rf = nullptr, *d_rl = nullptr;
  PS_CUDA(ps_alloc(&O, (size_t)(Rp * Sp), s));
  PS_CUDA(ps_alloc(&C, (size_t)(Rp * Rp), s));
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
    label_check_kernel<<<(unsigned)std::min<int64_t>(ps_ceil_div(W, 128), 1024), 128, 0, s>>>(
        a->d_bad, a->d_mask, W, F, lo, hi, ds->d_err);
    PS_LAUNCHED();
  }
  onehot_kernel<<<(unsigned)Rp, 256, 0, s>>>(a->d_codes, a->ldc, d_rf, d_rl, R, Sp, S, O);
  PS_LAUNCHED();
  // 128 x 256 tiles of C needed by pairs with g in [lo, hi): row tiles covering
  // off[lo] .. off[hi]-1, column tiles from the diagonal rightwards
  std::vector<int2> tl;
  if (R > 0) {
    const int64_t I0 = off[lo] / TM;
    const int64_t I1 = std::max<int64_t>(I0, (off[hi] - 1) / TM);
    for (int64_t I = I0; I <= I1; ++I)
      for (int64_t J = (I * TM) / TN; J < Rp / TN; ++J) tl.push_back(make_int2((int)I, (int)J));
  }
  int2* d_tiles = nullptr;
  if (!tl.empty()) {
    PS_CUDA(ps_alloc(&d_tiles, tl.size(), s));
    PS_CUDA(cudaMemcpyAsync(d_tiles, tl.data(), sizeof(int2) * tl.size(), cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaFuncSetAttribute(onehot_gemm_tc05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTc05Smem));
    CUtensorMap mapA, mapB;
    int rc = make_onehot_map(&mapA, O, Rp, Sp, TM);
    if (!rc) rc = make_onehot_map(&mapB, O, Rp, Sp, TN);
    if (rc) return rc;
    ps_prof_begin("chi2_gemm", s);
    onehot_gemm_tc05_kernel<<<(unsigned)tl.size(), TTH_WS, kTc05Smem, s>>>(mapA, mapB, Sp, d_tiles, C, Rp);
    ps_prof_end(s);
    PS_LAUNCHED();
  }
  int32_t* d_cat = a->d_cat;
  const int64_t total = (hi - lo) * F;
  const int blocks = (int)std::min<int64_t>(ps_ceil_div(total, 128), (int64_t)ds->num_sms * 16);
  if (a->cmax <= 16)
    chi2_finish_kernel<16><<<blocks, 128, 0, s>>>(C, Rp, d_off, d_cat, F, lo, hi, stat, p, phi, v, ds->d_err);
  else
    chi2_finish_kernel<256><<<blocks, 128, 0, s>>>(C, Rp, d_off, d_cat, F, lo, hi, stat, p, phi, v, ds->d_err);
  PS_LAUNCHED();
  ps_free(O, s);
  ps_free(C, s);
  ps_free(d_off, s);
  ps_free(d_rf, s);
  ps_free(d_rl, s);
  ps_free(d_tiles, s);
  return PS_OK;
}
