// ps_pearson.cu -- all-pairs Pearson with pairwise deletion on FP64 tensor cores.
//
// Replaces the reference's _pearson_block -> _pearson_rows -> _pearson_finish
// (engine.py:145-166, continuous.py:29-49, :77-103).  The two masked passes per
// pair become one masked-moment contraction over upper-triangular 64x64 tiles
// of features: with x' = (x - c_f) on present cells and 0 elsewhere, and m the
// 0/1 presence,
//     Sxy = X' X'^T,  Sx = X' M^T,  Sxx = X'^2 M^T,  Sy = M X'^T,  Syy = M X'^2^T
// run as DMMA.8x8x4 (mma.sync m8n8k4 f64 -- the only FP64 tensor path on
// sm_100a; tcgen05 has no f64 kind), and the pair count n = popc(m_g & m_h) on
// the integer pipe.  Centred sums then follow from
//     sxx = Sxx - Sx^2/n, syy = Syy - Sy^2/n, sxy = Sxy - Sx Sy/n.
// The epilogue (r, clamp, p = 2 beta_sym_sf(|r|, n/2 - 1), r^2) is fused into
// the same CTA.  Pairs where cancellation could flip the reference's
// degenerate-variance decision (sxx or syy <= 1e-3 of its raw second moment,
// or non-finite) are re-evaluated by an exact replay of the reference's
// sequential two-pass loop, so the NaN pattern is identical.
//
// Algorithmic work: 10 FP64 flops per pair-sample (5 masked MACs).
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include "ps_tc05.cuh"
#include <cudaTypedefs.h>
#include <algorithm>

namespace {

constexpr int T = 64;            // features per tile edge
constexpr int KC = 32;           // samples per k-chunk (one mask word)
constexpr int XS = KC + 4;       // padded smem row stride (doubles): 2 wavefronts per fragment load
#ifndef PS_PEARSON_WN
#define PS_PEARSON_WN 4
#endif
constexpr int WM = 2, WN = PS_PEARSON_WN;  // 8x8 accumulator blocks per warp (rows x cols)
constexpr int WJ = T / (8 * WN);           // column groups of warps
constexpr int NWARP = (T / (8 * WM)) * WJ;  // WN = 4: 4 x 2 warps of 16 x 32 pairs
constexpr int NTHR = NWARP * 32;
constexpr double kReplayTau = 1e-3;
constexpr int64_t kMomBlock = 12;  // tile columns per incremental int8 launch set

// MODE 0: raw values, centred and squared per use; 1: pre-centred x'
// (squared per use); 2: pre-centred x' and x'^2 (no FP64 ALU work in the
// DMMA loop; 222 KB of stages)
template <int MODE>
struct Stage {
  double xi[T][XS];
  double xj[T][XS];
  double qi[MODE == 2 ? T : 1][XS];
  double qj[MODE == 2 ? T : 1][XS];
  uint32_t mi[T];
  uint32_t mj[T];
};
// CPB chunks are computed per block barrier: CPB = 1 -> a 3-stage ring
// (prefetch distance 2 chunks), CPB = 2 -> a 4-stage ring filled in pairs
template <int CPB>
constexpr int nstage() { return CPB == 1 ? 3 : 2 * CPB; }
template <int MODE, int CPB = 1>
constexpr size_t smem_bytes() { return nstage<CPB>() * sizeof(Stage<MODE>); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

struct Outs {
  double* stat;
  double* p;
  double* r2;
  int2* replay;
  int* replay_count;
  int replay_cap;
  int* err;
  int defer_p;  // 1: the tile epilogue parks n in p; pearson_p_kernel evaluates the tail
  // moments path: the tiles store Sxy and n (F x F, upper pairs) for
  // pearson_pairs_kernel, which joins them with the int8 moments
  double* sxy = nullptr;
  int32_t* nn = nullptr;
};

// Pearson p = 2 I_{(1-|r|)/2}(n/2 - 1, n/2 - 1): the division-free continued
// fraction (PS_P_LENTZ: the reference's Lentz form, for A/B builds)
#ifdef PS_P_LENTZ
#define PS_BETA_SYM psf::beta_sym_sf
#else
#define PS_BETA_SYM psf::beta_sym_sf_nodiv
#endif

__device__ __forceinline__ void put(double* o, int64_t F, int64_t g, int64_t h, double v) {
  if (o) {
    o[g * F + h] = v;
    o[h * F + g] = v;
  }
}

// Exact replay of the pair (g, h): the replay kernel writes it.
__device__ __forceinline__ void replay_pair(int64_t g, int64_t h, int64_t F, const Outs& o) {
  int slot = atomicAdd(o.replay_count, 1);
  if (slot < o.replay_cap) o.replay[slot] = make_int2((int)g, (int)h);
  if (o.defer_p) put(o.p, F, g, h, PS_NAN);  // not a parked n: pearson_p_kernel skips it
}

// Digit-expansion moments (ps_moments.cu) carry a rigorous error bound: each
// expanded term is within 2^(e - 7 D) of x' (D = kMomentDigits; e: the row
// exponent of x', resp. x'^2), so |dSx| <= n 2^(e1 - 7 D), |dSxx| <= n 2^(e2 - 7 D) (+ the fp64 fold,
// 8 ulp).  A pair whose centred sums could move by more than 1e-12 of
// themselves (an outlier-dominated row exponent, a subset far smaller than the
// row's scale) is replayed exactly instead -- data-independent parity.
__device__ __forceinline__ bool moments_imprecise(int n, double sx, double sy, double qx, double qy, int e1g,
                                                  int e2g, int e1h, int e2h) {
  if (n <= 1) return false;
  const double fn = (double)n;
  // 4x the bound of Sxx: seven base-256 planes with a guard bit round at 2^(e - 55) (eight base-128
  // digits, PS_MOMENTS_B256=0: 2^(e - 56)); 8x the bound of Sx: six base-256 planes round at 2^(e - 47)
  // (base 128: truncated after digit 7, ~2^(e - 49)).  One bound for both forms.
  constexpr int kB = 53;
  constexpr int kB1 = 44;
  const double d1g = ldexp(1.0, e1g - kB1), d2g = ldexp(1.0, e2g - kB);
  const double d1h = ldexp(1.0, e1h - kB1), d2h = ldexp(1.0, e2h - kB);
  const double sxx = qx - sx * sx / fn, syy = qy - sy * sy / fn;
  if (!(sxx > 0.0) || !(syy > 0.0)) return false;  // the degenerate-variance rule replays it anyway
  const double exx = fn * d2g + 2.0 * fabs(sx) * d1g + 1e-15 * qx;
  const double eyy = fn * d2h + 2.0 * fabs(sy) * d1h + 1e-15 * qy;
  const double exy = fabs(sy) * d1g + fabs(sx) * d1h;
  return exx > 1e-12 * sxx || eyy > 1e-12 * syy || exy > 1e-12 * sqrt(sxx * syy);
}

// Sxy from int8 digit products (ps_moments.cu, s + t <= kSxyMaxOrder = 9): per
// element the expansion errors give |x eps_y| + |y eps_x| <= 2^(e_g + e_h - 55)
// and the dropped products < 2^(e_g + e_h - 53.1), together < 2^-54 of
// ag ah = 2^(e_g + e_h + 2); the fp64 fold of 36 scaled exact
// products errs by <= 36 * 2^-53 of the sum of their magnitudes, bounded (Cauchy-
// Schwarz over the joint samples, digit excess delta = 2^-7 of the row scale) by
// sqrt(qx qy) + delta 2^(e+1) sqrt(n q) terms.  The symmetric form (sum planes,
// ps_moments.cu: 24 products, each scaled term rounded once more) folds squares
// that cancel: |w (d_s d_s' + d_t d_t')| <= 2^-7 of ag ah per sample in at most
// nine partial sums, another n ag ah 2^-56.  The bound covers both forms.  4x
// margin; replay when it exceeds 1e-12 sqrt(sxx syy).
__device__ __forceinline__ bool sxy_imprecise(int n, double sx, double sy, double qx, double qy, int e1g, int e1h) {
  if (n <= 1) return false;
  const double fn = (double)n;
  const double sxx = qx - sx * sx / fn, syy = qy - sy * sy / fn;
  if (!(sxx > 0.0) || !(syy > 0.0)) return false;  // replayed by the degenerate-variance rule anyway
  const double ag = ldexp(1.0, e1g + 1), ah = ldexp(1.0, e1h + 1), dl = 0.0078125;
  const double trunc = fn * ag * ah * (ldexp(1.0, -54) + ldexp(1.0, -56));
  const double mag = sqrt(qx * qy) + dl * ag * sqrt(fn * qy) + dl * ah * sqrt(fn * qx) + fn * dl * dl * ag * ah;
  const double bound = 4.0 * (trunc + (double)kSxyFoldTerms * ldexp(mag, -53));
  return bound > 1e-12 * sqrt(sxx * syy);
}

// Moments -> outputs for one upper-triangular pair (g <= h).
__device__ void pearson_finish(int64_t g, int64_t h, int64_t F, int n, double sx, double sy,
                               double qx, double qy, double xy, const Outs& o) {
  double r = PS_NAN, p = PS_NAN;
  if (n > 1) {
    const double fn = (double)n;
    const bool diag = g == h;
    const double sxx = qx - sx * sx / fn;
    const double syy = diag ? sxx : qy - sy * sy / fn;
    if (!(sxx > kReplayTau * qx) || !(syy > kReplayTau * (diag ? qx : qy))) {
      replay_pair(g, h, F, o);
      return;
    }
    const double sxy = diag ? sxx : xy - sx * sy / fn;
    r = sxy / sqrt(sxx * syy);
    if (r > 1.0) r = 1.0;
    else if (r < -1.0) r = -1.0;
    if (n != 2) {
      if (o.defer_p) {
        p = fn;  // pearson_p_kernel: p from (r, n) at full occupancy
      } else {
        p = 2.0 * PS_BETA_SYM(fabs(r), 0.5 * fn - 1.0, o.err);
        if (p > 1.0) p = 1.0;
      }
    }
  }
  put(o.stat, F, g, h, r);
  put(o.p, F, g, h, p);
  put(o.r2, F, g, h, r * r);
}

// The p-values of the tiles' pairs (continuous.py:47): the tile epilogue
// parked n in p (NaN where p is NaN by rule, or the pair awaits the exact
// replay); here one thread per upper-triangle cell of rows [lo, hi) runs the
// beta continued fraction with the whole SM's warps in flight instead of
// inside the one-CTA-per-SM tile kernel, where the DMMA pipe idled meanwhile.
__global__ void pearson_p_kernel(const double* __restrict__ stat, double* __restrict__ pout, int64_t F, int64_t lo,
                                 int64_t hi, int* __restrict__ err) {
  // cells enumerated over the upper triangle only (no idle threads):
  // before(g) = cells of rows [lo, g)
  auto before = [&](int64_t g) { return (g - lo) * F - (g * (g - 1) - lo * (lo - 1)) / 2; };
  const int64_t total = before(hi);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = lo, b = hi - 1;  // last row g with before(g) <= it
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (before(mid) <= it) a = mid;
      else b = mid - 1;
    }
    const int64_t g = a, h = g + (it - before(g));
    const double fn = pout[g * F + h];
    if (fn != fn) continue;
    const double r = stat[g * F + h];
    double p = 2.0 * PS_BETA_SYM(fabs(r), 0.5 * fn - 1.0, err);
    if (p > 1.0) p = 1.0;
    pout[g * F + h] = p;
    pout[h * F + g] = p;
  }
}

// The moments path's pair epilogue: Sxy and n from the DMMA tiles, Sx / Sxx
// (and their transposes Sy / Syy) from the int8 contractions; one thread per
// upper-triangle cell of rows [lo, hi).  Pairs whose digit moments could move
// the centred sums by more than 1e-12 are replayed exactly.
__global__ void pearson_pairs_kernel(int64_t F, int64_t lo, int64_t hi, Outs o, const double* __restrict__ msx,
                                     const double* __restrict__ msq, const int32_t* __restrict__ me1,
                                     const int32_t* __restrict__ me2, int i8) {
  auto before = [&](int64_t g) { return (g - lo) * F - (g * (g - 1) - lo * (lo - 1)) / 2; };
  const int64_t total = before(hi);
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = lo, b = hi - 1;  // last row g with before(g) <= it
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (before(mid) <= it) a = mid;
      else b = mid - 1;
    }
    const int64_t g = a, h = g + (it - before(g));
    const int n = o.nn[g * F + h];
    const double sx = msx[g * F + h], sy = msx[h * F + g], qx = msq[g * F + h], qy = msq[h * F + g];
    const double xy = o.sxy[g * F + h];
    if (g != h && (moments_imprecise(n, sx, sy, qx, qy, me1[g], me2[g], me1[h], me2[h]) ||
                   (i8 && sxy_imprecise(n, sx, sy, qx, qy, me1[g], me1[h]))))
      replay_pair(g, h, F, o);
    else
      pearson_finish(g, h, F, n, sx, sy, qx, qy, xy, o);
  }
}

// x' = x - c_f on present cells, 0 elsewhere, for rows [f0, f0 + grid): the
// tile kernel's operands pre-centred once per element (the same fp64
// subtraction the tile kernel would do per use, so every bit is unchanged);
// the tile loop then feeds x' and x'^2 to the DMMAs without per-use
// subtract / select instructions on the FP64 pipe the DMMAs share.
__global__ void center_rows_kernel(const double* __restrict__ vals, int64_t ld, const uint32_t* __restrict__ mask,
                                   int64_t W, const double* __restrict__ center, double* __restrict__ out,
                                   double* __restrict__ out2, int64_t f0) {
  const int64_t f = f0 + blockIdx.x;
  const double c = center[f];
  const double* x = vals + f * ld;
  double* y = out + f * ld;
  const uint32_t* m = mask + f * W;
  for (int64_t s = threadIdx.x * 2; s < ld; s += blockDim.x * 2) {
    const uint32_t w = m[s >> 5];
    const double2 v = *reinterpret_cast<const double2*>(x + s);
    double2 r;
    r.x = ((w >> (s & 31)) & 1u) ? v.x - c : 0.0;
    r.y = ((w >> ((s + 1) & 31)) & 1u) ? v.y - c : 0.0;
    *reinterpret_cast<double2*>(y + s) = r;
    if (out2) *reinterpret_cast<double2*>(out2 + f * ld + s) = make_double2(r.x * r.x, r.y * r.y);
  }
}

// grid.x = tiles in range x nsplit.  Each CTA accumulates one 64x64 tile over
// its share of the k-chunks.  MODE >= 1: vals holds pre-centred x'
// (center_rows_kernel); MODE 2: sq holds x'^2.
template <int MODE, int CPB>
__global__ void __launch_bounds__(NTHR, 1)
pearson_tile_kernel(const double* __restrict__ vals, const double* __restrict__ sq, int64_t ld,
                    const uint32_t* __restrict__ mask, int64_t W, const double* __restrict__ center, int64_t F,
                    int64_t NT, int64_t tile0, int64_t lo, int64_t hi, int nsplit, int64_t chunks_per_split,
                    Outs o, double* __restrict__ ws, int colmajor) {
  constexpr bool PC = MODE >= 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Stage = ::Stage<MODE>;
  Stage* st = reinterpret_cast<Stage*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / WJ, wj = warp % WJ;
  const int64_t tile = tile0 + blockIdx.x / nsplit;
  const int split = blockIdx.x % nsplit;
  int64_t I, J;
  if (colmajor) ps_tri_tile_cm(tile, &I, &J);  // incremental launches: columns of uploaded rows
  else ps_tri_tile(tile, NT, &I, &J);
  const int64_t row0 = I * T, col0 = J * T;
  const int64_t c_begin = (int64_t)split * chunks_per_split;
  const int64_t c_end = min(W, c_begin + chunks_per_split);

  // per-lane fragment rows/cols and their pivots
  const int fr = lane >> 2, fk = lane & 3;
  double ci[WM], cj[WN];
#pragma unroll
  for (int q = 0; q < WM; ++q) {
    const int64_t gr = row0 + wi * 8 * WM + q * 8 + fr;
    ci[q] = gr < F ? center[gr] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < WN; ++q) {
    const int64_t gc = col0 + wj * 8 * WN + q * 8 + fr;
    cj[q] = gc < F ? center[gc] : 0.0;
  }

  double axy[WM][WN][2], asx[WM][WN][2], asxx[WM][WN][2], asy[WM][WN][2], asyy[WM][WN][2];
  int an[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        axy[i][j][e] = asx[i][j][e] = asxx[i][j][e] = asy[i][j][e] = asyy[i][j][e] = 0.0;
        an[i][j][e] = 0;
      }

  // global -> shared via cp.async (no register staging), NSTAGE-deep ring
  constexpr int LQ = (T * KC / 2) / NTHR;  // 16-byte copies per thread per operand tile
  auto issue = [&](int64_t c, Stage& sd) {
#pragma unroll
    for (int q = 0; q < LQ; ++q) {
      const int idx = tid + q * NTHR;
      const int r = idx >> 4, c2 = idx & 15;
      const int64_t gi = min(row0 + r, F - 1), gj = min(col0 + r, F - 1);
      const int64_t off = c * KC + c2 * 2;
      const unsigned si = (unsigned)__cvta_generic_to_shared(&sd.xi[r][c2 * 2]);
      const unsigned sj = (unsigned)__cvta_generic_to_shared(&sd.xj[r][c2 * 2]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(si), "l"(vals + gi * ld + off));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sj), "l"(vals + gj * ld + off));
      if constexpr (MODE == 2) {
        const unsigned qi = (unsigned)__cvta_generic_to_shared(&sd.qi[r][c2 * 2]);
        const unsigned qj = (unsigned)__cvta_generic_to_shared(&sd.qj[r][c2 * 2]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(qi), "l"(sq + gi * ld + off));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(qj), "l"(sq + gj * ld + off));
      }
    }
    if (tid < 2 * T) {
      const int64_t gr = (tid < T ? row0 : col0) + (tid & (T - 1));
      // rows past F get an all-zero mask, so their (clamped) values never count
      const uint32_t w = gr < F ? mask[gr * W + c] : 0u;
      if (tid < T) sd.mi[tid] = w;
      else sd.mj[tid - T] = w;
    }
    asm volatile("cp.async.commit_group;");
  };

  constexpr int NSTAGE = nstage<CPB>();
  constexpr int AHEAD = CPB == 1 ? NSTAGE - 1 : CPB;  // chunks loaded before the loop
  for (int q = 0; q < AHEAD; ++q) {
    if (c_begin + q < c_end) issue(c_begin + q, st[q]);
    else asm volatile("cp.async.commit_group;");
  }
  for (int64_t cb = c_begin; cb < c_end; cb += CPB) {
    // the chunks [cb, cb + CPB) have landed (CPB = 1: one newer group may
    // still be in flight)
    if (CPB == 1) asm volatile("cp.async.wait_group %0;" ::"n"(NSTAGE - 2));
    else asm volatile("cp.async.wait_group 0;");
    __syncthreads();
#pragma unroll
    for (int q = 0; q < CPB; ++q) {
      const int64_t cn = cb + (CPB == 1 ? NSTAGE - 1 : CPB) + q;
      if (cn < c_end) issue(cn, st[(int)((cn - c_begin) % NSTAGE)]);
      else asm volatile("cp.async.commit_group;");
    }
#pragma unroll 1
    for (int64_t c = cb; c < cb + CPB && c < c_end; ++c) {
    const int cur = (int)((c - c_begin) % NSTAGE);
    const Stage& s = st[cur];
    uint32_t mrow[WM], mcol[WN];
#pragma unroll
    for (int q = 0; q < WM; ++q) mrow[q] = s.mi[wi * 8 * WM + q * 8 + fr];
#pragma unroll
    for (int q = 0; q < WN; ++q) mcol[q] = s.mj[wj * 8 * WN + q * 8 + fr];
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      const int k = kk * 4 + fk;
      double xa[WM], ma[WM], xa2[WM], xb[WN], mb[WN], xb2[WN];
#pragma unroll
      for (int q = 0; q < WM; ++q) {
        const bool pa = (mrow[q] >> k) & 1u;
        const double va = s.xi[wi * 8 * WM + q * 8 + fr][k];
        xa[q] = PC ? va : (pa ? va - ci[q] : 0.0);
        ma[q] = pa ? 1.0 : 0.0;
        if constexpr (MODE == 2) xa2[q] = s.qi[wi * 8 * WM + q * 8 + fr][k];
        else xa2[q] = xa[q] * xa[q];
      }
#pragma unroll
      for (int q = 0; q < WN; ++q) {
        const bool pb = (mcol[q] >> k) & 1u;
        const double vb = s.xj[wj * 8 * WN + q * 8 + fr][k];
        xb[q] = PC ? vb : (pb ? vb - cj[q] : 0.0);
        mb[q] = pb ? 1.0 : 0.0;
        if constexpr (MODE == 2) xb2[q] = s.qj[wj * 8 * WN + q * 8 + fr][k];
        else xb2[q] = xb[q] * xb[q];
      }
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) {
          dmma(axy[i][j][0], axy[i][j][1], xa[i], xb[j]);
          dmma(asx[i][j][0], asx[i][j][1], xa[i], mb[j]);
          dmma(asxx[i][j][0], asxx[i][j][1], xa2[i], mb[j]);
          dmma(asy[i][j][0], asy[i][j][1], ma[i], xb[j]);
          dmma(asyy[i][j][0], asyy[i][j][1], ma[i], xb2[j]);
        }
    }
    // pair counts for the lane's accumulator positions (integer pipe)
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const uint32_t a = mrow[i];
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) an[i][j][e] += __popc(a & s.mj[wj * 8 * WN + j * 8 + 2 * fk + e]);
    }
    }  // chunks of this barrier
  }
  asm volatile("cp.async.wait_group 0;");

  if (nsplit > 1) {
    // partial moments -> workspace [tile-in-range][split][6][T][T]
    double* w = ws + ((blockIdx.x / nsplit) * (int64_t)nsplit + split) * 6 * T * T;
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wi * 8 * WM + i * 8 + fr, cc = wj * 8 * WN + j * 8 + 2 * fk + e;
          const int o2 = r * T + cc;
          w[0 * T * T + o2] = (double)an[i][j][e];
          w[1 * T * T + o2] = asx[i][j][e];
          w[2 * T * T + o2] = asy[i][j][e];
          w[3 * T * T + o2] = asxx[i][j][e];
          w[4 * T * T + o2] = asyy[i][j][e];
          w[5 * T * T + o2] = axy[i][j][e];
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t g = row0 + wi * 8 * WM + i * 8 + fr;
        const int64_t h = col0 + wj * 8 * WN + j * 8 + 2 * fk + e;
        if (g < lo || g >= hi || h < g || h >= F) continue;
        pearson_finish(g, h, F, an[i][j][e], asx[i][j][e], asy[i][j][e], asxx[i][j][e],
                       asyy[i][j][e], axy[i][j][e], o);
      }
}

// ---------------------------------------------------------------------------
// TMA-fed variant (no split-K): the pre-centred x' tiles arrive by
// cp.async.bulk.tensor in 128-byte-swizzled 64-row x 16-sample boxes and the
// presence words by a second tensor map, completion counted on per-stage
// `full` mbarriers; each warp releases a stage on its `empty` mbarrier and
// thread 0 -- the only producer -- refills a stage once all eight warps have
// released it, one stage behind, so no block-wide barrier sits in the loop.
// Same per-lane k order as pearson_tile_kernel: identical bits.
constexpr int TG = 64;                        // samples per stage (2 mask words)
constexpr int TBOX = 16;                      // doubles per box row (128 B, SW128)
constexpr int TNB = TG / TBOX;                // boxes per operand per stage
constexpr int TBOX_BYTES = T * TBOX * 8;      // 8 KB
constexpr int TMASK_WORDS = 2;                // presence words per row per stage (cp.async, 8 B)
constexpr int TSTAGE_BYTES = 2 * TNB * TBOX_BYTES + 2 * T * TMASK_WORDS * 4;
constexpr int TNS = 3;
constexpr size_t kTmaSmem = (size_t)TNS * TSTAGE_BYTES + 1024;
// PRE variant: 32-sample stages (one mask word), two CTAs per SM
constexpr size_t kTmaSmemPre = (size_t)TNS * (2 * (32 / TBOX) * TBOX_BYTES + 2 * T * 1 * 4) + 1024;
template <bool PRE>
constexpr size_t tma_smem() { return PRE ? kTmaSmemPre : kTmaSmem; }

// Whole-warp wait on an mbarrier phase: the try_wait loop is C++ (the
// compiler sees the branch) and the warp reconverges before the
// warp-synchronous DMMAs that follow -- an asm-internal spin loop would let
// lanes leave it at different times and reach mma.sync diverged.
__device__ __forceinline__ void mbar_wait_warp(uint64_t* mbar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(tc05::smem_u32(mbar)), "r"(parity)
        : "memory");
  } while (!done);
  __syncwarp();
}

__device__ __forceinline__ double ld_sw(uint32_t box_base, int r, int k) {
  // element (row r, sample k within the box) of a SWIZZLE_128B 64 x 16 double box
  const uint32_t a = box_base + tc05::sw128_offset((uint32_t)r, (uint32_t)(k >> 1)) + (uint32_t)(k & 1) * 8u;
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

// PRE: the first / second moments come from the int8 contractions
// (ps_moments.cu): the tiles run Sxy = X' X'^T alone -- one DMMA per fragment
// pair instead of five -- plus the pair counts, and store both for
// pearson_pairs_kernel (so they need no moments and overlap the upload)
template <bool PRE>
__global__ void __launch_bounds__(NTHR, PRE ? 2 : 1)
pearson_tma_kernel(const __grid_constant__ CUtensorMap xmap, const uint32_t* __restrict__ mpad, int64_t Wp,
                   int64_t W, int64_t F, int64_t NT, int64_t tile0, int64_t lo, int64_t hi, Outs o, int colmajor) {
  // PRE (one DMMA product): half-size stages (32 samples, one mask word) so
  // that two CTAs share an SM -- twice the warps to hide the DMMA latency
  constexpr int TG = PRE ? 32 : ::TG;
  constexpr int TNB = TG / TBOX;
  constexpr int TMASK_WORDS = TG / 32;
  constexpr int TSTAGE_BYTES = 2 * TNB * TBOX_BYTES + 2 * T * TMASK_WORDS * 4;
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  __shared__ uint64_t full[TNS], empty[TNS];
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc05::smem_u32(tsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / WJ, wj = warp % WJ;
  int64_t I, J;
  if (colmajor) ps_tri_tile_cm(tile0 + blockIdx.x, &I, &J);
  else ps_tri_tile(tile0 + blockIdx.x, NT, &I, &J);
  const int row0 = (int)(I * T), col0 = (int)(J * T);
  const int64_t ngroups = ps_ceil_div(W, TG / 32);
  if (tid == 0) {
    for (int i = 0; i < TNS; ++i) {
      tc05::mbar_init(&full[i], 1 + 32);  // lane 0's expect_tx + warp 0's cp.async arrivals
      tc05::mbar_init(&empty[i], NWARP);
    }
    tc05::fence_barrier_init();
    tc05::prefetch_tmap(&xmap);
  }
  __syncthreads();
  auto stage_addr = [&](int st) { return sbase + (uint32_t)st * TSTAGE_BYTES; };
  // warp 0, converged: lane 0 arms the stage's `full` barrier with the x'
  // bytes and issues the TMA boxes; every lane copies presence words of two
  // row-block and two column-block rows (8-byte cp.async, zero-filled past F)
  // and arrives on `full` when its copies land (noinc: counted in the init)
  auto issue = [&](int64_t g) {
    const int st = (int)(g % TNS);
    const uint32_t a = stage_addr(st);
    if (lane == 0) {
      tc05::mbar_arrive_expect_tx(&full[st], 2 * TNB * TBOX_BYTES);
      const int x0 = (int)(g * TG);
      for (int b = 0; b < TNB; ++b) {
        tc05::tma_load_2d(a + b * TBOX_BYTES, &xmap, x0 + b * TBOX, row0, &full[st]);
        tc05::tma_load_2d(a + (TNB + b) * TBOX_BYTES, &xmap, x0 + b * TBOX, col0, &full[st]);
      }
    }
    const uint32_t am = a + 2 * TNB * TBOX_BYTES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = lane + 32 * (q & 1);               // row within the block
      const int64_t gr = (q < 2 ? row0 : col0) + r;  // feature row
      const uint32_t dst = am + (uint32_t)((q < 2 ? 0 : T * TMASK_WORDS * 4) + r * TMASK_WORDS * 4);
      const uint32_t* src = mpad + (gr < F ? gr : 0) * Wp + TMASK_WORDS * g;
      const uint32_t nbytes = gr < F ? 4u * TMASK_WORDS : 0u;
      if constexpr (TMASK_WORDS == 2)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(nbytes) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(nbytes) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc05::smem_u32(&full[st])) : "memory");
  };
  if (warp == 0)
    for (int64_t g = 0; g < TNS - 1 && g < ngroups; ++g) issue(g);

  const int fr = lane >> 2, fk = lane & 3;
  double axy[WM][WN][2], asx[WM][WN][2], asxx[WM][WN][2], asy[WM][WN][2], asyy[WM][WN][2];
  int an[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        axy[i][j][e] = asx[i][j][e] = asxx[i][j][e] = asy[i][j][e] = asyy[i][j][e] = 0.0;
        an[i][j][e] = 0;
      }
  for (int64_t g = 0; g < ngroups; ++g) {
    if (warp == 0) {  // refill the stage the slowest warp released one group ago
      const int64_t gn = g + TNS - 1;
      if (gn < ngroups) {
        if (gn >= TNS && lane == 0) tc05::mbar_wait(&empty[gn % TNS], (uint32_t)(((gn / TNS) - 1) & 1));
        __syncwarp();
        issue(gn);
      }
    }
    const int st = (int)(g % TNS);
    mbar_wait_warp(&full[st], (uint32_t)((g / TNS) & 1));
    const uint32_t a = stage_addr(st);
    const uint32_t* smi = reinterpret_cast<const uint32_t*>(tsm + (size_t)st * TSTAGE_BYTES + 2 * TNB * TBOX_BYTES);
    const uint32_t* smj = smi + T * TMASK_WORDS;
#pragma unroll
    for (int h = 0; h < TG / 32; ++h) {
      uint32_t mrow[WM], mcol[WN];
#pragma unroll
      for (int q = 0; q < WM; ++q) mrow[q] = smi[(wi * 8 * WM + q * 8 + fr) * TMASK_WORDS + h];
#pragma unroll
      for (int q = 0; q < WN; ++q) mcol[q] = smj[(wj * 8 * WN + q * 8 + fr) * TMASK_WORDS + h];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = kk * 4 + fk;     // bit within the mask word
        const int ks = h * 32 + k;     // sample within the stage
        const uint32_t bi = a + (uint32_t)(ks / TBOX) * TBOX_BYTES;
        const uint32_t bj = a + (uint32_t)(TNB + ks / TBOX) * TBOX_BYTES;
        double xa[WM], xb[WN];
#pragma unroll
        for (int q = 0; q < WM; ++q) xa[q] = ld_sw(bi, wi * 8 * WM + q * 8 + fr, ks % TBOX);
#pragma unroll
        for (int q = 0; q < WN; ++q) xb[q] = ld_sw(bj, wj * 8 * WN + q * 8 + fr, ks % TBOX);
        if constexpr (PRE) {
#pragma unroll
          for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) dmma(axy[i][j][0], axy[i][j][1], xa[i], xb[j]);
        } else {
          double ma[WM], xa2[WM], mb[WN], xb2[WN];
#pragma unroll
          for (int q = 0; q < WM; ++q) {
            ma[q] = ((mrow[q] >> k) & 1u) ? 1.0 : 0.0;
            xa2[q] = xa[q] * xa[q];
          }
#pragma unroll
          for (int q = 0; q < WN; ++q) {
            mb[q] = ((mcol[q] >> k) & 1u) ? 1.0 : 0.0;
            xb2[q] = xb[q] * xb[q];
          }
#pragma unroll
          for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) {
              dmma(axy[i][j][0], axy[i][j][1], xa[i], xb[j]);
              dmma(asx[i][j][0], asx[i][j][1], xa[i], mb[j]);
              dmma(asxx[i][j][0], asxx[i][j][1], xa2[i], mb[j]);
              dmma(asy[i][j][0], asy[i][j][1], ma[i], xb[j]);
              dmma(asyy[i][j][0], asyy[i][j][1], ma[i], xb2[j]);
            }
        }
      }
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const uint32_t av = mrow[i];
#pragma unroll
        for (int j = 0; j < WN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            an[i][j][e] += __popc(av & smj[(wj * 8 * WN + j * 8 + 2 * fk + e) * TMASK_WORDS + h]);
      }
    }
    __syncwarp();
    if (lane == 0) tc05::mbar_arrive(&empty[st]);
  }
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t gg = row0 + wi * 8 * WM + i * 8 + fr;
        const int64_t hh = col0 + wj * 8 * WN + j * 8 + 2 * fk + e;
        if (gg < lo || gg >= hi || hh < gg || hh >= F) continue;
        if constexpr (PRE) {
          o.sxy[gg * F + hh] = axy[i][j][e];
          o.nn[gg * F + hh] = an[i][j][e];
        } else {
          pearson_finish(gg, hh, F, an[i][j][e], asx[i][j][e], asy[i][j][e], asxx[i][j][e], asyy[i][j][e],
                         axy[i][j][e], o);
        }
      }
}

// presence words with a 16-byte-aligned row stride (the mask tensor map's
// global stride must be a multiple of 16 bytes)
__global__ void pad_mask_kernel(const uint32_t* __restrict__ mask, int64_t W, int64_t Wp, uint32_t* __restrict__ out) {
  const int64_t f = blockIdx.x;
  for (int64_t w = threadIdx.x; w < Wp; w += blockDim.x) out[f * Wp + w] = w < W ? mask[f * W + w] : 0u;
}

// Split-K reduction (fixed split order => deterministic) + epilogue.
__global__ void pearson_splitk_finish_kernel(const double* __restrict__ ws, int64_t F, int64_t NT,
                                             int64_t tile0, int64_t ntiles, int nsplit, int64_t lo,
                                             int64_t hi, Outs o) {
  const int64_t total = ntiles * T * T;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tl = idx / (T * T);
    const int rc = (int)(idx % (T * T));
    int64_t I, J;
    ps_tri_tile(tile0 + tl, NT, &I, &J);
    const int64_t g = I * T + rc / T, h = J * T + rc % T;
    if (g < lo || g >= hi || h < g || h >= F) continue;
    double m[6] = {0, 0, 0, 0, 0, 0};
    for (int sp = 0; sp < nsplit; ++sp) {
      const double* w = ws + (tl * nsplit + sp) * 6 * T * T + rc;
#pragma unroll
      for (int q = 0; q < 6; ++q) m[q] += w[q * T * T];
    }
    pearson_finish(g, h, F, (int)m[0], m[1], m[2], m[3], m[4], m[5], o);
  }
}

// Exact replay of the reference's sequential two-pass loop (continuous.py:77-103)
// for pairs the fast path could not decide.  One thread per pair.
__global__ void pearson_replay_kernel(const double* __restrict__ vals, int64_t ld,
                                      const uint32_t* __restrict__ mask, int64_t W, int64_t S,
                                      int64_t F, const int2* __restrict__ list,
                                      const int* __restrict__ count_ptr, int cap, int64_t lo,
                                      int64_t hi, Outs o) {
  // The list length is only known on the device; an overflowing list falls
  // back to re-deciding every pair in range (pathological inputs only).
  const int count = *count_ptr;
  if (count == 0) return;
  const int all_pairs = count > cap;
  const int64_t n_items = all_pairs ? (hi - lo) * F : count;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    int64_t g, h;
    if (all_pairs) {
      g = lo + it / F;
      h = it % F;
      if (h < g) continue;
    } else {
      g = list[it].x;
      h = list[it].y;
    }
    const double* xg = vals + g * ld;
    const double* xh = vals + h * ld;
    const uint32_t* mg = mask + g * W;
    const uint32_t* mh = mask + h * W;
    int64_t n = 0;
    double sum_x = 0.0, sum_y = 0.0;
    for (int64_t s = 0; s < S; ++s) {
      if ((mg[s >> 5] & mh[s >> 5]) >> (s & 31) & 1u) {
        ++n;
        sum_x += xg[s];
        sum_y += xh[s];
      }
    }
    double r = PS_NAN, p = PS_NAN;
    if (n > 1) {
      const double mx = sum_x / (double)n, my = sum_y / (double)n;
      double sxx = 0.0, syy = 0.0, sxy = 0.0;
      for (int64_t s = 0; s < S; ++s) {
        if ((mg[s >> 5] & mh[s >> 5]) >> (s & 31) & 1u) {
          const double dx = xg[s] - mx, dy = xh[s] - my;
          sxx += dx * dx;
          syy += dy * dy;
          sxy += dx * dy;
        }
      }
      // the reference's test (continuous.py:34): NaN sums (NaN data under a
      // numeric sentinel) pass it and reach beta_sym_sf, which raises
      if (!(sxx <= 0.0 || syy <= 0.0)) {
        r = sxy / sqrt(sxx * syy);
        if (r > 1.0) r = 1.0;
        else if (r < -1.0) r = -1.0;
        if (n != 2) {
          if (o.defer_p) {
            p = (double)n;  // parked: pearson_p_kernel evaluates the tail from (r, n)
          } else {
            p = 2.0 * PS_BETA_SYM(fabs(r), 0.5 * (double)n - 1.0, o.err);
            if (p > 1.0) p = 1.0;
          }
        }
      }
    }
    put(o.stat, F, g, h, r);
    put(o.p, F, g, h, p);
    put(o.r2, F, g, h, r * r);
  }
}

}  // namespace

// default 1: x' once per element took the config-5 step 7209 -> 6627 ms
// (bitwise identical); precomputed squares (mode 2) measured no faster
// (613.6 vs 613.9 ms at 6000 x 10^5) and cost another F x ld buffer
// chunks per block barrier (PS_PEARSON_CPB: 1, 2 or 3; default 3: config-5
// recipe at 6000 x 10^5 614.4 (1) -> 603.0 (2) -> 600.0 ms (3, six stages,
// 224 KB), bitwise identical)
static int pearson_cpb() {
  const char* e = getenv("PS_PEARSON_CPB");
  const int v = e ? atoi(e) : 3;
  return v <= 1 ? 1 : v >= 3 ? 3 : 2;
}

static int pearson_mode() {
  const char* e = getenv("PS_PEARSON_MODE");
  const int m = e ? atoi(e) : 1;
  return m < 0 ? 0 : m > 2 ? 2 : m;
}

// (a function attribute is per device: set on every call)
template <int MODE, int CPB>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(pearson_tile_kernel<MODE, CPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes<MODE, CPB>());
}
static cudaError_t set_tile_attrs() {
  cudaError_t e = set_attr<0, 1>();
  if (e == cudaSuccess) e = set_attr<1, 1>();
  if (e == cudaSuccess) e = set_attr<2, 1>();
  if (e == cudaSuccess) e = set_attr<1, 2>();
  if (e == cudaSuccess) e = set_attr<1, 3>();
  return e;
}

static void launch_tiles(int mode, unsigned grid, cudaStream_t s, const double* vals, const double* sq, int64_t ld,
                         const uint32_t* mask, int64_t W, const double* center, int64_t F, int64_t NT, int64_t tile0,
                         int64_t lo, int64_t hi, int nsplit, int64_t cps, const Outs& o, double* ws, int colmajor) {
  const int cpb = pearson_cpb();
  if (mode == 1 && cpb == 3)
    pearson_tile_kernel<1, 3><<<grid, NTHR, smem_bytes<1, 3>(), s>>>(vals, sq, ld, mask, W, center, F, NT, tile0, lo,
                                                                     hi, nsplit, cps, o, ws, colmajor);
  else if (mode == 1 && cpb == 2)
    pearson_tile_kernel<1, 2><<<grid, NTHR, smem_bytes<1, 2>(), s>>>(vals, sq, ld, mask, W, center, F, NT, tile0, lo,
                                                                     hi, nsplit, cps, o, ws, colmajor);
  else if (mode == 2)
    pearson_tile_kernel<2, 1><<<grid, NTHR, smem_bytes<2, 1>(), s>>>(vals, sq, ld, mask, W, center, F, NT, tile0, lo,
                                                                     hi, nsplit, cps, o, ws, colmajor);
  else if (mode == 1)
    pearson_tile_kernel<1, 1><<<grid, NTHR, smem_bytes<1, 1>(), s>>>(vals, sq, ld, mask, W, center, F, NT, tile0, lo,
                                                                     hi, nsplit, cps, o, ws, colmajor);
  else
    pearson_tile_kernel<0, 1><<<grid, NTHR, smem_bytes<0, 1>(), s>>>(vals, sq, ld, mask, W, center, F, NT, tile0, lo,
                                                                     hi, nsplit, cps, o, ws, colmajor);
}

// TMA tensor maps of the pre-centred operands and the padded presence words
static PFN_cuTensorMapEncodeTiled_v12000 pearson_map_encoder() {
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

static int make_pearson_map(CUtensorMap* xmap, const double* xc, int64_t ld, int64_t F) {
  auto enc = pearson_map_encoder();
  if (!enc) return ps_fail(PS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)F};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {(cuuint32_t)TBOX, (cuuint32_t)T};
  cuuint32_t es[2] = {1, 1};
  if (enc(xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(xc), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return ps_fail(PS_ERR_CUDA, "pearson operand tensor map");
  return PS_OK;
}

// the TMA-fed tiles (PS_PEARSON_TMA=0: cp.async tiles) -- pre-centred
// operands, no split-K; the operand rows must be 16-byte multiples
static bool pearson_tma_on(int mode, int nsplit, int64_t ld) {
  const char* e = getenv("PS_PEARSON_TMA");
  const bool on = !(e && e[0] == '0');
  return on && mode == 1 && nsplit == 1 && (ld * 8) % 16 == 0;
}

// x' = x - c_f (0 where missing) for rows [f0, f1) of m into out (F x ld);
// shared with the ANOVA / t-test moment contraction (ps_group.cu)
int ps_center_rows(const ps_matrix* m, double* out, int64_t f0, int64_t f1, cudaStream_t s) {
  if (f1 <= f0) return PS_OK;
  center_rows_kernel<<<(unsigned)(f1 - f0), 256, 0, s>>>(m->d_vals, m->ld, m->d_mask, m->W, m->d_center, out, nullptr,
                                                         f0);
  PS_LAUNCHED();
  return PS_OK;
}

int ps_pearson_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* r2,
                   cudaStream_t s) {
  const int64_t F = a->F;
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(F, hi);
  if (hi <= lo || (!stat && !p && !r2)) return PS_OK;
  ps_device_state* ds = ps_state();
  const int64_t NT = ps_ceil_div(F, T);
  const int64_t I0 = lo / T, I1 = (hi - 1) / T;
  const int64_t tile0 = ps_tri_offset(I0, NT);
  const int64_t ntiles = ps_tri_offset(I1 + 1, NT) - tile0;
  const int64_t W = a->W;
  // split-K so that small problems still fill the machine (>= 2 CTAs per SM).
  // The split count is a function of the WHOLE triangle (F, S), never of the
  // range: a pair's k-order -- hence every bit of its result -- is the same
  // whichever range (rank, thread block of the reference) computes it.
  int nsplit = 1;
  const int64_t want = 2LL * ds->num_sms;
  const int64_t ntiles_all = NT * (NT + 1) / 2;
  if (ntiles_all < want) {
    nsplit = (int)std::min<int64_t>(ps_ceil_div(want, ntiles_all), std::max<int64_t>(1, W / 4));
    nsplit = std::max(1, nsplit);
  }
  const int64_t cps = ps_ceil_div(W, nsplit);
  nsplit = (int)ps_ceil_div(W, cps);

  const int64_t npairs = (hi - lo) * F;  // upper bound on pairs touched
  const int cap = (int)std::min<int64_t>(npairs, 1 << 22);
  // (the deferred tail needs r: only when stat is an output; PS_PEARSON_INLINE_P=1 keeps it in the tiles)
  // (deferred only when the tiles fill the GPU: config 5 6000 x 10^5 600.1 ->
  // 588.7 ms; at 200 x 1000 the extra launch costs more than it saves)
  const bool defer = p && stat && !getenv("PS_PEARSON_INLINE_P") && ntiles_all >= ds->num_sms;
  Outs o{stat, p, r2, nullptr, nullptr, cap, ds->d_err, defer ? 1 : 0};
  double* ws = nullptr;
  PS_CUDA(ps_alloc(&o.replay, (size_t)cap, s));
  PS_CUDA(ps_alloc(&o.replay_count, 1, s));
  PS_CUDA(cudaMemsetAsync(o.replay_count, 0, sizeof(int), s));
  if (nsplit > 1) PS_CUDA(ps_alloc(&ws, (size_t)(ntiles * nsplit * 6 * T * T), s));

  // operand mode (PS_PEARSON_MODE: 0 raw, 1 pre-centred x', 2 x' and x'^2)
  const int mode = pearson_mode();
  double *xc = nullptr, *xq = nullptr;
  if (mode >= 1) {
    PS_CUDA(ps_alloc(&xc, (size_t)(F * a->ld), s));
    if (mode == 2) PS_CUDA(ps_alloc(&xq, (size_t)(F * a->ld), s));
    center_rows_kernel<<<(unsigned)F, 256, 0, s>>>(a->d_vals, a->ld, a->d_mask, W, a->d_center, xc, xq, 0);
    PS_LAUNCHED();
  }
  PS_CUDA(set_tile_attrs());
  const int64_t grid = ntiles * nsplit;
  uint32_t* mpad = nullptr;
  if (pearson_tma_on(mode, nsplit, a->ld)) {
    const int64_t Wp = ps_round_up(W, 4);
    PS_CUDA(ps_alloc(&mpad, (size_t)(F * Wp), s));
    pad_mask_kernel<<<(unsigned)F, 256, 0, s>>>(a->d_mask, W, Wp, mpad);
    PS_LAUNCHED();
    CUtensorMap xmap;
    int rc = make_pearson_map(&xmap, xc, a->ld, F);
    if (rc) return rc;
    // large F: the four masked moments on the int8 tensor cores, Sxy alone on DMMA
    const bool mom = ps_moments_on(F, a->S);
    const bool i8 = mom && ps_sxy_int8(a->S);  // Sxy and n from int8 digit products too: no DMMA tiles
    if (mom) {
      PS_CUDA(ps_alloc(&o.sxy, (size_t)(F * F), s));
      PS_CUDA(ps_alloc(&o.nn, (size_t)(F * F), s));
    }
    PS_CUDA(cudaFuncSetAttribute(pearson_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTmaSmem));
    PS_CUDA(cudaFuncSetAttribute(pearson_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTmaSmemPre));
    if (!i8) {
      ps_prof_begin("pearson_tile", s);
      if (mom)
        pearson_tma_kernel<true><<<(unsigned)grid, NTHR, kTmaSmemPre, s>>>(xmap, mpad, Wp, W, F, NT, tile0, lo, hi, o,
                                                                           0);
      else
        pearson_tma_kernel<false><<<(unsigned)grid, NTHR, kTmaSmem, s>>>(xmap, mpad, Wp, W, F, NT, tile0, lo, hi, o,
                                                                         0);
      ps_prof_end(s);
      PS_LAUNCHED();
    }
    if (mom) {
      double *msx = nullptr, *msq = nullptr;
      int32_t *me1 = nullptr, *me2 = nullptr;
      rc = ps_pearson_moments(a, xc, lo, hi, &msx, &msq, &me1, &me2, i8 ? o.sxy : nullptr, i8 ? o.nn : nullptr, s);
      if (rc) return rc;
      pearson_pairs_kernel<<<ds->num_sms * 16, 128, 0, s>>>(F, lo, hi, o, msx, msq, me1, me2, i8 ? 1 : 0);
      PS_LAUNCHED();
      ps_free(msx, s);
      ps_free(msq, s);
      ps_free(me1, s);
      ps_free(me2, s);
      ps_free(o.sxy, s);
      ps_free(o.nn, s);
    }
  } else {
    ps_prof_begin("pearson_tile", s);
    launch_tiles(mode, (unsigned)grid, s, mode >= 1 ? xc : a->d_vals, xq, a->ld, a->d_mask, W, a->d_center, F, NT,
                 tile0, lo, hi, nsplit, cps, o, ws, 0);
    ps_prof_end(s);
    PS_LAUNCHED();
  }
  ps_free(mpad, s);
  ps_free(xc, s);
  ps_free(xq, s);
  if (nsplit > 1) {
    const int64_t total = ntiles * T * T;
    const int blocks = (int)std::min<int64_t>(ps_ceil_div(total, 256), (int64_t)ds->num_sms * 8);
    pearson_splitk_finish_kernel<<<blocks, 256, 0, s>>>(ws, F, NT, tile0, ntiles, nsplit, lo, hi,
                                                        o);
    PS_LAUNCHED();
  }
  {  // replays first: with deferred p they park n for the p-value pass
    const int blocks = ds->num_sms * 4;
    pearson_replay_kernel<<<blocks, 64, 0, s>>>(a->d_vals, a->ld, a->d_mask, W, a->S, F, o.replay,
                                                o.replay_count, cap, lo, hi, o);
    PS_LAUNCHED();
  }
  if (o.defer_p) {
    pearson_p_kernel<<<ds->num_sms * 16, 128, 0, s>>>(stat, p, F, lo, hi, ds->d_err);
    PS_LAUNCHED();
  }
  ps_free(o.replay, s);
  ps_free(o.replay_count, s);
  ps_free(ws, s);
  return PS_OK;
}

// ---------------------------------------------------------------------------
// Incremental Pearson (ps_run overlaps the tiles with the input upload): the
// tile columns J whose rows [0, (J+1) T) are uploaded run on the walk
// streams in column-major triangle order (no split-K: results are identical
// to the whole-matrix launch tile by tile); the replay of ill-conditioned
// pairs runs once all tiles are done.
struct ps_pearson_job {
  ps_matrix* a = nullptr;
  Outs o{};
  int mode = 0;            // operand mode (pearson_mode)
  bool tma = false;        // TMA-fed tiles (padded presence words + tensor maps)
  uint32_t* mpad = nullptr;
  int64_t Wp = 0;
  CUtensorMap xmap{};
  double* xc = nullptr;    // pre-centred x' (mode >= 1)
  double* xq = nullptr;    // x'^2 (mode 2)
  bool moments = false;    // large F: moments on the int8 tensor cores
  bool i8 = false;         // ... and Sxy / n too (no DMMA tiles): the int8 job follows the upload
  ps_moments_job* mj = nullptr;
  int64_t mcols = 0;       // 256-tile columns handed to the int8 job

  int64_t c_done = 0;      // rows centred
  int64_t J_done = 0;  // tile columns launched
  int nws = 0;
  cudaStream_t home = nullptr;
};

int ps_pearson_begin(ps_matrix* a, double* stat, double* p, double* r2, cudaStream_t s, ps_pearson_job** out) {
  *out = nullptr;
  ps_pearson_job* j = new ps_pearson_job();
  j->a = a;
  j->home = s;
  const int64_t F = a->F;
  const int cap = (int)std::min<int64_t>(F * F, 1 << 22);
  const int64_t nt = ps_ceil_div(F, T);
  j->o = Outs{stat, p, r2, nullptr, nullptr, cap, ps_state()->d_err,
              (p && stat && !getenv("PS_PEARSON_INLINE_P") && nt * (nt + 1) / 2 >= ps_state()->num_sms) ? 1 : 0};
  cudaError_t e = ps_alloc(&j->o.replay, (size_t)cap, s);
  if (e == cudaSuccess) e = ps_alloc(&j->o.replay_count, 1, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(j->o.replay_count, 0, sizeof(int), s);
  j->mode = pearson_mode();
  if (e == cudaSuccess && j->mode >= 1) e = ps_alloc(&j->xc, (size_t)(F * a->ld), s);
  if (e == cudaSuccess && j->mode == 2) e = ps_alloc(&j->xq, (size_t)(F * a->ld), s);
  if (e == cudaSuccess) e = set_tile_attrs();
  j->tma = pearson_tma_on(j->mode, 1, a->ld);
  if (e == cudaSuccess && j->tma) {
    j->Wp = ps_round_up(a->W, 4);
    e = ps_alloc(&j->mpad, (size_t)(F * j->Wp), s);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(pearson_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kTmaSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(pearson_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kTmaSmemPre);
    j->moments = ps_moments_on(F, a->S);
    j->i8 = j->moments && ps_sxy_int8(a->S);
    if (e == cudaSuccess && j->moments) e = ps_alloc(&j->o.sxy, (size_t)(F * F), s);
    if (e == cudaSuccess && j->moments) e = ps_alloc(&j->o.nn, (size_t)(F * F), s);
    // (after Sxy / n exist: the job writes them)
    if (e == cudaSuccess && j->i8 && ps_moments_job_begin(a, j->xc, j->o.sxy, j->o.nn, s, &j->mj) != PS_OK)
      e = cudaErrorMemoryAllocation;
    if (e == cudaSuccess && make_pearson_map(&j->xmap, j->xc, a->ld, F) != PS_OK)
      e = cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) {
    cudaStreamSynchronize(s);
    ps_free(j->o.replay, s);
    ps_free(j->o.replay_count, s);
    ps_free(j->xc, s);
    ps_free(j->xq, s);
    ps_free(j->mpad, s);
    ps_free(j->o.sxy, s);
    ps_free(j->o.nn, s);
    ps_moments_job_abort(j->mj, s);
    delete j;
    return ps_cuda_check(e, "pearson setup");
  }
  *out = j;
  return PS_OK;
}

// centre the rows [c_done, r1) on `s` -- the stream every later tile launch
// is ordered after (the incremental launches' walk streams wait on it)
static int pearson_center_upto(ps_pearson_job* j, int64_t r1, cudaStream_t s) {
  ps_matrix* a = j->a;
  r1 = std::min<int64_t>(a->F, r1);
  if (!j->xc || r1 <= j->c_done) return PS_OK;
  center_rows_kernel<<<(unsigned)(r1 - j->c_done), 256, 0, s>>>(a->d_vals, a->ld, a->d_mask, a->W, a->d_center, j->xc,
                                                                j->xq, j->c_done);
  PS_LAUNCHED();
  if (j->tma) {
    pad_mask_kernel<<<(unsigned)(r1 - j->c_done), 256, 0, s>>>(a->d_mask + j->c_done * a->W, a->W, j->Wp,
                                                              j->mpad + j->c_done * j->Wp);
    PS_LAUNCHED();
  }
  j->c_done = r1;
  return PS_OK;
}

static int pearson_columns(ps_pearson_job* j, int64_t J0, int64_t J1, cudaStream_t s) {
  if (J1 <= J0) return PS_OK;
  ps_matrix* a = j->a;
  const int64_t F = a->F, NT = ps_ceil_div(F, T), W = a->W;
  const int64_t t0 = J0 * (J0 + 1) / 2, t1 = J1 * (J1 + 1) / 2;
  ps_prof_begin("pearson_tile", s);
  if (j->tma && j->moments)
    pearson_tma_kernel<true><<<(unsigned)(t1 - t0), NTHR, kTmaSmemPre, s>>>(j->xmap, j->mpad, j->Wp, W, F, NT, t0, 0, F,
                                                                         j->o, 1);
  else if (j->tma)
    pearson_tma_kernel<false><<<(unsigned)(t1 - t0), NTHR, kTmaSmem, s>>>(j->xmap, j->mpad, j->Wp, W, F, NT, t0, 0, F,
                                                                          j->o, 1);
  else
    launch_tiles(j->mode, (unsigned)(t1 - t0), s, j->mode >= 1 ? j->xc : a->d_vals, j->xq, a->ld, a->d_mask, W,
                 a->d_center, F, NT, t0, 0, F, 1, W, j->o, nullptr, 1);
  ps_prof_end(s);
  PS_LAUNCHED();
  return PS_OK;
}

int ps_pearson_upto(ps_pearson_job* j, int64_t h1, cudaStream_t s) {
  const int64_t F = j->a->F;
  const int64_t J1 = h1 >= F ? ps_ceil_div(F, T) : h1 / T;  // whole tile columns only
  if (J1 <= j->J_done) return PS_OK;
  int rc0 = pearson_center_upto(j, J1 * T, s);
  if (rc0) return rc0;
  if (j->i8) {  // rows of the chunk, then the complete 256-tile columns on a walk stream
    const int64_t F = j->a->F, rows = j->c_done;  // centred rows only
    const int64_t NTm = ps_ceil_div(F, kMomentTile);
    const int64_t JM = rows >= F ? NTm : rows / kMomentTile;
    // the whole int8 job on ONE walk stream (in order: a column block reads
    // the digit planes of every earlier chunk), after the centring on `s`;
    // the high-priority upload stream only centres
    cudaStream_t w = ps_walk_stream(0, s);
    j->nws = std::max(j->nws, 1);
    int rc = ps_moments_job_rows(j->mj, rows, w);
    // column blocks of at least a few tiles: single tile columns are too small
    // launches (dozens of products each) to fill the GPU
    if (rc || JM - j->mcols < std::min<int64_t>(kMomBlock, NTm - j->mcols)) return rc;
    j->mcols = JM;
    return ps_moments_job_cols(j->mj, JM, w);
  }
  cudaStream_t w = ps_walk_stream(j->nws++, s);
  int rc = pearson_columns(j, j->J_done, J1, w);
  j->J_done = J1;
  return rc;
}

int ps_pearson_end(ps_pearson_job* j, cudaStream_t s, cudaEvent_t stat_ready) {
  ps_device_state* ds = ps_state();
  int rc = ps_walk_streams_join(j->nws, s);
  ps_matrix* a = j->a;
  if (!rc) rc = pearson_center_upto(j, a->F, s);
  if (!rc && !j->i8) rc = pearson_columns(j, j->J_done, ps_ceil_div(a->F, T), s);
  if (!rc && j->moments) {
    double *msx = nullptr, *msq = nullptr;
    int32_t *me1 = nullptr, *me2 = nullptr;
    if (j->i8) {
      rc = ps_moments_job_rows(j->mj, a->F, s);
      if (!rc) rc = ps_moments_job_cols(j->mj, ps_ceil_div(a->F, kMomentTile), s);
      if (!rc) rc = ps_moments_job_end(j->mj, &msx, &msq, &me1, &me2, j->home);
      j->mj = nullptr;
    } else {
      rc = ps_pearson_moments(a, j->xc, 0, a->F, &msx, &msq, &me1, &me2, nullptr, nullptr, s);
    }
    if (!rc) {
      pearson_pairs_kernel<<<ds->num_sms * 16, 128, 0, s>>>(a->F, 0, a->F, j->o, msx, msq, me1, me2, j->i8 ? 1 : 0);
      ps_count_launch();
      if (cudaGetLastError() != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "pearson pairs launch");
    }
    ps_free(msx, s);
    ps_free(msq, s);
    ps_free(me1, s);
    ps_free(me2, s);
  }
  // exact replays first (with deferred p they park n like the tiles), so the
  // statistic matrices are final before the p-value pass
  if (!rc) {
    pearson_replay_kernel<<<ds->num_sms * 4, 64, 0, s>>>(a->d_vals, a->ld, a->d_mask, a->W, a->S, a->F, j->o.replay,
                                                         j->o.replay_count, j->o.replay_cap, 0, a->F, j->o);
    ps_count_launch();
    if (cudaGetLastError() != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "pearson replay launch");
  }
  if (!rc && stat_ready) {
    const cudaError_t e = cudaEventRecord(stat_ready, s);
    if (e != cudaSuccess) rc = ps_cuda_check(e, "pearson stat event");
  }
  if (!rc && j->o.defer_p) {
    pearson_p_kernel<<<ds->num_sms * 16, 128, 0, s>>>(j->o.stat, j->o.p, a->F, 0, a->F, ds->d_err);
    ps_count_launch();
    if (cudaGetLastError() != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "pearson p launch");
  }
  ps_free(j->o.replay, j->home);
  ps_free(j->o.replay_count, j->home);
  ps_free(j->xc, j->home);
  ps_free(j->xq, j->home);
  ps_free(j->mpad, j->home);
  ps_free(j->o.sxy, j->home);
  ps_free(j->o.nn, j->home);
  delete j;
  return rc;
}

void ps_pearson_abort(ps_pearson_job* j, cudaStream_t s) {
  if (!j) return;
  cudaStreamSynchronize(s);
  cudaDeviceSynchronize();
  ps_free(j->o.replay, j->home);
  ps_free(j->o.replay_count, j->home);
  ps_free(j->xc, j->home);
  ps_free(j->xq, j->home);
  ps_free(j->mpad, j->home);
  ps_free(j->o.sxy, j->home);
  ps_free(j->o.nn, j->home);
  ps_moments_job_abort(j->mj, j->home);
  delete j;
}
