// ps_group.cu -- ANOVA and t-test: per-level moments as one FP64 tensor-core
// contraction of label one-hots against the continuous matrix.
//
// Replaces _anova_block -> _anova_rows -> _anova_finish and _ttest_block ->
// _ttest_rows -> _ttest_finish (engine.py:245-293; mixed.py:121-202,
// :453-520).  For label row j of feature g (level j; for the t-test the two
// rows are "label == 0" and "label != 0", mixed.py:192-201) and continuous
// feature h, over jointly present samples:
//     n_j = popc(onehot_gj & m_h),  S_j = sum x'_h,  Q_j = sum x'_h^2
// with x' = x - c_h (per-feature pivot) on present cells, 0 elsewhere.  S and
// Q are DMMA.8x8x4 contractions (one-hot x [X', X'^2]); n is exact on the
// integer pipe.  The epilogue evaluates the reference formulas in centred
// form (the pivot cancels from every deviation) and replays the reference's
// sequential raw one-pass loop exactly for pairs whose within-group sums are
// ill-conditioned, so degenerate-variance decisions (ssw_j > 0, SSW == 0,
// pooled == 0) match bit for bit.
//
// Algorithmic work: 4 k_g FP64 flops per pair-sample (ANOVA), 8 (t-test).
#include "ps_internal.cuh"
#include "ps_specfun.cuh"
#include <math_constants.h>
#include <algorithm>
#include <vector>

namespace {

constexpr int T = 64;        // rows (label levels) x cols (continuous features) per tile
constexpr int KC = 32;
constexpr int XS = KC + 4;
constexpr int NW = 8;        // 4 x 2 warps, 16 x 32 cells each
constexpr int NTH = NW * 32;
constexpr int WM = 2, WN = 4;
constexpr int NSTAGE = 3;
constexpr double kReplayTau = 1e-6;
constexpr double kCancelTau = 1e-5;  // mean differences below this fraction of the raw RMS are replayed
// The reference sums raw (uncentred) values in one pass, so its ssq - sum*mean
// and its group means carry a rounding error that grows ~ sqrt(n_j) eps raw:
// the replay thresholds grow with the group size so that any cell whose
// reference value could be off by more than ~1e-10 relative (data with a
// large offset over its spread, large groups) is replayed in the reference's
// own order (advisor finding; tests/test_gpu_mixed.py large-offset cases).
// Calibrated against the oracle by tests/calibrate_group_replay.py: outside
// the SSW rule no cell with error > 1e-10 has a mean spread above 6e-7
// sqrt(n) rms (2.5x margin).  Every replay costs a sequential pass over the
// pair's samples, so the margin is kept small: at 5e-6 config 4's ANOVA step
// went 6.4 -> 7.7 ms on replays of null pairs.
constexpr double kReplayK = 2.5e-6;   // gs replayed when <= kReplayK sqrt(n_j) raw
constexpr double kCancelK = 1.5e-6;   // SSB replayed when max |mean dev| <= kCancelK sqrt(n) rms
__device__ __forceinline__ double replay_tau(double n) { return fmax(kReplayTau, kReplayK * sqrt(n)); }
__device__ __forceinline__ double cancel_tau(double n) { return fmax(kCancelTau, kCancelK * sqrt(n)); }

struct Stage {
  double x[T][XS];
  uint32_t mh[T];
  uint32_t oh[T];
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// one-hot bit rows: row r = (feature row_feat[r], level row_level[r]); level
// -1 / -2 select the t-test rows (present && v == 0.0 / present && v != 0.0).
template <typename CT>
__global__ void onehot_bits_kernel(const CT* __restrict__ codes, int64_t ldc,
                                   const uint32_t* __restrict__ mask, const uint32_t* __restrict__ zero,
                                   int64_t W, const int32_t* __restrict__ row_feat,
                                   const int32_t* __restrict__ row_level, int64_t R, int64_t S,
                                   uint32_t* __restrict__ bits) {
  const int64_t r = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* out = bits + r * W;
  if (r >= R) {
    for (int64_t w = threadIdx.x; w < W; w += blockDim.x) out[w] = 0u;
    return;
  }
  const int f = row_feat[r], lev = row_level[r];
  if (lev < 0) {
    for (int64_t w = threadIdx.x; w < W; w += blockDim.x) {
      const uint32_t m = mask[f * W + w], z = zero[f * W + w];
      out[w] = lev == -1 ? (m & z) : (m & ~z);
    }
    return;
  }
  const CT* c = codes + f * ldc;
  for (int64_t w = warp; w < W; w += blockDim.x / 32) {
    const int64_t s = w * 32 + lane;
    const bool hit = s < S && c[s] == (CT)lev;
    const uint32_t b = __ballot_sync(PS_FULL, hit);
    if (lane == 0) out[w] = b;
  }
}

// M[r][h] moments over upper-left-aligned 64 x 64 tiles of (label rows x features)
// PC: vals holds the pre-centred x' (ps_center_rows; 0 where missing), so the
// DMMA loop skips the per-use subtract / select (bitwise the same operands)
template <bool PC>
__global__ void __launch_bounds__(NTH, 2)
group_gemm_kernel(const uint32_t* __restrict__ ohbits, int64_t Rp, const double* __restrict__ vals,
                  int64_t ld, const uint32_t* __restrict__ mask, const double* __restrict__ center,
                  int64_t W, int64_t Fq, int64_t row_tile0, int64_t col_tile0, int64_t col_tiles,
                  int32_t* __restrict__ Mn,
                  double* __restrict__ Ms, double* __restrict__ Mq, int64_t kparts, int64_t part_stride,
                  int64_t ldm, int64_t mcol0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // split-K (grids too small to fill the SMs): part y covers mask words
  // [W y / kparts, W (y + 1) / kparts) and writes its own partial moments
  const int64_t kc0 = W * blockIdx.y / kparts, kc1 = W * (blockIdx.y + 1) / kparts;
  Mn += blockIdx.y * part_stride;
  Ms += blockIdx.y * part_stride;
  Mq += blockIdx.y * part_stride;
  Stage* st = reinterpret_cast<Stage*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp >> 1, wj = warp & 1;
  const int64_t rt = row_tile0 + blockIdx.x / col_tiles, ct = col_tile0 + blockIdx.x % col_tiles;
  const int64_t row0 = rt * T, col0 = ct * T;
  const int fr = lane >> 2, fk = lane & 3;
  double cj[WN];
#pragma unroll
  for (int q = 0; q < WN; ++q) {
    const int64_t gc = col0 + wj * 8 * WN + q * 8 + fr;
    cj[q] = gc < Fq ? center[gc] : 0.0;
  }
  double as[WM][WN][2], aq[WM][WN][2];
  int an[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        as[i][j][e] = aq[i][j][e] = 0.0;
        an[i][j][e] = 0;
      }
  constexpr int LQ = (T * KC / 2) / NTH;
  auto issue = [&](int64_t c, Stage& sd) {
#pragma unroll
    for (int q = 0; q < LQ; ++q) {
      const int idx = tid + q * NTH;
      const int r = idx >> 4, c2 = idx & 15;
      const int64_t gj = min(col0 + r, Fq - 1);
      const unsigned sj = (unsigned)__cvta_generic_to_shared(&sd.x[r][c2 * 2]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sj), "l"(vals + gj * ld + c * KC + c2 * 2));
    }
    if (tid < T) {
      const int64_t gc = col0 + tid;
      sd.mh[tid] = gc < Fq ? mask[gc * W + c] : 0u;
    } else if (tid < 2 * T) {
      sd.oh[tid - T] = ohbits[(row0 + tid - T) * W + c];
    }
    asm volatile("cp.async.commit_group;");
  };
  for (int q = 0; q < NSTAGE - 1; ++q) {
    if (kc0 + q < kc1) issue(kc0 + q, st[q]);
    else asm volatile("cp.async.commit_group;");
  }
  for (int64_t c = kc0; c < kc1; ++c) {
    const int cur = (int)((c - kc0) % NSTAGE);
    asm volatile("cp.async.wait_group %0;" ::"n"(NSTAGE - 2));
    __syncthreads();
    {
      const int64_t cn = c + NSTAGE - 1;
      if (cn < kc1) issue(cn, st[(int)((cn - kc0) % NSTAGE)]);
      else asm volatile("cp.async.commit_group;");
    }
    const Stage& s = st[cur];
    uint32_t orow[WM], mcol[WN];
#pragma unroll
    for (int q = 0; q < WM; ++q) orow[q] = s.oh[wi * 8 * WM + q * 8 + fr];
#pragma unroll
    for (int q = 0; q < WN; ++q) mcol[q] = s.mh[wj * 8 * WN + q * 8 + fr];
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      const int k = kk * 4 + fk;
      double oa[WM], xb[WN], xb2[WN];
#pragma unroll
      for (int q = 0; q < WM; ++q) oa[q] = ((orow[q] >> k) & 1u) ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < WN; ++q) {
        const bool pb = (mcol[q] >> k) & 1u;
        xb[q] = PC ? s.x[wj * 8 * WN + q * 8 + fr][k] : (pb ? s.x[wj * 8 * WN + q * 8 + fr][k] - cj[q] : 0.0);
        xb2[q] = xb[q] * xb[q];
      }
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) {
          dmma(as[i][j][0], as[i][j][1], oa[i], xb[j]);
          dmma(aq[i][j][0], aq[i][j][1], oa[i], xb2[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) an[i][j][e] += __popc(orow[i] & s.mh[wj * 8 * WN + j * 8 + 2 * fk + e]);
  }
  asm volatile("cp.async.wait_group 0;");
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = row0 + wi * 8 * WM + i * 8 + fr;
        const int64_t h = col0 + wj * 8 * WN + j * 8 + 2 * fk + e;
        if (h >= Fq) continue;
        const int64_t o = r * ldm + (h - mcol0);  // M (ldm = Fq) or a column-window partial
        Mn[o] = an[i][j][e];
        Ms[o] = as[i][j][e];
        Mq[o] = aq[i][j][e];
      }
}

// Fixed-order sum of split-K partials of a column window [c0, c0 + width)
// (partials laid out rows x width) into M (rows x Fq).
__global__ void group_parts_reduce_cols_kernel(const int32_t* __restrict__ Pn, const double* __restrict__ Ps,
                                               const double* __restrict__ Pq, int64_t kparts, int64_t stride,
                                               int64_t rows, int64_t width, int64_t c0, int64_t Fq,
                                               int32_t* __restrict__ Mn, double* __restrict__ Ms,
                                               double* __restrict__ Mq) {
  const int64_t n = rows * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / width, c = i - r * width;
    if (c0 + c >= Fq) continue;
    int32_t cn = 0;
    double cs = 0.0, cq = 0.0;
    for (int64_t y = 0; y < kparts; ++y) {
      cn += Pn[y * stride + i];
      cs += Ps[y * stride + i];
      cq += Pq[y * stride + i];
    }
    const int64_t o = r * Fq + c0 + c;
    Mn[o] = cn;
    Ms[o] = cs;
    Mq[o] = cq;
  }
}

// Fixed-order sum of the split-K partial moments (deterministic).
__global__ void group_parts_reduce_kernel(const int32_t* __restrict__ Pn, const double* __restrict__ Ps,
                                          const double* __restrict__ Pq, int64_t kparts, int64_t stride,
                                          int64_t r0, int64_t r1, int64_t Fq, int32_t* __restrict__ Mn,
                                          double* __restrict__ Ms, double* __restrict__ Mq) {
  const int64_t n = (r1 - r0) * Fq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = r0 * Fq + i;
    int32_t cn = 0;
    double cs = 0.0, cq = 0.0;
    for (int64_t y = 0; y < kparts; ++y) {
      cn += Pn[y * stride + idx];
      cs += Ps[y * stride + idx];
      cq += Pq[y * stride + idx];
    }
    Mn[idx] = cn;
    Ms[idx] = cs;
    Mq[idx] = cq;
  }
}

struct Outs {
  double* stat;
  double* p;
  double* eff;
  int2* replay;
  int* replay_count;
  int replay_cap;
  int* err;
};

__device__ __forceinline__ void push_replay(const Outs& o, int64_t g, int64_t h) {
  const int slot = atomicAdd(o.replay_count, 1);
  if (slot < o.replay_cap) o.replay[slot] = make_int2((int)g, (int)h);
}

// element j of an array of GroupPart fields (stride = sizeof(GroupPart))
template <typename T>
struct Strided {
  const T* p;
  __device__ T operator[](int j) const;
};

// mixed.py:453-495 from raw (counts, sums, ssq) -- the exact reference form
template <typename CA, typename SA, typename QA>
__device__ void anova_finish_raw(CA counts, SA sums, QA ssq, int k, double* f_out, double* p_out, double* eta_out,
                                 int* err) {
  *f_out = *p_out = *eta_out = PS_NAN;
  if (k < 2) return;
  long long n = 0;
  double total = 0.0;
  for (int j = 0; j < k; ++j) {
    if (counts[j] == 0) return;
    n += counts[j];
    total += sums[j];
  }
  if (n <= k) return;
  const double grand = total / (double)n;
  double ssb = 0.0, ssw = 0.0, mlo = CUDART_INF, mhi = -CUDART_INF, scale = 0.0;
  for (int j = 0; j < k; ++j) {
    const double mj = sums[j] / (double)counts[j];
    const double dev = mj - grand;
    ssb += (double)counts[j] * dev * dev;
    const double gs = ssq[j] - sums[j] * mj;
    if (gs > 0.0) ssw += gs;
    if (mj < mlo) mlo = mj;
    if (mj > mhi) mhi = mj;
    if (fabs(mj) > scale) scale = fabs(mj);
  }
  if (ssw == 0.0) {
    if ((mhi - mlo) <= 1e-12 * scale) return;
    *f_out = CUDART_INF;
    *p_out = 0.0;
    *eta_out = 1.0;
    return;
  }
  const double f = (ssb / ((double)k - 1.0)) / (ssw / (double)(n - k));
  *f_out = f;
  *p_out = psf::f_sf(f, (double)k - 1.0, (double)(n - k), err);
  *eta_out = ssb / (ssb + ssw);
}

// mixed.py:121-157 from raw group sums -- the exact reference form
__device__ void ttest_finish_raw(long long n0, long long n1, double sum0, double sum1, double ss0,
                                 double ss1, int student, double* t_out, double* p_out, double* d_out,
                                 int* err) {
  *t_out = *p_out = *d_out = PS_NAN;
  if (n0 < 2 || n1 < 2 || n0 + n1 < 3) return;
  const double mean0 = sum0 / (double)n0, mean1 = sum1 / (double)n1;
  double var0 = (ss0 - sum0 * mean0) / (double)(n0 - 1);
  double var1 = (ss1 - sum1 * mean1) / (double)(n1 - 1);
  if (var0 < 0.0) var0 = 0.0;
  if (var1 < 0.0) var1 = 0.0;
  const double diff = mean0 - mean1;
  double t, dof, d;
  if (student) {
    const double pooled = ((double)(n0 - 1) * var0 + (double)(n1 - 1) * var1) / (double)(n0 + n1 - 2);
    if (pooled == 0.0) return;
    const double sp = sqrt(pooled);
    t = diff / (sp * sqrt(1.0 / (double)n0 + 1.0 / (double)n1));
    dof = (double)(n0 + n1 - 2);
    d = diff / sp;
  } else {
    if (var0 + var1 == 0.0) return;
    const double v0 = var0 / (double)n0, v1 = var1 / (double)n1;
    t = diff / sqrt(v0 + v1);
    dof = (v0 + v1) * (v0 + v1) / (v0 * v0 / (double)(n0 - 1) + v1 * v1 / (double)(n1 - 1));
    d = diff / sqrt(0.5 * (var0 + var1));
  }
  double p = 2.0 * psf::t_sf(fabs(t), dof, err);
  if (p > 1.0) p = 1.0;
  *t_out = t;
  *p_out = p;
  *d_out = d;
}

template <int KM>
__global__ void group_finish_kernel(int test, const int32_t* __restrict__ Mn, const double* __restrict__ Ms,
                                    const double* __restrict__ Mq, const int32_t* __restrict__ off,
                                    const int32_t* __restrict__ cat, const double* __restrict__ center,
                                    int64_t Fq, int64_t lo, int64_t hi, int student, Outs o) {
  for (int64_t idx = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < hi;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = idx / Fq, h = idx - g * Fq;
    const double c = center[h];
    double r0 = PS_NAN, r1 = PS_NAN, r2 = PS_NAN;
    if (test == PS_TEST_ANOVA) {
      const int k = cat[g];
      const int64_t base = (int64_t)off[g];
      if (k >= 2) {
        long long n = 0;
        double total = 0.0;
        bool empty = false, replay = false;
        for (int j = 0; j < k; ++j) {
          const int64_t cell = (base + j) * Fq + h;
          const long long nj = Mn[cell];
          if (nj == 0) empty = true;
          n += nj;
          total += Ms[cell];
        }
        if (!empty && n > k) {
          const double grand = total / (double)n;
          double ssb = 0.0, ssw = 0.0, mlo = CUDART_INF, mhi = -CUDART_INF, scale = 0.0;
          double maxdev = 0.0, rms = 0.0;
          for (int j = 0; j < k; ++j) {
            const int64_t cell = (base + j) * Fq + h;
            const double nj = (double)Mn[cell], sj = Ms[cell], qj = Mq[cell];
            const double mj = sj / nj;
            const double dev = mj - grand;
            ssb += nj * dev * dev;
            maxdev = fmax(maxdev, fabs(dev));
            rms = fmax(rms, sqrt(fmax(0.0, (qj + 2.0 * c * sj + nj * c * c) / nj)));  // raw-value RMS
            const double gs = qj - sj * mj;
            // the reference forms ssq - sum*mean in raw (uncentred) sums:
            // replay exactly whenever the sign of that could be in doubt
            if (!(gs > replay_tau(nj) * (qj + nj * c * c))) replay = true;
            ssw += gs;
            const double mr = mj + c;
            mlo = fmin(mlo, mr);
            mhi = fmax(mhi, mr);
            scale = fmax(scale, fabs(mr));
          }
          // group means that agree to ~1e-4 of the raw magnitudes: SSB is a
          // difference of nearly equal raw means, where the reference's own
          // one-pass rounding is ~1e-9 of it -- replay the reference exactly
          if (!(maxdev > cancel_tau((double)n) * rms)) replay = true;
          if (replay) {
            push_replay(o, g, h);
            continue;
          }
          const double f = (ssb / ((double)k - 1.0)) / (ssw / (double)(n - k));
          r0 = f;
          r1 = psf::f_sf(f, (double)k - 1.0, (double)(n - k), o.err);
          r2 = ssb / (ssb + ssw);
        }
      }
    } else {
      const int64_t c0 = (2 * g) * Fq + h, c1 = (2 * g + 1) * Fq + h;
      const long long n0 = Mn[c0], n1 = Mn[c1];
      if (!(n0 < 2 || n1 < 2 || n0 + n1 < 3)) {
        const double s0 = Ms[c0], s1 = Ms[c1], q0 = Mq[c0], q1 = Mq[c1];
        const double m0 = s0 / (double)n0, m1 = s1 / (double)n1;
        const double w0 = q0 - s0 * m0, w1 = q1 - s1 * m1;
        const double rms0 = sqrt(fmax(0.0, (q0 + 2.0 * c * s0 + (double)n0 * c * c) / (double)n0));
        const double rms1 = sqrt(fmax(0.0, (q1 + 2.0 * c * s1 + (double)n1 * c * c) / (double)n1));
        if (!(w0 > replay_tau((double)n0) * (q0 + (double)n0 * c * c)) ||
            !(w1 > replay_tau((double)n1) * (q1 + (double)n1 * c * c)) ||
            !(fabs(m0 - m1) > cancel_tau((double)(n0 + n1)) * fmax(rms0, rms1))) {  // (see the ANOVA SSB criterion)
          push_replay(o, g, h);
          continue;
        }
        const double var0 = w0 / (double)(n0 - 1), var1 = w1 / (double)(n1 - 1);
        const double diff = m0 - m1;
        double t, dof, d;
        if (student) {
          const double pooled = ((double)(n0 - 1) * var0 + (double)(n1 - 1) * var1) / (double)(n0 + n1 - 2);
          const double sp = sqrt(pooled);
          t = diff / (sp * sqrt(1.0 / (double)n0 + 1.0 / (double)n1));
          dof = (double)(n0 + n1 - 2);
          d = diff / sp;
        } else {
          const double v0 = var0 / (double)n0, v1 = var1 / (double)n1;
          t = diff / sqrt(v0 + v1);
          dof = (v0 + v1) * (v0 + v1) / (v0 * v0 / (double)(n0 - 1) + v1 * v1 / (double)(n1 - 1));
          d = diff / sqrt(0.5 * (var0 + var1));
        }
        double p = 2.0 * psf::t_sf(fabs(t), dof, o.err);
        if (p > 1.0) p = 1.0;
        r0 = t;
        r1 = p;
        r2 = d;
      }
    }
    if (o.stat) o.stat[idx] = r0;
    if (o.p) o.p[idx] = r1;
    if (o.eff) o.eff[idx] = r2;
  }
}

// Exact replay of _anova_rows / _ttest_rows (mixed.py:182-202, :498-520) for
// the ill-conditioned cells.  The reference sums every group sequentially in
// sample order; those per-group sums are independent, so one thread owns one
// (cell, group): it walks the jointly present samples of its group (one-hot
// row bits & the continuous mask, bit by bit in order) with raw fp64 one-pass
// sums in registers.  A second kernel applies the reference finish.
struct GroupPart {
  long long n;
  double sum, ssq;
};
template <typename T>
__device__ __forceinline__ T Strided<T>::operator[](int j) const {
  return *reinterpret_cast<const T*>(reinterpret_cast<const char*>(p) + (size_t)j * sizeof(GroupPart));
}

// One CTA of two warps per (cell, group) chain, 1024 samples per round:
// warp 0 compacts the group's jointly present values of round r+1 into one
// half of a shared double buffer, in sample order (coalesced loads issued one
// round ahead into registers, ballot-free shuffle compaction), while lane 0
// of warp 1 runs the reference's sequential one-pass sums over round r -- a
// chain of dependent DADDs (~8.3 cycles each on B200,
// tools/microbench/dadd_chain.cu), which is the kernel's floor.  One named
// barrier per round hands the halves over.
__global__ void __launch_bounds__(64)
group_replay_parts_kernel(const uint32_t* __restrict__ ohbits, const int32_t* __restrict__ off,
                          const double* __restrict__ vals, int64_t ld, const uint32_t* __restrict__ vmask, int64_t W,
                          const int2* __restrict__ items, int kslots, GroupPart* __restrict__ parts) {
  __shared__ __align__(16) double sbuf[2][1024];
  __shared__ uint32_t scnt[2];
  const int64_t t = blockIdx.x;
  const int it = (int)(t / kslots), j = (int)(t % kslots);
  const int64_t g = items[it].x, h = items[it].y;
  const int k = off[g + 1] - off[g];
  if (j >= k) return;  // block-uniform
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nr = ps_ceil_div(W, (int64_t)32);
  if (warp == 0) {
    const uint32_t* oh = ohbits + (int64_t)(off[g] + j) * W;
    const uint32_t* mh = vmask + h * W;
    const double* xv = vals + h * ld;
    const uint32_t lt = (1u << lane) - 1u;
    double v[32];
    uint32_t mw;
    auto fetch = [&](int64_t w0) {
      mw = w0 + lane < W ? __ldg(oh + w0 + lane) & __ldg(mh + w0 + lane) : 0u;
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = w0 + q < W ? __ldg(xv + (w0 + q) * 32 + lane) : 0.0;
    };
    fetch(0);
    for (int64_t r = 0; r < nr; ++r) {
      const uint32_t c = __popc(mw);
      uint32_t x = c;  // inclusive scan of the words' counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(PS_FULL, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t excl = x - c;
      double* buf = sbuf[r & 1];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t m = __shfl_sync(PS_FULL, mw, q);
        const uint32_t o = __shfl_sync(PS_FULL, excl, q);
        if ((m >> lane) & 1u) buf[o + __popc(m & lt)] = v[q];
      }
      if (lane == 31) scnt[r & 1] = x;
      if (r + 1 < nr) fetch((r + 1) * 32);
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
  } else {
    long long n = 0;
    double sum = 0.0, ssq = 0.0;
    for (int64_t r = 0; r < nr; ++r) {
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (lane == 0) {
        const double* buf = sbuf[r & 1];
        const uint32_t tot = scnt[r & 1];
        uint32_t i = 0;
        for (; i + 4 <= tot; i += 4) {
          const double v0 = buf[i], v1 = buf[i + 1], v2 = buf[i + 2], v3 = buf[i + 3];
          sum += v0;
          ssq += v0 * v0;
          sum += v1;
          ssq += v1 * v1;
          sum += v2;
          ssq += v2 * v2;
          sum += v3;
          ssq += v3 * v3;
        }
        for (; i < tot; ++i) {
          const double v = buf[i];
          sum += v;
          ssq += v * v;
        }
        n += tot;
      }
      __syncwarp();
    }
    if (lane == 0) parts[t] = GroupPart{n, sum, ssq};
  }
}

template <int KM>
__global__ void group_replay_finish_kernel(int test, const int2* __restrict__ items, int n_items, int kslots,
                                           const GroupPart* __restrict__ parts, const int32_t* __restrict__ off,
                                           int64_t Fq, int student, Outs o) {
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += gridDim.x * blockDim.x) {
    const int64_t g = items[it].x, h = items[it].y;
    const GroupPart* pp = parts + (int64_t)it * kslots;
    double r0, r1, r2;
    if (test == PS_TEST_ANOVA) {
      const int k = off[g + 1] - off[g];
      // the per-group sums stay in the parts array (any level count)
      anova_finish_raw(Strided<long long>{&pp[0].n}, Strided<double>{&pp[0].sum}, Strided<double>{&pp[0].ssq}, k,
                       &r0, &r1, &r2, o.err);
    } else {  // one-hot rows: "label == 0", "label != 0"
      ttest_finish_raw(pp[0].n, pp[1].n, pp[0].sum, pp[1].sum, pp[0].ssq, pp[1].ssq, student, &r0, &r1, &r2,
                       o.err);
    }
    const int64_t idx = g * Fq + h;
    if (o.stat) o.stat[idx] = r0;
    if (o.p) o.p[idx] = r1;
    if (o.eff) o.eff[idx] = r2;
  }
}

// LabelOutOfRange (mixed.py:511-515): a bad present label of a label row in
// [g0, g1) meeting a present value of any continuous feature in [h0, h1).
// (grid: x over mask words, y over chunks of 32 label rows)
__global__ void mixed_label_check_kernel(const uint32_t* __restrict__ bad, const uint32_t* __restrict__ vmask,
                                         int64_t W, int64_t g0, int64_t g1, int64_t h0, int64_t h1,
                                         int* __restrict__ err) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= W) return;
  const int64_t ga = g0 + (int64_t)blockIdx.y * 32, gb = min(g1, ga + 32);
  uint32_t anyb = 0;
  for (int64_t g = ga; g < gb; ++g) anyb |= bad[g * W + w];
  if (!anyb) return;
  uint32_t col = 0;
  for (int64_t h = h0; h < h1 && !(col & anyb); ++h) col |= vmask[h * W + w];
  if (col & anyb) ps_raise(err, PS_ERR_LABEL_OUT_OF_RANGE);
}

}  // namespace

static void launch_onehot_bits(ps_matrix* lab, int64_t W, const int32_t* rf, const int32_t* rl, int64_t R, int64_t Rp,
                               uint32_t* bits, cudaStream_t s) {
  if (lab->code_bytes == 2)
    onehot_bits_kernel<uint16_t><<<(unsigned)Rp, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(lab->d_codes), lab->ldc,
                                                             lab->d_mask, lab->d_zero, W, rf, rl, R, lab->S, bits);
  else
    onehot_bits_kernel<uint8_t><<<(unsigned)Rp, 256, 0, s>>>(lab->d_codes, lab->ldc, lab->d_mask, lab->d_zero, W, rf,
                                                            rl, R, lab->S, bits);
}

// LabelOutOfRange check of label rows [g0, g1) against continuous features
// [h0, h1) (also used by the Kruskal-Wallis walk, mixed.py:613-617).
int ps_mixed_label_check(ps_matrix* lab, ps_matrix* val, int64_t g0, int64_t g1, int64_t h0, int64_t h1,
                         cudaStream_t s) {
  if (g1 <= g0 || h1 <= h0) return PS_OK;
  const int64_t W = val->W;
  const dim3 grid((unsigned)ps_ceil_div(W, 128), (unsigned)ps_ceil_div(g1 - g0, 32));
  mixed_label_check_kernel<<<grid, 128, 0, s>>>(lab->d_bad, val->d_mask, W, g0, g1, h0, h1, ps_state()->d_err);
  PS_LAUNCHED();
  return PS_OK;
}

// Per-cell statistics from the moments of cells [lo, hi), then the exact
// in-order replay of the ill-conditioned cells (one host round trip for the
// replay count).  The replay list holds `cap` cells; when more cells need the
// replay (e.g. many constant continuous columns), the range is finished again
// in chunks of `cap` cells, each of which cannot overflow its list -- the
// reference answers every cell (mixed.py:453-495), so must we.
static int group_finish_chunk(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int student,
                              const int32_t* Mn, const double* Ms, const double* Mq, const int32_t* d_off,
                              const uint32_t* bits, int2* rep, int* repc, int cap, double* stat, double* p,
                              double* eff, int* count_out, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  const int64_t Fq = val->F, W = val->W;
  Outs o{stat, p, eff, rep, repc, cap, ds->d_err};
  PS_CUDA(cudaMemsetAsync(repc, 0, sizeof(int), s));
  const int blocks = (int)std::min<int64_t>(ps_ceil_div(hi - lo, 128), (int64_t)ds->num_sms * 16);
  const bool small = lab->cmax <= 16;
  if (small)
    group_finish_kernel<16><<<blocks, 128, 0, s>>>(test, Mn, Ms, Mq, d_off, lab->d_cat, val->d_center, Fq, lo,
                                                   hi, student, o);
  else
    group_finish_kernel<256><<<blocks, 128, 0, s>>>(test, Mn, Ms, Mq, d_off, lab->d_cat, val->d_center, Fq,
                                                    lo, hi, student, o);
  PS_LAUNCHED();
  int count = 0;
  PS_CUDA(cudaMemcpyAsync(&count, repc, sizeof(int), cudaMemcpyDeviceToHost, s));
  PS_CUDA(cudaStreamSynchronize(s));
  *count_out = count;
  if (count > cap) return PS_OK;  // the caller re-finishes in chunks
  const int n_items = count;
  if (n_items > 0) {
    const int kslots = test == PS_TEST_ANOVA ? std::max(2, lab->cmax) : 2;
    // batches of items so that the per-chain partials stay bounded (2^22
    // chains, 96 MiB) for any level count
    const int batch = (int)std::max<int64_t>(1, std::min<int64_t>(n_items, (1LL << 22) / kslots));
    GroupPart* parts = nullptr;
    PS_CUDA(ps_alloc(&parts, (size_t)batch * kslots, s));
    for (int b0 = 0; b0 < n_items; b0 += batch) {
      const int nb = std::min(batch, n_items - b0);
      group_replay_parts_kernel<<<(unsigned)((int64_t)nb * kslots), 64, 0, s>>>(
          bits, d_off, val->d_vals, val->ld, val->d_mask, W, rep + b0, kslots, parts);
      PS_LAUNCHED();
      const int fblocks = (int)std::min<int64_t>(ps_ceil_div(nb, 128), (int64_t)ds->num_sms * 4);
      if (small)
        group_replay_finish_kernel<16><<<fblocks, 128, 0, s>>>(test, rep + b0, nb, kslots, parts, d_off, Fq, student,
                                                               o);
      else
        group_replay_finish_kernel<256><<<fblocks, 128, 0, s>>>(test, rep + b0, nb, kslots, parts, d_off, Fq, student,
                                                                o);
      PS_LAUNCHED();
    }
    ps_free(parts, s);
  }
  return PS_OK;
}

static int group_finish_replay(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int student,
                               const int32_t* Mn, const double* Ms, const double* Mq, const int32_t* d_off,
                               const uint32_t* bits, int2* rep, int* repc, int cap, double* stat, double* p,
                               double* eff, cudaStream_t s) {
  int count = 0;
  int rc = group_finish_chunk(test, lab, val, lo, hi, student, Mn, Ms, Mq, d_off, bits, rep, repc, cap, stat, p, eff,
                              &count, s);
  for (int64_t c0 = lo; !rc && count > cap && c0 < hi; c0 += cap) {
    int cc = 0;
    rc = group_finish_chunk(test, lab, val, c0, std::min<int64_t>(hi, c0 + cap), student, Mn, Ms, Mq, d_off, bits,
                            rep, repc, cap, stat, p, eff, &cc, s);
  }
  return rc;
}

// replay list capacity (PS_REPLAY_CAP: tests shrink it to exercise the chunked re-finish)
static int replay_cap(int64_t cells) {
  int64_t lim = 1 << 22;
  if (const char* e = getenv("PS_REPLAY_CAP")) lim = std::max(1L, atol(e));
  return (int)std::max<int64_t>(1, std::min<int64_t>(cells, lim));
}

// Split-K factor of the moment contraction: enough K parts that two CTAs per
// SM are busy both for the whole (label rows x features) tile grid and for
// the column tiles of one upload chunk (run() contracts each staged chunk as
// it lands), at least 16 mask words per part.  A function of the matrices
// (R, Fq, S) only -- never of the launch -- so every cell's k-order, hence
// every bit, is the same for any range, rank or incremental launch.
static int64_t group_kparts(const ps_device_state* ds, int64_t R, int64_t Fq, int64_t W, int64_t ld) {
  const int64_t rtiles = ps_ceil_div(std::max<int64_t>(R, 1), T), ctiles = ps_ceil_div(Fq, T);
  const int64_t chunk_rows = (int64_t)std::max<size_t>(1, ps_stage_chunk_bytes() / (sizeof(double) * ld));
  const int64_t ct_chunk = std::min<int64_t>(ctiles, ps_ceil_div(chunk_rows, T));
  const int64_t want = 2 * (int64_t)ds->num_sms;
  const int64_t k = std::max(ps_ceil_div(want, rtiles * ctiles), ps_ceil_div(want, rtiles * ct_chunk));
  return std::max<int64_t>(1, std::min<int64_t>(k, W / 16));
}

int ps_group_moment_run(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int student,
                        double* stat, double* p, double* eff, cudaStream_t s) {
  const int64_t Fc = lab->F, Fq = val->F, S = val->S;
  if (lab->S != S) return ps_fail(PS_ERR_INVALID, "sample counts differ");
  lo = std::max<int64_t>(0, lo);
  hi = std::min<int64_t>(Fc * Fq, hi);
  if (hi <= lo || (!stat && !p && !eff)) return PS_OK;
  ps_device_state* ds = ps_state();
  const int64_t W = val->W;
  const int64_t g0 = lo / Fq, g1 = (hi - 1) / Fq + 1;
  // label rows of g0..g1-1
  std::vector<int32_t> off(Fc + 1, 0);
  std::vector<int32_t> rf, rl;
  for (int64_t g = 0; g < Fc; ++g) {
    const int k = test == PS_TEST_ANOVA ? (int)lab->h_cat[g] : 2;
    off[g + 1] = off[g] + k;
  }
  for (int64_t g = 0; g < Fc; ++g) {
    const int k = off[g + 1] - off[g];
    for (int j = 0; j < k; ++j) {
      rf.push_back((int32_t)g);
      rl.push_back(test == PS_TEST_ANOVA ? j : -1 - j);
    }
  }
  const int64_t R = off[Fc];
  const int64_t Rp = std::max<int64_t>(T, ps_round_up(R, T));
  const int64_t rtile0 = off[g0] / T;
  const int64_t rtile1 = off[g1] > 0 ? (off[g1] - 1) / T + 1 : rtile0;
  const int64_t ctiles = ps_ceil_div(Fq, T);

  uint32_t* bits = nullptr;
  int32_t *d_rf = nullptr, *d_rl = nullptr, *d_off = nullptr, *Mn = nullptr, *repc = nullptr;
  double *Ms = nullptr, *Mq = nullptr;
  int2* rep = nullptr;
  const int cap = replay_cap(hi - lo);
  PS_CUDA(ps_alloc(&bits, (size_t)(Rp * W), s));
  PS_CUDA(ps_alloc(&d_rf, (size_t)std::max<int64_t>(R, 1), s));
  PS_CUDA(ps_alloc(&d_rl, (size_t)std::max<int64_t>(R, 1), s));
  PS_CUDA(ps_alloc(&d_off, (size_t)(Fc + 1), s));
  PS_CUDA(ps_alloc(&Mn, (size_t)(Rp * Fq), s));
  PS_CUDA(ps_alloc(&Ms, (size_t)(Rp * Fq), s));
  PS_CUDA(ps_alloc(&Mq, (size_t)(Rp * Fq), s));
  PS_CUDA(ps_alloc(&rep, (size_t)cap, s));
  PS_CUDA(ps_alloc(&repc, 1, s));
  PS_CUDA(cudaMemsetAsync(repc, 0, sizeof(int), s));
  if (R > 0) {
    PS_CUDA(cudaMemcpyAsync(d_rf, rf.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaMemcpyAsync(d_rl, rl.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
  }
  PS_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * (Fc + 1), cudaMemcpyHostToDevice, s));
  if (test == PS_TEST_ANOVA) {
    const int64_t h0 = g1 - g0 > 1 ? 0 : lo - g0 * Fq;
    const int64_t h1 = g1 - g0 > 1 ? Fq : hi - g0 * Fq;
    const dim3 grid((unsigned)ps_ceil_div(W, 128), (unsigned)ps_ceil_div(g1 - g0, 32));
    mixed_label_check_kernel<<<grid, 128, 0, s>>>(lab->d_bad, val->d_mask, W, g0, g1, h0, h1, ds->d_err);
    PS_LAUNCHED();
  }
  launch_onehot_bits(lab, W, d_rf, d_rl, R, Rp, bits, s);
  PS_LAUNCHED();
  const size_t smem = NSTAGE * sizeof(Stage);
  PS_CUDA(cudaFuncSetAttribute(group_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PS_CUDA(cudaFuncSetAttribute(group_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = (rtile1 - rtile0) * ctiles;
  // pre-centred operands (PS_GROUP_RAW=1: centre inside the DMMA loop, A/B)
  double* xc = nullptr;
  const bool pc = !getenv("PS_GROUP_RAW");
  if (pc && grid > 0) {
    PS_CUDA(ps_alloc(&xc, (size_t)(Fq * val->ld), s));
    int crc = ps_center_rows(val, xc, 0, Fq, s);
    if (crc) return crc;
  }
  int32_t* Pn = nullptr;
  double *Ps = nullptr, *Pq = nullptr;
  if (grid > 0) {
    // split K when the WHOLE tile grid cannot fill two CTAs per SM (the split
    // is a function of the matrices, not of the range: every cell's k-order,
    // hence every bit, is the same for any range / rank / incremental launch)
    const int64_t kparts = group_kparts(ds, R, Fq, W, ps_round_up(val->S, 32));
    const int64_t stride = Rp * Fq;
    if (kparts > 1) {
      PS_CUDA(ps_alloc(&Pn, (size_t)(kparts * stride), s));
      PS_CUDA(ps_alloc(&Ps, (size_t)(kparts * stride), s));
      PS_CUDA(ps_alloc(&Pq, (size_t)(kparts * stride), s));
    }
    ps_prof_begin("group_gemm", s);
    if (pc)
      group_gemm_kernel<true><<<dim3((unsigned)grid, (unsigned)kparts), NTH, smem, s>>>(
          bits, Rp, xc, val->ld, val->d_mask, val->d_center, W, Fq, rtile0, 0, ctiles, kparts > 1 ? Pn : Mn,
          kparts > 1 ? Ps : Ms, kparts > 1 ? Pq : Mq, kparts, stride, Fq, 0);
    else
      group_gemm_kernel<false><<<dim3((unsigned)grid, (unsigned)kparts), NTH, smem, s>>>(
          bits, Rp, val->d_vals, val->ld, val->d_mask, val->d_center, W, Fq, rtile0, 0, ctiles, kparts > 1 ? Pn : Mn,
          kparts > 1 ? Ps : Ms, kparts > 1 ? Pq : Mq, kparts, stride, Fq, 0);
    ps_prof_end(s);
    PS_LAUNCHED();
    ps_free(xc, s);
    if (kparts > 1) {
      const int64_t r0 = rtile0 * T, r1 = rtile1 * T;
      const int blocks = (int)std::min<int64_t>(ps_ceil_div((r1 - r0) * Fq, 256), (int64_t)ds->num_sms * 8);
      group_parts_reduce_kernel<<<blocks, 256, 0, s>>>(Pn, Ps, Pq, kparts, stride, r0, r1, Fq, Mn, Ms, Mq);
      PS_LAUNCHED();
      ps_free(Pn, s);
      ps_free(Ps, s);
      ps_free(Pq, s);
    }
  }
  int frc = group_finish_replay(test, lab, val, lo, hi, student, Mn, Ms, Mq, d_off, bits, rep, repc, cap, stat, p, eff,
                                s);
  if (frc) return frc;
  ps_free(bits, s);
  ps_free(d_rf, s);
  ps_free(d_rl, s);
  ps_free(d_off, s);
  ps_free(Mn, s);
  ps_free(Ms, s);
  ps_free(Mq, s);
  ps_free(rep, s);
  ps_free(repc, s);
  return PS_OK;
}

// ---------------------------------------------------------------------------
// Incremental ANOVA / t-test (ps_run overlaps the moment contraction with the
// upload of the continuous matrix): every staged chunk of features whose
// column tiles are complete is contracted on a walk stream; the statistics,
// the label-range check and the replay run once all moments exist.
struct ps_group_job {
  int test = 0, student = 1;
  ps_matrix* lab = nullptr;
  ps_matrix* val = nullptr;
  int64_t R = 0, Rp = 0, h_done = 0;
  double* xc = nullptr;  // pre-centred x' (rows [0, c_done) ready)
  int64_t c_done = 0;
  uint32_t* bits = nullptr;
  int32_t *d_rf = nullptr, *d_rl = nullptr, *d_off = nullptr, *Mn = nullptr, *repc = nullptr;
  double *Ms = nullptr, *Mq = nullptr;
  int2* rep = nullptr;
  int cap = 0, nws = 0;
  cudaStream_t home = nullptr;
  // split-K partials of the incremental launches, one set per walk stream
  int32_t* pn[ps_device_state::kWalkStreams] = {};
  double* psum[ps_device_state::kWalkStreams] = {};
  double* pq[ps_device_state::kWalkStreams] = {};
  int64_t pcap = 0;  // elements per partial array
};

static void group_job_free(ps_group_job* j, cudaStream_t s) {
  ps_free(j->xc, s);
  ps_free(j->bits, s);
  ps_free(j->d_rf, s);
  ps_free(j->d_rl, s);
  ps_free(j->d_off, s);
  ps_free(j->Mn, s);
  ps_free(j->Ms, s);
  ps_free(j->Mq, s);
  ps_free(j->rep, s);
  ps_free(j->repc, s);
  for (int k = 0; k < ps_device_state::kWalkStreams; ++k) {
    ps_free(j->pn[k], s);
    ps_free(j->psum[k], s);
    ps_free(j->pq[k], s);
  }
  delete j;
}

// moments of all level rows x the column tiles [ct0, ct1); split K (fixed
// order) when the tile grid cannot fill two CTAs per SM, with partials laid
// out over the column window only
// `slot` >= 0: an incremental launch using the job's partial buffers of that
// walk-stream slot (allocated once, on the job's home stream); -1: a one-off
// launch on `s` with its own partial buffers.
static int group_gemm_cols(ps_group_job* j, int64_t ct0, int64_t ct1, cudaStream_t s, int slot = -1) {
  if (ct1 <= ct0 || j->R == 0) return PS_OK;
  ps_device_state* ds = ps_state();
  ps_matrix* val = j->val;
  const int64_t Fq = val->F, W = val->W, rtiles = ps_ceil_div(j->R, T), ctiles = ct1 - ct0;
  const size_t smem = NSTAGE * sizeof(Stage);
  PS_CUDA(cudaFuncSetAttribute(group_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PS_CUDA(cudaFuncSetAttribute(group_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = rtiles * ctiles;
  const int64_t kparts = group_kparts(ds, j->R, Fq, W, ps_round_up(val->S, 32));
  const int64_t rows = rtiles * T, width = ctiles * T, c0 = ct0 * T, stride = rows * width;
  // the slot's partial buffers hold a staging chunk's columns; a wider window
  // gets its own (same split, so the same bits)
  if (slot >= 0 && kparts * stride > j->pcap) slot = -1;
  int32_t* Pn = nullptr;
  double *Ps = nullptr, *Pq = nullptr;
  if (kparts > 1 && slot >= 0) {
    Pn = j->pn[slot];
    Ps = j->psum[slot];
    Pq = j->pq[slot];
  } else if (kparts > 1) {
    PS_CUDA(ps_alloc(&Pn, (size_t)(kparts * stride), s));
    PS_CUDA(ps_alloc(&Ps, (size_t)(kparts * stride), s));
    PS_CUDA(ps_alloc(&Pq, (size_t)(kparts * stride), s));
  }
  ps_prof_begin("group_gemm", s);
  auto kern = j->xc ? group_gemm_kernel<true> : group_gemm_kernel<false>;
  kern<<<dim3((unsigned)grid, (unsigned)kparts), NTH, smem, s>>>(
      j->bits, j->Rp, j->xc ? j->xc : val->d_vals, val->ld, val->d_mask, val->d_center, W, Fq, 0, ct0, ctiles,
      kparts > 1 ? Pn : j->Mn, kparts > 1 ? Ps : j->Ms, kparts > 1 ? Pq : j->Mq, kparts, stride,
      kparts > 1 ? width : Fq, kparts > 1 ? c0 : 0);
  ps_prof_end(s);
  PS_LAUNCHED();
  if (kparts > 1) {
    const int blocks = (int)std::min<int64_t>(ps_ceil_div(stride, 256), (int64_t)ds->num_sms * 8);
    group_parts_reduce_cols_kernel<<<blocks, 256, 0, s>>>(Pn, Ps, Pq, kparts, stride, rows, width, c0, Fq, j->Mn,
                                                          j->Ms, j->Mq);
    PS_LAUNCHED();
    if (slot < 0) {
      ps_free(Pn, s);
      ps_free(Ps, s);
      ps_free(Pq, s);
    }
  }
  return PS_OK;
}

int ps_group_moment_begin(int test, ps_matrix* lab, ps_matrix* val, int student, cudaStream_t s, ps_group_job** out) {
  *out = nullptr;
  const int64_t Fc = lab->F, Fq = val->F;
  if (lab->S != val->S) return ps_fail(PS_ERR_INVALID, "sample counts differ");
  ps_group_job* j = new ps_group_job();
  j->test = test;
  j->student = student;
  j->lab = lab;
  j->val = val;
  j->home = s;
  std::vector<int32_t> off(Fc + 1, 0), rf, rl;
  for (int64_t g = 0; g < Fc; ++g) off[g + 1] = off[g] + (test == PS_TEST_ANOVA ? (int)lab->h_cat[g] : 2);
  for (int64_t g = 0; g < Fc; ++g)
    for (int q = 0; q < off[g + 1] - off[g]; ++q) {
      rf.push_back((int32_t)g);
      rl.push_back(test == PS_TEST_ANOVA ? q : -1 - q);
    }
  j->R = off[Fc];
  j->Rp = std::max<int64_t>(T, ps_round_up(j->R, T));
  j->cap = replay_cap(Fc * Fq);
  const int64_t W = val->W;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { e = x; return x == cudaSuccess; };
  if (ok(ps_alloc(&j->bits, (size_t)(j->Rp * W), s)) && ok(ps_alloc(&j->d_rf, (size_t)std::max<int64_t>(j->R, 1), s)) &&
      ok(ps_alloc(&j->d_rl, (size_t)std::max<int64_t>(j->R, 1), s)) && ok(ps_alloc(&j->d_off, (size_t)(Fc + 1), s)) &&
      ok(ps_alloc(&j->Mn, (size_t)(j->Rp * Fq), s)) && ok(ps_alloc(&j->Ms, (size_t)(j->Rp * Fq), s)) &&
      ok(ps_alloc(&j->Mq, (size_t)(j->Rp * Fq), s)) && ok(ps_alloc(&j->rep, (size_t)j->cap, s)) &&
      ok(ps_alloc(&j->repc, 1, s)) && ok(cudaMemsetAsync(j->repc, 0, sizeof(int), s)) &&
      (j->R == 0 || (ok(cudaMemcpyAsync(j->d_rf, rf.data(), sizeof(int32_t) * j->R, cudaMemcpyHostToDevice, s)) &&
                     ok(cudaMemcpyAsync(j->d_rl, rl.data(), sizeof(int32_t) * j->R, cudaMemcpyHostToDevice, s)))) &&
      ok(cudaMemcpyAsync(j->d_off, off.data(), sizeof(int32_t) * (Fc + 1), cudaMemcpyHostToDevice, s))) {
    launch_onehot_bits(lab, W, j->d_rf, j->d_rl, j->R, j->Rp, j->bits, s);
    ps_count_launch();
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    cudaStreamSynchronize(s);
    group_job_free(j, s);
    return ps_cuda_check(e, "group test setup");
  }
  {
    // partial capacity per walk-stream slot: a staging chunk's columns (+ one
    // tile), split as far as a one-tile-column grid would be
    ps_device_state* ds = ps_state();
    const int64_t rtiles = ps_ceil_div(std::max<int64_t>(j->R, 1), T);
    const int64_t chunk_rows = (int64_t)std::max<size_t>(1, ps_stage_chunk_bytes() / (sizeof(double) * val->ld));
    const int64_t width_cap = (ps_ceil_div(chunk_rows, T) + 1) * T;
    const int64_t kp = group_kparts(ds, j->R, Fq, W, ps_round_up(val->S, 32));
    j->pcap = kp > 1 ? kp * rtiles * T * width_cap : 0;
  }
  if (!getenv("PS_GROUP_RAW") && j->R > 0) {
    e = ps_alloc(&j->xc, (size_t)(Fq * val->ld), s);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(s);
      group_job_free(j, s);
      return ps_cuda_check(e, "group test setup");
    }
  }
  // the pageable copies above are staged by the driver: the vectors may go
  *out = j;
  return PS_OK;
}

int ps_group_moment_upto(ps_group_job* j, int64_t h1, cudaStream_t s) {
  const int64_t Fq = j->val->F;
  h1 = h1 >= Fq ? Fq : h1 / T * T;  // whole column tiles only (a partial tile waits for its rows)
  if (h1 <= j->h_done) return PS_OK;
  const int slot = j->nws % ps_device_state::kWalkStreams;
  if (!j->pn[slot] && j->pcap > 0) {
    // first use of this slot: allocate on the home stream, order aux after it
    ps_device_state* ds = ps_state();
    PS_CUDA(ps_alloc(&j->pn[slot], (size_t)j->pcap, j->home));
    PS_CUDA(ps_alloc(&j->psum[slot], (size_t)j->pcap, j->home));
    PS_CUDA(ps_alloc(&j->pq[slot], (size_t)j->pcap, j->home));
    PS_CUDA(cudaEventRecord(ds->alloc_ev, j->home));
    PS_CUDA(cudaStreamWaitEvent(s, ds->alloc_ev, 0));
  }
  if (j->xc && h1 > j->c_done) {  // centre the new rows on s: every later launch is ordered after it
    int crc = ps_center_rows(j->val, j->xc, j->c_done, h1, s);
    if (crc) return crc;
    j->c_done = h1;
  }
  cudaStream_t w = ps_walk_stream(j->nws++, s);
  int rc = group_gemm_cols(j, j->h_done / T, ps_ceil_div(h1, T), w, j->pn[slot] ? slot : -1);
  j->h_done = h1;
  return rc;
}

int ps_group_moment_end(ps_group_job* j, double* stat, double* p, double* eff, cudaStream_t s) {
  ps_device_state* ds = ps_state();
  int rc = ps_walk_streams_join(j->nws, s);
  ps_matrix *lab = j->lab, *val = j->val;
  const int64_t Fc = lab->F, Fq = val->F;
  if (!rc && j->xc && Fq > j->c_done) {
    rc = ps_center_rows(val, j->xc, j->c_done, Fq, s);
    j->c_done = Fq;
  }
  if (!rc) rc = group_gemm_cols(j, j->h_done / T, ps_ceil_div(Fq, T), s);
  j->h_done = Fq;
  if (!rc && j->test == PS_TEST_ANOVA) {
    const dim3 grid((unsigned)ps_ceil_div(val->W, 128), (unsigned)ps_ceil_div(Fc, 32));
    mixed_label_check_kernel<<<grid, 128, 0, s>>>(lab->d_bad, val->d_mask, val->W, 0, Fc, 0, Fq, ds->d_err);
    ps_count_launch();
  }
  if (!rc && (stat || p || eff))
    rc = group_finish_replay(j->test, lab, val, 0, Fc * Fq, j->student, j->Mn, j->Ms, j->Mq, j->d_off, j->bits, j->rep,
                             j->repc, j->cap, stat, p, eff, s);
  if (j->home != s) {
    cudaEventRecord(ds->walk_ev[ps_device_state::kWalkStreams], s);
    cudaStreamWaitEvent(j->home, ds->walk_ev[ps_device_state::kWalkStreams], 0);
  }
  group_job_free(j, j->home);
  return rc;
}

void ps_group_moment_abort(ps_group_job* j, cudaStream_t s) {
  if (!j) return;
  cudaStreamSynchronize(s);
  cudaDeviceSynchronize();
  group_job_free(j, j->home);
}
