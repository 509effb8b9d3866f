// ps_specfun.cuh -- device fp64 special functions behind every p-value.
//
// Restates the reference's numba kernels (pkg/src/pairstat/specfun.py) on the
// device: Lanczos lnGamma (:19-70), the modified-Lentz incomplete-beta
// continued fraction (:73-108), reg_inc_beta with its symmetry switch
// (:111-148), the incomplete-gamma series / CF (:151-208) and the tails
// (:211-314).  Same 300-iteration cap and 1e-15 / 1e-300 constants, so the
// NonConvergence / DomainError behaviour matches; failures set the kernel's
// error word instead of throwing.  The library is compiled with -fmad=false so
// the operation order is the reference's; results differ from the CPU only
// through CUDA-vs-glibc log/exp/log1p/erfc ulps (tests/ pin 1e-12 relative
// against the golden grids).
#pragma once
#include "ps_common.cuh"
#include <math_constants.h>

namespace psf {

__device__ __forceinline__ double lanczos_lg(double x) {
  const double c0 = 0.99999999999980993, c1 = 676.5203681218851, c2 = -1259.1392167224028,
               c3 = 771.32342877765313, c4 = -176.61502916214059, c5 = 12.507343278686905,
               c6 = -0.13857109526572012, c7 = 9.9843695780195716e-6, c8 = 1.5056327351493116e-7;
  const double z = x - 1.0;
  double acc = c0;
  acc += c1 / (z + 1.0);
  acc += c2 / (z + 2.0);
  acc += c3 / (z + 3.0);
  acc += c4 / (z + 4.0);
  acc += c5 / (z + 5.0);
  acc += c6 / (z + 6.0);
  acc += c7 / (z + 7.0);
  acc += c8 / (z + 8.0);
  const double t = z + 7.0 + 0.5;
  const double half_log_two_pi = 0.9189385332046727;  // fl(0.5*log(fl(2*pi))), as the reference computes it
  return half_log_two_pi + (z + 0.5) * log(t) - t + log(acc);
}

__device__ __forceinline__ double ln_gamma(double x, int* err) {
  if (x <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x < 0.5) return log(CUDART_PI / sin(CUDART_PI * x)) - lanczos_lg(1.0 - x);
  return lanczos_lg(x);
}

static __device__ __noinline__ double beta_cf(double a, double b, double x, int* err) {
  const double tiny = 1e-300, eps = 1e-15;
  const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double c = 1.0;
  double d = 1.0 - qab * x / qap;
  if (fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 300; ++m) {
    const double fm = (double)m, m2 = (double)(2 * m);
    double aa = fm * (b - fm) * x / ((qam + m2) * (a + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    h *= d * c;
    aa = -(a + fm) * (qab + fm) * x / ((a + m2) * (qap + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double delta = d * c;
    h *= delta;
    if (fabs(delta - 1.0) < eps) return h;
  }
  ps_raise(err, PS_ERR_NONCONVERGENCE);
  return PS_NAN;
}

// The same continued fraction without divisions (Pearson p over ~2e8 pairs:
// the Lentz form spends three fp64 divisions per term).  Convergents A_k / B_k
// of 1 / (1 + d_1 / (1 + d_2 / ...)) by the forward recurrence, after the
// equivalence transformation that clears each term's denominator
// (d_k = num / den: A_k = den A_(k-1) + num A_(k-2), the pair (A_(k-1), B_(k-1))
// scaled by den as well, so every ratio is kept) and exact power-of-two
// rescaling once per iteration.  Same stopping rule as beta_cf --
// |f_k / f_(k-1) - 1| < 1e-15 after each odd term, written without the
// division.  Differs from the Lentz evaluation only by rounding (a few ulps per
// term; the stopping iteration can move by a few); a fraction not converged
// within kNodivIters (n beyond ~1.5e5 joint samples for Pearson) is evaluated
// by beta_cf itself, so the 300-iteration NonConvergence decision stays the
// reference's.
constexpr int kNodivIters = 240;
static __device__ __noinline__ double beta_cf_nodiv(double a, double b, double x, int* err) {
  const double eps = 1e-15;
  const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double A1 = 1.0, A0 = 0.0, B1 = 1.0, B0 = 1.0;  // (A_k, A_(k-1)), (B_k, B_(k-1))
  auto step = [&](double num, double den) {
    const double a1 = fma(num, A0, den * A1), b1 = fma(num, B0, den * B1);
    A0 = den * A1;
    B0 = den * B1;
    A1 = a1;
    B1 = b1;
  };
  step(-qab * x, qap);
#pragma unroll 1
  for (int m = 1; m <= kNodivIters; ++m) {
    const double fm = (double)m, m2 = (double)(2 * m);
    step(fm * (b - fm) * x, (qam + m2) * (a + m2));
    step(-(a + fm) * (qab + fm) * x, (a + m2) * (qap + m2));
    if (fabs(fma(A1, B0, -(A0 * B1))) < eps * fabs(A0 * B1)) return A1 / B1;
    // exact rescale by 2^-e (e: B_k's binary exponent) keeps the terms in range
    const int e = max(-1000, min(1000, ((__double2hiint(B1) >> 20) & 0x7FF) - 1023));
    const double sc = __hiloint2double((1023 - e) << 20, 0);
    A1 *= sc;
    A0 *= sc;
    B1 *= sc;
    B0 *= sc;
  }
  // near the cap the rounding of the stopping test could decide NonConvergence
  // differently from the reference: the Lentz form decides it
  return beta_cf(a, b, x, err);
}

__device__ __forceinline__ double reg_inc_beta(double x, double a, double b, int* err) {
  if (a <= 0.0 || b <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x < 0.0 || x > 1.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x == 0.0) return 0.0;
  if (x == 1.0) return 1.0;
  const double ln_front =
      ln_gamma(a + b, err) - ln_gamma(a, err) - ln_gamma(b, err) + a * log(x) + b * log1p(-x);
  const double front = exp(ln_front);
  if (x < (a + 1.0) / (a + b + 2.0)) return front * beta_cf(a, b, x, err) / a;
  return 1.0 - front * beta_cf(b, a, 1.0 - x, err) / b;
}

__device__ __forceinline__ double reg_inc_beta_nodiv(double x, double a, double b, int* err) {
  if (a <= 0.0 || b <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x < 0.0 || x > 1.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x == 0.0) return 0.0;
  if (x == 1.0) return 1.0;
  const double ln_front =
      ln_gamma(a + b, err) - ln_gamma(a, err) - ln_gamma(b, err) + a * log(x) + b * log1p(-x);
  const double front = exp(ln_front);
  if (x < (a + 1.0) / (a + b + 2.0)) return front * beta_cf_nodiv(a, b, x, err) / a;
  return 1.0 - front * beta_cf_nodiv(b, a, 1.0 - x, err) / b;
}

static __device__ __noinline__ double reg_inc_gamma_upper(double a, double x, int* err) {
  const double tiny = 1e-300, eps = 1e-15;
  if (a <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x < 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (x == 0.0) return 1.0;
  const double ln_front = -x + a * log(x) - ln_gamma(a, err);
  if (x < a + 1.0) {
    double term = 1.0 / a, total = term, ap = a;
    for (int i = 0; i < 300; ++i) {
      ap += 1.0;
      term *= x / ap;
      total += term;
      if (fabs(term) < fabs(total) * eps) return 1.0 - total * exp(ln_front);
    }
    ps_raise(err, PS_ERR_NONCONVERGENCE);
    return PS_NAN;
  }
  double b = x + 1.0 - a;
  double c = 1.0 / tiny;
  double d = 1.0 / b;
  double h = d;
  for (int i = 1; i <= 300; ++i) {
    const double an = -(double)i * ((double)i - a);
    b += 2.0;
    d = an * d + b;
    if (fabs(d) < tiny) d = tiny;
    c = b + an / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double delta = d * c;
    h *= delta;
    if (fabs(delta - 1.0) < eps) return h * exp(ln_front);
  }
  ps_raise(err, PS_ERR_NONCONVERGENCE);
  return PS_NAN;
}

__device__ __forceinline__ double normal_sf(double z) { return 0.5 * erfc(z / sqrt(2.0)); }

__device__ __forceinline__ double t_sf(double t, double dof, int* err) {
  if (dof <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  const double x = dof / (dof + t * t);
  const double tail = 0.5 * reg_inc_beta(x, 0.5 * dof, 0.5, err);
  return t >= 0.0 ? tail : 1.0 - tail;
}

__device__ __forceinline__ double chi2_sf(double x, double dof, int* err) {
  if (dof <= 0.0 || x < 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  return reg_inc_gamma_upper(0.5 * dof, 0.5 * x, err);
}

__device__ __forceinline__ double f_sf(double f, double d1, double d2, int* err) {
  if (d1 <= 0.0 || d2 <= 0.0 || f < 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (isinf(f)) return 0.0;
  return reg_inc_beta(d2 / (d2 + d1 * f), 0.5 * d2, 0.5 * d1, err);
}

__device__ __forceinline__ double beta_sym_sf(double r_abs, double a, int* err) {
  if (a <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (r_abs < 0.0 || r_abs > 1.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  return reg_inc_beta(0.5 * (1.0 - r_abs), a, a, err);
}

// beta_sym_sf through the division-free continued fraction (Pearson p)
__device__ __forceinline__ double beta_sym_sf_nodiv(double r_abs, double a, int* err) {
  if (a <= 0.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  if (r_abs < 0.0 || r_abs > 1.0) { ps_raise(err, PS_ERR_DOMAIN); return PS_NAN; }
  return reg_inc_beta_nodiv(0.5 * (1.0 - r_abs), a, a, err);
}

}  // namespace psf
