/*
 * oracle.c -- CPU restatement of the reference pair engine (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker and the CPU baseline ("port") for the B200
 * engine.  It is NOT part of the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Every function restates one reference function of /root/reference/pkg/src/
 * pairstat (a numba package, so there is no C source to compile; see
 * DESIGN.md "Oracle").  The floating-point operation order of the reference
 * is replayed exactly (compiled with -ffp-contract=off, no fast-math), so on
 * glibc this port reproduces the reference bit for bit; the golden fixtures
 * under tests/golden/ pin it (tests/test_oracle_golden.py).
 *
 * Parallelism: OpenMP over triangle rows / grid cells.  Every output cell is
 * written by exactly one iteration, so results do not depend on the thread
 * count (reference engine.py:10-18).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_LABEL 3
#define ORC_ERR_TIES 4
#define ORC_ERR_TABLE 5
#define ORC_ERR_NONCONV 6
#define ORC_ERR_DOMAIN 7

/* First error raised by any worker (reference: future.result(), engine.py:373-376). */
static int g_err = 0;
static void set_err(int code) {
#pragma omp critical(orc_err)
    {
        if (g_err == 0) g_err = code;
    }
}
static int take_err(void) {
    int e = g_err;
    g_err = 0;
    return e;
}

/* ------------------------------------------------------------------ */
/* Special functions: specfun.py                                       */
/* ------------------------------------------------------------------ */

static const double kLanczos[9] = {
    0.99999999999980993,  676.5203681218851,     -1259.1392167224028,
    771.32342877765313,   -176.61502916214059,   12.507343278686905,
    -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};
#define MAX_ITER 300
#define CONV_EPS 1e-15
#define TINY 1e-300

/* specfun.py:41-49 */
static double lanczos_lg(double x) {
    double z = x - 1.0;
    double acc = kLanczos[0];
    for (int i = 1; i < 9; ++i) acc += kLanczos[i] / (z + (double)i);
    double t = z + 7.0 + 0.5;
    double half_log_two_pi = 0.5 * log(2.0 * M_PI);
    return half_log_two_pi + (z + 0.5) * log(t) - t + log(acc);
}

/* specfun.py:52-70 */
double orc_ln_gamma(double x, int* err) {
    if (x <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x < 0.5) return log(M_PI / sin(M_PI * x)) - lanczos_lg(1.0 - x);
    return lanczos_lg(x);
}

/* specfun.py:73-108 (modified Lentz) */
static double beta_cf(double a, double b, double x, int* err) {
    double qab = a + b, qap = a + 1.0, qam = a - 1.0;
    double c = 1.0;
    double d = 1.0 - qab * x / qap;
    if (fabs(d) < TINY) d = TINY;
    d = 1.0 / d;
    double h = d;
    for (int m = 1; m <= MAX_ITER; ++m) {
        double fm = (double)m;
        double m2 = (double)(2 * m);
        double aa = fm * (b - fm) * x / ((qam + m2) * (a + m2));
        d = 1.0 + aa * d;
        if (fabs(d) < TINY) d = TINY;
        c = 1.0 + aa / c;
        if (fabs(c) < TINY) c = TINY;
        d = 1.0 / d;
        h *= d * c;
        aa = -(a + fm) * (qab + fm) * x / ((a + m2) * (qap + m2));
        d = 1.0 + aa * d;
        if (fabs(d) < TINY) d = TINY;
        c = 1.0 + aa / c;
        if (fabs(c) < TINY) c = TINY;
        d = 1.0 / d;
        double delta = d * c;
        h *= delta;
        if (fabs(delta - 1.0) < CONV_EPS) return h;
    }
    *err = ORC_ERR_NONCONV;
    return NAN;
}

/* specfun.py:111-148 */
double orc_reg_inc_beta(double x, double a, double b, int* err) {
    if (a <= 0.0 || b <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x < 0.0 || x > 1.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x == 0.0) return 0.0;
    if (x == 1.0) return 1.0;
    int e = 0;
    double ln_front = orc_ln_gamma(a + b, &e) - orc_ln_gamma(a, &e) - orc_ln_gamma(b, &e) +
                      a * log(x) + b * log1p(-x);
    if (e) { *err = e; return NAN; }
    double front = exp(ln_front);
    if (x < (a + 1.0) / (a + b + 2.0)) {
        double cf = beta_cf(a, b, x, err);
        return front * cf / a;
    }
    double cf = beta_cf(b, a, 1.0 - x, err);
    return 1.0 - front * cf / b;
}

/* specfun.py:151-208 */
double orc_reg_inc_gamma_upper(double a, double x, int* err) {
    if (a <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x < 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x == 0.0) return 1.0;
    int e = 0;
    double ln_front = -x + a * log(x) - orc_ln_gamma(a, &e);
    if (e) { *err = e; return NAN; }
    if (x < a + 1.0) {
        double term = 1.0 / a, total = term, ap = a;
        for (int i = 0; i < MAX_ITER; ++i) {
            ap += 1.0;
            term *= x / ap;
            total += term;
            if (fabs(term) < fabs(total) * CONV_EPS) return 1.0 - total * exp(ln_front);
        }
        *err = ORC_ERR_NONCONV;
        return NAN;
    }
    double b = x + 1.0 - a;
    double c = 1.0 / TINY;
    double d = 1.0 / b;
    double h = d;
    for (int i = 1; i <= MAX_ITER; ++i) {
        double an = -(double)i * ((double)i - a);
        b += 2.0;
        d = an * d + b;
        if (fabs(d) < TINY) d = TINY;
        c = b + an / c;
        if (fabs(c) < TINY) c = TINY;
        d = 1.0 / d;
        double delta = d * c;
        h *= delta;
        if (fabs(delta - 1.0) < CONV_EPS) return h * exp(ln_front);
    }
    *err = ORC_ERR_NONCONV;
    return NAN;
}

/* specfun.py:211-221 */
double orc_normal_sf(double z) { return 0.5 * erfc(z / sqrt(2.0)); }

/* specfun.py:224-244 */
double orc_t_sf(double t, double dof, int* err) {
    if (dof <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    double x = dof / (dof + t * t);
    double tail = 0.5 * orc_reg_inc_beta(x, 0.5 * dof, 0.5, err);
    if (t >= 0.0) return tail;
    return 1.0 - tail;
}

/* specfun.py:247-265 */
double orc_chi2_sf(double x, double dof, int* err) {
    if (dof <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (x < 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    return orc_reg_inc_gamma_upper(0.5 * dof, 0.5 * x, err);
}

/* specfun.py:268-289 */
double orc_f_sf(double f, double d1, double d2, int* err) {
    if (d1 <= 0.0 || d2 <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (f < 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (isinf(f)) return 0.0;
    return orc_reg_inc_beta(d2 / (d2 + d1 * f), 0.5 * d2, 0.5 * d1, err);
}

/* specfun.py:292-314 */
double orc_beta_sym_sf(double r_abs, double a, int* err) {
    if (a <= 0.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    if (r_abs < 0.0 || r_abs > 1.0) { *err = ORC_ERR_DOMAIN; return NAN; }
    return orc_reg_inc_beta(0.5 * (1.0 - r_abs), a, a, err);
}

/* ------------------------------------------------------------------ */
/* Pearson: continuous.py:29-49, :77-103; engine.py:145-166            */
/* ------------------------------------------------------------------ */

static void pearson_finish(int64_t n, double sxx, double syy, double sxy, double* r_out,
                           double* p_out, int* err) {
    if (n <= 1 || sxx <= 0.0 || syy <= 0.0) { *r_out = NAN; *p_out = NAN; return; }
    double r = sxy / sqrt(sxx * syy);
    if (r > 1.0) r = 1.0;
    else if (r < -1.0) r = -1.0;
    if (n == 2) { *r_out = r; *p_out = NAN; return; }
    double p = 2.0 * orc_beta_sym_sf(fabs(r), 0.5 * (double)n - 1.0, err);
    if (p > 1.0) p = 1.0;
    *r_out = r;
    *p_out = p;
}

void orc_pearson_pair(const double* xg, const uint8_t* pg, const double* xh, const uint8_t* ph,
                      int64_t S, double* r, double* p, int* err) {
    int64_t n = 0;
    double sum_x = 0.0, sum_y = 0.0;
    for (int64_t i = 0; i < S; ++i)
        if (pg[i] && ph[i]) { n++; sum_x += xg[i]; sum_y += xh[i]; }
    if (n <= 1) { *r = NAN; *p = NAN; return; }
    double mx = sum_x / (double)n, my = sum_y / (double)n;
    double sxx = 0.0, syy = 0.0, sxy = 0.0;
    for (int64_t i = 0; i < S; ++i)
        if (pg[i] && ph[i]) {
            double dx = xg[i] - mx, dy = xh[i] - my;
            sxx += dx * dx;
            syy += dy * dy;
            sxy += dx * dy;
        }
    pearson_finish(n, sxx, syy, sxy, r, p, err);
}

static inline void put_sym(double* out, int64_t F, int64_t g, int64_t h, double v) {
    if (!out) return;
    out[g * F + h] = v;
    out[h * F + g] = v;
}

int orc_pearson_block(const double* values, const uint8_t* present, int64_t F, int64_t S,
                      int64_t lo, int64_t hi, double* stat, double* p, double* r2,
                      int threads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t g = lo; g < hi; ++g) {
        for (int64_t h = g; h < F; ++h) {
            double r, pv;
            int e = 0;
            orc_pearson_pair(values + g * S, present + g * S, values + h * S, present + h * S, S,
                             &r, &pv, &e);
            if (e) set_err(e);
            put_sym(stat, F, g, h, r);
            put_sym(p, F, g, h, pv);
            put_sym(r2, F, g, h, r * r);
        }
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* Presort: ranking.py:30-53, engine.py:133-142, :379-400              */
/* ------------------------------------------------------------------ */

/* numpy's NaN-aware ordering: NaN sorts after every number. */
static inline int fless(double a, double b) { return a < b || (b != b && a == a); }

static void merge_sort_idx(int64_t* idx, const double* v, int64_t* tmp, int64_t n) {
    /* bottom-up stable merge sort of idx by v[idx] */
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * width) {
            int64_t mid = lo + width < n ? lo + width : n;
            int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            int64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                if (fless(v[idx[j]], v[idx[i]])) tmp[k++] = idx[j++];
                else tmp[k++] = idx[i++];
            }
            while (i < mid) tmp[k++] = idx[i++];
            while (j < hi) tmp[k++] = idx[j++];
        }
        memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
    }
}

int orc_presort(const double* values, const uint8_t* present, int64_t F, int64_t S,
                int64_t* orders, double* svals, int64_t* lengths, int threads) {
#pragma omp parallel num_threads(threads)
    {
        int64_t* idx = (int64_t*)malloc((size_t)S * sizeof(int64_t));
        int64_t* tmp = (int64_t*)malloc((size_t)S * sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
        for (int64_t f = 0; f < F; ++f) {
            const double* row = values + f * S;
            const uint8_t* pr = present + f * S;
            int64_t n = 0;
            for (int64_t i = 0; i < S; ++i)
                if (pr[i]) idx[n++] = i;
            merge_sort_idx(idx, row, tmp, n);
            lengths[f] = n;
            for (int64_t i = 0; i < n; ++i) {
                orders[f * S + i] = idx[i];
                svals[f * S + i] = row[idx[i]];
            }
        }
        free(idx);
        free(tmp);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Spearman: continuous.py:128-203; engine.py:169-205                  */
/* ------------------------------------------------------------------ */

static int64_t scatter_ranks(const int64_t* order, const double* sv, int64_t n_all,
                             const uint8_t* partner, double* out_ranks, int64_t* kept,
                             double* vals) {
    int64_t n = 0;
    for (int64_t i = 0; i < n_all; ++i) {
        int64_t s = order[i];
        kept[n] = s;
        vals[n] = sv[i];
        n += partner[s] ? 1 : 0;
    }
    int64_t i = 0;
    while (i < n) {
        double v = vals[i];
        int64_t j = i + 1;
        while (j < n && vals[j] == v) j++;
        double avg = 0.5 * (double)(i + j + 1);
        for (int64_t k = i; k < j; ++k) out_ranks[kept[k]] = avg;
        i = j;
    }
    return n;
}

void orc_spearman_pair(const int64_t* og, const double* svg, int64_t ng, const uint8_t* pg,
                       const int64_t* oh, const double* svh, int64_t nh, const uint8_t* ph,
                       double* rank_g, double* rank_h, int64_t* kept, double* vals, double* rho_out,
                       double* p_out, int* err) {
    int64_t n = scatter_ranks(og, svg, ng, ph, rank_g, kept, vals);
    scatter_ranks(oh, svh, nh, pg, rank_h, kept, vals);
    if (n <= 1) { *rho_out = NAN; *p_out = NAN; return; }
    double mean = 0.5 * (double)(n + 1);
    double sxx = 0.0, syy = 0.0, sxy = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = kept[i];
        double dx = rank_g[s] - mean, dy = rank_h[s] - mean;
        sxx += dx * dx;
        syy += dy * dy;
        sxy += dx * dy;
    }
    if (sxx <= 0.0 || syy <= 0.0) { *rho_out = NAN; *p_out = NAN; return; }
    double rho = sxy / sqrt(sxx * syy);
    if (rho > 1.0) rho = 1.0;
    else if (rho < -1.0) rho = -1.0;
    *rho_out = rho;
    if (n == 2) { *p_out = NAN; return; }
    if (rho == 1.0 || rho == -1.0) { *p_out = 0.0; return; }
    double t = rho * sqrt(((double)n - 2.0) / (1.0 - rho * rho));
    double p = 2.0 * orc_t_sf(fabs(t), (double)n - 2.0, err);
    if (p > 1.0) p = 1.0;
    *p_out = p;
}

int orc_spearman_block(const int64_t* orders, const double* svals, const int64_t* lengths,
                       const uint8_t* present, int64_t F, int64_t S, int64_t lo, int64_t hi,
                       double* stat, double* p, double* rho, int threads) {
#pragma omp parallel num_threads(threads)
    {
        double* rank_g = (double*)malloc((size_t)S * sizeof(double));
        double* rank_h = (double*)malloc((size_t)S * sizeof(double));
        int64_t* kept = (int64_t*)malloc((size_t)S * sizeof(int64_t));
        double* vals = (double*)malloc((size_t)S * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t g = lo; g < hi; ++g) {
            for (int64_t h = g; h < F; ++h) {
                double r, pv;
                int e = 0;
                orc_spearman_pair(orders + g * S, svals + g * S, lengths[g], present + g * S,
                                  orders + h * S, svals + h * S, lengths[h], present + h * S,
                                  rank_g, rank_h, kept, vals, &r, &pv, &e);
                if (e) set_err(e);
                put_sym(stat, F, g, h, r);
                put_sym(p, F, g, h, pv);
                put_sym(rho, F, g, h, r);
            }
        }
        free(rank_g);
        free(rank_h);
        free(kept);
        free(vals);
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* Chi-squared: categorical.py:31-94; engine.py:208-242                */
/* ------------------------------------------------------------------ */

static void chi2_finish(const int64_t* table, int64_t cg, int64_t ch, int64_t n, int64_t* rs,
                        int64_t* cs, double out[4], int* err) {
    out[0] = out[1] = out[2] = out[3] = NAN;
    if (n == 0) return;
    for (int64_t i = 0; i < cg; ++i) rs[i] = 0;
    for (int64_t j = 0; j < ch; ++j) cs[j] = 0;
    for (int64_t i = 0; i < cg; ++i)
        for (int64_t j = 0; j < ch; ++j) {
            int64_t c = table[i * ch + j];
            rs[i] += c;
            cs[j] += c;
        }
    for (int64_t i = 0; i < cg; ++i)
        if (rs[i] == 0) return;
    for (int64_t j = 0; j < ch; ++j)
        if (cs[j] == 0) return;
    double chi2 = 0.0;
    for (int64_t i = 0; i < cg; ++i)
        for (int64_t j = 0; j < ch; ++j) {
            double expected = (double)(rs[i] * cs[j]) / (double)n;
            if (expected > 0.0) {
                double diff = (double)table[i * ch + j] - expected;
                chi2 += diff * diff / expected;
            }
        }
    double phi = sqrt(chi2 / (double)n);
    int64_t cmin = cg < ch ? cg : ch;
    out[0] = chi2;
    out[2] = phi;
    if (cmin < 2) return;
    double dof = ((double)cg - 1.0) * ((double)ch - 1.0);
    out[1] = orc_chi2_sf(chi2, dof, err);
    out[3] = sqrt(chi2 / ((double)n * ((double)cmin - 1.0)));
}

int orc_chi2_pair(const double* g, const uint8_t* pg, const double* h, const uint8_t* ph,
                  int64_t S, int64_t cg, int64_t ch, int64_t* table, int64_t* rs, int64_t* cs,
                  double out[4], int* err) {
    for (int64_t i = 0; i < cg * ch; ++i) table[i] = 0;
    int64_t n = 0;
    for (int64_t s = 0; s < S; ++s) {
        if (pg[s] && ph[s]) {
            int64_t a = (int64_t)g[s], b = (int64_t)h[s];
            if (a < 0 || a >= cg || b < 0 || b >= ch) { *err = ORC_ERR_LABEL; return ORC_ERR_LABEL; }
            table[a * ch + b] += 1;
            n++;
        }
    }
    chi2_finish(table, cg, ch, n, rs, cs, out, err);
    return 0;
}

int orc_chi2_block(const double* values, const uint8_t* present, const int64_t* cat, int64_t F,
                   int64_t S, int64_t lo, int64_t hi, double* stat, double* p, double* phi,
                   double* v, int threads) {
    int64_t cmax = 0;
    for (int64_t f = 0; f < F; ++f)
        if (cat[f] > cmax) cmax = cat[f];
    if (cmax < 1) cmax = 1;
#pragma omp parallel num_threads(threads)
    {
        int64_t* table = (int64_t*)malloc((size_t)(cmax * cmax) * sizeof(int64_t));
        int64_t* rs = (int64_t*)malloc((size_t)cmax * sizeof(int64_t));
        int64_t* cs = (int64_t*)malloc((size_t)cmax * sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
        for (int64_t g = lo; g < hi; ++g) {
            for (int64_t h = g; h < F; ++h) {
                double out[4];
                int e = 0;
                orc_chi2_pair(values + g * S, present + g * S, values + h * S, present + h * S, S,
                              cat[g], cat[h], table, rs, cs, out, &e);
                if (e) { set_err(e); continue; }
                put_sym(stat, F, g, h, out[0]);
                put_sym(p, F, g, h, out[1]);
                put_sym(phi, F, g, h, out[2]);
                put_sym(v, F, g, h, out[3]);
            }
        }
        free(table);
        free(rs);
        free(cs);
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* t-test: mixed.py:121-202; engine.py:245-263                          */
/* ------------------------------------------------------------------ */

static void ttest_finish(int64_t n0, int64_t n1, double sum0, double sum1, double ss0, double ss1,
                         int student, double out[3], int* err) {
    out[0] = out[1] = out[2] = NAN;
    if (n0 < 2 || n1 < 2 || n0 + n1 < 3) return;
    double mean0 = sum0 / (double)n0, mean1 = sum1 / (double)n1;
    double var0 = (ss0 - sum0 * mean0) / (double)(n0 - 1);
    double var1 = (ss1 - sum1 * mean1) / (double)(n1 - 1);
    if (var0 < 0.0) var0 = 0.0;
    if (var1 < 0.0) var1 = 0.0;
    double diff = mean0 - mean1;
    double t, dof, d;
    if (student) {
        double pooled = ((double)(n0 - 1) * var0 + (double)(n1 - 1) * var1) / (double)(n0 + n1 - 2);
        if (pooled == 0.0) return;
        double sp = sqrt(pooled);
        t = diff / (sp * sqrt(1.0 / (double)n0 + 1.0 / (double)n1));
        dof = (double)(n0 + n1 - 2);
        d = diff / sp;
    } else {
        if (var0 + var1 == 0.0) return;
        double v0 = var0 / (double)n0, v1 = var1 / (double)n1;
        t = diff / sqrt(v0 + v1);
        dof = (v0 + v1) * (v0 + v1) / (v0 * v0 / (double)(n0 - 1) + v1 * v1 / (double)(n1 - 1));
        d = diff / sqrt(0.5 * (var0 + var1));
    }
    double p = 2.0 * orc_t_sf(fabs(t), dof, err);
    if (p > 1.0) p = 1.0;
    out[0] = t;
    out[1] = p;
    out[2] = d;
}

int orc_ttest_block(const double* lab, const uint8_t* labp, const double* val, const uint8_t* valp,
                    int64_t Fc, int64_t Fq, int64_t S, int64_t lo, int64_t hi, int student,
                    double* stat, double* p, double* dout, int threads) {
    (void)Fc;
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (int64_t idx = lo; idx < hi; ++idx) {
        int64_t g = idx / Fq, h = idx - g * Fq;
        const double* lg = lab + g * S;
        const uint8_t* lp = labp + g * S;
        const double* vh = val + h * S;
        const uint8_t* vp = valp + h * S;
        int64_t n0 = 0, n1 = 0;
        double sum0 = 0, sum1 = 0, ss0 = 0, ss1 = 0;
        for (int64_t i = 0; i < S; ++i) {
            if (lp[i] && vp[i]) {
                double v = vh[i];
                if (lg[i] == 0.0) { n0++; sum0 += v; ss0 += v * v; }
                else { n1++; sum1 += v; ss1 += v * v; }
            }
        }
        double out[3];
        int e = 0;
        ttest_finish(n0, n1, sum0, sum1, ss0, ss1, student, out, &e);
        if (e) set_err(e);
        if (stat) stat[g * Fq + h] = out[0];
        if (p) p[g * Fq + h] = out[1];
        if (dout) dout[g * Fq + h] = out[2];
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* ANOVA: mixed.py:453-520; engine.py:266-293                          */
/* ------------------------------------------------------------------ */

static void anova_finish(const int64_t* counts, const double* sums, const double* ssq, int64_t k,
                         double out[3], int* err) {
    out[0] = out[1] = out[2] = NAN;
    if (k < 2) return;
    int64_t n = 0;
    double total = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        if (counts[j] == 0) return;
        n += counts[j];
        total += sums[j];
    }
    if (n <= k) return;
    double grand = total / (double)n;
    double ssb = 0.0, ssw = 0.0, lo = INFINITY, hi = -INFINITY, scale = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double mj = sums[j] / (double)counts[j];
        double dev = mj - grand;
        ssb += (double)counts[j] * dev * dev;
        double gs = ssq[j] - sums[j] * mj;
        if (gs > 0.0) ssw += gs;
        if (mj < lo) lo = mj;
        if (mj > hi) hi = mj;
        if (fabs(mj) > scale) scale = fabs(mj);
    }
    if (ssw == 0.0) {
        if ((hi - lo) <= 1e-12 * scale) return;
        out[0] = INFINITY;
        out[1] = 0.0;
        out[2] = 1.0;
        return;
    }
    double f = (ssb / ((double)k - 1.0)) / (ssw / (double)(n - k));
    out[0] = f;
    out[1] = orc_f_sf(f, (double)k - 1.0, (double)(n - k), err);
    out[2] = ssb / (ssb + ssw);
}

int orc_anova_block(const double* lab, const uint8_t* labp, const int64_t* cat, const double* val,
                    const uint8_t* valp, int64_t Fc, int64_t Fq, int64_t S, int64_t lo, int64_t hi,
                    double* stat, double* p, double* eta, int threads) {
    int64_t kmax = 1;
    for (int64_t f = 0; f < Fc; ++f)
        if (cat[f] > kmax) kmax = cat[f];
#pragma omp parallel num_threads(threads)
    {
        int64_t* counts = (int64_t*)malloc((size_t)kmax * sizeof(int64_t));
        double* sums = (double*)malloc((size_t)kmax * sizeof(double));
        double* ssq = (double*)malloc((size_t)kmax * sizeof(double));
#pragma omp for schedule(dynamic, 64)
        for (int64_t idx = lo; idx < hi; ++idx) {
            int64_t g = idx / Fq, h = idx - g * Fq;
            int64_t k = cat[g];
            for (int64_t j = 0; j < k; ++j) { counts[j] = 0; sums[j] = 0.0; ssq[j] = 0.0; }
            const double* lg = lab + g * S;
            const uint8_t* lp = labp + g * S;
            const double* vh = val + h * S;
            const uint8_t* vp = valp + h * S;
            int bad = 0;
            for (int64_t i = 0; i < S; ++i) {
                if (lp[i] && vp[i]) {
                    int64_t j = (int64_t)lg[i];
                    if (j < 0 || j >= k) { bad = 1; break; }
                    double v = vh[i];
                    counts[j] += 1;
                    sums[j] += v;
                    ssq[j] += v * v;
                }
            }
            if (bad) { set_err(ORC_ERR_LABEL); continue; }
            double out[3];
            int e = 0;
            anova_finish(counts, sums, ssq, k, out, &e);
            if (e) set_err(e);
            if (stat) stat[g * Fq + h] = out[0];
            if (p) p[g * Fq + h] = out[1];
            if (eta) eta[g * Fq + h] = out[2];
        }
        free(counts);
        free(sums);
        free(ssq);
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* Mann-Whitney U: mixed.py:231-247, :305-403; engine.py:296-319        */
/* ------------------------------------------------------------------ */

#define EXACT_U_CAP 64
#define EXACT_U_AUTO_LIMIT 8

/* mixed.py:231-247 -- table is (n1+1) x (n1*n2+1) scratch, returns row n1 */
static void exact_u_counts(int64_t n1, int64_t n2, int64_t* table, int64_t* out_row) {
    int64_t umax = n1 * n2, w = umax + 1;
    memset(table, 0, (size_t)((n1 + 1) * w) * sizeof(int64_t));
    for (int64_t a = 0; a <= n1; ++a) table[a * w] = 1;
    for (int64_t b = 1; b <= n2; ++b)
        for (int64_t a = 1; a <= n1; ++a)
            for (int64_t u = b; u <= umax; ++u) table[a * w + u] += table[(a - 1) * w + u - b];
    memcpy(out_row, table + n1 * w, (size_t)w * sizeof(int64_t));
}

void orc_exact_u_counts(int64_t n1, int64_t n2, int64_t* out_row) {
    int64_t w = n1 * n2 + 1;
    int64_t* table = (int64_t*)malloc((size_t)((n1 + 1) * w) * sizeof(int64_t));
    exact_u_counts(n1, n2, table, out_row);
    free(table);
}

static void mwu_finish(int64_t n0, int64_t n1, double r0, double tie_term, int mode, double out[3],
                       int* err) {
    out[0] = out[1] = out[2] = NAN;
    if (n0 == 0 || n1 == 0) return;
    int64_t n = n0 + n1;
    double u = r0 - 0.5 * (double)n0 * (double)(n0 + 1);
    double mu = 0.5 * (double)n0 * (double)n1;
    double diff = u - mu;
    int use_exact = 0;
    if (mode == 0) {
        if (tie_term != 0.0) { *err = ORC_ERR_TIES; return; }
        if (n > EXACT_U_CAP) { *err = ORC_ERR_TABLE; return; }
        use_exact = 1;
    } else if (mode == 2) {
        int64_t mn = n0 < n1 ? n0 : n1;
        use_exact = tie_term == 0.0 && mn < EXACT_U_AUTO_LIMIT && n <= EXACT_U_CAP;
    }
    double sigma_sq = ((double)(n0 * n1) / 12.0) *
                      (((double)n + 1.0) - tie_term / ((double)n * ((double)n - 1.0)));
    out[0] = u;
    if (sigma_sq <= 0.0) return;
    double z = (fabs(diff) - 0.5) / sqrt(sigma_sq);
    if (z < 0.0) z = 0.0;
    double r;
    if (z == 0.0 || diff == 0.0) r = 0.0;
    else if (diff > 0.0) r = z / sqrt((double)n);
    else r = -z / sqrt((double)n);
    double p;
    if (use_exact) {
        int64_t umax = n0 * n1;
        int64_t* row = (int64_t*)malloc((size_t)(umax + 1) * sizeof(int64_t));
        orc_exact_u_counts(n0, n1, row);
        double m = u < (double)umax - u ? u : (double)umax - u;
        int64_t ulow = (int64_t)nearbyint(m);
        int64_t cum = 0, total = 0;
        for (int64_t i = 0; i <= umax; ++i) {
            total += row[i];
            if (i <= ulow) cum += row[i];
        }
        free(row);
        p = 2.0 * (double)cum / (double)total;
    } else {
        p = 2.0 * orc_normal_sf(z);
    }
    if (p > 1.0) p = 1.0;
    out[1] = p;
    out[2] = r;
}

int orc_mwu_block(const int64_t* orders, const double* svals, const int64_t* lengths,
                  const double* lab, const uint8_t* labp, int64_t Fc, int64_t Fq, int64_t S,
                  int64_t lo, int64_t hi, int mode, double* stat, double* p, double* rout,
                  int threads) {
    (void)Fq;
#pragma omp parallel num_threads(threads)
    {
        double* cv = (double*)malloc((size_t)S * sizeof(double));
        double* cl = (double*)malloc((size_t)S * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t h = lo; h < hi; ++h) {
            const int64_t* order = orders + h * S;
            const double* sv = svals + h * S;
            int64_t nall = lengths[h];
            for (int64_t g = 0; g < Fc; ++g) {
                const double* lg = lab + g * S;
                const uint8_t* lp = labp + g * S;
                int64_t m = 0;
                for (int64_t i = 0; i < nall; ++i) {
                    int64_t s = order[i];
                    cv[m] = sv[i];
                    cl[m] = lg[s];
                    m += lp[s] ? 1 : 0;
                }
                int64_t n0 = 0, n1 = 0;
                double r0 = 0.0, tie = 0.0;
                int64_t i = 0;
                while (i < m) {
                    double v = cv[i];
                    int64_t j = i + 1;
                    while (j < m && cv[j] == v) j++;
                    int64_t run = j - i, c0 = 0;
                    for (int64_t t = i; t < j; ++t) c0 += cl[t] == 0.0 ? 1 : 0;
                    double avg = 0.5 * (double)(i + j + 1);
                    r0 += avg * (double)c0;
                    n0 += c0;
                    n1 += run - c0;
                    if (run > 1) tie += (double)run * (double)run * (double)run - (double)run;
                    i = j;
                }
                double out[3];
                int e = 0;
                mwu_finish(n0, n1, r0, tie, mode, out, &e);
                if (e) { set_err(e); continue; }
                if (stat) stat[g * Fq + h] = out[0];
                if (p) p[g * Fq + h] = out[1];
                if (rout) rout[g * Fq + h] = out[2];
            }
        }
        free(cv);
        free(cl);
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* Kruskal-Wallis: mixed.py:550-623; engine.py:322-352                  */
/* ------------------------------------------------------------------ */

static void kruskal_finish(const double* rank_sums, const int64_t* counts, int64_t k, double tie,
                           double out[3], int* err) {
    out[0] = out[1] = out[2] = NAN;
    int64_t n = 0;
    for (int64_t j = 0; j < k; ++j) {
        if (counts[j] == 0) return;
        n += counts[j];
    }
    if (n < 2) return;
    double fn = (double)n;
    double tden = 1.0 - tie / (fn * fn * fn - fn);
    if (tden <= 0.0) return;
    double h = 0.0;
    for (int64_t j = 0; j < k; ++j) h += rank_sums[j] * rank_sums[j] / (double)counts[j];
    h = (12.0 / (fn * (fn + 1.0))) * h - 3.0 * (fn + 1.0);
    h /= tden;
    if (h < 0.0) h = 0.0;
    out[0] = h;
    if (k < 2) return;
    out[1] = orc_chi2_sf(h, (double)k - 1.0, err);
    if (n <= k) return;
    out[2] = (h - (double)k + 1.0) / (double)(n - k);
}

int orc_kruskal_block(const int64_t* orders, const double* svals, const int64_t* lengths,
                      const double* lab, const uint8_t* labp, const int64_t* cat, int64_t Fc,
                      int64_t Fq, int64_t S, int64_t lo, int64_t hi, double* stat, double* p,
                      double* eta, int threads) {
    int64_t kmax = 1;
    for (int64_t f = 0; f < Fc; ++f)
        if (cat[f] > kmax) kmax = cat[f];
#pragma omp parallel num_threads(threads)
    {
        double* cv = (double*)malloc((size_t)S * sizeof(double));
        double* cl = (double*)malloc((size_t)S * sizeof(double));
        double* rs = (double*)malloc((size_t)kmax * sizeof(double));
        int64_t* cnt = (int64_t*)malloc((size_t)kmax * sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
        for (int64_t h = lo; h < hi; ++h) {
            const int64_t* order = orders + h * S;
            const double* sv = svals + h * S;
            int64_t nall = lengths[h];
            for (int64_t g = 0; g < Fc; ++g) {
                int64_t k = cat[g];
                for (int64_t j = 0; j < k; ++j) { rs[j] = 0.0; cnt[j] = 0; }
                const double* lg = lab + g * S;
                const uint8_t* lp = labp + g * S;
                int64_t m = 0;
                for (int64_t i = 0; i < nall; ++i) {
                    int64_t s = order[i];
                    cv[m] = sv[i];
                    cl[m] = lg[s];
                    m += lp[s] ? 1 : 0;
                }
                double tie = 0.0;
                int bad = 0;
                int64_t i = 0;
                while (i < m && !bad) {
                    double v = cv[i];
                    int64_t j = i + 1;
                    while (j < m && cv[j] == v) j++;
                    int64_t run = j - i;
                    double avg = 0.5 * (double)(i + j + 1);
                    for (int64_t t = i; t < j; ++t) {
                        int64_t gi = (int64_t)cl[t];
                        if (gi < 0 || gi >= k) { bad = 1; break; }
                        rs[gi] += avg;
                        cnt[gi] += 1;
                    }
                    if (run > 1) tie += (double)run * (double)run * (double)run - (double)run;
                    i = j;
                }
                if (bad) { set_err(ORC_ERR_LABEL); continue; }
                double out[3];
                int e = 0;
                kruskal_finish(rs, cnt, k, tie, out, &e);
                if (e) set_err(e);
                if (stat) stat[g * Fq + h] = out[0];
                if (p) p[g * Fq + h] = out[1];
                if (eta) eta[g * Fq + h] = out[2];
            }
        }
        free(cv);
        free(cl);
        free(rs);
        free(cnt);
    }
    return take_err();
}

/* ------------------------------------------------------------------ */
/* Scalar entry points for the golden-vector tests                     */
/* ------------------------------------------------------------------ */

int orc_specfun(int which, const double* args, int64_t n, int nargs, double* out) {
    int first = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double* a = args + i * nargs;
        int e = 0;
        double r = NAN;
        switch (which) {
            case 0: r = orc_ln_gamma(a[0], &e); break;
            case 1: r = orc_reg_inc_beta(a[0], a[1], a[2], &e); break;
            case 2: r = orc_reg_inc_gamma_upper(a[0], a[1], &e); break;
            case 3: r = orc_normal_sf(a[0]); break;
            case 4: r = orc_t_sf(a[0], a[1], &e); break;
            case 5: r = orc_chi2_sf(a[0], a[1], &e); break;
            case 6: r = orc_f_sf(a[0], a[1], a[2], &e); break;
            case 7: r = orc_beta_sym_sf(a[0], a[1], &e); break;
            default: return ORC_ERR_DOMAIN;
        }
        out[i] = r;
        if (e && !first) first = e;
    }
    return first;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
