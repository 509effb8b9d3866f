/*
 * pairstat_b200.h -- C ABI of the B200-native all-pairs test engine.
 *
 * This is the drop-in boundary for the reference's compiled hot path.  The
 * reference (pkg/src/pairstat) binds its numba block kernels from Python:
 *
 *   engine._pearson_block(values, present, lo, hi, want.., out..)   engine.py:145-166
 *   engine._spearman_block(orders, svals, lengths, present, lo, hi, ..)  :169-205
 *   engine._chi2_block(values, present, cat_counts, lo, hi, ..)     :208-242
 *   engine._ttest_block(labels, lab_present, values, val_present, lo, hi, student, ..) :245-263
 *   engine._anova_block(labels, lab_present, cat_counts, values, val_present, lo, hi, ..) :266-293
 *   engine._mwu_block(orders, svals, lengths, labels, lab_present, lo, hi, mode, ..) :296-319
 *   engine._kruskal_block(orders, svals, lengths, labels, lab_present, cat_counts, lo, hi, ..) :322-352
 *   engine._presort_matrix(matrix, threads)                          :379-400
 *   adjust.adjust(p_matrix, method, symmetric)                       adjust.py:46-87
 *   engine.run(request, mat_a, mat_b)                                engine.py:415-557
 *
 * Each is replaced by one entry point below.  The precomputed inputs of the
 * reference kernels (present masks, presort tables, category counts) become
 * one opaque device-resident handle, ps_matrix, built by ps_matrix_create
 * (the device half of make_matrix + _presort_matrix).  Block entry points keep
 * the reference's range semantics: homogeneous tests compute triangle rows
 * g in [lo, hi) against h in [g, F) and mirror; ttest/anova compute flat grid
 * cells idx in [lo, hi) (g = idx / F_Q); mwu/kruskal compute continuous
 * features h in [lo, hi) against every label row.  A NULL output pointer is
 * the reference's want_* = False.  Output pointers are DEVICE pointers to
 * caller-owned, NaN-prefilled, row-major fp64 matrices (F x F or F_C x F_Q).
 *
 * ps_run is the host-buffer convenience used by the Python run(): it copies
 * host inputs to the device, runs the block(s) over the full range, applies
 * the requested adjustments on the device and copies every requested matrix
 * back into host memory.
 *
 * All functions return a status code (PS_OK or PS_ERR_*); ps_last_error()
 * returns a message for the calling thread's last failure.  The library holds
 * an internal lock, so concurrent callers are serialised.
 */
#ifndef PAIRSTAT_B200_H
#define PAIRSTAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (python: paper_2505_00448_b200/errors.py STATUS_TO_ERROR). */
#define PS_OK 0
#define PS_ERR_INVALID 1
#define PS_ERR_CUDA 2
#define PS_ERR_LABEL_OUT_OF_RANGE 3 /* LabelOutOfRange   categorical.py:88-91, mixed.py:512-515, :613-617 */
#define PS_ERR_EXACT_WITH_TIES 4    /* ExactModeWithTies mixed.py:316-320 */
#define PS_ERR_TABLE_TOO_LARGE 5    /* TableTooLarge     mixed.py:321-324 */
#define PS_ERR_NONCONVERGENCE 6     /* NonConvergence    specfun.py:108, :188, :208 */
#define PS_ERR_DOMAIN 7             /* DomainError       specfun.py */
#define PS_ERR_UNKNOWN_METHOD 8     /* UnknownMethod     adjust.py:66-70 */
#define PS_ERR_NON_SQUARE 9         /* NonSquareSymmetric adjust.py:77-81 */
#define PS_ERR_NO_DEVICE 10
#define PS_ERR_IO 11                /* OSError of matio.write_matrix / read_matrix */

/* Tests, in the reference's TESTS order (datamodel.py:47-57). */
#define PS_TEST_PEARSON 0
#define PS_TEST_SPEARMAN 1
#define PS_TEST_CHI2 2
#define PS_TEST_TTEST 3
#define PS_TEST_MWU 4
#define PS_TEST_ANOVA 5
#define PS_TEST_KRUSKAL 6

/* Matrix kinds (datamodel.py:40). */
#define PS_KIND_CONTINUOUS 0
#define PS_KIND_DICHOTOMOUS 1
#define PS_KIND_CATEGORICAL 2

/* Adjustment methods (adjust.py:20). */
#define PS_ADJ_BONFERRONI 0
#define PS_ADJ_BH 1
#define PS_ADJ_BY 2

/* U-test modes (mixed.py:36-40). */
#define PS_U_EXACT 0
#define PS_U_ASYMPTOTIC 1
#define PS_U_AUTO 2

/* Opaque device-resident prepared matrix (values, packed validity mask,
 * label codes, presort tables). */
typedef struct ps_matrix ps_matrix;

/* Description of a matrix as the reference's DataMatrix holds it
 * (datamodel.py:112-141): fp64 values, features x samples, row-major with
 * row stride `ld` elements, the missing-value sentinel, and for label kinds
 * the per-feature category counts (host pointer, length n_features). */
typedef struct ps_matrix_desc {
  const double* values;
  int64_t n_features;
  int64_t n_samples;
  int64_t ld;
  double na_sentinel;
  int kind;
  const int64_t* category_counts;
} ps_matrix_desc;

/* Library / device queries. */
const char* ps_version(void);
const char* ps_last_error(void);
int ps_device_count(int* count);
int ps_set_device(int device);

/* Build a device-resident prepared matrix.  `values_on_device` != 0 means
 * desc->values is a device pointer (no H2D copy).  `want_presort` builds the
 * per-feature sort tables needed by spearman / mwu / kruskal.  `stream` is a
 * cudaStream_t (NULL = legacy default stream). */
int ps_matrix_create(const ps_matrix_desc* desc, int values_on_device, int want_presort,
                     void* stream, ps_matrix** out);
int ps_matrix_destroy(ps_matrix* m);

/* Block kernels (device outputs; see file header for range semantics). */
int ps_pearson_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                     double* out_r2, void* stream);
/* The Pearson contraction path for an n_features x n_samples matrix, a
 * function of the shape alone (PS_PEARSON_MOMENTS=0/1 and PS_PEARSON_SXY=dmma
 * override), so every launch range and device count of one matrix takes the
 * same path: 0 = five-product FP64 DMMA tiles; 1 = masked moments as exact
 * int8 digit contractions + Sxy on DMMA tiles; 2 = moments, Sxy and pair
 * counts all as int8 digit contractions (ps_moments.cu). */
int ps_pearson_moments_used(int64_t n_features, int64_t n_samples);
int ps_spearman_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                      double* out_rho, void* stream);
int ps_chi2_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                  double* out_phi, double* out_v, void* stream);
int ps_ttest_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, int student,
                   double* out_stat, double* out_p, double* out_d, void* stream);
int ps_anova_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi,
                   double* out_stat, double* out_p, double* out_eta, void* stream);
int ps_mwu_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, int u_mode,
                 double* out_stat, double* out_p, double* out_r, void* stream);
int ps_kruskal_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi,
                     double* out_stat, double* out_p, double* out_eta, void* stream);

/* Multiple-testing adjustment of a device p matrix (adjust.py:46-87):
 * symmetric = strict upper triangle family mirrored with a NaN diagonal. */
int ps_adjust_device(const double* p, int64_t rows, int64_t cols, int method, int symmetric,
                     double* out, void* stream);

/* Host-buffer adjustment (the public adjust(), adjust.py:46-87). */
int ps_adjust(const double* p, int64_t rows, int64_t cols, int method, int symmetric, double* out);

/* Adjustment of an arbitrary device vector family (adjust.py:23-43).  Used by
 * the multi-GPU path after the p-values of all shards are gathered. */
int ps_adjust_family_device(const double* p, int64_t n, int method, double* out, void* stream);

/* Wait for `stream` and return the first error raised by a device kernel
 * since the last check (LabelOutOfRange, NonConvergence, ...). */
int ps_sync(void* stream);

/* Device special functions on a host batch (golden-grid tests): which =
 * 0 ln_gamma(x), 1 reg_inc_beta(x,a,b), 2 reg_inc_gamma_upper(a,x),
 * 3 normal_sf(z), 4 t_sf(t,dof), 5 chi2_sf(x,dof), 6 f_sf(f,d1,d2),
 * 7 beta_sym_sf(r,a) -- specfun.py:41-314.  args is n x nargs row-major. */
int ps_specfun_eval(int which, const double* args, int64_t n, int nargs, double* out);

/* numpy-identical BY harmonic factor c(m) (exposed for tests). */
double ps_by_factor(int64_t m);

/* Host-buffer end-to-end run (engine.py:415-557).  `b` is NULL for
 * homogeneous tests.  outs[0..3] are host pointers for the canonical raw
 * outputs ("stat", "p", effect 1, effect 2), adj_outs[0..2] for
 * p_bonferroni / p_bh / p_by; NULL = not requested.  Output matrices are
 * overwritten completely. */
int ps_run(int test, const ps_matrix_desc* a, const ps_matrix_desc* b, int t_variant, int u_mode,
           double* const* outs, double* const* adj_outs);

/* Instrumentation: number of kernels this library launched since the last
 * reset, and a device-time breakdown of the last block call. */
int64_t ps_kernel_launches(void);
void ps_reset_kernel_launches(void);

/* Kernel-level timing: when enabled, the dominant kernel of each block call
 * ("pearson_tile", "spearman_walk", "chi2_gemm", "group_gemm", "rank_mixed_walk")
 * is bracketed by CUDA events on its launch stream.  collect() sums them. */
void ps_profile_enable(int on);
int ps_profile_collect(const char* name, double* total_ms, int64_t* count);
/* The union of the launch intervals instead of their sum: the kernel's busy
 * time when launches of it run concurrently on several streams. */
int ps_profile_collect_union(const char* name, double* busy_ms, int64_t* count);

/* ---- presort tables in caller buffers (multi-GPU sharded presort) ----
 * Rank r presorts its own rows into buffers of F rows (ps_presort_layout gives
 * the row strides: order / inv uint16 x ldo, tb uint32 x ldt, lastb / nextb
 * uint16 x ldt, tied uint8, len int32), the ranks all-gather the rows (NCCL),
 * then ps_matrix_presort_done marks the tables complete.  Rows are
 * independent, so the gathered tables equal a single-GPU presort bit for bit. */
int ps_presort_layout(int64_t n_samples, int64_t* ldo, int64_t* ldt);
int ps_matrix_attach_presort(ps_matrix* m, void* order, void* inv, void* tb, void* lastb, void* nextb, void* tied,
                             void* len, void* stream);
int ps_matrix_presort_rows(ps_matrix* m, int64_t f0, int64_t f1, void* stream);
int ps_matrix_presort_done(ps_matrix* m, void* stream);

/* ---- multi-GPU result exchange (family = adjust.py:23-87) ----
 * A rank owning the reference partition [lo, hi) of `test` (triangle rows for
 * pearson / spearman / chi2, engine.py:93-125; flat cells for ttest / anova;
 * continuous features for mwu / kruskal, engine.py:70-90) packs the cells of
 * its range from a device rows x cols matrix into a dense device vector and,
 * after the ranks all-gathered the vectors, unpacks any rank's segment back
 * (mirrored for the symmetric layout).  Triangle rows hold the h > g cells
 * (diag = 0: the adjustment family; unpack writes a NaN diagonal) or h >= g
 * (diag = 1: raw outputs with their self-tests), row-major: one contiguous
 * segment of the reference's family order. */
/* Host rows -> device rows through the library's pinned, all-core staging
 * ring (each rank uploads its shard of the input); device padding columns
 * [width, dpitch) are zeroed.  Pitches and width in bytes. */
int ps_copy_h2d_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t rows,
                   void* stream);
int ps_cells_count(int test, int diag, int64_t rows, int64_t cols, int64_t lo, int64_t hi, int64_t* n);
int ps_cells_pack(int test, int diag, const double* mat, int64_t rows, int64_t cols, int64_t lo, int64_t hi,
                  double* vec, void* stream);
int ps_cells_unpack(int test, int diag, const double* vec, int64_t rows, int64_t cols, int64_t lo, int64_t hi,
                    double* mat, void* stream);

/* ---- delimited matrix files (matio.py:40-125; host code, no device) ----
 * ps_write_matrix: the reference's write_matrix byte for byte: header
 * delim-joined ["", col ids...], rows [row id, f"{v:.17g}"...] ("nan" for any
 * NaN), "\n" line ends.  row_ids / col_ids may be NULL (f0.., s0..). */
int ps_write_matrix(const char* path, const double* values, int64_t rows, int64_t cols,
                    const char* const* row_ids, const char* const* col_ids, char delim);

/* ps_read_matrix: read_matrix's parse (str.splitlines boundaries, empty lines
 * skipped, Python float() grammar).  On return `error` is 0 (ok), 1 (empty
 * file), 2 (ragged: err_row, err_count values) or 3 (malformed: err_row,
 * err_col, err_cell bytes); rows are 1-based file lines as in the reference's
 * messages.  ids are '\0'-terminated strings laid end to end.  Cells holding
 * non-ASCII bytes are listed in `fallback` (flat indices) for the caller to
 * parse.  Release with ps_matrix_file_free. */
typedef struct ps_matrix_file {
  int error;
  int os_errno;
  int64_t n_rows, n_cols;
  const double* values;
  const char* row_ids;
  int64_t row_ids_len;
  const char* col_ids;
  int64_t col_ids_len;
  const int64_t* fallback;
  int64_t n_fallback;
  int64_t err_row, err_col, err_count;
  const char* err_cell;
  int64_t err_cell_len;
  void* impl;
} ps_matrix_file;
int ps_read_matrix(const char* path, char delim, ps_matrix_file* out);
void ps_matrix_file_free(ps_matrix_file* f);

#ifdef __cplusplus
}
#endif
#endif /* PAIRSTAT_B200_H */
