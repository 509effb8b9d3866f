// ps_internal.cuh -- device-resident matrix handle and kernel entry points
// shared between the per-test translation units and the C-ABI layer.
#pragma once
#include <functional>
#include <utility>
#include <vector>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>
#include "ps_common.cuh"

// Device copy of one input matrix, prepared once per run (the device half of
// the reference's make_matrix + _presort_matrix, datamodel.py:144-196,
// engine.py:379-400).
struct ps_matrix {
  int kind = PS_KIND_CONTINUOUS;
  int device = 0;
  int64_t F = 0, S = 0;
  int64_t ld = 0;         // row stride of d_vals (doubles), multiple of 32
  int64_t W = 0;          // mask words per row = ceil(S/32)
  int64_t ldc = 0;        // row stride of d_codes (bytes), multiple of 16
  uint64_t sentinel_bits = 0;
  int sentinel_is_nan = 1;
  bool owns_vals = true;
  double* d_vals = nullptr;       // F x ld raw fp64 values (zero beyond S)
  uint32_t* d_mask = nullptr;     // F x W presence bits (bit s%32 of word s/32)
  double* d_center = nullptr;     // F per-feature pivot (mean of present values)
  int32_t* d_count = nullptr;     // F present counts
  // label kinds
  int64_t* h_cat = nullptr;       // host copy of category counts
  int32_t* d_cat = nullptr;       // F category counts (device)
  int cmax = 0;
  uint8_t* d_codes = nullptr;     // F x ldc: trunc(label) or 0xFE (present, out of range) / 0xFF (missing)
  int code_bytes = 1;             // 2 when some category count exceeds 254: uint16 codes, 0xFFFE / 0xFFFF
  uint32_t* d_zero = nullptr;     // F x W bits: present && value == 0.0 (ttest / mwu grouping)
  uint32_t* d_bad = nullptr;      // F x W bits: present && label out of [0, c_f)
  // presort tables (rank tests)
  bool has_presort = false;
  bool owns_presort = true;       // false: tables live in caller buffers (ps_matrix_attach_presort)
  int32_t* d_len = nullptr;       // F present counts (== d_count)
  int64_t ldo = 0;                // row stride of d_order / d_inv (uint16), multiple of 64
  int64_t ldt = 0;                // row stride of the tie tables (words), tie_words(S)
  uint16_t* d_order = nullptr;    // F x ldo: sample ids of present entries, ascending value, stable
  uint16_t* d_inv = nullptr;      // F x ldo: sorted position of sample s, 0xFFFF if missing
  uint32_t* d_tb = nullptr;       // F x ldt: tie-group boundary bits (ps_ties.cuh)
  uint16_t* d_lastb = nullptr;    // F x ldt: prefix-max boundary position per word
  uint16_t* d_nextb = nullptr;    // F x ldt: suffix-min boundary position per word
  uint8_t* d_tied = nullptr;      // F: 1 if the feature has a tie group of size > 1
  // tie-group index of the 16-bit tables (always library-owned): per word the
  // number of group starts before it, the start position of every group
  // (group D = the end sentinel n) and the group count D
  uint16_t* d_gp = nullptr;       // F x ldt
  uint16_t* d_bpos = nullptr;     // F x ldo
  int32_t* d_ngrp = nullptr;      // F
  uint32_t* d_ordgid = nullptr;   // F x ldo: order | group id << 16 (only when the Spearman walk streams g)
  // S > 65535 ("wide"): 32-bit orders and tie prefix tables instead of the
  // 16-bit ones (no inverse permutation); walked by the wide rank kernels
  bool wide = false;
  uint32_t* d_order32 = nullptr;  // F x ldo
  uint32_t* d_lastb32 = nullptr;  // F x ldt
  uint32_t* d_nextb32 = nullptr;  // F x ldt
  void* presort_scratch[4] = {nullptr, nullptr, nullptr, nullptr};  // global radix path (S > 20480)
  // device-side presort in row chunks on the auxiliary stream: (rows [0, r1)
  // presorted, event) -- rank walks start on the chunks already done
  std::vector<std::pair<int64_t, cudaEvent_t>> presort_marks;
  cudaEvent_t ready = nullptr;  // device-created matrices: values / codes prepared
};

// true when the matrix carries presort chunk marks some of which are still
// pending on the device (the walks can then overlap the presort)
// Pearson moments Sx = X' M^T and Sxx = X'^2 M^T on the int8 tensor cores
// (ps_moments.cu): rows / columns [lo, F) of two F x F fp64 matrices (freed
// by the caller); ps_moments_on: the large-F Pearson path uses them
bool ps_moments_on(int64_t F, int64_t S);
// digits of the expansion: each expanded term is within 2^(e - 7 kMomentDigits) of x'
constexpr int kMomentDigits = 8;
// Sx uses the top 7 digit planes (its truncation error 2^(e - 49) enters the
// centred sums only through Sx^2 / n and Sx Sy / n)
constexpr int kSxDigits = 7;
// Sxy keeps the digit products D_s D_t^T with s + t <= kSxyMaxOrder (36 of
// the 64).  The dropped ones (s + t >= 10, |d_s d_t| <= 4096) sum to below
// 7.06 * 2^-58 < 2^-55.1 of 2^(e_g + e_h + 2) per element; with the
// expansion error 2^(e_g + e_h - 55) the per-element error stays below
// 2^-54 of 2^(e_g + e_h + 2) (ps_pearson.cu sxy_imprecise).
constexpr int kSxyMaxOrder = 9;
constexpr int kSxyProducts = 36;  // pairs s, t in [1, 8] with s + t <= 9
// the symmetric form (S < 2^17) contracts 16 sum planes (D_s + D_t)(D_s + D_t)^T
// and the 8 squares D_s D_s^T instead: 24 products, 48 roundings in the fold
constexpr int kSxySymProducts = 24;
constexpr int kSxyFoldTerms = 48;
bool ps_sxy_sym(int64_t S);
int ps_pearson_moments(const ps_matrix* a, const double* xc, int64_t lo, int64_t hi, double** sx, double** sq,
                       int32_t** e1, int32_t** e2, double* sxy, int32_t* nn, cudaStream_t s);
// the large-F Pearson path also takes Sxy and n from int8 digit products (no
// FP64 tensor tiles); PS_PEARSON_SXY=dmma keeps the DMMA Sxy tiles
bool ps_sxy_int8(int64_t S);
// incremental form (ps_run follows the upload): rows, then tile columns of 256
struct ps_moments_job;
int ps_moments_job_begin(const ps_matrix* a, const double* xc, double* sxy, int32_t* nn, cudaStream_t s,
                         ps_moments_job** out);
int ps_moments_job_rows(ps_moments_job* j, int64_t r1, cudaStream_t s);
int ps_moments_job_cols(ps_moments_job* j, int64_t J1, cudaStream_t s);
int ps_moments_job_end(ps_moments_job* j, double** sx, double** sq, int32_t** e1, int32_t** e2, cudaStream_t s);
void ps_moments_job_abort(ps_moments_job* j, cudaStream_t s);
constexpr int kMomentTile = 256;
// true when the Spearman walk streams g's order (large S): d_ordgid is built
bool ps_spearman_streams_g(int64_t S);
// tie-group index (d_gp / d_bpos / d_ngrp) of rows [f0, f1) from the boundary bits
int ps_tie_index(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s);

bool ps_presort_pending(const ps_matrix* m);

// Per-device library state.
struct ps_device_state {
  int device = -1;
  int num_sms = 148;
  int* d_err = nullptr;           // device error word
  cudaStream_t stream = nullptr;  // library stream used by ps_run
  cudaStream_t aux = nullptr;     // second stream: per-chunk prep / presort during uploads
  cudaEvent_t aux_ev = nullptr;
  static constexpr int kWalkStreams = 4;
  cudaStream_t walk[kWalkStreams] = {};  // incremental rank walks during uploads
  cudaEvent_t walk_ev[kWalkStreams + 1] = {};
  cudaEvent_t alloc_ev = nullptr;  // orders allocations made on `stream` before work on `aux`
  cudaEvent_t stat_ev = nullptr;   // ps_run: a test's statistic matrix is final (early D2H)
};

ps_device_state* ps_state();                 // current device's state
void ps_count_launch(int n = 1);             // kernel-launch accounting
int ps_fail(int code, const std::string& msg);
int ps_cuda_check(cudaError_t e, const char* what);

#define PS_CUDA(call)                                              \
  do {                                                             \
    cudaError_t _e = (call);                                       \
    if (_e != cudaSuccess) return ps_cuda_check(_e, #call);        \
  } while (0)

#define PS_LAUNCHED()                                                      \
  do {                                                                     \
    ps_count_launch();                                                     \
    cudaError_t _e = cudaGetLastError();                                   \
    if (_e != cudaSuccess) return ps_cuda_check(_e, "kernel launch");     \
  } while (0)

// Kernel-level profiling: when enabled, the dominant kernel of each test
// records CUDA events on its launch stream (bench.py reads them back).
void ps_prof_begin(const char* name, cudaStream_t s);
void ps_prof_end(cudaStream_t s);

// Workspace allocation on the stream-ordered pool.
template <typename T>
inline cudaError_t ps_alloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync((void**)p, count * sizeof(T) + 16, s);
}
inline void ps_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// Kernel-family entry points (implemented per translation unit).
int ps_prepare_matrix(ps_matrix* m, cudaStream_t s);
int ps_mixed_label_check(ps_matrix* lab, ps_matrix* val, int64_t g0, int64_t g1, int64_t h0, int64_t h1,
                         cudaStream_t s);
int ps_prepare_alloc(ps_matrix* m, cudaStream_t s);
int ps_prepare_rows(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s);
int ps_presort_matrix(ps_matrix* m, cudaStream_t s);
int ps_presort_begin(ps_matrix* m, cudaStream_t s);
int ps_presort_attach(ps_matrix* m, uint16_t* order, uint16_t* inv, uint32_t* tb, uint16_t* lastb, uint16_t* nextb,
                      uint8_t* tied, int32_t* len, cudaStream_t s);
int ps_presort_rows(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s);
int ps_presort_end(ps_matrix* m, cudaStream_t s);
int ps_fill_nan(double* p, int64_t n, cudaStream_t s);
int ps_pearson_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* r2,
                   cudaStream_t s);
// pre-centred operands x' = x - c_f (0 where missing), rows [f0, f1) into out (F x ld)
int ps_center_rows(const ps_matrix* m, double* out, int64_t f0, int64_t f1, cudaStream_t s);
// Walk streams for incremental launches: launch k goes to stream k mod
// kWalkStreams after it waits on `after`; join makes `s` wait on every used one.
cudaStream_t ps_walk_stream(int k, cudaStream_t after);
int ps_walk_streams_join(int used, cudaStream_t s);
struct ps_pearson_job;
// Incremental Pearson tiles (outputs must exist when the job begins).
int ps_pearson_begin(ps_matrix* a, double* stat, double* p, double* r2, cudaStream_t s, ps_pearson_job** job);
int ps_pearson_upto(ps_pearson_job* job, int64_t h1, cudaStream_t s);
// stat_ready (optional): recorded on s once the statistic and effect-size
// matrices are final (before the deferred p-value pass)
int ps_pearson_end(ps_pearson_job* job, cudaStream_t s, cudaEvent_t stat_ready = nullptr);
void ps_pearson_abort(ps_pearson_job* job, cudaStream_t s);
struct ps_group_job;
// Incremental ANOVA / t-test moment contraction (as the Spearman job).
int ps_group_moment_begin(int test, ps_matrix* lab, ps_matrix* val, int student, cudaStream_t s, ps_group_job** job);
int ps_group_moment_upto(ps_group_job* job, int64_t h1, cudaStream_t s);
int ps_group_moment_end(ps_group_job* job, double* stat, double* p, double* eff, cudaStream_t s);
void ps_group_moment_abort(ps_group_job* job, cudaStream_t s);
struct ps_rank_job;
// Incremental Mann-Whitney / Kruskal-Wallis walks (as the Spearman job).
int ps_rank_mixed_begin(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int u_mode, cudaStream_t s,
                        ps_rank_job** job);
int ps_rank_mixed_walk_upto(ps_rank_job* job, int64_t h1, cudaStream_t s);
int ps_rank_mixed_end(ps_rank_job* job, double* stat, double* p, double* eff, cudaStream_t s);
void ps_rank_mixed_abort(ps_rank_job* job, cudaStream_t s);
struct ps_spearman_job;
// Incremental Spearman walk (ps_run overlaps it with the input upload):
// begin allocates, walk_upto walks the columns h < h1 whose rows are
// presorted, end walks the rest, folds and finishes (and frees the job).
int ps_spearman_begin(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho, cudaStream_t s,
                      ps_spearman_job** job);
int ps_spearman_walk_upto(ps_spearman_job* job, int64_t h1, cudaStream_t s);
int ps_spearman_end(ps_spearman_job* job, cudaStream_t s);
void ps_spearman_abort(ps_spearman_job* job, cudaStream_t s);
int ps_spearman_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* rho,
                    cudaStream_t s);
bool ps_spearman_wide(int64_t S);  // S beyond the shared-memory walk (wide walk, no upload overlap)
int ps_chi2_run(ps_matrix* a, int64_t lo, int64_t hi, double* stat, double* p, double* phi,
                double* v, cudaStream_t s);
int ps_group_moment_run(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi,
                        int student, double* stat, double* p, double* eff, cudaStream_t s);
int ps_rank_mixed_run(int test, ps_matrix* lab, ps_matrix* val, int64_t lo, int64_t hi, int u_mode,
                      double* stat, double* p, double* eff, cudaStream_t s);
int ps_adjust_run(const double* p, int64_t rows, int64_t cols, int method, int symmetric,
                  double* out, cudaStream_t s);
// on_rows(r0, nr, ev): called after the copy of rows [r0, r0 + nr) was issued;
// ev is recorded on the copy stream right after it
typedef std::function<int(int64_t, int64_t, cudaEvent_t)> ps_rows_done_fn;
int ps_stage_h2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                    cudaStream_t s, const ps_rows_done_fn& on_rows = nullptr);
int ps_stage_labels_h2d(const double* src, size_t spitch, int64_t F, int64_t S, uint64_t sent_bits, int sent_nan,
                        const int64_t* cat, uint8_t* d_codes, int64_t ldc, int code_bytes, uint32_t* d_zero,
                        int64_t W, cudaStream_t s);
int ps_prepare_labels_from_host(ps_matrix* m, const double* src, int64_t src_ld, cudaStream_t s);
int ps_stage_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
void ps_host_prefault(void* dst, size_t bytes);
size_t ps_stage_chunk_bytes();  // staging chunk size (bytes)
int ps_stage_d2h_many(int n, void* const* dst, const void* const* src, const size_t* bytes, cudaStream_t s);
int ps_adjust_family_run(const double* p, int64_t n, int method, double* out, cudaStream_t s);
