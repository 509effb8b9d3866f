// ps_api.cu -- the C ABI (include/pairstat_b200.h): device state, prepared
// matrices, block entry points and the host-buffer run() used by Python.
#include "ps_internal.cuh"
#include "ps_ties.cuh"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>
#include <vector>
#include <thread>

namespace {

// One lock per device: callers on the same device are serialised (its
// streams, pool and error word are shared), callers driving different
// devices -- a single-process multi-GPU run, one host thread per device --
// run concurrently.
std::recursive_mutex g_locks[64];
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
ps_device_state g_states[64];

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

struct Guard {
  std::lock_guard<std::recursive_mutex> lk{g_locks[current_device() & 63]};
};

int init_state(ps_device_state* st, int dev) {
  if (st->device == dev) return PS_OK;
  PS_CUDA(cudaSetDevice(dev));
  cudaDeviceProp prop;
  PS_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10) return ps_fail(PS_ERR_NO_DEVICE, "pair engine needs an sm_100 (B200) device");
  st->num_sms = prop.multiProcessorCount;
  PS_CUDA(cudaMalloc(&st->d_err, sizeof(int)));
  PS_CUDA(cudaMemset(st->d_err, 0, sizeof(int)));
  PS_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;
  PS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // aux carries the per-chunk prep / presort that incremental walks wait on
  PS_CUDA(cudaStreamCreateWithPriority(&st->aux, cudaStreamNonBlocking, prio_hi));
  PS_CUDA(cudaEventCreateWithFlags(&st->aux_ev, cudaEventDisableTiming));
  for (auto& w : st->walk) PS_CUDA(cudaStreamCreateWithFlags(&w, cudaStreamNonBlocking));
  for (auto& e : st->walk_ev) PS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  PS_CUDA(cudaEventCreateWithFlags(&st->alloc_ev, cudaEventDisableTiming));
  PS_CUDA(cudaEventCreateWithFlags(&st->stat_ev, cudaEventDisableTiming));
  // keep freed workspace cached in the stream-ordered pool between calls
  cudaMemPool_t pool;
  PS_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;
  PS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  st->device = dev;
  return PS_OK;
}

int ensure_state() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return ps_fail(PS_ERR_NO_DEVICE, "no CUDA device visible");
  }
  const int dev = current_device();
  return init_state(&g_states[dev], dev);
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Read and reset the device error word (synchronises the stream).
int drain_errors(cudaStream_t s) {
  ps_device_state* st = ps_state();
  int err = 0;
  PS_CUDA(cudaMemcpyAsync(&err, st->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  PS_CUDA(cudaStreamSynchronize(s));
  if (err) {
    PS_CUDA(cudaMemsetAsync(st->d_err, 0, sizeof(int), s));
    PS_CUDA(cudaStreamSynchronize(s));
    return ps_fail(err, "raised by a device kernel");
  }
  return PS_OK;
}

struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::atomic<bool> g_prof{false};
std::mutex g_prof_lock;  // guards g_prof_recs (any device's thread may record)
std::vector<ProfRec> g_prof_recs;
thread_local int64_t g_prof_open = -1;  // index of this thread's open record

}  // namespace

void ps_prof_begin(const char* name, cudaStream_t s) {
  if (!g_prof) return;
  ProfRec r;
  r.name = name;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  std::lock_guard<std::mutex> lk(g_prof_lock);
  g_prof_recs.push_back(r);
  g_prof_open = (int64_t)g_prof_recs.size() - 1;
}
void ps_prof_end(cudaStream_t s) {
  if (!g_prof || g_prof_open < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_lock);
  if (g_prof_open < (int64_t)g_prof_recs.size()) cudaEventRecord(g_prof_recs[g_prof_open].b, s);
  g_prof_open = -1;
}

ps_device_state* ps_state() { return &g_states[current_device()]; }
void ps_count_launch(int n) { g_launches += n; }
int ps_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int ps_cuda_check(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return PS_ERR_CUDA;
}

namespace {
// PS_TRACE=1: per-phase wall times of ps_run on stderr (synchronising)
struct Trace {
  bool on = getenv("PS_TRACE") != nullptr;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[ps_run] %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
// PS_TIMELINE=1: device timestamps (a one-thread kernel reads %globaltimer
// when its stream reaches the mark) and host enqueue times of the staging /
// presort / walk stages of ps_run, printed at the end of the run.
__global__ void stamp_kernel(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}
struct Timeline {
  bool on = getenv("PS_TIMELINE") != nullptr;
  std::vector<std::string> what;
  std::vector<double> host_ms;
  unsigned long long* d = nullptr;
  std::chrono::steady_clock::time_point t0;
  void mark(const std::string& w, cudaStream_t st) {
    if (!on) return;
    if (!d) {
      cudaMalloc(&d, 256 * sizeof(unsigned long long));
      t0 = std::chrono::steady_clock::now();
    }
    if (what.size() >= 256) return;
    stamp_kernel<<<1, 1, 0, st>>>(d + what.size());
    what.push_back(w);
    host_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  void dump() {
    if (!on || what.empty()) return;
    cudaDeviceSynchronize();
    std::vector<unsigned long long> t(what.size());
    cudaMemcpy(t.data(), d, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < t.size(); ++k)
      fprintf(stderr, "[timeline] %-28s gpu %8.3f ms   host %8.3f ms\n", what[k].c_str(), (t[k] - t[0]) * 1e-6,
              host_ms[k] - host_ms[0]);
    what.clear();
    host_ms.clear();
    cudaFree(d);
    d = nullptr;
  }
};
Timeline g_tl;
}  // namespace

extern "C" {

const char* ps_version(void) { return "paper_2505_00448_b200 0.1.0 (sm_100a)"; }
const char* ps_last_error(void) { return g_last_error.c_str(); }
int64_t ps_kernel_launches(void) { return g_launches.load(); }
void ps_reset_kernel_launches(void) { g_launches = 0; }

void ps_profile_enable(int on) { g_prof = on != 0; }

// Sum of event-timed milliseconds and launch count of kernel `name` since the
// last collect (synchronises on the recorded events); clears the records.
int ps_profile_collect(const char* name, double* total_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_prof_lock);
  double t = 0.0;
  int64_t c = 0;
  std::vector<ProfRec> keep;
  for (auto& r : g_prof_recs) {
    if (r.name == name) {
      cudaEventSynchronize(r.b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      t += ms;
      ++c;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    } else {
      keep.push_back(r);
    }
  }
  g_prof_recs.swap(keep);
  g_prof_open = -1;
  *total_ms = t;
  *count = c;
  return PS_OK;
}

// Union of the named kernel's launch intervals (concurrent launches on
// several streams count once): the kernel's busy time on the device.
int ps_profile_collect_union(const char* name, double* busy_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_prof_lock);
  std::vector<std::pair<double, double>> iv;
  std::vector<ProfRec> keep;
  cudaEvent_t base = nullptr;
  for (auto& r : g_prof_recs) {
    if (r.name != name) {
      keep.push_back(r);
      continue;
    }
    cudaEventSynchronize(r.b);
    if (!base) base = r.a;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, base, r.a);
    cudaEventElapsedTime(&b, base, r.b);
    iv.emplace_back(a, b);
  }
  std::sort(iv.begin(), iv.end());
  double busy = 0.0, cs = 0.0, ce = -1e300;
  for (const auto& x : iv) {
    if (x.first > ce) {
      if (ce > cs) busy += ce - cs;
      cs = x.first;
      ce = x.second;
    } else if (x.second > ce) {
      ce = x.second;
    }
  }
  if (!iv.empty() && ce > cs) busy += ce - cs;
  for (auto& r : g_prof_recs)
    if (r.name == name) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  g_prof_recs.swap(keep);
  g_prof_open = -1;
  *busy_ms = busy;
  *count = (int64_t)iv.size();
  return PS_OK;
}

int ps_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return PS_OK;
}

}  // extern "C"

cudaStream_t ps_walk_stream(int k, cudaStream_t after) {
  ps_device_state* st = ps_state();
  constexpr int K = ps_device_state::kWalkStreams;
  cudaStream_t w = st->walk[k % K];
  cudaEventRecord(st->walk_ev[K], after);
  cudaStreamWaitEvent(w, st->walk_ev[K], 0);
  if (g_tl.on) g_tl.mark("  walk launch " + std::to_string(k), after);
  return w;
}

int ps_walk_streams_join(int used, cudaStream_t s) {
  ps_device_state* st = ps_state();
  for (int k = 0; k < ps_device_state::kWalkStreams && k < used; ++k) {
    PS_CUDA(cudaEventRecord(st->walk_ev[k], st->walk[k]));
    PS_CUDA(cudaStreamWaitEvent(s, st->walk_ev[k], 0));
    if (g_tl.on) g_tl.mark("  walk stream " + std::to_string(k) + " done", st->walk[k]);
  }
  return PS_OK;
}

extern "C" {

int ps_set_device(int device) {
  Guard g;
  PS_CUDA(cudaSetDevice(device));
  return ensure_state();
}

}  // extern "C"

bool ps_presort_pending(const ps_matrix* m) {
  for (const auto& mk : m->presort_marks)
    if (cudaEventQuery(mk.second) == cudaErrorNotReady) return true;
  cudaGetLastError();
  return false;
}

// Device-resident presort in chunks of one CTA wave of features on the
// auxiliary stream, each chunk marked by an event; the main stream waits for
// the whole presort (every other consumer stays ordered), while the rank walks
// of a following block call may start on the chunks already presorted.
static int presort_in_chunks(ps_matrix* m, cudaStream_t s) {
  ps_device_state* st = ps_state();
  const int64_t step = st->num_sms;
  // (S > 32767: the walks run one CTA per SM from global orders and their
  // one-item-per-CTA launches cost more than the presort they hide: config
  // 5s step 449 ms presorted up front vs 497-779 ms in chunks)
  if (m->F < 2 * step || m->S > 32767 || getenv("PS_NO_OVERLAP")) return ps_presort_matrix(m, s);
  int rc = ps_presort_begin(m, s);
  if (rc) return rc;
  PS_CUDA(cudaEventRecord(st->aux_ev, s));
  PS_CUDA(cudaStreamWaitEvent(st->aux, st->aux_ev, 0));
  for (int64_t r0 = 0; r0 < m->F && !rc; r0 += step) {
    const int64_t r1 = std::min<int64_t>(m->F, r0 + step);
    rc = ps_presort_rows(m, r0, r1, st->aux);
    cudaEvent_t e = nullptr;
    cudaError_t ce = cudaSuccess;
    if (!rc) ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (!rc && ce == cudaSuccess) ce = cudaEventRecord(e, st->aux);
    if (e) m->presort_marks.emplace_back(r1, e);
    if (!rc && ce != cudaSuccess) rc = ps_cuda_check(ce, "presort mark");
  }
  if (rc) return rc;
  PS_CUDA(cudaEventRecord(st->aux_ev, st->aux));
  PS_CUDA(cudaStreamWaitEvent(s, st->aux_ev, 0));
  return ps_presort_end(m, s);
}

// Called on the auxiliary stream after each staged chunk of rows [0, r1) is
// prepared (and presorted): lets ps_run start computing on the rows already
// uploaded while the rest of the input is still in flight.
using RowsHook = std::function<int(ps_matrix*, int64_t r1, cudaStream_t aux)>;

static int matrix_create(const ps_matrix_desc* desc, int values_on_device, int want_presort, cudaStream_t s,
                         ps_matrix** out, const RowsHook* hook) {
  *out = nullptr;
  int rc = ensure_state();
  if (rc) return rc;
  if (!desc || desc->n_features <= 0 || desc->n_samples <= 0)
    return ps_fail(PS_ERR_INVALID, "expected a non-empty matrix");
  Trace tr;
  tr.s = s;
  ps_matrix* m = new ps_matrix();
  m->device = current_device();
  m->kind = desc->kind;
  m->F = desc->n_features;
  m->S = desc->n_samples;
  m->W = ps_ceil_div(m->S, 32);
  const double sent = desc->na_sentinel;
  m->sentinel_is_nan = std::isnan(sent) ? 1 : 0;
  std::memcpy(&m->sentinel_bits, &sent, sizeof(double));
  const int64_t src_ld = desc->ld > 0 ? desc->ld : m->S;
  if (m->kind != PS_KIND_CONTINUOUS) {
    if (!desc->category_counts) {
      delete m;
      return ps_fail(PS_ERR_INVALID, "label matrix without category counts");
    }
    m->h_cat = new int64_t[m->F];
    std::memcpy(m->h_cat, desc->category_counts, sizeof(int64_t) * m->F);
    int64_t cmax = 0;
    for (int64_t f = 0; f < m->F; ++f) cmax = std::max(cmax, m->h_cat[f]);
    if (cmax > 65534) {
      delete[] m->h_cat;
      delete m;
      return ps_fail(PS_ERR_INVALID, "category counts above 65534 are not supported by the device path");
    }
    m->cmax = (int)cmax;
    m->code_bytes = cmax > 254 ? 2 : 1;  // 16-bit label codes beyond 254 levels
    std::vector<int32_t> c32(m->h_cat, m->h_cat + m->F);
    rc = ps_alloc(&m->d_cat, (size_t)m->F, s) == cudaSuccess ? 0 : PS_ERR_CUDA;
    if (!rc) rc = cudaMemcpyAsync(m->d_cat, c32.data(), sizeof(int32_t) * m->F, cudaMemcpyHostToDevice, s)
                      == cudaSuccess ? 0 : PS_ERR_CUDA;
    if (!rc) rc = cudaStreamSynchronize(s) == cudaSuccess ? 0 : PS_ERR_CUDA;
    if (rc) {
      ps_matrix_destroy(m);
      return ps_fail(PS_ERR_CUDA, "category count upload failed");
    }
  }
  if (!values_on_device && m->kind != PS_KIND_CONTINUOUS) {
    // host labels: converted to device codes while staging; no fp64 copy
    m->ld = ps_round_up(m->S, 32);
    m->owns_vals = false;
    rc = ps_prepare_labels_from_host(m, desc->values, src_ld, s);
    tr.mark("  labels");
    if (rc) {
      ps_matrix_destroy(m);
      return rc;
    }
    *out = m;
    return PS_OK;
  }
  if (values_on_device && (src_ld % 32) == 0 && (reinterpret_cast<uintptr_t>(desc->values) % 256) == 0) {
    // use the caller's device buffer in place (must be zero-padded to ld)
    m->d_vals = const_cast<double*>(desc->values);
    m->ld = src_ld;
    m->owns_vals = false;
  } else {
    m->ld = ps_round_up(m->S, 32);
    if (ps_alloc(&m->d_vals, (size_t)(m->F * m->ld), s) != cudaSuccess) {
      ps_matrix_destroy(m);
      return ps_fail(PS_ERR_CUDA, "out of device memory for the input matrix");
    }
    cudaError_t e = cudaSuccess;
    if (m->ld != m->S && values_on_device) e = cudaMemsetAsync(m->d_vals, 0, sizeof(double) * m->F * m->ld, s);
    if (e == cudaSuccess && values_on_device)
      e = cudaMemcpy2DAsync(m->d_vals, sizeof(double) * m->ld, desc->values, sizeof(double) * src_ld,
                            sizeof(double) * m->S, m->F, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) {
      ps_matrix_destroy(m);
      return ps_cuda_check(e, "input upload");
    }
    if (!values_on_device) {
      // pinned, double-buffered, all-core staging of the pageable input; the
      // validity pass and the presort of each uploaded chunk of rows run on
      // the auxiliary stream while the next chunk is copied
      ps_device_state* st = ps_state();
      rc = ps_prepare_alloc(m, s);
      if (!rc && want_presort) rc = ps_presort_begin(m, s);
      if (!rc) {
        auto on_rows = [&](int64_t r0, int64_t nr, cudaEvent_t ev) -> int {
          PS_CUDA(cudaStreamWaitEvent(st->aux, ev, 0));
          g_tl.mark("rows " + std::to_string(r0 + nr) + " copied", st->aux);
          int c = ps_prepare_rows(m, r0, r0 + nr, st->aux);
          if (!c && want_presort) c = ps_presort_rows(m, r0, r0 + nr, st->aux);
          g_tl.mark("  presorted", st->aux);
          if (!c && hook) c = (*hook)(m, r0 + nr, st->aux);
          return c;
        };
        rc = ps_stage_h2d_2d(m->d_vals, sizeof(double) * m->ld, desc->values, sizeof(double) * src_ld,
                             sizeof(double) * m->S, m->F, s, on_rows);
      }
      if (!rc) {
        cudaError_t e2 = cudaEventRecord(st->aux_ev, st->aux);
        if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(s, st->aux_ev, 0);
        if (e2 != cudaSuccess) rc = ps_cuda_check(e2, "upload overlap");
      }
      if (!rc && want_presort) rc = ps_presort_end(m, s);
      tr.mark("  upload+prep");
      if (rc) {
        ps_matrix_destroy(m);
        return rc;
      }
      *out = m;
      return PS_OK;
    }
  }
  tr.mark("  upload");
  rc = ps_prepare_matrix(m, s);
  tr.mark("  prepare");
  // the prepared values / codes (before any presort wait on s)
  if (!rc && cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming) == cudaSuccess)
    cudaEventRecord(m->ready, s);
  if (!rc && want_presort) rc = presort_in_chunks(m, s);
  tr.mark("  presort");
  if (rc) {
    ps_matrix_destroy(m);
    return rc;
  }
  *out = m;
  return PS_OK;
}

extern "C" {

int ps_matrix_create(const ps_matrix_desc* desc, int values_on_device, int want_presort, void* stream,
                     ps_matrix** out) {
  Guard g;
  return matrix_create(desc, values_on_device, want_presort, as_stream(stream), out, nullptr);
}

int ps_pearson_moments_used(int64_t F, int64_t S) { return ps_moments_on(F, S) ? (ps_sxy_int8(S) ? 2 : 1) : 0; }

int ps_presort_layout(int64_t S, int64_t* ldo, int64_t* ldt) {
  if (S <= 0 || S > 65535) return ps_fail(PS_ERR_INVALID, "rank tests need 1 <= samples <= 65535");
  *ldo = ps_round_up(S + 1, 64);
  *ldt = tie_words(S);
  return PS_OK;
}

int ps_matrix_attach_presort(ps_matrix* m, void* order, void* inv, void* tb, void* lastb, void* nextb, void* tied,
                             void* len, void* stream) {
  Guard g;
  if (!m || m->has_presort || m->d_order) return ps_fail(PS_ERR_INVALID, "matrix already has presort tables");
  return ps_presort_attach(m, static_cast<uint16_t*>(order), static_cast<uint16_t*>(inv), static_cast<uint32_t*>(tb),
                           static_cast<uint16_t*>(lastb), static_cast<uint16_t*>(nextb), static_cast<uint8_t*>(tied),
                           static_cast<int32_t*>(len), as_stream(stream));
}

int ps_matrix_presort_rows(ps_matrix* m, int64_t f0, int64_t f1, void* stream) {
  Guard g;
  if (!m || !m->d_order) return ps_fail(PS_ERR_INVALID, "matrix has no presort tables attached");
  f0 = std::max<int64_t>(0, f0);
  f1 = std::min<int64_t>(m->F, f1);
  return ps_presort_rows(m, f0, f1, as_stream(stream));
}

int ps_matrix_presort_done(ps_matrix* m, void* stream) {
  Guard g;
  if (!m || !m->d_order) return ps_fail(PS_ERR_INVALID, "matrix has no presort tables attached");
  return ps_presort_end(m, as_stream(stream));
}

int ps_matrix_destroy(ps_matrix* m) {
  if (!m) return PS_OK;
  Guard g;
  cudaStream_t s = ps_state()->stream;
  if (m->owns_vals) ps_free(m->d_vals, s);
  ps_free(m->d_mask, s);
  ps_free(m->d_center, s);
  ps_free(m->d_count, s);
  ps_free(m->d_cat, s);
  ps_free(m->d_codes, s);
  ps_free(m->d_zero, s);
  ps_free(m->d_bad, s);
  ps_free(m->d_order32, s);
  ps_free(m->d_lastb32, s);
  ps_free(m->d_nextb32, s);
  ps_free(m->d_gp, s);
  ps_free(m->d_bpos, s);
  ps_free(m->d_ngrp, s);
  ps_free(m->d_ordgid, s);
  if (m->owns_presort) {
    ps_free(m->d_order, s);
    ps_free(m->d_inv, s);
    ps_free(m->d_tb, s);
    ps_free(m->d_lastb, s);
    ps_free(m->d_nextb, s);
    ps_free(m->d_tied, s);
    ps_free(m->d_len, s);
  }
  for (void* p : m->presort_scratch) ps_free(p, s);
  for (auto& mk : m->presort_marks) cudaEventDestroy(mk.second);
  if (m->ready) cudaEventDestroy(m->ready);
  delete[] m->h_cat;
  delete m;
  return PS_OK;
}

static int need_kind(ps_matrix* m, bool continuous, const char* what) {
  if (!m) return ps_fail(PS_ERR_INVALID, std::string(what) + ": missing matrix");
  if (continuous != (m->kind == PS_KIND_CONTINUOUS))
    return ps_fail(PS_ERR_INVALID, std::string(what) + ": wrong matrix kind");
  return PS_OK;
}

int ps_pearson_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                     double* out_r2, void* stream) {
  Guard g;
  int rc = need_kind(a, true, "pearson");
  if (!rc) rc = ps_pearson_run(a, lo, hi, out_stat, out_p, out_r2, as_stream(stream));
  return rc;
}

int ps_spearman_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                      double* out_rho, void* stream) {
  Guard g;
  int rc = need_kind(a, true, "spearman");
  if (!rc && !a->has_presort) rc = ps_presort_matrix(a, as_stream(stream));
  if (!rc) rc = ps_spearman_run(a, lo, hi, out_stat, out_p, out_rho, as_stream(stream));
  return rc;
}

int ps_chi2_block(ps_matrix* a, int64_t lo, int64_t hi, double* out_stat, double* out_p,
                  double* out_phi, double* out_v, void* stream) {
  Guard g;
  int rc = need_kind(a, false, "chi2");
  if (!rc) rc = ps_chi2_run(a, lo, hi, out_stat, out_p, out_phi, out_v, as_stream(stream));
  return rc;
}

int ps_ttest_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, int student,
                   double* out_stat, double* out_p, double* out_d, void* stream) {
  Guard g;
  int rc = need_kind(labels, false, "ttest");
  if (!rc) rc = need_kind(values, true, "ttest");
  if (!rc)
    rc = ps_group_moment_run(PS_TEST_TTEST, labels, values, lo, hi, student, out_stat, out_p, out_d,
                             as_stream(stream));
  return rc;
}

int ps_anova_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, double* out_stat,
                   double* out_p, double* out_eta, void* stream) {
  Guard g;
  int rc = need_kind(labels, false, "anova");
  if (!rc) rc = need_kind(values, true, "anova");
  if (!rc)
    rc = ps_group_moment_run(PS_TEST_ANOVA, labels, values, lo, hi, 1, out_stat, out_p, out_eta,
                             as_stream(stream));
  return rc;
}

int ps_mwu_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, int u_mode,
                 double* out_stat, double* out_p, double* out_r, void* stream) {
  Guard g;
  int rc = need_kind(labels, false, "mwu");
  if (!rc) rc = need_kind(values, true, "mwu");
  if (!rc && !values->has_presort) rc = ps_presort_matrix(values, as_stream(stream));
  if (!rc)
    rc = ps_rank_mixed_run(PS_TEST_MWU, labels, values, lo, hi, u_mode, out_stat, out_p, out_r,
                           as_stream(stream));
  return rc;
}

int ps_kruskal_block(ps_matrix* labels, ps_matrix* values, int64_t lo, int64_t hi, double* out_stat,
                     double* out_p, double* out_eta, void* stream) {
  Guard g;
  int rc = need_kind(labels, false, "kruskal");
  if (!rc) rc = need_kind(values, true, "kruskal");
  if (!rc && !values->has_presort) rc = ps_presort_matrix(values, as_stream(stream));
  if (!rc)
    rc = ps_rank_mixed_run(PS_TEST_KRUSKAL, labels, values, lo, hi, 0, out_stat, out_p, out_eta,
                           as_stream(stream));
  return rc;
}

int ps_adjust_device(const double* p, int64_t rows, int64_t cols, int method, int symmetric,
                     double* out, void* stream) {
  Guard g;
  int rc = ensure_state();
  if (!rc) rc = ps_adjust_run(p, rows, cols, method, symmetric, out, as_stream(stream));
  return rc;
}

int ps_adjust_family_device(const double* p, int64_t n, int method, double* out, void* stream) {
  Guard g;
  int rc = ensure_state();
  if (!rc) rc = ps_adjust_family_run(p, n, method, out, as_stream(stream));
  return rc;
}

int ps_sync(void* stream) {
  Guard g;
  int rc = ensure_state();
  if (!rc) rc = drain_errors(as_stream(stream));
  return rc;
}

// Host-buffer end-to-end run: engine.run (engine.py:415-557) on the device.

int ps_run(int test, const ps_matrix_desc* a, const ps_matrix_desc* b, int t_variant, int u_mode,
           double* const* outs, double* const* adj_outs) {
  Guard g;
  int rc = ensure_state();
  if (rc) return rc;
  ps_device_state* st = ps_state();
  cudaStream_t s = st->stream;
  Trace tr;
  tr.s = s;
  const bool homogeneous = test == PS_TEST_PEARSON || test == PS_TEST_SPEARMAN || test == PS_TEST_CHI2;
  if (!homogeneous && !b) return ps_fail(PS_ERR_INVALID, "mixed test needs a second matrix");
  const bool presort_a = test == PS_TEST_SPEARMAN;
  const bool presort_b = test == PS_TEST_MWU || test == PS_TEST_KRUSKAL;
  ps_matrix* ma = nullptr;
  ps_matrix* mb = nullptr;
  bool any_adj = adj_outs && (adj_outs[0] || adj_outs[1] || adj_outs[2]);
  const bool any_out = any_adj || (outs && (outs[0] || outs[1] || outs[2] || outs[3]));
  if (!a || a->n_features <= 0 || (!homogeneous && b->n_features <= 0))
    return ps_fail(PS_ERR_INVALID, "expected a non-empty matrix");
  // device outputs first: incremental kernels may write them during the upload
  const int64_t rows = a->n_features, cols = homogeneous ? a->n_features : b->n_features;
  const int64_t cells = rows * cols;
  double* d_out[4] = {nullptr, nullptr, nullptr, nullptr};
  auto free_outs = [&]() {
    for (int k = 0; k < 4; ++k) ps_free(d_out[k], s);
  };
  for (int k = 0; k < 4 && !rc; ++k) {
    const bool want = (outs && outs[k]) || (k == 1 && any_adj);
    if (!want) continue;
    if (ps_alloc(&d_out[k], (size_t)cells, s) != cudaSuccess) rc = ps_fail(PS_ERR_CUDA, "out of device memory");
    if (!rc) rc = ps_fill_nan(d_out[k], cells, s);
  }
  if (rc) {
    free_outs();
    return rc;
  }
  // Spearman: the walk over columns h < r1 starts as soon as rows [0, r1) are
  // uploaded and presorted, overlapping the rest of the upload
  // jobs allocate on the main stream (one stream for every large allocation
  // keeps the memory pool reusing its blocks from run to run); the auxiliary
  // stream then waits for those allocations
  auto after_alloc = [&](cudaStream_t aux) -> int {
    PS_CUDA(cudaEventRecord(st->alloc_ev, s));
    PS_CUDA(cudaStreamWaitEvent(aux, st->alloc_ev, 0));
    return PS_OK;
  };
  // Pearson: the tile columns of the uploaded rows
  ps_pearson_job* pjob = nullptr;
  RowsHook pearson_hook = [&](ps_matrix* m, int64_t r1, cudaStream_t aux) -> int {
    if (!pjob) {
      int c = ps_pearson_begin(m, d_out[0], d_out[1], d_out[2], s, &pjob);
      if (!c) c = after_alloc(aux);
      if (c) return c;
    }
    return ps_pearson_upto(pjob, r1, aux);
  };
  ps_spearman_job* sjob = nullptr;
  RowsHook walk_hook = [&](ps_matrix* m, int64_t r1, cudaStream_t aux) -> int {
    if (!sjob) {
      int c = ps_spearman_begin(m, 0, m->F, d_out[0], d_out[1], d_out[2], s, &sjob);
      if (!c) c = after_alloc(aux);
      if (c) return c;
    }
    return ps_spearman_walk_upto(sjob, r1, aux);
  };
  g_tl.mark("start", s);
  const bool no_overlap = getenv("PS_NO_OVERLAP") != nullptr;
  const bool overlap = test == PS_TEST_SPEARMAN && any_out && !no_overlap && !ps_spearman_wide(a->n_samples);
  // (only when the tile triangle alone fills the GPU: small matrices keep the
  // split-K whole-matrix launch)
  const int64_t nt_p = (rows + 63) / 64;
  const bool overlap_pearson =
      test == PS_TEST_PEARSON && any_out && !no_overlap && nt_p * (nt_p + 1) / 2 >= 8LL * st->num_sms;
  rc = matrix_create(a, 0, presort_a, s, &ma, overlap ? &walk_hook : overlap_pearson ? &pearson_hook : nullptr);
  // Mann-Whitney / Kruskal-Wallis: likewise, per uploaded chunk of features
  ps_rank_job* rjob = nullptr;
  RowsHook rank_hook = [&](ps_matrix* m, int64_t r1, cudaStream_t aux) -> int {
    if (!rjob) {
      int c = ps_rank_mixed_begin(test, ma, m, 0, m->F, test == PS_TEST_MWU ? u_mode : 0, s, &rjob);
      if (!c) c = after_alloc(aux);
      if (c) return c;
    }
    return ps_rank_mixed_walk_upto(rjob, r1, aux);
  };
  const bool overlap_rank = (test == PS_TEST_MWU || test == PS_TEST_KRUSKAL) && any_out && !getenv("PS_NO_OVERLAP");
  // ANOVA / t-test: the moment contraction of each uploaded chunk's columns
  ps_group_job* gjob = nullptr;
  RowsHook group_hook = [&](ps_matrix* m, int64_t r1, cudaStream_t aux) -> int {
    if (!gjob) {
      int c = ps_group_moment_begin(test, ma, m, test == PS_TEST_TTEST ? (t_variant == 0) : 1, s, &gjob);
      if (!c) c = after_alloc(aux);
      if (c) return c;
    }
    return ps_group_moment_upto(gjob, r1, aux);
  };
  const bool overlap_group = (test == PS_TEST_ANOVA || test == PS_TEST_TTEST) && any_out && !getenv("PS_NO_OVERLAP");
  if (!rc && !homogeneous)
    rc = matrix_create(b, 0, presort_b, s, &mb, overlap_rank ? &rank_hook : overlap_group ? &group_hook : nullptr);
  if (rc) {
    ps_pearson_abort(pjob, s);
    ps_spearman_abort(sjob, s);
    ps_rank_mixed_abort(rjob, s);
    ps_group_moment_abort(gjob, s);
    ps_matrix_destroy(ma);
    ps_matrix_destroy(mb);
    free_outs();
    return rc;
  }
  tr.mark("matrices");
  bool stat_early = false;  // the statistic matrices are final before the p-values
  if (!rc) {
    switch (test) {
      case PS_TEST_PEARSON:
        if (pjob) {
          rc = ps_pearson_end(pjob, s, st->stat_ev);
          stat_early = !rc;
          pjob = nullptr;
        } else {
          rc = ps_pearson_run(ma, 0, rows, d_out[0], d_out[1], d_out[2], s);
        }
        break;
      case PS_TEST_SPEARMAN:
        if (sjob) {
          rc = ps_spearman_end(sjob, s);
          sjob = nullptr;
        } else {
          rc = ps_spearman_run(ma, 0, rows, d_out[0], d_out[1], d_out[2], s);
        }
        break;
      case PS_TEST_CHI2: rc = ps_chi2_run(ma, 0, rows, d_out[0], d_out[1], d_out[2], d_out[3], s); break;
      case PS_TEST_TTEST:
      case PS_TEST_ANOVA:
        if (gjob) {
          rc = ps_group_moment_end(gjob, d_out[0], d_out[1], d_out[2], s);
          gjob = nullptr;
        } else {
          rc = ps_group_moment_run(test, ma, mb, 0, cells, test == PS_TEST_TTEST ? (t_variant == 0) : 1, d_out[0],
                                   d_out[1], d_out[2], s);
        }
        break;
      case PS_TEST_MWU:
      case PS_TEST_KRUSKAL:
        if (rjob) {
          rc = ps_rank_mixed_end(rjob, d_out[0], d_out[1], d_out[2], s);
          rjob = nullptr;
        } else {
          rc = ps_rank_mixed_run(test, ma, mb, 0, cols, test == PS_TEST_MWU ? u_mode : 0, d_out[0], d_out[1],
                                 d_out[2], s);
        }
        break;
      default: rc = ps_fail(PS_ERR_INVALID, "unknown test");
    }
  }
  if (pjob) ps_pearson_abort(pjob, s);  // not consumed (an earlier failure)
  if (sjob) ps_spearman_abort(sjob, s);
  if (rjob) ps_rank_mixed_abort(rjob, s);
  if (gjob) ps_group_moment_abort(gjob, s);
  // while the device computes: fault in the host output pages
  if (!rc && !getenv("PS_NO_PREFAULT")) {
    for (int k = 0; k < 4; ++k)
      if (outs && outs[k]) ps_host_prefault(outs[k], sizeof(double) * cells);
    for (int k = 0; k < 3; ++k)
      if (adj_outs && adj_outs[k]) ps_host_prefault(adj_outs[k], sizeof(double) * cells);
  }
  // Pearson: r (and r^2) are final before the p-value pass; their D2H runs
  // on a walk stream while the device evaluates the p-values
  bool early[4] = {false, false, false, false};
  if (!rc && stat_early && outs) {
    void* hd[2];
    const void* ds_[2];
    size_t nb[2];
    for (int q = 0; q < 2; ++q) {
      const int k = q ? 2 : 0;
      hd[q] = outs[k];
      ds_[q] = d_out[k];
      nb[q] = outs[k] && d_out[k] ? sizeof(double) * cells : 0;
      early[k] = nb[q] != 0;
    }
    cudaError_t e = cudaStreamWaitEvent(st->walk[0], st->stat_ev, 0);
    rc = e != cudaSuccess ? ps_cuda_check(e, "stat handoff") : ps_stage_d2h_many(2, hd, ds_, nb, st->walk[0]);
    g_tl.mark("stat d2h done", st->walk[0]);
  }
  if (!rc) rc = drain_errors(s);
  g_tl.mark("compute done", s);
  tr.mark("compute");
  // The p-value adjustments run on the auxiliary stream, driven by a helper
  // thread (the adjust path reads sizes back to the host), while this thread
  // stages the raw matrices to the host; the adjusted matrices follow.
  double* d_adjk[3] = {nullptr, nullptr, nullptr};
  int rc_adj = PS_OK;
  std::string adj_error;
  std::thread adj_thread;
  if (!rc && any_adj) {
    for (int k = 0; k < 3 && !rc; ++k)
      if (adj_outs[k] && ps_alloc(&d_adjk[k], (size_t)cells, s) != cudaSuccess)
        rc = ps_fail(PS_ERR_CUDA, "out of device memory");
    if (!rc) {
      cudaError_t e = cudaEventRecord(st->aux_ev, s);  // p (and the buffers) are ready
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st->aux, st->aux_ev, 0);
      if (e != cudaSuccess) rc = ps_cuda_check(e, "adjust handoff");
    }
    if (!rc) {
      const int dev = st->device;
      adj_thread = std::thread([&, dev] {
        cudaSetDevice(dev);
        for (int k = 0; k < 3 && rc_adj == PS_OK; ++k)
          if (adj_outs[k]) rc_adj = ps_adjust_run(d_out[1], rows, cols, k, homogeneous ? 1 : 0, d_adjk[k], st->aux);
        if (rc_adj) adj_error = g_last_error;  // thread_local: hand the message to the caller's thread
      });
    }
  }
  if (!rc && outs) {
    void* hd[4];
    const void* ds_[4];
    size_t nb[4];
    for (int k = 0; k < 4; ++k) {
      hd[k] = outs[k];
      ds_[k] = d_out[k];
      nb[k] = outs[k] && d_out[k] && !early[k] ? sizeof(double) * cells : 0;
    }
    rc = ps_stage_d2h_many(4, hd, ds_, nb, s);
  }
  tr.mark("d2h");
  if (adj_thread.joinable()) {
    adj_thread.join();
    // whatever happened, the main stream (which frees p, the adjusted buffers
    // and the adjust scratch) is ordered after everything issued on aux
    cudaError_t e = cudaEventRecord(st->aux_ev, st->aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, st->aux_ev, 0);
    if (e != cudaSuccess) cudaStreamSynchronize(st->aux);
    if (!rc && e != cudaSuccess) rc = ps_cuda_check(e, "adjust join");
  }
  if (!rc && rc_adj) rc = ps_fail(rc_adj, adj_error);
  if (!rc && any_adj) {
    {
      void* hd[3];
      const void* ds_[3];
      size_t nb[3];
      for (int k = 0; k < 3; ++k) {
        hd[k] = adj_outs[k];
        ds_[k] = d_adjk[k];
        nb[k] = adj_outs[k] && d_adjk[k] ? sizeof(double) * cells : 0;
      }
      rc = ps_stage_d2h_many(3, hd, ds_, nb, s);
    }
  }
  tr.mark("adjust");
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = ps_cuda_check(e, "run");
  }
  g_tl.mark("end", s);
  g_tl.dump();
  for (int k = 0; k < 3; ++k) ps_free(d_adjk[k], s);
  for (int k = 0; k < 4; ++k) ps_free(d_out[k], s);

  ps_matrix_destroy(ma);
  ps_matrix_destroy(mb);
  if (rc) cudaStreamSynchronize(s);
  return rc;
}

// Pageable host rows -> device rows through the pinned all-core staging ring
// (multi-GPU: each rank uploads its own shard of the input); the device
// padding columns [width, dpitch) are zeroed.  Returns once the host buffer
// may be reused (the last DMA may still be in flight on `stream`).
int ps_copy_h2d_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t rows,
                   void* stream) {
  Guard g;
  int rc = ensure_state();
  if (rc) return rc;
  if (rows <= 0 || width <= 0) return PS_OK;
  if (!dst || !src || dpitch < width || spitch < width) return ps_fail(PS_ERR_INVALID, "bad copy geometry");
  cudaStream_t s = as_stream(stream);
  rc = ps_stage_h2d_2d(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)rows, s);
  if (!rc && dpitch > width)
    PS_CUDA(cudaMemset2DAsync(static_cast<char*>(dst) + width, (size_t)dpitch, 0, (size_t)(dpitch - width),
                              (size_t)rows, s));
  return rc;
}

int ps_adjust(const double* p, int64_t rows, int64_t cols, int method, int symmetric, double* out) {
  Guard g;
  int rc = ensure_state();
  if (rc) return rc;
  cudaStream_t s = ps_state()->stream;
  const int64_t n = rows * cols;
  double* dp = nullptr;
  double* dout = nullptr;
  if (ps_alloc(&dp, (size_t)std::max<int64_t>(n, 1), s) != cudaSuccess ||
      ps_alloc(&dout, (size_t)std::max<int64_t>(n, 1), s) != cudaSuccess)
    return ps_fail(PS_ERR_CUDA, "out of device memory");
  cudaError_t e = cudaMemcpyAsync(dp, p, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) rc = ps_cuda_check(e, "adjust upload");
  if (!rc) rc = ps_adjust_run(dp, rows, cols, method, symmetric, dout, s);
  if (!rc) {
    e = cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) rc = ps_cuda_check(e, "adjust download");
  }
  cudaStreamSynchronize(s);
  ps_free(dp, s);
  ps_free(dout, s);
  return rc;
}

}  // extern "C"
