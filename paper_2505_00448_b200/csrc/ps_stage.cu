// ps_stage.cu -- host <-> device copies of pageable (numpy) buffers through a
// pinned, double-buffered staging ring.
//
// run() receives ordinary numpy arrays.  A pageable cudaMemcpy is staged by
// the driver through small bounce buffers on one CPU thread; here the host
// side of each 16 MiB chunk is copied by all host cores (OpenMP) into a pinned
// buffer while the DMA engine moves the previous chunk, so the PCIe link and
// the host copy overlap.  Small transfers go straight to cudaMemcpy.
#include "ps_internal.cuh"
#include <omp.h>
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <vector>

namespace {

// staging chunk (16 MiB measured best: 2-4 MiB chunks pay more per-chunk
// synchronisation than they save in pipeline fill); PS_STAGE_CHUNK_MB overrides
const size_t kChunk = []() -> size_t {
  const char* e = getenv("PS_STAGE_CHUNK_MB");
  const long v = e ? atol(e) : 16;
  return (size_t)std::max(1L, v) << 20;
}();
constexpr size_t kDirect = 4u << 20;  // below this, plain (pageable) copies

struct Ring {
  int device = -1;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t done = nullptr;
};
Ring g_ring[64];

int ring_for_device(Ring** out) {
  int dev = 0;
  PS_CUDA(cudaGetDevice(&dev));
  Ring& r = g_ring[dev];
  if (r.device != dev) {
    for (int b = 0; b < 2; ++b) {
      PS_CUDA(cudaHostAlloc(&r.buf[b], kChunk, cudaHostAllocDefault));
      PS_CUDA(cudaEventCreateWithFlags(&r.ev[b], cudaEventDisableTiming));
    }
    PS_CUDA(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    r.device = dev;
  }
  *out = &r;
  return PS_OK;
}

void par_copy(void* dst, const void* src, size_t bytes) {
  const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(bytes >> 18)));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int t = 0; t < nt; ++t) {
    const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  }
}

// One label row: the per-cell rules of prep_rows_kernel, branch-free so the
// compiler vectorises the code loop (AVX2 clone picked at load time).
template <typename CT>
__attribute__((target_clones("avx2", "default"))) void label_row(const double* row, int64_t S, int64_t W, double cf,
                                                                 uint64_t sent_bits, int sent_nan, CT* crow,
                                                                 uint32_t* zrow) {
  alignas(64) uint8_t zf[32];
  int64_t q0 = 0;
  for (int64_t w = 0; w < W; ++w, q0 += 32) {
    const int64_t len = std::min<int64_t>(S - q0, 32);
    for (int64_t q = 0; q < len; ++q) {
      const double v = row[q0 + q];
      uint64_t bits;
      std::memcpy(&bits, &v, sizeof(bits));
      const bool pres = sent_nan ? (v == v) : (bits != sent_bits);
      const bool ok = (v > -1.0) & (v < cf);  // false for NaN
      const int32_t lab = (int32_t)(ok ? v : 0.0);  // trunc toward zero (categorical.py:87)
      crow[q0 + q] = pres ? (ok ? (CT)lab : (CT)~(CT)1) : (CT)~(CT)0;
      zf[q] = pres & (v == 0.0);
    }
    uint32_t zw = 0;
    for (int64_t q = 0; q < len; ++q) zw |= (uint32_t)zf[q] << q;
    zrow[w] = zw;
  }
}

}  // namespace

// rows x width bytes from host (pitch spitch) to device (pitch dpitch)
int ps_stage_h2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                    cudaStream_t s, const ps_rows_done_fn& on_rows) {
  Ring* r = nullptr;
  int rc = ring_for_device(&r);
  if (rc) return rc;
  if (width * rows < kDirect || dpitch > kChunk) {
    PS_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, s));
    if (on_rows) {
      PS_CUDA(cudaEventRecord(r->done, s));
      return on_rows(0, (int64_t)rows, r->done);
    }
    return PS_OK;
  }
  const size_t rows_per = std::max<size_t>(1, kChunk / dpitch);
  // with a per-chunk consumer, the first chunks are smaller so that device
  // work on the first rows starts sooner (graduated 1/4, 1/4, 1/2, 1, 1 ...)
  auto chunk_rows = [&](int k) -> size_t {
    static const bool flat = getenv("PS_STAGE_FLAT") != nullptr;  // A/B switch
    if (!on_rows || k >= 3 || flat) return rows_per;
    return std::max<size_t>(1, rows_per / (k < 2 ? 4 : 2));
  };
  int b = 0, k = 0;
  for (size_t r0 = 0, nr = 0; r0 < rows; r0 += nr, b ^= 1, ++k) {
    nr = std::min(chunk_rows(k), rows - r0);
    PS_CUDA(cudaEventSynchronize(r->ev[b]));  // the DMA that last read this buffer is done
    char* pb = static_cast<char*>(r->buf[b]);
    const char* sp = static_cast<const char*>(src) + r0 * spitch;
    if (spitch == dpitch && width == dpitch) {
      par_copy(pb, sp, nr * width);
    } else {
      const int nt = std::max(1, std::min(omp_get_max_threads(), (int)nr));
#pragma omp parallel for num_threads(nt) schedule(static)
      for (long long i = 0; i < (long long)nr; ++i) std::memcpy(pb + i * dpitch, sp + i * spitch, width);
    }
    PS_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + r0 * dpitch, pb, nr * dpitch, cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaEventRecord(r->ev[b], s));
    if (on_rows) {
      rc = on_rows((int64_t)r0, (int64_t)nr, r->ev[b]);
      if (rc) return rc;
    }
  }
  return PS_OK;
}

// Label matrices from the host: every core converts its rows of fp64 labels
// into the device layout while staging -- uint8 codes (trunc(label), 0xFE
// present but outside [0, c_f) or NaN, 0xFF missing; padded with 0xFF to ldc)
// and the "present && label == 0.0" bit words -- with the same rules as
// prep_rows_kernel, so only ~1 B per cell crosses PCIe instead of 8.
template <typename CT>
static int stage_labels(const double* src, size_t spitch, int64_t F, int64_t S, uint64_t sent_bits, int sent_nan,
                        const int64_t* cat, CT* d_codes, int64_t ldc, uint32_t* d_zero, int64_t W, cudaStream_t s) {
  Ring* r = nullptr;
  int rc = ring_for_device(&r);
  if (rc) return rc;
  const size_t cb = sizeof(CT);
  const size_t row_bytes = (size_t)ldc * cb + (size_t)W * 4;
  int b = 0;
  if (row_bytes > kChunk) {
    // rows longer than a staging chunk (S of several million): each row in
    // segments of whole 32-sample words, all host cores per segment
    const int64_t seg_words = (int64_t)((kChunk - 256) / (32 * cb + 4));  // + room for the padding past S
    for (int64_t f = 0; f < F; ++f) {
      const double* row = src + (size_t)f * spitch;
      for (int64_t w0 = 0; w0 < W; w0 += seg_words, b ^= 1) {
        const int64_t nw = std::min<int64_t>(seg_words, W - w0);
        const int64_t q0 = w0 * 32, nq = std::min<int64_t>(S - q0, nw * 32);
        PS_CUDA(cudaEventSynchronize(r->ev[b]));
        CT* pc = static_cast<CT*>(r->buf[b]);
        uint32_t* pz = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(pc) + (size_t)seg_words * 32 * cb + 128);
        const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(nw / 1024) + 1));
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int t = 0; t < nt; ++t) {
          const int64_t a0 = nw * t / nt, e = nw * (t + 1) / nt;
          const int64_t qa = a0 * 32, qe = std::min<int64_t>(nq, e * 32);
          if (qe > qa)
            label_row<CT>(row + q0 + qa, qe - qa, e - a0, (double)cat[f], sent_bits, sent_nan, pc + qa, pz + a0);
        }
        // codes of the row's last word past S, and the padding to ldc
        const int64_t ccount = (w0 + nw == W) ? ldc - q0 : nw * 32;
        for (int64_t i = nq; i < ccount; ++i) pc[i] = (CT)~(CT)0;
        PS_CUDA(cudaMemcpyAsync(d_codes + (size_t)f * ldc + q0, pc, (size_t)ccount * cb, cudaMemcpyHostToDevice, s));
        PS_CUDA(cudaMemcpyAsync(d_zero + (size_t)f * W + w0, pz, (size_t)nw * 4, cudaMemcpyHostToDevice, s));
        PS_CUDA(cudaEventRecord(r->ev[b], s));
      }
    }
    return PS_OK;
  }
  const int64_t rows_per = std::max<int64_t>(1, (int64_t)(kChunk / row_bytes));
  for (int64_t r0 = 0; r0 < F; r0 += rows_per, b ^= 1) {
    const int64_t nr = std::min<int64_t>(rows_per, F - r0);
    PS_CUDA(cudaEventSynchronize(r->ev[b]));
    CT* pc = static_cast<CT*>(r->buf[b]);
    uint32_t* pz = reinterpret_cast<uint32_t*>(pc + (size_t)nr * ldc);  // ldc % 16 == 0: aligned
    const int nt = std::max(1, std::min(omp_get_max_threads(), (int)nr));
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t i = 0; i < nr; ++i) {
      const int64_t f = r0 + i;
      label_row<CT>(src + (size_t)f * spitch, S, W, (double)cat[f], sent_bits, sent_nan, pc + (size_t)i * ldc,
                    pz + (size_t)i * W);
      for (int64_t q = S; q < ldc; ++q) pc[(size_t)i * ldc + q] = (CT)~(CT)0;
    }
    PS_CUDA(cudaMemcpyAsync(d_codes + (size_t)r0 * ldc, pc, (size_t)nr * ldc * cb, cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaMemcpyAsync(d_zero + (size_t)r0 * W, pz, (size_t)nr * W * 4, cudaMemcpyHostToDevice, s));
    PS_CUDA(cudaEventRecord(r->ev[b], s));
  }
  return PS_OK;
}

int ps_stage_labels_h2d(const double* src, size_t spitch, int64_t F, int64_t S, uint64_t sent_bits, int sent_nan,
                        const int64_t* cat, uint8_t* d_codes, int64_t ldc, int code_bytes, uint32_t* d_zero,
                        int64_t W, cudaStream_t s) {
  if (code_bytes == 2)
    return stage_labels<uint16_t>(src, spitch, F, S, sent_bits, sent_nan, cat, reinterpret_cast<uint16_t*>(d_codes),
                                  ldc, d_zero, W, s);
  return stage_labels<uint8_t>(src, spitch, F, S, sent_bits, sent_nan, cat, d_codes, ldc, d_zero, W, s);
}

// contiguous device -> host copy; returns after dst is complete
size_t ps_stage_chunk_bytes() { return kChunk; }

// Touch every page of a host output buffer (one write per 4 KiB page, all
// cores) so that first-touch page faults are taken while the device computes,
// not inside the device-to-host copy.  The buffer is about to be overwritten.
void ps_host_prefault(void* dst, size_t bytes) {
  if (!dst || bytes == 0) return;
  char* p = static_cast<char*>(dst);
  const size_t page = 4096;
  const long long n = (long long)((bytes + page - 1) / page);
  const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(n / 256)));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (long long i = 0; i < n; ++i) static_cast<volatile char*>(p)[(size_t)i * page] = 0;
}

int ps_stage_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  void* d[1] = {dst};
  const void* sp[1] = {src};
  size_t b[1] = {bytes};
  return ps_stage_d2h_many(1, d, sp, b, s);
}

// Several device buffers to host memory as one pipeline of sub-chunks: the
// DMA of chunk i + 1 overlaps the host copy of chunk i, across buffers.
int ps_stage_d2h_many(int n, void* const* dst, const void* const* src, const size_t* bytes, cudaStream_t s) {
  struct Piece {
    char* d;
    const char* s;
    size_t len;
  };
  std::vector<Piece> pieces;
  for (int k = 0; k < n; ++k) {
    if (!dst[k] || !src[k] || !bytes[k]) continue;
    if (bytes[k] < kDirect) {
      PS_CUDA(cudaMemcpyAsync(dst[k], src[k], bytes[k], cudaMemcpyDeviceToHost, s));
      continue;
    }
    const size_t piece = std::min(kChunk, std::max<size_t>(2u << 20, bytes[k] / 4));
    for (size_t off = 0; off < bytes[k]; off += piece)
      pieces.push_back({static_cast<char*>(dst[k]) + off, static_cast<const char*>(src[k]) + off,
                        std::min(piece, bytes[k] - off)});
  }
  if (pieces.empty()) {
    PS_CUDA(cudaStreamSynchronize(s));
    return PS_OK;
  }
  Ring* r = nullptr;
  int rc = ring_for_device(&r);
  if (rc) return rc;
  auto issue = [&](size_t i) -> int {
    PS_CUDA(cudaMemcpyAsync(r->buf[i & 1], pieces[i].s, pieces[i].len, cudaMemcpyDeviceToHost, s));
    PS_CUDA(cudaEventRecord(r->ev[i & 1], s));
    return PS_OK;
  };
  rc = issue(0);
  for (size_t i = 0; i < pieces.size() && !rc; ++i) {
    if (i + 1 < pieces.size()) rc = issue(i + 1);  // next piece's DMA overlaps this piece's host copy
    if (rc) break;
    PS_CUDA(cudaEventSynchronize(r->ev[i & 1]));
    par_copy(pieces[i].d, r->buf[i & 1], pieces[i].len);
    // the buffer is reused by piece i + 2, issued after this copy returns
  }
  if (!rc) PS_CUDA(cudaStreamSynchronize(s));  // the direct (small) copies
  return rc;
}
