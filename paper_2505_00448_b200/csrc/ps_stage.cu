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

namespace {

constexpr size_t kChunk = 16u << 20;
constexpr size_t kDirect = 4u << 20;  // below this, plain (pageable) copies

struct Ring {
  int device = -1;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
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
    r.device = dev;
  }
  *out = &r;
  return PS_OK;
}

void par_copy(void* dst, const void* src, size_t bytes) {
  const int nt = std::max(1, std::min(omp_get_max_threads(), (int)(bytes >> 20)));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int t = 0; t < nt; ++t) {
    const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  }
}

}  // namespace

// rows x width bytes from host (pitch spitch) to device (pitch dpitch)
int ps_stage_h2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                    cudaStream_t s) {
  if (width * rows < kDirect || dpitch > kChunk) {
    PS_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, s));
    return PS_OK;
  }
  Ring* r = nullptr;
  int rc = ring_for_device(&r);
  if (rc) return rc;
  const size_t rows_per = std::max<size_t>(1, kChunk / dpitch);
  int b = 0;
  for (size_t r0 = 0; r0 < rows; r0 += rows_per, b ^= 1) {
    const size_t nr = std::min(rows_per, rows - r0);
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
  }
  return PS_OK;
}

// contiguous device -> host copy; returns after dst is complete
int ps_stage_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kDirect) {
    PS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    PS_CUDA(cudaStreamSynchronize(s));
    return PS_OK;
  }
  Ring* r = nullptr;
  int rc = ring_for_device(&r);
  if (rc) return rc;
  const size_t n = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) -> int {
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    PS_CUDA(cudaMemcpyAsync(r->buf[i & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
    PS_CUDA(cudaEventRecord(r->ev[i & 1], s));
    return PS_OK;
  };
  rc = issue(0);
  for (size_t i = 0; i < n && !rc; ++i) {
    if (i + 1 < n) rc = issue(i + 1);  // next chunk's DMA overlaps this chunk's host copy
    if (rc) break;
    PS_CUDA(cudaEventSynchronize(r->ev[i & 1]));
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    par_copy(static_cast<char*>(dst) + off, r->buf[i & 1], len);
    // the buffer is reused by chunk i + 2, issued after this copy returns
  }
  return rc;
}
