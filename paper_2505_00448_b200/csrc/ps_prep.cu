// ps_prep.cu -- one pass over each input matrix on the device: packed validity
// mask (reference present_mask, datamodel.py:86-104), per-feature present
// count and pivot (mean of present values, used to centre the moment
// contractions), and for label kinds the uint8 label codes the contingency /
// group kernels consume.  HBM-bound: reads 8 B/cell once, writes 1/8 B/cell
// of mask (+1 B/cell of codes for labels).
#include "ps_internal.cuh"
#include <math_constants.h>
#include <algorithm>
#include <limits>

namespace {

constexpr int kPrepThreads = 256;
// samples per CTA: a row is split into fixed segments so that a launch over a
// few rows (one upload chunk) still puts several CTAs -- several loads in
// flight -- on every SM.  The segment is a constant, so the pivot's summation
// order (segment partials added in order) never depends on the launch.
constexpr int64_t kPrepSeg = 8192;

// CT: uint8_t codes (0xFE out of range, 0xFF missing), or uint16_t when a
// category count exceeds 254 (0xFFFE / 0xFFFF)
template <typename CT>
__global__ void __launch_bounds__(kPrepThreads)
prep_rows_kernel(const double* __restrict__ vals, int64_t ld, int64_t S, int64_t W,
                 uint64_t sent_bits, int sent_nan, uint32_t* __restrict__ mask,
                 double* __restrict__ center, int32_t* __restrict__ count,
                 // label outputs (nullptr for continuous)
                 const int32_t* __restrict__ cat, CT* __restrict__ codes, int64_t ldc,
                 uint32_t* __restrict__ zero_bits, uint32_t* __restrict__ bad_bits, int64_t f0,
                 double* __restrict__ psum, int32_t* __restrict__ pcnt) {
  const int64_t f = f0 + blockIdx.x;
  const double* row = vals + f * ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cf = cat ? cat[f] : 0;
  const int64_t s_lo = (int64_t)blockIdx.y * kPrepSeg;
  const int64_t s_hi = min(S, s_lo + kPrepSeg);
  double sum = 0.0;
  int cnt = 0;
  // kU rows of the loop's loads in flight per thread (one 8-B load per thread
  // at a time leaves HBM mostly idle); processed in the original order
  constexpr int kU = 8;
  static_assert(kPrepSeg % (kPrepThreads * kU) == 0, "segments hold whole load rounds");
  for (int64_t base0 = s_lo + (int64_t)warp * 32; base0 < s_hi; base0 += (int64_t)kPrepThreads * kU) {
  double vu[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int64_t s = base0 + (int64_t)u * kPrepThreads + lane;
    vu[u] = s < S ? row[s] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int64_t base = base0 + (int64_t)u * kPrepThreads;
    if (base >= S) break;
    const int64_t s = base + lane;
    double v = 0.0;
    bool pres = false;
    if (s < S) {
      v = vu[u];
      pres = ps_is_present(v, sent_bits, sent_nan);
    }
    const uint32_t word = __ballot_sync(PS_FULL, pres);
    if (pres) { sum += v; }
    cnt += pres ? 1 : 0;
    if (codes) {
      CT code = (CT)~(CT)0;
      bool bad = false;
      if (pres) {
        // int(label) in the reference truncates toward zero (categorical.py:87).
        if (v != v || v <= -1.0 || v >= (double)cf) {
          bad = true;
        } else {
          code = (CT)(int)trunc(v);
        }
        if (bad) code = (CT)~(CT)1;
      }
      if (s < S) codes[f * ldc + s] = code;
      const uint32_t zw = __ballot_sync(PS_FULL, pres && v == 0.0);
      const uint32_t bw = __ballot_sync(PS_FULL, bad);
      if (lane == 0) {
        zero_bits[f * W + (base >> 5)] = zw;
        bad_bits[f * W + (base >> 5)] = bw;
      }
    }
    if (lane == 0) mask[f * W + (base >> 5)] = word;
  }
  }
  if (codes && blockIdx.y + 1 == gridDim.y)
    for (int64_t s = S + threadIdx.x; s < ldc; s += kPrepThreads) codes[f * ldc + s] = (CT)~(CT)0;
  // block reduction of (sum, cnt); order is fixed, so the pivot is reproducible.
  __shared__ double ssum[kPrepThreads / 32];
  __shared__ int scnt[kPrepThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(PS_FULL, sum, o);
    cnt += __shfl_xor_sync(PS_FULL, cnt, o);
  }
  if (lane == 0) { ssum[warp] = sum; scnt[warp] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    int c = 0;
    for (int w = 0; w < kPrepThreads / 32; ++w) { t += ssum[w]; c += scnt[w]; }
    if (psum) {  // several segments: partials, folded in order by prep_finish_kernel
      psum[blockIdx.x * gridDim.y + blockIdx.y] = t;
      pcnt[blockIdx.x * gridDim.y + blockIdx.y] = c;
    } else {
      count[f] = c;
      // pivot: any finite value works for centring; use the mean when finite.
      double piv = c > 0 ? t / (double)c : 0.0;
      if (!isfinite(piv)) piv = 0.0;
      center[f] = piv;
    }
  }
}

// Label matrices prepared from fp64 values on the device: presence / zero /
// out-of-range bit words and label codes only (the pivot is unused for
// labels: 0, as for host-staged codes).  Present counts are integer atomics
// (order-free); the caller zeroes count / center of the rows first.
template <typename CT>
__global__ void __launch_bounds__(kPrepThreads, 4)
prep_labels_kernel(const double* __restrict__ vals, int64_t ld, int64_t S, int64_t W, uint64_t sent_bits,
                   int sent_nan, uint32_t* __restrict__ mask, int32_t* __restrict__ count,
                   const int32_t* __restrict__ cat, CT* __restrict__ codes, int64_t ldc,
                   uint32_t* __restrict__ zero_bits, uint32_t* __restrict__ bad_bits, int64_t f0) {
  const int64_t f = f0 + blockIdx.x;
  const double* row = vals + f * ld;
  CT* crow = codes + f * ldc;
  uint32_t* mrow = mask + f * W;
  uint32_t* zrow = zero_bits + f * W;
  uint32_t* brow = bad_bits + f * W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double dcf = (double)cat[f];
  const int64_t s_lo = (int64_t)blockIdx.y * kPrepSeg;
  const int64_t s_hi = min(S, s_lo + kPrepSeg);
  constexpr CT kMiss = (CT)~(CT)0, kBad = (CT)~(CT)1;
  int cnt = 0;  // lane 0: present count of the warp's words
  constexpr int kU = 8;
  for (int64_t base0 = s_lo + (int64_t)warp * 32; base0 < s_hi; base0 += (int64_t)kPrepThreads * kU) {
    double vu[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t s = base0 + (int64_t)u * kPrepThreads + lane;
      vu[u] = s < S ? row[s] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t base = base0 + (int64_t)u * kPrepThreads;
      if (base >= S) break;
      const int64_t s = base + lane;
      const double v = vu[u];
      const bool pres = s < S && ps_is_present(v, sent_bits, sent_nan);
      // int(label) truncates toward zero (categorical.py:87); NaN fails both compares
      const bool ok = pres && v > -1.0 && v < dcf;
      if (s < S) crow[s] = ok ? (CT)(int)v : (pres ? kBad : kMiss);
      const uint32_t word = __ballot_sync(PS_FULL, pres);
      const uint32_t zw = __ballot_sync(PS_FULL, pres && v == 0.0);
      const uint32_t bw = __ballot_sync(PS_FULL, pres && !ok);
      if (lane == 0) {
        const int64_t w = base >> 5;
        mrow[w] = word;
        zrow[w] = zw;
        brow[w] = bw;
        cnt += __popc(word);
      }
    }
  }
  if (blockIdx.y + 1 == gridDim.y)
    for (int64_t s = S + threadIdx.x; s < ldc; s += kPrepThreads) crow[s] = kMiss;
  if (lane == 0 && cnt) atomicAdd(&count[f], cnt);
}

__global__ void prep_finish_kernel(const double* __restrict__ psum, const int32_t* __restrict__ pcnt, int nseg,
                                   int64_t nrows, int64_t f0, int32_t* __restrict__ count,
                                   double* __restrict__ center) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double t = 0.0;
  int c = 0;
  for (int y = 0; y < nseg; ++y) {
    t += psum[r * nseg + y];
    c += pcnt[r * nseg + y];
  }
  count[f0 + r] = c;
  double piv = c > 0 ? t / (double)c : 0.0;
  if (!isfinite(piv)) piv = 0.0;
  center[f0 + r] = piv;
}

// Label matrices staged from the host as codes: presence / out-of-range bit
// words and present counts from the codes (pivot unused for labels: 0).
template <typename CT>
__global__ void __launch_bounds__(kPrepThreads)
label_bits_kernel(const CT* __restrict__ codes, int64_t ldc, int64_t S, int64_t W,
                  uint32_t* __restrict__ mask, uint32_t* __restrict__ bad_bits, int32_t* __restrict__ count,
                  double* __restrict__ center) {
  const int64_t f = blockIdx.x;
  const CT* c = codes + f * ldc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int cnt = 0;
  for (int64_t base = (int64_t)warp * 32; base < S; base += (int64_t)kPrepThreads) {
    const int64_t s = base + lane;
    const CT code = s < S ? c[s] : (CT)~(CT)0;
    const uint32_t word = __ballot_sync(PS_FULL, code != (CT)~(CT)0);
    const uint32_t bw = __ballot_sync(PS_FULL, code == (CT)~(CT)1);
    if (lane == 0) {
      mask[f * W + (base >> 5)] = word;
      bad_bits[f * W + (base >> 5)] = bw;
      cnt += __popc(word);
    }
  }
  __shared__ int scnt[kPrepThreads / 32];
  if (lane == 0) scnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kPrepThreads / 32; ++w) t += scnt[w];
    count[f] = t;
    center[f] = 0.0;
  }
}

__global__ void fill_kernel(double* __restrict__ p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace

int ps_fill_nan(double* p, int64_t n, cudaStream_t s) {
  if (!p || n <= 0) return PS_OK;
  int blocks = (int)std::min<int64_t>(ps_ceil_div(n, 256), (int64_t)ps_state()->num_sms * 16);
  fill_kernel<<<blocks, 256, 0, s>>>(p, n, std::numeric_limits<double>::quiet_NaN());
  PS_LAUNCHED();
  return PS_OK;
}

// Host label matrix -> device codes + bits without a device copy of the values.
int ps_prepare_labels_from_host(ps_matrix* m, const double* src, int64_t src_ld, cudaStream_t s) {
  PS_CUDA(ps_alloc(&m->d_mask, (size_t)(m->F * m->W), s));
  PS_CUDA(ps_alloc(&m->d_center, (size_t)m->F, s));
  PS_CUDA(ps_alloc(&m->d_count, (size_t)m->F, s));
  m->ldc = ps_round_up(m->S + 1, 16);
  PS_CUDA(ps_alloc(&m->d_codes, (size_t)(m->F * m->ldc * m->code_bytes), s));
  PS_CUDA(ps_alloc(&m->d_zero, (size_t)(m->F * m->W), s));
  PS_CUDA(ps_alloc(&m->d_bad, (size_t)(m->F * m->W), s));
  int rc = ps_stage_labels_h2d(src, (size_t)src_ld, m->F, m->S, m->sentinel_bits, m->sentinel_is_nan, m->h_cat,
                               m->d_codes, m->ldc, m->code_bytes, m->d_zero, m->W, s);
  if (rc) return rc;
  if (m->code_bytes == 2)
    label_bits_kernel<uint16_t><<<(unsigned)m->F, kPrepThreads, 0, s>>>(
        reinterpret_cast<const uint16_t*>(m->d_codes), m->ldc, m->S, m->W, m->d_mask, m->d_bad, m->d_count,
        m->d_center);
  else
    label_bits_kernel<uint8_t><<<(unsigned)m->F, kPrepThreads, 0, s>>>(m->d_codes, m->ldc, m->S, m->W, m->d_mask,
                                                                       m->d_bad, m->d_count, m->d_center);
  PS_LAUNCHED();
  return PS_OK;
}

int ps_prepare_alloc(ps_matrix* m, cudaStream_t s) {
  PS_CUDA(ps_alloc(&m->d_mask, (size_t)(m->F * m->W), s));
  PS_CUDA(ps_alloc(&m->d_center, (size_t)m->F, s));
  PS_CUDA(ps_alloc(&m->d_count, (size_t)m->F, s));
  if (m->kind != PS_KIND_CONTINUOUS) {
    m->ldc = ps_round_up(m->S + 1, 16);  // code[S] = 0xFF: sentinel for padded walks
    PS_CUDA(ps_alloc(&m->d_codes, (size_t)(m->F * m->ldc * m->code_bytes), s));
    PS_CUDA(ps_alloc(&m->d_zero, (size_t)(m->F * m->W), s));
    PS_CUDA(ps_alloc(&m->d_bad, (size_t)(m->F * m->W), s));
  }
  return PS_OK;
}

int ps_prepare_rows(ps_matrix* m, int64_t f0, int64_t f1, cudaStream_t s) {
  if (f1 <= f0) return PS_OK;
  const bool labels = m->kind != PS_KIND_CONTINUOUS;
  const int64_t nrows = f1 - f0;
  const int nseg = (int)std::max<int64_t>(1, ps_ceil_div(m->S, kPrepSeg));
  double* psum = nullptr;
  int32_t* pcnt = nullptr;
  const dim3 grid((unsigned)nrows, (unsigned)nseg);
  if (labels) {
    PS_CUDA(cudaMemsetAsync(m->d_count + f0, 0, sizeof(int32_t) * nrows, s));
    PS_CUDA(cudaMemsetAsync(m->d_center + f0, 0, sizeof(double) * nrows, s));
    if (m->code_bytes == 2)
      prep_labels_kernel<uint16_t><<<grid, kPrepThreads, 0, s>>>(
          m->d_vals, m->ld, m->S, m->W, m->sentinel_bits, m->sentinel_is_nan, m->d_mask, m->d_count, m->d_cat,
          reinterpret_cast<uint16_t*>(m->d_codes), m->ldc, m->d_zero, m->d_bad, f0);
    else
      prep_labels_kernel<uint8_t><<<grid, kPrepThreads, 0, s>>>(
          m->d_vals, m->ld, m->S, m->W, m->sentinel_bits, m->sentinel_is_nan, m->d_mask, m->d_count, m->d_cat,
          m->d_codes, m->ldc, m->d_zero, m->d_bad, f0);
    PS_LAUNCHED();
    return PS_OK;
  }
  if (nseg > 1) {
    PS_CUDA(ps_alloc(&psum, (size_t)(nrows * nseg), s));
    PS_CUDA(ps_alloc(&pcnt, (size_t)(nrows * nseg), s));
  }
  if (labels && m->code_bytes == 2)
    prep_rows_kernel<uint16_t><<<grid, kPrepThreads, 0, s>>>(
        m->d_vals, m->ld, m->S, m->W, m->sentinel_bits, m->sentinel_is_nan, m->d_mask, m->d_center, m->d_count,
        m->d_cat, reinterpret_cast<uint16_t*>(m->d_codes), m->ldc, m->d_zero, m->d_bad, f0, psum, pcnt);
  else
    prep_rows_kernel<uint8_t><<<grid, kPrepThreads, 0, s>>>(
        m->d_vals, m->ld, m->S, m->W, m->sentinel_bits, m->sentinel_is_nan, m->d_mask, m->d_center, m->d_count,
        labels ? m->d_cat : nullptr, m->d_codes, m->ldc, m->d_zero, m->d_bad, f0, psum, pcnt);
  PS_LAUNCHED();
  if (nseg > 1) {
    prep_finish_kernel<<<(unsigned)ps_ceil_div(nrows, 128), 128, 0, s>>>(psum, pcnt, nseg, nrows, f0, m->d_count,
                                                                         m->d_center);
    PS_LAUNCHED();
    ps_free(psum, s);
    ps_free(pcnt, s);
  }
  return PS_OK;
}

int ps_prepare_matrix(ps_matrix* m, cudaStream_t s) {
  int rc = ps_prepare_alloc(m, s);
  if (!rc) rc = ps_prepare_rows(m, 0, m->F, s);
  return rc;
}
