// Shared-memory bandwidth on one B200 -- the denominator of the SMEM
// rooflines (Spearman / Kruskal-Wallis / Mann-Whitney walks).
//   lds128: conflict-free 16-byte loads (consecutive lanes, consecutive 16 B)
//   lds32 : conflict-free 4-byte loads
//   rnd16 : random 16-bit gathers (the walks' inv_h / R access pattern)
// 148 x 2 CTAs of 1024 threads, best of 5, CUDA events; prints JSON (B/s).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

constexpr int NT = 1024, BUF = 48 * 1024;

template <int ITERS>
__global__ void __launch_bounds__(NT, 2) lds128(uint32_t* out) {
  __shared__ uint4 buf[BUF / 16];
  for (int i = threadIdx.x; i < BUF / 16; i += NT) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 v = buf[(idx + u * NT) & (BUF / 16 - 1)];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    idx += 37;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = 1;
}

template <int ITERS>
__global__ void __launch_bounds__(NT, 2) lds32(uint32_t* out) {
  __shared__ uint32_t buf[BUF / 4];
  for (int i = threadIdx.x; i < BUF / 4; i += NT) buf[i] = i * 2654435761u;
  __syncthreads();
  uint32_t acc = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc ^= buf[(idx + u * NT) & (BUF / 4 - 1)];
    idx += 41;
  }
  if (acc == 0x12345678u) out[0] = 1;
}

template <int ITERS>
__global__ void __launch_bounds__(NT, 2) rnd16(uint32_t* out) {
  __shared__ uint16_t buf[BUF / 2];
  for (int i = threadIdx.x; i < BUF / 2; i += NT) buf[i] = (uint16_t)(i * 40503u);
  __syncthreads();
  uint32_t acc = 0, x = threadIdx.x * 2654435761u + 1u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x = x * 1664525u + 1013904223u;  // independent random index per lane
      acc += buf[(x >> 9) & (BUF / 2 - 1)];
    }
  }
  if (acc == 0x12345678u) out[0] = 1;
}

template <typename K>
static double best_bps(K kern, int blocks, double bytes) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  uint32_t* d;
  cudaMalloc(&d, 64);
  kern<<<blocks, NT>>>(d);
  cudaDeviceSynchronize();
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, NT>>>(d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = bytes / (ms * 1e-3) > best ? bytes / (ms * 1e-3) : best;
  }
  cudaFree(d);
  return best;
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  const int blocks = pr.multiProcessorCount * 2;
  constexpr int IT = 4096;
  const double b128 = best_bps(lds128<IT>, blocks, (double)blocks * NT * IT * 8 * 16);
  const double b32 = best_bps(lds32<IT>, blocks, (double)blocks * NT * IT * 16 * 4);
  const double r16 = best_bps(rnd16<IT>, blocks, (double)blocks * NT * IT * 16 * 2);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"smem_lds128_gbs\": %.1f, \"smem_lds32_gbs\": %.1f, "
         "\"smem_random_u16_gbs\": %.1f}\n",
         pr.multiProcessorCount, clk, b128 / 1e9, b32 / 1e9, r16 / 1e9);
  return 0;
}
