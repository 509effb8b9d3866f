// Latency of a dependent fp64 add chain (the exact-replay loops of
// ps_group.cu / ps_pearson.cu are such chains): one thread, N adds.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o dadd_chain dadd_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* __restrict__ x, int n, double* out, long long* cyc) {
  __shared__ double buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = x[i];
  __syncthreads();
  if (threadIdx.x) return;
  double sum = 0.0, ssq = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < n; r += 1024) {
    for (int i = 0; i < 1024; i += 4) {
      const double v0 = buf[i], v1 = buf[i + 1], v2 = buf[i + 2], v3 = buf[i + 3];
      sum += v0; ssq += v0 * v0; sum += v1; ssq += v1 * v1;
      sum += v2; ssq += v2 * v2; sum += v3; ssq += v3 * v3;
    }
  }
  long long t1 = clock64();
  out[0] = sum + ssq;
  cyc[0] = t1 - t0;
}

__global__ void chain_reg(int n, double a, double* out, long long* cyc) {
  double sum = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) sum += a;
  long long t1 = clock64();
  out[0] = sum;
  cyc[0] = t1 - t0;
}

int main() {
  double *x, *out;
  long long* cyc;
  cudaMalloc(&x, 1024 * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 1.0 + i * 1e-3;
  cudaMemcpy(x, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 1 << 20;
  long long c;
  chain_reg<<<1, 1>>>(n, 1.000001, out, cyc);
  chain_reg<<<1, 1>>>(n, 1.000001, out, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dadd_chain_cycles_per_add\": %.2f, ", (double)c / n);
  chain<<<1, 32>>>(x, n, out, cyc);
  chain<<<1, 32>>>(x, n, out, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("\"replay_loop_cycles_per_value\": %.2f}\n", (double)c / n);
  return 0;
}
