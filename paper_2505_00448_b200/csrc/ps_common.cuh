// ps_common.cuh -- shared device/host helpers of the B200 pair engine.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/pairstat_b200.h"

#define PS_WARP 32
#define PS_FULL 0xffffffffu

// Device-side error word: the first non-zero status code wins.  Kernels never
// throw; the host maps the word to the reference's exception classes
// (errors.py) after the stream drains.
__device__ __forceinline__ void ps_raise(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Bit-exact missingness rule of the reference (datamodel.py:86-104).
__device__ __forceinline__ bool ps_is_present(double v, uint64_t sentinel_bits, int sentinel_is_nan) {
  if (sentinel_is_nan) return !(v != v);
  return (uint64_t)__double_as_longlong(v) != sentinel_bits;
}

__host__ __device__ __forceinline__ int64_t ps_ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t ps_round_up(int64_t a, int64_t b) { return ps_ceil_div(a, b) * b; }

// Upper-triangular tile index t -> (I, J), I <= J, row-major over I.
// Row I holds (T - I) tiles.  Solved in closed form then corrected.
__host__ __device__ __forceinline__ void ps_tri_tile(int64_t t, int64_t T, int64_t* I, int64_t* J) {
  // offset(I) = I*T - I*(I-1)/2
  double b = 2.0 * (double)T + 1.0;
  int64_t i = (int64_t)((b - sqrt(b * b - 8.0 * (double)t)) * 0.5);
  if (i < 0) i = 0;
  if (i > T - 1) i = T - 1;
  while (i > 0 && i * T - i * (i - 1) / 2 > t) --i;
  while (i + 1 < T && (i + 1) * T - (i + 1) * i / 2 <= t) ++i;
  *I = i;
  *J = i + (t - (i * T - i * (i - 1) / 2));
}
// column-major upper triangle: tile t -> (I <= J), columns J in order
__host__ __device__ __forceinline__ void ps_tri_tile_cm(int64_t t, int64_t* I, int64_t* J) {
  int64_t j = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (j > 0 && j * (j + 1) / 2 > t) --j;
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  *J = j;
  *I = t - j * (j + 1) / 2;
}
__host__ __device__ __forceinline__ int64_t ps_tri_offset(int64_t I, int64_t T) {
  return I * T - I * (I - 1) / 2;
}

// numpy's NaN bit pattern (0x7ff8000000000000); CUDART_NAN is the negative one.
#define PS_NAN __longlong_as_double(0x7ff8000000000000LL)
