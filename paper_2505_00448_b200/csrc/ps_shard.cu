// ps_shard.cu -- the p-value exchange of the multi-GPU path.
//
// The reference adjusts one family per matrix (adjust.py:23-87): the strict
// upper triangle of a symmetric result, every cell of a mixed one.  When the
// pairs are sharded over GPUs by the reference's partitions (engine.py:70-125:
// triangle rows, flat cells, continuous features), each rank packs the family
// cells of ITS range into a dense vector, the ranks all-gather the vectors
// (NCCL), every rank adjusts the whole family on its device and unpacks its
// own segment back into its rows.  The same pack / all-gather / unpack with
// the diagonal included assembles full raw result matrices on every rank.  Homogeneous ranges are contiguous segments
// of the row-major upper triangle, so the concatenation is the reference's
// own family order; BH / BY / Bonferroni do not depend on the order anyway
// (tied p get identical adjusted values).  Bytes moved per rank: 8 per owned
// family cell -- half of an all-reduce of dense matrices.
#include "ps_internal.cuh"
#include <algorithm>

namespace {

enum Layout { kTriangle = 0, kFlat = 1, kColumns = 2 };

int layout_of(int test) {
  if (test == PS_TEST_PEARSON || test == PS_TEST_SPEARMAN || test == PS_TEST_CHI2) return kTriangle;
  if (test == PS_TEST_TTEST || test == PS_TEST_ANOVA) return kFlat;
  return kColumns;
}

// first packed index of triangle row g for a range starting at lo; a row
// holds the cells h > g (d = 0, the adjustment family) or h >= g (d = 1, raw
// outputs with their self-test diagonal)
__host__ __device__ __forceinline__ int64_t tri_row_offset(int64_t g, int64_t lo, int64_t F, int d) {
  // sum_{r=lo}^{g-1} (F - 1 + d - r)
  const int64_t k = g - lo;
  return k * (F - 1 + d - lo) - k * (k - 1) / 2;
}

// one CTA (grid-stride) per triangle row; threads over the row's cells
__global__ void tri_pack_kernel(const double* __restrict__ mat, int64_t F, int64_t lo, int64_t hi, int d,
                                double* __restrict__ vec) {
  for (int64_t g = lo + blockIdx.x; g < hi; g += gridDim.x) {
    const int64_t off = tri_row_offset(g, lo, F, d) - (g + 1 - d);
    const double* row = mat + g * F;
    for (int64_t h = g + 1 - d + threadIdx.x; h < F; h += blockDim.x) vec[off + h] = row[h];
  }
}

__global__ void tri_unpack_kernel(const double* __restrict__ vec, int64_t F, int64_t lo, int64_t hi, int d,
                                  double* __restrict__ mat) {
  for (int64_t g = lo + blockIdx.x; g < hi; g += gridDim.x) {
    const int64_t off = tri_row_offset(g, lo, F, d) - (g + 1 - d);
    if (!d && threadIdx.x == 0) mat[g * F + g] = PS_NAN;  // adjusted matrices blank the diagonal
    for (int64_t h = g + 1 - d + threadIdx.x; h < F; h += blockDim.x) {
      const double v = vec[off + h];
      mat[g * F + h] = v;
      mat[h * F + g] = v;
    }
  }
}

// flat cells [lo, hi) (ttest / anova) and column blocks (mwu / kruskal):
// index i of the packed vector <-> cell
__device__ __forceinline__ int64_t cell_of(int layout, int64_t i, int64_t cols, int64_t lo, int64_t hi) {
  if (layout == kFlat) return lo + i;
  const int64_t w = hi - lo;
  return (i / w) * cols + lo + i % w;
}

__global__ void cells_pack_kernel(int layout, const double* __restrict__ mat, int64_t cols, int64_t lo,
                                  int64_t hi, int64_t n, double* __restrict__ vec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    vec[i] = mat[cell_of(layout, i, cols, lo, hi)];
}

__global__ void cells_unpack_kernel(int layout, const double* __restrict__ vec, int64_t cols, int64_t lo,
                                    int64_t hi, int64_t n, double* __restrict__ mat) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mat[cell_of(layout, i, cols, lo, hi)] = vec[i];
}

int check_range(int test, int64_t rows, int64_t cols, int64_t* lo, int64_t* hi) {
  if (test < 0 || test > 6) return ps_fail(PS_ERR_INVALID, "unknown test");
  if (rows < 0 || cols < 0) return ps_fail(PS_ERR_INVALID, "negative shape");
  const int L = layout_of(test);
  if (L == kTriangle && rows != cols) return ps_fail(PS_ERR_NON_SQUARE, "homogeneous results are square");
  const int64_t units = L == kTriangle ? rows : L == kFlat ? rows * cols : cols;
  *lo = std::max<int64_t>(0, std::min(*lo, units));
  *hi = std::max<int64_t>(*lo, std::min(*hi, units));
  return PS_OK;
}

int64_t count_cells(int test, int d, int64_t rows, int64_t cols, int64_t lo, int64_t hi) {
  const int L = layout_of(test);
  if (L == kTriangle) return tri_row_offset(hi, lo, cols, d ? 1 : 0);
  if (L == kFlat) return hi - lo;
  return rows * (hi - lo);
}

}  // namespace

extern "C" {

int ps_cells_count(int test, int diag, int64_t rows, int64_t cols, int64_t lo, int64_t hi, int64_t* n) {
  int rc = check_range(test, rows, cols, &lo, &hi);
  if (rc) return rc;
  *n = count_cells(test, diag, rows, cols, lo, hi);
  return PS_OK;
}

int ps_cells_pack(int test, int diag, const double* mat, int64_t rows, int64_t cols, int64_t lo, int64_t hi,
                  double* vec, void* stream) {
  int rc = check_range(test, rows, cols, &lo, &hi);
  if (rc) return rc;
  const int64_t n = count_cells(test, diag, rows, cols, lo, hi);
  if (n == 0) return PS_OK;
  if (!mat || !vec) return ps_fail(PS_ERR_INVALID, "null buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int L = layout_of(test);
  if (L == kTriangle) {
    tri_pack_kernel<<<(unsigned)std::min<int64_t>(hi - lo, 4096), 256, 0, s>>>(mat, cols, lo, hi, diag ? 1 : 0, vec);
  } else {
    cells_pack_kernel<<<(unsigned)std::min<int64_t>(ps_ceil_div(n, 256), 4096), 256, 0, s>>>(L, mat, cols, lo, hi,
                                                                                           n, vec);
  }
  PS_LAUNCHED();
  return PS_OK;
}

int ps_cells_unpack(int test, int diag, const double* vec, int64_t rows, int64_t cols, int64_t lo, int64_t hi,
                    double* mat, void* stream) {
  int rc = check_range(test, rows, cols, &lo, &hi);
  if (rc) return rc;
  const int64_t n = count_cells(test, diag, rows, cols, lo, hi);
  if (!mat || (n && !vec)) return ps_fail(PS_ERR_INVALID, "null buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int L = layout_of(test);
  if (L == kTriangle) {
    if (hi > lo) {
      tri_unpack_kernel<<<(unsigned)std::min<int64_t>(hi - lo, 4096), 256, 0, s>>>(vec, cols, lo, hi, diag ? 1 : 0,
                                                                                    mat);
      PS_LAUNCHED();
    }
  } else if (n) {
    cells_unpack_kernel<<<(unsigned)std::min<int64_t>(ps_ceil_div(n, 256), 4096), 256, 0, s>>>(L, vec, cols, lo,
                                                                                             hi, n, mat);
    PS_LAUNCHED();
  }
  return PS_OK;
}

}  // extern "C"
