// ps_specfun_eval.cu -- batch evaluation of the device special functions
// (ps_specfun.cuh) for the golden-grid tests: the same functions the pair
// epilogues inline, evaluated on the device and copied back.
#include "ps_internal.cuh"
#include "ps_specfun.cuh"

namespace {

__global__ void specfun_kernel(int which, const double* __restrict__ args, int64_t n, int nargs,
                               double* __restrict__ out, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = args + i * nargs;
    double r = PS_NAN;
    switch (which) {
      case 0: r = psf::ln_gamma(a[0], err); break;
      case 1: r = psf::reg_inc_beta(a[0], a[1], a[2], err); break;
      case 2: r = psf::reg_inc_gamma_upper(a[0], a[1], err); break;
      case 3: r = psf::normal_sf(a[0]); break;
      case 4: r = psf::t_sf(a[0], a[1], err); break;
      case 5: r = psf::chi2_sf(a[0], a[1], err); break;
      case 6: r = psf::f_sf(a[0], a[1], a[2], err); break;
      case 7: r = psf::beta_sym_sf(a[0], a[1], err); break;
      default: ps_raise(err, PS_ERR_INVALID);
    }
    out[i] = r;
  }
}

}  // namespace

extern "C" int ps_specfun_eval(int which, const double* args, int64_t n, int nargs, double* out) {
  ps_device_state* st = ps_state();
  if (st->device < 0) {
    int rc = ps_set_device(0);
    if (rc) return rc;
    st = ps_state();
  }
  cudaStream_t s = st->stream;
  double *da = nullptr, *dout = nullptr;
  PS_CUDA(ps_alloc(&da, (size_t)(n * nargs + 1), s));
  PS_CUDA(ps_alloc(&dout, (size_t)(n + 1), s));
  PS_CUDA(cudaMemcpyAsync(da, args, sizeof(double) * n * nargs, cudaMemcpyHostToDevice, s));
  specfun_kernel<<<(unsigned)ps_ceil_div(n, 128) + 1, 128, 0, s>>>(which, da, n, nargs, dout, st->d_err);
  PS_LAUNCHED();
  PS_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  ps_free(da, s);
  ps_free(dout, s);
  return ps_sync(s);
}
