// The reference's pluggable real-FFT backend (transforms.py:9-12: rfftn /
// irfftn over every axis of a contiguous array) on the GPU.  Shapes whose
// axes factor into 2/3/5/7 with an even last axis run the hand-written
// engine (fft.cu / sfb_fft_reg.cuh); anything else goes to cuFFT.  Like
// scipy.fft, irfftn is normalised by 1/N and leaves its input untouched.
#include <cufft.h>

#include "sfb_fft.cuh"
#include "sfb_kernels.cuh"

struct sfb_fft {
  int dim = 0;
  int n[3] = {1, 1, 1};
  bool f64 = true;
  long long total = 0, ncomplex = 0;
  sfb::FftSolve F;
  cufftHandle fwd = 0, inv = 0;
  bool has_fwd = false, has_inv = false;
  void* scratch = nullptr;  // complex copy of the irfftn input
};

namespace sfb {
namespace {

int cufft_ok(cufftResult r, const char* what) {
  if (r == CUFFT_SUCCESS) return SFB_OK;
  return fail(SFB_ECUDA, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

template <typename T>
__global__ void k_scale(T* __restrict__ x, long long n, T s) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    x[t] *= s;
}

// the hand-written engine covers this shape (same admission as the
// spectral solver's setup_fft, poisson.cu)
int setup_own(sfb_fft* f) {
  FftSolve& F = f->F;
  const size_t csz = f->f64 ? 16 : 8;
  const int dim = f->dim, nlast = f->n[dim - 1];
  if (getenv("SFB_TRANSFORMS_CUFFT")) return SFB_OK;
  if (nlast % 2 != 0 || nlast < 4) return SFB_OK;
  FftLen half, ax[3];
  if (!fft_factor(nlast / 2, half) || 2 * (size_t)(nlast / 2) * csz > 200 * 1024) return SFB_OK;
  for (int a = 0; a < dim - 1; ++a)
    if (!fft_factor(f->n[a], ax[a]) || 2 * (size_t)f->n[a] * csz > 200 * 1024) return SFB_OK;
  int rc;
  if ((rc = (f->f64 ? fft_set_smem_limits<double>() : fft_set_smem_limits<float>()))) return rc;
  F.dim = dim;
  for (int a = 0; a < 3; ++a) F.n[a] = f->n[a];
  F.total = f->total;
  F.half = half;
  for (int a = 0; a < dim - 1; ++a) {
    F.ax[a] = ax[a];
    if ((rc = fft_upload_pass_twiddles(F.ax[a], f->f64, &F.tw_ax[a]))) return rc;
  }
  if ((rc = fft_upload_pass_twiddles(F.half, f->f64, &F.tw_half))) return rc;
  if ((rc = fft_upload_twiddles(nlast, f->f64, &F.tw_full))) return rc;
  fft_reg_assign(F);
  F.enabled = true;
  return SFB_OK;
}

int setup_cufft(sfb_fft* f) {
  int nn[3];
  for (int a = 0; a < f->dim; ++a) nn[a] = f->n[a];
  int rc;
  if ((rc = cufft_ok(cufftPlanMany(&f->fwd, f->dim, nn, nullptr, 1, 0, nullptr, 1, 0, f->f64 ? CUFFT_D2Z : CUFFT_R2C, 1),
                     "plan rfftn")))
    return rc;
  f->has_fwd = true;
  if ((rc = cufft_ok(cufftPlanMany(&f->inv, f->dim, nn, nullptr, 1, 0, nullptr, 1, 0, f->f64 ? CUFFT_Z2D : CUFFT_C2R, 1),
                     "plan irfftn")))
    return rc;
  f->has_inv = true;
  return SFB_OK;
}

template <typename T>
int run_forward(sfb_fft* f, const void* in, void* out, cudaStream_t st) {
  if (f->F.enabled) return fft_forward<T>(f->F, (const T*)in, out, st);
  int rc;
  if ((rc = cufft_ok(cufftSetStream(f->fwd, st), "stream"))) return rc;
  if (f->f64) return cufft_ok(cufftExecD2Z(f->fwd, (cufftDoubleReal*)in, (cufftDoubleComplex*)out), "D2Z");
  return cufft_ok(cufftExecR2C(f->fwd, (cufftReal*)in, (cufftComplex*)out), "R2C");
}

template <typename T>
int run_inverse(sfb_fft* f, const void* in, void* out, cudaStream_t st) {
  // both backends overwrite the complex input: work on a copy
  const size_t cb = (size_t)f->ncomplex * 2 * sizeof(T);
  int rc;
  if ((rc = cuda_check(cudaMemcpyAsync(f->scratch, in, cb, cudaMemcpyDeviceToDevice, st), "irfftn input copy")))
    return rc;
  if (f->F.enabled) {
    if ((rc = fft_inverse<T>(f->F, f->scratch, (T*)out, st))) return rc;
  } else {
    if ((rc = cufft_ok(cufftSetStream(f->inv, st), "stream"))) return rc;
    if (f->f64)
      rc = cufft_ok(cufftExecZ2D(f->inv, (cufftDoubleComplex*)f->scratch, (cufftDoubleReal*)out), "Z2D");
    else
      rc = cufft_ok(cufftExecC2R(f->inv, (cufftComplex*)f->scratch, (cufftReal*)out), "C2R");
    if (rc) return rc;
  }
  k_scale<T><<<148 * 4, 256, 0, st>>>((T*)out, f->total, (T)(1.0 / (double)f->total));
  SFB_LAUNCH_CHECK("irfftn normalisation");
  return SFB_OK;
}

}  // namespace
}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_fft_create(int dim, const int* n, int dtype, sfb_fft** out) {
  if (!n || !out) return fail(SFB_EINVAL, "null argument");
  *out = nullptr;
  if (dim < 1 || dim > 3) return fail(SFB_EINVAL, "rfftn: dimension must be 1, 2 or 3");
  if (dtype != SFB_F64 && dtype != SFB_F32) return fail(SFB_EINVAL, "rfftn: unknown dtype");
  sfb_fft* f = new sfb_fft();
  f->dim = dim;
  f->f64 = dtype == SFB_F64;
  f->total = 1;
  for (int a = 0; a < dim; ++a) {
    if (n[a] < 1) {
      delete f;
      return fail(SFB_EINVAL, "rfftn: extents must be positive");
    }
    f->n[a] = n[a];
    f->total *= n[a];
  }
  f->ncomplex = f->total / n[dim - 1] * (n[dim - 1] / 2 + 1);
  const size_t esz = f->f64 ? 8 : 4;
  int rc = cuda_check(cudaMalloc(&f->scratch, 2 * esz * (size_t)f->ncomplex), "cudaMalloc(rfftn scratch)");
  if (!rc) rc = setup_own(f);
  if (!rc && !f->F.enabled) rc = setup_cufft(f);
  if (rc) {
    sfb_fft_destroy(f);
    return rc;
  }
  *out = f;
  return SFB_OK;
}

int sfb_fft_destroy(sfb_fft* f) {
  if (!f) return SFB_OK;
  if (f->has_fwd) cufftDestroy(f->fwd);
  if (f->has_inv) cufftDestroy(f->inv);
  cudaFree(f->scratch);
  for (int a = 0; a < 3; ++a) cudaFree(f->F.tw_ax[a]);
  cudaFree(f->F.tw_half);
  cudaFree(f->F.tw_full);
  delete f;
  return SFB_OK;
}

int sfb_fft_uses_own(const sfb_fft* f) { return f && f->F.enabled ? 1 : 0; }

int sfb_rfftn(sfb_fft* f, const void* in, void* out, void* stream) {
  SFB_RANGE();
  if (!f || !in || !out) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  return f->f64 ? run_forward<double>(f, in, out, st) : run_forward<float>(f, in, out, st);
}

int sfb_irfftn(sfb_fft* f, const void* in, void* out, void* stream) {
  SFB_RANGE();
  if (!f || !in || !out) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  return f->f64 ? run_inverse<double>(f, in, out, st) : run_inverse<float>(f, in, out, st);
}

}  // extern "C"
