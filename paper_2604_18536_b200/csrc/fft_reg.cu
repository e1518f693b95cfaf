// Host dispatch of the register-resident FFT engine (sfb_fft_reg.cuh).
#include <cstdlib>
#include <mutex>

#include "sfb_fft_reg.cuh"

namespace sfb {

// lengths with an instantiated (A, B) engine (fft_reg_{d,f}{1,2}.cu)
bool reg_factor(int L, RegLen& R) {
  static const int tab[][3] = {{840, 28, 30}, {420, 20, 21}, {512, 16, 32}, {256, 16, 16}, {1024, 32, 32},
                               {1680, 40, 42},
                               {16, 4, 4},    {20, 4, 5},    {24, 4, 6},    {32, 4, 8},    {40, 5, 8},
                               {48, 6, 8},    {64, 8, 8},    {96, 8, 12},   {128, 8, 16},  {192, 12, 16},
                               {384, 16, 24}};
  R = RegLen{};
  if (getenv("SFB_FFT_STOCKHAM")) return false;
  for (const auto& e : tab)
    if (e[0] == L) {
      R.L = L;
      R.A = e[1];
      R.B = e[2];
      R.ok = true;
      return true;
    }
  return false;
}

// column width W of the strided kernels of length L (RegGeo<C, A, B>::W)
int reg_strided_w(int L, bool f64) {
  const size_t csz = f64 ? 16 : 8;
  const int w0 = (int)((f64 ? SFB_REG_SEG : SFB_REG_SEG_F32) / csz);
  return (size_t)L * w0 * csz <= 112 * 1024 ? w0 : w0 / 2;
}

int fft_reg_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SFB_ECUDA, "cudaGetDevice");
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev]) return SFB_OK;
  if (reg_tu_d1_init() || reg_tu_d2_init() || reg_tu_f1_init() || reg_tu_f2_init())
    return fail(SFB_ECUDA, "upload of the register-FFT twiddle tables failed");
  if (dev < 64) done[dev] = true;
  return SFB_OK;
}

template <>
int reg_run<double>(const RegLen& R, const RegCall& c, cudaStream_t st) {
  int rc = reg_tu_d1(R.L, c, st);
  if (rc == -1) rc = reg_tu_d2(R.L, c, st);
  if (rc == -1) return fail(SFB_EINVAL, "register FFT: length not instantiated");
  if (rc) return cuda_check(cudaGetLastError(), "register FFT launch");
  return SFB_OK;
}
template <>
int reg_run<float>(const RegLen& R, const RegCall& c, cudaStream_t st) {
  int rc = reg_tu_f1(R.L, c, st);
  if (rc == -1) rc = reg_tu_f2(R.L, c, st);
  if (rc == -1) return fail(SFB_EINVAL, "register FFT: length not instantiated");
  if (rc) return cuda_check(cudaGetLastError(), "register FFT launch");
  return SFB_OK;
}

}  // namespace sfb
