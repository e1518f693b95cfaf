// Register-FFT engine instantiations (double; see sfb_fft_reg.cuh).
#include "sfb_fft_reg.cuh"

namespace sfb {

int reg_tu_d1_init() { return reg_upload_tables(); }

int reg_tu_d1(int L, const RegCall& c, cudaStream_t st) {
  switch (L) {
    case 840: return reg_launch<double, 28, 30>(c, st);
    case 420: return reg_launch<double, 20, 21>(c, st);
    case 512: return reg_launch<double, 16, 32>(c, st);
    case 256: return reg_launch<double, 16, 16>(c, st);
    case 1024: return reg_launch<double, 32, 32>(c, st);
    case 1680: return reg_launch<double, 40, 42>(c, st);
    default: return -1;
  }
}

}  // namespace sfb
