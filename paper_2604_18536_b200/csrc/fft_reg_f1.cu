// Register-FFT engine instantiations (float; see sfb_fft_reg.cuh).
#include "sfb_fft_reg.cuh"

namespace sfb {

int reg_tu_f1_init() { return reg_upload_tables(); }

int reg_tu_f1(int L, const RegCall& c, cudaStream_t st) {
  switch (L) {
    case 840: return reg_launch<float, 28, 30>(c, st);
    case 420: return reg_launch<float, 20, 21>(c, st);
    case 512: return reg_launch<float, 16, 32>(c, st);
    case 256: return reg_launch<float, 16, 16>(c, st);
    case 1024: return reg_launch<float, 32, 32>(c, st);
    case 1680: return reg_launch<float, 40, 42>(c, st);
    default: return -1;
  }
}

}  // namespace sfb
