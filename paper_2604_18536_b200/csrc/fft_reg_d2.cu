// Register-FFT engine instantiations (double; see sfb_fft_reg.cuh).
#include "sfb_fft_reg.cuh"

namespace sfb {

int reg_tu_d2_init() { return reg_upload_tables(); }

int reg_tu_d2(int L, const RegCall& c, cudaStream_t st) {
  switch (L) {
    case 16: return reg_launch<double, 4, 4>(c, st);
    case 20: return reg_launch<double, 4, 5>(c, st);
    case 24: return reg_launch<double, 4, 6>(c, st);
    case 32: return reg_launch<double, 4, 8>(c, st);
    case 40: return reg_launch<double, 5, 8>(c, st);
    case 48: return reg_launch<double, 6, 8>(c, st);
    case 64: return reg_launch<double, 8, 8>(c, st);
    case 96: return reg_launch<double, 8, 12>(c, st);
    case 128: return reg_launch<double, 8, 16>(c, st);
    case 192: return reg_launch<double, 12, 16>(c, st);
    case 384: return reg_launch<double, 16, 24>(c, st);
    default: return -1;
  }
}

}  // namespace sfb
