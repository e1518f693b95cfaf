// Register-FFT engine instantiations (float; see sfb_fft_reg.cuh).
#include "sfb_fft_reg.cuh"

namespace sfb {

int reg_tu_f2_init() { return reg_upload_tables(); }

int reg_tu_f2(int L, const RegCall& c, cudaStream_t st) {
  switch (L) {
    case 16: return reg_launch<float, 4, 4>(c, st);
    case 20: return reg_launch<float, 4, 5>(c, st);
    case 24: return reg_launch<float, 4, 6>(c, st);
    case 32: return reg_launch<float, 4, 8>(c, st);
    case 40: return reg_launch<float, 5, 8>(c, st);
    case 48: return reg_launch<float, 6, 8>(c, st);
    case 64: return reg_launch<float, 8, 8>(c, st);
    case 96: return reg_launch<float, 8, 12>(c, st);
    case 128: return reg_launch<float, 8, 16>(c, st);
    case 192: return reg_launch<float, 12, 16>(c, st);
    case 384: return reg_launch<float, 16, 24>(c, st);
    default: return -1;
  }
}

}  // namespace sfb
