// Hand-written FFT engine (fft.cu) declarations.
#pragma once

#include "sfb_common.cuh"

namespace sfb {

struct FftLen {
  int L;          // complex transform length
  int np;         // number of Stockham passes
  int radix[12];  // radices in pass order
  int twoff[12];  // offset of each pass's twiddle table (after the plain table)
};

struct ScaleArgs {
  int dim;
  int nh;                     // half-spectrum extent of the last axis (3D column split)
  const double *l0, *l1, *l2; // per-axis eigenvalue tables (fp64)
  double invN;                // 1 / (n0 n1 n2): the irfftn normalisation
  int zero_ok;                // this chunk holds the k = 0 mode (zeroed)
};

struct FftSolve {
  bool enabled = false;
  int dim = 0;
  int n[3] = {1, 1, 1};
  long long total = 0;
  FftLen half{};       // length n_last/2 (real trick)
  FftLen ax[3]{};      // strided axes
  void* tw_half = nullptr;
  void* tw_full = nullptr;  // exp(-2 pi i k / n_last), k < n_last
  void* tw_ax[3] = {nullptr, nullptr, nullptr};
  ScaleArgs sc{};
};

bool fft_factor(int L, FftLen& P);
int fft_upload_twiddles(int L, bool f64, void** dev);
int fft_upload_pass_twiddles(FftLen& P, bool f64, void** dev);
// Spectral solve in place on rbuf.  When G/u are given, the right-hand side
// is the divergence of u, computed inside the first (R2C) pass.
template <typename T>
int fft_solve_inplace(FftSolve& F, T* rbuf, void* cbuf, cudaStream_t st, const Geo<T>* G = nullptr,
                      const void* const* u = nullptr);
template <typename T>
int fft_set_smem_limits();
template <typename T>
int fft_slab_forward(FftSolve& F, T* rbuf, void* cbuf, cudaStream_t st);
template <typename T>
int fft_slab_axis0(FftSolve& F, void* tbuf, int n1_chunk, cudaStream_t st);
template <typename T>
int fft_slab_inverse(FftSolve& F, void* cbuf, T* rbuf, cudaStream_t st);

}  // namespace sfb
