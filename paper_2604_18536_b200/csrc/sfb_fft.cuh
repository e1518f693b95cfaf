// Hand-written FFT engine (fft.cu) declarations.
#pragma once

#include <cuda.h>

#include "sfb_common.cuh"

namespace sfb {

struct FftLen {
  int L;          // complex transform length
  int np;         // number of Stockham passes
  int radix[12];  // radices in pass order
  int twoff[12];  // offset of each pass's twiddle table (after the plain table)
  int twn;        // total twiddle entries (plain + per-pass)
};

struct ScaleArgs {
  int dim;
  int nh;                     // half-spectrum extent of the last axis (3D column split)
  const double *l0, *l1, *l2; // per-axis eigenvalue tables (fp64)
  double invN;                // 1 / (n0 n1 n2): the irfftn normalisation
  int zero_ok;                // this chunk holds the k = 0 mode (zeroed)
  int tlog;                   // > 0: tiled spectrum (fft.cu): batch = k2 block of 2^tlog
                              // columns, column = k1 * 2^tlog + k2 % 2^tlog
};

// TMA description of one strided pass: a (2W x Lb [x batch]) box over the
// complex buffer viewed as reals; nbox boxes cover the transform length.
struct FftTma {
  CUtensorMap map;
  int rank = 0, nbox = 0, lb = 0, ncol = 0, nbatch = 0;
  bool ok = false;
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
  FftTma tma_ax1, tma_ax0;  // TMA maps of the axis-1 and axis-0 passes (3D)
  // register-resident engine (sfb_fft_reg.cuh) per pass, when instantiated
  int reg_half = 0, reg_ax[3] = {0, 0, 0};  // 0 = Stockham engine, else L
  int reg_a_half = 0, reg_b_half = 0, reg_a[3] = {0, 0, 0}, reg_b[3] = {0, 0, 0};
  // tiled half spectrum of the 3D solve (r2c_epilogue in sfb_fft_reg.cuh):
  // blocks of 2^tlog columns, block stride tks; 0 = natural layout
  int tlog = 0;
  long long tks = 0;
  // hybrid layout (default): the row passes keep the natural spectrum, the
  // axis-1 passes copy it to / from this tiled buffer, the axis-0 pass runs
  // on it in place (solver-owned; null = all passes on the tiled cbuf)
  void* tbuf = nullptr;
};

bool fft_factor(int L, FftLen& P);
// choose the register engine for every pass whose length is instantiated
void fft_reg_assign(FftSolve& F);
// column width of the register engine's strided kernels for length L (fft_reg.cu)
int reg_strided_w(int L, bool f64);
int fft_upload_twiddles(int L, bool f64, void** dev);
int fft_upload_pass_twiddles(FftLen& P, bool f64, void** dev);
// Spectral solve in place on rbuf.  When G/u are given, the right-hand side
// is the divergence of u, computed inside the first (R2C) pass.
// gradt: the right-hand side is -G^T(u)/W instead (the projection pullback)
template <typename T>
int fft_solve_inplace(FftSolve& F, T* rbuf, void* cbuf, cudaStream_t st, const Geo<T>* G = nullptr,
                      const void* const* u = nullptr, int gradt = 0);
template <typename T>
int fft_set_smem_limits();
// unnormalised real transforms of a contiguous array (fft.cu): forward
// R2C + C2C passes; inverse overwrites its complex input
template <typename T>
int fft_forward(FftSolve& F, const T* in, void* out, cudaStream_t st);
template <typename T>
int fft_inverse(FftSolve& F, void* in, T* out, cudaStream_t st);
// channel solve (fft.cu): R2C along z (of the divergence when G/u given,
// walls on y resolved inline) + forward FFT along x; inverse x + C2R; the
// tridiagonal solve along y runs between them (poisson.cu)
template <typename T>
int fft_channel_forward(FftSolve& F, const T* rbuf, void* cbuf, cudaStream_t st, const Geo<T>* G,
                        const void* const* u);
template <typename T>
int fft_channel_inverse(FftSolve& F, void* cbuf, T* rbuf, cudaStream_t st);
template <typename T>
bool fft_channel_divfuse_ok(const FftSolve& F, const Geo<T>& G);
// the register engine can fuse the divergence of u into the R2C pass
template <typename T>
bool fft_divfuse_ok(const FftSolve& F, const Geo<T>& G);
bool fft_tma_fits(int L, bool f64);
int fft_tma_make(FftTma& M, void* base, bool f64, int rank, long long inner_complex, long long rows, long long batch,
                 int L);
template <typename T, int MODE>
int fft_tma_pass(const FftTma& M, const FftLen& P, const void* tw, const ScaleArgs& sc, cudaStream_t st);
// slab-decomposed pieces (multi-GPU, fft.cu): R2C (divergence fused when
// G/u given), axis-1 FFT of a column chunk into / out of the all-to-all
// layout, axis-0 solve of a column chunk, C2R
template <typename T>
int fft_slab_r2c(FftSolve& F, T* rbuf, void* cbuf, cudaStream_t st, const Geo<T>* G, const void* const* u);
template <typename T>
int fft_slab_axis1(FftSolve& F, void* cbuf, void* xbuf, int nranks, int k, int K, bool inverse, cudaStream_t st);
template <typename T>
int fft_slab_axis0(FftSolve& F, void* tbuf, int n1_chunk, int nranks, int k, int K, cudaStream_t st);
template <typename T>
int fft_slab_c2r(FftSolve& F, void* cbuf, T* rbuf, cudaStream_t st);

}  // namespace sfb
