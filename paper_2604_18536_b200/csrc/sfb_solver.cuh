// Pressure solver object (opaque to C callers).
#pragma once

#include <cufft.h>

#include "sfb_common.cuh"
#include "sfb_fft.cuh"

namespace sfb {
template <typename T>
struct CT;
template <>
struct CT<double> {
  typedef double2 type;
};
template <>
struct CT<float> {
  typedef float2 type;
};

template <typename T>
int solve_inplace(sfb_solver* s, T* buf, cudaStream_t st);
// matrix-free CG (cg.cu)
template <typename T>
int cg_solve(sfb_solver* s, T* buf, cudaStream_t st);
int cg_setup(sfb_solver* s);
void cg_release(sfb_solver* s);
}  // namespace sfb

struct sfb_solver {
  sfb_plan* plan = nullptr;
  int kind = 0;
  cufftHandle fwd = 0, inv = 0;
  bool has_fwd = false, has_inv = false;
  void* work = nullptr;
  size_t work_size = 0;
  void* rbuf = nullptr;      // contiguous interior real array (rhs / solution)
  void* cbuf = nullptr;      // half spectrum
  double* cprime = nullptr;  // channel: Thomas c' scratch (fp64)
  double2* dscr = nullptr;   // channel, fp32 plans: fp64 forward-sweep scratch
  double* lam[3] = {nullptr, nullptr, nullptr};
  double *up = nullptr, *lo = nullptr, *di = nullptr, *dxy = nullptr;
  void* tmp = nullptr;       // pullback scratch (extended scalar)
  sfb::FftSolve fft;         // hand-written FFT path (spectral), when supported
  // slab decomposition (multi-GPU)
  bool slab = false;
  int n0g = 0, rank = 0, nranks = 1;
  void* tbuf = nullptr;      // transposed spectrum (n0 global, n1/P, nh); aliases cbuf when P = 1
  void* xbuf = nullptr;      // all-to-all send / receive buffer (P, m, n1/P, nh), P > 1
  // matrix-free CG (SFB_SOLVER_CG)
  double cg_tol = 0.0, cg_wtot = 0.0;
  int cg_max_iter = 0, cg_iters = 0, cg_nb = 0;
  void *cg_x = nullptr, *cg_r = nullptr, *cg_p = nullptr, *cg_ap = nullptr;
  double *cg_part = nullptr, *cg_dsc = nullptr, *cg_hsc = nullptr;
  std::vector<double> cg_hist;
  // device-driven iteration batches (cg.cu): residual history on the device,
  // a captured graph of kCgBatch iterations, the stream it was captured on
  double* cg_dhist = nullptr;
  int cg_dhist_cap = 0;
  void* cg_graph = nullptr;  // cudaGraphExec_t
  void* cg_cap_stream = nullptr;
  bool cg_graph_tried = false;
};
