// Shared pieces of the RK-stage kernels (stage.cu).
#pragma once

#include "sfb_kernels.cuh"

namespace sfb {

template <typename T>
struct StageArgs {
  CV<T> y, u0, s_in;
  MV<T> s_out, y_next, k_out;
  MV<T> u0_out;    // FL_U0P: the projected stage-0 state (u0 == y) is written here
  T cb, ca, nu;
  Force<T> F;
  const T* p_int;  // FL_PROJ: contiguous interior pressure; y is projected on the fly
  int has_s, has_next, has_k, s_from_u0, diff;
};

template <typename T>
__device__ __forceinline__ void cp_async_val(T* smem, const T* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? (int)sizeof(T) : 0;
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Coefficients of one axis at one index (operators.py:47-84 tables).
template <typename T>
struct Coef {
  T rdu, wlo, whi, ohi, olo, rdx, thi, tlo;
};
template <typename T>
__device__ __forceinline__ Coef<T> coef_at(const Geo<T>& G, int axis, int i) {
  Coef<T> c;
  c.rdu = tab(G, axis, T_RDU, i);
  c.wlo = tab(G, axis, T_WLO, i);
  c.whi = tab(G, axis, T_WHI, i);
  c.ohi = tab(G, axis, T_OHI, i);
  c.olo = tab(G, axis, T_OLO, i);
  c.rdx = tab(G, axis, T_RDX, i);
  c.thi = tab(G, axis, T_THI, i);
  c.tlo = tab(G, axis, T_TLO, i);
  return c;
}

// epilogue variants (compile-time): bit 1 k_out, bit 2 s_out, bit 4 s from
// u0 (else s_in), bit 8 y_next
// bit 16: y is unprojected, y - G p is formed in shared memory (all-periodic 3D)
// bit 32: every axis periodic (every interior cell is a DOF of every component):
// branch-free stencil evaluation, stores predicated on the tile bounds only
// bit 64 (with FL_PROJ, u0 == y): u0 is the stage state itself, projected in
// shared memory -- the combines take it from the ring centre and it is
// written once to u0_out (the deferred last projection of the previous step,
// timestep.py:208-210 fused into the next step's first stage)
// bit 128 (with FL_PROJ, u0 != y): the projected stage state (ring centre) is
// written to u0_out -- the VJP tape records it without a gradient-subtract pass
enum { FL_K = 1, FL_S = 2, FL_SU0 = 4, FL_NEXT = 8, FL_PROJ = 16, FL_PER = 32, FL_U0P = 64, FL_YOUT = 128 };



}  // namespace sfb
