// Device-side building blocks shared by the kernel translation units.
#pragma once

#include "sfb_common.cuh"

#define SFB_MAX_K 8

namespace sfb {

template <typename T>
struct CV {
  const T* c[3];
};
template <typename T>
struct MV {
  T* c[3];
};
// Body force: per-component constants f, or per-DOF fields a (extended
// arrays, sample_force of a callable, operators.py:241-259); a[c] == NULL
// means the constant.  Added after diffusion (operators.py:228-235).
template <typename T>
struct Force {
  T f[3];
  const T* a[3];
  const T* c[3];  // closure term (stage kernels): added after the force
};
template <typename T>
struct KList {
  const T* k[SFB_MAX_K][3];
  T coef[SFB_MAX_K];
};

// Momentum RHS of component ``a`` at extended linear index x (coords I),
// accumulated onto ``v`` in the reference's order: all convection terms
// (b = 0..D-1, operators.py:181-214), then all diffusion terms
// (operators.py:150-169), then the constant force (operators.py:228-235).
// Reads ghosts from memory (callers guarantee filled ghosts).
template <typename T, int D>
__device__ __forceinline__ T rhs_comp(const Geo<T>& G, const CV<T>& U, long long x, const int I[3], int a, T v,
                                      bool conv, bool diff, T nu, T fa) {
  const T* __restrict__ ua = U.c[a];
  const T uc = ua[x];
  T up[3], um[3];
#pragma unroll
  for (int b = 0; b < D; ++b) {
    up[b] = ua[x + G.s[b]];
    um[b] = ua[x - G.s[b]];
  }
  if (conv) {
#pragma unroll
    for (int b = 0; b < D; ++b) {
      const T tp = (uc + up[b]) * T(0.5);
      const T tm = (um[b] + uc) * T(0.5);
      T fl;
      if (b == a) {
        fl = (tp * tp - tm * tm) * tab(G, a, T_RDU, I[a]);
      } else {
        const T* __restrict__ ub = U.c[b];
        const T wl = tab(G, a, T_WLO, I[a]);
        const T wh = tab(G, a, T_WHI, I[a]);
        const long long sa = G.s[a], sb = G.s[b];
        const T vp = ub[x] * wl + ub[x + sa] * wh;
        const T vm = ub[x - sb] * wl + ub[x - sb + sa] * wh;
        fl = (tp * vp - tm * vm) * tab(G, b, T_RDX, I[b]);
      }
      v -= fl;
    }
  }
  if (diff) {
#pragma unroll
    for (int b = 0; b < D; ++b) {
      T khi, klo;
      if (b == a) {
        khi = tab(G, a, T_OHI, I[a]);
        klo = tab(G, a, T_OLO, I[a]);
      } else {
        khi = tab(G, b, T_THI, I[b]);
        klo = tab(G, b, T_TLO, I[b]);
      }
      v += nu * ((up[b] - uc) * khi - (uc - um[b]) * klo);
    }
  }
  if (fa != T(0)) v += fa;
  return v;
}

// u_a at I and I - e_a along its own axis with boundary entries resolved
// inline (what fill_ghosts_velocity would have written, fields.py:110-133)
template <typename T, int D>
__device__ __forceinline__ void own_pair(const Geo<T>& G, const T* __restrict__ ua, long long x, const int I[3], int a,
                                         T& cur, T& prev) {
  const int n = G.n[a];
  if (G.halo[a]) {
    cur = ua[x];
    prev = ua[x - G.s[a]];  // ghost plane supplied by the neighbouring slab
  } else if (G.per[a]) {
    cur = ua[x];
    prev = I[a] == 1 ? ua[x + (long long)(n - 1) * G.s[a]] : ua[x - G.s[a]];
  } else {
    cur = I[a] == n ? (G.bc_hi[a] == SFB_BC_DIRICHLET ? G.vhi[a][a] : T(0)) : ua[x];
    prev = I[a] == 1 ? (G.bc_lo[a] == SFB_BC_DIRICHLET ? G.vlo[a][a] : T(0)) : ua[x - G.s[a]];
  }
}

template <typename T>
int launch_planes(const Geo<T>& G, MV<T> U, int ncomp, int mode, cudaStream_t st);

}  // namespace sfb

#define SFB_TYPED(p, CALL)                                             \
  ((p)->dtype == SFB_F64 ? ([&]() { using T = double; return CALL; })() \
                         : ([&]() { using T = float; return CALL; })())
