// Hand-written pullback (VJP) kernels, gather form (adjoint.py:114-349).
//
// The reference scatters cotangents through mirrored slices into extended
// buffers and then folds ghosts back onto their fill sources
// (adjoint.py:53-111).  On periodic grids (the only ones the differentiable
// path accepts, adjoint.py:312-316) fill+fold is exactly periodic index
// wrapping, so every pullback here is a *gather*: each output DOF reads the
// cotangent / primal values it depends on (reach +-1 per axis, including the
// (-e_a+e_c) diagonals of the convective pullback) and writes once.  No
// atomics, so results are deterministic run to run.
#include <cstdlib>

#include "sfb_solver.cuh"
#include "sfb_stage.cuh"
#include "sfb_tma.cuh"

namespace sfb {

__device__ __forceinline__ int wr(int i, int n) { return i < 1 ? i + n : (i > n ? i - n : i); }

// read ptr at J + (o0, o1, o2) with periodic wrap
template <typename T, int D>
__device__ __forceinline__ T atw(const Geo<T>& G, const T* __restrict__ p, const int J[3], int o0, int o1, int o2) {
  int K[3] = {wr(J[0] + o0, G.n[0]), wr(J[1] + o1, G.n[1]), D == 3 ? wr(J[2] + o2, G.n[2]) : 0};
  return p[lin<T, D>(G, K)];
}

template <int D>
__device__ __forceinline__ void unit(int ax, int s, int o[3]) {
  o[0] = o[1] = o[2] = 0;
  o[ax] = s;
}

// divergence pullback (adjoint.py:114-128): out_a[J] = pb[J]/dx_a - pb[J+e_a]/dx_a(J_a+1)
template <typename T, int D>
__global__ void k_div_pb(Geo<T> G, const T* __restrict__ pb, MV<T> O, Box B) {
  int J[3];
  if (!box_coords<D>(B, J)) return;
  const long long x = lin<T, D>(G, J);
  const bool dof = is_pdof<T, D>(G, J);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T v = T(0);
    if (dof) {
      int o[3];
      unit<D>(a, 1, o);
      const int jp = wr(J[a] + 1, G.n[a]);
      v = pb[x] * tab(G, a, T_RDX, J[a]) - atw<T, D>(G, pb, J, o[0], o[1], o[2]) * tab(G, a, T_RDX, jp);
    }
    O.c[a][x] = v;
  }
}

// pressure-gradient pullback (adjoint.py:131-145), optional sign and
// 1/weight scaling for the projection pullback, ext or interior output
template <typename T, int D>
__global__ void k_grad_pb(Geo<T> G, CV<T> V, T* __restrict__ out, Box B, T sign, int interior_out, int divw) {
  int J[3];
  if (!box_coords<D>(B, J)) return;
  const bool dof = is_pdof<T, D>(G, J);
  T acc = T(0);
  if (dof) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int o[3];
      unit<D>(a, -1, o);
      const int jm = wr(J[a] - 1, G.n[a]);
      const T tm = atw<T, D>(G, V.c[a], J, o[0], o[1], o[2]) * tab(G, a, T_RDU, jm);
      const T t0 = V.c[a][lin<T, D>(G, J)] * tab(G, a, T_RDU, J[a]);
      acc += tm - t0;
    }
    acc = sign * acc;
    if (divw) {
      // 1 / W as the product of the reciprocal widths (no fp64 division)
      T rw = T(1);
#pragma unroll
      for (int b = 0; b < D; ++b) rw = rw * tab(G, b, T_RDX, J[b]);
      acc = acc * rw;
    }
  }
  if (interior_out) {
    if (!dof) return;
    long long o = (long long)(J[0] - 1) * G.n[1] + (J[1] - 1);
    if (D == 3) o = o * G.n[2] + (J[2] - 1);
    out[o] = acc;
  } else {
    out[lin<T, D>(G, J)] = acc;
  }
}

// diffusion pullback of component a at J (adjoint.py:148-173), gather form
template <typename T, int D>
__device__ __forceinline__ T diff_pb(const Geo<T>& G, const T* __restrict__ va, const int J[3], int a, T nu) {
  T acc = T(0);
  const T vc = va[lin<T, D>(G, J)];
#pragma unroll
  for (int b = 0; b < D; ++b) {
    const int ax = (b == a) ? a : b;
    const int shi = (b == a) ? T_OHI : T_THI, slo = (b == a) ? T_OLO : T_TLO;
    const int jm = wr(J[b] - 1, G.n[b]), jp = wr(J[b] + 1, G.n[b]);
    int om[3], op[3];
    unit<D>(b, -1, om);
    unit<D>(b, 1, op);
    const T vm = atw<T, D>(G, va, J, om[0], om[1], om[2]);
    const T vp = atw<T, D>(G, va, J, op[0], op[1], op[2]);
    acc += vm * tab(G, ax, shi, jm) - vc * (tab(G, ax, shi, J[b]) + tab(G, ax, slo, J[b])) + vp * tab(G, ax, slo, jp);
  }
  return nu * acc;
}

// convective pullback of component c at J (adjoint.py:176-227), gather form.
// Forward: out_a[I] = -sum_b (F_ab[I] - F_ab[I-e_b]) R_ab[I] with
// F_ab = T_ab * V_ab.  Cotangent of F: Fb_ab[K] = lam_ab[K+e_b] - lam_ab[K],
// lam_ab = vbar_a * R_ab.
template <typename T, int D>
__device__ __forceinline__ T conv_pb(const Geo<T>& G, const CV<T>& Vb, const CV<T>& U, const int J[3], int c) {
  T acc = T(0);
  const T* __restrict__ vc = Vb.c[c];
  const T* __restrict__ uc = U.c[c];
  const int nc = G.n[c];
  // (i) a = b = c
  {
    int m[3], p[3];
    unit<D>(c, -1, m);
    unit<D>(c, 1, p);
    const T l_m = atw<T, D>(G, vc, J, m[0], m[1], m[2]) * tab(G, c, T_RDU, wr(J[c] - 1, nc));
    const T l_0 = atw<T, D>(G, vc, J, 0, 0, 0) * tab(G, c, T_RDU, J[c]);
    const T l_p = atw<T, D>(G, vc, J, p[0], p[1], p[2]) * tab(G, c, T_RDU, wr(J[c] + 1, nc));
    const T u_m = atw<T, D>(G, uc, J, m[0], m[1], m[2]);
    const T u_0 = atw<T, D>(G, uc, J, 0, 0, 0);
    const T u_p = atw<T, D>(G, uc, J, p[0], p[1], p[2]);
    acc += (l_p - l_0) * ((u_0 + u_p) * T(0.5)) + (l_0 - l_m) * ((u_m + u_0) * T(0.5));
  }
#pragma unroll
  for (int b = 0; b < D; ++b) {
    if (b == c) continue;
    // (ii) a = c, b != c: transported pair
    {
      const T* __restrict__ ub = U.c[b];
      int m[3], p[3], mc[3];
      unit<D>(b, -1, m);
      unit<D>(b, 1, p);
      mc[0] = m[0];
      mc[1] = m[1];
      mc[2] = m[2];
      mc[c] += 1;  // -e_b + e_c
      int pc[3];
      unit<D>(c, 1, pc);
      const int nb = G.n[b];
      const T l_m = atw<T, D>(G, vc, J, m[0], m[1], m[2]) * tab(G, b, T_RDX, wr(J[b] - 1, nb));
      const T l_0 = atw<T, D>(G, vc, J, 0, 0, 0) * tab(G, b, T_RDX, J[b]);
      const T l_p = atw<T, D>(G, vc, J, p[0], p[1], p[2]) * tab(G, b, T_RDX, wr(J[b] + 1, nb));
      const T wl = tab(G, c, T_WLO, J[c]), wh = tab(G, c, T_WHI, J[c]);
      const T V0 = wl * atw<T, D>(G, ub, J, 0, 0, 0) + wh * atw<T, D>(G, ub, J, pc[0], pc[1], pc[2]);
      const T Vm = wl * atw<T, D>(G, ub, J, m[0], m[1], m[2]) + wh * atw<T, D>(G, ub, J, mc[0], mc[1], mc[2]);
      acc += T(0.5) * ((l_p - l_0) * V0 + (l_0 - l_m) * Vm);
    }
    // (iii) b' = c, a = b != c: transporting component c inside F_ac
    {
      const int a = b;
      const T* __restrict__ va = Vb.c[a];
      const T* __restrict__ ua = U.c[a];
      int pc[3], ma[3], mapc[3];
      unit<D>(c, 1, pc);
      unit<D>(a, -1, ma);
      mapc[0] = ma[0] + pc[0];
      mapc[1] = ma[1] + pc[1];
      mapc[2] = ma[2] + pc[2];
      const T rc0 = tab(G, c, T_RDX, J[c]);
      const T rcp = tab(G, c, T_RDX, wr(J[c] + 1, nc));
      // K = J
      {
        const T fb = atw<T, D>(G, va, J, pc[0], pc[1], pc[2]) * rcp - atw<T, D>(G, va, J, 0, 0, 0) * rc0;
        const T tt = (atw<T, D>(G, ua, J, 0, 0, 0) + atw<T, D>(G, ua, J, pc[0], pc[1], pc[2])) * T(0.5);
        acc += fb * tt * tab(G, a, T_WLO, J[a]);
      }
      // K = J - e_a
      {
        const T fb = atw<T, D>(G, va, J, mapc[0], mapc[1], mapc[2]) * rcp - atw<T, D>(G, va, J, ma[0], ma[1], ma[2]) * rc0;
        const T tt = (atw<T, D>(G, ua, J, ma[0], ma[1], ma[2]) + atw<T, D>(G, ua, J, mapc[0], mapc[1], mapc[2])) * T(0.5);
        acc += fb * tt * tab(G, a, T_WHI, wr(J[a] - 1, G.n[a]));
      }
    }
  }
  return acc;
}

// rhs pullback: out = scale*(conv_pb + diff_pb) [+ out]
template <typename T, int D>
__global__ void __launch_bounds__(256) k_rhs_pb(Geo<T> G, CV<T> Vb, CV<T> U, MV<T> O, Box B, T nu, int conv, int diff,
                                                int accumulate) {
  int J[3];
  if (!box_coords<D>(B, J)) return;
  const long long x = lin<T, D>(G, J);
  const bool dof = is_pdof<T, D>(G, J);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    if (!dof) {
      if (!accumulate) O.c[c][x] = T(0);
      continue;
    }
    T v = T(0);
    if (conv) v += conv_pb<T, D>(G, Vb, U, J, c);
    if (diff) v += diff_pb<T, D>(G, Vb.c[c], J, c, nu);
    if (accumulate) v += O.c[c][x];
    O.c[c][x] = v;
  }
}

// ---------------------------------------------------------------------------
// rhs pullback, 3D marching form: a CTA owns an 8 x 32 (j, k) tile and walks a
// chunk of planes; vbar and the primal u (6 components) stream through a
// 5-slot shared-memory ring whose halo rows / planes are loaded from the
// periodically wrapped source indices (so no ghost values are read).  Same
// arithmetic as conv_pb + diff_pb above.
// ---------------------------------------------------------------------------
#ifndef SFB_PB_TJ
#define SFB_PB_TJ 4
#endif
#ifndef SFB_PB_MINB
#define SFB_PB_MINB 3
#endif
constexpr int kPbTJ = SFB_PB_TJ, kPbTK = 32, kPbRing = 5;
// a field's plane tile in a ring slot: PS values at a 128-byte-aligned stride
// (kPbCS) so every TMA box lands aligned
constexpr int kPbPW = kPbTK + 2, kPbPH = kPbTJ + 2, kPbPS = kPbPW * kPbPH, kPbCS = (kPbPS + 15) / 16 * 16,
              kPbNE = 6 * kPbCS;
constexpr int kPbNT = kPbTJ * kPbTK, kPbNQ = (kPbNE + kPbNT - 1) / kPbNT;

// TMA descriptors of vbar0..2, u0..2: (TK+2) x (TJ+2) x 1 boxes of the
// extended arrays (fp64, ghosts holding the periodic images)
struct alignas(64) PbMaps {
  CUtensorMap m[6];
};

// TMA: every plane tile comes in as six boxes issued by one thread and
// completed on the slot's mbarrier; the halo is read from the ghost layers,
// which the caller fills with the periodic images first.  Otherwise the
// per-element cp.async fill reads the wrapped source indices.
#ifndef SFB_PB_MINB_TMA
#define SFB_PB_MINB_TMA 4  // 128 registers without spills: rhs pullback 3.81 -> 3.41 ms at 512^3
#endif
template <typename T, int ACC, bool TMA = false>
__global__ void __launch_bounds__(kPbNT, TMA ? SFB_PB_MINB_TMA : SFB_PB_MINB) k_rhs_pb_march(Geo<T> G, CV<T> Vb, CV<T> U, MV<T> O, T nu, int diff,
                                                            int chunk, const __grid_constant__ PbMaps M) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);  // [slot][6][CS]: vbar0..2, u0..2
  __shared__ __align__(8) unsigned long long pbar[kPbRing];
  // stencil tables staged in shared memory (wrapped indices, see below):
  // axis 1 per tile row, axis 2 per tile column, axis 0 per plane (two
  // alternating sets of planes i-1, i, i+1)
  T* tbj = ring + kPbRing * kPbNE;      // [SFB_NTAB][kPbPH]
  T* tbk = tbj + SFB_NTAB * kPbPH;      // [SFB_NTAB][kPbPW]
  T* tbi = tbk + SFB_NTAB * kPbPW;      // [2][SFB_NTAB][3]
  const int tk = threadIdx.x, tj = threadIdx.y, tid = tj * kPbTK + tk;
  const int k0 = 1 + blockIdx.x * kPbTK, j0 = 1 + blockIdx.y * kPbTJ;
  const int ib = 1 + blockIdx.z * chunk;
  const int ie = min(ib + chunk, G.n[0] + 1);
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const long long s0 = G.s[0], s1 = G.s[1];
  constexpr int NQ = TMA ? 1 : kPbNQ;
  const T* fsrc[NQ];
  bool fok[NQ];
  if constexpr (!TMA) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = tid + q * kPbNT;
      const int f = e / kPbCS;
      const int r = e - f * kPbCS;
      const int jj = r / kPbPW, kk = r - jj * kPbPW;
      const int gj = wr(j0 - 1 + jj, n1), gk = wr(k0 - 1 + kk, n2);  // periodic wrap of the halo
      fok[q] = e < kPbNE && r < kPbPS;
      const T* base = f < 3 ? Vb.c[f] : U.c[f < 6 ? f - 3 : 0];
      fsrc[q] = base + (fok[q] ? (long long)gj * s1 + gk : 0);
    }
  }
  unsigned yph = 0, ypend = 0;  // per-slot barrier parity / loads in flight (tracked by every thread)
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int b = 0; b < kPbRing; ++b) mbar_init(&pbar[b], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  auto ywait = [&](int slot) {
    if (TMA && ((ypend >> slot) & 1)) {
      mbar_wait(&pbar[slot], (yph >> slot) & 1);
      yph ^= 1u << slot;
      ypend &= ~(1u << slot);
    }
  };
  auto load_plane = [&](int ip, int slot) {
    if (ip < 0 || ip > n0 + 1) return;
    if constexpr (TMA) {
      ypend |= 1u << slot;
      if (tid == 0) {
        T* dst = ring + slot * kPbNE;
        mbar_arm(&pbar[slot], 6u * kPbPS * (unsigned)sizeof(T));
#pragma unroll
        for (int f = 0; f < 6; ++f) tma_load(&M.m[f], 3, dst + f * kPbCS, &pbar[slot], k0 - 1, j0 - 1, ip);
      }
    } else {
      const long long base = (long long)wr(ip, n0) * s0;
      T* dst = ring + slot * kPbNE + tid;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < NQ - 1 || tid + q * kPbNT < kPbNE) cp_async_val(dst + q * kPbNT, fsrc[q] + (fok[q] ? base : 0), fok[q]);
    }
  };
  const int j = j0 + tj, k = k0 + tk;
  const bool inside = j <= n1 && k <= n2;
  for (int e = tid; e < SFB_NTAB * kPbPH; e += kPbNT) {
    const int sl = e / kPbPH, r = e - sl * kPbPH;
    tbj[e] = tab(G, 1, sl, wr(min(j0 - 1 + r, n1 + 1), n1));
  }
  for (int e = tid; e < SFB_NTAB * kPbPW; e += kPbNT) {
    const int sl = e / kPbPW, r = e - sl * kPbPW;
    tbk[e] = tab(G, 2, sl, wr(min(k0 - 1 + r, n2 + 1), n2));
  }


  int sl_m = (ib - 1) % kPbRing;
  load_plane(ib - 1, sl_m);
  load_plane(ib, (sl_m + 1) % kPbRing);
  load_plane(ib + 1, (sl_m + 2) % kPbRing);
  cp_commit();
  load_plane(ib + 2, (sl_m + 3) % kPbRing);
  cp_commit();
  const int c0 = (tj + 1) * kPbPW + (tk + 1);
  long long x = (long long)ib * s0 + (long long)j * s1 + k;
  for (int i = ib; i < ie; ++i, x += s0) {
    if (tid < SFB_NTAB * 3) {
      const int sl = tid / 3, o = tid - sl * 3;
      tbi[((i & 1) * SFB_NTAB + sl) * 3 + o] = tab(G, 0, sl, wr(i - 1 + o, n0));
    }
    T accin[3] = {T(0), T(0), T(0)};
    if (ACC && inside) {
#pragma unroll
      for (int c = 0; c < 3; ++c) accin[c] = O.c[c][x];
    }
    int s1i = sl_m + 1, s2i = sl_m + 2;
    if (s1i >= kPbRing) s1i -= kPbRing;
    if (s2i >= kPbRing) s2i -= kPbRing;
    if (TMA) {
      if (i == ib) {
        ywait(sl_m);
        ywait(s1i);
      }
      ywait(s2i);
      // this thread's reads of the slot refilled below, before the TMA write
      fence_proxy_async_smem();
    } else {
      cp_wait<1>();
    }
    __syncthreads();
    int sl_l = sl_m + 4;
    if (sl_l >= kPbRing) sl_l -= kPbRing;
    load_plane(i + 3, sl_l);
    cp_commit();
    if (inside) {
      const T* P[3] = {ring + sl_m * kPbNE + c0, ring + s1i * kPbNE + c0, ring + s2i * kPbNE + c0};
      // field f at offset (d0, d1, d2), f in 0..2 vbar, 3..5 u
      auto R = [&](int f, int d0, int d1, int d2) -> T { return P[1 + d0][f * kPbCS + d1 * kPbPW + d2]; };
      // table value of axis ax, slot sl at the cell's index + off (wrapped)
      const T* ti = tbi + (i & 1) * SFB_NTAB * 3;
      auto TB = [&](int ax, int sl, int off) -> T {
        if (ax == 0) return ti[sl * 3 + 1 + off];
        if (ax == 1) return tbj[sl * kPbPH + tj + 1 + off];
        return tbk[sl * kPbPW + tk + 1 + off];
      };
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        int ec[3] = {0, 0, 0};
        ec[c] = 1;
        T acc = T(0);
        {  // (i) a = b = c
          const T l_m = R(c, -ec[0], -ec[1], -ec[2]) * TB(c, T_RDU, -1);
          const T l_0 = R(c, 0, 0, 0) * TB(c, T_RDU, 0);
          const T l_p = R(c, ec[0], ec[1], ec[2]) * TB(c, T_RDU, 1);
          const T u_m = R(3 + c, -ec[0], -ec[1], -ec[2]);
          const T u_0 = R(3 + c, 0, 0, 0);
          const T u_p = R(3 + c, ec[0], ec[1], ec[2]);
          acc += (l_p - l_0) * ((u_0 + u_p) * T(0.5)) + (l_0 - l_m) * ((u_m + u_0) * T(0.5));
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if (b == c) continue;
          int eb[3] = {0, 0, 0};
          eb[b] = 1;
          {  // (ii) a = c, b != c
            const T l_m = R(c, -eb[0], -eb[1], -eb[2]) * TB(b, T_RDX, -1);
            const T l_0 = R(c, 0, 0, 0) * TB(b, T_RDX, 0);
            const T l_p = R(c, eb[0], eb[1], eb[2]) * TB(b, T_RDX, 1);
            const T wl = TB(c, T_WLO, 0), wh = TB(c, T_WHI, 0);
            const T V0 = wl * R(3 + b, 0, 0, 0) + wh * R(3 + b, ec[0], ec[1], ec[2]);
            const T Vm = wl * R(3 + b, -eb[0], -eb[1], -eb[2]) + wh * R(3 + b, ec[0] - eb[0], ec[1] - eb[1], ec[2] - eb[2]);
            acc += T(0.5) * ((l_p - l_0) * V0 + (l_0 - l_m) * Vm);
          }
          {  // (iii) transporting component c inside F_ac, a = b
            const int a = b;
            const T rc0 = TB(c, T_RDX, 0);
            const T rcp = TB(c, T_RDX, 1);
            {
              const T fb = R(a, ec[0], ec[1], ec[2]) * rcp - R(a, 0, 0, 0) * rc0;
              const T tt = (R(3 + a, 0, 0, 0) + R(3 + a, ec[0], ec[1], ec[2])) * T(0.5);
              acc += fb * tt * TB(a, T_WLO, 0);
            }
            {
              const T fb = R(a, ec[0] - eb[0], ec[1] - eb[1], ec[2] - eb[2]) * rcp - R(a, -eb[0], -eb[1], -eb[2]) * rc0;
              const T tt = (R(3 + a, -eb[0], -eb[1], -eb[2]) + R(3 + a, ec[0] - eb[0], ec[1] - eb[1], ec[2] - eb[2])) * T(0.5);
              acc += fb * tt * TB(a, T_WHI, -1);
            }
          }
        }
        if (diff) {
          T ad = T(0);
          const T vc = R(c, 0, 0, 0);
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            int eb[3] = {0, 0, 0};
            eb[b] = 1;
            const int shi = (b == c) ? T_OHI : T_THI, slo = (b == c) ? T_OLO : T_TLO;
            const T vm = R(c, -eb[0], -eb[1], -eb[2]);
            const T vp = R(c, eb[0], eb[1], eb[2]);
            ad += vm * TB(b, shi, -1) - vc * (TB(b, shi, 0) + TB(b, slo, 0)) +
                  vp * TB(b, slo, 1);
          }
          acc += nu * ad;
        }
        if (ACC) acc += accin[c];
        O.c[c][x] = acc;
      }
    }
    sl_m = s1i;
  }
  cp_wait<0>();
  // no TMA write may still target this CTA's shared memory when it exits
#pragma unroll
  for (int b = 0; b < kPbRing; ++b) ywait(b);
}

// TMA maps of vbar and u for k_rhs_pb_march (fp64: a (TK+2)-wide fp32 box row
// is not a multiple of 16 bytes); false -> the cp.async fill
template <typename T>
static bool pb_maps(const Geo<T>& G, CV<T> V, CV<T> Uf, PbMaps& M) {
  static const bool off = env_int("SFB_PB_NOTMA") != 0;
  if (sizeof(T) != 8 || off || G.dim != 3) return false;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encode_fn();
  if (!enc) return false;
  const size_t esz = sizeof(T);
  if ((G.s[1] * esz) % 16 || (G.s[0] * esz) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)G.E[2], (cuuint64_t)G.E[1], (cuuint64_t)G.E[0]};
  cuuint64_t strides[2] = {(cuuint64_t)(G.s[1] * esz), (cuuint64_t)(G.s[0] * esz)};
  cuuint32_t box[3] = {(cuuint32_t)kPbPW, (cuuint32_t)kPbPH, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  for (int f = 0; f < 6; ++f) {
    const T* ptr = f < 3 ? V.c[f] : Uf.c[f - 3];
    if (!ptr || ((uintptr_t)ptr % 16)) return false;
    if (enc(&M.m[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)ptr, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// tma: the caller has filled the ghosts of V and Uf with their periodic images
template <typename T>
static int rhs_pb_march(const Geo<T>& G, CV<T> V, CV<T> Uf, MV<T> O, T nu, int diff, int accumulate, cudaStream_t st,
                        const PbMaps* maps = nullptr) {
  const size_t smem = ((size_t)kPbRing * kPbNE + SFB_NTAB * (kPbPH + kPbPW + 6)) * sizeof(T);
  cudaError_t e = ensure_smem((const void*)k_rhs_pb_march<T, 0>, smem);
  if (e == cudaSuccess) e = ensure_smem((const void*)k_rhs_pb_march<T, 1>, smem);
  if (e == cudaSuccess) e = ensure_smem((const void*)k_rhs_pb_march<T, 0, true>, smem);
  if (e == cudaSuccess) e = ensure_smem((const void*)k_rhs_pb_march<T, 1, true>, smem);
  if (e != cudaSuccess) return cuda_check(e, "rhs pullback: shared-memory attribute");
  const int bx = (G.n[2] + kPbTK - 1) / kPbTK, by = (G.n[1] + kPbTJ - 1) / kPbTJ;
  const long long bps = (long long)bx * by;
  // >= ~30 waves of resident CTAs (tail of the last partial wave), chunks of
  // >= 64 planes (stage.cu: the same split)
  long long want = (30LL * 148 * SFB_PB_MINB + bps - 1) / bps;
  if (want > G.n[0] / 64) want = G.n[0] / 64;
  if (want < 1) want = 1;
  int chunk = (int)((G.n[0] + want - 1) / want);
  if (chunk < 16) chunk = 16;
  const int bz = (G.n[0] + chunk - 1) / chunk;
  dim3 grid(bx, by, bz), blk(kPbTK, kPbTJ);
  static const PbMaps none{};
  const PbMaps& M = maps ? *maps : none;
  if (maps && accumulate) k_rhs_pb_march<T, 1, true><<<grid, blk, smem, st>>>(G, V, Uf, O, nu, diff, chunk, M);
  else if (maps) k_rhs_pb_march<T, 0, true><<<grid, blk, smem, st>>>(G, V, Uf, O, nu, diff, chunk, M);
  else if (accumulate) k_rhs_pb_march<T, 1><<<grid, blk, smem, st>>>(G, V, Uf, O, nu, diff, chunk, M);
  else k_rhs_pb_march<T, 0><<<grid, blk, smem, st>>>(G, V, Uf, O, nu, diff, chunk, M);
  SFB_LAUNCH_CHECK("rhs pullback (march)");
  if (!accumulate) return launch_planes<T>(G, O, 3, 2, st);  // non-DOF entries of the output are zero
  return SFB_OK;
}

// projection pullback tail: out_a = vbar_a + D^T(w * s)  (adjoint.py:335-349).
// With Kb (the sub-diagonal reverse sweep): the result r feeds only the next
// stage cotangent kbar = c1 ybar + c2 r (adjoint.py:400-419, the combine of
// step_backward fused here) and the g0 accumulation, so r itself is not stored.
template <typename T, int D>
__global__ void k_proj_pb_tail(Geo<T> G, const T* __restrict__ s, CV<T> Vb, MV<T> O, Box B, MV<T> Acc, CV<T> Yb,
                               T c1, T c2, MV<T> Kb) {
  int J[3];
  if (!box_coords<D>(B, J)) return;
  const long long x = lin<T, D>(G, J);
  if (!is_pdof<T, D>(G, J)) {
    if (O.c[0]) {
#pragma unroll
      for (int a = 0; a < D; ++a) O.c[a][x] = T(0);
    }
    if (Kb.c[0]) {
#pragma unroll
      for (int a = 0; a < D; ++a) Kb.c[a][x] = T(0);
    }
    return;
  }
  auto sbar = [&](const int K[3]) -> T {
    long long o = (long long)(K[0] - 1) * G.n[1] + (K[1] - 1);
    if (D == 3) o = o * G.n[2] + (K[2] - 1);
    T w = T(1);
#pragma unroll
    for (int b = 0; b < D; ++b) w = w * tab(G, b, T_DX, K[b]);
    return s[o] * w;
  };
  const T s0 = sbar(J);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int K[3] = {J[0], J[1], J[2]};
    K[a] = wr(J[a] + 1, G.n[a]);
    const T d = s0 * tab(G, a, T_RDX, J[a]) - sbar(K) * tab(G, a, T_RDX, K[a]);
    const T r = Vb.c[a][x] + d;
    if (O.c[0]) O.c[a][x] = r;
    if (Acc.c[0]) Acc.c[a][x] += r;  // g0 += ybar_j (adjoint.py:414-415)
    if (Kb.c[0]) {
      T v = Yb.c[a][x] * c1;  // k_combine's order: ybar term, then ybar_j term
      v += r * c2;
      Kb.c[a][x] = v;
    }
  }
}

// poisson_solve_transpose (adjoint.py:236-250): W S W^-1.  In: the interior
// of an extended cotangent divided by the pressure volume W (the reference's
// true division, W = dx0*dx1[*dx2] in the grid dtype); out: S's result times
// W on the interior of an extended array, ghosts zero.
template <typename T, int D>
__global__ void k_wconj(Geo<T> G, const T* __restrict__ src, T* __restrict__ dst, Box B, int into_ext) {
  int J[3];
  if (!box_coords<D>(B, J)) return;
  const bool dof = is_pdof<T, D>(G, J);
  long long o = 0;
  T w = T(1);
  if (dof) {
    o = (long long)(J[0] - 1) * G.n[1] + (J[1] - 1);
    if (D == 3) o = o * G.n[2] + (J[2] - 1);
#pragma unroll
    for (int b = 0; b < D; ++b) w = w * tab(G, b, T_DX, J[b]);
  }
  if (into_ext) dst[lin<T, D>(G, J)] = dof ? src[o] * w : T(0);
  else if (dof) dst[o] = src[lin<T, D>(G, J)] / w;
}

template <typename T>
static int solve_transpose(sfb_solver* s, const T* pbar, T* out, cudaStream_t st) {
  const Geo<T>& G = geo<T>(s->plan);
  T* rb = (T*)s->rbuf;
  Box B = int_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_wconj<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, pbar, rb, B, 0)));
  SFB_LAUNCH_CHECK("solve transpose: 1/W");
  if (int rc = solve_inplace<T>(s, rb, st)) return rc;
  Box E = ext_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_wconj<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, rb, out, E, 1)));
  SFB_LAUNCH_CHECK("solve transpose: W");
  return SFB_OK;
}

template <typename T>
static MV<T> mvp(const sfb_plan* p, void* const* u) {
  MV<T> r;
  for (int a = 0; a < 3; ++a) r.c[a] = (a < p->dim && u) ? (T*)u[a] : nullptr;
  return r;
}
template <typename T>
static CV<T> cvp(const sfb_plan* p, const void* const* u) {
  CV<T> r;
  for (int a = 0; a < 3; ++a) r.c[a] = (a < p->dim && u) ? (const T*)u[a] : nullptr;
  return r;
}

static int need_periodic(const sfb_plan* p) {
  if (!p->all_periodic) return fail(SFB_ECONFIG, "the differentiable path supports periodic boundaries only");
  return SFB_OK;
}

template <typename T>
static int project_pb(sfb_solver* s, void* const* vbar, void* const* out, void* const* acc, cudaStream_t st,
                      const void* const* ybar = nullptr, double c1 = 0.0, double c2 = 0.0, void* const* kb = nullptr) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  int rc;
  if ((rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st))) return rc;  // zero_non_dofs(vbar)
  Box B = int_box(G);
  T* rb = (T*)s->rbuf;
  static const bool nofuse = env_int("SFB_NO_PBFUSE") != 0;
  if (s->kind == SFB_SOLVER_SPECTRAL && s->fft.enabled && fft_divfuse_ok<T>(s->fft, G) && !nofuse) {
    // -G^T(vbar)/W formed inside the solve's first (R2C) pass
    if ((rc = fft_solve_inplace<T>(s->fft, rb, s->cbuf, st, &G, (const void* const*)vbar, 1))) return rc;
  } else {
    SFB_DISPATCH_DIM(G.dim, D, (k_grad_pb<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, cvp<T>(p, vbar), rb, B, T(-1), 1, 1)));
    SFB_LAUNCH_CHECK("project pullback: gradient pullback");
    if ((rc = solve_inplace<T>(s, rb, st))) return rc;
  }
  Box E = ext_box(G);
  MV<T> O = out ? mvp<T>(p, out) : MV<T>{{nullptr, nullptr, nullptr}};
  MV<T> Acc = acc ? mvp<T>(p, acc) : MV<T>{{nullptr, nullptr, nullptr}};
  MV<T> Kb = kb ? mvp<T>(p, kb) : MV<T>{{nullptr, nullptr, nullptr}};
  CV<T> Yb = ybar ? cvp<T>(p, ybar) : CV<T>{{nullptr, nullptr, nullptr}};
  SFB_DISPATCH_DIM(G.dim, D, (k_proj_pb_tail<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, rb, cvp<T>(p, vbar), O, E, Acc,
                                                                                          Yb, (T)c1, (T)c2, Kb)));
  SFB_LAUNCH_CHECK("project pullback: divergence pullback");
  return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

static bool okp(const sfb_plan* p, const void* const* u) {
  if (!u) return false;
  for (int a = 0; a < p->dim; ++a)
    if (!u[a]) return false;
  return true;
}

extern "C" {

int sfb_divergence_pullback(sfb_plan* p, void* pbar, void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !pbar || !okp(p, out)) return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(p)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    int rc = launch_planes<T>(G, MV<T>{{(T*)pbar, nullptr, nullptr}}, 1, 3, st);  // zero_ghosts_scalar(pbar)
    if (rc) return rc;
    Box E = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_div_pb<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, (const T*)pbar, mvp<T>(p, out), E)));
    SFB_LAUNCH_CHECK("divergence pullback");
    return (int)SFB_OK;
  })());
}

int sfb_pressure_gradient_pullback(sfb_plan* p, void* const* vbar, void* out, void* stream) {
  SFB_RANGE();
  if (!p || !okp(p, vbar) || !out) return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(p)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    int rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st);  // zero_non_dofs(vbar)
    if (rc) return rc;
    Box E = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_grad_pb<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, cvp<T>(p, vbar), (T*)out, E, T(1), 0, 0)));
    SFB_LAUNCH_CHECK("gradient pullback");
    return (int)SFB_OK;
  })());
}

int sfb_diffusion_pullback(sfb_plan* p, void* const* vbar, double nu, void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !okp(p, vbar) || !okp(p, out)) return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(p)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    int rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st);
    if (rc) return rc;
    Box E = ext_box(G);
    CV<T> V = cvp<T>(p, (const void* const*)vbar);
    SFB_DISPATCH_DIM(G.dim, D, (k_rhs_pb<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, V, V, mvp<T>(p, out), E, (T)nu, 0, 1, 0)));
    SFB_LAUNCH_CHECK("diffusion pullback");
    return (int)SFB_OK;
  })());
}

int sfb_convection_pullback(sfb_plan* p, void* const* vbar, const void* const* u, void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !okp(p, vbar) || !okp(p, u) || !okp(p, out)) return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(p)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    int rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st);
    if (rc) return rc;
    Box E = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_rhs_pb<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, cvp<T>(p, (const void* const*)vbar), cvp<T>(p, u), mvp<T>(p, out), E, T(0), 1, 0, 0)));
    SFB_LAUNCH_CHECK("convection pullback");
    return (int)SFB_OK;
  })());
}

int sfb_rhs_pullback(sfb_plan* p, void* const* vbar, const void* const* u, double nu, void* const* out, double scale,
                     int accumulate, void* stream) {
  SFB_RANGE();
  if (!p || !okp(p, vbar) || !okp(p, u) || !okp(p, out)) return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(p)) return rc;
  if (scale != 1.0) return fail(SFB_EINVAL, "scale must be 1 (reserved)");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    static const bool pb_generic = env_int("SFB_PB_GENERIC") != 0;
    PbMaps maps;
    if (G.dim == 3 && !pb_generic &&
        pb_maps<T>(G, cvp<T>(p, (const void* const*)vbar), cvp<T>(p, u), maps)) {
      // TMA tiles read the halo from the ghost layers: periodic images of
      // vbar and u first (the primal's refill is the reference's own,
      // adjoint.py:189); vbar's ghosts are zeroed afterwards, as the
      // reference leaves them (adjoint.py:119-136 zero_non_dofs)
      int rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 0, st);
      if (!rc) rc = launch_planes<T>(G, mvp<T>(p, (void* const*)u), p->dim, 0, st);
      if (!rc) rc = rhs_pb_march<T>(G, cvp<T>(p, (const void* const*)vbar), cvp<T>(p, u), mvp<T>(p, out), (T)nu,
                                    nu != 0.0, accumulate, st, &maps);
      if (!rc) rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st);
      return rc;
    }
    int rc = launch_planes<T>(G, mvp<T>(p, vbar), p->dim, 2, st);
    if (rc) return rc;
    if (G.dim == 3 && !pb_generic)
      return rhs_pb_march<T>(G, cvp<T>(p, (const void* const*)vbar), cvp<T>(p, u), mvp<T>(p, out), (T)nu, nu != 0.0,
                             accumulate, st);
    Box E = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_rhs_pb<T, D><<<box_grid(D, E), box_block(D), 0, st>>>(G, cvp<T>(p, (const void* const*)vbar), cvp<T>(p, u), mvp<T>(p, out), E, (T)nu, 1, nu != 0.0, accumulate)));
    SFB_LAUNCH_CHECK("rhs pullback");
    return (int)SFB_OK;
  })());
}

int sfb_solve_transpose(sfb_solver* s, const void* pbar, void* out, void* stream) {
  SFB_RANGE();
  if (!s || !pbar || !out) return fail(SFB_EINVAL, "null argument");
  if (s->slab) return fail(SFB_ECONFIG, "solve transpose: not available on a slab solver");
  return s->plan->dtype == SFB_F64 ? solve_transpose<double>(s, (const double*)pbar, (double*)out, (cudaStream_t)stream)
                                   : solve_transpose<float>(s, (const float*)pbar, (float*)out, (cudaStream_t)stream);
}

int sfb_project_pullback(sfb_solver* s, void* const* vbar, void* const* out, void* stream) {
  SFB_RANGE();
  return sfb_project_pullback_ex(s, vbar, out, nullptr, stream);
}

int sfb_project_pullback_ex(sfb_solver* s, void* const* vbar, void* const* out, void* const* acc, void* stream) {
  SFB_RANGE();
  if (!s || !okp(s->plan, vbar)) return fail(SFB_EINVAL, "null argument");
  if (out && !okp(s->plan, out)) return fail(SFB_EINVAL, "bad out");
  if (acc && !okp(s->plan, acc)) return fail(SFB_EINVAL, "bad acc");
  if (!out && !acc) return fail(SFB_EINVAL, "project pullback needs out or acc");
  if (int rc = need_periodic(s->plan)) return rc;
  return s->plan->dtype == SFB_F64 ? project_pb<double>(s, vbar, out, acc, (cudaStream_t)stream)
                                   : project_pb<float>(s, vbar, out, acc, (cudaStream_t)stream);
}

int sfb_project_pullback_kb(sfb_solver* s, void* const* vbar, void* const* acc, const void* const* ybar, double c1,
                            double c2, void* const* kb, void* stream) {
  SFB_RANGE();
  if (!s || !okp(s->plan, vbar) || !okp(s->plan, acc) || !okp(s->plan, ybar) || !okp(s->plan, kb))
    return fail(SFB_EINVAL, "null argument");
  if (int rc = need_periodic(s->plan)) return rc;
  return s->plan->dtype == SFB_F64
             ? project_pb<double>(s, vbar, nullptr, acc, (cudaStream_t)stream, ybar, c1, c2, kb)
             : project_pb<float>(s, vbar, nullptr, acc, (cudaStream_t)stream, ybar, c1, c2, kb);
}

}  // extern "C"
