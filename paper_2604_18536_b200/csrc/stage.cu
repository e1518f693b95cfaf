// Fused RK stage: momentum RHS + stage combine in one pass over HBM
// (operators.py:218-238 fused with timestep.py:186-207).
//
// Per velocity DOF:  k = F(y);  [k_out = k];  [s_out = s_in + k*cb];
//                    [y_next = u0 + k*ca]
// Because the reference accumulates acc = u0; acc += k_l*(dt*b_l) in stage
// order (timestep.py:203-207) and every explicit tableau with a single
// sub-diagonal (RK4) builds y_{j+1} = u0 + k_j*(dt*a_{j+1,j}), the running
// sum and the next stage state can be produced while k_j is still in
// registers -- k_j is never stored.  Four velocity registers suffice
// (u0, s, y, y_next), which is what lets 840^3 fp64 fit on one B200.
#include <cstdlib>

#include "sfb_stage.cuh"
#include "sfb_tma.cuh"

namespace sfb {

template <typename T, int D>
__global__ void __launch_bounds__(256) k_stage_generic(Geo<T> G, StageArgs<T> A, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    T k = rhs_comp<T, D>(G, A.y, x, I, a, T(0), true, A.diff, A.nu, A.F.f[a]);
    if (A.F.a[a]) k += A.F.a[a][x];
    if (A.F.c[a]) k += A.F.c[a][x];  // operators.py:236-237
    if (A.has_k) A.k_out.c[a][x] = k;
    if (A.has_s) {
      const T base = A.s_from_u0 ? A.u0.c[a][x] : A.s_in.c[a][x];
      A.s_out.c[a][x] = base + k * A.cb;
    }
    if (A.has_next) A.y_next.c[a][x] = A.u0.c[a][x] + k * A.ca;
  }
}

// ---------------------------------------------------------------------------
// 3D marching kernel: a CTA owns a TJ x TK column tile of the (j, k) plane and
// marches along axis 0 (the slowest, plane stride).  The three components of
// the stage state y stream through a 4-slot shared-memory ring of planes
// (i-1, i, i+1 in use, i+2 landing) filled with cp.async, each plane with a
// one-cell halo in j and k; every y value is read from HBM once per CTA and
// the stencil's 27 reads per cell come from shared memory.  u0 / s are read
// and s / y_next written once, coalesced, at the centre.
// ---------------------------------------------------------------------------
template <int TJ, int TK>
struct RingGeom {
  static constexpr int PW = TK + 2, PH = TJ + 2, PS = PW * PH, NT = TJ * TK;
  // component stride inside a plane slot, padded so each component's TMA box
  // lands 128-byte aligned
  static constexpr int CS = (PS + 15) / 16 * 16;
};

// TMA descriptors of the three stage-state components: (TK+2) x (TJ+2) x 1
// boxes over the extended array (fp64, even row pitch); ok = 0 -> cp.async fill
struct alignas(64) StageMaps {
  CUtensorMap y[3];
  int ok;
};

// Momentum RHS of component A at the thread's cell from the smem ring, same
// arithmetic and order as rhs_comp (sfb_kernels.cuh).  P[d] points at the
// component-0 centre of plane i-1+d; component c sits at +c*PS.
template <typename T, int A, int TJ, int TK>
__device__ __forceinline__ T rhs_ring(const T* const (&P)[3], const Coef<T> (&C)[3], bool diff, T nu, T fa) {
  typedef RingGeom<TJ, TK> RG;
  auto Y = [&](int c, int di, int dj, int dk) -> T { return P[1 + di][c * RG::CS + dj * RG::PW + dk]; };
  const T uc = Y(A, 0, 0, 0);
  T up[3], um[3];
  up[0] = Y(A, 1, 0, 0);
  um[0] = Y(A, -1, 0, 0);
  up[1] = Y(A, 0, 1, 0);
  um[1] = Y(A, 0, -1, 0);
  up[2] = Y(A, 0, 0, 1);
  um[2] = Y(A, 0, 0, -1);
  T v = T(0);
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const T tp = (uc + up[b]) * T(0.5);
    const T tm = (um[b] + uc) * T(0.5);
    T fl;
    if (b == A) {
      fl = (tp * tp - tm * tm) * C[A].rdu;
    } else {
      const T wl = C[A].wlo, wh = C[A].whi;
      const int eA0 = A == 0, eA1 = A == 1, eA2 = A == 2;
      const int eb0 = b == 0, eb1 = b == 1, eb2 = b == 2;
      const T vp = Y(b, 0, 0, 0) * wl + Y(b, eA0, eA1, eA2) * wh;
      const T vm = Y(b, -eb0, -eb1, -eb2) * wl + Y(b, eA0 - eb0, eA1 - eb1, eA2 - eb2) * wh;
      fl = (tp * vp - tm * vm) * C[b].rdx;
    }
    v -= fl;
  }
  if (diff) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const T khi = b == A ? C[A].ohi : C[b].thi;
      const T klo = b == A ? C[A].olo : C[b].tlo;
      v += nu * ((up[b] - uc) * khi - (uc - um[b]) * klo);
    }
  }
  if (fa != T(0)) v += fa;
  return v;
}

constexpr int kRing = 5;   // planes i-1, i, i+1 in use, i+2 landing, i+3 issued
constexpr int kPRing = 4;  // FL_PROJ: pressure planes, slot = plane & 3

template <typename T, int TJ, int TK, int CPT, int FL, int MINB>
__global__ void __launch_bounds__(TJ / CPT * TK, MINB)
    k_stage_march(Geo<T> G, StageArgs<T> A, int chunk, const __grid_constant__ StageMaps SM) {
  typedef RingGeom<TJ, TK> RG;
  constexpr bool PROJ = (FL & FL_PROJ) != 0;
  constexpr bool PER = (FL & FL_PER) != 0;
  constexpr bool U0P = (FL & FL_U0P) != 0;
  static_assert(!U0P || PROJ, "FL_U0P needs the on-the-fly projection");
  constexpr int NTH = TJ / CPT * TK;                // threads per CTA
  constexpr int NE = 3 * RG::CS;                    // values per plane slot (padded components)
  constexpr int NQ = (NE + NTH - 1) / NTH;          // fill copies per thread
  constexpr int RS = TJ / CPT;                      // row stride between a thread's cells
  constexpr int PPW = TK + 3, PPS = (TJ + 3) * PPW; // FL_PROJ pressure slot (j0-1 .. j0+TJ+1)
  constexpr int NQP = PROJ ? (PPS + NTH - 1) / NTH : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);         // [kRing][3][CS]
  __shared__ __align__(8) unsigned long long ybar[kRing];  // TMA completion of each plane slot
  Coef<T>* cj = reinterpret_cast<Coef<T>*>(ring + kRing * NE);  // axis-1 coefficients of the tile rows
  T* pring = reinterpret_cast<T*>(cj + TJ);         // FL_PROJ: [kPRing][PPS]
  const int tk = threadIdx.x, tq = threadIdx.y, tid = tq * TK + tk;
  const int k0 = 1 + blockIdx.x * TK, j0 = 1 + blockIdx.y * TJ;
  const int ib = 1 + blockIdx.z * chunk;
  const int ie = min(ib + chunk, G.n[0] + 1);
  const int k = k0 + tk;
  const long long s0 = G.s[0];
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];

  const T* fsrc[NQ];
  bool fok[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int e = tid + q * NTH;
    const int c = e / RG::CS;
    const int r = e - c * RG::CS;
    const int jj = r / RG::PW;
    const int kk = r - jj * RG::PW;
    int gj = j0 - 1 + jj, gk = k0 - 1 + kk;
    fok[q] = e < NE && r < RG::PS && gj < G.E[1] && gk < G.E[2];
    if (PROJ) {
      gj = wrap1(gj, n1);
      gk = wrap1(gk, n2);
    }
    fsrc[q] = A.y.c[c < 3 ? c : 0] + (fok[q] ? (long long)gj * G.s[1] + gk : 0);
  }
  const T* psrc[NQP];
  bool pok[NQP];
  if constexpr (PROJ) {
#pragma unroll
    for (int q = 0; q < NQP; ++q) {
      const int e = tid + q * NTH;
      const int jj = e / PPW, kk = e - (e / PPW) * PPW;
      const int gj = j0 - 1 + jj, gk = k0 - 1 + kk;
      pok[q] = e < PPS && gj <= n1 + 2 && gk <= n2 + 2;
      psrc[q] = A.p_int + (pok[q] ? (long long)(wrap1(gj, n1) - 1) * n2 + (wrap1(gk, n2) - 1) : 0);
    }
  }
  const long long ps0 = (long long)n1 * n2;
  // slab (halo axis 0): y ghost planes exchanged, pressure planes 0..m+2 stored
  // (sfb_slab_buffers p_slab); otherwise periodic wrap into the n0 planes
  const bool h0 = G.halo[0] != 0;
  // y planes by TMA (one thread, three boxes per plane, mbarrier completion)
  // unless the tile's halo wraps around a periodic edge of an unprojected
  // stage state (FL_PROJ: its ghosts are never filled) -- those edge tiles
  // keep the per-element wrapped cp.async fill
  const bool tma = SM.ok && (!PROJ || (blockIdx.x > 0 && k0 + TK <= n2 && blockIdx.y > 0 && j0 + TJ <= n1));
  unsigned yph = 0, ypend = 0;  // per-slot barrier parity / loads in flight (tracked by every thread)
  if (tma && tid == 0) {
#pragma unroll
    for (int b = 0; b < kRing; ++b) mbar_init(&ybar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto ywait = [&](int slot) {
    if (tma && ((ypend >> slot) & 1)) {
      mbar_wait(&ybar[slot], (yph >> slot) & 1);
      yph ^= 1u << slot;
      ypend &= ~(1u << slot);
    }
  };
  auto load_p = [&](int ip) {
    if constexpr (PROJ) {
      // slab: planes 0..m+2 = 0..E[0] exist; periodic: wrap1 covers 1-n0..2n0.
      // Prefetches past that (m == 1 slabs, n0 == 1 grids) are never consumed.
      if (h0 ? (ip < 0 || ip > G.E[0]) : (ip < 1 - n0 || ip > 2 * n0)) return;
      T* dst = pring + (ip & (kPRing - 1)) * PPS + tid;
      const long long base = (long long)(h0 ? ip : wrap1(ip, n0) - 1) * ps0;
#pragma unroll
      for (int q = 0; q < NQP; ++q)
        if (q < NQP - 1 || tid + q * NTH < PPS) cp_async_val(dst + q * NTH, psrc[q] + (pok[q] ? base : 0), pok[q]);
    }
  };
  auto load_plane = [&](int ip, int slot, bool with_p = true) {
    if (ip < 0 || ip >= G.E[0]) return;
    const int pl = PROJ && !h0 ? wrap1(ip, n0) : ip;
    if (tma) {
      ypend |= 1u << slot;
      if (tid == 0) {
        T* dst = ring + slot * NE;
        mbar_arm(&ybar[slot], 3u * RG::PS * (unsigned)sizeof(T));
#pragma unroll
        for (int c = 0; c < 3; ++c) tma_load(&SM.y[c], 3, dst + c * RG::CS, &ybar[slot], k0 - 1, j0 - 1, pl);
      }
    } else {
      T* dst = ring + slot * NE + tid;
      const long long base = (long long)pl * s0;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < NQ - 1 || tid + q * NTH < NE) cp_async_val(dst + q * NTH, fsrc[q] + (fok[q] ? base : 0), fok[q]);
    }
    if (with_p) load_p(ip + 1);  // the pressure plane this y plane's projection needs besides its own
  };
  // y -= G p on one freshly landed plane slot (poisson.py:334-339 arithmetic).
  // A thread owns the same in-plane positions r = tid + q*NTH of every plane:
  // their pressure-slot offsets are fixed, the axis-1/2 reciprocal widths
  // come from two small shared tables filled once.
  constexpr int NR = (RG::PS + NTH - 1) / NTH;
  T* rdj = pring + kPRing * PPS;  // [TJ+2] 1/du_1 of the slot rows (wrapped)
  T* rdk = rdj + (TJ + 2);        // [TK+2] 1/du_2 of the slot columns
  int rpo[NR];
  if constexpr (PROJ) {
    for (int e = tid; e < TJ + 2; e += NTH) rdj[e] = tab(G, 1, T_RDU, wrap1(min(j0 - 1 + e, n1 + 1), n1));
    for (int e = tid; e < TK + 2; e += NTH) rdk[e] = tab(G, 2, T_RDU, wrap1(min(k0 - 1 + e, n2 + 1), n2));
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = tid + q * NTH;
      const int jj = r / RG::PW, kk = r - (r / RG::PW) * RG::PW;
      rpo[q] = (jj << 16) | kk;
    }
  }
  auto project_plane = [&](int ip, int slot) {
    if constexpr (PROJ) {
      T* ys = ring + slot * NE;
      const T* pc = pring + (ip & (kPRing - 1)) * PPS;
      const T* pn = pring + ((ip + 1) & (kPRing - 1)) * PPS;
      const T r0 = tab(G, 0, T_RDU, h0 ? ip : wrap1(ip, n0));
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int r = tid + q * NTH;
        if (q < NR - 1 || r < RG::PS) {
          const int jj = rpo[q] >> 16, kk = rpo[q] & 0xffff;
          const int po = jj * PPW + kk;
          const T p0 = pc[po];
          ys[r] -= (pn[po] - p0) * r0;
          ys[RG::CS + r] -= (pc[po + PPW] - p0) * rdj[jj];
          ys[2 * RG::CS + r] -= (pc[po + 1] - p0) * rdk[kk];
        }
      }
    }
  };
  if (tid < TJ) cj[tid] = coef_at(G, 1, min(j0 + tid, G.n[1]));
  Coef<T> C[3];
  C[2] = coef_at(G, 2, min(k, G.n[2]));

  int sl_m = (ib - 1) % kRing;
  if (PROJ) load_p(ib - 1);
  load_plane(ib - 1, sl_m);
  load_plane(ib, (sl_m + 1) % kRing);
  load_plane(ib + 1, (sl_m + 2) % kRing);
  cp_commit();
  // FL_PROJ: pressure plane ib+3 would land in the slot of ib-1, still needed
  // by the first projection; it is loaded in the first iteration instead
  load_plane(ib + 2, (sl_m + 3) % kRing, !PROJ);
  cp_commit();

  bool inside[CPT];
  int jr[CPT];
#pragma unroll
  for (int r = 0; r < CPT; ++r) {
    jr[r] = j0 + tq + r * RS;
    inside[r] = (k <= G.n[2]) && (jr[r] <= G.n[1]);
  }
  const bool wall0 = !G.per[0], wall1 = !G.per[1], wall2 = !G.per[2];
  long long x0 = (long long)ib * s0 + (long long)jr[0] * G.s[1] + k;
  const long long rstep = (long long)RS * G.s[1];
  for (int i = ib; i < ie; ++i, x0 += s0) {
    T b0[CPT][3], bs[CPT][3];
    bool dof[CPT][3];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const long long x = x0 + r * rstep;
      dof[r][0] = inside[r] && (PER || !(wall0 && i == G.n[0]));
      dof[r][1] = inside[r] && (PER || !(wall1 && jr[r] == G.n[1]));
      dof[r][2] = inside[r] && (PER || !(wall2 && k == G.n[2]));
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        b0[r][a] = T(0);
        bs[r][a] = T(0);
        if (dof[r][a]) {
          if (!U0P && ((FL & FL_NEXT) || ((FL & FL_S) && (FL & FL_SU0)))) b0[r][a] = A.u0.c[a][x];
          if ((FL & FL_S) && !(FL & FL_SU0)) bs[r][a] = A.s_in.c[a][x];
        }
      }
    }
    C[0] = coef_at(G, 0, i);
    int sl_l = sl_m + 4;
    if (sl_l >= kRing) sl_l -= kRing;
    int s1i = sl_m + 1, s2i = sl_m + 2;
    if (s1i >= kRing) s1i -= kRing;
    if (s2i >= kRing) s2i -= kRing;
    if (i == ib) {
      ywait(sl_m);
      ywait(s1i);
    }
    ywait(s2i);
    if (PROJ && i == ib + 1) cp_wait<0>();
    else cp_wait<1>();
    // this thread's generic-proxy accesses of the slot refilled below (read by
    // the stencil, rewritten by the projection) ordered before the TMA overwrite
    if (tma) fence_proxy_async_smem();
    __syncthreads();
    if constexpr (PROJ) {
      if (i == ib) {
        project_plane(i - 1, sl_m);
        project_plane(i, s1i);
      }
      project_plane(i + 1, s2i);
      __syncthreads();
      if (i == ib) load_p(ib + 3);
    }
    load_plane(i + 3, sl_l);
    cp_commit();
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const int c0 = (tq + r * RS + 1) * RG::PW + (tk + 1);
      const T* const P[3] = {ring + sl_m * NE + c0, ring + s1i * NE + c0, ring + s2i * NE + c0};
      C[1] = cj[tq + r * RS];
      T kv[3];
      if constexpr (PER) {
        kv[0] = rhs_ring<T, 0, TJ, TK>(P, C, A.diff, A.nu, A.F.f[0]);
        kv[1] = rhs_ring<T, 1, TJ, TK>(P, C, A.diff, A.nu, A.F.f[1]);
        kv[2] = rhs_ring<T, 2, TJ, TK>(P, C, A.diff, A.nu, A.F.f[2]);
      } else {
        kv[0] = dof[r][0] ? rhs_ring<T, 0, TJ, TK>(P, C, A.diff, A.nu, A.F.f[0]) : T(0);
        kv[1] = dof[r][1] ? rhs_ring<T, 1, TJ, TK>(P, C, A.diff, A.nu, A.F.f[1]) : T(0);
        kv[2] = dof[r][2] ? rhs_ring<T, 2, TJ, TK>(P, C, A.diff, A.nu, A.F.f[2]) : T(0);
      }
      const long long x = x0 + r * rstep;
      if (A.F.c[0]) {  // closure term after the force (operators.py:236-237)
        if (A.F.a[0]) {
#pragma unroll
          for (int a = 0; a < 3; ++a)
            if (dof[r][a]) kv[a] += A.F.a[a][x];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (dof[r][a]) kv[a] += A.F.c[a][x];
      } else if (A.F.a[0]) {  // per-DOF force fields (sample_force of a callable)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (dof[r][a]) kv[a] += A.F.a[a][x];
      }
      if constexpr (U0P) {
#pragma unroll
        for (int a = 0; a < 3; ++a) b0[r][a] = P[1][a * RG::CS];  // projected y at the centre
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!dof[r][a]) continue;
        if (U0P) A.u0_out.c[a][x] = b0[r][a];
        if (FL & FL_YOUT) A.u0_out.c[a][x] = P[1][a * RG::CS];  // projected y at the centre (tape)
        if (FL & FL_K) A.k_out.c[a][x] = kv[a];
        if (FL & FL_S) A.s_out.c[a][x] = ((FL & FL_SU0) ? b0[r][a] : bs[r][a]) + kv[a] * A.cb;
        if (FL & FL_NEXT) A.y_next.c[a][x] = b0[r][a] + kv[a] * A.ca;
      }
    }
    sl_m = s1i;
  }
  cp_wait<0>();
  // no TMA write may still target this CTA's shared memory when it exits
#pragma unroll
  for (int b = 0; b < kRing; ++b) ywait(b);
}

#ifndef SFB_STAGE_TJ
#define SFB_STAGE_TJ 8
#endif
#ifndef SFB_STAGE_CPT
#define SFB_STAGE_CPT 2
#endif
#ifndef SFB_STAGE_TK
#define SFB_STAGE_TK 32
#endif
constexpr int kTJ = SFB_STAGE_TJ, kTK = SFB_STAGE_TK, kCPT = SFB_STAGE_CPT;

// TMA maps of the stage state y (fp64 only: a (TK+2)-wide fp32 box row is not
// a multiple of 16 bytes); SM.ok = 0 keeps the cp.async fill
template <typename T, int TJ>
static void stage_maps(const Geo<T>& G, const StageArgs<T>& A, StageMaps& SM) {
  SM.ok = 0;
  static const bool off = env_int("SFB_STAGE_NOTMA") != 0;
  if (sizeof(T) != 8 || off || G.dim != 3) return;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encode_fn();
  if (!enc) return;
  const size_t esz = sizeof(T);
  if ((G.s[1] * esz) % 16 || (G.s[0] * esz) % 16) return;
  cuuint64_t dims[3] = {(cuuint64_t)G.E[2], (cuuint64_t)G.E[1], (cuuint64_t)G.E[0]};
  cuuint64_t strides[2] = {(cuuint64_t)(G.s[1] * esz), (cuuint64_t)(G.s[0] * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(kTK + 2), (cuuint32_t)(TJ + 2), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  for (int c = 0; c < 3; ++c) {
    if (!A.y.c[c] || ((uintptr_t)A.y.c[c] % 16)) return;
    if (enc(&SM.y[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A.y.c[c], dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return;
  }
  SM.ok = 1;
}

template <typename T, int FL>
static int stage_march_launch(const Geo<T>& G, const StageArgs<T>& A, cudaStream_t st) {
#ifndef SFB_STAGE_MINB
#define SFB_STAGE_MINB 3
#endif
#ifndef SFB_STAGE_MINB_PROJ
#define SFB_STAGE_MINB_PROJ 3
#endif
  // the deferred-projection stage 0 (FL_U0P: three field writes, no TMA) runs
  // 4 x 32 tiles, one cell per thread, 4 CTAs per SM (840^3: 18.1 -> 17.4 ms;
  // the other variants lost with that tile, profiles/r2/stage_tiles)
#ifndef SFB_U0P_TJ
#define SFB_U0P_TJ 4
#endif
#ifndef SFB_U0P_CPT
#define SFB_U0P_CPT 1
#endif
#ifndef SFB_U0P_MINB
#define SFB_U0P_MINB 4
#endif
  constexpr bool U0P = (FL & FL_U0P) != 0;
  constexpr int TJ = U0P ? SFB_U0P_TJ : kTJ, CPT = U0P ? SFB_U0P_CPT : kCPT;
  constexpr int MINB = U0P ? SFB_U0P_MINB : ((FL & FL_PROJ) ? SFB_STAGE_MINB_PROJ : SFB_STAGE_MINB);
  typedef RingGeom<TJ, kTK> RG;
  const size_t smem = (size_t)kRing * 3 * RG::CS * sizeof(T) + TJ * sizeof(Coef<T>) +
                      ((FL & FL_PROJ) ? ((size_t)kPRing * (TJ + 3) * (kTK + 3) + TJ + kTK + 4) * sizeof(T) : 0);
  if (cudaError_t e = ensure_smem((const void*)k_stage_march<T, TJ, kTK, CPT, FL, MINB>, smem))
    return cuda_check(e, "rk stage: shared-memory attribute");
  const int bx = (G.n[2] + kTK - 1) / kTK, by = (G.n[1] + TJ - 1) / TJ;
  const long long bps = (long long)bx * by;
  // split the march into bz chunks so the launch is >= ~30 waves of resident
  // CTAs: with one chunk (840^3: 2835 CTAs = 6.4 waves of 444) the last
  // partial wave idled most of the GPU for a whole CTA lifetime (stage
  // kernels 62.2 -> 57.4 ms per step at bz = 5); chunks stay >= 64 planes so
  // the 3-plane ring refill per chunk costs < 5 %
  long long want = (30LL * 148 * MINB + bps - 1) / bps;
  // the deferred stage 0 (three field writes) re-reads less DRAM with shorter
  // chunks: the resident tiles then span fewer planes, so their halo rows stay
  // in L2 (840^3: 8 chunks instead of 4, 67.6 -> 65.0 GB, 16.89 -> 16.54 ms)
  if (U0P && want < 8) want = 8;
  if (want > G.n[0] / 64) want = G.n[0] / 64;
  if (want < 1) want = 1;
  static const int bz_env = env_int("SFB_STAGE_BZ");
  if (bz_env > 0) want = bz_env;
  int chunk = (int)((G.n[0] + want - 1) / want);
  if (chunk < 16) chunk = 16;
  const int bz = (G.n[0] + chunk - 1) / chunk;
  // TMA fill for the on-the-fly-projection stages: stages 1-3 (17.8 -> 16.3,
  // 13.8 -> 12.8 ms at 840^3) and the deferred stage 0 on its 4 x 32 tiles
  // (17.4 -> 16.8 ms).  The plain stage 0 of a projected state (FL46) stays
  // on cp.async: with TMA it re-read more DRAM and stalled longer on 8 x 32
  // tiles (11.3 -> 13.0 ms; profiles/r2/stage_tma)
  StageMaps SM;
  SM.ok = 0;
  static const bool tma_all = env_int("SFB_STAGE_TMA_ALL") != 0;
  if (tma_all || ((FL & FL_PROJ) && (!(FL & FL_SU0) || (FL & FL_U0P)))) stage_maps<T, TJ>(G, A, SM);
  k_stage_march<T, TJ, kTK, CPT, FL, MINB><<<dim3(bx, by, bz), dim3(kTK, TJ / CPT), smem, st>>>(G, A, chunk, SM);
  SFB_LAUNCH_CHECK("rk stage (march)");
  return SFB_OK;
}

template <typename T>
static int stage_march(const Geo<T>& G, const StageArgs<T>& A, cudaStream_t st, bool allow_per = true) {
  // a halo axis 0 (z-slab) has no walls either: every local cell is a DOF, so
  // the branch-free variant applies (its ring reads the exchanged ghost planes)
  static const bool noper = env_int("SFB_STAGE_NOPER") != 0;
  const bool per = allow_per && G.per[0] && G.per[1] && G.per[2] && !G.halo[1] && !G.halo[2] && !noper;
  const int fl = (A.has_k ? FL_K : 0) | (A.has_s ? FL_S : 0) | (A.has_s && A.s_from_u0 ? FL_SU0 : 0) |
                 (A.has_next ? FL_NEXT : 0) | (A.p_int ? FL_PROJ : 0) | (per ? FL_PER : 0) |
                 (A.u0_out.c[0] && A.u0.c[0] == A.y.c[0] ? FL_U0P : 0) |
                 (A.u0_out.c[0] && A.u0.c[0] != A.y.c[0] ? FL_YOUT : 0);
  switch (fl) {
    // VJP tape: stages 1-3 also record the projected stage state
    case FL_PER | FL_S | FL_NEXT | FL_PROJ | FL_YOUT:
      return stage_march_launch<T, FL_PER | FL_S | FL_NEXT | FL_PROJ | FL_YOUT>(G, A, st);
    case FL_PER | FL_S | FL_PROJ | FL_YOUT: return stage_march_launch<T, FL_PER | FL_S | FL_PROJ | FL_YOUT>(G, A, st);
    case FL_PER | FL_S | FL_SU0 | FL_NEXT | FL_PROJ | FL_U0P:
      return stage_march_launch<T, FL_PER | FL_S | FL_SU0 | FL_NEXT | FL_PROJ | FL_U0P>(G, A, st);
    case FL_S | FL_SU0 | FL_NEXT | FL_PROJ | FL_U0P:
      return stage_march_launch<T, FL_S | FL_SU0 | FL_NEXT | FL_PROJ | FL_U0P>(G, A, st);
    case FL_PER | FL_S | FL_NEXT | FL_PROJ: return stage_march_launch<T, FL_PER | FL_S | FL_NEXT | FL_PROJ>(G, A, st);
    case FL_PER | FL_S | FL_PROJ: return stage_march_launch<T, FL_PER | FL_S | FL_PROJ>(G, A, st);
    case FL_PER | FL_S | FL_SU0 | FL_NEXT: return stage_march_launch<T, FL_PER | FL_S | FL_SU0 | FL_NEXT>(G, A, st);
    case FL_PER | FL_S | FL_NEXT: return stage_march_launch<T, FL_PER | FL_S | FL_NEXT>(G, A, st);
    case FL_PER | FL_S: return stage_march_launch<T, FL_PER | FL_S>(G, A, st);
    case FL_S | FL_NEXT | FL_PROJ: return stage_march_launch<T, FL_S | FL_NEXT | FL_PROJ>(G, A, st);
    case FL_S | FL_PROJ: return stage_march_launch<T, FL_S | FL_PROJ>(G, A, st);
    case FL_S | FL_SU0 | FL_NEXT: return stage_march_launch<T, FL_S | FL_SU0 | FL_NEXT>(G, A, st);
    case FL_S | FL_NEXT: return stage_march_launch<T, FL_S | FL_NEXT>(G, A, st);
    case FL_S: return stage_march_launch<T, FL_S>(G, A, st);
    case FL_S | FL_SU0: return stage_march_launch<T, FL_S | FL_SU0>(G, A, st);
    case FL_K: return stage_march_launch<T, FL_K>(G, A, st);
    case FL_NEXT: return stage_march_launch<T, FL_NEXT>(G, A, st);
    default:
      if (fl & FL_PER) return stage_march<T>(G, A, st, false);  // rarer variants: general-BC kernels
      return -1;  // uncommon combination: generic kernel
  }
}

template <typename T>
static int run_stage(sfb_plan* p, const sfb_stage_args* a, cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  StageArgs<T> A;
  for (int c = 0; c < 3; ++c) {
    bool on = c < p->dim;
    A.y.c[c] = on ? (const T*)a->y[c] : nullptr;
    A.u0.c[c] = on ? (const T*)a->u0[c] : nullptr;
    A.s_in.c[c] = on ? (const T*)a->s_in[c] : nullptr;
    A.s_out.c[c] = on ? (T*)a->s_out[c] : nullptr;
    A.y_next.c[c] = on ? (T*)a->y_next[c] : nullptr;
    A.k_out.c[c] = on ? (T*)a->k_out[c] : nullptr;
    A.u0_out.c[c] = on ? (T*)a->u0_out[c] : nullptr;
    A.F.a[c] = on ? (const T*)a->force_field[c] : nullptr;
    A.F.c[c] = on ? (const T*)a->closure_term[c] : nullptr;
    A.F.f[c] = (on && !A.F.a[c]) ? (T)a->force[c] : T(0);
  }
  A.cb = (T)a->cb;
  A.ca = (T)a->ca;
  A.nu = (T)a->nu;
  A.diff = a->nu != 0.0;
  A.has_k = a->k_out[0] != nullptr;
  A.has_s = a->s_out[0] != nullptr;
  A.has_next = a->y_next[0] != nullptr;
  A.s_from_u0 = a->s_in[0] == nullptr;
  A.p_int = (const T*)a->p_int;
  if (A.p_int && !(G.dim == 3 && G.per[0] && G.per[1] && G.per[2] && !G.halo[1] && !G.halo[2]))
    return fail(SFB_ECONFIG, "on-the-fly projection needs a periodic (or z-slab) 3D plan");
  if ((A.F.a[0] != nullptr) != (G.dim < 2 || A.F.a[1] != nullptr) ||
      (G.dim == 3 && (A.F.a[0] != nullptr) != (A.F.a[2] != nullptr)))
    return fail(SFB_EINVAL, "force fields: give all components or none");
  if (A.has_next && !a->u0[0]) return fail(SFB_EINVAL, "y_next requires u0");
  if (A.u0_out.c[0] && a->u0[0] != a->y[0]) {
    if (!A.p_int || A.has_k)
      return fail(SFB_EINVAL, "u0_out with u0 != y: the projected stage state of an on-the-fly projection only");
  } else if (A.u0_out.c[0]) {
    if (!A.p_int || a->u0[0] != a->y[0] || !A.has_s || !A.s_from_u0 || A.has_k)
      return fail(SFB_EINVAL, "u0_out: stage 0 of a deferred projection only (p_int set, u0 == y, s from u0)");
    for (int c = 0; c < G.dim; ++c)
      if (A.u0_out.c[c] == (const T*)a->y[c] || A.u0_out.c[c] == A.s_out.c[c] || A.u0_out.c[c] == A.y_next.c[c])
        return fail(SFB_EINVAL, "u0_out must not alias y, s_out or y_next");
  }
  if (A.has_s && A.s_from_u0 && !a->u0[0]) return fail(SFB_EINVAL, "s_out requires s_in or u0");
  static const bool generic = env_int("SFB_STAGE_GENERIC") != 0;
  if (G.dim == 3 && (!generic || A.p_int)) {
    const int rc = stage_march<T>(G, A, st);
    if (rc >= 0) return rc;
    if (A.p_int) return fail(SFB_ECONFIG, "on-the-fly projection: unsupported stage variant");
  }
  Box B = int_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_stage_generic<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, A, B)));
  SFB_LAUNCH_CHECK("rk stage");
  return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_rk_stage(sfb_plan* p, const sfb_stage_args* a, void* stream) {
  SFB_RANGE();
  if (!p || !a || !a->y[0]) return fail(SFB_EINVAL, "null argument");
  if (a->nu < 0) return fail(SFB_EINVAL, "viscosity must be nonnegative");
  return SFB_TYPED(p, run_stage<T>(p, a, (cudaStream_t)stream));
}
