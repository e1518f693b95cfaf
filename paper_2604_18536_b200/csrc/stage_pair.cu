// Fused RK stage, fp64 periodic fast path: two adjacent-k cells per thread.
//
// Same contract as k_stage_march (stage.cu): k = F(y) (operators.py:218-238,
// reference order of convection / diffusion / force terms) fused with the RK
// stage combine (timestep.py:186-207).  Differences that cut instructions:
//   * each thread owns the cell pair (k, k+1) with k even in the extended
//     index: the smem ring rows are 16-byte aligned, so a stencil row window
//     (k-1 .. k+2) is 2-3 LDS.128 shared by both cells, and the epilogue
//     (u0 / s reads, s / y_next writes) is 16-byte vectorised;
//   * the ring is filled with 16-byte cp.async copies whose per-thread
//     source offsets are precomputed once;
//   * periodic axes only (plus the slab halo axis): every interior cell is a
//     DOF of every component, so there is no per-component DOF logic.
// Used when all axes are periodic/halo, the dtype is fp64 and n2 is even.
#include <cstdlib>

#include "sfb_stage.cuh"

namespace sfb {

namespace {
constexpr int PTK = 32;             // cells per tile along k (16 pairs)
constexpr int PTJ = 8;              // rows per tile along j
constexpr int PNT = PTK / 2 * PTJ;  // 128 threads
constexpr int PPW = PTK + 4;        // ring row: ext k from kb-2 to kb+33 (36 values, 16B aligned)
constexpr int PPH = PTJ + 2;        // ring rows: j0-1 .. j0+8
constexpr int PPS = PPW * PPH;      // one component of one plane
constexpr int PNE = 3 * PPS;        // one plane slot
constexpr int PRING = 5;
constexpr int PNPAIR = PPW / 2;                 // 16B copies per ring row
constexpr int PNCOPY = 3 * PPH * PNPAIR;        // per plane
constexpr int PNQ = (PNCOPY + PNT - 1) / PNT;   // per thread
}  // namespace

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <int FL>
__global__ void __launch_bounds__(PNT, 4) k_stage_pair(Geo<double> G, StageArgs<double> A, int chunk) {
  typedef double T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);                      // [PRING][3][PPH][PPW]
  Coef<T>* cj = reinterpret_cast<Coef<T>*>(ring + PRING * PNE);  // axis-1 coefficients of the tile rows
  Coef<T>* ck = cj + PTJ;                                        // axis-2 coefficients of the tile cells
  const int tp = threadIdx.x, tq = threadIdx.y, tid = tq * (PTK / 2) + tp;
  const int kb = blockIdx.x * PTK;  // even extended k of the tile start
  const int j0 = 1 + blockIdx.y * PTJ;
  const int ib = 1 + blockIdx.z * chunk;
  const int ie = min(ib + chunk, G.n[0] + 1);
  const long long s0 = G.s[0], s1 = G.s[1];

  // plane-invariant ring fill descriptors
  int goff[PNQ], soff[PNQ];
  const T* gbase[PNQ];
  bool gok[PNQ];
#pragma unroll
  for (int q = 0; q < PNQ; ++q) {
    const int e = tid + q * PNT;
    const int row = e / PNPAIR;
    const int pr = e - row * PNPAIR;
    const int c = row / PPH;
    const int jj = row - c * PPH;
    const int gj = j0 - 1 + jj;
    const int gk = kb - 2 + 2 * pr;
    gok[q] = e < PNCOPY && gj < G.E[1] && gk >= 0 && gk + 1 < G.E[2];
    goff[q] = gok[q] ? (int)(gj * s1 + gk) : 0;
    soff[q] = c * PPS + jj * PPW + 2 * pr;
    gbase[q] = A.y.c[c < 3 ? c : 0];
  }
  auto load_plane = [&](int ip, int slot) {
    if (ip < 0 || ip >= G.E[0]) return;
    T* dst = ring + slot * PNE;
    const long long base = (long long)ip * s0;
#pragma unroll
    for (int q = 0; q < PNQ; ++q)
      if (q < PNQ - 1 || tid + q * PNT < PNCOPY) cp_async16(dst + soff[q], gbase[q] + (gok[q] ? base + goff[q] : 0), gok[q]);
  };
  if (tid < PTJ) cj[tid] = coef_at(G, 1, min(j0 + tid, G.n[1]));

  const int k = kb + 2 * tp;  // cells k and k+1
  const int j = j0 + tq;
  const bool jin = j <= G.n[1];
  const bool v0 = jin && k >= 1 && k <= G.n[2];
  const bool v1 = jin && k + 1 >= 1 && k + 1 <= G.n[2];
  if (tid < PTK) ck[tid] = coef_at(G, 2, min(max(kb + tid, 1), G.n[2]));

  int sl_m = (ib - 1) % PRING;
  load_plane(ib - 1, sl_m);
  load_plane(ib, (sl_m + 1) % PRING);
  load_plane(ib + 1, (sl_m + 2) % PRING);
  cp_commit();
  load_plane(ib + 2, (sl_m + 3) % PRING);
  cp_commit();

  const int cofs = (tq + 1) * PPW + 2 + 2 * tp;  // ring offset of cell k (component 0)
  long long x = (long long)ib * s0 + (long long)j * s1 + k;  // even: 16B aligned pair
  const T nu = A.nu;
  for (int i = ib; i < ie; ++i, x += s0) {
    // epilogue operands (vector loads), issued before the ring wait
    double2 b0[3], bs[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      b0[a] = make_double2(0.0, 0.0);
      bs[a] = make_double2(0.0, 0.0);
      if (v0 || v1) {
        if ((FL & FL_NEXT) || ((FL & FL_S) && (FL & FL_SU0))) b0[a] = *reinterpret_cast<const double2*>(A.u0.c[a] + x);
        if ((FL & FL_S) && !(FL & FL_SU0)) bs[a] = *reinterpret_cast<const double2*>(A.s_in.c[a] + x);
      }
    }
    const Coef<T> C0 = coef_at(G, 0, i);
    cp_wait<1>();
    __syncthreads();
    int sl_l = sl_m + 4;
    if (sl_l >= PRING) sl_l -= PRING;
    load_plane(i + 3, sl_l);
    cp_commit();
    int s1i = sl_m + 1, s2i = sl_m + 2;
    if (s1i >= PRING) s1i -= PRING;
    if (s2i >= PRING) s2i -= PRING;
    const Coef<T> C1 = cj[tq];
    const T* Pm = ring + sl_m * PNE + cofs;  // plane i-1
    const T* P0 = ring + s1i * PNE + cofs;   // plane i
    const T* Pp = ring + s2i * PNE + cofs;   // plane i+1
    // row windows; (x, y) of a double2 are the values at k, k+1 (offset 0),
    // k-2, k-1 (offset -2) or k+2, k+3 (offset +2)
    T ctr[3][4];  // centre row: k-1, k, k+1, k+2
    T ipv[3][2], imv[3][2], jpv[3][2], jmv[3][2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double2 a = lds2(P0 + c * PPS - 2), b = lds2(P0 + c * PPS), d = lds2(P0 + c * PPS + 2);
      ctr[c][0] = a.y;
      ctr[c][1] = b.x;
      ctr[c][2] = b.y;
      ctr[c][3] = d.x;
      double2 t = lds2(Pp + c * PPS);
      ipv[c][0] = t.x;
      ipv[c][1] = t.y;
      t = lds2(Pm + c * PPS);
      imv[c][0] = t.x;
      imv[c][1] = t.y;
      t = lds2(P0 + c * PPS + PPW);
      jpv[c][0] = t.x;
      jpv[c][1] = t.y;
      t = lds2(P0 + c * PPS - PPW);
      jmv[c][0] = t.x;
      jmv[c][1] = t.y;
    }
    // cross-term windows
    const double2 ipjm1 = lds2(Pp + 1 * PPS - PPW);                 // u1 (i+1, j-1) k, k+1
    const double2 imjp0 = lds2(Pm + 0 * PPS + PPW);                 // u0 (i-1, j+1) k, k+1
    const T ip2m = lds2(Pp + 2 * PPS - 2).y;                        // u2 (i+1, j, k-1)
    const T jp2m = lds2(P0 + 2 * PPS + PPW - 2).y;                  // u2 (i, j+1, k-1)
    const T im0p = lds2(Pm + 0 * PPS + 2).x;                        // u0 (i-1, j, k+2)
    const T jm1p = lds2(P0 + 1 * PPS - PPW + 2).x;                  // u1 (i, j-1, k+2)
    T kv[2][3];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const Coef<T> Ck = ck[2 * tp + q];
      // neighbours of component a at cell q along axis b: up/um
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const T uc = ctr[a][1 + q];
        const T up[3] = {ipv[a][q], jpv[a][q], ctr[a][2 + q]};
        const T um[3] = {imv[a][q], jmv[a][q], ctr[a][q]};
        const Coef<T>& Ca = a == 0 ? C0 : (a == 1 ? C1 : Ck);
        T v = T(0);
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const T tp_ = (uc + up[b]) * T(0.5);
          const T tm_ = (um[b] + uc) * T(0.5);
          T fl;
          if (b == a) {
            fl = (tp_ * tp_ - tm_ * tm_) * Ca.rdu;
          } else {
            const Coef<T>& Cb = b == 0 ? C0 : (b == 1 ? C1 : Ck);
            const T ub0 = ctr[b][1 + q];
            // u_b at +e_a
            const T ubA = a == 0 ? ipv[b][q] : (a == 1 ? jpv[b][q] : ctr[b][2 + q]);
            // u_b at -e_b
            const T ubm = b == 0 ? imv[0][q] : (b == 1 ? jmv[1][q] : ctr[2][q]);
            // u_b at -e_b + e_a
            T ubmA;
            if (a == 0 && b == 1) ubmA = q == 0 ? ipjm1.x : ipjm1.y;
            else if (a == 0 && b == 2) ubmA = q == 0 ? ip2m : ipv[2][0];
            else if (a == 1 && b == 0) ubmA = q == 0 ? imjp0.x : imjp0.y;
            else if (a == 1 && b == 2) ubmA = q == 0 ? jp2m : jpv[2][0];
            else if (a == 2 && b == 0) ubmA = q == 0 ? imv[0][1] : im0p;
            else ubmA = q == 0 ? jmv[1][1] : jm1p;  // a == 2, b == 1
            const T vp = ub0 * Ca.wlo + ubA * Ca.whi;
            const T vm = ubm * Ca.wlo + ubmA * Ca.whi;
            fl = (tp_ * vp - tm_ * vm) * Cb.rdx;
          }
          v -= fl;
        }
        if (A.diff) {
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const Coef<T>& Cb = b == 0 ? C0 : (b == 1 ? C1 : Ck);
            const T khi = b == a ? Ca.ohi : Cb.thi;
            const T klo = b == a ? Ca.olo : Cb.tlo;
            v += nu * ((up[b] - uc) * khi - (uc - um[b]) * klo);
          }
        }
        const T fa = A.F.f[a];
        if (fa != T(0)) v += fa;
        kv[q][a] = v;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double2 so, yo;
      if (FL & FL_S) {
        const double2 bb = (FL & FL_SU0) ? b0[a] : bs[a];
        so = make_double2(bb.x + kv[0][a] * A.cb, bb.y + kv[1][a] * A.cb);
      }
      if (FL & FL_NEXT) yo = make_double2(b0[a].x + kv[0][a] * A.ca, b0[a].y + kv[1][a] * A.ca);
      if (v0 && v1) {
        if (FL & FL_S) *reinterpret_cast<double2*>(A.s_out.c[a] + x) = so;
        if (FL & FL_NEXT) *reinterpret_cast<double2*>(A.y_next.c[a] + x) = yo;
        if (FL & FL_K) *reinterpret_cast<double2*>(A.k_out.c[a] + x) = make_double2(kv[0][a], kv[1][a]);
      } else if (v0) {
        if (FL & FL_S) A.s_out.c[a][x] = so.x;
        if (FL & FL_NEXT) A.y_next.c[a][x] = yo.x;
        if (FL & FL_K) A.k_out.c[a][x] = kv[0][a];
      } else if (v1) {
        if (FL & FL_S) A.s_out.c[a][x + 1] = so.y;
        if (FL & FL_NEXT) A.y_next.c[a][x + 1] = yo.y;
        if (FL & FL_K) A.k_out.c[a][x + 1] = kv[1][a];
      }
    }
    sl_m = s1i;
  }
  cp_wait<0>();
}

template <int FL>
static int pair_launch(const Geo<double>& G, const StageArgs<double>& A, cudaStream_t st) {
  const size_t smem = (size_t)PRING * PNE * sizeof(double) + (PTJ + PTK) * sizeof(Coef<double>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_stage_pair<FL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int bx = (G.E[2] + PTK - 1) / PTK, by = (G.n[1] + PTJ - 1) / PTJ;
  const long long bps = (long long)bx * by;
  long long want = (4LL * 148 * 4 + bps - 1) / bps;
  int chunk = (int)((G.n[0] + want - 1) / want);
  if (chunk < 16) chunk = 16;
  const int bz = (G.n[0] + chunk - 1) / chunk;
  k_stage_pair<FL><<<dim3(bx, by, bz), dim3(PTK / 2, PTJ), smem, st>>>(G, A, chunk);
  SFB_LAUNCH_CHECK("rk stage (pair)");
  return SFB_OK;
}

template <>
int stage_pair<double>(const Geo<double>& G, const StageArgs<double>& A, cudaStream_t st) {
  for (int a = 0; a < 3; ++a)
    if (!G.per[a]) return -1;  // periodic / halo axes only
  if (G.E[2] % 2 != 0) return -1;
  const int fl = (A.has_k ? FL_K : 0) | (A.has_s ? FL_S : 0) | (A.has_s && A.s_from_u0 ? FL_SU0 : 0) |
                 (A.has_next ? FL_NEXT : 0);
  switch (fl) {
    case FL_S | FL_SU0 | FL_NEXT: return pair_launch<FL_S | FL_SU0 | FL_NEXT>(G, A, st);
    case FL_S | FL_NEXT: return pair_launch<FL_S | FL_NEXT>(G, A, st);
    case FL_S: return pair_launch<FL_S>(G, A, st);
    case FL_K: return pair_launch<FL_K>(G, A, st);
    default: return -1;
  }
}

template <>
int stage_pair<float>(const Geo<float>&, const StageArgs<float>&, cudaStream_t) {
  return -1;
}

}  // namespace sfb
