// Pressure Poisson solvers and the projection (poisson.py:152-348).
//
// SPECTRAL  (poisson.py:167-200): cuFFT D2Z/Z2D (raw transforms only) +
//           hand-written eigenvalue scaling (separable 1D tables, the
//           irfftn 1/N folded in, k = 0 zeroed).
// CHANNEL   (replaces DirectPoissonSolver, poisson.py:203-229, on grids
//           periodic+uniform in x/z with walls on y): batched 2D D2Z over
//           (x, z) -> per-(kx,kz) tridiagonal along y (Thomas, one thread per
//           system, coalesced over kz; fp64 arithmetic) -> Z2D.  The (0,0)
//           mode is closed by the weighted-zero-mean gauge of the augmented
//           system (poisson.py:211-229).
// project   (poisson.py:321-341): div with inline boundary resolution ->
//           solve -> gradient subtract (periodic wrap inline) -> ghost fill.
#include <cufft.h>

#include <cmath>
#include <cstdlib>
#include <vector>

#include "sfb_kernels.cuh"
#include "sfb_solver.cuh"

namespace sfb {

static int cufft_check(cufftResult r, const char* what) {
  if (r == CUFFT_SUCCESS) return SFB_OK;
  return fail(SFB_ECUDA, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

// ---------------------------------------------------------------------------
// projection kernels
// ---------------------------------------------------------------------------

// divergence into a contiguous interior array (operators.py:108-122)
template <typename T, int D>
__global__ void k_div_int(Geo<T> G, CV<T> U, T* __restrict__ out, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  T acc = T(0);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T cur, prev;
    own_pair<T, D>(G, U.c[a], x, I, a, cur, prev);
    acc += (cur - prev) * tab(G, a, T_RDX, I[a]);
  }
  long long o = (long long)(I[0] - 1) * G.n[1] + (I[1] - 1);
  if (D == 3) o = o * G.n[2] + (I[2] - 1);
  out[o] = acc;
}

// 3D marching divergence: a thread owns a (j, k) column and walks a chunk of
// planes, carrying u_0 of the previous plane in a register (one fewer load per
// cell, loads of consecutive planes in flight together).
template <typename T>
__global__ void __launch_bounds__(256) k_div_march(Geo<T> G, CV<T> U, T* __restrict__ out, int chunk) {
  const int k = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int j = 1 + blockIdx.y * blockDim.y + threadIdx.y;
  if (k > G.n[2] || j > G.n[1]) return;
  const int ib = 1 + blockIdx.z * chunk;
  const int ie = min(ib + chunk, G.n[0] + 1);
  const long long s0 = G.s[0], s1 = G.s[1];
  const T* __restrict__ u0 = U.c[0];
  const T* __restrict__ u1 = U.c[1];
  const T* __restrict__ u2 = U.c[2];
  const T r1 = tab(G, 1, T_RDX, j), r2 = tab(G, 2, T_RDX, k);
  // axis-1 / axis-2 neighbour offsets with inline boundary resolution
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const bool w1lo = !G.per[1] && !G.halo[1] && j == 1, w1hi = !G.per[1] && !G.halo[1] && j == n1;
  const bool w2lo = !G.per[2] && !G.halo[2] && k == 1, w2hi = !G.per[2] && !G.halo[2] && k == n2;
  const long long o1m = (G.per[1] && !G.halo[1] && j == 1) ? (long long)(n1 - 1) * s1 : -s1;
  const long long o2m = (G.per[2] && !G.halo[2] && k == 1) ? (long long)(n2 - 1) : -1;
  const T v1lo = G.bc_lo[1] == SFB_BC_DIRICHLET ? G.vlo[1][1] : T(0), v1hi = G.bc_hi[1] == SFB_BC_DIRICHLET ? G.vhi[1][1] : T(0);
  const T v2lo = G.bc_lo[2] == SFB_BC_DIRICHLET ? G.vlo[2][2] : T(0), v2hi = G.bc_hi[2] == SFB_BC_DIRICHLET ? G.vhi[2][2] : T(0);
  const bool wall0 = !G.per[0] && !G.halo[0];
  long long x = (long long)ib * s0 + (long long)j * s1 + k;
  T prev0;
  if (ib == 1) {
    if (G.halo[0]) prev0 = u0[x - s0];
    else if (G.per[0]) prev0 = u0[x + (long long)(n0 - 1) * s0];
    else prev0 = G.bc_lo[0] == SFB_BC_DIRICHLET ? G.vlo[0][0] : T(0);
  } else {
    prev0 = u0[x - s0];
  }
  long long o = ((long long)(ib - 1) * n1 + (j - 1)) * n2 + (k - 1);
  const long long os = (long long)n1 * n2;
#pragma unroll 4
  for (int i = ib; i < ie; ++i, x += s0, o += os) {
    const T m0 = u0[x];
    const T c0 = (wall0 && i == n0) ? (G.bc_hi[0] == SFB_BC_DIRICHLET ? G.vhi[0][0] : T(0)) : m0;
    const T c1 = w1hi ? v1hi : u1[x];
    const T p1 = w1lo ? v1lo : u1[x + o1m];
    const T c2 = w2hi ? v2hi : u2[x];
    const T p2 = w2lo ? v2lo : u2[x + o2m];
    T acc = (c0 - prev0) * tab(G, 0, T_RDX, i);
    acc += (c1 - p1) * r1;
    acc += (c2 - p2) * r2;
    out[o] = acc;
    prev0 = m0;
  }
}

// u_a[DOF] -= (p[I+e_a] - p[I]) / du_a   (poisson.py:334-339), p interior
template <typename T, int D>
__global__ void k_grad_sub(Geo<T> G, const T* __restrict__ p, MV<T> U, Box B, T* __restrict__ pe) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  long long o = (long long)(I[0] - 1) * G.n[1] + (I[1] - 1);
  long long ps[3];
  if (D == 3) {
    o = o * G.n[2] + (I[2] - 1);
    ps[0] = (long long)G.n[1] * G.n[2];
    ps[1] = G.n[2];
    ps[2] = 1;
  } else {
    ps[0] = G.n[1];
    ps[1] = 1;
  }
  const T pc = p[o];
  if (pe) pe[x] = pc;  // extended pressure interior (ghosts: scalar fill after)
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    // only periodic axes reach I_a = n for their own component; a halo axis
    // reads the next slab's first plane, stored after the local planes
    const long long on = (I[a] == G.n[a] && !G.halo[a]) ? o - (long long)(G.n[a] - 1) * ps[a] : o + ps[a];
    const T g = (p[on] - pc) * tab(G, a, T_RDU, I[a]);
    U.c[a][x] -= g;
  }
}

// 3D marching gradient-subtract (+ extended pressure interior): a thread owns
// a (j, k) column and walks a chunk of planes carrying p of the next plane.
template <typename T>
__global__ void __launch_bounds__(256) k_grad_march(Geo<T> G, const T* __restrict__ p, MV<T> U, int chunk,
                                                     T* __restrict__ pe) {
  const int k = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int j = 1 + blockIdx.y * blockDim.y + threadIdx.y;
  if (k > G.n[2] || j > G.n[1]) return;
  const int ib = 1 + blockIdx.z * chunk;
  const int ie = min(ib + chunk, G.n[0] + 1);
  const int n0 = G.n[0], n1 = G.n[1], n2 = G.n[2];
  const long long s0 = G.s[0], s1 = G.s[1];
  const long long os = (long long)n1 * n2;
  T* __restrict__ u0 = U.c[0];
  T* __restrict__ u1 = U.c[1];
  T* __restrict__ u2 = U.c[2];
  const bool per1 = G.per[1] && !G.halo[1], per2 = G.per[2] && !G.halo[2];
  const bool dof1 = !(!G.per[1] && j == n1), dof2 = !(!G.per[2] && k == n2);
  const long long oj = (j == n1 && per1) ? -(long long)(n1 - 1) * n2 : n2;
  const long long ok = (k == n2 && per2) ? -(long long)(n2 - 1) : 1;
  const T r1 = tab(G, 1, T_RDU, j), r2 = tab(G, 2, T_RDU, k);
  const bool per0 = G.per[0] && !G.halo[0], wall0 = !G.per[0];
  long long x = (long long)ib * s0 + (long long)j * s1 + k;
  long long o = ((long long)(ib - 1) * n1 + (j - 1)) * n2 + (k - 1);
  T pc = p[o];
#pragma unroll 4
  for (int i = ib; i < ie; ++i, x += s0, o += os) {
    // next plane (periodic wrap at i = n0; a halo axis reads the stored halo plane)
    const long long on = (i == n0 && per0) ? o - (long long)(n0 - 1) * os : o + os;
    const bool has_next = !(wall0 && i == n0);
    const T pn = (has_next || i < n0) ? p[on] : pc;
    const T pj = dof1 ? p[o + oj] : pc;
    const T pk = dof2 ? p[o + ok] : pc;
    if (pe) pe[x] = pc;
    if (has_next) u0[x] -= (pn - pc) * tab(G, 0, T_RDU, i);
    if (dof1) u1[x] -= (pj - pc) * r1;
    if (dof2) u2[x] -= (pk - pc) * r2;
    pc = pn;
  }
}

template <typename T>
static int launch_grad(const Geo<T>& G, const T* p, MV<T> U, T* pe, cudaStream_t st);

// extended, ghost-filled pressure from the interior solution (fields.py:81-93)
template <typename T, int D>
__global__ void k_p_ext(Geo<T> G, const T* __restrict__ p, T* __restrict__ pe, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  int J[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int n = G.n[a];
    int i = I[a];
    if (G.halo[a]) {
      if (i == 0) return;  // previous slab's plane: exchanged by the caller
      J[a] = i - 1;        // i == n + 1 reads the halo plane stored after the slab
      continue;
    }
    if (i == 0) i = G.per[a] ? n : 1;
    else if (i == n + 1) i = G.per[a] ? 1 : n;
    J[a] = i - 1;
  }
  long long o = (long long)J[0] * G.n[1] + J[1];
  if (D == 3) o = o * G.n[2] + J[2];
  pe[lin<T, D>(G, I)] = p[o];
}

template <typename T>
static int launch_grad(const Geo<T>& G, const T* p, MV<T> U, T* pe, cudaStream_t st) {
  static const bool grad_march = env_int("SFB_GRAD_MARCH") != 0;
  if (G.dim == 3 && grad_march) {
    dim3 blk(64, 4);
    const int bx = (G.n[2] + 63) / 64, by = (G.n[1] + 3) / 4;
    const long long bps = (long long)bx * by;
    long long want = (30LL * 148 * 8 + bps - 1) / bps;  // >= ~30 waves (stage.cu)
    if (want > G.n[0] / 32) want = G.n[0] / 32;
    if (want < 1) want = 1;
    int chunk = (int)((G.n[0] + want - 1) / want);
    if (chunk < 8) chunk = 8;
    const int bz = (G.n[0] + chunk - 1) / chunk;
    k_grad_march<T><<<dim3(bx, by, bz), blk, 0, st>>>(G, p, U, chunk, pe);
    SFB_LAUNCH_CHECK("gradient subtract (march)");
    return SFB_OK;
  }
  Box B = int_box(G);
  if (G.dim == 3) {
    // 128 x 2 blocks along the contiguous axis (vs the generic 32 x 4 x 2):
    // longer contiguous runs per warp pair, 840^3 fp64 8.18 -> 7.65 ms
    // SFB_GRAD_BLK: a power of two in [32, 256], else the measured default
    static const int bxk = [] {
      const int v = env_int("SFB_GRAD_BLK", 128);
      return (v >= 32 && v <= 256 && (v & (v - 1)) == 0) ? v : 128;
    }();
    dim3 blk(bxk, 256 / bxk, 1);
    dim3 grid((B.cnt[2] + blk.x - 1) / blk.x, (B.cnt[1] + blk.y - 1) / blk.y, B.cnt[0]);
    k_grad_sub<T, 3><<<grid, blk, 0, st>>>(G, p, U, B, pe);
    SFB_LAUNCH_CHECK("gradient subtract");
    return SFB_OK;
  }
  SFB_DISPATCH_DIM(G.dim, D, (k_grad_sub<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, p, U, B, pe)));
  SFB_LAUNCH_CHECK("gradient subtract");
  return SFB_OK;
}

template <typename T>
static int launch_div(const Geo<T>& G, CV<T> C, T* out, cudaStream_t st) {
  static const bool div_march = env_int("SFB_DIV_MARCH") != 0;
  if (G.dim == 3 && div_march) {
    dim3 blk(64, 4);
    const int bx = (G.n[2] + 63) / 64, by = (G.n[1] + 3) / 4;
    const long long bps = (long long)bx * by;
    long long want = (4LL * 148 * 8 + bps - 1) / bps;
    int chunk = (int)((G.n[0] + want - 1) / want);
    if (chunk < 8) chunk = 8;
    const int bz = (G.n[0] + chunk - 1) / chunk;
    k_div_march<T><<<dim3(bx, by, bz), blk, 0, st>>>(G, C, out, chunk);
    SFB_LAUNCH_CHECK("divergence (march)");
    return SFB_OK;
  }
  Box B = int_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_div_int<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, C, out, B)));
  SFB_LAUNCH_CHECK("projection divergence");
  return SFB_OK;
}

// ---------------------------------------------------------------------------
// spectral scaling (poisson.py:179-199)
// ---------------------------------------------------------------------------
template <typename T, int D>
__global__ void k_spec_scale(typename CT<T>::type* __restrict__ c, const double* __restrict__ l0,
                             const double* __restrict__ l1, const double* __restrict__ l2, int m0, int m1, int mh,
                             T invN) {
  const long long total = (long long)m0 * (D == 3 ? (long long)m1 * mh : mh);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int k0, k1, k2;
    if (D == 3) {
      k2 = (int)(t % mh);
      long long r = t / mh;
      k1 = (int)(r % m1);
      k0 = (int)(r / m1);
    } else {
      k1 = (int)(t % mh);
      k0 = (int)(t / mh);
      k2 = 0;
    }
    // lam accumulated in fp64 in axis order, then cast (poisson.py:179-192)
    double lam = l0[k0] + l1[k1];
    if (D == 3) lam = lam + l2[k2];
    typename CT<T>::type v = c[t];
    if (t == 0) {
      v.x = T(0);
      v.y = T(0);
    } else {
      const T lt = (T)lam;
      v.x = v.x / lt * invN;
      v.y = v.y / lt * invN;
    }
    c[t] = v;
  }
}

// ---------------------------------------------------------------------------
// channel: batched tridiagonal along y per (kx, kz)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_tridiag(typename CT<T>::type* c, double2* dd, double* __restrict__ cp,
                          const double* __restrict__ up, const double* __restrict__ lo, const double* __restrict__ di,
                          const double* __restrict__ dxy, const double* __restrict__ lx, const double* __restrict__ lz,
                          int n0, int n1, int nh, double invN) {
  // dd: fp64 forward-sweep storage; aliases c for fp64 plans (so neither is
  // __restrict__: the chunked loads must stay ahead of the aliased stores)
  const int kz = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = blockIdx.y;
  if (kz >= nh) return;
  const long long base = (long long)k0 * n1 * nh + kz;
  const long long st = nh;
  const bool zero_mode = (k0 == 0 && kz == 0);
  const double lam = lx[k0] + lz[kz];
  double mr = 0.0, mi = 0.0;
  if (zero_mode) {
    // remove the dx-weighted mean: the (0,0)-mode image of the weighted-mean
    // removal of the augmented system (poisson.py:211-229)
    double sw = 0.0;
    for (int j = 0; j < n1; ++j) {
      const typename CT<T>::type v = c[base + j * st];
      mr += dxy[j] * (double)v.x;
      mi += dxy[j] * (double)v.y;
      sw += dxy[j];
    }
    mr /= sw;
    mi /= sw;
  }
  // (0,0): consistent singular Neumann system; drop the last row and pin
  // x_{n1-1} = 0, then restore the weighted zero mean below
  const int m = zero_mode ? n1 - 1 : n1;
  // the sweeps are serial in j: loads are issued kTdU rows ahead so only one
  // memory latency is exposed per kTdU steps
  constexpr int kTdU = 8;
  double cprev = 0.0, dr = 0.0, dm = 0.0;
  for (int j0 = 0; j0 < m; j0 += kTdU) {
    typename CT<T>::type vb[kTdU];
#pragma unroll
    for (int u = 0; u < kTdU; ++u)
      if (j0 + u < m) vb[u] = c[base + (long long)(j0 + u) * st];
#pragma unroll
    for (int u = 0; u < kTdU; ++u) {
      const int j = j0 + u;
      if (j >= m) break;
      const double l = lo[j + 1];
      double b = di[j + 1] + (zero_mode ? 0.0 : lam);
      if (j > 0) b -= l * cprev;
      const double ib = 1.0 / b;
      const double cj = up[j + 1] * ib;
      dr = ((double)vb[u].x - mr - l * dr) * ib;
      dm = ((double)vb[u].y - mi - l * dm) * ib;
      cp[base + (long long)j * st] = cj;
      cprev = cj;
      dd[base + (long long)j * st] = make_double2(dr, dm);
    }
  }
  double xr = 0.0, xi = 0.0;
  double sr = 0.0, si = 0.0, sw = 0.0;
  for (int j1 = m - 1; j1 >= 0; j1 -= kTdU) {
    double2 db[kTdU];
    double cb[kTdU];
#pragma unroll
    for (int u = 0; u < kTdU; ++u)
      if (j1 - u >= 0) {
        db[u] = dd[base + (long long)(j1 - u) * st];
        cb[u] = cp[base + (long long)(j1 - u) * st];
      }
#pragma unroll
    for (int u = 0; u < kTdU; ++u) {
      const int j = j1 - u;
      if (j < 0) break;
      const double2 v = db[u];
      if (j == m - 1) {
        xr = v.x;
        xi = v.y;
      } else {
        xr = v.x - cb[u] * xr;
        xi = v.y - cb[u] * xi;
      }
      if (zero_mode) {
        dd[base + (long long)j * st] = make_double2(xr, xi);
        sr += dxy[j] * xr;
        si += dxy[j] * xi;
      } else {
        typename CT<T>::type w;
        w.x = (T)(xr * invN);
        w.y = (T)(xi * invN);
        c[base + (long long)j * st] = w;
      }
    }
  }
  if (zero_mode) {
    for (int j = 0; j < n1; ++j) sw += dxy[j];
    sr /= sw;
    si /= sw;
    for (int j = 0; j < n1; ++j) {
      double2 v = j < m ? dd[base + j * st] : make_double2(0.0, 0.0);
      typename CT<T>::type w;
      w.x = (T)((v.x - sr) * invN);
      w.y = (T)((v.y - si) * invN);
      c[base + j * st] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// solver object
// ---------------------------------------------------------------------------
static int make_plans(sfb_solver* s) {
  sfb_plan* p = s->plan;
  const bool f64 = p->dtype == SFB_F64;
  cufftType tf = f64 ? CUFFT_D2Z : CUFFT_R2C, ti = f64 ? CUFFT_Z2D : CUFFT_C2R;
  int rc;
  if ((rc = cufft_check(cufftCreate(&s->fwd), "cufftCreate"))) return rc;
  s->has_fwd = true;
  if ((rc = cufft_check(cufftCreate(&s->inv), "cufftCreate"))) return rc;
  s->has_inv = true;
  cufftSetAutoAllocation(s->fwd, 0);
  cufftSetAutoAllocation(s->inv, 0);
  size_t w1 = 0, w2 = 0;
  if (s->kind == SFB_SOLVER_SPECTRAL) {
    int nn[3] = {p->n[0], p->n[1], p->n[2]};
    if ((rc = cufft_check(cufftMakePlanMany(s->fwd, p->dim, nn, nullptr, 1, 0, nullptr, 1, 0, tf, 1, &w1), "plan fwd")))
      return rc;
    if ((rc = cufft_check(cufftMakePlanMany(s->inv, p->dim, nn, nullptr, 1, 0, nullptr, 1, 0, ti, 1, &w2), "plan inv")))
      return rc;
  } else {
    const int n0 = p->n[0], n1 = p->n[1], n2 = p->n[2], nh = n2 / 2 + 1;
    int nn[2] = {n0, n2};
    int ie[2] = {n0, n1 * n2};
    int oe[2] = {n0, n1 * nh};
    if ((rc = cufft_check(cufftMakePlanMany(s->fwd, 2, nn, ie, 1, n2, oe, 1, nh, tf, n1, &w1), "plan fwd"))) return rc;
    if ((rc = cufft_check(cufftMakePlanMany(s->inv, 2, nn, oe, 1, nh, ie, 1, n2, ti, n1, &w2), "plan inv"))) return rc;
  }
  s->work_size = w1 > w2 ? w1 : w2;
  if (s->work_size) {
    if ((rc = cuda_check(cudaMalloc(&s->work, s->work_size), "cudaMalloc(cufft work)"))) return rc;
  }
  cufftSetWorkArea(s->fwd, s->work);
  cufftSetWorkArea(s->inv, s->work);
  return SFB_OK;
}

template <typename T>
static int exec_fwd(sfb_solver* s, const T* in, cudaStream_t st) {
  cufftSetStream(s->fwd, st);
  if (sizeof(T) == 8)
    return cufft_check(cufftExecD2Z(s->fwd, (cufftDoubleReal*)in, (cufftDoubleComplex*)s->cbuf), "D2Z");
  return cufft_check(cufftExecR2C(s->fwd, (cufftReal*)in, (cufftComplex*)s->cbuf), "R2C");
}
template <typename T>
static int exec_inv(sfb_solver* s, T* out, cudaStream_t st) {
  cufftSetStream(s->inv, st);
  if (sizeof(T) == 8)
    return cufft_check(cufftExecZ2D(s->inv, (cufftDoubleComplex*)s->cbuf, (cufftDoubleReal*)out), "Z2D");
  return cufft_check(cufftExecC2R(s->inv, (cufftComplex*)s->cbuf, (cufftReal*)out), "C2R");
}

template <typename T>
static int launch_tridiag(sfb_solver* s, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const int n0 = p->n[0], n1 = p->n[1], nh = p->n[2] / 2 + 1;
  dim3 grid((nh + 63) / 64, n0);
  double2* dd = sizeof(T) == 8 ? (double2*)s->cbuf : s->dscr;
  k_tridiag<T><<<grid, 64, 0, st>>>((typename CT<T>::type*)s->cbuf, dd, s->cprime, s->up, s->lo, s->di, s->dxy,
                                    s->lam[0], s->lam[2], n0, n1, nh, 1.0 / ((double)n0 * p->n[2]));
  SFB_LAUNCH_CHECK("tridiagonal");
  return SFB_OK;
}

// channel solve on the register FFT engine: FFT(x, z) -> tridiagonal(y) ->
// inverse; the divergence of u fused into the R2C when G/u are given
template <typename T>
static int channel_fft_solve(sfb_solver* s, T* buf, cudaStream_t st, const Geo<T>* G = nullptr,
                             const void* const* u = nullptr) {
  int rc;
  if ((rc = fft_channel_forward<T>(s->fft, buf, s->cbuf, st, G, u))) return rc;
  if ((rc = launch_tridiag<T>(s, st))) return rc;
  return fft_channel_inverse<T>(s->fft, s->cbuf, buf, st);
}

template <typename T>
int solve_inplace(sfb_solver* s, T* buf, cudaStream_t st) {
  // buf: contiguous interior rhs in, solution out
  sfb_plan* p = s->plan;
  int rc;
  if (s->kind == SFB_SOLVER_CG) return cg_solve<T>(s, buf, st);
  if (s->kind == SFB_SOLVER_CHANNEL && s->fft.enabled) return channel_fft_solve<T>(s, buf, st);
  if (s->fft.enabled) return fft_solve_inplace<T>(s->fft, buf, s->cbuf, st);
  if ((rc = exec_fwd<T>(s, buf, st))) return rc;
  if (s->kind == SFB_SOLVER_SPECTRAL) {
    const int m0 = p->n[0], m1 = p->n[1];
    const int mh = p->n[p->dim - 1] / 2 + 1;
    const double N = (double)p->int_count;
    const T invN = (T)(1.0 / N);
    int nb = 148 * 8;
    SFB_DISPATCH_DIM(p->dim, D,
                     (k_spec_scale<T, D><<<nb, 256, 0, st>>>((typename CT<T>::type*)s->cbuf, s->lam[0], s->lam[1],
                                                             s->lam[2], m0, m1, mh, invN)));
    SFB_LAUNCH_CHECK("spectral scale");
  } else if ((rc = launch_tridiag<T>(s, st))) {
    return rc;
  }
  return exec_inv<T>(s, buf, st);
}
template int solve_inplace<double>(sfb_solver*, double*, cudaStream_t);
template int solve_inplace<float>(sfb_solver*, float*, cudaStream_t);

template <typename T>
static bool divfused(const sfb_solver* s) {
  if (s->kind == SFB_SOLVER_CHANNEL) return s->fft.enabled && fft_channel_divfuse_ok<T>(s->fft, geo<T>(s->plan));
  return s->fft.enabled && (fft_divfuse_ok<T>(s->fft, geo<T>(s->plan)) || getenv("SFB_DIVFUSE"));
}

// divergence -> solve; the pressure interior is left in s->rbuf
template <typename T>
static int project_solve(sfb_solver* s, const void* const* u, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  CV<T> C;
  for (int a = 0; a < 3; ++a) C.c[a] = a < p->dim ? (const T*)u[a] : nullptr;
  T* rb = (T*)s->rbuf;
  int rc;
  if (divfused<T>(s)) {
    // divergence fused into the first FFT pass
    if (s->kind == SFB_SOLVER_CHANNEL) {
      if ((rc = channel_fft_solve<T>(s, rb, st, &G, u))) return rc;
    } else if ((rc = fft_solve_inplace<T>(s->fft, rb, s->cbuf, st, &G, u))) {
      return rc;
    }
  } else {
    if ((rc = launch_div<T>(G, C, rb, st))) return rc;
    if ((rc = solve_inplace<T>(s, rb, st))) return rc;
  }
  return SFB_OK;
}

template <typename T>
static int project(sfb_solver* s, void* const* u, void* p_ext, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  MV<T> U;
  for (int a = 0; a < 3; ++a) U.c[a] = a < p->dim ? (T*)u[a] : nullptr;
  int rc;
  if ((rc = project_solve<T>(s, (const void* const*)u, st))) return rc;
  if ((rc = launch_grad<T>(G, (T*)s->rbuf, U, (T*)p_ext, st))) return rc;
  if ((rc = launch_planes<T>(G, U, p->dim, 0, st))) return rc;
  if (p_ext) {
    // pressure ghosts (fields.py:81-93) from the interior just written
    if ((rc = launch_planes<T>(G, MV<T>{{(T*)p_ext, nullptr, nullptr}}, 1, 1, st))) return rc;
  }
  return SFB_OK;
}

// Register-engine FFT(x, z) for the channel solver when the x length and the
// half z length have an instantiated engine (else cuFFT plans, make_plans)
static int setup_fft_channel(sfb_solver* s) {
  sfb_plan* p = s->plan;
  FftSolve& F = s->fft;
  const bool f64 = p->dtype == SFB_F64;
  const int n0 = p->n[0], n2 = p->n[2];
  if (p->dim != 3 || n2 % 2 != 0) return SFB_OK;
  FftLen half, ax0;
  if (!fft_factor(n2 / 2, half) || !fft_factor(n0, ax0)) return SFB_OK;
  int rc;
  if ((rc = (f64 ? fft_set_smem_limits<double>() : fft_set_smem_limits<float>()))) return rc;
  F.dim = 3;
  for (int a = 0; a < 3; ++a) F.n[a] = p->n[a];
  F.total = p->int_count;
  F.half = half;
  F.ax[0] = ax0;
  F.ax[1] = ax0;  // unused (the y direction is the tridiagonal solve)
  if ((rc = fft_upload_pass_twiddles(F.ax[0], f64, &F.tw_ax[0]))) return rc;
  if ((rc = fft_upload_pass_twiddles(F.half, f64, &F.tw_half))) return rc;
  if ((rc = fft_upload_twiddles(n2, f64, &F.tw_full))) return rc;
  fft_reg_assign(F);
  if (!F.reg_half || !F.reg_ax[0]) return SFB_OK;
  F.enabled = true;
  return SFB_OK;
}

// Hand-written FFT path for the spectral solve when every axis length
// factors into 2/3/5/7, the last axis is even and a tile fits in smem.
static int setup_fft(sfb_solver* s) {
  sfb_plan* p = s->plan;
  FftSolve& F = s->fft;
  const bool f64 = p->dtype == SFB_F64;
  const size_t csz = f64 ? 16 : 8;
  const int dim = p->dim, nlast = p->n[dim - 1];
  if (nlast % 2 != 0 || nlast < 2) return SFB_OK;
  FftLen half, ax[3];
  if (!fft_factor(nlast / 2, half)) return SFB_OK;
  if (2 * (size_t)(nlast / 2) * csz > 200 * 1024) return SFB_OK;
  for (int a = 0; a < dim - 1; ++a) {
    if (!fft_factor(p->n[a], ax[a])) return SFB_OK;
    if (2 * (size_t)p->n[a] * csz > 200 * 1024) return SFB_OK;
  }
  int rc;
  if ((rc = (f64 ? fft_set_smem_limits<double>() : fft_set_smem_limits<float>()))) return rc;
  F.dim = dim;
  for (int a = 0; a < 3; ++a) F.n[a] = a < dim ? p->n[a] : 1;
  F.total = p->int_count;
  F.half = half;
  for (int a = 0; a < dim - 1; ++a) {
    F.ax[a] = ax[a];
    if ((rc = fft_upload_pass_twiddles(F.ax[a], f64, &F.tw_ax[a]))) return rc;
  }
  if ((rc = fft_upload_pass_twiddles(F.half, f64, &F.tw_half))) return rc;
  if ((rc = fft_upload_twiddles(nlast, f64, &F.tw_full))) return rc;
  F.sc.dim = dim;
  F.sc.nh = dim == 3 ? nlast / 2 + 1 : 0;
  F.sc.l0 = s->lam[0];
  F.sc.l1 = s->lam[1];
  F.sc.l2 = s->lam[2];
  F.sc.invN = 1.0 / (double)p->int_count;
  F.sc.zero_ok = 1;
  fft_reg_assign(F);
  F.enabled = true;
  // tiled spectrum when every pass runs in the register engine (fft.cu)
  F.tlog = 0;
  if (dim == 3 && F.reg_half && F.reg_ax[0] && F.reg_ax[1] && !getenv("SFB_FFT_NATURAL")) {
    const int w1 = reg_strided_w(p->n[1], f64);
    const int tw = env_int("SFB_FFT_TILE", w1);
    int lg = 0;
    while ((1 << lg) < tw) ++lg;
    // the row kernels' tiled walk (sfb_fft_reg.cuh kTileIt) covers blocks of
    // 4 or 8 columns, at most one block per thread group of a row
    const int tt = F.reg_a_half > F.reg_b_half ? F.reg_a_half : F.reg_b_half;
    if ((1 << lg) == tw && (tw == 4 || tw == 8) && tw <= tt && tw % w1 == 0) {
      F.tlog = lg;
      F.tks = (long long)p->n[0] * p->n[1] * tw;
      // hybrid (default, axis-1 kernel width only): a separate tiled copy;
      // SFB_FFT_TILED_ROWS=1 tiles the row passes' spectrum too (measured
      // slower: the row kernels lose more than the copy costs)
      if (tw == w1 && !getenv("SFB_FFT_TILED_ROWS")) {
        const long long nblk = (p->n[2] / 2 + 1 + tw - 1) / tw;
        const size_t bytes = (f64 ? 16 : 8) * (size_t)nblk * F.tks;
        if ((rc = cuda_check(cudaMalloc(&s->tbuf, bytes), "cudaMalloc(tiled spectrum)"))) return rc;
        if ((rc = cuda_check(cudaMemset(s->tbuf, 0, bytes), "cudaMemset(tiled spectrum)"))) return rc;
        F.tbuf = s->tbuf;
      }
    }
  }
  if (dim == 3 && !getenv("SFB_NO_TMA") && !F.tlog) {
    const int n0 = p->n[0], n1 = p->n[1];
    const long long nh = nlast / 2 + 1;
    // axis-1 pass: box over (nh complex columns, n1 rows, n0 batch); axis-0: (n1*nh, n0)
    if (fft_tma_fits(n1, f64) && (rc = fft_tma_make(F.tma_ax1, s->cbuf, f64, 3, nh, n1, n0, n1))) return rc;
    if (fft_tma_fits(n0, f64) && (rc = fft_tma_make(F.tma_ax0, s->cbuf, f64, 2, (long long)n1 * nh, n0, 1, n0)))
      return rc;
  }
  return SFB_OK;
}

static bool axis_uniform(const std::vector<double>& dx) {
  // grid.py:177-183: allclose(widths, widths[0], rtol=1e-12) on interior widths
  const size_t n = dx.size() - 2;
  for (size_t i = 1; i <= n; ++i)
    if (std::fabs(dx[i] - dx[1]) > 1e-12 * std::fabs(dx[1])) return false;
  return true;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_solver_create(sfb_plan* p, int kind, sfb_solver** out) {
  if (!p || !out) return fail(SFB_EINVAL, "null argument");
  *out = nullptr;
  if (kind == SFB_SOLVER_SPECTRAL) {
    if (!p->all_periodic) return fail(SFB_ECONFIG, "spectral pressure solver requires periodic axes");
    for (int a = 0; a < p->dim; ++a)
      if (!axis_uniform(p->hdx[a])) return fail(SFB_ECONFIG, "spectral pressure solver requires uniform axes");
  } else if (kind == SFB_SOLVER_CHANNEL) {
    if (p->dim != 3 || p->bc_lo[0] != SFB_BC_PERIODIC || p->bc_lo[2] != SFB_BC_PERIODIC ||
        p->bc_lo[1] == SFB_BC_PERIODIC)
      return fail(SFB_ECONFIG, "channel pressure solver requires periodic x/z and walls on y");
    if (!axis_uniform(p->hdx[0]) || !axis_uniform(p->hdx[2]))
      return fail(SFB_ECONFIG, "channel pressure solver requires uniform x/z");
  } else if (kind == SFB_SOLVER_CG) {
    for (int a = 0; a < p->dim; ++a)
      if (p->bc_lo[a] == SFB_BC_HALO) return fail(SFB_ECONFIG, "the CG solver does not run on slab plans");
    sfb_solver* s = new sfb_solver();
    s->plan = p;
    s->kind = kind;
    const size_t esz = p->dtype == SFB_F64 ? 8 : 4;
    int rc = cuda_check(cudaMalloc(&s->rbuf, esz * p->int_count), "cudaMalloc(rbuf)");
    if (!rc) rc = cg_setup(s);
    if (rc) {
      sfb_solver_destroy(s);
      return rc;
    }
    *out = s;
    return SFB_OK;
  } else {
    return fail(SFB_ECONFIG, "unknown pressure solver kind");
  }
  sfb_solver* s = new sfb_solver();
  s->plan = p;
  s->kind = kind;
  const size_t esz = p->dtype == SFB_F64 ? 8 : 4;
  const int dlast = p->dim - 1;
  const long long nh = p->n[dlast] / 2 + 1;
  const long long ncomplex = p->int_count / p->n[dlast] * nh;
  int rc;
  std::vector<double> host[3];
  if ((rc = cuda_check(cudaMalloc(&s->rbuf, esz * p->int_count), "cudaMalloc(rbuf)"))) goto bad;
  // room for the tiled spectrum (fft.cu): nh padded to a multiple of the
  // widest column block (8); zeroed once so the padding columns the axis-0
  // pass transforms are finite
  {
    const long long cpad = kind == SFB_SOLVER_SPECTRAL ? p->int_count / p->n[dlast] * ((nh + 7) / 8 * 8) : ncomplex;
    if ((rc = cuda_check(cudaMalloc(&s->cbuf, 2 * esz * cpad), "cudaMalloc(cbuf)"))) goto bad;
    if ((rc = cuda_check(cudaMemset(s->cbuf, 0, 2 * esz * cpad), "cudaMemset(cbuf)"))) goto bad;
  }
  // eigenvalue tables lam_a[k] = (2 cos(2 pi k / n) - 2) / h^2 (poisson.py:180-186)
  for (int a = 0; a < 3; ++a) {
    int n = a < p->dim ? p->n[a] : 1;
    host[a].resize(n);
    double h = p->width0[a];
    for (int k = 0; k < n; ++k)
      host[a][k] = a < p->dim && !(kind == SFB_SOLVER_CHANNEL && a == 1)
                       ? (2.0 * std::cos(2.0 * M_PI * k / n) - 2.0) / (h * h)
                       : 0.0;
    if ((rc = cuda_check(cudaMalloc(&s->lam[a], sizeof(double) * n), "cudaMalloc(lam)"))) goto bad;
    if ((rc = cuda_check(cudaMemcpy(s->lam[a], host[a].data(), sizeof(double) * n, cudaMemcpyHostToDevice), "upload")))
      goto bad;
  }
  if (kind == SFB_SOLVER_SPECTRAL && !getenv("SFB_FORCE_CUFFT")) {
    if ((rc = setup_fft(s))) goto bad;
  }
  if (kind == SFB_SOLVER_CHANNEL && !getenv("SFB_FORCE_CUFFT")) {
    if ((rc = setup_fft_channel(s))) goto bad;
  }
  if (!s->fft.enabled && (rc = make_plans(s))) goto bad;
  if (kind == SFB_SOLVER_CHANNEL) {
    // tridiagonal coefficients from the reference's y tables (fp64)
    const int n1 = p->n[1];
    std::vector<double> up(n1 + 2, 0.0), lo(n1 + 2, 0.0), di(n1 + 2, 0.0), dxy(n1);
    const std::vector<double>& dx = p->hdx[1];
    const std::vector<double>& du = p->hdu[1];
    for (int j = 1; j < n1; ++j) up[j] = 1.0 / (du[j] * dx[j]);
    for (int j = 2; j <= n1; ++j) lo[j] = 1.0 / (du[j - 1] * dx[j]);
    for (int j = 1; j <= n1; ++j) {
      di[j] = -(up[j] + lo[j]);
      dxy[j - 1] = dx[j];
    }
    double** dst[4] = {&s->up, &s->lo, &s->di, &s->dxy};
    std::vector<double>* src[4] = {&up, &lo, &di, &dxy};
    for (int t = 0; t < 4; ++t) {
      size_t bytes = sizeof(double) * src[t]->size();
      if ((rc = cuda_check(cudaMalloc(dst[t], bytes), "cudaMalloc(tri)"))) goto bad;
      if ((rc = cuda_check(cudaMemcpy(*dst[t], src[t]->data(), bytes, cudaMemcpyHostToDevice), "upload"))) goto bad;
    }
    if ((rc = cuda_check(cudaMalloc(&s->cprime, sizeof(double) * ncomplex), "cudaMalloc(cprime)"))) goto bad;
    if (p->dtype == SFB_F32 &&
        (rc = cuda_check(cudaMalloc(&s->dscr, sizeof(double2) * ncomplex), "cudaMalloc(dscr)")))
      goto bad;
  }
  *out = s;
  return SFB_OK;
bad:
  sfb_solver_destroy(s);
  return rc;
}

int sfb_solver_uses_own_fft(const sfb_solver* s) { return s && s->fft.enabled ? 1 : 0; }

int sfb_solver_destroy(sfb_solver* s) {
  if (!s) return SFB_OK;
  if (s->has_fwd) cufftDestroy(s->fwd);
  if (s->has_inv) cufftDestroy(s->inv);
  cg_release(s);
  if (s->tbuf == s->cbuf) s->tbuf = nullptr;  // P = 1 alias
  void* bufs[] = {s->tbuf, s->xbuf, s->work, s->rbuf, s->cbuf, s->cprime, s->dscr, s->lam[0], s->lam[1], s->lam[2],
                  s->up, s->lo, s->di, s->dxy, s->tmp, s->fft.tw_half, s->fft.tw_full,
                  s->fft.tw_ax[0], s->fft.tw_ax[1], s->fft.tw_ax[2]};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete s;
  return SFB_OK;
}

int sfb_solver_solve(sfb_solver* s, const void* rhs, void* out, void* stream) {
  SFB_RANGE();
  if (!s || !rhs || !out) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  sfb_plan* p = s->plan;
  const size_t bytes = (p->dtype == SFB_F64 ? 8 : 4) * (size_t)p->int_count;
  int rc;
  if ((rc = cuda_check(cudaMemcpyAsync(s->rbuf, rhs, bytes, cudaMemcpyDeviceToDevice, st), "copy rhs"))) return rc;
  rc = p->dtype == SFB_F64 ? solve_inplace<double>(s, (double*)s->rbuf, st) : solve_inplace<float>(s, (float*)s->rbuf, st);
  if (rc) return rc;
  return cuda_check(cudaMemcpyAsync(out, s->rbuf, bytes, cudaMemcpyDeviceToDevice, st), "copy out");
}

int sfb_project_solve(sfb_solver* s, const void* const* u, const void** p_int, void* stream) {
  SFB_RANGE();
  if (!s || !u || !p_int) return fail(SFB_EINVAL, "null argument");
  if (s->slab) return fail(SFB_ECONFIG, "sfb_project_solve: slab solvers use the sfb_slab_* sequence");
  for (int a = 0; a < s->plan->dim; ++a)
    if (!u[a]) return fail(SFB_EINVAL, "null velocity component");
  const int rc = s->plan->dtype == SFB_F64 ? project_solve<double>(s, u, (cudaStream_t)stream)
                                           : project_solve<float>(s, u, (cudaStream_t)stream);
  *p_int = rc ? nullptr : s->rbuf;
  return rc;
}

int sfb_project_finish(sfb_solver* s, void* const* u, void* p_ext, void* stream) {
  SFB_RANGE();
  if (!s || !u) return fail(SFB_EINVAL, "null argument");
  if (s->slab) return fail(SFB_ECONFIG, "sfb_project_finish: slab solvers use sfb_slab_correct");
  for (int a = 0; a < s->plan->dim; ++a)
    if (!u[a]) return fail(SFB_EINVAL, "null velocity component");
  return SFB_TYPED(s->plan, ([&]() {
    sfb_plan* p = s->plan;
    const Geo<T>& G = geo<T>(p);
    cudaStream_t st = (cudaStream_t)stream;
    MV<T> U;
    for (int a = 0; a < 3; ++a) U.c[a] = a < p->dim ? (T*)u[a] : nullptr;
    int rc;
    if ((rc = launch_grad<T>(G, (T*)s->rbuf, U, (T*)p_ext, st))) return rc;
    if ((rc = launch_planes<T>(G, U, p->dim, 0, st))) return rc;
    if (p_ext && (rc = launch_planes<T>(G, MV<T>{{(T*)p_ext, nullptr, nullptr}}, 1, 1, st))) return rc;
    return (int)SFB_OK;
  })());
}

int sfb_project_launches(const sfb_solver* s, int mode) {
  if (!s) return 0;
  const bool fused = s->plan->dtype == SFB_F64 ? divfused<double>(s) : divfused<float>(s);
  if (mode == 3) return fused ? 1 : 2;  // sfb_slab_r2c
  int n;
  if (s->fft.enabled) n = (s->plan->dim == 3 ? 5 : 3) + (fused ? 0 : 1);
  else if (s->kind == SFB_SOLVER_CG) n = 1 + 4 + 7 * s->cg_iters;  // divergence, CG init, CG iterations
  else n = 2;  // divergence + eigenvalue scaling / tridiagonal (cuFFT transforms not counted)
  if (mode == 2) return n;
  return n + 2 + (mode == 1 ? 1 : 0);  // gradient subtract, velocity ghosts (+ pressure ghosts)
}

int sfb_project(sfb_solver* s, void* const* u, void* p_ext, void* stream) {
  SFB_RANGE();
  if (!s || !u) return fail(SFB_EINVAL, "null argument");
  for (int a = 0; a < s->plan->dim; ++a)
    if (!u[a]) return fail(SFB_EINVAL, "null velocity component");
  return s->plan->dtype == SFB_F64 ? project<double>(s, u, p_ext, (cudaStream_t)stream)
                                   : project<float>(s, u, p_ext, (cudaStream_t)stream);
}


// ---------------------------------------------------------------------------
// slab-decomposed spectral solve (multi-GPU)
// ---------------------------------------------------------------------------
int sfb_slab_solver_create(sfb_plan* p, int n0g, int rank, int nranks, sfb_solver** out) {
  if (!p || !out) return fail(SFB_EINVAL, "null argument");
  *out = nullptr;
  if (p->dim != 3 || p->bc_lo[0] != SFB_BC_HALO || p->bc_lo[1] != SFB_BC_PERIODIC || p->bc_lo[2] != SFB_BC_PERIODIC)
    return fail(SFB_ECONFIG, "slab solver needs a 3D plan with a halo axis 0 and periodic axes 1, 2");
  const int m = p->n[0], n1 = p->n[1], n2 = p->n[2];
  if (nranks < 1 || rank < 0 || rank >= nranks || n0g != m * nranks || n1 % nranks != 0 || n2 % 2 != 0)
    return fail(SFB_ECONFIG, "slab solver needs n0 = m*P, n1 % P == 0 and an even n2");
  for (int a = 1; a < 3; ++a)
    if (!axis_uniform(p->hdx[a])) return fail(SFB_ECONFIG, "spectral pressure solver requires uniform axes");
  FftLen half, a0, a1;
  if (!fft_factor(n2 / 2, half) || !fft_factor(n0g, a0) || !fft_factor(n1, a1) || n0g > 3584 || n1 > 3584 ||
      n2 / 2 > 2048)
    return fail(SFB_ECONFIG, "slab solver: axis lengths must factor into 2, 3, 5, 7");
  sfb_solver* s = new sfb_solver();
  s->plan = p;
  s->kind = SFB_SOLVER_SPECTRAL;
  s->slab = true;
  s->n0g = n0g;
  s->rank = rank;
  s->nranks = nranks;
  const bool f64 = p->dtype == SFB_F64;
  const size_t esz = f64 ? 8 : 4;
  const long long nh = n2 / 2 + 1;
  const long long ncomplex = (long long)m * n1 * nh;
  int rc;
  double h[3] = {p->width0[0], p->width0[1], p->width0[2]};
  int ng[3] = {n0g, n1, n2};
  FftSolve& F = s->fft;
  // pressure planes [prev's last | m local | next's first two] (ext indices 0..m+2)
  if ((rc = cuda_check(cudaMalloc(&s->rbuf, esz * (size_t)(m + 3) * n1 * n2), "cudaMalloc(rbuf)"))) goto bad;
  if ((rc = cuda_check(cudaMalloc(&s->cbuf, 2 * esz * ncomplex), "cudaMalloc(spec)"))) goto bad;
  if (nranks > 1) {
    if ((rc = cuda_check(cudaMalloc(&s->tbuf, 2 * esz * ncomplex), "cudaMalloc(trans)"))) goto bad;
    if ((rc = cuda_check(cudaMalloc(&s->xbuf, 2 * esz * ncomplex), "cudaMalloc(exchange)"))) goto bad;
  } else {
    s->tbuf = s->cbuf;  // one rank: the axis-0 pass runs on the spectrum in place
  }
  for (int a = 0; a < 3; ++a) {
    std::vector<double> lam(ng[a]);
    for (int k = 0; k < ng[a]; ++k) lam[k] = (2.0 * std::cos(2.0 * M_PI * k / ng[a]) - 2.0) / (h[a] * h[a]);
    if ((rc = cuda_check(cudaMalloc(&s->lam[a], sizeof(double) * ng[a]), "cudaMalloc(lam)"))) goto bad;
    if ((rc = cuda_check(cudaMemcpy(s->lam[a], lam.data(), sizeof(double) * ng[a], cudaMemcpyHostToDevice), "upload")))
      goto bad;
  }
  if ((rc = (f64 ? fft_set_smem_limits<double>() : fft_set_smem_limits<float>()))) goto bad;
  F.dim = 3;
  F.n[0] = m;
  F.n[1] = n1;
  F.n[2] = n2;
  F.total = (long long)m * n1 * n2;
  F.half = half;
  F.ax[0] = a0;
  F.ax[1] = a1;
  if ((rc = fft_upload_pass_twiddles(F.ax[0], f64, &F.tw_ax[0]))) goto bad;
  if ((rc = fft_upload_pass_twiddles(F.ax[1], f64, &F.tw_ax[1]))) goto bad;
  if ((rc = fft_upload_pass_twiddles(F.half, f64, &F.tw_half))) goto bad;
  if ((rc = fft_upload_twiddles(n2, f64, &F.tw_full))) goto bad;
  F.sc.dim = 3;
  F.sc.nh = (int)nh;
  F.sc.l0 = s->lam[0];
  F.sc.l1 = s->lam[1] + (long long)rank * (n1 / nranks);
  F.sc.l2 = s->lam[2];
  F.sc.invN = 1.0 / ((double)n0g * n1 * n2);
  F.sc.zero_ok = rank == 0;
  fft_reg_assign(F);
  F.enabled = true;
  if (!getenv("SFB_NO_TMA")) {
    if (fft_tma_fits(n1, f64) && (rc = fft_tma_make(F.tma_ax1, s->cbuf, f64, 3, nh, n1, m, n1))) goto bad;
    if (fft_tma_fits(n0g, f64) &&
        (rc = fft_tma_make(F.tma_ax0, s->tbuf, f64, 2, (long long)(n1 / nranks) * nh, n0g, 1, n0g)))
      goto bad;
  }
  *out = s;
  return SFB_OK;
bad:
  sfb_solver_destroy(s);
  return rc;
}

int sfb_slab_buffers(sfb_solver* s, void** spec, void** trans, void** xchg, void** p_slab, void** p_local,
                     void** p_halo) {
  if (!s || !s->slab) return fail(SFB_EINVAL, "not a slab solver");
  sfb_plan* p = s->plan;
  const size_t esz = p->dtype == SFB_F64 ? 8 : 4;
  if (spec) *spec = s->cbuf;
  if (trans) *trans = s->tbuf;
  if (xchg) *xchg = s->xbuf;
  const size_t plane = esz * (size_t)p->n[1] * p->n[2];
  if (p_slab) *p_slab = s->rbuf;
  if (p_local) *p_local = (char*)s->rbuf + plane;
  if (p_halo) *p_halo = (char*)s->rbuf + plane * (1 + (size_t)p->n[0]);
  return SFB_OK;
}

}  // extern "C"

namespace sfb {
// the local pressure planes start one plane into the slab pressure buffer
template <typename T>
static T* slab_local(sfb_solver* s) {
  return (T*)s->rbuf + (size_t)s->plan->n[1] * s->plan->n[2];
}

template <typename T>
static int slab_r2c(sfb_solver* s, void* const* u, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  if (fft_divfuse_ok<T>(s->fft, G))
    return fft_slab_r2c<T>(s->fft, slab_local<T>(s), s->cbuf, st, &G, (const void* const*)u);
  CV<T> C;
  for (int a = 0; a < 3; ++a) C.c[a] = (const T*)u[a];
  int rc = launch_div<T>(G, C, slab_local<T>(s), st);
  if (rc) return rc;
  return fft_slab_r2c<T>(s->fft, slab_local<T>(s), s->cbuf, st, nullptr, nullptr);
}

template <typename T>
static int slab_correct(sfb_solver* s, void* const* u, void* p_ext, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  MV<T> U;
  for (int a = 0; a < 3; ++a) U.c[a] = (T*)u[a];
  Box B = int_box(G);
  int rc = launch_grad<T>(G, (const T*)slab_local<T>(s), U, (T*)p_ext, st);
  if (rc) return rc;
  rc = launch_planes<T>(G, U, 3, 0, st);
  if (rc) return rc;
  if (p_ext && (rc = launch_planes<T>(G, MV<T>{{(T*)p_ext, nullptr, nullptr}}, 1, 1, st))) return rc;
  return SFB_OK;
}
}  // namespace sfb

extern "C" {

int sfb_slab_r2c(sfb_solver* s, void* const* u, void* stream) {
  SFB_RANGE();
  if (!s || !s->slab || !u || !u[0] || !u[1] || !u[2]) return fail(SFB_EINVAL, "bad slab call");
  return s->plan->dtype == SFB_F64 ? slab_r2c<double>(s, u, (cudaStream_t)stream)
                                   : slab_r2c<float>(s, u, (cudaStream_t)stream);
}

int sfb_slab_max_chunks(const sfb_solver* s) {
  if (!s || !s->slab) return 0;
  return s->fft.reg_ax[1] ? s->plan->n[2] / 2 + 1 : 1;
}

int sfb_slab_axis1(sfb_solver* s, int chunk, int nchunks, int inverse, void* stream) {
  SFB_RANGE();
  if (!s || !s->slab || nchunks < 1 || chunk < 0 || chunk >= nchunks) return fail(SFB_EINVAL, "bad slab call");
  return s->plan->dtype == SFB_F64
             ? fft_slab_axis1<double>(s->fft, s->cbuf, s->xbuf, s->nranks, chunk, nchunks, inverse != 0,
                                      (cudaStream_t)stream)
             : fft_slab_axis1<float>(s->fft, s->cbuf, s->xbuf, s->nranks, chunk, nchunks, inverse != 0,
                                     (cudaStream_t)stream);
}

int sfb_slab_axis0(sfb_solver* s, int chunk, int nchunks, void* stream) {
  SFB_RANGE();
  if (!s || !s->slab || nchunks < 1 || chunk < 0 || chunk >= nchunks) return fail(SFB_EINVAL, "bad slab call");
  const int c = s->plan->n[1] / s->nranks;
  return s->plan->dtype == SFB_F64
             ? fft_slab_axis0<double>(s->fft, s->tbuf, c, s->nranks, chunk, nchunks, (cudaStream_t)stream)
             : fft_slab_axis0<float>(s->fft, s->tbuf, c, s->nranks, chunk, nchunks, (cudaStream_t)stream);
}

int sfb_slab_c2r(sfb_solver* s, void* stream) {
  SFB_RANGE();
  if (!s || !s->slab) return fail(SFB_EINVAL, "bad slab call");
  return s->plan->dtype == SFB_F64 ? fft_slab_c2r<double>(s->fft, s->cbuf, slab_local<double>(s), (cudaStream_t)stream)
                                   : fft_slab_c2r<float>(s->fft, s->cbuf, slab_local<float>(s), (cudaStream_t)stream);
}

int sfb_slab_correct(sfb_solver* s, void* const* u, void* p_ext, void* stream) {
  SFB_RANGE();
  if (!s || !s->slab || !u || !u[0] || !u[1] || !u[2]) return fail(SFB_EINVAL, "bad slab call");
  return s->plan->dtype == SFB_F64 ? slab_correct<double>(s, u, p_ext, (cudaStream_t)stream)
                                   : slab_correct<float>(s, u, p_ext, (cudaStream_t)stream);
}

}  // extern "C"
