// Forward stencils, ghost fills, RK combines and reductions (sm_100a).
//
// Reference: operators.py:108-301 (stencils), fields.py:81-140 (fills),
// timestep.py:140-250 (axpy / stage combine / CFL).  The hot fused RK-stage
// kernel lives in stage.cu; this file holds the generic (any BC, 2D/3D)
// kernels behind the drop-in operator API.
#include <cmath>
#include <vector>

#include "sfb_kernels.cuh"

namespace sfb {

// ---------------------------------------------------------------------------
// Ghost fill as a composed affine map (fields.py:81-140).
//
// The reference fills axis 0, then 1, then 2; each fill copies whole planes
// (incl. ghosts of the other axes).  The final value of a boundary entry is
// therefore  v = k_a0 + s_a0*( ... (k_aN + s_aN * x) )  where the chain walks
// the axes whose fill targets the entry from the last axis back to the first
// and x is a DOF value.  We evaluate that chain directly per entry, so one
// launch fills every plane of every component, reading only DOF entries.
// ---------------------------------------------------------------------------

template <typename T, int D>
__device__ __forceinline__ T ghost_value(const Geo<T>& G, const T* __restrict__ u, int c, const int I[3], bool scalar) {
  int J[3] = {I[0], I[1], I[2]};
  T kst[3];
  signed char sst[3];
  int nst = 0;
  bool constant = false;
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    if (constant) break;
    const int n = G.n[a];
    const int i = J[a];
    int src = i;
    signed char s = 1;
    T k = T(0);
    bool tgt = false;
    if (G.halo[a]) {
      // ghost planes supplied by the neighbouring slab: not a fill target
    } else if (G.per[a]) {
      if (i == 0) { tgt = true; src = n; }
      else if (i == n + 1) { tgt = true; src = 1; }
    } else if (scalar) {
      if (i == 0) { tgt = true; src = 1; }
      else if (i == n + 1) { tgt = true; src = n; }
    } else {
      const bool normal = (c == a);
      if (i == 0) {
        tgt = true;
        if (G.bc_lo[a] == SFB_BC_DIRICHLET) {
          if (normal) { s = 0; k = G.vlo[a][c]; }
          else { src = 1; s = -1; k = G.c2lo[a][c]; }
        } else {  // symmetric
          if (normal) { s = 0; k = T(0); }
          else { src = 1; s = 1; }
        }
      } else if (i == n + 1) {
        tgt = true;
        if (G.bc_hi[a] == SFB_BC_DIRICHLET) {
          src = normal ? n - 1 : n; s = -1; k = G.c2hi[a][c];
        } else {
          if (normal) { src = n - 1; s = -1; k = T(0); }
          else { src = n; s = 1; }
        }
      } else if (i == n && normal) {
        tgt = true;
        s = 0;
        k = (G.bc_hi[a] == SFB_BC_DIRICHLET) ? G.vhi[a][c] : T(0);
      }
    }
    if (tgt) {
      kst[nst] = k;
      sst[nst] = s;
      ++nst;
      if (s == 0) constant = true;
      else J[a] = src;
    }
  }
  T v = T(0);
  if (!constant) v = u[lin<T, D>(G, J)];
  for (int t = nst - 1; t >= 0; --t) {
    if (sst[t] == 0) v = kst[t];
    else if (sst[t] < 0) v = kst[t] - v;
  }
  return v;
}

struct PlaneSet {
  int count;
  int comp[32];
  int axis[32];
  int idx[32];
  int size[32];
};

// mode 0: velocity fill, 1: scalar fill, 2: zero velocity non-DOFs
// (adjoint.py:40-50), 3: zero scalar ghosts (adjoint.py:32-37)
template <typename T, int D>
__global__ void k_planes(Geo<T> G, MV<T> U, PlaneSet P, int mode) {
  const int pl = blockIdx.y;
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= P.size[pl]) return;
  const int c = P.comp[pl], ax = P.axis[pl];
  int I[3] = {0, 0, 0};
  I[ax] = P.idx[pl];
  int rem = pos;
#pragma unroll
  for (int b = D - 1; b >= 0; --b) {
    if (b == ax) continue;
    I[b] = rem % G.E[b];
    rem /= G.E[b];
  }
  T* __restrict__ u = U.c[c];
  const long long x = lin<T, D>(G, I);
  if (mode >= 2) u[x] = T(0);
  else u[x] = ghost_value<T, D>(G, u, c, I, mode == 1);
}

template <typename T>
static PlaneSet make_planes(const Geo<T>& G, int ncomp, bool boundary_faces) {
  PlaneSet P;
  P.count = 0;
  for (int c = 0; c < ncomp; ++c)
    for (int a = 0; a < G.dim; ++a) {
      if (G.halo[a]) continue;
      int idxs[3] = {0, G.n[a] + 1, G.n[a]};
      int ni = (boundary_faces && !G.per[a] && c == a) ? 3 : 2;
      int sz = 1;
      for (int b = 0; b < G.dim; ++b)
        if (b != a) sz *= G.E[b];
      for (int t = 0; t < ni; ++t) {
        P.comp[P.count] = c;
        P.axis[P.count] = a;
        P.idx[P.count] = idxs[t];
        P.size[P.count] = sz;
        ++P.count;
      }
    }
  return P;
}

template <typename T>
int launch_planes(const Geo<T>& G, MV<T> U, int ncomp, int mode, cudaStream_t st) {
  PlaneSet P = make_planes(G, ncomp, mode == 0 || mode == 2);
  if (P.count == 0) return SFB_OK;
  int mx = 0;
  for (int i = 0; i < P.count; ++i) mx = P.size[i] > mx ? P.size[i] : mx;
  dim3 grid((mx + 255) / 256, P.count);
  SFB_DISPATCH_DIM(G.dim, D, (k_planes<T, D><<<grid, 256, 0, st>>>(G, U, P, mode)));
  SFB_LAUNCH_CHECK("fill/zero planes");
  return SFB_OK;
}
template int launch_planes<double>(const Geo<double>&, MV<double>, int, int, cudaStream_t);
template int launch_planes<float>(const Geo<float>&, MV<float>, int, int, cudaStream_t);

// ---------------------------------------------------------------------------
// Adjoint of the ghost fills (adjoint.py:53-111): for one axis a, every
// position of the other axes' extended plane folds its two ghost entries
// onto their sources, statement for statement in the reference's order (a
// thread owns the whole line along a, so n == 1 aliasing is exact).  The
// host walks the axes in reverse, one launch per axis, as the reference
// does; blockIdx.y is the component (comp < 0: the scalar rules).
// ---------------------------------------------------------------------------
template <typename T, int D>
__global__ void k_fold(Geo<T> G, MV<T> U, int axis, int scalar) {
  const int c = blockIdx.y;
  int sz = 1;
#pragma unroll
  for (int b = 0; b < D; ++b)
    if (b != axis) sz *= G.E[b];
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= sz) return;
  int I[3] = {0, 0, 0};
  int rem = pos;
#pragma unroll
  for (int b = D - 1; b >= 0; --b) {
    if (b == axis) continue;
    I[b] = rem % G.E[b];
    rem /= G.E[b];
  }
  T* __restrict__ u = U.c[c];
  const int n = G.n[axis];
  const long long st = G.s[axis];
  const long long x0 = lin<T, D>(G, I);  // I[axis] == 0
  T* g_lo = u + x0;
  T* g_hi = u + x0 + (long long)(n + 1) * st;
  auto at = [&](int i) -> T& { return u[x0 + (long long)i * st]; };
  if (G.per[axis]) {
    at(n) += *g_lo;
    at(1) += *g_hi;
    *g_lo = T(0);
    *g_hi = T(0);
    return;
  }
  if (scalar) {
    at(1) += *g_lo;
    at(n) += *g_hi;
    *g_lo = T(0);
    *g_hi = T(0);
    return;
  }
  const bool normal = c == axis;
  if (!normal) {
    if (G.bc_lo[axis] == SFB_BC_DIRICHLET) at(1) -= *g_lo;
    else if (G.bc_lo[axis] == SFB_BC_SYMMETRIC) at(1) += *g_lo;
  }
  *g_lo = T(0);
  if (G.bc_hi[axis] == SFB_BC_DIRICHLET || G.bc_hi[axis] == SFB_BC_SYMMETRIC) {
    if (normal) {
      at(n - 1) -= *g_hi;
      at(n) = T(0);
    } else if (G.bc_hi[axis] == SFB_BC_DIRICHLET) {
      at(n) -= *g_hi;
    } else {
      at(n) += *g_hi;
    }
  }
  *g_hi = T(0);
}

template <typename T>
int launch_fold(const Geo<T>& G, MV<T> U, int ncomp, bool scalar, cudaStream_t st) {
  for (int a = G.dim - 1; a >= 0; --a) {
    if (G.halo[a]) continue;  // slab ghost planes belong to the neighbouring rank
    int sz = 1;
    for (int b = 0; b < G.dim; ++b)
      if (b != a) sz *= G.E[b];
    dim3 grid((sz + 255) / 256, ncomp);
    SFB_DISPATCH_DIM(G.dim, D, (k_fold<T, D><<<grid, 256, 0, st>>>(G, U, a, scalar ? 1 : 0)));
    SFB_LAUNCH_CHECK("fold ghosts");
  }
  return SFB_OK;
}

// ---------------------------------------------------------------------------
// divergence (operators.py:108-122): whole extended output, ghosts zero
// ---------------------------------------------------------------------------
template <typename T, int D>
__global__ void k_divergence(Geo<T> G, CV<T> U, T* __restrict__ out, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  T acc = T(0);
  if (is_pdof<T, D>(G, I)) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const T* __restrict__ ua = U.c[a];
      acc += (ua[x] - ua[x - G.s[a]]) * tab(G, a, T_RDX, I[a]);
    }
  }
  out[x] = acc;
}

// pressure_gradient (operators.py:125-137)
template <typename T, int D>
__global__ void k_gradient(Geo<T> G, const T* __restrict__ p, MV<T> O, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  const T pc = p[x];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T v = T(0);
    if (is_udof<T, D>(G, I, a)) v = (p[x + G.s[a]] - pc) * tab(G, a, T_RDU, I[a]);
    O.c[a][x] = v;
  }
}

// convection / diffusion / momentum_rhs (operators.py:140-238)
template <typename T, int D>
__global__ void k_rhs(Geo<T> G, CV<T> U, MV<T> O, Box B, T nu, Force<T> F, int flags) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  const bool conv = flags & 1, diff = flags & 2, accum = flags & 4;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T* __restrict__ o = O.c[a];
    if (is_udof<T, D>(G, I, a)) {
      T v = accum ? o[x] : T(0);
      v = rhs_comp<T, D>(G, U, x, I, a, v, conv, diff, nu, F.f[a]);
      if (F.a[a]) v += F.a[a][x];
      o[x] = v;
    } else if (!accum) {
      o[x] = T(0);
    }
  }
}

// dst = base + sum_l k_l * c_l on DOFs (timestep.py:190-207, 166-172)
template <typename T, int D>
__global__ void k_combine(Geo<T> G, MV<T> Dst, CV<T> Base, KList<T> K, int nk, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    T v = Base.c[a] ? Base.c[a][x] : T(0);
    for (int l = 0; l < nk; ++l) v += K.k[l][a][x] * K.coef[l];
    Dst.c[a][x] = v;
  }
}

// Wray3 register update (timestep.py:231-238)
template <typename T, int D>
__global__ void k_wray(Geo<T> G, MV<T> U, MV<T> Fn, MV<T> Fo, T g, T z, int has_fold, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    T f = Fn.c[a][x] * g;
    Fn.c[a][x] = f;
    T u = U.c[a][x] + f;
    if (has_fold) {
      T fo = Fo.c[a][x] * z;
      Fo.c[a][x] = fo;
      u += fo;
    }
    U.c[a][x] = u;
  }
}

// out_a = W_u,a * u_a on DOFs, zero elsewhere (kinetic_energy_pullback,
// adjoint.py:264-273; weights as operators.py:262-272)
template <typename T, int D>
__global__ void k_wscale(Geo<T> G, CV<T> U, MV<T> O, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T v = T(0);
    if (is_udof<T, D>(G, I, a)) {
      T w = T(1);
#pragma unroll
      for (int b = 0; b < D; ++b) w = w * tab(G, b, b == a ? T_DU : T_DX, I[b]);
      v = w * U.c[a][x];
    }
    O.c[a][x] = v;
  }
}

// ---------------------------------------------------------------------------
// reductions: kinetic energy / weighted inner product / CFL (deterministic
// two-pass: fixed per-block partials, then one block in fixed order)
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  return v;
}
template <int NT>
__device__ __forceinline__ double block_min(double v) {
  __shared__ double sh[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < NT / 32 ? sh[threadIdx.x] : INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  }
  return v;
}

// mode 0: sum w*u*v  (KE when v == u), mode 1: min du/|u|, reduced as
// min(-|u|/du) = -max(|u| * (1/du)) (no fp64 division per point; the finish
// inverts once)
template <typename T, int D>
__global__ void __launch_bounds__(256) k_reduce(Geo<T> G, CV<T> U, CV<T> V, int mode, double* __restrict__ part) {
  const long long total = (long long)G.n[0] * G.n[1] * (D == 3 ? G.n[2] : 1);
  const bool small = total < (1LL << 32);
  double acc = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    if (small) {  // 32-bit index arithmetic (64-bit division is a long sequence)
      unsigned r = (unsigned)t;
      if (D == 3) {
        I[2] = 1 + (int)(r % (unsigned)G.n[2]);
        r /= (unsigned)G.n[2];
      } else {
        I[2] = 0;
      }
      I[1] = 1 + (int)(r % (unsigned)G.n[1]);
      I[0] = 1 + (int)(r / (unsigned)G.n[1]);
    } else {
      long long r = t;
      if (D == 3) {
        I[2] = 1 + (int)(r % G.n[2]);
        r /= G.n[2];
      } else {
        I[2] = 0;
      }
      I[1] = 1 + (int)(r % G.n[1]);
      I[0] = 1 + (int)(r / G.n[1]);
    }
    const long long x = lin<T, D>(G, I);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (!is_udof<T, D>(G, I, a)) continue;
      const T ua = U.c[a][x];
      if (mode == 0) {
        T w = T(1);
#pragma unroll
        for (int b = 0; b < D; ++b) w = w * tab(G, b, b == a ? T_DU : T_DX, I[b]);
        acc += (double)(w * ua * V.c[a][x]);
      } else {
        const T sp = ua < T(0) ? -ua : ua;
        acc = fmin(acc, -(double)(sp * tab(G, a, T_RDU, I[a])));
      }
    }
  }
  double r = mode == 0 ? block_sum<256>(acc) : block_min<256>(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void k_finish(const double* __restrict__ part, int n, int mode, double* __restrict__ out) {
  double acc = mode == 0 ? 0.0 : INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = mode == 0 ? acc + part[i] : fmin(acc, part[i]);
  double r = mode == 0 ? block_sum<256>(acc) : block_min<256>(acc);
  if (threadIdx.x == 0) out[0] = mode == 0 ? r : (r < 0.0 ? -1.0 / r : INFINITY);
}

template <typename T>
static int reduce(sfb_plan* p, CV<T> U, CV<T> V, int mode, double* out, cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  int nb = p->red_blocks;
  long long need = (p->int_count + 255) / 256;
  if (need < nb) nb = (int)(need > 0 ? need : 1);
  SFB_DISPATCH_DIM(G.dim, D, (k_reduce<T, D><<<nb, 256, 0, st>>>(G, U, V, mode, p->d_red)));
  SFB_LAUNCH_CHECK("reduce");
  k_finish<<<1, 256, 0, st>>>(p->d_red, nb, mode, p->d_red + p->red_blocks);
  SFB_LAUNCH_CHECK("reduce finish");
  int rc = cuda_check(cudaMemcpyAsync(p->h_red, p->d_red + p->red_blocks, sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
  if (rc) return rc;
  rc = cuda_check(cudaStreamSynchronize(st), "sync");
  if (rc) return rc;
  *out = p->h_red[0];
  return SFB_OK;
}

// ---------------------------------------------------------------------------
// host entry helpers
// ---------------------------------------------------------------------------
template <typename T>
static CV<T> cv(const sfb_plan* p, const void* const* u) {
  CV<T> r;
  for (int a = 0; a < 3; ++a) r.c[a] = (a < p->dim && u) ? (const T*)u[a] : nullptr;
  return r;
}
template <typename T>
static MV<T> mv(const sfb_plan* p, void* const* u) {
  MV<T> r;
  for (int a = 0; a < 3; ++a) r.c[a] = (a < p->dim && u) ? (T*)u[a] : nullptr;
  return r;
}

static bool ptrs_ok(const sfb_plan* p, const void* const* u) {
  if (!u) return false;
  for (int a = 0; a < p->dim; ++a)
    if (!u[a]) return false;
  return true;
}

template <typename T>
static int do_rhs(sfb_plan* p, const void* const* u, void* const* out, double nu, const double* force,
                  const void* const* field, int flags, cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  Force<T> F;
  for (int a = 0; a < 3; ++a) {
    F.a[a] = (field && a < p->dim) ? (const T*)field[a] : nullptr;
    F.c[a] = nullptr;
    F.f[a] = (force && a < p->dim && !F.a[a]) ? (T)force[a] : T(0);
  }
  Box B = ext_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_rhs<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, cv<T>(p, u), mv<T>(p, out), B, (T)nu, F, flags)));
  SFB_LAUNCH_CHECK("momentum rhs");
  return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_fill_ghosts_velocity(sfb_plan* p, void* const* u, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u)) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_planes<T>(geo<T>(p), mv<T>(p, u), p->dim, 0, (cudaStream_t)stream));
}

int sfb_fill_ghosts_scalar(sfb_plan* p, void* f, void* stream) {
  SFB_RANGE();
  if (!p || !f) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_planes<T>(geo<T>(p), MV<T>{{(T*)f, nullptr, nullptr}}, 1, 1, (cudaStream_t)stream));
}

int sfb_fold_ghosts_velocity(sfb_plan* p, void* const* u, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u)) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_fold<T>(geo<T>(p), mv<T>(p, u), p->dim, false, (cudaStream_t)stream));
}

int sfb_fold_ghosts_scalar(sfb_plan* p, void* f, void* stream) {
  SFB_RANGE();
  if (!p || !f) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_fold<T>(geo<T>(p), MV<T>{{(T*)f, nullptr, nullptr}}, 1, true, (cudaStream_t)stream));
}

int sfb_zero_non_dofs_velocity(sfb_plan* p, void* const* u, void* stream) {
  if (!p || !ptrs_ok(p, u)) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_planes<T>(geo<T>(p), mv<T>(p, u), p->dim, 2, (cudaStream_t)stream));
}

int sfb_zero_ghosts_scalar(sfb_plan* p, void* f, void* stream) {
  if (!p || !f) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, launch_planes<T>(geo<T>(p), MV<T>{{(T*)f, nullptr, nullptr}}, 1, 3, (cudaStream_t)stream));
}

int sfb_divergence(sfb_plan* p, const void* const* u, void* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !out) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    Box B = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_divergence<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, cv<T>(p, u), (T*)out, B)));
    SFB_LAUNCH_CHECK("divergence");
    return (int)SFB_OK;
  })());
}

int sfb_pressure_gradient(sfb_plan* p, const void* pf, void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !pf || !ptrs_ok(p, out)) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    Box B = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_gradient<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, (const T*)pf, mv<T>(p, out), B)));
    SFB_LAUNCH_CHECK("pressure gradient");
    return (int)SFB_OK;
  })());
}

int sfb_convection(sfb_plan* p, const void* const* u, void* const* out, int accumulate, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, out)) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, do_rhs<T>(p, u, out, 0.0, nullptr, nullptr, 1 | (accumulate ? 4 : 0), (cudaStream_t)stream));
}

int sfb_diffusion(sfb_plan* p, const void* const* u, double nu, void* const* out, int accumulate, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, out)) return fail(SFB_EINVAL, "null argument");
  if (nu < 0) return fail(SFB_EINVAL, "viscosity must be nonnegative");
  return SFB_TYPED(p, do_rhs<T>(p, u, out, nu, nullptr, nullptr, 2 | (accumulate ? 4 : 0), (cudaStream_t)stream));
}

int sfb_momentum_rhs(sfb_plan* p, const void* const* u, double nu, const double* force, const void* const* force_field,
                     void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, out)) return fail(SFB_EINVAL, "null argument");
  if (nu < 0) return fail(SFB_EINVAL, "viscosity must be nonnegative");
  int flags = 1 | (nu != 0.0 ? 2 : 0);
  return SFB_TYPED(p, do_rhs<T>(p, u, out, nu, force, force_field, flags, (cudaStream_t)stream));
}

int sfb_combine(sfb_plan* p, void* const* dst, const void* const* base, int nk, const void* const* k,
                const double* coef, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, dst) || nk < 0 || nk > SFB_MAX_K) return fail(SFB_EINVAL, "bad combine args");
  if (base && !base[0]) base = nullptr;  // all-NULL base: zero
  if (base && !ptrs_ok(p, base)) return fail(SFB_EINVAL, "bad combine base");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    KList<T> K;
    for (int l = 0; l < nk; ++l) {
      for (int a = 0; a < 3; ++a) K.k[l][a] = a < p->dim ? (const T*)k[3 * l + a] : nullptr;
      K.coef[l] = (T)coef[l];
    }
    Box B = int_box(G);
    CV<T> bb = base ? cv<T>(p, base) : CV<T>{{nullptr, nullptr, nullptr}};
    SFB_DISPATCH_DIM(G.dim, D, (k_combine<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, mv<T>(p, dst), bb, K, nk, B)));
    SFB_LAUNCH_CHECK("combine");
    return (int)SFB_OK;
  })());
}

int sfb_wray_update(sfb_plan* p, void* const* u, void* const* fnew, void* const* fold, double g, double z, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, fnew)) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int has_fold = fold && fold[0];
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    Box B = int_box(G);
    MV<T> fo = has_fold ? mv<T>(p, fold) : mv<T>(p, fnew);
    SFB_DISPATCH_DIM(G.dim, D, (k_wray<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, mv<T>(p, u), mv<T>(p, fnew), fo, (T)g, (T)z, has_fold, B)));
    SFB_LAUNCH_CHECK("wray update");
    return (int)SFB_OK;
  })());
}

int sfb_weighted_scale(sfb_plan* p, const void* const* u, void* const* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, out)) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() {
    const Geo<T>& G = geo<T>(p);
    Box B = ext_box(G);
    SFB_DISPATCH_DIM(G.dim, D, (k_wscale<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, cv<T>(p, u), mv<T>(p, out), B)));
    SFB_LAUNCH_CHECK("weighted scale");
    return (int)SFB_OK;
  })());
}

int sfb_kinetic_energy(sfb_plan* p, const void* const* u, double* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !out) return fail(SFB_EINVAL, "null argument");
  double s = 0;
  int rc = SFB_TYPED(p, reduce<T>(p, cv<T>(p, u), cv<T>(p, u), 0, &s, (cudaStream_t)stream));
  if (rc) return rc;
  *out = 0.5 * s;
  return SFB_OK;
}

int sfb_weighted_inner(sfb_plan* p, const void* const* u, const void* const* v, double* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !ptrs_ok(p, v) || !out) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, reduce<T>(p, cv<T>(p, u), cv<T>(p, v), 0, out, (cudaStream_t)stream));
}

int sfb_cfl_conv(sfb_plan* p, const void* const* u, double* out, void* stream) {
  SFB_RANGE();
  if (!p || !ptrs_ok(p, u) || !out) return fail(SFB_EINVAL, "null argument");
  return SFB_TYPED(p, reduce<T>(p, cv<T>(p, u), cv<T>(p, u), 1, out, (cudaStream_t)stream));
}

}  // extern "C"
