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
#include "sfb_kernels.cuh"

namespace sfb {

template <typename T>
struct StageArgs {
  CV<T> y, u0, s_in;
  MV<T> s_out, y_next, k_out;
  T cb, ca, nu;
  Force<T> F;
  int has_s, has_next, has_k, s_from_u0, diff;
};

template <typename T, int D>
__global__ void __launch_bounds__(256) k_stage_generic(Geo<T> G, StageArgs<T> A, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    const T k = rhs_comp<T, D>(G, A.y, x, I, a, T(0), true, A.diff, A.nu, A.F.f[a]);
    if (A.has_k) A.k_out.c[a][x] = k;
    if (A.has_s) {
      const T base = A.s_from_u0 ? A.u0.c[a][x] : A.s_in.c[a][x];
      A.s_out.c[a][x] = base + k * A.cb;
    }
    if (A.has_next) A.y_next.c[a][x] = A.u0.c[a][x] + k * A.ca;
  }
}

template <typename T>
int stage_fast_3d(const Geo<T>& G, const StageArgs<T>& A, cudaStream_t st);

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
    A.F.f[c] = on ? (T)a->force[c] : T(0);
  }
  A.cb = (T)a->cb;
  A.ca = (T)a->ca;
  A.nu = (T)a->nu;
  A.diff = a->nu != 0.0;
  A.has_k = a->k_out[0] != nullptr;
  A.has_s = a->s_out[0] != nullptr;
  A.has_next = a->y_next[0] != nullptr;
  A.s_from_u0 = a->s_in[0] == nullptr;
  if (A.has_next && !a->u0[0]) return fail(SFB_EINVAL, "y_next requires u0");
  if (A.has_s && A.s_from_u0 && !a->u0[0]) return fail(SFB_EINVAL, "s_out requires s_in or u0");
  Box B = int_box(G);
  SFB_DISPATCH_DIM(G.dim, D, (k_stage_generic<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, A, B)));
  SFB_LAUNCH_CHECK("rk stage");
  return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_rk_stage(sfb_plan* p, const sfb_stage_args* a, void* stream) {
  if (!p || !a || !a->y[0]) return fail(SFB_EINVAL, "null argument");
  if (a->nu < 0) return fail(SFB_EINVAL, "viscosity must be nonnegative");
  return SFB_TYPED(p, run_stage<T>(p, a, (cudaStream_t)stream));
}
