// Matrix-free conjugate-gradient pressure solve on the GPU
// (CGPoissonSolver, poisson.py:232-308), for the grids the FFT paths do not
// cover: stretched axes, symmetric or mixed walls, any periodicity pattern.
//
// The operator is the reference's _LaplacianApply (poisson.py:43-68) --
// scalar ghost fill, gradient on the velocity DOFs, homogeneous velocity
// fill, divergence -- evaluated as one 7-point stencil per cell: with
// homogeneous conditions every non-periodic boundary face carries zero
// normal velocity (Dirichlet and Symmetric alike, fields.py:96-140), and a
// periodic axis's face 0 is the copy of face n.  Weighted by the pressure
// volumes W it is symmetric negative semi-definite; CG runs on -W L.
//
// One iteration = 4 fused passes over the interior arrays (apply + p.Ap,
// update + sums, centre + |r|^2, new direction) with deterministic two-pass
// fp64 reductions that stay on the device.  The stopping test
// (poisson.py:289-297) runs on the device too: iterations are enqueued in
// batches of kCgBatch (one captured CUDA graph), every kernel of an
// iteration after convergence returns at once, and the host reads the
// done flag once per batch -- same iterates, same iteration count and
// residual history as one host round trip per iteration.
#include <cmath>
#include <cstdlib>

#include "sfb_kernels.cuh"
#include "sfb_solver.cuh"

namespace sfb {

namespace {
constexpr int kCgNT = 256;
constexpr int kCgBatch = 16;
// device scalar slots
enum { S_DENOM = 0, S_ALPHA, S_MX, S_MR, S_RR, S_BETA, S_TOLB, S_IT, S_DONE, S_FAIL, S_N };

template <int NT>
__device__ __forceinline__ double bsum(double v) {
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
  __syncthreads();
  return v;
}

// interior cell t (row-major over n) -> 1-based indices
template <int D>
__device__ __forceinline__ void cell(const int n[3], long long t, int I[3]) {
  if (t < (1LL << 32)) {  // 32-bit index arithmetic (64-bit division is a long sequence)
    unsigned r = (unsigned)t;
    if (D == 3) {
      I[2] = 1 + (int)(r % (unsigned)n[2]);
      r /= (unsigned)n[2];
    } else {
      I[2] = 0;
    }
    I[1] = 1 + (int)(r % (unsigned)n[1]);
    I[0] = 1 + (int)(r / (unsigned)n[1]);
    return;
  }
  if (D == 3) {
    I[2] = 1 + (int)(t % n[2]);
    t /= n[2];
  } else {
    I[2] = 0;
  }
  I[1] = 1 + (int)(t % n[1]);
  I[0] = 1 + (int)(t / n[1]);
}

// pressure volume W = dx_0 dx_1 (dx_2) in axis order (operators.py:275-281)
template <typename T, int D>
__device__ __forceinline__ T weight(const Geo<T>& G, const int I[3]) {
  T w = T(1);
#pragma unroll
  for (int a = 0; a < D; ++a) w = w * tab(G, a, T_DX, I[a]);
  return w;
}
}  // namespace

// ap = -W L p ; partial sums of p.ap
template <typename T, int D>
__global__ void __launch_bounds__(kCgNT) k_cg_apply(Geo<T> G, const T* __restrict__ p, T* __restrict__ ap,
                                                    double* __restrict__ part, const double* __restrict__ sc) {
  if (sc[S_DONE] != 0.0) return;
  const long long total = (long long)G.n[0] * G.n[1] * (D == 3 ? G.n[2] : 1);
  long long ps[3];
  ps[D - 1] = 1;
  if (D == 3) ps[1] = G.n[2];
  ps[0] = (long long)G.n[1] * (D == 3 ? G.n[2] : 1);
  double acc = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    cell<D>(G.n, t, I);
    const T pc = p[t];
    T L = T(0);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int n = G.n[a], i = I[a];
      T ghi, glo;
      if (G.per[a]) {
        const long long up = i == n ? t - (long long)(n - 1) * ps[a] : t + ps[a];
        ghi = (p[up] - pc) * tab(G, a, T_RDU, i);
        if (i == 1) {
          const long long last = t + (long long)(n - 1) * ps[a];
          glo = (pc - p[last]) * tab(G, a, T_RDU, n);  // face 0 = copy of face n
        } else {
          glo = (pc - p[t - ps[a]]) * tab(G, a, T_RDU, i - 1);
        }
      } else {
        ghi = i == n ? T(0) : (p[t + ps[a]] - pc) * tab(G, a, T_RDU, i);
        glo = i == 1 ? T(0) : (pc - p[t - ps[a]]) * tab(G, a, T_RDU, i - 1);
      }
      L += (ghi - glo) * tab(G, a, T_RDX, i);
    }
    const T v = -(L * weight<T, D>(G, I));
    ap[t] = v;
    acc += (double)pc * (double)v;
  }
  const double r = bsum<kCgNT>(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// mode 0: sum W*b ; mode 1: r = -(b - m) W, p = r, sum r^2 ; mode 3: sum W*x, sum r (after update)
// mode 4: centre x, r and sum r^2
template <typename T, int D, int MODE>
__global__ void __launch_bounds__(kCgNT) k_cg_vec(Geo<T> G, const T* __restrict__ b, T* __restrict__ x,
                                                  T* __restrict__ r, T* __restrict__ p, const T* __restrict__ ap,
                                                  const double* __restrict__ sc, double* __restrict__ part, int nb) {
  if ((MODE == 3 || MODE == 4) && sc[S_DONE] != 0.0) return;
  const long long total = (long long)G.n[0] * G.n[1] * (D == 3 ? G.n[2] : 1);
  double a0 = 0.0, a1 = 0.0;
  T alpha = T(0), mx = T(0), mr = T(0), m = T(0);
  if (MODE == 1) m = (T)sc[S_MX];
  if (MODE == 3) alpha = (T)sc[S_ALPHA];
  if (MODE == 4) {
    mx = (T)sc[S_MX];
    mr = (T)sc[S_MR];
  }
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    cell<D>(G.n, t, I);
    if (MODE == 0) {
      a0 += (double)(weight<T, D>(G, I) * b[t]);
    } else if (MODE == 1) {
      T v = b[t] - m;
      v = v * weight<T, D>(G, I);
      v = -v;
      r[t] = v;
      p[t] = v;
      a0 += (double)v * (double)v;
    } else if (MODE == 3) {
      // t = p*alpha; x += t ; ap *= alpha ; r -= ap  (poisson.py:284-288)
      const T xn = x[t] + p[t] * alpha;
      x[t] = xn;
      const T rn = r[t] - ap[t] * alpha;
      r[t] = rn;
      a0 += (double)(weight<T, D>(G, I) * xn);
      a1 += (double)rn;
    } else {
      x[t] = x[t] - mx;
      const T rn = r[t] - mr;
      r[t] = rn;
      a0 += (double)rn * (double)rn;
    }
  }
  const double s0 = bsum<kCgNT>(a0);
  if (threadIdx.x == 0) part[blockIdx.x] = s0;
  if (MODE == 3) {
    const double s1 = bsum<kCgNT>(a1);
    if (threadIdx.x == 0) part[nb + blockIdx.x] = s1;
  }
}

// p = p*beta + r
template <typename T>
__global__ void __launch_bounds__(kCgNT) k_cg_dir(T* __restrict__ p, const T* __restrict__ r,
                                                  const double* __restrict__ sc, long long total) {
  if (sc[S_DONE] != 0.0) return;
  const T beta = (T)sc[S_BETA];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x)
    p[t] = p[t] * beta + r[t];
}

// second pass of the reductions; what = which scalars to form
//  0: S_MX = sum/wtot (weighted mean of b)   1: S_RR = sum (|b|^2)
//  2: S_DENOM, S_ALPHA = S_RR / S_DENOM       3: S_MX = sum0/wtot, S_MR = sum1/N
//  4: the end of an iteration (poisson.py:289-297): a non-positive p.Ap
//     fails; else record |r|, stop at |r| <= tol |b|, else
//     beta = |r_new|^2 / |r|^2
__global__ void __launch_bounds__(kCgNT) k_cg_finish(const double* __restrict__ part, int nb, int what, double wtot,
                                                     double ntot, double* __restrict__ sc, double* __restrict__ hist) {
  if (what >= 2 && sc[S_DONE] != 0.0) return;
  double a0 = 0.0, a1 = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a0 += part[i];
    if (what == 3) a1 += part[nb + i];
  }
  a0 = bsum<kCgNT>(a0);
  if (what == 3) a1 = bsum<kCgNT>(a1);
  if (threadIdx.x != 0) return;
  switch (what) {
    case 0: sc[S_MX] = a0 / wtot; break;
    case 1: sc[S_RR] = a0; break;
    case 2: sc[S_DENOM] = a0; sc[S_ALPHA] = sc[S_RR] / a0; break;  // r.r of the previous iterate
    case 3: sc[S_MX] = a0 / wtot; sc[S_MR] = a1 / ntot; break;
    default: {
      if (!(sc[S_DENOM] > 0.0)) {
        sc[S_FAIL] = 1.0;
        sc[S_DONE] = 1.0;
        break;
      }
      const int it = (int)sc[S_IT] + 1;
      sc[S_IT] = it;
      const double res = sqrt(a0);
      hist[it] = res;
      if (res <= sc[S_TOLB]) {
        sc[S_DONE] = 1.0;
      } else {
        sc[S_BETA] = a0 / sc[S_RR];
        sc[S_RR] = a0;
      }
      break;
    }
  }
}

// arm the device-side stopping test after the initial residual
__global__ void k_cg_arm(double* __restrict__ sc, double* __restrict__ hist, double tol) {
  const double b_norm = sqrt(sc[S_RR]);
  hist[0] = b_norm;
  sc[S_TOLB] = tol * b_norm;
  sc[S_IT] = 0.0;
  sc[S_DONE] = 0.0;
  sc[S_FAIL] = 0.0;
}

template <typename T>
static void cg_iteration(sfb_solver* s, const Geo<T>& G, int nb, cudaStream_t st) {
  T* x = (T*)s->cg_x;
  T* r = (T*)s->cg_r;
  T* pd = (T*)s->cg_p;
  T* ap = (T*)s->cg_ap;
  double* part = s->cg_part;
  double* sc = s->cg_dsc;
  const double wtot = s->cg_wtot, ntot = (double)s->plan->int_count;
  SFB_DISPATCH_DIM(G.dim, D, (k_cg_apply<T, D><<<nb, kCgNT, 0, st>>>(G, pd, ap, part, sc)));
  k_cg_finish<<<1, kCgNT, 0, st>>>(part, nb, 2, wtot, ntot, sc, s->cg_dhist);
  SFB_DISPATCH_DIM(G.dim, D, (k_cg_vec<T, D, 3><<<nb, kCgNT, 0, st>>>(G, x, x, r, pd, ap, sc, part, nb)));
  k_cg_finish<<<1, kCgNT, 0, st>>>(part, nb, 3, wtot, ntot, sc, s->cg_dhist);
  SFB_DISPATCH_DIM(G.dim, D, (k_cg_vec<T, D, 4><<<nb, kCgNT, 0, st>>>(G, x, x, r, pd, ap, sc, part, nb)));
  k_cg_finish<<<1, kCgNT, 0, st>>>(part, nb, 4, wtot, ntot, sc, s->cg_dhist);
  k_cg_dir<T><<<nb, kCgNT, 0, st>>>(pd, r, sc, s->plan->int_count);
}

// capture kCgBatch iterations once per solver (all pointers are solver-owned)
template <typename T>
static void cg_capture(sfb_solver* s, const Geo<T>& G, int nb) {
  s->cg_graph_tried = true;
  if (getenv("SFB_CG_NOGRAPH")) return;
  // one capture stream per solver, created on the first capture and reused
  // when sfb_cg_configure forces a re-capture (destroyed with the solver)
  cudaStream_t cap = (cudaStream_t)s->cg_cap_stream;
  if (!cap) {
    if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    s->cg_cap_stream = cap;
  }
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  for (int k = 0; k < kCgBatch; ++k) cg_iteration<T>(s, G, nb, cap);
  cudaGraphExec_t ex = nullptr;
  if (cudaStreamEndCapture(cap, &g) == cudaSuccess && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess)
    s->cg_graph = ex;
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
}

template <typename T>
int cg_solve(sfb_solver* s, T* buf, cudaStream_t st) {
  sfb_plan* p = s->plan;
  const Geo<T>& G = geo<T>(p);
  const long long total = p->int_count;
  int nb = (int)((total + kCgNT - 1) / kCgNT);
  if (nb > s->cg_nb) nb = s->cg_nb;
  T* x = (T*)s->cg_x;
  T* r = (T*)s->cg_r;
  T* pd = (T*)s->cg_p;
  T* ap = (T*)s->cg_ap;
  double* part = s->cg_part;
  double* sc = s->cg_dsc;
  double* hs = s->cg_hsc;
  const double wtot = s->cg_wtot, ntot = (double)total;
  int rc;
  if (s->cg_dhist_cap < s->cg_max_iter + 1) {
    if (s->cg_dhist) cudaFree(s->cg_dhist);
    s->cg_dhist = nullptr;
    // the captured batch holds the old history pointer
    if (s->cg_graph) cudaGraphExecDestroy((cudaGraphExec_t)s->cg_graph);
    s->cg_graph = nullptr;
    s->cg_graph_tried = false;
    s->cg_dhist_cap = 0;
    if ((rc = cuda_check(cudaMalloc(&s->cg_dhist, sizeof(double) * (s->cg_max_iter + 1)), "cudaMalloc(cg history)")))
      return rc;
    s->cg_dhist_cap = s->cg_max_iter + 1;
  }
  auto pull = [&]() -> int {
    int rc2 = cuda_check(cudaMemcpyAsync(hs, sc, sizeof(double) * S_N, cudaMemcpyDeviceToHost, st), "cg d2h");
    if (rc2) return rc2;
    return cuda_check(cudaStreamSynchronize(st), "cg sync");
  };
  auto history = [&](int n) -> int {
    s->cg_hist.assign(n + 1, 0.0);
    int rc2 = cuda_check(cudaMemcpyAsync(s->cg_hist.data(), s->cg_dhist, sizeof(double) * (n + 1),
                                         cudaMemcpyDeviceToHost, st), "cg history");
    if (rc2) return rc2;
    s->cg_iters = n;
    return cuda_check(cudaStreamSynchronize(st), "cg sync");
  };
  s->cg_hist.clear();
  s->cg_iters = 0;
  // b = -W (rhs - wmean(rhs)),  p = r = b
  SFB_DISPATCH_DIM(G.dim, D, (k_cg_vec<T, D, 0><<<nb, kCgNT, 0, st>>>(G, buf, x, r, pd, ap, sc, part, nb)));
  k_cg_finish<<<1, kCgNT, 0, st>>>(part, nb, 0, wtot, ntot, sc, s->cg_dhist);
  SFB_DISPATCH_DIM(G.dim, D, (k_cg_vec<T, D, 1><<<nb, kCgNT, 0, st>>>(G, buf, x, r, pd, ap, sc, part, nb)));
  k_cg_finish<<<1, kCgNT, 0, st>>>(part, nb, 1, wtot, ntot, sc, s->cg_dhist);
  if ((rc = cuda_check(cudaMemsetAsync(x, 0, sizeof(T) * total, st), "cg x = 0"))) return rc;
  k_cg_arm<<<1, 1, 0, st>>>(sc, s->cg_dhist, s->cg_tol);
  SFB_LAUNCH_CHECK("cg init");
  if ((rc = pull())) return rc;
  if (std::sqrt(hs[S_RR]) == 0.0) {
    s->cg_hist.assign(1, 0.0);
    return cuda_check(cudaMemsetAsync(buf, 0, sizeof(T) * total, st), "cg zero");
  }
  if (!s->cg_graph_tried) cg_capture<T>(s, G, nb);
  int issued = 0;
  while (issued < s->cg_max_iter) {
    const int k = std::min(kCgBatch, s->cg_max_iter - issued);
    if (k == kCgBatch && s->cg_graph) {
      if ((rc = cuda_check(cudaGraphLaunch((cudaGraphExec_t)s->cg_graph, st), "cg graph launch"))) return rc;
    } else {
      for (int i = 0; i < k; ++i) cg_iteration<T>(s, G, nb, st);
      SFB_LAUNCH_CHECK("cg iterations");
    }
    issued += k;
    if ((rc = pull())) return rc;
    if (hs[S_FAIL] != 0.0) {
      if ((rc = history((int)hs[S_IT]))) return rc;
      return fail(SFB_ENUMERIC, "pressure operator lost positive definiteness");
    }
    if (hs[S_DONE] != 0.0) {
      if ((rc = history((int)hs[S_IT]))) return rc;
      return cuda_check(cudaMemcpyAsync(buf, x, sizeof(T) * total, cudaMemcpyDeviceToDevice, st), "cg out");
    }
  }
  if ((rc = history((int)hs[S_IT]))) return rc;
  char msg[160];
  snprintf(msg, sizeof msg, "pressure CG did not reach tol=%g in %d iterations", s->cg_tol, s->cg_max_iter);
  return fail(SFB_ECONVERGE, msg);
}
template int cg_solve<double>(sfb_solver*, double*, cudaStream_t);
template int cg_solve<float>(sfb_solver*, float*, cudaStream_t);

int cg_setup(sfb_solver* s) {
  sfb_plan* p = s->plan;
  const size_t esz = p->dtype == SFB_F64 ? 8 : 4;
  const long long total = p->int_count;
  s->cg_nb = p->red_blocks;
  int rc;
  void** bufs[4] = {&s->cg_x, &s->cg_r, &s->cg_p, &s->cg_ap};
  for (void** b : bufs)
    if ((rc = cuda_check(cudaMalloc(b, esz * total), "cudaMalloc(cg)"))) return rc;
  if ((rc = cuda_check(cudaMalloc(&s->cg_part, sizeof(double) * 2 * s->cg_nb), "cudaMalloc(cg part)"))) return rc;
  if ((rc = cuda_check(cudaMalloc(&s->cg_dsc, sizeof(double) * S_N), "cudaMalloc(cg scalars)"))) return rc;
  // every slot defined before the first host read (compute-sanitizer initcheck)
  if ((rc = cuda_check(cudaMemset(s->cg_dsc, 0, sizeof(double) * S_N), "cudaMemset(cg scalars)"))) return rc;
  if ((rc = cuda_check(cudaMallocHost(&s->cg_hsc, sizeof(double) * S_N), "cudaMallocHost(cg)"))) return rc;
  // total pressure volume (poisson.py:158, np.sum of the weights)
  double wtot = 0.0;
  const int n0 = p->n[0], n1 = p->n[1], n2 = p->dim == 3 ? p->n[2] : 1;
  for (int i = 1; i <= n0; ++i)
    for (int j = 1; j <= n1; ++j) {
      const double w01 = p->hdx[0][i] * p->hdx[1][j];
      if (p->dim == 3)
        for (int k = 1; k <= n2; ++k) wtot += w01 * p->hdx[2][k];
      else
        wtot += w01;
    }
  s->cg_wtot = wtot;
  const double n = (double)total;
  s->cg_tol = p->dtype == SFB_F64 ? 1e-10 : 1e-5;
  const int m = (int)std::ceil(std::pow(n, 1.0 / p->dim));
  s->cg_max_iter = std::min(10000, 10 * m + 10);
  return SFB_OK;
}

void cg_release(sfb_solver* s) {
  void* bufs[] = {s->cg_x, s->cg_r, s->cg_p, s->cg_ap, s->cg_part, s->cg_dsc, s->cg_dhist};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (s->cg_graph) cudaGraphExecDestroy((cudaGraphExec_t)s->cg_graph);
  if (s->cg_cap_stream) cudaStreamDestroy((cudaStream_t)s->cg_cap_stream);
  if (s->cg_hsc) cudaFreeHost(s->cg_hsc);
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_cg_configure(sfb_solver* s, double tol, int max_iter) {
  if (!s || s->kind != SFB_SOLVER_CG) return fail(SFB_EINVAL, "not a CG solver");
  if (!(tol > 0.0)) return fail(SFB_EINVAL, "tolerance must be positive");
  if (max_iter < 1) return fail(SFB_EINVAL, "max_iter must be positive");
  s->cg_tol = tol;
  s->cg_max_iter = max_iter;
  return SFB_OK;
}

int sfb_cg_info(const sfb_solver* s, int* iterations, double* history, int cap, int* count) {
  if (!s || s->kind != SFB_SOLVER_CG) return fail(SFB_EINVAL, "not a CG solver");
  if (iterations) *iterations = s->cg_iters;
  const int n = (int)s->cg_hist.size();
  if (count) *count = n;
  if (history)
    for (int i = 0; i < n && i < cap; ++i) history[i] = s->cg_hist[i];
  return SFB_OK;
}

}  // extern "C"
