// Hand-written FFT engine for the spectral pressure solve (sm_100a).
//
// Replaces the raw cuFFT transforms of poisson.py:196,199 on the hot path.
// One HBM pass per axis: a CTA stages a tile (the full transform length L x
// W columns) in shared memory, runs a mixed-radix Stockham FFT (radices
// 8/4/2/7/5/3, natural-order output) and writes it back.
//
// 3D solve = 5 passes over the half spectrum:
//   R2C along axis 2 (real trick: length-n2/2 complex FFT + post-twiddle)
//   C2C fwd along axis 1
//   C2C fwd along axis 0 -> eigenvalue scaling 1/(Lambda N) -> C2C inv (fused)
//   C2C inv along axis 1
//   C2R along axis 2 (pre-twiddle + length-n2/2 inverse FFT)
// (2D: R2C axis 1, fused axis 0, C2R axis 1.)
#include <cmath>
#include <cstdlib>
#include <vector>

#include "sfb_fft.cuh"
#include "sfb_fft_dev.cuh"
#include "sfb_fft_reg.cuh"
#include "sfb_kernels.cuh"

namespace sfb {

// ---------------------------------------------------------------------------
// strided C2C pass (optionally fused forward -> scale -> inverse)
//   element (m, col) at base + m*S + col, col in [0, ncol), tile W columns
// ---------------------------------------------------------------------------
template <typename T, int MODE, int W>  // MODE 0 fwd, 1 inv, 2 fwd+scale+inv
__global__ void __launch_bounds__(256, 4) k_fft_strided(typename CX<T>::t* __restrict__ data, FftLen P,
                                                     long long S, int ncol, long long bstride,
                                                     const typename CX<T>::t* __restrict__ tw, ScaleArgs sc) {
  typedef typename CX<T>::t C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + (size_t)P.L * W;
  const int c0 = blockIdx.x * W;
  C* base = data + (long long)blockIdx.y * bstride;
  const int L = P.L;
  const int tot = L * W;
  // thread-fixed column; rows m = m0 + s*ms (strength-reduced addressing)
  const int w = threadIdx.x % W, m0 = threadIdx.x / W, ms = blockDim.x / W;
  const int col = c0 + w;
  const bool ok = col < ncol;
  {
    const C* g = base + (ok ? (long long)m0 * S + col : 0);
    const long long gs = ok ? (long long)ms * S : 0;
    C* sd = bufA + m0 * W + w;
#pragma unroll 4
    for (int m = m0; m < L; m += ms, g += gs, sd += ms * W) cp_async_elem(sd, g, ok);
  }
  cp_async_wait_all();
  C* res;
  if (MODE == 1) res = run_fft<C, true, W>(bufA, bufB, P, tw);
  else res = run_fft<C, false, W>(bufA, bufB, P, tw);
  if (MODE == 2) {
    // eigenvalue scaling (poisson.py:179-199): lam in fp64, cast to T
    if (ok) {
      double lc;
      if (sc.dim == 3) {
        const int k1 = col / sc.nh, k2 = col - k1 * sc.nh;
        lc = sc.l1[k1] + 0.0;
        // (l0[m] + l1[k1]) + l2[k2], accumulated in axis order
        for (int m = m0; m < L; m += ms) {
          const double lam = (sc.l0[m] + lc) + sc.l2[k2];
          C v = res[m * W + w];
          if (m == 0 && col == 0 && blockIdx.y == 0 && sc.zero_ok) {
            v.x = 0;
            v.y = 0;
          } else {
            const T f = spec_rcp<T>(lam) * (T)sc.invN;
            v.x *= f;
            v.y *= f;
          }
          res[m * W + w] = v;
        }
      } else {
        lc = sc.l1[col];
        for (int m = m0; m < L; m += ms) {
          const double lam = sc.l0[m] + lc;
          C v = res[m * W + w];
          if (m == 0 && col == 0 && blockIdx.y == 0 && sc.zero_ok) {
            v.x = 0;
            v.y = 0;
          } else {
            const T f = spec_rcp<T>(lam) * (T)sc.invN;
            v.x *= f;
            v.y *= f;
          }
          res[m * W + w] = v;
        }
      }
    }
    C* other = (res == bufA) ? bufB : bufA;
    res = run_fft<C, true, W>(res, other, P, tw);
  }
  if (ok) {
    C* g = base + (long long)m0 * S + col;
    const long long gs = (long long)ms * S;
    const C* sd = res + m0 * W + w;
#pragma unroll 4
    for (int m = m0; m < L; m += ms, g += gs, sd += ms * W) *g = *sd;
  }
}

// ---------------------------------------------------------------------------
// contiguous-axis real transforms: one row per CTA, M = N/2 complex points
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) k_fft_r2c(const T* __restrict__ in, typename CX<T>::t* __restrict__ out, FftLen P,
                                                 const typename CX<T>::t* __restrict__ tw,
                                                 const typename CX<T>::t* __restrict__ tw2, long long in_row,
                                                 long long out_row) {
  typedef typename CX<T>::t C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + P.L;
  const int M = P.L;
  const C* row = reinterpret_cast<const C*>(in + (long long)blockIdx.x * in_row);
  for (int m = threadIdx.x; m < M; m += blockDim.x) cp_async_elem(bufA + m, row + m, true);
  cp_async_wait_all();
  C* Z = run_fft<C, false, 1>(bufA, bufB, P, tw);
  C* o = out + (long long)blockIdx.x * out_row;
  // X[k] = E[k] + w^k O[k],  E = (Z[k] + conj Z[M-k]) / 2,  O = (Z[k] - conj Z[M-k]) / (2i)
  for (int k = threadIdx.x; k <= M; k += blockDim.x) {
    const C zk = Z[k == M ? 0 : k];
    const C zc = Z[k == 0 ? 0 : M - k];
    C e, od;
    e.x = T(0.5) * (zk.x + zc.x);
    e.y = T(0.5) * (zk.y - zc.y);
    // (zk - conj(zc)) / (2i) = (a + ib)/(2i) = (b - ia)/2 with a = zk.x - zc.x, b = zk.y + zc.y
    od.x = T(0.5) * (zk.y + zc.y);
    od.y = -T(0.5) * (zk.x - zc.x);
    const C w = tw2[k];  // exp(-2 pi i k / N)
    o[k] = cadd(e, cmul(w, od));
  }
}

// R2C of one row of the divergence, computed on the fly from the velocity
// (operators.py:108-122 fused into the first FFT pass of poisson.py:196):
// the five velocity rows the row's divergence needs are staged into shared
// memory with cp.async (all in flight at once), the divergence is formed
// there, and the divergence field is never written to HBM.
template <typename T>
__device__ __forceinline__ void cp_async_scalar(T* smem, const T* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}

template <typename T, int D>
__global__ void __launch_bounds__(128) k_fft_r2c_div(Geo<T> G, CV<T> U, typename CX<T>::t* __restrict__ out, FftLen P,
                                                     const typename CX<T>::t* __restrict__ tw,
                                                     const typename CX<T>::t* __restrict__ tw2, long long out_row) {
  typedef typename CX<T>::t C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + P.L;
  T* xr = reinterpret_cast<T*>(bufA);
  const int M = P.L;
  const int nl = G.n[D - 1];
  T* rows = reinterpret_cast<T*>(bufB + P.L);  // [2*D-1][nl]: a=0 cur/prev, (a=1 cur/prev), last cur
  int i0, i1 = 0;
  if (D == 3) {
    i0 = 1 + blockIdx.x / G.n[1];
    i1 = 1 + blockIdx.x % G.n[1];
  } else {
    i0 = 1 + blockIdx.x;
  }
  // source rows (element k=1 of each row); boundary rows resolved like own_pair
  const long long sa0 = G.s[0];
  const long long base = (long long)i0 * G.s[0] + (D == 3 ? (long long)i1 * G.s[1] : 0) + 1;
  const T* src[5];
  int nsrc = 0;
  bool c0_const = false, p0_const = false, c1_const = false, p1_const = false;
  // axis 0 (component 0)
  {
    const int n = G.n[0];
    src[nsrc++] = U.c[0] + base;  // cur
    if (G.per[0]) src[nsrc++] = U.c[0] + base + (i0 == 1 ? (long long)(n - 1) * sa0 : -sa0);
    else src[nsrc++] = U.c[0] + base - sa0;
    if (!G.per[0]) {
      c0_const = i0 == n;
      p0_const = i0 == 1;
    }
  }
  if (D == 3) {
    const int n = G.n[1];
    const long long sa1 = G.s[1];
    src[nsrc++] = U.c[1] + base;
    if (G.per[1]) src[nsrc++] = U.c[1] + base + (i1 == 1 ? (long long)(n - 1) * sa1 : -sa1);
    else src[nsrc++] = U.c[1] + base - sa1;
    if (!G.per[1]) {
      c1_const = i1 == n;
      p1_const = i1 == 1;
    }
  }
  src[nsrc++] = U.c[D - 1] + base;  // last component along the row
  for (int r = 0; r < nsrc; ++r)
    for (int m = threadIdx.x; m < nl; m += 128) cp_async_scalar(rows + r * nl + m, src[r] + m);
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const T rd0 = tab(G, 0, T_RDX, i0);
  const T rd1 = D == 3 ? tab(G, 1, T_RDX, i1) : T(0);
  const T* rl = rows + (nsrc - 1) * nl;
  const int al = D - 1;
  for (int m = threadIdx.x; m < nl; m += 128) {
    T c = c0_const ? (G.bc_hi[0] == SFB_BC_DIRICHLET ? G.vhi[0][0] : T(0)) : rows[m];
    T pv = p0_const ? (G.bc_lo[0] == SFB_BC_DIRICHLET ? G.vlo[0][0] : T(0)) : rows[nl + m];
    T acc = (c - pv) * rd0;
    if (D == 3) {
      c = c1_const ? (G.bc_hi[1] == SFB_BC_DIRICHLET ? G.vhi[1][1] : T(0)) : rows[2 * nl + m];
      pv = p1_const ? (G.bc_lo[1] == SFB_BC_DIRICHLET ? G.vlo[1][1] : T(0)) : rows[3 * nl + m];
      acc += (c - pv) * rd1;
    }
    // last axis: within the row
    T cl, pl;
    if (G.per[al]) {
      cl = rl[m];
      pl = rl[m == 0 ? nl - 1 : m - 1];
    } else {
      cl = m == nl - 1 ? (G.bc_hi[al] == SFB_BC_DIRICHLET ? G.vhi[al][al] : T(0)) : rl[m];
      pl = m == 0 ? (G.bc_lo[al] == SFB_BC_DIRICHLET ? G.vlo[al][al] : T(0)) : rl[m - 1];
    }
    acc += (cl - pl) * tab(G, al, T_RDX, m + 1);
    xr[m] = acc;
  }
  C* Z = run_fft<C, false, 1>(bufA, bufB, P, tw);
  C* o = out + (long long)blockIdx.x * out_row;
  for (int k = threadIdx.x; k <= M; k += blockDim.x) {
    const C zk = Z[k == M ? 0 : k];
    const C zc = Z[k == 0 ? 0 : M - k];
    C e, od;
    e.x = T(0.5) * (zk.x + zc.x);
    e.y = T(0.5) * (zk.y - zc.y);
    od.x = T(0.5) * (zk.y + zc.y);
    od.y = -T(0.5) * (zk.x - zc.x);
    const C w = tw2[k];
    o[k] = cadd(e, cmul(w, od));
  }
}

template <typename T>
__global__ void __launch_bounds__(128) k_fft_c2r(const typename CX<T>::t* __restrict__ in, T* __restrict__ out, FftLen P,
                                                 const typename CX<T>::t* __restrict__ tw,
                                                 const typename CX<T>::t* __restrict__ tw2, long long in_row,
                                                 long long out_row) {
  typedef typename CX<T>::t C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + P.L;
  const int M = P.L;
  const C* Xg = in + (long long)blockIdx.x * in_row;
  C* X = bufB;  // staged row (M+1 values; the smem allocation has 2M+2)
  for (int k = threadIdx.x; k <= M; k += blockDim.x) cp_async_elem(X + k, Xg + k, true);
  cp_async_wait_all();
  __syncthreads();
  // Z[k] = (X[k] + conj X[M-k]) + i (X[k] - conj X[M-k]) exp(+2 pi i k / N)
  for (int k = threadIdx.x; k < M; k += blockDim.x) {
    const C xk = X[k];
    const C xc = X[M - k];
    C fe, fo, d;
    fe.x = xk.x + xc.x;
    fe.y = xk.y - xc.y;
    d.x = xk.x - xc.x;
    d.y = xk.y + xc.y;
    C w = tw2[k];
    w.y = -w.y;
    fo = cmul(d, w);
    C z;
    z.x = fe.x - fo.y;
    z.y = fe.y + fo.x;
    bufA[k] = z;
  }
  C* z = run_fft<C, true, 1>(bufA, bufB, P, tw);
  C* row = reinterpret_cast<C*>(out + (long long)blockIdx.x * out_row);
  for (int m = threadIdx.x; m < M; m += blockDim.x) row[m] = z[m];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool fft_factor(int L, FftLen& P) {
  P.L = L;
  P.np = 0;
  int r = L;
  const int order[6] = {8, 4, 2, 7, 5, 3};
  // prefer radix 8; use one 4 or 2 for the power-of-two remainder
  while (r > 1) {
    bool ok = false;
    for (int q : order) {
      if (r % q == 0) {
        if (P.np >= 12) return false;
        P.radix[P.np++] = q;
        r /= q;
        ok = true;
        break;
      }
    }
    if (!ok) return false;
  }
  return true;
}

void fft_reg_assign(FftSolve& F) {
  RegLen R;
  F.reg_half = 0;
  if (reg_factor(F.half.L, R)) {
    F.reg_half = R.L;
    F.reg_a_half = R.A;
    F.reg_b_half = R.B;
  }
  for (int a = 0; a < 3; ++a) {
    F.reg_ax[a] = 0;
    if (a < F.dim - 1 && reg_factor(F.ax[a].L, R)) {
      F.reg_ax[a] = R.L;
      F.reg_a[a] = R.A;
      F.reg_b[a] = R.B;
    }
  }
}

static int upload(const std::vector<double>& t, bool f64, void** dev) {
  size_t bytes;
  std::vector<float> tf;
  const void* src;
  if (f64) {
    bytes = sizeof(double) * t.size();
    src = t.data();
  } else {
    tf.assign(t.begin(), t.end());
    bytes = sizeof(float) * tf.size();
    src = tf.data();
  }
  int rc = cuda_check(cudaMalloc(dev, bytes), "cudaMalloc(twiddles)");
  if (rc) return rc;
  return cuda_check(cudaMemcpy(*dev, src, bytes, cudaMemcpyHostToDevice), "upload twiddles");
}

static void push_root(std::vector<double>& t, long long num, long long den) {
  const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)(num % den) / (long double)den;
  t.push_back((double)cosl(a));
  t.push_back((double)sinl(a));
}

int fft_upload_twiddles(int L, bool f64, void** dev) {
  std::vector<double> t;
  for (int m = 0; m < (L > 0 ? L : 1); ++m) push_root(t, m, L > 0 ? L : 1);
  return upload(t, f64, dev);
}

// plain table (L entries) followed by per-pass tables [k][r-1]
int fft_upload_pass_twiddles(FftLen& P, bool f64, void** dev) {
  std::vector<double> t;
  const int L = P.L > 0 ? P.L : 1;
  for (int m = 0; m < L; ++m) push_root(t, m, L);
  int Ns = 1;
  for (int p = 0; p < P.np; ++p) {
    const int R = P.radix[p];
    P.twoff[p] = (int)(t.size() / 2);
    const int step = L / (Ns * R);
    if (Ns > 1)
      for (int k = 0; k < Ns; ++k)
        for (int r = 1; r < R; ++r) push_root(t, (long long)k * r * step, L);
    Ns *= R;
  }
  P.twn = (int)(t.size() / 2);
  return upload(t, f64, dev);
}

static int pick_w(int L, size_t csz) {
  static int wmax = getenv("SFB_FFT_WMAX") ? atoi(getenv("SFB_FFT_WMAX")) : 8;
  int W = wmax;
  while (W > 1 && 2 * (size_t)L * W * csz > 110 * 1024) W /= 2;
  return W;
}

static RegLen reg_of(int L, int A, int B) {
  RegLen R;
  R.L = L;
  R.A = A;
  R.B = B;
  R.ok = L > 0;
  return R;
}

template <typename T, int MODE>
static int launch_strided(typename CX<T>::t* data, const FftLen& P, int W, long long S, int ncol, long long bstride,
                          int nbatch, const typename CX<T>::t* tw, const ScaleArgs& sc, cudaStream_t st,
                          const FftTma* tma = nullptr, RegLen reg = RegLen{}) {
  typedef typename CX<T>::t C;
  if (reg.ok) {
    RegCall c{};
    c.kind = MODE;
    c.out = data;
    c.S = S;
    c.ncol = ncol;
    c.bstride = bstride;
    c.nbatch = nbatch;
    c.twL = tw;
    c.sc = sc;
    return reg_run<T>(reg, c, st);
  }
  if (tma && tma->ok && !getenv("SFB_NO_TMA")) return fft_tma_pass<T, MODE>(*tma, P, tw, sc, st);
  dim3 grid((ncol + W - 1) / W, nbatch);
  const size_t sm = 2 * (size_t)P.L * W * sizeof(C);
  switch (W) {
    case 8: k_fft_strided<T, MODE, 8><<<grid, 256, sm, st>>>(data, P, S, ncol, bstride, tw, sc); break;
    case 4: k_fft_strided<T, MODE, 4><<<grid, 256, sm, st>>>(data, P, S, ncol, bstride, tw, sc); break;
    case 2: k_fft_strided<T, MODE, 2><<<grid, 256, sm, st>>>(data, P, S, ncol, bstride, tw, sc); break;
    default: k_fft_strided<T, MODE, 1><<<grid, 256, sm, st>>>(data, P, S, ncol, bstride, tw, sc); break;
  }
  SFB_LAUNCH_CHECK("fft strided pass");
  return SFB_OK;
}

template <typename T>
static int launch_r2c(FftSolve& F, const T* rbuf, typename CX<T>::t* cbuf, long long rows, cudaStream_t st,
                      bool tiled = false) {
  typedef typename CX<T>::t C;
  const int nlast = F.n[F.dim - 1], M = nlast / 2, nh = M + 1;
  if (F.reg_half) {
    RegCall c{};
    c.kind = 3;
    c.in = rbuf;
    c.out = cbuf;
    c.rows = rows;
    c.in_row = nlast;
    c.out_row = nh;
    c.tlog = tiled ? F.tlog : 0;
    c.ks = F.tks;
    c.twL = F.tw_half;
    c.twN = F.tw_full;
    return reg_run<T>(reg_of(F.reg_half, F.reg_a_half, F.reg_b_half), c, st);
  }
  k_fft_r2c<T><<<(unsigned)rows, 128, 2 * (size_t)M * sizeof(C), st>>>(rbuf, cbuf, F.half, (const C*)F.tw_half,
                                                                       (const C*)F.tw_full, nlast, nh);
  SFB_LAUNCH_CHECK("fft r2c");
  return SFB_OK;
}

template <typename T>
static int launch_c2r(FftSolve& F, const typename CX<T>::t* cbuf, T* rbuf, long long rows, cudaStream_t st,
                      bool tiled = false) {
  typedef typename CX<T>::t C;
  const int nlast = F.n[F.dim - 1], M = nlast / 2, nh = M + 1;
  if (F.reg_half) {
    RegCall c{};
    c.kind = 4;
    c.in = cbuf;
    c.out = rbuf;
    c.rows = rows;
    c.in_row = nh;
    c.out_row = nlast;
    c.tlog = tiled ? F.tlog : 0;
    c.ks = F.tks;
    c.twL = F.tw_half;
    c.twN = F.tw_full;
    return reg_run<T>(reg_of(F.reg_half, F.reg_a_half, F.reg_b_half), c, st);
  }
  k_fft_c2r<T><<<(unsigned)rows, 128, (2 * (size_t)M + 2) * sizeof(C), st>>>(cbuf, rbuf, F.half, (const C*)F.tw_half,
                                                                             (const C*)F.tw_full, nh, nlast);
  SFB_LAUNCH_CHECK("fft c2r");
  return SFB_OK;
}

template <typename T>
bool fft_divfuse_ok(const FftSolve& F, const Geo<T>& G) {
  if (getenv("SFB_NO_DIVFUSE")) return false;
  return F.reg_half && G.dim == 3 && F.dim == 3 && G.per[1] && !G.halo[1] && G.per[2] && !G.halo[2] &&
         (G.per[0] || G.halo[0]) && F.n[0] == G.n[0] && F.n[1] == G.n[1] && F.n[2] == G.n[2];
}
template bool fft_divfuse_ok<double>(const FftSolve&, const Geo<double>&);
template bool fft_divfuse_ok<float>(const FftSolve&, const Geo<float>&);

#define SFB_REG(F, a) reg_of((F).reg_ax[a], (F).reg_a[a], (F).reg_b[a])

// ---- channel solve (poisson.py:203-229 on separable channel grids): the
// register engine does the raw FFT(x, z) passes, the batched tridiagonal
// solve along y (poisson.cu k_tridiag) runs between them on the natural
// half spectrum (n0, n1, nh)
template <typename T>
bool fft_channel_divfuse_ok(const FftSolve& F, const Geo<T>& G) {
  if (getenv("SFB_NO_DIVFUSE")) return false;
  return F.reg_half && F.reg_ax[0] && G.dim == 3 && F.dim == 3 && G.per[0] && !G.halo[0] && G.per[2] && !G.halo[2] &&
         !G.per[1] && F.n[0] == G.n[0] && F.n[1] == G.n[1] && F.n[2] == G.n[2];
}
template bool fft_channel_divfuse_ok<double>(const FftSolve&, const Geo<double>&);
template bool fft_channel_divfuse_ok<float>(const FftSolve&, const Geo<float>&);

template <typename T>
int fft_channel_forward(FftSolve& F, const T* rbuf, void* cbuf_v, cudaStream_t st, const Geo<T>* G,
                        const void* const* u) {
  typedef typename CX<T>::t C;
  C* cbuf = (C*)cbuf_v;
  const int n0 = F.n[0], n1 = F.n[1], nlast = F.n[2], nh = nlast / 2 + 1;
  const long long rows = (long long)n0 * n1;
  if (G) {
    // R2C along z of the divergence (walls on y resolved inline)
    RegCall c{};
    c.kind = 5;
    c.out = cbuf;
    c.rows = rows;
    c.out_row = nh;
    c.twL = F.tw_half;
    c.twN = F.tw_full;
    c.geo = G;
    c.wall1 = 1;
    for (int a = 0; a < 3; ++a) c.u[a] = u[a];
    if (int rc = reg_run<T>(reg_of(F.reg_half, F.reg_a_half, F.reg_b_half), c, st)) return rc;
  } else if (int rc = launch_r2c<T>(F, rbuf, cbuf, rows, st)) {
    return rc;
  }
  ScaleArgs none{};
  return launch_strided<T, 0>(cbuf, F.ax[0], 0, (long long)n1 * nh, n1 * nh, 0, 1, (const C*)F.tw_ax[0], none, st,
                              nullptr, SFB_REG(F, 0));
}

template <typename T>
int fft_channel_inverse(FftSolve& F, void* cbuf_v, T* rbuf, cudaStream_t st) {
  typedef typename CX<T>::t C;
  C* cbuf = (C*)cbuf_v;
  const int n0 = F.n[0], n1 = F.n[1], nh = F.n[2] / 2 + 1;
  ScaleArgs none{};
  if (int rc = launch_strided<T, 1>(cbuf, F.ax[0], 0, (long long)n1 * nh, n1 * nh, 0, 1, (const C*)F.tw_ax[0], none,
                                    st, nullptr, SFB_REG(F, 0)))
    return rc;
  return launch_c2r<T>(F, cbuf, rbuf, (long long)n0 * n1, st);
}
template int fft_channel_forward<double>(FftSolve&, const double*, void*, cudaStream_t, const Geo<double>*,
                                         const void* const*);
template int fft_channel_forward<float>(FftSolve&, const float*, void*, cudaStream_t, const Geo<float>*,
                                        const void* const*);
template int fft_channel_inverse<double>(FftSolve&, void*, double*, cudaStream_t);
template int fft_channel_inverse<float>(FftSolve&, void*, float*, cudaStream_t);

template <typename T>
int fft_solve_inplace(FftSolve& F, T* rbuf, void* cbuf_v, cudaStream_t st, const Geo<T>* G, const void* const* u,
                      int gradt) {
  typedef typename CX<T>::t C;
  C* cbuf = (C*)cbuf_v;
  const size_t csz = sizeof(C);
  const int dim = F.dim;
  const int nlast = F.n[dim - 1];
  const int M = nlast / 2;
  const int nh = M + 1;
  const long long rows = F.total / nlast;
  // tiled spectrum (every pass in the register engine, r2c_epilogue): the
  // R2C writes it, the strided passes run on contiguous column blocks, the
  // C2R reads it
  // hybrid: natural rows, the strided passes on a tiled copy (F.tbuf)
  const bool hybrid = F.tlog > 0 && dim == 3 && F.tbuf;
  const bool tiled = F.tlog > 0 && dim == 3 && !F.tbuf && (!G || fft_divfuse_ok(F, *G));
  // 1. R2C along the contiguous axis (optionally of the divergence of u)
  if (G && fft_divfuse_ok(F, *G)) {
    RegCall c{};
    c.kind = 5;
    c.out = cbuf;
    c.rows = rows;
    c.out_row = nh;
    c.tlog = tiled ? F.tlog : 0;
    c.ks = F.tks;
    c.gradt = gradt;
    c.twL = F.tw_half;
    c.twN = F.tw_full;
    c.geo = G;
    for (int a = 0; a < 3; ++a) c.u[a] = u[a];
    int rc = reg_run<T>(reg_of(F.reg_half, F.reg_a_half, F.reg_b_half), c, st);
    if (rc) return rc;
  } else if (G) {
    if (gradt) return fail(SFB_EINVAL, "fused projection-pullback input needs the register R2C");
    size_t sm = 2 * (size_t)M * csz;
    CV<T> U;
    for (int a = 0; a < 3; ++a) U.c[a] = a < dim ? (const T*)u[a] : nullptr;
    const size_t smd = sm + (size_t)(2 * dim - 1) * nlast * sizeof(T);
    SFB_DISPATCH_DIM(dim, D,
                     (k_fft_r2c_div<T, D><<<(unsigned)rows, 128, smd, st>>>(*G, U, cbuf, F.half, (const C*)F.tw_half,
                                                                            (const C*)F.tw_full, nh)));
    SFB_LAUNCH_CHECK("fft r2c (fused divergence)");
  } else {
    int rc = launch_r2c<T>(F, rbuf, cbuf, rows, st, tiled);
    if (rc) return rc;
  }
  ScaleArgs none{};
  if (hybrid) {
    const int n0 = F.n[0], n1 = F.n[1], tw = 1 << F.tlog, nblk = (nh + tw - 1) / tw;
    C* tb = (C*)F.tbuf;
    int rc;
    // 2. axis 1 forward, natural -> tiled: each CTA reads 4-column segments of
    //    one plane and writes one contiguous (n1, tw) block
    RegCall c{};
    c.kind = 0;
    c.in = cbuf;
    c.out = tb;
    c.S_in = nh;
    c.bstride_in = (long long)n1 * nh;
    c.cbs_in = tw;
    c.S = tw;
    c.bstride = (long long)n1 * tw;
    c.cbs_out = F.tks;
    c.ncol = nh;
    c.nbatch = n0;
    c.twL = F.tw_ax[1];
    if ((rc = reg_run<T>(SFB_REG(F, 1), c, st))) return rc;
    // 3. axis 0 forward + scale + inverse in place on the tiled copy
    ScaleArgs sc = F.sc;
    sc.tlog = F.tlog;
    if ((rc = launch_strided<T, 2>(tb, F.ax[0], 0, (long long)n1 * tw, n1 * tw, F.tks, nblk, (const C*)F.tw_ax[0],
                                   sc, st, nullptr, SFB_REG(F, 0))))
      return rc;
    // 4. axis 1 inverse, tiled -> natural
    c.kind = 1;
    c.in = tb;
    c.out = cbuf;
    c.S_in = tw;
    c.bstride_in = (long long)n1 * tw;
    c.cbs_in = F.tks;
    c.S = nh;
    c.bstride = (long long)n1 * nh;
    c.cbs_out = tw;
    if ((rc = reg_run<T>(SFB_REG(F, 1), c, st))) return rc;
    return launch_c2r<T>(F, cbuf, rbuf, rows, st);
  }
  if (tiled) {
    const int n0 = F.n[0], n1 = F.n[1], tw = 1 << F.tlog, nblk = (nh + tw - 1) / tw;
    int rc;
    // 2. axis 1 forward: batch (block, k0) = one contiguous (n1, tw) array
    if ((rc = launch_strided<T, 0>(cbuf, F.ax[1], 0, tw, tw, (long long)n1 * tw, nblk * n0, (const C*)F.tw_ax[1],
                                   none, st, nullptr, SFB_REG(F, 1))))
      return rc;
    // 3. axis 0 forward + scale + inverse: batch = block, columns (k1, w) contiguous
    ScaleArgs sc = F.sc;
    sc.tlog = F.tlog;
    if ((rc = launch_strided<T, 2>(cbuf, F.ax[0], 0, (long long)n1 * tw, n1 * tw, F.tks, nblk, (const C*)F.tw_ax[0],
                                   sc, st, nullptr, SFB_REG(F, 0))))
      return rc;
    // 4. axis 1 inverse
    if ((rc = launch_strided<T, 1>(cbuf, F.ax[1], 0, tw, tw, (long long)n1 * tw, nblk * n0, (const C*)F.tw_ax[1],
                                   none, st, nullptr, SFB_REG(F, 1))))
      return rc;
    return launch_c2r<T>(F, cbuf, rbuf, rows, st, true);
  }
  if (dim == 3) {
    const int n0 = F.n[0], n1 = F.n[1];
    // 2. axis 1 forward: S = nh, columns k2 < nh, batch over k0
    int rc;
    if ((rc = launch_strided<T, 0>(cbuf, F.ax[1], pick_w(n1, csz), nh, nh, (long long)n1 * nh, n0,
                                   (const C*)F.tw_ax[1], none, st, &F.tma_ax1, SFB_REG(F, 1))))
      return rc;
    // 3. axis 0 forward + scale + inverse: S = n1*nh, columns (k1,k2)
    if ((rc = launch_strided<T, 2>(cbuf, F.ax[0], pick_w(n0, csz), (long long)n1 * nh, n1 * nh, 0, 1,
                                   (const C*)F.tw_ax[0], F.sc, st, &F.tma_ax0, SFB_REG(F, 0))))
      return rc;
    // 4. axis 1 inverse
    if ((rc = launch_strided<T, 1>(cbuf, F.ax[1], pick_w(n1, csz), nh, nh, (long long)n1 * nh, n0,
                                   (const C*)F.tw_ax[1], none, st, &F.tma_ax1, SFB_REG(F, 1))))
      return rc;
  } else {
    const int n0 = F.n[0];
    int rc;
    if ((rc = launch_strided<T, 2>(cbuf, F.ax[0], pick_w(n0, csz), nh, nh, 0, 1, (const C*)F.tw_ax[0], F.sc, st,
                                   nullptr, SFB_REG(F, 0))))
      return rc;
  }
  // 5. C2R along the contiguous axis
  return launch_c2r<T>(F, cbuf, rbuf, rows, st);
}
template int fft_solve_inplace<double>(FftSolve&, double*, void*, cudaStream_t, const Geo<double>*, const void* const*,
                                       int);
template int fft_solve_inplace<float>(FftSolve&, float*, void*, cudaStream_t, const Geo<float>*, const void* const*,
                                      int);

// Standalone unnormalised real transforms (the `transforms.rfftn/irfftn`
// plugin, transforms.py:9-12): R2C along the contiguous axis, then forward
// C2C passes along axes d-2 .. 0; the inverse runs the mirror image and
// overwrites its complex input.
template <typename T>
int fft_forward(FftSolve& F, const T* in, void* out_v, cudaStream_t st) {
  typedef typename CX<T>::t C;
  C* out = (C*)out_v;
  const size_t csz = sizeof(C);
  const int dim = F.dim, nlast = F.n[dim - 1], nh = nlast / 2 + 1;
  int rc;
  if ((rc = launch_r2c<T>(F, in, out, F.total / nlast, st))) return rc;
  ScaleArgs none{};
  if (dim == 3) {
    const int n0 = F.n[0], n1 = F.n[1];
    if ((rc = launch_strided<T, 0>(out, F.ax[1], pick_w(n1, csz), nh, nh, (long long)n1 * nh, n0,
                                   (const C*)F.tw_ax[1], none, st, nullptr, SFB_REG(F, 1))))
      return rc;
    return launch_strided<T, 0>(out, F.ax[0], pick_w(n0, csz), (long long)n1 * nh, n1 * nh, 0, 1,
                                (const C*)F.tw_ax[0], none, st, nullptr, SFB_REG(F, 0));
  }
  if (dim == 2)
    return launch_strided<T, 0>(out, F.ax[0], pick_w(F.n[0], csz), nh, nh, 0, 1, (const C*)F.tw_ax[0], none, st,
                                nullptr, SFB_REG(F, 0));
  return SFB_OK;
}
template int fft_forward<double>(FftSolve&, const double*, void*, cudaStream_t);
template int fft_forward<float>(FftSolve&, const float*, void*, cudaStream_t);

template <typename T>
int fft_inverse(FftSolve& F, void* in_v, T* out, cudaStream_t st) {
  typedef typename CX<T>::t C;
  C* in = (C*)in_v;
  const size_t csz = sizeof(C);
  const int dim = F.dim, nlast = F.n[dim - 1], nh = nlast / 2 + 1;
  int rc;
  ScaleArgs none{};
  if (dim == 3) {
    const int n0 = F.n[0], n1 = F.n[1];
    if ((rc = launch_strided<T, 1>(in, F.ax[0], pick_w(n0, csz), (long long)n1 * nh, n1 * nh, 0, 1,
                                   (const C*)F.tw_ax[0], none, st, nullptr, SFB_REG(F, 0))))
      return rc;
    if ((rc = launch_strided<T, 1>(in, F.ax[1], pick_w(n1, csz), nh, nh, (long long)n1 * nh, n0,
                                   (const C*)F.tw_ax[1], none, st, nullptr, SFB_REG(F, 1))))
      return rc;
  } else if (dim == 2) {
    if ((rc = launch_strided<T, 1>(in, F.ax[0], pick_w(F.n[0], csz), nh, nh, 0, 1, (const C*)F.tw_ax[0], none, st,
                                   nullptr, SFB_REG(F, 0))))
      return rc;
  }
  return launch_c2r<T>(F, in, out, F.total / nlast, st);
}
template int fft_inverse<double>(FftSolve&, void*, double*, cudaStream_t);
template int fft_inverse<float>(FftSolve&, void*, float*, cudaStream_t);

// ---- slab-decomposed pieces (multi-GPU): F.n = {m local planes, n1, n2},
// F.ax[0] is the global axis-0 length, F.sc.l1 offset to this rank's k1 chunk.
// chunked exchange layout of the slab all-to-all: (P, m, c, nh), c = n1 / P;
// element (q, i, r, k2) = k1 = q c + r of plane i
template <typename T>
__global__ void k_chunk_permute(const typename CX<T>::t* __restrict__ nat, typename CX<T>::t* __restrict__ xch, int m,
                                int n1, int c, int nh, int to_xchg) {
  typedef typename CX<T>::t C;
  const long long total = (long long)m * n1 * nh;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int k2 = (int)(t % nh);
    const long long r0 = t / nh;
    const int k1 = (int)(r0 % n1), i = (int)(r0 / n1);
    const long long x = (((long long)(k1 / c) * m + i) * c + (k1 % c)) * nh + k2;
    if (to_xchg) xch[x] = nat[t];
    else ((C*)nat)[t] = xch[x];
  }
}

// column chunk k of K over the nh half-spectrum columns
static void chunk_cols(int nh, int k, int K, int& c0, int& w) {
  const int base = (nh + K - 1) / K;
  c0 = k * base;
  w = nh - c0 < base ? nh - c0 : base;
}

template <typename T>
int fft_slab_r2c(FftSolve& F, T* rbuf, void* cbuf_v, cudaStream_t st, const Geo<T>* G, const void* const* u) {
  typedef typename CX<T>::t C;
  C* cbuf = (C*)cbuf_v;
  const int m = F.n[0], n1 = F.n[1], nh = F.n[2] / 2 + 1;
  const long long rows = (long long)m * n1;
  if (G && fft_divfuse_ok(F, *G)) {
    RegCall c{};
    c.kind = 5;
    c.out = cbuf;
    c.rows = rows;
    c.out_row = nh;
    c.twL = F.tw_half;
    c.twN = F.tw_full;
    c.geo = G;
    for (int a = 0; a < 3; ++a) c.u[a] = u[a];
    return reg_run<T>(reg_of(F.reg_half, F.reg_a_half, F.reg_b_half), c, st);
  }
  return launch_r2c<T>(F, rbuf, cbuf, rows, st);
}

// Axis-1 FFT of column chunk k of K.  One rank: in place on the natural
// spectrum (the whole width).  P ranks: forward writes / inverse reads the
// chunk's all-to-all block of xbuf, laid out (P, m, n1/P, w) (rank q's k1
// range contiguous), so the exchange needs no packing.
template <typename T>
int fft_slab_axis1(FftSolve& F, void* cbuf_v, void* xbuf, int nranks, int k, int K, bool inverse, cudaStream_t st) {
  typedef typename CX<T>::t C;
  C* cbuf = (C*)cbuf_v;
  const int m = F.n[0], n1 = F.n[1], nh = F.n[2] / 2 + 1;
  ScaleArgs none{};
  if (!xbuf || nranks <= 1) {
    if (inverse)
      return launch_strided<T, 1>(cbuf, F.ax[1], pick_w(n1, sizeof(C)), nh, nh, (long long)n1 * nh, m,
                                  (const C*)F.tw_ax[1], none, st, &F.tma_ax1, SFB_REG(F, 1));
    return launch_strided<T, 0>(cbuf, F.ax[1], pick_w(n1, sizeof(C)), nh, nh, (long long)n1 * nh, m,
                                (const C*)F.tw_ax[1], none, st, &F.tma_ax1, SFB_REG(F, 1));
  }
  const int c = n1 / nranks;
  int c0, w;
  chunk_cols(nh, k, K, c0, w);
  if (w <= 0) return SFB_OK;
  C* xk = (C*)xbuf + (long long)nranks * m * c * c0;
  if (!F.reg_ax[1]) {
    // Stockham / cuFFT-length fallback: whole-width transform + permute copy
    if (K != 1) return fail(SFB_EINVAL, "chunked slab exchange needs the register FFT engine");
    if (inverse) {
      k_chunk_permute<T><<<148 * 8, 256, 0, st>>>(cbuf, xk, m, n1, c, nh, 0);
      SFB_LAUNCH_CHECK("slab unpack");
      return launch_strided<T, 1>(cbuf, F.ax[1], pick_w(n1, sizeof(C)), nh, nh, (long long)n1 * nh, m,
                                  (const C*)F.tw_ax[1], none, st, &F.tma_ax1, RegLen{});
    }
    int rc = launch_strided<T, 0>(cbuf, F.ax[1], pick_w(n1, sizeof(C)), nh, nh, (long long)n1 * nh, m,
                                  (const C*)F.tw_ax[1], none, st, &F.tma_ax1, RegLen{});
    if (rc) return rc;
    k_chunk_permute<T><<<148 * 8, 256, 0, st>>>(cbuf, xk, m, n1, c, nh, 1);
    SFB_LAUNCH_CHECK("slab pack");
    return SFB_OK;
  }
  RegCall rc{};
  rc.kind = inverse ? 7 : 6;
  rc.in = inverse ? (const void*)xk : (const void*)(cbuf + c0);
  rc.out = inverse ? (void*)(cbuf + c0) : (void*)xk;
  rc.ncol = w;
  rc.nbatch = m;
  rc.S = nh;  // the natural side's row stride
  rc.map_c = c;
  rc.map_sq = (long long)m * c * w;
  rc.map_s = w;
  rc.bstride_in = inverse ? (long long)c * w : (long long)n1 * nh;
  rc.bstride = inverse ? (long long)n1 * nh : (long long)c * w;
  rc.twL = F.tw_ax[1];
  return reg_run<T>(SFB_REG(F, 1), rc, st);
}

// Axis-0 forward -> 1/(Lambda N) -> inverse on column chunk k of K of the
// transposed spectrum (n0, n1/P, w) (the whole spectrum in place when P = 1)
template <typename T>
int fft_slab_axis0(FftSolve& F, void* tbuf_v, int n1_chunk, int nranks, int k, int K, cudaStream_t st) {
  typedef typename CX<T>::t C;
  const int nh = F.n[2] / 2 + 1;
  int c0 = 0, w = nh;
  if (nranks > 1) chunk_cols(nh, k, K, c0, w);
  if (w <= 0) return SFB_OK;
  C* tk = (C*)tbuf_v + (long long)F.ax[0].L * n1_chunk * c0;
  ScaleArgs sc = F.sc;
  sc.nh = w;
  sc.l2 = F.sc.l2 + c0;
  sc.zero_ok = F.sc.zero_ok && c0 == 0;
  const int ncol = n1_chunk * w;
  return launch_strided<T, 2>(tk, F.ax[0], pick_w(F.ax[0].L, sizeof(C)), ncol, ncol, 0, 1, (const C*)F.tw_ax[0], sc,
                              st, K == 1 ? &F.tma_ax0 : nullptr, SFB_REG(F, 0));
}

template <typename T>
int fft_slab_c2r(FftSolve& F, void* cbuf, T* rbuf, cudaStream_t st) {
  typedef typename CX<T>::t C;
  return launch_c2r<T>(F, (const C*)cbuf, rbuf, (long long)F.n[0] * F.n[1], st);
}

#define SFB_SLAB_INST(T)                                                                                          \
  template int fft_slab_r2c<T>(FftSolve&, T*, void*, cudaStream_t, const Geo<T>*, const void* const*);            \
  template int fft_slab_axis1<T>(FftSolve&, void*, void*, int, int, int, bool, cudaStream_t);                     \
  template int fft_slab_axis0<T>(FftSolve&, void*, int, int, int, int, cudaStream_t);                             \
  template int fft_slab_c2r<T>(FftSolve&, void*, T*, cudaStream_t);
SFB_SLAB_INST(double)
SFB_SLAB_INST(float)
#undef SFB_SLAB_INST

template <typename T>
int fft_set_smem_limits() {
  if (int rc = fft_reg_init()) return rc;
  const int big = 200 * 1024;
  cudaError_t e = cudaSuccess;
#define SFB_SMEM(K) \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, big)
  SFB_SMEM((k_fft_strided<T, 0, 1>));
  SFB_SMEM((k_fft_strided<T, 0, 2>));
  SFB_SMEM((k_fft_strided<T, 0, 4>));
  SFB_SMEM((k_fft_strided<T, 0, 8>));
  SFB_SMEM((k_fft_strided<T, 1, 1>));
  SFB_SMEM((k_fft_strided<T, 1, 2>));
  SFB_SMEM((k_fft_strided<T, 1, 4>));
  SFB_SMEM((k_fft_strided<T, 1, 8>));
  SFB_SMEM((k_fft_strided<T, 2, 1>));
  SFB_SMEM((k_fft_strided<T, 2, 2>));
  SFB_SMEM((k_fft_strided<T, 2, 4>));
  SFB_SMEM((k_fft_strided<T, 2, 8>));
  SFB_SMEM(k_fft_r2c<T>);
  SFB_SMEM((k_fft_r2c_div<T, 2>));
  SFB_SMEM((k_fft_r2c_div<T, 3>));
  SFB_SMEM(k_fft_c2r<T>);
#undef SFB_SMEM
  return cuda_check(e, "cudaFuncSetAttribute(fft smem)");
}
template int fft_set_smem_limits<double>();
template int fft_set_smem_limits<float>();

}  // namespace sfb
