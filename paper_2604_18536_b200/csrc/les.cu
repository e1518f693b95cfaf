// Eddy-viscosity closures on the GPU (les.py:58-417): the velocity gradient
// at the pressure points, the six models' nu_t, and the divergence of the
// modelled stress 2 nu_t S on the velocity DOFs.  One thread per cell; every
// formula keeps the reference's operands and order (the four-corner
// averages, the degenerate-denominator rules); divisions by the width tables
// are multiplications by their reciprocal tables (one rounding apart).
// The sigma model's singular values are formed in fp64 from the
// characteristic invariants (the reference uses numpy longdouble, les.py:168).
#include <cmath>

#include "sfb_kernels.cuh"

namespace sfb {

enum { LES_SMAG = 1, LES_VREMAN, LES_QR, LES_WALE, LES_SIGMA, LES_S3PQR };

// velocity gradient at cell I (extended indices), les.py:58-88
template <typename T, int D>
__device__ __forceinline__ void grad_tensor(const Geo<T>& G, const CV<T>& U, const int I[3], long long x, T A[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[i][j] = T(0);
#pragma unroll
  for (int i = 0; i < D; ++i) A[i][i] = (U.c[i][x] - U.c[i][x - G.s[i]]) * tab(G, i, T_RDX, I[i]);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (i == j) continue;
      // corner (ci, cj) = (I_i - 1 + oi, I_j - 1 + oj): (u_i[.., cj+1] - u_i[.., cj]) / du_j[cj]
      T acc = T(0);
      bool first = true;
#pragma unroll
      for (int oi = 0; oi < 2; ++oi)
#pragma unroll
        for (int oj = 0; oj < 2; ++oj) {
          const long long c = x + (long long)(oi - 1) * G.s[i] + (long long)(oj - 1) * G.s[j];
          const T part = (U.c[i][c + G.s[j]] - U.c[i][c]) * tab(G, j, T_RDU, I[j] - 1 + oj);
          acc = first ? part : acc + part;
          first = false;
        }
      A[i][j] = T(0.25) * acc;
    }
}

// closed-form eigenvalues of a symmetric 3x3 (two leading), les.py:122-148
__device__ __forceinline__ void sym_eigs(const double m[3][3], double& e1, double& e2) {
  const double m00 = m[0][0], m11 = m[1][1], m22 = m[2][2], m01 = m[0][1], m02 = m[0][2], m12 = m[1][2];
  const double off = m01 * m01 + m02 * m02 + m12 * m12;
  const double q = (m00 + m11 + m22) / 3.0;
  const double p2 = (m00 - q) * (m00 - q) + (m11 - q) * (m11 - q) + (m22 - q) * (m22 - q) + 2.0 * off;
  const double pp = sqrt(fmax(p2 / 6.0, 0.0));
  if (!(pp > 0)) {
    e1 = q;
    e2 = q;
    return;
  }
  const double b00 = (m00 - q) / pp, b11 = (m11 - q) / pp, b22 = (m22 - q) / pp;
  const double b01 = m01 / pp, b02 = m02 / pp, b12 = m12 / pp;
  const double det = b00 * (b11 * b22 - b12 * b12) - b01 * (b01 * b22 - b12 * b02) + b02 * (b01 * b12 - b11 * b02);
  const double phi = acos(fmin(fmax(det / 2.0, -1.0), 1.0)) / 3.0;
  e1 = q + 2.0 * pp * cos(phi);
  const double e3 = q + 2.0 * pp * cos(phi + 2.0 * M_PI / 3.0);
  e2 = 3.0 * q - e1 - e3;
}

// x^e on x > 0 (else 0); a negative exponent on x <= 0 flags a degenerate point
template <typename T>
__device__ __forceinline__ T pow_or_flag(T x, T e, bool& bad) {
  if (e == T(0)) return T(1);
  if (x > T(0)) return pow(x, e);
  if (e < T(0)) bad = true;
  return T(0);
}

template <typename T, int D, int KIND>
__global__ void __launch_bounds__(256) k_nut(Geo<T> G, CV<T> U, T c, T pexp, T* __restrict__ nut, Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
  T A[3][3];
  grad_tensor<T, D>(G, U, I, x, A);
  T S[3][3], W[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      S[i][j] = T(0.5) * (A[i][j] + A[j][i]);
      W[i][j] = T(0.5) * (A[i][j] - A[j][i]);
    }
  // filter width (les.py:297-305): (prod dx)^(1/d)
  T prod = T(1);
#pragma unroll
  for (int a = 0; a < D; ++a) prod = prod * tab(G, a, T_DX, I[a]);
  const T delta = D == 3 ? cbrt(prod) : D == 2 ? sqrt(prod) : prod;
  const T cd2 = (c * delta) * (c * delta);
  T val = T(0);
  if (KIND == LES_SMAG || KIND == LES_QR) {
    T qs = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) qs += S[i][j] * S[j][i];
    qs = T(-0.5) * qs;
    if (KIND == LES_SMAG) {
      val = cd2 * sqrt(fmax(T(-4) * qs, T(0)));
    } else {
      T rs;
      // structurally two-component tensor: third row and column zero (les.py:101-108)
      const bool planar = D == 2 || (A[2][0] == T(0) && A[2][1] == T(0) && A[2][2] == T(0) && A[0][2] == T(0) &&
                                     A[1][2] == T(0));
      if (planar) {
        const T t2 = S[0][0] + S[1][1];
        const T det2 = S[0][0] * S[1][1] - S[0][1] * S[1][0];
        rs = t2 * (t2 * t2 - T(3) * det2) / T(3);
      } else {
        rs = T(0);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) rs += S[i][j] * S[j][k] * S[k][i];
        rs = rs / T(3);
      }
      val = qs < T(0) ? cd2 * (fabs(rs) / -qs) : T(0);
    }
  } else if (KIND == LES_VREMAN) {
    T dm[3] = {T(0), T(0), T(0)};
#pragma unroll
    for (int m = 0; m < D; ++m) dm[m] = tab(G, m, T_DX, I[m]);
    T rows[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int m = 0; m < 3; ++m) rows[i][m] = A[i][m] * dm[m];
    T b = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i + 1; j < 3; ++j) {
        const T c0 = rows[i][1] * rows[j][2] - rows[i][2] * rows[j][1];
        const T c1 = rows[i][2] * rows[j][0] - rows[i][0] * rows[j][2];
        const T c2 = rows[i][0] * rows[j][1] - rows[i][1] * rows[j][0];
        b = b + (c0 * c0 + c1 * c1 + c2 * c2);
      }
    T paa = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) paa += A[i][j] * A[i][j];
    const T den = paa / T(2);
    val = den > T(0) ? c * c * sqrt(b / den) : T(0);
  } else if (KIND == LES_WALE) {
    T A2[3][3], sd[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        T s = T(0);
#pragma unroll
        for (int j = 0; j < 3; ++j) s += A[i][j] * A[j][k];
        A2[i][k] = s;
      }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) sd[i][j] = T(0.5) * (A2[i][j] + A2[j][i]);
    const T tr = sd[0][0] + sd[1][1] + sd[2][2];
#pragma unroll
    for (int i = 0; i < 3; ++i) sd[i][i] -= tr / T(3);
    T sdsd = T(0), ss = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        sdsd += sd[i][j] * sd[i][j];
        ss += S[i][j] * S[i][j];
      }
    const T den = pow(ss, T(2.5)) + pow(sdsd, T(1.25));
    val = den > T(0) ? cd2 * (pow(sdsd, T(1.5)) / den) : T(0);
  } else if (KIND == LES_SIGMA) {
    // singular values (les.py:160-179).  The reference evaluates the closed-form
    // eigenvalues of A^T A in longdouble; in fp64 the second eigenvalue of a
    // nearly two-component gradient would cancel, so it is formed here from
    // the characteristic invariants instead: e2 + e3 = (I2 - e2 e3) / e1,
    // e2 e3 = I3 / e1, with I2 = sum |c_i x c_j|^2 over the columns of A
    // (Lagrange identity, no cancellation) and I3 = det(A)^2.
    double ata[3][3], col[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) col[i][k] = (double)A[k][i];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) ata[i][j] = col[i][0] * col[j][0] + col[i][1] * col[j][1] + col[i][2] * col[j][2];
    double e1, e2x;
    sym_eigs(ata, e1, e2x);
    const double a00 = A[0][0], a01 = A[0][1], a02 = A[0][2], a10 = A[1][0], a11 = A[1][1], a12 = A[1][2];
    const double a20 = A[2][0], a21 = A[2][1], a22 = A[2][2];
    const double dt = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20);
    const double det = fabs(dt);
    double i2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i + 1; j < 3; ++j) {
        const double x0 = col[i][1] * col[j][2] - col[i][2] * col[j][1];
        const double x1 = col[i][2] * col[j][0] - col[i][0] * col[j][2];
        const double x2 = col[i][0] * col[j][1] - col[i][1] * col[j][0];
        i2 += x0 * x0 + x1 * x1 + x2 * x2;
      }
    double e2 = 0.0;
    if (e1 > 0.0) {
      const double pr23 = det * det / e1;
      const double sum23 = fmax((i2 - pr23) / e1, 0.0);
      e2 = 0.5 * (sum23 + sqrt(fmax(sum23 * sum23 - 4.0 * pr23, 0.0)));
    }
    (void)e2x;
    const double s1 = sqrt(fmax(e1, 0.0)), s2 = sqrt(fmax(e2, 0.0));
    const double pr = s1 * s2;
    const double s3 = fmin(pr > 0.0 ? det / pr : 0.0, s2);
    if (s1 > 0.0) {
      const double v = s3 * (s1 - s2) * (s2 - s3) / (s1 * s1);
      val = cd2 * (T)fmax(v, 0.0);
    }
  } else {  // S3PQR
    T qa = T(0), paa = T(0), ra = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        qa += A[i][j] * A[j][i];
        paa += A[i][j] * A[i][j];
#pragma unroll
        for (int k = 0; k < 3; ++k) ra += A[i][j] * A[j][k] * A[k][i];
      }
    qa = T(-0.5) * qa;
    ra = ra / T(3);
    const T om[3] = {W[2][1], W[0][2], W[1][0]};
    T v2 = T(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const T so = S[i][0] * om[0] + S[i][1] * om[1] + S[i][2] * om[2];
      v2 += so * so;
    }
    v2 = T(4) * v2;
    const T qaa = v2 + qa * qa, raa = ra * ra;
    bool bad = false;
    const T f1 = pow_or_flag(paa, pexp, bad);
    const T f2 = pow_or_flag(qaa, -(pexp + T(1)), bad);
    const T f3 = pow_or_flag(raa, (pexp + T(2.5)) / T(3), bad);
    val = bad ? T(0) : cd2 * (f1 * f2 * f3);
  }
  nut[x] = val;
}

// out_a (+)= div(2 nu_t S)_a on the velocity DOFs (les.py:343-417); nut with
// filled ghosts
template <typename T, int D>
__global__ void __launch_bounds__(256) k_eddy(Geo<T> G, CV<T> U, const T* __restrict__ nut, MV<T> out, int accumulate,
                                              Box B) {
  int I[3];
  if (!box_coords<D>(B, I)) return;
  const long long x = lin<T, D>(G, I);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (!is_udof<T, D>(G, I, a)) continue;
    const T* __restrict__ ua = U.c[a];
    const long long sa = G.s[a];
    T v = accumulate ? out.c[a][x] : T(0);
#pragma unroll
    for (int b = 0; b < D; ++b) {
      T t;
      if (b == a) {
        // centre fluxes 2 nu_t A_aa at I and I + e_a
        T fl[2];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const long long c = x + o * sa;
          T g = (ua[c] - ua[c - sa]) * tab(G, a, T_RDX, I[a] + o);
          g = g * nut[c];
          fl[o] = g * T(2);
        }
        t = (fl[1] - fl[0]) * tab(G, a, T_RDU, I[a]);
      } else {
        // corner fluxes 2 nu_t S_ab at corners I_b - 1 and I_b along b
        const T* __restrict__ ub = U.c[b];
        const long long sb = G.s[b];
        T fl[2];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const long long c = x + (long long)(o - 1) * sb;
          T sab = (ua[c + sb] - ua[c]) * tab(G, b, T_RDU, I[b] - 1 + o);
          sab = sab + (ub[c + sa] - ub[c]) * tab(G, a, T_RDU, I[a]);
          T nc = nut[c] + nut[c + sa];
          nc = nc + (nut[c + sb] + nut[c + sa + sb]);
          nc = nc * T(0.25);
          fl[o] = sab * nc;
        }
        t = (fl[1] - fl[0]) * tab(G, b, T_RDX, I[b]);
      }
      v += t;
    }
    out.c[a][x] = v;
  }
}

// min / max of a scalar's interior (deterministic two-pass)
template <typename T, int D>
__global__ void __launch_bounds__(256) k_minmax(Geo<T> G, const T* __restrict__ f, double* __restrict__ part) {
  const long long total = (long long)G.n[0] * G.n[1] * (D == 3 ? G.n[2] : 1);
  double mn = INFINITY, mx = -INFINITY;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    long long r = t;
    if (D == 3) {
      I[2] = 1 + (int)(r % G.n[2]);
      r /= G.n[2];
    } else {
      I[2] = 0;
    }
    I[1] = 1 + (int)(r % G.n[1]);
    I[0] = 1 + (int)(r / G.n[1]);
    const double v = (double)f[lin<T, D>(G, I)];
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  __shared__ double smn[8], smx[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    part[2 * blockIdx.x] = mn;
    part[2 * blockIdx.x + 1] = mx;
  }
}

__global__ void k_minmax_finish(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double mn = INFINITY, mx = -INFINITY;
  for (int i = 0; i < nb; ++i) {
    mn = fmin(mn, part[2 * i]);
    mx = fmax(mx, part[2 * i + 1]);
  }
  out[0] = mn;
  out[1] = mx;
}

template <typename T>
static int closure_nut_run(sfb_plan* p, int kind, double c, double pexp, const void* const* u, void* nut,
                           cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  CV<T> U;
  for (int a = 0; a < 3; ++a) U.c[a] = a < p->dim ? (const T*)u[a] : nullptr;
  Box B = int_box(G);
  T* f = (T*)nut;
#define SFB_NUT(K) \
  SFB_DISPATCH_DIM(G.dim, D, (k_nut<T, D, K><<<box_grid(D, B), box_block(D), 0, st>>>(G, U, (T)c, (T)pexp, f, B)))
  switch (kind) {
    case LES_SMAG: SFB_NUT(LES_SMAG); break;
    case LES_VREMAN: SFB_NUT(LES_VREMAN); break;
    case LES_QR: SFB_NUT(LES_QR); break;
    case LES_WALE: SFB_NUT(LES_WALE); break;
    case LES_SIGMA: SFB_NUT(LES_SIGMA); break;
    default: SFB_NUT(LES_S3PQR); break;
  }
#undef SFB_NUT
  SFB_LAUNCH_CHECK("closure nu_t");
  return SFB_OK;
}

// ---------------------------------------------------------------------------
// Pullback of the Smagorinsky closure term E(u) = div(2 nu_t(u) S(u)) on a
// periodic 3D grid: out += (dE/du)^T Ebar, both through the resolved
// gradients (nu_t fixed) and through nu_t = (c Delta)^2 |S|.  The reference's
// tape leaves closures out (adjoint.py:374); this is the a-posteriori
// training extension.  Three gather passes over intermediate
// cell fields (periodic ghosts filled between them, so every stencil reach
// is a plain +-1 read), no atomics: the result is deterministic.
//   K1 (cell c): centre flux cotangents Fbar_a = Ebar_a[c-e_a]/du_a[c_a-1]
//       - Ebar_a[c]/du_a[c_a] -> gbar_a = 2 nu Fbar_a, nud = sum 2 g_a Fbar_a;
//       corner (a<b) cotangents Fcbar from E_a and E_b -> sbar = Fcbar nc,
//       W = Fcbar sab (for the four nu_t of the corner average)
//   K2 (cell c): nubar = nud + 1/4 sum_pairs W over the corners touching c;
//       Abar_ij = nubar (c Delta)^2 2 S_ij / |S| (symmetric, 6 fields)
//   K3 (velocity DOF J): the transposes of the centre / corner differences
//       and of grad_tensor, gathered from gbar, sbar, Abar
// scratch layout (extended scalars): 0-2 gbar, 3-5 sbar (pairs 01, 02, 12),
// 6 nud, 7-9 W, 10-15 Abar (00, 11, 22, 01, 02, 12)
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int pair_a(int p) { return p < 2 ? 0 : 1; }  // pairs (0,1) (0,2) (1,2)
__host__ __device__ constexpr int pair_b(int p) { return p == 0 ? 1 : 2; }
__host__ __device__ constexpr int pair_of(int a, int b) { return a + b - 1; }  // (0,1)->0 (0,2)->1 (1,2)->2

template <typename T>
__global__ void __launch_bounds__(256) k_cpb1(Geo<T> G, CV<T> U, const T* __restrict__ nut, CV<T> Eb,
                                              T* __restrict__ scr, long long fs, Box B) {
  int I[3];
  if (!box_coords<3>(B, I)) return;
  const long long x = lin<T, 3>(G, I);
  T nud = T(0);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long sa = G.s[a];
    const T fb = Eb.c[a][x - sa] * tab(G, a, T_RDU, I[a] - 1) - Eb.c[a][x] * tab(G, a, T_RDU, I[a]);
    const T g = (U.c[a][x] - U.c[a][x - sa]) * tab(G, a, T_RDX, I[a]);
    scr[a * fs + x] = T(2) * nut[x] * fb;
    nud += T(2) * g * fb;
  }
  scr[6 * fs + x] = nud;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int a = pair_a(p), b = pair_b(p);
    const long long sa = G.s[a], sb = G.s[b];
    const T fcb = (Eb.c[a][x] * tab(G, b, T_RDX, I[b]) - Eb.c[a][x + sb] * tab(G, b, T_RDX, I[b] + 1)) +
                  (Eb.c[b][x] * tab(G, a, T_RDX, I[a]) - Eb.c[b][x + sa] * tab(G, a, T_RDX, I[a] + 1));
    const T sab = (U.c[a][x + sb] - U.c[a][x]) * tab(G, b, T_RDU, I[b]) +
                  (U.c[b][x + sa] - U.c[b][x]) * tab(G, a, T_RDU, I[a]);
    const T nc = T(0.25) * ((nut[x] + nut[x + sa]) + (nut[x + sb] + nut[x + sa + sb]));
    scr[(3 + p) * fs + x] = fcb * nc;
    scr[(7 + p) * fs + x] = fcb * sab;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_cpb2(Geo<T> G, CV<T> U, T c, T* __restrict__ scr, long long fs, Box B) {
  int I[3];
  if (!box_coords<3>(B, I)) return;
  const long long x = lin<T, 3>(G, I);
  T nub = scr[6 * fs + x];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const long long sa = G.s[pair_a(p)], sb = G.s[pair_b(p)];
    const T* W = scr + (7 + p) * fs;
    nub += T(0.25) * ((W[x] + W[x - sa]) + (W[x - sb] + W[x - sa - sb]));
  }
  T A[3][3];
  grad_tensor<T, 3>(G, U, I, x, A);
  T S[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) S[i][j] = T(0.5) * (A[i][j] + A[j][i]);
  T q = T(0);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) q += S[i][j] * S[j][i];
  const T mag = sqrt(fmax(T(2) * q, T(0)));  // |S| = sqrt(-4 qs), qs = -q/2 (k_nut)
  T prod = T(1);
#pragma unroll
  for (int a = 0; a < 3; ++a) prod = prod * tab(G, a, T_DX, I[a]);
  const T delta = cbrt(prod);
  const T cd2 = (c * delta) * (c * delta);
  // d|S|/dA_ij = 2 S_ij / |S| (zero where |S| = 0: the subgradient the
  // forward's max(., 0) takes)
  const T f = mag > T(0) ? nub * cd2 * T(2) / mag : T(0);
  scr[10 * fs + x] = f * S[0][0];
  scr[11 * fs + x] = f * S[1][1];
  scr[12 * fs + x] = f * S[2][2];
  scr[13 * fs + x] = f * S[0][1];
  scr[14 * fs + x] = f * S[0][2];
  scr[15 * fs + x] = f * S[1][2];
}

template <typename T>
__device__ __forceinline__ int abar_slot(int i, int j) {
  return i == j ? 10 + i : 13 + pair_of(i < j ? i : j, i < j ? j : i);
}

template <typename T>
__global__ void __launch_bounds__(256) k_cpb3(Geo<T> G, const T* __restrict__ scr, long long fs, MV<T> out, Box B) {
  int I[3];
  if (!box_coords<3>(B, I)) return;
  const long long x = lin<T, 3>(G, I);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const long long si = G.s[i];
    // centre differences: eddy flux gradients and grad_tensor's diagonal
    const T* gb = scr + i * fs;
    const T* Ad = scr + (10 + i) * fs;
    T v = (gb[x] + Ad[x]) * tab(G, i, T_RDX, I[i]) - (gb[x + si] + Ad[x + si]) * tab(G, i, T_RDX, I[i] + 1);
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      if (o == i) continue;
      const long long so = G.s[o];
      // corner strain 2 S_io of the eddy fluxes
      const T* sb = scr + (3 + pair_of(i < o ? i : o, i < o ? o : i)) * fs;
      v += sb[x - so] * tab(G, o, T_RDU, I[o] - 1) - sb[x] * tab(G, o, T_RDU, I[o]);
      // grad_tensor's four-corner average of du_i / dx_o
      const T* Ab = scr + abar_slot<T>(i, o) * fs;
      const T lo = (Ab[x] + Ab[x + si]) + (Ab[x - so] + Ab[x + si - so]);
      const T hi = (Ab[x] + Ab[x + si]) + (Ab[x + so] + Ab[x + si + so]);
      v += T(0.25) * (lo * tab(G, o, T_RDU, I[o] - 1) - hi * tab(G, o, T_RDU, I[o]));
    }
    out.c[i][x] += v;
  }
}

template <typename T>
static int closure_pullback_run(sfb_plan* p, double c, const void* const* u, const void* nut, const void* const* vbar,
                                void* const* out, void* scratch, cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  CV<T> U, Eb;
  MV<T> O;
  for (int a = 0; a < 3; ++a) {
    U.c[a] = (const T*)u[a];
    Eb.c[a] = (const T*)vbar[a];
    O.c[a] = (T*)out[a];
  }
  T* scr = (T*)scratch;
  const long long fs = p->ext_count;
  Box B = int_box(G);
  k_cpb1<T><<<box_grid(3, B), box_block(3), 0, st>>>(G, U, (const T*)nut, Eb, scr, fs, B);
  SFB_LAUNCH_CHECK("closure pullback 1");
  for (int f = 0; f < 10; f += 3)
    if (int rc = launch_planes<T>(G, MV<T>{{scr + f * fs, f + 1 < 10 ? scr + (f + 1) * fs : nullptr,
                                              f + 2 < 10 ? scr + (f + 2) * fs : nullptr}},
                                  f + 3 <= 10 ? 3 : 10 - f, 1, st))
      return rc;
  k_cpb2<T><<<box_grid(3, B), box_block(3), 0, st>>>(G, U, (T)c, scr, fs, B);
  SFB_LAUNCH_CHECK("closure pullback 2");
  for (int f = 10; f < 16; f += 3)
    if (int rc = launch_planes<T>(G, MV<T>{{scr + f * fs, scr + (f + 1) * fs, scr + (f + 2) * fs}}, 3, 1, st))
      return rc;
  k_cpb3<T><<<box_grid(3, B), box_block(3), 0, st>>>(G, scr, fs, O, B);
  SFB_LAUNCH_CHECK("closure pullback 3");
  return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_closure_nut(sfb_plan* p, int kind, double c, double pexp, const void* const* u, void* nut, void* stream) {
  SFB_RANGE();
  if (!p || !u || !nut) return fail(SFB_EINVAL, "null argument");
  for (int a = 0; a < p->dim; ++a)
    if (!u[a]) return fail(SFB_EINVAL, "null velocity component");
  if (kind < LES_SMAG || kind > LES_S3PQR) return fail(SFB_ECONFIG, "unknown closure kind");
  if (c < 0) return fail(SFB_EINVAL, "closure constant must be nonnegative");
  return SFB_TYPED(p, closure_nut_run<T>(p, kind, c, pexp, u, nut, (cudaStream_t)stream));
}

int sfb_eddy_stress_divergence(sfb_plan* p, const void* const* u, const void* nut, void* const* out, int accumulate,
                               void* stream) {
  SFB_RANGE();
  if (!p || !u || !nut || !out) return fail(SFB_EINVAL, "null argument");
  for (int a = 0; a < p->dim; ++a)
    if (!u[a] || !out[a]) return fail(SFB_EINVAL, "null velocity component");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() -> int {
    const Geo<T>& G = geo<T>(p);
    CV<T> U;
    MV<T> O;
    for (int a = 0; a < 3; ++a) {
      U.c[a] = a < p->dim ? (const T*)u[a] : nullptr;
      O.c[a] = a < p->dim ? (T*)out[a] : nullptr;
    }
    if (!accumulate)
      for (int a = 0; a < p->dim; ++a)
        if (int rc = cuda_check(cudaMemsetAsync(O.c[a], 0, sizeof(T) * p->ext_count, st), "zero out")) return rc;
    Box B = int_box(G);
    SFB_DISPATCH_DIM(G.dim, D,
                     (k_eddy<T, D><<<box_grid(D, B), box_block(D), 0, st>>>(G, U, (const T*)nut, O, accumulate, B)));
    SFB_LAUNCH_CHECK("eddy stress divergence");
    return SFB_OK;
  }()));
}

int sfb_closure_pullback(sfb_plan* p, int kind, double c, const void* const* u, const void* nut,
                         const void* const* vbar, void* const* out, void* scratch, void* stream) {
  SFB_RANGE();
  if (!p || !u || !nut || !vbar || !out || !scratch) return fail(SFB_EINVAL, "null argument");
  if (kind != LES_SMAG) return fail(SFB_ECONFIG, "closure pullback: Smagorinsky only");
  if (p->dim != 3 || !p->all_periodic) return fail(SFB_ECONFIG, "closure pullback: periodic 3D grids only");
  for (int a = 0; a < 3; ++a)
    if (!u[a] || !vbar[a] || !out[a]) return fail(SFB_EINVAL, "null velocity component");
  return SFB_TYPED(p, closure_pullback_run<T>(p, c, u, nut, vbar, out, scratch, (cudaStream_t)stream));
}

int sfb_scalar_minmax(sfb_plan* p, const void* f, double* mn, double* mx, void* stream) {
  SFB_RANGE();
  if (!p || !f || !mn || !mx) return fail(SFB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int nb = p->red_blocks / 2;
  const long long need = (p->int_count + 255) / 256;
  if (need < nb) nb = (int)(need > 0 ? need : 1);
  int rc = SFB_TYPED(p, ([&]() -> int {
    const Geo<T>& G = geo<T>(p);
    SFB_DISPATCH_DIM(G.dim, D, (k_minmax<T, D><<<nb, 256, 0, st>>>(G, (const T*)f, p->d_red)));
    SFB_LAUNCH_CHECK("scalar min/max");
    return SFB_OK;
  }()));
  if (rc) return rc;
  // partials occupy d_red[0 .. 2 nb); the result goes to the two slots after
  k_minmax_finish<<<1, 32, 0, st>>>(p->d_red, nb, p->d_red + 2 * nb);
  if ((rc = cuda_check(cudaGetLastError(), "min/max finish"))) return rc;
  if ((rc = cuda_check(cudaMemcpyAsync(p->h_red, p->d_red + 2 * nb, 2 * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "d2h")))
    return rc;
  if ((rc = cuda_check(cudaStreamSynchronize(st), "sync"))) return rc;
  *mn = p->h_red[0];
  *mx = p->h_red[1];
  return SFB_OK;
}

}  // extern "C"
