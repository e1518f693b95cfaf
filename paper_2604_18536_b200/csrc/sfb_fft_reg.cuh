// Register-resident two-level FFT engine (sm_100a) for the spectral solve.
//
// A length-L transform with L = A*B (A, B <= 32) is done as one "four-step":
//   n = B*n1 + n2, k = k1 + A*k2
//   phase 1: B threads, thread n2 holds x[B*n1 + n2] (n1 < A) in registers,
//            A-point DFT, twiddle W_L^(n2*k1)
//   exchange through shared memory (the only one)
//   phase 2: A threads, thread k1 holds the B values of its k1, B-point DFT,
//            result X[k1 + A*k2] (natural order) in registers
// The A- and B-point DFTs are themselves four-steps over the radices
// 8/7/5/4/3/2 with compile-time indices, so the data never leaves registers
// inside a phase; twiddles of the sub-DFTs come from the constant bank.
//
// Compared with the shared-memory Stockham engine (fft.cu: one smem round trip
// and one __syncthreads per radix pass) this does one exchange per transform,
// loads straight from HBM into registers and stores straight back, which is
// what lets the strided passes run at HBM speed.  The fused
// forward -> eigenvalue scaling -> inverse pass (axis 0) keeps the spectrum of
// a column in registers between the forward phase 2 and the inverse phase 1.
#pragma once

#include "sfb_fft.cuh"
#include "sfb_fft_dev.cuh"
#include "sfb_kernels.cuh"

#include <cstdlib>

// minimum resident CTAs of the row kernels.  fp64: 2 CTAs of 192 threads.
// At 3 CTAs x 6 warps one SM sub-partition holds 5 warps, so ptxas caps the
// row kernels at 96 registers and spills (the C2R's 104-byte stack); at 2 CTAs
// they get 168 (840^3 step, 4 launches each: R2C+div 20.7 -> 19.0 ms, C2R
// 9.4 -> 7.7 ms).  fp32 fits 96 registers without spills: 3 CTAs.
#ifndef SFB_R2CDIV_MINB
#define SFB_R2CDIV_MINB 2
#endif
#ifndef SFB_ROW_MINB
#define SFB_ROW_MINB 2
#endif
#ifndef SFB_ROW_MINB_F32
#define SFB_ROW_MINB_F32 3
#endif
#define SFB_ROW_MINB_T(T, M) (sizeof(T) == 8 ? (M) : SFB_ROW_MINB_F32)

namespace sfb {

// W_N^j = exp(-2 pi i j / N) for sub-DFT sizes N <= kTwN (index N*kTwN + j).
// Internal linkage: every translation unit that instantiates kernels owns a
// copy and uploads it through its reg_tu_*_init() (fft_reg.cu calls them all).
constexpr int kTwN = 42;  // largest sub-DFT (1680 = 40 x 42)
static __constant__ double2 c_twd[(kTwN + 1) * kTwN];
static __constant__ float2 c_twf[(kTwN + 1) * kTwN];

template <typename C>
__device__ __forceinline__ C ctw(int N, int j);
template <>
__device__ __forceinline__ double2 ctw<double2>(int N, int j) { return c_twd[N * kTwN + j]; }
template <>
__device__ __forceinline__ float2 ctw<float2>(int N, int j) { return c_twf[N * kTwN + j]; }

__host__ __device__ constexpr bool rdft_base(int N) { return N == 2 || N == 3 || N == 4 || N == 5 || N == 7 || N == 8; }

// factor p of a composite N (base radix closest to sqrt(N), N/p > 1)
__host__ __device__ constexpr int rdft_pick(int N) {
  int best = 0, bd = 1 << 30;
  const int cand[6] = {8, 7, 5, 4, 3, 2};
  for (int i = 0; i < 6; ++i) {
    const int p = cand[i];
    if (N % p == 0 && N / p > 1) {
      const int q = N / p;
      const int d = p > q ? p - q : q - p;
      if (d < bd) {
        bd = d;
        best = p;
      }
    }
  }
  return best;
}

// x * W_N^j (forward) or x * conj(W_N^j) (INV); j a compile-time constant
// after unrolling; multiples of N/4 are done exactly.
template <typename C, int N, bool INV>
__device__ __forceinline__ C twmul_c(C x, int j) {
  j %= N;
  if (j == 0) return x;
  if ((4 * j) % N == 0) {
    const int q = 4 * j / N;  // W^(q N/4) = (-i)^q
    if (q == 2) {
      x.x = -x.x;
      x.y = -x.y;
      return x;
    }
    const bool mi = (q == 1) != INV;  // multiply by -i ?
    C r;
    if (mi) {
      r.x = x.y;
      r.y = -x.x;
    } else {
      r.x = -x.y;
      r.y = x.x;
    }
    return r;
  }
  C w = ctw<C>(N, j);
  if (INV) w.y = -w.y;
  return cmul(x, w);
}

// In-register DFT of N points (natural order in, natural order out).
template <typename C, int N, bool INV>
__device__ __forceinline__ void rdft(C* v) {
  static_assert(N <= kTwN, "rdft: sub-DFT larger than the twiddle table");
#ifdef SFB_REG_NOCOMPUTE
  if (true) return;
#endif
  if constexpr (N == 1) {
  } else if constexpr (rdft_base(N)) {
    dft<C, N, INV>(v);
  } else {
    constexpr int p = rdft_pick(N), q = N / p;
    static_assert(p > 1 && p * q == N, "rdft: unsupported length");
    C t[N];
#pragma unroll
    for (int n2 = 0; n2 < q; ++n2) {
      C a[p];
#pragma unroll
      for (int n1 = 0; n1 < p; ++n1) a[n1] = v[q * n1 + n2];
      rdft<C, p, INV>(a);
#pragma unroll
      for (int k1 = 0; k1 < p; ++k1) t[n2 * p + k1] = twmul_c<C, N, INV>(a[k1], n2 * k1);
    }
#pragma unroll
    for (int k1 = 0; k1 < p; ++k1) {
      C b[q];
#pragma unroll
      for (int n2 = 0; n2 < q; ++n2) b[n2] = t[n2 * p + k1];
      rdft<C, q, INV>(b);
#pragma unroll
      for (int k2 = 0; k2 < q; ++k2) v[k1 + p * k2] = b[k2];
    }
  }
}

// compile-time tile geometry of an (A, B) engine for element type C
template <typename C, int A, int B>
struct RegGeo {
  static constexpr int L = A * B;
  static constexpr int TT = A > B ? A : B;  // threads per transform
  // strided passes: W contiguous columns per CTA (SFB_REG_SEG-byte segments)
#ifndef SFB_REG_SEG
#define SFB_REG_SEG 64
#endif
#ifndef SFB_REG_MINB
#define SFB_REG_MINB 3
#endif
  static constexpr int E = (int)(128 / sizeof(C));  // elements per 128-byte wavefront
#ifndef SFB_REG_SEG_F32
#define SFB_REG_SEG_F32 SFB_REG_SEG
#endif
#ifndef SFB_REG_MINB_F32
#define SFB_REG_MINB_F32 SFB_REG_MINB
#endif
#ifndef SFB_REG_MINB2
#define SFB_REG_MINB2 SFB_REG_MINB
#endif
#ifndef SFB_REG_MINB2_F32
#define SFB_REG_MINB2_F32 2
#endif
  static constexpr int SEG = sizeof(C) == 16 ? SFB_REG_SEG : SFB_REG_SEG_F32;
  static constexpr int MB = sizeof(C) == 16 ? SFB_REG_MINB : SFB_REG_MINB_F32;
  static constexpr int W0 = (int)(SEG / sizeof(C));
  static constexpr int W = (size_t)L * W0 * sizeof(C) <= 112 * 1024 ? W0 : W0 / 2;
  static constexpr int XS = A * W + (W < E ? ((W - (A * W) % E) % E + E) % E : 0);
  static constexpr int NT_S = W * TT;
  static constexpr size_t SMEM_S = ((size_t)B * XS + 32 + (L + 31) / 32) * sizeof(C);
  static constexpr int MINB_S = SMEM_S * MB <= 220 * 1024 ? MB : 1;
  // the fused fwd-scale-inverse axis-0 pass (MODE 2) holds two transforms'
  // state; in fp32 it spills at 3 CTAs (80 registers at 8 warps per CTA)
  static constexpr int MB2 = sizeof(C) == 16 ? SFB_REG_MINB2 : SFB_REG_MINB2_F32;
  // MODE 2 also stages the axis-0 eigenvalues (L doubles) in shared memory
  static constexpr size_t SMEM_S2 = SMEM_S + (size_t)L * sizeof(double);
  static constexpr int MINB_S2 = SMEM_S2 * MB2 <= 220 * 1024 ? MB2 : 1;
  // row passes: RP rows per CTA; exchange rows padded to an odd stride
  static constexpr int AP = (A % 2 == 0) ? A + 1 : A;
  static constexpr int ROWBUF = (B * AP > L + 1 ? B * AP : L + 1);
#ifndef SFB_ROW_NT
#define SFB_ROW_NT 192
#endif
  static constexpr int RP = (SFB_ROW_NT / TT) > 0 ? SFB_ROW_NT / TT : 1;
  static constexpr int NT_R = RP * TT;
  static constexpr size_t SMEM_R = (size_t)RP * ROWBUF * sizeof(C);
};

template <typename C>
__device__ __forceinline__ C czero() {
  C z;
  z.x = 0;
  z.y = 0;
  return z;
}

// Two-level twiddle W_L^m = hi[m >> 5] * lo[m & 31] from shared memory (m < L):
// 1 KB instead of an L-entry table, so the tile keeps the SM's smem.
template <typename C>
__device__ __forceinline__ void tw_fill(C* lo, C* hi, const C* __restrict__ twL, int L) {
  const int nhi = (L + 31) / 32;
  for (int j = threadIdx.x; j < 32 + nhi; j += blockDim.x) {
    if (j < 32) lo[j] = __ldg(twL + (j < L ? j : 0));
    else hi[j - 32] = __ldg(twL + 32 * (j - 32));
  }
}
template <typename C, bool INV>
__device__ __forceinline__ C tw_mul(C x, const C* lo, const C* hi, int m) {
  C w = cmul(hi[m >> 5], lo[m & 31]);
  if (INV) w.y = -w.y;
  return cmul(x, w);
}

// ---------------------------------------------------------------------------
// strided C2C pass over columns: element (m, col) at data + b*bstride + m*S + col
// MODE 0 forward, 1 inverse, 2 forward -> 1/(Lambda N) -> inverse (axis 0)
// Exchange layout: slot (n2, k1, w) at n2*XS + k1*W + w, XS padded so the
// rows of one 128-byte shared-memory wavefront fall in distinct banks.
// ---------------------------------------------------------------------------
// MODE 3 / 4: forward / inverse out of place, with the transform rows of the
// output (3) or input (4) placed by a chunked map (slab all-to-all layout,
// distributed.py): row r at (r / mp.c) * mp.sq + (r % mp.c) * mp.s
struct RowSplit {
  int c;
  long long sq, s;
};

template <typename T, int A, int B, int MODE>
__global__ void __launch_bounds__(RegGeo<typename CX<T>::t, A, B>::NT_S,
                                  MODE == 2 ? RegGeo<typename CX<T>::t, A, B>::MINB_S2 : RegGeo<typename CX<T>::t, A, B>::MINB_S)
    k_rfft_strided(const typename CX<T>::t* __restrict__ in, typename CX<T>::t* __restrict__ data, long long S,
                   int ncol, long long bin, long long bstride, RowSplit mp, const typename CX<T>::t* __restrict__ twL,
                   ScaleArgs sc, int swap, long long S_in, long long cbs_in, long long cbs_out) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  constexpr int W = RG::W, XS = RG::XS;
  constexpr bool MAP_OUT = MODE == 3, MAP_IN = MODE == 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* buf = reinterpret_cast<C*>(smem_raw);
  C* twlo = buf + B * XS;
  C* twhi = twlo + 32;
  const int w = threadIdx.x % W, t = threadIdx.x / W;
  // grid: (column blocks, batches), or swapped when the batches exceed grid.y
  const int cblk = swap ? blockIdx.y : blockIdx.x, bat = swap ? blockIdx.x : blockIdx.y;
  const int col = cblk * W + w;
  const bool ok = col < ncol;
  // column block cblk at cblk * cbs (natural layout: cbs = W, i.e. column
  // col; tiled spectrum: the block stride); input rows S_in apart, output S
  C* base = data + (long long)bat * bstride + (ok ? cblk * cbs_out + w : 0);
  const C* ibase = in + (long long)bat * bin + (ok ? cblk * cbs_in + w : 0);
  constexpr bool INV1 = MODE == 1 || MODE == 4;
  const long long gs = (long long)B * S;
  auto mapped = [&](int r) -> long long { return (long long)(r / mp.c) * mp.sq + (long long)(r % mp.c) * mp.s; };
  C v[A > B ? A : B];
  // phase 1: thread n2 = t loads its column straight into registers
  if (t < B) {
    if constexpr (MAP_IN) {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) v[n1] = ok ? __ldcs(ibase + mapped(B * n1 + t)) : czero<C>();
    } else {
      const C* g = ibase + (long long)t * S_in;
      const long long gsi = (long long)B * S_in;
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) v[n1] = ok ? __ldcs(g + n1 * gsi) : czero<C>();
    }
  }
  tw_fill(twlo, twhi, twL, A * B);
  // MODE 2: the axis-0 eigenvalues in shared memory (kept out of registers:
  // a per-thread preload of B of them spilled the fused pass)
  double* l0s = reinterpret_cast<double*>(twhi + (A * B + 31) / 32);
  if constexpr (MODE == 2) {
    for (int i = threadIdx.x; i < A * B; i += blockDim.x) l0s[i] = __ldg(sc.l0 + i);
  }
  __syncthreads();
  if (t < B) {
    const int n2 = t;
    rdft<C, A, INV1>(v);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      C x = v[k1];
      if (k1 > 0) x = tw_mul<C, INV1>(x, twlo, twhi, n2 * k1);
      buf[n2 * XS + k1 * W + w] = x;
    }
  }
  __syncthreads();
  if (t < A) {
    const int k1 = t;
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) v[n2] = buf[n2 * XS + k1 * W + w];
    rdft<C, B, INV1>(v);
    if constexpr (MODE == 2) {
      // eigenvalue scaling (poisson.py:179-199): lam in fp64, cast to T
      double lc = 0.0, l2v = 0.0;
      if (sc.dim == 3) {
        int c1, c2;
        if (sc.tlog > 0) {  // tiled spectrum: batch = k2 block; padding columns clamp (never read back)
          c1 = col >> sc.tlog;
          c2 = min((bat << sc.tlog) + (col & ((1 << sc.tlog) - 1)), sc.nh - 1);
        } else {
          c1 = col / sc.nh;
          c2 = col - c1 * sc.nh;
        }
        lc = ok ? sc.l1[c1] : 0.0;
        l2v = ok ? sc.l2[c2] : 0.0;
      } else {
        lc = ok ? sc.l1[col] : 0.0;
      }
      const bool zmode = col == 0 && bat == 0 && sc.zero_ok;
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) {
        const int m = k1 + A * k2;
        const double l0 = l0s[m];
        const double lam = sc.dim == 3 ? (l0 + lc) + l2v : l0 + lc;
        if (m == 0 && zmode) {
          v[k2] = czero<C>();
        } else {
          const T f = spec_rcp<T>(lam) * (T)sc.invN;
          v[k2].x *= f;
          v[k2].y *= f;
        }
      }
      // inverse: B-point inverse DFT over k2 in registers, conj twiddle,
      // back into the same smem slots this thread read
      rdft<C, B, true>(v);
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) {
        C x = v[n2];
        if (k1 > 0) x = tw_mul<C, true>(x, twlo, twhi, n2 * k1);
        buf[n2 * XS + k1 * W + w] = x;
      }
    } else if (ok) {
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2)
        __stcs(base + (MAP_OUT ? mapped(k1 + A * k2) : (long long)(k1 + A * k2) * S), v[k2]);
    }
  }
  if constexpr (MODE == 2) {
    __syncthreads();
    if (t < B) {
      const int n2 = t;
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) v[k1] = buf[n2 * XS + k1 * W + w];
      rdft<C, A, true>(v);
      if (ok) {
        C* g = base + (long long)n2 * S;
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) __stcs(g + n1 * gs, v[n1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// contiguous-axis real transforms, M = A*B complex points per row (N = 2M reals)
// ---------------------------------------------------------------------------
// loads per thread of the tiled C2R staging: blocks of tw >= 4 columns, RP
// rows per CTA, NT_R = RP * TT threads walking TT / tw blocks at a time
// (tw <= TT; fft.cu falls back to the natural layout otherwise)
template <int M, int TT>
constexpr int kTileIt = ((M + 4) / 4 + TT / 4 - 1) / (TT / 4) > ((M + 8) / 8 + TT / 8 - 1) / (TT / 8 > 0 ? TT / 8 : 1)
                            ? ((M + 4) / 4 + TT / 4 - 1) / (TT / 4)
                            : ((M + 8) / 8 + TT / 8 - 1) / (TT / 8 > 0 ? TT / 8 : 1);

// Tiled half spectrum (single-GPU spectral solve, fft.cu): element (row, k) of
// the natural (rows, M+1) layout sits at (k >> tlog) * ks + row * 2^tlog +
// (k & (2^tlog - 1)) -- blocks of 2^tlog columns, each block a contiguous
// (rows, 2^tlog) array.  The strided passes then read contiguous 2^tlog-wide
// column blocks (axis 1: one whole block per CTA; axis 0: rows of the block
// 64 bytes x n1 apart instead of a 64-byte segment per plane, 5.7 MB apart).
// tlog <= 0: natural layout.
//
// R2C epilogue: X[k] = E[k] + w^k O[k], E = (Z[k] + conj Z[M-k]) / 2,
// O = (Z[k] - conj Z[M-k]) / (2i), from the CTA's rows in shared memory (row
// r at r * ROWBUF).  Tiled stores run over (block, row, w) with w fastest, so
// a warp writes the CTA's consecutive rows of one block contiguously.
template <typename T, int A, int B>
__device__ __forceinline__ void r2c_epilogue(const typename CX<T>::t* __restrict__ sbuf, typename CX<T>::t* __restrict__ out,
                                             long long row0, long long rows, long long out_row,
                                             const typename CX<T>::t* __restrict__ twN, int tlog, long long ks) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  constexpr int M = A * B, TT = RG::TT;
  auto val = [&](const C* buf, int k) -> C {
    const C zk = buf[k == M ? 0 : k];
    const C zc = buf[k == 0 ? 0 : M - k];
    C e, od;
    e.x = T(0.5) * (zk.x + zc.x);
    e.y = T(0.5) * (zk.y - zc.y);
    od.x = T(0.5) * (zk.y + zc.y);
    od.y = -T(0.5) * (zk.x - zc.x);
    const C w = __ldg(twN + k);
    return cadd(e, cmul(w, od));
  };
  if (tlog > 0) {
    // a thread owns one (row, w) slot of every block it walks (see k_rfft_c2r)
    const int tw = 1 << tlog, nslot = RG::RP << tlog, ng = RG::NT_R / nslot, nblk = (M + tw) >> tlog;
    const int slot = threadIdx.x % nslot, g = threadIdx.x / nslot;
    const int r = slot >> tlog, w = slot & (tw - 1);
    const long long row = row0 + r;
    if (g >= ng || row >= rows) return;
    C* dst = out + row * tw + w;
    const C* sb = sbuf + r * RG::ROWBUF;
    for (int K = g; K < nblk; K += ng) {
      const int k = (K << tlog) + w;
      if (k <= M) __stcs(dst + K * ks, val(sb, k));
    }
    return;
  }
  const int r = threadIdx.x / TT, t = threadIdx.x % TT;
  const long long row = row0 + r;
  if (row >= rows) return;
  C* o = out + row * out_row;
  for (int k = t; k <= M; k += TT) __stcs(o + k, val(sbuf + r * RG::ROWBUF, k));
}

template <typename T, int A, int B>
__global__ void __launch_bounds__(RegGeo<typename CX<T>::t, A, B>::NT_R, SFB_ROW_MINB_T(T, SFB_ROW_MINB))
    k_rfft_r2c(const T* __restrict__ in, typename CX<T>::t* __restrict__ out, long long rows, long long in_row,
               long long out_row, const typename CX<T>::t* __restrict__ twM, const typename CX<T>::t* __restrict__ twN,
               int tlog, long long ks) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  constexpr int M = A * B, TT = RG::TT, AP = RG::AP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int r = threadIdx.x / TT, t = threadIdx.x % TT;
  const long long row = (long long)blockIdx.x * RG::RP + r;
  const bool okr = row < rows;
  C* buf = reinterpret_cast<C*>(smem_raw) + r * RG::ROWBUF;
  if (t < B) {
    const int n2 = t;
    const C* x = reinterpret_cast<const C*>(in + (okr ? row : 0) * in_row);
    C v[A];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) v[n1] = okr ? __ldcs(x + B * n1 + n2) : czero<C>();
    rdft<C, A, false>(v);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      C y = v[k1];
      if (k1 > 0) y = cmul(y, __ldg(twM + n2 * k1));
      buf[n2 * AP + k1] = y;
    }
  }
  __syncthreads();
  C v[B];
  if (t < A) {
    const int k1 = t;
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) v[n2] = buf[n2 * AP + k1];
    rdft<C, B, false>(v);
  }
  __syncthreads();
  if (t < A) {
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) buf[t + A * k2] = v[k2];
  }
  __syncthreads();
  r2c_epilogue<T, A, B>(reinterpret_cast<const C*>(smem_raw), out, (long long)blockIdx.x * RG::RP, rows, out_row, twN,
                        tlog, ks);
}

// R2C of the projection right-hand side computed on the fly: the real input
// at interior cell (i, j, k) is the divergence of the velocity
// (operators.py:108-122, same operation order as k_div_int), read from the
// extended velocity arrays; the divergence field never touches HBM.
// Axes 1 and 2 periodic, axis 0 periodic or a halo axis (slab).
// WALL1 (channel: walls on axis 1): the two axis-1 faces of a wall-adjacent
// row are resolved inline like k_div_int / k_div_march (the wall face carries
// the Dirichlet value, zero for a symmetric wall): w1lo -> u_1 below = v1lo,
// w1hi -> u_1 at the cell's upper face = v1hi
template <typename T, bool WALL1 = false>
__device__ __forceinline__ T div_at(const Geo<T>& G, const T* __restrict__ u0, const T* __restrict__ u1,
                                    const T* __restrict__ u2, long long x, long long o0m, long long o1m, T r0, T r1,
                                    int kk, bool w1lo = false, bool w1hi = false, T v1lo = T(0), T v1hi = T(0)) {
  const long long xk = x + kk;
  const long long o2m = kk == 1 ? (long long)(G.n[2] - 1) : -1;
  T acc = (__ldg(u0 + xk) - __ldg(u0 + xk + o0m)) * r0;
  if constexpr (WALL1) {
    const T c1 = w1hi ? v1hi : __ldg(u1 + xk);
    const T p1 = w1lo ? v1lo : __ldg(u1 + xk + o1m);
    acc += (c1 - p1) * r1;
  } else {
    acc += (__ldg(u1 + xk) - __ldg(u1 + xk + o1m)) * r1;
  }
  acc += (__ldg(u2 + xk) - __ldg(u2 + xk + o2m)) * tab(G, 2, T_RDX, kk);
  return acc;
}

// GT: the input of the projection pullback's solve instead of a divergence,
// -G^T(v) / W at the pressure point (adjoint.cu k_grad_pb with sign -1 and
// the 1/W weight, periodic axes), same operation order
template <typename T>
__device__ __forceinline__ T gradT_at(const Geo<T>& G, const T* __restrict__ v0, const T* __restrict__ v1,
                                      const T* __restrict__ v2, long long x, long long o0m, long long o1m, T q0m, T q0,
                                      T q1m, T q1, T rw01, int kk) {
  const long long xk = x + kk;
  const long long o2m = kk == 1 ? (long long)(G.n[2] - 1) : -1;
  const int km = kk == 1 ? G.n[2] : kk - 1;
  T acc = T(0);
  acc += __ldg(v0 + xk + o0m) * q0m - __ldg(v0 + xk) * q0;
  acc += __ldg(v1 + xk + o1m) * q1m - __ldg(v1 + xk) * q1;
  acc += __ldg(v2 + xk + o2m) * tab(G, 2, T_RDU, km) - __ldg(v2 + xk) * tab(G, 2, T_RDU, kk);
  acc = T(-1) * acc;
  return acc * (rw01 * tab(G, 2, T_RDX, kk));
}

template <typename T, int A, int B, bool WALL1 = false, bool GT = false>
__global__ void __launch_bounds__(RegGeo<typename CX<T>::t, A, B>::NT_R, SFB_ROW_MINB_T(T, SFB_R2CDIV_MINB))
    k_rfft_r2c_div(Geo<T> G, CV<T> U, typename CX<T>::t* __restrict__ out, long long rows, long long out_row,
                   const typename CX<T>::t* __restrict__ twM, const typename CX<T>::t* __restrict__ twN, int tlog,
                   long long ks) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  constexpr int M = A * B, TT = RG::TT, AP = RG::AP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int r = threadIdx.x / TT, t = threadIdx.x % TT;
  const long long row = (long long)blockIdx.x * RG::RP + r;
  const bool okr = row < rows;
  C* buf = reinterpret_cast<C*>(smem_raw) + r * RG::ROWBUF;
  if (t < B) {
    const int n2 = t;
    C v[A];
    if (okr) {
      const int i = 1 + (int)(row / G.n[1]), j = 1 + (int)(row % G.n[1]);
      const long long x = (long long)i * G.s[0] + (long long)j * G.s[1];
      const long long o0m = (i == 1 && !G.halo[0]) ? (long long)(G.n[0] - 1) * G.s[0] : -G.s[0];
      const long long o1m = (!WALL1 && j == 1) ? (long long)(G.n[1] - 1) * G.s[1] : -G.s[1];
      const T r0 = tab(G, 0, T_RDX, i), r1 = tab(G, 1, T_RDX, j);
      const bool w1lo = WALL1 && j == 1, w1hi = WALL1 && j == G.n[1];
      const T v1lo = (WALL1 && G.bc_lo[1] == SFB_BC_DIRICHLET) ? G.vlo[1][1] : T(0);
      const T v1hi = (WALL1 && G.bc_hi[1] == SFB_BC_DIRICHLET) ? G.vhi[1][1] : T(0);
      if constexpr (GT) {
        const int im = i == 1 ? G.n[0] : i - 1, jm = j == 1 ? G.n[1] : j - 1;
        const T q0m = tab(G, 0, T_RDU, im), q0 = tab(G, 0, T_RDU, i);
        const T q1m = tab(G, 1, T_RDU, jm), q1 = tab(G, 1, T_RDU, j);
        const T rw01 = (T(1) * r0) * r1;
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int m = B * n1 + n2;
          v[n1].x = gradT_at(G, U.c[0], U.c[1], U.c[2], x, o0m, o1m, q0m, q0, q1m, q1, rw01, 2 * m + 1);
          v[n1].y = gradT_at(G, U.c[0], U.c[1], U.c[2], x, o0m, o1m, q0m, q0, q1m, q1, rw01, 2 * m + 2);
        }
      } else {
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
          const int m = B * n1 + n2;
          v[n1].x = div_at<T, WALL1>(G, U.c[0], U.c[1], U.c[2], x, o0m, o1m, r0, r1, 2 * m + 1, w1lo, w1hi, v1lo, v1hi);
          v[n1].y = div_at<T, WALL1>(G, U.c[0], U.c[1], U.c[2], x, o0m, o1m, r0, r1, 2 * m + 2, w1lo, w1hi, v1lo, v1hi);
        }
      }
    } else {
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) v[n1] = czero<C>();
    }
    rdft<C, A, false>(v);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      C y = v[k1];
      if (k1 > 0) y = cmul(y, __ldg(twM + n2 * k1));
      buf[n2 * AP + k1] = y;
    }
  }
  __syncthreads();
  C v[B];
  if (t < A) {
    const int k1 = t;
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) v[n2] = buf[n2 * AP + k1];
    rdft<C, B, false>(v);
  }
  __syncthreads();
  if (t < A) {
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) buf[t + A * k2] = v[k2];
  }
  __syncthreads();
  r2c_epilogue<T, A, B>(reinterpret_cast<const C*>(smem_raw), out, (long long)blockIdx.x * RG::RP, rows, out_row, twN,
                        tlog, ks);
}

template <typename T, int A, int B>
__global__ void __launch_bounds__(RegGeo<typename CX<T>::t, A, B>::NT_R, SFB_ROW_MINB_T(T, SFB_ROW_MINB))
    k_rfft_c2r(const typename CX<T>::t* __restrict__ in, T* __restrict__ out, long long rows, long long in_row,
               long long out_row, const typename CX<T>::t* __restrict__ twM, const typename CX<T>::t* __restrict__ twN,
               int tlog, long long ks) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  constexpr int M = A * B, TT = RG::TT, AP = RG::AP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int r = threadIdx.x / TT, t = threadIdx.x % TT;
  const long long row = (long long)blockIdx.x * RG::RP + r;
  const bool okr = row < rows;
  C* buf = reinterpret_cast<C*>(smem_raw) + r * RG::ROWBUF;
  const C* X = in + (okr ? row : 0) * in_row;
  if (tlog > 0) {
    // tiled spectrum (see r2c_epilogue): stage the CTA's rows through shared
    // memory, each block's rows read contiguously
    // a thread owns one (row, w) slot of every block it walks (the CTA's
    // rows of one block are contiguous): no per-element index division, and
    // all of its loads are issued before the first shared store
    const int tw = 1 << tlog, nslot = RG::RP << tlog, ng = RG::NT_R / nslot, nblk = (M + tw) >> tlog;
    const int slot = threadIdx.x % nslot, g = threadIdx.x / nslot;
    const int rr = slot >> tlog, w = slot & (tw - 1);
    const long long rowt = (long long)blockIdx.x * RG::RP + rr;
    const bool okt = g < ng && rowt < rows;
    const C* src = in + rowt * tw + w;
    C* sb = reinterpret_cast<C*>(smem_raw) + rr * RG::ROWBUF + w;
    C tmp[kTileIt<M, TT>];
#pragma unroll
    for (int q = 0; q < kTileIt<M, TT>; ++q) {
      const int K = g + q * ng, k = (K << tlog) + w;
      tmp[q] = okt && K < nblk && k <= M ? __ldcs(src + K * ks) : czero<C>();
    }
#pragma unroll
    for (int q = 0; q < kTileIt<M, TT>; ++q) {
      const int K = g + q * ng;
      if (okt && K < nblk && (K << tlog) + w <= M) sb[K << tlog] = tmp[q];
    }
    __syncthreads();
    X = buf;
  }
  C v[A];
  if (t < B) {
    const int n2 = t;
    // Z[k] = (X[k] + conj X[M-k]) + i (X[k] - conj X[M-k]) exp(+2 pi i k / N)
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) {
      const int k = B * n1 + n2;
      C z = czero<C>();
      if (okr) {
        const C xk = X[k];
        const C xc = X[M - k];
        C fe, d, w;
        fe.x = xk.x + xc.x;
        fe.y = xk.y - xc.y;
        d.x = xk.x - xc.x;
        d.y = xk.y + xc.y;
        w = __ldg(twN + k);
        w.y = -w.y;
        const C fo = cmul(d, w);
        z.x = fe.x - fo.y;
        z.y = fe.y + fo.x;
      }
      v[n1] = z;
    }
  }
  if (tlog > 0) __syncthreads();  // every staged row read before the exchange overwrites it
  if (t < B) {
    const int n2 = t;
    rdft<C, A, true>(v);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      C y = v[k1];
      if (k1 > 0) {
        C tw = __ldg(twM + n2 * k1);
        tw.y = -tw.y;
        y = cmul(y, tw);
      }
      buf[n2 * AP + k1] = y;
    }
  }
  __syncthreads();
  if (t < A && okr) {
    const int k1 = t;
    C v[B];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) v[n2] = buf[n2 * AP + k1];
    rdft<C, B, true>(v);
    C* o = reinterpret_cast<C*>(out + row * out_row);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) __stcs(o + k1 + A * k2, v[k2]);
  }
}

// ---- host side ----
struct RegLen {
  int L = 0, A = 0, B = 0;
  bool ok = false;
};
// one launch request: kind 0/1/2 strided MODE, 3 R2C, 4 C2R, 5 R2C of the divergence,
// 6 / 7 strided forward / inverse out of place with the output / input rows
// split into chunks (map_c rows per chunk, chunk stride map_sq, row stride map_s)
struct RegCall {
  int kind;
  const void* in;
  void* out;  // strided: in == out (in place)
  long long S, bstride, rows, in_row, out_row;
  long long bstride_in, map_sq, map_s;
  int map_c;
  int ncol, nbatch;
  const void* twL;  // plain table exp(-2 pi i m / L), m < L
  const void* twN;  // real trick: exp(-2 pi i k / 2L), k <= L
  ScaleArgs sc;
  long long S_in, cbs_in, cbs_out;  // strided kinds: input row stride, column-block strides (0 = natural)
  const void* geo;     // kind 5: host Geo<T> of the velocity plan
  const void* u[3];    // kind 5: extended velocity components
  int tlog;            // kinds 3-5: tiled spectrum (r2c_epilogue), 0 = natural
  int wall1;           // kind 5: walls on axis 1 (channel), resolved inline
  int gradt;           // kind 5: -G^T(v)/W (projection pullback) instead of div(v)
  long long ks;        //   its block stride
};

static int reg_upload_tables() {
  static double2 hd[(kTwN + 1) * kTwN];
  static float2 hf[(kTwN + 1) * kTwN];
  for (int N = 1; N <= kTwN; ++N)
    for (int j = 0; j < kTwN; ++j) {
      const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)(j % N) / (long double)N;
      hd[N * kTwN + j] = make_double2((double)cosl(a), (double)sinl(a));
      hf[N * kTwN + j] = make_float2((float)cosl(a), (float)sinl(a));
    }
  if (cudaMemcpyToSymbol(c_twd, hd, sizeof(hd)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_twf, hf, sizeof(hf)) != cudaSuccess) return -1;
  return 0;
}

template <typename T, int A, int B>
static int reg_launch(const RegCall& c, cudaStream_t st) {
  typedef typename CX<T>::t C;
  typedef RegGeo<C, A, B> RG;
  {
    cudaError_t e = cudaSuccess;
#define SFB_ATTR(K, B) \
  if (e == cudaSuccess) e = ensure_smem((const void*)K, (B))
    SFB_ATTR((k_rfft_strided<T, A, B, 0>), RG::SMEM_S);
    SFB_ATTR((k_rfft_strided<T, A, B, 1>), RG::SMEM_S);
    SFB_ATTR((k_rfft_strided<T, A, B, 2>), RG::SMEM_S2);
    SFB_ATTR((k_rfft_strided<T, A, B, 3>), RG::SMEM_S);
    SFB_ATTR((k_rfft_strided<T, A, B, 4>), RG::SMEM_S);
    SFB_ATTR((k_rfft_r2c<T, A, B>), RG::SMEM_R);
    SFB_ATTR((k_rfft_c2r<T, A, B>), RG::SMEM_R);
    SFB_ATTR((k_rfft_r2c_div<T, A, B>), RG::SMEM_R);
    SFB_ATTR((k_rfft_r2c_div<T, A, B, true>), RG::SMEM_R);
    SFB_ATTR((k_rfft_r2c_div<T, A, B, false, true>), RG::SMEM_R);
#undef SFB_ATTR
    if (e != cudaSuccess) return -2;
  }
  if (c.kind <= 2 || c.kind == 6 || c.kind == 7) {
    const unsigned nblk = (unsigned)((c.ncol + RG::W - 1) / RG::W);
    const int swap = c.nbatch > 65535;  // grid.y limit: batches on x
    const dim3 grid = swap ? dim3(c.nbatch, nblk) : dim3(nblk, c.nbatch);
    C* d = (C*)c.out;
    const C* src = c.in ? (const C*)c.in : d;
    const long long bin = c.in ? c.bstride_in : c.bstride;
    const RowSplit mp{c.map_c > 0 ? c.map_c : 1, c.map_sq, c.map_s};
    const long long sin = c.S_in ? c.S_in : c.S, cbi = c.cbs_in ? c.cbs_in : RG::W, cbo = c.cbs_out ? c.cbs_out : RG::W;
    const C* tw = (const C*)c.twL;
#define SFB_STRIDED(M)                                                                                     \
  k_rfft_strided<T, A, B, M><<<grid, RG::NT_S, M == 2 ? RG::SMEM_S2 : RG::SMEM_S, st>>>(src, d, c.S, c.ncol, bin, c.bstride, mp, tw, \
                                                                 c.sc, swap, sin, cbi, cbo)
    switch (c.kind) {
      case 0: SFB_STRIDED(0); break;
      case 1: SFB_STRIDED(1); break;
      case 2: SFB_STRIDED(2); break;
      case 6: SFB_STRIDED(3); break;
      default: SFB_STRIDED(4); break;
    }
#undef SFB_STRIDED
  } else {
    const unsigned nb = (unsigned)((c.rows + RG::RP - 1) / RG::RP);
    if (c.kind == 3)
      k_rfft_r2c<T, A, B><<<nb, RG::NT_R, RG::SMEM_R, st>>>((const T*)c.in, (C*)c.out, c.rows, c.in_row, c.out_row,
                                                          (const C*)c.twL, (const C*)c.twN, c.tlog, c.ks);
    else if (c.kind == 4)
      k_rfft_c2r<T, A, B><<<nb, RG::NT_R, RG::SMEM_R, st>>>((const C*)c.in, (T*)c.out, c.rows, c.in_row, c.out_row,
                                                          (const C*)c.twL, (const C*)c.twN, c.tlog, c.ks);
    else {
      CV<T> U;
      for (int a = 0; a < 3; ++a) U.c[a] = (const T*)c.u[a];
      if (c.gradt)
        k_rfft_r2c_div<T, A, B, false, true><<<nb, RG::NT_R, RG::SMEM_R, st>>>(
            *(const Geo<T>*)c.geo, U, (C*)c.out, c.rows, c.out_row, (const C*)c.twL, (const C*)c.twN, c.tlog, c.ks);
      else if (c.wall1)
        k_rfft_r2c_div<T, A, B, true><<<nb, RG::NT_R, RG::SMEM_R, st>>>(*(const Geo<T>*)c.geo, U, (C*)c.out, c.rows,
                                                                      c.out_row, (const C*)c.twL, (const C*)c.twN,
                                                                      c.tlog, c.ks);
      else
        k_rfft_r2c_div<T, A, B><<<nb, RG::NT_R, RG::SMEM_R, st>>>(*(const Geo<T>*)c.geo, U, (C*)c.out, c.rows,
                                                                c.out_row, (const C*)c.twL, (const C*)c.twN, c.tlog,
                                                                c.ks);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// dispatch (fft_reg.cu); the per-unit entry points return -1 when the length
// is not instantiated in that unit
bool reg_factor(int L, RegLen& R);
int fft_reg_init();
template <typename T>
int reg_run(const RegLen& R, const RegCall& c, cudaStream_t st);
int reg_tu_d1(int L, const RegCall& c, cudaStream_t st);
int reg_tu_d2(int L, const RegCall& c, cudaStream_t st);
int reg_tu_f1(int L, const RegCall& c, cudaStream_t st);
int reg_tu_f2(int L, const RegCall& c, cudaStream_t st);
int reg_tu_d1_init();
int reg_tu_d2_init();
int reg_tu_f1_init();
int reg_tu_f2_init();

}  // namespace sfb
