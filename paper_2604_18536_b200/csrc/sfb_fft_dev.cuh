// Device building blocks of the hand-written FFT engine (shared by fft.cu
// and fft_tma.cu): complex helpers, small DFTs, Stockham passes.
#pragma once

#include "sfb_fft.cuh"

namespace sfb {

template <typename T>
struct CX;
template <>
struct CX<double> {
  typedef double2 t;
};
template <>
struct CX<float> {
  typedef float2 t;
};

// cp.async (LDGSTS) of one complex element into shared memory; pred=false
// zero-fills.  All loads of a tile are issued back to back, then waited on.
template <typename C>
__device__ __forceinline__ void cp_async_elem(C* smem, const C* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? (int)sizeof(C) : 0;
  if constexpr (sizeof(C) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) {
  C r;
  r.x = a.x + b.x;
  r.y = a.y + b.y;
  return r;
}
template <typename C>
__device__ __forceinline__ C csub(C a, C b) {
  C r;
  r.x = a.x - b.x;
  r.y = a.y - b.y;
  return r;
}
// multiply by -i (forward) or +i (inverse)
template <typename C, bool INV>
__device__ __forceinline__ C mul_mi(C a) {
  C r;
  if (INV) {
    r.x = -a.y;
    r.y = a.x;
  } else {
    r.x = a.y;
    r.y = -a.x;
  }
  return r;
}

// ---------------------------------------------------------------------------
// small DFTs, forward sign exp(-2 pi i k m / R); INV uses the + sign
// ---------------------------------------------------------------------------
template <typename C, bool INV>
__device__ __forceinline__ void dft2(C* v) {
  C a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <typename C, bool INV>
__device__ __forceinline__ void dft4(C* v) {
  C s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  C s13 = cadd(v[1], v[3]), d13 = mul_mi<C, INV>(csub(v[1], v[3]));
  v[0] = cadd(s02, s13);
  v[2] = csub(s02, s13);
  v[1] = cadd(d02, d13);
  v[3] = csub(d02, d13);
}

template <typename C, bool INV>
__device__ __forceinline__ void dft8(C* v) {
  typedef decltype(v[0].x) R;
  const R h = (R)0.70710678118654752440084436210484903928;
  // radix-2 first stage over pairs (m, m+4)
  C a[4], b[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    a[m] = cadd(v[m], v[m + 4]);
    b[m] = csub(v[m], v[m + 4]);
  }
  // twiddle b[m] by w8^m (forward w8 = exp(-i pi/4))
  {
    C t = b[1];
    // w8^1 = h - i h (fwd), h + i h (inv)
    b[1].x = h * (t.x + (INV ? -t.y : t.y));
    b[1].y = h * (t.y + (INV ? t.x : -t.x));
    b[2] = mul_mi<C, INV>(b[2]);
    t = b[3];
    // w8^3 = -h - i h (fwd), -h + i h (inv)
    b[3].x = h * (-t.x + (INV ? -t.y : t.y));
    b[3].y = h * (-t.y + (INV ? t.x : -t.x));
  }
  dft4<C, INV>(a);
  dft4<C, INV>(b);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    v[2 * m] = a[m];
    v[2 * m + 1] = b[m];
  }
}

// odd radix R in {3, 5, 7}: pairwise-symmetric direct DFT.
// cos/sin(2 pi j / R) for j = 1..(R-1)/2 (the rest by symmetry)
__device__ __forceinline__ double odd_cos(int R, int j) {
  if (R == 3) return -0.5;
  if (R == 5) return j == 1 ? 0.30901699437494742410229341718281905886 : -0.80901699437494742410229341718281905886;
  return j == 1 ? 0.62348980185873353052500488400423981063
                : (j == 2 ? -0.22252093395631440428890256449679475947 : -0.90096886790241912623610231950744505117);
}
__device__ __forceinline__ double odd_sin(int R, int j) {
  if (R == 3) return 0.86602540378443864676372317075293618347;
  if (R == 5) return j == 1 ? 0.95105651629515357211643933337938214340 : 0.58778525229247312916870595463907276860;
  return j == 1 ? 0.78183148246802980870844452667405775023
                : (j == 2 ? 0.97492791218182360701813168299393121723 : 0.43388373911755812047576833284835875461);
}

template <typename C, int R, bool INV>
__device__ __forceinline__ void dft_odd(C* v) {
  typedef decltype(v[0].x) RT;
  constexpr int H = (R - 1) / 2;
  // cos/sin(2 pi j / R), j = 0..R-1 (compile-time after unrolling)
  RT cs[R], sn[R];
  cs[0] = (RT)1;
  sn[0] = (RT)0;
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    cs[j] = (RT)odd_cos(R, j);
    sn[j] = (RT)odd_sin(R, j);
    cs[R - j] = cs[j];
    sn[R - j] = -sn[j];
  }
  C sp[H], dm[H];
#pragma unroll
  for (int m = 1; m <= H; ++m) {
    sp[m - 1] = cadd(v[m], v[R - m]);
    dm[m - 1] = csub(v[m], v[R - m]);
  }
  C y0 = v[0];
#pragma unroll
  for (int m = 0; m < H; ++m) y0 = cadd(y0, sp[m]);
  C out[R];
  out[0] = y0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    C A = v[0], B;
    B.x = 0;
    B.y = 0;
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      const int j = (k * m) % R;
      A.x += sp[m - 1].x * cs[j];
      A.y += sp[m - 1].y * cs[j];
      B.x += dm[m - 1].x * sn[j];
      B.y += dm[m - 1].y * sn[j];
    }
    // forward: y_k = A - i B, y_{R-k} = A + i B
    C iB;
    iB.x = -B.y;
    iB.y = B.x;
    if (INV) {
      out[k] = cadd(A, iB);
      out[R - k] = csub(A, iB);
    } else {
      out[k] = csub(A, iB);
      out[R - k] = cadd(A, iB);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = out[k];
}

template <typename C, int R, bool INV>
__device__ __forceinline__ void dft(C* v) {
  if constexpr (R == 2) dft2<C, INV>(v);
  else if constexpr (R == 4) dft4<C, INV>(v);
  else if constexpr (R == 8) dft8<C, INV>(v);
  else dft_odd<C, R, INV>(v);
}

// j / Ns and j % Ns for j < 2^24 without an integer divide
__device__ __forceinline__ void divmod_ns(int j, int Ns, float inv, int& q, int& r) {
  q = __float2int_rz(__int2float_rn(j) * inv);
  r = j - q * Ns;
  if (r < 0) {
    --q;
    r += Ns;
  } else if (r >= Ns) {
    ++q;
    r -= Ns;
  }
}

// One Stockham pass over a tile stored [m][w] (m < L, w < W): src -> dst.
// Thread t owns column t % W and butterflies j = t / W + s * (NT / W).
// twp: this pass's twiddles laid out [k][r-1] (contiguous per butterfly).
template <typename C, int R, bool INV, int W, bool TWS = false>
__device__ __forceinline__ void stockham(const C* __restrict__ src, C* __restrict__ dst, int L, int Ns,
                                         const C* __restrict__ twp) {
  const int nb = L / R;
  const int col = threadIdx.x % W;
  const int jstride = blockDim.x / W;
  const int nbW = nb * W, NsW = Ns * W;
  const float inv = 1.0f / (float)Ns;
  const C* s0 = src + col;
  C* d0 = dst + col;
  for (int j = threadIdx.x / W; j < nb; j += jstride) {
    int g, k;
    divmod_ns(j, Ns, inv, g, k);
    const C* sp = s0 + j * W;
    C v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = sp[r * nbW];
    if (Ns > 1) {
      const C* tp = twp + k * (R - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        C w = TWS ? tp[r - 1] : __ldg(tp + (r - 1));
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    dft<C, R, INV>(v);
    C* dp = d0 + (g * Ns * R + k) * W;
#pragma unroll
    for (int r = 0; r < R; ++r) dp[r * NsW] = v[r];
  }
}

// Run all passes of a length-L plan; returns the buffer holding the result.
// tw: plain table exp(-2 pi i m / L) followed by the per-pass tables.
template <typename C, bool INV, int W, bool TWS = false>
__device__ __forceinline__ C* run_fft(C* a, C* b, const FftLen& P, const C* __restrict__ tw) {
  int Ns = 1;
  for (int p = 0; p < P.np; ++p) {
    __syncthreads();
    const C* twp = tw + P.twoff[p];
    switch (P.radix[p]) {
      case 8: stockham<C, 8, INV, W, TWS>(a, b, P.L, Ns, twp); break;
      case 4: stockham<C, 4, INV, W, TWS>(a, b, P.L, Ns, twp); break;
      case 2: stockham<C, 2, INV, W, TWS>(a, b, P.L, Ns, twp); break;
      case 7: stockham<C, 7, INV, W, TWS>(a, b, P.L, Ns, twp); break;
      case 5: stockham<C, 5, INV, W, TWS>(a, b, P.L, Ns, twp); break;
      default: stockham<C, 3, INV, W, TWS>(a, b, P.L, Ns, twp); break;
    }
    Ns *= P.radix[p];
    C* t = a;
    a = b;
    b = t;
  }
  __syncthreads();
  return a;
}


}  // namespace sfb
