// TMA-pipelined strided FFT passes (sm_100a).
//
// The smem Stockham passes of fft.cu are latency-bound: a CTA alternates
// between loading its tile, computing and storing it, and with two tiles per
// SM the HBM traffic stalls while both compute.  Here each CTA is persistent
// and owns three tile buffers: tile t+1 is brought in by TMA
// (cp.async.bulk.tensor, mbarrier completion) and the result of tile t-1
// drains to HBM by TMA bulk stores while all warps compute tile t.  The loads
// and stores cost the warps no instructions, out-of-range rows/columns are
// zero-filled / clipped by the tensor map.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sfb_fft.cuh"
#include "sfb_fft_dev.cuh"
#include "sfb_kernels.cuh"
#include "sfb_tma.cuh"

namespace sfb {

struct TmaTile {
  int rank;   // 3: (2W, rows, batch) map; 2: (2W, rows) map
  int nbox;   // boxes per tile along the FFT axis
  int lb;     // rows per box
  int ncol;   // complex columns
  int nbatch;
};

template <typename T, int MODE, int W, int NT>
__global__ void __launch_bounds__(NT, 1) k_fft_tma(const __grid_constant__ CUtensorMap tm, TmaTile tt, FftLen P,
                                                   const typename CX<T>::t* __restrict__ tw, ScaleArgs sc) {
  typedef typename CX<T>::t C;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int rows = tt.nbox * tt.lb;  // >= L
  const size_t bufc = (size_t)rows * W;
  C* buf[3] = {reinterpret_cast<C*>(smem_raw), reinterpret_cast<C*>(smem_raw) + bufc,
               reinterpret_cast<C*>(smem_raw) + 2 * bufc};
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw + 3 * bufc * sizeof(C));
  C* stw = reinterpret_cast<C*>(smem_raw + 3 * bufc * sizeof(C) + 64);  // twiddle tables staged once per CTA
  for (int e = threadIdx.x; e < P.twn; e += NT) stw[e] = tw[e];
  const unsigned tile_bytes = (unsigned)(bufc * sizeof(C));
  const int ntx = (tt.ncol + W - 1) / W;
  const int ntiles = ntx * tt.nbatch;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t, int b) {
    const int bx = t % ntx, by = t / ntx;
    mbar_arm(&bars[b], tile_bytes);
    for (int q = 0; q < tt.nbox; ++q)
      tma_load(&tm, tt.rank, buf[b] + (size_t)q * tt.lb * W, &bars[b], 2 * bx * W, q * tt.lb, by);
  };
  int cur = 0, tmp = 1, pre = 2;
  unsigned phase[3] = {0, 0, 0};
  int t = blockIdx.x;
  if (threadIdx.x == 0) {
    if (t < ntiles) issue(t, cur);
    if (t + (int)gridDim.x < ntiles) issue(t + gridDim.x, pre);
  }
  for (; t < ntiles; t += gridDim.x) {
    mbar_wait(&bars[cur], phase[cur]);
    phase[cur] ^= 1;
    C* res;
#ifdef SFB_TMA_NOCOMPUTE
    res = buf[cur];
#else
    if (MODE == 1) res = run_fft<C, true, W, true>(buf[cur], buf[tmp], P, stw);
    else res = run_fft<C, false, W, true>(buf[cur], buf[tmp], P, stw);
#endif
    const int bx = t % ntx, by = t / ntx;
    const int c0 = bx * W;
    if (MODE == 2) {
      const int w = threadIdx.x % W, m0 = threadIdx.x / W, ms = NT / W;
      const int col = c0 + w;
      if (col < tt.ncol) {
        double lc;
        int k2 = 0;
        if (sc.dim == 3) {
          const int k1 = col / sc.nh;
          k2 = col - k1 * sc.nh;
          lc = sc.l1[k1];
        } else {
          lc = sc.l1[col];
        }
        for (int m = m0; m < P.L; m += ms) {
          const double lam = sc.dim == 3 ? (sc.l0[m] + lc) + sc.l2[k2] : sc.l0[m] + lc;
          C v = res[m * W + w];
          if (m == 0 && col == 0 && by == 0 && sc.zero_ok) {
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
#ifndef SFB_TMA_NOCOMPUTE
      C* other = (res == buf[cur]) ? buf[tmp] : buf[cur];
      res = run_fft<C, true, W, true>(res, other, P, stw);
#endif
    }
    // results of this tile -> HBM by TMA; smem writes must be visible to the async proxy
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    const int rb = (res == buf[cur]) ? cur : tmp;
    const int ob = (rb == cur) ? tmp : cur;
    if (threadIdx.x == 0) {
      for (int q = 0; q < tt.nbox; ++q) tma_store(&tm, tt.rank, res + (size_t)q * tt.lb * W, 2 * c0, q * tt.lb, by);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      const int tn = t + 2 * (int)gridDim.x;
      if (tn < ntiles) {
        // the result buffer becomes the next prefetch target once drained
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        issue(tn, rb);
      }
    }
    cur = pre;
    tmp = ob;
    pre = rb;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launches
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000)p;
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

static constexpr int kTmaNT = 512;

static int tma_w(bool f64) { return f64 ? 4 : 8; }

// (2W x rows [x batch]) box over a complex array viewed as doubles/floats
int fft_tma_make(FftTma& M, void* base, bool f64, int rank, long long inner_complex, long long rows,
                 long long batch, int L) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encode_fn();
  if (!enc) return fail(SFB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int W = tma_w(f64);
  const size_t esz = f64 ? 8 : 4;
  const int nbox = (L + 255) / 256;
  const int lb = (((L + nbox - 1) / nbox) + 1) & ~1;  // even: 128-byte aligned box destinations
  cuuint64_t dims[3] = {(cuuint64_t)(2 * inner_complex), (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(2 * inner_complex * esz), (cuuint64_t)(2 * inner_complex * esz * rows)};
  cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)lb, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  M.ok = false;
  // TMA needs 16-byte multiples for the global strides; otherwise keep the
  // cp.async path for this pass
  if ((strides[0] % 16) != 0 || (rank == 3 && (strides[1] % 16) != 0) || ((uintptr_t)base % 16) != 0) return SFB_OK;
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(&M.map), f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   (cuuint32_t)rank, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return SFB_OK;  // unsupported geometry: cp.async path
  M.rank = rank;
  M.nbox = nbox;
  M.lb = lb;
  M.ncol = (int)inner_complex;
  M.nbatch = rank == 3 ? (int)batch : 1;
  M.ok = true;
  return SFB_OK;
}

template <typename T, int MODE>
int fft_tma_pass(const FftTma& M, const FftLen& P, const void* tw, const ScaleArgs& sc, cudaStream_t st) {
  typedef typename CX<T>::t C;
  constexpr int W = sizeof(T) == 8 ? 4 : 8;
  static int nsm = 0;
  const size_t smem = 3 * (size_t)M.nbox * M.lb * W * sizeof(C) + 64 + (size_t)P.twn * sizeof(C);
  if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  if (cudaError_t e = ensure_smem((const void*)k_fft_tma<T, MODE, W, kTmaNT>, 227 * 1024))
    return cuda_check(e, "fft tma: shared-memory attribute");
  TmaTile tt{M.rank, M.nbox, M.lb, M.ncol, M.nbatch};
  const long long ntiles = (long long)((M.ncol + W - 1) / W) * M.nbatch;
  const int g = (int)(ntiles < nsm ? ntiles : nsm);
  const CUtensorMap* map = reinterpret_cast<const CUtensorMap*>(&M.map);
  k_fft_tma<T, MODE, W, kTmaNT><<<g, kTmaNT, smem, st>>>(*map, tt, P, (const C*)tw, sc);
  SFB_LAUNCH_CHECK("fft tma pass");
  return SFB_OK;
}
template int fft_tma_pass<double, 0>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);
template int fft_tma_pass<double, 1>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);
template int fft_tma_pass<double, 2>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);
template int fft_tma_pass<float, 0>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);
template int fft_tma_pass<float, 1>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);
template int fft_tma_pass<float, 2>(const FftTma&, const FftLen&, const void*, const ScaleArgs&, cudaStream_t);

bool fft_tma_fits(int L, bool f64) {
  const int W = tma_w(f64);
  const int nbox = (L + 255) / 256;
  const int lb = (((L + nbox - 1) / nbox) + 1) & ~1;
  const size_t bytes = 3 * (size_t)nbox * lb * W * (f64 ? 16 : 8) + 64 + 2 * (size_t)L * (f64 ? 16 : 8);
  return bytes <= 227 * 1024;
}

}  // namespace sfb
