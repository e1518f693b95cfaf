// Plane-averaged channel statistics on the GPU (stats.py:55-167): per
// wall-normal index, deterministic two-pass fp64 sums over the homogeneous
// planes, so a snapshot never leaves the device; the host forms the profile
// and the snapshot average (in long double, like the reference).
#include "sfb_kernels.cuh"

namespace sfb {

namespace {
constexpr int kStNT = 256, kStChunks = 32;  // blocks per plane

template <int NT>
__device__ __forceinline__ double st_bsum(double v) {
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

// interior position t of the homogeneous plane at wall index j -> cell I
template <int D>
__device__ __forceinline__ void plane_cell(const int n[3], int wall, int j, long long t, int I[3]) {
  int ax[2], c = 0;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (a != wall) ax[c++] = a;
  I[0] = I[1] = I[2] = 0;
  I[wall] = j;
  if (D == 3) {
    I[ax[1]] = 1 + (int)(t % n[ax[1]]);
    I[ax[0]] = 1 + (int)(t / n[ax[1]]);
  } else {
    I[ax[0]] = 1 + (int)t;
  }
}
}  // namespace

// NQ quantities per wall index j = 1..n_wall, summed over the plane
//  MODE 0: raw component sums  q_a = u_a                           (NQ = D)
//  MODE 1: fluctuation moments (u = fluctuation, ghosts filled with the
//          homogeneous conditions): q0 = f_0^2, q1 = f_o^2 (o the other
//          homogeneous axis, 3D), q2 = c_w^2, q3 = f_0^3, q4 = f_0^4,
//          q5 = c_0 c_0 c_w, q6 = c_0 c_o'   (c = centred, o' = 2 in 3D else 1)
template <typename T, int D, int MODE>
__global__ void __launch_bounds__(kStNT) k_plane_sums(Geo<T> G, CV<T> U, int wall, double* __restrict__ part) {
  constexpr int NQ = MODE == 0 ? D : 7;
  const int j = 1 + blockIdx.y;
  long long plane = 1;
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (a != wall) plane *= G.n[a];
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const int oth = D == 3 ? (wall == 2 ? 1 : 2) : 1;   // the rms of u_oth (3D), stats.py:105-113
  const int cross = D == 3 ? 2 : 1;                    // uw partner (stats.py:122-123)
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < plane; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    plane_cell<D>(G.n, wall, j, t, I);
    const long long x = lin<T, D>(G, I);
    if (MODE == 0) {
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += (double)U.c[a][x];
    } else {
      const T f0 = U.c[0][x];
      const T c0 = T(0.5) * (U.c[0][x - G.s[0]] + f0);
      const T cw = T(0.5) * (U.c[wall][x - G.s[wall]] + U.c[wall][x]);
      const T cc = T(0.5) * (U.c[cross][x - G.s[cross]] + U.c[cross][x]);
      const T fo = D == 3 ? U.c[oth][x] : T(0);
      acc[0] += (double)(f0 * f0);
      acc[1] += (double)(fo * fo);
      acc[2] += (double)(cw * cw);
      acc[3] += (double)(f0 * f0 * f0);
      acc[4] += (double)(f0 * f0 * f0 * f0);
      acc[5] += (double)(c0 * c0 * cw);
      acc[6] += (double)(c0 * cc);
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = st_bsum<kStNT>(acc[q]);
    if (threadIdx.x == 0) part[((long long)q * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void k_plane_finish(const double* __restrict__ part, int nq, int nj, int nb, double* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nq * nj) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(long long)idx * nb + b];
  out[idx] = s;
}

// u_a -= mean_a[j] at every position of wall index j = 1..n_wall
template <typename T, int D>
__global__ void k_sub_plane_mean(Geo<T> G, MV<T> U, int wall, const double* __restrict__ mean) {
  const long long total = (long long)G.E[0] * G.E[1] * (D == 3 ? G.E[2] : 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int I[3];
    long long r = t;
    if (D == 3) {
      I[2] = (int)(r % G.E[2]);
      r /= G.E[2];
    } else {
      I[2] = 0;
    }
    I[1] = (int)(r % G.E[1]);
    I[0] = (int)(r / G.E[1]);
    const int j = I[wall];
    if (j < 1 || j > G.n[wall]) continue;
#pragma unroll
    for (int a = 0; a < D; ++a) U.c[a][t] -= (T)mean[a * G.n[wall] + (j - 1)];
  }
}

template <typename T>
static int plane_sums_run(sfb_plan* p, int wall, const void* const* u, int mode, double* out, cudaStream_t st) {
  const Geo<T>& G = geo<T>(p);
  CV<T> U;
  for (int a = 0; a < 3; ++a) U.c[a] = a < p->dim ? (const T*)u[a] : nullptr;
  const int nj = G.n[wall];
  const int nq = mode == 0 ? p->dim : 7;
  double* part = nullptr;
  int rc = cuda_check(cudaMallocAsync(&part, sizeof(double) * (size_t)nq * nj * kStChunks, st), "stats scratch");
  if (rc) return rc;
  dim3 grid(kStChunks, nj);
  if (mode == 0)
    SFB_DISPATCH_DIM(G.dim, D, (k_plane_sums<T, D, 0><<<grid, kStNT, 0, st>>>(G, U, wall, part)));
  else
    SFB_DISPATCH_DIM(G.dim, D, (k_plane_sums<T, D, 1><<<grid, kStNT, 0, st>>>(G, U, wall, part)));
  k_plane_finish<<<(nq * nj + 127) / 128, 128, 0, st>>>(part, nq, nj, kStChunks, out);
  rc = cuda_check(cudaGetLastError(), "plane sums");
  cudaFreeAsync(part, st);
  return rc;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_plane_sums(sfb_plan* p, int wall_axis, const void* const* u, int mode, double* out, void* stream) {
  SFB_RANGE();
  if (!p || !u || !out) return fail(SFB_EINVAL, "null argument");
  if (wall_axis < 0 || wall_axis >= p->dim) return fail(SFB_EINVAL, "wall axis out of range");
  if (mode != 0 && mode != 1) return fail(SFB_EINVAL, "unknown plane-sum mode");
  for (int a = 0; a < p->dim; ++a)
    if (!u[a]) return fail(SFB_EINVAL, "null velocity component");
  return SFB_TYPED(p, plane_sums_run<T>(p, wall_axis, u, mode, out, (cudaStream_t)stream));
}

int sfb_sub_plane_mean(sfb_plan* p, int wall_axis, void* const* u, const double* mean, void* stream) {
  SFB_RANGE();
  if (!p || !u || !mean) return fail(SFB_EINVAL, "null argument");
  if (wall_axis < 0 || wall_axis >= p->dim) return fail(SFB_EINVAL, "wall axis out of range");
  cudaStream_t st = (cudaStream_t)stream;
  return SFB_TYPED(p, ([&]() -> int {
    const Geo<T>& G = geo<T>(p);
    MV<T> U;
    for (int a = 0; a < 3; ++a) U.c[a] = a < p->dim ? (T*)u[a] : nullptr;
    SFB_DISPATCH_DIM(G.dim, D, (k_sub_plane_mean<T, D><<<148 * 8, 256, 0, st>>>(G, U, wall_axis, mean)));
    SFB_LAUNCH_CHECK("subtract plane mean");
    return SFB_OK;
  }()));
}

}  // extern "C"
