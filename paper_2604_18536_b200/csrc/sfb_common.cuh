// Shared definitions for the stagflow_b200 kernels (sm_100a).
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <vector>

#include "../../include/stagflow_b200.h"

namespace sfb {

// table slots (order fixed by the ABI, stagflow_b200.h)
enum { T_DX = 0, T_DU, T_RDX, T_RDU, T_WLO, T_WHI, T_OHI, T_OLO, T_THI, T_TLO };

// Per-launch geometry + device table pointers.  Passed by value.
template <typename T>
struct Geo {
  int dim;
  int n[3];        // interior extents
  int E[3];        // extended extents (n+2); unused axes = 1
  long long s[3];  // element strides of the extended array
  int per[3];      // periodic flags (DOF semantics; also set for halo axes)
  int halo[3];     // ghost planes supplied externally (slab decomposition)
  int bc_lo[3], bc_hi[3];
  T c2lo[3][3], c2hi[3][3];  // (T)(2*val) for tangential reflections [axis][comp]
  T vlo[3][3], vhi[3][3];    // (T)val for normal boundary faces
  const T* tab[3][SFB_NTAB];
};

}  // namespace sfb

// The plan (opaque to C callers).
struct sfb_plan {
  int dim = 0;
  int dtype = SFB_F64;
  int n[3] = {1, 1, 1};
  int bc_lo[3] = {0, 0, 0}, bc_hi[3] = {0, 0, 0};
  double val_lo[3][3] = {}, val_hi[3][3] = {};
  double width0[3] = {0, 0, 0};
  std::string bc_sig;
  void* d_tables = nullptr;     // SFB_NTAB * sum(n+2) values of T
  double* d_red = nullptr;      // reduction partials (fp64)
  double* h_red = nullptr;      // pinned host scalar
  int red_blocks = 0;
  sfb::Geo<double> g64;
  sfb::Geo<float> g32;
  bool all_periodic = true;
  long long ext_count = 0;      // elements of one extended array
  long long int_count = 0;      // interior cells
  std::vector<double> hdx[3], hdu[3];  // host copies of the dx/du tables
};

namespace sfb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
// cudaFuncAttributeMaxDynamicSharedMemorySize for kernel `func` on the
// current device, set once per (kernel, device) under a mutex (plan.cu):
// a process may drive several devices, and plans are used from any thread.
cudaError_t ensure_smem(const void* func, size_t bytes);
// Tuning knob from the environment, read once (thread-safe static init in the
// caller): 0 if unset.
inline int env_int(const char* name, int dflt = 0) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <typename T>
inline const Geo<T>& geo(const sfb_plan* p);
template <>
inline const Geo<double>& geo<double>(const sfb_plan* p) { return p->g64; }
template <>
inline const Geo<float>& geo<float>(const sfb_plan* p) { return p->g32; }

// Generic cell launch: D-dimensional box [lo, lo+cnt) of the extended index
// space.  x runs over the fastest axis (D-1) for coalescing.
struct Box {
  int lo[3];
  int cnt[3];
};

inline dim3 box_block(int dim) { return dim == 3 ? dim3(32, 4, 2) : dim3(32, 8, 1); }
inline dim3 box_grid(int dim, const Box& b) {
  dim3 blk = box_block(dim);
  if (dim == 3)
    return dim3((b.cnt[2] + blk.x - 1) / blk.x, (b.cnt[1] + blk.y - 1) / blk.y, (b.cnt[0] + blk.z - 1) / blk.z);
  return dim3((b.cnt[1] + blk.x - 1) / blk.x, (b.cnt[0] + blk.y - 1) / blk.y, 1);
}

// coordinates of this thread in the box; returns false when outside
template <int D>
__device__ __forceinline__ bool box_coords(const Box& b, int I[3]) {
  if (D == 3) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    int j = blockIdx.y * blockDim.y + threadIdx.y;
    int i = blockIdx.z * blockDim.z + threadIdx.z;
    if (k >= b.cnt[2] || j >= b.cnt[1] || i >= b.cnt[0]) return false;
    I[0] = i + b.lo[0];
    I[1] = j + b.lo[1];
    I[2] = k + b.lo[2];
  } else {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    int i = blockIdx.y * blockDim.y + threadIdx.y;
    if (j >= b.cnt[1] || i >= b.cnt[0]) return false;
    I[0] = i + b.lo[0];
    I[1] = j + b.lo[1];
    I[2] = 0;
  }
  return true;
}

template <typename T, int D>
__device__ __forceinline__ long long lin(const Geo<T>& G, const int I[3]) {
  long long r = (long long)I[0] * G.s[0] + (long long)I[1] * G.s[1];
  if (D == 3) r += (long long)I[2] * G.s[2];
  return r;
}

// Is I a degree of freedom of velocity component c (grid.py:197-209)?
template <typename T, int D>
__device__ __forceinline__ bool is_udof(const Geo<T>& G, const int I[3], int c) {
#pragma unroll
  for (int b = 0; b < D; ++b) {
    int hi = (b == c && !G.per[b]) ? G.n[b] - 1 : G.n[b];
    if (I[b] < 1 || I[b] > hi) return false;
  }
  return true;
}

template <typename T, int D>
__device__ __forceinline__ bool is_pdof(const Geo<T>& G, const int I[3]) {
#pragma unroll
  for (int b = 0; b < D; ++b)
    if (I[b] < 1 || I[b] > G.n[b]) return false;
  return true;
}

template <typename T>
__device__ __forceinline__ T tab(const Geo<T>& G, int axis, int slot, int i) {
  return __ldg(G.tab[axis][slot] + i);
}

// periodic wrap of an interior index that stepped one past the range
// 1 / lam of the spectral scaling.  fp64: the MUFU seed and two Newton
// steps (within one ulp of the IEEE quotient, a handful of instructions
// instead of the division's ~25-instruction sequence, which dominated the
// fused axis-0 pass); fp32: the correctly rounded reciprocal (== 1.0f / x).
template <typename T>
__device__ __forceinline__ T spec_rcp(double lam);
template <>
__device__ __forceinline__ double spec_rcp<double>(double lam) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(lam));
  double e = fma(-lam, r, 1.0);
  r = fma(r, e, r);
  e = fma(-lam, r, 1.0);
  return fma(r, e, r);
}
template <>
__device__ __forceinline__ float spec_rcp<float>(double lam) {
  return __frcp_rn((float)lam);
}

__device__ __forceinline__ int wrap1(int i, int n) { return i < 1 ? i + n : (i > n ? i - n : i); }

// Launch-configuration helpers for the host.
template <typename T>
Box ext_box(const Geo<T>& G) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = 0;
    b.cnt[a] = a < G.dim ? G.E[a] : 1;
  }
  return b;
}
template <typename T>
Box int_box(const Geo<T>& G) {
  Box b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = a < G.dim ? 1 : 0;
    b.cnt[a] = a < G.dim ? G.n[a] : 1;
  }
  return b;
}

// NVTX range over one C-ABI call (tracing): the host span in which
// the call enqueues its kernels, named after the entry point; free when no
// tool is attached (NVTX3 is header-only)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};
#define SFB_RANGE() ::sfb::NvtxScope sfb_nvtx_scope_(__func__)

}  // namespace sfb

#define SFB_DISPATCH_DIM(dim, D, ...) \
  do {                                \
    if ((dim) == 3) {                 \
      constexpr int D = 3;            \
      __VA_ARGS__;                    \
    } else {                          \
      constexpr int D = 2;            \
      __VA_ARGS__;                    \
    }                                 \
  } while (0)

#define SFB_LAUNCH_CHECK(what)                                           \
  do {                                                                   \
    cudaError_t _e = cudaGetLastError();                                 \
    if (_e != cudaSuccess) return sfb::cuda_check(_e, what);             \
  } while (0)
