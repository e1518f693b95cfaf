// Plan creation: grid tables and boundary metadata on the device
// (replaces grid.py:115-223 + operators.py:38-90 as seen by the kernels).
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <map>
#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include "sfb_common.cuh"

namespace sfb {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SFB_OK;
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  g_err = m;
  return SFB_ECUDA;
}

cudaError_t ensure_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[std::make_pair(func, dev)];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

template <typename T>
static void fill_geo(Geo<T>& G, const sfb_plan* p, const T* dtab) {
  memset(&G, 0, sizeof(G));
  G.dim = p->dim;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = a < p->dim ? p->n[a] : 1;
    G.E[a] = a < p->dim ? p->n[a] + 2 : 1;
    G.per[a] = a < p->dim ? (p->bc_lo[a] == SFB_BC_PERIODIC || p->bc_lo[a] == SFB_BC_HALO) : 1;
    G.halo[a] = a < p->dim ? (p->bc_lo[a] == SFB_BC_HALO) : 0;
    G.bc_lo[a] = p->bc_lo[a];
    G.bc_hi[a] = p->bc_hi[a];
    for (int c = 0; c < 3; ++c) {
      // (T)(2.0*val): the reference forms 2.0*val in Python floats and the
      // subtraction happens in the array dtype (fields.py:120,130,133)
      G.c2lo[a][c] = (T)(2.0 * p->val_lo[a][c]);
      G.c2hi[a][c] = (T)(2.0 * p->val_hi[a][c]);
      G.vlo[a][c] = (T)p->val_lo[a][c];
      G.vhi[a][c] = (T)p->val_hi[a][c];
    }
  }
  if (p->dim == 3) {
    G.s[2] = 1;
    G.s[1] = G.E[2];
    G.s[0] = (long long)G.E[1] * G.E[2];
  } else {
    G.s[2] = 0;
    G.s[1] = 1;
    G.s[0] = G.E[1];
  }
  size_t off = 0;
  for (int a = 0; a < p->dim; ++a) {
    for (int t = 0; t < SFB_NTAB; ++t) {
      G.tab[a][t] = dtab + off;
      off += G.E[a];
    }
  }
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_abi_version(void) { return SFB_ABI_VERSION; }

const char* sfb_last_error(void) { return g_err.c_str(); }

int sfb_plan_create(const sfb_grid_desc* d, sfb_plan** out) {
  if (!d || !out) return fail(SFB_EINVAL, "null argument");
  *out = nullptr;
  if (d->dim != 2 && d->dim != 3) return fail(SFB_ECONFIG, "unsupported dimension; need 2 or 3");
  if (d->dtype != SFB_F64 && d->dtype != SFB_F32) return fail(SFB_EINVAL, "dtype must be float64 or float32");
  for (int a = 0; a < d->dim; ++a) {
    if (d->n[a] < 1) return fail(SFB_EINVAL, "need at least one volume per axis");
    bool plo = d->bc_lo[a] == SFB_BC_PERIODIC, phi = d->bc_hi[a] == SFB_BC_PERIODIC;
    if (plo != phi) return fail(SFB_EINVAL, "periodic must be declared on both sides or neither");
    if ((d->bc_lo[a] == SFB_BC_HALO) != (d->bc_hi[a] == SFB_BC_HALO))
      return fail(SFB_EINVAL, "halo must be declared on both sides or neither");
    const bool wall = !plo && d->bc_lo[a] != SFB_BC_HALO;
    if (wall && d->n[a] < 2) return fail(SFB_ECONFIG, "a wall axis needs at least two volumes");
    for (int s = 0; s < 2; ++s) {
      int k = s ? d->bc_hi[a] : d->bc_lo[a];
      if (k < 0 || k > 3) return fail(SFB_EINVAL, "unknown boundary kind");
    }
  }
  if (!d->tables) return fail(SFB_EINVAL, "missing grid tables");

  sfb_plan* p = new sfb_plan();
  p->dim = d->dim;
  p->dtype = d->dtype;
  p->ext_count = 1;
  p->int_count = 1;
  size_t ntab = 0;
  for (int a = 0; a < 3; ++a) {
    p->n[a] = a < d->dim ? d->n[a] : 1;
    p->bc_lo[a] = a < d->dim ? d->bc_lo[a] : SFB_BC_PERIODIC;
    p->bc_hi[a] = a < d->dim ? d->bc_hi[a] : SFB_BC_PERIODIC;
    p->width0[a] = d->width0[a];
    for (int c = 0; c < 3; ++c) {
      p->val_lo[a][c] = d->val_lo[a][c];
      p->val_hi[a][c] = d->val_hi[a][c];
    }
    if (a < d->dim) {
      p->ext_count *= (p->n[a] + 2);
      p->int_count *= p->n[a];
      ntab += (size_t)SFB_NTAB * (p->n[a] + 2);
      if (p->bc_lo[a] != SFB_BC_PERIODIC) p->all_periodic = false;
    }
  }
  size_t esz = d->dtype == SFB_F64 ? 8 : 4;
  std::vector<unsigned char> host(ntab * esz);
  for (size_t i = 0; i < ntab; ++i) {
    if (esz == 8)
      reinterpret_cast<double*>(host.data())[i] = d->tables[i];
    else
      reinterpret_cast<float*>(host.data())[i] = (float)d->tables[i];
  }
  int rc = SFB_OK;
  if ((rc = cuda_check(cudaMalloc(&p->d_tables, host.size()), "cudaMalloc(tables)")) != SFB_OK) goto bad;
  if ((rc = cuda_check(cudaMemcpy(p->d_tables, host.data(), host.size(), cudaMemcpyHostToDevice), "upload tables")) != SFB_OK)
    goto bad;
  p->red_blocks = 1184;  // 8 x 148 SMs
  if ((rc = cuda_check(cudaMalloc(&p->d_red, sizeof(double) * (p->red_blocks + 8)), "cudaMalloc(red)")) != SFB_OK) goto bad;
  if ((rc = cuda_check(cudaMallocHost(&p->h_red, sizeof(double) * 8), "cudaMallocHost")) != SFB_OK) goto bad;
  {
    size_t off = 0;
    for (int a = 0; a < d->dim; ++a) {
      const size_t E = p->n[a] + 2;
      p->hdx[a].assign(d->tables + off + T_DX * E, d->tables + off + (T_DX + 1) * E);
      p->hdu[a].assign(d->tables + off + T_DU * E, d->tables + off + (T_DU + 1) * E);
      off += SFB_NTAB * E;
    }
  }
  if (d->dtype == SFB_F64)
    fill_geo<double>(p->g64, p, (const double*)p->d_tables);
  else
    fill_geo<float>(p->g32, p, (const float*)p->d_tables);
  *out = p;
  return SFB_OK;
bad:
  sfb_plan_destroy(p);
  return rc;
}

// Dirichlet wall values of a plan whose walls move (a callable Dirichlet
// evaluated at a new time, fields.py:72-76); kernels take the plan's Geo by
// value at launch, so every launch after this call sees the new values
int sfb_plan_set_walls(sfb_plan* p, const double* val_lo, const double* val_hi) {
  if (!p || !val_lo || !val_hi) return fail(SFB_EINVAL, "null argument");
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      p->val_lo[a][c] = val_lo[3 * a + c];
      p->val_hi[a][c] = val_hi[3 * a + c];
    }
  auto put = [&](auto& G) {
    typedef typename std::remove_reference<decltype(G.vlo[0][0])>::type T;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        G.c2lo[a][c] = (T)(2.0 * p->val_lo[a][c]);
        G.c2hi[a][c] = (T)(2.0 * p->val_hi[a][c]);
        G.vlo[a][c] = (T)p->val_lo[a][c];
        G.vhi[a][c] = (T)p->val_hi[a][c];
      }
  };
  put(p->g64);
  put(p->g32);
  return SFB_OK;
}

int sfb_plan_destroy(sfb_plan* p) {
  if (!p) return SFB_OK;
  if (p->d_tables) cudaFree(p->d_tables);
  if (p->d_red) cudaFree(p->d_red);
  if (p->h_red) cudaFreeHost(p->h_red);
  delete p;
  return SFB_OK;
}

}  // extern "C"
