// NCCL communicator of the z-slab decomposition behind the C ABI
// (SURVEY 8(b) comm_create, 8(e)): ghost-plane exchange, the spectral
// solve's all-to-all transposes and fp64 all-reduces, all enqueued on the
// caller's CUDA stream -- no host synchronisation.
//
// NCCL is resolved at sfb_comm_create time with dlopen("libnccl.so.2"): the
// copy the process has already loaded (PyTorch's) is reused, so one NCCL
// runs per process, and the core library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "sfb_common.cuh"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SFB_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    SFB_SYM(GetUniqueId);
    SFB_SYM(CommInitRank);
    SFB_SYM(CommDestroy);
    SFB_SYM(GroupStart);
    SFB_SYM(GroupEnd);
    SFB_SYM(Send);
    SFB_SYM(Recv);
    SFB_SYM(AllReduce);
    SFB_SYM(GetErrorString);
#undef SFB_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
             api.Recv && api.AllReduce && api.GetErrorString;
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SFB_OK;
  return sfb::fail(SFB_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

struct sfb_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

using namespace sfb;

extern "C" {

int sfb_comm_unique_id(void* id) {
  if (!id) return fail(SFB_EINVAL, "null argument");
  if (!nccl().ok) return fail(SFB_ECONFIG, "libnccl.so.2 not found");
  ncclUniqueId u;
  if (int rc = nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId")) return rc;
  std::memcpy(id, &u, sizeof(u));
  return SFB_OK;
}

int sfb_comm_create(const void* id, int nranks, int rank, sfb_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(SFB_EINVAL, "bad communicator arguments");
  *out = nullptr;
  if (!nccl().ok) return fail(SFB_ECONFIG, "libnccl.so.2 not found");
  sfb_comm* c = new sfb_comm();
  c->rank = rank;
  c->nranks = nranks;
  cudaGetDevice(&c->device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  if (int rc = nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank")) {
    delete c;
    return rc;
  }
  *out = c;
  return SFB_OK;
}

int sfb_comm_destroy(sfb_comm* c) {
  if (!c) return SFB_OK;
  int rc = c->comm ? nccl_check(nccl().CommDestroy(c->comm), "ncclCommDestroy") : SFB_OK;
  delete c;
  return rc;
}

int sfb_comm_rank(const sfb_comm* c) { return c ? c->rank : -1; }

// send `bytes` of `send` to peer_send and receive as many into `recv` from
// peer_recv, one NCCL group (either side may be skipped with a null pointer)
int sfb_comm_sendrecv(sfb_comm* c, const void* send, int peer_send, void* recv, int peer_recv, size_t bytes,
                      void* stream) {
  SFB_RANGE();
  if (!c) return fail(SFB_EINVAL, "null communicator");
  cudaStream_t st = (cudaStream_t)stream;
  if (c->nranks == 1) {  // periodic self-exchange
    if (send && recv && send != recv)
      return cuda_check(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st), "self send/recv");
    return SFB_OK;
  }
  NcclApi& n = nccl();
  if (int rc = nccl_check(n.GroupStart(), "ncclGroupStart")) return rc;
  if (send) n.Send(send, bytes, ncclChar, peer_send, c->comm, st);
  if (recv) n.Recv(recv, bytes, ncclChar, peer_recv, c->comm, st);
  return nccl_check(n.GroupEnd(), "ncclSend/ncclRecv");
}

// ghost planes along axis 0 of nf extended fields of m local planes
// (plane_bytes each): plane 0 <- prev rank's plane m, plane m+1 <- next
// rank's plane 1; one group for all fields
int sfb_comm_halo(sfb_comm* c, void* const* fields, int nf, size_t plane_bytes, int m, void* stream) {
  SFB_RANGE();
  if (!c || !fields || nf < 1 || m < 1) return fail(SFB_EINVAL, "bad halo arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (c->nranks == 1) {
    for (int f = 0; f < nf; ++f) {
      char* b = (char*)fields[f];
      if (int rc = cuda_check(cudaMemcpyAsync(b, b + (size_t)m * plane_bytes, plane_bytes, cudaMemcpyDeviceToDevice, st),
                              "halo (self)"))
        return rc;
      if (int rc = cuda_check(cudaMemcpyAsync(b + (size_t)(m + 1) * plane_bytes, b + plane_bytes, plane_bytes,
                                              cudaMemcpyDeviceToDevice, st),
                              "halo (self)"))
        return rc;
    }
    return SFB_OK;
  }
  const int prev = (c->rank + c->nranks - 1) % c->nranks, next = (c->rank + 1) % c->nranks;
  NcclApi& n = nccl();
  if (int rc = nccl_check(n.GroupStart(), "ncclGroupStart")) return rc;
  for (int f = 0; f < nf; ++f) {
    char* b = (char*)fields[f];
    n.Send(b + (size_t)m * plane_bytes, plane_bytes, ncclChar, next, c->comm, st);
    n.Recv(b, plane_bytes, ncclChar, prev, c->comm, st);
    n.Send(b + plane_bytes, plane_bytes, ncclChar, prev, c->comm, st);
    n.Recv(b + (size_t)(m + 1) * plane_bytes, plane_bytes, ncclChar, next, c->comm, st);
  }
  return nccl_check(n.GroupEnd(), "halo exchange");
}

// equal-split all-to-all: block q (bytes_per_peer) of send goes to rank q,
// block q of recv comes from rank q
int sfb_comm_alltoall(sfb_comm* c, const void* send, void* recv, size_t bytes_per_peer, void* stream) {
  SFB_RANGE();
  if (!c || !send || !recv) return fail(SFB_EINVAL, "bad all-to-all arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (c->nranks == 1)
    return send == recv ? SFB_OK
                        : cuda_check(cudaMemcpyAsync(recv, send, bytes_per_peer, cudaMemcpyDeviceToDevice, st),
                                     "all-to-all (self)");
  NcclApi& n = nccl();
  if (int rc = nccl_check(n.GroupStart(), "ncclGroupStart")) return rc;
  for (int q = 0; q < c->nranks; ++q) {
    n.Send((const char*)send + (size_t)q * bytes_per_peer, bytes_per_peer, ncclChar, q, c->comm, st);
    n.Recv((char*)recv + (size_t)q * bytes_per_peer, bytes_per_peer, ncclChar, q, c->comm, st);
  }
  return nccl_check(n.GroupEnd(), "all-to-all");
}

// in-place all-reduce of count fp64 values in device memory: op 0 sum,
// 1 min, 2 max
int sfb_comm_allreduce_f64(sfb_comm* c, double* buf, size_t count, int op, void* stream) {
  SFB_RANGE();
  if (!c || !buf || op < 0 || op > 2) return fail(SFB_EINVAL, "bad all-reduce arguments");
  if (c->nranks == 1) return SFB_OK;
  const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
  return nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat64, o, c->comm, (cudaStream_t)stream),
                    "ncclAllReduce");
}

}  // extern "C"
