// Time-rank hand-offs over NCCL for non-Python hosts:
// the C-ABI equivalent of the exchanges the controller needs -- C1 fine
// payload + flag and C2 coarse payload rank n -> n+1 (ncclSend/ncclRecv,
// pfasst.py:107-118, 189-202), C3 the block-boundary broadcast
// (pfasst.py:272-278).  libnccl is opened with dlopen on first use, so the
// library has no link-time NCCL dependency and still loads on CPU-only hosts;
// the Python package's "nccl" executor uses torch.distributed instead and
// does not call these.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/pintlab_b200.h"
#include "common.cuh"

namespace pl {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                        cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

template <typename F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

int nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return 0;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error("libnccl.so.2 not found (%s)", dlerror());
    return PL_ERR_UNSUPPORTED;
  }
  NcclApi a;
  a.h = h;
  bool ok = sym(h, "ncclGetUniqueId", a.get_unique_id) &&
            sym(h, "ncclCommInitRank", a.comm_init_rank) &&
            sym(h, "ncclCommDestroy", a.comm_destroy) && sym(h, "ncclSend", a.send) &&
            sym(h, "ncclRecv", a.recv) && sym(h, "ncclBroadcast", a.bcast) &&
            sym(h, "ncclGroupStart", a.group_start) && sym(h, "ncclGroupEnd", a.group_end) &&
            sym(h, "ncclGetErrorString", a.error_string);
  if (!ok) {
    set_error("libnccl is missing a required symbol");
    return PL_ERR_UNSUPPORTED;
  }
  g_nccl = a;
  return 0;
}

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  set_error("NCCL error in %s: %s", what, g_nccl.error_string ? g_nccl.error_string(r) : "?");
  return PL_ERR_CUDA;
}

}  // namespace
}  // namespace pl

struct pl_comm {
  ncclComm_t comm;
  int rank, nranks, device;
};

extern "C" {

int pl_comm_unique_id(char* id) {
  if (!id) {
    pl::set_error("null id buffer");
    return PL_ERR_ARG;
  }
  PL_TRY(pl::nccl_api());
  ncclUniqueId u;
  PL_TRY(pl::nccl_status(pl::g_nccl.get_unique_id(&u), "ncclGetUniqueId"));
  std::memcpy(id, u.internal, PL_COMM_ID_BYTES);
  return PL_OK;
}

int pl_comm_init(pl_comm** out, const char* id, int rank, int nranks, int device) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks || device < 0) {
    pl::set_error("bad communicator arguments (rank %d of %d, device %d)", rank, nranks,
                  device);
    return PL_ERR_ARG;
  }
  PL_TRY(pl::nccl_api());
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return pl::cuda_status(e, "cudaSetDevice");
  ncclUniqueId u;
  std::memcpy(u.internal, id, PL_COMM_ID_BYTES);
  pl_comm* c = new pl_comm;
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  int rc = pl::nccl_status(pl::g_nccl.comm_init_rank(&c->comm, nranks, u, rank),
                           "ncclCommInitRank");
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return PL_OK;
}

int pl_comm_destroy(pl_comm* c) {
  if (!c) return PL_OK;
  int rc = pl::nccl_status(pl::g_nccl.comm_destroy(c->comm), "ncclCommDestroy");
  delete c;
  return rc;
}

int pl_comm_group_start(void) {
  PL_TRY(pl::nccl_api());
  return pl::nccl_status(pl::g_nccl.group_start(), "ncclGroupStart");
}

int pl_comm_group_end(void) {
  PL_TRY(pl::nccl_api());
  return pl::nccl_status(pl::g_nccl.group_end(), "ncclGroupEnd");
}

int pl_comm_send(pl_comm* c, const void* buf, size_t bytes, int peer, void* stream) {
  if (!c || (!buf && bytes) || peer < 0 || peer >= c->nranks) {
    pl::set_error("bad send arguments");
    return PL_ERR_ARG;
  }
  return pl::nccl_status(pl::g_nccl.send(buf, bytes, ncclUint8, peer, c->comm,
                                         (cudaStream_t)stream),
                         "ncclSend");
}

int pl_comm_recv(pl_comm* c, void* buf, size_t bytes, int peer, void* stream) {
  if (!c || (!buf && bytes) || peer < 0 || peer >= c->nranks) {
    pl::set_error("bad recv arguments");
    return PL_ERR_ARG;
  }
  return pl::nccl_status(pl::g_nccl.recv(buf, bytes, ncclUint8, peer, c->comm,
                                         (cudaStream_t)stream),
                         "ncclRecv");
}

int pl_comm_bcast(pl_comm* c, void* buf, size_t bytes, int root, void* stream) {
  if (!c || (!buf && bytes) || root < 0 || root >= c->nranks) {
    pl::set_error("bad broadcast arguments");
    return PL_ERR_ARG;
  }
  return pl::nccl_status(pl::g_nccl.bcast(buf, buf, bytes, ncclUint8, root, c->comm,
                                          (cudaStream_t)stream),
                         "ncclBroadcast");
}

}  // extern "C"
