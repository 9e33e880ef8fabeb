// NCCL communicators and the per-sweep node-RHS all-gather behind the C ABI
// (include/sdcsw.h, "NCCL transport").  Replaces the reference's per-sweep
// thread-pool barrier (pkg/src/parsdc/integrators.py:278-288: every node's
// future.result() before the next quadrature) when the nodes of a sweep live
// on different GPUs: one ncclAllGather of the (f_E, f_I) pairs per sweep, and
// with a spectral split one more of the Fourier parts per f_E.
//
// torch.distributed is used only to carry the 128-byte unique id from rank 0
// to the others (bootstrap); communicator creation, splitting and every
// collective on the data path are these calls.  All collectives are
// stream-ordered and capturable into CUDA graphs (the node-parallel step
// replays as one graph with the all-gathers inside).
//
// NCCL is bound at first use with dlopen("libnccl.so.2"), not at link time:
// the process's NCCL is then the one PyTorch already loaded (same soname), so
// loading libsdcsw.so can never put a second, older NCCL in front of
// libtorch_cuda (which needs its own version's symbols).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/sdcsw.h"
#include "internal.cuh"

struct sdcsw_comm {
  ncclComm_t comm = nullptr;
  int world = 0;
  int rank = 0;
  int device = 0;
};

namespace {

struct Nccl {
  bool ok = false;
  std::string why;
  decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&::ncclCommInitRank) CommInitRank = nullptr;
  decltype(&::ncclCommInitAll) CommInitAll = nullptr;
  decltype(&::ncclCommSplit) CommSplit = nullptr;
  decltype(&::ncclCommCount) CommCount = nullptr;
  decltype(&::ncclCommUserRank) CommUserRank = nullptr;
  decltype(&::ncclAllGather) AllGather = nullptr;
  decltype(&::ncclCommDestroy) CommDestroy = nullptr;
  decltype(&::ncclGetErrorString) GetErrorString = nullptr;
  decltype(&::ncclGetVersion) GetVersion = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    bool all = true;
    auto bind = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      all = all && fn != nullptr;
    };
    bind(n.GetUniqueId, "ncclGetUniqueId");
    bind(n.CommInitRank, "ncclCommInitRank");
    bind(n.CommInitAll, "ncclCommInitAll");
    bind(n.CommSplit, "ncclCommSplit");
    bind(n.CommCount, "ncclCommCount");
    bind(n.CommUserRank, "ncclCommUserRank");
    bind(n.AllGather, "ncclAllGather");
    bind(n.CommDestroy, "ncclCommDestroy");
    bind(n.GetErrorString, "ncclGetErrorString");
    bind(n.GetVersion, "ncclGetVersion");
    n.ok = all;
    if (!all) n.why = "libnccl.so.2 lacks a required symbol (NCCL >= 2.18 needed)";
  });
  return n;
}

int nccl_missing(const char* where) {
  const Nccl& n = nccl();
  if (n.ok) return SDCSW_OK;
  sdcsw::set_error(std::string(where) + ": " + n.why);
  return SDCSW_ERR_CUDA;
}

int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return SDCSW_OK;
  sdcsw::set_error(std::string(where) + ": " + nccl().GetErrorString(r) +
                   (r == ncclInvalidArgument || r == ncclInvalidUsage ? "" : " (NCCL)"));
  return (r == ncclInvalidArgument || r == ncclInvalidUsage) ? SDCSW_ERR_PARAM : SDCSW_ERR_CUDA;
}

}  // namespace

extern "C" {

int sdcsw_comm_unique_id(void* id, int bytes) {
  if (id == nullptr || bytes < (int)sizeof(ncclUniqueId)) {
    sdcsw::set_error("sdcsw_comm_unique_id: need a buffer of SDCSW_COMM_ID_BYTES bytes");
    return SDCSW_ERR_PARAM;
  }
  if (int st = nccl_missing("sdcsw_comm_unique_id")) return st;
  ncclUniqueId uid;
  const int st = nccl_status(nccl().GetUniqueId(&uid), "sdcsw_comm_unique_id");
  if (st == SDCSW_OK) memcpy(id, &uid, sizeof(uid));
  return st;
}

int sdcsw_comm_create(const void* id, int bytes, int world, int rank, int device,
                      sdcsw_comm** out) {
  if (id == nullptr || out == nullptr || bytes < (int)sizeof(ncclUniqueId) || world < 1 ||
      rank < 0 || rank >= world) {
    sdcsw::set_error("sdcsw_comm_create: bad unique id, world or rank");
    return SDCSW_ERR_PARAM;
  }
  *out = nullptr;
  if (int st = nccl_missing("sdcsw_comm_create")) return st;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    sdcsw::set_error(std::string("sdcsw_comm_create: ") + cudaGetErrorString(e));
    return SDCSW_ERR_CUDA;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  sdcsw_comm* c = new sdcsw_comm;
  const int st = nccl_status(nccl().CommInitRank(&c->comm, world, uid, rank), "sdcsw_comm_create");
  if (st != SDCSW_OK) {
    delete c;
    return st;
  }
  c->world = world;
  c->rank = rank;
  c->device = device;
  *out = c;
  return SDCSW_OK;
}

int sdcsw_comm_init_all(int ndev, const int* devs, sdcsw_comm** out) {
  if (ndev < 1 || ndev > 64 || devs == nullptr || out == nullptr) {
    sdcsw::set_error("sdcsw_comm_init_all: bad device list");
    return SDCSW_ERR_PARAM;
  }
  if (int st = nccl_missing("sdcsw_comm_init_all")) return st;
  ncclComm_t comms[64];
  const int st = nccl_status(nccl().CommInitAll(comms, ndev, devs), "sdcsw_comm_init_all");
  if (st != SDCSW_OK) return st;
  for (int i = 0; i < ndev; ++i) {
    out[i] = new sdcsw_comm;
    out[i]->comm = comms[i];
    out[i]->world = ndev;
    out[i]->rank = i;
    out[i]->device = devs[i];
  }
  return SDCSW_OK;
}

int sdcsw_comm_split(sdcsw_comm* parent, int color, int key, sdcsw_comm** out) {
  if (parent == nullptr || parent->comm == nullptr || out == nullptr || color < 0) {
    sdcsw::set_error("sdcsw_comm_split: bad communicator or color");
    return SDCSW_ERR_PARAM;
  }
  *out = nullptr;
  sdcsw_comm* c = new sdcsw_comm;
  int st = nccl_status(nccl().CommSplit(parent->comm, color, key, &c->comm, nullptr), "sdcsw_comm_split");
  if (st == SDCSW_OK) st = nccl_status(nccl().CommCount(c->comm, &c->world), "sdcsw_comm_split");
  if (st == SDCSW_OK) st = nccl_status(nccl().CommUserRank(c->comm, &c->rank), "sdcsw_comm_split");
  if (st != SDCSW_OK) {
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
    return st;
  }
  c->device = parent->device;
  *out = c;
  return SDCSW_OK;
}

int sdcsw_comm_info(sdcsw_comm* c, int* world, int* rank) {
  if (c == nullptr || c->comm == nullptr) return SDCSW_ERR_STATE;
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return SDCSW_OK;
}

int sdcsw_allgather_rhs(sdcsw_comm* c, const double* send, double* recv, long long count,
                        void* stream) {
  if (c == nullptr || c->comm == nullptr) {
    sdcsw::set_error("sdcsw_allgather_rhs: destroyed communicator");
    return SDCSW_ERR_STATE;
  }
  if (count < 0 || (count > 0 && (send == nullptr || recv == nullptr))) {
    sdcsw::set_error("sdcsw_allgather_rhs: bad buffer");
    return SDCSW_ERR_PARAM;
  }
  if (count == 0) return SDCSW_OK;
  return nccl_status(nccl().AllGather(send, recv, (size_t)count, ncclDouble, c->comm,
                                   (cudaStream_t)stream),
                     "sdcsw_allgather_rhs");
}

int sdcsw_comm_destroy(sdcsw_comm* c) {
  if (c == nullptr) return SDCSW_OK;
  int st = SDCSW_OK;
  if (c->comm != nullptr) st = nccl_status(nccl().CommDestroy(c->comm), "sdcsw_comm_destroy");
  delete c;
  return st;
}

int sdcsw_nccl_version(void) {  // 0 if no NCCL can be loaded
  int v = 0;
  if (nccl().ok) nccl().GetVersion(&v);
  return v;
}

}  // extern "C"
