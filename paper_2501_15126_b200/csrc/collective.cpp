// collective.cpp -- the path's one exchange step: an NCCL
// all-gather of every rank's 8/16-byte unscaled partial, issued by libperm on
// the plan's stream, followed by the fixed-order fold kernel.  Multi-GPU is
// future work in the paper.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): when torch has
// already loaded its NCCL, that same library instance is returned (matching
// soname), so communicators created through it and through libperm are the
// same kind; otherwise the system libnccl is used.  Only the five entry points
// below are needed, so no NCCL header or link-time dependency is required.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "perm.h"

namespace {

typedef int nccl_result;  // ncclResult_t; 0 = ncclSuccess
struct nccl_uid { char internal[128]; };  // ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128)
constexpr int kNcclUint8 = 1;             // ncclDataType_t ncclUint8

struct Nccl {
  void* h = nullptr;
  nccl_result (*get_unique_id)(nccl_uid*) = nullptr;
  nccl_result (*comm_init_rank)(void**, int, nccl_uid, int) = nullptr;
  nccl_result (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  nccl_result (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  std::string err;
};

Nccl& nccl() {
  static Nccl N;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      N.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
    N.h = h;
    N.get_unique_id = (nccl_result(*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
    N.comm_init_rank = (nccl_result(*)(void**, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
    N.all_gather = (nccl_result(*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(h, "ncclAllGather");
    N.comm_destroy = (nccl_result(*)(void*))dlsym(h, "ncclCommDestroy");
    N.error_string = (const char* (*)(nccl_result))dlsym(h, "ncclGetErrorString");
    if (!N.get_unique_id || !N.comm_init_rank || !N.all_gather || !N.comm_destroy) {
      N.err = "libnccl.so.2 lacks an expected entry point";
      N.h = nullptr;
    }
  });
  return N;
}

std::string nerr(nccl_result r) {
  Nccl& N = nccl();
  return N.error_string ? N.error_string(r) : ("ncclResult " + std::to_string(r));
}

}  // namespace

// internal (runtime.cpp): in-place all-gather of `bytes` per rank on `st`
// (rank r's contribution at recv + r * bytes).  Returns a perm_status; msg set
// on error.
int libperm_allgather(void* comm, void* recv, size_t bytes, int rank, cudaStream_t st, std::string& msg) {
  Nccl& N = nccl();
  if (!N.h) { msg = N.err; return PERM_ENCCL; }
  const nccl_result r = N.all_gather(static_cast<char*>(recv) + (size_t)rank * bytes, recv, bytes, kNcclUint8,
                                     comm, st);
  if (r != 0) { msg = "ncclAllGather: " + nerr(r); return PERM_ENCCL; }
  return PERM_OK;
}

int libperm_nccl_available(std::string& msg) {
  Nccl& N = nccl();
  if (!N.h) msg = N.err;
  return N.h != nullptr;
}

int libperm_comm_unique_id(void* id128, std::string& msg) {
  Nccl& N = nccl();
  if (!N.h) { msg = N.err; return PERM_ENCCL; }
  nccl_uid u;
  const nccl_result r = N.get_unique_id(&u);
  if (r != 0) { msg = "ncclGetUniqueId: " + nerr(r); return PERM_ENCCL; }
  std::memcpy(id128, u.internal, 128);
  return PERM_OK;
}

int libperm_comm_init(int world, int rank, const void* id128, int device, void** comm, std::string& msg) {
  Nccl& N = nccl();
  if (!N.h) { msg = N.err; return PERM_ENCCL; }
  if (cudaSetDevice(device) != cudaSuccess) { msg = "cudaSetDevice failed"; return PERM_ECUDA; }
  nccl_uid u;
  std::memcpy(u.internal, id128, 128);
  const nccl_result r = N.comm_init_rank(comm, world, u, rank);
  if (r != 0) { msg = "ncclCommInitRank: " + nerr(r); return PERM_ENCCL; }
  return PERM_OK;
}

int libperm_comm_destroy(void* comm, std::string& msg) {
  Nccl& N = nccl();
  if (!N.h) { msg = N.err; return PERM_ENCCL; }
  if (!comm) return PERM_OK;
  const nccl_result r = N.comm_destroy(comm);
  if (r != 0) { msg = "ncclCommDestroy: " + nerr(r); return PERM_ENCCL; }
  return PERM_OK;
}
