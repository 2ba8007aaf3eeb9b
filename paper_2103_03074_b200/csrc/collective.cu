// collective.cu -- the multi-GPU path's one collective over NCCL:
// the sum over ranks of the partials of disjoint slice ranges.  libnccl.so.2
// is dlopen'd on first use (torch's bundled copy when torch is loaded, the
// system one otherwise), so libtnb.so itself has no NCCL dependency.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "tnb_internal.h"

namespace tnb {
namespace {

// the few NCCL entry points used (nccl.h 2.x ABI)
typedef struct { char internal[128]; } NcclUniqueId;
typedef void* NcclComm;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0 };
struct Nccl {
  int (*get_unique_id)(NcclUniqueId*) = nullptr;
  int (*comm_init_rank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
  int (*comm_destroy)(NcclComm) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { err = "libnccl.so.2 not found"; return; }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce)
    throw Error(TNB_ERR_CUDA, err.empty() ? "NCCL entry points missing" : err);
  return n;
}

void nccl_check(int r, const char* what) {
  if (r != 0) {
    const Nccl& n = nccl();
    throw Error(TNB_ERR_CUDA, std::string(what) + ": " + (n.error_string ? n.error_string(r) : "NCCL error"));
  }
}

}  // namespace

void nccl_unique_id(uint8_t* out) {
  NcclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void* nccl_comm_create(int nranks, const uint8_t* idb, int rank, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(TNB_ERR_ARG, "bad NCCL rank / size");
  TNB_CUDA(cudaSetDevice(device));
  NcclUniqueId id;
  std::memcpy(id.internal, idb, 128);
  NcclComm c = nullptr;
  nccl_check(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_comm_destroy(void* c) {
  if (c) nccl_check(nccl().comm_destroy(c), "ncclCommDestroy");
}

void nccl_allreduce_sum(void* c, int precision, void* buf, int64_t n, void* stream) {
  if (!c || !buf || n < 0) throw Error(TNB_ERR_ARG, "bad allreduce arguments");
  const int dt = precision == TNB_SINGLE ? kNcclFloat32 : kNcclFloat64;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  nccl_check(nccl().all_reduce(buf, buf, (size_t)(2 * n), dt, kNcclSum, c, s), "ncclAllReduce");
  TNB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace tnb
