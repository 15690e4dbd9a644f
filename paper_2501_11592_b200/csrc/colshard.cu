// colshard.cu — one very large dictionary sharded by columns over GPUs
// (north star "Multi-GPU partitioning").
//
// Rank r of W owns atoms [r n/W, (r+1) n/W) for the correlation GEMM and
// learns signals [r B/W, (r+1) B/W); every rank keeps the whole dictionary for
// the support gathers (256 MB fp32 at config 3).  Per outer iteration:
//   K1 on the local atom shard for all B residuals -> per (signal, tile)
//   candidate records (Cand: top-2 atoms + third value);  ncclAllGather of
//   those (B x tiles x 32 bytes: ~0.5 MB at config 3, W = 8);  the selection rule then runs on the
//   owner rank over the complete candidate table exactly as on one GPU (the
//   per-signal (max, index) reduction plus the top-2 gap that decides whether
//   the fp64 rescan is needed);  learning on the owner;  ncclAllGather of the
//   new residual rows (tf32 hi/lo) for the next K1;  ncclAllReduce(sum) of the
//   active-signal count.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, so the copy torch has
// already loaded is reused) and only column-sharded contexts touch it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "clomp_internal.cuh"

namespace clb {

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.handle = h;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
  });
  return api;
}

// cand[b][r*ntl + tl] <- gathered[r][b][tl], atoms shifted to global numbers.
__global__ void k_cand_exchange(const Cand* __restrict__ g, Cand* __restrict__ cand, int64_t B,
                                int64_t ntl, int world, int64_t atoms_per_rank) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)world * B * ntl;
  if (e >= total) return;
  const int64_t r = e / (B * ntl), rem = e % (B * ntl), b = rem / ntl, tl = rem % ntl;
  Cand c = g[e];
  const int32_t sh = (int32_t)(r * atoms_per_rank);
  if (c.i1 >= 0 && c.i1 != 0x7fffffff) c.i1 += sh;
  if (c.i2 >= 0 && c.i2 != 0x7fffffff) c.i2 += sh;
  cand[b * (world * ntl) + r * ntl + tl] = c;
}

}  // namespace

bool nccl_available() {
  NcclApi& a = nccl();
  return a.getUniqueId && a.commInitRank && a.allGather && a.allReduce;
}

int nccl_unique_id(void* out) {
  NcclApi& a = nccl();
  if (!a.getUniqueId) return 1;
  ncclUniqueId id;
  if (a.getUniqueId(&id) != ncclSuccess) return 1;
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

void* nccl_comm_init(int world, int rank, const void* id, std::string* err) {
  NcclApi& a = nccl();
  if (!a.commInitRank) {
    *err = "libnccl.so.2 not loadable";
    return nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = a.commInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") + (a.errorString ? a.errorString(r) : "error");
    return nullptr;
  }
  return comm;
}

void nccl_comm_destroy(void* comm) {
  NcclApi& a = nccl();
  if (comm && a.commDestroy) a.commDestroy(static_cast<ncclComm_t>(comm));
}

// In-place all-gather of `count_per_rank` elements (rank r's slice at r*count).
bool nccl_allgather_inplace(void* comm, void* buf, size_t count_per_rank, int bytes_per_elem,
                            int rank, cudaStream_t s) {
  NcclApi& a = nccl();
  const ncclDataType_t t =
      bytes_per_elem == 8 ? ncclFloat64 : (bytes_per_elem == 4 ? ncclInt32 : ncclUint8);
  char* base = static_cast<char*>(buf);
  return a.allGather(base + (size_t)rank * count_per_rank * bytes_per_elem, buf, count_per_rank,
                     t, static_cast<ncclComm_t>(comm), s) == ncclSuccess;
}

bool nccl_allgather(void* comm, const void* send, void* recv, size_t count, int bytes_per_elem,
                    cudaStream_t s) {
  NcclApi& a = nccl();
  ncclDataType_t t = bytes_per_elem == 8 ? ncclFloat64 : (bytes_per_elem == 4 ? ncclInt32 : ncclUint8);
  return a.allGather(send, recv, count, t, static_cast<ncclComm_t>(comm), s) == ncclSuccess;
}

bool nccl_allreduce_sum_i32(void* comm, int32_t* buf, size_t count, cudaStream_t s) {
  NcclApi& a = nccl();
  return a.allReduce(buf, buf, count, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm), s) ==
         ncclSuccess;
}

void launch_cand_exchange(const Cand* g, Cand* cand, int64_t B, int64_t ntl, int world,
                          int64_t atoms_per_rank, cudaStream_t s) {
  const int64_t total = (int64_t)world * B * ntl;
  k_cand_exchange<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(g, cand, B, ntl, world,
                                                                   atoms_per_rank);
}

}  // namespace clb
