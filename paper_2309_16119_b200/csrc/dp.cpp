// dp.cpp — the data-parallel exchange of SURVEY §8(e) behind the C ABI
// (include/mlra.h, mlra_dp_* / mlra_allreduce_lora_grads): one sum all-reduce
// of the flat fp32 LoRA-gradient bucket per step over NCCL (NVLink / NVSwitch
// on the box), for C++ callers that do not run torch.distributed.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): in a process that
// already loaded one (e.g. torch's) the same library is reused, and libmlra has
// no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/mlra.h"

namespace mlra {
mlra_status set_error(mlra_status st, const std::string& msg);
}  // namespace mlra

namespace {

// The few NCCL entry points used, with their public C signatures (nccl.h).
typedef struct { char internal[128]; } NcclUniqueId;
typedef void* NcclComm;
typedef int (*GetUniqueIdFn)(NcclUniqueId*);
typedef int (*CommInitRankFn)(NcclComm*, int, NcclUniqueId, int);
typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*CommDestroyFn)(NcclComm);
typedef const char* (*GetErrorStringFn)(int);
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclSum = 0;      // ncclSum

struct Nccl {
  bool ok = false;
  std::string why;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  AllReduceFn all_reduce = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  GetErrorStringFn error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      n.why = e ? e : "libnccl.so.2 not found";
      return;
    }
    n.get_unique_id = reinterpret_cast<GetUniqueIdFn>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<CommInitRankFn>(dlsym(h, "ncclCommInitRank"));
    n.all_reduce = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
    n.comm_destroy = reinterpret_cast<CommDestroyFn>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<GetErrorStringFn>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy;
    if (!n.ok) n.why = "libnccl.so.2 lacks the expected symbols";
  });
  return n;
}

mlra_status nccl_fail(int rc, const char* what) {
  const Nccl& n = nccl();
  return mlra::set_error(MLRA_ERR_CUDA, std::string(what) + ": NCCL error " + std::to_string(rc) +
                                            (n.error_string ? std::string(" (") + n.error_string(rc) + ")"
                                                            : std::string()));
}

}  // namespace

struct mlra_dp {
  NcclComm comm = nullptr;
  int rank = 0, world = 1;
};

extern "C" {

mlra_status mlra_dp_unique_id(void* id_out) {
  if (!id_out) return mlra::set_error(MLRA_ERR_CONTRACT, "dp: null id buffer");
  const Nccl& n = nccl();
  if (!n.ok) return mlra::set_error(MLRA_ERR_UNSUPPORTED, "dp: " + n.why);
  NcclUniqueId id;
  if (int rc = n.get_unique_id(&id)) return nccl_fail(rc, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return MLRA_OK;
}

mlra_status mlra_dp_init(int rank, int world, const void* id, mlra_dp** out) {
  if (!out || !id) return mlra::set_error(MLRA_ERR_CONTRACT, "dp: null argument");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world)
    return mlra::set_error(MLRA_ERR_CONFIG, "dp: rank " + std::to_string(rank) +
                                                " out of [0, " + std::to_string(world) + ")");
  const Nccl& n = nccl();
  if (!n.ok) return mlra::set_error(MLRA_ERR_UNSUPPORTED, "dp: " + n.why);
  NcclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* d = new mlra_dp();
  d->rank = rank;
  d->world = world;
  if (int rc = n.comm_init_rank(&d->comm, world, uid, rank)) {
    delete d;
    return nccl_fail(rc, "ncclCommInitRank");
  }
  *out = d;
  return MLRA_OK;
}

mlra_status mlra_allreduce_lora_grads(mlra_dp* dp, float* bucket, uint64_t count, void* stream) {
  if (!dp) return mlra::set_error(MLRA_ERR_CONTRACT, "dp: null communicator");
  if (count == 0) return MLRA_OK;
  if (!bucket) return mlra::set_error(MLRA_ERR_CONTRACT, "dp: null gradient bucket");
  if (int rc = nccl().all_reduce(bucket, bucket, count, kNcclFloat32, kNcclSum, dp->comm,
                                 static_cast<cudaStream_t>(stream)))
    return nccl_fail(rc, "ncclAllReduce");
  return MLRA_OK;
}

void mlra_dp_destroy(mlra_dp* dp) {
  if (!dp) return;
  if (dp->comm && nccl().ok) nccl().comm_destroy(dp->comm);
  delete dp;
}

}  // extern "C"
