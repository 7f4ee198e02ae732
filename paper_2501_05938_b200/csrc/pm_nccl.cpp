// pm_nccl.cpp -- see pm_nccl.h.  The NCCL C API (nccl.h, 2.x) is declared here
// by hand: the handful of entry points the row-sharded solve needs.
#include "pm_nccl.h"

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace pmnccl {
namespace {

struct UniqueId {
  char internal[kUniqueIdBytes];
};
// ncclDataType_t values of nccl.h 2.x
constexpr int kNcclFloat32 = 7;
constexpr int kNcclFloat64 = 8;

using GetVersionFn = int (*)(int*);
using GetUniqueIdFn = int (*)(UniqueId*);
using CommInitRankFn = int (*)(void**, int, UniqueId, int);
using CommDestroyFn = int (*)(void*);
using CommCountFn = int (*)(const void*, int*);
using CommUserRankFn = int (*)(const void*, int*);
using AllGatherFn = int (*)(const void*, void*, size_t, int, void*, void*);
using GetErrorStringFn = const char* (*)(int);

struct Api {
  void* lib = nullptr;
  std::string error;
  int version = -1;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  CommCountFn comm_count = nullptr;
  CommUserRankFn comm_user_rank = nullptr;
  AllGatherFn all_gather = nullptr;
  GetErrorStringFn error_string = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("PM_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm || !*nm) continue;
      a.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
      if (a.lib) break;
    }
    if (!a.lib) {
      const char* e = dlerror();
      a.error = std::string("cannot load NCCL (PM_NCCL_LIB / libnccl.so.2): ") + (e ? e : "");
      return;
    }
    auto sym = [&](const char* s) { return dlsym(a.lib, s); };
    a.get_unique_id = reinterpret_cast<GetUniqueIdFn>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<CommInitRankFn>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<CommDestroyFn>(sym("ncclCommDestroy"));
    a.comm_count = reinterpret_cast<CommCountFn>(sym("ncclCommCount"));
    a.comm_user_rank = reinterpret_cast<CommUserRankFn>(sym("ncclCommUserRank"));
    a.all_gather = reinterpret_cast<AllGatherFn>(sym("ncclAllGather"));
    a.error_string = reinterpret_cast<GetErrorStringFn>(sym("ncclGetErrorString"));
    auto gv = reinterpret_cast<GetVersionFn>(sym("ncclGetVersion"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.comm_count || !a.comm_user_rank ||
        !a.all_gather || !gv) {
      a.error = "the loaded NCCL lacks a required symbol";
      dlclose(a.lib);
      a.lib = nullptr;
      return;
    }
    int v = 0;
    a.version = gv(&v) == 0 ? v : -1;
  });
  return a;
}

int result(int r, const char* what, std::string* why) {
  if (r != 0 && why) {
    const char* s = api().error_string ? api().error_string(r) : "";
    *why = std::string(what) + " failed: " + (s ? s : "") + " (ncclResult " + std::to_string(r) + ")";
  }
  return r;
}

bool ready(std::string* why) {
  if (api().lib) return true;
  if (why) *why = api().error;
  return false;
}

}  // namespace

bool load(std::string* why) { return ready(why); }
int version() { return api().lib ? api().version : -1; }

int get_unique_id(void* id_out, std::string* why) {
  if (!ready(why)) return -1;
  UniqueId id;
  const int r = api().get_unique_id(&id);
  if (r == 0) std::memcpy(id_out, id.internal, kUniqueIdBytes);
  return result(r, "ncclGetUniqueId", why);
}

int comm_init_rank(void** comm_out, int nranks, const void* id, int rank, std::string* why) {
  if (!ready(why)) return -1;
  UniqueId u;
  std::memcpy(u.internal, id, kUniqueIdBytes);
  return result(api().comm_init_rank(comm_out, nranks, u, rank), "ncclCommInitRank", why);
}

int comm_destroy(void* comm, std::string* why) {
  if (!ready(why)) return -1;
  return result(api().comm_destroy(comm), "ncclCommDestroy", why);
}

int comm_count(void* comm, int* count, std::string* why) {
  if (!ready(why)) return -1;
  return result(api().comm_count(comm, count), "ncclCommCount", why);
}

int comm_user_rank(void* comm, int* rank, std::string* why) {
  if (!ready(why)) return -1;
  return result(api().comm_user_rank(comm, rank), "ncclCommUserRank", why);
}

int all_gather(const void* send, void* recv, size_t count, bool f64, void* comm, void* stream,
               std::string* why) {
  if (!ready(why)) return -1;
  return result(api().all_gather(send, recv, count, f64 ? kNcclFloat64 : kNcclFloat32, comm, stream),
                "ncclAllGather", why);
}

}  // namespace pmnccl
