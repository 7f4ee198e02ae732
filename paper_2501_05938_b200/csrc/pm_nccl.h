// pm_nccl.h -- NCCL loaded at run time (dlopen), for the C-ABI collective
// entry pm_solve_dist_nccl_* (include/pm_tridiag.h).  The library does not
// link NCCL: a process that never calls these never loads it, and a process
// that already has NCCL loaded (e.g. PyTorch's bundled libnccl.so.2) shares
// that one copy, because dlopen of the soname returns the loaded object.
#pragma once

#include <cstddef>
#include <string>

namespace pmnccl {

constexpr int kUniqueIdBytes = 128;  // sizeof(ncclUniqueId)

// Loads NCCL once (PM_NCCL_LIB, else libnccl.so.2, else libnccl.so).
// Returns false and sets `why` when it cannot be loaded.
bool load(std::string* why);
int version();  // NCCL_VERSION_CODE of the loaded library, -1 if absent

// Thin calls; return 0 on ncclSuccess, else the ncclResult_t, with the
// library's message in `why`.
int get_unique_id(void* id_out, std::string* why);
int comm_init_rank(void** comm_out, int nranks, const void* id, int rank, std::string* why);
int comm_destroy(void* comm, std::string* why);
int comm_count(void* comm, int* count, std::string* why);
int comm_user_rank(void* comm, int* rank, std::string* why);
// ncclAllGather of `count` elements of FP64 (f64 = true) or FP32 per rank.
int all_gather(const void* send, void* recv, size_t count, bool f64, void* comm, void* stream,
               std::string* why);

}  // namespace pmnccl
