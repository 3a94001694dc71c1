// comm.cpp -- NCCL binding for the Ulysses all-to-all (rows a2 / a6).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") -- the NCCL
// 2.28 that torch already loaded in the process, or TM_NCCL_LIB -- so that a
// single-GPU ctx never needs it.  One communicator per tm_ctx, created from
// a 128-byte unique id the harness broadcasts over torch.distributed.
#include "comm.h"

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace tmk {
namespace {

using ncclComm_t = void*;
using ncclResult_t = int;
struct ncclUniqueId { char internal[128]; };

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AlltoAll)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {getenv("TM_NCCL_LIB"), "libnccl.so.2", "libnccl.so", TM_NCCL_DEFAULT};
        for (const char* nm : names) {
            if (!nm || !*nm) continue;
            n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
#define SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.h, "nccl" #f))
        SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(CommGetAsyncError);
        SYM(AlltoAll); SYM(Send); SYM(Recv); SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
    });
    return (n.h && n.GetUniqueId && n.CommInitRank && n.Send && n.Recv) ? &n : nullptr;
}

thread_local char g_msg[256];

const char* err(ncclResult_t r) {
    Nccl* n = nccl();
    snprintf(g_msg, sizeof g_msg, "NCCL error %d: %s", r,
             (n && n->GetErrorString) ? n->GetErrorString(r) : "?");
    return g_msg;
}

}  // namespace

const char* comm_unique_id(uint8_t id[128]) {
    Nccl* n = nccl();
    if (!n) return "NCCL library not found (dlopen libnccl.so.2 failed)";
    ncclUniqueId u;
    ncclResult_t r = n->GetUniqueId(&u);
    if (r) return err(r);
    memcpy(id, u.internal, 128);
    return nullptr;
}

const char* comm_init(void** comm, int world, int rank, const uint8_t id[128]) {
    Nccl* n = nccl();
    if (!n) return "NCCL library not found (dlopen libnccl.so.2 failed)";
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclResult_t r = n->CommInitRank(comm, world, u, rank);
    return r ? err(r) : nullptr;
}

void comm_destroy(void* comm) {
    Nccl* n = nccl();
    if (n && comm && n->CommDestroy) n->CommDestroy(comm);
}

const char* comm_async_error(void* comm) {
    Nccl* n = nccl();
    if (!n || !comm || !n->CommGetAsyncError) return nullptr;
    ncclResult_t st = 0;
    const ncclResult_t r = n->CommGetAsyncError(comm, &st);
    if (r) return err(r);
    return st ? err(st) : nullptr;
}

// Block p of `send` (count_bytes bytes) goes to rank p; block q of `recv`
// comes from rank q.  ncclAlltoAll when the library has it, else grouped
// send/recv (same semantics, nccl.h:460 / :507 / :526).
const char* comm_alltoall(void* comm, const void* send, void* recv, size_t count_bytes, int world,
                          cudaStream_t s) {
    Nccl* n = nccl();
    if (!n) return "NCCL library not found";
    const int kInt8 = 0;
    ncclResult_t r;
    if (n->AlltoAll) {
        r = n->AlltoAll(send, recv, count_bytes, kInt8, comm, s);
        return r ? err(r) : nullptr;
    }
    r = n->GroupStart();
    for (int p = 0; p < world && !r; ++p) {
        r = n->Send(static_cast<const char*>(send) + p * count_bytes, count_bytes, kInt8, p, comm, s);
        if (!r) r = n->Recv(static_cast<char*>(recv) + p * count_bytes, count_bytes, kInt8, p, comm, s);
    }
    ncclResult_t r2 = n->GroupEnd();
    if (!r) r = r2;
    return r ? err(r) : nullptr;
}

}  // namespace tmk
