// comm.cu — the library's own NCCL communicator for the view-parallel exchange.
//
// libnccl is bound at run time (dlopen), so the library has no link-time NCCL dependency and
// shares the NCCL already loaded into a process (e.g. torch's bundled libnccl.so.2, found with
// RTLD_NOLOAD) instead of loading a second copy next to it.  Only the handful of entry points the
// exchange uses are resolved; the types come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "internal.h"

namespace splat_b200 {

namespace {

struct NcclApi {
    bool loaded = false;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

NcclApi g_nccl;

bool load_nccl(std::string* err) {
    if (g_nccl.loaded) return true;
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch's NCCL)
        if (h) break;
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        *err = std::string("NCCL not found: ") + dlerror();
        return false;
    }
#define SPLAT_NCCL_SYM(field, name)                                      \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) {                                                 \
        *err = std::string("NCCL symbol missing: ") + name;              \
        return false;                                                    \
    }
    SPLAT_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
    SPLAT_NCCL_SYM(init_rank, "ncclCommInitRank");
    SPLAT_NCCL_SYM(destroy, "ncclCommDestroy");
    SPLAT_NCCL_SYM(reduce_scatter, "ncclReduceScatter");
    SPLAT_NCCL_SYM(all_gather, "ncclAllGather");
    SPLAT_NCCL_SYM(all_reduce, "ncclAllReduce");
    SPLAT_NCCL_SYM(error_string, "ncclGetErrorString");
#undef SPLAT_NCCL_SYM
    g_nccl.loaded = true;
    return true;
}

int nccl_status(ncclResult_t r, const char* where, std::string* err) {
    if (r == ncclSuccess) return 0;
    *err = std::string(where) + ": " + g_nccl.error_string(r);
    return -1;
}

}  // namespace

struct Comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
};

int comm_unique_id(void* id_out, std::string* err) {
    if (!load_nccl(err)) return -1;
    ncclUniqueId id;
    if (nccl_status(g_nccl.get_unique_id(&id), "ncclGetUniqueId", err)) return -1;
    std::memcpy(id_out, &id, sizeof(id));
    return 0;
}

Comm* comm_create(int nranks, int rank, const void* id_in, std::string* err) {
    if (!load_nccl(err)) return nullptr;
    ncclUniqueId id;
    std::memcpy(&id, id_in, sizeof(id));
    Comm* c = new Comm;
    c->nranks = nranks;
    c->rank = rank;
    if (nccl_status(g_nccl.init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank", err)) {
        delete c;
        return nullptr;
    }
    return c;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->comm) g_nccl.destroy(c->comm);
    delete c;
}

int comm_ranks(const Comm* c) { return c ? c->nranks : 1; }
int comm_rank(const Comm* c) { return c ? c->rank : 0; }

int comm_reduce_scatter(Comm* c, const float* send, float* recv, size_t recv_count, cudaStream_t s, std::string* err) {
    return nccl_status(g_nccl.reduce_scatter(send, recv, recv_count, ncclFloat32, ncclSum, c->comm, s),
                       "ncclReduceScatter", err);
}

int comm_all_gather(Comm* c, const float* send, float* recv, size_t send_count, cudaStream_t s, std::string* err) {
    return nccl_status(g_nccl.all_gather(send, recv, send_count, ncclFloat32, c->comm, s), "ncclAllGather", err);
}

int comm_all_reduce(Comm* c, const void* send, void* recv, size_t count, int dtype, int op, cudaStream_t s,
                    std::string* err) {
    return nccl_status(g_nccl.all_reduce(send, recv, count, static_cast<ncclDataType_t>(dtype),
                                         static_cast<ncclRedOp_t>(op), c->comm, s),
                       "ncclAllReduce", err);
}

}  // namespace splat_b200
