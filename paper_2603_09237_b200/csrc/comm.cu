#include <dlfcn.h>

#include <string>

#include "comm.h"
#include "common.cuh"

namespace mb200 {

namespace {
typedef struct { char internal[128]; } ncclUniqueId;
typedef void* ncclComm_t;
typedef int ncclResult_t;
enum { ncclUint8 = 1, ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0 };
struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n;
    if (!n.lib) {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.lib) break;
        }
        if (!n.lib) throw ConfigError("NCCL (libnccl.so.2) not found; multi-GPU needs NCCL");
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(n.lib, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(n.lib, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(n.lib, "ncclCommDestroy");
        n.allGather = (decltype(n.allGather))dlsym(n.lib, "ncclAllGather");
        n.allReduce = (decltype(n.allReduce))dlsym(n.lib, "ncclAllReduce");
        n.getErrorString = (decltype(n.getErrorString))dlsym(n.lib, "ncclGetErrorString");
    }
    return n;
}
void check(ncclResult_t r, const char* what) {
    if (r != 0)
        throw CudaError(std::string("NCCL ") + what + " failed: " +
                        (nccl().getErrorString ? nccl().getErrorString(r) : "?"));
}
}  // namespace

struct Comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
};

int comm_unique_id(void* out) {
    ncclUniqueId id;
    check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    memcpy(out, &id, sizeof(id));
    return 0;
}
Comm* comm_create(int world, int rank, const void* id128) {
    if (!id128) throw ConfigError("multi-GPU trainer needs an NCCL unique id");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    Comm* c = new Comm;
    c->world = world;
    c->rank = rank;
    check(nccl().commInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    return c;
}
void comm_destroy(Comm* c) {
    if (c && c->comm) nccl().commDestroy(c->comm);
    delete c;
}
void comm_allreduce_f32(Comm* c, float* buf, size_t count, cudaStream_t s) {
    check(nccl().allReduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, s), "ncclAllReduce");
}
void comm_allreduce_f64(Comm* c, double* buf, size_t count, cudaStream_t s) {
    check(nccl().allReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, s), "ncclAllReduce");
}
void comm_allgather_bytes(Comm* c, void* buf, size_t bytes, cudaStream_t s) {
    uint8_t* b = static_cast<uint8_t*>(buf);
    check(nccl().allGather(b + (size_t)c->rank * bytes, b, bytes, ncclUint8, c->comm, s), "ncclAllGather");
}

}  // namespace mb200
