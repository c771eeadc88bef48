#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"

namespace mb200 {

namespace {
typedef struct { char internal[128]; } ncclUniqueId;
typedef void* ncclComm_t;
typedef int ncclResult_t;
enum { ncclUint8 = 1, ncclFloat64 = 8, ncclSum = 0 };
struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static std::once_flag once;
    static Nccl n;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.lib) break;
        }
        if (!n.lib) return;
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(n.lib, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(n.lib, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(n.lib, "ncclCommDestroy");
        n.commSplit = (decltype(n.commSplit))dlsym(n.lib, "ncclCommSplit");
        n.allGather = (decltype(n.allGather))dlsym(n.lib, "ncclAllGather");
        n.allReduce = (decltype(n.allReduce))dlsym(n.lib, "ncclAllReduce");
        n.send = (decltype(n.send))dlsym(n.lib, "ncclSend");
        n.recv = (decltype(n.recv))dlsym(n.lib, "ncclRecv");
        n.groupStart = (decltype(n.groupStart))dlsym(n.lib, "ncclGroupStart");
        n.groupEnd = (decltype(n.groupEnd))dlsym(n.lib, "ncclGroupEnd");
        n.getErrorString = (decltype(n.getErrorString))dlsym(n.lib, "ncclGetErrorString");
    });
    if (!n.lib) throw ConfigError("NCCL (libnccl.so.2) not found; multi-GPU needs NCCL");
    return n;
}
void check(ncclResult_t r, const char* what) {
    if (r != 0)
        throw CudaError(std::string("NCCL ") + what + " failed: " +
                        (nccl().getErrorString ? nccl().getErrorString(r) : "?"));
}

constexpr int kMaxLoop = 16;
struct SumSrc {
    const double* p[kMaxLoop];
};
// out[i] = sum over ranks in rank order (every rank computes the same sum)
__global__ void k_sum_ranks(SumSrc src, int world, size_t n, double* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = src.p[0][i];
        for (int r = 1; r < world; ++r) s += src.p[r][i];
        out[i] = s;
    }
}
}  // namespace

// ------------------------------------------------------------------ loopback group
struct LoopGroup {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    struct Slot {
        const void* send = nullptr;
        void* recv = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Slot> slot;
    LoopGroup* child = nullptr;  // comm_split's group (created by the first caller)
    ~LoopGroup() { delete child; }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

LoopGroup* loop_group_create(int world) {
    if (world < 1 || world > kMaxLoop) throw ConfigError("loopback group: world must be in [1, 16]");
    LoopGroup* g = new LoopGroup;
    g->world = world;
    g->slot.resize(world);
    return g;
}
void loop_group_destroy(LoopGroup* g) { delete g; }
int comm_world_of(const LoopGroup* g) { return g->world; }

struct Comm {
    int world = 1, rank = 0;
    ncclComm_t nc = nullptr;     // NCCL backend
    LoopGroup* lg = nullptr;     // loopback backend
    double* tmp = nullptr;       // loopback all-reduce staging
    size_t tmp_n = 0;
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
    check(nccl().commInitRank(&c->nc, world, id, rank), "ncclCommInitRank");
    return c;
}
Comm* comm_create_loopback(LoopGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->world) throw ConfigError("loopback communicator: bad rank");
    Comm* c = new Comm;
    c->world = g->world;
    c->rank = rank;
    c->lg = g;
    LoopGroup::Slot& s = g->slot[rank];
    if (!s.ready) {
        MB_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
        MB_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }
    return c;
}
Comm* comm_split(Comm* c) {
    if (c->nc) {
        Nccl& n = nccl();
        if (!n.commSplit) throw ConfigError("NCCL without ncclCommSplit (needs >= 2.18)");
        Comm* d = new Comm;
        d->world = c->world;
        d->rank = c->rank;
        check(n.commSplit(c->nc, 0, c->rank, &d->nc, nullptr), "ncclCommSplit");
        return d;
    }
    LoopGroup* g = c->lg;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (!g->child) g->child = loop_group_create(g->world);
    }
    return comm_create_loopback(g->child, c->rank);
}
int comm_world(const Comm* c) { return c->world; }
int comm_rank(const Comm* c) { return c->rank; }
void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->nc) nccl().commDestroy(c->nc);
    if (c->lg) {
        LoopGroup::Slot& s = c->lg->slot[c->rank];
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.done) cudaEventDestroy(s.done);
        s.ready = s.done = nullptr;
    }
    if (c->tmp) cudaFree(c->tmp);
    delete c;
}

namespace {
// loopback protocol around one collective: publish (pointers + a ready event
// on this rank's stream), barrier, wait for every rank's ready event, run
// this rank's part, record done, barrier, wait for every rank's done event
// (so no rank overwrites a buffer another rank is still reading).
template <typename Body>
void loop_collective(Comm* c, const void* send, void* recv, cudaStream_t s, Body body) {
    LoopGroup& g = *c->lg;
    LoopGroup::Slot& me = g.slot[c->rank];
    me.send = send;
    me.recv = recv;
    MB_CUDA(cudaEventRecord(me.ready, s));
    g.barrier();
    for (int q = 0; q < g.world; ++q)
        if (q != c->rank) MB_CUDA(cudaStreamWaitEvent(s, g.slot[q].ready, 0));
    body(g);
    MB_CUDA(cudaEventRecord(me.done, s));
    g.barrier();
    for (int q = 0; q < g.world; ++q)
        if (q != c->rank) MB_CUDA(cudaStreamWaitEvent(s, g.slot[q].done, 0));
}
}  // namespace

void comm_allreduce_f64(Comm* c, double* buf, size_t count, cudaStream_t s) {
    if (count == 0) return;
    if (c->nc) {
        check(nccl().allReduce(buf, buf, count, ncclFloat64, ncclSum, c->nc, s), "ncclAllReduce");
        return;
    }
    if (c->tmp_n < count) {
        if (c->tmp) cudaFree(c->tmp);
        MB_CUDA(cudaMalloc(&c->tmp, sizeof(double) * count));
        c->tmp_n = count;
    }
    loop_collective(c, buf, buf, s, [&](LoopGroup& g) {
        SumSrc src{};
        for (int q = 0; q < g.world; ++q) src.p[q] = static_cast<const double*>(g.slot[q].send);
        k_sum_ranks<<<(unsigned)std::min<size_t>((count + 255) / 256, 1024), 256, 0, s>>>(src, g.world, count, c->tmp);
        MB_LAUNCH();
    });
    // every rank has summed the unmodified buffers: now overwrite its own
    MB_CUDA(cudaMemcpyAsync(buf, c->tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
}

void comm_allgather_bytes(Comm* c, void* buf, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    uint8_t* b = static_cast<uint8_t*>(buf);
    if (c->nc) {
        check(nccl().allGather(b + (size_t)c->rank * bytes, b, bytes, ncclUint8, c->nc, s), "ncclAllGather");
        return;
    }
    loop_collective(c, buf, buf, s, [&](LoopGroup& g) {
        for (int q = 0; q < g.world; ++q)
            if (q != c->rank)
                MB_CUDA(cudaMemcpyAsync(b + (size_t)q * bytes, static_cast<const uint8_t*>(g.slot[q].send) + (size_t)q * bytes,
                                        bytes, cudaMemcpyDeviceToDevice, s));
    });
}

void comm_alltoall_bytes(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    const uint8_t* sb = static_cast<const uint8_t*>(send);
    uint8_t* rb = static_cast<uint8_t*>(recv);
    if (c->nc) {
        Nccl& n = nccl();
        check(n.groupStart(), "ncclGroupStart");
        for (int p = 0; p < c->world; ++p) {
            check(n.send(sb + (size_t)p * bytes, bytes, ncclUint8, p, c->nc, s), "ncclSend");
            check(n.recv(rb + (size_t)p * bytes, bytes, ncclUint8, p, c->nc, s), "ncclRecv");
        }
        check(n.groupEnd(), "ncclGroupEnd");
        return;
    }
    loop_collective(c, send, recv, s, [&](LoopGroup& g) {
        for (int q = 0; q < g.world; ++q)
            MB_CUDA(cudaMemcpyAsync(rb + (size_t)q * bytes, static_cast<const uint8_t*>(g.slot[q].send) + (size_t)c->rank * bytes,
                                    bytes, cudaMemcpyDeviceToDevice, s));
    });
}

}  // namespace mb200
