// Communicator of one rank of the sharded training step.
//
// Two backends behind one interface:
//  * NCCL (dlopen'd libnccl.so.2, so the library has no link-time NCCL
//    dependency and single-GPU runs never touch it): one process per GPU.
//  * Loopback: W ranks as W host threads of one process on ONE device. The
//    collectives are device-to-device copies / a fixed-order sum kernel,
//    ordered with CUDA events and a host barrier (no kernel ever waits on
//    another rank's kernel, so nothing spins). It exists to run the sharded
//    data plane at W = 2, 4, ... on a single GPU in tests, where it must
//    reproduce the W = 1 result bit for bit.
//
// Every collective is issued by all ranks of a communicator in the same
// order on one stream per communicator (the trainer keeps one communicator
// per update chain, so the actor and critic exchanges overlap).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace mb200 {
struct Comm;
struct LoopGroup;  // shared state of a loopback group (W ranks, one device)

int comm_unique_id(void* out128);  // 0 ok
Comm* comm_create(int world, int rank, const void* id128);  // NCCL
Comm* comm_create_loopback(LoopGroup* g, int rank);
LoopGroup* loop_group_create(int world);
void loop_group_destroy(LoopGroup* g);
int comm_world_of(const LoopGroup* g);
// a second communicator over the same ranks (collective: every rank calls it)
Comm* comm_split(Comm* c);
int comm_world(const Comm* c);
int comm_rank(const Comm* c);
void comm_destroy(Comm* c);

void comm_allreduce_f64(Comm* c, double* buf, size_t count, cudaStream_t s);  // sum, in place
// in place: rank r's bytes_per_rank at buf + r * bytes_per_rank, gathered in rank order
void comm_allgather_bytes(Comm* c, void* buf, size_t bytes_per_rank, cudaStream_t s);
// send + p * bytes_per_peer goes to rank p; recv + q * bytes_per_peer comes from rank q
void comm_alltoall_bytes(Comm* c, const void* send, void* recv, size_t bytes_per_peer, cudaStream_t s);
}  // namespace mb200
