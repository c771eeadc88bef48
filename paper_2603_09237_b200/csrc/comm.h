// Minimal NCCL binding (dlopen'd libnccl.so.2, so the library has no
// link-time NCCL dependency and single-GPU runs never touch it). Used for
// the per-minibatch hypernetwork-gradient all-reduce (each rank's partial
// sums over its own clusters) and the tiny normalisation-statistics and
// loss all-reduces.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace mb200 {
struct Comm;
int comm_unique_id(void* out128);  // 0 ok
Comm* comm_create(int world, int rank, const void* id128);
void comm_destroy(Comm* c);
void comm_allreduce_f32(Comm* c, float* buf, size_t count, cudaStream_t s);   // sum, in place
void comm_allreduce_f64(Comm* c, double* buf, size_t count, cudaStream_t s);  // sum, in place
}  // namespace mb200
