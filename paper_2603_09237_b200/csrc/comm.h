// Minimal NCCL binding (dlopen'd libnccl.so.2, so the library has no
// link-time NCCL dependency and single-GPU runs never touch it). Used for
// the per-minibatch all-gather of the per-cluster theta gradients (bf16
// rows), the small feature-map / b gradient all-reduces, and the tiny
// normalisation-statistics and loss all-reduces.
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
// in place: rank r's bytes_per_rank at buf + r * bytes_per_rank, gathered in rank order
void comm_allgather_bytes(Comm* c, void* buf, size_t bytes_per_rank, cudaStream_t s);
}  // namespace mb200
