// Tiled bf16 "image" storage shared by every tensor-core operand of the
// update (activations, gradients, generated weights, hypernet M, gtheta).
//
// A logical matrix X[R][C] is stored as 128 x 128 chunks (32 KB, contiguous)
// of 8 x 16 B UMMA core matrices:
//   chunk (rt, ct) at ((rt * CT) + ct) * 32768,  CT = ceil(C / 128)
//   element (r, c) within the chunk at
//       ((r % 128) / 8) * 2048 + ((c % 128) / 8) * 128 + (r % 8) * 16 + (c % 8) * 2
// The SAME chunk is a valid tcgen05 operand in both orientations:
//   view 0 (MMA row = r, K = c): K-major,  SBO = 2048, LBO = 128,  K-step 16 -> +256 B
//   view 1 (MMA row = c, K = r): MN-major, SBO = 128,  LBO = 2048, K-step 16 -> +4096 B
// so forward (X W^T), data-gradient (G W) and weight-gradient (G^T X)
// GEMMs all read the same buffers, one bulk copy per chunk. Padding (to 128
// in both dims) is zero-filled once at allocation and never written.
#pragma once
#include <stdint.h>

namespace mb200 {

struct Img {
    uint8_t* p = nullptr;
    int R = 0, C = 0;  // logical extent
    long gs = 0;       // byte stride between per-group images
};

__host__ __device__ __forceinline__ int img_ct(int C) { return (C + 127) >> 7; }
__host__ __device__ __forceinline__ int img_rt(int R) { return (R + 127) >> 7; }
__host__ __device__ __forceinline__ long img_bytes(int R, int C) { return (long)img_rt(R) * img_ct(C) * 32768; }
__host__ __device__ __forceinline__ long img_off(long r, long c, int CT) {
    return ((r >> 7) * CT + (c >> 7)) * 32768 + ((r & 127) >> 3) * 2048 + ((c & 127) >> 3) * 128 + (r & 7) * 16 +
           (c & 7) * 2;
}

}  // namespace mb200
