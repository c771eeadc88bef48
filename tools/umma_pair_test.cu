// Feasibility / layout check of the 2-CTA tcgen05 MMA (cta_group::2):
// D[256 x N] = A[256 x K] B[N x K]^T with A rows 0-127 in CTA 0's shared
// memory and 128-255 in CTA 1's (same offsets), B split along N (columns
// [0, N/2) in CTA 0, [N/2, N) in CTA 1), each CTA's TMEM holding its 128 rows
// of D. Checked against a CPU product; then a timing loop (cycles per MMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_09237_b200/csrc tools/umma_pair_test.cu -o tools/umma_pair_test.bin
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "umma.cuh"

using namespace mb200;

constexpr int N = 256, K = 64;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            umma::smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// K-major SWIZZLE_NONE core-matrix layout, rows x K bf16: element (r, k) at
// (r/8)*(K*16) + (k/8)*128 + (r%8)*16 + (k%8)*2  (SBO = K*16, LBO = 128)
__device__ __forceinline__ int off(int r, int k) { return (r / 8) * (K * 16) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_pair(const float* A, const float* B, float* D, int reps, long long* cyc) {
    __shared__ __align__(1024) uint8_t sa[128 * K * 2];
    __shared__ __align__(1024) uint8_t sb[(N / 2) * K * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this CTA's A rows and B columns
    for (int e = threadIdx.x; e < 128 * K; e += 128) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<__nv_bfloat16*>(sa + off(r, k)) = __float2bfloat16(A[(rank * 128 + r) * K + k]);
    }
    for (int e = threadIdx.x; e < (N / 2) * K; e += 128) {
        const int n = e / K, k = e % K;
        *reinterpret_cast<__nv_bfloat16*>(sb + off(n, k)) = __float2bfloat16(B[(rank * (N / 2) + n) * K + k]);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(umma::smem_u32(&tslot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        umma::mbar_init(&bar, 1);
        umma::fence_barrier_init();
    }
    umma::fence_proxy_async();
    umma::fence_before_sync();
    cluster_sync();
    umma::fence_after_sync();
    const uint32_t tb = tslot;
    const uint32_t idesc = umma::idesc_bf16(256, N, false, false);
    const uint64_t ad = umma::smem_desc(umma::smem_u32(sa), 128, K * 16);
    const uint64_t bd = umma::smem_desc(umma::smem_u32(sb), 128, K * 16);
    long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
        const int nk = rep == 0 ? K / 16 : reps;
        if (rank == 0 && warp == 1) {
            t0 = clock64();
            if (umma::elect_one()) {
                for (int i = 0; i < nk; ++i) {
                    const int kk = i % (K / 16);
                    mma2(tb, ad + 16 * kk, bd + 16 * kk, idesc, i ? 1u : 0u);
                }
                commit2(&bar);
            }
            __syncwarp();
        }
        umma::mbar_wait(&bar, (uint32_t)rep);
        if (rank == 0 && warp == 1) t1 = clock64();
        umma::fence_after_sync();
        if (rep == 0) {  // D rows of this CTA: lane quadrant = warp
            for (int c0 = 0; c0 < N; c0 += 16) {
                float v[16];
                umma::tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c0, v);
                const int row = rank * 128 + warp * 32 + lane;
                for (int i = 0; i < 16; ++i) D[row * N + c0 + i] = v[i];
            }
        }
        umma::fence_before_sync();
        cluster_sync();
        umma::fence_after_sync();
    }
    if (rank == 0 && threadIdx.x == 32) *cyc = t1 - t0;
    umma::fence_before_sync();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

int main() {
    std::vector<float> A(256 * K), B(N * K), D(256 * N, -1.f), R(256 * N, 0.f);
    for (int i = 0; i < 256 * K; ++i) A[i] = (float)((i * 7 + 3) % 9 - 4);
    for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5 + 1) % 7 - 3);
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dD;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice);
    const int reps = 512;
    k_pair<<<2, 128>>>(dA, dB, dD, reps, dc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    long long cyc = 0;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxe = 0;
    for (int i = 0; i < 256 * N; ++i) {
        const double d = std::abs((double)D[i] - R[i]);
        maxe = d > maxe ? d : maxe;
        if (d > 1e-3 && bad++ < 5) printf("  mismatch row %d col %d: got %g want %g\n", i / N, i % N, D[i], R[i]);
    }
    printf("2-CTA M=256 N=%d K=%d: %d mismatches (max err %g); %d MMAs in %lld cycles = %.1f cycles/MMA (floor %d)\n", N, K,
           bad, maxe, reps, cyc, (double)cyc / reps, 256 * N / 512);
    return bad ? 2 : 0;
}
