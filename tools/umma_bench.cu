// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1) issue-to-completion
// cycles per instruction for the operand layouts the rollout and the GEMMs
// use. One CTA per SM issues NI back-to-back MMAs on resident SMEM operands
// (contents irrelevant), commits, waits; reports cycles / MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_09237_b200/csrc tools/umma_bench.cu -o /tmp/umma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "umma.cuh"

using namespace mb200;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t swz) {
    uint64_t d = umma::smem_desc(saddr, lbo, sbo);
    d |= (uint64_t)swz << 61;
    return d;
}

struct Cfg {
    int M, N, a_mn, b_mn, swz, background;  // background: 8 warps of epilogue-like work (tcgen05.ld, tanh, STS)
    int chunk;  // > 0: the rollout's issue pattern, `chunk` MMAs then a commit (+ a ready-barrier wait and fence)
    int parts = 7;  // chunk mode: 1 ready-barrier wait, 2 tcgen05.fence::after_thread_sync, 4 commit per chunk,
                    // 8: the whole loop on lane 0 (no per-chunk warp reconvergence)
                    // 16: the whole loop inside one elect.sync region
                    // 32: per chunk elect, compile-time chunk of 4 MMAs (fully unrolled)
};

__global__ void k_bench(Cfg c, int NI, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, ebar[4], rbar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) umma::tmem_alloc(&tslot, 512);
    if (threadIdx.x == 32) {
        umma::mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) umma::mbar_init(&ebar[i], 1);
        umma::mbar_init(&rbar, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = tslot;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (warp >= 4 && c.background) {  // epilogue-like load on the other warps until the MMA warp is done
        uint8_t* sb = smem + 131072 + (warp - 4) * 2048;
        float acc = 0.f;
        while (!stop) {
            uint32_t r[16];
            umma::tmem_ld16_async(tb + 256 + ((uint32_t)((warp & 3) * 32) << 16), r);
            umma::tmem_wait_ld();
            float f[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = umma::tanh_approx(__uint_as_float(r[i]) + acc);
            uint4 q;
            q.x = umma::pack_bf16(f[0], f[1]); q.y = umma::pack_bf16(f[2], f[3]);
            q.z = umma::pack_bf16(f[4], f[5]); q.w = umma::pack_bf16(f[6], f[7]);
            *reinterpret_cast<uint4*>(sb + (threadIdx.x & 31) * 16) = q;
            acc += f[15] * 1e-9f;
        }
        if (acc == 12345.f) out[1] = 1;
    }
    if (warp == 1) {
        const uint32_t a0 = umma::smem_u32(smem), b0 = a0 + 65536;
        // SWIZZLE_NONE: interleaved core matrices (LBO 128 between K blocks, SBO 1024 between 8-row groups)
        // SWIZZLE_128B K-major: 8-row x 128 B atoms, SBO 1024, K step +32 B
        const uint32_t swz = c.swz ? 2u : 0u;
        const uint32_t kstep = c.swz ? 32 : 256;
        const uint64_t ad = desc_sw(a0, c.swz ? 16 : 128, 1024, swz);
        const uint64_t bd = desc_sw(b0, c.swz ? 16 : 128, 1024, swz);
        const uint32_t idesc = umma::idesc_bf16(c.M, c.N, c.a_mn, c.b_mn);
        long long t0 = 0, t1 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            __syncwarp();
            t0 = clock64();
            if (c.chunk == 0) {
                if (umma::elect_one()) {
                    for (int i = 0; i < NI; ++i) {
                        const int kk = i & 3;
                        umma::mma_bf16(tb, ad + (uint64_t)((kk * kstep) >> 4), bd + (uint64_t)((kk * kstep) >> 4),
                                       idesc, i ? 1u : 0u);
                    }
                    umma::commit(&bar);
                }
                __syncwarp();
            } else {
                if (rep == 0 && umma::elect_one()) umma::mbar_arrive(&rbar);  // a barrier that is already complete
                __syncwarp();
                if ((c.parts & 8) && (threadIdx.x & 31) == 0) {
                    for (int i0 = 0; i0 < NI; i0 += c.chunk) {
                        if (c.parts & 1) umma::mbar_wait(&rbar, 0u);
                        if (c.parts & 2) umma::fence_after_sync();
                        for (int i = i0; i < i0 + c.chunk; ++i) {
                            const int kk = i & 3;
                            umma::mma_bf16(tb, ad + (uint64_t)((kk * kstep) >> 4), bd + (uint64_t)((kk * kstep) >> 4),
                                           idesc, i ? 1u : 0u);
                        }
                        if (c.parts & 4) umma::commit(&ebar[(i0 / c.chunk) & 3]);
                    }
                }
                if (c.parts & 16) {
                    if (umma::elect_one()) {
                        for (int i0 = 0; i0 < NI; i0 += c.chunk) {
                            if (c.parts & 1) umma::mbar_wait(&rbar, 0u);
                            if (c.parts & 2) umma::fence_after_sync();
                            for (int i = i0; i < i0 + c.chunk; ++i) {
                                const int kk = i & 3;
                                umma::mma_bf16(tb, ad + (uint64_t)((kk * kstep) >> 4),
                                               bd + (uint64_t)((kk * kstep) >> 4), idesc, i ? 1u : 0u);
                            }
                            if (c.parts & 4) umma::commit(&ebar[(i0 / c.chunk) & 3]);
                        }
                    }
                    __syncwarp();
                }
                if (c.parts & 32) {
                    for (int i0 = 0; i0 < NI; i0 += 4) {
                        if (c.parts & 1) umma::mbar_wait(&rbar, 0u);
                        if (c.parts & 2) umma::fence_after_sync();
                        if (umma::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma::mma_bf16(tb, ad + (uint64_t)((kk * kstep) >> 4), bd + (uint64_t)((kk * kstep) >> 4),
                                               idesc, (i0 | kk) ? 1u : 0u);
                            if (c.parts & 4) umma::commit(&ebar[(i0 >> 2) & 3]);
                        }
                        __syncwarp();
                    }
                }
                if (!(c.parts & 56))
                for (int i0 = 0; i0 < NI; i0 += c.chunk) {
                    if (c.parts & 1) umma::mbar_wait(&rbar, 0u);
                    if (c.parts & 2) umma::fence_after_sync();
                    if (umma::elect_one()) {
                        for (int i = i0; i < i0 + c.chunk; ++i) {
                            const int kk = i & 3;
                            umma::mma_bf16(tb, ad + (uint64_t)((kk * kstep) >> 4), bd + (uint64_t)((kk * kstep) >> 4),
                                           idesc, i ? 1u : 0u);
                        }
                        if (c.parts & 4) umma::commit(&ebar[(i0 / c.chunk) & 3]);
                    }
                    __syncwarp();
                }
                if (umma::elect_one()) umma::commit(&bar);
                __syncwarp();
            }
            umma::mbar_wait(&bar, (uint32_t)rep);
            t1 = clock64();
        }
        if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = t1 - t0;
        if (threadIdx.x == 32) stop = 1;
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 512);
}

int main() {
    long long* d_out;
    cudaMalloc(&d_out, 16);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const Cfg cfgs[] = {
        {128, 64, 0, 1, 0, 0, 0},       // rollout hidden layer: A K-major, B MN-major, no swizzle
        {128, 64, 0, 1, 0, 0, 4, 7},    // the rollout's pattern: wait + fence + 4 MMAs + commit, per chunk elect
        {128, 64, 0, 1, 0, 0, 4, 39},   // the same with a compile-time unrolled chunk
        {128, 64, 0, 1, 0, 0, 4, 36},   // unrolled chunk + commit
        {128, 64, 0, 1, 0, 0, 4, 32},   // unrolled chunk only
        {128, 128, 0, 0, 0, 0, 4, 39},  // N = 128, unrolled 4 + wait + fence + commit
    };
    for (const Cfg& c : cfgs) {
        for (int grid : {1}) {
            const int NI = 512;
            k_bench<<<grid, 384, 200 * 1024>>>(c, NI, d_out);
            cudaError_t e = cudaDeviceSynchronize();
            long long cyc = 0;
            cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
            const double flop_per = 2.0 * c.M * c.N * 16;
            printf("M %3d N %3d a_mn %d b_mn %d swz %d bg %d chunk %2d parts %d grid %3d: %.1f cycles/MMA (floor %d) %s\n",
                   c.M, c.N, c.a_mn, c.b_mn, c.swz, c.background, c.chunk, c.parts, grid, (double)cyc / NI, (c.M < 128 ? 128 : c.M) * c.N / 256,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
            (void)flop_per;
        }
    }
    return 0;
}
