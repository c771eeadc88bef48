// Hypernetwork M-block gradient fused with its Adam step (single rank: no
// gradient exchange sits between the backward and the optimizer, and the
// reference applies no gradient clipping, train.cpp:170-180). The reference
// computes dM = sum_g gtheta_g f_g^T (hypernet.cpp:124-160), stores it, and
// Adam reads it back (train.cpp:28-39). Here
//   dM[p][f] = sum_{g < G} gtheta[g][p] f[g][f]     (K = G clusters, 128 per stage)
// is a 64 x 32 register tile per 4-warp step of a persistent block on
// mma.sync (bf16 operands, fp32 accumulation, like the tcgen05 GEMM it
// replaces), and is consumed in registers by Adam: p, m1, m2 are streamed in
// by cp.async one tile ahead and written once, the bf16 image of the new M is written for the next theta
// GEMM, and dM itself never touches HBM. Bytes per element of M: 12 in, 12 +
// 2 out (the unfused pair moved 4 + 28 + 2). The tensor work is ~1% of the
// launch: this kernel is HBM-bound, not a tcgen05 candidate.
//
// Operands are the update's existing tiled bf16 images (img.cuh): gimg
// (rows g, cols p) and fimg (rows g, cols f). Both are K(=g)-outer, so the
// fragments come from ldmatrix.trans on a shared-memory copy of the core
// matrices (one contiguous run per 8 rows of g).
#include <algorithm>

#include "common.cuh"
#include "img.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

namespace {
constexpr int TP = 64, TF = 32;  // tile: 64 rows of M (p) x 32 columns (f)
constexpr int NT = TF / 8;       // n-tiles per warp (warp w: rows 16w..16w+15)
constexpr int KC = 128;          // groups (K) per pipeline stage; K loops over 128-group chunks
constexpr int LDP = TF + 8;      // smem row stride (floats) of the p / m1 / m2 tiles: conflict-free float2
constexpr int SA = KC / 8 * TP * 16, SB = KC / 8 * TF * 16, SP = TP * LDP * 4;
constexpr int STAGE = SA + SB;   // one K chunk of the gtheta / f slabs
constexpr int PMV = 3 * SP;      // one tile's p, m1, m2
constexpr int SMEM = 2 * STAGE + 2 * PMV;

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 16 B global -> shared, asynchronous; src_bytes 0 zero-fills (rows past P)
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {  // MUFU.SQRT; sqrt(0) = 0
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// W-column slab [c0, c0 + W) of image rows [8 kb0, 8 (kb0 + nkb)) (W = 32 or
// 64) -> smem: core matrix (row block kb - kb0, column block cb) at
// ((kb - kb0) * W/8 + cb) * 128 bytes. Thread t copies unit w = t % W of row
// blocks t / W, + 128 / W, ...
template <int W>
__device__ __forceinline__ void slab_async(uint32_t dst, const Img& im, int c0, int kb0, int nkb, int tl) {
    const int CT = img_ct(im.C);
    const int w = tl % W;
    const uint8_t* src = im.p + (long)(c0 >> 7) * 32768 + ((c0 & 127) >> 3) * 128 + w * 16;
    for (int j = tl / W; j < nkb; j += 128 / W) {
        const int kb = kb0 + j;
        cp16(dst + (j * W + w) * 16, src + (long)(kb >> 4) * CT * 32768 + (kb & 15) * 2048, 16);
    }
}

// the p, m1, m2 rows of tile t (thread t: column quad t % 8 of rows t / 8 + 16 k)
__device__ __forceinline__ void load_pmv(const DmAdam& a, int t, int ntf, uint32_t dst, int tl) {
    const int p0 = (t / ntf) * TP, f0 = (t % ntf) * TF;
    const int c4 = tl & 7, r0 = tl >> 3;
#pragma unroll
    for (int k = 0; k < TP / 16; ++k) {
        const int r = r0 + 16 * k;
        const bool ok = p0 + r < a.P;
        const long e = (long)(ok ? p0 + r : 0) * a.F + f0 + c4 * 4;
        const uint32_t d = dst + (r * LDP + c4 * 4) * 4;
        cp16(d, a.p + e, ok ? 16 : 0);
        cp16(d + SP, a.m1 + e, ok ? 16 : 0);
        cp16(d + 2 * SP, a.m2 + e, ok ? 16 : 0);
    }
}

// K = G <= 128 (a single rank's clusters, the bench launch): one stage per
// tile holding its gtheta / f slabs AND its p / m1 / m2 (2 stages: the next
// tile streams in while this one computes). 9 % faster than the K-chunked
// walker below at G = 128 (ncu, 92-94 vs 101-103 us).
constexpr int STAGE1 = SA + SB + PMV;
__global__ void __launch_bounds__(128) k_dm_adam_k1(const __grid_constant__ DmAdam a, int ntiles, int ntf) {
    extern __shared__ __align__(128) uint8_t smem[];
    pdl_enter();
    if (*a.err) return;  // non-finite loss: no update (k_adam_img)
    const int tl = threadIdx.x, lane = tl & 31, warp = tl >> 5;
    const int rq = lane >> 2, q = lane & 3, mi = lane >> 3, mr = lane & 7;
    const int Kp = (a.G + 15) & ~15;
    const int CT = img_ct(a.F);
    const uint32_t s0 = umma::smem_u32(smem);
    auto load = [&](int t, uint32_t st) {
        const int p0 = (t / ntf) * TP, f0 = (t % ntf) * TF;
        slab_async<TP>(st, a.gimg, p0, 0, Kp / 8, tl);
        slab_async<TF>(st + SA, a.fimg, f0, 0, Kp / 8, tl);
        load_pmv(a, t, ntf, st + SA + SB, tl);
    };
    int t = blockIdx.x;
    if (t < ntiles) load(t, s0);
    cp_commit();
    for (int i = 0; t < ntiles; t += gridDim.x, ++i) {
        const int tn = t + gridDim.x;
        const uint32_t st = s0 + (i & 1) * STAGE1;
        if (tn < ntiles) load(tn, s0 + ((i + 1) & 1) * STAGE1);
        cp_commit();
        cp_wait1();
        __syncthreads();
        float c[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
        for (int s = 0; s < Kp / 16; ++s) {
            uint32_t af[4];
            ldsm_x4_t(st + (((2 * s + (mi >> 1)) * (TP / 8) + 2 * warp + (mi & 1)) * 128 + mr * 16), af[0], af[1],
                      af[2], af[3]);
#pragma unroll
            for (int jp = 0; jp < NT / 2; ++jp) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(st + SA + (((2 * s + (mi & 1)) * (TF / 8) + 2 * jp + (mi >> 1)) * 128 + mr * 16), b0, b1, b2,
                          b3);
                mma16816(c[2 * jp], af, b0, b1);
                mma16816(c[2 * jp + 1], af, b2, b3);
            }
        }
        const int p0 = (t / ntf) * TP, f0 = (t % ntf) * TF;
        const float* sp = reinterpret_cast<const float*>(smem + (i & 1) * STAGE1 + SA + SB);
        const float lr1 = a.lr * a.ibc1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = warp * 16 + rq + 8 * h, row = p0 + r;
            if (row >= a.P) continue;
            float* prow = a.p + (long)row * a.F + f0 + 2 * q;
            float* arow = a.m1 + (long)row * a.F + f0 + 2 * q;
            float* brow = a.m2 + (long)row * a.F + f0 + 2 * q;
            uint8_t* irow = a.mimg.p + img_off(row, f0 + 2 * q, CT);
            const float* srow = sp + r * LDP + 2 * q;
#pragma unroll
            for (int jj = 0; jj < NT; ++jj) {
                float2 P2 = *reinterpret_cast<const float2*>(srow + 8 * jj);
                float2 A2 = *reinterpret_cast<const float2*>(srow + SP / 4 + 8 * jj);
                float2 B2 = *reinterpret_cast<const float2*>(srow + 2 * (SP / 4) + 8 * jj);
                const float g[2] = {c[jj][2 * h], c[jj][2 * h + 1]};
                float* P = &P2.x;
                float* A = &A2.x;
                float* B = &B2.x;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    A[k] = 0.9f * A[k] + 0.1f * g[k];
                    B[k] = 0.999f * B[k] + 0.001f * g[k] * g[k];
                    P[k] -= __fdividef(lr1 * A[k], sqrt_approx(B[k] * a.ibc2) + 1e-8f);
                }
                *reinterpret_cast<float2*>(prow + 8 * jj) = P2;
                *reinterpret_cast<float2*>(arow + 8 * jj) = A2;
                *reinterpret_cast<float2*>(brow + 8 * jj) = B2;
                *reinterpret_cast<uint32_t*>(irow + 128 * jj) = umma::pack_bf16(P[0], P[1]);
            }
        }
        __syncthreads();
    }
}

// persistent: block b walks tiles t = b, b + gridDim.x, ...; each tile is
// nk K-chunks of <= 128 groups. A load unit is (tile, chunk): the gtheta / f
// slabs of the chunk, plus the tile's p, m1, m2 with its first chunk. Two
// units are in flight (cp.async groups, wait_group 1), so the next chunk or
// tile streams in while this one's MMAs / Adam run. The accumulators live in
// registers across the chunks of a tile and are summed in the same k order
// for every chunking (identical results for any number of ranks).
__global__ void __launch_bounds__(128) k_dm_adam(const __grid_constant__ DmAdam a, int ntiles, int ntf) {
    extern __shared__ __align__(128) uint8_t smem[];
    pdl_enter();
    if (*a.err) return;  // non-finite loss: no update (k_adam_img)
    const int tl = threadIdx.x;
    const int vb = blockIdx.x, vgrid = gridDim.x;
    auto sync = [] { __syncthreads(); };
    const int lane = tl & 31, warp = tl >> 5;
    const int rq = lane >> 2, q = lane & 3, mi = lane >> 3, mr = lane & 7;
    const int Kp = (a.G + 15) & ~15;
    const int nk = (Kp + KC - 1) / KC;
    const int CT = img_ct(a.F);
    const uint32_t s0 = umma::smem_u32(smem);
    const uint32_t pmv0 = s0 + 2 * STAGE;
    const int my_tiles = vb < ntiles ? (ntiles - 1 - vb) / vgrid + 1 : 0;
    const int units = my_tiles * nk;
    auto issue = [&](int u) {  // load unit u of this block
        const int j = u / nk, kc = u - j * nk;
        const int t = vb + j * vgrid;
        const int p0 = (t / ntf) * TP, f0 = (t % ntf) * TF;
        const int kb0 = kc * (KC / 8), nkb = min(KC, Kp - kc * KC) / 8;
        const uint32_t st = s0 + (u & 1) * STAGE;
        slab_async<TP>(st, a.gimg, p0, kb0, nkb, tl);
        slab_async<TF>(st + SA, a.fimg, f0, kb0, nkb, tl);
        if (kc == 0) load_pmv(a, t, ntf, pmv0 + (j & 1) * PMV, tl);
    };
    if (units > 0) issue(0);
    cp_commit();
    float c[NT][4];
    for (int u = 0; u < units; ++u) {
        const int j = u / nk, kc = u - j * nk;
        const int t = vb + j * vgrid;
        if (u + 1 < units) issue(u + 1);
        cp_commit();
        cp_wait1();  // unit u has landed (unit u + 1 may be in flight)
        sync();
        if (kc == 0) {
#pragma unroll
            for (int jj = 0; jj < NT; ++jj) c[jj][0] = c[jj][1] = c[jj][2] = c[jj][3] = 0.f;
        }
        const uint32_t st = s0 + (u & 1) * STAGE;
        const int ks = min(KC, Kp - kc * KC) / 16;
        for (int s = 0; s < ks; ++s) {
            // A (m = p, k = g): matrices (g-block 2s + (mi >> 1), p-block 2 warp + (mi & 1))
            uint32_t af[4];
            ldsm_x4_t(st + (((2 * s + (mi >> 1)) * (TP / 8) + 2 * warp + (mi & 1)) * 128 + mr * 16), af[0], af[1],
                      af[2], af[3]);
#pragma unroll
            for (int jp = 0; jp < NT / 2; ++jp) {  // n-tiles 2 jp, 2 jp + 1
                // B (k = g, n = f): matrices (g-block 2s + (mi & 1), f-block 2 jp + (mi >> 1))
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(st + SA + (((2 * s + (mi & 1)) * (TF / 8) + 2 * jp + (mi >> 1)) * 128 + mr * 16), b0, b1, b2,
                          b3);
                mma16816(c[2 * jp], af, b0, b1);
                mma16816(c[2 * jp + 1], af, b2, b3);
            }
        }
        if (kc == nk - 1) {
            const int p0 = (t / ntf) * TP, f0 = (t % ntf) * TF;
            const float* sp = reinterpret_cast<const float*>(smem + 2 * STAGE + (j & 1) * PMV);
            // Adam in fp32 with hardware sqrt / reciprocal (a few ulp from the IEEE
            // forms of k_adam_img; far inside the bf16-operand tolerance)
            const float lr1 = a.lr * a.ibc1;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = warp * 16 + rq + 8 * h, row = p0 + r;
                if (row >= a.P) continue;
                float* prow = a.p + (long)row * a.F + f0 + 2 * q;
                float* arow = a.m1 + (long)row * a.F + f0 + 2 * q;
                float* brow = a.m2 + (long)row * a.F + f0 + 2 * q;
                uint8_t* irow = a.mimg.p + img_off(row, f0 + 2 * q, CT);  // + 128 B per n-tile (8 columns)
                const float* srow = sp + r * LDP + 2 * q;
#pragma unroll
                for (int jj = 0; jj < NT; ++jj) {
                    float2 P2 = *reinterpret_cast<const float2*>(srow + 8 * jj);
                    float2 A2 = *reinterpret_cast<const float2*>(srow + SP / 4 + 8 * jj);
                    float2 B2 = *reinterpret_cast<const float2*>(srow + 2 * (SP / 4) + 8 * jj);
                    const float g[2] = {c[jj][2 * h], c[jj][2 * h + 1]};
                    float* P = &P2.x;
                    float* A = &A2.x;
                    float* B = &B2.x;
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        A[k] = 0.9f * A[k] + 0.1f * g[k];
                        B[k] = 0.999f * B[k] + 0.001f * g[k] * g[k];
                        P[k] -= __fdividef(lr1 * A[k], sqrt_approx(B[k] * a.ibc2) + 1e-8f);
                    }
                    *reinterpret_cast<float2*>(prow + 8 * jj) = P2;
                    *reinterpret_cast<float2*>(arow + 8 * jj) = A2;
                    *reinterpret_cast<float2*>(brow + 8 * jj) = B2;
                    *reinterpret_cast<uint32_t*>(irow + 128 * jj) = umma::pack_bf16(P[0], P[1]);
                }
            }
        }
        sync();  // this stage (and, after the last chunk, this p / m1 / m2 buffer) is refilled next
    }
}
}  // namespace

void dm_adam(const DmAdam& a, cudaStream_t s) {
    if (a.F % TF || a.G < 1 || a.P < 1) throw ShapeError("dm_adam: F % 32 == 0, groups >= 1, rows >= 1 required");
    if (a.P <= 0) return;
    const uintptr_t al = reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m1) |
                         reinterpret_cast<uintptr_t>(a.m2);
    if (al & 15) throw ShapeError("dm_adam: parameter block must be 16-byte aligned");
    ensure_smem((const void*)k_dm_adam, SMEM);
    const int ntf = a.F / TF, ntiles = (a.P + TP - 1) / TP * ntf;
    // two 108 KB blocks per SM. (One double-width block on a subset of the
    // SMs, leaving the rest to the other update chain, was measured slower:
    // the optimizer loses more bandwidth than the other chain gains.)
    const int grid = std::min(ntiles, 2 * device_sms());
    if (a.G <= KC) {  // one K chunk: one stage per tile
        ensure_smem((const void*)k_dm_adam_k1, 2 * STAGE1);
        launch_pdl(k_dm_adam_k1, dim3(grid), dim3(128), 2 * STAGE1, s, a, ntiles, ntf);
    } else {  // K chunks (more clusters than one rank's 128)
        launch_pdl(k_dm_adam, dim3(grid), dim3(128), SMEM, s, a, ntiles, ntf);
    }
    MB_LAUNCH();
}

}  // namespace mb200
