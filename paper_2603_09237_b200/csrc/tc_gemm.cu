// tcgen05 GEMM for every GEMM-shaped step of the training iteration
// (hypernet theta generation, dM, df split-K, feature MLP, grouped policy /
// critic MLP forward, dX and per-cluster dW). Drop-in for the strided /
// grouped GemmDesc of gemm_simt:
//   * 128 x BN output tile per CTA, fp32 accumulators in TMEM (BN columns);
//   * operands read from fp32 global memory (any layout with one unit
//     stride), rounded to bf16 and staged in shared memory in the canonical
//     no-swizzle UMMA layout -- K-major when the K stride is 1, MN-major
//     when the M/N stride is 1 (umma.cuh), so no transposes are ever
//     materialised;
//   * 2-stage pipeline: all 256 threads stage K-tile k+1 while the single
//     issuing thread's tcgen05.mma of tile k runs; tcgen05.commit ->
//     mbarrier releases a stage;
//   * epilogue: tcgen05.ld (32 lanes x 16 cols per warp) -> bias / tanh /
//     tanh-derivative / accumulate -> global.
#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

namespace {
constexpr int TM = 128, TK = 64, NTH = 256;
constexpr int A_STAGE = TM * TK * 2;  // 16 KB

template <int BN>
struct Smem {
    static constexpr int B_STAGE = BN * TK * 2;
    static constexpr int BYTES = 2 * A_STAGE + 2 * B_STAGE + 64;
};

// stage one operand tile (ROWS x 64 K) of fp32 global data as bf16 UMMA core
// matrices. All global loads of the tile are issued before any conversion /
// shared store so each thread keeps PER independent requests in flight.
template <int ROWS>
__device__ __forceinline__ void stage(uint8_t* dst, const float* __restrict__ src, long s_mn, long s_k,
                                      bool mn_major, int mn0, int mn_hi, int k0, int k_hi) {
    constexpr int NCH = ROWS * (TK / 8);
    constexpr int PER = (NCH + NTH - 1) / NTH;
    float v[PER][8];
    int off[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int c = threadIdx.x + q * NTH;
        off[q] = -1;
        if (c >= NCH) continue;
        const int r8 = c & 7, rest = c >> 3, kb = rest & 7, grp = rest >> 3;
        off[q] = grp * 1024 + kb * 128 + r8 * 16;
        if (!mn_major) {  // 8 consecutive k of one row
            const int mn = mn0 + grp * 8 + r8, k = k0 + kb * 8;
            const float* p = src + (long)mn * s_mn + (long)k * s_k;
            if (mn < mn_hi && k + 8 <= k_hi && s_k == 1 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(p));
                const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
                v[q][0] = a.x; v[q][1] = a.y; v[q][2] = a.z; v[q][3] = a.w;
                v[q][4] = b.x; v[q][5] = b.y; v[q][6] = b.z; v[q][7] = b.w;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[q][e] = (mn < mn_hi && k + e < k_hi) ? __ldg(p + (long)e * s_k) : 0.f;
            }
        } else {  // 8 consecutive mn of one k
            const int mn = mn0 + grp * 8, k = k0 + kb * 8 + r8;
            const float* p = src + (long)mn * s_mn + (long)k * s_k;
            if (k < k_hi && mn + 8 <= mn_hi && s_mn == 1 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(p));
                const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
                v[q][0] = a.x; v[q][1] = a.y; v[q][2] = a.z; v[q][3] = a.w;
                v[q][4] = b.x; v[q][5] = b.y; v[q][6] = b.z; v[q][7] = b.w;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[q][e] = (k < k_hi && mn + e < mn_hi) ? __ldg(p + (long)e * s_mn) : 0.f;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (off[q] < 0) continue;
        uint4 w;
        w.x = umma::pack_bf16(v[q][0], v[q][1]);
        w.y = umma::pack_bf16(v[q][2], v[q][3]);
        w.z = umma::pack_bf16(v[q][4], v[q][5]);
        w.w = umma::pack_bf16(v[q][6], v[q][7]);
        *reinterpret_cast<uint4*>(dst + off[q]) = w;
    }
}

template <int BN>
__global__ void __launch_bounds__(NTH) k_tc_gemm(GemmDesc d, int a_mn_major, int b_mn_major) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + 2 * A_STAGE;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sB + 2 * Smem<BN>::B_STAGE);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 2);

    const int z = blockIdx.z;
    int m_lo = 0, m_hi = d.M, k_lo = 0, k_hi = d.K;
    const float* A = d.A;
    const float* B = d.B;
    float* C = d.C;
    const float* bias = d.bias;
    if (d.gmode == 0) {
        A += z * d.a_bz;
        B += z * d.b_bz;
        C += z * d.c_bz;
        if (bias) bias += z * d.bias_bz;
    } else if (d.gmode == 1) {
        m_lo = d.goff[z];
        m_hi = d.goff[z + 1];
        B += z * d.b_bz;
        if (bias) bias += z * d.bias_bz;
    } else {
        k_lo = d.goff[z];
        k_hi = d.goff[z + 1];
        C += z * d.c_bz;
    }
    const int m0 = m_lo + blockIdx.y * TM;
    const int n0 = blockIdx.x * BN;
    if (m0 >= m_hi || n0 >= d.N) return;  // block-uniform

    constexpr uint32_t kCols = BN < 32 ? 32 : BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(tslot, kCols);
    if (threadIdx.x == 32) {
        umma::mbar_init(&mbar[0], 1);
        umma::mbar_init(&mbar[1], 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tbase = *tslot;
    const uint32_t idesc = umma::idesc_bf16(TM, BN, a_mn_major, b_mn_major);
    const int nk = (k_hi - k_lo + TK - 1) / TK;

    for (int kt = 0; kt < nk; ++kt) {
        const int s = kt & 1;
        if (kt >= 2) umma::mbar_wait(&mbar[s], ((kt - 2) >> 1) & 1);
        const int k0 = k_lo + kt * TK;
        stage<TM>(sA + s * A_STAGE, A, d.am, d.ak, a_mn_major, m0, m_hi, k0, k_hi);
        stage<BN>(sB + s * Smem<BN>::B_STAGE, B, d.bn, d.bk, b_mn_major, n0, d.N, k0, k_hi);
        umma::fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            umma::fence_after_sync();
            const uint32_t a0 = umma::smem_u32(sA + s * A_STAGE), b0 = umma::smem_u32(sB + s * Smem<BN>::B_STAGE);
#pragma unroll
            for (int kk = 0; kk < TK / 16; ++kk)
                umma::mma_bf16(tbase, umma::smem_desc(a0 + kk * 256, 128, 1024),
                               umma::smem_desc(b0 + kk * 256, 128, 1024), idesc, (kt | kk) ? 1u : 0u);
            umma::commit(&mbar[s]);
        }
    }
    if (nk > 0) {
        umma::mbar_wait(&mbar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
        umma::fence_after_sync();
    }

    // epilogue: warp w reads TMEM lanes 32*(w%4).. and column half w/4
    const int lg = warp & 3, ch = warp >> 2;
    const int m = m0 + lg * 32 + lane;
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const bool active = BN >= 32 || ch == 0;
    if (active) {
        for (int c0 = ch * HALF; c0 < ch * HALF + HALF; c0 += 16) {
            float v[16];
            if (nk > 0) {
                umma::tmem_ld16(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)c0, v);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            if (m < m_hi) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int n = n0 + c0 + i;
                    if (n >= d.N) continue;
                    float x = v[i];
                    if (d.bias_mode == 1) x += bias[n];
                    else if (d.bias_mode == 2) x += bias[m];
                    float* cp = C + (long)m * d.cm + (long)n * d.cn;
                    if (d.accumulate) x += *cp;
                    if (d.act == 1) {
                        if (d.C2) d.C2[(long)m * d.c2m + (long)n * d.c2n] = x;
                        x = tanhf(x);
                    } else if (d.act == 2) {
                        const float a = d.aux[(long)m * d.xm + (long)n * d.xn];
                        x *= 1.f - a * a;
                    }
                    *cp = x;
                }
            }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tbase, kCols);
}

template <int BN>
void launch(const GemmDesc& d, int a_mn, int b_mn, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        MB_CUDA(cudaFuncSetAttribute(k_tc_gemm<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::BYTES));
        configured = true;
    }
    const int mext = d.gmode == 1 ? d.max_group : d.M;
    dim3 grid((d.N + BN - 1) / BN, (mext + TM - 1) / TM, d.Z);
    k_tc_gemm<BN><<<grid, NTH, Smem<BN>::BYTES, s>>>(d, a_mn, b_mn);
    MB_LAUNCH();
}
}  // namespace

bool gemm_tc_eligible(const GemmDesc& d) {
    return (d.ak == 1 || d.am == 1) && (d.bk == 1 || d.bn == 1);
}

void gemm_tc(const GemmDesc& d, cudaStream_t s) {
    if (d.M <= 0 || d.N <= 0 || d.Z <= 0) return;
    if (d.gmode == 1 && d.max_group <= 0) return;
    if (!gemm_tc_eligible(d)) throw ShapeError("gemm_tc: operands need a unit stride along K or M/N");
    const int a_mn = d.ak == 1 ? 0 : 1;
    const int b_mn = d.bk == 1 ? 0 : 1;
    if (d.N <= 16) launch<16>(d, a_mn, b_mn, s);
    else if (d.N <= 32) launch<32>(d, a_mn, b_mn, s);
    else if (d.N <= 64) launch<64>(d, a_mn, b_mn, s);
    else if (d.N <= 128) launch<128>(d, a_mn, b_mn, s);
    else launch<256>(d, a_mn, b_mn, s);
}

}  // namespace mb200
