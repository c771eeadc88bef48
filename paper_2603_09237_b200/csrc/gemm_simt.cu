// Generic strided / grouped fp32 SIMT GEMM with fused epilogues. First
// correct implementation of every GEMM-shaped step of the update (grouped
// MLP forward/backward, hypernet feature MLP); tcgen05 kernels
// (tc_gemm.cu) replace it on the hot shapes.
#include "common.cuh"
#include "kernels.h"

namespace mb200 {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

__global__ void __launch_bounds__(NT) k_gemm_simt(GemmDesc d) {
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BN + 4];
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
    const int m0 = m_lo + blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    if (m0 >= m_hi || n0 >= d.N) return;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    float acc[4][4] = {};
    const bool a_kc = (d.ak == 1), b_nc = (d.bn == 1);
    for (int k0 = k_lo; k0 < k_hi; k0 += BK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + NT * q;
            int mm, kk;
            if (a_kc) { mm = e >> 4; kk = e & 15; } else { kk = e >> 6; mm = e & 63; }
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < m_hi && gk < k_hi) ? A[gm * d.am + gk * d.ak] : 0.f;
            int nn, kb;
            if (b_nc) { kb = e >> 6; nn = e & 63; } else { nn = e >> 4; kb = e & 15; }
            const int gn = n0 + nn, gkb = k0 + kb;
            Bs[kb][nn] = (gn < d.N && gkb < k_hi) ? B[gkb * d.bk + gn * d.bn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
            const float a[4] = {a4.x, a4.y, a4.z, a4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= m_hi) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= d.N) continue;
            float v = acc[i][j];
            if (d.bias_mode == 1) v += bias[gn];
            else if (d.bias_mode == 2) v += bias[gm];
            float* cp = C + gm * d.cm + gn * d.cn;
            if (d.accumulate) v += *cp;
            if (d.act == 1) {
                if (d.C2) d.C2[gm * d.c2m + gn * d.c2n] = v;
                v = tanhf(v);
            } else if (d.act == 2) {
                const float a = d.aux[gm * d.xm + gn * d.xn];
                v *= 1.f - a * a;
            }
            *cp = v;
        }
    }
}
}  // namespace

void gemm_simt(const GemmDesc& d, cudaStream_t s) {
    if (d.M <= 0 || d.N <= 0 || d.Z <= 0) return;
    const int mext = d.gmode == 1 ? d.max_group : d.M;
    if (mext <= 0) return;
    dim3 grid((d.N + BN - 1) / BN, (mext + BM - 1) / BM, d.Z);
    k_gemm_simt<<<grid, NT, 0, s>>>(d);
    MB_LAUNCH();
}

}  // namespace mb200
