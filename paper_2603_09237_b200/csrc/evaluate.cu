// evaluate_params / eval_point (reference evaluate.cpp:17-101) on the device:
// for every preference w_g of the simplex grid, `episodes` fresh instances of
// the environment are reset from Rng(key).split(g) (instance i streams from
// .split(i), env.cpp:51-58) and stepped with the deterministic policy --
// the generated MLP's output activation, tanh of the Gaussian mean -- until
// every instance finished its first episode or max_episode_steps; the
// undiscounted returns of that first episode are averaged per objective.
//
// One CTA per (grid point, block of 8 or 16 instances): the point's generated
// weights theta_g (from the hypernet GEMM) are staged ONCE into shared
// memory as bf16 (transposed, [in][out], so thread j reads W[k][j]
// conflict-free) and stay resident for all steps; activations ping-pong in
// shared memory as [k][instance]; env state lives in shared memory. Each
// step: thread j computes output j of a layer for all the CTA's instances (the
// instance values are shared-memory broadcasts), then the instance threads
// step the environment. fp32 arithmetic, fp64 return sums.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mb200 {

namespace {
constexpr int kEvalE = 16;  // max instances per CTA
constexpr int kEvalThreads = 256;

template <int E>  // instances per CTA (8 or 16)
__global__ void __launch_bounds__(kEvalThreads) k_eval(const __grid_constant__ EvalArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    const NetDims& nd = a.pol;
    const int g = blockIdx.x / a.cpp, cb = blockIdx.x % a.cpp;
    const int i0 = cb * E, n = min(E, a.episodes - i0);
    const float* th = a.theta + (long)g * a.ld;
    // ---- shared-memory carve-up (host sizes the same)
    uint8_t* p = sm;
    float* S = reinterpret_cast<float*>(p); p += sizeof(float) * a.sdim * E;
    float* act[2];
    act[0] = reinterpret_cast<float*>(p); p += sizeof(float) * a.maxw * E;
    act[1] = reinterpret_cast<float*>(p); p += sizeof(float) * a.maxw * E;
    double* tot = reinterpret_cast<double*>(p); p += sizeof(double) * E * 8;
    float* bias = reinterpret_cast<float*>(p); p += sizeof(float) * a.nbias;
    __nv_bfloat16* WT = reinterpret_cast<__nv_bfloat16*>(p);  // per layer [in][out]
    __shared__ int alive[E], steps[E];
    // ---- weights: theta (fp32, W_l [out][in] then b_l) -> WT_l (bf16, [in][out])
    {
        long wo = 0, bo = 0;
        for (int l = 0; l < nd.L; ++l) {
            const int in = nd.sz[l], out = nd.sz[l + 1];
            for (int e = threadIdx.x; e < in * out; e += blockDim.x) {
                const int j = e / in, k = e - j * in;
                WT[wo + (long)k * out + j] = __float2bfloat16_rn(th[nd.woff[l] + e]);
            }
            for (int j = threadIdx.x; j < out; j += blockDim.x) bias[bo + j] = th[nd.boff[l] + j];
            wo += (long)in * out;
            bo += out;
        }
    }
    // ---- fresh instances: BatchedEnv::reset(rng.split(g)) (env.cpp:51-58)
    const uint64_t gkey = split_key(a.key, (uint64_t)g);
    if (threadIdx.x < E) {
        const int r = threadIdx.x;
        alive[r] = r < n;
        steps[r] = 0;
        for (int k = 0; k < 8; ++k) tot[r * 8 + k] = 0.0;
        if (r < n) {
            uint64_t ctr = 0;
            env_do_reset(a.kind, S + r, E, split_key(gkey, (uint64_t)(i0 + r)), &ctr);
        } else {
            for (int k = 0; k < a.sdim; ++k) S[k * E + r] = 0.f;
        }
    }
    __syncthreads();
    for (int t = 0; t < a.max_steps; ++t) {
        const int any = __syncthreads_or(threadIdx.x < E ? alive[threadIdx.x] : 0);
        if (!any) break;  // evaluate.cpp:57
        for (int e = threadIdx.x; e < a.od * E; e += blockDim.x) act[0][e] = S[e];  // obs = state[0:od]
        __syncthreads();
        int cur = 0;
        long wo = 0, bo = 0;
        for (int l = 0; l < nd.L; ++l) {  // mlp_forward_cached (nn.cpp:60-92), tanh every layer
            const int in = nd.sz[l], out = nd.sz[l + 1];
            const float* ai = act[cur];
            float* ao = act[cur ^ 1];
            for (int j = threadIdx.x; j < out; j += blockDim.x) {
                float z[E];
#pragma unroll
                for (int r = 0; r < E; ++r) z[r] = bias[bo + j];
#pragma unroll 4
                for (int k = 0; k < in; ++k) {
                    const float w = __bfloat162float(WT[wo + (long)k * out + j]);
                    const float4* x4 = reinterpret_cast<const float4*>(ai + k * E);
#pragma unroll
                    for (int q = 0; q < E / 4; ++q) {
                        const float4 x = x4[q];
                        z[4 * q + 0] = fmaf(w, x.x, z[4 * q + 0]);
                        z[4 * q + 1] = fmaf(w, x.y, z[4 * q + 1]);
                        z[4 * q + 2] = fmaf(w, x.z, z[4 * q + 2]);
                        z[4 * q + 3] = fmaf(w, x.w, z[4 * q + 3]);
                    }
                }
                const bool squash = l < nd.L - 1 || nd.out_tanh;
#pragma unroll
                for (int r = 0; r < E; ++r) ao[j * E + r] = squash ? tanhf(z[r]) : z[r];
            }
            __syncthreads();
            cur ^= 1;
            wo += (long)in * out;
            bo += out;
        }
        // ---- step the alive instances (env.cpp:60-92), first-episode returns
        if (threadIdx.x < n && alive[threadIdx.x]) {
            const int r = threadIdx.x;
            float ac[16], rw[8];
            for (int d = 0; d < a.ad; ++d) {
                const float x = act[cur][d * E + r];
                if (!isfinite(x)) atomicExch(a.err, 3);
                ac[d] = fminf(fmaxf(x, -1.f), 1.f);
            }
            const bool tm = env_do_step(a.kind, S + r, E, ac, rw);
            const int st = steps[r] + 1;
            steps[r] = st;
            const bool tr = !tm && st >= a.max_steps;
            for (int k = 0; k < a.m; ++k) tot[r * 8 + k] += (double)rw[k];
            if (tm || tr) alive[r] = 0;
        }
        __syncthreads();
    }
    if (threadIdx.x < a.m) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += tot[r * 8 + threadIdx.x];
        a.part[((long)g * a.cpp + cb) * a.m + threadIdx.x] = s;
    }
}

__global__ void k_eval_mean(const double* part, int ng, int cpp, int m, int episodes, double* mean) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ng * m) return;
    const int g = e / m, k = e - g * m;
    double s = 0.0;
    for (int c = 0; c < cpp; ++c) s += part[((long)g * cpp + c) * m + k];
    mean[e] = s / (double)episodes;
}
}  // namespace

size_t eval_smem(const EvalArgs& a, int E) {
    size_t w = 0;
    for (int l = 0; l < a.pol.L; ++l) w += (size_t)a.pol.sz[l] * a.pol.sz[l + 1];
    return sizeof(float) * a.sdim * E + 2 * sizeof(float) * a.maxw * E + sizeof(double) * E * 8 +
           sizeof(float) * a.nbias + 2 * w;
}

void evaluate(EvalArgs a, int n_points, double* d_mean, cudaStream_t s) {
    const int E = a.episodes <= 8 ? 8 : kEvalE;
    a.cpp = (a.episodes + E - 1) / E;
    a.maxw = 0;
    a.nbias = 0;
    for (int l = 0; l <= a.pol.L; ++l) a.maxw = std::max(a.maxw, (a.pol.sz[l] + 3) / 4 * 4);
    for (int l = 0; l < a.pol.L; ++l) a.nbias += a.pol.sz[l + 1];
    if (a.ad > 16 || a.m > 8) throw ShapeError("evaluate: act_dim <= 16 and m <= 8 on the device");
    const size_t smem = (eval_smem(a, E) + 15) / 16 * 16;
    if (smem > 220 * 1024) throw ShapeError("evaluate: the policy does not fit in shared memory (bf16)");
    auto kern = E == 8 ? k_eval<8> : k_eval<16>;
    MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<n_points * a.cpp, kEvalThreads, smem, s>>>(a);
    MB_LAUNCH();
    const int n = n_points * a.m;
    k_eval_mean<<<(n + 255) / 256, 256, 0, s>>>(a.part, n_points, a.cpp, a.m, a.episodes, d_mean);
    MB_LAUNCH();
}

}  // namespace mb200
