// K3 on the tensor cores: the fused rollout (rollout.cpp:37-161) with every
// policy / critic layer as tcgen05.mma.
//
// * One persistent CTA owns <= 64 instances of ONE preference cluster for
//   all T steps; env state stays in shared memory.
// * The cluster's generated weights theta_c (fp32, from the hypernet GEMM)
//   are packed once per iteration by k_pack_theta into bf16 "blobs" already
//   in the UMMA K-major core-matrix image, one contiguous chunk per
//   128-feature tile of each hidden layer plus one chunk for the output
//   layer. Every step the CTA streams its chunks L2 -> SMEM with the TMA
//   bulk-copy engine (cp.async.bulk, mbarrier complete_tx) through a 2-slot
//   ring, two chunks ahead of the MMA.
// * Hidden layers: D[feature][env] = W_l (A, K-major) x act^T (B, MN-major),
//   M = 128 features per tile, N = envs; the epilogue (tcgen05.ld) adds the
//   fp32 bias, applies tanh and writes the next layer's bf16 operand.
// * Output layer: D[env][out] = act (A, MN-major, M = 64 envs) x W_out^T
//   (B, K-major, N = 16), so each env-owning thread gets its own outputs
//   and goes straight on to sampling / the env step.
// * The N(0,1) draws do not depend on the policy: k_rollout_noise computes
//   all T steps' fp64 Box-Muller draws ahead at full occupancy (bit-identical
//   words, rounded to fp32 exactly where the sequential sampler rounds), and
//   the sampler only reads them.
// * Critic: once per step at the pre-reset final observation; at the
//   current observation only when the previous step reset an instance (or
//   t = 0), because V(o_{t+1}) = next_value_t otherwise.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

namespace {
constexpr int RNT = 256;  // threads
constexpr int RE = 64;    // instances per CTA
constexpr int OUT_COL = 128;

#ifdef MB_ROLL_PROF  // phase timing of CTA 0 (debug builds only: NVCC="nvcc -DMB_ROLL_PROF")
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define RPROF(k)                                            \
    if (blockIdx.x == 0 && threadIdx.x == 0) {              \
        const unsigned long long now_ = gtimer();           \
        prof_[k] += now_ - prof_last_;                      \
        prof_last_ = now_;                                  \
    }
#else
#define RPROF(k)
#endif

__device__ __forceinline__ float sech2(float z) {
    const float e = __expf(-2.f * fabsf(z));
    const float d = 1.f + e;
    return 4.f * e / (d * d);
}

struct Ctx {
    uint8_t* ring0;  // 2 weight slots: ring0 + slot * ring_stride (no indexed pointer array: registers)
    int ring_stride;
    uint8_t* xb;     // layer-0 operand (MN-major, env x obs_pad)
    uint8_t* hb0;  // 2 hidden-activation buffers (MN-major, env x hpad): hb0 + i * hb_stride
    int hb_stride;
    uint64_t* fullb;
    uint64_t* mmad;
    uint32_t tbase;
    int nepad;
    // issue state (thread 0 only)
    long issued;  // chunks issued so far
    long consumed;
};

__device__ __forceinline__ void chunk_at(const RolloutTcArgs& a, int vflag, int pos, int* net, int* c) {
    if (pos < a.pol_plan.nchunks) { *net = 0; *c = pos; return; }
    pos -= a.pol_plan.nchunks;
    *net = 1;
    *c = vflag ? (pos % a.cri_plan.nchunks) : pos;
}
__device__ __forceinline__ int step_len(const RolloutTcArgs& a, int vflag) {
    return a.pol_plan.nchunks + (vflag ? 2 : 1) * a.cri_plan.nchunks;
}

// thread 0: issue the bulk copy of the J-th chunk of the CTA's sequence.
// The sequence position is tracked by (step, pos); vflag of the issuing
// step is known because the issuer runs at most 2 chunks ahead and every
// step starts with >= 2 policy chunks.
struct Issuer {
    int step, pos;
};

__device__ __forceinline__ void issue_next(const RolloutTcArgs& a, Ctx& x, Issuer& is, const int* vflags, int group) {
    if (is.step >= a.T) return;
    int net, c;
    chunk_at(a, vflags[is.step & 1], is.pos, &net, &c);
    const NetPlan& pl = net ? a.cri_plan : a.pol_plan;
    const uint8_t* src = (net ? a.cri_blob : a.pol_blob) + (long)group * pl.blob_bytes + pl.chunk_off[c];
    const int slot = (int)(x.issued & 1);
    umma::mbar_arrive_expect_tx(&x.fullb[slot], (uint32_t)pl.chunk_bytes[c]);
    umma::bulk_g2s(x.ring0 + slot * x.ring_stride, src, (uint32_t)pl.chunk_bytes[c], &x.fullb[slot]);
    x.issued++;
    if (++is.pos >= step_len(a, vflags[is.step & 1])) {
        is.pos = 0;
        is.step++;
    }
}

// Run one net (all chunks) on the layer-0 operand xb. Result: output layer
// accumulators in TMEM columns [OUT_COL, OUT_COL+16) (M = 64 env layout).
__device__ __forceinline__ void run_net(const RolloutTcArgs& a, Ctx& x, Issuer& is, const int* vflags, int group, int net,
                        const float* theta) {
    const NetPlan& pl = net ? a.cri_plan : a.pol_plan;
    const NetDims& nd = net ? a.cri : a.pol;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int c = 0;
    int cur = -1;  // -1: input is xb, else hb[cur]
    for (int l = 0; l < nd.L; ++l) {
        const bool last = (l == nd.L - 1);
        const int kin = pl.kin_pad[l];
        const uint32_t sbo = (uint32_t)kin * 16;  // 8-row block stride of every operand of this layer
        const uint8_t* inb = cur < 0 ? x.xb : x.hb0 + cur * x.hb_stride;
        const int ntiles = last ? 1 : pl.tiles[l];
        for (int t = 0; t < ntiles; ++t, ++c) {
            if (threadIdx.x == 0) {
                const int slot = (int)(x.consumed & 1);
                umma::mbar_wait(&x.fullb[slot], (uint32_t)((x.consumed >> 1) & 1));
                umma::fence_after_sync();
                const uint32_t w0 = umma::smem_u32(x.ring0 + slot * x.ring_stride), i0 = umma::smem_u32(inb);
                if (!last) {
                    const uint32_t idesc = umma::idesc_bf16(128, x.nepad, false, true);
                    for (int k = 0; k < kin / 16; ++k)
                        umma::mma_bf16(x.tbase + (uint32_t)(t * x.nepad), umma::smem_desc(w0 + k * 256, 128, sbo),
                                       umma::smem_desc(i0 + k * 256, 128, sbo), idesc, k ? 1u : 0u);
                } else {
                    const uint32_t idesc = umma::idesc_bf16(64, 16, true, false);
                    for (int k = 0; k < kin / 16; ++k)
                        umma::mma_bf16(x.tbase + OUT_COL, umma::smem_desc(i0 + k * 256, 128, sbo),
                                       umma::smem_desc(w0 + k * 256, 128, sbo), idesc, k ? 1u : 0u);
                }
                umma::commit(x.mmad);
                umma::mbar_wait(x.mmad, (uint32_t)(x.consumed & 1));
                x.consumed++;
                issue_next(a, x, is, vflags, group);  // slot is free again
            }
        }
        __syncthreads();
        umma::fence_after_sync();
        if (!last) {  // epilogue: bias + tanh -> next operand (MN-major, env x hpad)
            const int nxt = cur < 0 ? 0 : (cur ^ 1);
            uint8_t* ob = x.hb0 + nxt * x.hb_stride;
            const uint32_t osbo = (uint32_t)pl.kin_pad[l + 1] * 16;
            const int tile = warp >> 2, lg = warp & 3;
            const int out = nd.sz[l + 1];
            if (tile < ntiles && tile * 128 + lg * 32 < out) {
                const int j = tile * 128 + lg * 32 + lane;
                const float bj = j < out ? theta[nd.boff[l] + j] : 0.f;
                for (int n0 = 0; n0 < x.nepad; n0 += 16) {
                    float v[16];
                    umma::tmem_ld16(x.tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(tile * x.nepad + n0), v);
                    if (j < out) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint4 q;
                            // MUFU tanh (rel err < 2^-10.99): below the bf16 rounding of the operand
                            q.x = umma::pack_bf16(umma::tanh_approx(v[8 * h + 0] + bj), umma::tanh_approx(v[8 * h + 1] + bj));
                            q.y = umma::pack_bf16(umma::tanh_approx(v[8 * h + 2] + bj), umma::tanh_approx(v[8 * h + 3] + bj));
                            q.z = umma::pack_bf16(umma::tanh_approx(v[8 * h + 4] + bj), umma::tanh_approx(v[8 * h + 5] + bj));
                            q.w = umma::pack_bf16(umma::tanh_approx(v[8 * h + 6] + bj), umma::tanh_approx(v[8 * h + 7] + bj));
                            const int nb = (n0 >> 3) + h;
                            *reinterpret_cast<uint4*>(ob + nb * osbo + (j >> 3) * 128 + (j & 7) * 16) = q;
                        }
                    }
                }
            }
            umma::fence_before_sync();
            umma::fence_proxy_async();
            __syncthreads();
            cur = nxt;
        }
    }
}

__global__ void __launch_bounds__(RNT, 1) k_rollout_tc(const __grid_constant__ RolloutTcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int cpg = (a.reps + RE - 1) / RE;
    const int c = blockIdx.x / cpg, ch = blockIdx.x % cpg;
    const int i0 = c * a.reps + ch * RE;
    const int nr = min(RE, a.reps - ch * RE);
    const int od = a.od, ad = a.ad, m = a.m, sd = a.sdim;
    const int tid = threadIdx.x;
    // ---- shared memory carve-up (host computes the same total)
    Ctx x;
    uint8_t* p = smem;
    x.ring0 = p; x.ring_stride = a.slot_bytes; p += 2 * a.slot_bytes;
    x.xb = p; p += a.xb_bytes;
    x.hb0 = p; x.hb_stride = a.hb_bytes; p += 2 * a.hb_bytes;
    float* S = reinterpret_cast<float*>(p); p += sizeof(float) * sd * RE;      // env state [k][env]
    float* MU = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 16;     // policy mean
    float* ZS = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 16;     // pre-tanh sample
    float* VV = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 8;      // value
    float* NV = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 8;      // next value
    float* TRK = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 8;     // running returns
    float* LS = reinterpret_cast<float*>(p); p += sizeof(float) * 16;
    uint64_t* EK = reinterpret_cast<uint64_t*>(p); p += 8 * RE;
    uint64_t* EC = reinterpret_cast<uint64_t*>(p); p += 8 * RE;
    int* STP = reinterpret_cast<int*>(p); p += 4 * RE;
    int* NEED = reinterpret_cast<int*>(p); p += 4 * RE;
    int* VF = reinterpret_cast<int*>(p); p += 16;   // vflag of step t (index t & 1)
    x.fullb = reinterpret_cast<uint64_t*>(p); p += 16;
    x.mmad = reinterpret_cast<uint64_t*>(p); p += 8;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(p);
    x.nepad = a.nepad;
    x.issued = x.consumed = 0;

    const float* th = a.theta + (long)c * a.theta_ld;
    const float* ph = a.phi + (long)c * a.phi_ld;
    // zero the operand buffers once: padded K rows / env columns stay zero
    for (int e = tid; e < (a.xb_bytes + 2 * a.hb_bytes) / 16; e += RNT)
        reinterpret_cast<uint4*>(x.xb)[e] = make_uint4(0, 0, 0, 0);
    for (int e = tid; e < sd * nr; e += RNT) {
        const int k = e / nr, r = e % nr;
        S[k * RE + r] = a.state[(long)k * a.N + i0 + r];
    }
    for (int r = tid; r < RE; r += RNT) {
        NEED[r] = 1;
        if (r < nr) {
            EK[r] = a.env_key[i0 + r];
            EC[r] = a.env_ctr[i0 + r];
            STP[r] = a.steps[i0 + r];
            for (int k = 0; k < m; ++k) TRK[r * 8 + k] = a.tracker[(long)(i0 + r) * m + k];
        }
    }
    if (tid < ad) LS[tid] = fminf(fmaxf(th[a.pol.mlp_n + tid], -5.f), 1.f);  // nn.cpp:185-188
    if (tid == 0) { VF[0] = 1; VF[1] = 1; }
    if ((tid >> 5) == 0) umma::tmem_alloc(tslot, 256);
    if (tid == 32) {
        umma::mbar_init(&x.fullb[0], 1);
        umma::mbar_init(&x.fullb[1], 1);
        umma::mbar_init(x.mmad, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    x.tbase = *tslot;
    Issuer is{0, 0};
    if (tid == 0) {
        issue_next(a, x, is, VF, c);
        issue_next(a, x, is, VF, c);
    }
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t xsbo = (uint32_t)a.pol_plan.kin_pad[0] * 16;

#ifdef MB_ROLL_PROF
    unsigned long long prof_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, prof_last_ = gtimer();
#endif
    for (int t = 0; t < a.T; ++t) {
        // ---- observation -> layer-0 operand (bf16, MN-major) + batch.obs
        for (int q = tid; q < nr * 4; q += RNT)  // 4 threads per instance (no div / mod)
            for (int r = q >> 2, k = q & 3; k < od; k += 4) {
                const float v = S[k * RE + r];
                a.obs[((long)(i0 + r) * a.T + t) * od + k] = v;
                *reinterpret_cast<__nv_bfloat16*>(x.xb + (r >> 3) * xsbo + (k >> 3) * 128 + (k & 7) * 16 +
                                                  (r & 7) * 2) = __float2bfloat16_rn(v);
            }
        umma::fence_proxy_async();
        __syncthreads();
        RPROF(0);
        // ---- policy
        run_net(a, x, is, VF, c, 0, th);
        RPROF(1);
        if (warp < 4) {  // M = 64 output layout: env = 16*warp + lane (lanes < 16)
            float v[16];
            umma::tmem_ld16(x.tbase + ((uint32_t)(warp * 32) << 16) + OUT_COL, v);
            const int r = warp * 16 + lane;
            if (lane < 16 && r < nr)
                for (int d = 0; d < ad; ++d) MU[r * 16 + d] = v[d] + th[a.pol.boff[a.pol.L - 1] + d];
        }
        umma::fence_before_sync();
        __syncthreads();
        RPROF(2);
        // ---- Gaussian sample (nn.cpp:192-202): the precomputed draw of (t, instance, dim)
        const float* eps_t = a.eps + ((long)t * a.N + i0) * ad;
        for (int e = tid; e < nr * ad; e += RNT) {
            const int r = e / ad, d = e - r * ad;
            const float sig = __expf(LS[d]);
            const float mu = MU[r * 16 + d];
            const float z = mu + sig * eps_t[e];
            a.act_pre[((long)(i0 + r) * a.T + t) * ad + d] = z;
            // action_logprob's per-dim term (nn.cpp:204-219), summed per row below; the
            // squashed action tanh(z) for the env step: both per (env, dim) item here
            // rather than in the one-thread-per-env loops
            const float zn = (z - mu) / sig;
            MU[r * 16 + d] = (-0.5f * zn * zn - LS[d] - 0.9189385332046727f) - __logf(sech2(z) + 1e-6f);
            ZS[r * 16 + d] = tanhf(z);
        }
        __syncthreads();
        for (int r = tid; r < nr; r += RNT) {  // action_logprob: the dims' terms in order
            float lp = 0.f;
            for (int d = 0; d < ad; ++d) lp += MU[r * 16 + d];
            a.logprob[(long)(i0 + r) * a.T + t] = lp;
        }
        RPROF(3);
        // ---- critic at the current obs, only if some instance reset (or t = 0)
        if (VF[t & 1]) {
            run_net(a, x, is, VF, c, 1, ph);
            if (warp < 4) {
                float v[16];
                umma::tmem_ld16(x.tbase + ((uint32_t)(warp * 32) << 16) + OUT_COL, v);
                const int r = warp * 16 + lane;
                if (lane < 16 && r < nr)
                    for (int k = 0; k < m; ++k) VV[r * 8 + k] = v[k] + ph[a.cri.boff[a.cri.L - 1] + k];
            }
            umma::fence_before_sync();
        }
        __syncthreads();
        RPROF(4);
        // ---- value, env step (env.cpp:60-92), tracker (rollout.cpp:143-148)
        int any_reset = 0;
        for (int r = tid; r < nr; r += RNT) {
            const long row = (long)(i0 + r) * a.T + t;
            for (int k = 0; k < m; ++k) a.value[row * m + k] = NEED[r] ? VV[r * 8 + k] : NV[r * 8 + k];
            float act[16], rw[8];  // compile-time indexed (predicated): registers, not local memory
            bool anyc = false;
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                act[d] = 0.f;
                if (d < ad) {
                    const float xx = ZS[r * 16 + d];  // tanh(z), from the sampling pass
                    if (!isfinite(xx)) atomicExch(a.err, 3);
                    act[d] = fminf(fmaxf(xx, -1.f), 1.f);
                    anyc |= act[d] != xx;
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) rw[k] = 0.f;
            if (anyc) atomicAdd(a.clamp_count, 1ULL);
            float* s = S + r;
            const bool tm = env_do_step(a.kind, s, RE, act, rw);
            const int st = STP[r] + 1;
            const bool tr = !tm && st >= a.max_steps;
            a.term[row] = tm;
            a.trunc[row] = tr;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < m) {
                    a.reward[row * m + k] = rw[k];
                    TRK[r * 8 + k] += rw[k];
                }
            if (tm || tr) {
                double ret = 0.0;
                for (int k = 0; k < m; ++k) {
                    ret += (double)a.cluster_w[c * m + k] * TRK[r * 8 + k];
                    TRK[r * 8 + k] = 0.f;
                }
                a.ret_sum[i0 + r] += ret;
                a.ret_cnt[i0 + r] += 1;
                STP[r] = 0;  // (the reset itself after the final-obs operand pass below)
                NEED[r] = 1;
                any_reset = 1;
            } else {
                STP[r] = st;
                NEED[r] = 0;
            }
        }
        any_reset = __syncthreads_or(any_reset);
        if (tid == 0) VF[(t + 1) & 1] = any_reset;
        // pre-reset final obs -> critic operand, 4 threads per instance
        for (int r = tid >> 2; r < nr; r += RNT / 4)
            for (int k = tid & 3; k < od; k += 4)
                *reinterpret_cast<__nv_bfloat16*>(x.xb + (r >> 3) * xsbo + (k >> 3) * 128 + (k & 7) * 16 +
                                                  (r & 7) * 2) = __float2bfloat16_rn(S[k * RE + r]);
        if (any_reset) {  // auto-reset from the instance's persistent stream (env.cpp:84-92)
            __syncthreads();
            for (int r = tid; r < nr; r += RNT)
                if (NEED[r]) {
                    uint64_t cc = EC[r];
                    env_do_reset(a.kind, S + r, RE, EK[r], &cc);
                    EC[r] = cc;
                }
        }
        umma::fence_proxy_async();
        __syncthreads();
        RPROF(5);
        // ---- critic at the pre-reset final obs -> next_value
        run_net(a, x, is, VF, c, 1, ph);
        RPROF(6);
        if (warp < 4) {
            float v[16];
            umma::tmem_ld16(x.tbase + ((uint32_t)(warp * 32) << 16) + OUT_COL, v);
            const int r = warp * 16 + lane;
            if (lane < 16 && r < nr)
                for (int k = 0; k < m; ++k) {
                    const float nv = v[k] + ph[a.cri.boff[a.cri.L - 1] + k];
                    NV[r * 8 + k] = nv;
                    a.next_value[((long)(i0 + r) * a.T + t) * m + k] = nv;
                }
        }
        umma::fence_before_sync();
        __syncthreads();
    }
#ifdef MB_ROLL_PROF
    if (blockIdx.x == 0 && tid == 0)
        printf("rollout CTA0 us (thread 0's clock): obs %.1f policy %.1f pol_out %.1f sample+logprob(own rows) %.1f "
               "critic_cur(+wait) %.1f env %.1f "
               "critic_final %.1f tail %.1f\n",
               prof_[0] * 1e-3, prof_[1] * 1e-3, prof_[2] * 1e-3, prof_[3] * 1e-3, prof_[4] * 1e-3, prof_[5] * 1e-3,
               prof_[6] * 1e-3, prof_[7] * 1e-3);
#endif
    for (int e = tid; e < sd * nr; e += RNT) {
        const int k = e / nr, r = e % nr;
        a.state[(long)k * a.N + i0 + r] = S[k * RE + r];
    }
    for (int r = tid; r < nr; r += RNT) {
        a.env_ctr[i0 + r] = EC[r];
        a.steps[i0 + r] = STP[r];
        for (int k = 0; k < m; ++k) a.tracker[(long)(i0 + r) * m + k] = TRK[r * 8 + k];
    }
    __syncthreads();
    if (warp == 0) umma::tmem_free(x.tbase, 256);
}

// theta (fp32, reference flat layout) -> bf16 blob in the UMMA K-major image:
// hidden layer l, tile t: rows [128t, 128t+128) x kin_pad(l); output layer:
// 16 rows x kin_pad(L-1). Element (r, k) of a chunk at
// (r/8)*kin_pad*16 + (k/8)*128 + (r%8)*16 + (k%8)*2.
__global__ void k_pack_theta(const float* __restrict__ theta, long P, NetDims nd, NetPlan pl, uint8_t* blob) {
    const int g = blockIdx.y;
    const float* th = theta + (long)g * P;
    uint8_t* out = blob + (long)g * pl.blob_bytes;
    const long units = pl.blob_bytes / 16;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < units; u += (long)gridDim.x * blockDim.x) {
        const long byte = u * 16;
        int c = 0;
        while (c + 1 < pl.nchunks && byte >= pl.chunk_off[c + 1]) ++c;
        const int l = pl.chunk_layer[c], tile = pl.chunk_tile[c];
        const int kin = pl.kin_pad[l];
        const int within = (int)(byte - pl.chunk_off[c]);
        const int rblk = within / (kin * 16), rem = within % (kin * 16);
        const int kb = rem / 128, r8 = (rem % 128) / 16;
        const int row = tile * 128 + rblk * 8 + r8;
        const int in = nd.sz[l], outd = nd.sz[l + 1];
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = kb * 8 + e;
            v[e] = (row < outd && k < in) ? th[nd.woff[l] + (long)row * in + k] : 0.f;
        }
        uint4 q;
        q.x = umma::pack_bf16(v[0], v[1]);
        q.y = umma::pack_bf16(v[2], v[3]);
        q.z = umma::pack_bf16(v[4], v[5]);
        q.w = umma::pack_bf16(v[6], v[7]);
        *reinterpret_cast<uint4*>(out + byte) = q;
    }
}

// one thread per (step, instance, dim): the fp64 Box-Muller draw of words
// 2 (t ad + d) + 1, + 2 of the instance's rollout stream, rounded to fp32
__global__ void k_rollout_noise(uint64_t roll_key, int inst_base, int N, int T, int ad, float* __restrict__ eps) {
    const long n = (long)T * N * ad;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
        const long ti = e / ad;
        const int d = (int)(e - ti * ad);
        const int t = (int)(ti / N), i = (int)(ti - (long)t * N);
        const uint64_t key = split_key(roll_key, (uint64_t)(inst_base + i));  // rollout.cpp:101
        const uint64_t base = 2ull * ((uint64_t)t * ad + d);
        eps[e] = (float)box_muller(rng_word(key, base + 1), rng_word(key, base + 2));
    }
}
}  // namespace

static int pad16(int x) { return (x + 15) / 16 * 16; }
static int pad128(int x) { return (x + 127) / 128 * 128; }

NetPlan make_plan(const NetDims& nd) {
    NetPlan pl{};
    if (nd.L < 2) throw ShapeError("tensor-core rollout needs at least one hidden layer");
    if (nd.sz[nd.L] > 16) throw ShapeError("tensor-core rollout supports output dims <= 16");
    long off = 0;
    int c = 0;
    for (int l = 0; l < nd.L; ++l) {
        pl.kin_pad[l] = l == 0 ? pad16(nd.sz[0]) : pad128(nd.sz[l]);
        if (nd.sz[l + 1] > 256 && l < nd.L - 1) throw ShapeError("tensor-core rollout supports hidden widths <= 256");
        const bool last = l == nd.L - 1;
        pl.tiles[l] = last ? 1 : pad128(nd.sz[l + 1]) / 128;
        for (int t = 0; t < pl.tiles[l]; ++t, ++c) {
            pl.chunk_off[c] = (int)off;
            pl.chunk_bytes[c] = (last ? 16 : 128) * pl.kin_pad[l] * 2;
            pl.chunk_layer[c] = l;
            pl.chunk_tile[c] = t;
            off += pl.chunk_bytes[c];
        }
    }
    pl.nchunks = c;
    pl.blob_bytes = (int)off;
    return pl;
}

void pack_theta(const float* theta, long ld, int G, const NetDims& nd, const NetPlan& pl, uint8_t* blob, cudaStream_t s) {
    dim3 grid((unsigned)((pl.blob_bytes / 16 + 255) / 256), G);
    k_pack_theta<<<grid, 256, 0, s>>>(theta, ld, nd, pl, blob);
    MB_LAUNCH();
}

void rollout_noise(uint64_t roll_key, int inst_base, int N, int T, int ad, float* eps, cudaStream_t s) {
    const long n = (long)T * N * ad;
    if (n == 0) return;
    k_rollout_noise<<<(unsigned)std::min<long>((n + 255) / 256, (long)device_sms() * 16), 256, 0, s>>>(
        roll_key, inst_base, N, T, ad, eps);
    MB_LAUNCH();
}

size_t rollout_tc_smem(const RolloutTcArgs& a) {
    return 2ull * a.slot_bytes + a.xb_bytes + 2ull * a.hb_bytes + sizeof(float) * a.sdim * RE +
           sizeof(float) * RE * (16 + 16 + 8 + 8 + 8) + 64 + 2 * 8 * RE + 2 * 4 * RE + 16 + 16 + 8 + 16;
}

void rollout_tc(RolloutTcArgs a, cudaStream_t s) {
    int slot = 0;
    for (int c = 0; c < a.pol_plan.nchunks; ++c) slot = slot > a.pol_plan.chunk_bytes[c] ? slot : a.pol_plan.chunk_bytes[c];
    for (int c = 0; c < a.cri_plan.nchunks; ++c) slot = slot > a.cri_plan.chunk_bytes[c] ? slot : a.cri_plan.chunk_bytes[c];
    a.slot_bytes = slot;
    a.xb_bytes = RE * a.pol_plan.kin_pad[0] * 2;
    int hmax = 128;
    for (int l = 1; l < a.pol.L; ++l) hmax = hmax > a.pol_plan.kin_pad[l] ? hmax : a.pol_plan.kin_pad[l];
    for (int l = 1; l < a.cri.L; ++l) hmax = hmax > a.cri_plan.kin_pad[l] ? hmax : a.cri_plan.kin_pad[l];
    a.hb_bytes = RE * hmax * 2;
    const int ne = a.reps < RE ? a.reps : RE;
    a.nepad = pad16(ne);
    const size_t bytes = rollout_tc_smem(a);
    if (bytes > 227 * 1024) throw ShapeError("tensor-core rollout: shared-memory plan exceeds 227 KB");
    ensure_smem((const void*)k_rollout_tc, bytes);
    const int cpg = (a.reps + RE - 1) / RE;
    k_rollout_tc<<<a.K * cpg, RNT, bytes, s>>>(a);
    MB_LAUNCH();
}

}  // namespace mb200
