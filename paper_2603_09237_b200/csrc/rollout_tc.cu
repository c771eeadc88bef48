// K3 on the tensor cores: the fused rollout (rollout.cpp:37-161) with every
// policy / critic layer as tcgen05.mma.
//
// * One persistent CTA owns <= 64 instances of ONE preference cluster for
//   all T steps; env state stays in shared memory.
// * The cluster's generated weights theta_c (fp32, from the hypernet GEMM)
//   are packed once per iteration by k_pack_theta into bf16 "blobs" already
//   in the UMMA K-major core-matrix image, one contiguous <= 16 KB chunk per
//   (128-feature tile, 64-wide K piece) of each hidden layer plus one chunk
//   for the output layer. Every step the CTA streams its chunks L2 -> SMEM
//   with the TMA bulk-copy engine (cp.async.bulk, mbarrier complete_tx).
// * Hidden layers: D[feature][env] = W_l (A, K-major) x act^T (B, MN-major),
//   M = 128 features per tile, N = envs; the epilogue (tcgen05.ld) adds the
//   fp32 bias, applies tanh and writes the next layer's bf16 operand, in
//   place (the layer's MMAs have consumed their input when it runs).
// * Output layer: D[env][out] = act (A, MN-major, M = 64 envs) x W_out^T
//   (B, K-major, N = 16), so each env-owning thread gets its own outputs.
// * Warp-specialised, two independent chains per CTA:
//     warps 0-7    policy group: policy epilogues (one 128-feature tile per
//                  warp quadrant pair), Gaussian sample, log-prob, env step,
//                  auto-reset, operand writes (the critical path);
//     warps 8-11   critic group: critic epilogues, value / next value;
//     warps 12/13  policy bulk-copy producer / policy MMA issuer;
//     warps 14/15  critic bulk-copy producer / critic MMA issuer.
//   Each net has its own weight ring and TMEM columns, so the critic at the
//   final observation of step t runs while the policy chain goes on to step
//   t + 1 (both depend only on the env step), and weights of the next pass
//   stream in while the current one computes. All hand-offs are mbarriers
//   (parity-tracked; every buffer a chain reuses is released explicitly).
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
constexpr int RE = 64;           // instances per CTA
constexpr int PGROUP = 256;      // policy group: 8 warps (two per TMEM lane quadrant, one tile each)
constexpr int CGROUP = 128;      // critic group: 4 warps
constexpr int RNT = PGROUP + CGROUP + 128;  // + 4 issue warps
constexpr int W_CRI = PGROUP / 32, W_ISSUE = W_CRI + CGROUP / 32;  // first warp of each role
constexpr int MAX_SLOTS = 4;     // weight-ring slots per net
constexpr int SLOT_MAX = 16384;  // bytes per ring slot (largest chunk)
constexpr uint32_t POL_COL = 0, CRI_COL = 256, OUT_OFF = 128;  // TMEM columns (512 allocated)
constexpr int BAR_POL = 1, BAR_CRI = 2;                        // named barriers of the two groups
// mo-humanoid6 joint scratch in the policy hidden buffer, after the sampling scratch (MU, ZS)
constexpr int H6_SCRATCH_OFF = 2 * RE * 16 * 4, H6_SCRATCH_BYTES = 4 * RE * 12 * 4;

#ifdef MB_ROLL_PROF  // phase timing in CTA 0 (debug builds only: NVCC="nvcc -DMB_ROLL_PROF")
__shared__ unsigned long long g_rp[4][16], g_rp_last[4];  // (CTA 0 prints them)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// thread slot j: 0 policy group thread 0, 2 critic group thread 0
__device__ __forceinline__ int rprof_slot() {
    if (blockIdx.x != 0) return -1;
    return threadIdx.x == 0 ? 0 : threadIdx.x == PGROUP ? 2 : threadIdx.x == (W_ISSUE + 1) * 32 ? 1 : -1;
}
#define RPROF(k)                                          \
    {                                                     \
        const int j_ = rprof_slot();                      \
        if (j_ >= 0) {                                    \
            const unsigned long long now_ = gtimer();     \
            if (g_rp_last[j_]) g_rp[j_][k] += now_ - g_rp_last[j_]; \
            g_rp_last[j_] = now_;                         \
        }                                                 \
    }
#else
#define RPROF(k)
#endif

struct Bars {
    uint64_t pfull[MAX_SLOTS], pempty[MAX_SLOTS], cfull[MAX_SLOTS], cempty[MAX_SLOTS];
    uint64_t pacc, cacc;               // MMA issuer -> group: a layer's accumulators are complete
    uint64_t php, chp;                 // group -> MMA issuer: a layer's epilogue wrote the next operand
    uint64_t xp_ready[2], xp_free[2];  // observation operand of step t (buffer t & 1)
    uint64_t xc_ready, xc_free;        // final-observation operand
    uint64_t vf_ready[2];              // NEED / VF of step s (s & 1) published
    uint64_t cdone[2];                 // critic group done reading NEED / VF of step s
};

struct Ring {
    uint8_t* base;
    uint64_t* full;
    uint64_t* empty;
    int nslots, slot_bytes;
    int slot, round;  // position of the issuing thread
    __device__ __forceinline__ void advance() {
        if (++slot == nslots) {
            slot = 0;
            ++round;
        }
    }
};

// sech^2 z = 4 e / (1 + e)^2, e = exp(-2 |z|) (= 1 - tanh^2 z without its
// cancellation at large |z|); the fast MUFU division: it only feeds a log
__device__ __forceinline__ float sech2(float z) {
    const float e = __expf(-2.f * fabsf(z));
    const float d = 1.f + e;
    return __fdividef(4.f * e, d * d);
}

__device__ __forceinline__ void wait_phase(uint64_t* b, int n) { umma::mbar_wait(b, (uint32_t)(n & 1)); }

// producer warp (converged; one elected lane issues): the bulk copies of
// one pass of a net, in chunk order
__device__ __forceinline__ void produce_pass(const NetPlan& pl, const uint8_t* blob, Ring& r) {
    for (int c = 0; c < pl.nchunks; ++c) {
        if (r.round > 0) wait_phase(&r.empty[r.slot], r.round - 1);  // the MMAs of the slot's last chunk are done
        if (umma::elect_one()) {
            umma::mbar_arrive_expect_tx(&r.full[r.slot], (uint32_t)pl.chunk_bytes[c]);
            umma::bulk_g2s(r.base + r.slot * r.slot_bytes, blob + pl.chunk_off[c], (uint32_t)pl.chunk_bytes[c],
                           &r.full[r.slot]);
        }
        __syncwarp();
        r.advance();
    }
}

// the MMA warp's copy of a net's plan, one chunk per lane (chunks 32.. in
// the second word): nk | k0 / 16 << 5 | tile << 10 | last-of-layer << 15;
// per layer (lanes < 8) the input's padded K x 16 (its 8-env block stride).
// Read with one shuffle per chunk instead of indexed constant loads.
struct LanePlan {
    uint32_t c0, c1, sbo;
};
__device__ __forceinline__ LanePlan lane_plan(const NetPlan& pl, int L, int lane) {
    auto pack = [&](int c) -> uint32_t {
        if (c >= pl.nchunks) return 0u;
        const bool last = c + 1 == pl.nchunks || pl.chunk_layer[c + 1] != pl.chunk_layer[c];
        return (uint32_t)(pl.chunk_kw[c] / 16) | (uint32_t)(pl.chunk_k0[c] / 16) << 5 |
               (uint32_t)pl.chunk_tile[c] << 10 | (last ? 1u : 0u) << 15;
    };
    LanePlan lp;
    lp.c0 = pack(lane);
    lp.c1 = pack(lane + 32);
    lp.sbo = lane < L ? (uint32_t)pl.kin_pad[lane] * 16 : 0u;
    return lp;
}

// MMA warp (converged; one elected lane issues): one pass of a net on the
// operand at smem address `in0`. Layer l > 0 waits for the group's epilogue
// of layer l - 1 (`hready`); each layer ends with a commit to `acc`; the
// layer-0 MMAs also release the input operand through `xfree` (when given).
// Descriptors are built once per chunk and advanced by 256 B (+16 in the
// address field) per K = 16 step.
__device__ __forceinline__ void mma_pass(const LanePlan& lp, int L, Ring& r, uint32_t tbase, uint32_t in0,
                                         uint32_t hb0, int nepad, uint64_t* acc, uint64_t* hready, int& hph,
                                         uint64_t* xfree) {
#ifdef MB_ROLL_PROF
    long long cw_h = 0, cw_f = 0, c_all = clock64();
#endif
    const uint32_t ring0 = umma::smem_u32(r.base);
    int c = 0;
    for (int l = 0; l < L; ++l) {
        if (l > 0) {
#ifdef MB_ROLL_PROF
            const long long q0 = clock64();
#endif
            wait_phase(hready, hph++);
#ifdef MB_ROLL_PROF
            cw_h += clock64() - q0;
#endif
            umma::fence_after_sync();
        }
        const bool last = l == L - 1;
        // input operand at K = 0; its 8-env block stride is this layer's padded K
        const uint64_t in_desc = umma::smem_desc(l == 0 ? in0 : hb0, 128, __shfl_sync(0xffffffffu, lp.sbo, l));
        const uint32_t idesc =
            last ? umma::idesc_bf16(64, 16, true, false) : umma::idesc_bf16(128, nepad, false, true);
        for (;; ++c) {
            const uint32_t info = __shfl_sync(0xffffffffu, c < 32 ? lp.c0 : lp.c1, c & 31);
            const int nk = (int)(info & 31), k0s = (int)((info >> 5) & 31), tile = (int)((info >> 10) & 1);
#ifdef MB_ROLL_PROF
            const long long q0 = clock64();
#endif
            wait_phase(&r.full[r.slot], r.round);
#ifdef MB_ROLL_PROF
            cw_f += clock64() - q0;
#endif
            umma::fence_after_sync();
            // SWIZZLE_NONE descriptor: address >> 4, LBO 128 B, SBO = the chunk's K x 16 B, version 1
            const uint64_t w_desc = (uint64_t)(((ring0 + (uint32_t)(r.slot * r.slot_bytes)) >> 4) & 0x3FFF) |
                                    ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(nk * 16) << 32) | ((uint64_t)1 << 46);
            const uint64_t x_desc = in_desc + (uint64_t)(k0s * 16);  // k0 / 16 steps of 16
            const int k0 = k0s;  // only its zero-ness matters for the accumulate flag
            if (umma::elect_one()) {
                // the common chunk widths as straight-line code: a runtime-trip MMA loop
                // issues at about half the rate (tools/umma_bench.cu)
                if (!last) {
                    const uint32_t d = tbase + (uint32_t)(tile * nepad);
                    if (nk == 4) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma::mma_bf16(d, w_desc + 16 * kk, x_desc + 16 * kk, idesc, (k0 | kk) ? 1u : 0u);
                    } else {
                        for (int kk = 0; kk < nk; ++kk)
                            umma::mma_bf16(d, w_desc + 16 * kk, x_desc + 16 * kk, idesc, (k0 | kk) ? 1u : 0u);
                    }
                } else if (nk == 16) {
#pragma unroll
                    for (int kk = 0; kk < 16; ++kk)
                        umma::mma_bf16(tbase + OUT_OFF, x_desc + 16 * kk, w_desc + 16 * kk, idesc,
                                       (k0 | kk) ? 1u : 0u);
                } else {
                    for (int kk = 0; kk < nk; ++kk)
                        umma::mma_bf16(tbase + OUT_OFF, x_desc + 16 * kk, w_desc + 16 * kk, idesc,
                                       (k0 | kk) ? 1u : 0u);
                }
                umma::commit(&r.empty[r.slot]);
            }
            __syncwarp();
            r.advance();
            if (info >> 15) {
                ++c;
                break;
            }
        }
        if (umma::elect_one()) {
            if (l == 0 && xfree) umma::commit(xfree);
            umma::commit(acc);
        }
        __syncwarp();
    }
#ifdef MB_ROLL_PROF
    if (rprof_slot() == 1) {
        g_rp[1][0] += clock64() - c_all;
        g_rp[1][1] += cw_h;
        g_rp[1][2] += cw_f;
        g_rp[1][3] += 1;
    }
#endif
}

// group epilogue of hidden layer l: bias + tanh -> the next layer's bf16
// operand (MN-major, env x kin_pad(l+1)); zeros in the padded features
__device__ __forceinline__ void hidden_epi(const NetPlan& pl, const NetDims& nd, int l, const float* theta,
                                           uint8_t* hb, uint32_t tacc, int nepad, int gw, int lane, int tile0,
                                           int tstep) {
    const uint32_t osbo = (uint32_t)pl.kin_pad[l + 1] * 16;
    const int out = nd.sz[l + 1];
    for (int tile = tile0; tile < pl.tiles[l]; tile += tstep) {
        const int j = tile * 128 + gw * 32 + lane;
        const bool live = j < out;
        const float bj = live ? theta[nd.boff[l] + j] : 0.f;
        const uint32_t ta = tacc + ((uint32_t)(gw * 32) << 16) + (uint32_t)(tile * nepad);
        uint8_t* ob = hb + (j >> 3) * 128 + (j & 7) * 16;
        for (int n0 = 0; n0 < nepad; n0 += 32) {
            uint32_t v[32];
            const bool two = n0 + 16 < nepad;  // warp-uniform
            umma::tmem_ld16_async(ta + n0, v);
            if (two) umma::tmem_ld16_async(ta + n0 + 16, v + 16);
            umma::tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (h >= 2 && !two) break;
                uint4 q = make_uint4(0, 0, 0, 0);
                if (live) {
                    // MUFU tanh (rel err < 2^-10.99): below the bf16 rounding of the operand
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) f[e] = umma::tanh_approx(__uint_as_float(v[8 * h + e]) + bj);
                    q.x = umma::pack_bf16(f[0], f[1]);
                    q.y = umma::pack_bf16(f[2], f[3]);
                    q.z = umma::pack_bf16(f[4], f[5]);
                    q.w = umma::pack_bf16(f[6], f[7]);
                }
                *reinterpret_cast<uint4*>(ob + ((n0 >> 3) + h) * osbo) = q;
            }
        }
    }
}

// the group's hidden layers of one pass (warp quadrant gw; tiles tile0,
// tile0 + tstep, ...); warps with out_reader get the output layer's 16
// accumulators of env (gw * 16 + lane) (lanes < 16) in v
__device__ __forceinline__ void group_pass(const NetPlan& pl, const NetDims& nd, const float* theta, uint8_t* hb,
                                           uint32_t tacc, int nepad, uint64_t* acc, int& aph, uint64_t* hready,
                                           int gw, int lane, int tile0, int tstep, bool out_reader, int bar,
                                           int nthr, bool leader, float* v) {
    for (int l = 0; l + 1 < nd.L; ++l) {
        RPROF(5);
        wait_phase(acc, aph++);
        RPROF(6);
        umma::fence_after_sync();
        hidden_epi(pl, nd, l, theta, hb, tacc, nepad, gw, lane, tile0, tstep);
        umma::fence_proxy_async();  // generic-proxy operand writes -> the MMA's async proxy
        umma::fence_before_sync();
        umma::bar_sync(bar, nthr);  // the whole group's writes, then one arrival
        if (leader) umma::mbar_arrive(hready);
    }
    RPROF(5);
    wait_phase(acc, aph++);
    RPROF(6);
    if (out_reader) {
        umma::fence_after_sync();
        uint32_t r[16];
        umma::tmem_ld16_async(tacc + OUT_OFF + ((uint32_t)(gw * 32) << 16), r);
        umma::tmem_wait_ld();
        umma::fence_before_sync();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
    }
}

// observation of the instances (state in S) -> bf16 MN-major operands,
// PGROUP / RE threads per instance: xa (all instances, if given) and xb
// plus the batch's obs rows at step t (if given) for the instances whose
// need[] flag equals `sel` (all instances when need is null)
__device__ __forceinline__ void write_operands(const float* S, int nr, int od, uint8_t* xa, uint8_t* xb,
                                               const int* need, int sel, uint32_t xsbo, float* obs_out, long T,
                                               long t, long i0, int gtid) {
    constexpr int TPI = PGROUP / RE;
    for (int r = gtid / TPI; r < nr; r += RE) {
        const bool wb = xb && (!need || need[r] == sel);
        if (!xa && !wb) continue;
        for (int k = gtid % TPI; k < od; k += TPI) {
            const float v = S[k * RE + r];
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const int off = (r >> 3) * xsbo + (k >> 3) * 128 + (k & 7) * 16 + (r & 7) * 2;
            if (xa) *reinterpret_cast<__nv_bfloat16*>(xa + off) = h;
            if (wb) {
                *reinterpret_cast<__nv_bfloat16*>(xb + off) = h;
                if (obs_out) obs_out[((i0 + r) * T + t) * od + k] = v;
            }
        }
    }
}

__global__ void __launch_bounds__(RNT, 1) k_rollout_tc(const __grid_constant__ RolloutTcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int cpg = (a.reps + RE - 1) / RE;
    const int c = blockIdx.x / cpg, ch = blockIdx.x % cpg;
    const int i0 = c * a.reps + ch * RE;
    const int nr = min(RE, a.reps - ch * RE);
    const int od = a.od, ad = a.ad, m = a.m, sd = a.sdim, T = a.T, nepad = a.nepad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- shared memory carve-up (host computes the same total)
    uint8_t* p = smem;
    uint8_t* pring = p; p += a.pol_slots * a.slot_bytes;
    uint8_t* cring = p; p += a.cri_slots * a.slot_bytes;
    uint8_t* xp = p; p += 2 * a.xb_bytes;  // observation operand, by step parity
    uint8_t* xc = p; p += a.xb_bytes;      // final-observation operand
    uint8_t* hp = p; p += a.hb_bytes;      // policy hidden activations (in place across layers)
    uint8_t* hc = p; p += a.hb_bytes;      // critic hidden activations
    float* S = reinterpret_cast<float*>(p); p += sizeof(float) * sd * RE;  // env state [k][env]
    float* TRK = reinterpret_cast<float*>(p); p += sizeof(float) * RE * 8;  // running returns
    float* LS = reinterpret_cast<float*>(p); p += sizeof(float) * 16;
    uint64_t* EK = reinterpret_cast<uint64_t*>(p); p += 8 * RE;
    uint64_t* EC = reinterpret_cast<uint64_t*>(p); p += 8 * RE;
    int* STP = reinterpret_cast<int*>(p); p += 4 * RE;
    int* NEED = reinterpret_cast<int*>(p); p += 4 * 2 * RE;  // [s & 1][env]: reset before step s
    int* VF = reinterpret_cast<int*>(p); p += 16;            // [s & 1]: any NEED at step s
    Bars* B = reinterpret_cast<Bars*>(p); p += sizeof(Bars);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(p);
    // the policy group's sampling scratch lives in its hidden buffer, idle
    // between the output layer and the next layer-0 epilogue
    float* MU = reinterpret_cast<float*>(hp);
    float* ZS = MU + RE * 16;

#ifdef MB_ROLL_PROF
    if (rprof_slot() >= 0) {
        for (int k = 0; k < 16; ++k) g_rp[rprof_slot()][k] = 0;
        g_rp_last[rprof_slot()] = 0;
    }
#endif
    const float* th = a.theta + (long)c * a.theta_ld;
    const float* ph = a.phi + (long)c * a.phi_ld;
    const uint32_t xsbo = (uint32_t)a.pol_plan.kin_pad[0] * 16;
    // zero the operand buffers once: padded K rows / env columns stay zero
    for (int e = tid; e < (3 * a.xb_bytes + 2 * a.hb_bytes) / 16; e += RNT)
        reinterpret_cast<uint4*>(xp)[e] = make_uint4(0, 0, 0, 0);
    for (int e = tid; e < sd * nr; e += RNT) {
        const int k = e / nr, r = e % nr;
        S[k * RE + r] = a.state[(long)k * a.N + i0 + r];
    }
    for (int r = tid; r < RE; r += RNT) {
        NEED[r] = 1;
        NEED[RE + r] = 0;
        if (r < nr) {
            EK[r] = a.env_key[i0 + r];
            EC[r] = a.env_ctr[i0 + r];
            STP[r] = a.steps[i0 + r];
            for (int k = 0; k < m; ++k) TRK[r * 8 + k] = a.tracker[(long)(i0 + r) * m + k];
        }
    }
    if (tid < ad) LS[tid] = fminf(fmaxf(th[a.pol.mlp_n + tid], -5.f), 1.f);  // nn.cpp:185-188
    if (tid == 0) { VF[0] = 1; VF[1] = 0; }
    if (warp == 0) umma::tmem_alloc(tslot, 512);
    if (tid == 32) {
        for (int i = 0; i < MAX_SLOTS; ++i) {
            umma::mbar_init(&B->pfull[i], 1);
            umma::mbar_init(&B->pempty[i], 1);
            umma::mbar_init(&B->cfull[i], 1);
            umma::mbar_init(&B->cempty[i], 1);
        }
        umma::mbar_init(&B->pacc, 1);
        umma::mbar_init(&B->cacc, 1);
        umma::mbar_init(&B->php, 1);
        umma::mbar_init(&B->chp, 1);
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&B->xp_ready[i], 1);
            umma::mbar_init(&B->xp_free[i], 1);
            umma::mbar_init(&B->vf_ready[i], 1);
            umma::mbar_init(&B->cdone[i], 1);
        }
        umma::mbar_init(&B->xc_ready, 1);
        umma::mbar_init(&B->xc_free, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tbase = *tslot;
    const NetPlan& PP = a.pol_plan;
    const NetPlan& CP = a.cri_plan;
    const uint8_t* pblob = a.pol_blob + (long)c * PP.blob_bytes;
    const uint8_t* cblob = a.cri_blob + (long)c * CP.blob_bytes;

    if (warp >= W_ISSUE) {
        // ================= issue warps (converged; elected lanes issue)
        {
            Ring pr{pring, B->pfull, B->pempty, a.pol_slots, a.slot_bytes, 0, 0};
            Ring cr{cring, B->cfull, B->cempty, a.cri_slots, a.slot_bytes, 0, 0};
            if (warp == W_ISSUE) {  // policy producer: P(0..T-1)
                for (int t = 0; t < T; ++t) produce_pass(PP, pblob, pr);
            } else if (warp == W_ISSUE + 1) {  // policy MMA
                int hph = 0;
                const LanePlan plp = lane_plan(PP, a.pol.L, lane);
                for (int t = 0; t < T; ++t) {
                    wait_phase(&B->xp_ready[t & 1], t >> 1);
                    umma::fence_after_sync();
                    mma_pass(plp, a.pol.L, pr, tbase + POL_COL, umma::smem_u32(xp + (t & 1) * a.xb_bytes),
                             umma::smem_u32(hp), nepad, &B->pacc, &B->php, hph, nullptr);
                }
            } else if (warp == W_ISSUE + 2) {  // critic producer: [C_final(s-1)], [C_cur(s) if VF(s)], ..., C_final(T-1)
                for (int s = 0; s < T; ++s) {
                    if (s > 0) produce_pass(CP, cblob, cr);
                    wait_phase(&B->vf_ready[s & 1], s >> 1);
                    if (VF[s & 1]) produce_pass(CP, cblob, cr);
                }
                produce_pass(CP, cblob, cr);
            } else {  // critic MMA, same sequence
                int hph = 0;
                const LanePlan clp = lane_plan(CP, a.cri.L, lane);
                for (int s = 0; s <= T; ++s) {
                    if (s > 0) {
                        wait_phase(&B->xc_ready, s - 1);
                        umma::fence_after_sync();
                        mma_pass(clp, a.cri.L, cr, tbase + CRI_COL, umma::smem_u32(xc), umma::smem_u32(hc), nepad,
                                 &B->cacc, &B->chp, hph, &B->xc_free);
                    }
                    if (s == T) break;
                    wait_phase(&B->vf_ready[s & 1], s >> 1);
                    if (VF[s & 1]) {
                        wait_phase(&B->xp_ready[s & 1], s >> 1);
                        umma::fence_after_sync();
                        mma_pass(clp, a.cri.L, cr, tbase + CRI_COL, umma::smem_u32(xp + (s & 1) * a.xb_bytes),
                                 umma::smem_u32(hc), nepad, &B->cacc, &B->chp, hph, &B->xp_free[s & 1]);
                    } else {
                        if (umma::elect_one()) umma::mbar_arrive(&B->xp_free[s & 1]);
                        __syncwarp();
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp >= W_CRI) {
        // ================= critic group: epilogues, value / next value
        const int gw = warp & 3;
        const bool cleader = tid == PGROUP;
        const int rr = gw * 16 + lane;  // env of this lane in the M = 64 output layout
        const bool own = lane < 16 && rr < nr;
        const float* cb = ph + a.cri.boff[a.cri.L - 1];
        int aph = 0;
        float v[16];
        for (int s = 0; s <= T; ++s) {
            if (s < T) wait_phase(&B->vf_ready[s & 1], s >> 1);  // NEED / VF of step s
            if (s > 0) {  // C_final(s-1) -> next_value[s-1]; value[s] where no reset
                group_pass(CP, a.cri, ph, hc, tbase + CRI_COL, nepad, &B->cacc, aph, &B->chp, gw, lane, 0, 1, true, BAR_CRI,
                           CGROUP, cleader, v);
                if (own) {
                    const long row = (long)(i0 + rr) * T + (s - 1);
                    const bool cont = s < T && !NEED[(s & 1) * RE + rr];
#pragma unroll
                    for (int k = 0; k < 8; ++k)  // compile-time indices: v stays in registers
                        if (k < m) {
                            const float nv = v[k] + cb[k];
                            a.next_value[row * m + k] = nv;
                            if (cont) a.value[(row + 1) * m + k] = nv;
                        }
                }
            }
            if (s == T) break;
            if (VF[s & 1]) {  // C_cur(s) -> value[s] of the instances reset before step s
                group_pass(CP, a.cri, ph, hc, tbase + CRI_COL, nepad, &B->cacc, aph, &B->chp, gw, lane, 0, 1, true, BAR_CRI,
                           CGROUP, cleader, v);
                if (own && NEED[(s & 1) * RE + rr]) {
                    const long row = (long)(i0 + rr) * T + s;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k < m) a.value[row * m + k] = v[k] + cb[k];
                }
            }
            umma::bar_sync(BAR_CRI, CGROUP);  // the group is done with NEED / VF of step s
            if (cleader) umma::mbar_arrive(&B->cdone[s & 1]);
        }
    } else {
        // ================= policy group: the critical path
        const int gtid = tid, gw = warp & 3;
        const int rr = gw * 16 + lane;  // env of this lane in the M = 64 output layout (warps 0-3)
        const float* pb = th + a.pol.boff[a.pol.L - 1];
        int aph = 0;
        float v[16];
        write_operands(S, nr, od, nullptr, xp, nullptr, 0, xsbo, a.obs, T, 0, i0, gtid);
        umma::fence_proxy_async();
        umma::bar_sync(BAR_POL, PGROUP);
        if (gtid == 0) {
            umma::mbar_arrive(&B->xp_ready[0]);
            umma::mbar_arrive(&B->vf_ready[0]);
        }  // NEED / VF of step 0 were set before the sync
        constexpr int EPT = RE * 16 / PGROUP;  // sampling items per thread
        float epsr[EPT];
        auto load_eps = [&](int t) {
            const float* eps_t = a.eps + ((long)t * a.N + i0) * ad;
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const int e = gtid + k * PGROUP;
                epsr[k] = e < nr * ad ? __ldg(eps_t + e) : 0.f;
            }
        };
        load_eps(0);
        // this thread's sampling items (instance, dim) and their step-invariant terms
        int s_row[EPT], s_dim[EPT];
        float s_sig[EPT], s_isig[EPT], s_ls[EPT];
        bool s_ok[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int e = gtid + k * PGROUP;
            s_ok[k] = e < nr * ad;
            const int ee = s_ok[k] ? e : 0;
            s_row[k] = ee / ad;
            s_dim[k] = ee - s_row[k] * ad;
            s_ls[k] = LS[s_dim[k]];
            s_sig[k] = __expf(s_ls[k]);
            s_isig[k] = 1.f / s_sig[k];
        }
        for (int t = 0; t < T; ++t) {
            // ---- policy(obs_t)
            group_pass(PP, a.pol, th, hp, tbase + POL_COL, nepad, &B->pacc, aph, &B->php, gw, lane, warp >> 2, 2,
                       warp < 4, BAR_POL, PGROUP, gtid == 0, v);
            if (warp < 4 && lane < 16 && rr < nr)
#pragma unroll
                for (int d = 0; d < 16; ++d)
                    if (d < ad) MU[rr * 16 + d] = v[d] + pb[d];
            umma::bar_sync(BAR_POL, PGROUP);
            RPROF(1);
            // ---- Gaussian sample (nn.cpp:192-202): the precomputed draw of (t, instance, dim),
            // loaded into registers one step ahead
            // all items' math first (independent chains the compiler can interleave),
            // then the stores of the items that exist
            float s_z[EPT], s_lp[EPT], s_tz[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const float mu = MU[s_row[k] * 16 + s_dim[k]];
                const float z = mu + s_sig[k] * epsr[k];
                // action_logprob's per-dim term (nn.cpp:204-219), summed per row below; the
                // squashed action tanh(z) for the env step
                const float zn = (z - mu) * s_isig[k];
                s_z[k] = z;
                s_lp[k] = (-0.5f * zn * zn - s_ls[k] - 0.9189385332046727f) - __logf(sech2(z) + 1e-6f);
                s_tz[k] = tanhf(z);
            }
#pragma unroll
            for (int k = 0; k < EPT; ++k)
                if (s_ok[k]) {
                    const int r = s_row[k], d = s_dim[k];
                    a.act_pre[((long)(i0 + r) * T + t) * ad + d] = s_z[k];
                    MU[r * 16 + d] = s_lp[k];
                    ZS[r * 16 + d] = s_tz[k];
                }
            RPROF(9);
            if (t + 1 < T) load_eps(t + 1);
            RPROF(10);
            umma::bar_sync(BAR_POL, PGROUP);
            RPROF(2);
            // NEED / VF of step t - 1 are reused for step t + 1: the critic group must be done with them
            if (t > 0) wait_phase(&B->cdone[(t - 1) & 1], (t - 1) >> 1);
            RPROF(7);
            int any_reset = 0;
            // mo-humanoid6 (when the scratch fits the policy hidden buffer): the twelve joints on
            // the instance's 4 threads, the body update / bookkeeping on its first thread
            const bool split = a.kind == ENV_HUMANOID6 && a.hb_bytes >= H6_SCRATCH_OFF + H6_SCRATCH_BYTES;
            float* h6s = reinterpret_cast<float*>(hp + H6_SCRATCH_OFF);  // [4][RE][12]: s_j, e_j, a_j, qd_j
            const int r_own = split ? gtid >> 2 : gtid;
            const bool owner = split ? ((gtid & 3) == 0 && r_own < nr) : gtid < nr;
            bool anyc = false;
            if (split) {
                if (r_own < nr) {
#pragma unroll
                    for (int jj = 0; jj < 3; ++jj) {
                        const int j = (gtid & 3) + 4 * jj;
                        const float xx = ZS[r_own * 16 + j];  // tanh(z), from the sampling pass
                        if (!isfinite(xx)) atomicExch(a.err, 3);
                        const float aj = fminf(fmaxf(xx, -1.f), 1.f);
                        anyc |= aj != xx;
                        float e, qd, sj;
                        h6_joint(S + r_own, RE, j, aj, &e, &qd, &sj);
                        h6s[(0 * RE + r_own) * 12 + j] = sj;
                        h6s[(1 * RE + r_own) * 12 + j] = e;
                        h6s[(2 * RE + r_own) * 12 + j] = aj;
                        h6s[(3 * RE + r_own) * 12 + j] = qd;
                    }
                }
                // the instance's 4 threads are adjacent lanes
                anyc |= __shfl_xor_sync(0xffffffffu, anyc, 1);
                anyc |= __shfl_xor_sync(0xffffffffu, anyc, 2);
                RPROF(11);
                umma::bar_sync(BAR_POL, PGROUP);
                RPROF(12);
            }
            if (owner) {
                const int r = r_own;
                float lp = 0.f;  // action_logprob: the dims' terms in order
                for (int d = 0; d < ad; ++d) lp += MU[r * 16 + d];
                const long row = (long)(i0 + r) * T + t;
                a.logprob[row] = lp;
                RPROF(14);
                // ---- env step (env.cpp:60-92), tracker (rollout.cpp:143-148)
                float rw[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) rw[k] = 0.f;
                bool tm;
                if (split) {
                    tm = h6_body(S + r, RE, h6s + (0 * RE + r) * 12, h6s + (1 * RE + r) * 12,
                                 h6s + (2 * RE + r) * 12, h6s + (3 * RE + r) * 12, 1, rw);
                } else {
                    float act[16];  // compile-time indexed (predicated): registers, not local memory
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
                    tm = env_do_step(a.kind, S + r, RE, act, rw);
                }
                RPROF(15);
                if (anyc) atomicAdd(a.clamp_count, 1ULL);
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
                const bool done = tm || tr;
                if (done) {
                    double ret = 0.0;
                    for (int k = 0; k < m; ++k) {
                        ret += (double)a.cluster_w[c * m + k] * TRK[r * 8 + k];
                        TRK[r * 8 + k] = 0.f;
                    }
                    a.ret_sum[i0 + r] += ret;
                    a.ret_cnt[i0 + r] += 1;
                }
                STP[r] = done ? 0 : st;  // (the reset itself after the final-obs operand pass below)
                NEED[((t + 1) & 1) * RE + r] = done;
                any_reset |= done;
            }
            RPROF(13);
            any_reset = umma::bar_sync_or(BAR_POL, PGROUP, any_reset);
            RPROF(3);
            // ---- pre-reset final obs -> critic operand (once C_final(t-1) has consumed the
            // buffer) and, for the instances that did not reset, obs_{t+1} -> policy operand
            // (buffer (t+1) & 1, once step t-1's readers are done) in the same pass
            const bool nxt = t + 1 < T;
            if (t > 0) wait_phase(&B->xc_free, t - 1);
            if (nxt && t + 1 >= 2) wait_phase(&B->xp_free[(t + 1) & 1], ((t + 1) >> 1) - 1);
            RPROF(8);
            if (gtid == 0) {
                VF[(t + 1) & 1] = any_reset;
                umma::mbar_arrive(&B->vf_ready[(t + 1) & 1]);
            }
            const int* need = NEED + ((t + 1) & 1) * RE;
            uint8_t* xpn = nxt ? xp + ((t + 1) & 1) * a.xb_bytes : nullptr;
            write_operands(S, nr, od, xc, xpn, need, 0, xsbo, a.obs, T, t + 1, i0, gtid);
            umma::fence_proxy_async();
            umma::bar_sync(BAR_POL, PGROUP);
            if (gtid == 0) {
                umma::mbar_arrive(&B->xc_ready);
                if (nxt && !any_reset) umma::mbar_arrive(&B->xp_ready[(t + 1) & 1]);
            }
            if (any_reset) {  // auto-reset from the instance's persistent stream (env.cpp:84-92)
                for (int r = gtid; r < nr; r += PGROUP)
                    if (need[r]) {
                        uint64_t cc = EC[r];
                        env_do_reset(a.kind, S + r, RE, EK[r], &cc);
                        EC[r] = cc;
                    }
                umma::bar_sync(BAR_POL, PGROUP);
                if (nxt) {
                    write_operands(S, nr, od, nullptr, xpn, need, 1, xsbo, a.obs, T, t + 1, i0, gtid);
                    umma::fence_proxy_async();
                    umma::bar_sync(BAR_POL, PGROUP);
                    if (gtid == 0) umma::mbar_arrive(&B->xp_ready[(t + 1) & 1]);
                }
            }
            RPROF(4);
        }
#ifdef MB_ROLL_PROF
        if (blockIdx.x == 0 && gtid == 0) {
            const unsigned long long* q = g_rp[0];
            printf("rollout CTA0 policy group us: out+MU %.1f sample %.1f (math %.1f eps-loads %.1f bar %.1f) "
                   "wait-cdone %.1f env %.1f wait-free %.1f operands+reset %.1f epilogues %.1f wait-acc %.1f\n",
                   q[1] * 1e-3, (q[9] + q[10] + q[2]) * 1e-3, q[9] * 1e-3, q[10] * 1e-3, q[2] * 1e-3, q[7] * 1e-3,
                   q[3] * 1e-3, q[8] * 1e-3, q[4] * 1e-3, q[5] * 1e-3, q[6] * 1e-3);
            printf("rollout CTA0 env: joints %.1f bar %.1f owner: logprob-sum %.1f body %.1f bookkeeping %.1f; "
                   "bar-or %.1f\n", q[11] * 1e-3, q[12] * 1e-3, q[14] * 1e-3, q[15] * 1e-3, q[13] * 1e-3,
                   q[3] * 1e-3);
        }
#endif
        umma::bar_sync(BAR_POL, PGROUP);
        for (int e = gtid; e < sd * nr; e += PGROUP) {
            const int k = e / nr, r = e % nr;
            a.state[(long)k * a.N + i0 + r] = S[k * RE + r];
        }
        for (int r = gtid; r < nr; r += PGROUP) {
            a.env_ctr[i0 + r] = EC[r];
            a.steps[i0 + r] = STP[r];
            for (int k = 0; k < m; ++k) a.tracker[(long)(i0 + r) * m + k] = TRK[r * 8 + k];
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
#ifdef MB_ROLL_PROF
    if (blockIdx.x == 0 && tid == 0) {
        const unsigned long long* q = g_rp[2];
        printf("rollout CTA0 critic group us: epilogues+rest %.1f wait-acc %.1f\n", q[5] * 1e-3, q[6] * 1e-3);
        q = g_rp[1];
        printf("rollout CTA0 policy MMA warp, cycles per pass: total %.0f wait-epilogue %.0f wait-weights %.0f "
               "issue %.0f (%llu passes)\n", (double)q[0] / q[3], (double)q[1] / q[3], (double)q[2] / q[3],
               (double)(q[0] - q[1] - q[2]) / q[3], q[3]);
    }
#endif
    if (warp == 0) umma::tmem_free(tbase, 512);
}

// theta (fp32, reference flat layout) -> bf16 blob in the UMMA K-major image.
// Chunk c holds rows [128 tile, +rows) x K columns [k0, k0 + kw) of its
// layer; element (r, k0 + kk) at (r/8)*kw*16 + (kk/8)*128 + (r%8)*16 + (kk%8)*2.
__global__ void k_pack_theta(const float* __restrict__ theta, long P, NetDims nd, NetPlan pl, uint8_t* blob) {
    const int g = blockIdx.y;
    const float* th = theta + (long)g * P;
    uint8_t* out = blob + (long)g * pl.blob_bytes;
    const long units = pl.blob_bytes / 16;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < units; u += (long)gridDim.x * blockDim.x) {
        const long byte = u * 16;
        int lo = 0, hi = pl.nchunks - 1;  // last chunk with chunk_off <= byte
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pl.chunk_off[mid] <= byte) lo = mid; else hi = mid - 1;
        }
        const int c = lo;
        const int l = pl.chunk_layer[c], tile = pl.chunk_tile[c];
        const int kw = pl.chunk_kw[c], k0 = pl.chunk_k0[c];
        const int within = (int)(byte - pl.chunk_off[c]);
        const int rblk = within / (kw * 16), rem = within % (kw * 16);
        const int kb = rem / 128, r8 = (rem % 128) / 16;
        const int row = tile * 128 + rblk * 8 + r8;
        const int in = nd.sz[l], outd = nd.sz[l + 1];
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = k0 + kb * 8 + e;
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
        const int rows = last ? 16 : 128;
        const int kwmax = SLOT_MAX / (rows * 2);  // a chunk fills at most one ring slot
        pl.tiles[l] = last ? 1 : pad128(nd.sz[l + 1]) / 128;
        for (int t = 0; t < pl.tiles[l]; ++t)
            for (int k0 = 0; k0 < pl.kin_pad[l]; k0 += kwmax, ++c) {
                if (c >= ROLL_MAX_CHUNKS) throw ShapeError("tensor-core rollout: too many weight chunks");
                const int kw = std::min(kwmax, pl.kin_pad[l] - k0);
                pl.chunk_off[c] = (int)off;
                pl.chunk_bytes[c] = rows * kw * 2;
                pl.chunk_layer[c] = l;
                pl.chunk_tile[c] = t;
                pl.chunk_k0[c] = k0;
                pl.chunk_kw[c] = kw;
                pl.max_chunk = std::max(pl.max_chunk, pl.chunk_bytes[c]);
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

// everything but the two weight rings
static size_t rollout_fixed_smem(const RolloutTcArgs& a) {
    return 3ull * a.xb_bytes + 2ull * a.hb_bytes + sizeof(float) * a.sdim * RE + sizeof(float) * RE * 8 +
           sizeof(float) * 16 + 2 * 8 * RE + 4 * RE + 4 * 2 * RE + 16 + sizeof(Bars) + 16;
}

void rollout_tc(RolloutTcArgs a, cudaStream_t s) {
    if (a.T <= 0 || a.K <= 0) return;
    if (a.pol_plan.kin_pad[0] != a.cri_plan.kin_pad[0])
        throw ShapeError("tensor-core rollout: policy and critic inputs differ");
    a.slot_bytes = std::max(a.pol_plan.max_chunk, a.cri_plan.max_chunk);
    a.xb_bytes = RE * a.pol_plan.kin_pad[0] * 2;
    int hmax = 128;
    for (int l = 1; l < a.pol.L; ++l) hmax = std::max(hmax, a.pol_plan.kin_pad[l]);
    for (int l = 1; l < a.cri.L; ++l) hmax = std::max(hmax, a.cri_plan.kin_pad[l]);
    a.hb_bytes = RE * hmax * 2;
    const int ne = a.reps < RE ? a.reps : RE;
    a.nepad = pad16(ne);
    const size_t limit = 227 * 1024, fixed = rollout_fixed_smem(a);
    const int slots = fixed < limit ? (int)((limit - fixed) / a.slot_bytes) : 0;
    a.pol_slots = std::min(MAX_SLOTS, (slots + 1) / 2);  // the policy chain is the critical path
    a.cri_slots = std::min(MAX_SLOTS, slots - a.pol_slots);
    if (a.cri_slots < 2) throw ShapeError("tensor-core rollout: shared-memory plan exceeds 227 KB");
    const size_t bytes = fixed + (size_t)(a.pol_slots + a.cri_slots) * a.slot_bytes;
    ensure_smem((const void*)k_rollout_tc, bytes);
    const int cpg = (a.reps + RE - 1) / RE;
    k_rollout_tc<<<a.K * cpg, RNT, bytes, s>>>(a);
    MB_LAUNCH();
}

}  // namespace mb200
