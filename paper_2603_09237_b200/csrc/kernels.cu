// Device kernels of the MORLAX B200 training step (everything except the
// GEMMs and Pareto): K1 env step, K3 fused rollout, K4 GAE scan +
// normalise/scalarise, K5 per-row PPO losses, K7 Adam, reductions.
// Reference semantics are cited per kernel (paths under /root/reference/proj).
#include <map>
#include <mutex>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

std::atomic<long> g_kernel_launches{0};
int device_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 0;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = sms;
    return sms;
}
void ensure_smem(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cache;
    int dev = 0;
    MB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = cache[{dev, func}];
    if (bytes <= have) return;
    MB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
}
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MORLAX_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// =========================================================================
// K1: BatchedEnv reset / step (env.cpp:44-106). SoA state [sdim][N].
// =========================================================================
__global__ void k_env_reset(int kind, int N, float* state, uint64_t* keys, uint64_t* ctrs, int* steps,
                            uint64_t parent, int base) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint64_t k = split_key(parent, (uint64_t)(base + i));  // env.cpp:53-54 (global lane)
    uint64_t c = 0;
    env_do_reset(kind, state + i, N, k, &c);
    keys[i] = k;
    ctrs[i] = c;
    steps[i] = 0;
}

__global__ void k_env_step(int kind, int N, int ad, int od, int m, int max_steps, float* state,
                           uint64_t* keys, uint64_t* ctrs, int* steps, const float* actions, float* obs,
                           float* reward, uint8_t* term, uint8_t* trunc,
                           unsigned long long* clamp_count, int* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    float a[16], r[8];
    bool any = false;
    for (int d = 0; d < ad; ++d) {  // env.cpp:63-72
        const float x = actions[(long)i * ad + d];
        if (!isfinite(x)) atomicExch(err, 3);
        a[d] = fminf(fmaxf(x, -1.f), 1.f);
        any |= a[d] != x;
    }
    if (any) atomicAdd(clamp_count, 1ULL);
    float* s = state + i;
    const bool t = env_do_step(kind, s, N, a, r);
    const int st = steps[i] + 1;
    const bool tr = !t && st >= max_steps;  // env.cpp:80
    for (int k = 0; k < m; ++k) reward[(long)i * m + k] = r[k];
    term[i] = t;
    trunc[i] = tr;
    for (int k = 0; k < od; ++k) obs[(long)i * od + k] = s[(long)k * N];  // pre-reset final obs
    if (t || tr) {
        uint64_t c = ctrs[i];
        env_do_reset(kind, s, N, keys[i], &c);
        ctrs[i] = c;
        steps[i] = 0;
    } else {
        steps[i] = st;
    }
}

__global__ void k_env_obs(int N, int od, const float* state, float* obs) {
    const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (e >= (long)N * od) return;
    const int i = e / od, k = e % od;
    obs[e] = state[(long)k * N + i];
}

void env_reset(int kind, int N, float* state, uint64_t* keys, uint64_t* ctrs, int* steps,
               uint64_t parent_key, int inst_base, cudaStream_t s) {
    k_env_reset<<<(N + 255) / 256, 256, 0, s>>>(kind, N, state, keys, ctrs, steps, parent_key, inst_base);
    MB_LAUNCH();
}
void env_step(int kind, int N, float* state, uint64_t* keys, uint64_t* ctrs, int* steps,
              const float* actions, float* obs, float* reward, uint8_t* term, uint8_t* trunc,
              unsigned long long* clamp_count, int* err, cudaStream_t s) {
    const EnvSpecB es = env_spec_of(kind);
    k_env_step<<<(N + 255) / 256, 256, 0, s>>>(kind, N, es.act_dim, es.obs_dim, es.m, es.max_steps,
                                                state, keys, ctrs, steps, actions, obs, reward, term,
                                                trunc, clamp_count, err);
    MB_LAUNCH();
}
void env_obs(int kind, int N, const float* state, float* obs, cudaStream_t s) {
    const int od = env_spec_of(kind).obs_dim;
    k_env_obs<<<(int)(((long)N * od + 255) / 256), 256, 0, s>>>(N, od, state, obs);
    MB_LAUNCH();
}

__device__ __forceinline__ float sech2_f(float z) {
    // 1 - tanh(z)^2 without cancellation: 4 e^{-2|z|} / (1 + e^{-2|z|})^2
    const float e = __expf(-2.f * fabsf(z));
    const float d = 1.f + e;
    return __fdividef(4.f * e, d * d);  // the fast MUFU division: it only feeds a log
}

// =========================================================================
// K4: per-objective GAE (gae.cpp:26-66) as a warp-shuffle scan over T.
// One warp per (instance, objective). The backward recurrence
// A_t = delta_t + c_t A_{t+1} is an affine map per step; each lane composes
// its time chunk, a suffix scan of (C, D) pairs across lanes supplies the
// carry, and the lane replays its chunk.
// =========================================================================
__global__ void k_gae(int N, int T, int m, const float* __restrict__ rew, const float* __restrict__ val,
                      const float* __restrict__ nval, const uint8_t* __restrict__ term,
                      const uint8_t* __restrict__ trunc, float gamma, float lambda, float* adv,
                      float* tgt) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= N * m) return;
    const int i = warp / m, k = warp % m;
    const int tc = (T + 31) / 32;
    const int t0 = min(T, lane * tc), t1 = min(T, t0 + tc);
    const float gl = gamma * lambda;
    float C = 1.f, D = 0.f;
    for (int t = t1 - 1; t >= t0; --t) {  // compose f_t o (current): x -> delta + c x
        const long r = (long)i * T + t;
        const float boot = term[r] ? 0.f : 1.f;
        const float cont = (term[r] || trunc[r]) ? 0.f : 1.f;
        const long idx = r * m + k;
        const float delta = rew[idx] + gamma * nval[idx] * boot - val[idx];
        const float c = gl * cont;
        D = delta + c * D;
        C = c * C;
    }
    // inclusive suffix scan: lane L <- f_L o f_{L+1} o ... o f_31
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float C2 = __shfl_down_sync(0xffffffffu, C, off);
        const float D2 = __shfl_down_sync(0xffffffffu, D, off);
        if (lane + off < 32) {
            D = D + C * D2;
            C = C * C2;
        }
    }
    float carry = __shfl_down_sync(0xffffffffu, D, 1);
    if (lane == 31) carry = 0.f;
    for (int t = t1 - 1; t >= t0; --t) {
        const long r = (long)i * T + t;
        const float boot = term[r] ? 0.f : 1.f;
        const float cont = (term[r] || trunc[r]) ? 0.f : 1.f;
        const long idx = r * m + k;
        const float delta = rew[idx] + gamma * nval[idx] * boot - val[idx];
        carry = delta + gl * cont * carry;
        adv[idx] = carry;
        tgt[idx] = carry + val[idx];
    }
}

// The same recurrence for short horizons, one block per kGaeInst instances:
// their T x m blocks of every input (contiguous in the row-major [row][m]
// layout) are staged through shared memory with coalesced loads, then one
// thread per (instance, objective) runs the backward recurrence
// sequentially from shared memory (instance stride padded so the m x
// kGaeInst threads hit distinct banks), and advantages / targets leave with
// coalesced stores. (The warp-scan kernel above reads m-strided words and
// spends its issue slots on shuffles; at T = 64 the sequential pass is
// shorter than the scan.) Same arithmetic per (instance, objective).
constexpr int kGaeInst = 8;
__global__ void __launch_bounds__(256) k_gae_inst(int N, int T, int m, int stride, const float* __restrict__ rew,
                                                   const float* __restrict__ val, const float* __restrict__ nval,
                                                   const uint8_t* __restrict__ term,
                                                   const uint8_t* __restrict__ trunc, float gamma, float lambda,
                                                   float* adv, float* tgt) {
    extern __shared__ float gsm[];
    const int tm = T * m;
    float* R = gsm;  // rew -> adv
    float* V = R + kGaeInst * stride;
    float* X = V + kGaeInst * stride;  // next value -> target
    uint8_t* FL = reinterpret_cast<uint8_t*>(X + kGaeInst * stride);  // bit 0 term, bit 1 trunc
    const int i0 = blockIdx.x * kGaeInst;
    const int ni = min(kGaeInst, N - i0);
    const long b = (long)i0 * tm;
    const int n = ni * tm;
    for (int e0 = 0; e0 < n; e0 += 256 * 4) {  // 12 loads in flight per thread before the smem stores
        float lr[4], lv[4], lx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * 256 + threadIdx.x;
            if (e < n) {
                lr[u] = rew[b + e];
                lv[u] = val[b + e];
                lx[u] = nval[b + e];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * 256 + threadIdx.x;
            if (e < n) {
                const int w = e / tm, o = w * stride + (e - w * tm);
                R[o] = lr[u];
                V[o] = lv[u];
                X[o] = lx[u];
            }
        }
    }
    for (int e = threadIdx.x; e < ni * T; e += blockDim.x)
        FL[e] = (term[(long)i0 * T + e] ? 1 : 0) | (trunc[(long)i0 * T + e] ? 2 : 0);
    __syncthreads();
    if (threadIdx.x < ni * m) {
        const int w = threadIdx.x / m, k = threadIdx.x - w * m;
        float* r = R + w * stride + k;
        const float* v = V + w * stride + k;
        float* x = X + w * stride + k;
        const uint8_t* fl = FL + w * T;
        const float gl = gamma * lambda;
        float carry = 0.f;  // gae.cpp:40-60
#pragma unroll 8
        for (int t = T - 1; t >= 0; --t) {
            const int f = fl[t];
            const float boot = (f & 1) ? 0.f : 1.f;
            const float cont = f ? 0.f : 1.f;
            const float vt = v[t * m];
            const float delta = r[t * m] + gamma * x[t * m] * boot - vt;
            carry = delta + gl * cont * carry;
            r[t * m] = carry;
            x[t * m] = carry + vt;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ni * tm; e += blockDim.x) {
        const int w = e / tm, o = w * stride + (e - w * tm);
        adv[b + e] = R[o];
        tgt[b + e] = X[o];
    }
}

void gae_scan(int N, int T, int m, const float* reward, const float* value, const float* next_value,
              const uint8_t* term, const uint8_t* trunc, float gamma, float lambda, float* adv,
              float* targets, cudaStream_t s) {
    const int tm = T * m, stride = tm + ((m - tm) % 32 + 32) % 32;  // stride = m (mod 32)
    const size_t sm = sizeof(float) * 3 * (size_t)kGaeInst * stride + (size_t)kGaeInst * T;
    if (T <= 256 && m * kGaeInst <= 256 && sm <= 48 * 1024) {
        k_gae_inst<<<(N + kGaeInst - 1) / kGaeInst, 256, sm, s>>>(N, T, m, stride, reward, value, next_value, term,
                                                                   trunc, gamma, lambda, adv, targets);
        MB_LAUNCH();
        return;
    }
    const long warps = (long)N * m;
    k_gae<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(N, T, m, reward, value, next_value, term,
                                                          trunc, gamma, lambda, adv, targets);
    MB_LAUNCH();
}

// Normalisation statistics (gae.cpp:79-96): deterministic fp64 reductions in
// a fixed two-level order that does not depend on how the rows are spread
// over GPUs: one partial per group of consecutive rows (a preference
// cluster's reps * T rows in the trainer: whole clusters live on one rank),
// then the group partials summed in group order. pass 1 (mean == nullptr):
// sum x; pass 2: sum (x - mean)^2.
__global__ void __launch_bounds__(256) k_chan_part(const float* __restrict__ x, long rows_per_group, int m,
                                                   const double* mean, double* part) {
    __shared__ double red[256 * 8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const float* xg = x + (long)blockIdx.x * rows_per_group * m;
    double mu[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) mu[k] = (mean && k < m) ? mean[k] : 0.0;
    for (long r = threadIdx.x; r < rows_per_group; r += blockDim.x)
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < m) {
                double v = xg[r * m + k];
                if (mean) {
                    v -= mu[k];
                    v *= v;
                }
                acc[k] += v;
            }
#pragma unroll
    for (int k = 0; k < 8; ++k) red[k * 256 + threadIdx.x] = acc[k];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int k = 0; k < m; ++k) red[k * 256 + threadIdx.x] += red[k * 256 + threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 8) part[blockIdx.x * 8 + threadIdx.x] = threadIdx.x < m ? red[threadIdx.x * 256] : 0.0;
}
// out[k] = sum_g part[g][k]: warp k, lane-strided partial sums in g order,
// then a fixed butterfly (the same order for any group count split)
__global__ void k_chan_total(const double* __restrict__ part, int groups, int m, double* out) {
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (k >= m) return;
    double s = 0.0;
    for (int g = lane; g < groups; g += 32) s += part[g * 8 + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[k] = s;
}
void channel_partials(const float* x, int groups, long rows_per_group, int m, const double* mean, double* part,
                      cudaStream_t s) {
    if (m > 8) throw ShapeError("normalize: at most 8 objectives on the device");
    if (groups <= 0) return;
    k_chan_part<<<groups, 256, 0, s>>>(x, rows_per_group, m, mean, part);
    MB_LAUNCH();
}
void channel_total(const double* part, int groups, int m, double* out, cudaStream_t s) {
    k_chan_total<<<1, 256, 0, s>>>(part, groups, m, out);
    MB_LAUNCH();
}

__global__ void k_stats_finalize(const double* s, double rows, int m, double* out, int mode) {
    const int k = threadIdx.x;
    if (k >= m) return;
    out[k] = mode == 0 ? s[k] / rows : 1.0 / (sqrt(s[k] / rows) + 1e-8);  // gae.cpp:91-96
}
void stats_finalize(const double* sums, double rows, int m, double* out, int mode, cudaStream_t s) {
    k_stats_finalize<<<1, 32, 0, s>>>(sums, rows, m, out, mode);
    MB_LAUNCH();
}

// scalarise (gae.cpp:98-115): s = sum_k w_k (A_k - mu_k) inv_k
__global__ void k_scalarize(int N, int T, int m, const float* adv, const float* cw, int reps,
                            const double* mean, const double* inv, float* out) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= (long)N * T) return;
    const int i = r / T, c = i / reps;
    double s = 0.0;
    for (int k = 0; k < m; ++k) s += (double)cw[c * m + k] * (((double)adv[r * m + k] - mean[k]) * inv[k]);
    out[r] = (float)s;
}
void scalarize(int N, int T, int m, const float* adv, const float* cluster_w, int reps,
               const double* mean, const double* inv_std, float* sadv, cudaStream_t s) {
    const long R = (long)N * T;
    k_scalarize<<<(int)((R + 255) / 256), 256, 0, s>>>(N, T, m, adv, cluster_w, reps, mean, inv_std, sadv);
    MB_LAUNCH();
}

__global__ void k_check_finite(const double* x, int n, int* err, int code) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && !isfinite(x[i])) atomicExch(err, code);
}
void check_finite_f64(const double* x, int n, int* err, int code, cudaStream_t s) {
    k_check_finite<<<(n + 255) / 256, 256, 0, s>>>(x, n, err, code);
    MB_LAUNCH();
}

// image-output variants (tcgen05 update path): one block = one 128-row tile;
// padded rows (rows[q] < 0) get zero loss and zero gradient. Per-tile column
// sums of the output gradient (bias grads) and of the log-std terms go to
// psum / psls [tile][16] (deterministic, summed per cluster by k_segsum_multi);
// loss_rows[tile] = the tile's loss sum (fp64).
__device__ __forceinline__ void tile_colsum(const float* g, int width, float* red, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = 0; d < width; ++d) {
        float x = g[d];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[warp * 16 + d] = x;
    }
    __syncthreads();
    if (threadIdx.x < width) out[threadIdx.x] = red[threadIdx.x] + red[16 + threadIdx.x] + red[32 + threadIdx.x] +
                                                red[48 + threadIdx.x];
    __syncthreads();
}

// fp64 sum of one value per thread of a 128-thread block -> *out (thread 0)
__device__ __forceinline__ void tile_sum_f64(double x, double* out) {
    __shared__ double wsum[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) *out = (wsum[0] + wsum[1]) + (wsum[2] + wsum[3]);
}

__global__ void __launch_bounds__(128) k_actor_rows_img(int ad, const int* rows, const int* rg, const float* theta,
                                                        long P, long mlp_n, const float* mu, int ldmu,
                                                        const float* z, const float* lp_old, const float* sadv,
                                                        float clip, float ent, float inv_B, Img gimg, float* psum,
                                                        float* psls, double* loss_rows, int* err) {
    __shared__ float red[64];
    const int q = blockIdx.x * 128 + threadIdx.x;
    float g[16], gl[16];
    for (int d = 0; d < 16; ++d) g[d] = gl[d] = 0.f;
    double lrow = 0.0;
    if (rows[q] >= 0) {
        const float* th = theta + (long)rg[q] * P + mlp_n;
        float lp = 0.f, ls[16], zn[16], sig[16], ent_h = 0.f;
        for (int d = 0; d < ad; ++d) {  // action_logprob (nn.cpp:204-219)
            ls[d] = fminf(fmaxf(th[d], -5.f), 1.f);
            sig[d] = __expf(ls[d]);
            const float zz = z[(long)q * ad + d];
            zn[d] = (zz - mu[(long)q * ldmu + d]) / sig[d];
            lp += -0.5f * zn[d] * zn[d] - ls[d] - 0.9189385332046727f;
            lp -= __logf(sech2_f(zz) + 1e-6f);
            ent_h += ls[d] + 0.5f * (1.f + 1.8378770664093453f);
        }
        const float ratio = __expf(lp - lp_old[q]);
        if (!isfinite(ratio)) atomicExch(err, 3);
        const float adv = sadv[q];
        const float unc = ratio * adv;
        const float clp = fminf(fmaxf(ratio, 1.f - clip), 1.f + clip) * adv;
        lrow = (double)(-fminf(unc, clp) * inv_B) - (double)(ent * ent_h * inv_B);
        const float glp = unc <= clp ? -ratio * adv * inv_B : 0.f;  // losses.cpp:116
        for (int d = 0; d < ad; ++d) {
            g[d] = glp * zn[d] / sig[d];
            const float raw = th[d];  // clamp mask (losses.cpp:124-128)
            gl[d] = (raw >= -5.f && raw <= 1.f) ? glp * (zn[d] * zn[d] - 1.f) - ent * inv_B : 0.f;
        }
    }
    tile_sum_f64(lrow, loss_rows + blockIdx.x);  // per-tile loss partial
    const int CT = img_ct(gimg.C);
    for (int h = 0; h < (ad + 7) / 8; ++h) {
        uint4 w;
        w.x = umma::pack_bf16(g[8 * h + 0], g[8 * h + 1]);
        w.y = umma::pack_bf16(g[8 * h + 2], g[8 * h + 3]);
        w.z = umma::pack_bf16(g[8 * h + 4], g[8 * h + 5]);
        w.w = umma::pack_bf16(g[8 * h + 6], g[8 * h + 7]);
        *reinterpret_cast<uint4*>(gimg.p + img_off(q, 8 * h, CT)) = w;
    }
    tile_colsum(g, ad, red, psum + blockIdx.x * 16);
    tile_colsum(gl, ad, red, psls + blockIdx.x * 16);
}
void actor_rows_img(int Bp, int ad, const int* rows, const int* row_group, const float* theta, long P, long mlp_n,
                    const float* mu, int ldmu, const float* z, const float* lp_old, const float* sadv, float clip,
                    float ent, float inv_B, const Img& g_out, float* psum, float* psls, double* loss_rows, int* err,
                    cudaStream_t s) {
    k_actor_rows_img<<<Bp / 128, 128, 0, s>>>(ad, rows, row_group, theta, P, mlp_n, mu, ldmu, z, lp_old, sadv, clip,
                                              ent, inv_B, g_out, psum, psls, loss_rows, err);
    MB_LAUNCH();
}

__global__ void __launch_bounds__(128) k_critic_rows_img(int m, const int* rows, const float* v, int ldv,
                                                         const float* tgt, float inv_B, Img gimg, float* psum,
                                                         double* loss_rows) {
    __shared__ float red[64];
    const int q = blockIdx.x * 128 + threadIdx.x;
    float g[16];
    for (int k = 0; k < 16; ++k) g[k] = 0.f;
    double l = 0.0;
    if (rows[q] >= 0)
        for (int k = 0; k < m; ++k) {
            const float e = v[(long)q * ldv + k] - tgt[(long)q * m + k];
            l += (double)e * e * inv_B;
            g[k] = 2.f * e * inv_B;  // losses.cpp:179-181 (no 1/2)
        }
    tile_sum_f64(l, loss_rows + blockIdx.x);  // per-tile loss partial
    const int CT = img_ct(gimg.C);
    for (int h = 0; h < (m + 7) / 8; ++h) {
        uint4 w;
        w.x = umma::pack_bf16(g[8 * h + 0], g[8 * h + 1]);
        w.y = umma::pack_bf16(g[8 * h + 2], g[8 * h + 3]);
        w.z = umma::pack_bf16(g[8 * h + 4], g[8 * h + 5]);
        w.w = umma::pack_bf16(g[8 * h + 6], g[8 * h + 7]);
        *reinterpret_cast<uint4*>(gimg.p + img_off(q, 8 * h, CT)) = w;
    }
    tile_colsum(g, m, red, psum + blockIdx.x * 16);
}
void critic_rows_img(int Bp, int m, const int* rows, const float* v, int ldv, const float* tgt, float inv_B,
                     const Img& g_out, float* psum, double* loss_rows, cudaStream_t s) {
    k_critic_rows_img<<<Bp / 128, 128, 0, s>>>(m, rows, v, ldv, tgt, inv_B, g_out, psum, loss_rows);
    MB_LAUNCH();
}

// =========================================================================
// K5 head: the output layer of the generated MLP, the per-row loss and the
// output layer's backward in one pass over a 128-row tile of one cluster
// (losses.cpp:87-132 / 165-185 with nn.cpp:60-92, 111-160 for the last
// layer):
//   o      = b_L + W_L a          (a = last hidden activation row, bf16 image)
//   g      = dloss/do             (actor: clipped surrogate + entropy;
//                                  critic: 2 e / B)
//   g_prev = (W_L^T g) * (1 - a^2)  -> bf16 image (input of the dW / dX GEMMs)
// plus per-tile column sums of g (output bias grads), of the log-std terms
// and of g_prev (bias grads of the last hidden layer), and the tile's loss.
// The output layer is only act_dim / m (<= 16) wide: both contractions run
// on mma.sync m16n8k16 (bf16 operands, fp32 accumulation), each warp owning
// two 16-row m-tiles. tcgen05 would accept the shape (M = 128, N = 16), but
// the kernel is bound by the activation-image read and the per-row loss
// math: ~12 x 256 MACs per row fill the tensor pipe for a few % of the
// kernel either way, and register fragments loaded straight from the image
// need no shared-memory staging, TMEM allocation or commit round trips.
// The accumulator fragment of the forward (rows x out) is exactly the A
// fragment of the backward (rows x K = out), and the forward's A fragments
// (the activations) are exactly the tanh' operands of the backward's
// accumulator, so the activations are read once and nothing is staged.
// In the forward W_L enters as a two-term bf16 split (hi + lo: ~16 mantissa
// bits, the accuracy of the fp32 SIMT form this replaced -- the PPO ratio is
// sensitive to the output mean; the activations are the bf16 image either
// way); the backward uses bf16 g and W_L like the other data-gradient GEMMs.
// W_L sits in shared memory in fragment order for both products. Padded rows
// (rows[q] < 0) contribute zeros.
// =========================================================================
__device__ __forceinline__ void mma_bf16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t bf2_pack(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// the bf16 residual x - bf16(x) (the "lo" half of a two-term bf16 split)
__device__ __forceinline__ float bf_lo(float x) { return x - __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float2 bf2_unpack(uint32_t u) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}

// NT = n-tiles of the output (out <= 8 * NT)
template <bool ACTOR, int NT>
__global__ void __launch_bounds__(128, 4) k_head(HeadArgs a) {
    // forward W_L = hi + lo (two bf16 terms: ~16 mantissa bits, as the fp32
    // form this replaced: the PPO ratio is sensitive to the output mean)
    __shared__ uint2 swf[2][16][NT][32];  // forward B: (k = h pair, n = d) per k-step / n-tile / lane
    __shared__ uint2 swb[32][32];         // backward B: (k = d pair, n = h) per h n-tile / lane
    __shared__ float sb[16], red[4][16], redl[4][16];
    __shared__ float red2[4][256];
    pdl_enter();
    const int H = a.H, out = a.out, KS = H >> 4, HT = H >> 3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, rq = lane >> 2, q = lane & 3;
    const int z = a.rg[blockIdx.x * 128];  // groups are 128-row padded: one cluster per tile
    const float* th = a.theta + (long)z * a.ld;
    const float* W = th + a.woff;  // W_L [out][H] fp32
    for (int e = threadIdx.x; e < KS * NT * 32; e += 128) {
        const int l = e & 31, j = (e >> 5) % NT, st = e / (32 * NT);
        const int n = j * 8 + (l >> 2), k = st * 16 + 2 * (l & 3);
        float w0 = 0.f, w1 = 0.f, w8 = 0.f, w9 = 0.f;
        if (n < out) {
            w0 = W[(long)n * H + k]; w1 = W[(long)n * H + k + 1];
            w8 = W[(long)n * H + k + 8]; w9 = W[(long)n * H + k + 9];
        }
        swf[0][st][j][l] = make_uint2(bf2_pack(w0, w1), bf2_pack(w8, w9));
        swf[1][st][j][l] = make_uint2(bf2_pack(bf_lo(w0), bf_lo(w1)), bf2_pack(bf_lo(w8), bf_lo(w9)));
    }
    for (int e = threadIdx.x; e < HT * 32; e += 128) {
        const int l = e & 31, nt = e >> 5;
        const int hcol = nt * 8 + (l >> 2), d = 2 * (l & 3);
        auto w = [&](int dd) { return dd < out ? W[(long)dd * H + hcol] : 0.f; };
        swb[nt][l] = make_uint2(bf2_pack(w(d), w(d + 1)), bf2_pack(w(d + 8), w(d + 9)));
    }
    __shared__ float sinv[16], smask[16], sconst[2];  // actor: 1 / sigma_d, clamp mask; sum_d lp / entropy terms
    if (threadIdx.x < 16) {
        const int d = threadIdx.x;
        sb[d] = d < out ? th[a.boff + d] : 0.f;
        if (ACTOR) {
            const float raw = d < out ? th[a.mlp_n + d] : 0.f;
            const float ls = fminf(fmaxf(raw, -5.f), 1.f);
            sinv[d] = d < out ? __expf(-ls) : 0.f;
            smask[d] = (d < out && raw >= -5.f && raw <= 1.f) ? 1.f : 0.f;
            float c1 = d < out ? -ls - 0.9189385332046727f : 0.f;
            float c2 = d < out ? ls + 0.5f * (1.f + 1.8378770664093453f) : 0.f;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {  // fixed-order sums over d (lanes 0-15)
                c1 += __shfl_xor_sync(0x0000ffffu, c1, o);
                c2 += __shfl_xor_sync(0x0000ffffu, c2, o);
            }
            if (d == 0) {
                sconst[0] = c1;
                sconst[1] = c2;
            }
        }
    }
    __syncthreads();
    const int CTa = img_ct(a.A.C), CTg = img_ct(a.Gprev.C), CTo = img_ct(a.Gout.C);
    float cs[NT][2], csl[NT][2];  // this lane's column sums (lanes rq == 0 hold the warp's)
#pragma unroll
    for (int j = 0; j < NT; ++j) cs[j][0] = cs[j][1] = csl[j][0] = csl[j][1] = 0.f;
    double lrow = 0.0;
#pragma unroll 1
    for (int mt = 0; mt < 2; ++mt) {
        const int r0 = blockIdx.x * 128 + warp * 32 + mt * 16 + rq;  // rows r0, r0 + 8
        uint32_t af[16][4];
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (s < KS) {
                const uint8_t* p0 = a.A.p + img_off(r0, s * 16, CTa) + q * 4;
                const uint8_t* p1 = a.A.p + img_off(r0, s * 16 + 8, CTa) + q * 4;
                af[s][0] = *reinterpret_cast<const uint32_t*>(p0);
                af[s][1] = *reinterpret_cast<const uint32_t*>(p0 + 2048);  // row + 8: next core-matrix row group
                af[s][2] = *reinterpret_cast<const uint32_t*>(p1);
                af[s][3] = *reinterpret_cast<const uint32_t*>(p1 + 2048);
            }
        // per-row loss inputs of this lane's (row, column) slots, in flight under the MMAs
        bool live[2];
        float zin[2][NT][2], lpo[2], adv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = r0 + 8 * h;
            live[h] = a.rows[r] >= 0;
            lpo[h] = ACTOR ? a.lp_old[r] : 0.f;
            adv[h] = ACTOR ? a.sadv[r] : 0.f;
            const float* src = ACTOR ? a.z : a.tgt;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int d = 8 * j + 2 * q + e;
                    zin[h][j][e] = d < out ? src[(long)r * out + d] : 0.f;
                }
        }
        // ---- forward of the output layer: c[j] = (rows r0 / r0 + 8, columns 8j + 2q, + 1)
        float c[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            c[j][0] = c[j][2] = sb[8 * j + 2 * q];
            c[j][1] = c[j][3] = sb[8 * j + 2 * q + 1];
        }
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (s < KS)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const uint2 b = swf[0][s][j][lane], bl = swf[1][s][j][lane];
                    mma_bf16_16816(c[j], af[s][0], af[s][1], af[s][2], af[s][3], b.x, b.y);
                    mma_bf16_16816(c[j], af[s][0], af[s][1], af[s][2], af[s][3], bl.x, bl.y);
                }
        // ---- per-row loss and dloss/do (the row's columns are spread over the 4 q-lanes)
        float g[2][NT][2], gl[2][NT][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool lv = live[h];
            if (ACTOR) {  // losses.cpp:87-129 (action_logprob nn.cpp:204-219)
                // lp = sum_d [-zn^2 / 2 - ls_d - log sqrt(2 pi) - log(sech^2 z_d + 1e-6)]; the
                // sigma / entropy terms depend on the cluster only (sconst)
                float lp = 0.f, zn[NT][2];
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int d = 8 * j + 2 * q + e;
                        zn[j][e] = 0.f;
                        if (d < out && lv) {
                            const float zz = zin[h][j][e];
                            zn[j][e] = (zz - c[j][2 * h + e]) * sinv[d];
                            lp += -0.5f * zn[j][e] * zn[j][e] - __logf(sech2_f(zz) + 1e-6f);
                        }
                    }
                lp += __shfl_xor_sync(0xffffffffu, lp, 1);
                lp += __shfl_xor_sync(0xffffffffu, lp, 2);
                lp += sconst[0];
                const float ent_h = sconst[1];
                float glp = 0.f;
                if (lv) {
                    const float ratio = __expf(lp - lpo[h]);
                    if (!isfinite(ratio)) atomicExch(a.err, 3);
                    const float unc = ratio * adv[h];
                    const float clp = fminf(fmaxf(ratio, 1.f - a.clip), 1.f + a.clip) * adv[h];
                    if (q == 0) lrow += (double)(-fminf(unc, clp) * a.inv_B) - (double)(a.ent * ent_h * a.inv_B);
                    glp = unc <= clp ? -ratio * adv[h] * a.inv_B : 0.f;  // losses.cpp:116
                }
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int d = 8 * j + 2 * q + e;
                        const bool ok = d < out && lv;
                        g[h][j][e] = ok ? glp * zn[j][e] * sinv[d] : 0.f;
                        // clamp mask (losses.cpp:124-128)
                        gl[h][j][e] = ok ? smask[d] * (glp * (zn[j][e] * zn[j][e] - 1.f) - a.ent * a.inv_B) : 0.f;
                    }
            } else {  // losses.cpp:170-185: sum_k (v - tgt)^2 / B, grad 2 e / B
                float sq = 0.f;
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int d = 8 * j + 2 * q + e;
                        const bool ok = d < out && lv;
                        const float er = ok ? c[j][2 * h + e] - zin[h][j][e] : 0.f;
                        sq += er * er;
                        g[h][j][e] = 2.f * er * a.inv_B;
                        gl[h][j][e] = 0.f;
                    }
                sq += __shfl_xor_sync(0xffffffffu, sq, 1);
                sq += __shfl_xor_sync(0xffffffffu, sq, 2);
                if (q == 0 && lv) lrow += (double)sq * a.inv_B;
            }
        }
        // ---- output-layer gradient image (dW_L GEMM operand) and its column sums
        uint32_t ga[2][2];  // backward A fragment: (row h, k = 8j + 2q pair)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                ga[j][h] = j < NT ? bf2_pack(g[h][j < NT ? j : 0][0], g[h][j < NT ? j : 0][1]) : 0u;
                if (j < NT) *reinterpret_cast<uint32_t*>(a.Gout.p + img_off(r0 + 8 * h, 8 * j + 2 * q, CTo)) = ga[j][h];
            }
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float x = g[0][j][e] + g[1][j][e], y = gl[0][j][e] + gl[1][j][e];
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    x += __shfl_xor_sync(0xffffffffu, x, o);
                    if (ACTOR) y += __shfl_xor_sync(0xffffffffu, y, o);
                }
                cs[j][e] += x;
                csl[j][e] += y;
            }
        // ---- backward: (rows x out) g times W_L -> (rows x H), times tanh'(a);
        // groups of 4 n-tiles (32 columns): this lane's 8 row-pair sums are
        // reduce-scattered over the 8 lanes sharing q (xor 16, 8, 4: 7 shuffles),
        // leaving lane (rq, q) with the warp's sum of column 8 (rq >> 1) + 2q + (rq & 1)
        uint8_t* gp0 = a.Gprev.p + img_off(r0, 2 * q, CTg);  // + 128 B per n-tile, + 32 KB per 128 columns
#pragma unroll
        for (int n4 = 0; n4 < 8; ++n4) {
            if (4 * n4 >= HT) break;
            float cs8[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int nt = 4 * n4 + u;
                if (nt >= HT) {  // H % 32 == 16: the last group is half full
                    cs8[2 * u] = cs8[2 * u + 1] = 0.f;
                    continue;
                }
                const uint2 b = swb[nt][lane];
                float v[4] = {0.f, 0.f, 0.f, 0.f};
                mma_bf16_16816(v, ga[0][0], ga[0][1], ga[1][0], ga[1][1], b.x, b.y);
                // activations at (rows r0 / r0 + 8, columns 8 nt + 2q, + 1): the forward's A fragments
                const float2 x0 = bf2_unpack(af[nt >> 1][(nt & 1) ? 2 : 0]);
                const float2 x1 = bf2_unpack(af[nt >> 1][(nt & 1) ? 3 : 1]);
                v[0] *= 1.f - x0.x * x0.x;
                v[1] *= 1.f - x0.y * x0.y;
                v[2] *= 1.f - x1.x * x1.x;
                v[3] *= 1.f - x1.y * x1.y;
                uint8_t* gp = gp0 + (nt >> 4) * 32768 + (nt & 15) * 128;
                *reinterpret_cast<uint32_t*>(gp) = bf2_pack(v[0], v[1]);
                *reinterpret_cast<uint32_t*>(gp + 2048) = bf2_pack(v[2], v[3]);
                cs8[2 * u] = v[0] + v[2];
                cs8[2 * u + 1] = v[1] + v[3];
            }
            // slot k = 2u + e (column 8 (4 n4 + u) + 2q + e); halve the slots per step
#pragma unroll
            for (int w = 4; w >= 1; w >>= 1) {
                const int bit = w == 4 ? 16 : w == 2 ? 8 : 4;  // lane bit paired at this step
                const bool up = (lane & bit) != 0;
#pragma unroll
                for (int i = 0; i < w; ++i) {
                    const float mine = up ? cs8[w + i] : cs8[i];
                    const float other = up ? cs8[i] : cs8[w + i];
                    cs8[i] = mine + __shfl_xor_sync(0xffffffffu, other, bit);
                }
            }
            // lane keeps slot k = 4 (lane>>4 & 1) + 2 (lane>>3 & 1) + (lane>>2 & 1) = rq bit-reversed
            const int k = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
            const int col = 8 * (4 * n4 + (k >> 1)) + 2 * q + (k & 1);
            if (col < H) {
                if (mt == 0) red2[warp][col] = cs8[0];
                else red2[warp][col] += cs8[0];
            }
        }
    }
    if (rq == 0)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                red[warp][8 * j + 2 * q + e] = cs[j][e];
                redl[warp][8 * j + 2 * q + e] = csl[j][e];
            }
    tile_sum_f64(lrow, a.loss_rows + blockIdx.x);  // includes a __syncthreads
    if (threadIdx.x < out) {
        const int d = threadIdx.x;
        a.psum[blockIdx.x * 16 + d] = (red[0][d] + red[1][d]) + (red[2][d] + red[3][d]);
        if (ACTOR) a.psls[blockIdx.x * 16 + d] = (redl[0][d] + redl[1][d]) + (redl[2][d] + redl[3][d]);
    }
    for (int j = threadIdx.x; j < H; j += 128)
        a.psum_prev[(long)blockIdx.x * a.psum_prev_ld + j] = (red2[0][j] + red2[1][j]) + (red2[2][j] + red2[3][j]);
}
void head(const HeadArgs& a, bool actor, cudaStream_t s) {
    if (a.Bp <= 0) return;
    if (a.H > 256 || a.H % 16 || a.out > 16 || a.out < 1)
        throw ShapeError("head: needs hidden width % 16 == 0 (<= 256), 1 <= out <= 16");
    const unsigned tiles = (unsigned)(a.Bp / 128);
    if (a.out <= 8) {
        if (actor) launch_pdl(k_head<true, 1>, dim3(tiles), dim3(128), 0, s, a);
        else launch_pdl(k_head<false, 1>, dim3(tiles), dim3(128), 0, s, a);
    } else {
        if (actor) launch_pdl(k_head<true, 2>, dim3(tiles), dim3(128), 0, s, a);
        else launch_pdl(k_head<false, 2>, dim3(tiles), dim3(128), 0, s, a);
    }
    MB_LAUNCH();
}

// =========================================================================
// K7: Adam (adam.cpp:8-26), eps after sqrt(v_hat); bias corrections from
// the host in fp64. Skipped entirely once a numeric error is flagged, so
// the parameters stay at the last healthy state (train.cpp:197-206).
// =========================================================================
__global__ void k_adam(long n, float4* p, const float4* g, float4* m1, float4* m2, float lr, float ibc1,
                       float ibc2, const int* err) {
    if (*err) return;
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 pp = p[i], gg = g[i], a = m1[i], b = m2[i];
    float* P = &pp.x;
    const float* G = &gg.x;
    float* A = &a.x;
    float* Bv = &b.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        A[k] = 0.9f * A[k] + 0.1f * G[k];
        Bv[k] = 0.999f * Bv[k] + 0.001f * G[k] * G[k];
        P[k] -= lr * (A[k] * ibc1) / (sqrtf(Bv[k] * ibc2) + 1e-8f);
    }
    p[i] = pp;
    m1[i] = a;
    m2[i] = b;
}
__global__ void k_adam_tail(long lo, long n, float* p, const float* g, float* m1, float* m2, float lr,
                            float ibc1, float ibc2, const int* err) {
    if (*err) return;
    const long i = lo + threadIdx.x;
    if (i >= n) return;
    m1[i] = 0.9f * m1[i] + 0.1f * g[i];
    m2[i] = 0.999f * m2[i] + 0.001f * g[i] * g[i];
    p[i] -= lr * (m1[i] * ibc1) / (sqrtf(m2[i] * ibc2) + 1e-8f);
}
void adam(long n, float* p, const float* g, float* m1, float* m2, float lr, float bc1, float bc2,
          const int* err, cudaStream_t s) {
    const long n4 = n / 4;
    if (n4) {
        k_adam<<<(int)((n4 + 255) / 256), 256, 0, s>>>(n4, (float4*)p, (const float4*)g, (float4*)m1,
                                                      (float4*)m2, lr, 1.f / bc1, 1.f / bc2, err);
        MB_LAUNCH();
    }
    if (n4 * 4 < n) {
        k_adam_tail<<<1, 32, 0, s>>>(n4 * 4, n, p, g, m1, m2, lr, 1.f / bc1, 1.f / bc2, err);
        MB_LAUNCH();
    }
}

// Adam that also refreshes the bf16 image of the hypernet M block
// (flat indices [m_lo, m_lo + P*F) -> image (p, f)), used as the operand of
// the next theta-generation and df GEMMs. 4 parameters per thread; m_lo and
// F are multiples of 4 so a quad never straddles an 8-column image group.
__global__ void k_adam_img(long n4, float4* p, const float4* g, float4* m1, float4* m2, float lr, float ibc1,
                           float ibc2, const int* err, long m_lo, long m_hi, int F, Img mimg, long n, long hole_lo,
                           long hole_len) {
    pdl_enter();
    if (*err) return;
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n4) {  // the n % 4 scalar tail (never inside the M block: it ends at b, after M)
        long e = 4 * n4 + (i - n4);
        if (e >= hole_lo) e += hole_len;
        if (i - n4 < 4 && e < n) {
            float* ps = reinterpret_cast<float*>(p);
            const float* gs = reinterpret_cast<const float*>(g);
            float* as = reinterpret_cast<float*>(m1);
            float* bs = reinterpret_cast<float*>(m2);
            as[e] = 0.9f * as[e] + 0.1f * gs[e];
            bs[e] = 0.999f * bs[e] + 0.001f * gs[e] * gs[e];
            ps[e] -= lr * (as[e] * ibc1) / (sqrtf(bs[e] * ibc2) + 1e-8f);
        }
        return;
    }
    if (4 * i >= hole_lo) i += hole_len / 4;  // the skipped range (4-aligned)
    float4 pp = p[i], gg = g[i], a = m1[i], b = m2[i];
    float* P = &pp.x;
    const float* G = &gg.x;
    float* A = &a.x;
    float* Bv = &b.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        A[k] = 0.9f * A[k] + 0.1f * G[k];
        Bv[k] = 0.999f * Bv[k] + 0.001f * G[k] * G[k];
        P[k] -= lr * (A[k] * ibc1) / (sqrtf(Bv[k] * ibc2) + 1e-8f);
    }
    p[i] = pp;
    m1[i] = a;
    m2[i] = b;
    const long e = 4 * i;
    if (e >= m_lo && e < m_hi) {
        const long r = (e - m_lo) / F, c = (e - m_lo) - r * F;
        uint2 q;
        q.x = umma::pack_bf16(P[0], P[1]);
        q.y = umma::pack_bf16(P[2], P[3]);
        *reinterpret_cast<uint2*>(mimg.p + img_off(r, c, img_ct(F))) = q;
    }
}
void adam_img(long n, float* p, const float* g, float* m1, float* m2, float lr, float bc1, float bc2, const int* err,
              long m_lo, int F, const Img& mimg, cudaStream_t s, long hole_lo, long hole_len) {
    const long m_hi = m_lo + (long)mimg.R * F;
    if (m_lo % 4 || F % 8) throw ShapeError("adam_img: M block must be 4-aligned with F % 8 == 0");
    if (hole_lo % 4 || hole_len % 4 || hole_len < 0 || (hole_len && mimg.R))
        throw ShapeError("adam_img: the skipped range must be 4-aligned (and excludes the image)");
    const long n_all = n;  // the tail's bound is in unshifted element indices
    n -= hole_len;         // elements updated
    if (n <= 0) return;
    const long n4 = n / 4, threads = n4 + (n - 4 * n4);
    launch_pdl(k_adam_img, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s, n4, (float4*)p,
               (const float4*)g, (float4*)m1, (float4*)m2, lr, 1.f / bc1, 1.f / bc2, err, m_lo, m_hi, F, mimg, n_all,
               hole_lo, hole_len);
    MB_LAUNCH();
}

// =========================================================================
// RNG test kernels (rng.hpp words / Box-Muller on the device)
// =========================================================================
__global__ void k_rng_words(uint64_t key, uint64_t ctr, long n, uint64_t* out) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = rng_word(key, ctr + 1 + i);
}
__global__ void k_rng_gauss(uint64_t key, uint64_t ctr, long n, double* out) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = box_muller(rng_word(key, ctr + 2 * i + 1), rng_word(key, ctr + 2 * i + 2));
}
void rng_words(uint64_t key, uint64_t ctr, long n, uint64_t* out, cudaStream_t s) {
    k_rng_words<<<(int)((n + 255) / 256), 256, 0, s>>>(key, ctr, n, out);
    MB_LAUNCH();
}
void rng_gaussians(uint64_t key, uint64_t ctr, long n, double* out, cudaStream_t s) {
    k_rng_gauss<<<(int)((n + 255) / 256), 256, 0, s>>>(key, ctr, n, out);
    MB_LAUNCH();
}

}  // namespace mb200
