// Device kernels of the MORLAX B200 training step (everything except the
// GEMMs and Pareto): K1 env step, K3 fused rollout, K4 GAE scan +
// normalise/scalarise, K5 per-row PPO losses, K7 Adam, reductions.
// Reference semantics are cited per kernel (paths under /root/reference/proj).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

std::atomic<long> g_kernel_launches{0};

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
    return 4.f * e / (d * d);
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

void gae_scan(int N, int T, int m, const float* reward, const float* value, const float* next_value,
              const uint8_t* term, const uint8_t* trunc, float gamma, float lambda, float* adv,
              float* targets, cudaStream_t s) {
    const long warps = (long)N * m;
    k_gae<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(N, T, m, reward, value, next_value, term,
                                                          trunc, gamma, lambda, adv, targets);
    MB_LAUNCH();
}

// Normalisation statistics (gae.cpp:79-96): deterministic two-level fp64
// reductions. pass 1 (mean == nullptr): sum x; pass 2: sum (x - mean)^2.
constexpr int kRedBlocks = 148 * 2;
__global__ void k_chan_partial(const float* x, long rows, int m, const double* mean, double* part) {
    extern __shared__ double red[];  // [blockDim][m]
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < rows; r += (long)gridDim.x * blockDim.x)
        for (int k = 0; k < m; ++k) {
            double v = x[r * m + k];
            if (mean) {
                v -= mean[k];
                v *= v;
            }
            acc[k] += v;
        }
    for (int k = 0; k < m; ++k) red[threadIdx.x * m + k] = acc[k];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int k = 0; k < m; ++k) red[threadIdx.x * m + k] += red[(threadIdx.x + s) * m + k];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < m; ++k) part[blockIdx.x * m + k] = red[k];
}
__global__ void k_chan_final(const double* part, int nb, int m, double* out) {
    const int k = threadIdx.x;
    if (k >= m) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b * m + k];
    out[k] = s;
}
void channel_sums(const float* x, long rows, int m, const double* mean, double* out, double* scratch,
                  cudaStream_t s) {
    k_chan_partial<<<kRedBlocks, 256, 256 * m * sizeof(double), s>>>(x, rows, m, mean, scratch);
    MB_LAUNCH();
    k_chan_final<<<1, 32, 0, s>>>(scratch, kRedBlocks, m, out);
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

// =========================================================================
// K5 pieces: minibatch gather and per-row loss heads (losses.cpp:87-129,
// 170-185).
// =========================================================================
__global__ void k_gather(const int* rows, int B, const float* src, int width, float* dst) {
    const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (e >= (long)B * width) return;
    const int q = e / width, j = e % width;
    dst[e] = src[(long)rows[q] * width + j];
}
void gather_rows(const int* rows, int B, const float* src, int width, float* dst, cudaStream_t s) {
    const long n = (long)B * width;
    if (n == 0) return;
    k_gather<<<(int)((n + 255) / 256), 256, 0, s>>>(rows, B, src, width, dst);
    MB_LAUNCH();
}

__global__ void k_fill_row_group(const int* goff, int G, int* rg) {
    const int g = blockIdx.x;
    for (int q = goff[g] + threadIdx.x; q < goff[g + 1]; q += blockDim.x) rg[q] = g;
}
void fill_row_group(const int* goff, int G, int* row_group, int B, cudaStream_t s) {
    (void)B;
    k_fill_row_group<<<G, 256, 0, s>>>(goff, G, row_group);
    MB_LAUNCH();
}

__global__ void k_actor_rows(int B, int ad, const int* rg, const float* theta, long P, long mlp_n,
                             const float* mu, const float* z, const float* lp_old, const float* sadv,
                             float clip, float ent, float inv_B, float* g_mu, float* lsg, double* loss_rows,
                             int* err) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B) return;
    const float* th = theta + (long)rg[q] * P + mlp_n;
    float lp = 0.f, ls[16], zn[16], sig[16];
    float ent_h = 0.f;
    for (int d = 0; d < ad; ++d) {  // action_logprob (nn.cpp:204-219) with the recomputed mean
        const float raw = th[d];
        ls[d] = fminf(fmaxf(raw, -5.f), 1.f);
        sig[d] = __expf(ls[d]);
        const float zz = z[(long)q * ad + d];
        zn[d] = (zz - mu[(long)q * ad + d]) / sig[d];
        lp += -0.5f * zn[d] * zn[d] - ls[d] - 0.9189385332046727f;
        lp -= __logf(sech2_f(zz) + 1e-6f);
        ent_h += ls[d] + 0.5f * (1.f + 1.8378770664093453f);  // gaussian_entropy
    }
    const float ratio = __expf(lp - lp_old[q]);
    if (!isfinite(ratio)) atomicExch(err, 3);  // losses.cpp:103-105
    const float adv = sadv[q];
    const float unc = ratio * adv;
    const float clp = fminf(fmaxf(ratio, 1.f - clip), 1.f + clip) * adv;
    loss_rows[q] = (double)(-fminf(unc, clp) * inv_B) - (double)(ent * ent_h * inv_B);
    const float glp = unc <= clp ? -ratio * adv * inv_B : 0.f;  // losses.cpp:116
    for (int d = 0; d < ad; ++d) {
        g_mu[(long)q * ad + d] = glp * zn[d] / sig[d];  // pre-activation gradient (no tanh')
        const float raw = th[d];
        lsg[(long)q * ad + d] = (raw >= -5.f && raw <= 1.f) ? glp * (zn[d] * zn[d] - 1.f) - ent * inv_B : 0.f;
    }
}
void actor_rows(int B, int ad, const int* row_group, const float* theta, long P, long mlp_n,
                const float* mu, const float* z, const float* lp_old, const float* sadv, float clip,
                float ent, float inv_B, float* g_mu, float* lsg, double* loss_rows, int* err,
                cudaStream_t s) {
    k_actor_rows<<<(B + 255) / 256, 256, 0, s>>>(B, ad, row_group, theta, P, mlp_n, mu, z, lp_old, sadv,
                                                 clip, ent, inv_B, g_mu, lsg, loss_rows, err);
    MB_LAUNCH();
}

__global__ void k_critic_rows(int B, int m, const float* v, const float* tgt, float inv_B, float* g,
                              double* loss_rows) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B) return;
    double l = 0.0;
    for (int k = 0; k < m; ++k) {
        const float e = v[(long)q * m + k] - tgt[(long)q * m + k];
        l += (double)e * e * inv_B;
        g[(long)q * m + k] = 2.f * e * inv_B;  // losses.cpp:179-181 (no 1/2)
    }
    loss_rows[q] = l;
}
void critic_rows(int B, int m, const float* v, const float* tgt, float inv_B, float* g_out,
                 double* loss_rows, cudaStream_t s) {
    k_critic_rows<<<(B + 255) / 256, 256, 0, s>>>(B, m, v, tgt, inv_B, g_out, loss_rows);
    MB_LAUNCH();
}

// out[z][j] (+)= sum_{q in [goff[z], goff[z+1])} x[q][j]; one block per (z, 128-col tile)
__global__ void k_segcolsum(const float* x, int width, const int* goff, float* out, long out_bz, int acc) {
    const int z = blockIdx.y;
    const int j = blockIdx.x * 128 + (threadIdx.x & 127);
    const int half = threadIdx.x >> 7;  // 2 row-halves
    __shared__ float red[256];
    const int lo = goff[z], hi = goff[z + 1];
    float s = 0.f;
    if (j < width)
        for (int q = lo + half; q < hi; q += 2) s += x[(long)q * width + j];
    red[threadIdx.x] = s;
    __syncthreads();
    if (half == 0 && j < width) {
        const float v = red[threadIdx.x] + red[threadIdx.x + 128];
        float* o = out + z * out_bz + j;
        *o = acc ? *o + v : v;
    }
}
void segmented_colsum(const float* x, int width, const int* goff, int G, float* out, long out_bz,
                      int accumulate, cudaStream_t s) {
    dim3 grid((width + 127) / 128, G);
    k_segcolsum<<<grid, 256, 0, s>>>(x, width, goff, out, out_bz, accumulate);
    MB_LAUNCH();
}

// out[j] = sum_r x[r][j]
__global__ void k_colsum(const float* __restrict__ x, int rows, long width, long ld, float* out) {
    const long j = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (j >= width) return;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // 8 independent chains: loads stay in flight
    int r = 0;
    for (; r + 8 <= rows; r += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += x[(long)(r + u) * ld + j];
    for (; r < rows; ++r) a[0] += x[(long)r * ld + j];
    out[j] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}
void colsum_rows(const float* x, int rows, long width, long ld, float* out, cudaStream_t s) {
    k_colsum<<<(int)((width + 255) / 256), 256, 0, s>>>(x, rows, width, ld, out);
    MB_LAUNCH();
}

__global__ void k_sum_f64(const double* __restrict__ x, long n, double* out, int acc) {
    __shared__ double red[1024];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    long i = threadIdx.x;
    for (; i + 3 * (long)blockDim.x < n; i += 4 * (long)blockDim.x) {
        s0 += x[i];
        s1 += x[i + blockDim.x];
        s2 += x[i + 2 * (long)blockDim.x];
        s3 += x[i + 3 * (long)blockDim.x];
    }
    for (; i < n; i += blockDim.x) s0 += x[i];
    double s = (s0 + s1) + (s2 + s3);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = acc ? *out + red[0] : red[0];
}
void sum_f64(const double* x, long n, double* out, int accumulate, cudaStream_t s) {
    k_sum_f64<<<1, 1024, 0, s>>>(x, n, out, accumulate);
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

__global__ void k_reduce_splits(const float* __restrict__ parts, int S, long n, float* out) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int k = 0;
    for (; k + 8 <= S; k += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += parts[(long)(k + u) * n + i];
    for (; k < S; ++k) a[0] += parts[(long)k * n + i];
    out[i] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}
void reduce_splits(const float* parts, int S, long n, float* out, cudaStream_t s) {
    k_reduce_splits<<<(int)((n + 255) / 256), 256, 0, s>>>(parts, S, n, out);
    MB_LAUNCH();
}

__global__ void k_mul_dtanh(float* g, const float* a, long n) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i < n) g[i] *= 1.f - a[i] * a[i];
}
void mul_dtanh(float* g, const float* a, long n, cudaStream_t s) {
    k_mul_dtanh<<<(int)((n + 255) / 256), 256, 0, s>>>(g, a, n);
    MB_LAUNCH();
}

// image-output variants (tcgen05 update path): one block = one 128-row tile;
// padded rows (rows[q] < 0) get zero loss and zero gradient. Per-tile column
// sums of the output gradient (bias grads) and of the log-std terms go to
// psum / psls [tile][16] (deterministic, summed per cluster by tile_segsum);
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
// layer). The output layer is only act_dim (12) or m (6) wide -- too narrow
// for the tensor cores -- so it runs on the CUDA cores in fp32 from the
// fp32 generated weights W_L [out][H] (staged in shared memory):
//   o      = b_L + W_L a          (a = last hidden activation row, bf16 image)
//   g      = dloss/do             (actor: clipped surrogate + entropy;
//                                  critic: 2 e / B)
//   g_prev = (W_L^T g) * (1 - a^2)  -> bf16 image (input of the dW / dX GEMMs)
// plus per-tile column sums of g (output bias grads), of the log-std terms
// and of g_prev (bias grads of the last hidden layer), and the tile's loss.
// Padded rows (rows[q] < 0) contribute zeros.
// =========================================================================
// OUT = output width (compile time: the per-row arrays stay in registers)
template <bool ACTOR, int OUT>
__global__ void __launch_bounds__(128) k_head(HeadArgs a) {
    __shared__ __align__(16) float sw[16 * 256];
    __shared__ float sb[16];
    __shared__ float red[64];
    __shared__ float red2[4 * 256];
    const int H = a.H;
    constexpr int out = OUT;
    const int q = blockIdx.x * 128 + threadIdx.x;
    const int z = a.rg[blockIdx.x * 128];  // groups are 128-row padded: one cluster per tile
    const float* th = a.theta + (long)z * a.ld;
    for (int e = threadIdx.x; e < out * H; e += 128) sw[e] = th[a.woff + e];
    if (threadIdx.x < out) sb[threadIdx.x] = th[a.boff + threadIdx.x];
    __syncthreads();
    const bool live = a.rows[q] >= 0;
    const int CTa = img_ct(a.A.C), CTg = img_ct(a.Gprev.C), CTo = img_ct(a.Gout.C);
    // ---- forward of the output layer
    float o[OUT];
#pragma unroll
    for (int j = 0; j < OUT; ++j) o[j] = 0.f;
    // activation row: 4 16-byte units (32 columns) in flight per step
    auto fwd8 = [&](const uint4& u, int c) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
        float x[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(b2[e]);
            x[2 * e] = f.x;
            x[2 * e + 1] = f.y;
        }
#pragma unroll
        for (int j = 0; j < OUT; ++j) {
            const float4 w0 = *reinterpret_cast<const float4*>(sw + j * H + c);
            const float4 w1 = *reinterpret_cast<const float4*>(sw + j * H + c + 4);
            o[j] = fmaf(x[0], w0.x, o[j]);
            o[j] = fmaf(x[1], w0.y, o[j]);
            o[j] = fmaf(x[2], w0.z, o[j]);
            o[j] = fmaf(x[3], w0.w, o[j]);
            o[j] = fmaf(x[4], w1.x, o[j]);
            o[j] = fmaf(x[5], w1.y, o[j]);
            o[j] = fmaf(x[6], w1.z, o[j]);
            o[j] = fmaf(x[7], w1.w, o[j]);
        }
    };
    int c = 0;
    for (; c + 32 <= H; c += 32) {
        uint4 u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = *reinterpret_cast<const uint4*>(a.A.p + img_off(q, c + 8 * k, CTa));
#pragma unroll
        for (int k = 0; k < 4; ++k) fwd8(u[k], c + 8 * k);
    }
    for (; c < H; c += 8) fwd8(*reinterpret_cast<const uint4*>(a.A.p + img_off(q, c, CTa)), c);
    float g[16], gl[16];  // 16: the image / column-sum code below works in 8-wide groups
#pragma unroll
    for (int j = 0; j < 16; ++j) g[j] = gl[j] = 0.f;
    double lrow = 0.0;
    if (live) {
        if (ACTOR) {  // losses.cpp:87-129 (action_logprob nn.cpp:204-219)
            const float* ls_raw = th + a.mlp_n;
            float lp = 0.f, zn[OUT], sig[OUT], ent_h = 0.f;
#pragma unroll
            for (int d = 0; d < OUT; ++d) {
                const float ls = fminf(fmaxf(ls_raw[d], -5.f), 1.f);
                sig[d] = __expf(ls);
                const float zz = a.z[(long)q * out + d];
                zn[d] = (zz - (o[d] + sb[d])) / sig[d];
                lp += -0.5f * zn[d] * zn[d] - ls - 0.9189385332046727f;
                lp -= __logf(sech2_f(zz) + 1e-6f);
                ent_h += ls + 0.5f * (1.f + 1.8378770664093453f);
            }
            const float ratio = __expf(lp - a.lp_old[q]);
            if (!isfinite(ratio)) atomicExch(a.err, 3);
            const float adv = a.sadv[q];
            const float unc = ratio * adv;
            const float clp = fminf(fmaxf(ratio, 1.f - a.clip), 1.f + a.clip) * adv;
            lrow = (double)(-fminf(unc, clp) * a.inv_B) - (double)(a.ent * ent_h * a.inv_B);
            const float glp = unc <= clp ? -ratio * adv * a.inv_B : 0.f;  // losses.cpp:116
#pragma unroll
            for (int d = 0; d < OUT; ++d) {
                g[d] = glp * zn[d] / sig[d];
                const float raw = ls_raw[d];  // clamp mask (losses.cpp:124-128)
                gl[d] = (raw >= -5.f && raw <= 1.f) ? glp * (zn[d] * zn[d] - 1.f) - a.ent * a.inv_B : 0.f;
            }
        } else {  // losses.cpp:170-185: sum_k (v - tgt)^2 / B, grad 2 e / B
#pragma unroll
            for (int k = 0; k < OUT; ++k) {
                const float e = (o[k] + sb[k]) - a.tgt[(long)q * out + k];
                lrow += (double)e * e * a.inv_B;
                g[k] = 2.f * e * a.inv_B;
            }
        }
    }
    tile_sum_f64(lrow, a.loss_rows + blockIdx.x);
    for (int h = 0; h < (out + 7) / 8; ++h) {  // output-layer gradient image (dW_L GEMM operand)
        uint4 w;
        w.x = umma::pack_bf16(g[8 * h + 0], g[8 * h + 1]);
        w.y = umma::pack_bf16(g[8 * h + 2], g[8 * h + 3]);
        w.z = umma::pack_bf16(g[8 * h + 4], g[8 * h + 5]);
        w.w = umma::pack_bf16(g[8 * h + 6], g[8 * h + 7]);
        *reinterpret_cast<uint4*>(a.Gout.p + img_off(q, 8 * h, CTo)) = w;
    }
    {  // per-tile column sums of the output gradient (bias) and the log-std terms, fixed order
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int d = 0; d < OUT; ++d) {
            float x1 = g[d], x2 = gl[d];
#pragma unroll
            for (int k = 16; k > 0; k >>= 1) {
                x1 += __shfl_xor_sync(0xffffffffu, x1, k);
                if (ACTOR) x2 += __shfl_xor_sync(0xffffffffu, x2, k);
            }
            if (lane == 0) {
                red[warp * 16 + d] = x1;
                if (ACTOR) red2[warp * 16 + d] = x2;  // red2 is free until the backward below
            }
        }
        __syncthreads();
        if (threadIdx.x < OUT) {
            a.psum[blockIdx.x * 16 + threadIdx.x] =
                red[threadIdx.x] + red[16 + threadIdx.x] + red[32 + threadIdx.x] + red[48 + threadIdx.x];
            if (ACTOR)
                a.psls[blockIdx.x * 16 + threadIdx.x] =
                    red2[threadIdx.x] + red2[16 + threadIdx.x] + red2[32 + threadIdx.x] + red2[48 + threadIdx.x];
        }
        __syncthreads();
    }
    // ---- backward of the output layer into the last hidden layer
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4 nxt[2];
    nxt[0] = *reinterpret_cast<const uint4*>(a.A.p + img_off(q, 0, CTa));
    nxt[1] = *reinterpret_cast<const uint4*>(a.A.p + img_off(q, 8, CTa));
    for (int c = 0; c < H; c += 16) {
        const uint4 cur[2] = {nxt[0], nxt[1]};
        if (c + 16 < H) {  // next 16 columns' activations load under this step's FMAs
            nxt[0] = *reinterpret_cast<const uint4*>(a.A.p + img_off(q, c + 16, CTa));
            nxt[1] = *reinterpret_cast<const uint4*>(a.A.p + img_off(q, c + 24, CTa));
        }
        float v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = 0.f;
#pragma unroll
        for (int j = 0; j < OUT; ++j) {  // W_L^T g: rows of W_L as float4 broadcasts
            const float4* w4 = reinterpret_cast<const float4*>(sw + j * H + c);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 w = w4[k];
                v[4 * k + 0] = fmaf(g[j], w.x, v[4 * k + 0]);
                v[4 * k + 1] = fmaf(g[j], w.y, v[4 * k + 1]);
                v[4 * k + 2] = fmaf(g[j], w.z, v[4 * k + 2]);
                v[4 * k + 3] = fmaf(g[j], w.w, v[4 * k + 3]);
            }
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&cur[hh]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(b2[e]);
                v[8 * hh + 2 * e] *= 1.f - f.x * f.x;
                v[8 * hh + 2 * e + 1] *= 1.f - f.y * f.y;
            }
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            uint4 w;
            w.x = umma::pack_bf16(v[8 * hh + 0], v[8 * hh + 1]);
            w.y = umma::pack_bf16(v[8 * hh + 2], v[8 * hh + 3]);
            w.z = umma::pack_bf16(v[8 * hh + 4], v[8 * hh + 5]);
            w.w = umma::pack_bf16(v[8 * hh + 6], v[8 * hh + 7]);
            *reinterpret_cast<uint4*>(a.Gprev.p + img_off(q, c + 8 * hh, CTg)) = w;
        }
        // warp reduce-scatter of 16 columns over 32 rows (deterministic order)
        int col = 0;
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1) {
            const bool up = (lane & (2 * w)) != 0;
            col += up ? w : 0;
#pragma unroll
            for (int i = 0; i < w; ++i) {
                const float mine = up ? v[w + i] : v[i];
                const float other = up ? v[i] : v[w + i];
                v[i] = mine + __shfl_xor_sync(0xffffffffu, other, 2 * w);
            }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        if ((lane & 1) == 0) red2[warp * 256 + c + col] = v[0];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += 128)
        a.psum_prev[(long)blockIdx.x * a.psum_prev_ld + j] =
            (red2[j] + red2[256 + j]) + (red2[512 + j] + red2[768 + j]);
}
void head(const HeadArgs& a, bool actor, cudaStream_t s) {
    if (a.Bp <= 0) return;
    if (a.H > 256 || a.H % 16 || a.out > 16) throw ShapeError("head: needs hidden width % 16 == 0 (<= 256), out <= 16");
#define MB_HEAD(O)                                                              \
    case O:                                                                     \
        if (actor) k_head<true, O><<<a.Bp / 128, 128, 0, s>>>(a);               \
        else k_head<false, O><<<a.Bp / 128, 128, 0, s>>>(a);                    \
        break;
    switch (a.out) {
        MB_HEAD(1) MB_HEAD(2) MB_HEAD(3) MB_HEAD(4) MB_HEAD(5) MB_HEAD(6) MB_HEAD(7) MB_HEAD(8)
        MB_HEAD(9) MB_HEAD(10) MB_HEAD(11) MB_HEAD(12) MB_HEAD(13) MB_HEAD(14) MB_HEAD(15) MB_HEAD(16)
        default: throw ShapeError("head: output width must be in [1, 16]");
    }
#undef MB_HEAD
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
    n -= hole_len;  // elements updated
    const long n4 = n / 4, threads = n4 + (n - 4 * n4);
    k_adam_img<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n4, (float4*)p, (const float4*)g, (float4*)m1,
                                                                (float4*)m2, lr, 1.f / bc1, 1.f / bc2, err, m_lo, m_hi,
                                                                F, mimg, n, hole_lo, hole_len);
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
