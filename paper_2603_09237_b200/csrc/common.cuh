// Shared device/host helpers for the MORLAX B200 path: error taxonomy,
// the counter-based RNG (bit-identical u64 words to include/morlax/rng.hpp
// of the reference) and the environment dynamics (fp32 state).
#pragma once

#include <atomic>

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "humanoid6_params.h"

namespace mb200 {

// ---- error taxonomy (reference include/morlax/errors.hpp:10-30) ----------
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

#define MB_CUDA(x)                                                                   \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess)                                                       \
            throw ::mb200::CudaError(std::string("CUDA error ") + cudaGetErrorString(_e) + \
                                     " at " __FILE__ ":" + std::to_string(__LINE__)); \
    } while (0)
// every kernel launch of the library goes through MB_LAUNCH: the counter is
// the bench's gpu_launches figure (kernels.cu defines it)
extern std::atomic<long> g_kernel_launches;
#define MB_LAUNCH()                                                        \
    do {                                                                   \
        g_kernel_launches.fetch_add(1, std::memory_order_relaxed);         \
        MB_CUDA(cudaGetLastError());                                       \
    } while (0)

// ---- per-device launch facts ---------------------------------------------------
// The SM count and the one-time cudaFuncSetAttribute(MaxDynamicSharedMemory)
// of the >48 KB kernels are cached per CUDA device (keyed by cudaGetDevice, a
// mutex around the cache): one process may drive several GPUs from several
// host threads (kernels.cu).
// Host-side ordering rule: every stream of ours is non-blocking, so work on
// the legacy default stream (the synchronous-API cudaMemset, and cudaMemcpy
// from pageable host memory, which may return before its DMA lands) is not
// ordered before it. Such calls are followed by cudaStreamSynchronize(0).
int device_sms();
void ensure_smem(const void* func, size_t bytes);

// ---- programmatic dependent launch ------------------------------------------
// The update chain's kernels are launched with programmatic stream
// serialization (launch_pdl): a kernel's launch is processed while its
// predecessor drains (the predecessor's implicit trigger at completion), and
// the kernel waits for the predecessor's completion and memory
// (griddepcontrol.wait) only after its prologue. Measured: 22.9 vs 23.5 ms /
// iteration. An early explicit trigger (griddepcontrol.launch_dependents at
// kernel entry) was slower (24.0): waiting CTAs hold SMs the other update
// stream could use. Without the launch attribute the wait is a no-op.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();  // MORLAX_PDL != "0" (kernels.cu)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MB_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

// ---- RNG: include/morlax/rng.hpp:18-93 -----------------------------------
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kSeedTag = 0x5851F42D4C957F2DULL;
constexpr uint64_t kSplitTag = 0xA0761D6478BD642FULL;
constexpr uint64_t kLaneTag = 0xE7037ED1A0B428DBULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t seed_key(uint64_t seed) { return mix64(seed ^ kSeedTag); }
__host__ __device__ __forceinline__ uint64_t split_key(uint64_t key, uint64_t lane) {
    return mix64(mix64(key ^ kSplitTag) + mix64(lane ^ kLaneTag));
}
// the word returned when the (pre-incremented) counter equals `ctr`
__host__ __device__ __forceinline__ uint64_t rng_word(uint64_t key, uint64_t ctr) {
    return mix64(key + kGamma * ctr);
}
__host__ __device__ __forceinline__ double word_double(uint64_t w) {
    return (double)(w >> 11) * 0x1.0p-53;
}
__host__ __device__ __forceinline__ double word_open(uint64_t w) {
    return (double)((w >> 11) + 1) * 0x1.0p-53;
}
#ifdef __CUDACC__
__device__ __forceinline__ double uniform_rn(double lo, double hi, uint64_t w) {
    // lo + (hi - lo) * u with the reference's separate rounding (no FMA)
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), word_double(w)));
}
__device__ __forceinline__ double box_muller(uint64_t w1, uint64_t w2) {
    const double u1 = word_open(w1), u2 = word_double(w2);
    return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(2.0 * 3.141592653589793, u2)));
}
#endif

struct HostRng {  // host mirror with the reference's member semantics
    uint64_t key = 0, ctr = 0;
    static HostRng seeded(uint64_t seed) { return HostRng{seed_key(seed), 0}; }
    HostRng split(uint64_t lane) const { return HostRng{split_key(key, lane), 0}; }
    uint64_t next_u64() { return rng_word(key, ++ctr); }
    double next_double() { return word_double(next_u64()); }
    double next_open() { return word_open(next_u64()); }
    uint64_t next_below(uint64_t n) {
        return (uint64_t)(((unsigned __int128)next_u64() * n) >> 64);
    }
};

// ---- environments ---------------------------------------------------------
enum EnvKind { ENV_LQR = 0, ENV_LQR_M1 = 1, ENV_POINTMASS = 2, ENV_DST = 3, ENV_HUMANOID6 = 4 };

struct EnvSpecB {
    int kind, obs_dim, act_dim, m, max_steps, state_dim, reset_words;
};

inline EnvSpecB env_spec_of(int kind) {
    switch (kind) {  // envs.hpp / env_*.cpp make_spec
        case ENV_LQR: return {ENV_LQR, 1, 1, 2, 200, 1, 1};
        case ENV_LQR_M1: return {ENV_LQR_M1, 1, 1, 1, 200, 1, 1};
        case ENV_POINTMASS: return {ENV_POINTMASS, 4, 2, 2, 200, 4, 2};
        case ENV_DST: return {ENV_DST, 1, 1, 2, 50, 1, 0};
        case ENV_HUMANOID6: return {ENV_HUMANOID6, H6_OBS, H6_ACT, H6_M, H6_HORIZON, H6_OBS, H6_OBS};
    }
    throw ConfigError("unknown environment kind " + std::to_string(kind));
}
inline int env_kind_of(const std::string& n) {  // registry.cpp:17-23 (+ mo-humanoid6)
    if (n == "mo-lqr1d") return ENV_LQR;
    if (n == "mo-lqr1d-m1") return ENV_LQR_M1;
    if (n == "mo-pointmass") return ENV_POINTMASS;
    if (n == "mo-dst-continuous") return ENV_DST;
    if (n == "mo-humanoid6") return ENV_HUMANOID6;
    throw ConfigError("unknown environment: " + n);
}

#ifdef __CUDACC__
__constant__ float c_h6[6][12] = {H6_CX, H6_CY, H6_CZ, H6_CR, H6_CP, H6_CW};
__constant__ float c_dst_depth[10] = {1, 6, 7, 9, 10, 11, 14, 15, 18, 20};
__constant__ float c_dst_value[10] = {0.7f, 8.2f, 11.5f, 14.0f, 15.1f, 16.1f, 19.6f, 20.3f, 22.4f, 23.7f};

// do_reset: state element k lives at s[k * ss]. Consumes the instance
// stream (key, *ctr) exactly like the reference do_reset.
__device__ __forceinline__ void env_do_reset(int kind, float* s, int ss, uint64_t key, uint64_t* ctr) {
    switch (kind) {
        case ENV_LQR:
        case ENV_LQR_M1:  // env_lqr.cpp:20-22
            s[0] = (float)uniform_rn(-1.0, 1.0, rng_word(key, ++*ctr));
            break;
        case ENV_POINTMASS:  // env_pointmass.cpp:22-28
            s[0] = (float)uniform_rn(-0.1, 0.1, rng_word(key, ++*ctr));
            s[ss] = (float)uniform_rn(-0.1, 0.1, rng_word(key, ++*ctr));
            s[2 * ss] = 0.f;
            s[3 * ss] = 0.f;
            break;
        case ENV_DST: s[0] = 0.f; break;  // env_deepsea.cpp:33-37
        case ENV_HUMANOID6:
            for (int k = 0; k < H6_OBS; ++k)
                s[k * ss] = (float)uniform_rn(-H6_INIT, H6_INIT, rng_word(key, ++*ctr));
            break;
    }
}

// mo-humanoid6 step, split so the twelve joints can run on several threads
// (csrc/humanoid6_params.h): joint j's actuator / joint update; returns the
// new actuator state e, joint velocity qd and s_j = tanh(qd)
__device__ __forceinline__ void h6_joint(float* s, int ss, int j, float aj, float* e_out, float* qd_out,
                                         float* sj_out) {
    const float dt = (float)H6_DT;
    float e = s[(24 + j) * ss], qd = s[(12 + j) * ss], q = s[j * ss];
    e = __fadd_rn(e, __fmul_rn((float)H6_ALPHA, __fsub_rn(aj, e)));
    qd = __fadd_rn(qd, __fmul_rn(dt, __fsub_rn(__fsub_rn(__fmul_rn((float)H6_KT, e), __fmul_rn((float)H6_KP, q)),
                                               __fmul_rn((float)H6_KD, qd))));
    q = __fadd_rn(q, __fmul_rn(dt, qd));
    s[(24 + j) * ss] = e;
    s[(12 + j) * ss] = qd;
    s[j * ss] = q;
    *e_out = e;
    *qd_out = qd;
    *sj_out = tanhf(qd);
}
// the body update from the twelve joints' (s_j, e_j, a_j, qd_j) (element j at
// [j * stride]), summed in joint order; writes the 6 rewards, returns fallen
__device__ __forceinline__ bool h6_body(float* s, int ss, const float* sjv, const float* ev, const float* av,
                                        const float* qdv, int stride, float* r) {
    const float dt = (float)H6_DT;
    float sx = 0, sy = 0, sz = 0, sr = 0, sp = 0, sw = 0, asq = 0, qsq = 0;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
        const float sj = sjv[j * stride], e = ev[j * stride], aj = av[j * stride], qd = qdv[j * stride];
        sx += c_h6[0][j] * sj;
        sy += c_h6[1][j] * sj;
        sw += c_h6[5][j] * sj;
        sz += c_h6[2][j] * e;
        sr += c_h6[3][j] * e;
        sp += c_h6[4][j] * e;
        asq += aj * aj;
        qsq += qd * qd;
    }
    float h = s[36 * ss], vx = s[37 * ss], vy = s[38 * ss], vz = s[39 * ss];
    float roll = s[40 * ss], pitch = s[41 * ss], wx = s[42 * ss], wy = s[43 * ss], wz = s[44 * ss];
    vx += dt * (sx - (float)H6_DRAG * vx);
    vy += dt * (sy - (float)H6_DRAG * vy);
    vz += dt * (sz - (float)H6_KH * h - (float)H6_DZ * vz);
    h += dt * vz;
    wx += dt * (sr - (float)H6_KA * roll - (float)H6_DA * wx);
    roll += dt * wx;
    wy += dt * (sp - (float)H6_KA * pitch - (float)H6_DA * wy);
    pitch += dt * wy;
    wz += dt * (sw - (float)H6_DRAG * wz);
    s[36 * ss] = h; s[37 * ss] = vx; s[38 * ss] = vy; s[39 * ss] = vz;
    s[40 * ss] = roll; s[41 * ss] = pitch; s[42 * ss] = wx; s[43 * ss] = wy; s[44 * ss] = wz;
    r[0] = vx;
    r[1] = -asq / 12.f;
    r[2] = -(roll * roll + pitch * pitch);
    r[3] = vy;
    r[4] = -0.1f * qsq / 12.f;
    r[5] = -(h * h + 0.1f * wz * wz);
    return fabsf(roll) > (float)H6_FALL || fabsf(pitch) > (float)H6_FALL;
}

// do_step with a pre-clamped action; writes m rewards, returns terminated.
__device__ __forceinline__ bool env_do_step(int kind, float* s, int ss, const float* a, float* r) {
    switch (kind) {
        case ENV_LQR:
        case ENV_LQR_M1: {  // env_lqr.cpp:25-37
            const float x = s[0], u = a[0];
            r[0] = -x * x;
            if (kind == ENV_LQR) r[1] = -u * u;
            s[0] = __fadd_rn(__fmul_rn(0.9f, x), __fmul_rn(0.5f, u));
            return false;
        }
        case ENV_POINTMASS: {  // env_pointmass.cpp:30-41, semi-implicit Euler
            const float vx = __fadd_rn(s[2 * ss], __fmul_rn(0.05f, a[0]));
            const float vy = __fadd_rn(s[3 * ss], __fmul_rn(0.05f, a[1]));
            s[2 * ss] = vx;
            s[3 * ss] = vy;
            s[0] = __fadd_rn(s[0], __fmul_rn(0.05f, vx));
            s[ss] = __fadd_rn(s[ss], __fmul_rn(0.05f, vy));
            r[0] = vx;
            r[1] = -__fadd_rn(__fmul_rn(a[0], a[0]), __fmul_rn(a[1], a[1]));
            return false;
        }
        case ENV_DST: {  // env_deepsea.cpp:39-59
            const float p = __fadd_rn(s[0], a[0]);
            s[0] = p;
            r[0] = 0.f;
            r[1] = -1.f;
            for (int t = 0; t < 10; ++t)
                if (fabsf(p - c_dst_depth[t]) <= 0.25f) {
                    r[0] = c_dst_value[t];
                    return true;
                }
            return false;
        }
        case ENV_HUMANOID6: {  // csrc/humanoid6_params.h
            float sjv[12], ev[12], qdv[12];
#pragma unroll
            for (int j = 0; j < 12; ++j) h6_joint(s, ss, j, a[j], &ev[j], &qdv[j], &sjv[j]);
            return h6_body(s, ss, sjv, ev, a, qdv, 1, r);
        }
    }
    return false;
}
#endif

}  // namespace mb200
