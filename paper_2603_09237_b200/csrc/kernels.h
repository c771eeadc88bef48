// Host-side launch wrappers for every device kernel of the MORLAX B200 path.
// All take an explicit stream; none synchronise.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "img.cuh"

namespace mb200 {

// all layers' generated weights of groups [g0, g0+ng) -> per-group layer images
struct PackDims {
    int L = 0;
    int in[8] = {}, out[8] = {};
    long woff[8] = {}, ioff[8] = {};
    long ustart[9] = {};  // (8-row-padded) 8-column units per group before layer l
};

// ---------------------------------------------------------------- tcgen05 GEMM v2
// D(m,n) = sum_k A(m,k) B(n,k) over tiled bf16 images (img.cuh), operands
// streamed by the bulk-copy engine (img_gemm.cu). view 0: (row, col) =
// (m|n, k) K-major; view 1: (row, col) = (k, m|n) MN-major.
struct IGemm {
    Img A; int a_view = 0;
    Img B; int b_view = 0;
    int M = 0, N = 0, K = 0, Z = 1;
    const int* goff = nullptr;  // 128-aligned group offsets (gmode 1: rows, 2: K)
    int gmode = 0, max_group = 0;
    const float* bias = nullptr; long bias_gs = 0; int bias_mode = 0;  // 1: bias[n], 2: bias[m]
    int act = 0;                 // 0 none, 1 tanh (C2 <- pre-activation), 2 x *= 1 - aux(m,n)^2
    Img aux;                     // rows view (row = m, col = n), aux.gs ignored for gmode 1
    float* C = nullptr; long cm = 0, cn = 0, c_gs = 0;
    float* C2 = nullptr; long c2m = 0, c2n = 0, c2_gs = 0;
    int accumulate = 0;
    Img O; int o_mode = 0;       // 0 none, 1 image (row = m, col = n)
    int N_tile = 0;              // set by the launcher
    float* psum = nullptr;       // act 2: per-128-row-tile column sums [Bp/128][psum_ld]
    long psum_ld = 0;
    // act 0: a bf16 copy of C (row stride c16m elements, cn == 1); 16-column
    // chunks entirely inside one of the nbf column ranges [bf_lo, bf_hi) are
    // written only there (their fp32 C is left as it was)
    uint16_t* C16 = nullptr;
    long c16m = 0;
    int nbf = 0;
    long bf_lo[7] = {}, bf_hi[7] = {};
    // b_tma: B chunks come straight from row-major bf16 rows through a tiled
    // tensor map (make_weight_map) instead of the packed image B.p: per group
    // z a [B.R][B.C] matrix; a 128 x 128 chunk lands as two 128-row x 64-column
    // boxes in the 128-byte-swizzled layout (K-major for view 0, MN-major for
    // view 1). B.R / B.C still give the extents.
    int b_tma = 0;
    alignas(64) CUtensorMap bmap;
};
// tensor map over rows [z][R][C] of bf16 (row stride C, group stride gs
// elements; C % 8 == 0, base 16-byte aligned) for b_tma: 64 x 128 x 1 boxes,
// SWIZZLE_128B, zero fill past R and C
bool make_weight_map(CUtensorMap* map, const uint16_t* base, int R, int C, long gs, int Z);
// out[z*out_gs + j] = sum over row tiles t of group z (goff/128) of psum[t*ld + j]
void img_gemm(const IGemm& d, cudaStream_t s);
// 1-3 independent GEMMs with the same epilogue kind in one persistent launch
void img_gemm_batch(const IGemm* ds, int n, cudaStream_t s);
// several per-cluster segment-sum jobs (+ the per-tile loss partials) in one launch
struct SegJob {
    const float* psum = nullptr;
    long ld = 0;
    int width = 0;
    float* out = nullptr;
    long out_gs = 0;
};
struct SegLoss {
    const double* tiles = nullptr;  // [n] per-tile loss partials -> *out
    long n = 0;
    double* out = nullptr;
};
struct SegJobs {
    int n = 0;
    SegJob job[16];
    int nloss = 0;
    SegLoss loss[2];
};
void segsum_multi(const SegJobs& jb, const int* goff, int G, cudaStream_t s);
// dst(r, c) <- src[z*src_gs + r*ld + c] for z < G (dst.gs per z)
void to_img(const float* src, long ld, long src_gs, int R, int C, const Img& dst, int G, cudaStream_t s);
void pack_weights(const float* theta, long ld, int g0, int ng, const PackDims& pd, uint8_t* wimg, long gs,
                  cudaStream_t s);
// the same from the bf16 copy of theta (a relayout, no rounding)
void pack_weights16(const uint16_t* theta16, long ld, int g0, int ng, const PackDims& pd, uint8_t* wimg, long gs,
                    cudaStream_t s);
// gtheta [G][ld] -> bf16 image + column sums db[P] in one pass (db may be null)
void gtheta_prep(const float* gt, long ld, int G, int P, const Img& gimg, float* db, cudaStream_t s);
// sharded optimizer: the local clusters' gtheta rows [Kl][ld] split by
// column shard into send[W][Kl][S] (columns past ld zero-filled)
void pack_shards(const float* gt, long ld, int Kl, long S, int W, float* send, cudaStream_t s);
struct MbGather {
    int Bp = 0, G = 0, od = 0, ad = 0, m = 0;
    const int *rows = nullptr, *goff = nullptr;
    const float *obs = nullptr, *act = nullptr, *lp = nullptr, *sadv = nullptr, *tgt = nullptr;
    Img Xi;
    float *act_o = nullptr, *lp_o = nullptr, *sadv_o = nullptr, *tgt_o = nullptr;
    int* rg = nullptr;
};
void gather_minibatch(const MbGather& a, cudaStream_t s);
void gather_img(const int* rows, int Bp, const float* src, int width, const Img& dst, cudaStream_t s);
// per-row loss heads writing the output-layer gradient into an image
// psum / psls: per-128-row-tile column sums [Bp/128][16] of the output
// gradient (bias grads) and of the log-std gradient terms
void actor_rows_img(int Bp, int ad, const int* rows, const int* row_group, const float* theta, long P, long mlp_n,
                    const float* mu, int ldmu, const float* z, const float* lp_old, const float* sadv, float clip,
                    float ent, float inv_B, const Img& g_out, float* psum, float* psls, double* loss_rows, int* err,
                    cudaStream_t s);
void critic_rows_img(int Bp, int m, const int* rows, const float* v, int ldv, const float* tgt, float inv_B,
                     const Img& g_out, float* psum, double* loss_rows, cudaStream_t s);
// fused output layer + per-row loss + output-layer backward (kernels.cu k_head)
struct HeadArgs {
    int Bp = 0, H = 0, out = 0;
    const int *rows = nullptr, *rg = nullptr;
    const float* theta = nullptr;  // local clusters' generated params [G][ld]
    long ld = 0, woff = 0, boff = 0, mlp_n = 0;
    Img A;                         // last hidden activation image (rows x H)
    Img Gout, Gprev;               // output-layer gradient image, last-hidden pre-activation gradient image
    // actor
    const float *z = nullptr, *lp_old = nullptr, *sadv = nullptr;
    float clip = 0.f, ent = 0.f;
    int* err = nullptr;
    // critic
    const float* tgt = nullptr;
    float inv_B = 0.f;
    float *psum = nullptr, *psls = nullptr, *psum_prev = nullptr;  // [tile][16], [tile][16], [tile][psum_prev_ld]
    long psum_prev_ld = 0;
    double* loss_rows = nullptr;
};
void head(const HeadArgs& a, bool actor, cudaStream_t s);
// Adam over n elements (minus the 4-aligned range [hole_lo, hole_lo + hole_len),
// left untouched); elements in the M block [m_lo, m_lo + mimg.R * F) also
// refresh the bf16 image
void adam_img(long n, float* p, const float* g, float* m1, float* m2, float lr, float bc1, float bc2, const int* err,
              long m_lo, int F, const Img& mimg, cudaStream_t s, long hole_lo = 0, long hole_len = 0);
// dM = gtheta^T f consumed in registers by Adam on the M block (dm_adam.cu)
struct DmAdam {
    Img gimg, fimg;        // gtheta (rows g, cols p), f (rows g, cols f)
    int G = 0, P = 0, F = 0;
    float *p = nullptr, *m1 = nullptr, *m2 = nullptr;  // M block [P][F] fp32
    Img mimg;              // bf16 image of M (rows p, cols f)
    float lr = 0.f, ibc1 = 0.f, ibc2 = 0.f;
    const int* err = nullptr;
};
void dm_adam(const DmAdam& a, cudaStream_t s);

// ---------------------------------------------------------------- env (K1)
void env_reset(int kind, int N, float* state, uint64_t* keys, uint64_t* ctrs, int* steps,
               uint64_t parent_key, int inst_base, cudaStream_t s);
void env_step(int kind, int N, float* state, uint64_t* keys, uint64_t* ctrs, int* steps,
              const float* actions, float* obs, float* reward, uint8_t* term, uint8_t* trunc,
              unsigned long long* clamp_count, int* err, cudaStream_t s);
void env_obs(int kind, int N, const float* state, float* obs, cudaStream_t s);

// ---------------------------------------------------------------- rollout (K3+K1)
struct NetDims {
    int L;             // layers
    int sz[9];         // sizes[0..L]
    long woff[8], boff[8];
    long mlp_n, P;
    int out_tanh, has_log_std;
};
// evaluate_params (evaluate.cu): deterministic first-episode returns per
// simplex-grid preference; theta [n_points][ld] from the hypernet forward
struct EvalArgs {
    int kind = 0, od = 0, ad = 0, m = 0, sdim = 0, max_steps = 0;
    int episodes = 0;
    int cpp = 0, maxw = 0, nbias = 0;  // set by evaluate()
    NetDims pol{};
    const float* theta = nullptr;
    long ld = 0;
    uint64_t key = 0;                  // Rng(key): point g resets from split(g)
    double* part = nullptr;            // [n_points][ceil(episodes / 16)][m] scratch
    int* err = nullptr;
};
void evaluate(EvalArgs a, int n_points, double* d_mean, cudaStream_t s);

struct RolloutArgs {
    int kind, N, T, K, reps, od, ad, m, sdim, max_steps;
    const float* theta;  // [K][theta_ld] (first Pa used)
    const float* phi;    // [K][phi_ld]
    long theta_ld, phi_ld;
    NetDims pol, cri;
    float* state; uint64_t* env_key; uint64_t* env_ctr; int* steps;
    uint64_t roll_key;
    int roll_inst_base;  // global instance index of local instance 0 (sharding)
    float *obs, *act_pre, *logprob, *reward, *value, *next_value;
    uint8_t *term, *trunc;
    float* tracker;      // [N][m]
    const float* cluster_w;  // [K][m]
    double* ret_sum; int* ret_cnt;  // [N] completed scalarised returns
    unsigned long long* clamp_count; int* err;
};

// tensor-core rollout (rollout_tc.cu): per-cluster weights packed as bf16
// UMMA images, streamed per step by the bulk-copy engine. A chunk is one
// bulk copy: rows [128 tile, +128) (16 for the output layer) x K columns
// [k0, k0 + kw) of layer `layer`, K-major core matrices with SBO = kw * 16.
constexpr int ROLL_MAX_CHUNKS = 48;
struct NetPlan {
    int nchunks, blob_bytes, max_chunk;
    int kin_pad[8], tiles[8];
    int chunk_off[ROLL_MAX_CHUNKS], chunk_bytes[ROLL_MAX_CHUNKS], chunk_layer[ROLL_MAX_CHUNKS],
        chunk_tile[ROLL_MAX_CHUNKS], chunk_k0[ROLL_MAX_CHUNKS], chunk_kw[ROLL_MAX_CHUNKS];
};
NetPlan make_plan(const NetDims& nd);
void pack_theta(const float* theta, long ld, int G, const NetDims& nd, const NetPlan& pl, uint8_t* blob, cudaStream_t s);
struct RolloutTcArgs : RolloutArgs {
    NetPlan pol_plan, cri_plan;
    const uint8_t* pol_blob;  // [K][pol_plan.blob_bytes]
    const uint8_t* cri_blob;
    const float* eps;         // [T][N][ad] the rollout's N(0,1) draws (rollout_noise)
    // filled by rollout_tc: ring slot size and slots per net, operand buffer sizes, padded env count
    int slot_bytes, pol_slots, cri_slots, xb_bytes, hb_bytes, nepad;
};
void rollout_tc(RolloutTcArgs a, cudaStream_t s);
// the N(0,1) draws of a whole rollout, ahead of it and in parallel:
// eps[t][i][d] = (float) Box-Muller of words 2 (t ad + d) + 1, + 2 of instance
// i's stream roll_key.split(inst_base + i) (rollout.cpp:101, nn.cpp:192-202,
// rng.hpp:55-60) -- the exact value the sequential sampler adds to the mean
void rollout_noise(uint64_t roll_key, int inst_base, int N, int T, int ad, float* eps, cudaStream_t s);

// ---------------------------------------------------------------- GAE + normalise (K4)
void gae_scan(int N, int T, int m, const float* reward, const float* value, const float* next_value,
              const uint8_t* term, const uint8_t* trunc, float gamma, float lambda, float* adv,
              float* targets, cudaStream_t s);
// per-group partial sums part[g][8] (fp64) of x[r*m+k] (pass 1) or
// (x - mean)^2 (pass 2) over the group's consecutive rows; channel_total sums
// the partials in group order (rank-count invariant: gae.cpp:79-96)
void channel_partials(const float* x, int groups, long rows_per_group, int m, const double* mean, double* part,
                      cudaStream_t s);
void channel_total(const double* part, int groups, int m, double* out, cudaStream_t s);
// mean[k] = sums[k] / rows (mode 0); inv[k] = 1/(sqrt(sums[k]/rows) + 1e-8) (mode 1)
void stats_finalize(const double* sums, double rows, int m, double* out, int mode, cudaStream_t s);
void scalarize(int N, int T, int m, const float* adv, const float* cluster_w, int reps,
               const double* mean, const double* inv_std, float* sadv, cudaStream_t s);

// ---------------------------------------------------------------- PPO (K5)
// out[z*out_bz + j] (+)= sum_{rows in group z} x[row*width + j]
void check_finite_f64(const double* x, int n, int* err, int code, cudaStream_t s);

// hypernetwork feature map (feature.cu): fused tanh MLP over the cluster rows
constexpr int kMaxFeatLayers = 8;
struct FeatDims {
    int L = 0;
    int sz[kMaxFeatLayers + 1] = {};
    long woff[kMaxFeatLayers] = {}, boff[kMaxFeatLayers] = {};
    float* act[kMaxFeatLayers + 1] = {};   // activations [G][sz[l]] (act[0] = w)
    float* gz[kMaxFeatLayers] = {};        // pre-activation gradients [G][sz[l+1]]
};
// act[1..L] for all G rows of the cluster weights w [G][m]; fimg (bf16 image
// of f) gets rows [r0, r0 + rn) as image rows 0..rn-1
// df = sum of the split-K partials [splits][G][F]; writes dW/db of every layer into gout (flat layout)
// the same for up to two feature maps of equal depth in lockstep (one launch per layer)
struct FeatJob {
    const FeatDims* fd;
    const float* p;
    const float* w;
    int G;
    Img fimg;  // forward: image rows [r0, r0 + rn)
    int r0, rn;
    const float* parts;  // backward: split-K partials of M^T gtheta
    int splits;
    float* gout;
};
void feature_forward_multi(const FeatJob* jobs, int nj, cudaStream_t s);
// stage 0: df split-K sum * tanh' (gz of the last layer) and the dense
// backward; 1: the first part only; 2: the dense backward only
void feature_backward_multi(const FeatJob* jobs, int nj, cudaStream_t s, int stage = 0);

// ---------------------------------------------------------------- Adam (K7)
void adam(long n, float* p, const float* g, float* m1, float* m2, float lr, float bc1, float bc2,
          const int* err, cudaStream_t s);

// ---------------------------------------------------------------- Pareto (K8/K9)
void pareto_mask(int n, int m, const double* pts, uint8_t* mask, uint8_t* uniq, double* sums,
                 cudaStream_t s);
// linear_dominance_filter's selection on the nondominated set nd [nn][m]
// (device): keep[q] = 1 for survivors; scratch >= 2 nn ints (m == 2)
void linear_dominance(int nn, int m, const double* nd, uint8_t* keep, int* scratch, cudaStream_t s);
// exact hypervolume (WFG recursion, any m <= 8) of the points >= ref;
// value and clipped count written to host memory (synchronises `s`)
void hv_exact(int n, int m, const double* d_pts, const double* d_ref, double* value, int* clipped, cudaStream_t s);
void hv_mc(int n, int m, const double* pts, const double* ref, uint64_t samples, uint64_t key,
           uint64_t ctr, unsigned long long* hits, double* hi_out, cudaStream_t s);
void rng_words(uint64_t key, uint64_t ctr, long n, uint64_t* out, cudaStream_t s);
void rng_gaussians(uint64_t key, uint64_t ctr, long n, double* out, cudaStream_t s);

}  // namespace mb200
