// Host C++ side of the MORLAX B200 path: device-resident hypernetworks,
// batched env, and the train-iteration orchestration. Mirrors the
// reference API (include/morlax/trainer.hpp, hypernet.hpp, env.hpp) with
// device buffers; C-ABI wrappers live in capi.cu.
#pragma once

#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace mb200 {

struct Comm;       // communicator of one rank (comm.cu), null when single-GPU without one
struct LoopGroup;  // in-process loopback group (comm.cu)

// Per-kernel-class device timing with CUDA events on the launching stream,
// plus the algorithmic FLOPs / bytes of every launch (for the roofline).
struct Profiler {
    struct Cls {
        std::string name;
        double flops = 0, bytes = 0, ms = 0;
        long count = 0;
    };
    bool on = false;
    std::string phase = "iteration";  // class key prefix: the phase being enqueued
    std::vector<Cls> cls;
    std::vector<cudaEvent_t> pool;
    struct Pending { int c; cudaEvent_t a, b; cudaStream_t s; };
    std::vector<Pending> pending;
    size_t used = 0;
    // per-launch timeline of the last collect(): class, stream, start / end
    // (ms from the first recorded launch)
    struct Span { int c; int stream; double t0, t1; };
    std::vector<Span> timeline;
    std::vector<cudaStream_t> streams;
    int begin(const char* name, double flops, double bytes, cudaStream_t s);
    void end(int h, cudaStream_t s);
    void collect();  // synchronises the recorded events
    void reset();
    ~Profiler();
};

struct TrainConfig {  // trainer.hpp:21-77 (TrainerConfig + HypernetArch)
    int env_kind = ENV_POINTMASS;
    int N = 256, K = 16, kappa = 0, T = 32, epochs = 4, minibatch_count = 4;
    double gamma = 0.99, lambda = 0.95, clip_eps = 0.2, actor_lr = 3e-4, critic_lr = 3e-4,
           entropy_coef = 0.1;
    uint64_t seed = 0;
    int F = 64;
    std::vector<int> feat_hidden{64}, actor_hidden{64, 64}, critic_hidden{64, 64};
    void validate(int m) const;  // config.cpp:17-45 semantics
};

// Device-resident affine hypernetwork theta(w) = M f(w) + b (hypernet.hpp:20-75)
// for one target net, with fp32 master params, grads and Adam moments in the
// reference flat layout [feature | M (P x F) | b (P)].
struct HyperNet {
    int m = 0, F = 0, G = 0;  // G: groups (clusters) this hypernet serves
    std::vector<int> fsz;     // feature sizes [m, hidden..., F]
    std::vector<long> fwoff, fboff;
    NetDims tgt{};
    long nf = 0, P = 0, n = 0;
    long ld = 0;  // row stride of theta / gtheta (P rounded up to 8: aligned vector stores)
    float *p = nullptr, *g = nullptr, *m1 = nullptr, *m2 = nullptr;
    long steps[3] = {0, 0, 0};
    std::vector<float*> fact;  // feature activations [G][fsz[l]], l = 0..Lf
    float *theta = nullptr, *gtheta = nullptr, *gf = nullptr, *parts = nullptr;
    // the update forward's theta: bf16 for the hidden layers' weights (only the
    // weight packing reads them), fp32 kept for biases, the output layer and
    // the log-std (theta16_last: the last forward wrote the weights here only)
    uint16_t* theta16 = nullptr;
    bool theta16_last = false;
    // the update's weight GEMMs read the layers whose rows are 16-byte
    // aligned in theta16 through tensor maps (no packing): wmap_ok[l]; built
    // for the clusters [wmap_g0, wmap_g0 + wmap_ng)
    std::vector<CUtensorMap> wmap;
    std::vector<int> wmap_ok;
    int wmap_g0 = -1, wmap_ng = -1;
    bool weight_tma(int l) const { return theta16_last && l < (int)wmap_ok.size() && wmap_ok[l]; }
    std::vector<float*> fgz;   // feature pre-activation gradients [G][fsz[l+1]]
    FeatDims fd{};             // device view of the feature MLP (feature.cu)
    const float* w_last = nullptr;  // cluster weights of the last forward (feature-map input)
    int fg0 = 0, fng = 0;           // clusters [fg0, fg0 + fng) of the last forward (this rank's)
    int splits = 1;
    int* d_split_bounds = nullptr;
    // bf16 tiled images (img.cuh) feeding the tcgen05 GEMMs
    Img mimg;                    // M [P][F]      (refreshed by Adam)
    Img fimg;                    // f(w) [G][F]
    Img gimg;                    // gtheta [G][P]
    Img wimg;                    // generated weights, per group (wimg.gs): layer l at wimg_off[l]
    std::vector<long> wimg_off;
    void refresh_images(cudaStream_t s);                 // p (M block) -> mimg after external loads

    // world > 1 (or a single-rank communicator): the optimizer is sharded --
    // this rank owns M rows and b entries [row_lo, row_hi)
    void init(int m_, int F_, const std::vector<int>& fh, const std::vector<int>& target_sizes,
              bool out_tanh, bool has_log_std, int G_, Comm* comm_ = nullptr, int Kl_ = 0);
    void free_all();
    void init_params(uint64_t key, cudaStream_t s);  // init_hypernet (hypernet.cpp:124-145)
    // f (all G clusters), theta for groups [g0, g0+ng) of the G cluster weights w[G][m]
    // upd: the update's forward (hidden-layer weights of theta in bf16 only)
    void forward(const float* w, int g0, int ng, cudaStream_t s, bool upd = false);
    // the same for nh (1 or 2) hypernetworks in lockstep, one launch per stage
    static void forward_multi(HyperNet* const* hs, int nh, const float* w, int g0, int ng, cudaStream_t s,
                              bool upd = false);
    // part 0: all; 1: the gradient passes (gtheta image, shard exchange, df,
    // feature map: no parameter is written); 2: dM (+ the fused M-block Adam)
    static void backward_multi(HyperNet* const* hs, int nh, cudaStream_t s, int part = 0);
    // grads from gtheta [G][P] (all groups) -> g
    void backward(cudaStream_t s);
    void adam_step(double lr, const int* err, cudaStream_t s);
    // fused update: called before backward, which then applies Adam to the
    // M block inside the dM kernel (dM is never stored); adam_step finishes
    // the feature / b blocks
    void adam_begin(double lr, const int* err);
    bool adam_fused = false;
    float ad_lr = 0.f, ad_ibc1 = 0.f, ad_ibc2 = 0.f;
    const int* ad_err = nullptr;
    // ---- sharded optimizer, comm != null:
    // per minibatch the local clusters' fp32 gtheta rows are split by column
    // shard and exchanged all-to-all (grecv = every cluster's gtheta on this
    // rank's shard), db and dM + Adam run on the shard only, and the
    // refreshed bf16 M image rows and b entries are all-gathered. The
    // feature-map gradient of each cluster (gz) is all-gathered and the
    // feature map's backward + Adam run replicated over all clusters. Every
    // reduction keeps the single-rank order, so any rank count gives the
    // single-rank result bit for bit.
    Comm* comm = nullptr;
    // the gtheta exchange (all-to-all + this shard's gtheta pass) and the gz
    // all-gather run on xs, beside the df GEMM and the local feature-map
    // backward (xev: fork / join)
    cudaStream_t xs = nullptr;
    cudaEvent_t xev[2] = {nullptr, nullptr};
    int world = 1, rank = 0, Kl = 0;
    long S = 0, row_lo = 0, row_hi = 0;  // shard width (multiple of 128) and this rank's rows
    float *gsend = nullptr, *grecv = nullptr;  // [W][Kl][S] fp32
    Img gshard;                                 // bf16 [G][S]: this shard's gtheta, all clusters
    Img fall;                                   // bf16 [G][F]: f(w) of all clusters
    void gather_params(cudaStream_t s);         // all-gather the fp32 M rows (export / checkpoints)
};

NetDims make_dims(const std::vector<int>& sizes, bool out_tanh, bool has_log_std);

struct IterStats {
    double actor_loss = 0, critic_loss = 0;  // summed over minibatch steps
    double seconds = 0;
    int minibatches = 0;
    int numeric_error = 0;
    std::vector<double> cluster_returns;     // mean completed return per cluster (NaN if none)
};

// Minibatch row selection for one rank (host, pure): rows of perm[lo:hi)
// whose instance lies in [inst_lo, inst_lo + n_inst), converted to local row
// ids and stably grouped by cluster (losses.cpp:21-33 ordering).
void shard_minibatch(const int* perm, int lo, int hi, int T, int inst_lo, int n_inst, int reps,
                     int n_groups, int* rows_out, int* goff_out, int* n_rows_out, int* max_group);
int pad_groups(const int* rows, int* goff, int G, int* rows_out, int* n_out);
// the sharded optimizer's M-row partition (HyperNet::init)
void shard_rows(long P, int world, int rank, long* S, long* lo, long* hi);

class Trainer {
public:
    Trainer(const TrainConfig& cfg, int world = 1, int rank = 0, const void* nccl_id = nullptr,
            LoopGroup* loop = nullptr);
    ~Trainer();
    void iteration(int it, IterStats* st);

    // phases (for tests / bench breakdowns); iteration() runs all of them
    void phase_plans(int it);  // minibatch plans only (update of an externally set batch)
    void phase_rollout(int it);
    void phase_advantages();
    void phase_update(int it, int max_minibatches = -1);
    void finish(IterStats* st);
    // actor_loss + critic_loss (+ hypernet backward) on global rows of the
    // current batch, no Adam (parity tests; losses.cpp:46-189)
    void losses_only(const int* rows, int n, double* actor_loss, double* critic_loss);
    void set_clusters(const float* cw);

    // accessors
    const TrainConfig& config() const { return cfg_; }
    const EnvSpecB& env() const { return es_; }
    HyperNet& actor() { return actor_; }
    HyperNet& critic() { return critic_; }
    int local_envs() const { return Nl_; }
    int local_groups() const { return Kl_; }
    cudaStream_t stream() const { return s_; }
    const std::vector<int>& perm() const { return perm_; }
    void set_perm(const int* p);  // invalidates the look-ahead plan
    const std::vector<float>& clusters_host() const { return cw_h_; }
    // device batch
    float *d_obs = nullptr, *d_act = nullptr, *d_lp = nullptr, *d_rew = nullptr, *d_val = nullptr,
          *d_nval = nullptr, *d_adv = nullptr, *d_tgt = nullptr, *d_sadv = nullptr;
    uint8_t *d_term = nullptr, *d_trunc = nullptr;
    float* d_state = nullptr;
    float* d_eps = nullptr;  // [T][local N][act_dim] the rollout's N(0,1) draws
    uint64_t *d_ekey = nullptr, *d_ectr = nullptr;
    int* d_steps = nullptr;
    float* d_tracker = nullptr;
    int* d_err = nullptr;
    unsigned long long* d_clamps = nullptr;
    double* d_retsum = nullptr;  // per instance: sum of completed-episode scalarised returns (rollout.cpp:150-159)
    int* d_retcnt = nullptr;     // per instance: completed episodes this iteration
    long kernel_launches() const { return g_kernel_launches.load(); }  // process-wide
    Profiler& profiler() { return prof_; }

private:
    void alloc();
    void prepare_perms(int it);
    // Minibatch plan of one iteration (train.cpp:156-169): the shuffled
    // persistent permutation and every minibatch's sharded, group-padded row
    // map. Pure host work keyed by the iteration's RNG lane, so the plan for
    // it+1 is built on a worker thread while the GPU runs iteration it.
    struct PermPlan {
        int it = -1;
        long version = -1;       // perm_version_ it was built from
        std::vector<int> perm;   // permutation after this iteration's shuffles
        int* rows = nullptr;     // pinned [slots][Bpmax]
        int* goff = nullptr;     // pinned [slots][Kl+1]
        std::vector<int> B, Bglob, maxg, tmp;
        cudaEvent_t uploaded = nullptr;  // last upload from these pinned buffers
    } plan_[2];
    void build_plan(PermPlan& p, int it, const std::vector<int>& perm_before, long version);
    void join_worker();
    std::thread worker_;
    int worker_plan_ = -1;
    long perm_version_ = 0;
    void minibatch(int slot, int B, int Bglob, int maxg, const int* d_rows, const int* d_goff);
    void net_step(HyperNet* const* hs, const bool* actor, int nn, int Bp, float inv_B, int maxg, const int* rows,
                  const int* d_goff, int slot, cudaStream_t s);

    TrainConfig cfg_;
    EnvSpecB es_{};
    int world_ = 1, rank_ = 0;
    Comm* comm_ = nullptr;   // actor chain + per-iteration collectives (stream s_)
    Comm* comm2_ = nullptr;  // critic chain (stream s2_): the two chains' exchanges overlap
    int Nl_ = 0, Kl_ = 0, reps_ = 0, inst_lo_ = 0, g_lo_ = 0;
    long Rl_ = 0;
    HostRng root_;
    HyperNet actor_, critic_;
    cudaStream_t s_ = nullptr;
    std::vector<float> cw_h_;
    float* d_cw = nullptr;
    float* h_cw_pinned = nullptr;
    std::vector<int> perm_;
    int* h_rows_pinned = nullptr;  // [epochs*mbs][Bmax]
    int* h_goff_pinned = nullptr;  // [epochs*mbs][Kl+1]
    int *d_rows = nullptr, *d_goff = nullptr, *d_rowgroup = nullptr;
    std::vector<int> mb_B_, mb_Bglob_, mb_maxg_;
    int Bmax_ = 0, Bpmax_ = 0;  // real / group-padded (128-aligned) rows per minibatch
    struct UpdBufs {            // per-net tcgen05 update buffers
        std::vector<Img> A;     // [Bp][h_l] hidden activations (post-tanh)
        std::vector<Img> G;     // [Bp][out_l] gradient at the pre-activation of layer l
        float* Zf = nullptr;    // [Bp][16] output layer (policy mean / values), fp32
        float* psls = nullptr;      // per-128-row-tile column sums of the log-std gradient terms
        std::vector<float*> pbias;  // per layer l: per-tile column sums of G_l (bias grads of layer l)
        double* lossrows = nullptr;
    } ub_[2];
    cudaStream_t s2_ = nullptr;  // critic chain of the update
    cudaEvent_t ev_gather_ = nullptr, ev_c_net_ = nullptr, ev_chk_ = nullptr;
    // the minibatch inputs (gathered rows) are double-buffered by minibatch
    // parity: the gather of minibatch i+1 (stream s3_) waits only for the two
    // chains' losses of minibatch i-1 (ev_ad_ / ev_cd_[parity])
    cudaEvent_t ev_cd_[2] = {nullptr, nullptr}, ev_ad_[2] = {nullptr, nullptr};  // critic / actor done with set p
    cudaEvent_t ev_cfin_ = nullptr;  // the critic chain's last Adam
    cudaStream_t s3_ = nullptr;      // the minibatch gathers
    // per update chain (0: actor on s_, 1: critic on s2_) a side stream for
    // the kernels that are independent of the chain's next one (the bias-
    // gradient sums beside the weight-gradient GEMMs, the feature / b Adam
    // beside the fused dM + Adam), forked and joined by events
    cudaStream_t side_[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork_[2] = {nullptr, nullptr}, ev_join_[2] = {nullptr, nullptr};
    void fork(cudaStream_t s);            // side stream of s waits for s's work so far
    void join(cudaStream_t s);            // s waits for its side stream's work so far
    cudaStream_t side_of(cudaStream_t s) const { return s == s2_ ? side_[1] : side_[0]; }
    int mb_par_ = 0;
    struct MbBufs {
        Img Xi;
        float *Z = nullptr, *lpo = nullptr, *sa = nullptr, *tg = nullptr;
        int* rg = nullptr;
    } mbb_[2];
    void use_mb_bufs(int parity);  // point Xi_ / d_Z / ... at buffer set `parity`
    Img Xi_;                    // [Bp][obs] gathered observations (bf16 image)
    std::vector<uint8_t*> img_allocs_;
    std::vector<int> rows_tmp_;
    Img new_img(int R, int C);
    // update buffers
    float *d_Z = nullptr, *d_lpo = nullptr, *d_sa = nullptr, *d_tg = nullptr;
    float *d_lsg = nullptr;
    double *d_lossrows = nullptr, *d_mbloss = nullptr, *d_stats = nullptr, *d_scratch = nullptr;
    double* d_part = nullptr;  // [K][8] per-cluster normalisation partials (all ranks' after the all-gather)
    NetPlan pol_plan_{}, cri_plan_{};
    uint8_t *d_pol_blob = nullptr, *d_cri_blob = nullptr;
    int mb_done_ = 0;
    Profiler prof_;
};

}  // namespace mb200
