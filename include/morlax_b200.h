/* morlax_b200: C-ABI of the B200-native MORLAX data-parallel training step.
 *
 * The reference (/root/reference/proj) is a C++20 library whose hot path is
 * reached through its header API; it has no FFI of its own. Each entry point
 * below replaces the reference interface cited beside it, over plain
 * pointers and sizes (no C++ or torch types), so a C, C++ (see
 * INTEGRATION.md), ctypes, cgo or JNI caller can bind it.
 *
 * Status convention (reference tools/commands.hpp:12-32 exit codes):
 *   0 ok, 2 ConfigError / ShapeError / DomainError, 3 NumericError,
 *   1 other (CUDA / internal). morlax_last_error() returns the message and
 *   morlax_last_error_kind() the reference exception class name.
 * Host-buffer entry points copy host<->device inside the call; *_device
 * entry points take device pointers and a cudaStream_t (as void*).
 * All float state is fp32 on the device; reference-layout exports are fp64.
 */
#ifndef MORLAX_B200_H
#define MORLAX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MORLAX_OK 0
#define MORLAX_ERR_OTHER 1
#define MORLAX_ERR_CONFIG 2
#define MORLAX_ERR_NUMERIC 3

const char* morlax_last_error(void);
/* "ConfigError" | "ShapeError" | "DomainError" | "NumericError" | "CudaError" | "" */
const char* morlax_last_error_kind(void);
int morlax_version(void);
int morlax_device_count(void);

/* ---- RNG (replaces include/morlax/rng.hpp:18-93 on the device) --------- */
/* words ctr+1 .. ctr+n of stream `key` (Rng::next_u64) */
int morlax_rng_words(uint64_t key, uint64_t ctr, int64_t n, uint64_t* host_out);
/* n Box-Muller gaussians (Rng::next_gaussian, 2 words each) */
int morlax_rng_gaussians(uint64_t key, uint64_t ctr, int64_t n, double* host_out);

/* ---- Environment (replaces BatchedEnv, include/morlax/env.hpp:37-99,
 *      and make_env / env_spec, src/registry.cpp:17-35) ------------------ */
typedef struct morlax_env morlax_env;
int morlax_env_spec(const char* name, int* obs_dim, int* act_dim, int* m, int* max_episode_steps);
int morlax_env_create(const char* name, int num_envs, morlax_env** out);
void morlax_env_destroy(morlax_env* env);
/* BatchedEnv::reset(const Rng&): instance i streams from split(i) */
int morlax_env_reset(morlax_env* env, uint64_t key, uint64_t ctr, float* obs_out /* N*obs or NULL */);
/* BatchedEnv::step(span actions, StepOut&): host buffers */
int morlax_env_step(morlax_env* env, const float* actions, float* obs, float* reward, uint8_t* terminated,
                    uint8_t* truncated);
/* same on device buffers, async on `stream` */
int morlax_env_step_device(morlax_env* env, const float* d_actions, float* d_obs, float* d_reward,
                           uint8_t* d_terminated, uint8_t* d_truncated, void* stream);
int morlax_env_current_obs(morlax_env* env, float* obs_out);
uint64_t morlax_env_clamp_count(morlax_env* env);

/* ---- Hypernetwork (replaces hypernet_forward / hypernet_backward /
 *      init_hypernet, include/morlax/hypernet.hpp:52-75) ------------------ */
typedef struct {
    int m, F;
    int n_feature_hidden;
    int feature_hidden[8];
    int n_target_sizes; /* [in, hidden..., out] */
    int target_sizes[9];
    int target_tanh;    /* policy head (tanh) vs critic (identity) */
    int has_log_std;
} morlax_hypernet_spec;
int64_t morlax_hypernet_param_count(const morlax_hypernet_spec* spec);
int64_t morlax_hypernet_target_count(const morlax_hypernet_spec* spec);
/* flat = [feature | M (P x F) | b], reference flatten_hypernet order */
int morlax_init_hypernet(const morlax_hypernet_spec* spec, uint64_t key, uint64_t ctr, double* flat_out);
/* theta[g] = M f(w_g) + b for G preference vectors w [G][m] */
int morlax_hypernet_forward(const morlax_hypernet_spec* spec, const double* flat, const double* w, int G,
                            double* theta_out /* G*P */);
/* sum_g hypernet_backward(w_g, gtheta_g) into grad_out (overwritten) */
int morlax_hypernet_backward(const morlax_hypernet_spec* spec, const double* flat, const double* w, int G,
                             const double* gtheta /* G*P */, double* grad_out);

/* ---- Per-preference-group policy forward (replaces policy_forward,
 *      src/nn.cpp:162-190, over hypernet_forward's generated weights,
 *      src/hypernet.cpp:69-90, for G preferences x R observations each) --- */
typedef struct morlax_policy morlax_policy;
int morlax_policy_create(const morlax_hypernet_spec* spec, int groups, int rows_per_group, morlax_policy** out);
void morlax_policy_destroy(morlax_policy* p);
/* flat = [feature | M | b] (reference flatten_hypernet order) */
int morlax_policy_set_params(morlax_policy* p, const double* flat);
/* w [G][m] on the simplex (ShapeError/DomainError as hypernet_forward),
 * obs [G*R][obs_dim] grouped by preference -> pre [G*R][out]: the Gaussian
 * mean before the tanh squash (GaussianAction::pre); host buffers */
int morlax_policy_forward(morlax_policy* p, const double* w, const float* obs, float* pre_out);
/* same on device buffers (w as fp32), async on `stream` */
int morlax_policy_forward_device(morlax_policy* p, const float* d_w, const float* d_obs, float* d_pre, void* stream);
/* algorithmic FLOPs of one forward (feature MLP + theta GEMM + per-row MLP) */
double morlax_policy_flops(morlax_policy* p);

/* ---- Evaluation (replaces evaluate_params / eval_point,
 *      src/evaluate.cpp:17-101, and simplex_grid_size, simplex.cpp:119) --- */
int64_t morlax_simplex_grid_size(int m, int resolution);
/* for every w of simplex_grid(m, resolution) (reference order) the
 * deterministic policy (tanh of the mean) of the actor hypernet `flat` runs
 * episodes_per_point fresh instances reset from Rng(key).split(g) for one
 * episode each; w_out / mean_return_out are [n_points][m] */
int morlax_evaluate_params(const morlax_hypernet_spec* actor_spec, const double* flat, const char* env_name,
                           int grid_resolution, int episodes_per_point, uint64_t key, double* w_out,
                           double* mean_return_out, int64_t* n_points);

/* ---- Advantage estimation (replaces gae_per_objective /
 *      normalize_and_scalarize, include/morlax/trainer.hpp:154-161) ------ */
int morlax_gae(int N, int T, int m, const float* reward, const float* value, const float* next_value,
               const uint8_t* terminated, const uint8_t* truncated, double gamma, double lambda,
               float* advantages_out, float* value_targets_out);
int morlax_normalize_scalarize(int N, int T, int m, const float* advantages,
                               const double* tradeoffs /* N*m */, float* out);

/* ---- Adam (replaces adam_apply, include/morlax/trainer.hpp:211-212) ----- */
int morlax_adam(int64_t n, double* params, const double* grad, double* m1, double* m2, int64_t* step,
                double lr);

/* ---- Trainer (replaces train(), include/morlax/trainer.hpp:256-257, and
 *      the loop body of src/train.cpp:118-184: collect_rollouts,
 *      gae_per_objective, normalize_and_scalarize, actor_loss,
 *      critic_loss, adam_apply) --------------------------------------------- */
typedef struct {
    const char* env_name;
    int N, K, kappa, T, epochs, minibatch_count;
    double gamma, gae_lambda, clip_eps, actor_lr, critic_lr, entropy_coef;
    uint64_t seed;
    int F;
    int n_feature_hidden;
    int feature_hidden[8];
    int n_actor_hidden;
    int actor_hidden[8];
    int n_critic_hidden;
    int critic_hidden[8];
} morlax_train_config;

typedef struct {
    double actor_loss;  /* summed over minibatch steps (IterationStats) */
    double critic_loss;
    int minibatches;
    int numeric_error;
    int64_t kernel_launches; /* cumulative */
} morlax_iter_stats;

typedef struct morlax_trainer morlax_trainer;
/* world > 1: one trainer per GPU/rank; nccl_id = 128 bytes from
 * morlax_nccl_unique_id() on rank 0, broadcast by the caller. A non-NULL
 * nccl_id with world == 1 builds a single-rank communicator (the
 * multi-GPU code path on one GPU; results identical to nccl_id == NULL). */
int morlax_nccl_unique_id(void* out128);
int morlax_trainer_create(const morlax_train_config* cfg, int world, int rank, const void* nccl_id,
                          morlax_trainer** out);
void morlax_trainer_destroy(morlax_trainer* t);
/* In-process loopback group: `world` ranks as host threads of ONE process
 * on ONE device (comm.h). Each rank's trainer runs the sharded multi-GPU
 * data plane (all-to-all of the per-cluster gradient shards, sharded dM +
 * Adam, all-gathers of the M image / b / feature gradients) with
 * device-to-device copies in place of NCCL; every rank must drive its
 * trainer from its own thread (the collectives meet at host barriers).
 * Results equal the single-rank trainer's bit for bit (tests only: it
 * measures nothing about NVLink). */
typedef struct morlax_loopback morlax_loopback;
int morlax_loopback_create(int world, morlax_loopback** out);
void morlax_loopback_destroy(morlax_loopback* g); /* after every trainer of the group */
int morlax_trainer_create_loopback(const morlax_train_config* cfg, morlax_loopback* group, int rank,
                                   morlax_trainer** out);
/* one full training iteration `it` (host-facing: H2D of sampled
 * preferences and minibatch indices, D2H of the stats, inside the call) */
int morlax_trainer_iteration(morlax_trainer* t, int it, morlax_iter_stats* stats);
/* phases: 1 sampling + rollout, 2 GAE + normalise, 3 update (first
 * max_minibatches, -1 = all), 4 finish (sync, stats, NumericError),
 * 5 minibatch plans only (instead of 1 when the batch and the clusters were
 * set through morlax_trainer_set: the GAE + PPO update of config 4) */
int morlax_trainer_phase(morlax_trainer* t, int it, int phase, int max_minibatches, morlax_iter_stats* stats);
int morlax_trainer_sizes(morlax_trainer* t, int64_t* actor_params, int64_t* critic_params, int* local_envs,
                         int* local_clusters, int* rows_per_iteration);
/* which: 0 actor, 1 critic. fp64 reference flat layout */
int morlax_trainer_get_params(morlax_trainer* t, int which, double* out);
int morlax_trainer_set_params(morlax_trainer* t, int which, const double* in);
/* flat hypernet gradient of the last backward pass (morlax_trainer_losses
 * or the last minibatch of an iteration) */
int morlax_trainer_get_grad(morlax_trainer* t, int which, double* out);
/* Checkpoint wire format of the reference (save_checkpoint / load_checkpoint,
 * src/checkpoint.cpp:15-241; "MRLXCKPT" v1, little-endian fixed width): the
 * trainer's RunConfig, specs, fp64 params in flatten_hypernet order,
 * `iteration`, root Rng(seed) key / counter. The RunConfig fields the
 * trainer does not hold come from `extra` (NULL = the reference defaults:
 * iterations 300, eval grid 10 / 8 episodes / interval 10, empty pareto
 * reference). Loading checks magic, version, architecture and counts
 * (ConfigError) and sets both hypernets' params (like the reference, no
 * Adam state is stored). */
typedef struct {
    int iterations;
    int grid_resolution, episodes_per_point, log_interval;
    int n_pareto_reference;
    const double* pareto_reference;
} morlax_checkpoint_extra;
int morlax_trainer_save_checkpoint(morlax_trainer* t, const char* path, int64_t iteration,
                                   const morlax_checkpoint_extra* extra);
int morlax_trainer_load_checkpoint(morlax_trainer* t, const char* path, int64_t* iteration_out);

/* ---- Training loop (replaces train(RunConfig, TrainOptions,
 *      IterationCallback), include/morlax/trainer.hpp:237-257 and
 *      src/train.cpp:55-229, single rank): iterations of the device loop
 *      body; every log_interval (and the last) iteration evaluate_params ->
 *      archive -> nondominated_filter -> hypervolume; out_dir/metrics.csv
 *      (iteration,wall_ms,cluster_<c>_return...,archive_hypervolume; "%.17g")
 *      and out_dir/checkpoint.bin (MRLXCKPT v1: the final params, or on a
 *      NumericError the last healthy iteration's, then status 3). `out`
 *      (optional) receives the trained trainer (free with
 *      morlax_trainer_destroy); NULL destroys it. */
typedef struct {
    const char* out_dir; /* NULL / "" disables checkpoint.bin and metrics.csv (TrainOptions::out_dir) */
    int iterations;      /* TrainerConfig::iterations */
    int grid_resolution, episodes_per_point, log_interval; /* EvalConfig */
    int n_pareto_reference;
    const double* pareto_reference; /* NULL: the env's hv_reference */
    int deterministic;   /* wall_ms logged as 0 (TrainOptions::deterministic) */
} morlax_run_options;
typedef struct {         /* IterationStats (trainer.hpp:243-249) */
    int iteration;
    double actor_loss, critic_loss, archive_hypervolume;
    int n_clusters;
    const double* cluster_returns; /* valid during the callback */
} morlax_iteration_stats;
/* a non-zero return stops training (train() propagates a callback's
 * exception): morlax_train returns 1, last error "iteration callback failed" */
typedef int (*morlax_iteration_callback)(const morlax_iteration_stats* stats, void* user);
int morlax_train(const morlax_train_config* cfg, const morlax_run_options* opts, morlax_iteration_callback cb,
                 void* user, morlax_trainer** out);

int morlax_trainer_get_theta(morlax_trainer* t, int which, float* out /* local K x P */);
/* field: obs action_pre logprob reward value next_value advantages
 * value_targets scalar_advantage (float) | terminated truncated (uint8) |
 * clusters (float K*m) | perm (int32 N*T) | env_state (float sdim*N) */
int morlax_trainer_get(morlax_trainer* t, const char* field, void* out);
int morlax_trainer_set(morlax_trainer* t, const char* field, const void* in);
/* actor_loss + critic_loss through the hypernetwork on global rows
 * `rows` of the current batch; leaves grads in get_grad; no Adam */
int morlax_trainer_losses(morlax_trainer* t, const int32_t* rows, int n_rows, double* actor_loss,
                          double* critic_loss);
int64_t morlax_trainer_kernel_launches(morlax_trainer* t);
/* per-kernel-class CUDA-event timing (+ algorithmic FLOPs / bytes) of the
 * launches made while enabled; enabling resets the tallies */
int morlax_trainer_profile_enable(morlax_trainer* t, int on);
int morlax_trainer_profile_count(morlax_trainer* t);
int morlax_trainer_profile_get(morlax_trainer* t, int i, char* name64, double* ms, double* flops, double* bytes,
                               int64_t* count);
/* per-launch timeline of the profiled iteration (class, stream index,
 * start / end in ms from its first launch; CUDA events around each launch) */
int morlax_trainer_profile_timeline_count(morlax_trainer* t);
int morlax_trainer_profile_timeline(morlax_trainer* t, int i, char* name64, int* stream, double* t0_ms,
                                    double* t1_ms);
void* morlax_trainer_stream(morlax_trainer* t);

/* host-side sharding helper (pure): rows of perm[lo:hi) that belong to
 * instances [inst_lo, inst_lo+n_inst), local row ids grouped by cluster */
/* host helper: the sharded optimizer's partition of the P hypernet rows
 * (M rows and b entries): shard width S (a multiple of 128), rank's rows
 * [row_lo, row_hi) */
int morlax_shard_rows(int64_t P, int world, int rank, int64_t* S, int64_t* row_lo, int64_t* row_hi);
int morlax_shard_minibatch(const int32_t* perm, int lo, int hi, int T, int inst_lo, int n_inst, int reps,
                           int n_groups, int32_t* rows_out, int32_t* goff_out, int* n_rows_out,
                           int* max_group_out);

/* ---- test hook: C[M][N] = A(m,k) B(k,n) with strided fp32 operands, on the
 *      tcgen05 path (use_tc must be 1; the SIMT path was removed: ConfigError) */
int morlax_gemm_test(int M, int N, int K, const float* A, long am, long ak, const float* B, long bk, long bn,
                     float* C, int use_tc);

/* microbenchmark hook for the tcgen05 GEMM (tools/gemm_bench.py): ms per launch */
/* test hook: fused hypernet M-block gradient + Adam (dm_adam.cu) on host
 * arrays: dM = gtheta^T f (bf16 operands, fp32 accumulation; G groups in
 * 128-group K chunks) and Adam on p / m1 / m2 [P][F] (hypernet.cpp:92-122 dM,
 * adam.cpp:8-26); also returns the bf16 bits of the refreshed M image rows */
int morlax_dm_adam_test(int G, int P, int F, const float* gtheta, const float* f, float* p, float* m1, float* m2,
                        float lr, float ibc1, float ibc2, uint16_t* mimg_rows);
int morlax_gemm_bench(int M, int N, int K, int a_view, int b_view, int act, int iters, double* ms);

/* ---- Pareto (replaces nondominated_filter / hypervolume_mc /
 *      hypervolume_detailed, include/morlax/pareto.hpp:21-56) ------------ */
/* survivors of nondominated_filter as a mask over the input order */
int morlax_pareto_mask(int n, int m, const double* points, uint8_t* mask_out);
int morlax_pareto_mask_device(int n, int m, const double* d_points, uint8_t* d_mask, void* stream);
/* survivors of linear_dominance_filter (pareto.cpp:79-139) as a mask over
 * the input order: nondominated points that attain max_w w.J (m == 2: the
 * upper hull, collinear kept; m >= 3: the simplex_grid(m, 60) sweep) */
int morlax_linear_dominance_mask(int n, int m, const double* points, uint8_t* mask_out);
int morlax_hypervolume_mc(int n, int m, const double* points, const double* reference, uint64_t samples,
                          uint64_t key, uint64_t ctr, double* value, double* stderr_out, uint64_t* hits);
/* hypervolume_detailed (pareto.cpp:209-230): exact for m <= 4 (device WFG
 * recursion, same value as the reference's slicing recursion to fp64
 * rounding), above that the reference's Monte-Carlo with `samples` and
 * Rng(seed) on the device (bit-identical hit count) */
int morlax_hypervolume_detailed(int n, int m, const double* points, const double* reference,
                                uint64_t samples, uint64_t seed, double* value, double* stderr_out,
                                int* exact, int* clipped);

/* exact hypervolume for any m <= 8 (new: the reference has no exact
 * algorithm above m = 4): WFG exclusive-volume recursion on the device,
 * fp64; points below the reference are clipped (pareto.cpp:191-205) and
 * counted. The _device form takes device pointers and synchronises `stream`. */
int morlax_hypervolume_exact(int n, int m, const double* points, const double* reference, double* value,
                             int* clipped);
int morlax_hypervolume_exact_device(int n, int m, const double* d_points, const double* d_reference,
                                    double* value, int* clipped, void* stream);

#ifdef __cplusplus
}
#endif
#endif
