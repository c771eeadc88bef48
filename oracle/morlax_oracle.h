/* TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * morlax_oracle: a plain-C, fp64 restatement of the MORLAX reference
 * (/root/reference/proj) hot path: counter RNG, preference sampling,
 * batched envs, flat-parameter MLPs, the affine hypernetwork, rollouts,
 * per-objective GAE + normalise/scalarise, clipped-PPO actor / vector
 * critic losses through the hypernetwork, Adam, the train-iteration body,
 * Pareto dominance and hypervolume. Each function cites the reference
 * file:line it restates. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may call it.
 *
 * Pinning: tests/test_oracle_vs_ref.py checks every entry point against the
 * compiled reference (oracle/_ref/libmorlax_ref.so, built from the
 * reference sources in place by oracle/Makefile) and against the
 * known-answer fixtures of the reference tests (tests/golden/).
 *
 * Error convention (mirrors include/morlax/errors.hpp + tools/commands.hpp):
 * return 0 ok, 2 Config/Shape/Domain error, 3 NumericError; message via
 * mo_last_error().
 */
#ifndef MORLAX_ORACLE_H
#define MORLAX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MO_OK 0
#define MO_ERR 2
#define MO_NUMERIC 3

const char* mo_last_error(void);

/* ---- RNG (rng.hpp:18-93) ---------------------------------------------- */
typedef struct { uint64_t key, ctr; } mo_rng;
mo_rng mo_rng_seed(uint64_t seed);
mo_rng mo_rng_split(mo_rng r, uint64_t lane);
uint64_t mo_rng_next_u64(mo_rng* r);
double mo_rng_next_double(mo_rng* r);
double mo_rng_next_open(mo_rng* r);
double mo_rng_uniform(mo_rng* r, double lo, double hi);
double mo_rng_next_gaussian(mo_rng* r);
uint64_t mo_rng_next_below(mo_rng* r, uint64_t n);
void mo_rng_shuffle_i32(mo_rng* r, int32_t* v, int64_t n);
/* ctypes-friendly wrappers */
void mo_rng_seed_state(uint64_t seed, uint64_t* key, uint64_t* ctr);
uint64_t mo_rng_split_key(uint64_t key, uint64_t lane);
void mo_rng_words(uint64_t key, uint64_t ctr, int64_t n, uint64_t* out);
void mo_rng_gaussians(uint64_t key, uint64_t ctr, int64_t n, double* out);
void mo_rng_shuffle(uint64_t key, uint64_t* ctr, int32_t* v, int64_t n);

/* ---- specs --------------------------------------------------------------- */
#define MO_MAX_LAYERS 8
typedef struct {
    int n_sizes;               /* layer_sizes.size() */
    int sizes[MO_MAX_LAYERS + 1];
    int out_tanh;              /* output activation tanh (else identity) */
} mo_mlp;
typedef struct {
    int m, F;
    int n_feat_hidden;
    int feat_hidden[MO_MAX_LAYERS];
    mo_mlp target;
    int has_log_std;
} mo_hspec;

int64_t mo_mlp_param_count(const mo_mlp* s);
int64_t mo_hspec_feature_count(const mo_hspec* h);
int64_t mo_hspec_target_count(const mo_hspec* h);
int64_t mo_hspec_param_count(const mo_hspec* h);
void mo_hspec_feature_spec(const mo_hspec* h, mo_mlp* out);

/* ---- NN (nn.cpp) ----------------------------------------------------------- */
int mo_mlp_forward(const mo_mlp* s, const double* params, const double* in, double* out);
int mo_init_mlp(const mo_mlp* s, uint64_t key, uint64_t ctr, double* out);

/* ---- Hypernet (hypernet.cpp), flat = [feature | M (P x F) | b (P)] ------- */
int mo_init_hypernet(const mo_hspec* h, uint64_t key, uint64_t ctr, double* flat);
int mo_hypernet_forward(const mo_hspec* h, const double* flat, const double* w, double* theta);
int mo_hypernet_features(const mo_hspec* h, const double* flat, const double* w, double* f);
int mo_hypernet_backward(const mo_hspec* h, const double* flat, const double* w,
                         const double* gtheta, double* gflat);

/* ---- Envs (env.cpp, env_*.cpp; humanoid6 defined in csrc/humanoid6_params.h) */
enum { MO_ENV_LQR = 0, MO_ENV_LQR_M1 = 1, MO_ENV_POINTMASS = 2, MO_ENV_DST = 3,
       MO_ENV_HUMANOID6 = 4 };
typedef struct { int kind, obs_dim, act_dim, m, max_steps; } mo_envspec;
int mo_env_spec(int kind, mo_envspec* out);
int mo_env_kind_from_name(const char* name);
typedef struct mo_env mo_env;
mo_env* mo_env_create(int kind, int n);
void mo_env_destroy(mo_env* e);
int mo_env_reset(mo_env* e, uint64_t key, uint64_t ctr, double* obs_out);
int mo_env_step(mo_env* e, const double* actions, double* obs, double* reward,
                uint8_t* term, uint8_t* trunc);
void mo_env_current_obs(const mo_env* e, double* out);
uint64_t mo_env_clamp_count(const mo_env* e);
/* streams (key, ctr) and step counters per instance */
void mo_env_get_streams(const mo_env* e, uint64_t* keys, uint64_t* ctrs, int32_t* steps);
/* test hook: restart instances from given states / counters (teacher forcing) */
void mo_env_set_instances(mo_env* e, const double* state, const int32_t* steps, const uint64_t* keys,
                          const uint64_t* ctrs);

/* ---- Rollout (rollout.cpp:37-161) ---------------------------------------- */
typedef struct {
    double *obs, *action_pre, *logprob, *reward, *value, *next_value;
    uint8_t *term, *trunc;
} mo_batch;
int mo_collect_rollouts(const mo_hspec* a, const double* aflat,
                        const mo_hspec* c, const double* cflat, mo_env* env,
                        const double* cluster_w, int K, int reps, int T,
                        uint64_t key, uint64_t ctr, mo_batch* out,
                        double* tracker_running /* N*m, may be NULL */);

/* ---- GAE (gae.cpp:26-117) ---------------------------------------------- */
int mo_gae(int N, int T, int m, const double* reward, const double* value,
           const double* next_value, const uint8_t* term, const uint8_t* trunc,
           double gamma, double lambda, double* adv, double* targets);
int mo_normalize_scalarize(int N, int T, int m, const double* adv,
                           const double* tradeoffs /* N*m */, double* out);

/* ---- Losses (losses.cpp:46-189) ---------------------------------------- */
int mo_actor_loss(const mo_hspec* h, const double* flat, int N, int T,
                  const double* obs, const double* action_pre,
                  const double* logprob_old, const double* tradeoffs /* N*m */,
                  const int32_t* cluster /* N */, const int32_t* rows, int n_rows,
                  const double* sadv, double clip_eps, double entropy_coef,
                  double* loss, double* gflat);
int mo_critic_loss(const mo_hspec* h, const double* flat, int N, int T,
                   const double* obs, const double* tradeoffs, const int32_t* cluster,
                   const int32_t* rows, int n_rows, const double* targets,
                   double* loss, double* gflat);

/* ---- Adam (adam.cpp:8-26) ------------------------------------------------ */
int mo_adam(int64_t n, double* p, const double* g, double* m1, double* m2,
            int64_t* step, double lr);

/* ---- Train iteration (train.cpp:55-229, loop body :118-184) -------------- */
typedef struct {
    int env_kind;
    int N, K, kappa, T, epochs, minibatch_count;
    double gamma, lambda, clip_eps, actor_lr, critic_lr, entropy_coef;
    uint64_t seed;
    int F;
    int n_feat_hidden, feat_hidden[MO_MAX_LAYERS];
    int n_actor_hidden, actor_hidden[MO_MAX_LAYERS];
    int n_critic_hidden, critic_hidden[MO_MAX_LAYERS];
} mo_train_cfg;
typedef struct mo_trainer mo_trainer;
mo_trainer* mo_trainer_create(const mo_train_cfg* cfg);
void mo_trainer_destroy(mo_trainer* t);
void mo_trainer_specs(const mo_trainer* t, mo_hspec* actor, mo_hspec* critic);
/* phases: 1 = sampling+rollout only, 2 = + gae/normalise, 3 = full update.
 * `max_minibatches` < 0 runs all; otherwise stops after that many (for
 * bounded CPU-baseline samples). */
int mo_trainer_iteration(mo_trainer* t, int it, int max_minibatches,
                         double* actor_loss_sum, double* critic_loss_sum);
double* mo_trainer_actor_params(mo_trainer* t);
double* mo_trainer_critic_params(mo_trainer* t);
int32_t* mo_trainer_perm(mo_trainer* t);
mo_env* mo_trainer_env(mo_trainer* t);
/* last iteration's batch / gae outputs (valid after an iteration) */
const mo_batch* mo_trainer_batch(const mo_trainer* t);
const double* mo_trainer_advantages(const mo_trainer* t);
const double* mo_trainer_targets(const mo_trainer* t);
const double* mo_trainer_sadv(const mo_trainer* t);
const double* mo_trainer_clusters(const mo_trainer* t);
const double* mo_trainer_tracker(const mo_trainer* t);

/* ---- Pareto (pareto.cpp) ------------------------------------------------- */
int mo_dominates(int m, const double* a, const double* b);
int mo_nondominated_mask(int n, int m, const double* pts, uint8_t* mask);
int mo_hypervolume_exact(int n, int m, const double* pts, const double* ref,
                         double* value, int* clipped);
int mo_hypervolume_mc(int n, int m, const double* pts, const double* ref,
                      uint64_t samples, uint64_t key, uint64_t ctr, double* value,
                      double* stderr_out, uint64_t* hits);
/* hypervolume_detailed (pareto.cpp:209-230): exact for m <= 4 else MC */
int mo_hypervolume_detailed(int n, int m, const double* pts, const double* ref,
                            uint64_t samples, uint64_t seed, double* value,
                            double* stderr_out, int* exact, int* clipped);
/* ---- simplex_grid (simplex.cpp:108-130) and evaluate_params
 * (evaluate.cpp:17-101): w_out [n_points][m], mean_out [n_points][m] */
int64_t mo_simplex_grid_size(int m, int res);
int mo_simplex_grid(int m, int res, double* out);
int mo_evaluate_params(const mo_hspec* h, const double* flat, int env_kind, int res, int episodes,
                       uint64_t key, double* w_out, double* mean_out, int64_t* n_points);
/* linear_dominance_filter (pareto.cpp:79-139) as a survivor mask over the
 * input order (duplicates: first occurrence) */
int mo_linear_dominance_mask(int n, int m, const double* pts, uint8_t* mask);
/* New exact algorithm for any m (WFG-style exclusive-volume recursion). Not
 * in the reference (which has no exact algorithm above m = 4). */
int mo_hypervolume_wfg(int n, int m, const double* pts, const double* ref, double* value);

#ifdef __cplusplus
}
#endif
#endif
