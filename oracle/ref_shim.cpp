// TEST INFRASTRUCTURE ONLY. extern "C" shim over the COMPILED REFERENCE
// (/root/reference/proj/src/*.cpp built in place by oracle/Makefile into
// oracle/_ref/libmorlax_ref.so). It exposes the reference's own functions
// with the same flat signatures as the C oracle (prefix mref_ instead of
// mo_), so tests can pin the oracle against the reference, and bench.py's
// `--impl reference` arm can time the reference CPU path.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "morlax/env.hpp"
#include "morlax/envs.hpp"
#include "morlax/errors.hpp"
#include "morlax/hypernet.hpp"
#include "morlax/nn.hpp"
#include "morlax/pareto.hpp"
#include "morlax/rng.hpp"
#include "morlax/simplex.hpp"
#include "morlax/trainer.hpp"

extern "C" {
#include "morlax_oracle.h"
}

using namespace morlax;

std::unique_ptr<BatchedEnv> make_humanoid6_env(int n);  // ref_humanoid6.cpp

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {  // tools/commands.hpp:12-32 exit-code mapping
    try {
        fn();
        return 0;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const DomainError& e) {
        g_err = e.what();
        return 2;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

HypernetSpec to_spec(const mo_hspec* h) {
    HypernetSpec s;
    s.m = h->m;
    s.F = h->F;
    for (int i = 0; i < h->n_feat_hidden; ++i) s.feature_hidden.push_back(h->feat_hidden[i]);
    for (int i = 0; i < h->target.n_sizes; ++i) s.target_spec.layer_sizes.push_back(h->target.sizes[i]);
    s.target_spec.output_activation = h->target.out_tanh ? Activation::kTanh : Activation::kIdentity;
    s.target_has_log_std = h->has_log_std != 0;
    return s;
}

const char* env_name(int kind) {
    switch (kind) {
        case MO_ENV_LQR: return "mo-lqr1d";
        case MO_ENV_LQR_M1: return "mo-lqr1d-m1";
        case MO_ENV_POINTMASS: return "mo-pointmass";
        case MO_ENV_DST: return "mo-dst-continuous";
    }
    return "mo-humanoid6";
}

std::unique_ptr<BatchedEnv> make_any_env(int kind, int n) {
    if (kind == MO_ENV_HUMANOID6) return make_humanoid6_env(n);
    return make_env(env_name(kind), n);
}

struct RefEnv {
    std::unique_ptr<BatchedEnv> env;
};

}  // namespace

extern "C" {

const char* mref_last_error(void) { return g_err.c_str(); }

void mref_rng_words(uint64_t key, uint64_t ctr, int64_t n, uint64_t* out) {
    Rng r = Rng::from_state(key, ctr);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void mref_rng_gaussians(uint64_t key, uint64_t ctr, int64_t n, double* out) {
    Rng r = Rng::from_state(key, ctr);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_gaussian();
}
void mref_rng_seed_state(uint64_t seed, uint64_t* key, uint64_t* ctr) {
    Rng r(seed);
    *key = r.key();
    *ctr = r.counter();
}
uint64_t mref_rng_split_key(uint64_t key, uint64_t lane) {
    return Rng::from_state(key, 0).split(lane).key();
}
void mref_rng_shuffle(uint64_t key, uint64_t* ctr, int32_t* v, int64_t n) {
    Rng r = Rng::from_state(key, *ctr);
    std::vector<int> p(v, v + n);
    r.shuffle(p);
    std::copy(p.begin(), p.end(), v);
    *ctr = r.counter();
}
void mref_dirichlet(uint64_t key, uint64_t ctr, int m, int n, double* out) {
    Rng r = Rng::from_state(key, ctr);
    auto v = dirichlet_sample(r, m, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < m; ++j) out[i * m + j] = v[i].weights[j];
}

int mref_init_hypernet(const mo_hspec* h, uint64_t key, uint64_t ctr, double* flat) {
    return guarded([&] {
        Rng r = Rng::from_state(key, ctr);
        auto f = flatten_hypernet(init_hypernet(to_spec(h), r));
        std::copy(f.begin(), f.end(), flat);
    });
}
int mref_hypernet_forward(const mo_hspec* h, const double* flat, const double* w, double* theta) {
    return guarded([&] {
        const HypernetSpec s = to_spec(h);
        const auto hp = unflatten_hypernet(s, {flat, (size_t)hypernet_param_count(s)});
        auto th = hypernet_forward(s, hp, TradeoffVector{std::vector<double>(w, w + h->m)});
        std::copy(th.begin(), th.end(), theta);
    });
}
int mref_hypernet_backward(const mo_hspec* h, const double* flat, const double* w,
                           const double* gtheta, double* gflat) {
    return guarded([&] {
        const HypernetSpec s = to_spec(h);
        const auto hp = unflatten_hypernet(s, {flat, (size_t)hypernet_param_count(s)});
        HypernetGrad g;
        g.resize_like(s);
        hypernet_backward(s, hp, TradeoffVector{std::vector<double>(w, w + h->m)},
                          {gtheta, s.target_param_count()}, g);
        auto f = flatten_hypernet_grad(g);
        for (size_t i = 0; i < f.size(); ++i) gflat[i] += f[i];
    });
}

void* mref_env_create(int kind, int n) {
    try {
        auto* e = new RefEnv{make_any_env(kind, n)};
        return e;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}
void mref_env_destroy(void* e) { delete static_cast<RefEnv*>(e); }
int mref_env_reset(void* e, uint64_t key, uint64_t ctr, double* obs) {
    return guarded([&] {
        auto o = static_cast<RefEnv*>(e)->env->reset(Rng::from_state(key, ctr));
        if (obs) std::copy(o.begin(), o.end(), obs);
    });
}
int mref_env_step(void* e, const double* actions, double* obs, double* reward, uint8_t* term,
                  uint8_t* trunc) {
    return guarded([&] {
        BatchedEnv& env = *static_cast<RefEnv*>(e)->env;
        const size_t na = (size_t)env.num_envs() * env.spec().act_dim;
        BatchedEnv::StepOut out;
        env.step({actions, na}, out);
        std::copy(out.obs.begin(), out.obs.end(), obs);
        std::copy(out.reward.begin(), out.reward.end(), reward);
        std::copy(out.terminated.begin(), out.terminated.end(), term);
        std::copy(out.truncated.begin(), out.truncated.end(), trunc);
    });
}
void mref_env_current_obs(void* e, double* out) {
    auto o = static_cast<RefEnv*>(e)->env->current_obs();
    std::copy(o.begin(), o.end(), out);
}
uint64_t mref_env_clamp_count(void* e) { return static_cast<RefEnv*>(e)->env->clamp_count(); }

static void fill_batch(const RolloutBatch& b, mo_batch* o) {
    std::copy(b.obs.begin(), b.obs.end(), o->obs);
    std::copy(b.action_pre.begin(), b.action_pre.end(), o->action_pre);
    std::copy(b.logprob_old.begin(), b.logprob_old.end(), o->logprob);
    std::copy(b.reward.begin(), b.reward.end(), o->reward);
    std::copy(b.value.begin(), b.value.end(), o->value);
    std::copy(b.next_value.begin(), b.next_value.end(), o->next_value);
    std::copy(b.terminated.begin(), b.terminated.end(), o->term);
    std::copy(b.truncated.begin(), b.truncated.end(), o->trunc);
}

int mref_collect_rollouts(const mo_hspec* a, const double* aflat, const mo_hspec* c,
                          const double* cflat, void* env, const double* cw, int K, int reps,
                          int T, uint64_t key, uint64_t ctr, mo_batch* out, int threads) {
    return guarded([&] {
        const HypernetSpec as = to_spec(a), cs = to_spec(c);
        const auto ap = unflatten_hypernet(as, {aflat, (size_t)hypernet_param_count(as)});
        const auto cp = unflatten_hypernet(cs, {cflat, (size_t)hypernet_param_count(cs)});
        std::vector<TradeoffVector> cl;
        for (int k = 0; k < K; ++k) cl.push_back(TradeoffVector{std::vector<double>(cw + k * a->m, cw + (k + 1) * a->m)});
        RolloutBatch b = collect_rollouts(as, ap, cs, cp, *static_cast<RefEnv*>(env)->env, cl, reps, T,
                                          Rng::from_state(key, ctr), threads);
        fill_batch(b, out);
    });
}

static RolloutBatch gae_batch(int N, int T, int m, const double* reward, const double* value,
                              const double* next_value, const uint8_t* term, const uint8_t* trunc) {
    RolloutBatch b;
    b.resize(N, T, m, 1, 1);
    const size_t r = (size_t)N * T;
    std::copy(reward, reward + r * m, b.reward.begin());
    std::copy(value, value + r * m, b.value.begin());
    std::copy(next_value, next_value + r * m, b.next_value.begin());
    std::copy(term, term + r, b.terminated.begin());
    std::copy(trunc, trunc + r, b.truncated.begin());
    return b;
}

int mref_gae(int N, int T, int m, const double* reward, const double* value, const double* next_value,
             const uint8_t* term, const uint8_t* trunc, double gamma, double lambda, double* adv,
             double* targets) {
    return guarded([&] {
        RolloutBatch b = gae_batch(N, T, m, reward, value, next_value, term, trunc);
        GaeResult g = gae_per_objective(b, gamma, lambda);
        std::copy(g.advantages.begin(), g.advantages.end(), adv);
        std::copy(g.value_targets.begin(), g.value_targets.end(), targets);
    });
}
int mref_normalize_scalarize(int N, int T, int m, const double* adv, const double* tw, double* out) {
    return guarded([&] {
        RolloutBatch b;
        b.resize(N, T, m, 1, 1);
        for (int i = 0; i < N; ++i) b.tradeoffs.push_back(TradeoffVector{std::vector<double>(tw + i * m, tw + (i + 1) * m)});
        std::vector<double> a(adv, adv + (size_t)N * T * m);
        auto s = normalize_and_scalarize(a, b);
        std::copy(s.begin(), s.end(), out);
    });
}

static RolloutBatch loss_batch(const mo_hspec* h, int N, int T, int m, const double* obs,
                               const double* action_pre, const double* logprob_old,
                               const double* tw, const int32_t* cluster) {
    const int od = h->target.sizes[0];
    const int ad = h->has_log_std ? h->target.sizes[h->target.n_sizes - 1] : 1;
    RolloutBatch b;
    b.resize(N, T, m, od, ad);
    const size_t r = (size_t)N * T;
    std::copy(obs, obs + r * od, b.obs.begin());
    if (action_pre) std::copy(action_pre, action_pre + r * ad, b.action_pre.begin());
    if (logprob_old) std::copy(logprob_old, logprob_old + r, b.logprob_old.begin());
    for (int i = 0; i < N; ++i) {
        b.tradeoffs.push_back(TradeoffVector{std::vector<double>(tw + i * m, tw + (i + 1) * m)});
        b.cluster[i] = cluster[i];
    }
    return b;
}

int mref_actor_loss(const mo_hspec* h, const double* flat, int N, int T, const double* obs,
                    const double* action_pre, const double* logprob_old, const double* tw,
                    const int32_t* cluster, const int32_t* rows, int n_rows, const double* sadv,
                    double clip, double ent, double* loss, double* gflat) {
    return guarded([&] {
        const HypernetSpec s = to_spec(h);
        const auto hp = unflatten_hypernet(s, {flat, (size_t)hypernet_param_count(s)});
        RolloutBatch b = loss_batch(h, N, T, h->m, obs, action_pre, logprob_old, tw, cluster);
        std::vector<double> sa(sadv, sadv + (size_t)N * T);
        Minibatch mb;
        mb.batch = &b;
        mb.rows.assign(rows, rows + n_rows);
        mb.scalar_advantage = &sa;
        LossResult lr = actor_loss(s, hp, mb, clip, ent);
        *loss = lr.loss;
        auto g = flatten_hypernet_grad(lr.grad);
        std::copy(g.begin(), g.end(), gflat);
    });
}
int mref_critic_loss(const mo_hspec* h, const double* flat, int N, int T, const double* obs,
                     const double* tw, const int32_t* cluster, const int32_t* rows, int n_rows,
                     const double* targets, double* loss, double* gflat) {
    return guarded([&] {
        const HypernetSpec s = to_spec(h);
        const auto hp = unflatten_hypernet(s, {flat, (size_t)hypernet_param_count(s)});
        RolloutBatch b = loss_batch(h, N, T, h->m, obs, nullptr, nullptr, tw, cluster);
        std::vector<double> tg(targets, targets + (size_t)N * T * h->m);
        Minibatch mb;
        mb.batch = &b;
        mb.rows.assign(rows, rows + n_rows);
        mb.value_targets = &tg;
        LossResult lr = critic_loss(s, hp, mb);
        *loss = lr.loss;
        auto g = flatten_hypernet_grad(lr.grad);
        std::copy(g.begin(), g.end(), gflat);
    });
}
int mref_adam(int64_t n, double* p, const double* g, double* m1, double* m2, int64_t* step, double lr) {
    return guarded([&] {
        AdamState st;
        st.m1.assign(m1, m1 + n);
        st.m2.assign(m2, m2 + n);
        st.step = *step;
        adam_apply(st, {p, (size_t)n}, {g, (size_t)n}, lr);
        std::copy(st.m1.begin(), st.m1.end(), m1);
        std::copy(st.m2.begin(), st.m2.end(), m2);
        *step = st.step;
    });
}

// The full reference train() (train.cpp:55-229) for built-in envs; returns
// the final flattened params. Evaluation/archive side effects are
// separate RNG lanes and do not touch the params.
int mref_train(const mo_train_cfg* c, int iterations, double* actor_out, double* critic_out) {
    return guarded([&] {
        RunConfig cfg;
        cfg.env_name = env_name(c->env_kind);
        TrainerConfig& t = cfg.trainer;
        t.N = c->N; t.K = c->K; t.kappa = c->kappa; t.T = c->T;
        t.gamma = c->gamma; t.gae_lambda = c->lambda; t.clip_eps = c->clip_eps;
        t.epochs = c->epochs; t.minibatch_count = c->minibatch_count;
        t.actor_lr = c->actor_lr; t.critic_lr = c->critic_lr; t.entropy_coef = c->entropy_coef;
        t.iterations = iterations; t.seed = c->seed;
        cfg.hypernet.F = c->F;
        cfg.hypernet.feature_hidden.assign(c->feat_hidden, c->feat_hidden + c->n_feat_hidden);
        cfg.hypernet.actor_hidden.assign(c->actor_hidden, c->actor_hidden + c->n_actor_hidden);
        cfg.hypernet.critic_hidden.assign(c->critic_hidden, c->critic_hidden + c->n_critic_hidden);
        cfg.eval.grid_resolution = 2;
        cfg.eval.episodes_per_point = 1;
        cfg.eval.log_interval = 1000000;
        TrainOptions opts;
        opts.threads = 1;
        opts.deterministic = true;
        Checkpoint ck = train(cfg, opts);
        std::copy(ck.actor_params.begin(), ck.actor_params.end(), actor_out);
        std::copy(ck.critic_params.begin(), ck.critic_params.end(), critic_out);
    });
}

// The reference train() with files and evaluation (train.cpp:55-229):
// out_dir gets metrics.csv / checkpoint.bin; archive_hv_out[it] from the
// callback; final params out.
int mref_train_run(const mo_train_cfg* c, int iterations, int grid, int episodes, int log_interval,
                   const char* out_dir, double* archive_hv_out, double* actor_out, double* critic_out) {
    return guarded([&] {
        RunConfig cfg;
        cfg.env_name = env_name(c->env_kind);
        TrainerConfig& t = cfg.trainer;
        t.N = c->N; t.K = c->K; t.kappa = c->kappa; t.T = c->T;
        t.gamma = c->gamma; t.gae_lambda = c->lambda; t.clip_eps = c->clip_eps;
        t.epochs = c->epochs; t.minibatch_count = c->minibatch_count;
        t.actor_lr = c->actor_lr; t.critic_lr = c->critic_lr; t.entropy_coef = c->entropy_coef;
        t.iterations = iterations; t.seed = c->seed;
        cfg.hypernet.F = c->F;
        cfg.hypernet.feature_hidden.assign(c->feat_hidden, c->feat_hidden + c->n_feat_hidden);
        cfg.hypernet.actor_hidden.assign(c->actor_hidden, c->actor_hidden + c->n_actor_hidden);
        cfg.hypernet.critic_hidden.assign(c->critic_hidden, c->critic_hidden + c->n_critic_hidden);
        cfg.eval.grid_resolution = grid;
        cfg.eval.episodes_per_point = episodes;
        cfg.eval.log_interval = log_interval;
        TrainOptions opts;
        opts.threads = 1;
        opts.deterministic = true;
        opts.out_dir = out_dir ? out_dir : "";
        Checkpoint ck = train(cfg, opts, [&](const IterationStats& s) {
            archive_hv_out[s.iteration] = s.archive_hypervolume;
        });
        std::copy(ck.actor_params.begin(), ck.actor_params.end(), actor_out);
        std::copy(ck.critic_params.begin(), ck.critic_params.end(), critic_out);
    });
}

// ---- Timed harness: exactly the train() loop body (train.cpp:118-184) on
// reference functions, any env including mo-humanoid6, `threads` rollout
// workers. Used by bench.py --impl reference / cpu_baseline.
struct RefTrainer {
    RunConfig cfg;
    HypernetSpec as, cs;
    HypernetParams a, c;
    AdamState af, aM, ab, cf, cM, cb;
    std::unique_ptr<BatchedEnv> env;
    EpisodeTracker tracker;
    std::vector<int> perm;
    Rng root;
    int threads = 1;
};

void* mref_trainer_create(const mo_train_cfg* c, int threads) {
    try {
        auto* t = new RefTrainer;
        HypernetArch arch;
        arch.F = c->F;
        arch.feature_hidden.assign(c->feat_hidden, c->feat_hidden + c->n_feat_hidden);
        arch.actor_hidden.assign(c->actor_hidden, c->actor_hidden + c->n_actor_hidden);
        arch.critic_hidden.assign(c->critic_hidden, c->critic_hidden + c->n_critic_hidden);
        t->env = make_any_env(c->env_kind, c->N);
        const EnvSpec es = t->env->spec();
        t->as = arch.actor_spec(es);
        t->cs = arch.critic_spec(es);
        t->root = Rng(c->seed);
        Rng ai = t->root.split(0xA1), ci = t->root.split(0xA2);
        t->a = init_hypernet(t->as, ai);
        t->c = init_hypernet(t->cs, ci);
        t->af = AdamState(t->a.feature_params.size()); t->aM = AdamState(t->a.M.size()); t->ab = AdamState(t->a.b.size());
        t->cf = AdamState(t->c.feature_params.size()); t->cM = AdamState(t->c.M.size()); t->cb = AdamState(t->c.b.size());
        t->env->reset(t->root.split(0xE0));
        t->tracker.reset(c->N, es.m);
        t->perm.resize((size_t)c->N * c->T);
        std::iota(t->perm.begin(), t->perm.end(), 0);
        TrainerConfig& tc = t->cfg.trainer;
        tc.N = c->N; tc.K = c->K; tc.kappa = c->kappa; tc.T = c->T;
        tc.gamma = c->gamma; tc.gae_lambda = c->lambda; tc.clip_eps = c->clip_eps;
        tc.epochs = c->epochs; tc.minibatch_count = c->minibatch_count;
        tc.actor_lr = c->actor_lr; tc.critic_lr = c->critic_lr; tc.entropy_coef = c->entropy_coef;
        t->threads = threads;
        return t;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void mref_trainer_destroy(void* t) { delete static_cast<RefTrainer*>(t); }

// phase timings (seconds) out: [sampling+rollout, gae+normalise, update]
int mref_trainer_iteration(void* tp, int it, int max_minibatches, int rollout_instances,
                           double* seconds_out, double* actor_loss_out, double* critic_loss_out) {
    return guarded([&] {
        RefTrainer& t = *static_cast<RefTrainer*>(tp);
        const TrainerConfig& tc = t.cfg.trainer;
        const int m = t.env->spec().m;
        const int reps = tc.N / tc.K;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto t0 = now();
        const Rng iter_rng = t.root.split(0x1000'0000ULL + (uint64_t)it);
        std::vector<TradeoffVector> clusters;
        SamplingConfig sc;
        sc.m = m; sc.K = tc.K; sc.kappa = tc.kappa; sc.N = tc.N;
        Rng sample_rng = iter_rng.split(0);
        const auto per_instance = build_tradeoff_batch(sc, sample_rng);
        for (int k = 0; k < tc.K; ++k) clusters.push_back(per_instance[(size_t)k * reps]);
        (void)rollout_instances;
        RolloutBatch batch;
        batch = collect_rollouts(t.as, t.a, t.cs, t.c, *t.env, clusters, reps, tc.T,
                                 iter_rng.split(1), t.threads, &t.tracker);
        auto t1 = now();
        const GaeResult gae = gae_per_objective(batch, tc.gamma, tc.gae_lambda);
        const std::vector<double> sadv = normalize_and_scalarize(gae.advantages, batch);
        auto t2 = now();
        Rng shuffle_rng = iter_rng.split(2);
        Minibatch mb;
        mb.batch = &batch;
        mb.scalar_advantage = &sadv;
        mb.value_targets = &gae.value_targets;
        const int rows = tc.N * tc.T;
        int done = 0;
        double al_sum = 0, cl_sum = 0, loss_s = 0, adam_s = 0;
        for (int e = 0; e < tc.epochs; ++e) {
            shuffle_rng.shuffle(t.perm);
            for (int s = 0; s < tc.minibatch_count; ++s) {
                if (max_minibatches >= 0 && done >= max_minibatches) break;
                const int lo = (int)((long long)rows * s / tc.minibatch_count);
                const int hi = (int)((long long)rows * (s + 1) / tc.minibatch_count);
                if (lo == hi) continue;
                mb.rows.assign(t.perm.begin() + lo, t.perm.begin() + hi);
                auto l0 = now();
                const LossResult al = actor_loss(t.as, t.a, mb, tc.clip_eps, tc.entropy_coef);
                const LossResult cl = critic_loss(t.cs, t.c, mb);
                auto l1 = now();
                loss_s += std::chrono::duration<double>(l1 - l0).count();
                if (!std::isfinite(al.loss) || !std::isfinite(cl.loss)) throw NumericError("non-finite loss");
                adam_apply(t.af, t.a.feature_params, al.grad.feature_params, tc.actor_lr);
                adam_apply(t.aM, t.a.M, al.grad.M, tc.actor_lr);
                adam_apply(t.ab, t.a.b, al.grad.b, tc.actor_lr);
                adam_apply(t.cf, t.c.feature_params, cl.grad.feature_params, tc.critic_lr);
                adam_apply(t.cM, t.c.M, cl.grad.M, tc.critic_lr);
                adam_apply(t.cb, t.c.b, cl.grad.b, tc.critic_lr);
                adam_s += std::chrono::duration<double>(now() - l1).count();
                al_sum += al.loss;
                cl_sum += cl.loss;
                done++;
            }
        }
        auto t3 = now();
        if (seconds_out) {
            seconds_out[0] = std::chrono::duration<double>(t1 - t0).count();
            seconds_out[1] = std::chrono::duration<double>(t2 - t1).count();
            seconds_out[2] = std::chrono::duration<double>(t3 - t2).count();
            seconds_out[3] = done;
            seconds_out[4] = loss_s;
            seconds_out[5] = adam_s;
        }
        if (actor_loss_out) *actor_loss_out = al_sum;
        if (critic_loss_out) *critic_loss_out = cl_sum;
    });
}
void mref_trainer_params(void* tp, double* actor_out, double* critic_out) {
    RefTrainer& t = *static_cast<RefTrainer*>(tp);
    auto a = flatten_hypernet(t.a), c = flatten_hypernet(t.c);
    if (actor_out) std::copy(a.begin(), a.end(), actor_out);
    if (critic_out) std::copy(c.begin(), c.end(), critic_out);
}
void mref_trainer_perm(void* tp, int32_t* out) {
    RefTrainer& t = *static_cast<RefTrainer*>(tp);
    std::copy(t.perm.begin(), t.perm.end(), out);
}

// load_checkpoint + save_checkpoint of the reference (checkpoint.cpp:200-241):
// reads `in`, returns the params and iteration, writes the same checkpoint to `out`
int mref_checkpoint_resave(const char* in, const char* out, double* actor_out, int64_t cap_a, double* critic_out,
                           int64_t cap_c, int64_t* iteration) {
    return guarded([&] {
        const Checkpoint ck = load_checkpoint(in);
        if ((int64_t)ck.actor_params.size() > cap_a || (int64_t)ck.critic_params.size() > cap_c)
            throw ShapeError("checkpoint_resave: output buffers too small");
        std::copy(ck.actor_params.begin(), ck.actor_params.end(), actor_out);
        std::copy(ck.critic_params.begin(), ck.critic_params.end(), critic_out);
        *iteration = ck.iteration;
        save_checkpoint(ck, out);
    });
}
int64_t mref_simplex_grid_size(int m, int res) { return (int64_t)simplex_grid_size(m, res); }
int mref_evaluate_params(const mo_hspec* h, const double* flat, int env_kind, int res, int episodes,
                         uint64_t key, double* w_out, double* mean_out, int64_t* n_points) {
    return guarded([&] {  // the reference registry: lqr / pointmass / dst only
        const HypernetSpec s = to_spec(h);
        const auto hp = unflatten_hypernet(s, {flat, (size_t)hypernet_param_count(s)});
        const EvalTable tab = evaluate_params(s, hp, env_name(env_kind), res, episodes, Rng::from_state(key, 0), 1);
        for (size_t g = 0; g < tab.rows.size(); ++g)
            for (int k = 0; k < tab.m; ++k) {
                w_out[g * tab.m + k] = tab.rows[g].w.weights[k];
                mean_out[g * tab.m + k] = tab.rows[g].mean_return[k];
            }
        *n_points = (int64_t)tab.rows.size();
    });
}
int mref_linear_dominance_mask(int n, int m, const double* pts, uint8_t* mask) {
    return guarded([&] {
        std::vector<ObjectiveVector> p;
        for (int i = 0; i < n; ++i) p.emplace_back(pts + (size_t)i * m, pts + (size_t)(i + 1) * m);
        auto out = linear_dominance_filter(p);
        size_t k = 0;
        for (int i = 0; i < n; ++i) {
            mask[i] = 0;
            if (k < out.size() && out[k] == p[i]) {
                mask[i] = 1;
                ++k;
            }
        }
    });
}
int mref_nondominated_mask(int n, int m, const double* pts, uint8_t* mask) {
    return guarded([&] {
        std::vector<ObjectiveVector> p;
        for (int i = 0; i < n; ++i) p.emplace_back(pts + (size_t)i * m, pts + (size_t)(i + 1) * m);
        auto out = nondominated_filter(p);
        size_t k = 0;
        for (int i = 0; i < n; ++i) {
            mask[i] = 0;
            if (k < out.size() && out[k] == p[i]) {
                mask[i] = 1;
                ++k;
            }
        }
    });
}
int mref_hypervolume_detailed(int n, int m, const double* pts, const double* ref, uint64_t samples,
                              uint64_t seed, double* value, double* se, int* exact, int* clipped) {
    return guarded([&] {
        ParetoFront f;
        for (int i = 0; i < n; ++i) f.points.emplace_back(pts + (size_t)i * m, pts + (size_t)(i + 1) * m);
        f.reference.assign(ref, ref + m);
        auto r = hypervolume_detailed(f, samples, seed);
        *value = r.value;
        if (se) *se = r.stderr_est;
        if (exact) *exact = r.exact ? 1 : 0;
        if (clipped) *clipped = r.clipped;
    });
}
int mref_hypervolume_mc(int n, int m, const double* pts, const double* ref, uint64_t samples,
                        uint64_t key, uint64_t ctr, double* value, double* se) {
    return guarded([&] {
        ParetoFront f;
        for (int i = 0; i < n; ++i) f.points.emplace_back(pts + (size_t)i * m, pts + (size_t)(i + 1) * m);
        f.reference.assign(ref, ref + m);
        *value = hypervolume_mc(f, samples, Rng::from_state(key, ctr), se);
    });
}

}  // extern "C"
