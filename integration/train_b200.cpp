// Reference-side adapter over the C-ABI (include/morlax_b200.h): maps the
// reference's configuration and callback types onto morlax_train /
// morlax_pareto_mask / morlax_evaluate_params and rethrows the library's
// status codes as the reference's exception classes (errors.hpp:10-30), so
// the CLI's exit codes (tools/commands.hpp:12-32) are unchanged.
#include "train_b200.hpp"

#include <exception>
#include <stdexcept>

#include "morlax/envs.hpp"
#include "morlax/errors.hpp"
#include "morlax/rng.hpp"
#include "morlax_b200.h"

namespace morlax {
namespace {
void check(int rc) {
    if (rc == MORLAX_OK) return;
    const std::string kind = morlax_last_error_kind(), msg = morlax_last_error();
    if (kind == "NumericError") throw NumericError(msg);
    if (kind == "ShapeError") throw ShapeError(msg);
    if (kind == "DomainError") throw DomainError(msg);
    if (kind == "ConfigError") throw ConfigError(msg);
    throw std::runtime_error(msg);
}
template <size_t N>
void fill_sizes(int* n, int (&dst)[N], const std::vector<int>& v) {
    if (v.size() > N) throw ConfigError("too many layers for the B200 path");
    *n = (int)v.size();
    for (size_t i = 0; i < v.size(); ++i) dst[i] = v[i];
}
}  // namespace

Checkpoint train_b200(const RunConfig& cfg, const TrainOptions& opts, const IterationCallback& cb) {
    cfg.validate();  // config.cpp:17-45: the same ConfigError messages as train()
    const TrainerConfig& t = cfg.trainer;
    morlax_train_config c{};
    c.env_name = cfg.env_name.c_str();
    c.N = t.N; c.K = t.K; c.kappa = t.kappa; c.T = t.T;
    c.epochs = t.epochs; c.minibatch_count = t.minibatch_count;
    c.gamma = t.gamma; c.gae_lambda = t.gae_lambda; c.clip_eps = t.clip_eps;
    c.actor_lr = t.actor_lr; c.critic_lr = t.critic_lr; c.entropy_coef = t.entropy_coef;
    c.seed = t.seed; c.F = cfg.hypernet.F;
    fill_sizes(&c.n_feature_hidden, c.feature_hidden, cfg.hypernet.feature_hidden);
    fill_sizes(&c.n_actor_hidden, c.actor_hidden, cfg.hypernet.actor_hidden);
    fill_sizes(&c.n_critic_hidden, c.critic_hidden, cfg.hypernet.critic_hidden);
    morlax_run_options o{};
    o.out_dir = opts.out_dir.empty() ? nullptr : opts.out_dir.c_str();
    o.iterations = t.iterations;
    o.grid_resolution = cfg.eval.grid_resolution;
    o.episodes_per_point = cfg.eval.episodes_per_point;
    o.log_interval = cfg.eval.log_interval;
    o.n_pareto_reference = (int)cfg.pareto_reference.size();
    o.pareto_reference = cfg.pareto_reference.empty() ? nullptr : cfg.pareto_reference.data();
    o.deterministic = opts.deterministic;
    struct Bridge {
        const IterationCallback* cb;
        std::exception_ptr err;
    } bridge{&cb, nullptr};
    auto trampoline = [](const morlax_iteration_stats* s, void* u) -> int {
        auto* b = static_cast<Bridge*>(u);
        if (!*b->cb) return 0;
        IterationStats st;
        st.iteration = s->iteration;
        st.actor_loss = s->actor_loss;
        st.critic_loss = s->critic_loss;
        st.archive_hypervolume = s->archive_hypervolume;
        st.cluster_returns.assign(s->cluster_returns, s->cluster_returns + s->n_clusters);
        try {
            (*b->cb)(st);
        } catch (...) {
            b->err = std::current_exception();
            return 1;
        }
        return 0;
    };
    morlax_trainer* tr = nullptr;
    const int rc = morlax_train(&c, &o, trampoline, &bridge, &tr);
    if (bridge.err) std::rethrow_exception(bridge.err);  // the callback's own exception
    check(rc);                                           // NumericError etc., as the reference
    int64_t na = 0, nc = 0;
    int le = 0, lc = 0, rows = 0;
    check(morlax_trainer_sizes(tr, &na, &nc, &le, &lc, &rows));
    Checkpoint ck;
    ck.config = cfg;
    ck.actor_spec = cfg.hypernet.actor_spec(env_spec(cfg.env_name));
    ck.critic_spec = cfg.hypernet.critic_spec(env_spec(cfg.env_name));
    ck.actor_params.resize(na);
    ck.critic_params.resize(nc);
    check(morlax_trainer_get_params(tr, 0, ck.actor_params.data()));  // flatten_hypernet order, fp64
    check(morlax_trainer_get_params(tr, 1, ck.critic_params.data()));
    ck.iteration = t.iterations;
    const Rng root(t.seed);
    ck.rng_key = root.key();
    ck.rng_counter = root.counter();
    morlax_trainer_destroy(tr);
    return ck;
}

std::vector<ObjectiveVector> nondominated_filter_b200(const std::vector<ObjectiveVector>& pts) {
    if (pts.empty()) return {};
    const int n = (int)pts.size(), m = (int)pts[0].size();
    std::vector<double> flat;
    flat.reserve((size_t)n * m);
    for (const auto& p : pts) {
        if ((int)p.size() != m) throw ShapeError("nondominated_filter: objective vectors differ in length");
        flat.insert(flat.end(), p.begin(), p.end());
    }
    std::vector<uint8_t> mask(n);
    check(morlax_pareto_mask(n, m, flat.data(), mask.data()));
    std::vector<ObjectiveVector> out;
    for (int i = 0; i < n; ++i)
        if (mask[i]) out.push_back(pts[i]);
    return out;
}

EvalTable evaluate_params_b200(const HypernetSpec& spec, const HypernetParams& params, const std::string& env_name,
                               int res, int episodes, const Rng& rng) {
    morlax_hypernet_spec s{};
    s.m = spec.m;
    s.F = spec.F;
    fill_sizes(&s.n_feature_hidden, s.feature_hidden, spec.feature_hidden);
    fill_sizes(&s.n_target_sizes, s.target_sizes, spec.target_spec.layer_sizes);
    s.target_tanh = spec.target_spec.output_activation == Activation::kTanh;
    s.has_log_std = spec.target_has_log_std;
    const std::vector<double> flat = flatten_hypernet(params);
    const int64_t n = spec.m == 1 ? 1 : morlax_simplex_grid_size(spec.m, res);
    std::vector<double> w((size_t)n * spec.m), r((size_t)n * spec.m);
    int64_t got = 0;
    // Rng::split is a pure function of the key (rng.hpp:35-40): the key alone
    // fixes every point's reset streams
    check(morlax_evaluate_params(&s, flat.data(), env_name.c_str(), res, episodes, rng.key(), w.data(), r.data(),
                                 &got));
    EvalTable tab;
    tab.m = spec.m;
    for (int64_t g = 0; g < got; ++g)
        tab.rows.push_back(EvalRow{TradeoffVector{{w.begin() + g * spec.m, w.begin() + (g + 1) * spec.m}},
                                   {r.begin() + g * spec.m, r.begin() + (g + 1) * spec.m}});
    return tab;
}

}  // namespace morlax
