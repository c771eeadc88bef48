// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile `adapter` into
// oracle/_ref/, run by tests/test_gpu_adapter.py): drives the reference-side
// adapter integration/train_b200.cpp -- the code a maintainer adds next to
// proj/src/train.cpp -- and the compiled reference's own entry points on the
// same inputs, and prints one JSON line for the test to check:
//   * train_b200 vs train (trainer.hpp:256-257) on a tiny config: per-
//     iteration losses, archive hypervolume and cluster returns through the
//     IterationCallback, final parameters (written raw to argv[1] prefix);
//   * the CLI exit-code contract (tools/commands.hpp:12-32) through
//     morlax::cli::guarded for a ConfigError (K does not divide N) and a
//     NumericError (a diverging learning rate), for both implementations;
//   * nondominated_filter_b200 vs nondominated_filter (pareto.hpp:24-28);
//   * evaluate_params_b200 vs evaluate_params (trainer.hpp:271-276).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "../integration/train_b200.hpp"
#include "commands.hpp"
#include "morlax/envs.hpp"
#include "morlax/hypernet.hpp"
#include "morlax/pareto.hpp"

using namespace morlax;

static RunConfig tiny() {
    RunConfig c;
    c.env_name = "mo-pointmass";
    TrainerConfig& t = c.trainer;
    t.N = 16; t.K = 2; t.kappa = 0; t.T = 12; t.epochs = 2; t.minibatch_count = 2;
    t.iterations = 3; t.seed = 5; t.entropy_coef = 0.1;
    c.hypernet.F = 16;
    c.hypernet.feature_hidden = {16};
    c.hypernet.actor_hidden = {16, 16};
    c.hypernet.critic_hidden = {16, 16};
    c.eval.grid_resolution = 3;
    c.eval.episodes_per_point = 2;
    c.eval.log_interval = 2;
    return c;
}

static void dump(const std::string& path, const std::vector<double>& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(double)));
}

static std::string arr(const std::vector<double>& v) {
    std::string s = "[";
    char b[64];
    for (size_t i = 0; i < v.size(); ++i) {
        std::snprintf(b, sizeof b, "%s%.17g", i ? "," : "", std::isnan(v[i]) ? -1e300 : v[i]);
        s += b;
    }
    return s + "]";
}

int main(int argc, char** argv) {
    const std::string prefix = argc > 1 ? argv[1] : "adapter";
    // ---- train_b200 vs train
    const RunConfig cfg = tiny();
    TrainOptions opts;
    opts.deterministic = true;
    std::vector<double> la_b, lc_b, hv_b, la_r, lc_r, hv_r, ret_b, ret_r;
    const Checkpoint ck_b = train_b200(cfg, opts, [&](const IterationStats& s) {
        la_b.push_back(s.actor_loss);
        lc_b.push_back(s.critic_loss);
        hv_b.push_back(s.archive_hypervolume);
        ret_b.insert(ret_b.end(), s.cluster_returns.begin(), s.cluster_returns.end());
    });
    const Checkpoint ck_r = train(cfg, opts, [&](const IterationStats& s) {
        la_r.push_back(s.actor_loss);
        lc_r.push_back(s.critic_loss);
        hv_r.push_back(s.archive_hypervolume);
        ret_r.insert(ret_r.end(), s.cluster_returns.begin(), s.cluster_returns.end());
    });
    dump(prefix + "_actor_b200.bin", ck_b.actor_params);
    dump(prefix + "_critic_b200.bin", ck_b.critic_params);
    dump(prefix + "_actor_ref.bin", ck_r.actor_params);
    dump(prefix + "_critic_ref.bin", ck_r.critic_params);
    // ---- exit codes through the CLI's guarded()
    RunConfig bad = tiny();
    bad.trainer.N = 15;  // K does not divide N: ConfigError -> 2
    const int cfg_b = cli::guarded([&] { train_b200(bad, opts); return 0; });
    const int cfg_r = cli::guarded([&] { train(bad, opts); return 0; });
    RunConfig blow = tiny();
    blow.trainer.actor_lr = 1e300;  // one Adam step moves every weight by ~1e300: the next losses overflow
    blow.trainer.critic_lr = 1e300; // in fp64 as in fp32 -> NumericError -> 3
    const int num_b = cli::guarded([&] { train_b200(blow, opts); return 0; });
    const int num_r = cli::guarded([&] { train(blow, opts); return 0; });
    // ---- nondominated_filter
    std::vector<ObjectiveVector> pts;
    Rng rng(17);
    for (int i = 0; i < 400; ++i) {
        ObjectiveVector p(3);
        for (double& x : p) x = std::round(rng.next_double() * 20.0) / 10.0;  // ties and duplicates
        pts.push_back(p);
    }
    const bool nd_equal = nondominated_filter_b200(pts) == nondominated_filter(pts);
    // ---- evaluate_params on the reference-trained actor
    const HypernetSpec as = cfg.hypernet.actor_spec(env_spec(cfg.env_name));
    const HypernetParams hp = unflatten_hypernet(as, ck_r.actor_params);
    const Rng erng(0x1234);
    const EvalTable eb = evaluate_params_b200(as, hp, cfg.env_name, 4, 3, erng);
    const EvalTable er = evaluate_params(as, hp, cfg.env_name, 4, 3, erng, 1);
    double emax = 0.0, escale = 0.0;
    bool ew = eb.rows.size() == er.rows.size();
    for (size_t g = 0; ew && g < eb.rows.size(); ++g) {
        ew = ew && eb.rows[g].w.weights == er.rows[g].w.weights;
        for (size_t k = 0; k < er.rows[g].mean_return.size(); ++k) {
            emax = std::fmax(emax, std::fabs(eb.rows[g].mean_return[k] - er.rows[g].mean_return[k]));
            escale = std::fmax(escale, std::fabs(er.rows[g].mean_return[k]));
        }
    }
    std::printf(
        "{\"actor_loss_b200\": %s, \"actor_loss_ref\": %s, \"critic_loss_b200\": %s, \"critic_loss_ref\": %s, "
        "\"hv_b200\": %s, \"hv_ref\": %s, \"returns_b200\": %s, \"returns_ref\": %s, \"iteration_b200\": %lld, "
        "\"iteration_ref\": %lld, \"n_actor\": %zu, \"n_critic\": %zu, \"config_exit_b200\": %d, "
        "\"config_exit_ref\": %d, \"numeric_exit_b200\": %d, \"numeric_exit_ref\": %d, \"nondominated_equal\": %s, "
        "\"eval_grid_equal\": %s, \"eval_max_abs\": %.17g, \"eval_scale\": %.17g}\n",
        arr(la_b).c_str(), arr(la_r).c_str(), arr(lc_b).c_str(), arr(lc_r).c_str(), arr(hv_b).c_str(),
        arr(hv_r).c_str(), arr(ret_b).c_str(), arr(ret_r).c_str(), (long long)ck_b.iteration,
        (long long)ck_r.iteration, ck_b.actor_params.size(), ck_b.critic_params.size(), cfg_b, cfg_r, num_b, num_r,
        nd_equal ? "true" : "false", ew ? "true" : "false", emax, escale);
    return 0;
}
