// extern "C" boundary (include/morlax_b200.h). Every entry point maps the
// reference's C++ exceptions to the CLI's status codes
// (tools/commands.hpp:12-32) and records a thread-local message.
#include <cmath>
#include <cstdio>
#include <functional>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "../../include/morlax_b200.h"
#include "comm.h"
#include "policy.h"
#include "trainer.h"

using namespace mb200;

namespace {
thread_local std::string g_err, g_kind;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        g_kind.clear();
        return MORLAX_OK;
    } catch (const NumericError& e) {
        g_err = e.what(); g_kind = "NumericError";
        return MORLAX_ERR_NUMERIC;
    } catch (const ConfigError& e) {
        g_err = e.what(); g_kind = "ConfigError";
        return MORLAX_ERR_CONFIG;
    } catch (const ShapeError& e) {
        g_err = e.what(); g_kind = "ShapeError";
        return MORLAX_ERR_CONFIG;
    } catch (const DomainError& e) {
        g_err = e.what(); g_kind = "DomainError";
        return MORLAX_ERR_CONFIG;
    } catch (const CudaError& e) {
        g_err = e.what(); g_kind = "CudaError";
        return MORLAX_ERR_OTHER;
    } catch (const std::exception& e) {
        g_err = e.what(); g_kind = "Error";
        return MORLAX_ERR_OTHER;
    }
}

template <typename T>
struct DBuf {  // scoped device buffer
    T* p = nullptr;
    size_t n = 0;
    explicit DBuf(size_t n_) : n(n_) { MB_CUDA(cudaMalloc(&p, (n ? n : 1) * sizeof(T))); }
    DBuf(const T* host, size_t n_) : DBuf(n_) {
        if (n) {
            MB_CUDA(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
            MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
        }
    }
    ~DBuf() { cudaFree(p); }
    void get(T* host) const {
        if (n) MB_CUDA(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
};

std::vector<int> vec(int n, const int* a) { return std::vector<int>(a, a + n); }

void check_simplex(int m, const double* w) {  // TradeoffVector::checked (simplex.cpp:18-30)
    double s = 0.0;
    for (int i = 0; i < m; ++i) {
        if (!(w[i] >= 0.0)) throw DomainError("trade-off entries must be nonnegative");
        s += w[i];
    }
    if (std::fabs(s - 1.0) > 1e-9) throw DomainError("trade-off entries must sum to 1 (got " + std::to_string(s) + ")");
}

struct HyperHandle {
    HyperNet h;
    explicit HyperHandle(const morlax_hypernet_spec* s, int G) {
        if (s->n_target_sizes < 2 || s->n_target_sizes > 9) throw ShapeError("MlpSpec needs at least input and output sizes");
        h.init(s->m, s->F, vec(s->n_feature_hidden, s->feature_hidden), vec(s->n_target_sizes, s->target_sizes),
               s->target_tanh != 0, s->has_log_std != 0, G);
    }
    ~HyperHandle() { h.free_all(); }
    void load(const double* flat) {
        std::vector<float> f(flat, flat + h.n);
        MB_CUDA(cudaMemcpy(h.p, f.data(), sizeof(float) * h.n, cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
        h.refresh_images(0);
    }
};
}  // namespace

struct morlax_env {
    EnvSpecB es;
    int N;
    float* state = nullptr;
    uint64_t *keys = nullptr, *ctrs = nullptr;
    int* steps = nullptr;
    int* err = nullptr;
    unsigned long long* clamps = nullptr;
    cudaStream_t s = nullptr;
};

struct morlax_trainer {
    Trainer* t = nullptr;
};

struct morlax_policy {
    GroupPolicy* p = nullptr;
    int m = 0;
};

namespace mb200 {
// ---- checkpoint wire format (checkpoint.cpp:15-241): "MRLXCKPT", u32 v1,
// RunConfig, actor / critic HypernetSpec, fp64 params (flatten_hypernet
// order), i64 iteration, root Rng key / counter; little-endian fixed width
namespace {
const char* env_name_of(int kind) {
    switch (kind) {
        case ENV_LQR: return "mo-lqr1d";
        case ENV_LQR_M1: return "mo-lqr1d-m1";
        case ENV_POINTMASS: return "mo-pointmass";
        case ENV_DST: return "mo-dst-continuous";
    }
    return "mo-humanoid6";
}
struct CkWriter {
    std::string buf;
    void raw(const void* p, size_t n) { buf.append(static_cast<const char*>(p), n); }
    template <typename T>
    void put(T v) { raw(&v, sizeof(T)); }
    void str(const std::string& s) { put<uint64_t>(s.size()); raw(s.data(), s.size()); }
    void vec_i32(const std::vector<int>& v) { put<uint64_t>(v.size()); for (int x : v) put<int32_t>(x); }
    void vec_f64(const std::vector<double>& v) { put<uint64_t>(v.size()); raw(v.data(), v.size() * 8); }
};
struct CkReader {
    const std::string& b;
    size_t o = 0;
    std::string path;
    void raw(void* p, size_t n) {
        if (o + n > b.size()) throw ConfigError("checkpoint truncated: " + path);
        std::memcpy(p, b.data() + o, n);
        o += n;
    }
    template <typename T>
    T get() { T v; raw(&v, sizeof(T)); return v; }
    uint64_t len(uint64_t cap) {
        const uint64_t n = get<uint64_t>();
        if (n > cap) throw ConfigError("checkpoint corrupt (oversized field): " + path);
        return n;
    }
    std::string str() { const uint64_t n = len(1u << 20); std::string s(n, '\0'); raw(&s[0], n); return s; }
    std::vector<int> vec_i32() { const uint64_t n = len(1u << 20); std::vector<int> v(n); for (auto& x : v) x = get<int32_t>(); return v; }
    std::vector<double> vec_f64() { const uint64_t n = len(1u << 28); std::vector<double> v(n); raw(v.data(), n * 8); return v; }
};
void write_spec(CkWriter& w, const HyperNet& h, const std::vector<int>& fh) {  // write_hypernet_spec
    w.put<int32_t>(h.m);
    w.put<int32_t>(h.F);
    w.vec_i32(fh);
    w.vec_i32(std::vector<int>(h.tgt.sz, h.tgt.sz + h.tgt.L + 1));
    w.put<uint8_t>(h.tgt.out_tanh ? 1 : 0);
    w.put<uint8_t>(h.tgt.has_log_std ? 1 : 0);
}
std::vector<double> params_f64(const HyperNet& h, const float* dev, cudaStream_t s) {
    std::vector<float> f(h.n);
    MB_CUDA(cudaStreamSynchronize(s));
    MB_CUDA(cudaMemcpy(f.data(), dev, sizeof(float) * h.n, cudaMemcpyDeviceToHost));
    return std::vector<double>(f.begin(), f.end());
}
// save_checkpoint (checkpoint.cpp:200-213) of the trainer's config with the
// params read from the device buffers actor_dev / critic_dev (the live
// params, or train()'s last-healthy snapshot)
void write_checkpoint(Trainer& tr, const char* path, int64_t iteration, const morlax_checkpoint_extra* x,
                      const float* actor_dev, const float* critic_dev) {
    const TrainConfig& c = tr.config();
    const morlax_checkpoint_extra def{300, 10, 8, 10, 0, nullptr};  // trainer.hpp:39, 59-62 defaults
    const morlax_checkpoint_extra& e = x ? *x : def;
    CkWriter w;
    w.raw("MRLXCKPT", 8);
    w.put<uint32_t>(1);
    w.str(env_name_of(c.env_kind));  // write_run_config (checkpoint.cpp:137-163)
    w.put<int32_t>(c.N); w.put<int32_t>(c.K); w.put<int32_t>(c.kappa); w.put<int32_t>(c.T);
    w.put<double>(c.gamma); w.put<double>(c.lambda); w.put<double>(c.clip_eps);
    w.put<int32_t>(c.epochs); w.put<int32_t>(c.minibatch_count);
    w.put<double>(c.actor_lr); w.put<double>(c.critic_lr); w.put<double>(c.entropy_coef);
    w.put<int32_t>(e.iterations);
    w.put<uint64_t>(c.seed);
    w.put<int32_t>(c.F);
    w.vec_i32(c.feat_hidden); w.vec_i32(c.actor_hidden); w.vec_i32(c.critic_hidden);
    w.put<int32_t>(e.grid_resolution); w.put<int32_t>(e.episodes_per_point); w.put<int32_t>(e.log_interval);
    w.vec_f64(std::vector<double>(e.pareto_reference, e.pareto_reference + (e.pareto_reference ? e.n_pareto_reference : 0)));
    write_spec(w, tr.actor(), c.feat_hidden);
    write_spec(w, tr.critic(), c.feat_hidden);
    w.vec_f64(params_f64(tr.actor(), actor_dev, tr.stream()));
    w.vec_f64(params_f64(tr.critic(), critic_dev, tr.stream()));
    w.put<int64_t>(iteration);
    w.put<uint64_t>(seed_key(c.seed));  // the root Rng(seed) is only ever split: counter 0
    w.put<uint64_t>(0);
    FILE* f = std::fopen(path, "wb");
    if (!f) throw ConfigError(std::string("cannot open checkpoint for writing: ") + path);
    const size_t n = std::fwrite(w.buf.data(), 1, w.buf.size(), f);
    if (std::fclose(f) != 0 || n != w.buf.size()) throw ConfigError(std::string("failed writing checkpoint: ") + path);
}
}  // namespace
}  // namespace mb200

extern "C" {

const char* morlax_last_error(void) { return g_err.c_str(); }
const char* morlax_last_error_kind(void) { return g_kind.c_str(); }
int morlax_version(void) { return 1; }
int morlax_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int morlax_rng_words(uint64_t key, uint64_t ctr, int64_t n, uint64_t* out) {
    return guarded([&] {
        DBuf<uint64_t> d(n);
        rng_words(key, ctr, n, d.p, 0);
        d.get(out);
    });
}
int morlax_rng_gaussians(uint64_t key, uint64_t ctr, int64_t n, double* out) {
    return guarded([&] {
        DBuf<double> d(n);
        rng_gaussians(key, ctr, n, d.p, 0);
        d.get(out);
    });
}

// ------------------------------------------------------------------ env
int morlax_env_spec(const char* name, int* od, int* ad, int* m, int* ms) {
    return guarded([&] {
        const EnvSpecB es = env_spec_of(env_kind_of(name));
        if (od) *od = es.obs_dim;
        if (ad) *ad = es.act_dim;
        if (m) *m = es.m;
        if (ms) *ms = es.max_steps;
    });
}
int morlax_env_create(const char* name, int n, morlax_env** out) {
    return guarded([&] {
        if (n < 1) throw ShapeError("BatchedEnv: num_envs must be >= 1");
        auto* e = new morlax_env;
        e->es = env_spec_of(env_kind_of(name));
        e->N = n;
        MB_CUDA(cudaMalloc(&e->state, sizeof(float) * e->es.state_dim * n));
        MB_CUDA(cudaMalloc(&e->keys, sizeof(uint64_t) * n));
        MB_CUDA(cudaMalloc(&e->ctrs, sizeof(uint64_t) * n));
        MB_CUDA(cudaMalloc(&e->steps, sizeof(int) * n));
        MB_CUDA(cudaMalloc(&e->err, sizeof(int)));
        MB_CUDA(cudaMalloc(&e->clamps, sizeof(unsigned long long)));
        MB_CUDA(cudaMemset(e->state, 0, sizeof(float) * e->es.state_dim * n));
        MB_CUDA(cudaMemset(e->steps, 0, sizeof(int) * n));
        MB_CUDA(cudaMemset(e->err, 0, sizeof(int)));
        MB_CUDA(cudaMemset(e->clamps, 0, sizeof(unsigned long long)));
        MB_CUDA(cudaStreamSynchronize(0));  // the legacy-stream fills, before e->s (non-blocking) uses them
        MB_CUDA(cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking));
        *out = e;
    });
}
void morlax_env_destroy(morlax_env* e) {
    if (!e) return;
    cudaFree(e->state); cudaFree(e->keys); cudaFree(e->ctrs); cudaFree(e->steps); cudaFree(e->err);
    cudaFree(e->clamps);
    cudaStreamDestroy(e->s);
    delete e;
}
int morlax_env_reset(morlax_env* e, uint64_t key, uint64_t ctr, float* obs_out) {
    return guarded([&] {
        (void)ctr;  // split() ignores the parent counter (rng.hpp:35-40)
        env_reset(e->es.kind, e->N, e->state, e->keys, e->ctrs, e->steps, key, 0, e->s);
        if (obs_out) {
            DBuf<float> o((size_t)e->N * e->es.obs_dim);
            env_obs(e->es.kind, e->N, e->state, o.p, e->s);
            MB_CUDA(cudaStreamSynchronize(e->s));
            o.get(obs_out);
        }
        MB_CUDA(cudaStreamSynchronize(e->s));
    });
}
int morlax_env_step_device(morlax_env* e, const float* a, float* obs, float* rew, uint8_t* term, uint8_t* trunc,
                           void* stream) {
    return guarded([&] {
        env_step(e->es.kind, e->N, e->state, e->keys, e->ctrs, e->steps, a, obs, rew, term, trunc, e->clamps, e->err,
                 (cudaStream_t)stream);
    });
}
int morlax_env_step(morlax_env* e, const float* actions, float* obs, float* reward, uint8_t* term,
                    uint8_t* trunc) {
    return guarded([&] {
        const EnvSpecB& es = e->es;
        const size_t N = e->N;
        for (size_t i = 0; i < N * es.act_dim; ++i)  // env.cpp:66-68 (checked before any state change)
            if (!std::isfinite(actions[i]))
                throw NumericError("non-finite action for environment instance " + std::to_string(i / es.act_dim));
        DBuf<float> da(actions, N * es.act_dim), dobs(N * es.obs_dim), drew(N * es.m);
        DBuf<uint8_t> dt(N), dr(N);
        env_step(es.kind, e->N, e->state, e->keys, e->ctrs, e->steps, da.p, dobs.p, drew.p, dt.p, dr.p, e->clamps,
                 e->err, e->s);
        MB_CUDA(cudaStreamSynchronize(e->s));
        dobs.get(obs);
        drew.get(reward);
        dt.get(term);
        dr.get(trunc);
    });
}
int morlax_env_current_obs(morlax_env* e, float* out) {
    return guarded([&] {
        DBuf<float> o((size_t)e->N * e->es.obs_dim);
        env_obs(e->es.kind, e->N, e->state, o.p, e->s);
        MB_CUDA(cudaStreamSynchronize(e->s));
        o.get(out);
    });
}
uint64_t morlax_env_clamp_count(morlax_env* e) {
    unsigned long long c = 0;
    cudaStreamSynchronize(e->s);  // the env kernels run on e->s (non-blocking)
    cudaMemcpy(&c, e->clamps, sizeof(c), cudaMemcpyDeviceToHost);
    return c;
}

// ------------------------------------------------------------------ hypernet
int64_t morlax_hypernet_target_count(const morlax_hypernet_spec* s) {
    NetDims d = make_dims(vec(s->n_target_sizes, s->target_sizes), s->target_tanh, s->has_log_std);
    return d.P;
}
int64_t morlax_hypernet_param_count(const morlax_hypernet_spec* s) {
    std::vector<int> fs{s->m};
    for (int i = 0; i < s->n_feature_hidden; ++i) fs.push_back(s->feature_hidden[i]);
    fs.push_back(s->F);
    long nf = 0;
    for (size_t l = 0; l + 1 < fs.size(); ++l) nf += (long)(fs[l] + 1) * fs[l + 1];
    const long P = morlax_hypernet_target_count(s);
    return nf + P * s->F + P;
}
int morlax_init_hypernet(const morlax_hypernet_spec* s, uint64_t key, uint64_t ctr, double* out) {
    return guarded([&] {
        (void)ctr;
        HyperHandle hh(s, 1);
        hh.h.init_params(key, 0);
        std::vector<float> f(hh.h.n);
        MB_CUDA(cudaMemcpy(f.data(), hh.h.p, sizeof(float) * hh.h.n, cudaMemcpyDeviceToHost));
        for (long i = 0; i < hh.h.n; ++i) out[i] = f[i];
    });
}
int morlax_hypernet_forward(const morlax_hypernet_spec* s, const double* flat, const double* w, int G,
                            double* theta) {
    return guarded([&] {
        for (int g = 0; g < G; ++g) check_simplex(s->m, w + (size_t)g * s->m);
        HyperHandle hh(s, G);
        hh.load(flat);
        std::vector<float> wf(w, w + (size_t)G * s->m);
        DBuf<float> dw(wf.data(), wf.size());
        hh.h.forward(dw.p, 0, G, 0);
        std::vector<float> th((size_t)G * hh.h.P);
        MB_CUDA(cudaMemcpy2D(th.data(), sizeof(float) * hh.h.P, hh.h.theta, sizeof(float) * hh.h.ld,
                             sizeof(float) * hh.h.P, G, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < th.size(); ++i) {
            if (!std::isfinite(th[i]))
                throw NumericError("hypernet_forward produced a non-finite parameter at index " +
                                   std::to_string(i % hh.h.P));
            theta[i] = th[i];
        }
    });
}
int morlax_policy_create(const morlax_hypernet_spec* s, int groups, int rows_per_group, morlax_policy** out) {
    return guarded([&] {
        if (s->n_target_sizes < 2 || s->n_target_sizes > 9) throw ShapeError("MlpSpec needs at least input and output sizes");
        auto* h = new morlax_policy;
        try {
            h->p = new GroupPolicy(s->m, s->F, vec(s->n_feature_hidden, s->feature_hidden),
                                   vec(s->n_target_sizes, s->target_sizes), s->target_tanh != 0, s->has_log_std != 0,
                                   groups, rows_per_group);
        } catch (...) {
            delete h;
            throw;
        }
        h->m = s->m;
        *out = h;
    });
}
void morlax_policy_destroy(morlax_policy* h) {
    if (!h) return;
    delete h->p;
    delete h;
}
int morlax_policy_set_params(morlax_policy* h, const double* flat) {
    return guarded([&] {
        HyperNet& hn = h->p->h;
        std::vector<float> f(flat, flat + hn.n);
        MB_CUDA(cudaMemcpy(hn.p, f.data(), sizeof(float) * hn.n, cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
        hn.refresh_images(0);
        MB_CUDA(cudaDeviceSynchronize());
    });
}
int morlax_policy_forward(morlax_policy* h, const double* w, const float* obs, float* pre) {
    return guarded([&] {
        GroupPolicy& gp = *h->p;
        for (int g = 0; g < gp.G; ++g) check_simplex(h->m, w + (size_t)g * h->m);
        const int od = gp.h.tgt.sz[0], out = gp.h.tgt.sz[gp.h.tgt.L];
        std::vector<float> wf(w, w + (size_t)gp.G * h->m);
        DBuf<float> dw(wf.data(), wf.size()), dobs(obs, (size_t)gp.G * gp.R * od), dpre((size_t)gp.G * gp.R * out);
        gp.forward(dw.p, dobs.p, dpre.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        dpre.get(pre);
    });
}
int morlax_policy_forward_device(morlax_policy* h, const float* d_w, const float* d_obs, float* d_pre,
                                 void* stream) {
    return guarded([&] { h->p->forward(d_w, d_obs, d_pre, (cudaStream_t)stream); });
}
double morlax_policy_flops(morlax_policy* h) { return h ? h->p->flops() : 0.0; }
int64_t morlax_simplex_grid_size(int m, int res) {  // simplex.cpp:119-130
    if (m < 1 || res < 1) return 0;
    int64_t r = 1;
    for (int i = 1; i <= m - 1; ++i) r = r * (res + i) / i;
    return r;
}
int morlax_evaluate_params(const morlax_hypernet_spec* s, const double* flat, const char* env_name,
                           int grid_resolution, int episodes, uint64_t key, double* w_out, double* mean_out,
                           int64_t* n_points) {
    return guarded([&] {  // evaluate.cpp:68-101
        if (episodes < 1) throw ConfigError("evaluate: episodes_per_point must be >= 1");
        const EnvSpecB es = env_spec_of(env_kind_of(env_name));
        if (s->m != es.m) throw ShapeError("evaluate: hypernet trade-off dim does not match env");
        if (s->n_target_sizes < 2 || s->target_sizes[0] != es.obs_dim ||
            s->target_sizes[s->n_target_sizes - 1] != es.act_dim)
            throw ShapeError("evaluate: policy spec does not match the environment");
        // simplex_grid (simplex.cpp:88-117): compositions of res into m parts,
        // first coordinate from res down to 0
        std::vector<double> W;
        if (es.m == 1) {
            W.push_back(1.0);
        } else {
            if (grid_resolution < 1) throw ConfigError("evaluate: grid_resolution must be >= 1");
            std::vector<int> k(es.m, 0);
            std::function<void(int, int)> rec = [&](int depth, int rem) {
                if (depth == es.m - 1) {
                    k[depth] = rem;
                    for (int j = 0; j < es.m; ++j) W.push_back((double)k[j] / grid_resolution);
                    return;
                }
                for (int v = rem; v >= 0; --v) {
                    k[depth] = v;
                    rec(depth + 1, rem - v);
                }
            };
            rec(0, grid_resolution);
        }
        const int ng = (int)(W.size() / es.m);
        HyperHandle hh(s, ng);
        hh.load(flat);
        std::vector<float> wf(W.begin(), W.end());
        DBuf<float> dw(wf.data(), wf.size());
        hh.h.forward(dw.p, 0, ng, 0);  // theta for every grid point (hypernet.cpp:69-90)
        const int cpp = (episodes + 15) / 16;
        DBuf<double> part((size_t)ng * cpp * es.m), mean((size_t)ng * es.m);
        DBuf<int> err(1);
        MB_CUDA(cudaMemset(err.p, 0, sizeof(int)));
        EvalArgs a;
        a.kind = es.kind; a.od = es.obs_dim; a.ad = es.act_dim; a.m = es.m; a.sdim = es.state_dim;
        a.max_steps = es.max_steps; a.episodes = episodes; a.pol = hh.h.tgt;
        a.theta = hh.h.theta; a.ld = hh.h.ld; a.key = key; a.part = part.p; a.err = err.p;
        evaluate(a, ng, mean.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        int e = 0;
        err.get(&e);
        if (e) throw NumericError("evaluate: non-finite action");
        std::copy(W.begin(), W.end(), w_out);
        mean.get(mean_out);
        *n_points = ng;
    });
}
int morlax_hypernet_backward(const morlax_hypernet_spec* s, const double* flat, const double* w, int G,
                             const double* gtheta, double* out) {
    return guarded([&] {
        for (int g = 0; g < G; ++g) check_simplex(s->m, w + (size_t)g * s->m);
        HyperHandle hh(s, G);
        hh.load(flat);
        std::vector<float> wf(w, w + (size_t)G * s->m);
        DBuf<float> dw(wf.data(), wf.size());
        hh.h.forward(dw.p, 0, G, 0);
        std::vector<float> gt(gtheta, gtheta + (size_t)G * hh.h.P);
        MB_CUDA(cudaMemcpy2D(hh.h.gtheta, sizeof(float) * hh.h.ld, gt.data(), sizeof(float) * hh.h.P,
                             sizeof(float) * hh.h.P, G, cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
        hh.h.backward(0);
        std::vector<float> g(hh.h.n);
        MB_CUDA(cudaMemcpy(g.data(), hh.h.g, sizeof(float) * g.size(), cudaMemcpyDeviceToHost));
        for (long i = 0; i < hh.h.n; ++i) out[i] = g[i];
    });
}

// ------------------------------------------------------------------ GAE / Adam
int morlax_gae(int N, int T, int m, const float* rew, const float* val, const float* nval, const uint8_t* term,
               const uint8_t* trunc, double gamma, double lambda, float* adv, float* tgt) {
    return guarded([&] {
        if (N <= 0 || T <= 0 || m <= 0) throw ShapeError("gae: batch dimensions must be positive");
        if (!(gamma >= 0.0 && gamma <= 1.0)) throw DomainError("gae: gamma must lie in [0, 1], got " + std::to_string(gamma));
        if (!(lambda >= 0.0 && lambda <= 1.0)) throw DomainError("gae: lambda must lie in [0, 1], got " + std::to_string(lambda));
        const size_t R = (size_t)N * T;
        DBuf<float> r(rew, R * m), v(val, R * m), nv(nval, R * m), a(R * m), tg(R * m);
        DBuf<uint8_t> te(term, R), tr(trunc, R);
        gae_scan(N, T, m, r.p, v.p, nv.p, te.p, tr.p, (float)gamma, (float)lambda, a.p, tg.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        a.get(adv);
        tg.get(tgt);
    });
}
int morlax_normalize_scalarize(int N, int T, int m, const float* adv, const double* tw, float* out) {
    return guarded([&] {
        const size_t R = (size_t)N * T;
        DBuf<float> a(adv, R * m), o(R);
        std::vector<float> twf(tw, tw + (size_t)N * m);
        DBuf<float> w(twf.data(), twf.size());
        DBuf<double> st(32), part((size_t)N * 8);  // partials per instance (T rows each)
        channel_partials(a.p, N, T, m, nullptr, part.p, 0);
        channel_total(part.p, N, m, st.p, 0);
        stats_finalize(st.p, (double)R, m, st.p + 8, 0, 0);
        channel_partials(a.p, N, T, m, st.p + 8, part.p, 0);
        channel_total(part.p, N, m, st.p + 16, 0);
        stats_finalize(st.p + 16, (double)R, m, st.p + 24, 1, 0);
        scalarize(N, T, m, a.p, w.p, 1, st.p + 8, st.p + 24, o.p, 0);  // reps = 1: per-instance weights
        MB_CUDA(cudaDeviceSynchronize());
        o.get(out);
    });
}
int morlax_adam(int64_t n, double* p, const double* g, double* m1, double* m2, int64_t* step, double lr) {
    return guarded([&] {
        std::vector<float> pf(p, p + n), gf(g, g + n), af(m1, m1 + n), bf(m2, m2 + n);
        DBuf<float> dp(pf.data(), n), dg(gf.data(), n), da(af.data(), n), db(bf.data(), n);
        DBuf<int> err(1);
        MB_CUDA(cudaMemset(err.p, 0, sizeof(int)));
        *step += 1;
        const double bc1 = 1.0 - std::pow(0.9, (double)*step), bc2 = 1.0 - std::pow(0.999, (double)*step);
        adam(n, dp.p, dg.p, da.p, db.p, (float)lr, (float)bc1, (float)bc2, err.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        dp.get(pf.data());
        da.get(af.data());
        db.get(bf.data());
        for (int64_t i = 0; i < n; ++i) {
            p[i] = pf[i];
            m1[i] = af[i];
            m2[i] = bf[i];
        }
    });
}

// ------------------------------------------------------------------ trainer
int morlax_nccl_unique_id(void* out) {
    return guarded([&] { comm_unique_id(out); });
}
struct morlax_loopback {
    LoopGroup* g = nullptr;
};
int morlax_loopback_create(int world, morlax_loopback** out) {
    return guarded([&] {
        auto* h = new morlax_loopback;
        h->g = loop_group_create(world);
        *out = h;
    });
}
void morlax_loopback_destroy(morlax_loopback* g) {
    if (!g) return;
    loop_group_destroy(g->g);
    delete g;
}
static int trainer_create(const morlax_train_config* c, int world, int rank, const void* id, LoopGroup* loop,
                          morlax_trainer** out);
int morlax_trainer_create(const morlax_train_config* c, int world, int rank, const void* id, morlax_trainer** out) {
    return trainer_create(c, world, rank, id, nullptr, out);
}
int morlax_trainer_create_loopback(const morlax_train_config* c, morlax_loopback* g, int rank, morlax_trainer** out) {
    if (!g) return guarded([] { throw ConfigError("loopback group is null"); });
    return trainer_create(c, comm_world_of(g->g), rank, nullptr, g->g, out);
}
static int trainer_create(const morlax_train_config* c, int world, int rank, const void* id, LoopGroup* loop,
                          morlax_trainer** out) {
    return guarded([&] {
        TrainConfig tc;
        tc.env_kind = env_kind_of(c->env_name ? c->env_name : "");
        tc.N = c->N; tc.K = c->K; tc.kappa = c->kappa; tc.T = c->T;
        tc.epochs = c->epochs; tc.minibatch_count = c->minibatch_count;
        tc.gamma = c->gamma; tc.lambda = c->gae_lambda; tc.clip_eps = c->clip_eps;
        tc.actor_lr = c->actor_lr; tc.critic_lr = c->critic_lr; tc.entropy_coef = c->entropy_coef;
        tc.seed = c->seed; tc.F = c->F;
        tc.feat_hidden = vec(c->n_feature_hidden, c->feature_hidden);
        tc.actor_hidden = vec(c->n_actor_hidden, c->actor_hidden);
        tc.critic_hidden = vec(c->n_critic_hidden, c->critic_hidden);
        auto* h = new morlax_trainer;
        try {
            h->t = new Trainer(tc, world, rank, id, loop);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
void morlax_trainer_destroy(morlax_trainer* t) {
    if (!t) return;
    delete t->t;
    delete t;
}
static void fill_stats(morlax_trainer* t, const IterStats& st, morlax_iter_stats* out) {
    if (!out) return;
    out->actor_loss = st.actor_loss;
    out->critic_loss = st.critic_loss;
    out->minibatches = st.minibatches;
    out->numeric_error = st.numeric_error;
    out->kernel_launches = t->t->kernel_launches();
}
int morlax_trainer_iteration(morlax_trainer* t, int it, morlax_iter_stats* stats) {
    IterStats st;
    const int rc = guarded([&] { t->t->iteration(it, &st); });
    fill_stats(t, st, stats);
    return rc;
}
int morlax_trainer_phase(morlax_trainer* t, int it, int phase, int max_mb, morlax_iter_stats* stats) {
    IterStats st;
    const int rc = guarded([&] {
        switch (phase) {
            case 1: t->t->phase_rollout(it); break;
            case 2: t->t->phase_advantages(); break;
            case 3: t->t->phase_update(it, max_mb); break;
            case 4: t->t->finish(&st); break;
            case 5: t->t->phase_plans(it); break;
            default: throw ConfigError("unknown phase");
        }
    });
    if (phase == 4) fill_stats(t, st, stats);
    return rc;
}
int morlax_trainer_sizes(morlax_trainer* t, int64_t* ap, int64_t* cp, int* le, int* lc, int* rows) {
    return guarded([&] {
        Trainer& tr = *t->t;
        if (ap) *ap = tr.actor().n;
        if (cp) *cp = tr.critic().n;
        if (le) *le = tr.local_envs();
        if (lc) *lc = tr.local_groups();
        if (rows) *rows = tr.local_envs() * tr.config().T;
    });
}

int morlax_trainer_save_checkpoint(morlax_trainer* t, const char* path, int64_t iteration,
                                   const morlax_checkpoint_extra* x) {
    return guarded([&] {
        Trainer& tr = *t->t;
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
        tr.actor().gather_params(tr.stream());  // sharded optimizer: every rank's M rows (collective)
        tr.critic().gather_params(tr.stream());
        write_checkpoint(tr, path, iteration, x, tr.actor().p, tr.critic().p);
    });
}

// train() (train.cpp:55-229) over the device trainer: per iteration the
// device loop body (sampling, rollout, GAE, PPO update), every log_interval
// (and the last iteration) evaluate_params of the actor -> archive ->
// nondominated_filter -> hypervolume (exact m <= 4, else MC 1e6 / seed
// 0x9E3779B9), one metrics.csv row ("%.17g", wall_ms 0 when deterministic),
// the callback, and a last-healthy snapshot (device copy of both hypernets'
// params, taken after each iteration). On NumericError the snapshot is saved
// as checkpoint.bin and the error returned (3); at the end the final params.
int morlax_train(const morlax_train_config* cfg, const morlax_run_options* o, morlax_iteration_callback cb,
                 void* user, morlax_trainer** out) {
    morlax_trainer* t = nullptr;
    int rc = morlax_trainer_create(cfg, 1, 0, nullptr, &t);
    if (rc) return rc;
    float *snap_a = nullptr, *snap_c = nullptr;
    rc = guarded([&] {
        Trainer& tr = *t->t;
        const TrainConfig& c = tr.config();
        const morlax_run_options def{nullptr, 300, 10, 8, 10, 0, nullptr, 0};  // trainer.hpp:39, 59-62
        const morlax_run_options& op = o ? *o : def;
        if (op.iterations < 1) throw ConfigError("trainer.iterations must be >= 1");
        if (op.grid_resolution < 1 || op.episodes_per_point < 1 || op.log_interval < 1)
            throw ConfigError("eval: grid_resolution, episodes_per_point and log_interval must be >= 1");
        const EnvSpecB es = env_spec_of(c.env_kind);
        std::vector<double> ref(op.pareto_reference, op.pareto_reference + (op.pareto_reference ? op.n_pareto_reference : 0));
        if (ref.empty()) {  // EnvSpec::hv_reference (env_lqr.cpp:15, env_pointmass.cpp:14, env_deepsea.cpp:31)
            switch (c.env_kind) {
                case ENV_LQR: ref = {-50.0, -20.0}; break;
                case ENV_LQR_M1: ref = {-50.0}; break;
                case ENV_POINTMASS: ref = {-1100.0, -450.0}; break;
                case ENV_DST: ref = {-1.0, -55.0}; break;
                default: ref = H6_HV_REF; break;
            }
        }
        if ((int)ref.size() != es.m) throw ConfigError("pareto_reference length must equal the number of objectives");
        const morlax_checkpoint_extra ex{op.iterations, op.grid_resolution, op.episodes_per_point, op.log_interval,
                                         op.pareto_reference ? op.n_pareto_reference : 0, op.pareto_reference};
        const bool files = op.out_dir && op.out_dir[0];
        std::string dir = files ? std::string(op.out_dir) : std::string();
        FILE* metrics = nullptr;
        if (files) {
            std::filesystem::create_directories(dir);
            metrics = std::fopen((dir + "/metrics.csv").c_str(), "w");
            if (!metrics) throw ConfigError("cannot open metrics log in '" + dir + "'");
            std::fprintf(metrics, "iteration,wall_ms");
            for (int k = 0; k < c.K; ++k) std::fprintf(metrics, ",cluster_%d_return", k);
            std::fprintf(metrics, ",archive_hypervolume\n");
        }
        struct Closer {
            FILE*& f;
            ~Closer() { if (f) std::fclose(f); }
        } closer{metrics};
        const HyperNet& A = tr.actor();
        const HyperNet& Cn = tr.critic();
        MB_CUDA(cudaMalloc(&snap_a, sizeof(float) * A.n));
        MB_CUDA(cudaMalloc(&snap_c, sizeof(float) * Cn.n));
        auto snapshot = [&] {
            MB_CUDA(cudaMemcpyAsync(snap_a, A.p, sizeof(float) * A.n, cudaMemcpyDeviceToDevice, tr.stream()));
            MB_CUDA(cudaMemcpyAsync(snap_c, Cn.p, sizeof(float) * Cn.n, cudaMemcpyDeviceToDevice, tr.stream()));
        };
        snapshot();
        int64_t last_it = 0;
        // actor spec for evaluate_params (HypernetArch::actor_spec)
        morlax_hypernet_spec as{};
        as.m = A.m; as.F = A.F;
        as.n_feature_hidden = (int)c.feat_hidden.size();
        for (size_t k = 0; k < c.feat_hidden.size(); ++k) as.feature_hidden[k] = c.feat_hidden[k];
        as.n_target_sizes = A.tgt.L + 1;
        for (int k = 0; k <= A.tgt.L; ++k) as.target_sizes[k] = A.tgt.sz[k];
        as.target_tanh = A.tgt.out_tanh ? 1 : 0;
        as.has_log_std = A.tgt.has_log_std ? 1 : 0;
        std::vector<double> archive;  // [n][m]
        double archive_hv = 0.0;
        const HostRng root = HostRng::seeded(c.seed);
        for (int it = 0; it < op.iterations; ++it) {
            const auto t0 = std::chrono::steady_clock::now();
            IterStats st;
            try {
                tr.iteration(it, &st);
                if (it % op.log_interval == 0 || it == op.iterations - 1) {
                    const std::vector<double> flat = params_f64(A, A.p, tr.stream());
                    const int64_t np = morlax_simplex_grid_size(es.m, op.grid_resolution);
                    std::vector<double> w((size_t)np * es.m), mr((size_t)np * es.m);
                    int64_t n = 0;
                    const uint64_t key = root.split(0x20000000ULL + (uint64_t)it).key;  // kLaneEvalBase + it
                    if (morlax_evaluate_params(&as, flat.data(), env_name_of(c.env_kind), op.grid_resolution,
                                               op.episodes_per_point, key, w.data(), mr.data(), &n))
                        throw std::runtime_error(g_err);
                    archive.insert(archive.end(), mr.begin(), mr.begin() + n * es.m);
                    const int na = (int)(archive.size() / es.m);
                    std::vector<uint8_t> keep(na);
                    if (morlax_pareto_mask(na, es.m, archive.data(), keep.data())) throw std::runtime_error(g_err);
                    std::vector<double> kept;
                    for (int i = 0; i < na; ++i)
                        if (keep[i]) kept.insert(kept.end(), archive.begin() + (size_t)i * es.m, archive.begin() + (size_t)(i + 1) * es.m);
                    archive.swap(kept);
                    double se = 0;
                    int exact = 0, clipped = 0;
                    if (morlax_hypervolume_detailed((int)(archive.size() / es.m), es.m, archive.data(), ref.data(),
                                                    1000000, 0x9E3779B9ULL, &archive_hv, &se, &exact, &clipped))
                        throw std::runtime_error(g_err);
                }
            } catch (const NumericError&) {  // keep the last healthy state on disk, then rethrow
                if (files) {
                    write_checkpoint(tr, (dir + "/checkpoint.bin").c_str(), last_it, &ex, snap_a, snap_c);
                    std::fflush(metrics);
                }
                throw;
            }
            const double wall_ms =
                op.deterministic ? 0.0
                                 : std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (metrics) {
                std::fprintf(metrics, "%d,%.17g", it, wall_ms);
                for (double r : st.cluster_returns) std::fprintf(metrics, ",%.17g", r);
                std::fprintf(metrics, ",%.17g\n", archive_hv);
                std::fflush(metrics);
            }
            if (cb) {
                morlax_iteration_stats s{it, st.actor_loss, st.critic_loss, archive_hv, (int)st.cluster_returns.size(),
                                         st.cluster_returns.data()};
                if (cb(&s, user)) throw std::runtime_error("iteration callback failed");
            }
            snapshot();
            last_it = it + 1;
        }
        if (files) write_checkpoint(tr, (dir + "/checkpoint.bin").c_str(), last_it, &ex, A.p, Cn.p);
    });
    cudaFree(snap_a);
    cudaFree(snap_c);
    if (rc == 0 && out) {
        *out = t;
    } else {
        morlax_trainer_destroy(t);
        if (out) *out = nullptr;
    }
    return rc;
}

int morlax_trainer_load_checkpoint(morlax_trainer* t, const char* path, int64_t* iteration) {
    return guarded([&] {  // load_checkpoint (checkpoint.cpp:215-241) + the params into the trainer
        FILE* f = std::fopen(path, "rb");
        if (!f) throw ConfigError(std::string("cannot open checkpoint: ") + path);
        std::string b;
        char tmp[1 << 16];
        size_t k;
        while ((k = std::fread(tmp, 1, sizeof(tmp), f)) > 0) b.append(tmp, k);
        std::fclose(f);
        CkReader r{b, 0, path};
        char magic[8];
        r.raw(magic, 8);
        if (std::memcmp(magic, "MRLXCKPT", 8) != 0) throw ConfigError(std::string("not a checkpoint file: ") + path);
        const uint32_t ver = r.get<uint32_t>();
        if (ver != 1) throw ConfigError("unsupported checkpoint version " + std::to_string(ver) + ": " + path);
        r.str();
        for (int i = 0; i < 4; ++i) r.get<int32_t>();
        for (int i = 0; i < 3; ++i) r.get<double>();
        for (int i = 0; i < 2; ++i) r.get<int32_t>();
        for (int i = 0; i < 3; ++i) r.get<double>();
        r.get<int32_t>();
        r.get<uint64_t>();
        r.get<int32_t>();
        for (int i = 0; i < 3; ++i) r.vec_i32();
        for (int i = 0; i < 3; ++i) r.get<int32_t>();
        r.vec_f64();
        Trainer& tr = *t->t;
        for (HyperNet* h : {&tr.actor(), &tr.critic()}) {  // read_hypernet_spec, checked against the trainer
            const int m = r.get<int32_t>(), F = r.get<int32_t>();
            const std::vector<int> fh = r.vec_i32(), ts = r.vec_i32();
            r.get<uint8_t>();
            r.get<uint8_t>();
            const std::vector<int> mine(h->tgt.sz, h->tgt.sz + h->tgt.L + 1);
            std::vector<int> fmine(h->fsz.begin() + 1, h->fsz.end() - 1);
            if (m != h->m || F != h->F || ts != mine || fh != fmine)
                throw ConfigError(std::string("checkpoint architecture does not match the trainer: ") + path);
        }
        const std::vector<double> a = r.vec_f64(), c = r.vec_f64();
        if ((long)a.size() != tr.actor().n || (long)c.size() != tr.critic().n)
            throw ConfigError(std::string("checkpoint parameter count mismatch: ") + path);
        const int64_t it = r.get<int64_t>();
        if (iteration) *iteration = it;
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
        for (int w = 0; w < 2; ++w) {
            HyperNet& h = w ? tr.critic() : tr.actor();
            const std::vector<double>& v = w ? c : a;
            std::vector<float> fl(v.begin(), v.end());
            MB_CUDA(cudaMemcpy(h.p, fl.data(), sizeof(float) * h.n, cudaMemcpyHostToDevice));
            MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
            h.refresh_images(tr.stream());
        }
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
    });
}

int morlax_trainer_get_params(morlax_trainer* t, int which, double* out) {
    return guarded([&] {
        HyperNet& h = which ? t->t->critic() : t->t->actor();
        std::vector<float> f(h.n);
        MB_CUDA(cudaStreamSynchronize(t->t->stream()));
        h.gather_params(t->t->stream());  // sharded optimizer: every rank's M rows (collective)
        MB_CUDA(cudaMemcpy(f.data(), h.p, sizeof(float) * h.n, cudaMemcpyDeviceToHost));
        for (long i = 0; i < h.n; ++i) out[i] = f[i];
    });
}
int morlax_trainer_set_params(morlax_trainer* t, int which, const double* in) {
    return guarded([&] {
        HyperNet& h = which ? t->t->critic() : t->t->actor();
        std::vector<float> f(in, in + h.n);
        MB_CUDA(cudaStreamSynchronize(t->t->stream()));
        MB_CUDA(cudaMemcpy(h.p, f.data(), sizeof(float) * h.n, cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
        h.refresh_images(t->t->stream());
        MB_CUDA(cudaStreamSynchronize(t->t->stream()));
    });
}
int morlax_trainer_get_grad(morlax_trainer* t, int which, double* out) {
    return guarded([&] {
        HyperNet& h = which ? t->t->critic() : t->t->actor();
        std::vector<float> f(h.n);
        MB_CUDA(cudaStreamSynchronize(t->t->stream()));
        h.gather_params(t->t->stream());  // sharded optimizer: every rank's M rows (collective)
        MB_CUDA(cudaMemcpy(f.data(), h.g, sizeof(float) * h.n, cudaMemcpyDeviceToHost));
        for (long i = 0; i < h.n; ++i) out[i] = f[i];
    });
}
int morlax_trainer_get_theta(morlax_trainer* t, int which, float* out) {
    return guarded([&] {
        Trainer& tr = *t->t;
        HyperNet& h = which ? tr.critic() : tr.actor();
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
        const int g0 = (tr.local_groups() == tr.config().K) ? 0 : 0;
        MB_CUDA(cudaMemcpy2D(out, sizeof(float) * h.P, h.theta + (long)g0 * h.ld, sizeof(float) * h.ld,
                             sizeof(float) * h.P, tr.local_groups(), cudaMemcpyDeviceToHost));
        if (h.theta16_last) {  // the update forward kept the hidden layers' weights in bf16 only
            const int G = tr.local_groups();
            std::vector<uint16_t> w((size_t)G * h.P);
            MB_CUDA(cudaMemcpy2D(w.data(), sizeof(uint16_t) * h.P, h.theta16 + (long)g0 * h.ld,
                                 sizeof(uint16_t) * h.ld, sizeof(uint16_t) * h.P, G, cudaMemcpyDeviceToHost));
            for (int g = 0; g < G; ++g)
                for (int l = 0; l + 1 < h.tgt.L; ++l)
                    for (long p = h.tgt.woff[l]; p < h.tgt.woff[l] + (long)h.tgt.sz[l] * h.tgt.sz[l + 1]; ++p) {
                        const uint32_t u = (uint32_t)w[(size_t)g * h.P + p] << 16;
                        std::memcpy(&out[(size_t)g * h.P + p], &u, 4);
                    }
        }
    });
}

static void field_info(Trainer& tr, const std::string& f, void** dev, size_t* bytes) {
    const long R = (long)tr.local_envs() * tr.config().T;
    const EnvSpecB& es = tr.env();
    *dev = nullptr;
    if (f == "obs") { *dev = tr.d_obs; *bytes = sizeof(float) * R * es.obs_dim; }
    else if (f == "action_pre") { *dev = tr.d_act; *bytes = sizeof(float) * R * es.act_dim; }
    else if (f == "logprob") { *dev = tr.d_lp; *bytes = sizeof(float) * R; }
    else if (f == "reward") { *dev = tr.d_rew; *bytes = sizeof(float) * R * es.m; }
    else if (f == "value") { *dev = tr.d_val; *bytes = sizeof(float) * R * es.m; }
    else if (f == "next_value") { *dev = tr.d_nval; *bytes = sizeof(float) * R * es.m; }
    else if (f == "advantages") { *dev = tr.d_adv; *bytes = sizeof(float) * R * es.m; }
    else if (f == "value_targets") { *dev = tr.d_tgt; *bytes = sizeof(float) * R * es.m; }
    else if (f == "scalar_advantage") { *dev = tr.d_sadv; *bytes = sizeof(float) * R; }
    else if (f == "terminated") { *dev = tr.d_term; *bytes = R; }
    else if (f == "truncated") { *dev = tr.d_trunc; *bytes = R; }
    else if (f == "env_state") { *dev = tr.d_state; *bytes = sizeof(float) * es.state_dim * tr.local_envs(); }
    else if (f == "tracker") { *dev = tr.d_tracker; *bytes = sizeof(float) * es.m * tr.local_envs(); }
    else if (f == "env_ctr") { *dev = tr.d_ectr; *bytes = sizeof(uint64_t) * tr.local_envs(); }
    else if (f == "env_steps") { *dev = tr.d_steps; *bytes = sizeof(int) * tr.local_envs(); }
    else if (f == "env_key") { *dev = tr.d_ekey; *bytes = sizeof(uint64_t) * tr.local_envs(); }
    else if (f == "ret_sum") { *dev = tr.d_retsum; *bytes = sizeof(double) * tr.local_envs(); }
    else if (f == "ret_cnt") { *dev = tr.d_retcnt; *bytes = sizeof(int) * tr.local_envs(); }
    else if (f != "clusters" && f != "perm") throw ConfigError("unknown field: " + f);
}
int morlax_trainer_get(morlax_trainer* t, const char* field, void* out) {
    return guarded([&] {
        Trainer& tr = *t->t;
        const std::string f(field);
        if (f == "clusters") {
            std::memcpy(out, tr.clusters_host().data(), sizeof(float) * tr.clusters_host().size());
            return;
        }
        if (f == "perm") {
            std::memcpy(out, tr.perm().data(), sizeof(int) * tr.perm().size());
            return;
        }
        void* dev;
        size_t bytes;
        field_info(tr, f, &dev, &bytes);
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
        MB_CUDA(cudaMemcpy(out, dev, bytes, cudaMemcpyDeviceToHost));
    });
}
int morlax_trainer_set(morlax_trainer* t, const char* field, const void* in) {
    return guarded([&] {
        Trainer& tr = *t->t;
        const std::string f(field);
        if (f == "perm") {
            tr.set_perm(static_cast<const int*>(in));
            return;
        }
        if (f == "clusters") {
            tr.set_clusters((const float*)in);
            return;
        }
        void* dev;
        size_t bytes;
        field_info(tr, f, &dev, &bytes);
        if (!dev) throw ConfigError("field is read-only: " + f);
        MB_CUDA(cudaStreamSynchronize(tr.stream()));
        MB_CUDA(cudaMemcpy(dev, in, bytes, cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
    });
}
int morlax_trainer_losses(morlax_trainer* t, const int32_t* rows, int n, double* al, double* cl) {
    return guarded([&] { t->t->losses_only(rows, n, al, cl); });
}
int64_t morlax_trainer_kernel_launches(morlax_trainer* t) { return t->t->kernel_launches(); }
int morlax_trainer_profile_enable(morlax_trainer* t, int on) {
    return guarded([&] {
        Profiler& p = t->t->profiler();
        p.collect();
        p.reset();
        p.on = on != 0;
    });
}
int morlax_trainer_profile_count(morlax_trainer* t) {
    int n = 0;
    guarded([&] {
        t->t->profiler().collect();
        n = (int)t->t->profiler().cls.size();
    });
    return n;
}
int morlax_trainer_profile_get(morlax_trainer* t, int i, char* name64, double* ms, double* flops, double* bytes,
                               int64_t* count) {
    return guarded([&] {
        Profiler& p = t->t->profiler();
        p.collect();
        if (i < 0 || i >= (int)p.cls.size()) throw ShapeError("profile index out of range");
        const auto& c = p.cls[i];
        std::strncpy(name64, c.name.c_str(), 63);
        name64[63] = 0;
        *ms = c.ms;
        *flops = c.flops;
        *bytes = c.bytes;
        *count = c.count;
    });
}
int morlax_trainer_profile_timeline(morlax_trainer* t, int i, char* name64, int* stream, double* t0_ms,
                                    double* t1_ms) {
    return guarded([&] {
        Profiler& p = t->t->profiler();
        p.collect();
        if (i < 0 || i >= (int)p.timeline.size()) throw ShapeError("timeline index out of range");
        const auto& sp = p.timeline[i];
        std::strncpy(name64, p.cls[sp.c].name.c_str(), 63);
        name64[63] = 0;
        *stream = sp.stream;
        *t0_ms = sp.t0;
        *t1_ms = sp.t1;
    });
}
int morlax_trainer_profile_timeline_count(morlax_trainer* t) {
    int n = 0;
    guarded([&] {
        t->t->profiler().collect();
        n = (int)t->t->profiler().timeline.size();
    });
    return n;
}
void* morlax_trainer_stream(morlax_trainer* t) { return (void*)t->t->stream(); }

int morlax_shard_rows(int64_t P, int world, int rank, int64_t* S, int64_t* row_lo, int64_t* row_hi) {
    return guarded([&] {
        if (P < 1 || world < 1 || rank < 0 || rank >= world) throw ConfigError("shard_rows: bad arguments");
        long s = 0, lo = 0, hi = 0;
        shard_rows(P, world, rank, &s, &lo, &hi);
        *S = s;
        *row_lo = lo;
        *row_hi = hi;
    });
}
int morlax_shard_minibatch(const int32_t* perm, int lo, int hi, int T, int inst_lo, int n_inst, int reps,
                           int n_groups, int32_t* rows_out, int32_t* goff_out, int* n_rows, int* max_group) {
    return guarded([&] {
        shard_minibatch(perm, lo, hi, T, inst_lo, n_inst, reps, n_groups, rows_out, goff_out, n_rows, max_group);
    });
}

// ------------------------------------------------------------------ GEMM test hook
int morlax_gemm_test(int M, int N, int K, const float* A, long am, long ak, const float* B, long bk, long bn,
                     float* C, int use_tc) {
    return guarded([&] {
        long amax = (long)(M - 1) * am + (long)(K - 1) * ak + 1;
        long bmax = (long)(K - 1) * bk + (long)(N - 1) * bn + 1;
        DBuf<float> da(A, amax), db(B, bmax), dc((size_t)M * N);
        if (use_tc) {
            // operands -> tiled bf16 images in the orientation their strides
            // describe (unit stride along K: view 0; along M/N: view 1)
            const int a_view = ak == 1 ? 0 : 1, b_view = bk == 1 ? 0 : 1;
            const int aR = a_view ? K : M, aC = a_view ? M : K, bR = b_view ? K : N, bC = b_view ? N : K;
            DBuf<uint8_t> ia(img_bytes(aR, aC)), ib(img_bytes(bR, bC));
            MB_CUDA(cudaMemset(ia.p, 0, img_bytes(aR, aC)));
            MB_CUDA(cudaMemset(ib.p, 0, img_bytes(bR, bC)));
            Img IA{ia.p, aR, aC, 0}, IB{ib.p, bR, bC, 0};
            to_img(da.p, a_view ? am * 0 + (ak == 1 ? 1 : ak) : am, 0, aR, aC, IA, 1, 0);
            to_img(db.p, b_view ? bn * 0 + bk : bn, 0, bR, bC, IB, 1, 0);
            IGemm d;
            d.A = IA; d.a_view = a_view;
            d.B = IB; d.b_view = b_view;
            d.M = M; d.N = N; d.K = K;
            d.C = dc.p; d.cm = N; d.cn = 1;
            img_gemm(d, 0);
        } else {
            throw ConfigError("gemm_test: the SIMT GEMM was removed; use_tc must be 1");
        }
        MB_CUDA(cudaDeviceSynchronize());
        dc.get(C);
    });
}

// test hook: the fused hypernet M-block gradient + Adam (dm_adam.cu) on host
// arrays at any (G, P, F): dM = gtheta^T f over the bf16 images of gtheta
// [G][P] and f [G][F], Adam on p / m1 / m2 [P][F]; returns the updated
// fp32 state and the bf16 bits of the refreshed M image as rows [P][F]
int morlax_dm_adam_test(int G, int P, int F, const float* gtheta, const float* f, float* p, float* m1, float* m2,
                        float lr, float ibc1, float ibc2, uint16_t* mimg_rows) {
    return guarded([&] {
        DBuf<float> dg(gtheta, (size_t)G * P), dfv(f, (size_t)G * F), dp(p, (size_t)P * F), da(m1, (size_t)P * F),
            db(m2, (size_t)P * F);
        DBuf<uint8_t> gi(img_bytes(G, P)), fi(img_bytes(G, F)), mi(img_bytes(P, F));
        DBuf<int> err(1);
        MB_CUDA(cudaMemset(gi.p, 0, img_bytes(G, P)));
        MB_CUDA(cudaMemset(fi.p, 0, img_bytes(G, F)));
        MB_CUDA(cudaMemset(mi.p, 0, img_bytes(P, F)));
        MB_CUDA(cudaMemset(err.p, 0, sizeof(int)));
        DmAdam a;
        a.gimg = Img{gi.p, G, P, 0};
        a.fimg = Img{fi.p, G, F, 0};
        a.mimg = Img{mi.p, P, F, 0};
        to_img(dg.p, P, 0, G, P, a.gimg, 1, 0);
        to_img(dfv.p, F, 0, G, F, a.fimg, 1, 0);
        a.G = G; a.P = P; a.F = F;
        a.p = dp.p; a.m1 = da.p; a.m2 = db.p;
        a.lr = lr; a.ibc1 = ibc1; a.ibc2 = ibc2; a.err = err.p;
        dm_adam(a, 0);
        MB_CUDA(cudaDeviceSynchronize());
        dp.get(p);
        da.get(m1);
        db.get(m2);
        if (mimg_rows) {
            std::vector<uint8_t> im(img_bytes(P, F));
            MB_CUDA(cudaMemcpy(im.data(), mi.p, im.size(), cudaMemcpyDeviceToHost));
            const int CT = img_ct(F);
            for (long r = 0; r < P; ++r)
                for (int c = 0; c < F; ++c)
                    std::memcpy(mimg_rows + r * F + c, im.data() + img_off(r, c, CT), 2);
        }
    });
}

// microbenchmark hook: D = A(view a) B(view b)^T over random bf16 images,
// epilogue `act` (0 fp32 out, 1 tanh -> image, 2 tanh' -> image); returns ms/launch
int morlax_gemm_bench(int M, int N, int K, int a_view, int b_view, int act, int iters, double* ms) {
    return guarded([&] {
        const int aR = a_view ? K : M, aC = a_view ? M : K, bR = b_view ? K : N, bC = b_view ? N : K;
        DBuf<uint8_t> ia(img_bytes(aR, aC)), ib(img_bytes(bR, bC)), io(img_bytes(M, N)), ix(img_bytes(M, N));
        DBuf<float> c((size_t)M * N);
        MB_CUDA(cudaMemset(ia.p, 0x3c, img_bytes(aR, aC)));
        MB_CUDA(cudaMemset(ib.p, 0x3c, img_bytes(bR, bC)));
        MB_CUDA(cudaMemset(ix.p, 0x3c, img_bytes(M, N)));
        IGemm d;
        d.A = Img{ia.p, aR, aC, 0}; d.a_view = a_view;
        d.B = Img{ib.p, bR, bC, 0}; d.b_view = b_view;
        d.M = M; d.N = N; d.K = K;
        if (act == 0) { d.C = c.p; d.cm = N; d.cn = 1; }
        else { d.act = act; d.O = Img{io.p, M, N, 0}; d.o_mode = 1; d.aux = Img{ix.p, M, N, 0}; }
        // MORLAX_BENCH_TMA=1: B from row-major bf16 rows through a tensor map (the update's weight path)
        const char* te = std::getenv("MORLAX_BENCH_TMA");
        DBuf<uint16_t> brow((size_t)bR * bC);
        if (te && te[0] == '1') {
            MB_CUDA(cudaMemset(brow.p, 0x3c, sizeof(uint16_t) * (size_t)bR * bC));
            MB_CUDA(cudaStreamSynchronize(0));
            if (!make_weight_map(&d.bmap, brow.p, bR, bC, (long)bR * bC, 1)) throw ConfigError("gemm_bench: tensor map");
            d.b_tma = 1;
        }
        img_gemm(d, 0);
        cudaEvent_t e0, e1;
        MB_CUDA(cudaEventCreate(&e0));
        MB_CUDA(cudaEventCreate(&e1));
        MB_CUDA(cudaEventRecord(e0, 0));
        for (int i = 0; i < iters; ++i) img_gemm(d, 0);
        MB_CUDA(cudaEventRecord(e1, 0));
        MB_CUDA(cudaEventSynchronize(e1));
        float t = 0;
        MB_CUDA(cudaEventElapsedTime(&t, e0, e1));
        *ms = t / iters;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

// ------------------------------------------------------------------ pareto
int morlax_pareto_mask_device(int n, int m, const double* d_pts, uint8_t* d_mask, void* stream) {
    return guarded([&] {
        if (m < 1 || m > 8) throw ShapeError("pareto: objective count must be in [1, 8]");
        DBuf<uint8_t> uq(n);
        DBuf<double> sums(n);
        pareto_mask(n, m, d_pts, d_mask, uq.p, sums.p, (cudaStream_t)stream);
        MB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    });
}
int morlax_pareto_mask(int n, int m, const double* pts, uint8_t* mask) {
    return guarded([&] {
        if (n <= 0) return;
        if (m < 1 || m > 8) throw ShapeError("pareto: objective count must be in [1, 8]");
        DBuf<double> p(pts, (size_t)n * m);
        DBuf<uint8_t> mk(n), uq(n);
        DBuf<double> sums(n);
        pareto_mask(n, m, p.p, mk.p, uq.p, sums.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        mk.get(mask);
    });
}
int morlax_linear_dominance_mask(int n, int m, const double* pts, uint8_t* mask) {
    return guarded([&] {  // pareto.cpp:79-139
        if (m < 1 || m > 8) throw ShapeError("linear_dominance_filter: objective count must be in [1, 8]");
        if (n <= 0) return;
        DBuf<double> p(pts, (size_t)n * m);
        DBuf<uint8_t> mk(n), uq(n);
        DBuf<double> sums(n);
        pareto_mask(n, m, p.p, mk.p, uq.p, sums.p, 0);  // nd = nondominated_filter(points)
        MB_CUDA(cudaDeviceSynchronize());
        mk.get(mask);
        std::vector<int> idx;
        for (int i = 0; i < n; ++i)
            if (mask[i]) idx.push_back(i);
        const int nn = (int)idx.size();
        if (nn <= 2 || m == 1) return;
        std::vector<double> nd((size_t)nn * m);
        for (int q = 0; q < nn; ++q) std::memcpy(&nd[(size_t)q * m], pts + (size_t)idx[q] * m, sizeof(double) * m);
        DBuf<double> dnd(nd.data(), nd.size());
        DBuf<uint8_t> keep(nn);
        DBuf<int> scratch(2 * (size_t)nn);
        linear_dominance(nn, m, dnd.p, keep.p, scratch.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        std::vector<uint8_t> k(nn);
        keep.get(k.data());
        for (int q = 0; q < nn; ++q) mask[idx[q]] = k[q];
    });
}
int morlax_hypervolume_mc(int n, int m, const double* pts, const double* ref, uint64_t samples, uint64_t key,
                          uint64_t ctr, double* value, double* se, uint64_t* hits_out) {
    return guarded([&] {
        if (samples == 0) throw ShapeError("hypervolume_mc: samples must be > 0");
        if (m < 1 || m > 8) throw ShapeError("hypervolume: objective count must be in [1, 8]");
        *value = 0.0;
        if (se) *se = 0.0;
        if (hits_out) *hits_out = 0;
        if (n <= 0) return;
        DBuf<double> p(pts, (size_t)n * m), r(ref, m), scratch((size_t)n * m + 8 + n + 8);
        DBuf<unsigned long long> hits(1);
        hv_mc(n, m, p.p, r.p, samples, key, ctr, hits.p, scratch.p, 0);
        MB_CUDA(cudaDeviceSynchronize());
        unsigned long long h = 0;
        hits.get(&h);
        double hi[8];
        MB_CUDA(cudaMemcpy(hi, scratch.p, sizeof(double) * m, cudaMemcpyDeviceToHost));
        int k = 0;
        MB_CUDA(cudaMemcpy(&k, (int*)(scratch.p + 8 + (size_t)n * m), sizeof(int), cudaMemcpyDeviceToHost));
        if (k == 0) return;
        double box = 1.0;  // pareto.cpp:253-254, same order -> bit-identical
        for (int j = 0; j < m; ++j) box *= hi[j] - ref[j];
        if (box == 0.0) return;
        const double frac = (double)h / (double)samples;
        if (se) *se = box * std::sqrt(frac * (1.0 - frac) / (double)samples);
        *value = box * frac;
        if (hits_out) *hits_out = h;
    });
}
int morlax_hypervolume_exact(int n, int m, const double* pts, const double* ref, double* value, int* clipped) {
    return guarded([&] {
        if (m < 1 || m > 8) throw ShapeError("hypervolume: objective count must be in [1, 8]");
        *value = 0.0;
        if (clipped) *clipped = 0;
        if (n <= 0) return;
        DBuf<double> p(pts, (size_t)n * m), r(ref, m);
        int c = 0;
        hv_exact(n, m, p.p, r.p, value, &c, 0);
        if (clipped) *clipped = c;
    });
}
int morlax_hypervolume_exact_device(int n, int m, const double* d_pts, const double* d_ref, double* value,
                                    int* clipped, void* stream) {
    return guarded([&] {
        if (m < 1 || m > 8) throw ShapeError("hypervolume: objective count must be in [1, 8]");
        *value = 0.0;
        int c = 0;
        if (n > 0) hv_exact(n, m, d_pts, d_ref, value, &c, (cudaStream_t)stream);
        if (clipped) *clipped = c;
    });
}
int morlax_hypervolume_detailed(int n, int m, const double* pts, const double* ref, uint64_t samples, uint64_t seed,
                                double* value, double* se, int* exact, int* clipped) {
    return guarded([&] {
        if (m < 1) throw ShapeError("hypervolume: empty reference point");
        int cl = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < m; ++j)
                if (pts[(size_t)i * m + j] < ref[j]) { ++cl; break; }
        if (clipped) *clipped = cl;
        if (m > 8) throw ShapeError("hypervolume: objective count must be in [1, 8]");
        if (m <= 4) {  // pareto.cpp:217-219: exact for m <= 4 (device WFG recursion)
            if (exact) *exact = 1;
            if (se) *se = 0.0;
            *value = 0.0;
            if (n <= 0) return;
            DBuf<double> p(pts, (size_t)n * m), r(ref, m);
            int c2 = 0;
            hv_exact(n, m, p.p, r.p, value, &c2, 0);
            return;
        }
        if (exact) *exact = 0;
        const uint64_t key = seed_key(seed);
        const int rc = morlax_hypervolume_mc(n, m, pts, ref, samples, key, 0, value, se, nullptr);
        if (rc) throw std::runtime_error(g_err);
    });
}

}  // extern "C"
