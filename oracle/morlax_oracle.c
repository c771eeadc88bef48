/* TEST INFRASTRUCTURE ONLY -- see morlax_oracle.h. fp64 restatement of the
 * MORLAX reference hot path. Every function cites the reference lines it
 * restates (paths relative to /root/reference/proj). Build flags must keep
 * -ffp-contract=off so that a + b*c rounds exactly like the reference's
 * x86-64 build (no FMA). */
#include "morlax_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2603_09237_b200/csrc/humanoid6_params.h"

static __thread char g_err[512];
const char* mo_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

/* ========================================================================= */
/* RNG: include/morlax/rng.hpp:18-93                                          */
/* ========================================================================= */
#define K_GAMMA 0x9E3779B97F4A7C15ULL
#define K_SEED 0x5851F42D4C957F2DULL
#define K_SPLIT 0xA0761D6478BD642FULL
#define K_LANE 0xE7037ED1A0B428DBULL

static inline uint64_t mix64(uint64_t z) { /* rng.hpp:85-89 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
mo_rng mo_rng_seed(uint64_t seed) { /* rng.hpp:21 */
    mo_rng r = {mix64(seed ^ K_SEED), 0};
    return r;
}
mo_rng mo_rng_split(mo_rng r, uint64_t lane) { /* rng.hpp:35-40 */
    mo_rng c = {mix64(mix64(r.key ^ K_SPLIT) + mix64(lane ^ K_LANE)), 0};
    return c;
}
uint64_t mo_rng_next_u64(mo_rng* r) { return mix64(r->key + K_GAMMA * ++r->ctr); } /* :42 */
double mo_rng_next_double(mo_rng* r) { /* :45 */
    return (double)(mo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}
double mo_rng_next_open(mo_rng* r) { /* :48-50 */
    return (double)((mo_rng_next_u64(r) >> 11) + 1) * 0x1.0p-53;
}
double mo_rng_uniform(mo_rng* r, double lo, double hi) { /* :52 */
    return lo + (hi - lo) * mo_rng_next_double(r);
}
double mo_rng_next_gaussian(mo_rng* r) { /* :55-60 Box-Muller, 2 words */
    const double u1 = mo_rng_next_open(r);
    const double u2 = mo_rng_next_double(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}
uint64_t mo_rng_next_below(mo_rng* r, uint64_t n) { /* :64-67 */
    return (uint64_t)(((unsigned __int128)mo_rng_next_u64(r) * n) >> 64);
}
void mo_rng_shuffle_i32(mo_rng* r, int32_t* v, int64_t n) { /* :71-76 */
    for (int64_t i = n; i > 1; --i) {
        int64_t j = (int64_t)mo_rng_next_below(r, (uint64_t)i);
        int32_t t = v[i - 1];
        v[i - 1] = v[j];
        v[j] = t;
    }
}
void mo_rng_seed_state(uint64_t seed, uint64_t* key, uint64_t* ctr) {
    mo_rng r = mo_rng_seed(seed);
    *key = r.key;
    *ctr = r.ctr;
}
uint64_t mo_rng_split_key(uint64_t key, uint64_t lane) {
    mo_rng r = {key, 0};
    return mo_rng_split(r, lane).key;
}
void mo_rng_words(uint64_t key, uint64_t ctr, int64_t n, uint64_t* out) {
    mo_rng r = {key, ctr};
    for (int64_t i = 0; i < n; ++i) out[i] = mo_rng_next_u64(&r);
}
void mo_rng_gaussians(uint64_t key, uint64_t ctr, int64_t n, double* out) {
    mo_rng r = {key, ctr};
    for (int64_t i = 0; i < n; ++i) out[i] = mo_rng_next_gaussian(&r);
}
void mo_rng_shuffle(uint64_t key, uint64_t* ctr, int32_t* v, int64_t n) {
    mo_rng r = {key, *ctr};
    mo_rng_shuffle_i32(&r, v, n);
    *ctr = r.ctr;
}

/* ========================================================================= */
/* NN: src/nn.cpp                                                             */
/* ========================================================================= */
#define LOG_STD_MIN (-5.0)
#define LOG_STD_MAX (1.0)
#define TANH_EPS 1e-6
#define LOG_SQRT_2PI 0.9189385332046727 /* nn.cpp:14 */
#define HYPER_INIT_SCALE 0.01           /* hypernet.hpp:67 */
#define LOG_STD_INIT (-1.0)             /* hypernet.hpp:68 */

static inline double clampd(double x, double lo, double hi) {
    return x < lo ? lo : (hi < x ? hi : x); /* std::clamp semantics */
}

int64_t mo_mlp_param_count(const mo_mlp* s) { /* nn.cpp:29-36 */
    int64_t n = 0;
    for (int l = 0; l + 1 < s->n_sizes; ++l) n += (int64_t)(s->sizes[l] + 1) * s->sizes[l + 1];
    return n;
}
static int mlp_width_max(const mo_mlp* s) {
    int w = 0;
    for (int l = 0; l < s->n_sizes; ++l) w = s->sizes[l] > w ? s->sizes[l] : w;
    return w;
}

/* Cached forward (nn.cpp:60-92). acts: (n_sizes) rows of width wmax;
 * acts[0] = input; preact = last layer pre-activation. */
typedef struct {
    int L, wmax;
    double* acts;   /* (L+1) * wmax */
    double* preact; /* wmax */
    double* g;      /* scratch */
    double* gprev;
} mlp_work;
static void work_init(mlp_work* w, const mo_mlp* s) {
    w->L = s->n_sizes - 1;
    w->wmax = mlp_width_max(s);
    w->acts = (double*)calloc((size_t)(w->L + 1) * w->wmax, sizeof(double));
    w->preact = (double*)calloc(w->wmax, sizeof(double));
    w->g = (double*)calloc(w->wmax, sizeof(double));
    w->gprev = (double*)calloc(w->wmax, sizeof(double));
}
static void work_free(mlp_work* w) {
    free(w->acts);
    free(w->preact);
    free(w->g);
    free(w->gprev);
}
static inline double* act_row(mlp_work* w, int l) { return w->acts + (size_t)l * w->wmax; }

static void mlp_forward_cached(const mo_mlp* s, const double* params, const double* input,
                               mlp_work* w) {
    const int L = s->n_sizes - 1;
    memcpy(act_row(w, 0), input, sizeof(double) * s->sizes[0]);
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        const int in = s->sizes[l], out = s->sizes[l + 1];
        const double* W = params + off;
        const double* b = W + (size_t)in * out;
        const double* a = act_row(w, l);
        double* next = act_row(w, l + 1);
        const int last = (l == L - 1);
        for (int j = 0; j < out; ++j) {
            double z = b[j];
            const double* wr = W + (size_t)j * in;
            for (int i = 0; i < in; ++i) z += wr[i] * a[i];
            if (last) {
                w->preact[j] = z;
                next[j] = s->out_tanh ? tanh(z) : z;
            } else {
                next[j] = tanh(z);
            }
        }
        off += (size_t)(in + 1) * out;
    }
}

static int all_finite(const double* v, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

int mo_mlp_forward(const mo_mlp* s, const double* params, const double* in, double* out) {
    /* nn.cpp:94-109 (validating) */
    if (s->n_sizes < 2) return fail(MO_ERR, "MlpSpec needs at least input and output sizes");
    if (!all_finite(params, mo_mlp_param_count(s))) return fail(MO_NUMERIC, "non-finite value in mlp params");
    if (!all_finite(in, s->sizes[0])) return fail(MO_NUMERIC, "non-finite value in mlp input");
    mlp_work w;
    work_init(&w, s);
    mlp_forward_cached(s, params, in, &w);
    memcpy(out, act_row(&w, w.L), sizeof(double) * s->sizes[s->n_sizes - 1]);
    work_free(&w);
    return MO_OK;
}

/* nn.cpp:111-160 */
static void mlp_backward(const mo_mlp* s, const double* params, mlp_work* w,
                         const double* grad_out, int grad_at_preact, double* gparams,
                         double* grad_input /* may be NULL */) {
    const int L = s->n_sizes - 1;
    const int od = s->sizes[L];
    double* g = w->g;
    memcpy(g, grad_out, sizeof(double) * od);
    if (!grad_at_preact && s->out_tanh) {
        const double* aL = act_row(w, L);
        for (int j = 0; j < od; ++j) g[j] *= 1.0 - aL[j] * aL[j];
    }
    size_t offs[MO_MAX_LAYERS + 1];
    size_t off = 0;
    for (int l = 0; l < L; ++l) {
        offs[l] = off;
        off += (size_t)(s->sizes[l] + 1) * s->sizes[l + 1];
    }
    for (int l = L - 1; l >= 0; --l) {
        const int in = s->sizes[l], out = s->sizes[l + 1];
        const double* W = params + offs[l];
        double* gW = gparams + offs[l];
        double* gb = gW + (size_t)in * out;
        const double* a = act_row(w, l);
        for (int j = 0; j < out; ++j) {
            const double gj = g[j];
            double* gr = gW + (size_t)j * in;
            for (int i = 0; i < in; ++i) gr[i] += gj * a[i];
            gb[j] += gj;
        }
        if (l == 0 && grad_input == NULL) break;
        double* gp = w->gprev;
        for (int i = 0; i < in; ++i) gp[i] = 0.0;
        for (int j = 0; j < out; ++j) {
            const double gj = g[j];
            const double* wr = W + (size_t)j * in;
            for (int i = 0; i < in; ++i) gp[i] += gj * wr[i];
        }
        if (l > 0)
            for (int i = 0; i < in; ++i) gp[i] *= 1.0 - a[i] * a[i];
        memcpy(g, gp, sizeof(double) * in);
    }
    if (grad_input) memcpy(grad_input, g, sizeof(double) * s->sizes[0]);
}

/* nn.cpp:260-274 */
static void init_mlp(const mo_mlp* s, mo_rng* rng, double* out) {
    size_t off = 0;
    for (int l = 0; l + 1 < s->n_sizes; ++l) {
        const int in = s->sizes[l], out_ = s->sizes[l + 1];
        const double bound = 1.0 / sqrt((double)in);
        const size_t n = (size_t)(in + 1) * out_;
        for (size_t k = 0; k < n; ++k) out[off + k] = mo_rng_uniform(rng, -bound, bound);
        off += n;
    }
}
int mo_init_mlp(const mo_mlp* s, uint64_t key, uint64_t ctr, double* out) {
    mo_rng r = {key, ctr};
    init_mlp(s, &r, out);
    return MO_OK;
}

/* nn.cpp:192-219: log-density of tanh(z) under the squashed Gaussian */
static double action_logprob(int d, const double* mu, const double* ls, const double* z) {
    double lp = 0.0;
    for (int i = 0; i < d; ++i) {
        const double sigma = exp(ls[i]);
        const double zn = (z[i] - mu[i]) / sigma;
        const double a = tanh(z[i]);
        lp += -0.5 * zn * zn - ls[i] - LOG_SQRT_2PI;
        lp -= log(1.0 - a * a + TANH_EPS);
    }
    return lp;
}
static double gaussian_entropy(int d, const double* ls) { /* nn.cpp:221-226 */
    double h = 0.0;
    for (int i = 0; i < d; ++i) h += ls[i] + 0.5 * (1.0 + log(2.0 * 3.141592653589793));
    return h;
}

/* ========================================================================= */
/* Hypernet: src/hypernet.cpp                                                 */
/* ========================================================================= */
void mo_hspec_feature_spec(const mo_hspec* h, mo_mlp* fs) { /* hypernet.cpp:10-17 */
    fs->n_sizes = 0;
    fs->sizes[fs->n_sizes++] = h->m;
    for (int i = 0; i < h->n_feat_hidden; ++i) fs->sizes[fs->n_sizes++] = h->feat_hidden[i];
    fs->sizes[fs->n_sizes++] = h->F;
    fs->out_tanh = 1;
}
int64_t mo_hspec_feature_count(const mo_hspec* h) {
    mo_mlp fs;
    mo_hspec_feature_spec(h, &fs);
    return mo_mlp_param_count(&fs);
}
int64_t mo_hspec_target_count(const mo_hspec* h) { /* hypernet.cpp:19-22 */
    return mo_mlp_param_count(&h->target) +
           (h->has_log_std ? h->target.sizes[h->target.n_sizes - 1] : 0);
}
int64_t mo_hspec_param_count(const mo_hspec* h) { /* hypernet.cpp:44-48 */
    return mo_hspec_feature_count(h) + mo_hspec_target_count(h) * h->F + mo_hspec_target_count(h);
}

static int check_simplex(int m, const double* w) { /* simplex.cpp:18-30 */
    double sum = 0.0;
    for (int i = 0; i < m; ++i) {
        if (!(w[i] >= 0.0)) return fail(MO_ERR, "trade-off entries must be nonnegative");
        sum += w[i];
    }
    if (fabs(sum - 1.0) > 1e-9) return fail(MO_ERR, "trade-off entries must sum to 1 (got %f)", sum);
    return MO_OK;
}

int mo_hypernet_features(const mo_hspec* h, const double* flat, const double* w, double* f) {
    int rc = check_simplex(h->m, w);
    if (rc) return rc;
    mo_mlp fs;
    mo_hspec_feature_spec(h, &fs);
    mlp_work wk;
    work_init(&wk, &fs);
    mlp_forward_cached(&fs, flat, w, &wk);
    memcpy(f, act_row(&wk, wk.L), sizeof(double) * h->F);
    work_free(&wk);
    return MO_OK;
}

int mo_hypernet_forward(const mo_hspec* h, const double* flat, const double* w, double* theta) {
    /* hypernet.cpp:69-90 */
    const int64_t nf = mo_hspec_feature_count(h), P = mo_hspec_target_count(h);
    const int F = h->F;
    double* f = (double*)malloc(sizeof(double) * F);
    int rc = mo_hypernet_features(h, flat, w, f);
    if (rc) { free(f); return rc; }
    const double* M = flat + nf;
    const double* b = M + P * F;
    for (int64_t j = 0; j < P; ++j) {
        double z = b[j];
        const double* row = M + j * F;
        for (int k = 0; k < F; ++k) z += row[k] * f[k];
        theta[j] = z;
        if (!isfinite(z)) {
            free(f);
            return fail(MO_NUMERIC, "hypernet_forward produced a non-finite parameter at index %lld",
                        (long long)j);
        }
    }
    free(f);
    return MO_OK;
}

int mo_hypernet_backward(const mo_hspec* h, const double* flat, const double* w,
                         const double* gtheta, double* gflat) {
    /* hypernet.cpp:92-122 -- accumulates into gflat */
    int rc = check_simplex(h->m, w);
    if (rc) return rc;
    const int64_t nf = mo_hspec_feature_count(h), P = mo_hspec_target_count(h);
    const int F = h->F;
    mo_mlp fs;
    mo_hspec_feature_spec(h, &fs);
    mlp_work wk;
    work_init(&wk, &fs);
    mlp_forward_cached(&fs, flat, w, &wk);
    const double* f = act_row(&wk, wk.L);
    const double* M = flat + nf;
    double* gM = gflat + nf;
    double* gb = gM + P * F;
    double* gf = (double*)calloc(F, sizeof(double));
    for (int64_t j = 0; j < P; ++j) {
        const double gj = gtheta[j];
        gb[j] += gj;
        const double* Mr = M + j * F;
        double* gMr = gM + j * F;
        for (int k = 0; k < F; ++k) {
            gMr[k] += gj * f[k];
            gf[k] += gj * Mr[k];
        }
    }
    mlp_backward(&fs, flat, &wk, gf, 0, gflat, NULL);
    free(gf);
    work_free(&wk);
    return MO_OK;
}

int mo_init_hypernet(const mo_hspec* h, uint64_t key, uint64_t ctr, double* flat) {
    /* hypernet.cpp:124-145 */
    mo_rng rng = {key, ctr};
    mo_rng frng = mo_rng_split(rng, 0), mrng = mo_rng_split(rng, 1), brng = mo_rng_split(rng, 2);
    const int64_t nf = mo_hspec_feature_count(h), P = mo_hspec_target_count(h);
    const int F = h->F;
    mo_mlp fs;
    mo_hspec_feature_spec(h, &fs);
    init_mlp(&fs, &frng, flat);
    double* M = flat + nf;
    const double m_std = HYPER_INIT_SCALE / sqrt((double)F);
    for (int64_t i = 0; i < P * F; ++i) M[i] = m_std * mo_rng_next_gaussian(&mrng);
    double* b = M + P * F;
    init_mlp(&h->target, &brng, b);
    for (int64_t j = mo_mlp_param_count(&h->target); j < P; ++j) b[j] = LOG_STD_INIT;
    return MO_OK;
}

/* ========================================================================= */
/* Envs: src/env.cpp, env_lqr.cpp, env_pointmass.cpp, env_deepsea.cpp        */
/* ========================================================================= */
static const double kDstDepths[10] = {1, 6, 7, 9, 10, 11, 14, 15, 18, 20};   /* env_deepsea.cpp:15 */
static const double kDstValues[10] = {0.7, 8.2, 11.5, 14.0, 15.1, 16.1, 19.6, 20.3, 22.4, 23.7};
static const double H6cx[12] = H6_CX, H6cy[12] = H6_CY, H6cz[12] = H6_CZ, H6cr[12] = H6_CR,
                    H6cp[12] = H6_CP, H6cw[12] = H6_CW;

int mo_env_spec(int kind, mo_envspec* o) {
    o->kind = kind;
    switch (kind) {
        case MO_ENV_LQR: o->obs_dim = 1; o->act_dim = 1; o->m = 2; o->max_steps = 200; return MO_OK;
        case MO_ENV_LQR_M1: o->obs_dim = 1; o->act_dim = 1; o->m = 1; o->max_steps = 200; return MO_OK;
        case MO_ENV_POINTMASS: o->obs_dim = 4; o->act_dim = 2; o->m = 2; o->max_steps = 200; return MO_OK;
        case MO_ENV_DST: o->obs_dim = 1; o->act_dim = 1; o->m = 2; o->max_steps = 50; return MO_OK;
        case MO_ENV_HUMANOID6:
            o->obs_dim = H6_OBS; o->act_dim = H6_ACT; o->m = H6_M; o->max_steps = H6_HORIZON;
            return MO_OK;
    }
    return fail(MO_ERR, "unknown environment kind %d", kind);
}
int mo_env_kind_from_name(const char* n) { /* registry.cpp:17-23 */
    if (!strcmp(n, "mo-lqr1d")) return MO_ENV_LQR;
    if (!strcmp(n, "mo-lqr1d-m1")) return MO_ENV_LQR_M1;
    if (!strcmp(n, "mo-pointmass")) return MO_ENV_POINTMASS;
    if (!strcmp(n, "mo-dst-continuous")) return MO_ENV_DST;
    if (!strcmp(n, "mo-humanoid6")) return MO_ENV_HUMANOID6;
    return -1;
}

struct mo_env {
    mo_envspec spec;
    int n;
    int sdim;        /* physical state width */
    double* state;   /* n * sdim */
    mo_rng* streams; /* n */
    int32_t* steps;  /* n */
    double* cur_obs; /* n * obs_dim */
    uint64_t clamps;
};

static int env_state_dim(int kind) {
    switch (kind) {
        case MO_ENV_POINTMASS: return 4;
        case MO_ENV_HUMANOID6: return H6_OBS;
        default: return 1;
    }
}

mo_env* mo_env_create(int kind, int n) {
    mo_envspec sp;
    if (mo_env_spec(kind, &sp) || n < 1) return NULL;
    mo_env* e = (mo_env*)calloc(1, sizeof(mo_env));
    e->spec = sp;
    e->n = n;
    e->sdim = env_state_dim(kind);
    e->state = (double*)calloc((size_t)n * e->sdim, sizeof(double));
    e->streams = (mo_rng*)calloc(n, sizeof(mo_rng));
    e->steps = (int32_t*)calloc(n, sizeof(int32_t));
    e->cur_obs = (double*)calloc((size_t)n * sp.obs_dim, sizeof(double));
    return e;
}
void mo_env_destroy(mo_env* e) {
    if (!e) return;
    free(e->state);
    free(e->streams);
    free(e->steps);
    free(e->cur_obs);
    free(e);
}

static void do_reset(mo_env* e, int i) {
    double* s = e->state + (size_t)i * e->sdim;
    mo_rng* st = &e->streams[i];
    switch (e->spec.kind) {
        case MO_ENV_LQR:
        case MO_ENV_LQR_M1: s[0] = mo_rng_uniform(st, -1.0, 1.0); break; /* env_lqr.cpp:20-22 */
        case MO_ENV_POINTMASS:                                              /* env_pointmass.cpp:22-28 */
            s[0] = mo_rng_uniform(st, -0.1, 0.1);
            s[1] = mo_rng_uniform(st, -0.1, 0.1);
            s[2] = 0.0;
            s[3] = 0.0;
            break;
        case MO_ENV_DST: s[0] = 0.0; break; /* env_deepsea.cpp:33-37 */
        case MO_ENV_HUMANOID6:
            for (int k = 0; k < H6_OBS; ++k) s[k] = mo_rng_uniform(st, -H6_INIT, H6_INIT);
            break;
    }
}
static void write_obs(const mo_env* e, int i, double* out) {
    const double* s = e->state + (size_t)i * e->sdim;
    memcpy(out, s, sizeof(double) * e->spec.obs_dim); /* obs == state for all envs */
}
static void do_step(mo_env* e, int i, const double* a, double* r, int* term) {
    double* s = e->state + (size_t)i * e->sdim;
    *term = 0;
    switch (e->spec.kind) {
        case MO_ENV_LQR:
        case MO_ENV_LQR_M1: { /* env_lqr.cpp:25-37 */
            const double u = a[0];
            r[0] = -s[0] * s[0];
            if (e->spec.kind == MO_ENV_LQR) r[1] = -u * u;
            s[0] = 0.9 * s[0] + 0.5 * u;
            break;
        }
        case MO_ENV_POINTMASS: /* env_pointmass.cpp:30-41 */
            s[2] += 0.05 * a[0];
            s[3] += 0.05 * a[1];
            s[0] += 0.05 * s[2];
            s[1] += 0.05 * s[3];
            r[0] = s[2];
            r[1] = -(a[0] * a[0] + a[1] * a[1]);
            break;
        case MO_ENV_DST: /* env_deepsea.cpp:39-59 */
            s[0] += a[0];
            r[0] = 0.0;
            r[1] = -1.0;
            for (int t = 0; t < 10; ++t)
                if (fabs(s[0] - kDstDepths[t]) <= 0.25) {
                    r[0] = kDstValues[t];
                    *term = 1;
                    break;
                }
            break;
        case MO_ENV_HUMANOID6: { /* csrc/humanoid6_params.h */
            double* q = s;
            double* qd = s + 12;
            double* ee = s + 24;
            double sx = 0, sy = 0, sz = 0, sr = 0, sp = 0, sw = 0, asq = 0, qsq = 0;
            for (int j = 0; j < 12; ++j) {
                ee[j] += H6_ALPHA * (a[j] - ee[j]);
                qd[j] += H6_DT * (H6_KT * ee[j] - H6_KP * q[j] - H6_KD * qd[j]);
                q[j] += H6_DT * qd[j];
                const double sj = tanh(qd[j]);
                sx += H6cx[j] * sj;
                sy += H6cy[j] * sj;
                sw += H6cw[j] * sj;
                sz += H6cz[j] * ee[j];
                sr += H6cr[j] * ee[j];
                sp += H6cp[j] * ee[j];
                asq += a[j] * a[j];
                qsq += qd[j] * qd[j];
            }
            double *h = s + 36, *vx = s + 37, *vy = s + 38, *vz = s + 39, *roll = s + 40,
                   *pitch = s + 41, *wx = s + 42, *wy = s + 43, *wz = s + 44;
            *vx += H6_DT * (sx - H6_DRAG * *vx);
            *vy += H6_DT * (sy - H6_DRAG * *vy);
            *vz += H6_DT * (sz - H6_KH * *h - H6_DZ * *vz);
            *h += H6_DT * *vz;
            *wx += H6_DT * (sr - H6_KA * *roll - H6_DA * *wx);
            *roll += H6_DT * *wx;
            *wy += H6_DT * (sp - H6_KA * *pitch - H6_DA * *wy);
            *pitch += H6_DT * *wy;
            *wz += H6_DT * (sw - H6_DRAG * *wz);
            r[0] = *vx;
            r[1] = -asq / 12.0;
            r[2] = -(*roll * *roll + *pitch * *pitch);
            r[3] = *vy;
            r[4] = -0.1 * qsq / 12.0;
            r[5] = -(*h * *h + 0.1 * *wz * *wz);
            *term = (fabs(*roll) > H6_FALL || fabs(*pitch) > H6_FALL) ? 1 : 0;
            break;
        }
    }
}
static void reset_instance(mo_env* e, int i) { /* env.cpp:44-49 */
    do_reset(e, i);
    e->steps[i] = 0;
    write_obs(e, i, e->cur_obs + (size_t)i * e->spec.obs_dim);
}
int mo_env_reset(mo_env* e, uint64_t key, uint64_t ctr, double* obs_out) { /* env.cpp:51-58 */
    mo_rng r = {key, ctr};
    for (int i = 0; i < e->n; ++i) {
        e->streams[i] = mo_rng_split(r, (uint64_t)i);
        reset_instance(e, i);
    }
    if (obs_out) memcpy(obs_out, e->cur_obs, sizeof(double) * e->n * e->spec.obs_dim);
    return MO_OK;
}
static int step_instance(mo_env* e, int i, const double* action, double* reward, uint8_t* term,
                         uint8_t* trunc, double* final_obs) { /* env.cpp:60-92 */
    double cl[16];
    int any = 0;
    for (int d = 0; d < e->spec.act_dim; ++d) {
        if (!isfinite(action[d])) return fail(MO_NUMERIC, "non-finite action for environment instance %d", i);
        cl[d] = clampd(action[d], -1.0, 1.0);
        any |= cl[d] != action[d];
    }
    if (any) e->clamps++;
    int t = 0;
    do_step(e, i, cl, reward, &t);
    e->steps[i] += 1;
    const int tr = !t && e->steps[i] >= e->spec.max_steps;
    *term = (uint8_t)t;
    *trunc = (uint8_t)tr;
    write_obs(e, i, final_obs);
    if (t || tr)
        reset_instance(e, i);
    else
        memcpy(e->cur_obs + (size_t)i * e->spec.obs_dim, final_obs, sizeof(double) * e->spec.obs_dim);
    return MO_OK;
}
int mo_env_step(mo_env* e, const double* actions, double* obs, double* reward, uint8_t* term,
                uint8_t* trunc) { /* env.cpp:94-106 */
    const mo_envspec* s = &e->spec;
    for (int i = 0; i < e->n; ++i) {
        int rc = step_instance(e, i, actions + (size_t)i * s->act_dim, reward + (size_t)i * s->m,
                               term + i, trunc + i, obs + (size_t)i * s->obs_dim);
        if (rc) return rc;
    }
    return MO_OK;
}
void mo_env_current_obs(const mo_env* e, double* out) {
    memcpy(out, e->cur_obs, sizeof(double) * e->n * e->spec.obs_dim);
}
uint64_t mo_env_clamp_count(const mo_env* e) { return e->clamps; }
void mo_env_get_streams(const mo_env* e, uint64_t* keys, uint64_t* ctrs, int32_t* steps) {
    for (int i = 0; i < e->n; ++i) {
        if (keys) keys[i] = e->streams[i].key;
        if (ctrs) ctrs[i] = e->streams[i].ctr;
        if (steps) steps[i] = e->steps[i];
    }
}

/* Test hook (teacher forcing; not a reference entry point): overwrite every
 * instance's state, step counter and stream position, so a parity test can
 * restart the oracle from the device's recorded observation each step
 * (obs == state for every env, write_obs above). Streams keep their keys
 * unless keys is non-NULL. */
void mo_env_set_instances(mo_env* e, const double* state, const int32_t* steps, const uint64_t* keys,
                          const uint64_t* ctrs) {
    for (int i = 0; i < e->n; ++i) {
        if (state) {
            memcpy(e->state + (size_t)i * e->sdim, state + (size_t)i * e->sdim, sizeof(double) * e->sdim);
            write_obs(e, i, e->cur_obs + (size_t)i * e->spec.obs_dim);
        }
        if (steps) e->steps[i] = steps[i];
        if (keys) e->streams[i].key = keys[i];
        if (ctrs) e->streams[i].ctr = ctrs[i];
    }
}

/* ========================================================================= */
/* Rollout: src/rollout.cpp:37-161                                            */
/* ========================================================================= */
int mo_collect_rollouts(const mo_hspec* ah, const double* aflat, const mo_hspec* ch,
                        const double* cflat, mo_env* env, const double* cw, int K, int reps,
                        int T, uint64_t key, uint64_t ctr, mo_batch* out, double* tracker) {
    const mo_envspec* es = &env->spec;
    const int N = K * reps, od = es->obs_dim, ad = es->act_dim, m = es->m;
    if (K < 1 || reps < 1) return fail(MO_ERR, "collect_rollouts: need at least one cluster and one repeat");
    if (N != env->n) return fail(MO_ERR, "collect_rollouts: K * reps (%d) does not match env instances (%d)", N, env->n);
    if (T < 1) return fail(MO_ERR, "collect_rollouts: T must be >= 1");
    const int64_t Pa = mo_hspec_target_count(ah), Pc = mo_hspec_target_count(ch);
    const int64_t mlp_a = mo_mlp_param_count(&ah->target);
    double* theta = (double*)malloc(sizeof(double) * Pa * K);
    double* phi = (double*)malloc(sizeof(double) * Pc * K);
    for (int c = 0; c < K; ++c) { /* :66-75 */
        int rc = mo_hypernet_forward(ah, aflat, cw + (size_t)c * m, theta + Pa * c);
        if (!rc) rc = mo_hypernet_forward(ch, cflat, cw + (size_t)c * m, phi + Pc * c);
        if (rc) { free(theta); free(phi); return rc; }
    }
    mo_rng root = {key, ctr};
    mlp_work wa, wc;
    work_init(&wa, &ah->target);
    work_init(&wc, &ch->target);
    double fobs[64], act[16], z[16], ls[16], rew[16];
    int rc = MO_OK;
    for (int i = 0; i < N && !rc; ++i) { /* :98-151, thread-count invariant */
        mo_rng stream = mo_rng_split(root, (uint64_t)i);
        const int c = i / reps;
        const double* pol = theta + Pa * c;
        const double* val = phi + Pc * c;
        const double* w = cw + (size_t)c * m;
        for (int k = 0; k < ad; ++k) ls[k] = clampd(pol[mlp_a + k], LOG_STD_MIN, LOG_STD_MAX);
        for (int t = 0; t < T; ++t) {
            const int64_t r = (int64_t)i * T + t;
            const double* o = env->cur_obs + (size_t)i * od;
            memcpy(out->obs + r * od, o, sizeof(double) * od);
            if (!all_finite(pol, Pa) || !all_finite(o, od)) { rc = fail(MO_NUMERIC, "non-finite value in policy params"); break; }
            mlp_forward_cached(&ah->target, pol, o, &wa); /* policy_forward nn.cpp:162-190 */
            const double* mu = wa.preact;
            for (int d = 0; d < ad; ++d) { /* sample_and_logprob nn.cpp:192-202 */
                const double sigma = exp(ls[d]);
                z[d] = mu[d] + sigma * mo_rng_next_gaussian(&stream);
                act[d] = tanh(z[d]);
            }
            memcpy(out->action_pre + r * ad, z, sizeof(double) * ad);
            out->logprob[r] = action_logprob(ad, mu, ls, z);
            mlp_forward_cached(&ch->target, val, o, &wc); /* critic_forward */
            memcpy(out->value + r * m, act_row(&wc, wc.L), sizeof(double) * m);
            double* rw = out->reward + r * m;
            rc = step_instance(env, i, act, rw, out->term + r, out->trunc + r, fobs);
            if (rc) break;
            mlp_forward_cached(&ch->target, val, fobs, &wc);
            memcpy(out->next_value + r * m, act_row(&wc, wc.L), sizeof(double) * m);
            if (tracker) { /* :143-148 */
                double* run = tracker + (size_t)i * m;
                for (int k = 0; k < m; ++k) run[k] += rw[k];
                if (out->term[r] || out->trunc[r])
                    for (int k = 0; k < m; ++k) run[k] = 0.0;
            }
            (void)w;
            (void)rew;
        }
    }
    work_free(&wa);
    work_free(&wc);
    free(theta);
    free(phi);
    return rc;
}

/* ========================================================================= */
/* GAE: src/gae.cpp:26-117                                                    */
/* ========================================================================= */
int mo_gae(int N, int T, int m, const double* reward, const double* value, const double* next_value,
           const uint8_t* term, const uint8_t* trunc, double gamma, double lambda, double* adv,
           double* targets) {
    if (N <= 0 || T <= 0 || m <= 0) return fail(MO_ERR, "gae: batch dimensions must be positive");
    if (!(gamma >= 0.0 && gamma <= 1.0)) return fail(MO_ERR, "gae: gamma must lie in [0, 1], got %f", gamma);
    if (!(lambda >= 0.0 && lambda <= 1.0)) return fail(MO_ERR, "gae: lambda must lie in [0, 1], got %f", lambda);
    double carry[64];
    for (int i = 0; i < N; ++i) {
        for (int k = 0; k < m; ++k) carry[k] = 0.0;
        for (int t = T - 1; t >= 0; --t) {
            const int64_t r = (int64_t)i * T + t;
            const double bootstrap = term[r] ? 0.0 : 1.0;
            const double carry_on = (term[r] || trunc[r]) ? 0.0 : 1.0;
            for (int k = 0; k < m; ++k) {
                const int64_t idx = r * m + k;
                const double delta = reward[idx] + gamma * next_value[idx] * bootstrap - value[idx];
                carry[k] = delta + gamma * lambda * carry_on * carry[k];
                adv[idx] = carry[k];
                targets[idx] = adv[idx] + value[idx];
            }
        }
    }
    return MO_OK;
}
int mo_normalize_scalarize(int N, int T, int m, const double* adv, const double* tw, double* out) {
    const int64_t rows = (int64_t)N * T;
    double mean[64] = {0}, var[64] = {0}, inv[64];
    for (int64_t r = 0; r < rows; ++r)
        for (int k = 0; k < m; ++k) mean[k] += adv[r * m + k];
    for (int k = 0; k < m; ++k) mean[k] /= (double)rows;
    for (int64_t r = 0; r < rows; ++r)
        for (int k = 0; k < m; ++k) {
            const double d = adv[r * m + k] - mean[k];
            var[k] += d * d;
        }
    for (int k = 0; k < m; ++k) inv[k] = 1.0 / (sqrt(var[k] / (double)rows) + 1e-8);
    for (int i = 0; i < N; ++i) {
        const double* w = tw + (size_t)i * m;
        for (int t = 0; t < T; ++t) {
            const int64_t r = (int64_t)i * T + t;
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += w[k] * (adv[r * m + k] - mean[k]) * inv[k];
            out[r] = s;
        }
    }
    return MO_OK;
}

/* ========================================================================= */
/* Losses: src/losses.cpp                                                     */
/* ========================================================================= */
/* group_by_cluster (losses.cpp:21-33): ordered by cluster id, rows kept in
 * minibatch order. Returns order[] (row positions) and group starts. */
static int group_rows(int N, int T, const int32_t* cluster, const int32_t* rows, int n_rows,
                      int32_t** sorted, int32_t** starts, int* ngroups, int32_t** gid) {
    int maxc = 0;
    for (int q = 0; q < n_rows; ++q) {
        if (rows[q] < 0 || rows[q] >= N * T) return fail(MO_ERR, "minibatch row index out of range");
        const int c = cluster[rows[q] / T];
        if (c > maxc) maxc = c;
    }
    int* cnt = (int*)calloc(maxc + 2, sizeof(int));
    for (int q = 0; q < n_rows; ++q) cnt[cluster[rows[q] / T] + 1]++;
    for (int c = 0; c <= maxc; ++c) cnt[c + 1] += cnt[c];
    *sorted = (int32_t*)malloc(sizeof(int32_t) * (n_rows ? n_rows : 1));
    int* pos = (int*)malloc(sizeof(int) * (maxc + 1));
    for (int c = 0; c <= maxc; ++c) pos[c] = cnt[c];
    for (int q = 0; q < n_rows; ++q) {
        const int c = cluster[rows[q] / T];
        (*sorted)[pos[c]++] = rows[q];
    }
    int ng = 0;
    *starts = (int32_t*)malloc(sizeof(int32_t) * (maxc + 2));
    *gid = (int32_t*)malloc(sizeof(int32_t) * (maxc + 1));
    for (int c = 0; c <= maxc; ++c)
        if (cnt[c + 1] > cnt[c]) {
            (*starts)[ng] = cnt[c];
            (*gid)[ng] = c;
            ng++;
        }
    (*starts)[ng] = n_rows;
    *ngroups = ng;
    free(cnt);
    free(pos);
    return MO_OK;
}

int mo_actor_loss(const mo_hspec* h, const double* flat, int N, int T, const double* obs,
                  const double* action_pre, const double* logprob_old, const double* tw,
                  const int32_t* cluster, const int32_t* rows, int n_rows, const double* sadv,
                  double clip_eps, double ent, double* loss_out, double* gflat) {
    /* losses.cpp:46-137 */
    if (n_rows <= 0) return fail(MO_ERR, "minibatch has no rows");
    if (!h->has_log_std) return fail(MO_ERR, "actor_loss: hypernet target must be a policy");
    if (!(clip_eps > 0.0)) return fail(MO_ERR, "actor_loss: clip_eps must be positive");
    const mo_mlp* net = &h->target;
    const int od = net->sizes[0], ad = net->sizes[net->n_sizes - 1];
    const int64_t mlp_n = mo_mlp_param_count(net), pol_n = mo_hspec_target_count(h);
    const double inv_B = 1.0 / (double)n_rows;
    memset(gflat, 0, sizeof(double) * mo_hspec_param_count(h));
    int32_t *sorted, *starts, *gid;
    int ng;
    int rc = group_rows(N, T, cluster, rows, n_rows, &sorted, &starts, &ng, &gid);
    if (rc) return rc;
    double* theta = (double*)malloc(sizeof(double) * pol_n);
    double* gth = (double*)malloc(sizeof(double) * pol_n);
    mlp_work wk;
    work_init(&wk, net);
    double loss = 0.0, ls[16], gmu[16];
    for (int g = 0; g < ng && !rc; ++g) {
        const int first = sorted[starts[g]] / T;
        const double* w = tw + (size_t)first * h->m;
        rc = mo_hypernet_forward(h, flat, w, theta);
        if (rc) break;
        memset(gth, 0, sizeof(double) * pol_n);
        for (int d = 0; d < ad; ++d) ls[d] = clampd(theta[mlp_n + d], LOG_STD_MIN, LOG_STD_MAX);
        for (int q = starts[g]; q < starts[g + 1]; ++q) {
            const int r = sorted[q];
            mlp_forward_cached(net, theta, obs + (size_t)r * od, &wk);
            const double* mu = wk.preact;
            const double* z = action_pre + (size_t)r * ad;
            const double lp_new = action_logprob(ad, mu, ls, z);
            const double ratio = exp(lp_new - logprob_old[r]);
            if (!isfinite(ratio)) { rc = fail(MO_NUMERIC, "actor_loss: non-finite ratio at row %d", r); break; }
            const double adv = sadv[r];
            const double unclipped = ratio * adv;
            const double clipped = clampd(ratio, 1.0 - clip_eps, 1.0 + clip_eps) * adv;
            const double mn = clipped < unclipped ? clipped : unclipped;
            loss += -mn * inv_B;
            loss -= ent * gaussian_entropy(ad, ls) * inv_B;
            const double glp = unclipped <= clipped ? -ratio * adv * inv_B : 0.0;
            for (int d = 0; d < ad; ++d) {
                const double sigma = exp(ls[d]);
                const double zn = (z[d] - mu[d]) / sigma;
                gmu[d] = glp * zn / sigma;
                const double raw = theta[mlp_n + d];
                if (raw >= LOG_STD_MIN && raw <= LOG_STD_MAX) {
                    gth[mlp_n + d] += glp * (zn * zn - 1.0);
                    gth[mlp_n + d] -= ent * inv_B;
                }
            }
            mlp_backward(net, theta, &wk, gmu, 1, gth, NULL);
        }
        if (!rc) rc = mo_hypernet_backward(h, flat, w, gth, gflat);
    }
    *loss_out = loss;
    work_free(&wk);
    free(theta);
    free(gth);
    free(sorted);
    free(starts);
    free(gid);
    return rc;
}

int mo_critic_loss(const mo_hspec* h, const double* flat, int N, int T, const double* obs,
                   const double* tw, const int32_t* cluster, const int32_t* rows, int n_rows,
                   const double* targets, double* loss_out, double* gflat) {
    /* losses.cpp:139-189 */
    if (n_rows <= 0) return fail(MO_ERR, "minibatch has no rows");
    if (h->has_log_std) return fail(MO_ERR, "critic_loss: hypernet target must be a value net");
    const mo_mlp* net = &h->target;
    const int od = net->sizes[0], m = net->sizes[net->n_sizes - 1];
    const int64_t mlp_n = mo_mlp_param_count(net);
    const double inv_B = 1.0 / (double)n_rows;
    memset(gflat, 0, sizeof(double) * mo_hspec_param_count(h));
    int32_t *sorted, *starts, *gid;
    int ng;
    int rc = group_rows(N, T, cluster, rows, n_rows, &sorted, &starts, &ng, &gid);
    if (rc) return rc;
    double* phi = (double*)malloc(sizeof(double) * mlp_n);
    double* gphi = (double*)malloc(sizeof(double) * mlp_n);
    mlp_work wk;
    work_init(&wk, net);
    double loss = 0.0, gout[64];
    for (int g = 0; g < ng && !rc; ++g) {
        const int first = sorted[starts[g]] / T;
        const double* w = tw + (size_t)first * h->m;
        rc = mo_hypernet_forward(h, flat, w, phi);
        if (rc) break;
        memset(gphi, 0, sizeof(double) * mlp_n);
        for (int q = starts[g]; q < starts[g + 1]; ++q) {
            const int r = sorted[q];
            mlp_forward_cached(net, phi, obs + (size_t)r * od, &wk);
            const double* v = act_row(&wk, wk.L);
            const double* tg = targets + (size_t)r * m;
            for (int k = 0; k < m; ++k) {
                const double e = v[k] - tg[k];
                loss += e * e * inv_B;
                gout[k] = 2.0 * e * inv_B;
            }
            mlp_backward(net, phi, &wk, gout, 0, gphi, NULL);
        }
        rc = mo_hypernet_backward(h, flat, w, gphi, gflat);
    }
    *loss_out = loss;
    work_free(&wk);
    free(phi);
    free(gphi);
    free(sorted);
    free(starts);
    free(gid);
    return rc;
}

/* ========================================================================= */
/* Adam: src/adam.cpp:8-26                                                    */
/* ========================================================================= */
int mo_adam(int64_t n, double* p, const double* g, double* m1, double* m2, int64_t* step, double lr) {
    *step += 1;
    const double bc1 = 1.0 - pow(0.9, (double)*step);
    const double bc2 = 1.0 - pow(0.999, (double)*step);
    for (int64_t i = 0; i < n; ++i) {
        const double gi = g[i];
        m1[i] = 0.9 * m1[i] + (1.0 - 0.9) * gi;
        m2[i] = 0.999 * m2[i] + (1.0 - 0.999) * gi * gi;
        const double mhat = m1[i] / bc1;
        const double vhat = m2[i] / bc2;
        p[i] -= lr * mhat / (sqrt(vhat) + 1e-8);
    }
    return MO_OK;
}

/* ========================================================================= */
/* Train iteration: src/train.cpp:55-229                                      */
/* ========================================================================= */
struct mo_trainer {
    mo_train_cfg cfg;
    mo_envspec es;
    mo_hspec ah, ch;
    mo_rng root;
    double *ap, *cp;               /* flat params */
    double *am1, *am2, *cm1, *cm2; /* Adam moments (flat; blocks share layout) */
    int64_t astep[3], cstep[3];
    mo_env* env;
    double* tracker;
    int32_t* perm;
    int64_t rows;
    mo_batch b;
    double *adv, *tgt, *sadv, *clusters, *tw;
    int32_t* cluster_of;
};

static void make_specs(const mo_train_cfg* c, const mo_envspec* es, mo_hspec* a, mo_hspec* cr) {
    /* config.cpp:59-83 (HypernetArch::actor_spec / critic_spec) */
    memset(a, 0, sizeof(*a));
    a->m = es->m;
    a->F = c->F;
    a->n_feat_hidden = c->n_feat_hidden;
    for (int i = 0; i < c->n_feat_hidden; ++i) a->feat_hidden[i] = c->feat_hidden[i];
    *cr = *a;
    a->target.n_sizes = 0;
    a->target.sizes[a->target.n_sizes++] = es->obs_dim;
    for (int i = 0; i < c->n_actor_hidden; ++i) a->target.sizes[a->target.n_sizes++] = c->actor_hidden[i];
    a->target.sizes[a->target.n_sizes++] = es->act_dim;
    a->target.out_tanh = 1;
    a->has_log_std = 1;
    cr->target.n_sizes = 0;
    cr->target.sizes[cr->target.n_sizes++] = es->obs_dim;
    for (int i = 0; i < c->n_critic_hidden; ++i) cr->target.sizes[cr->target.n_sizes++] = c->critic_hidden[i];
    cr->target.sizes[cr->target.n_sizes++] = es->m;
    cr->target.out_tanh = 0;
    cr->has_log_std = 0;
}

mo_trainer* mo_trainer_create(const mo_train_cfg* cfg) {
    mo_trainer* t = (mo_trainer*)calloc(1, sizeof(mo_trainer));
    t->cfg = *cfg;
    if (mo_env_spec(cfg->env_kind, &t->es)) { free(t); return NULL; }
    if (cfg->N % cfg->K != 0) { fail(MO_ERR, "K must divide N"); free(t); return NULL; }
    make_specs(cfg, &t->es, &t->ah, &t->ch);
    t->root = mo_rng_seed(cfg->seed);
    const int64_t na = mo_hspec_param_count(&t->ah), nc = mo_hspec_param_count(&t->ch);
    t->ap = (double*)malloc(sizeof(double) * na);
    t->cp = (double*)malloc(sizeof(double) * nc);
    mo_rng ai = mo_rng_split(t->root, 0xA1), ci = mo_rng_split(t->root, 0xA2); /* train.cpp:67-70 */
    mo_init_hypernet(&t->ah, ai.key, ai.ctr, t->ap);
    mo_init_hypernet(&t->ch, ci.key, ci.ctr, t->cp);
    t->am1 = (double*)calloc(na, sizeof(double));
    t->am2 = (double*)calloc(na, sizeof(double));
    t->cm1 = (double*)calloc(nc, sizeof(double));
    t->cm2 = (double*)calloc(nc, sizeof(double));
    t->env = mo_env_create(cfg->env_kind, cfg->N);
    mo_rng er = mo_rng_split(t->root, 0xE0); /* train.cpp:74-75 */
    mo_env_reset(t->env, er.key, er.ctr, NULL);
    const int m = t->es.m;
    t->tracker = (double*)calloc((size_t)cfg->N * m, sizeof(double));
    t->rows = (int64_t)cfg->N * cfg->T;
    t->perm = (int32_t*)malloc(sizeof(int32_t) * t->rows);
    for (int64_t i = 0; i < t->rows; ++i) t->perm[i] = (int32_t)i; /* :112-114 */
    const int64_t R = t->rows;
    t->b.obs = (double*)calloc(R * t->es.obs_dim, sizeof(double));
    t->b.action_pre = (double*)calloc(R * t->es.act_dim, sizeof(double));
    t->b.logprob = (double*)calloc(R, sizeof(double));
    t->b.reward = (double*)calloc(R * m, sizeof(double));
    t->b.value = (double*)calloc(R * m, sizeof(double));
    t->b.next_value = (double*)calloc(R * m, sizeof(double));
    t->b.term = (uint8_t*)calloc(R, 1);
    t->b.trunc = (uint8_t*)calloc(R, 1);
    t->adv = (double*)calloc(R * m, sizeof(double));
    t->tgt = (double*)calloc(R * m, sizeof(double));
    t->sadv = (double*)calloc(R, sizeof(double));
    t->clusters = (double*)calloc((size_t)cfg->K * m, sizeof(double));
    t->tw = (double*)calloc((size_t)cfg->N * m, sizeof(double));
    t->cluster_of = (int32_t*)calloc(cfg->N, sizeof(int32_t));
    return t;
}
void mo_trainer_destroy(mo_trainer* t) {
    if (!t) return;
    free(t->ap); free(t->cp); free(t->am1); free(t->am2); free(t->cm1); free(t->cm2);
    mo_env_destroy(t->env);
    free(t->tracker); free(t->perm);
    free(t->b.obs); free(t->b.action_pre); free(t->b.logprob); free(t->b.reward);
    free(t->b.value); free(t->b.next_value); free(t->b.term); free(t->b.trunc);
    free(t->adv); free(t->tgt); free(t->sadv); free(t->clusters); free(t->tw); free(t->cluster_of);
    free(t);
}
void mo_trainer_specs(const mo_trainer* t, mo_hspec* a, mo_hspec* c) {
    if (a) *a = t->ah;
    if (c) *c = t->ch;
}

static void hyper_adam(const mo_hspec* h, double* p, const double* g, double* m1, double* m2,
                       int64_t* steps, double lr) { /* train.cpp:28-39: feature, M, b */
    const int64_t nf = mo_hspec_feature_count(h), P = mo_hspec_target_count(h);
    const int64_t nM = P * h->F;
    mo_adam(nf, p, g, m1, m2, &steps[0], lr);
    mo_adam(nM, p + nf, g + nf, m1 + nf, m2 + nf, &steps[1], lr);
    mo_adam(P, p + nf + nM, g + nf + nM, m1 + nf + nM, m2 + nf + nM, &steps[2], lr);
}

int mo_trainer_iteration(mo_trainer* t, int it, int max_mb, double* als, double* cls) {
    const mo_train_cfg* c = &t->cfg;
    const int m = t->es.m, K = c->K, N = c->N, T = c->T, reps = N / K;
    mo_rng iter = mo_rng_split(t->root, 0x10000000ULL + (uint64_t)it); /* :120 */
    if (m == 1) {
        for (int k = 0; k < K; ++k) t->clusters[k] = 1.0;
    } else { /* simplex.cpp:55-87 via train.cpp:128-138 */
        mo_rng srng = mo_rng_split(iter, 0);
        const int nd = K - c->kappa;
        for (int k = 0; k < nd; ++k) {
            double* w = t->clusters + (size_t)k * m;
            double sum = 0.0;
            for (int j = 0; j < m; ++j) {
                w[j] = -log(mo_rng_next_open(&srng));
                sum += w[j];
            }
            for (int j = 0; j < m; ++j) w[j] /= sum;
        }
        for (int k = 0; k < c->kappa; ++k) {
            double* w = t->clusters + (size_t)(nd + k) * m;
            for (int j = 0; j < m; ++j) w[j] = (j == k) ? 1.0 : 0.0;
        }
    }
    for (int i = 0; i < N; ++i) {
        t->cluster_of[i] = i / reps;
        memcpy(t->tw + (size_t)i * m, t->clusters + (size_t)(i / reps) * m, sizeof(double) * m);
    }
    mo_rng roll = mo_rng_split(iter, 1);
    int rc = mo_collect_rollouts(&t->ah, t->ap, &t->ch, t->cp, t->env, t->clusters, K, reps, T,
                                 roll.key, roll.ctr, &t->b, t->tracker);
    if (rc) return rc;
    rc = mo_gae(N, T, m, t->b.reward, t->b.value, t->b.next_value, t->b.term, t->b.trunc, c->gamma,
                c->lambda, t->adv, t->tgt);
    if (rc) return rc;
    mo_normalize_scalarize(N, T, m, t->adv, t->tw, t->sadv);
    mo_rng shuf = mo_rng_split(iter, 2);
    const int64_t na = mo_hspec_param_count(&t->ah), nc = mo_hspec_param_count(&t->ch);
    double* ga = (double*)malloc(sizeof(double) * na);
    double* gc = (double*)malloc(sizeof(double) * nc);
    double asum = 0.0, csum = 0.0;
    int done = 0;
    for (int e = 0; e < c->epochs && !rc; ++e) {
        mo_rng_shuffle_i32(&shuf, t->perm, t->rows);
        for (int s = 0; s < c->minibatch_count; ++s) {
            if (max_mb >= 0 && done >= max_mb) break;
            const int lo = (int)(t->rows * s / c->minibatch_count);
            const int hi = (int)(t->rows * (s + 1) / c->minibatch_count);
            if (lo == hi) continue;
            double al = 0.0, cl = 0.0;
            rc = mo_actor_loss(&t->ah, t->ap, N, T, t->b.obs, t->b.action_pre, t->b.logprob, t->tw,
                               t->cluster_of, t->perm + lo, hi - lo, t->sadv, c->clip_eps,
                               c->entropy_coef, &al, ga);
            if (!rc)
                rc = mo_critic_loss(&t->ch, t->cp, N, T, t->b.obs, t->tw, t->cluster_of, t->perm + lo,
                                    hi - lo, t->tgt, &cl, gc);
            if (rc) break;
            if (!isfinite(al) || !isfinite(cl)) {
                rc = fail(MO_NUMERIC, "non-finite loss at iteration %d, epoch %d, minibatch %d", it, e, s);
                break;
            }
            hyper_adam(&t->ah, t->ap, ga, t->am1, t->am2, t->astep, c->actor_lr);
            hyper_adam(&t->ch, t->cp, gc, t->cm1, t->cm2, t->cstep, c->critic_lr);
            asum += al;
            csum += cl;
            done++;
        }
    }
    free(ga);
    free(gc);
    if (als) *als = asum;
    if (cls) *cls = csum;
    return rc;
}
double* mo_trainer_actor_params(mo_trainer* t) { return t->ap; }
double* mo_trainer_critic_params(mo_trainer* t) { return t->cp; }
int32_t* mo_trainer_perm(mo_trainer* t) { return t->perm; }
mo_env* mo_trainer_env(mo_trainer* t) { return t->env; }
const mo_batch* mo_trainer_batch(const mo_trainer* t) { return &t->b; }
const double* mo_trainer_advantages(const mo_trainer* t) { return t->adv; }
const double* mo_trainer_targets(const mo_trainer* t) { return t->tgt; }
const double* mo_trainer_sadv(const mo_trainer* t) { return t->sadv; }
const double* mo_trainer_clusters(const mo_trainer* t) { return t->clusters; }
const double* mo_trainer_tracker(const mo_trainer* t) { return t->tracker; }

/* ========================================================================= */
/* Pareto: src/pareto.cpp                                                     */
/* ========================================================================= */
int mo_dominates(int m, const double* a, const double* b) { /* pareto.cpp:27-36 */
    int strict = 0;
    for (int i = 0; i < m; ++i) {
        if (a[i] < b[i]) return 0;
        if (a[i] > b[i]) strict = 1;
    }
    return strict;
}
static int vec_eq(int m, const double* a, const double* b) {
    for (int i = 0; i < m; ++i)
        if (!(a[i] == b[i])) return 0;
    return 1;
}

/* nondominated_filter (pareto.cpp:38-77) as a mask over the input order. */
int mo_nondominated_mask(int n, int m, const double* pts, uint8_t* mask) {
    if (n <= 0) return MO_OK;
    int* uniq = (int*)malloc(sizeof(int) * n);
    int nu = 0;
    for (int i = 0; i < n; ++i) {
        int dup = 0;
        for (int q = 0; q < nu; ++q)
            if (vec_eq(m, pts + (size_t)uniq[q] * m, pts + (size_t)i * m)) { dup = 1; break; }
        if (!dup) uniq[nu++] = i;
    }
    double* sums = (double*)calloc(n, sizeof(double));
    for (int q = 0; q < nu; ++q) {
        double s = 0.0;
        for (int j = 0; j < m; ++j) s += pts[(size_t)uniq[q] * m + j];
        sums[uniq[q]] = s;
    }
    /* stable sort of uniq by sum descending (insertion sort keeps it stable) */
    int* order = (int*)malloc(sizeof(int) * (nu ? nu : 1));
    for (int q = 0; q < nu; ++q) {
        int v = uniq[q], p = q;
        while (p > 0 && sums[order[p - 1]] < sums[v]) { order[p] = order[p - 1]; --p; }
        order[p] = v;
    }
    int* kept = (int*)malloc(sizeof(int) * (nu ? nu : 1));
    int nk = 0;
    for (int q = 0; q < nu; ++q) {
        const int i = order[q];
        int dom = 0;
        for (int z = 0; z < nk; ++z)
            if (mo_dominates(m, pts + (size_t)kept[z] * m, pts + (size_t)i * m)) { dom = 1; break; }
        if (!dom) kept[nk++] = i;
    }
    memset(mask, 0, n);
    for (int z = 0; z < nk; ++z) mask[kept[z]] = 1;
    free(uniq); free(sums); free(order); free(kept);
    return MO_OK;
}

/* hv_recursive (pareto.cpp:145-189); pts clipped already, n x m, may be
 * modified. Sorting ties are broken by index (std::sort leaves them
 * unspecified; values agree to rounding). */
static int g_sort_dim;
static int g_sort_m;
static int cmp_desc(const void* a, const void* b) {
    const double x = ((const double*)a)[g_sort_dim], y = ((const double*)b)[g_sort_dim];
    return (x > y) ? -1 : (x < y) ? 1 : 0;
}
static double hv_rec(double* pts, int n, const double* ref, int m, int stride) {
    /* nondominated filter first (on the leading m coords of each row) */
    double* buf = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1) * m);
    for (int i = 0; i < n; ++i) memcpy(buf + (size_t)i * m, pts + (size_t)i * stride, sizeof(double) * m);
    uint8_t* mask = (uint8_t*)malloc(n ? n : 1);
    mo_nondominated_mask(n, m, buf, mask);
    int k = 0;
    for (int i = 0; i < n; ++i)
        if (mask[i]) { memmove(buf + (size_t)k * m, buf + (size_t)i * m, sizeof(double) * m); k++; }
    free(mask);
    n = k;
    double vol = 0.0;
    if (n == 0) { free(buf); return 0.0; }
    if (m == 1) {
        double best = ref[0];
        for (int i = 0; i < n; ++i) best = buf[i] > best ? buf[i] : best;
        free(buf);
        return best - ref[0];
    }
    g_sort_dim = (m == 2) ? 0 : m - 1;
    g_sort_m = m;
    qsort(buf, n, sizeof(double) * m, cmp_desc);
    if (m == 2) {
        double area = 0.0, yprev = ref[1];
        for (int i = 0; i < n; ++i) {
            area += (buf[(size_t)i * m] - ref[0]) * (buf[(size_t)i * m + 1] - yprev);
            yprev = buf[(size_t)i * m + 1];
        }
        free(buf);
        return area;
    }
    double* active = (double*)malloc(sizeof(double) * (size_t)n * (m - 1));
    int na = 0, i = 0;
    while (i < n) {
        const double ztop = buf[(size_t)i * m + m - 1];
        while (i < n && buf[(size_t)i * m + m - 1] == ztop) {
            memcpy(active + (size_t)na * (m - 1), buf + (size_t)i * m, sizeof(double) * (m - 1));
            na++;
            i++;
        }
        const double zbot = (i < n) ? buf[(size_t)i * m + m - 1] : ref[m - 1];
        const double height = ztop - zbot;
        if (height > 0.0) vol += height * hv_rec(active, na, ref, m - 1, m - 1);
    }
    free(active);
    free(buf);
    return vol;
}

static double* clip_points(int n, int m, const double* pts, const double* ref, int* nout, int* clipped) {
    /* pareto.cpp:191-205 */
    double* out = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1) * m);
    int k = 0, c = 0;
    for (int i = 0; i < n; ++i) {
        int ok = 1;
        for (int j = 0; j < m; ++j)
            if (pts[(size_t)i * m + j] < ref[j]) { ok = 0; break; }
        if (ok) memcpy(out + (size_t)(k++) * m, pts + (size_t)i * m, sizeof(double) * m);
        else c++;
    }
    *nout = k;
    if (clipped) *clipped = c;
    return out;
}

int mo_hypervolume_exact(int n, int m, const double* pts, const double* ref, double* value, int* clipped) {
    int k;
    double* c = clip_points(n, m, pts, ref, &k, clipped);
    *value = k ? hv_rec(c, k, ref, m, m) : 0.0;
    free(c);
    return MO_OK;
}

int mo_hypervolume_mc(int n, int m, const double* pts, const double* ref, uint64_t samples,
                      uint64_t key, uint64_t ctr, double* value, double* se, uint64_t* hits) {
    /* pareto.cpp:236-277 */
    if (samples == 0) return fail(MO_ERR, "hypervolume_mc: samples must be > 0");
    int k;
    double* p = clip_points(n, m, pts, ref, &k, NULL);
    *value = 0.0;
    if (se) *se = 0.0;
    if (hits) *hits = 0;
    if (k == 0) { free(p); return MO_OK; }
    double hi[64], x[64];
    for (int j = 0; j < m; ++j) {
        hi[j] = ref[j];
        for (int i = 0; i < k; ++i) hi[j] = p[(size_t)i * m + j] > hi[j] ? p[(size_t)i * m + j] : hi[j];
    }
    double box = 1.0;
    for (int j = 0; j < m; ++j) box *= hi[j] - ref[j];
    if (box == 0.0) { free(p); return MO_OK; }
    mo_rng r = {key, ctr};
    uint64_t covered = 0;
    for (uint64_t s = 0; s < samples; ++s) {
        for (int j = 0; j < m; ++j) x[j] = ref[j] + (hi[j] - ref[j]) * mo_rng_next_double(&r);
        for (int i = 0; i < k; ++i) {
            int inside = 1;
            for (int j = 0; j < m; ++j)
                if (x[j] > p[(size_t)i * m + j]) { inside = 0; break; }
            if (inside) { ++covered; break; }
        }
    }
    const double frac = (double)covered / (double)samples;
    if (se) *se = box * sqrt(frac * (1.0 - frac) / (double)samples);
    *value = box * frac;
    if (hits) *hits = covered;
    free(p);
    return MO_OK;
}

int mo_hypervolume_detailed(int n, int m, const double* pts, const double* ref, uint64_t samples,
                            uint64_t seed, double* value, double* se, int* exact, int* clipped) {
    /* pareto.cpp:209-230 */
    int cl = 0, k;
    double* c = clip_points(n, m, pts, ref, &k, &cl);
    if (clipped) *clipped = cl;
    *value = 0.0;
    if (se) *se = 0.0;
    if (exact) *exact = 1;
    if (k == 0) { free(c); return MO_OK; }
    if (m <= 4) {
        *value = hv_rec(c, k, ref, m, m);
    } else {
        mo_rng r = mo_rng_seed(seed);
        int rc = mo_hypervolume_mc(k, m, c, ref, samples, r.key, r.ctr, value, se, NULL);
        if (exact) *exact = 0;
        free(c);
        return rc;
    }
    free(c);
    return MO_OK;
}

/* ---- simplex_grid (simplex.cpp:88-117): compositions of `res` into m parts,
 * first coordinate from res down to 0, recursively; entries k / res. */
static void grid_rec_c(int m, int res, int remaining, int depth, double* prefix, double* out, int64_t* n) {
    if (depth == m - 1) {
        prefix[depth] = (double)remaining / res;
        memcpy(out + (size_t)(*n) * m, prefix, sizeof(double) * m);
        (*n)++;
        return;
    }
    for (int k = remaining; k >= 0; --k) {
        prefix[depth] = (double)k / res;
        grid_rec_c(m, res, remaining - k, depth + 1, prefix, out, n);
    }
}
int64_t mo_simplex_grid_size(int m, int res) {
    int64_t r = 1;
    for (int i = 1; i <= m - 1; ++i) r = r * (res + i) / i;
    return r;
}
int mo_simplex_grid(int m, int res, double* out) {
    if (m < 1 || res < 1) return fail(MO_ERR, "simplex_grid: bad arguments");
    if (m == 1) { out[0] = 1.0; return MO_OK; }
    double prefix[64];
    int64_t n = 0;
    grid_rec_c(m, res, res, 0, prefix, out, &n);
    return MO_OK;
}

/* ---- evaluate_params / eval_point (evaluate.cpp:17-101): for every simplex
 * grid point g, a fresh env of `episodes` instances reset from
 * Rng(key).split(g); the deterministic policy (tanh of the mean, the
 * target MLP's output activation) steps the still-alive instances for up to
 * max_episode_steps; first-episode undiscounted returns, averaged. Dead
 * instances are stepped too (their own streams only) and masked out. */
int mo_evaluate_params(const mo_hspec* h, const double* flat, int env_kind, int res, int episodes,
                       uint64_t key, double* w_out, double* mean_out, int64_t* n_points) {
    mo_envspec es;
    if (mo_env_spec(env_kind, &es)) return MO_ERR;
    if (episodes < 1) return fail(MO_ERR, "evaluate: episodes_per_point must be >= 1");
    if (h->m != es.m) return fail(MO_ERR, "evaluate: hypernet trade-off dim does not match env");
    if (es.m > 1 && res < 1) return fail(MO_ERR, "evaluate: grid_resolution must be >= 1");
    const int64_t ng = es.m == 1 ? 1 : mo_simplex_grid_size(es.m, res);
    if (es.m == 1) w_out[0] = 1.0; else mo_simplex_grid(es.m, res, w_out);
    const int64_t P = mo_hspec_target_count(h);
    double* theta = (double*)malloc(sizeof(double) * P);
    double* obs = (double*)malloc(sizeof(double) * (size_t)episodes * es.obs_dim);
    double* act = (double*)calloc((size_t)episodes * es.act_dim, sizeof(double));
    double* nobs = (double*)malloc(sizeof(double) * (size_t)episodes * es.obs_dim);
    double* rew = (double*)malloc(sizeof(double) * (size_t)episodes * es.m);
    uint8_t* term = (uint8_t*)malloc(episodes);
    uint8_t* trunc = (uint8_t*)malloc(episodes);
    uint8_t* alive = (uint8_t*)malloc(episodes);
    double* tot = (double*)malloc(sizeof(double) * (size_t)episodes * es.m);
    int rc = MO_OK;
    for (int64_t g = 0; g < ng && rc == MO_OK; ++g) {
        rc = mo_hypernet_forward(h, flat, w_out + (size_t)g * es.m, theta);
        if (rc) break;
        mo_env* env = mo_env_create(env_kind, episodes);
        mo_rng root = {key, 0};
        mo_env_reset(env, mo_rng_split(root, (uint64_t)g).key, 0, NULL);
        for (int i = 0; i < episodes; ++i) alive[i] = 1;
        memset(tot, 0, sizeof(double) * (size_t)episodes * es.m);
        for (int t = 0; t < es.max_steps; ++t) {
            int any = 0;
            mo_env_current_obs(env, obs);
            for (int i = 0; i < episodes; ++i) {
                if (!alive[i]) continue;
                any = 1;
                mo_mlp_forward(&h->target, theta, obs + (size_t)i * es.obs_dim, act + (size_t)i * es.act_dim);
            }
            if (!any) break;
            rc = mo_env_step(env, act, nobs, rew, term, trunc);
            if (rc) break;
            for (int i = 0; i < episodes; ++i) {
                if (!alive[i]) continue;
                for (int k = 0; k < es.m; ++k) tot[(size_t)i * es.m + k] += rew[(size_t)i * es.m + k];
                if (term[i] || trunc[i]) alive[i] = 0;
            }
        }
        for (int k = 0; k < es.m; ++k) {
            double mean = 0.0;
            for (int i = 0; i < episodes; ++i) mean += tot[(size_t)i * es.m + k];
            mean_out[(size_t)g * es.m + k] = mean / (double)episodes;
        }
        mo_env_destroy(env);
    }
    *n_points = ng;
    free(theta); free(obs); free(act); free(nobs); free(rew); free(term); free(trunc); free(alive); free(tot);
    return rc;
}

/* ---- linear_dominance_filter (pareto.cpp:79-139) as a mask over the input:
 * nd = nondominated_filter; |nd| <= 2 or m == 1 -> nd; m == 2 -> upper hull
 * of nd sorted by J1 ascending, collinear points kept (cross > 0 pops);
 * m >= 3 -> a point survives if w.p >= best - 1e-9 max(1, |best|) for some
 * w on simplex_grid(m, 60) (simplex.cpp:108-117; w_j = k_j / 60, dot in
 * coordinate order, simplex.cpp:10-16). */
static const double* g_ldf_pts;
static int cmp_j1_asc(const void* a, const void* b) {
    const double x = g_ldf_pts[(size_t)(*(const int*)a) * 2], y = g_ldf_pts[(size_t)(*(const int*)b) * 2];
    return x < y ? -1 : x > y ? 1 : 0;
}
static void ldf_grid_rec(int m, int res, int remaining, int depth, int* k, const double* nd, int nn,
                         uint8_t* keep) {
    if (depth == m - 1) {
        k[depth] = remaining;
        double best = -INFINITY;
        for (int i = 0; i < nn; ++i) {
            double acc = 0.0;
            for (int j = 0; j < m; ++j) acc += ((double)k[j] / res) * nd[(size_t)i * m + j];
            best = acc > best ? acc : best;
        }
        const double tol = 1e-9 * (fabs(best) > 1.0 ? fabs(best) : 1.0);
        for (int i = 0; i < nn; ++i) {
            double acc = 0.0;
            for (int j = 0; j < m; ++j) acc += ((double)k[j] / res) * nd[(size_t)i * m + j];
            if (acc >= best - tol) keep[i] = 1;
        }
        return;
    }
    for (int v = remaining; v >= 0; --v) {
        k[depth] = v;
        ldf_grid_rec(m, res, remaining - v, depth + 1, k, nd, nn, keep);
    }
}
int mo_linear_dominance_mask(int n, int m, const double* pts, uint8_t* mask) {
    if (n <= 0) return MO_OK;
    if (m < 1) return fail(MO_ERR, "linear_dominance_filter: empty points");
    mo_nondominated_mask(n, m, pts, mask);
    int nn = 0;
    for (int i = 0; i < n; ++i) nn += mask[i] != 0;
    if (nn <= 2 || m == 1) return MO_OK;
    int* idx = (int*)malloc(sizeof(int) * nn);
    double* nd = (double*)malloc(sizeof(double) * (size_t)nn * m);
    for (int i = 0, q = 0; i < n; ++i)
        if (mask[i]) {
            idx[q] = i;
            memcpy(nd + (size_t)q * m, pts + (size_t)i * m, sizeof(double) * m);
            ++q;
        }
    uint8_t* keep = (uint8_t*)calloc(nn, 1);
    if (m == 2) {
        int* order = (int*)malloc(sizeof(int) * nn);
        int* hull = (int*)malloc(sizeof(int) * nn);
        for (int q = 0; q < nn; ++q) order[q] = q;
        g_ldf_pts = nd;
        qsort(order, nn, sizeof(int), cmp_j1_asc);  /* J1 values are distinct in nd */
        int h = 0;
        for (int q = 0; q < nn; ++q) {
            const int id = order[q];
            while (h >= 2) {
                const double* p1 = nd + (size_t)hull[h - 2] * 2;
                const double* p2 = nd + (size_t)hull[h - 1] * 2;
                const double* p3 = nd + (size_t)id * 2;
                const double cross = (p2[0] - p1[0]) * (p3[1] - p2[1]) - (p2[1] - p1[1]) * (p3[0] - p2[0]);
                if (cross > 0.0) --h; else break;
            }
            hull[h++] = id;
        }
        for (int q = 0; q < h; ++q) keep[hull[q]] = 1;
        free(order);
        free(hull);
    } else {
        int k[64];
        ldf_grid_rec(m, 60, 60, 0, k, nd, nn, keep);
    }
    for (int q = 0; q < nn; ++q) mask[idx[q]] = keep[q];
    free(keep);
    free(nd);
    free(idx);
    return MO_OK;
}

/* ---- WFG exact hypervolume (any m). New algorithm, not in the reference:
 * hv(S) = sum_k [ inclhv(s_k) - hv(nd(limit(s_k, S[k+1:]))) ] with points
 * sorted by the last objective descending; m == 2 base case is the sweep
 * of pareto.cpp:154-166. Maximisation w.r.t. `ref`. */
static double wfg_hv(double* pts, int n, int m, const double* ref);
static double wfg_2d(double* pts, int n, const double* ref) {
    g_sort_dim = 0;
    qsort(pts, n, sizeof(double) * 2, cmp_desc);
    double area = 0.0, yprev = ref[1];
    for (int i = 0; i < n; ++i) {
        const double y = pts[2 * i + 1];
        if (y > yprev) {
            area += (pts[2 * i] - ref[0]) * (y - yprev);
            yprev = y;
        }
    }
    return area;
}
static int nd_compact(double* pts, int n, int m) {
    /* keep points not weakly dominated by another kept point (dups collapse) */
    uint8_t* keep = (uint8_t*)malloc(n ? n : 1);
    for (int i = 0; i < n; ++i) keep[i] = 1;
    for (int i = 0; i < n; ++i) {
        if (!keep[i]) continue;
        for (int j = 0; j < n; ++j) {
            if (i == j || !keep[j]) continue;
            /* does j weakly dominate i ? */
            int ge = 1;
            for (int d = 0; d < m; ++d)
                if (pts[(size_t)j * m + d] < pts[(size_t)i * m + d]) { ge = 0; break; }
            if (ge) { keep[i] = 0; break; }
        }
    }
    int k = 0;
    for (int i = 0; i < n; ++i)
        if (keep[i]) { memmove(pts + (size_t)k * m, pts + (size_t)i * m, sizeof(double) * m); k++; }
    free(keep);
    return k;
}
static double wfg_hv(double* pts, int n, int m, const double* ref) {
    if (n == 0) return 0.0;
    if (m == 2) return wfg_2d(pts, n, ref);
    if (n == 1) {
        double v = 1.0;
        for (int d = 0; d < m; ++d) v *= pts[d] - ref[d];
        return v;
    }
    g_sort_dim = m - 1;
    qsort(pts, n, sizeof(double) * m, cmp_desc);
    double total = 0.0;
    double* lim = (double*)malloc(sizeof(double) * (size_t)n * m);
    for (int k = 0; k < n; ++k) {
        const double* p = pts + (size_t)k * m;
        double incl = 1.0;
        for (int d = 0; d < m; ++d) incl *= p[d] - ref[d];
        int nl = 0;
        for (int q = k + 1; q < n; ++q) {
            const double* s = pts + (size_t)q * m;
            double* o = lim + (size_t)nl * m;
            for (int d = 0; d < m; ++d) o[d] = s[d] < p[d] ? s[d] : p[d];
            nl++;
        }
        nl = nd_compact(lim, nl, m);
        total += incl - wfg_hv(lim, nl, m, ref);
    }
    free(lim);
    return total;
}
int mo_hypervolume_wfg(int n, int m, const double* pts, const double* ref, double* value) {
    int k;
    double* c = clip_points(n, m, pts, ref, &k, NULL);
    k = nd_compact(c, k, m);
    *value = wfg_hv(c, k, m, ref);
    free(c);
    return MO_OK;
}
