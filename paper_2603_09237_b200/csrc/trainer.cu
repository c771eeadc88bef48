// Host orchestration of one MORLAX training iteration on the GPU
// (reference src/train.cpp:118-184): preference sampling -> hypernet
// generation -> fused rollout -> GAE / normalise / scalarise -> epochs x
// minibatches of {actor loss, critic loss through the hypernetwork, Adam}.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "comm.h"
#include "trainer.h"

namespace mb200 {

// ------------------------------------------------------------------ helpers
template <typename T>
static T* dalloc(size_t n) {
    T* p = nullptr;
    if (n == 0) n = 1;
    MB_CUDA(cudaMalloc(&p, n * sizeof(T)));
    // cudaMemset runs asynchronously on the legacy default stream, which does
    // not order against our non-blocking streams: wait for it, or a kernel or
    // copy on another stream can land before the zero fill
    MB_CUDA(cudaMemset(p, 0, n * sizeof(T)));
    MB_CUDA(cudaStreamSynchronize(0));
    return p;
}
template <typename T>
static void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

NetDims make_dims(const std::vector<int>& s, bool out_tanh, bool has_log_std) {
    NetDims d{};
    d.L = (int)s.size() - 1;
    if (d.L < 1 || d.L > 8) throw ShapeError("MlpSpec needs at least input and output sizes");
    long off = 0;
    for (int l = 0; l <= d.L; ++l) d.sz[l] = s[l];
    for (int l = 0; l < d.L; ++l) {  // nn.cpp:38-58 flat layout: W (out x in) then b
        d.woff[l] = off;
        d.boff[l] = off + (long)s[l] * s[l + 1];
        off += (long)(s[l] + 1) * s[l + 1];
    }
    d.mlp_n = off;
    d.P = off + (has_log_std ? s[d.L] : 0);
    d.out_tanh = out_tanh;
    d.has_log_std = has_log_std;
    return d;
}

void TrainConfig::validate(int m) const {  // config.cpp:17-45, simplex.cpp:44-53
    if (N < 1) throw ConfigError("trainer.N must be >= 1");
    if (T < 1) throw ConfigError("trainer.T must be >= 1");
    if (!(gamma >= 0.0 && gamma < 1.0)) throw ConfigError("trainer.gamma must lie in [0, 1)");
    if (!(lambda >= 0.0 && lambda <= 1.0)) throw ConfigError("trainer.gae_lambda must lie in [0, 1]");
    if (!(clip_eps > 0.0)) throw ConfigError("trainer.clip_eps must be > 0");
    if (epochs < 1) throw ConfigError("trainer.epochs must be >= 1");
    if (minibatch_count < 1) throw ConfigError("trainer.minibatch_count must be >= 1");
    if (!(actor_lr > 0.0)) throw ConfigError("trainer.actor_lr must be > 0");
    if (!(critic_lr > 0.0)) throw ConfigError("trainer.critic_lr must be > 0");
    if (entropy_coef < 0.0) throw ConfigError("trainer.entropy_coef must be >= 0");
    if (F < 1) throw ConfigError("hypernet.F must be >= 1");
    for (int h : feat_hidden)
        if (h < 1) throw ConfigError("hypernet.feature_hidden sizes must be >= 1");
    for (int h : actor_hidden)
        if (h < 1) throw ConfigError("hypernet.actor_hidden sizes must be >= 1");
    for (int h : critic_hidden)
        if (h < 1) throw ConfigError("hypernet.critic_hidden sizes must be >= 1");
    if (m == 1) {
        if (K != N) throw ConfigError("trainer.K must equal trainer.N when the environment has one objective");
        return;
    }
    if (K <= 1) throw ConfigError("K must be > 1");
    if (N % K != 0)
        throw ConfigError("K must divide N (got K=" + std::to_string(K) + ", N=" + std::to_string(N) + ")");
    if (kappa < 0 || kappa > K) throw ConfigError("kappa must be in [0, K]");
    if (kappa > m) throw ConfigError("kappa must be <= m");
}

// ------------------------------------------------------------------ init kernels
// init_mlp_params (nn.cpp:260-274): one stream, entry e uses word e+1,
// U(-1/sqrt(fan_in), +1/sqrt(fan_in)) for weights and biases alike.
struct InitLayers {
    int L;
    long end[9];
    double bound[9];
};
__global__ void k_init_mlp(float* out, long n, uint64_t key, InitLayers il, long fill_from, float fill) {
    const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (e >= n) return;
    if (e >= fill_from) {
        out[e] = fill;  // policy log-std slots (hypernet.cpp:140-142)
        return;
    }
    int l = 0;
    while (l < il.L - 1 && e >= il.end[l]) ++l;
    const double b = il.bound[l];
    out[e] = (float)uniform_rn(-b, b, rng_word(key, (uint64_t)e + 1));
}
// M ~ N(0, (0.01/sqrt(F))^2): entry i consumes words 2i+1, 2i+2 (Box-Muller)
__global__ void k_init_gauss(float* out, long n, uint64_t key, double sd) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = (float)__dmul_rn(sd, box_muller(rng_word(key, 2 * (uint64_t)i + 1), rng_word(key, 2 * (uint64_t)i + 2)));
}
static InitLayers init_layers(const std::vector<int>& s) {
    InitLayers il{};
    il.L = (int)s.size() - 1;
    long off = 0;
    for (int l = 0; l < il.L; ++l) {
        off += (long)(s[l] + 1) * s[l + 1];
        il.end[l] = off;
        il.bound[l] = 1.0 / std::sqrt((double)s[l]);
    }
    return il;
}

// ------------------------------------------------------------------ profiler
int Profiler::begin(const char* name, double flops, double bytes, cudaStream_t s) {
    if (!on) return -1;
    const std::string key = phase + "/" + name;  // the iteration phase the launch belongs to
    int c = -1;
    for (size_t i = 0; i < cls.size(); ++i)
        if (cls[i].name == key) c = (int)i;
    if (c < 0) {
        cls.push_back(Cls{key});
        c = (int)cls.size() - 1;
    }
    cls[c].flops += flops;
    cls[c].bytes += bytes;
    cls[c].count += 1;
    while (pool.size() < used + 2) {
        cudaEvent_t e;
        MB_CUDA(cudaEventCreate(&e));
        pool.push_back(e);
    }
    Pending p{c, pool[used], pool[used + 1], s};
    used += 2;
    MB_CUDA(cudaEventRecord(p.a, s));
    pending.push_back(p);
    return (int)pending.size() - 1;
}
void Profiler::end(int h, cudaStream_t s) {
    if (h >= 0) MB_CUDA(cudaEventRecord(pending[h].b, s));
}
void Profiler::collect() {
    if (!pending.empty()) timeline.clear();
    for (auto& p : pending) {
        MB_CUDA(cudaEventSynchronize(p.b));
        float ms = 0;
        MB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        cls[p.c].ms += ms;
        float t0 = 0;
        MB_CUDA(cudaEventElapsedTime(&t0, pending[0].a, p.a));
        int sid = -1;
        for (size_t i = 0; i < streams.size(); ++i)
            if (streams[i] == p.s) sid = (int)i;
        if (sid < 0) {
            streams.push_back(p.s);
            sid = (int)streams.size() - 1;
        }
        timeline.push_back(Span{p.c, sid, t0, t0 + ms});
    }
    pending.clear();
    used = 0;
}
void Profiler::reset() {
    pending.clear();
    used = 0;
    cls.clear();
}
Profiler::~Profiler() {
    for (auto e : pool) cudaEventDestroy(e);
}
static Profiler* g_prof = nullptr;  // the active trainer's profiler (launch sites below)
struct ProfScope {
    int h;
    cudaStream_t s;
    ProfScope(const char* n, double f, double b, cudaStream_t s_) : s(s_) {
        h = g_prof ? g_prof->begin(n, f, b, s_) : -1;
    }
    ~ProfScope() {
        if (g_prof) g_prof->end(h, s);
    }
};

// ------------------------------------------------------------------ HyperNet
void HyperNet::init(int m_, int F_, const std::vector<int>& fh, const std::vector<int>& ts, bool out_tanh,
                    bool has_log_std, int G_, Comm* comm_, int Kl_) {
    m = m_;
    F = F_;
    G = G_;
    comm = comm_;
    if (comm && !xs) {
        MB_CUDA(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
        for (auto& e : xev) MB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    world = comm ? comm_world(comm) : 1;
    rank = comm ? comm_rank(comm) : 0;
    Kl = comm ? Kl_ : G_;
    fsz.clear();
    fsz.push_back(m);
    for (int h : fh) fsz.push_back(h);
    fsz.push_back(F);
    nf = 0;
    fwoff.clear();
    fboff.clear();
    for (size_t l = 0; l + 1 < fsz.size(); ++l) {
        fwoff.push_back(nf);
        fboff.push_back(nf + (long)fsz[l] * fsz[l + 1]);
        nf += (long)(fsz[l] + 1) * fsz[l + 1];
    }
    tgt = make_dims(ts, out_tanh, has_log_std);
    P = tgt.P;
    ld = (P + 7) / 8 * 8;
    n = nf + P * F + P;
    shard_rows(P, world, rank, &S, &row_lo, &row_hi);
    if (comm && (nf % 4 || (P * F) % 4))
        throw ShapeError("sharded optimizer: feature-map and M block sizes must be multiples of 4");
    const long pad = comm ? (long)world * S - P : 0;  // b is all-gathered in place (rank r at b + r S)
    p = dalloc<float>(n + pad);
    g = dalloc<float>(n + pad);
    m1 = dalloc<float>(n + pad);
    m2 = dalloc<float>(n + pad);
    fact.assign(fsz.size(), nullptr);
    int maxw = 0;
    for (size_t l = 0; l < fsz.size(); ++l) {
        fact[l] = dalloc<float>((size_t)G * fsz[l]);
        maxw = std::max(maxw, fsz[l]);
    }
    const int Lf = (int)fsz.size() - 1;
    if (Lf < 1 || Lf > kMaxFeatLayers) throw ConfigError("feature map must have 1.." + std::to_string(kMaxFeatLayers) + " layers");
    fgz.assign(Lf, nullptr);
    fd = FeatDims{};
    fd.L = Lf;
    for (int l = 0; l <= Lf; ++l) {
        fd.sz[l] = fsz[l];
        fd.act[l] = fact[l];
    }
    for (int l = 0; l < Lf; ++l) {
        fgz[l] = dalloc<float>((size_t)G * fsz[l + 1]);
        fd.gz[l] = fgz[l];
        fd.woff[l] = fwoff[l];
        fd.boff[l] = fboff[l];
    }
    theta = dalloc<float>((size_t)G * ld);
    theta16 = dalloc<uint16_t>((size_t)G * ld);
    gtheta = dalloc<float>((size_t)G * ld);
    gf = dalloc<float>((size_t)G * F);
    splits = (int)std::min<long>(64, std::max<long>(1, P / 1024));
    parts = dalloc<float>((size_t)splits * G * F);
    std::vector<int> bounds(splits + 1);
    for (int z = 0; z <= splits; ++z) bounds[z] = (int)(P * z / splits);
    d_split_bounds = dalloc<int>(splits + 1);
    MB_CUDA(cudaMemcpy(d_split_bounds, bounds.data(), sizeof(int) * (splits + 1), cudaMemcpyHostToDevice));
    MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
    // images (zero-filled: padding stays zero forever)
    auto mk = [](int R, int C, long gs, int groups) {
        Img im;
        im.R = R;
        im.C = C;
        im.gs = gs;
        im.p = dalloc<uint8_t>((size_t)(groups > 1 ? gs * groups : img_bytes(R, C)));
        return im;
    };
    mimg = mk((int)(comm ? world * S : P), F, 0, 1);  // rows [r S, r S + S): rank r's all-gather block
    mimg.R = (int)P;
    fimg = mk(G, F, 0, 1);
    if (comm) {
        gsend = dalloc<float>((size_t)world * Kl * S);
        grecv = dalloc<float>((size_t)world * Kl * S);
        gshard = mk(G, (int)S, 0, 1);
        fall = mk(G, F, 0, 1);
    }
    gimg = mk(G, (int)P, 0, 1);
    wimg_off.clear();
    long ws = 0;
    for (int l = 0; l < tgt.L; ++l) {
        wimg_off.push_back(ws);
        ws += img_bytes(tgt.sz[l + 1], tgt.sz[l]);
    }
    wimg.R = wimg.C = 0;
    wimg.gs = ws;
    wimg.p = dalloc<uint8_t>((size_t)ws * G);
    // 128-aligned K splits of P for the df GEMM (split-K over tcgen05 CTAs)
    const int kchunks = (int)((P + 127) / 128);
    static const int max_splits = [] {  // MORLAX_DF_SPLITS: A/B of the split-K width
        const char* e = std::getenv("MORLAX_DF_SPLITS");
        return e ? std::max(1, std::atoi(e)) : 64;  // 148 -> 64: -0.2 ms / iteration (fewer partials)
    }();
    splits = std::max(1, std::min(kchunks, max_splits));
    std::vector<int> kb(splits + 1);
    for (int z = 0; z <= splits; ++z) kb[z] = (int)std::min<long>(P, 128L * ((long)kchunks * z / splits));
    kb[splits] = (int)(((P + 127) / 128) * 128);
    cudaFree(d_split_bounds);
    d_split_bounds = dalloc<int>(splits + 1);
    MB_CUDA(cudaMemcpy(d_split_bounds, kb.data(), sizeof(int) * (splits + 1), cudaMemcpyHostToDevice));
    MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
    cudaFree(parts);
    parts = dalloc<float>((size_t)splits * G * F);
}

void HyperNet::free_all() {
    if (xs) cudaStreamDestroy(xs);
    for (auto& e : xev)
        if (e) cudaEventDestroy(e);
    xs = nullptr;
    xev[0] = xev[1] = nullptr;
    dfree(gshard.p); dfree(fall.p); dfree(gsend); dfree(grecv);
    dfree(p); dfree(g); dfree(m1); dfree(m2);
    for (auto& a : fact) dfree(a);
    for (auto& a : fgz) dfree(a);
    dfree(theta); dfree(theta16); dfree(gtheta); dfree(gf); dfree(parts); dfree(d_split_bounds);
    dfree(mimg.p); dfree(fimg.p); dfree(gimg.p); dfree(wimg.p);
}

void HyperNet::init_params(uint64_t key, cudaStream_t s) {  // hypernet.cpp:124-145
    const uint64_t kf = split_key(key, 0), km = split_key(key, 1), kb = split_key(key, 2);
    InitLayers fl = init_layers(fsz);
    k_init_mlp<<<(int)((nf + 255) / 256), 256, 0, s>>>(p, nf, kf, fl, nf, 0.f);
    MB_LAUNCH();
    const long nM = P * F;
    k_init_gauss<<<(int)((nM + 255) / 256), 256, 0, s>>>(p + nf, nM, km, 0.01 / std::sqrt((double)F));
    MB_LAUNCH();
    std::vector<int> ts(tgt.sz, tgt.sz + tgt.L + 1);
    InitLayers tl = init_layers(ts);
    k_init_mlp<<<(int)((P + 255) / 256), 256, 0, s>>>(p + nf + nM, P, kb, tl, tgt.mlp_n, -1.f);
    MB_LAUNCH();
    MB_CUDA(cudaMemsetAsync(m1, 0, n * sizeof(float), s));
    MB_CUDA(cudaMemsetAsync(m2, 0, n * sizeof(float), s));
    steps[0] = steps[1] = steps[2] = 0;
    to_img(p + nf, F, 0, (int)P, F, mimg, 1, s);
}

// algorithmic bytes of one tcgen05 GEMM of this dataflow: the bf16 operand
// images (B once per group for the row-grouped GEMMs), the tanh' operand,
// and the output (bf16 image or fp32, per group for the K-grouped ones)
static double igemm_bytes(const IGemm& d) {
    const double M = d.M, N = d.N, K = d.K, Z = d.Z;
    double b = 2.0 * M * K;                        // A
    b += 2.0 * N * K * (d.gmode == 1 ? Z : 1.0);   // B (per group weights when rows are grouped)
    if (d.act == 2) b += 2.0 * M * N;              // tanh' operand image
    const double outs = M * N * (d.gmode == 2 ? Z : (d.gmode == 0 ? Z : 1.0));
    if (d.o_mode) b += 2.0 * outs;
    if (d.C) {
        double bf = 0;  // columns written in bf16 only
        for (int k = 0; d.C16 && k < d.nbf; ++k) bf += (double)(d.bf_hi[k] - d.bf_lo[k]);
        b += (d.C16 ? 2.0 * outs : 0.0) + 4.0 * outs * (1.0 - bf / N);
    }
    return b;
}
static void igemm(const char* cls, const IGemm& d, cudaStream_t s) {
    const double f = 2.0 * d.M * d.N * d.K * (d.gmode == 0 ? d.Z : 1);
    ProfScope p(cls, f, igemm_bytes(d), s);
    img_gemm(d, s);
}

// feature map f(w) for all G groups (SIMT: K = m is tiny), then on the tensor
// cores theta[g][p] = b[p] + sum_k M[p][k] f[g][k] (hypernet.cpp:73-88) for
// this rank's clusters [g0, g0+ng) only (theta rows keep global indices).
void HyperNet::forward(const float* w, int g0, int ng, cudaStream_t s, bool upd) {
    HyperNet* self = this;
    forward_multi(&self, 1, w, g0, ng, s, upd);
}

// the forward of one or two hypernetworks (actor and critic) in lockstep:
// each stage is one launch covering both
void HyperNet::forward_multi(HyperNet* const* hs, int nh, const float* w, int g0, int ng, cudaStream_t s,
                             bool upd) {
    {
        double fl = 0;
        FeatJob jobs[2];
        for (int k = 0; k < nh; ++k) {
            HyperNet& h = *hs[k];
            for (size_t l = 0; l + 1 < h.fsz.size(); ++l) fl += 2.0 * h.G * h.fsz[l] * h.fsz[l + 1];
            h.w_last = w;
            h.fg0 = g0;
            h.fng = ng;
            jobs[k] = FeatJob{&h.fd, h.p, w, h.G, h.fimg, g0, ng, nullptr, 0, nullptr};
        }
        ProfScope ps("feature_fwd", fl, 0, s);
        feature_forward_multi(jobs, nh, s);  // tanh MLP incl. tanh output (hypernet.cpp:10-17)
    }
    {
        IGemm ds[2];
        double fl = 0, by = 0;
        for (int k = 0; k < nh; ++k) {
            HyperNet& h = *hs[k];
            IGemm& d = ds[k];  // theta[g][p] = b[p] + sum_k f[g][k] M[p][k]: rows = clusters
            d.A = h.fimg; d.a_view = 0;  // (m = g, k = f)
            d.B = h.mimg; d.b_view = 0;  // (n = p, k = f)
            d.M = ng; d.N = (int)h.P; d.K = h.F;
            d.bias = h.p + h.nf + h.P * h.F; d.bias_mode = 1;
            d.C = h.theta + (long)g0 * h.ld; d.cm = h.ld; d.cn = 1;
            h.theta16_last = upd;
            if (upd) {  // the hidden layers' weights only feed the bf16 weight packing
                d.C16 = h.theta16 + (long)g0 * h.ld;
                d.c16m = h.ld;
                for (int l = 0; l + 1 < h.tgt.L && d.nbf < 7; ++l) {
                    d.bf_lo[d.nbf] = h.tgt.woff[l];
                    d.bf_hi[d.nbf] = h.tgt.woff[l] + (long)h.tgt.sz[l] * h.tgt.sz[l + 1];
                    ++d.nbf;
                }
            }
            fl += 2.0 * d.M * d.N * d.K;
            by += igemm_bytes(d);
        }
        ProfScope ps("hyper_theta", fl, by, s);
        img_gemm_batch(ds, nh, s);
    }
    for (int k = 0; k < nh; ++k) {
        HyperNet& h = *hs[k];
        if (upd && (h.wmap_g0 != g0 || h.wmap_ng != ng)) {  // tensor maps over theta16 (once per cluster range)
            h.wmap.assign(h.tgt.L, CUtensorMap{});
            h.wmap_ok.assign(h.tgt.L, 0);
            static const bool tma = [] {
                const char* e = std::getenv("MORLAX_WEIGHT_TMA");  // "0": pack every layer (A/B, tests)
                return !(e && e[0] == '0');
            }();
            for (int l = 0; tma && l < h.tgt.L; ++l)
                h.wmap_ok[l] = make_weight_map(&h.wmap[l], h.theta16 + (long)g0 * h.ld + h.tgt.woff[l],
                                               h.tgt.sz[l + 1], h.tgt.sz[l], h.ld, ng);
            h.wmap_g0 = g0;
            h.wmap_ng = ng;
        }
        PackDims pd;  // generated weights of this rank's clusters -> per-layer bf16 images
        long units = 0;
        for (int l = 0; l < h.tgt.L; ++l) {
            if (upd && h.wmap_ok[l]) continue;  // read through its tensor map instead
            const int q = pd.L++;
            pd.in[q] = h.tgt.sz[l];
            pd.out[q] = h.tgt.sz[l + 1];
            pd.woff[q] = h.tgt.woff[l];
            pd.ioff[q] = h.wimg_off[l];
            pd.ustart[q + 1] = pd.ustart[q] + (long)((h.tgt.sz[l + 1] + 7) / 8 * 8) * ((h.tgt.sz[l] + 7) / 8);
            units += (long)h.tgt.sz[l] * h.tgt.sz[l + 1];
        }
        if (pd.L == 0) continue;
        ProfScope ps("pack_weights", 0, (upd ? 4.0 : 6.0) * ng * units, s);
        if (upd) pack_weights16(h.theta16, h.ld, g0, ng, pd, h.wimg.p, h.wimg.gs, s);
        else pack_weights(h.theta, h.ld, g0, ng, pd, h.wimg.p, h.wimg.gs, s);
    }
}

void HyperNet::refresh_images(cudaStream_t s) { to_img(p + nf, F, 0, (int)P, F, mimg, 1, s); }

// hypernet_backward (hypernet.cpp:92-122) summed over the clusters:
// db = sum_g gtheta_g, dM = sum_g gtheta_g f_g^T, df_g = M^T gtheta_g, then
// the feature-map backward. Writes (not accumulates) the flat grad g. This
// rank's clusters are [fg0, fg0 + fng) (all of them without a communicator).
// Sharded (comm set): the local gtheta rows are exchanged all-to-all by
// column shard, so db and dM of this rank's M rows [row_lo, row_hi) sum over
// every cluster in the single-rank order; each cluster's df-derived feature
// gradient (gz) is all-gathered and the feature-map backward runs over all
// clusters on every rank. No collective sums floating-point partials, so the
// result is the single-rank one bit for bit.
void HyperNet::backward(cudaStream_t s) {
    HyperNet* self = this;
    backward_multi(&self, 1, s);
}

static Img img_rows(const Img& im, long r0, int R) {  // rows [r0, r0 + R) of an image (r0 % 128 == 0)
    Img v = im;
    v.p = im.p + (r0 / 128) * (long)img_ct(im.C) * 32768;
    v.R = R;
    return v;
}

void HyperNet::backward_multi(HyperNet* const* hs, int nh, cudaStream_t s, int part) {
    if (part != 2) {  // the gradient passes (no parameter is written)
        for (int k = 0; k < nh; ++k) {  // local gimg (df operand) + db (single rank) in one pass
            HyperNet& h = *hs[k];
            ProfScope ps("gtheta_prep", 0, 6.0 * h.fng * h.P + (h.comm ? 8.0 * h.world * h.Kl * h.S : 4.0 * h.P), s);
            gtheta_prep(h.gtheta + (long)h.fg0 * h.ld, h.ld, h.fng, (int)h.P, h.gimg,
                        h.comm ? nullptr : h.g + h.nf + h.P * h.F, s);
            if (h.comm) {
                pack_shards(h.gtheta + (long)h.fg0 * h.ld, h.ld, h.fng, h.S, h.world, h.gsend, s);
                // the exchange starts now on xs, beside the df GEMM and the local feature backward
                MB_CUDA(cudaEventRecord(h.xev[0], s));
                MB_CUDA(cudaStreamWaitEvent(h.xs, h.xev[0], 0));
                ProfScope ps2("exchange", 0, 4.0 * h.world * h.Kl * h.S, h.xs);
                // every cluster's gtheta on this rank's shard, then its image and db (all clusters, in order)
                comm_alltoall_bytes(h.comm, h.gsend, h.grecv, sizeof(float) * (size_t)h.Kl * h.S, h.xs);
                if (h.row_hi > h.row_lo)
                    gtheta_prep(h.grecv, h.S, h.G, (int)(h.row_hi - h.row_lo), h.gshard,
                                h.g + h.nf + h.P * h.F + h.row_lo, h.xs);
            }
        }
        {
            IGemm ds[2];
            double fl = 0, by = 0;
            for (int k = 0; k < nh; ++k) {
                HyperNet& h = *hs[k];
                IGemm& d = ds[k];  // gf[g][k] = sum_p gtheta[g][p] M[p][k], split-K over 128-aligned P ranges
                d.A = h.gimg; d.a_view = 0;  // (m = g, k = p)
                d.B = h.mimg; d.b_view = 1;  // (n = f, k = p)
                d.M = h.fng; d.N = h.F; d.K = (int)h.P; d.Z = h.splits;
                d.gmode = 2; d.goff = h.d_split_bounds;
                d.C = h.parts; d.cm = h.F; d.cn = 1; d.c_gs = (long)h.fng * h.F;
                fl += 2.0 * d.M * d.N * d.K;
                by += igemm_bytes(d);
            }
            ProfScope ps("hyper_df", fl, by, s);
            img_gemm_batch(ds, nh, s);
        }
        FeatDims loc[2], all[2];
        FeatJob jl[2], ja[2];
        bool any_comm = false;
        for (int k = 0; k < nh; ++k) {
            HyperNet& h = *hs[k];
            any_comm |= h.comm != nullptr;
            loc[k] = h.fd;  // this rank's clusters: df split-K sum * tanh' -> gz rows [fg0, fg0 + fng)
            for (int l = 0; l <= h.fd.L; ++l) loc[k].act[l] = h.fd.act[l] + (long)h.fg0 * h.fd.sz[l];
            for (int l = 0; l < h.fd.L; ++l) loc[k].gz[l] = h.fd.gz[l] + (long)h.fg0 * h.fd.sz[l + 1];
            jl[k] = FeatJob{&loc[k], h.p, h.w_last + (long)h.fg0 * h.m, h.fng, Img{}, 0, 0, h.parts, h.splits, h.g};
            all[k] = h.fd;  // all clusters: the feature map's weight gradients
            ja[k] = FeatJob{&all[k], h.p, h.w_last, h.G, Img{}, 0, 0, h.parts, h.splits, h.g};
        }
        if (!any_comm) {
            double fl = 0;
            for (int k = 0; k < nh; ++k)
                for (size_t l = 0; l + 1 < hs[k]->fsz.size(); ++l) fl += 4.0 * hs[k]->G * hs[k]->fsz[l] * hs[k]->fsz[l + 1];
            ProfScope ps("feature_bwd", fl, 0, s);
            feature_backward_multi(jl, nh, s, 0);
        } else {
            feature_backward_multi(jl, nh, s, 1);
            for (int k = 0; k < nh; ++k) {
                HyperNet& h = *hs[k];
                // the local gz rows are done: all-gather them behind the exchange on xs
                // (one communicator, the same order on every rank), then rejoin
                MB_CUDA(cudaEventRecord(h.xev[0], s));
                MB_CUDA(cudaStreamWaitEvent(h.xs, h.xev[0], 0));
                {
                    ProfScope ps("exchange", 0, 4.0 * h.G * h.F, h.xs);
                    comm_allgather_bytes(h.comm, h.fd.gz[h.fd.L - 1], sizeof(float) * (size_t)h.Kl * h.F, h.xs);
                }
                MB_CUDA(cudaEventRecord(h.xev[1], h.xs));
                MB_CUDA(cudaStreamWaitEvent(s, h.xev[1], 0));
            }
            double fl = 0;
            for (int k = 0; k < nh; ++k)
                for (size_t l = 0; l + 1 < hs[k]->fsz.size(); ++l) fl += 4.0 * hs[k]->G * hs[k]->fsz[l] * hs[k]->fsz[l + 1];
            ProfScope ps("feature_bwd", fl, 0, s);
            feature_backward_multi(ja, nh, s, 2);
        }
    }
    if (part != 1) {  // dM and, fused, the M-block Adam (after the losses' finiteness check)
        for (int k = 0; k < nh; ++k) {
            HyperNet& h = *hs[k];
            if (h.comm) to_img(h.fact.back(), h.F, 0, h.G, h.F, h.fall, 1, s);  // f(w) of every cluster
        }
        {
            IGemm ds[2];
            double fl = 0, by = 0;
            int nd = 0;
            for (int k = 0; k < nh; ++k) {
                HyperNet& h = *hs[k];
                if (h.adam_fused || h.row_hi <= h.row_lo) continue;
                IGemm& d = ds[nd++];  // dM[p][k] = sum_g gtheta[g][p] f[g][k] over this rank's rows
                d.A = h.comm ? h.gshard : h.gimg; d.a_view = 1;  // (m = p, k = g)
                d.B = h.comm ? h.fall : h.fimg; d.b_view = 1;    // (n = f, k = g)
                d.M = (int)(h.row_hi - h.row_lo); d.N = h.F; d.K = h.comm ? h.G : h.fng;
                d.C = h.g + h.nf + h.row_lo * h.F; d.cm = h.F; d.cn = 1;
                fl += 2.0 * d.M * d.N * d.K;
                by += igemm_bytes(d);
            }
            if (nd) {
                ProfScope ps("hyper_dM", fl, by, s);
                img_gemm_batch(ds, nd, s);
            }
        }
        for (int k = 0; k < nh; ++k) {  // dM consumed by Adam in registers (dm_adam.cu)
            HyperNet& h = *hs[k];
            if (!h.adam_fused || h.row_hi <= h.row_lo) continue;
            DmAdam a;
            a.gimg = h.comm ? h.gshard : h.gimg; a.fimg = h.comm ? h.fall : h.fimg;
            a.G = h.comm ? h.G : h.fng; a.P = (int)(h.row_hi - h.row_lo); a.F = h.F;
            const long off = h.nf + h.row_lo * h.F;
            a.p = h.p + off; a.m1 = h.m1 + off; a.m2 = h.m2 + off;
            a.mimg = img_rows(h.mimg, h.row_lo, a.P);
            a.lr = h.ad_lr; a.ibc1 = h.ad_ibc1; a.ibc2 = h.ad_ibc2; a.err = h.ad_err;
            // HBM-bound: p, m1, m2 in + out (fp32), M image out (bf16), gtheta image in
            ProfScope ps("dm_adam", 0, 26.0 * a.P * h.F + 2.0 * a.P * a.G, s);
            dm_adam(a, s);
        }
    }
}

void HyperNet::adam_begin(double lr, const int* err) {
    for (long& st : steps) ++st;
    const double bc1 = 1.0 - std::pow(0.9, (double)steps[0]);
    const double bc2 = 1.0 - std::pow(0.999, (double)steps[0]);
    ad_lr = (float)lr;
    ad_ibc1 = 1.f / (float)bc1;  // as adam_img
    ad_ibc2 = 1.f / (float)bc2;
    ad_err = err;
    adam_fused = true;
}

void HyperNet::adam_step(double lr, const int* err, cudaStream_t s) {
    // three blocks (feature, M, b) with their own step counters (train.cpp:28-39);
    // they always advance together, so one launch covers the flat vector.
    if (!adam_fused)
        for (long& st : steps) ++st;
    const double bc1 = 1.0 - std::pow(0.9, (double)steps[0]);
    const double bc2 = 1.0 - std::pow(0.999, (double)steps[0]);
    const long b0 = nf + P * F;
    Img none;
    if (!comm) {
        if (adam_fused) {  // M was updated inside the dM kernel: the feature and b blocks remain
            ProfScope ps("adam", 0, 28.0 * (nf + P), s);
            adam_img(n, p, g, m1, m2, (float)lr, (float)bc1, (float)bc2, err, 0, F, none, s, nf, b0 - nf);
        } else {
            ProfScope ps("adam", 0, 28.0 * n + 2.0 * P * F, s);  // p,g,m1,m2 in; p,m1,m2 out; M image (bf16)
            adam_img(n, p, g, m1, m2, (float)lr, (float)bc1, (float)bc2, err, nf, F, mimg, s);
        }
        adam_fused = false;
        return;
    }
    // sharded: the replicated feature block and this rank's M rows / b entries
    {
        ProfScope ps("adam", 0, 28.0 * (nf + (row_hi - row_lo) * (adam_fused ? 1 : F + 1)), s);
        if (adam_fused) {  // feature block + b shard (M shard done in dm_adam)
            adam_img(b0 + row_hi, p, g, m1, m2, (float)lr, (float)bc1, (float)bc2, err, 0, F, none, s, nf,
                     b0 + row_lo - nf);
        } else {
            adam_img(nf + row_hi * F, p, g, m1, m2, (float)lr, (float)bc1, (float)bc2, err, 0, F, none, s, nf,
                     row_lo * F);  // feature block + M shard
            if (row_hi > row_lo)
                to_img(p + nf + row_lo * F, F, 0, (int)(row_hi - row_lo), F, img_rows(mimg, row_lo, (int)(row_hi - row_lo)),
                       1, s);
            adam_img(b0 + row_hi, p, g, m1, m2, (float)lr, (float)bc1, (float)bc2, err, 0, F, none, s, 0,
                     b0 + row_lo);  // b shard
        }
    }
    adam_fused = false;
    ProfScope ps("exchange", 0, 2.0 * world * S * F + 4.0 * world * S, s);
    // every rank's refreshed M image rows and b entries (rank r's block at row / entry r S)
    comm_allgather_bytes(comm, mimg.p, (size_t)(S / 128) * img_ct(F) * 32768, s);
    comm_allgather_bytes(comm, p + b0, sizeof(float) * (size_t)S, s);
}

void HyperNet::gather_params(cudaStream_t s) {
    if (!comm) return;
    float* tmp = dalloc<float>((size_t)world * S * F);
    MB_CUDA(cudaMemcpyAsync(tmp + (size_t)rank * S * F, p + nf + row_lo * F, sizeof(float) * (row_hi - row_lo) * F,
                            cudaMemcpyDeviceToDevice, s));
    comm_allgather_bytes(comm, tmp, sizeof(float) * (size_t)S * F, s);
    MB_CUDA(cudaMemcpyAsync(p + nf, tmp, sizeof(float) * P * F, cudaMemcpyDeviceToDevice, s));
    MB_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
}

// ------------------------------------------------------------------ sharding
// optimizer shards: whole 128-row chunks of the M image per rank; rank r
// owns rows [r S, r S + S) clipped to P (the last ranks may own none)
void shard_rows(long P, int world, int rank, long* S, long* lo, long* hi) {
    const long rt = (P + 127) / 128;
    *S = ((rt + world - 1) / world) * 128;
    *lo = std::min<long>(P, (long)rank * *S);
    *hi = std::min<long>(P, *lo + *S);
}

void shard_minibatch(const int* perm, int lo, int hi, int T, int inst_lo, int n_inst, int reps, int n_groups,
                     int* rows_out, int* goff_out, int* n_rows_out, int* max_group) {
    // stable counting sort by (local) cluster id; rows keep minibatch order
    std::vector<int> cnt(n_groups + 1, 0);
    for (int q = lo; q < hi; ++q) {
        const int i = perm[q] / T - inst_lo;
        if (i < 0 || i >= n_inst) continue;
        cnt[i / reps + 1]++;
    }
    int mx = 0;
    for (int c = 0; c < n_groups; ++c) {
        mx = std::max(mx, cnt[c + 1]);
        cnt[c + 1] += cnt[c];
    }
    for (int c = 0; c <= n_groups; ++c) goff_out[c] = cnt[c];
    std::vector<int> pos(cnt.begin(), cnt.end() - 1);
    for (int q = lo; q < hi; ++q) {
        const int r = perm[q];
        const int i = r / T - inst_lo;
        if (i < 0 || i >= n_inst) continue;
        rows_out[pos[i / reps]++] = r - inst_lo * T;
    }
    *n_rows_out = cnt[n_groups];
    *max_group = mx;
}

// pad every cluster's row range to a multiple of 128 (row id -1 = padding);
// rewrites goff in place, returns the max padded group size
int pad_groups(const int* rows, int* goff, int G, int* rows_out, int* n_out) {
    int q = 0, mx = 0;
    std::vector<int> og(goff, goff + G + 1);
    for (int z = 0; z < G; ++z) {
        const int cnt = og[z + 1] - og[z];
        const int pc = (cnt + 127) / 128 * 128;
        goff[z] = q;
        for (int i = 0; i < cnt; ++i) rows_out[q + i] = rows[og[z] + i];
        for (int i = cnt; i < pc; ++i) rows_out[q + i] = -1;
        q += pc;
        mx = std::max(mx, pc);
    }
    goff[G] = q;
    *n_out = q;
    return mx;
}

// ------------------------------------------------------------------ Trainer
Trainer::Trainer(const TrainConfig& cfg, int world, int rank, const void* nccl_id, LoopGroup* loop)
    : cfg_(cfg), world_(world), rank_(rank) {
    es_ = env_spec_of(cfg.env_kind);
    cfg_.validate(es_.m);
    if (es_.obs_dim > 64 || es_.act_dim > 16 || es_.m > 8)
        throw ShapeError("env dims exceed the device bounds (obs 64, act 16, m 8)");
    for (int h : cfg.actor_hidden)
        if (h > 256) throw ShapeError("hidden widths above 256 are not supported on the device path");
    for (int h : cfg.critic_hidden)
        if (h > 256) throw ShapeError("hidden widths above 256 are not supported on the device path");
    if (world < 1 || rank < 0 || rank >= world) throw ConfigError("bad world/rank");
    if (cfg.K % world != 0) throw ConfigError("K must be divisible by the number of GPUs");
    Kl_ = cfg.K / world;
    reps_ = cfg.N / cfg.K;
    Nl_ = Kl_ * reps_;
    inst_lo_ = rank * Nl_;
    g_lo_ = rank * Kl_;
    Rl_ = (long)Nl_ * cfg.T;
    MB_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    MB_CUDA(cudaStreamCreateWithFlags(&s2_, cudaStreamNonBlocking));
    MB_CUDA(cudaStreamCreateWithFlags(&s3_, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&ev_gather_, &ev_c_net_, &ev_chk_, &ev_cd_[0], &ev_cd_[1], &ev_ad_[0], &ev_ad_[1],
                           &ev_cfin_})
        MB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int c = 0; c < 2; ++c) {
        MB_CUDA(cudaStreamCreateWithFlags(&side_[c], cudaStreamNonBlocking));
        MB_CUDA(cudaEventCreateWithFlags(&ev_fork_[c], cudaEventDisableTiming));
        MB_CUDA(cudaEventCreateWithFlags(&ev_join_[c], cudaEventDisableTiming));
    }
    for (cudaEvent_t e : {ev_cd_[0], ev_cd_[1], ev_cfin_}) MB_CUDA(cudaEventRecord(e, s2_));
    for (cudaEvent_t e : {ev_ad_[0], ev_ad_[1]}) MB_CUDA(cudaEventRecord(e, s_));
    // a communicator whenever an NCCL id or a loopback group is given (world
    // == 1 included: the single-rank collectives run the sharded code path
    // on one GPU); one per update chain so the two chains' exchanges overlap
    if (loop) {
        comm_ = comm_create_loopback(loop, rank);
        if (comm_world(comm_) != world) throw ConfigError("loopback group size != world");
    } else if (world > 1 || nccl_id) {
        comm_ = comm_create(world, rank, nccl_id);
    }
    if (comm_) comm2_ = comm_split(comm_);
    root_ = HostRng::seeded(cfg.seed);
    std::vector<int> as{es_.obs_dim}, cs{es_.obs_dim};
    for (int h : cfg.actor_hidden) as.push_back(h);
    as.push_back(es_.act_dim);
    for (int h : cfg.critic_hidden) cs.push_back(h);
    cs.push_back(es_.m);
    actor_.init(es_.m, cfg.F, cfg.feat_hidden, as, true, true, cfg.K, comm_, Kl_);     // config.cpp:59-70
    critic_.init(es_.m, cfg.F, cfg.feat_hidden, cs, false, false, cfg.K, comm2_, Kl_); // config.cpp:72-83
    actor_.init_params(root_.split(0xA1).key, s_);                        // train.cpp:67-70
    critic_.init_params(root_.split(0xA2).key, s_);
    alloc();
    env_reset(es_.kind, Nl_, d_state, d_ekey, d_ectr, d_steps, root_.split(0xE0).key, inst_lo_, s_);
    perm_.resize((size_t)cfg.N * cfg.T);
    std::iota(perm_.begin(), perm_.end(), 0);  // train.cpp:112-114
    MB_CUDA(cudaStreamSynchronize(s_));
}

Trainer::~Trainer() {
    join_worker();
    for (auto& p : plan_) {
        if (p.rows) cudaFreeHost(p.rows);
        if (p.goff) cudaFreeHost(p.goff);
        if (p.uploaded) cudaEventDestroy(p.uploaded);
    }
    if (g_prof == &prof_) g_prof = nullptr;
    actor_.free_all();
    critic_.free_all();
    for (auto* p : {d_obs, d_act, d_eps, d_lp, d_rew, d_val, d_nval, d_adv, d_tgt, d_sadv, d_state, d_tracker, d_cw,
                    d_lsg, mbb_[0].Z, mbb_[0].lpo, mbb_[0].sa, mbb_[0].tg, mbb_[1].Z, mbb_[1].lpo, mbb_[1].sa,
                    mbb_[1].tg})
        if (p) cudaFree(p);
    for (auto& b : mbb_) cudaFree(b.rg);
    for (auto* p : img_allocs_) cudaFree(p);
    for (auto& u : ub_) {
        for (float* q : u.pbias) cudaFree(q);
        cudaFree(u.psls);
        cudaFree(u.lossrows);
    }
    for (auto e : {ev_gather_, ev_c_net_, ev_chk_, ev_cd_[0], ev_cd_[1], ev_ad_[0], ev_ad_[1], ev_cfin_})
        if (e) cudaEventDestroy(e);
    if (s2_) cudaStreamDestroy(s2_);
    if (s3_) cudaStreamDestroy(s3_);
    for (int c = 0; c < 2; ++c) {
        if (side_[c]) cudaStreamDestroy(side_[c]);
        if (ev_fork_[c]) cudaEventDestroy(ev_fork_[c]);
        if (ev_join_[c]) cudaEventDestroy(ev_join_[c]);
    }
    for (auto& u : ub_) cudaFree(u.Zf);
    for (void* p : {(void*)d_term, (void*)d_trunc, (void*)d_ekey, (void*)d_ectr, (void*)d_steps, (void*)d_err,
                    (void*)d_clamps, (void*)d_rows, (void*)d_goff, (void*)d_lossrows,
                    (void*)d_mbloss, (void*)d_stats, (void*)d_scratch, (void*)d_part, (void*)d_retsum, (void*)d_retcnt,
                    (void*)d_pol_blob, (void*)d_cri_blob})
        if (p) cudaFree(p);
    if (h_cw_pinned) cudaFreeHost(h_cw_pinned);
    if (h_rows_pinned) cudaFreeHost(h_rows_pinned);
    if (h_goff_pinned) cudaFreeHost(h_goff_pinned);
    if (comm2_) comm_destroy(comm2_);
    if (comm_) comm_destroy(comm_);
    if (s_) cudaStreamDestroy(s_);
}

void Trainer::alloc() {
    const int od = es_.obs_dim, ad = es_.act_dim, m = es_.m;
    d_obs = dalloc<float>(Rl_ * od);
    d_act = dalloc<float>(Rl_ * ad);
    d_eps = dalloc<float>(Rl_ * ad);
    d_lp = dalloc<float>(Rl_);
    d_rew = dalloc<float>(Rl_ * m);
    d_val = dalloc<float>(Rl_ * m);
    d_nval = dalloc<float>(Rl_ * m);
    d_adv = dalloc<float>(Rl_ * m);
    d_tgt = dalloc<float>(Rl_ * m);
    d_sadv = dalloc<float>(Rl_);
    d_term = dalloc<uint8_t>(Rl_);
    d_trunc = dalloc<uint8_t>(Rl_);
    d_state = dalloc<float>((size_t)es_.state_dim * Nl_);
    d_ekey = dalloc<uint64_t>(Nl_);
    d_ectr = dalloc<uint64_t>(Nl_);
    d_steps = dalloc<int>(Nl_);
    d_tracker = dalloc<float>((size_t)Nl_ * m);
    d_err = dalloc<int>(1);
    d_clamps = dalloc<unsigned long long>(1);
    d_cw = dalloc<float>((size_t)cfg_.K * m);
    MB_CUDA(cudaMallocHost(&h_cw_pinned, sizeof(float) * cfg_.K * m));
    const long R = (long)cfg_.N * cfg_.T;
    Bmax_ = (int)((R + cfg_.minibatch_count - 1) / cfg_.minibatch_count);
    const int slots = cfg_.epochs * cfg_.minibatch_count;
    MB_CUDA(cudaMallocHost(&h_rows_pinned, sizeof(int) * (size_t)slots * Bmax_));
    MB_CUDA(cudaMallocHost(&h_goff_pinned, sizeof(int) * (size_t)slots * (Kl_ + 1)));
    d_rows = dalloc<int>((size_t)slots * Bmax_);
    d_goff = dalloc<int>((size_t)slots * (Kl_ + 1));
    d_rowgroup = dalloc<int>(Bmax_);
    d_Z = dalloc<float>((size_t)Bmax_ * ad);
    d_lpo = dalloc<float>(Bmax_);
    d_sa = dalloc<float>(Bmax_);
    d_tg = dalloc<float>((size_t)Bmax_ * m);
    d_lsg = dalloc<float>((size_t)Bmax_ * ad);
    // tcgen05 update path: group-padded (128-aligned) minibatch rows
    Bpmax_ = ((Bmax_ + 127) / 128 + Kl_) * 128;
    MB_CUDA(cudaFreeHost(h_rows_pinned));
    MB_CUDA(cudaMallocHost(&h_rows_pinned, sizeof(int) * (size_t)slots * Bpmax_));
    cudaFree(d_rows);
    d_rows = dalloc<int>((size_t)slots * Bpmax_);
    cudaFree(d_rowgroup);
    for (float** f : {&d_Z, &d_lpo, &d_sa, &d_tg, &d_lsg}) cudaFree(*f);
    for (auto& b : mbb_) {  // double-buffered minibatch inputs (see mbb_)
        b.rg = dalloc<int>(Bpmax_);
        b.Z = dalloc<float>((size_t)Bpmax_ * ad);
        b.lpo = dalloc<float>(Bpmax_);
        b.sa = dalloc<float>(Bpmax_);
        b.tg = dalloc<float>((size_t)Bpmax_ * m);
        b.Xi = new_img(Bpmax_, od);
    }
    d_lsg = dalloc<float>((size_t)Bpmax_ * ad);
    use_mb_bufs(0);
    for (int w = 0; w < 2; ++w) {
        const NetDims& nd = w == 0 ? actor_.tgt : critic_.tgt;
        for (int l = 0; l < nd.L; ++l) {
            if (l < nd.L - 1) ub_[w].A.push_back(new_img(Bpmax_, nd.sz[l + 1]));
            ub_[w].G.push_back(new_img(Bpmax_, nd.sz[l + 1]));
        }
        ub_[w].Zf = dalloc<float>((size_t)Bpmax_ * 16);
    }
    d_lossrows = dalloc<double>(Bpmax_);
    {
        int wmax = 16;
        for (int l = 1; l <= actor_.tgt.L; ++l) wmax = std::max(wmax, actor_.tgt.sz[l]);
        for (int l = 1; l <= critic_.tgt.L; ++l) wmax = std::max(wmax, critic_.tgt.sz[l]);
        for (auto& u : ub_) {
            const int L = (&u == &ub_[0] ? actor_ : critic_).tgt.L;
            for (int l = 0; l < L; ++l) u.pbias.push_back(dalloc<float>((size_t)(Bpmax_ / 128) * wmax));
            u.psls = dalloc<float>((size_t)(Bpmax_ / 128) * 16);
            u.lossrows = dalloc<double>(Bpmax_);
        }
    }
    rows_tmp_.assign((size_t)Bmax_ + 1, 0);
    for (auto& p : plan_) {
        MB_CUDA(cudaMallocHost(&p.rows, sizeof(int) * (size_t)slots * Bpmax_));
        MB_CUDA(cudaMallocHost(&p.goff, sizeof(int) * (size_t)slots * (Kl_ + 1)));
        p.B.assign(slots, 0);
        p.Bglob.assign(slots, 0);
        p.maxg.assign(slots, 0);
        p.tmp.assign((size_t)Bmax_ + 1, 0);
        MB_CUDA(cudaEventCreateWithFlags(&p.uploaded, cudaEventDisableTiming));
    }
    d_mbloss = dalloc<double>((size_t)slots * 2 + 2);
    d_stats = dalloc<double>(4 * 8);
    d_part = dalloc<double>((size_t)cfg_.K * 8);
    d_scratch = dalloc<double>(148 * 2 * 8);
    d_retsum = dalloc<double>(Nl_);
    pol_plan_ = make_plan(actor_.tgt);
    cri_plan_ = make_plan(critic_.tgt);
    if (pol_plan_.kin_pad[0] != cri_plan_.kin_pad[0]) throw ShapeError("policy/critic input padding mismatch");
    d_pol_blob = dalloc<uint8_t>((size_t)Kl_ * pol_plan_.blob_bytes);
    d_cri_blob = dalloc<uint8_t>((size_t)Kl_ * cri_plan_.blob_bytes);
    d_retcnt = dalloc<int>(Nl_);
    mb_B_.assign(slots, 0);
    mb_Bglob_.assign(slots, 0);
    mb_maxg_.assign(slots, 0);
}

Img Trainer::new_img(int R, int C) {
    Img im;
    im.R = R;
    im.C = C;
    im.p = dalloc<uint8_t>((size_t)img_bytes(R, C));
    img_allocs_.push_back(im.p);
    return im;
}

void Trainer::phase_rollout(int it) {
    g_prof = &prof_;
    prof_.phase = "rollout";
    const int m = es_.m, K = cfg_.K;
    const HostRng iter = root_.split(0x10000000ULL + (uint64_t)it);  // train.cpp:120
    cw_h_.assign((size_t)K * m, 0.f);
    if (m == 1) {
        for (int k = 0; k < K; ++k) cw_h_[k] = 1.f;
    } else {  // build_tradeoff_batch (simplex.cpp:55-87): K-kappa Dirichlet draws + vertices
        HostRng sr = iter.split(0);
        const int nd = K - cfg_.kappa;
        std::vector<double> w(m);
        for (int k = 0; k < nd; ++k) {
            double sum = 0.0;
            for (int j = 0; j < m; ++j) {
                w[j] = -std::log(sr.next_open());
                sum += w[j];
            }
            for (int j = 0; j < m; ++j) cw_h_[(size_t)k * m + j] = (float)(w[j] / sum);
        }
        for (int k = 0; k < cfg_.kappa; ++k) cw_h_[(size_t)(nd + k) * m + k] = 1.f;
    }
    std::memcpy(h_cw_pinned, cw_h_.data(), sizeof(float) * K * m);
    MB_CUDA(cudaMemcpyAsync(d_cw, h_cw_pinned, sizeof(float) * K * m, cudaMemcpyHostToDevice, s_));
    MB_CUDA(cudaMemsetAsync(d_retsum, 0, sizeof(double) * Nl_, s_));
    MB_CUDA(cudaMemsetAsync(d_retcnt, 0, sizeof(int) * Nl_, s_));
    MB_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s_));
    {
        HyperNet* both[2] = {&actor_, &critic_};
        HyperNet::forward_multi(both, 2, d_cw, g_lo_, Kl_, s_);
    }
    {
        ProfScope ps("pack_theta", 0, (double)Kl_ * (actor_.P * 4 + pol_plan_.blob_bytes + critic_.P * 4 +
                                                       cri_plan_.blob_bytes), s_);
        pack_theta(actor_.theta + (long)g_lo_ * actor_.ld, actor_.ld, Kl_, actor_.tgt, pol_plan_, d_pol_blob, s_);
        pack_theta(critic_.theta + (long)g_lo_ * critic_.ld, critic_.ld, Kl_, critic_.tgt, cri_plan_, d_cri_blob, s_);
    }
    RolloutTcArgs a{};
    a.pol_plan = pol_plan_;
    a.cri_plan = cri_plan_;
    a.pol_blob = d_pol_blob;
    a.cri_blob = d_cri_blob;
    a.kind = es_.kind; a.N = Nl_; a.T = cfg_.T; a.K = Kl_; a.reps = reps_;
    a.od = es_.obs_dim; a.ad = es_.act_dim; a.m = m; a.sdim = es_.state_dim; a.max_steps = es_.max_steps;
    a.theta = actor_.theta + (long)g_lo_ * actor_.ld;
    a.theta_ld = actor_.ld;
    a.phi = critic_.theta + (long)g_lo_ * critic_.ld;
    a.phi_ld = critic_.ld;
    a.pol = actor_.tgt; a.cri = critic_.tgt;
    a.state = d_state; a.env_key = d_ekey; a.env_ctr = d_ectr; a.steps = d_steps;
    a.roll_key = iter.split(1).key;  // train.cpp:146
    a.roll_inst_base = inst_lo_;
    {
        ProfScope ps("noise", 0, 4.0 * Rl_ * es_.act_dim, s_);
        rollout_noise(a.roll_key, inst_lo_, Nl_, cfg_.T, es_.act_dim, d_eps, s_);
    }
    a.eps = d_eps;
    a.obs = d_obs; a.act_pre = d_act; a.logprob = d_lp; a.reward = d_rew; a.value = d_val; a.next_value = d_nval;
    a.term = d_term; a.trunc = d_trunc; a.tracker = d_tracker;
    a.cluster_w = d_cw + (size_t)g_lo_ * m;
    a.ret_sum = d_retsum; a.ret_cnt = d_retcnt;
    a.clamp_count = d_clamps; a.err = d_err;
    {
        // algorithmic work per env-step: policy MLP + ONE critic MLP (the
        // reference's second critic call per step is reused)
        double macs = 0;
        for (int l = 0; l < a.pol.L; ++l) macs += (double)a.pol.sz[l] * a.pol.sz[l + 1];
        for (int l = 0; l < a.cri.L; ++l) macs += (double)a.cri.sz[l] * a.cri.sz[l + 1];
        // batch writes (obs, pre-tanh action, log-prob, reward / value / next value, flags)
        const double by = (double)Rl_ * (4.0 * (a.od + a.ad + 1 + 3 * m) + 2);
        ProfScope ps("rollout", 2.0 * macs * Rl_, by, s_);
        rollout_tc(a, s_);
    }
    prepare_perms(it);  // host work overlaps the rollout on the GPU
}

// the update of an externally provided batch (set via the field setters):
// only the iteration's minibatch plans and the per-iteration resets; the
// clusters are whatever set_clusters() left (train.cpp:156-169)
void Trainer::phase_plans(int it) {
    g_prof = &prof_;
    MB_CUDA(cudaMemsetAsync(d_retsum, 0, sizeof(double) * Nl_, s_));
    MB_CUDA(cudaMemsetAsync(d_retcnt, 0, sizeof(int) * Nl_, s_));
    MB_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s_));
    prepare_perms(it);
}

void Trainer::build_plan(PermPlan& p, int it, const std::vector<int>& perm_before, long version) {
    if (p.uploaded) MB_CUDA(cudaEventSynchronize(p.uploaded));  // pinned buffers free again
    p.it = -1;
    p.perm = perm_before;
    const HostRng iter = root_.split(0x10000000ULL + (uint64_t)it);
    HostRng sh = iter.split(2);  // train.cpp:156
    const long R = (long)cfg_.N * cfg_.T;
    const int mbs = cfg_.minibatch_count;
    int* perm = p.perm.data();
    for (int e = 0; e < cfg_.epochs; ++e) {
        for (long i = R; i > 1; --i) {  // rng.hpp:71-76 Fisher-Yates
            const long j = (long)sh.next_below((uint64_t)i);
            std::swap(perm[i - 1], perm[j]);
        }
        for (int s = 0; s < mbs; ++s) {
            const int slot = e * mbs + s;
            const int lo = (int)(R * s / mbs), hi = (int)(R * (s + 1) / mbs);  // train.cpp:163-169
            int nrows = 0, mx = 0;
            int* goff = p.goff + (size_t)slot * (Kl_ + 1);
            shard_minibatch(perm, lo, hi, cfg_.T, inst_lo_, Nl_, reps_, Kl_, p.tmp.data(), goff, &nrows, &mx);
            p.Bglob[slot] = hi - lo;
            p.maxg[slot] = pad_groups(p.tmp.data(), goff, Kl_, p.rows + (size_t)slot * Bpmax_, &p.B[slot]);
        }
    }
    p.version = version;
    p.it = it;
}

void Trainer::join_worker() {
    if (worker_.joinable()) worker_.join();
}

void Trainer::set_perm(const int* in) {
    join_worker();
    std::memcpy(perm_.data(), in, sizeof(int) * perm_.size());
    ++perm_version_;
}

void Trainer::prepare_perms(int it) {
    join_worker();
    int use = -1;
    for (int b = 0; b < 2; ++b)
        if (plan_[b].it == it && plan_[b].version == perm_version_) use = b;
    if (use < 0) {  // no look-ahead plan (first iteration, perm set externally, iteration skipped)
        use = worker_plan_ >= 0 ? worker_plan_ : 0;
        build_plan(plan_[use], it, perm_, perm_version_);
    }
    PermPlan& p = plan_[use];
    perm_.swap(p.perm);
    p.perm.clear();
    p.it = -1;  // consumed
    ++perm_version_;
    mb_B_ = p.B;
    mb_Bglob_ = p.Bglob;
    mb_maxg_ = p.maxg;
    const int slots = cfg_.epochs * cfg_.minibatch_count;
    MB_CUDA(cudaMemcpyAsync(d_rows, p.rows, sizeof(int) * (size_t)slots * Bpmax_, cudaMemcpyHostToDevice, s_));
    MB_CUDA(cudaMemcpyAsync(d_goff, p.goff, sizeof(int) * (size_t)slots * (Kl_ + 1), cudaMemcpyHostToDevice, s_));
    MB_CUDA(cudaEventRecord(p.uploaded, s_));
    // look ahead: the next iteration's plan on the other buffer, from the
    // permutation this iteration leaves behind
    const int nxt = use ^ 1;
    worker_plan_ = nxt;
    const long ver = perm_version_;
    std::vector<int> base = perm_;
    worker_ = std::thread([this, nxt, it, ver, base = std::move(base)]() {
        try {
            build_plan(plan_[nxt], it + 1, base, ver);
        } catch (...) {
            plan_[nxt].it = -1;  // rebuilt (and the error raised) synchronously when needed
        }
    });
}

void Trainer::phase_advantages() {
    g_prof = &prof_;
    prof_.phase = "advantages";
    const int m = es_.m;
    {
        ProfScope ps("gae", 0, (double)Rl_ * (5.0 * m * 4 + 2), s_);  // r,V,V' in; A,target out; flags
        gae_scan(Nl_, cfg_.T, m, d_rew, d_val, d_nval, d_term, d_trunc, (float)cfg_.gamma, (float)cfg_.lambda,
                 d_adv, d_tgt, s_);
    }
    // global per-channel statistics (gae.cpp:79-96): one partial per cluster
    // (whole clusters live on one rank), all-gathered, summed in cluster order
    const double rows = (double)cfg_.N * cfg_.T;
    double* sum1 = d_stats;
    double* mean = d_stats + 8;
    double* sum2 = d_stats + 16;
    double* inv = d_stats + 24;
    const long rpg = (long)reps_ * cfg_.T;
    channel_partials(d_adv, Kl_, rpg, m, nullptr, d_part + (size_t)g_lo_ * 8, s_);
    if (comm_) comm_allgather_bytes(comm_, d_part, sizeof(double) * 8 * Kl_, s_);
    channel_total(d_part, cfg_.K, m, sum1, s_);
    stats_finalize(sum1, rows, m, mean, 0, s_);
    channel_partials(d_adv, Kl_, rpg, m, mean, d_part + (size_t)g_lo_ * 8, s_);
    if (comm_) comm_allgather_bytes(comm_, d_part, sizeof(double) * 8 * Kl_, s_);
    channel_total(d_part, cfg_.K, m, sum2, s_);
    stats_finalize(sum2, rows, m, inv, 1, s_);
    scalarize(Nl_, cfg_.T, m, d_adv, d_cw + (size_t)g_lo_ * m, reps_, mean, inv, d_sadv, s_);
}

// One net's loss + backward through its generated weights on one minibatch
// (losses.cpp:46-189), every contraction on the tensor cores over bf16
// images: forward Z_l = A_{l-1} W_l^T (grouped rows), per-row loss head,
// dW_l = G_l^T A_{l-1} (K = the cluster's rows), dX = (G_l W_l) * tanh'.
// Leaves gtheta [local clusters][P] (fp32, reference flat layout) complete.
// One or two nets' loss + backward through their generated weights on one
// minibatch (losses.cpp:46-189); with two nets (actor + critic) every stage
// is one launch covering both. Contractions on the tensor cores over bf16
// images: forward Z_l = A_{l-1} W_l^T (grouped rows), per-row loss head,
// dW_l = G_l^T A_{l-1} (K = the cluster's rows), dX = (G_l W_l) * tanh'.
// Leaves gtheta [local clusters][P] (fp32, reference flat layout) complete.
void Trainer::net_step(HyperNet* const* hs, const bool* actor, int nn, int Bp, float inv_B, int maxg, const int* rows,
                       const int* goff, int slot, cudaStream_t s_) {
    struct Net {
        HyperNet* h;
        bool actor;
        UpdBufs* u;
        float* gth;
        const float* th;
        bool fused_head;
        int Lg;
    } N[2];
    for (int k = 0; k < nn; ++k) {
        Net& n = N[k];
        n.h = hs[k];
        n.actor = actor[k];
        n.u = &ub_[n.actor ? 0 : 1];
        n.gth = n.h->gtheta + (long)g_lo_ * n.h->ld;
        n.th = n.h->theta + (long)g_lo_ * n.h->ld;
        const NetDims& nd = n.h->tgt;
        const int L = nd.L;
        // the output layer, the loss and the output layer's backward run fused
        // in k_head on the CUDA cores when there is a hidden layer to feed it
        n.fused_head = L >= 2 && nd.sz[L - 1] % 16 == 0 && nd.sz[L - 1] <= 256 && nd.sz[L] <= 16;
        n.Lg = n.fused_head ? L - 1 : L;  // layers run as tensor-core GEMMs in the forward
        if (Bp == 0) {
            MB_CUDA(cudaMemsetAsync(n.gth, 0, sizeof(float) * Kl_ * n.h->ld, s_));
            MB_CUDA(cudaMemsetAsync(d_mbloss + slot * 2 + (n.actor ? 0 : 1), 0, sizeof(double), s_));
        }
    }
    if (Bp == 0) return;
    // the generated weight images (h.wimg) were written by the forward's theta GEMM
    auto wl = [](const HyperNet& h, int l) {
        Img w = h.wimg;
        w.p = h.wimg.p + h.wimg_off[l];
        w.R = h.tgt.sz[l + 1];
        w.C = h.tgt.sz[l];
        return w;
    };
    auto set_w = [&](IGemm& d, const HyperNet& h, int l) {  // layer l's weights as the B operand
        d.B = wl(h, l);
        if (h.weight_tma(l)) {
            d.b_tma = 1;
            d.bmap = h.wmap[l];
        }
    };
    auto batch = [&](const char* cls, const IGemm* ds, int n) {
        double fl = 0, by = 0;
        for (int k = 0; k < n; ++k) {
            fl += 2.0 * ds[k].M * ds[k].N * ds[k].K * (ds[k].gmode == 0 ? ds[k].Z : 1);
            by += igemm_bytes(ds[k]);
        }
        ProfScope ps(cls, fl, by, s_);
        img_gemm_batch(ds, n, s_);
    };
    const int Lmax = std::max(N[0].h->tgt.L, nn > 1 ? N[1].h->tgt.L : 0);
    for (int l = 0; l < Lmax; ++l) {  // forward, layer by layer over the nets
        IGemm ds[2];
        int n = 0;
        for (int k = 0; k < nn; ++k) {
            const Net& t = N[k];
            const NetDims& nd = t.h->tgt;
            if (l >= t.Lg) continue;
            const bool last = (l == nd.L - 1);
            IGemm& d = ds[n++];
            d.A = l == 0 ? Xi_ : t.u->A[l - 1]; d.a_view = 0;  // (m = row, k = in)
            set_w(d, *t.h, l); d.b_view = 0;                   // (n = out, k = in)
            d.M = Bp; d.N = nd.sz[l + 1]; d.K = nd.sz[l]; d.Z = Kl_;
            d.gmode = 1; d.goff = goff; d.max_group = maxg;
            d.bias = t.th + nd.boff[l]; d.bias_gs = t.h->ld; d.bias_mode = 1;
            if (last) {
                d.C = t.u->Zf; d.cm = 16; d.cn = 1;  // Gaussian mean / values (pre-activation)
            } else {
                d.act = 1; d.O = t.u->A[l]; d.o_mode = 1;
            }
        }
        // a tanh layer and a plain output layer cannot share a launch
        if (n == 2 && ds[0].act != ds[1].act) {
            batch("mlp_fwd", &ds[0], 1);
            batch("mlp_fwd", &ds[1], 1);
        } else if (n) {
            batch("mlp_fwd", ds, n);
        }
    }
    for (int k = 0; k < nn; ++k) {
        const Net& t = N[k];
        const NetDims& nd = t.h->tgt;
        const int L = nd.L;
        UpdBufs& u = *t.u;
        if (t.fused_head) {
            HeadArgs ha;
            ha.Bp = Bp; ha.H = nd.sz[L - 1]; ha.out = nd.sz[L];
            ha.rows = rows; ha.rg = d_rowgroup;
            ha.theta = t.th; ha.ld = t.h->ld; ha.woff = nd.woff[L - 1]; ha.boff = nd.boff[L - 1]; ha.mlp_n = nd.mlp_n;
            ha.A = u.A[L - 2]; ha.Gout = u.G[L - 1]; ha.Gprev = u.G[L - 2];
            ha.z = d_Z; ha.lp_old = d_lpo; ha.sadv = d_sa; ha.clip = (float)cfg_.clip_eps;
            ha.ent = (float)cfg_.entropy_coef; ha.err = d_err;
            ha.tgt = d_tg; ha.inv_B = inv_B;
            ha.psum = u.pbias[L - 1]; ha.psls = u.psls; ha.psum_prev = u.pbias[L - 2]; ha.psum_prev_ld = nd.sz[L - 1];
            ha.loss_rows = u.lossrows;
            const double fl = 4.0 * Bp * nd.sz[L - 1] * nd.sz[L];  // forward + backward of the output layer
            // last hidden activation image in, its gradient image out, the row inputs and output-layer gradient
            const double by = 4.0 * Bp * nd.sz[L - 1] + 4.0 * Bp * (nd.sz[L] + 4) + 2.0 * Bp * nd.sz[L];
            ProfScope ps("mlp_head", fl, by, s_);
            head(ha, t.actor, s_);
        } else if (t.actor) {  // losses.cpp:87-129
            actor_rows_img(Bp, es_.act_dim, rows, d_rowgroup, t.th, t.h->ld, nd.mlp_n, u.Zf, 16, d_Z, d_lpo, d_sa,
                           (float)cfg_.clip_eps, (float)cfg_.entropy_coef, inv_B, u.G[L - 1], u.pbias[L - 1], u.psls,
                           u.lossrows, d_err, s_);
        } else {  // losses.cpp:170-185
            critic_rows_img(Bp, es_.m, rows, u.Zf, 16, d_tg, inv_B, u.G[L - 1], u.pbias[L - 1], u.lossrows, s_);
        }
    }
    // backward (nn.cpp:111-160): the data-gradient chain first (each dX needs
    // the previous one), then every layer's weight gradient -- independent
    // of each other -- batched three per launch
    for (int l = Lmax - 1; l > 0; --l) {
        IGemm ds[2];
        int n = 0;
        for (int k = 0; k < nn; ++k) {
            const Net& t = N[k];
            const NetDims& nd = t.h->tgt;
            if (l >= nd.L || (t.fused_head && l == nd.L - 1)) continue;  // k_head produced G_{L-2}
            IGemm& e = ds[n++];  // G_{l-1}[q][i] = (sum_j G_l[q][j] W_l[z][j][i]) (1 - A_{l-1}[q][i]^2)
            e.A = t.u->G[l]; e.a_view = 0;  // (m = q, k = j)
            set_w(e, *t.h, l); e.b_view = 1;  // (n = i, k = j)
            e.M = Bp; e.N = nd.sz[l]; e.K = nd.sz[l + 1]; e.Z = Kl_;
            e.gmode = 1; e.goff = goff; e.max_group = maxg;
            e.act = 2; e.aux = t.u->A[l - 1];
            e.O = t.u->G[l - 1]; e.o_mode = 1;
            e.psum = t.u->pbias[l - 1]; e.psum_ld = nd.sz[l];  // per-tile column sums -> bias grads of layer l-1
        }
        if (n) batch("mlp_dX", ds, n);
    }
    // every bias gradient (per-tile column sums of G_l -> per cluster), the
    // log-std gradients and the minibatch losses need only the epilogues'
    // partials, all written by now: one launch on the side stream, beside
    // the weight-gradient GEMMs (both feed the gtheta pass)
    SegJobs jb;
    for (int k = 0; k < nn; ++k) {
        const Net& t = N[k];
        const NetDims& nd = t.h->tgt;
        const int L = nd.L;
        for (int l = 0; l < L; ++l)  // output layer partials are written with a row stride of 16
            jb.job[jb.n++] = SegJob{t.u->pbias[l], l == L - 1 ? 16 : nd.sz[l + 1], nd.sz[l + 1],
                                    t.gth + nd.boff[l], t.h->ld};
        if (t.actor) jb.job[jb.n++] = SegJob{t.u->psls, 16, es_.act_dim, t.gth + nd.mlp_n, t.h->ld};
        jb.loss[jb.nloss++] = SegLoss{t.u->lossrows, Bp / 128, d_mbloss + slot * 2 + (t.actor ? 0 : 1)};
    }
    fork(s_);
    {
        ProfScope ps("segsum", 0, 4.0 * (Bp / 128) * 16 * 2 * 8 + 8.0 * Bp, side_of(s_));  // per-tile partials -> per cluster
        segsum_multi(jb, goff, Kl_, side_of(s_));
    }
    std::vector<IGemm> dws;
    for (int k = 0; k < nn; ++k) {
        const Net& t = N[k];
        const NetDims& nd = t.h->tgt;
        for (int l = nd.L - 1; l >= 0; --l) {
            const Img& ain = l == 0 ? Xi_ : t.u->A[l - 1];
            IGemm d;  // dW_l[z][j][i] = sum_{q in z} G_l[q][j] A_{l-1}[q][i]
            d.A = t.u->G[l]; d.a_view = 1;  // (m = j, k = q)
            d.B = ain; d.b_view = 1;        // (n = i, k = q)
            d.M = nd.sz[l + 1]; d.N = nd.sz[l]; d.K = Bp; d.Z = Kl_;
            d.gmode = 2; d.goff = goff;
            d.C = t.gth + nd.woff[l]; d.cm = nd.sz[l]; d.cn = 1; d.c_gs = t.h->ld;
            dws.push_back(d);
        }
    }
    for (size_t k0 = 0; k0 < dws.size(); k0 += 3) batch("mlp_dW", &dws[k0], (int)std::min<size_t>(3, dws.size() - k0));
    join(s_);
}

// a chain's side stream: fork = it waits for the chain's work so far; join =
// the chain waits for the side stream's work so far
void Trainer::fork(cudaStream_t s) {
    const int c = s == s2_ ? 1 : 0;
    MB_CUDA(cudaEventRecord(ev_fork_[c], s));
    MB_CUDA(cudaStreamWaitEvent(side_[c], ev_fork_[c], 0));
}
void Trainer::join(cudaStream_t s) {
    const int c = s == s2_ ? 1 : 0;
    MB_CUDA(cudaEventRecord(ev_join_[c], side_[c]));
    MB_CUDA(cudaStreamWaitEvent(s, ev_join_[c], 0));
}

void Trainer::use_mb_bufs(int p) {
    const MbBufs& b = mbb_[p];
    Xi_ = b.Xi; d_Z = b.Z; d_lpo = b.lpo; d_sa = b.sa; d_tg = b.tg; d_rowgroup = b.rg;
}

// One PPO minibatch (train.cpp:163-180). Default: one stream per net (actor
// on s_, critic on s2_): the two losses / backward passes / Adam steps are
// independent, so one net's HBM-bound Adam overlaps the other net's GEMMs.
// Joins: both losses are checked for finiteness before either Adam
// (train.cpp:174-178), and the next minibatch's gather waits for the last
// readers of its input buffer set. Single rank: each chain's bias-gradient
// sums and feature / b Adam run on its side stream. MORLAX_FUSED_NETS=1: both
// nets in lockstep on one stream, every stage one launch covering both
// (fewer, fuller launches but no overlap; slower).
void Trainer::minibatch(int slot, int Bp, int Bglob, int maxg, const int* rows, const int* goff) {
    const int od = es_.obs_dim, ad = es_.act_dim, m = es_.m;
    const float inv_B = (float)(1.0 / (double)Bglob);  // global 1/B (losses.cpp:66,155)
    static const bool two = [] {
        const char* e = std::getenv("MORLAX_FUSED_NETS");
        return !(e && e[0] == '1');
    }();
    cudaStream_t sc = two ? s2_ : s_;
    const char* fe = std::getenv("MORLAX_FUSED_ADAM");  // "0": the unfused dM GEMM + Adam (A/B, tests)
    const bool fuse_env = !(fe && fe[0] == '0');
    // dm_adam's tile width (K: any cluster count, in 128-cluster chunks)
    const bool fuse = fuse_env && actor_.F % 64 == 0 && critic_.F % 64 == 0;
    if (fuse) {  // host-side Adam step counters / bias corrections for the fused M-block update
        actor_.adam_begin(cfg_.actor_lr, d_err);
        critic_.adam_begin(cfg_.critic_lr, d_err);
    }
    // the minibatch rows are gathered on their own stream into the input
    // buffer set of this parity, once both chains' losses of two minibatches
    // back (the set's last readers) are done; each chain waits only for it
    mb_par_ ^= 1;
    use_mb_bufs(mb_par_);
    MB_CUDA(cudaStreamWaitEvent(s3_, ev_ad_[mb_par_], 0));
    MB_CUDA(cudaStreamWaitEvent(s3_, ev_cd_[mb_par_], 0));
    if (Bp > 0) {
        MbGather ga;
        ga.Bp = Bp; ga.G = Kl_; ga.od = od; ga.ad = ad; ga.m = m;
        ga.rows = rows; ga.goff = goff;
        ga.obs = d_obs; ga.act = d_act; ga.lp = d_lp; ga.sadv = d_sadv; ga.tgt = d_tgt;
        ga.Xi = Xi_; ga.act_o = d_Z; ga.lp_o = d_lpo; ga.sadv_o = d_sa; ga.tgt_o = d_tg; ga.rg = d_rowgroup;
        ProfScope ps("gather", 0, (double)Bp * (4.0 * od + 2.0 * od + 8.0 * ad + 16.0 + 8.0 * m + 4.0), s3_);
        gather_minibatch(ga, s3_);
    }
    MB_CUDA(cudaEventRecord(ev_gather_, s3_));
    HyperNet* both[2] = {&actor_, &critic_};
    const bool roles[2] = {true, false};
    if (!two) {
        HyperNet::forward_multi(both, 2, d_cw, g_lo_, Kl_, s_, true);  // hypernet_forward per loss (losses.cpp:79,167)
        MB_CUDA(cudaStreamWaitEvent(s_, ev_gather_, 0));
        net_step(both, roles, 2, Bp, inv_B, maxg, rows, goff, slot, s_);
        MB_CUDA(cudaEventRecord(ev_ad_[mb_par_], s_));
        MB_CUDA(cudaEventRecord(ev_cd_[mb_par_], s_));
        if (comm_) comm_allreduce_f64(comm_, d_mbloss + slot * 2, 2, s_);
        check_finite_f64(d_mbloss + slot * 2, 2, d_err, 3, s_);  // train.cpp:174-178
        HyperNet::backward_multi(both, 2, s_);  // (with an exchange: its collectives inside, on s_)
        actor_.adam_step(cfg_.actor_lr, d_err, s_);  // train.cpp:179-180
        critic_.adam_step(cfg_.critic_lr, d_err, s_);
        MB_CUDA(cudaEventRecord(ev_cfin_, s_));
        return;
    }
    // the forwards (feature map, theta, weight packing) need no minibatch rows
    critic_.forward(d_cw, g_lo_, Kl_, sc, true);
    MB_CUDA(cudaStreamWaitEvent(sc, ev_gather_, 0));
    net_step(&both[1], &roles[1], 1, Bp, inv_B, maxg, rows, goff, slot, sc);
    MB_CUDA(cudaEventRecord(ev_c_net_, sc));
    MB_CUDA(cudaEventRecord(ev_cd_[mb_par_], sc));
    // the gradient passes of the backward write no parameter (with a
    // communicator they hold the chain's exchange collectives): each chain
    // runs them before the finiteness join
    HyperNet::backward_multi(&both[1], 1, sc, 1);
    actor_.forward(d_cw, g_lo_, Kl_, s_, true);
    MB_CUDA(cudaStreamWaitEvent(s_, ev_gather_, 0));
    net_step(&both[0], &roles[0], 1, Bp, inv_B, maxg, rows, goff, slot, s_);
    MB_CUDA(cudaEventRecord(ev_ad_[mb_par_], s_));
    HyperNet::backward_multi(&both[0], 1, s_, 1);
    MB_CUDA(cudaStreamWaitEvent(s_, ev_c_net_, 0));
    if (comm_) comm_allreduce_f64(comm_, d_mbloss + slot * 2, 2, s_);
    check_finite_f64(d_mbloss + slot * 2, 2, d_err, 3, s_);  // train.cpp:174-178
    MB_CUDA(cudaEventRecord(ev_chk_, s_));
    MB_CUDA(cudaStreamWaitEvent(sc, ev_chk_, 0));
    // single rank, fused dM + Adam: the feature / b Adam (adam_img) runs on
    // the side stream beside it (disjoint parameter ranges, inputs complete;
    // unfused, adam_img also updates M from the dM GEMM and must follow it)
    const bool side = comm_ == nullptr && fuse;
    for (int k = 1; k >= 0; --k) {  // critic chain, then actor chain
        cudaStream_t st = k ? sc : s_;
        if (side) fork(st);
        HyperNet::backward_multi(&both[k], 1, st, 2);  // (+ the chain's all-gathers on its communicator)
        both[k]->adam_step(k ? cfg_.critic_lr : cfg_.actor_lr, d_err, side ? side_of(st) : st);  // train.cpp:179-180
        if (side) join(st);
        if (k) MB_CUDA(cudaEventRecord(ev_cfin_, sc));
    }
}

void Trainer::phase_update(int it, int max_minibatches) {
    g_prof = &prof_;
    prof_.phase = "update";
    (void)it;
    const int mbs = cfg_.minibatch_count;
    mb_done_ = 0;
    // the gathers (stream s3_) read the rollout / advantages and the uploaded
    // minibatch index lists, all produced on s_
    MB_CUDA(cudaEventRecord(ev_gather_, s_));
    MB_CUDA(cudaStreamWaitEvent(s3_, ev_gather_, 0));
    // every rank refreshes theta for its clusters from the current params
    for (int e = 0; e < cfg_.epochs; ++e)
        for (int s = 0; s < mbs; ++s) {
            if (max_minibatches >= 0 && mb_done_ >= max_minibatches) return;
            const int slot = e * mbs + s;
            if (mb_Bglob_[slot] == 0) continue;  // lo == hi
            minibatch(slot, mb_B_[slot], mb_Bglob_[slot], mb_maxg_[slot], d_rows + (size_t)slot * Bpmax_,
                      d_goff + (size_t)slot * (Kl_ + 1));
            ++mb_done_;
        }
}

void Trainer::finish(IterStats* st) {
    MB_CUDA(cudaStreamWaitEvent(s_, ev_cfin_, 0));  // the critic chain's last Adam
    const int slots = cfg_.epochs * cfg_.minibatch_count;
    std::vector<double> losses((size_t)slots * 2);
    std::vector<double> rs(Nl_);
    std::vector<int> rc(Nl_);
    int err = 0;
    MB_CUDA(cudaMemcpyAsync(losses.data(), d_mbloss, sizeof(double) * slots * 2, cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaMemcpyAsync(rs.data(), d_retsum, sizeof(double) * Nl_, cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaMemcpyAsync(rc.data(), d_retcnt, sizeof(int) * Nl_, cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaStreamSynchronize(s_));
    if (st) {
        st->actor_loss = st->critic_loss = 0;
        int done = 0;
        for (int e = 0, k = 0; e < cfg_.epochs; ++e)
            for (int s = 0; s < cfg_.minibatch_count; ++s, ++k) {
                if (done >= mb_done_) break;
                if (mb_Bglob_[k] == 0) continue;
                st->actor_loss += losses[k * 2];
                st->critic_loss += losses[k * 2 + 1];
                ++done;
            }
        st->minibatches = mb_done_;
        st->numeric_error = err;
        st->cluster_returns.assign(Kl_, std::nan(""));
        for (int c = 0; c < Kl_; ++c) {
            double s = 0;
            int n = 0;
            for (int r = 0; r < reps_; ++r) {
                s += rs[c * reps_ + r];
                n += rc[c * reps_ + r];
            }
            if (n) st->cluster_returns[c] = s / n;
        }
    }
    if (err) throw NumericError("non-finite value during the training iteration (loss, ratio or action)");
}

void Trainer::set_clusters(const float* cw) {
    cw_h_.assign(cw, cw + (size_t)cfg_.K * es_.m);
    MB_CUDA(cudaMemcpy(d_cw, cw, sizeof(float) * cfg_.K * es_.m, cudaMemcpyHostToDevice));
    MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
}

void Trainer::losses_only(const int* rows, int n, double* al, double* cl) {
    g_prof = &prof_;
    if (n <= 0) throw ShapeError("minibatch has no rows");
    if (n > Bmax_) throw ShapeError("losses_only: more rows than one minibatch buffer holds");
    for (int q = 0; q < n; ++q)
        if (rows[q] < 0 || rows[q] >= cfg_.N * cfg_.T) throw ShapeError("minibatch row index out of range");
    int B = 0, mx = 0, Bp = 0;
    shard_minibatch(rows, 0, n, cfg_.T, inst_lo_, Nl_, reps_, Kl_, rows_tmp_.data(), h_goff_pinned, &B, &mx);
    mx = pad_groups(rows_tmp_.data(), h_goff_pinned, Kl_, h_rows_pinned, &Bp);
    MB_CUDA(cudaMemcpyAsync(d_rows, h_rows_pinned, sizeof(int) * (Bp ? Bp : 1), cudaMemcpyHostToDevice, s_));
    MB_CUDA(cudaMemcpyAsync(d_goff, h_goff_pinned, sizeof(int) * (Kl_ + 1), cudaMemcpyHostToDevice, s_));
    MB_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s_));
    {
        HyperNet* both[2] = {&actor_, &critic_};
        HyperNet::forward_multi(both, 2, d_cw, g_lo_, Kl_, s_);
    }
    const int od = es_.obs_dim, ad = es_.act_dim, m = es_.m;
    const float inv_B = (float)(1.0 / (double)n);
    if (Bp > 0) {
        MbGather ga;
        ga.Bp = Bp; ga.G = Kl_; ga.od = od; ga.ad = ad; ga.m = m;
        ga.rows = d_rows; ga.goff = d_goff;
        ga.obs = d_obs; ga.act = d_act; ga.lp = d_lp; ga.sadv = d_sadv; ga.tgt = d_tgt;
        ga.Xi = Xi_; ga.act_o = d_Z; ga.lp_o = d_lpo; ga.sadv_o = d_sa; ga.tgt_o = d_tg; ga.rg = d_rowgroup;
        gather_minibatch(ga, s_);
    }
    HyperNet* both[2] = {&actor_, &critic_};
    const bool roles[2] = {true, false};
    net_step(both, roles, 2, Bp, inv_B, mx, d_rows, d_goff, 0, s_);
    if (comm_) comm_allreduce_f64(comm_, d_mbloss, 2, s_);
    {  // (with an exchange: its collectives inside, on s_)
        HyperNet* both[2] = {&actor_, &critic_};
        HyperNet::backward_multi(both, 2, s_);
    }
    double l[2];
    int err = 0;
    MB_CUDA(cudaMemcpyAsync(l, d_mbloss, sizeof(l), cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s_));
    MB_CUDA(cudaStreamSynchronize(s_));
    if (err) throw NumericError("actor_loss: non-finite ratio");
    *al = l[0];
    *cl = l[1];
}

void Trainer::iteration(int it, IterStats* st) {
    g_prof = &prof_;
    static const bool host_timing = [] {  // MORLAX_HOST_TIMING=1: host enqueue time per phase (stderr)
        const char* e = std::getenv("MORLAX_HOST_TIMING");
        return e && e[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    phase_rollout(it);
    const auto t1 = clk::now();
    phase_advantages();
    const auto t2 = clk::now();
    phase_update(it);
    const auto t3 = clk::now();
    finish(st);
    if (host_timing) {
        const auto ms = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        std::fprintf(stderr, "host enqueue ms: rollout %.3f advantages %.3f update %.3f | total with sync %.3f\n",
                     ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t0, clk::now()));
    }
}

}  // namespace mb200
