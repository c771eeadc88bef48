// Per-preference-group policy forward (BASELINE config 2; reference
// policy_forward nn.cpp:162-190 over the weights hypernet_forward
// hypernet.cpp:69-90 generates for each preference): for G preference
// vectors w_g and R observations per group,
//   theta_g = M f(w_g) + b                      (feature MLP + tcgen05 GEMM)
//   pre[g, r] = W_L tanh(... tanh(W_1 obs[g, r] + b_1) ...) + b_L
// with every layer one grouped tcgen05 GEMM over all G*R rows (the rows of
// group g multiply group g's generated weights), bf16 operands and fp32
// accumulation. pre is the Gaussian mean before the tanh squash
// (GaussianAction::pre); the deterministic action is tanh(pre).
#include <algorithm>
#include <vector>

#include "kernels.h"
#include "policy.h"

namespace mb200 {

namespace {
// d_pre[g*R + r][j] <- out[g*Rp + r][j] (drop the 128-row group padding)
__global__ void k_unpad(const float* __restrict__ src, int ld, int R, int Rp, int out, long n, float* dst) {
    const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const long row = e / out;
    const int j = (int)(e - row * out);
    const long g = row / R, r = row - g * R;
    dst[e] = src[(g * Rp + r) * ld + j];
}
// group-padded row map: q = g*Rp + r -> g*R + r (r < R), -1 for padding
__global__ void k_rowmap(int G, int R, int Rp, int* rows) {
    const long q = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (q >= (long)G * Rp) return;
    const int g = (int)(q / Rp), r = (int)(q - (long)g * Rp);
    rows[q] = r < R ? g * R + r : -1;
}
}  // namespace

GroupPolicy::GroupPolicy(int m, int F, const std::vector<int>& fh, const std::vector<int>& sizes, bool out_tanh,
                         bool has_log_std, int G_, int R_)
    : G(G_), R(R_) {
    if (G < 1 || R < 1) throw ShapeError("policy forward: need >= 1 group and >= 1 row per group");
    h.init(m, F, fh, sizes, out_tanh, has_log_std, G);
    if (h.tgt.sz[h.tgt.L] > 16) throw ShapeError("policy forward: output width must be <= 16");
    Rp = (R + 127) / 128 * 128;
    const long rows = (long)G * Rp;
    if (rows > (1L << 30)) throw ShapeError("policy forward: too many rows");
    auto img = [&](int C) {
        Img im;
        im.R = (int)rows;
        im.C = C;
        MB_CUDA(cudaMalloc(&im.p, (size_t)img_bytes((int)rows, C)));
        MB_CUDA(cudaMemset(im.p, 0, (size_t)img_bytes((int)rows, C)));
        return im;
    };
    X = img(h.tgt.sz[0]);
    for (int l = 0; l + 1 < h.tgt.L; ++l) A.push_back(img(h.tgt.sz[l + 1]));
    MB_CUDA(cudaMalloc(&out_pad, sizeof(float) * rows * 16));
    MB_CUDA(cudaMalloc(&rowmap, sizeof(int) * rows));
    std::vector<int> go(G + 1);
    for (int g = 0; g <= G; ++g) go[g] = g * Rp;
    MB_CUDA(cudaMalloc(&goff, sizeof(int) * (G + 1)));
    MB_CUDA(cudaMemcpy(goff, go.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice));
    k_rowmap<<<(unsigned)((rows + 255) / 256), 256>>>(G, R, Rp, rowmap);
    MB_LAUNCH();
    MB_CUDA(cudaDeviceSynchronize());
}

GroupPolicy::~GroupPolicy() {
    h.free_all();
    cudaFree(X.p);
    for (auto& a : A) cudaFree(a.p);
    cudaFree(out_pad);
    cudaFree(rowmap);
    cudaFree(goff);
}

void GroupPolicy::forward(const float* d_w, const float* d_obs, float* d_pre, cudaStream_t s) {
    const NetDims& nd = h.tgt;
    h.forward(d_w, 0, G, s);                                    // theta + per-layer weight images
    gather_img(rowmap, G * Rp, d_obs, nd.sz[0], X, s);           // observations -> bf16 image
    for (int l = 0; l < nd.L; ++l) {
        const bool last = l == nd.L - 1;
        IGemm d;
        d.A = l == 0 ? X : A[l - 1]; d.a_view = 0;
        d.B = h.wimg; d.B.p = h.wimg.p + h.wimg_off[l]; d.B.R = nd.sz[l + 1]; d.B.C = nd.sz[l]; d.b_view = 0;
        d.M = G * Rp; d.N = nd.sz[l + 1]; d.K = nd.sz[l]; d.Z = G;
        d.gmode = 1; d.goff = goff; d.max_group = Rp;
        d.bias = h.theta + nd.boff[l]; d.bias_gs = h.ld; d.bias_mode = 1;
        if (last) {
            d.C = out_pad; d.cm = 16; d.cn = 1;
        } else {
            d.act = 1; d.O = A[l]; d.o_mode = 1;
        }
        img_gemm(d, s);
    }
    const int out = nd.sz[nd.L];
    const long n = (long)G * R * out;
    k_unpad<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out_pad, 16, R, Rp, out, n, d_pre);
    MB_LAUNCH();
}

double GroupPolicy::flops() const {
    const NetDims& nd = h.tgt;
    double f = 0;
    for (int l = 0; l < nd.L; ++l) f += 2.0 * G * R * nd.sz[l] * nd.sz[l + 1];  // per-row MLP
    f += 2.0 * G * h.P * h.F;                                                    // theta = M f + b
    for (size_t l = 0; l + 1 < h.fsz.size(); ++l) f += 2.0 * G * h.fsz[l] * h.fsz[l + 1];
    return f;
}

}  // namespace mb200
