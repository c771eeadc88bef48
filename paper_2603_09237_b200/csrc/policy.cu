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

#include "img.cuh"
#include "kernels.h"
#include "policy.h"
#include "umma.cuh"

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
// output layer on the CUDA cores (OUT <= 16 outputs: too narrow for a
// 128-wide MMA tile): one 128-row tile of one group per block, W_L (fp32,
// from theta) in shared memory, the last hidden activation row from its bf16
// image; writes the unpadded pre-squash means directly
template <int OUT>
__global__ void __launch_bounds__(128) k_out_forward(const float* __restrict__ theta, long ld, long woff, long boff,
                                                     int H, Img A, int R, int Rp, float* __restrict__ pre) {
    __shared__ __align__(16) float sw[OUT * 256];
    __shared__ float sb[OUT];
    const int q = blockIdx.x * 128 + threadIdx.x;
    const int g = (blockIdx.x * 128) / Rp, r = q - g * Rp;
    const float* th = theta + (long)g * ld;
    for (int e = threadIdx.x; e < OUT * H; e += 128) sw[e] = th[woff + e];
    if (threadIdx.x < OUT) sb[threadIdx.x] = th[boff + threadIdx.x];
    __syncthreads();
    if (r >= R) return;
    const int CT = img_ct(A.C);
    float o[OUT];
#pragma unroll
    for (int j = 0; j < OUT; ++j) o[j] = sb[j];
    for (int c = 0; c < H; c += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(A.p + img_off(q, c, CT));
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
        float x[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(b2[e]);
            x[2 * e] = f.x;
            x[2 * e + 1] = f.y;
        }
#pragma unroll
        for (int j = 0; j < OUT; ++j) {
            const float4 w0 = *reinterpret_cast<const float4*>(sw + j * H + c);
            const float4 w1 = *reinterpret_cast<const float4*>(sw + j * H + c + 4);
            o[j] = fmaf(x[0], w0.x, fmaf(x[1], w0.y, fmaf(x[2], w0.z, fmaf(x[3], w0.w, o[j]))));
            o[j] = fmaf(x[4], w1.x, fmaf(x[5], w1.y, fmaf(x[6], w1.z, fmaf(x[7], w1.w, o[j]))));
        }
    }
    float* dst = pre + ((long)g * R + r) * OUT;
#pragma unroll
    for (int j = 0; j < OUT; ++j) dst[j] = o[j];
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
    MB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    MB_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    MB_CUDA(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
    MB_CUDA(cudaDeviceSynchronize());
}

GroupPolicy::~GroupPolicy() {
    h.free_all();
    cudaFree(X.p);
    for (auto& a : A) cudaFree(a.p);
    cudaFree(out_pad);
    cudaFree(rowmap);
    cudaFree(goff);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_x) cudaEventDestroy(ev_x);
    if (s2) cudaStreamDestroy(s2);
}

void GroupPolicy::forward(const float* d_w, const float* d_obs, float* d_pre, cudaStream_t s) {
    const NetDims& nd = h.tgt;
    // observations -> bf16 image on a side stream, concurrently with theta generation
    MB_CUDA(cudaEventRecord(ev_in, s));
    MB_CUDA(cudaStreamWaitEvent(s2, ev_in, 0));
    gather_img(rowmap, G * Rp, d_obs, nd.sz[0], X, s2);
    MB_CUDA(cudaEventRecord(ev_x, s2));
    h.forward(d_w, 0, G, s);                                    // theta + per-layer weight images
    MB_CUDA(cudaStreamWaitEvent(s, ev_x, 0));
    const int H = nd.sz[nd.L - 1], out = nd.sz[nd.L];
    const bool simt_out = nd.L >= 2 && H % 8 == 0 && H <= 256 && out <= 16;
    for (int l = 0; l < nd.L - (simt_out ? 1 : 0); ++l) {
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
    if (simt_out) {
        const long woff = nd.woff[nd.L - 1], boff = nd.boff[nd.L - 1];
        const Img& a = A[nd.L - 2];
        const unsigned tiles = (unsigned)((long)G * Rp / 128);
#define MB_OUT(O) \
    case O: k_out_forward<O><<<tiles, 128, 0, s>>>(h.theta, h.ld, woff, boff, H, a, R, Rp, d_pre); break;
        switch (out) {
            MB_OUT(1) MB_OUT(2) MB_OUT(3) MB_OUT(4) MB_OUT(5) MB_OUT(6) MB_OUT(7) MB_OUT(8)
            MB_OUT(9) MB_OUT(10) MB_OUT(11) MB_OUT(12) MB_OUT(13) MB_OUT(14) MB_OUT(15) MB_OUT(16)
        }
#undef MB_OUT
        MB_LAUNCH();
        return;
    }
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
