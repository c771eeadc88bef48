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
// output layer (OUT <= 16 outputs: too narrow for a 128-wide tcgen05 tile)
// on mma.sync m16n8k16: one 128-row tile of one group per 4-warp block, each
// warp two 16-row m-tiles; A fragments straight from the bf16 image (one
// 8 x 16 B core matrix = one coalesced 128 B warp load per fragment pair),
// W_L (bf16-rounded from theta, as the weight image) staged in shared memory in
// fragment order; writes the unpadded pre-squash means plus bias directly
template <int NT>
__global__ void __launch_bounds__(128) k_out_forward(const float* __restrict__ theta, long ld, long woff, long boff,
                                                     int H, Img A, int R, int Rp, int OUT, float* __restrict__ pre) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile_r = blockIdx.x * 128;
    const int g = tile_r / Rp;
    const float* th = theta + (long)g * ld;
    const int KS = H >> 4, kq = 2 * (lane & 3), rq = lane >> 2;
    // W_L fragments in mma order: sb[s][j][lane] = {k pair, k pair + 8} of row n
    __shared__ uint2 sb[16][NT][32];
    for (int e = threadIdx.x; e < KS * NT * 32; e += 128) {
        const int l = e & 31, j = (e >> 5) % NT, st = e / (32 * NT);
        const int n = j * 8 + (l >> 2), k = st * 16 + 2 * (l & 3);
        float2 lo = make_float2(0.f, 0.f), hi = lo;
        if (n < OUT) {
            const float* w = th + woff + (long)n * H + k;
            lo = make_float2(w[0], w[1]);
            hi = make_float2(w[8], w[9]);
        }
        const __nv_bfloat162 l2 = __float22bfloat162_rn(lo), h2 = __float22bfloat162_rn(hi);
        sb[st][j][l] = make_uint2(*reinterpret_cast<const uint32_t*>(&l2), *reinterpret_cast<const uint32_t*>(&h2));
    }
    float bias[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int n = j * 8 + kq + e;
            bias[j][e] = n < OUT ? th[boff + n] : 0.f;
        }
    const int CT = img_ct(A.C);
    __syncthreads();
#pragma unroll 1
    for (int mt = 0; mt < 2; ++mt) {
        const int row = tile_r + warp * 32 + mt * 16 + rq;  // and row + 8
        uint32_t af[16][4];
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (s < KS) {
                const uint8_t* p0 = A.p + img_off(row, s * 16, CT) + kq * 2;
                const uint8_t* p1 = A.p + img_off(row, s * 16 + 8, CT) + kq * 2;
                af[s][0] = *reinterpret_cast<const uint32_t*>(p0);
                af[s][1] = *reinterpret_cast<const uint32_t*>(p0 + 2048);  // row + 8: next core-matrix row group
                af[s][2] = *reinterpret_cast<const uint32_t*>(p1);
                af[s][3] = *reinterpret_cast<const uint32_t*>(p1 + 2048);
            }
        float c[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (s < KS)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const uint2 b = sb[s][j][lane];
                    asm volatile(
                        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                        "{%8,%9}, {%0,%1,%2,%3};\n"
                        : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                        : "r"(af[s][0]), "r"(af[s][1]), "r"(af[s][2]), "r"(af[s][3]), "r"(b.x), "r"(b.y));
                }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = row + 8 * h - g * Rp;
            if (r >= R) continue;
            float* dst = pre + ((long)g * R + r) * OUT;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int n = j * 8 + kq + e;
                    if (n < OUT) dst[n] = c[j][2 * h + e] + bias[j][e];
                }
        }
    }
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
        MB_CUDA(cudaStreamSynchronize(0));  // legacy-stream fill, before the non-blocking streams use it
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
    MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
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
    const bool mma_out = nd.L >= 2 && H % 16 == 0 && H <= 256 && out <= 16;
    for (int l = 0; l < nd.L - (mma_out ? 1 : 0); ++l) {
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
    if (mma_out) {
        const long woff = nd.woff[nd.L - 1], boff = nd.boff[nd.L - 1];
        const Img& a = A[nd.L - 2];
        const unsigned tiles = (unsigned)((long)G * Rp / 128);
        if (out <= 8)
            k_out_forward<1><<<tiles, 128, 0, s>>>(h.theta, h.ld, woff, boff, H, a, R, Rp, out, d_pre);
        else
            k_out_forward<2><<<tiles, 128, 0, s>>>(h.theta, h.ld, woff, boff, H, a, R, Rp, out, d_pre);
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
