// Hypernetwork feature map f(w) (hypernet.cpp:10-17, 92-122): a tanh MLP
// (tanh on the output too) over the K cluster weight vectors. The work is
// tiny (K = 128 rows, widths of a few hundred) and sits on the critical path
// of every minibatch, so the limit is L2 latency, not bandwidth or flops.
// fp32 throughout.
//   forward : all layers in one launch (k_feat_fwd, a block per 4 clusters,
//             activations in shared memory): per layer Y = tanh(X W^T + b);
//             the last layer also writes the bf16 image of f for the theta GEMM;
//   backward: every contraction is one launch of k_dense16, a 16 x 16 output
//             tile per CTA (>= 128 CTAs per layer) that stages its whole K
//             extent (in 256-wide slices) of both operands in shared memory
//             with one round of loads, then one FMA chain per thread;
//             gz_L = (sum of the split-K partials of M^T gtheta) * tanh';
//             per layer gz_{l-1} = (gz_l W_l) * tanh'(a_l);
//             dW_l = gz_l^T a_l with db_l as an extra all-ones column.
#include <algorithm>

#include "common.cuh"
#include "img.cuh"
#include "kernels.h"

namespace mb200 {

namespace {
constexpr int KC = 64;  // K slice staged per round (8.5 KB of shared memory: fits beside the optimizer)

struct Dense16 {
    const float* A;  // A(r, k) = A[r * ar + k * ak]
    long ar, ak;
    const float* B;  // B(c, k) = B[c * bc + k * bk]; c == N -> 1 when ones_col
    long bc, bk;
    int R, N, K;
    const float* bias;  // [N] or null
    int act;            // 0 none, 1 tanh, 2 * (1 - aux^2)
    const float* aux;   // aux(r, c) = aux[r * xr + c]
    long xr;
    float* C;           // C(r, c) = C[r * cr + c * cc]
    long cr, cc;
    int ones_col;       // column N of the output = sum_k A(r, k) -> Cb[r]
    float* Cb;
    Img img;            // optional bf16 image copy of the output (row r - img_r0, col c)
    int img_r0, img_rn; // rows [img_r0, img_r0 + img_rn) go to the image
};

// 16 rows x kn (<= KC) of one operand into smem, all of a thread's loads in
// flight before the stores; k-fast thread mapping when k is the unit-stride
// index (coalesced), row-fast when the row is (the transposed operands of dW)
__device__ __forceinline__ void stage16(const float* __restrict__ P, long pr, long pk, int r0, int rlim, int k0,
                                        int kn, int ones_row, float (*S)[KC + 4]) {
    constexpr int PER = 16 * KC / 256;  // elements per thread
    float v[PER];
    const bool kfast = pk == 1 || pr != 1;
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = t + 256 * i;
        const int rr = kfast ? e / KC : (e & 15), kk = kfast ? e % KC : (e >> 4);
        const int r = r0 + rr;
        float x = 0.f;
        if (kk < kn) {
            if (r < rlim) x = P[r * pr + (long)(k0 + kk) * pk];
            else if (r == ones_row) x = 1.f;
        }
        v[i] = x;
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = t + 256 * i;
        const int rr = kfast ? e / KC : (e & 15), kk = kfast ? e % KC : (e >> 4);
        S[rr][kk] = v[i];
    }
}

__device__ void dense16_tile(const Dense16& d, int bx, int by, float (*As)[KC + 4], float (*Bs)[KC + 4]) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int r0 = by * 16, c0 = bx * 16;
    const int ncols = d.N + (d.ones_col ? 1 : 0);
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    for (int k0 = 0; k0 < d.K; k0 += KC) {
        const int kn = min(KC, d.K - k0);
        stage16(d.A, d.ar, d.ak, r0, d.R, k0, kn, -1, As);
        stage16(d.B, d.bc, d.bk, c0, d.N, k0, kn, d.ones_col ? d.N : -1, Bs);
        __syncthreads();
        const float4* a4 = reinterpret_cast<const float4*>(As[ty]);
        const float4* b4 = reinterpret_cast<const float4*>(Bs[tx]);
        for (int q = 0; q < (kn + 3) / 4; ++q) {  // zero-filled past kn
            const float4 a = a4[q], b = b4[q];
            acc0 = fmaf(a.x, b.x, acc0);
            acc1 = fmaf(a.y, b.y, acc1);
            acc2 = fmaf(a.z, b.z, acc2);
            acc3 = fmaf(a.w, b.w, acc3);
        }
        __syncthreads();
    }
    const float acc = (acc0 + acc1) + (acc2 + acc3);
    const int r = r0 + ty, c = c0 + tx;
    if (r >= d.R || c >= ncols) return;
    float v = acc;
    if (c == d.N) {  // ones column: row sums of A (bias gradients)
        d.Cb[r] = v;
        return;
    }
    if (d.bias) v += d.bias[c];
    if (d.act == 1) {
        v = tanhf(v);
    } else if (d.act == 2) {
        const float a = d.aux[r * d.xr + c];
        v *= 1.f - a * a;
    }
    d.C[r * d.cr + c * d.cc] = v;
    if (d.img.p && r >= d.img_r0 && r < d.img_r0 + d.img_rn)
        *reinterpret_cast<__nv_bfloat16*>(d.img.p + img_off(r - d.img_r0, c, img_ct(d.img.C))) = __float2bfloat16_rn(v);
}

__global__ void __launch_bounds__(256) k_dense16(Dense16 d) {
    __shared__ __align__(16) float As[16][KC + 4];
    __shared__ __align__(16) float Bs[16][KC + 4];
    dense16_tile(d, blockIdx.x, blockIdx.y, As, Bs);
}

// up to 4 independent contractions in one launch (tile ranges per descriptor)
struct DenseBatch {
    Dense16 d[4];
    int n = 0;
    int base[5] = {0, 0, 0, 0, 0};
    int nx[4] = {1, 1, 1, 1};
};
__global__ void __launch_bounds__(256) k_dense16_multi(const __grid_constant__ DenseBatch b) {
    pdl_enter();
    __shared__ __align__(16) float As[16][KC + 4];
    __shared__ __align__(16) float Bs[16][KC + 4];
    const int t = blockIdx.x;
    int k = 0;
    while (k + 1 < b.n && t >= b.base[k + 1]) ++k;
    const int u = t - b.base[k];
    dense16_tile(b.d[k], u % b.nx[k], u / b.nx[k], As, Bs);
}
void dense16_multi(const Dense16* ds, int n, cudaStream_t s) {
    DenseBatch b;
    b.n = n;
    for (int k = 0; k < n; ++k) {
        b.d[k] = ds[k];
        b.nx[k] = (ds[k].N + (ds[k].ones_col ? 1 : 0) + 15) / 16;
        b.base[k + 1] = b.base[k] + b.nx[k] * ((ds[k].R + 15) / 16);
    }
    if (b.base[n] == 0) return;
    launch_pdl(k_dense16_multi, dim3(b.base[n]), dim3(256), 0, s, b);
    MB_LAUNCH();
}

// gz[g][j] = (sum_k parts[k][g][j]) * (1 - f[g][j]^2); 4 threads per output
// (split slices) so 4x more loads are in flight, combined in a fixed order
__global__ void __launch_bounds__(256) k_split_dtanh(const float* __restrict__ parts, int splits, long n,
                                                     const float* __restrict__ f, float* gz) {
    pdl_enter();
    __shared__ float part[4][64];
    const int ol = threadIdx.x & 63, sl = threadIdx.x >> 6;
    const long i = blockIdx.x * 64L + ol;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if (i < n) {
        const int ks = (splits + 3) / 4, k0 = sl * ks, k1 = min(splits, k0 + ks);
        int k = k0;
        for (; k + 4 <= k1; k += 4) {
            a0 += parts[(long)k * n + i];
            a1 += parts[(long)(k + 1) * n + i];
            a2 += parts[(long)(k + 2) * n + i];
            a3 += parts[(long)(k + 3) * n + i];
        }
        for (; k < k1; ++k) a0 += parts[(long)k * n + i];
    }
    part[sl][ol] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (sl == 0 && i < n) {
        const float x = f[i];
        gz[i] = ((part[0][ol] + part[1][ol]) + (part[2][ol] + part[3][ol])) * (1.f - x * x);
    }
}

// The whole forward of the feature map in one launch (hypernet.cpp:10-17):
// a block per kFfClusters clusters (both maps' blocks side by side in y)
// keeps its rows' activations in shared memory, layer after layer. A warp
// computes kFfRows output features of the block's clusters at a time: lanes
// split K in float4 pieces (scalar when a row is not 16-byte aligned), the
// 16 partial dot products per lane go through one reduce-scatter shuffle
// tree (16 shuffles), and lane 2q ends with (feature q / kFfClusters,
// cluster q % kFfClusters). Little shared memory (4 KB at width 256).
constexpr int kFfClusters = 2, kFfWarps = 16, kFfRows = 16 / kFfClusters;
struct FeatFwdJob {
    FeatDims fd;
    const float* p;
    const float* w;
    int G;
    Img fimg;
    int r0, rn;
};
struct FeatFwdArgs {
    FeatFwdJob job[2];
    int nj = 1, maxw = 0;
};
__global__ void __launch_bounds__(32 * kFfWarps) k_feat_fwd(const __grid_constant__ FeatFwdArgs a) {
    extern __shared__ __align__(16) float fsm[];
    const FeatFwdJob& J = a.job[blockIdx.y];
    const FeatDims& fd = J.fd;
    const int g0 = blockIdx.x * kFfClusters;
    if (g0 >= J.G) return;
    const int nc = min(kFfClusters, J.G - g0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* cur = fsm;                            // [kFfClusters][maxw]
    float* nxt = fsm + kFfClusters * a.maxw;
    pdl_enter();
    for (int e = threadIdx.x; e < kFfClusters * a.maxw; e += blockDim.x) {
        const int c = e / a.maxw, k = e - c * a.maxw;
        cur[e] = (c < nc && k < fd.sz[0]) ? J.w[(long)(g0 + c) * fd.sz[0] + k] : 0.f;
    }
    __syncthreads();
    for (int l = 0; l < fd.L; ++l) {
        const int in = fd.sz[l], out = fd.sz[l + 1];
        const float* W = J.p + fd.woff[l];
        const float* bias = J.p + fd.boff[l];
        const bool vec = (in & 3) == 0 && (fd.woff[l] & 3) == 0;
        for (int j0 = warp * kFfRows; j0 < out; j0 += kFfWarps * kFfRows) {
            float s[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) s[q] = 0.f;
            if (vec) {
                for (int k = lane * 4; k < in; k += 128) {
                    float4 xv[kFfClusters];
#pragma unroll
                    for (int c = 0; c < kFfClusters; ++c) xv[c] = *reinterpret_cast<const float4*>(cur + c * a.maxw + k);
#pragma unroll
                    for (int r = 0; r < kFfRows; ++r) {
                        const float4 wv = j0 + r < out ? __ldg(reinterpret_cast<const float4*>(W + (long)(j0 + r) * in + k))
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < kFfClusters; ++c) {
                            float t = s[r * kFfClusters + c];
                            t = fmaf(wv.x, xv[c].x, t);
                            t = fmaf(wv.y, xv[c].y, t);
                            t = fmaf(wv.z, xv[c].z, t);
                            t = fmaf(wv.w, xv[c].w, t);
                            s[r * kFfClusters + c] = t;
                        }
                    }
                }
            } else {
                for (int k = lane; k < in; k += 32) {
#pragma unroll
                    for (int r = 0; r < kFfRows; ++r) {
                        const float wv = j0 + r < out ? __ldg(W + (long)(j0 + r) * in + k) : 0.f;
#pragma unroll
                        for (int c = 0; c < kFfClusters; ++c)
                            s[r * kFfClusters + c] = fmaf(wv, cur[c * a.maxw + k], s[r * kFfClusters + c]);
                    }
                }
            }
            // reduce-scatter of the 16 sums over the warp (fixed order)
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1) {
                const bool up = (lane & (2 * w)) != 0;
#pragma unroll
                for (int i = 0; i < w; ++i) {
                    const float mine = up ? s[w + i] : s[i];
                    const float other = up ? s[i] : s[w + i];
                    s[i] = mine + __shfl_xor_sync(0xffffffffu, other, 2 * w);
                }
            }
            s[0] += __shfl_xor_sync(0xffffffffu, s[0], 1);
            const int q = (lane >> 1) & 15, r = q / kFfClusters, c = q % kFfClusters, j = j0 + r;
            if ((lane & 1) == 0 && j < out && c < nc) {
                const float v = tanhf(s[0] + bias[j]);
                nxt[c * a.maxw + j] = v;
                const int g = g0 + c;
                fd.act[l + 1][(long)g * out + j] = v;
                if (l == fd.L - 1 && J.fimg.p && g >= J.r0 && g < J.r0 + J.rn)
                    *reinterpret_cast<__nv_bfloat16*>(J.fimg.p + img_off(g - J.r0, j, img_ct(J.fimg.C))) =
                        __float2bfloat16_rn(v);
            }
        }
        __syncthreads();
        float* t = cur;  // (rows of clusters >= nc are never written: they only feed sums that are dropped)
        cur = nxt;
        nxt = t;
    }
}
}  // namespace

void feature_forward_multi(const FeatJob* jobs, int nj, cudaStream_t s) {
    if (nj < 1 || nj > 2) throw ShapeError("feature_forward_multi: one or two feature maps");
    FeatFwdArgs a;
    a.nj = nj;
    int maxw = 0, nb = 0;
    for (int k = 0; k < nj; ++k) {
        const FeatJob& j = jobs[k];
        if (j.fd->L != jobs[0].fd->L) throw ShapeError("feature_forward_multi: the feature maps must have equal depth");
        a.job[k] = FeatFwdJob{*j.fd, j.p, j.w, j.G, j.fimg, j.r0, j.rn};
        for (int l = 0; l <= j.fd->L; ++l) maxw = std::max(maxw, j.fd->sz[l]);
        nb = std::max(nb, (j.G + kFfClusters - 1) / kFfClusters);
    }
    a.maxw = (maxw + 3) & ~3;
    if (nb == 0) return;
    const size_t smem = sizeof(float) * 2 * kFfClusters * a.maxw;
    if (smem > 48 * 1024) throw ShapeError("feature_forward_multi: feature width above 1536");
    launch_pdl(k_feat_fwd, dim3((unsigned)nb, (unsigned)nj), dim3(32 * kFfWarps), smem, s, a);
    MB_LAUNCH();
}

void feature_backward_multi(const FeatJob* jobs, int nj, cudaStream_t s, int stage) {
    const int L = jobs[0].fd->L;
    for (int k = 0; k < nj; ++k) {
        const FeatJob& j = jobs[k];
        if (j.fd->L != L) throw ShapeError("feature_backward_multi: the feature maps must have equal depth");
        if (stage == 2) continue;
        const long n = (long)j.G * j.fd->sz[L];
        launch_pdl(k_split_dtanh, dim3((unsigned)((n + 63) / 64)), dim3(256), 0, s, j.parts, j.splits, n,
                   (const float*)j.fd->act[L], j.fd->gz[L - 1]);
        MB_LAUNCH();
    }
    if (stage == 1) return;
    for (int l = L - 1; l >= 0; --l) {
        Dense16 ds[4];
        int nd = 0;
        for (int k = 0; k < nj; ++k) {
            const FeatJob& j = jobs[k];
            const FeatDims& fd = *j.fd;
            const int in = fd.sz[l], out = fd.sz[l + 1];
            const float* a_in = l == 0 ? j.w : fd.act[l];
            Dense16 d{};  // dW[j][i] = sum_g gz[g][j] a[g][i]; db[j] = sum_g gz[g][j]
            d.A = fd.gz[l]; d.ar = 1; d.ak = out;
            d.B = a_in; d.bc = 1; d.bk = in;
            d.R = out; d.N = in; d.K = j.G;
            d.C = j.gout + fd.woff[l]; d.cr = in; d.cc = 1;
            d.ones_col = 1; d.Cb = j.gout + fd.boff[l];
            ds[nd++] = d;
            if (l > 0) {  // independent of dW_l: same launch
                Dense16 e{};  // gz_{l-1}[g][i] = (sum_j gz_l[g][j] W[j][i]) (1 - a_l[g][i]^2)
                e.A = fd.gz[l]; e.ar = out; e.ak = 1;
                e.B = j.p + fd.woff[l]; e.bc = 1; e.bk = in;
                e.R = j.G; e.N = in; e.K = out;
                e.act = 2; e.aux = fd.act[l]; e.xr = in;
                e.C = fd.gz[l - 1]; e.cr = in; e.cc = 1;
                ds[nd++] = e;
            }
        }
        dense16_multi(ds, nd, s);
    }
}

}  // namespace mb200
