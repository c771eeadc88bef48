// Hypernetwork feature map f(w) (hypernet.cpp:10-17, 92-122): a tanh MLP
// (tanh on the output too) over the K cluster weight vectors. The work is
// tiny (K = 128 rows, widths of a few hundred) and sits on the critical path
// of every minibatch, so the limit is L2 latency, not bandwidth or flops:
// every contraction is one launch of k_dense16, a 16 x 16 output tile per
// CTA (>= 128 CTAs per layer) that stages its whole K extent (in 256-wide
// slices) of both operands in shared memory with one round of loads, then
// one FMA chain per thread. fp32 throughout.
//   forward : per layer Y = tanh(X W^T + b); the last layer also writes the
//             bf16 image of f for the theta GEMM;
//   backward: gz_L = (sum of the split-K partials of M^T gtheta) * tanh';
//             per layer gz_{l-1} = (gz_l W_l) * tanh'(a_l);
//             dW_l = gz_l^T a_l with db_l as an extra all-ones column.
#include <algorithm>

#include "common.cuh"
#include "img.cuh"
#include "kernels.h"

namespace mb200 {

namespace {
constexpr int KC = 256;  // K slice staged per round

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

// 16 rows x kn (<= KC) of one operand into smem, all 16 loads in flight
// before the stores; k-fast thread mapping when k is the unit-stride index
// (coalesced), row-fast when the row is (the transposed operands of dW)
__device__ __forceinline__ void stage16(const float* __restrict__ P, long pr, long pk, int r0, int rlim, int k0,
                                        int kn, int ones_row, float (*S)[KC + 4]) {
    float v[16];
    const bool kfast = pk == 1 || pr != 1;
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int rr = kfast ? i : (t & 15), kk = kfast ? t : (t >> 4) + 16 * i;
        const int r = r0 + rr;
        float x = 0.f;
        if (kk < kn) {
            if (r < rlim) x = P[r * pr + (long)(k0 + kk) * pk];
            else if (r == ones_row) x = 1.f;
        }
        v[i] = x;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int rr = kfast ? i : (t & 15), kk = kfast ? t : (t >> 4) + 16 * i;
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

void dense16(const Dense16& d, cudaStream_t s) {
    const int ncols = d.N + (d.ones_col ? 1 : 0);
    dim3 grid((ncols + 15) / 16, (d.R + 15) / 16);
    k_dense16<<<grid, 256, 0, s>>>(d);
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
// The whole two-layer feature map (one hidden layer: [m, H, F]) in ONE
// launch: block (row block rb of 8 clusters, column block cb of 64 outputs,
// net z) computes the hidden layer for its 8 rows (K = m: a few FMAs per
// output, recomputed by the F / 64 column blocks instead of a second launch)
// and its 64 outputs of the last layer from a transposed shared-memory copy
// of the W_1 slice (coalesced loads, conflict-free reads). Every output is a
// fixed-order fp32 FMA chain. Writes act[1] (column block 0), act[2] and the
// bf16 image of f.
constexpr int F2_ROWS = 8, F2_COLS = 64, F2_HMAX = 256;
struct Feat2Job {
    const float* p;  // flat hypernet params (feature block first)
    const float* w;  // cluster weights [G][m]
    int G, m, H, F;
    long woff0, boff0, woff1, boff1;
    float *act1, *act2;  // [G][H], [G][F]
    Img fimg;
    int r0, rn;
};
struct Feat2Batch {
    Feat2Job j[2];
};
__global__ void __launch_bounds__(256) k_feature_fwd2(const __grid_constant__ Feat2Batch b) {
    extern __shared__ float fsm[];
    const Feat2Job& J = b.j[blockIdx.z];
    const int H = J.H, m = J.m;
    float* Ws = fsm;                           // [H][F2_COLS + 1] W_1 slice, transposed
    float* A1 = fsm + F2_HMAX * (F2_COLS + 1);  // [F2_ROWS][H]
    float* Wv = A1 + F2_ROWS * F2_HMAX;         // [F2_ROWS][m]
    const int r0 = blockIdx.x * F2_ROWS, c0 = blockIdx.y * F2_COLS;
    const int t = threadIdx.x;
    if (r0 >= J.G || c0 >= J.F) return;
    pdl_enter();
    // W_1 [F][H] rows c0.. (k fastest: coalesced) -> Ws[k][c]
    const float* W1 = J.p + J.woff1;
    for (int e = t; e < F2_COLS * H; e += 256) {
        const int c = e / H, k = e - c * H;
        Ws[k * (F2_COLS + 1) + c] = c0 + c < J.F ? W1[(long)(c0 + c) * H + k] : 0.f;
    }
    for (int e = t; e < F2_ROWS * m; e += 256) {
        const int r = e / m;
        Wv[e] = r0 + r < J.G ? J.w[(long)(r0 + r) * m + (e - r * m)] : 0.f;
    }
    __syncthreads();
    // hidden layer: a1[r][k] = tanh(b0[k] + sum_i W0[k][i] w[r][i])
    const float* W0 = J.p + J.woff0;
    const float* b0 = J.p + J.boff0;
    for (int e = t; e < F2_ROWS * H; e += 256) {
        const int r = e / H, k = e - r * H;
        float acc = b0[k];
        for (int i = 0; i < m; ++i) acc = fmaf(W0[(long)k * m + i], Wv[r * m + i], acc);
        const float a = tanhf(acc);
        A1[r * F2_HMAX + k] = a;
        if (blockIdx.y == 0 && r0 + r < J.G) J.act1[(long)(r0 + r) * H + k] = a;
    }
    __syncthreads();
    // last layer: thread (c = t % 64, rows 2 (t / 64), + 1)
    const int c = t & (F2_COLS - 1), rp = (t >> 6) * 2;
    const int col = c0 + c;
    if (col >= J.F) return;
    const float bb = J.p[J.boff1 + col];
    float acc0 = bb, acc1 = bb;
    const float* x0 = A1 + rp * F2_HMAX;
    const float* x1 = x0 + F2_HMAX;
    for (int k = 0; k < H; ++k) {
        const float wk = Ws[k * (F2_COLS + 1) + c];
        acc0 = fmaf(wk, x0[k], acc0);
        acc1 = fmaf(wk, x1[k], acc1);
    }
    const int CT = img_ct(J.fimg.C);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = r0 + rp + h;
        if (r >= J.G) continue;
        const float f = tanhf(h ? acc1 : acc0);
        J.act2[(long)r * J.F + col] = f;
        if (J.fimg.p && r >= J.r0 && r < J.r0 + J.rn)
            *reinterpret_cast<__nv_bfloat16*>(J.fimg.p + img_off(r - J.r0, col, CT)) = __float2bfloat16_rn(f);
    }
}
// The dense part of the two-layer feature map's backward in ONE launch
// (after gz_1 = (sum of the split-K partials of M^T gtheta) * tanh'):
//   type A blocks (32 x 32 tiles): dW_1[f][h] = sum_g gz_1[g][f] a_1[g][h],
//     db_1[f] = sum_g gz_1[g][f] (the h-tile-0 blocks);
//   type B blocks (8 hidden columns h): gz_0[g][h] = (sum_f gz_1[g][f]
//     W_1[f][h]) (1 - a_1[g][h]^2) for every cluster g, then
//     dW_0[h][i] = sum_g gz_0[g][h] w[g][i] and db_0[h] = sum_g gz_0[g][h]
//     in the same block (the dependency that took a second launch).
// Every sum runs over g (or f) in order with one fp32 FMA chain.
constexpr int B2_T = 32, B2_H = 8, B2_G = 32;
struct Bwd2Job {
    const float* p;   // flat params
    const float* w;   // [G][m]
    const float* gz1; // [G][F]
    const float* a1;  // [G][H]
    float* gz0;       // [G][H] (written for inspection)
    float* gout;      // flat grad
    int G, m, H, F;
    long woff0, boff0, woff1, boff1;
};
struct Bwd2Batch {
    Bwd2Job j[2];
    int nA[2];  // type A blocks of each job (the rest of grid.x are type B)
};
constexpr size_t B2_SMEM = sizeof(float) * (F2_HMAX * (B2_H + 1) + B2_G * (F2_HMAX + 1) + 1024 * B2_H);
__global__ void __launch_bounds__(256) k_feature_bwd2(const __grid_constant__ Bwd2Batch b) {
    extern __shared__ float bsm[];
    // type A: two staged [32][33] tiles; type B: W_1 columns, gz_1 rows, gz_0 (G <= 1024)
    float(*sA)[B2_T + 1] = reinterpret_cast<float(*)[B2_T + 1]>(bsm);
    float(*sB)[B2_T + 1] = reinterpret_cast<float(*)[B2_T + 1]>(bsm + B2_G * (B2_T + 1));
    float(*sW)[B2_H + 1] = reinterpret_cast<float(*)[B2_H + 1]>(bsm);
    float(*sGz)[F2_HMAX + 1] = reinterpret_cast<float(*)[F2_HMAX + 1]>(bsm + F2_HMAX * (B2_H + 1));
    float(*sG0)[B2_H] = reinterpret_cast<float(*)[B2_H]>(bsm + F2_HMAX * (B2_H + 1) + B2_G * (F2_HMAX + 1));
    const Bwd2Job& J = b.j[blockIdx.z];
    const int nA = b.nA[blockIdx.z];
    const int t = threadIdx.x;
    const int G = J.G, H = J.H, F = J.F, m = J.m;
    pdl_enter();
    if ((int)blockIdx.x < nA) {  // ---- type A: dW_1 tile (+ db_1)
        const int ntf = (F + B2_T - 1) / B2_T;
        const int f0 = (blockIdx.x % ntf) * B2_T, h0 = (blockIdx.x / ntf) * B2_T;
        const int fl = t >> 3, hl = (t & 7) * 4;
        float acc[4] = {0.f, 0.f, 0.f, 0.f}, accb = 0.f;
        for (int g0 = 0; g0 < G; g0 += B2_G) {
            for (int e = t; e < B2_G * B2_T; e += 256) {
                const int gg = e / B2_T, c = e - gg * B2_T;
                const bool ok = g0 + gg < G;
                sA[gg][c] = ok && f0 + c < F ? J.gz1[(long)(g0 + gg) * F + f0 + c] : 0.f;
                sB[gg][c] = ok && h0 + c < H ? J.a1[(long)(g0 + gg) * H + h0 + c] : 0.f;
            }
            __syncthreads();
            const int gn = min(B2_G, G - g0);
            for (int gg = 0; gg < gn; ++gg) {
                const float x = sA[gg][fl];
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[i] = fmaf(x, sB[gg][hl + i], acc[i]);
                accb += x;
            }
            __syncthreads();
        }
        const int f = f0 + fl;
        if (f < F) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (h0 + hl + i < H) J.gout[J.woff1 + (long)f * H + h0 + hl + i] = acc[i];
            if (h0 == 0 && hl == 0) J.gout[J.boff1 + f] = accb;
        }
        return;
    }
    // ---- type B: gz_0 for hidden columns [h0, h0 + 8) of every cluster, then dW_0 / db_0
    const int h0 = ((int)blockIdx.x - nA) * B2_H;
    const float* W1 = J.p + J.woff1;  // [F][H]
    for (int e = t; e < F * B2_H; e += 256) {
        const int f = e / B2_H, hh = e - f * B2_H;
        sW[f][hh] = h0 + hh < H ? W1[(long)f * H + h0 + hh] : 0.f;
    }
    const int hh = t & (B2_H - 1), gl = t >> 3;  // 8 columns x 32 clusters per pass
    for (int g0 = 0; g0 < G; g0 += B2_G) {
        __syncthreads();
        for (int e = t; e < B2_G * F; e += 256) {
            const int gg = e / F, f = e - gg * F;
            sGz[gg][f] = g0 + gg < G ? J.gz1[(long)(g0 + gg) * F + f] : 0.f;
        }
        __syncthreads();
        const int g = g0 + gl;
        if (g < G && h0 + hh < H) {
            float acc = 0.f;
            for (int f = 0; f < F; ++f) acc = fmaf(sGz[gl][f], sW[f][hh], acc);
            const float a = J.a1[(long)g * H + h0 + hh];
            const float v = acc * (1.f - a * a);
            sG0[g][hh] = v;
            J.gz0[(long)g * H + h0 + hh] = v;
        }
    }
    __syncthreads();
    // dW_0[h][i] = sum_g gz_0[g][h] w[g][i]; db_0[h] (i == m): one output per thread
    for (int e = t; e < B2_H * (m + 1); e += 256) {
        const int hc = e / (m + 1), i = e - hc * (m + 1);
        const int h = h0 + hc;
        if (h >= H) continue;
        float acc = 0.f;
        if (i < m)
            for (int g = 0; g < G; ++g) acc = fmaf(sG0[g][hc], J.w[(long)g * m + i], acc);
        else
            for (int g = 0; g < G; ++g) acc += sG0[g][hc];
        if (i < m)
            J.gout[J.woff0 + (long)h * m + i] = acc;
        else
            J.gout[J.boff0 + h] = acc;
    }
}
}  // namespace

void feature_forward_multi(const FeatJob* jobs, int nj, cudaStream_t s) {
    const int L = jobs[0].fd->L;
    for (int k = 1; k < nj; ++k)
        if (jobs[k].fd->L != L) throw ShapeError("feature_forward_multi: the feature maps must have equal depth");
    bool fused = L == 2 && nj <= 2;
    for (int k = 0; k < nj; ++k) fused = fused && jobs[k].fd->sz[1] <= F2_HMAX && jobs[k].fd->sz[0] <= 8;
    if (fused) {  // one launch for the whole map (both nets)
        Feat2Batch fb{};
        int gmax = 0, fmax = 0;
        for (int k = 0; k < nj; ++k) {
            const FeatJob& j = jobs[k];
            const FeatDims& fd = *j.fd;
            fb.j[k] = Feat2Job{j.p, j.w, j.G, fd.sz[0], fd.sz[1], fd.sz[2], fd.woff[0], fd.boff[0], fd.woff[1],
                               fd.boff[1], fd.act[1], fd.act[2], j.fimg, j.r0, j.rn};
            gmax = std::max(gmax, j.G);
            fmax = std::max(fmax, fd.sz[2]);
        }
        const size_t smem = sizeof(float) * (F2_HMAX * (F2_COLS + 1) + F2_ROWS * F2_HMAX + F2_ROWS * 8);
        ensure_smem((const void*)k_feature_fwd2, smem);
        launch_pdl(k_feature_fwd2, dim3((gmax + F2_ROWS - 1) / F2_ROWS, (fmax + F2_COLS - 1) / F2_COLS, nj),
                   dim3(256), smem, s, fb);
        MB_LAUNCH();
        return;
    }
    for (int l = 0; l < L; ++l) {
        Dense16 ds[4];
        for (int k = 0; k < nj; ++k) {
            const FeatJob& j = jobs[k];
            const FeatDims& fd = *j.fd;
            Dense16 d{};
            d.A = l == 0 ? j.w : fd.act[l];  // act[0] is not materialised: w is the input
            d.ar = fd.sz[l]; d.ak = 1;
            d.B = j.p + fd.woff[l]; d.bc = fd.sz[l]; d.bk = 1;  // W [out][in]
            d.R = j.G; d.N = fd.sz[l + 1]; d.K = fd.sz[l];
            d.bias = j.p + fd.boff[l];
            d.act = 1;
            d.C = fd.act[l + 1]; d.cr = fd.sz[l + 1]; d.cc = 1;
            if (l == L - 1) {
                d.img = j.fimg;
                d.img_r0 = j.r0;
                d.img_rn = j.rn;
            }
            ds[k] = d;
        }
        dense16_multi(ds, nj, s);
    }
}

void feature_forward(const FeatDims& fd, const float* p, const float* w, int G, const Img& fimg, int r0, int rn,
                     cudaStream_t s) {
    FeatJob j{&fd, p, w, G, fimg, r0, rn, nullptr, 0, nullptr};
    feature_forward_multi(&j, 1, s);
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
    bool fused = L == 2 && nj <= 2;
    for (int k = 0; k < nj; ++k)
        fused = fused && jobs[k].fd->sz[1] <= F2_HMAX && jobs[k].fd->sz[2] <= F2_HMAX && jobs[k].G <= 1024;
    if (fused) {  // the dense part in one launch (both nets)
        Bwd2Batch bb{};
        int nmax = 0;
        for (int k = 0; k < nj; ++k) {
            const FeatJob& j = jobs[k];
            const FeatDims& fd = *j.fd;
            const int H = fd.sz[1], F = fd.sz[2];
            bb.j[k] = Bwd2Job{j.p, j.w, fd.gz[1], fd.act[1], fd.gz[0], j.gout, j.G, fd.sz[0], H, F,
                              fd.woff[0], fd.boff[0], fd.woff[1], fd.boff[1]};
            bb.nA[k] = ((F + B2_T - 1) / B2_T) * ((H + B2_T - 1) / B2_T);
            nmax = std::max(nmax, bb.nA[k] + (H + B2_H - 1) / B2_H);
        }
        ensure_smem((const void*)k_feature_bwd2, B2_SMEM);
        launch_pdl(k_feature_bwd2, dim3(nmax, 1, nj), dim3(256), B2_SMEM, s, bb);
        MB_LAUNCH();
        return;
    }
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

void feature_backward(const FeatDims& fd, const float* p, const float* w, const float* parts, int splits, int G,
                      float* gout, cudaStream_t s) {
    FeatJob j{&fd, p, w, G, Img{}, 0, 0, parts, splits, gout};
    feature_backward_multi(&j, 1, s, 0);
}

}  // namespace mb200
