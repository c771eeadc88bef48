// tcgen05 GEMM v2: D(m, n) = sum_k A(m, k) B(n, k) over tiled bf16 images
// (img.cuh), every operand chunk brought in by the TMA bulk-copy engine.
//
//   * CTA tile 128 x BN (BN <= 256), K in chunks of 128, S-stage smem ring;
//   * thread 0 = producer: cp.async.bulk of the A chunk and the B chunk(s)
//     of K-chunk kc into stage kc % S, completion on full[s] (expect_tx);
//   * thread 32 = MMA issuer: waits full[s], issues 8 x (K = 16)
//     tcgen05.mma per B chunk, tcgen05.commit -> empty[s] frees the stage,
//     a final commit -> done;
//   * all 8 warps: epilogue from TMEM (32 lanes x 16 columns per tcgen05.ld)
//     with bias / tanh / tanh-derivative (aux image) / accumulate, writing
//     fp32 (strided) and/or a bf16 image (for the next GEMM).
// Grouped modes: gmode 1 = rows grouped (A rows and output rows start at
// goff[z], 128-aligned; B / bias per group), gmode 2 = K grouped (K range
// [goff[z], goff[z+1]), 128-aligned; output per group).
#include "common.cuh"
#include "img.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

namespace {
constexpr int NT = 256;
constexpr int CHUNK = 32768;

template <int BN>
struct Cfg {
    static constexpr int NB = BN > 128 ? 2 : 1;          // B chunks per stage
    static constexpr int STAGES = BN > 128 ? 2 : 3;
    static constexpr int STAGE = CHUNK * (1 + NB);
    static constexpr int SMEM = STAGES * STAGE + 256;
    static constexpr int NMMA = BN > 128 ? 128 : BN;      // N per MMA instruction
};

__device__ __forceinline__ long chunk_index(int view, int mt, int kc, int CT) {
    // view 0: (row tile = mt, col tile = kc); view 1: (row tile = kc, col tile = mt)
    return view == 0 ? (long)mt * CT + kc : (long)kc * CT + mt;
}

template <int BN>
__global__ void __launch_bounds__(NT, 1) k_img_gemm(IGemm d) {
    using C = Cfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* done = empty + C::STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

    const int z = blockIdx.z;
    int m_lo = 0, m_hi = d.M, k_lo = 0, k_hi = d.K;
    const uint8_t* Ab = d.A.p;
    const uint8_t* Bb = d.B.p;
    const float* bias = d.bias;
    long cz = 0, oz = 0;
    if (d.gmode == 0) {
        Ab += z * d.A.gs;
        Bb += z * d.B.gs;
        if (bias) bias += z * d.bias_gs;
        cz = z;
    } else if (d.gmode == 1) {
        m_lo = d.goff[z];
        m_hi = d.goff[z + 1];
        Bb += z * d.B.gs;
        if (bias) bias += z * d.bias_gs;
    } else {
        k_lo = d.goff[z];
        k_hi = d.goff[z + 1];
        cz = z;
    }
    oz = z;
    const int m0 = m_lo + blockIdx.y * 128;
    const int n0 = blockIdx.x * BN;
    if (m0 >= m_hi || n0 >= d.N) return;
    const int nk = (k_hi - k_lo + 127) >> 7;
    const int kc0 = k_lo >> 7;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kCols = BN < 32 ? 32 : BN;

    if (warp == 0) umma::tmem_alloc(tslot, kCols);
    if (threadIdx.x == 32) {
        for (int s = 0; s < C::STAGES; ++s) {
            umma::mbar_init(&full[s], 1);
            umma::mbar_init(&empty[s], 1);
        }
        umma::mbar_init(done, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tbase = *tslot;
    const int CTa = img_ct(d.A.C), CTb = img_ct(d.B.C);
    const int mt = m0 >> 7;
    const int nt0 = n0 >> 7;

    if (threadIdx.x == 0) {  // ---------------- producer
        // B bytes per chunk: a row-view operand narrower than 128 only needs
        // the first BN/8 row blocks of its chunk
        const uint32_t bbytes = (d.b_view == 0 && BN < 128) ? (uint32_t)BN * 256 : (uint32_t)CHUNK;
        for (int kc = 0; kc < nk; ++kc) {
            const int s = kc % C::STAGES;
            if (kc >= C::STAGES) umma::mbar_wait(&empty[s], ((kc / C::STAGES) - 1) & 1);
            uint8_t* st = smem + s * C::STAGE;
            umma::mbar_arrive_expect_tx(&full[s], CHUNK + C::NB * bbytes);
            umma::bulk_g2s(st, Ab + chunk_index(d.a_view, mt, kc0 + kc, CTa) * CHUNK, CHUNK, &full[s]);
            for (int j = 0; j < C::NB; ++j)
                umma::bulk_g2s(st + CHUNK * (1 + j), Bb + chunk_index(d.b_view, nt0 + j, kc0 + kc, CTb) * CHUNK,
                               bbytes, &full[s]);
        }
    } else if (threadIdx.x == 32) {  // ---------------- MMA issuer
        const uint32_t idesc = umma::idesc_bf16(128, C::NMMA, d.a_view == 1, d.b_view == 1);
        const uint32_t a_lbo = d.a_view ? 2048 : 128, a_sbo = d.a_view ? 128 : 2048, a_step = d.a_view ? 4096 : 256;
        const uint32_t b_lbo = d.b_view ? 2048 : 128, b_sbo = d.b_view ? 128 : 2048, b_step = d.b_view ? 4096 : 256;
        for (int kc = 0; kc < nk; ++kc) {
            const int s = kc % C::STAGES;
            umma::mbar_wait(&full[s], (kc / C::STAGES) & 1);
            umma::fence_after_sync();
            const uint32_t a0 = umma::smem_u32(smem + s * C::STAGE);
#pragma unroll
            for (int j = 0; j < C::NB; ++j) {
                const uint32_t b0 = a0 + CHUNK * (1 + j);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma::mma_bf16(tbase + j * 128, umma::smem_desc(a0 + kk * a_step, a_lbo, a_sbo),
                                   umma::smem_desc(b0 + kk * b_step, b_lbo, b_sbo), idesc, (kc | kk) ? 1u : 0u);
            }
            umma::commit(&empty[s]);
        }
        umma::commit(done);
    }
    __syncwarp();
    // ---------------- epilogue (all warps)
    if (nk > 0) umma::mbar_wait(done, 0);
    umma::fence_after_sync();
    const int lg = warp & 3, half = warp >> 2;
    const int m = m0 + lg * 32 + lane;
    constexpr int HALF = BN >= 32 ? BN / 2 : BN;
    const bool active = BN >= 32 || half == 0;
    const int CTo = img_ct(d.O.C), CTx = img_ct(d.aux.C);
    if (active) {
        for (int c0 = half * HALF; c0 < half * HALF + HALF; c0 += 16) {
            float v[16];
            if (nk > 0) {
                umma::tmem_ld16(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)c0, v);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            if (m >= m_hi) continue;
            const int nb = n0 + c0;
            // aux (tanh-derivative) values for these 16 columns
            float ax[16];
            if (d.act == 2) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint8_t* ap = d.aux.p + oz * d.aux.gs + img_off(m, nb + 8 * h, CTx);
                    const uint4 q = *reinterpret_cast<const uint4*>(ap);
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __bfloat1622float2(b2[e]);
                        ax[8 * h + 2 * e] = f.x;
                        ax[8 * h + 2 * e + 1] = f.y;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int n = nb + i;
                float x = v[i];
                if (d.bias_mode == 1) x += n < d.N ? bias[n] : 0.f;
                else if (d.bias_mode == 2) x += bias[m];
                if (d.C && d.accumulate && n < d.N) x += d.C[cz * d.c_gs + (long)m * d.cm + (long)n * d.cn];
                if (d.act == 1) {
                    if (d.C2 && n < d.N) d.C2[cz * d.c2_gs + (long)m * d.c2m + (long)n * d.c2n] = x;
                    x = tanhf(x);
                } else if (d.act == 2) {
                    x *= 1.f - ax[i] * ax[i];
                }
                v[i] = x;
                if (d.C && n < d.N) d.C[cz * d.c_gs + (long)m * d.cm + (long)n * d.cn] = x;
            }
            if (d.o_mode == 1) {  // image (row = m, col = n): two 16-B stores
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (nb + 8 * h >= d.N) continue;
                    uint4 q;
                    q.x = umma::pack_bf16(v[8 * h + 0], v[8 * h + 1]);
                    q.y = umma::pack_bf16(v[8 * h + 2], v[8 * h + 3]);
                    q.z = umma::pack_bf16(v[8 * h + 4], v[8 * h + 5]);
                    q.w = umma::pack_bf16(v[8 * h + 6], v[8 * h + 7]);
                    if (nb + 8 * h + 8 > d.N) {  // partial: keep padding columns zero
                        float t[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) t[e] = (nb + 8 * h + e < d.N) ? v[8 * h + e] : 0.f;
                        q.x = umma::pack_bf16(t[0], t[1]);
                        q.y = umma::pack_bf16(t[2], t[3]);
                        q.z = umma::pack_bf16(t[4], t[5]);
                        q.w = umma::pack_bf16(t[6], t[7]);
                    }
                    *reinterpret_cast<uint4*>(d.O.p + oz * d.O.gs + img_off(m, nb + 8 * h, CTo)) = q;
                }
            }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tbase, kCols);
}

template <int BN>
void launch(const IGemm& d, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        MB_CUDA(cudaFuncSetAttribute(k_img_gemm<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
        configured = true;
    }
    const int mext = d.gmode == 1 ? d.max_group : d.M;
    dim3 grid((d.N + BN - 1) / BN, (mext + 127) / 128, d.Z);
    k_img_gemm<BN><<<grid, NT, Cfg<BN>::SMEM, s>>>(d);
    MB_LAUNCH();
}
}  // namespace

void img_gemm(const IGemm& d, cudaStream_t s) {
    if (d.M <= 0 || d.N <= 0 || d.Z <= 0) return;
    if (d.gmode == 1 && d.max_group <= 0) return;
    if (d.N <= 16) launch<16>(d, s);
    else if (d.N <= 32) launch<32>(d, s);
    else if (d.N <= 64) launch<64>(d, s);
    else if (d.N <= 128) launch<128>(d, s);
    else launch<256>(d, s);
}

// ---- image packing / unpacking helpers ------------------------------------
// dst image (row r, col c) <- src[r * ld + c] (fp32), r < R, c < C
__global__ void k_to_img(const float* __restrict__ src, long ld, long src_gs, int R, int C, Img dst) {
    const int z = blockIdx.y;
    const int CT = img_ct(C);
    const long units = (long)R * ((C + 7) / 8);
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < units; u += (long)gridDim.x * blockDim.x) {
        const int r = (int)(u / ((C + 7) / 8)), c = (int)(u % ((C + 7) / 8)) * 8;
        const float* sp = src + z * src_gs + (long)r * ld + c;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = c + e < C ? sp[e] : 0.f;
        uint4 q;
        q.x = umma::pack_bf16(v[0], v[1]);
        q.y = umma::pack_bf16(v[2], v[3]);
        q.z = umma::pack_bf16(v[4], v[5]);
        q.w = umma::pack_bf16(v[6], v[7]);
        *reinterpret_cast<uint4*>(dst.p + z * dst.gs + img_off(r, c, CT)) = q;
    }
}
void to_img(const float* src, long ld, long src_gs, int R, int C, const Img& dst, int G, cudaStream_t s) {
    const long units = (long)R * ((C + 7) / 8);
    if (units == 0) return;
    dim3 grid((unsigned)std::min<long>((units + 255) / 256, 4096), G);
    k_to_img<<<grid, 256, 0, s>>>(src, ld, src_gs, R, C, dst);
    MB_LAUNCH();
}

// gather minibatch rows (row map, -1 = padding) of src[.][width] into an image
__global__ void k_gather_img(const int* rows, int Bp, const float* __restrict__ src, int width, Img dst) {
    const int CT = img_ct(width);
    const int cpr = (width + 7) / 8;
    const long units = (long)Bp * cpr;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < units; u += (long)gridDim.x * blockDim.x) {
        const int q = (int)(u / cpr), c = (int)(u % cpr) * 8;
        const int r = rows[q];
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = (r >= 0 && c + e < width) ? src[(long)r * width + c + e] : 0.f;
        uint4 w;
        w.x = umma::pack_bf16(v[0], v[1]);
        w.y = umma::pack_bf16(v[2], v[3]);
        w.z = umma::pack_bf16(v[4], v[5]);
        w.w = umma::pack_bf16(v[6], v[7]);
        *reinterpret_cast<uint4*>(dst.p + img_off(q, c, CT)) = w;
    }
}
void gather_img(const int* rows, int Bp, const float* src, int width, const Img& dst, cudaStream_t s) {
    const long units = (long)Bp * ((width + 7) / 8);
    if (units == 0) return;
    k_gather_img<<<(unsigned)std::min<long>((units + 255) / 256, 8192), 256, 0, s>>>(rows, Bp, src, width, dst);
    MB_LAUNCH();
}

// fp32 gather with padding (-1 -> 0)
__global__ void k_gather_pad(const int* rows, int Bp, const float* __restrict__ src, int width, float* dst) {
    const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (e >= (long)Bp * width) return;
    const int q = (int)(e / width), j = (int)(e % width);
    const int r = rows[q];
    dst[e] = r >= 0 ? src[(long)r * width + j] : 0.f;
}
void gather_pad(const int* rows, int Bp, const float* src, int width, float* dst, cudaStream_t s) {
    const long n = (long)Bp * width;
    if (n == 0) return;
    k_gather_pad<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rows, Bp, src, width, dst);
    MB_LAUNCH();
}

// per-group column sums of an image's rows [goff[z], goff[z+1]) for columns
// [0, width): out fp32 [z*out_gs + j] and, if gimg.p, the gtheta image at
// (row z, col c0 + j)
__global__ void k_img_segcolsum(Img x, int width, const int* goff, float* out, long out_gs, Img gimg, long c0) {
    const int z = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= width) return;
    const int CT = img_ct(x.C);
    float s = 0.f;
    for (int q = goff[z]; q < goff[z + 1]; ++q)
        s += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(x.p + img_off(q, j, CT)));
    out[z * out_gs + j] = s;
    if (gimg.p)
        *reinterpret_cast<__nv_bfloat16*>(gimg.p + img_off(z, c0 + j, img_ct(gimg.C))) = __float2bfloat16_rn(s);
}
void img_segcolsum(const Img& x, int width, const int* goff, int G, float* out, long out_gs, const Img& gimg, long c0,
                   cudaStream_t s) {
    dim3 grid((width + 127) / 128, G);
    k_img_segcolsum<<<grid, 128, 0, s>>>(x, width, goff, out, out_gs, gimg, c0);
    MB_LAUNCH();
}

// fp32 per-group column sums (log-std gradients) -> fp32 flat + image
__global__ void k_segcolsum_f32(const float* x, int width, const int* goff, float* out, long out_gs, Img gimg,
                                long c0) {
    const int z = blockIdx.y;
    const int j = threadIdx.x;
    if (j >= width) return;
    float s = 0.f;
    for (int q = goff[z]; q < goff[z + 1]; ++q) s += x[(long)q * width + j];
    out[z * out_gs + j] = s;
    if (gimg.p)
        *reinterpret_cast<__nv_bfloat16*>(gimg.p + img_off(z, c0 + j, img_ct(gimg.C))) = __float2bfloat16_rn(s);
}
void segcolsum_f32(const float* x, int width, const int* goff, int G, float* out, long out_gs, const Img& gimg,
                   long c0, cudaStream_t s) {
    k_segcolsum_f32<<<dim3(1, G), 32, 0, s>>>(x, width, goff, out, out_gs, gimg, c0);
    MB_LAUNCH();
}

}  // namespace mb200
