// tcgen05 GEMM v3: D(m, n) = sum_k A(m, k) B(n, k) over tiled bf16 images
// (img.cuh). Persistent, warp-specialised, double-buffered accumulators:
//
//   * grid = min(#tiles, #SMs); each CTA walks output tiles (128 x BN)
//     round-robin (tile order: N fastest, then M, then group z);
//   * warp 0 / lane 0 = producer: cp.async.bulk of the A chunk and B
//     chunk(s) of every 128-wide K chunk into an S-stage smem ring
//     (full[s] expect_tx, empty[s] released by tcgen05.commit);
//   * warp 1 / lane 0 = MMA issuer: 8 x (K = 16) tcgen05.mma per B chunk
//     into TMEM accumulator buffer (tile & 1); tcgen05.commit -> tfull;
//   * warps 4.. = epilogue (8 or 16; TMEM lanes 32*(w%4).., column part (w-4)/4): tcgen05.ld 16 columns at
//     a time, fused bias / tanh / tanh' / fp32 + bf16-image stores, then
//     arrive tempty so the MMA warp can reuse the buffer -- the epilogue of
//     tile i overlaps the loads and MMAs of tile i+1.
// Grouped modes: gmode 1 = rows grouped (A/output rows start at goff[z],
// 128-aligned; B / bias per group), gmode 2 = K grouped (K range
// [goff[z], goff[z+1]), 128-aligned; output per group).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "img.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace mb200 {

namespace {
#ifdef MB_GEMM_PROF  // role timing of CTA 0 (NVCC="nvcc -DMB_GEMM_PROF")
#define GPROF_BEGIN const long long gp_start = clock64(); long long gp_wait = 0, gp_t0 = 0
#define GPROF_T0 gp_t0 = clock64()
#define GPROF_ADD(v) v += clock64() - gp_t0
#define GPROF_END(role, what)                                                                                  \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                                                            \
        printf("gemm CTA0 %s: total %lld cycles, %s %lld\n", role, clock64() - gp_start, what, gp_wait)
#else
#define GPROF_BEGIN
#define GPROF_T0
#define GPROF_ADD(v)
#define GPROF_END(role, what)
#endif
constexpr int CHUNK = 32768;
constexpr int EPI_WARP0 = 4;

template <int BN, int EPI>
struct Cfg {
    static constexpr int NB = BN > 128 ? 2 : 1;      // B chunks per stage
    static constexpr int STAGE = CHUNK * (1 + NB);
    static constexpr int STAGES = BN > 128 ? 2 : 3;
    static constexpr int NMMA = BN > 128 ? 128 : BN;  // N per MMA instruction
    static constexpr int ACC = BN < 32 ? 32 : BN;     // TMEM columns per accumulator buffer
    static constexpr int TCOLS = 2 * ACC;             // double buffered (<= 512)
    // epilogue warps: 4 lane quadrants x NEPI/4 column parts. The image
    // epilogues (tanh / tanh') are issue-latency bound with 2 warps per
    // SMSP, so wide tiles get 16 warps; fp32-output tiles keep 8 and the
    // smem staging area of their transposed stores
    static constexpr int NEPI = (EPI == 1 && BN >= 64) ? 16 : 8;
    static constexpr int NT = 128 + 32 * NEPI;
    static constexpr int SMEM = STAGES * STAGE + 1024 + 4 * BN + 16 * BN + (EPI == 0 ? 8 * 512 * 4 : 0);
};

__device__ __forceinline__ long chunk_index(int view, int mt, int kc, int CT) {
    // view 0: (row tile = mt, col tile = kc); view 1: (row tile = kc, col tile = mt)
    return view == 0 ? (long)mt * CT + kc : (long)kc * CT + mt;
}

struct TileInfo {
    int z, m0, n0, m_hi, k_lo, nk;
    bool valid;
};

__device__ __forceinline__ TileInfo tile_info(const IGemm& d, int t, int ntn, int ntm) {
    TileInfo ti;
    const int x = t % ntn, y = (t / ntn) % ntm;
    ti.z = t / (ntn * ntm);
    int m_lo = 0, m_hi = d.M, k_lo = 0, k_hi = d.K;
    if (d.gmode == 1) {
        m_lo = d.goff[ti.z];
        m_hi = d.goff[ti.z + 1];
    } else if (d.gmode == 2) {
        k_lo = d.goff[ti.z];
        k_hi = d.goff[ti.z + 1];
    }
    ti.m0 = m_lo + y * 128;
    ti.n0 = x * (d.N_tile);
    ti.m_hi = m_hi;
    ti.k_lo = k_lo;
    ti.nk = (k_hi - k_lo + 127) >> 7;
    ti.valid = ti.m0 < m_hi;
    return ti;
}

// up to 3 independent GEMMs of the same epilogue kind in one persistent
// launch: tile t belongs to g[k] with base[k] <= t < base[k+1]
struct GemmBatch {
    IGemm g[3];
    int n = 1;
    int base[4] = {0, 0, 0, 0};
    int ntn[3] = {1, 1, 1}, ntm[3] = {1, 1, 1};
};
__device__ __forceinline__ int batch_of(const GemmBatch& bt, int t) { return t < bt.base[1] ? 0 : t < bt.base[2] ? 1 : 2; }

// EPI: 0 = fp32 out (bias optional), 1 = tanh -> image (+ optional fp32 pre-act),
//      2 = tanh' (aux image) -> image
template <int BN, int EPI>
__global__ void __launch_bounds__(Cfg<BN, EPI>::NT, 1) k_img_gemm(const __grid_constant__ GemmBatch bt) {
    const int ntiles = bt.base[bt.n];
    using C = Cfg<BN, EPI>;
    constexpr int NEPI = C::NEPI, ET = 32 * NEPI;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sbias = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 1024);  // [BN]
    float* sred = sbias + BN;                                                        // [4][BN] column partials
    float* sstg = sred + 4 * BN;  // [8 warps][32 x 16] fp32 store staging

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(tslot, C::TCOLS);
    if (threadIdx.x == 32) {
        for (int s = 0; s < C::STAGES; ++s) {
            umma::mbar_init(&full[s], 1);
            umma::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            umma::mbar_init(&tfull[b], 1);
            umma::mbar_init(&tempty[b], ET);
        }
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    pdl_enter();  // prologue done: wait for the predecessor's data
    const uint32_t tbase = *tslot;
    // the descriptor and tile coordinates of batch tile t
#define MB_TILE(t)                                  \
    const int bk_ = batch_of(bt, t);                \
    const IGemm& d = bt.g[bk_];                     \
    const TileInfo ti = tile_info(d, t - bt.base[bk_], bt.ntn[bk_], bt.ntm[bk_])

    if (warp == 0) {
        {  // ---------------- producer (converged warp; one elected lane issues)
            GPROF_BEGIN;
            long g = 0;  // global chunk counter
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                MB_TILE(t);
                if (!ti.valid) continue;
                const int CTa = img_ct(d.A.C), CTb = img_ct(d.B.C);
                const uint32_t bbytes =
                    (d.b_view == 0 && BN < 128 && !d.b_tma) ? (uint32_t)BN * 256 : (uint32_t)CHUNK;
                const uint8_t* Ab = d.A.p + (d.gmode == 0 ? ti.z * d.A.gs : 0);
                const uint8_t* Bb = d.B.p + (d.gmode != 2 ? ti.z * d.B.gs : 0);
                const int mt = ti.m0 >> 7, nt0 = ti.n0 >> 7, kc0 = ti.k_lo >> 7;
                // B chunks that exist for this N tile (a narrow GEMM batched with BN > N)
                const int nbv = min(C::NB, (d.b_view ? CTb : img_rt(d.B.R)) - nt0);
                for (int kc = 0; kc < ti.nk; ++kc, ++g) {
                    const int s = (int)(g % C::STAGES);
                    GPROF_T0;
                    umma::mbar_wait(&empty[s], (uint32_t)(((g / C::STAGES) & 1) ^ 1));
                    GPROF_ADD(gp_wait);
                    uint8_t* st = smem + s * C::STAGE;
                    if (umma::elect_one()) {
                        umma::mbar_arrive_expect_tx(&full[s], CHUNK + nbv * bbytes);
                        umma::bulk_g2s(st, Ab + chunk_index(d.a_view, mt, kc0 + kc, CTa) * CHUNK, CHUNK, &full[s]);
#pragma unroll
                        for (int j = 0; j < C::NB; ++j) {
                            if (j >= nbv) continue;
                            if (d.b_tma) {  // (row chunk, column chunk) of B's [R][C] rows: two 64-column boxes
                                const int rc = d.b_view ? kc0 + kc : nt0 + j, cc = d.b_view ? nt0 + j : kc0 + kc;
                                const int z = d.gmode != 2 ? ti.z : 0;
                                umma::tma_load_3d(st + CHUNK * (1 + j), &d.bmap, cc * 128, rc * 128, z, &full[s]);
                                umma::tma_load_3d(st + CHUNK * (1 + j) + CHUNK / 2, &d.bmap, cc * 128 + 64, rc * 128, z,
                                                  &full[s]);
                            } else {
                                umma::bulk_g2s(st + CHUNK * (1 + j),
                                               Bb + chunk_index(d.b_view, nt0 + j, kc0 + kc, CTb) * CHUNK, bbytes,
                                               &full[s]);
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            GPROF_END("producer", "wait-stage");
        }
        __syncwarp();
    } else if (warp == 1) {
        {  // ---------------- MMA issuer (converged warp; one elected lane issues)
            GPROF_BEGIN;
#ifdef MB_GEMM_PROF
            long long gp_wait2 = 0;
#endif
            long g = 0;
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                MB_TILE(t);
                if (!ti.valid) continue;
                const uint32_t idesc = umma::idesc_bf16(128, C::NMMA, d.a_view == 1, d.b_view == 1);
                const uint32_t a_lbo = d.a_view ? 2048 : 128, a_sbo = d.a_view ? 128 : 2048;
                const uint32_t a_step = d.a_view ? 4096 : 256;
                const uint32_t b_lbo = d.b_view ? 2048 : 128, b_sbo = d.b_view ? 128 : 2048;
                const uint32_t b_step = d.b_view ? 4096 : 256;
                const int nbv = min(C::NB, (d.b_view ? img_ct(d.B.C) : img_rt(d.B.R)) - (ti.n0 >> 7));
                const int acc = it & 1;
                GPROF_T0;
                umma::mbar_wait(&tempty[acc], (uint32_t)(((it >> 1) & 1) ^ 1));
                GPROF_ADD(gp_wait2);
                umma::fence_after_sync();
                const uint32_t dcol = tbase + (uint32_t)(acc * C::ACC);
                // descriptors of stage 0's A and first B chunk; a stage / chunk / K step
                // only moves the start address (+bytes >> 4 in the low field)
                const uint64_t a_desc0 = umma::smem_desc(umma::smem_u32(smem), a_lbo, a_sbo);
                // tensor-map B chunks: 128-byte swizzle, two 64-column halves 16 KB apart;
                // K-major (view 0): SBO 1024 (8-row groups), K step +32 B inside a half;
                // MN-major (view 1): LBO 16 KB (the halves), SBO 1024, K step +2 KB
                const uint64_t b_desc0 =
                    d.b_tma ? (umma::smem_desc(umma::smem_u32(smem) + CHUNK, d.b_view ? CHUNK / 2 : 16, 1024) |
                               ((uint64_t)2 << 61))
                            : umma::smem_desc(umma::smem_u32(smem) + CHUNK, b_lbo, b_sbo);
                auto b_koff = [&](int kk) -> uint32_t {
                    if (!d.b_tma) return (uint32_t)kk * b_step;
                    return d.b_view ? (uint32_t)kk * 2048 : (uint32_t)((kk >> 2) * (CHUNK / 2) + (kk & 3) * 32);
                };
                for (int kc = 0; kc < ti.nk; ++kc, ++g) {
                    const int s = (int)(g % C::STAGES);
                    GPROF_T0;
                    umma::mbar_wait(&full[s], (uint32_t)((g / C::STAGES) & 1));
                    GPROF_ADD(gp_wait);
                    umma::fence_after_sync();
                    if (umma::elect_one()) {
                        const uint64_t ad = a_desc0 + (uint64_t)((s * C::STAGE) >> 4);
#pragma unroll
                        for (int j = 0; j < C::NB; ++j) {
                            if (j >= nbv) break;
                            const uint64_t bd = b_desc0 + (uint64_t)((s * C::STAGE + j * CHUNK) >> 4);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)
                                umma::mma_bf16(dcol + j * 128, ad + (uint64_t)(kk * (a_step >> 4)),
                                               bd + (uint64_t)(b_koff(kk) >> 4), idesc, (kc | kk) ? 1u : 0u);
                        }
                        umma::commit(&empty[s]);
                    }
                    __syncwarp();
                }
                if (umma::elect_one()) umma::commit(&tfull[acc]);
                __syncwarp();
                ++it;
            }
#ifdef MB_GEMM_PROF
            if (blockIdx.x == 0 && lane == 0) printf("gemm CTA0 mma: wait-accumulator %lld cycles\n", gp_wait2);
#endif
            GPROF_END("mma", "wait-data");
        }
        __syncwarp();
    } else if (warp >= EPI_WARP0) {  // ---------------- epilogue (NEPI warps)
        const int ew = warp - EPI_WARP0;           // 0..NEPI-1
        GPROF_BEGIN;
        const int lg = ew & 3, half = ew >> 2;     // TMEM lane quadrant, column part
        const int et = threadIdx.x - EPI_WARP0 * 32;  // 0..ET-1
        constexpr int NPART = NEPI / 4;
        constexpr int HALF = BN >= 16 * NPART ? BN / NPART : BN;  // columns per part
        const bool active = BN >= 16 * NPART || half == 0;
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            MB_TILE(t);
            if (!ti.valid) continue;
            const int acc = it & 1;
            const float* bias = d.bias ? d.bias + (d.gmode != 2 ? ti.z * d.bias_gs : 0) : nullptr;
            // per-n bias -> smem (the previous tile's readers passed this barrier already)
            asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
            if (d.bias_mode == 1)
                for (int j = et; j < BN; j += ET) sbias[j] = (ti.n0 + j < d.N) ? bias[ti.n0 + j] : 0.f;
            asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
            const int m = ti.m0 + lg * 32 + lane;
            const bool mrow = m < ti.m_hi;
            const float bm = (d.bias_mode == 2 && mrow) ? bias[m] : 0.f;
            const long cz = d.gmode == 1 ? 0 : ti.z;
            float* crow = d.C ? d.C + cz * d.c_gs + (long)m * d.cm : nullptr;
            const int CTo = img_ct(d.O.C), CTx = img_ct(d.aux.C);
            // full tile (every grouped tile: groups are 128-row padded): no
            // per-chunk guards, addresses = per-thread base + compile-time offset
            const bool fast = ti.m0 + 128 <= ti.m_hi && ti.n0 + BN <= d.N && !d.accumulate &&
                              (EPI != 0 || (d.cn == 1 && (d.cm & 3) == 0 && (d.c_gs & 3) == 0 &&
                                            (reinterpret_cast<uintptr_t>(d.C) & 15) == 0)) &&
                              (EPI != 1 || !d.C2);
            if (active && fast) {
                constexpr int NCH = HALF / 16;
                // image byte offset of (row m, column n0 + half * HALF); + chunk offset below
                const long rowo_x = ((long)(m >> 7) * CTx) * 32768 + ((m & 127) >> 3) * 2048 + (m & 7) * 16;
                const long rowo_o = ((long)(m >> 7) * CTo) * 32768 + ((m & 127) >> 3) * 2048 + (m & 7) * 16;
                const int cb = ti.n0 + half * HALF;  // multiple of 16; chunks below never cross 128
                const long colo = (long)(cb >> 7) * 32768 + ((cb & 127) >> 3) * 128;
                const uint8_t* xb = d.aux.p + rowo_x + colo;
                uint8_t* ob = d.O.p + rowo_o + colo;
                // EPI 0: first row of this warp's 32-row slab, first column of the half
                const long wofs = cz * d.c_gs + (long)(ti.m0 + lg * 32) * d.cm + cb;
                float* stg = sstg + ew * 512;
                // transpose the warp's 32 rows x 16 columns through shared memory
                // (XOR-swizzled float4 slots, conflict-free both ways) so every
                // store instruction writes 8 rows x 64 contiguous bytes
                auto stage_store = [&](float* dst, const float* x) {
#pragma unroll
                    for (int h = 0; h < 4; ++h)
                        *reinterpret_cast<float4*>(stg + lane * 16 + ((h ^ ((lane >> 1) & 3)) << 2)) =
                            make_float4(x[4 * h], x[4 * h + 1], x[4 * h + 2], x[4 * h + 3]);
                    __syncwarp();
#pragma unroll
                    for (int s8 = 0; s8 < 4; ++s8) {
                        const int r = s8 * 8 + (lane >> 2), h = lane & 3;
                        const float4 y = *reinterpret_cast<const float4*>(stg + r * 16 + ((h ^ ((r >> 1) & 3)) << 2));
                        *reinterpret_cast<float4*>(dst + (long)r * d.cm + h * 4) = y;
                    }
                    __syncwarp();
                };
                // bf16 copy: the warp's 32 rows x 16 columns (32 B per row) through the
                // same staging area, each store instruction writing 16 rows x 32 B
                auto stage_store16 = [&](uint16_t* dst, const float* x) {
                    uint32_t* st32 = reinterpret_cast<uint32_t*>(stg);
                    uint4 q0, q1;
                    q0.x = umma::pack_bf16(x[0], x[1]);
                    q0.y = umma::pack_bf16(x[2], x[3]);
                    q0.z = umma::pack_bf16(x[4], x[5]);
                    q0.w = umma::pack_bf16(x[6], x[7]);
                    q1.x = umma::pack_bf16(x[8], x[9]);
                    q1.y = umma::pack_bf16(x[10], x[11]);
                    q1.z = umma::pack_bf16(x[12], x[13]);
                    q1.w = umma::pack_bf16(x[14], x[15]);
                    *reinterpret_cast<uint4*>(st32 + lane * 8) = q0;
                    *reinterpret_cast<uint4*>(st32 + lane * 8 + 4) = q1;
                    __syncwarp();
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        const int piece = s2 * 32 + lane, r = piece >> 1, h = piece & 1;
                        const uint4 y = *reinterpret_cast<const uint4*>(st32 + r * 8 + h * 4);
                        *reinterpret_cast<uint4*>(dst + (long)r * d.c16m + h * 8) = y;
                    }
                    __syncwarp();
                };
                auto bf_only = [&](int n0c) {  // columns [n0c, n0c + 16) all inside one bf16-only range
                    for (int k = 0; k < d.nbf; ++k)
                        if (n0c >= d.bf_lo[k] && n0c + 16 <= d.bf_hi[k]) return true;
                    return false;
                };
                // chunk ci = columns cb + 16 ci .. +15, inside one 128-column chunk
                // for every BN ((cb & 127) + 16 ci <= 112): 2 core-matrix columns
                auto coff = [](int ci) -> long { return (long)ci * 256; };
                // one 16-column chunk: TMEM -> bias -> activation -> bf16 image (or
                // fp32 via the staging transpose); ax = this chunk's tanh' operand
                auto chunk = [&](int ci, const uint4* ax) {
                    const int c0 = half * HALF + ci * 16;
                    float v[16];
                    if (ti.nk > 0) {
                        umma::tmem_ld16(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * C::ACC + c0), v);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = 0.f;
                    }
                    if (d.bias_mode == 1) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] += sbias[c0 + i];
                    } else if (d.bias_mode == 2) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] += bm;
                    }
                    if (EPI == 0) {
                        if (d.C16) {
                            stage_store16(d.C16 + cz * d.c_gs + (long)(ti.m0 + lg * 32) * d.c16m + cb + ci * 16, v);
                            if (bf_only(cb + ci * 16)) return;
                        }
                        stage_store(d.C + wofs + ci * 16, v);
                        return;
                    }
                    if (EPI == 1) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = umma::tanh_approx(v[i]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&ax[h]);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f = __bfloat1622float2(b2[e]);
                                v[8 * h + 2 * e] *= 1.f - f.x * f.x;
                                v[8 * h + 2 * e + 1] *= 1.f - f.y * f.y;
                            }
                        }
                        if (d.psum) {  // warp reduce-scatter of 16 columns over 32 rows
                            float a2[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) a2[i] = v[i];
                            int col = 0;
#pragma unroll
                            for (int w = 8; w >= 1; w >>= 1) {
                                const bool up = (lane & (2 * w)) != 0;
                                col += up ? w : 0;
#pragma unroll
                                for (int i = 0; i < w; ++i) {
                                    const float mine = up ? a2[w + i] : a2[i];
                                    const float other = up ? a2[i] : a2[w + i];
                                    a2[i] = mine + __shfl_xor_sync(0xffffffffu, other, 2 * w);
                                }
                            }
                            a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 1);
                            if ((lane & 1) == 0) sred[lg * BN + c0 + col] = a2[0];
                        }
                    }
                    uint4 q0, q1;
                    q0.x = umma::pack_bf16(v[0], v[1]);
                    q0.y = umma::pack_bf16(v[2], v[3]);
                    q0.z = umma::pack_bf16(v[4], v[5]);
                    q0.w = umma::pack_bf16(v[6], v[7]);
                    q1.x = umma::pack_bf16(v[8], v[9]);
                    q1.y = umma::pack_bf16(v[10], v[11]);
                    q1.z = umma::pack_bf16(v[12], v[13]);
                    q1.w = umma::pack_bf16(v[14], v[15]);
                    *reinterpret_cast<uint4*>(ob + coff(ci)) = q0;
                    *reinterpret_cast<uint4*>(ob + coff(ci) + 128) = q1;
                };
                // pairs of chunks, the next pair's tanh' operands in flight under
                // this pair's math; kept rolled (the fully unrolled epilogue did
                // not fit the instruction cache: "no_instructions" stalls)
                auto aux = [&](int ci, uint4* dst) {
                    if (EPI == 2 && ci < NCH) {
                        dst[0] = *reinterpret_cast<const uint4*>(xb + coff(ci));
                        dst[1] = *reinterpret_cast<const uint4*>(xb + coff(ci) + 128);
                    }
                };
                // the tanh' operands two chunk pairs ahead (their L2 latency is longer than
                // one pair's math); the first two pairs are in flight under the accumulator wait
                uint4 cur[4], nxt[4], nx2[4];
                aux(0, cur);
                aux(1, cur + 2);
                aux(2, nxt);
                aux(3, nxt + 2);
                GPROF_T0;
                umma::mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
                GPROF_ADD(gp_wait);
                umma::fence_after_sync();
#pragma unroll 1
                for (int ci = 0; ci < NCH; ci += 2) {
                    aux(ci + 4, nx2);
                    aux(ci + 5, nx2 + 2);
                    chunk(ci, cur);
                    if (ci + 1 < NCH) chunk(ci + 1, cur + 2);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        cur[q] = nxt[q];
                        nxt[q] = nx2[q];
                    }
                }
            } else if (active) {
                // partial tiles (edges of M or N): guarded, rolled
                constexpr int NCH = HALF / 16;
                auto aux_load = [&](int ci, uint4* dst) {
                    const int nb2 = ti.n0 + half * HALF + ci * 16;
                    dst[0] = dst[1] = make_uint4(0, 0, 0, 0);
                    if (EPI == 2 && mrow && nb2 < d.N) {
                        dst[0] = *reinterpret_cast<const uint4*>(d.aux.p + img_off(m, nb2, CTx));
                        if (nb2 + 8 < d.N) dst[1] = *reinterpret_cast<const uint4*>(d.aux.p + img_off(m, nb2 + 8, CTx));
                    }
                };
                umma::mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));  // committed even when nk == 0
                umma::fence_after_sync();
#pragma unroll 1
                for (int ci = 0; ci < NCH; ++ci) {
                    const int c0 = half * HALF + ci * 16;
                    const int nb = ti.n0 + c0;
                    const bool full = mrow && nb + 16 <= d.N;
                    const bool any = mrow && nb < d.N;
                    uint4 ax[2];
                    aux_load(ci, ax);
                    float v[16];
                    if (ti.nk > 0) {
                        umma::tmem_ld16(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * C::ACC + c0), v);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = 0.f;
                    }
                    if (d.bias_mode == 1) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] += sbias[c0 + i];
                    } else if (d.bias_mode == 2) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] += bm;
                    }
                    if (EPI == 0) {
                        if (!any) continue;
                        if (d.C16) {
                            uint16_t* r16 = d.C16 + cz * d.c_gs + (long)m * d.c16m;
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (nb + i < d.N) {
                                    const __nv_bfloat16 b = __float2bfloat16_rn(v[i]);
                                    r16[nb + i] = *reinterpret_cast<const uint16_t*>(&b);
                                }
                            bool only = false;
                            for (int k = 0; k < d.nbf; ++k)
                                if (nb >= d.bf_lo[k] && nb + 16 <= d.bf_hi[k]) only = true;
                            if (only) continue;
                        }
                        if (d.accumulate)
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (nb + i < d.N) v[i] += crow[(long)(nb + i) * d.cn];
                        if (full && d.cn == 1 && ((reinterpret_cast<uintptr_t>(crow + nb) & 15) == 0)) {
                            float4* q = reinterpret_cast<float4*>(crow + nb);
#pragma unroll
                            for (int h = 0; h < 4; ++h)
                                q[h] = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (nb + i < d.N) crow[(long)(nb + i) * d.cn] = v[i];
                        }
                        continue;
                    }
                    if (EPI == 1) {
                        if (d.C2 && any)
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (nb + i < d.N) d.C2[(long)m * d.c2m + (long)(nb + i) * d.c2n] = v[i];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = umma::tanh_approx(v[i]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&ax[h]);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f = __bfloat1622float2(b2[e]);
                                v[8 * h + 2 * e] *= 1.f - f.x * f.x;
                                v[8 * h + 2 * e + 1] *= 1.f - f.y * f.y;
                            }
                        }
                        if (d.psum) {  // warp reduce-scatter of 16 columns over 32 rows: 16 shuffles
                            float a2[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) a2[i] = (full || (any && nb + i < d.N)) ? v[i] : 0.f;
                            int col = 0;
#pragma unroll
                            for (int w = 8; w >= 1; w >>= 1) {  // keep w columns, 2x rows each step
                                const int sel = (lane & (2 * w)) ? w : 0;
                                col += sel;
#pragma unroll
                                for (int i = 0; i < w; ++i) {
                                    const float mine = sel ? a2[w + i] : a2[i];
                                    const float other = sel ? a2[i] : a2[w + i];
                                    a2[i] = mine + __shfl_xor_sync(0xffffffffu, other, 2 * w);
                                }
                            }
                            a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 1);
                            if ((lane & 1) == 0) sred[lg * BN + c0 + col] = a2[0];
                        }
                    }
                    if (!any) continue;
                    if (!full)
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (nb + i >= d.N) v[i] = 0.f;  // keep padding zero
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!full && nb + 8 * h >= d.N) continue;
                        uint4 q;
                        q.x = umma::pack_bf16(v[8 * h + 0], v[8 * h + 1]);
                        q.y = umma::pack_bf16(v[8 * h + 2], v[8 * h + 3]);
                        q.z = umma::pack_bf16(v[8 * h + 4], v[8 * h + 5]);
                        q.w = umma::pack_bf16(v[8 * h + 6], v[8 * h + 7]);
                        *reinterpret_cast<uint4*>(d.O.p + img_off(m, nb + 8 * h, CTo)) = q;
                    }
                }
            }
            umma::fence_before_sync();
            umma::mbar_arrive(&tempty[acc]);
            if (EPI == 2 && d.psum) {  // psum[m-tile][n] = sum over the tile's 128 rows
                asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
                for (int j = et; j < BN; j += ET)
                    if (ti.n0 + j < d.N)
                        d.psum[(long)(ti.m0 >> 7) * d.psum_ld + ti.n0 + j] =
                            sred[j] + sred[BN + j] + sred[2 * BN + j] + sred[3 * BN + j];
            }
            ++it;
        }
        if (ew == 0) GPROF_END("epilogue", "wait-accumulator");
    }
    __syncthreads();
    if (warp == 0) umma::tmem_free(tbase, C::TCOLS);
#undef MB_TILE
}

template <int BN, int EPI>
void launch(const IGemm* ds, int n, cudaStream_t s) {
    using C = Cfg<BN, EPI>;
    ensure_smem((const void*)k_img_gemm<BN, EPI>, C::SMEM);
    GemmBatch bt;
    bt.n = n;
    for (int k = 0; k < n; ++k) {
        IGemm d = ds[k];
        d.N_tile = BN;
        const int mext = d.gmode == 1 ? d.max_group : d.M;
        bt.ntn[k] = (d.N + BN - 1) / BN;
        bt.ntm[k] = (mext + 127) / 128;
        bt.base[k + 1] = bt.base[k] + bt.ntn[k] * bt.ntm[k] * d.Z;
        bt.g[k] = d;
    }
    const int ntiles = bt.base[n];
    if (ntiles == 0) return;
    const int sms = device_sms();
    const int grid = ntiles < sms ? ntiles : sms;
    launch_pdl(k_img_gemm<BN, EPI>, dim3(grid), dim3(C::NT), C::SMEM, s, bt);
    MB_LAUNCH();
}

template <int EPI>
void dispatch_bn(const IGemm* ds, int n, cudaStream_t s) {
    int N = 0;
    for (int k = 0; k < n; ++k) N = std::max(N, ds[k].N);
    if (N <= 16) launch<16, EPI>(ds, n, s);
    else if (N <= 32) launch<32, EPI>(ds, n, s);
    else if (N <= 64) launch<64, EPI>(ds, n, s);
    else if (N <= 128) launch<128, EPI>(ds, n, s);
    else launch<256, EPI>(ds, n, s);
}
}  // namespace

void img_gemm_batch(const IGemm* ds, int n, cudaStream_t s) {
    if (n < 1 || n > 3) throw ShapeError("img_gemm_batch: 1 to 3 GEMMs per launch");
    std::vector<IGemm> live;
    for (int k = 0; k < n; ++k) {
        const IGemm& d = ds[k];
        if (d.M <= 0 || d.N <= 0 || d.Z <= 0 || (d.gmode == 1 && d.max_group <= 0)) continue;
        if (d.act != ds[0].act || d.o_mode != ds[0].o_mode)
            throw ShapeError("img_gemm_batch: the batched GEMMs must share the epilogue kind");
        live.push_back(d);
    }
    if (live.empty()) return;
    const IGemm& d0 = live[0];
    if (d0.act == 0) {
        if (d0.o_mode != 0) throw ShapeError("img_gemm: image output needs an activation epilogue");
        dispatch_bn<0>(live.data(), (int)live.size(), s);
    } else if (d0.act == 1) {
        dispatch_bn<1>(live.data(), (int)live.size(), s);
    } else {
        dispatch_bn<2>(live.data(), (int)live.size(), s);
    }
}

void img_gemm(const IGemm& d, cudaStream_t s) { img_gemm_batch(&d, 1, s); }

bool make_weight_map(CUtensorMap* map, const uint16_t* base, int R, int C, long gs, int Z) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode enc = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<Encode>(f);
    }();
    if (!enc || C % 8 || gs % 8 || (reinterpret_cast<uintptr_t>(base) & 15) || R < 1 || Z < 1) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)R, (cuuint64_t)Z};
    const cuuint64_t strides[2] = {(cuuint64_t)C * 2, (cuuint64_t)gs * 2};
    const cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// every per-cluster segment sum of one net's minibatch step in one launch:
// block z < G sums job j's tiles of cluster z (fixed order), block G sums
// the per-tile loss partials (fp64, fixed tree) into *loss_out
__global__ void k_segsum_multi(const __grid_constant__ SegJobs jb, const int* goff, int G) {
    pdl_enter();
    const int z = blockIdx.x;
    if (z >= G) {  // one block per loss
        const SegLoss& L = jb.loss[z - G];
        __shared__ double red[256];
        double s = 0.0;
        for (long i = threadIdx.x; i < L.n; i += blockDim.x) s += L.tiles[i];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int k = blockDim.x / 2; k > 0; k >>= 1) {
            if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
            __syncthreads();
        }
        if (threadIdx.x == 0) *L.out = red[0];
        return;
    }
    const int t0 = goff[z] >> 7, t1 = goff[z + 1] >> 7;
    for (int q = 0; q < jb.n; ++q) {
        const SegJob& j = jb.job[q];
        for (int c = threadIdx.x; c < j.width; c += blockDim.x) {
            float acc = 0.f;
            for (int t = t0; t < t1; ++t) acc += j.psum[(long)t * j.ld + c];
            j.out[(long)z * j.out_gs + c] = acc;
        }
    }
}
void segsum_multi(const SegJobs& jb, const int* goff, int G, cudaStream_t s) {
    launch_pdl(k_segsum_multi, dim3(G + jb.nloss), dim3(256), 0, s, jb, goff, G);
    MB_LAUNCH();
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

// local clusters' gtheta rows [Kl][ld] -> send[W][Kl][S]: destination
// rank d gets columns [d S, d S + S) of every local row (the all-to-all
// payload of the sharded optimizer); one float4 per thread
__global__ void k_pack_shards(const float* __restrict__ gt, long ld, int Kl, long S, int W, float* __restrict__ send) {
    pdl_enter();
    const long s4 = S / 4, units = (long)W * Kl * s4;
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < units; u += (long)gridDim.x * blockDim.x) {
        const long d = u / ((long)Kl * s4), rem = u - d * Kl * s4;
        const long k = rem / s4, c = d * S + (rem - k * s4) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < ld) v = *reinterpret_cast<const float4*>(gt + k * ld + c);
        reinterpret_cast<float4*>(send)[u] = v;
    }
}
void pack_shards(const float* gt, long ld, int Kl, long S, int W, float* send, cudaStream_t s) {
    if (ld % 8 || S % 128) throw ShapeError("pack_shards: row stride % 8 and shard width % 128 required");
    const long units = (long)W * Kl * (S / 4);
    if (units == 0) return;
    launch_pdl(k_pack_shards, dim3((unsigned)std::min<long>((units + 255) / 256, 148L * 8)), dim3(256), 0, s, gt, ld,
               Kl, S, W, send);
    MB_LAUNCH();
}

// generated weights theta[g0 + z][woff_l + j * in_l + i] -> layer images of
// group z (row j, col i), every layer of every group in one launch; one thread
// per 8-column unit (32-byte fp32 reads, one 16-byte image store)
__global__ void k_pack_weights(const float* __restrict__ theta, long ld, int g0, int ng, PackDims pd, uint8_t* wimg,
                               long gs) {
    pdl_enter();
    const long per = pd.ustart[pd.L];
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < per * ng; u += (long)gridDim.x * blockDim.x) {
        const int z = (int)(u / per);
        const long r = u - (long)z * per;
        int l = 0;
        while (r >= pd.ustart[l + 1]) ++l;
        const int in = pd.in[l], cpr = (in + 7) >> 3;
        const int e = (int)(r - pd.ustart[l]);
        // consecutive threads = consecutive 8-column units of one row: each
        // warp reads a contiguous 1 KB of theta (two float4 per thread)
        const int j = e / cpr, c = (e - j * cpr) * 8;
        if (j >= pd.out[l]) continue;  // rows padded to a multiple of 8
        const float* src = theta + (long)(g0 + z) * ld + pd.woff[l] + (long)j * in + c;
        float v[8];
        if (c + 8 <= in && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = c + q < in ? src[q] : 0.f;
        }
        uint4 w;
        w.x = umma::pack_bf16(v[0], v[1]);
        w.y = umma::pack_bf16(v[2], v[3]);
        w.z = umma::pack_bf16(v[4], v[5]);
        w.w = umma::pack_bf16(v[6], v[7]);
        *reinterpret_cast<uint4*>(wimg + (long)z * gs + pd.ioff[l] + img_off(j, c, img_ct(in))) = w;
    }
}
void pack_weights(const float* theta, long ld, int g0, int ng, const PackDims& pd, uint8_t* wimg, long gs,
                  cudaStream_t s) {
    const long n = pd.ustart[pd.L] * ng;
    if (n == 0) return;
    launch_pdl(k_pack_weights, dim3((unsigned)std::min<long>((n + 255) / 256, 148 * 16)), dim3(256), 0, s, theta, ld,
               g0, ng, pd, wimg, gs);
    MB_LAUNCH();
}

// the same from the bf16 copy of theta: one 16-byte read and one 16-byte
// image store per 8-column unit
__global__ void k_pack_weights16(const uint16_t* __restrict__ theta16, long ld, int g0, int ng, PackDims pd,
                                 uint8_t* wimg, long gs) {
    pdl_enter();
    const long per = pd.ustart[pd.L];
    for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < per * ng; u += (long)gridDim.x * blockDim.x) {
        const int z = (int)(u / per);
        const long r = u - (long)z * per;
        int l = 0;
        while (r >= pd.ustart[l + 1]) ++l;
        const int in = pd.in[l], cpr = (in + 7) >> 3;
        const int e = (int)(r - pd.ustart[l]);
        const int j = e / cpr, c = (e - j * cpr) * 8;
        if (j >= pd.out[l]) continue;
        const uint16_t* src = theta16 + (long)(g0 + z) * ld + pd.woff[l] + (long)j * in + c;
        uint4 w;
        if (c + 8 <= in && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            w = *reinterpret_cast<const uint4*>(src);
        } else {
            uint16_t v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = c + q < in ? src[q] : (uint16_t)0;
            w.x = v[0] | (uint32_t)v[1] << 16;
            w.y = v[2] | (uint32_t)v[3] << 16;
            w.z = v[4] | (uint32_t)v[5] << 16;
            w.w = v[6] | (uint32_t)v[7] << 16;
        }
        *reinterpret_cast<uint4*>(wimg + (long)z * gs + pd.ioff[l] + img_off(j, c, img_ct(in))) = w;
    }
}
void pack_weights16(const uint16_t* theta16, long ld, int g0, int ng, const PackDims& pd, uint8_t* wimg, long gs,
                    cudaStream_t s) {
    const long n = pd.ustart[pd.L] * ng;
    if (n == 0) return;
    launch_pdl(k_pack_weights16, dim3((unsigned)std::min<long>((n + 255) / 256, 148 * 16)), dim3(256), 0, s,
               theta16, ld, g0, ng, pd, wimg, gs);
    MB_LAUNCH();
}

// gtheta [G][ld] (fp32) -> bf16 image (row g, col p) for the dM / df GEMMs and
// db[p] = sum_g gtheta[g][p] (hypernet.cpp:92-122) in one read. A block step
// covers 32 8-column units x 32 row slices (1024 threads, <= 32 registers: two
// blocks fill an SM, so 64 warps x 32 B per lane keep enough bytes in flight);
// persistent over the unit groups (no tail wave); the slices' sums combine in
// a fixed order.
constexpr int kGtSlices = 32, kGtUnits = 32;
__global__ void __launch_bounds__(kGtUnits * kGtSlices, 2) k_gtheta_prep(const float* __restrict__ gt, long ld, int G,
                                                                         int P, Img gimg, float* db) {
    pdl_enter();
    __shared__ float part[kGtSlices][kGtUnits][9];
    const int ul = threadIdx.x % kGtUnits, sl = threadIdx.x / kGtUnits;
    const int CT = img_ct(gimg.C);
    const int rs = (G + kGtSlices - 1) / kGtSlices, r0 = sl * rs, r1 = min(G, r0 + rs);
    const long ngroups = ((P + 7) / 8 + kGtUnits - 1) / kGtUnits;
    for (long ug = blockIdx.x; ug < ngroups; ug += gridDim.x) {
        const int p0 = (int)((ug * kGtUnits + ul) * 8);
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (p0 < P) {
            const bool full = p0 + 8 <= P;
            for (int g = r0; g < r1; ++g) {
                const float* src = gt + (long)g * ld + p0;
                float v[8];
                if (full) {
                    const float4 a = *reinterpret_cast<const float4*>(src);
                    const float4 b = *reinterpret_cast<const float4*>(src + 4);
                    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[e] = p0 + e < P ? src[e] : 0.f;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += v[e];
                uint4 w;
                w.x = umma::pack_bf16(v[0], v[1]);
                w.y = umma::pack_bf16(v[2], v[3]);
                w.z = umma::pack_bf16(v[4], v[5]);
                w.w = umma::pack_bf16(v[6], v[7]);
                *reinterpret_cast<uint4*>(gimg.p + img_off(g, p0, CT)) = w;
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) part[sl][ul][e] = acc[e];
        __syncthreads();
        if (db && sl == 0 && p0 < P)
            for (int e = 0; e < 8 && p0 + e < P; ++e) {
                float t = 0.f;
                for (int q = 0; q < kGtSlices; ++q) t += part[q][ul][e];
                db[p0 + e] = t;
            }
        __syncthreads();
    }
}
void gtheta_prep(const float* gt, long ld, int G, int P, const Img& gimg, float* db, cudaStream_t s) {
    if (ld % 8) throw ShapeError("gtheta_prep: row stride must be a multiple of 8");
    const long ngroups = ((P + 7) / 8 + kGtUnits - 1) / kGtUnits;
    const int sms = device_sms();
    launch_pdl(k_gtheta_prep, dim3((unsigned)std::min<long>(ngroups, 2L * sms)), dim3(kGtUnits * kGtSlices), 0, s, gt,
               ld, G, P, gimg, db);
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

// the whole minibatch in one launch (losses.cpp:21-33 row selection), one
// block per 128-row tile (groups are 128-row padded: a tile is one cluster,
// found once by a warp-wide count of the offsets <= the tile start). Per padded
// row q (row map rows[q], -1 = padding -> zeros): observation row -> bf16
// image (threads walk the tile's 8-column units row-major: coalesced 32 B
// reads, 16 B image stores), actions / old log-prob / scalar advantage / value
// targets -> fp32 rows, the cluster -> rg
__global__ void __launch_bounds__(128) k_gather_minibatch(const __grid_constant__ MbGather a) {
    __shared__ int srow[128], sz;
    pdl_enter();
    const int q0 = blockIdx.x * 128, t = threadIdx.x;
    const int q = q0 + t;
    const int r = a.rows[q];
    srow[t] = r;
    if (t < 32) {
        int cnt = 0;
        for (int b = 0; b < a.G; b += 32) {
            const int i = b + t;
            cnt += __popc(__ballot_sync(0xffffffffu, i < a.G && a.goff[i] <= q0));
        }
        if (t == 0) sz = cnt - 1;
    }
    const bool ok = r >= 0;
    a.lp_o[q] = ok ? a.lp[r] : 0.f;
    a.sadv_o[q] = ok ? a.sadv[r] : 0.f;
    __syncthreads();
    a.rg[q] = sz;
    const int CT = img_ct(a.od), cpr = (a.od + 7) >> 3;
    const bool vec = (a.od & 3) == 0;
    // 4 units per thread per round: all 8 loads in flight before the stores
    for (int u0 = t; u0 < 128 * cpr; u0 += 4 * 128) {
        float v[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int u = u0 + k * 128;
            const int rl = u / cpr, c = (u - rl * cpr) * 8;
            const int rr = u < 128 * cpr ? srow[rl] : -1;
            const float* src = a.obs + (long)(rr >= 0 ? rr : 0) * a.od;
            if (rr >= 0 && vec && c + 8 <= a.od) {
                const float4 x = *reinterpret_cast<const float4*>(src + c);
                const float4 y = *reinterpret_cast<const float4*>(src + c + 4);
                v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w;
                v[k][4] = y.x; v[k][5] = y.y; v[k][6] = y.z; v[k][7] = y.w;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[k][e] = (rr >= 0 && c + e < a.od) ? src[c + e] : 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int u = u0 + k * 128;
            if (u >= 128 * cpr) break;
            const int rl = u / cpr, c = (u - rl * cpr) * 8;
            uint4 w;
            w.x = umma::pack_bf16(v[k][0], v[k][1]);
            w.y = umma::pack_bf16(v[k][2], v[k][3]);
            w.z = umma::pack_bf16(v[k][4], v[k][5]);
            w.w = umma::pack_bf16(v[k][6], v[k][7]);
            *reinterpret_cast<uint4*>(a.Xi.p + img_off(q0 + rl, c, CT)) = w;
        }
    }
    for (int u = t; u < 128 * a.ad; u += 128) {
        const int rl = u / a.ad, e = u - rl * a.ad, rr = srow[rl];
        a.act_o[(long)q0 * a.ad + u] = rr >= 0 ? a.act[(long)rr * a.ad + e] : 0.f;
    }
    for (int u = t; u < 128 * a.m; u += 128) {
        const int rl = u / a.m, e = u - rl * a.m, rr = srow[rl];
        a.tgt_o[(long)q0 * a.m + u] = rr >= 0 ? a.tgt[(long)rr * a.m + e] : 0.f;
    }
}
void gather_minibatch(const MbGather& a, cudaStream_t s) {
    if (a.Bp <= 0) return;
    if (a.Bp % 128) throw ShapeError("gather_minibatch: rows must be 128-padded per cluster");
    launch_pdl(k_gather_minibatch, dim3(a.Bp / 128), dim3(128), 0, s, a);
    MB_LAUNCH();
}

}  // namespace mb200
