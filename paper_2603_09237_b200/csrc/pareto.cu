// K8 / K9: Pareto dominance mask and Monte-Carlo hypervolume (fp64).
// nondominated_filter (pareto.cpp:38-77) is a sequential sum-ordered sweep;
// it is equivalent to the data-parallel rule
//   keep(i) = first-occurrence(i) and no first-occurrence j that precedes i
//             in the (sum desc, index asc) order dominates i
// (a removed dominator implies an earlier kept dominator by transitivity),
// so every point is decided independently. Sums are accumulated in the
// reference's order with round-to-nearest adds, so the order -- and hence
// the mask -- is bit-identical, including fp ties.
// hypervolume_mc (pareto.cpp:236-277): sample s uses words s*m+j+1 of the
// stream; coordinates use explicit __dmul_rn/__dadd_rn (no FMA) so every
// sample point and the hit count are bit-identical to the reference.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace mb200 {

__global__ void k_pareto_prep(int n, int m, const double* __restrict__ p, uint8_t* uniq, double* sums) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* pi = p + (long)i * m;
    bool u = true;
    for (int j = 0; j < i && u; ++j) {
        const double* pj = p + (long)j * m;
        bool eq = true;
        for (int k = 0; k < m; ++k)
            if (!(pj[k] == pi[k])) { eq = false; break; }
        if (eq) u = false;
    }
    uniq[i] = u;
    double s = 0.0;
    for (int k = 0; k < m; ++k) s = __dadd_rn(s, pi[k]);
    sums[i] = s;
}

__global__ void k_pareto_mask(int n, int m, const double* __restrict__ p, const uint8_t* __restrict__ uniq,
                              const double* __restrict__ sums, uint8_t* mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!uniq[i]) { mask[i] = 0; return; }
    const double* pi = p + (long)i * m;
    const double si = sums[i];
    bool keep = true;
    for (int j = 0; j < n && keep; ++j) {
        if (j == i || !uniq[j]) continue;
        const double sj = sums[j];
        if (!(sj > si || (sj == si && j < i))) continue;
        const double* pj = p + (long)j * m;
        bool ge = true, strict = false;  // dominates(pj, pi): pareto.cpp:27-36
        for (int k = 0; k < m; ++k) {
            if (pj[k] < pi[k]) { ge = false; break; }
            if (pj[k] > pi[k]) strict = true;
        }
        if (ge && strict) keep = false;
    }
    mask[i] = keep;
}

void pareto_mask(int n, int m, const double* pts, uint8_t* mask, uint8_t* uniq, double* sums,
                 cudaStream_t s) {
    if (n <= 0) return;
    k_pareto_prep<<<(n + 127) / 128, 128, 0, s>>>(n, m, pts, uniq, sums);
    MB_LAUNCH();
    k_pareto_mask<<<(n + 127) / 128, 128, 0, s>>>(n, m, pts, uniq, sums, mask);
    MB_LAUNCH();
}

// ---- linear_dominance_filter (pareto.cpp:79-139) on the nondominated set
// nd [nn][m] (input order). m == 2: one block sorts by J1 (rank scatter;
// J1 values are distinct in nd) and thread 0 runs the upper-hull scan with
// the reference's cross product (explicit _rn ops: no FMA contraction).
// m >= 3: every weight of simplex_grid(m, 60) (simplex.cpp:108-117) is
// unranked from its index (stars and bars, grid_rec order), w_j = k_j / 60,
// dots in coordinate order (simplex.cpp:10-16); the points within
// 1e-9 max(1, |best|) of the best are kept. Bit-identical keep decisions.
__global__ void k_ldf_hull2(int nn, const double* __restrict__ nd, int* order, uint8_t* keep) {
    for (int q = threadIdx.x; q < nn; q += blockDim.x) {
        const double x = nd[2 * q];
        int rank = 0;
        for (int r = 0; r < nn; ++r) rank += nd[2 * r] < x || (nd[2 * r] == x && r < q);
        order[rank] = q;
        keep[q] = 0;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    int h = 0;
    int* hull = order + nn;
    for (int q = 0; q < nn; ++q) {
        const int id = order[q];
        while (h >= 2) {
            const double* p1 = nd + 2 * hull[h - 2];
            const double* p2 = nd + 2 * hull[h - 1];
            const double* p3 = nd + 2 * id;
            const double cross = __dsub_rn(__dmul_rn(__dsub_rn(p2[0], p1[0]), __dsub_rn(p3[1], p2[1])),
                                           __dmul_rn(__dsub_rn(p2[1], p1[1]), __dsub_rn(p3[0], p2[0])));
            if (cross > 0.0) --h;
            else break;
        }
        hull[h++] = id;
    }
    for (int q = 0; q < h; ++q) keep[hull[q]] = 1;
}

constexpr int kLdfRes = 60;
constexpr int kLdfThreads = 256;
__device__ __forceinline__ double ldf_dot(const int* k, const double* p, int m) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn((double)k[j], (double)kLdfRes), p[j]));
    return acc;
}
// binom[n][r] for n <= kLdfRes + 8, r <= 8 (uint64, exact)
__global__ void __launch_bounds__(kLdfThreads) k_ldf_sweep(int nn, int m, const double* __restrict__ nd,
                                                           const unsigned long long* __restrict__ binom,
                                                           unsigned long long nw, uint8_t* keep_g) {
    extern __shared__ double sp[];  // [nn][m]
    uint8_t* keep = reinterpret_cast<uint8_t*>(sp + (size_t)nn * m);
    for (int e = threadIdx.x; e < nn * m; e += blockDim.x) sp[e] = nd[e];
    for (int e = threadIdx.x; e < nn; e += blockDim.x) keep[e] = 0;
    __syncthreads();
    for (unsigned long long w = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; w < nw;
         w += (unsigned long long)gridDim.x * blockDim.x) {
        // unrank: grid_rec enumerates k_0 from R down to 0, then recurses
        int k[8];
        unsigned long long idx = w;
        int R = kLdfRes;
        for (int j = 0; j < m - 1; ++j) {
            const int q = m - j;  // parts left including this one
            int v = R;
            for (;; --v) {
                const unsigned long long cnt = binom[(R - v + q - 2) * 9 + (q - 2)];  // compositions of R-v into q-1
                if (idx < cnt) break;
                idx -= cnt;
            }
            k[j] = v;
            R -= v;
        }
        k[m - 1] = R;
        double best = -INFINITY;
        for (int i = 0; i < nn; ++i) best = fmax(best, ldf_dot(k, sp + i * m, m));
        const double tol = __dmul_rn(1e-9, fmax(1.0, fabs(best)));
        const double thr = __dsub_rn(best, tol);
        for (int i = 0; i < nn; ++i)
            if (ldf_dot(k, sp + i * m, m) >= thr) keep[i] = 1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nn; e += blockDim.x)
        if (keep[e]) keep_g[e] = 1;
}

void linear_dominance(int nn, int m, const double* nd, uint8_t* keep, int* scratch, cudaStream_t s) {
    if (m == 2) {
        k_ldf_hull2<<<1, 256, 0, s>>>(nn, nd, scratch, keep);
        MB_LAUNCH();
        return;
    }
    // compositions of r into q parts = C(r + q - 1, q - 1); table over n <= 68, r <= 8
    static unsigned long long* d_binom = nullptr;
    std::vector<unsigned long long> b(69 * 9, 0);
    for (int n = 0; n <= 68; ++n) {
        b[n * 9] = 1;
        for (int r = 1; r <= 8 && r <= n; ++r) b[n * 9 + r] = b[(n - 1) * 9 + r - 1] + (r <= n - 1 ? b[(n - 1) * 9 + r] : 0);
    }
    if (!d_binom) {
        MB_CUDA(cudaMalloc(&d_binom, sizeof(unsigned long long) * b.size()));
        MB_CUDA(cudaMemcpy(d_binom, b.data(), sizeof(unsigned long long) * b.size(), cudaMemcpyHostToDevice));
        MB_CUDA(cudaStreamSynchronize(0));  // a pageable H2D copy may return before its DMA lands
    }
    const unsigned long long nw = b[(kLdfRes + m - 1) * 9 + (m - 1)];  // C(60 + m - 1, m - 1)
    MB_CUDA(cudaMemsetAsync(keep, 0, nn, s));
    const size_t smem = sizeof(double) * (size_t)nn * m + nn;
    if (smem > 200 * 1024) throw ShapeError("linear_dominance_filter: too many nondominated points for the device sweep");
    ensure_smem((const void*)k_ldf_sweep, smem);
    const unsigned long long blocks = std::min<unsigned long long>((nw + kLdfThreads - 1) / kLdfThreads, 148ull * 8);
    k_ldf_sweep<<<(unsigned)blocks, kLdfThreads, smem, s>>>(nn, m, nd, d_binom, nw, keep);
    MB_LAUNCH();
}

// single block: compact points that are >= ref in every coordinate
// (clip_to_reference, pareto.cpp:191-205) and compute hi (pareto.cpp:248-252)
__global__ void k_hv_prep(int n, int m, const double* p, const double* ref, double* cp, int* k_out,
                          double* hi) {
    __shared__ int cnt;
    if (threadIdx.x == 0) {
        int k = 0;
        for (int i = 0; i < n; ++i) {
            bool ok = true;
            for (int j = 0; j < m; ++j)
                if (p[(long)i * m + j] < ref[j]) { ok = false; break; }
            if (ok) {
                for (int j = 0; j < m; ++j) cp[(long)k * m + j] = p[(long)i * m + j];
                ++k;
            }
        }
        cnt = k;
        *k_out = k;
        for (int j = 0; j < m; ++j) {
            double h = ref[j];
            for (int i = 0; i < k; ++i) h = fmax(h, cp[(long)i * m + j]);
            hi[j] = h;
        }
    }
    __syncthreads();
    (void)cnt;
}

constexpr int kHvThreads = 256;
template <int M>  // objectives (compile time: the sample point stays in registers)
__global__ void __launch_bounds__(kHvThreads) k_hv_mc(const double* __restrict__ cp, const int* kp,
                                                      const double* __restrict__ ref,
                                                      const double* __restrict__ hi, uint64_t samples,
                                                      uint64_t key, uint64_t ctr, unsigned long long* hits) {
    constexpr int m = M;
    extern __shared__ double pts[];  // [k][m]
    const int k = *kp;
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) pts[e] = cp[e];
    double r[M], span[M];
#pragma unroll
    for (int j = 0; j < m; ++j) {
        r[j] = ref[j];
        span[j] = __dsub_rn(hi[j], ref[j]);
    }
    __syncthreads();
    unsigned long long local = 0;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < samples;
         s += (uint64_t)gridDim.x * blockDim.x) {
        double x[M];
#pragma unroll
        for (int j = 0; j < m; ++j)
            x[j] = __dadd_rn(r[j], __dmul_rn(span[j], word_double(rng_word(key, ctr + s * m + j + 1))));
        for (int i = 0; i < k; ++i) {
            const double* pi = pts + i * m;
            bool inside = true;
#pragma unroll
            for (int j = 0; j < m; ++j) inside = inside && !(x[j] > pi[j]);
            if (inside) { ++local; break; }
        }
    }
    // warp + block reduction of an integer count: order-independent, exact
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    __shared__ unsigned long long wsum[kHvThreads / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kHvThreads / 32; ++w) t += wsum[w];
        atomicAdd(hits, t);
    }
}

void hv_mc(int n, int m, const double* pts, const double* ref, uint64_t samples, uint64_t key, uint64_t ctr,
           unsigned long long* hits, double* hi_out, cudaStream_t s) {
    // scratch: compacted points + count live right after hi_out (caller sizes it n*m + 2m + 2)
    double* cp = hi_out + 8;
    int* kp = reinterpret_cast<int*>(cp + (long)n * m);
    k_hv_prep<<<1, 32, 0, s>>>(n, m, pts, ref, cp, kp, hi_out);
    MB_LAUNCH();
    MB_CUDA(cudaMemsetAsync(hits, 0, sizeof(unsigned long long), s));
    const size_t smem = (size_t)n * m * sizeof(double);
#define MB_HV(M_)                                                                                      \
    case M_:                                                                                           \
        MB_CUDA(cudaFuncSetAttribute(k_hv_mc<M_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        k_hv_mc<M_><<<148 * 8, kHvThreads, smem, s>>>(cp, kp, ref, hi_out, samples, key, ctr, hits);       \
        break;
    switch (m) {
        MB_HV(1) MB_HV(2) MB_HV(3) MB_HV(4) MB_HV(5) MB_HV(6) MB_HV(7) MB_HV(8)
        default: throw ShapeError("hypervolume: objective count must be in [1, 8]");
    }
#undef MB_HV
    MB_LAUNCH();
}

}  // namespace mb200
