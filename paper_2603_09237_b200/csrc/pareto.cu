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
__global__ void __launch_bounds__(kHvThreads) k_hv_mc(int m, const double* __restrict__ cp, const int* kp,
                                                      const double* __restrict__ ref,
                                                      const double* __restrict__ hi, uint64_t samples,
                                                      uint64_t key, uint64_t ctr, unsigned long long* hits) {
    extern __shared__ double pts[];  // [k][m]
    const int k = *kp;
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) pts[e] = cp[e];
    double r[8], span[8];
    for (int j = 0; j < m; ++j) {
        r[j] = ref[j];
        span[j] = __dsub_rn(hi[j], ref[j]);
    }
    __syncthreads();
    unsigned long long local = 0;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < samples;
         s += (uint64_t)gridDim.x * blockDim.x) {
        double x[8];
        for (int j = 0; j < m; ++j)
            x[j] = __dadd_rn(r[j], __dmul_rn(span[j], word_double(rng_word(key, ctr + s * m + j + 1))));
        for (int i = 0; i < k; ++i) {
            const double* pi = pts + i * m;
            bool inside = true;
            for (int j = 0; j < m; ++j)
                if (x[j] > pi[j]) { inside = false; break; }
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
    static size_t configured = 0;
    if (smem > configured) {
        MB_CUDA(cudaFuncSetAttribute(k_hv_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    k_hv_mc<<<148 * 8, kHvThreads, smem, s>>>(m, cp, kp, ref, hi_out, samples, key, ctr, hits);
    MB_LAUNCH();
}

}  // namespace mb200
