// K9b: exact hypervolume on the device for any m <= 8 (fp64).
//
// The reference is exact only for m <= 4 (hv_recursive, pareto.cpp:145-189,
// slicing along the last objective) and falls back to Monte-Carlo above
// (pareto.cpp:209-230). Here one algorithm serves every m: the WFG
// exclusive-volume recursion
//     hv(S) = sum_k [ box(s_k) - hv( nd( limit(s_k, S[k+1:]) ) ) ]
// (S sorted by the last objective, descending; limit(p, X) = {min(x, p)};
// nd = nondominated with duplicates collapsed), with the m == 2 base case
// the reference's sweep (pareto.cpp:154-166) and m == 1 its maximum. The
// oracle (oracle/morlax_oracle.c mo_hypervolume_wfg) is the same recursion on
// the host; for m <= 4 both are checked against the reference's own exact
// recursion.
//
// Work shape (config 5: 1020 nondominated 6-D points): the top-level limit
// sets have ~1000 points before nd and 4..90 after; below that the
// recursion is ~15 M small nodes (a few to a few dozen points each). So:
//   1. k_hv_top     (one block)  clip (pareto.cpp:191-205) + nd + sort the
//                                input: one rank-scatter;
//   2. k_hv_level1  (block per top term k) L1_k = nd(limit(top_k, top[k+1:]))
//                                -- the large O(c^2 m) dominance tests;
//   3. k_hv_sub     (persistent, one WARP per subtask (k, j), ~40 k of
//                                them) incl(L1_k[j]) - hv(nd(limit(L1_k[j],
//                                L1_k[j+1:]))) by a depth-first recursion
//                                with warp-synchronous limit / nd / sort
//                                steps and a per-warp global arena;
//   4. k_hv_reduce  (one block)  ordered sums: hv(L1_k) = sum_j sub(k, j),
//                                total = sum_k box(top_k) - hv(L1_k).
// Every sum is in a fixed order, so the value is deterministic. A warp
// arena overflow (adversarial fronts whose limit sets do not shrink) sets a
// flag and the host re-runs step 3 with the worst-case arena.
#include <map>
#include <mutex>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mb200 {

namespace {
constexpr int kHvMaxM = 8;
constexpr int kHvMaxN = 4096;
constexpr int kSubWarps = 8;  // warps per k_hv_sub block

struct HvFrame {
    long off;      // arena offset (doubles) of this frame's point set
    int size, k;   // set size, next term index
    double total;  // sum of finished terms
    double incl;   // box volume of the term being expanded
};

__device__ __forceinline__ double box_vol(const double* p, const double* ref, int m) {
    double v = 1.0;
    for (int d = 0; d < m; ++d) v = __dmul_rn(v, __dsub_rn(p[d], ref[d]));
    return v;
}

// weak domination by a different vector, or an equal vector earlier
__device__ __forceinline__ bool dropped_by(const double* pr, const double* pq, int m, bool earlier) {
    bool ne = false;
    for (int d = 0; d < m; ++d) {
        if (pr[d] < pq[d]) return false;
        if (pr[d] != pq[d]) ne = true;
    }
    return ne || earlier;
}

// ---- block-wide: dst <- nd(raw[0..c)) sorted by `key` desc (ties: index asc)
__device__ int block_nd_sort(const double* raw, int c, int m, int key, double* dst, int* flag) {
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
        const double* pq = raw + (long)q * m;
        bool keep = true;
        for (int r = 0; r < c && keep; ++r)
            if (r != q && dropped_by(raw + (long)r * m, pq, m, r < q)) keep = false;
        flag[q] = keep;
    }
    __syncthreads();
    int kept = 0;
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
        if (!flag[q]) continue;
        ++kept;
        const double kq = raw[(long)q * m + key];
        int rank = 0;
        for (int r = 0; r < c; ++r) {
            if (!flag[r]) continue;
            const double kr = raw[(long)r * m + key];
            rank += (kr > kq || (kr == kq && r < q));
        }
        for (int d = 0; d < m; ++d) dst[(long)rank * m + d] = raw[(long)q * m + d];
    }
    if (kept) atomicAdd(&s_cnt, kept);
    __syncthreads();
    const int n = s_cnt;
    __syncthreads();
    return n;
}

// ---- warp-wide version (M objectives at compile time: the tested point in
// registers); bits: per-warp keep mask (c <= kHvMaxN)
template <int M>
__device__ int warp_nd_sort(const double* raw, int c, int key, double* dst, unsigned* bits) {
    constexpr int m = M;
    const int lane = threadIdx.x & 31;
    const int words = (c + 31) >> 5;
    for (int w = 0; w < words; ++w) {
        const int q = w * 32 + lane;
        bool keep = q < c;
        if (keep) {
            double pq[M];
#pragma unroll
            for (int d = 0; d < M; ++d) pq[d] = raw[(long)q * m + d];
            for (int r = 0; r < c && keep; ++r) {
                if (r == q) continue;
                const double* pr = raw + (long)r * m;
                bool ge = true, ne = false;
#pragma unroll
                for (int d = 0; d < M; ++d) {
                    const double x = pr[d];
                    ge = ge && x >= pq[d];
                    ne = ne || x != pq[d];
                }
                if (ge && (ne || r < q)) keep = false;
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) bits[w] = b;
    }
    __syncwarp();
    int n = 0;
    for (int w = 0; w < words; ++w) n += __popc(bits[w]);
    for (int w = 0; w < words; ++w) {
        const int q = w * 32 + lane;
        if (q >= c || !((bits[w] >> lane) & 1u)) continue;
        const double kq = raw[(long)q * m + key];
        int rank = 0;
        for (int r = 0; r < c; ++r) {
            if (!((bits[r >> 5] >> (r & 31)) & 1u)) continue;
            const double kr = raw[(long)r * m + key];
            rank += (kr > kq || (kr == kq && r < q));
        }
        for (int d = 0; d < m; ++d) dst[(long)rank * m + d] = raw[(long)q * m + d];
    }
    __syncwarp();
    return n;
}

// 2-D sweep of a set sorted by x descending (pareto.cpp:154-166)
__device__ double sweep2(const double* X, int n, const double* ref) {
    double area = 0.0, yprev = ref[1];
    for (int i = 0; i < n; ++i) {
        const double y = X[2 * i + 1];
        if (y > yprev) {
            area = __dadd_rn(area, __dmul_rn(__dsub_rn(X[2 * i], ref[0]), __dsub_rn(y, yprev)));
            yprev = y;
        }
    }
    return area;
}

// 1. top-level set: clip, nd, sort. One block of 1024.
__global__ void __launch_bounds__(1024) k_hv_top(int n, int m, const double* __restrict__ pts,
                                                 const double* __restrict__ ref, double* raw, double* top,
                                                 int* s0_out, int* clipped_out, int* flag) {
    __shared__ int cnt;
    if (threadIdx.x == 0) {  // clip keeping input order (serial prefix, n <= 4096)
        int k = 0, c = 0;
        for (int i = 0; i < n; ++i) {
            bool ok = true;
            for (int j = 0; j < m; ++j)
                if (pts[(long)i * m + j] < ref[j]) { ok = false; break; }
            if (ok) {
                for (int j = 0; j < m; ++j) raw[(long)k * m + j] = pts[(long)i * m + j];
                ++k;
            } else {
                ++c;
            }
        }
        cnt = k;
        *clipped_out = c;
    }
    __syncthreads();
    const int s0 = block_nd_sort(raw, cnt, m, m == 2 ? 0 : m - 1, top, flag);
    if (threadIdx.x == 0) *s0_out = s0;
}

// 2. L1_k = nd(limit(top_k, top[k+1:])) into L1 + k * s0 * m (block per k)
__global__ void __launch_bounds__(256) k_hv_level1(const double* __restrict__ top, const int* s0p, int m,
                                                   double* L1, double* raw_all, int* sz1, int* flag_all) {
    const int s0 = *s0p;
    const int k = blockIdx.x;
    if (k >= s0) return;
    const int c = s0 - k - 1;
    double* raw = raw_all + (long)k * s0 * m;
    int* flag = flag_all + (long)k * s0;
    const double* p = top + (long)k * m;
    for (int q = threadIdx.x; q < c; q += blockDim.x)
        for (int d = 0; d < m; ++d) raw[(long)q * m + d] = fmin(top[(long)(k + 1 + q) * m + d], p[d]);
    __syncthreads();
    const int n1 = block_nd_sort(raw, c, m, m - 1, L1 + (long)k * s0 * m, flag);
    if (threadIdx.x == 0) sz1[k] = n1;
}

// subtask offsets: off[k] = sum_{k' < k} sz1[k'] (one block, ordered)
__global__ void k_hv_offsets(const int* s0p, const int* sz1, int* off, int* nsub, int* cmax) {
    if (threadIdx.x != 0) return;
    int acc = 0, mx = 0;
    for (int k = 0; k < *s0p; ++k) {
        off[k] = acc;
        acc += sz1[k];
        mx = max(mx, sz1[k]);
    }
    off[*s0p] = acc;
    *nsub = acc;
    *cmax = mx;
}

// 3. subtask (k, j): incl(L1_k[j]) - hv(nd(limit(L1_k[j], L1_k[j+1:]))),
// one warp each, depth-first over an explicit frame stack
template <int M>
__global__ void __launch_bounds__(kSubWarps * 32) k_hv_sub(const double* __restrict__ L1, const int* s0p,
                                                            const int* __restrict__ sz1,
                                                            const int* __restrict__ off, const int* nsubp, int m,
                                                            const double* __restrict__ ref_g, double* arena_base,
                                                            long arena_cap, HvFrame* frames_base, int frame_stride, int* task_ctr,
                                                            double* sub, int* overflow) {
    __shared__ unsigned bits_all[kSubWarps][kHvMaxN / 32];
    __shared__ double ref[kHvMaxM];
    if (threadIdx.x < m) ref[threadIdx.x] = ref_g[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long wid = (long)blockIdx.x * kSubWarps + wib;
    unsigned* bits = bits_all[wib];
    double* arena = arena_base + wid * arena_cap;
    const int s0 = *s0p, nsub = *nsubp;
    HvFrame* st = frames_base + wid * (long)frame_stride;
    const int key = m - 1;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(task_ctr, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nsub) break;
        int lo = 0, hi = s0;  // off[lo] <= t < off[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= t) lo = mid;
            else hi = mid;
        }
        const int k = lo, j = t - off[k];
        const double* X0 = L1 + (long)k * s0 * m;
        const int c0 = sz1[k];
        const double* p0 = X0 + (long)j * m;
        const double incl0 = box_vol(p0, ref, m);
        const int cc0 = c0 - j - 1;
        double hv = 0.0;
        bool ovf = 2L * cc0 * m > arena_cap;
        if (!ovf && cc0 > 0) {
            double* raw = arena + (long)cc0 * m;
            for (int q = lane; q < cc0; q += 32)
                for (int d = 0; d < m; ++d) raw[(long)q * m + d] = fmin(X0[(long)(j + 1 + q) * m + d], p0[d]);
            __syncwarp();
            const int n1 = warp_nd_sort<M>(raw, cc0, key, arena, bits);
            if (n1 == 1) {
                hv = box_vol(arena, ref, m);
            } else if (n1 > 1) {
                if (lane == 0) st[0] = HvFrame{0, n1, 0, 0.0, 0.0};
                int depth = 0;
                __syncwarp();
                for (;;) {
                    const HvFrame F = st[depth];
                    if (F.k == F.size) {
                        if (depth == 0) {
                            hv = F.total;
                            break;
                        }
                        if (lane == 0) {
                            HvFrame& P = st[depth - 1];
                            P.total = __dadd_rn(P.total, __dsub_rn(P.incl, F.total));
                            P.k += 1;
                        }
                        --depth;
                        __syncwarp();
                        continue;
                    }
                    const double* X = arena + F.off;
                    const double* p = X + (long)F.k * m;
                    const double incl = box_vol(p, ref, m);
                    const int cc = F.size - F.k - 1;
                    const long child = F.off + (long)F.size * m;
                    if (child + 2L * cc * m > arena_cap) {
                        ovf = true;
                        break;
                    }
                    int n2 = 0;
                    if (cc > 0) {
                        double* raw2 = arena + child + (long)cc * m;
                        for (int q = lane; q < cc; q += 32)
                            for (int d = 0; d < m; ++d)
                                raw2[(long)q * m + d] = fmin(X[(long)(F.k + 1 + q) * m + d], p[d]);
                        __syncwarp();
                        n2 = warp_nd_sort<M>(raw2, cc, key, arena + child, bits);
                    }
                    if (n2 >= 2) {
                        if (lane == 0) {
                            st[depth].incl = incl;
                            st[depth + 1] = HvFrame{child, n2, 0, 0.0, 0.0};
                        }
                        ++depth;
                    } else if (lane == 0) {
                        HvFrame& G = st[depth];
                        const double sub_hv = n2 == 1 ? box_vol(arena + child, ref, m) : 0.0;
                        G.total = __dadd_rn(G.total, __dsub_rn(incl, sub_hv));
                        G.k += 1;
                    }
                    __syncwarp();
                }
            }
        }
        if (lane == 0) {
            if (ovf) atomicExch(overflow, 1);
            sub[t] = __dsub_rn(incl0, hv);
        }
        __syncwarp();
    }
}

// 4. ordered sums (one block): per k in parallel, then the total in order
__global__ void k_hv_reduce(const double* __restrict__ top, const int* s0p, const int* __restrict__ off,
                            const double* __restrict__ sub, int m, const double* __restrict__ ref, double* term,
                            double* out) {
    const int s0 = *s0p;
    for (int k = threadIdx.x; k < s0; k += blockDim.x) {
        double h = 0.0;
        for (int t = off[k]; t < off[k + 1]; ++t) h = __dadd_rn(h, sub[t]);
        term[k] = __dsub_rn(box_vol(top + (long)k * m, ref, m), h);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < s0; ++k) s = __dadd_rn(s, term[k]);
        *out = s;
    }
}

__global__ void k_hv_small(const double* top, const int* s0p, int m, const double* ref, double* out) {
    if (threadIdx.x != 0) return;
    const int s0 = *s0p;
    if (s0 == 0) {
        *out = 0.0;
    } else if (m == 1) {
        double best = ref[0];
        for (int i = 0; i < s0; ++i) best = fmax(best, top[i]);
        *out = __dsub_rn(best, ref[0]);
    } else {
        *out = sweep2(top, s0, ref);
    }
}

// device scratch reused across calls (grown on demand, never shrunk): the
// recursion arenas are hundreds of MB and cudaMalloc / cudaFree of that size
// per call cost more than the computation
struct ScratchPool {
    void* p[16] = {};
    size_t cap[16] = {};
    void* get(int slot, size_t bytes) {
        if (bytes == 0) bytes = 1;
        if (bytes > cap[slot]) {
            if (p[slot]) cudaFree(p[slot]);
            MB_CUDA(cudaMalloc(&p[slot], bytes));
            cap[slot] = bytes;
        }
        return p[slot];
    }
};
// one pool per device; hv_exact holds the pool's mutex for the whole call
// (it is synchronous), so concurrent host threads never share scratch
struct DevicePools {
    std::mutex mu;
    std::map<int, ScratchPool> pools;
};
DevicePools g_pools;
thread_local ScratchPool* t_pool = nullptr;
template <typename T>
struct DevScratch {
    T* p = nullptr;
    DevScratch(int slot, size_t n) { p = static_cast<T*>(t_pool->get(slot, sizeof(T) * (n ? n : 1))); }
};
}  // namespace

void hv_exact(int n, int m, const double* d_pts, const double* d_ref, double* value, int* clipped,
              cudaStream_t s) {
    if (m < 1 || m > kHvMaxM) throw ShapeError("hypervolume: objective count must be in [1, 8]");
    if (n > kHvMaxN) throw ShapeError("exact hypervolume: at most 4096 points");
    int cur_dev = 0;
    MB_CUDA(cudaGetDevice(&cur_dev));
    std::lock_guard<std::mutex> lk(g_pools.mu);
    t_pool = &g_pools.pools[cur_dev];
    const long nn = n > 0 ? n : 1;
    DevScratch<double> raw(0, nn * m), top(1, nn * m), out(2, 1);
    DevScratch<int> ints(3, 8), flag(4, nn);
    int *s0p = ints.p, *clp = ints.p + 1, *ctr = ints.p + 2, *ovf = ints.p + 3, *nsubp = ints.p + 4,
        *cmaxp = ints.p + 5;
    MB_CUDA(cudaMemsetAsync(ints.p, 0, sizeof(int) * 8, s));
    k_hv_top<<<1, 1024, 0, s>>>(n, m, d_pts, d_ref, raw.p, top.p, s0p, clp, flag.p);
    MB_LAUNCH();
    int s0 = 0;
    MB_CUDA(cudaMemcpyAsync(&s0, s0p, sizeof(int), cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(clipped, clp, sizeof(int), cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaStreamSynchronize(s));
    if (m <= 2 || s0 == 0) {
        k_hv_small<<<1, 32, 0, s>>>(top.p, s0p, m, d_ref, out.p);
        MB_LAUNCH();
        MB_CUDA(cudaMemcpyAsync(value, out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        MB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // 2. level-1 limit sets (worst case s0 points each)
    DevScratch<double> L1(5, (size_t)s0 * s0 * m), raw1(6, (size_t)s0 * s0 * m);
    DevScratch<int> sz1(7, s0), off(8, s0 + 1), flag1(9, (size_t)s0 * s0);
    k_hv_level1<<<s0, 256, 0, s>>>(top.p, s0p, m, L1.p, raw1.p, sz1.p, flag1.p);
    MB_LAUNCH();
    k_hv_offsets<<<1, 32, 0, s>>>(s0p, sz1.p, off.p, nsubp, cmaxp);
    MB_LAUNCH();
    int nsub = 0, cmax = 0;
    MB_CUDA(cudaMemcpyAsync(&nsub, nsubp, sizeof(int), cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaMemcpyAsync(&cmax, cmaxp, sizeof(int), cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaStreamSynchronize(s));
    DevScratch<double> sub(10, nsub), term(11, s0);
    // 3. warp subtasks; arena per warp: sets on the recursion path + scratch
    int dev = 0, sms = 148;
    MB_CUDA(cudaGetDevice(&dev));
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long worst = ((long)cmax * (cmax + 1) / 2 + 2L * cmax) * m;
    long cap = std::min<long>(worst, (64L + 2L) * cmax * m);
    int blocks = std::max(1, std::min(sms * 4, (nsub + kSubWarps - 1) / kSubWarps));
    for (int attempt = 0; attempt < 2; ++attempt) {
        const long warps = (long)blocks * kSubWarps;
        DevScratch<double> arena(12, (size_t)(cap > 0 ? cap : 1) * warps);
        DevScratch<HvFrame> frames(13, (size_t)warps * (cmax + 1));
        MB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int) * 2, s));
        auto sub_kernel = m == 3 ? k_hv_sub<3> : m == 4 ? k_hv_sub<4> : m == 5 ? k_hv_sub<5> : m == 6 ? k_hv_sub<6>
                        : m == 7 ? k_hv_sub<7> : k_hv_sub<8>;
        sub_kernel<<<blocks, kSubWarps * 32, 0, s>>>(L1.p, s0p, sz1.p, off.p, nsubp, m, d_ref, arena.p, cap,
                                                    frames.p, cmax + 1, ctr, sub.p, ovf);
        MB_LAUNCH();
        int of = 0;
        MB_CUDA(cudaMemcpyAsync(&of, ovf, sizeof(int), cudaMemcpyDeviceToHost, s));
        MB_CUDA(cudaStreamSynchronize(s));
        if (!of) break;
        if (cap == worst) throw ShapeError("exact hypervolume: recursion arena exhausted");
        cap = worst;
        // keep the worst-case arena within ~4 GB
        blocks = (int)std::max<long>(1, std::min<long>(blocks, (4L << 30) / (8L * worst * kSubWarps)));
    }
    k_hv_reduce<<<1, 256, 0, s>>>(top.p, s0p, off.p, sub.p, m, d_ref, term.p, out.p);
    MB_LAUNCH();
    MB_CUDA(cudaMemcpyAsync(value, out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    MB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mb200
