// Per-preference-group policy forward through generated weights (policy.cu).
#pragma once
#include <vector>

#include "trainer.h"

namespace mb200 {

struct GroupPolicy {
    HyperNet h;
    int G = 0, R = 0, Rp = 0;  // groups, rows per group, rows per group padded to 128
    Img X;                     // observation image [G*Rp][obs]
    std::vector<Img> A;        // hidden activations [G*Rp][width]
    float* out_pad = nullptr;  // [G*Rp][16] output layer (pre-squash means)
    int* rowmap = nullptr;     // padded row -> input row (-1 = padding)
    int* goff = nullptr;       // group row offsets (g * Rp)
    cudaStream_t s2 = nullptr;  // side stream: the observation image while theta is generated
    cudaEvent_t ev_in = nullptr, ev_x = nullptr;
    GroupPolicy(int m, int F, const std::vector<int>& fh, const std::vector<int>& sizes, bool out_tanh,
                bool has_log_std, int G, int R);
    ~GroupPolicy();
    GroupPolicy(const GroupPolicy&) = delete;
    GroupPolicy& operator=(const GroupPolicy&) = delete;
    // d_w [G][m] (simplex rows), d_obs [G*R][obs] fp32 -> d_pre [G*R][out] fp32
    void forward(const float* d_w, const float* d_obs, float* d_pre, cudaStream_t s);
    double flops() const;  // algorithmic FLOPs of one forward
};

}  // namespace mb200
