// TEST INFRASTRUCTURE ONLY. The mo-humanoid6 synthetic environment as a
// reference-side BatchedEnv subclass (env.hpp:37-99 contract), so the
// COMPILED REFERENCE's collect_rollouts / train loop can run configs 3/5
// for the CPU baseline. Dynamics are defined once in
// paper_2603_09237_b200/csrc/humanoid6_params.h (fp64 here).
#include <cmath>
#include <memory>
#include <vector>

#include "morlax/env.hpp"
#include "../paper_2603_09237_b200/csrc/humanoid6_params.h"

using namespace morlax;

namespace {
constexpr double kCx[12] = H6_CX, kCy[12] = H6_CY, kCz[12] = H6_CZ, kCr[12] = H6_CR,
                 kCp[12] = H6_CP, kCw[12] = H6_CW;

class Humanoid6Env final : public BatchedEnv {
public:
    explicit Humanoid6Env(int n) : BatchedEnv(make_spec(), n), s_((size_t)n * H6_OBS, 0.0) {}
    static EnvSpec make_spec() {
        EnvSpec s;
        s.name = "mo-humanoid6";
        s.obs_dim = H6_OBS;
        s.act_dim = H6_ACT;
        s.m = H6_M;
        s.max_episode_steps = H6_HORIZON;
        s.objective_names = {"forward", "energy", "upright", "lateral", "smooth", "height"};
        s.hv_reference = H6_HV_REF;
        return s;
    }

protected:
    void do_reset(int i, Rng& st) override {
        double* s = s_.data() + (size_t)i * H6_OBS;
        for (int k = 0; k < H6_OBS; ++k) s[k] = st.uniform(-H6_INIT, H6_INIT);
    }
    void do_step(int i, const double* a, double* r, bool* term) override {
        double* s = s_.data() + (size_t)i * H6_OBS;
        double* q = s;
        double* qd = s + 12;
        double* ee = s + 24;
        double sx = 0, sy = 0, sz = 0, sr = 0, sp = 0, sw = 0, asq = 0, qsq = 0;
        for (int j = 0; j < 12; ++j) {
            ee[j] += H6_ALPHA * (a[j] - ee[j]);
            qd[j] += H6_DT * (H6_KT * ee[j] - H6_KP * q[j] - H6_KD * qd[j]);
            q[j] += H6_DT * qd[j];
            const double sj = std::tanh(qd[j]);
            sx += kCx[j] * sj;
            sy += kCy[j] * sj;
            sw += kCw[j] * sj;
            sz += kCz[j] * ee[j];
            sr += kCr[j] * ee[j];
            sp += kCp[j] * ee[j];
            asq += a[j] * a[j];
            qsq += qd[j] * qd[j];
        }
        double &h = s[36], &vx = s[37], &vy = s[38], &vz = s[39], &roll = s[40], &pitch = s[41],
               &wx = s[42], &wy = s[43], &wz = s[44];
        vx += H6_DT * (sx - H6_DRAG * vx);
        vy += H6_DT * (sy - H6_DRAG * vy);
        vz += H6_DT * (sz - H6_KH * h - H6_DZ * vz);
        h += H6_DT * vz;
        wx += H6_DT * (sr - H6_KA * roll - H6_DA * wx);
        roll += H6_DT * wx;
        wy += H6_DT * (sp - H6_KA * pitch - H6_DA * wy);
        pitch += H6_DT * wy;
        wz += H6_DT * (sw - H6_DRAG * wz);
        r[0] = vx;
        r[1] = -asq / 12.0;
        r[2] = -(roll * roll + pitch * pitch);
        r[3] = vy;
        r[4] = -0.1 * qsq / 12.0;
        r[5] = -(h * h + 0.1 * wz * wz);
        *term = std::fabs(roll) > H6_FALL || std::fabs(pitch) > H6_FALL;
    }
    void write_obs(int i, double* out) const override {
        const double* s = s_.data() + (size_t)i * H6_OBS;
        for (int k = 0; k < H6_OBS; ++k) out[k] = s[k];
    }

private:
    std::vector<double> s_;
};
}  // namespace

std::unique_ptr<BatchedEnv> make_humanoid6_env(int n) { return std::make_unique<Humanoid6Env>(n); }
