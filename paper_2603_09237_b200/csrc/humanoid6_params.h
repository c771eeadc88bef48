/* mo-humanoid6: the "humanoid-scale synthetic 6-objective env" named by
 * BASELINE.json configs 3/5. It does not exist in the reference
 * (SURVEY.md Appendix A.3), so it is DEFINED here, once, and included by
 * the CUDA kernels (fp32), the C oracle (fp64) and the reference-side
 * BatchedEnv subclass used for the CPU baseline (oracle/ref_humanoid6.cpp).
 *
 * Design follows the reference's environment contract (env.hpp:26-36):
 * deterministic dynamics, all stochasticity in the initial state
 * (45 uniform draws in [-0.1, 0.1] from the instance stream, index order),
 * actions clamped to [-1, 1] by the BatchedEnv wrapper.
 *
 * State == observation (45):
 *   [ 0,12) q   joint angles          [12,24) qd  joint velocities
 *   [24,36) e   actuator (lagged torque) states
 *   36 h  torso height deviation      37 vx  38 vy  39 vz  (torso velocity)
 *   40 roll  41 pitch                 42 wx  43 wy  (roll / pitch rates)
 *   44 wz yaw rate
 * Step (dt = H6_DT), pre-clamped action a[12]:
 *   e  += H6_ALPHA (a - e)
 *   qd += dt (H6_KT e - H6_KP q - H6_KD qd);  q += dt qd   (semi-implicit)
 *   s_j = tanh(qd_j)
 *   vx += dt (sum CX_j s_j - H6_DRAG vx)
 *   vy += dt (sum CY_j s_j - H6_DRAG vy)
 *   vz += dt (sum CZ_j e_j - H6_KH h - H6_DZ vz);  h += dt vz
 *   wx += dt (sum CR_j e_j - H6_KA roll  - H6_DA wx); roll  += dt wx
 *   wy += dt (sum CP_j e_j - H6_KA pitch - H6_DA wy); pitch += dt wy
 *   wz += dt (sum CW_j s_j - H6_DRAG wz)
 * Rewards (6, on the post-step state):
 *   r0 = vx                         forward speed
 *   r1 = -(sum a_j^2) / 12          energy
 *   r2 = -(roll^2 + pitch^2)        uprightness
 *   r3 = vy                         lateral speed
 *   r4 = -0.1 (sum qd_j^2) / 12     joint smoothness
 *   r5 = -(h^2 + 0.1 wz^2)          height / heading stability
 * Terminated when |roll| > 1 or |pitch| > 1 (fall). Truncation at
 * H6_HORIZON steps (BatchedEnv).
 */
#ifndef MORLAX_HUMANOID6_PARAMS_H
#define MORLAX_HUMANOID6_PARAMS_H

#define H6_OBS 45
#define H6_ACT 12
#define H6_M 6
#define H6_HORIZON 1000
#define H6_INIT 0.1
#define H6_DT 0.05
#define H6_ALPHA 0.25
#define H6_KT 4.0
#define H6_KP 2.0
#define H6_KD 0.5
#define H6_DRAG 0.5
#define H6_KH 2.0
#define H6_DZ 1.0
#define H6_KA 1.5
#define H6_DA 0.5
#define H6_FALL 1.0

/* Coupling tables (joint -> torso). Exactly representable in fp32. */
#define H6_CX {0.25, -0.125, 0.25, -0.0625, 0.1875, -0.125, 0.25, -0.125, 0.25, -0.0625, 0.1875, -0.125}
#define H6_CY {0.125, 0.1875, -0.125, -0.1875, 0.125, -0.125, -0.125, -0.1875, 0.125, 0.1875, -0.125, 0.125}
#define H6_CZ {0.125, 0.125, 0.0625, 0.0625, -0.0625, -0.0625, 0.125, 0.125, 0.0625, 0.0625, -0.0625, -0.0625}
#define H6_CR {0.25, -0.25, 0.125, -0.125, 0.0625, -0.0625, -0.25, 0.25, -0.125, 0.125, -0.0625, 0.0625}
#define H6_CP {0.125, 0.125, -0.25, -0.25, 0.125, 0.125, 0.0625, 0.0625, -0.125, -0.125, 0.0625, 0.0625}
#define H6_CW {0.0625, -0.0625, 0.125, -0.125, 0.0625, -0.0625, -0.0625, 0.0625, -0.125, 0.125, -0.0625, 0.0625}

/* Hypervolume reference point: worst bounded per-objective return over a
 * 1000-step episode is far below these; they bound T=64 windows. */
#define H6_HV_REF {-100.0, -100.0, -100.0, -100.0, -100.0, -100.0}

#endif
