// qb_k_adjoint.cu -- K1 adjoint kernels: BPTT over a whole horizon in one
// launch (gradients.rollout_grad, gradients.py:218-237) and the single-step
// VJP.  One env per thread walks t = T-1 .. 0 keeping lambda (17) in
// registers; per step it reads the saved pre-step state (17 planes) and the
// action (16 B), and writes the action gradient (16 B): ~236 B/env-step of
// HBM traffic, plus the optional deterministic env-sum of the action
// gradient (k_env_sum) that feeds the multi-GPU all-reduce of a shared
// open-loop action sequence.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "qb_adjoint.cuh"
#include "qb_internal.h"

namespace {

// A/B switch: QB_ADJOINT_FUSED=1 keeps the one-thread-per-env adjoint
bool getenv_flag(const char *name) {
    const char *v = std::getenv(name);
    return v && std::strcmp(v, "0") != 0 && v[0] != 0;
}

template <class R, int KIND, int SUB>
__global__ void __launch_bounds__(128) k_rollout_bwd(DynConsts<R> C, long long n, long long ld, int T,
                                                     const typename storage_of<R>::type *tape,
                                                     const typename storage_of<R>::type *actions,
                                                     const typename storage_of<R>::type *g_traj,
                                                     typename storage_of<R>::type *grad_actions,
                                                     typename storage_of<R>::type *grad_init, uint8_t *boundary) {
    using S = typename storage_of<R>::type;
    // FP32 2-substep build: the first substep's stages go through shared
    // memory (one column of 52 floats per thread) instead of being recomputed
    constexpr bool kCache = SUB == 2 && std::is_same<R, float>::value;
    __shared__ float stage_s[kCache ? 52 * 128 : 1];
    StageCache<R> cache{nullptr, 0};
    if constexpr (kCache) cache = StageCache<R>{reinterpret_cast<R *>(stage_s) + threadIdx.x, 128};
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < n;
    const long long ii = live ? i : 0;
    const bool single = T < 0;
    const int steps = single ? 1 : T;
    const long long block = 17 * ld;
    R lam[17];
    const S *g_last = single ? g_traj : g_traj + (long long)T * block;
#pragma unroll
    for (int k = 0; k < 17; ++k) lam[k] = R(g_last[k * ld + ii]);
    bool flag = false;
    // software pipeline: step t-1's tape state and action and step t's
    // trajectory gradient are loaded while step t is computed (at C4 sizes
    // each SM sub-partition runs about one warp, so nothing else hides the
    // L2 latency)
    S xn[17], an[4], gn[17];
    auto load_step = [&](int t) {
        const S *xs = tape + (long long)t * block;
#pragma unroll
        for (int k = 0; k < 17; ++k) xn[k] = xs[k * ld + ii];
        const S *ap = actions + ((long long)t * n + ii) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) an[k] = ap[k];
    };
    load_step(steps - 1);
    for (int t = steps - 1; t >= 0; --t) {
        R x[17], a[4], cmd[4];
#pragma unroll
        for (int k = 0; k < 17; ++k) x[k] = R(xn[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = R(an[k]);
        if (t > 0) load_step(t - 1);
        if (!single) {
            const S *gt = g_traj + (long long)t * block;
#pragma unroll
            for (int k = 0; k < 17; ++k) gn[k] = gt[k * ld + ii];
        }
        command_to_speeds<R, KIND>(C, x, a, cmd);
        R cb[4] = {R(0.0), R(0.0), R(0.0), R(0.0)};
        dyn_step_vjp<R, SUB>(C, x, cmd, lam, cb, flag, cache);  // lam <- J^T lam (dynamics part)
        R ga[4];
        if constexpr (KIND == QB_CMD_ROTOR) {
#pragma unroll
            for (int k = 0; k < 4; ++k) ga[k] = cb[k];
        } else if constexpr (KIND == QB_CMD_SRT) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                bool f2 = false;
                R m = clip_mask(a[k], C.flo, C.fhi, f2);
                ga[k] = cb[k] * m * speed_of_thrust_grad(C, np_clip(a[k], C.flo, C.fhi));
            }
        } else {  // CTBR: through the rate loop + mixer; also adds d/d omega to lam
            ctbr_vjp(C, x, a[0], a[1], a[2], a[3], cb, ga, lam);
        }
        S *gp = grad_actions + ((long long)t * n + ii) * 4;
        if (live) {
#pragma unroll
            for (int k = 0; k < 4; ++k) gp[k] = to_store(ga[k]);
        }
        if (!single) {
#pragma unroll
            for (int k = 0; k < 17; ++k) lam[k] = lam[k] + R(gn[k]);
        }
    }
    if (live) {
#pragma unroll
        for (int k = 0; k < 17; ++k) grad_init[k * ld + i] = to_store(lam[k]);
        if (boundary) boundary[i] = flag ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// Split adjoint (FP32, RK4, 2 substeps: the production configuration).  At
// config 4 (16,384 envs) one thread per env gives a single warp per SM
// sub-partition, so the reverse sweep is a latency-bound chain of ~3.5k
// dependent-ish instructions per env-step.  Here every env is served by TWO
// warps of one 64-thread block, split along the structure of the rigid-body
// equations (dynamics.py:154-200):
//   T (warp 0): translational part -- p, v and their adjoints; the drag /
//               thrust force in the body frame, rotated into the world frame
//               (v' = g + M(q) F(M(q)^T v) / m), and its VJP in matrix form
//               (M = to_matrix(q), dL/dq through dM/dq);
//   R (warp 1): rotational part -- q, omega, rotors: quaternion kinematics,
//               Euler's equations, rotor lag, clamps, renormalisation, the
//               controller (CTBR / SRT) and the action gradient.
// q and omega never depend on p or v, so R runs the forward recompute of
// step t-1 while T works on step t, and T's backward never waits for R; R
// consumes T's dL/dq contributions (4 floats per RK4 stage) and thrust
// cotangent (1 per substep) one step later.  Exchange: shared memory,
// double-buffered by step parity, one __syncthreads per step.
// Same derivative conventions (clip masks, boundary flag) as dyn_step_vjp.
namespace tr {

constexpr int NS = 2;  // substeps
constexpr int NK = 4;  // RK4 stages

struct Smem {
    float q[2][NS][NK][4][32];    // R -> T: q at each stage argument (stage 1 = substep input)
    float fsm[2][NS][32];         // R -> T: fsum / m of each substep
    float qb[2][NS][NK][4][32];   // T -> R: dL/dq of each stage from the translational equations
    float fbz[2][NS][32];         // T -> R: thrust cotangent of each substep (sum over stages, x 1/m)
    float w[2][NS][NK][3][32];    // R private: omega at each stage argument
    float qraw[2][NS][4][32];     // R private: unnormalised q after each substep
    float rot[2][NS][4][32];      // R private: rotor speeds after the lag (w of dynamics.py:245)
    float rin[2][4][32];          // R private: rotor state entering the step
    float cmd[2][4][32];          // R private: commanded rotor speeds (clamped) + raw
    float craw[2][4][32];
    float om0[2][3][32];          // R private: omega entering the step (controller VJP)
};

__device__ __forceinline__ void qmat(const float *q, float m[3][3]) { q_matrix<float>(q, m); }

// dL/dq of M(q) = q_matrix(q) given A = dL/dM (FP32 form of quatmath.py:75-81)
__device__ __forceinline__ void qmat_vjp(const float *q, const float A[3][3], float *qb) {
    const float w = q[0], x = q[1], y = q[2], z = q[3];
    const float s01 = A[0][1] + A[1][0], s02 = A[0][2] + A[2][0], s12 = A[1][2] + A[2][1];
    const float d10 = A[1][0] - A[0][1], d02 = A[0][2] - A[2][0], d21 = A[2][1] - A[1][2];
    qb[0] = 2.0f * (z * d10 + y * d02 + x * d21);
    qb[1] = 2.0f * (y * s01 + z * s02 + w * d21 - 2.0f * x * (A[1][1] + A[2][2]));
    qb[2] = 2.0f * (x * s01 + z * s12 + w * d02 - 2.0f * y * (A[0][0] + A[2][2]));
    qb[3] = 2.0f * (x * s02 + y * s12 + w * d10 - 2.0f * z * (A[0][0] + A[1][1]));
}

// translational rates at one stage: dv = g + M f(M^T v), f = ndm b|b| + (0,0,fsum/m)
__device__ __forceinline__ void t_rhs(const DynConsts<float> &C, const float *q, const float *v, float fsm, float *dv) {
    float m[3][3];
    qmat(q, m);
    const float bx = m[0][0] * v[0] + m[1][0] * v[1] + m[2][0] * v[2];
    const float by = m[0][1] * v[0] + m[1][1] * v[1] + m[2][1] * v[2];
    const float bz = m[0][2] * v[0] + m[1][2] * v[1] + m[2][2] * v[2];
    const float fx = C.ndm[0] * bx * fabsf(bx), fy = C.ndm[1] * by * fabsf(by), fz = C.ndm[2] * bz * fabsf(bz) + fsm;
    dv[0] = C.g[0] + m[0][0] * fx + m[0][1] * fy + m[0][2] * fz;
    dv[1] = C.g[1] + m[1][0] * fx + m[1][1] * fy + m[1][2] * fz;
    dv[2] = C.g[2] + m[2][0] * fx + m[2][1] * fy + m[2][2] * fz;
}

// VJP of t_rhs for cotangent av (of dv) and kp (of dp = v): adds to vb, qb, returns dL/d(fsum/m)
__device__ __forceinline__ float t_vjp(const DynConsts<float> &C, const float *q, const float *v, float fsm,
                                       const float *av, float *vb, float *qb) {
    float m[3][3];
    qmat(q, m);
    const float bx = m[0][0] * v[0] + m[1][0] * v[1] + m[2][0] * v[2];
    const float by = m[0][1] * v[0] + m[1][1] * v[1] + m[2][1] * v[2];
    const float bz = m[0][2] * v[0] + m[1][2] * v[1] + m[2][2] * v[2];
    const float f[3] = {C.ndm[0] * bx * fabsf(bx), C.ndm[1] * by * fabsf(by), C.ndm[2] * bz * fabsf(bz) + fsm};
    float Fb[3], gb[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) Fb[j] = m[0][j] * av[0] + m[1][j] * av[1] + m[2][j] * av[2];
    gb[0] = Fb[0] * 2.0f * C.ndm[0] * fabsf(bx);
    gb[1] = Fb[1] * 2.0f * C.ndm[1] * fabsf(by);
    gb[2] = Fb[2] * 2.0f * C.ndm[2] * fabsf(bz);
    float A[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        vb[i] += m[i][0] * gb[0] + m[i][1] * gb[1] + m[i][2] * gb[2];
#pragma unroll
        for (int j = 0; j < 3; ++j) A[i][j] = av[i] * f[j] + v[i] * gb[j];
    }
    float g4[4];
    qmat_vjp(q, A, g4);
#pragma unroll
    for (int k = 0; k < 4; ++k) qb[k] += g4[k];
    return Fb[2];
}

// rotational rates (FP32 ode_rhs rows 6..12)
__device__ __forceinline__ void r_rhs(const DynConsts<float> &C, const float *q, const float *o, const float *tqJ,
                                      float *dq, float *dw) {
    dq[0] = 0.5f * (-q[1] * o[0] - q[2] * o[1] - q[3] * o[2]);
    dq[1] = 0.5f * (q[0] * o[0] + q[2] * o[2] - q[3] * o[1]);
    dq[2] = 0.5f * (q[0] * o[1] - q[1] * o[2] + q[3] * o[0]);
    dq[3] = 0.5f * (q[0] * o[2] + q[1] * o[1] - q[2] * o[0]);
    dw[0] = tqJ[0] - C.cJ[0] * (o[1] * o[2]);
    dw[1] = tqJ[1] - C.cJ[1] * (o[2] * o[0]);
    dw[2] = tqJ[2] - C.cJ[2] * (o[0] * o[1]);
}

// VJP of r_rhs: aq (4), aw (3) cotangents -> adds to qb, ob, fb (thrust, 4)
__device__ __forceinline__ void r_vjp(const DynConsts<float> &C, const float *q, const float *o, const float *aq,
                                      const float *aw, float *qb, float *ob, float *fb) {
    const float h0 = 0.5f * aq[0], h1 = 0.5f * aq[1], h2 = 0.5f * aq[2], h3 = 0.5f * aq[3];
    qb[0] += h1 * o[0] + h2 * o[1] + h3 * o[2];
    qb[1] += -h0 * o[0] - h2 * o[2] + h3 * o[1];
    qb[2] += -h0 * o[1] + h1 * o[2] - h3 * o[0];
    qb[3] += -h0 * o[2] - h1 * o[1] + h2 * o[0];
    ob[0] += -h0 * q[1] + h1 * q[0] + h2 * q[3] - h3 * q[2] - aw[1] * C.cJ[1] * o[2] - aw[2] * C.cJ[2] * o[1];
    ob[1] += -h0 * q[2] - h1 * q[3] + h2 * q[0] + h3 * q[1] - aw[0] * C.cJ[0] * o[2] - aw[2] * C.cJ[2] * o[0];
    ob[2] += -h0 * q[3] + h1 * q[2] - h2 * q[1] + h3 * q[0] - aw[0] * C.cJ[0] * o[1] - aw[1] * C.cJ[1] * o[0];
    const float b0 = aw[0] * C.invJ[0], b1 = aw[1] * C.invJ[1], b2 = aw[2] * C.invJ[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) fb[i] += C.arms[i][0] * b0 + C.arms[i][1] * b1 + C.arms[i][2] * b2;
}

// RK4 stage weights of the reverse sweep: kb_k = cy_k * yb_out + cs_k * sb_{k+1}
__device__ __forceinline__ float cy_of(const DynConsts<float> &C, int k) {
    return (k == 0 || k == 3) ? C.sixth_h : 2.0f * C.sixth_h;
}
__device__ __forceinline__ float cs_of(const DynConsts<float> &C, int k) {  // k = 0..2 (stage k+1 feeds stage k)
    return k == 2 ? C.h : C.half_h;
}

}  // namespace tr

template <int KIND>
__global__ void __launch_bounds__(64) k_rollout_bwd_tr(DynConsts<float> C, long long n, long long ld, int T,
                                                       const float *tape, const float *actions, const float *g_traj,
                                                       float *grad_actions, float *grad_init, uint8_t *boundary) {
    using namespace tr;
    __shared__ Smem sm;
    const int lane = threadIdx.x & 31;
    const bool is_r = threadIdx.x >= 32;
    const long long i = (long long)blockIdx.x * 32 + lane;
    const bool live = i < n;
    const long long ii = live ? i : 0;
    const long long block = 17 * ld;

    if (!is_r) {
        // =================== T: p, v ===================
        float lam[6];
        const float *gl = g_traj + (long long)T * block;
#pragma unroll
        for (int k = 0; k < 6; ++k) lam[k] = gl[k * ld + ii];
        // step t's inputs (tape p, v and the loss gradient) are loaded one
        // iteration ahead: at 7 warps per SM nothing else hides their latency
        float pvn[6], gtn[6];
        if (T > 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                pvn[k] = tape[(long long)(T - 1) * block + k * ld + ii];
                gtn[k] = g_traj[(long long)(T - 1) * block + k * ld + ii];
            }
        }
        __syncthreads();  // R's forward of step T-1
        for (int t = T - 1; t >= -1; --t) {
            if (t >= 0) {
                const int bf = t & 1;
                float vs[NS][NK][3];  // v at each stage argument
                float pv[6], gtc[6];
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    pv[k] = pvn[k];
                    gtc[k] = gtn[k];
                }
                if (t >= 1) {
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        pvn[k] = tape[(long long)(t - 1) * block + k * ld + ii];
                        gtn[k] = g_traj[(long long)(t - 1) * block + k * ld + ii];
                    }
                }
                // forward recompute of the translational stages
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const float fsm = sm.fsm[bf][s][lane];
                    float acc[6], y[6], tt[6];
#pragma unroll
                    for (int k = 0; k < 6; ++k) y[k] = tt[k] = pv[k];
#pragma unroll
                    for (int k = 0; k < NK; ++k) {
                        float q[4], d[6];
#pragma unroll
                        for (int c = 0; c < 4; ++c) q[c] = sm.q[bf][s][k][c][lane];
#pragma unroll
                        for (int c = 0; c < 3; ++c) vs[s][k][c] = tt[3 + c];
                        d[0] = tt[3]; d[1] = tt[4]; d[2] = tt[5];
                        t_rhs(C, q, tt + 3, fsm, d + 3);
                        if (k == 0) {
#pragma unroll
                            for (int c = 0; c < 6; ++c) acc[c] = d[c];
                        } else if (k < 3) {
#pragma unroll
                            for (int c = 0; c < 6; ++c) acc[c] = fmaf(2.0f, d[c], acc[c]);
                        } else {
#pragma unroll
                            for (int c = 0; c < 6; ++c) acc[c] = acc[c] + d[c];
                        }
                        const float hk = k == 2 ? C.h : C.half_h;
                        if (k < 3) {
#pragma unroll
                            for (int c = 0; c < 6; ++c) tt[c] = fmaf(hk, d[c], y[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 6; ++c) pv[c] = fmaf(C.sixth_h, acc[c], y[c]);
                }
                // reverse sweep (renormalisation does not touch p, v)
#pragma unroll
                for (int s = NS - 1; s >= 0; --s) {
                    const float fsm = sm.fsm[bf][s][lane];
                    float yb[6], sb[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, fz = 0.f;
#pragma unroll
                    for (int c = 0; c < 6; ++c) yb[c] = lam[c];
#pragma unroll
                    for (int k = NK - 1; k >= 0; --k) {
                        float kb[6];
                        const float cy = cy_of(C, k);
#pragma unroll
                        for (int c = 0; c < 6; ++c) kb[c] = k == NK - 1 ? cy * lam[c] : fmaf(cs_of(C, k), sb[c], cy * lam[c]);
                        float q[4], qb[4] = {0.f, 0.f, 0.f, 0.f}, vb[3] = {0.f, 0.f, 0.f};
#pragma unroll
                        for (int c = 0; c < 4; ++c) q[c] = sm.q[bf][s][k][c][lane];
                        fz += t_vjp(C, q, vs[s][k], fsm, kb + 3, vb, qb);
#pragma unroll
                        for (int c = 0; c < 4; ++c) sm.qb[bf][s][k][c][lane] = qb[c];
                        // sb: d(stage rates)/d(stage state)^T kb -- p: none; v: dp = v, plus vb
                        sb[0] = sb[1] = sb[2] = 0.f;
#pragma unroll
                        for (int c = 0; c < 3; ++c) sb[3 + c] = kb[c] + vb[c];
#pragma unroll
                        for (int c = 3; c < 6; ++c) yb[c] += sb[c];
                    }
                    sm.fbz[bf][s][lane] = fz * C.inv_mass;
#pragma unroll
                    for (int c = 0; c < 6; ++c) lam[c] = yb[c];
                }
#pragma unroll
                for (int k = 0; k < 6; ++k) lam[k] += gtc[k];
            }
            __syncthreads();
        }
        if (live) {
#pragma unroll
            for (int k = 0; k < 6; ++k) grad_init[k * ld + i] = lam[k];
        }
        return;
    }

    // =================== R: q, omega, rotors, controller ===================
    float lam[11];  // 6..16
    bool flag = false;
    {
        const float *gl = g_traj + (long long)T * block;
#pragma unroll
        for (int k = 0; k < 11; ++k) lam[k] = gl[(6 + k) * ld + ii];
    }
    // forward recompute of the rotational stages of step t into buffer t & 1
    // (x, a: step t's tape row and action, loaded by the caller ahead of time)
    auto load_step = [&](int t, float *x, float *a) {
        const float *xs = tape + (long long)t * block;
#pragma unroll
        for (int k = 0; k < 17; ++k) x[k] = xs[k * ld + ii];
        const float *ap = actions + ((long long)t * n + ii) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = ap[k];
    };
    auto forward = [&](int t, float *x, const float *a) {
        const int bf = t & 1;
        float cmd[4];
        command_to_speeds<float, KIND>(C, x, a, cmd);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            sm.craw[bf][k][lane] = cmd[k];
            cmd[k] = p_clip(cmd[k], C.rlo, C.rhi);
            sm.cmd[bf][k][lane] = cmd[k];
            sm.rin[bf][k][lane] = x[13 + k];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.om0[bf][c][lane] = x[10 + c];
        float q[4] = {x[6], x[7], x[8], x[9]}, o[3] = {x[10], x[11], x[12]}, rot[4] = {x[13], x[14], x[15], x[16]};
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            float w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                w[k] = p_clip(cmd[k] + (rot[k] - cmd[k]) * C.alpha, C.rlo, C.rhi);
                sm.rot[bf][s][k][lane] = w[k];
            }
            Wrench<float> W;
            make_wrench(C, w, W);
            sm.fsm[bf][s][lane] = W.fsum_m;
            float aq[4], aw[3], tq[4], tw[3];
#pragma unroll
            for (int c = 0; c < 4; ++c) tq[c] = q[c];
#pragma unroll
            for (int c = 0; c < 3; ++c) tw[c] = o[c];
#pragma unroll
            for (int k = 0; k < NK; ++k) {
#pragma unroll
                for (int c = 0; c < 4; ++c) sm.q[bf][s][k][c][lane] = tq[c];
#pragma unroll
                for (int c = 0; c < 3; ++c) sm.w[bf][s][k][c][lane] = tw[c];
                float dq[4], dw[3];
                r_rhs(C, tq, tw, W.tqJ, dq, dw);
                if (k == 0) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) aq[c] = dq[c];
#pragma unroll
                    for (int c = 0; c < 3; ++c) aw[c] = dw[c];
                } else if (k < 3) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) aq[c] = fmaf(2.0f, dq[c], aq[c]);
#pragma unroll
                    for (int c = 0; c < 3; ++c) aw[c] = fmaf(2.0f, dw[c], aw[c]);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) aq[c] = aq[c] + dq[c];
#pragma unroll
                    for (int c = 0; c < 3; ++c) aw[c] = aw[c] + dw[c];
                }
                if (k < 3) {
                    const float hk = k == 2 ? C.h : C.half_h;
#pragma unroll
                    for (int c = 0; c < 4; ++c) tq[c] = fmaf(hk, dq[c], q[c]);
#pragma unroll
                    for (int c = 0; c < 3; ++c) tw[c] = fmaf(hk, dw[c], o[c]);
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                q[c] = fmaf(C.sixth_h, aq[c], q[c]);
                sm.qraw[bf][s][c][lane] = q[c];
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) o[c] = fmaf(C.sixth_h, aw[c], o[c]);
            q_normalize(q);
#pragma unroll
            for (int k = 0; k < 4; ++k) rot[k] = w[k];
        }
    };
    if (T > 0) {
        float x[17], a[4];
        load_step(T - 1, x, a);
        forward(T - 1, x, a);
    }
    __syncthreads();
    for (int t = T - 1; t >= -1; --t) {
        const int tb = t + 1;  // the step whose reverse sweep R finishes now (T processed it last iteration)
        // this iteration's global inputs, issued before the sweep hides their latency:
        // the next forward's tape row / action, step tb's action and loss gradient
        float xn[17], an[4], atb[4], gtb[11];
        if (t >= 1) load_step(t - 1, xn, an);
        if (tb <= T - 1) {
            const float *ap = actions + ((long long)tb * n + ii) * 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) atb[k] = ap[k];
            const float *gt = g_traj + (long long)tb * block;
#pragma unroll
            for (int k = 0; k < 11; ++k) gtb[k] = gt[(6 + k) * ld + ii];
        }
        if (tb <= T - 1) {
            const int bf = tb & 1;
            float cb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int s = NS - 1; s >= 0; --s) {
                // renormalisation q = q_raw / |q_raw| (gradients.py:130-133)
                float yo[7];
                {
                    float u[4], n2 = 0.f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        u[c] = sm.qraw[bf][s][c][lane];
                        n2 = fmaf(u[c], u[c], n2);
                    }
                    const float inv = rsqrtf(n2);
                    float ul = 0.f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        u[c] *= inv;
                        ul = fmaf(u[c], lam[c], ul);
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) yo[c] = (lam[c] - u[c] * ul) * inv;
#pragma unroll
                    for (int c = 0; c < 3; ++c) yo[4 + c] = lam[4 + c];
                }
                float yb[7], sb[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, fb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 7; ++c) yb[c] = yo[c];
#pragma unroll
                for (int k = NK - 1; k >= 0; --k) {
                    float kb[7];
                    const float cy = cy_of(C, k);
#pragma unroll
                    for (int c = 0; c < 7; ++c) kb[c] = k == NK - 1 ? cy * yo[c] : fmaf(cs_of(C, k), sb[c], cy * yo[c]);
                    float q[4], o[3], qb[4], ob[3] = {0.f, 0.f, 0.f};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        q[c] = sm.q[bf][s][k][c][lane];
                        qb[c] = sm.qb[bf][s][k][c][lane];  // translational share (T)
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) o[c] = sm.w[bf][s][k][c][lane];
                    r_vjp(C, q, o, kb, kb + 4, qb, ob, fb);
#pragma unroll
                    for (int c = 0; c < 4; ++c) sb[c] = qb[c];
#pragma unroll
                    for (int c = 0; c < 3; ++c) sb[4 + c] = ob[c];
#pragma unroll
                    for (int c = 0; c < 7; ++c) yb[c] += sb[c];
                }
                // thrust -> rotor speed of this substep, lag and its clamp (dynamics.py:109-114)
                const float fz = sm.fbz[bf][s][lane];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float w = sm.rot[bf][s][k][lane];
                    const float cmd = sm.cmd[bf][k][lane];
                    const float rin = s == 0 ? sm.rin[bf][k][lane] : sm.rot[bf][0][k][lane];
                    const float raw = cmd + (rin - cmd) * C.alpha;
                    const float lm = clip_mask(raw, C.rlo, C.rhi, flag);
                    const float wb = (fb[k] + fz) * (2.0f * C.k2 * w + C.k1) + lam[7 + k];
                    const float rb = lm * wb;
                    lam[7 + k] = C.alpha * rb;
                    cb[k] = cb[k] + (1.0f - C.alpha) * rb;
                }
#pragma unroll
                for (int c = 0; c < 7; ++c) lam[c] = yb[c];
            }
            // command clamp + controller (control.py:101-158)
            float ga[4];
            {
                float cbm[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) cbm[k] = clip_mask(sm.craw[bf][k][lane], C.rlo, C.rhi, flag) * cb[k];
                const float *a = atb;
                if constexpr (KIND == QB_CMD_ROTOR) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) ga[k] = cbm[k];
                } else if constexpr (KIND == QB_CMD_SRT) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        bool f2 = false;
                        const float m = clip_mask(a[k], C.flo, C.fhi, f2);
                        ga[k] = cbm[k] * m * speed_of_thrust_grad(C, np_clip(a[k], C.flo, C.fhi));
                    }
                } else {
                    float x[17], xb[17];
#pragma unroll
                    for (int k = 0; k < 17; ++k) x[k] = xb[k] = 0.f;
#pragma unroll
                    for (int c = 0; c < 3; ++c) x[10 + c] = sm.om0[bf][c][lane];
                    ctbr_vjp(C, x, a[0], a[1], a[2], a[3], cbm, ga, xb);
#pragma unroll
                    for (int c = 0; c < 3; ++c) lam[4 + c] += xb[10 + c];
                }
            }
            if (live) {
                float *gp = grad_actions + ((long long)tb * n + ii) * 4;
#pragma unroll
                for (int k = 0; k < 4; ++k) gp[k] = ga[k];
            }
#pragma unroll
            for (int k = 0; k < 11; ++k) lam[k] += gtb[k];
        }
        if (t >= 1) forward(t - 1, xn, an);
        __syncthreads();
    }
    if (live) {
#pragma unroll
        for (int k = 0; k < 11; ++k) grad_init[(6 + k) * ld + i] = lam[k];
        if (boundary) boundary[i] = flag ? 1 : 0;
    }
}

// env-sum of the action gradient (shared open-loop parameters, config 4):
// sum[4 t + k] += sum_i grad[t][i][k] in double, one block per step, a fixed
// summation order (strided per-thread sums, then a shared-memory tree), so
// the result is bitwise reproducible run to run -- unlike atomics
template <class S>
__global__ void __launch_bounds__(256) k_env_sum(long long n, const S *grad, double *sum) {
    __shared__ double red[4][256];
    const int t = blockIdx.x;
    const S *g = grad + (long long)t * n * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] += (double)g[4 * i + k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) red[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
#pragma unroll
            for (int k = 0; k < 4; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) sum[4 * t + threadIdx.x] += red[threadIdx.x][0];
}

template <class R>
int dispatch(const qb_params *p, int kind, long long n, long long ld, int T, const void *tape, const void *actions,
             const void *gtraj, void *ga, void *gi, uint8_t *boundary, double *sum, cudaStream_t st) {
    using S = typename storage_of<R>::type;
    DynConsts<R> C = make_consts<R>(*p);
    if (C.substeps > 8) {
        qb::set_error("adjoint supports up to 8 substeps (got %d)", C.substeps);
        return QB_EINVAL;
    }
    const int B = 128;
    dim3 g(qb::env_grid(n, B));
    auto *x = static_cast<const S *>(tape);
    auto *a = static_cast<const S *>(actions);
    auto *gt = static_cast<const S *>(gtraj);
    auto *gA = static_cast<S *>(ga);
    auto *gI = static_cast<S *>(gi);
    // FP32, RK4, 2 substeps (the production setting), a whole horizon: the
    // two-warp split adjoint (one T and one R warp per 32 envs)
    if constexpr (std::is_same<R, float>::value) {
        // the split pays off while the batch leaves the SMs under-subscribed (config 4: 16,384 envs = 3.5
        // warps per SM; 1.46x at 16,384 and 2.1x at 2,048 envs); beyond ~256 envs per SM the one-thread
        // kernel's lower instruction count wins (0.75x at 131,072)
        if (C.substeps == 2 && C.integrator == QB_RK4 && T >= 1 && n <= 256LL * qb::sm_count() &&
            !getenv_flag("QB_ADJOINT_FUSED")) {
            dim3 g2((unsigned)((n + 31) / 32));
#define QB_BWD_TR(K) k_rollout_bwd_tr<K><<<g2, 64, 0, st>>>(C, n, ld, T, x, a, gt, gA, gI, boundary)
            switch (kind) {
                case QB_CMD_ROTOR: QB_BWD_TR(QB_CMD_ROTOR); break;
                case QB_CMD_CTBR: QB_BWD_TR(QB_CMD_CTBR); break;
                case QB_CMD_SRT: QB_BWD_TR(QB_CMD_SRT); break;
                default: qb::set_error("command kind %d is not differentiable", kind); return QB_EINVAL;
            }
#undef QB_BWD_TR
            int rc = qb::check_launch("rollout_backward");
            if (rc || !sum) return rc;
            k_env_sum<S><<<T, 256, 0, st>>>(n, gA, sum);
            return qb::check_launch("action_grad_sum");
        }
    }
    // the default 2 substeps get a compile-time specialisation (FP32 only)
    const bool sub2 = std::is_same<R, float>::value && C.substeps == 2;
#define QB_BWD(K)                                                                                    \
    (sub2 ? (k_rollout_bwd<R, K, 2><<<g, B, 0, st>>>(C, n, ld, T, x, a, gt, gA, gI, boundary), 0) \
          : (k_rollout_bwd<R, K, 0><<<g, B, 0, st>>>(C, n, ld, T, x, a, gt, gA, gI, boundary), 0))
    switch (kind) {
        case QB_CMD_ROTOR: QB_BWD(QB_CMD_ROTOR); break;
        case QB_CMD_CTBR: QB_BWD(QB_CMD_CTBR); break;
        case QB_CMD_SRT: QB_BWD(QB_CMD_SRT); break;
        default: qb::set_error("command kind %d is not differentiable", kind); return QB_EINVAL;
    }
#undef QB_BWD
    int rc = qb::check_launch("rollout_backward");
    if (rc || !sum) return rc;
    k_env_sum<S><<<T < 0 ? 1 : T, 256, 0, st>>>(n, gA, sum);
    return qb::check_launch("action_grad_sum");
}

}  // namespace

namespace qb {
int launch_vjp(const qb_params *p, int kind, int dtype, long long n, long long ld, int T, const void *states_tape,
               const void *actions, const void *g_traj, void *grad_actions, void *grad_init, uint8_t *boundary,
               double *action_grad_sum, cudaStream_t st) {
    if (n == 0) return QB_OK;
    if (dtype == QB_F32)
        return dispatch<float>(p, kind, n, ld, T, states_tape, actions, g_traj, grad_actions, grad_init, boundary,
                               action_grad_sum, st);
    return dispatch<xd>(p, kind, n, ld, T, states_tape, actions, g_traj, grad_actions, grad_init, boundary, action_grad_sum,
                        st);
}
}  // namespace qb
