// qb_k_adjoint.cu -- K1 adjoint kernels: BPTT over a whole horizon in one
// launch (gradients.rollout_grad, gradients.py:218-237) and the single-step
// VJP.  One env per thread walks t = T-1 .. 0 keeping lambda (17) in
// registers; per step it reads the saved pre-step state (17 planes) and the
// action (16 B), and writes the action gradient (16 B): ~236 B/env-step of
// HBM traffic, plus the optional deterministic env-sum of the action
// gradient (k_env_sum) that feeds the multi-GPU all-reduce of a shared
// open-loop action sequence.
#include <type_traits>

#include "qb_adjoint.cuh"
#include "qb_internal.h"

namespace {

constexpr unsigned FULL = 0xffffffffu;

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
