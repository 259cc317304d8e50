// qb_k_dynamics.cu -- K1 forward: fused controller + mixer + motor lag +
// Euler/RK4 + drag + renormalisation, one env per thread.
//
// Memory: the 17 state planes are read and written once per env-step (each
// warp touches one contiguous 128 B line per plane), the action as one
// 16 B vector per env: 152 B/env-step in FP32 (K1 roofline).
// Everything else stays in registers; for a horizon rollout the state never
// leaves registers between steps and only the tape is written.
#include <type_traits>

#include "qb_dynamics.cuh"
#include "qb_internal.h"

#ifndef QB_DYN_MINB
#define QB_DYN_MINB 6  // single-step kernel: min resident 128-thread blocks/SM (register cap, no spills)
#endif

namespace {

template <class S> struct Vec4Load;
template <> struct Vec4Load<float> {
    static __device__ __forceinline__ void load(const float *p, float *o) {
        float4 v = __ldg(reinterpret_cast<const float4 *>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
    static __device__ __forceinline__ void store(float *p, const float *o) {
        *reinterpret_cast<float4 *>(p) = make_float4(o[0], o[1], o[2], o[3]);
    }
};
template <> struct Vec4Load<double> {
    static __device__ __forceinline__ void load(const double *p, double *o) {
        double2 a = __ldg(reinterpret_cast<const double2 *>(p)), b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
    static __device__ __forceinline__ void store(double *p, const double *o) {
        reinterpret_cast<double2 *>(p)[0] = make_double2(o[0], o[1]);
        reinterpret_cast<double2 *>(p)[1] = make_double2(o[2], o[3]);
    }
};

template <class R, class S> __device__ __forceinline__ void load4(const S *p, R *o) {
    S t[4];
    Vec4Load<S>::load(p, t);
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = R(t[k]);
}
template <class R, class S> __device__ __forceinline__ void store4(S *p, const R *o) {
    S t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = to_store(o[k]);
    Vec4Load<S>::store(p, t);
}

// step (T == 0) or horizon rollout (T > 0: state = tape block 0, actions_seq
// (T,n,4), block t+1 written after step t).
template <class R, int KIND, int SUB = 0>
__device__ __forceinline__ void dyn_body(const DynConsts<R> &C, long long n, long long ld,
                                         typename storage_of<R>::type *state,
                                         const typename storage_of<R>::type *action,
                                         typename storage_of<R>::type *rotor_out, uint8_t *nonfinite, int T) {
    using S = typename storage_of<R>::type;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R x[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) x[k] = R(state[k * ld + i]);
    const int steps = T > 0 ? T : 1;
    bool ok_all = true;
    R a_next[4];
    load4<R, S>(action + i * 4, a_next);
    for (int t = 0; t < steps; ++t) {
        R a[4], cmd[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = a_next[k];
        // rollouts: the next step's action is in flight during this step
        if (t + 1 < steps) load4<R, S>(action + ((long long)(t + 1) * n + i) * 4, a_next);
        command_to_speeds<R, KIND>(C, x, a, cmd);
        if (rotor_out && T == 0) store4<R, S>(rotor_out + i * 4, cmd);
        ok_all &= dyn_step<R, SUB>(C, x, cmd);
        // a NaN action propagates to a NaN state in the reference (np.clip keeps NaN)
        ok_all &= !(r_isnan(a[0]) || r_isnan(a[1]) || r_isnan(a[2]) || r_isnan(a[3]));
        S *dst = T > 0 ? state + (long long)(t + 1) * 17 * ld : state;
#pragma unroll
        for (int k = 0; k < 17; ++k) dst[k * ld + i] = to_store(x[k]);
    }
    if (nonfinite) nonfinite[i] = ok_all ? 0 : 1;
}

// one step over many envs: HBM-bound design point -> cap registers for 6 blocks/SM
// (measured: 6 beats 8 (spills) and 5; an env-pair FFMA2 variant needed 158
// registers and lost on occupancy)
// SUB = 2 (the default SimConfig) unrolls the substep loop at compile time.
template <class R, int KIND, int SUB>
__global__ void __launch_bounds__(128, QB_DYN_MINB) k_dyn_step(DynConsts<R> C, long long n, long long ld,
                                                     typename storage_of<R>::type *state,
                                                     const typename storage_of<R>::type *action,
                                                     typename storage_of<R>::type *rotor_out, uint8_t *nonfinite, int T) {
    dyn_body<R, KIND, SUB>(C, n, ld, state, action, rotor_out, nonfinite, T);
}

// horizon rollout: few envs, long per-thread loop -> no register cap (no spills)
template <class R, int KIND, int SUB>
__global__ void __launch_bounds__(128) k_rollout_fwd(DynConsts<R> C, long long n, long long ld,
                                                     typename storage_of<R>::type *state,
                                                     const typename storage_of<R>::type *action,
                                                     typename storage_of<R>::type *rotor_out, uint8_t *nonfinite, int T) {
    dyn_body<R, KIND, SUB>(C, n, ld, state, action, rotor_out, nonfinite, T);
}

template <class R, int KIND>
__global__ void __launch_bounds__(128) k_command(DynConsts<R> C, long long n, long long ld,
                                                 const typename storage_of<R>::type *state,
                                                 const typename storage_of<R>::type *action,
                                                 typename storage_of<R>::type *out) {
    using S = typename storage_of<R>::type;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R x[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) x[k] = R(state[k * ld + i]);
    R a[4], cmd[4];
    load4<R, S>(action + i * 4, a);
    command_to_speeds<R, KIND>(C, x, a, cmd);
    store4<R, S>(out + i * 4, cmd);
}

template <class R, int KIND>
void launch_step(const DynConsts<R> &C, dim3 g, int B, cudaStream_t st, long long n, long long ld,
                 typename storage_of<R>::type *x, const typename storage_of<R>::type *a,
                 typename storage_of<R>::type *o, uint8_t *nonfinite, int T) {
    if (T > 0) {
        if (std::is_same<R, float>::value && C.substeps == 2)
            k_rollout_fwd<R, KIND, 2><<<g, B, 0, st>>>(C, n, ld, x, a, o, nonfinite, T);
        else
            k_rollout_fwd<R, KIND, 0><<<g, B, 0, st>>>(C, n, ld, x, a, o, nonfinite, T);
        return;
    }
    if constexpr (std::is_same<R, float>::value) {
        if (C.substeps == 2) {
            k_dyn_step<R, KIND, 2><<<g, B, 0, st>>>(C, n, ld, x, a, o, nonfinite, T);
            return;
        }
    }
    k_dyn_step<R, KIND, 0><<<g, B, 0, st>>>(C, n, ld, x, a, o, nonfinite, T);
}

template <class R>
int dispatch_step(const qb_params *p, int kind, long long n, long long ld, void *state, const void *action,
                  void *rotor_out, uint8_t *nonfinite, int T, cudaStream_t st) {
    using S = typename storage_of<R>::type;
    DynConsts<R> C = make_consts<R>(*p);
    const int B = 128;
    dim3 g(qb::env_grid(n, B));
    auto *x = static_cast<S *>(state);
    auto *a = static_cast<const S *>(action);
    auto *o = static_cast<S *>(rotor_out);
#define QB_LAUNCH(K) launch_step<R, K>(C, g, B, st, n, ld, x, a, o, nonfinite, T)
    switch (kind) {
        case QB_CMD_SRT: QB_LAUNCH(QB_CMD_SRT); break;
        case QB_CMD_CTBR: QB_LAUNCH(QB_CMD_CTBR); break;
        case QB_CMD_PS: QB_LAUNCH(QB_CMD_PS); break;
        case QB_CMD_LV: QB_LAUNCH(QB_CMD_LV); break;
        case QB_CMD_ROTOR: QB_LAUNCH(QB_CMD_ROTOR); break;
        default: qb::set_error("unknown command kind %d", kind); return QB_EINVAL;
    }
#undef QB_LAUNCH
    return qb::check_launch("dynamics_step");
}

// controller stages (control.py:101-139): 0 mixer (in [F, tau] -> thrusts +
// saturated), 1 LV -> CTBR, 2 PS -> CTBR (out [collective, rates])
template <class R>
__global__ void __launch_bounds__(128) k_control_stage(DynConsts<R> C, int stage, long long n, long long ld,
                                                       const typename storage_of<R>::type *state,
                                                       const typename storage_of<R>::type *in,
                                                       typename storage_of<R>::type *out, uint8_t *flags) {
    using S = typename storage_of<R>::type;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R a[4], o[4];
    load4<R, S>(in + i * 4, a);
    if (stage == 0) {
        bool sat;
        mixer(C, a[0], a + 1, o, &sat);
        if (flags) flags[i] = sat;
    } else {
        R x[17];
#pragma unroll
        for (int k = 0; k < 17; ++k) x[k] = R(state[k * ld + i]);
        if (stage == 1)
            to_ctbr<R, QB_CMD_LV>(C, x, a, o[0], o + 1);
        else
            to_ctbr<R, QB_CMD_PS>(C, x, a, o[0], o + 1);
    }
    store4<R, S>(out + i * 4, o);
}

template <class R>
int dispatch_stage(const qb_params *p, int stage, long long n, long long ld, const void *state, const void *in, void *out,
                   uint8_t *flags, cudaStream_t st) {
    using S = typename storage_of<R>::type;
    k_control_stage<R><<<qb::env_grid(n, 128), 128, 0, st>>>(make_consts<R>(*p), stage, n, ld,
                                                              static_cast<const S *>(state), static_cast<const S *>(in),
                                                              static_cast<S *>(out), flags);
    return qb::check_launch("control_stage");
}

template <class R>
int dispatch_command(const qb_params *p, int kind, long long n, long long ld, const void *state, const void *action,
                     void *out, cudaStream_t st) {
    using S = typename storage_of<R>::type;
    DynConsts<R> C = make_consts<R>(*p);
    const int B = 128;
    dim3 g(qb::env_grid(n, B));
    auto *x = static_cast<const S *>(state);
    auto *a = static_cast<const S *>(action);
    auto *o = static_cast<S *>(out);
    switch (kind) {
        case QB_CMD_SRT: k_command<R, QB_CMD_SRT><<<g, B, 0, st>>>(C, n, ld, x, a, o); break;
        case QB_CMD_CTBR: k_command<R, QB_CMD_CTBR><<<g, B, 0, st>>>(C, n, ld, x, a, o); break;
        case QB_CMD_PS: k_command<R, QB_CMD_PS><<<g, B, 0, st>>>(C, n, ld, x, a, o); break;
        case QB_CMD_LV: k_command<R, QB_CMD_LV><<<g, B, 0, st>>>(C, n, ld, x, a, o); break;
        case QB_CMD_ROTOR: k_command<R, QB_CMD_ROTOR><<<g, B, 0, st>>>(C, n, ld, x, a, o); break;
        default: qb::set_error("unknown command kind %d", kind); return QB_EINVAL;
    }
    return qb::check_launch("command_to_rotor_speeds");
}

}  // namespace

namespace qb {
int launch_dynamics_step(const qb_params *p, int kind, int dtype, long long n, long long ld, void *state,
                         const void *action, void *rotor_out, uint8_t *nonfinite, int T, const void *actions_seq,
                         cudaStream_t st) {
    const void *a = T > 0 ? actions_seq : action;
    if (dtype == QB_F32) return dispatch_step<float>(p, kind, n, ld, state, a, rotor_out, nonfinite, T, st);
    return dispatch_step<xd>(p, kind, n, ld, state, a, rotor_out, nonfinite, T, st);
}

int launch_control_stage(const qb_params *p, int stage, int dtype, long long n, long long ld, const void *state,
                         const void *in, void *out, uint8_t *flags, cudaStream_t st) {
    if (n == 0) return QB_OK;
    if (dtype == QB_F32) return dispatch_stage<float>(p, stage, n, ld, state, in, out, flags, st);
    return dispatch_stage<xd>(p, stage, n, ld, state, in, out, flags, st);
}

int launch_command(const qb_params *p, int kind, int dtype, long long n, long long ld, const void *state,
                   const void *action, void *out, cudaStream_t st) {
    if (dtype == QB_F32) return dispatch_command<float>(p, kind, n, ld, state, action, out, st);
    return dispatch_command<xd>(p, kind, n, ld, state, action, out, st);
}
}  // namespace qb
