// qb_k_env.cu -- K1+K3 fused env step and the device-side reset.
//
// One thread per env runs QuadEnvBase.step (env/base.py:156-210) minus the
// observation render, in reference order:
//   lazy auto-reset of envs finished last step  base.py:170-173 (+_spawn_agent :114-147)
//   prev_state <- state                          base.py:175
//   controller -> dynamics (K1)                  base.py:176-179
//   non-finite -> freeze at prev_state           base.py:180-185
//   step_count += 1                              base.py:186
//   proximity / collision / out-of-bounds        base.py:214-224 (kernels.py:120-182)
//   task success + reward                        tasks.py:45-56, 97-111
//   terminated / truncated / needs_respawn       base.py:193-209
// Proximity, flags and rewards are evaluated in exact double (qb_real.cuh xd)
// on the stored state, so collision/done flags are bit-identical to the
// reference evaluated on the same state.  Spawns draw from per-env PCG64
// streams identical to default_rng(seed + i) (qb_rng.cuh).
#include "qb_dynamics.cuh"
#include "qb_geometry.cuh"
#include "qb_checks.cuh"
#include "qb_internal.h"
#include "qb_rng.cuh"

#ifndef QB_ENV_MINB
#define QB_ENV_MINB 6  // measured at 4M envs: 6 blocks (80 regs) beats 5 (96) by 2% and 8 (64, spills) by 19%
#endif

namespace {

template <class R> struct EnvArgs {
    DynConsts<R> C;
    qb_task T;
    qb_env_buffers B;
    DevScene S;
};

__device__ __forceinline__ void sample_dist(const qb_dist &d, Pcg64 &r, double *out) {
    if (d.kind == QB_DIST_FIXED) {
        for (int k = 0; k < 3; ++k) out[k] = d.a[k];
    } else if (d.kind == QB_DIST_UNIFORM) {
        for (int k = 0; k < 3; ++k) out[k] = uniform_draw(r, d.a[k], d.b[k]);
    } else {
        for (int k = 0; k < 3; ++k) out[k] = __dadd_rn(d.a[k], __dmul_rn(d.b[k], normal_draw(r)));
    }
}

// base.py:313-319 -- qz (x) qy (x) qx from intrinsic roll-pitch-yaw
__device__ __forceinline__ void quat_from_rpy(const double *rpy, double *q) {
    double cr = cos(0.5 * rpy[0]), sr = sin(0.5 * rpy[0]);
    double cp = cos(0.5 * rpy[1]), sp = sin(0.5 * rpy[1]);
    double cyw = cos(0.5 * rpy[2]), syw = sin(0.5 * rpy[2]);
    // qy (x) qx with qx = (cr, sr, 0, 0), qy = (cp, 0, sp, 0)
    xd a0 = xd(cp) * xd(cr), a1 = xd(cp) * xd(sr), a2 = xd(sp) * xd(cr), a3 = -(xd(sp) * xd(sr));
    // qz (x) a with qz = (cyw, 0, 0, syw)
    xd w(cyw), z(syw);
    q[0] = (w * a0 - z * a3).v;
    q[1] = (w * a1 - z * a2).v;
    q[2] = (w * a2 + z * a1).v;
    q[3] = (w * a3 + z * a0).v;
}

template <class R> __device__ __forceinline__ void hover_state(const DynConsts<R> &C, R *x) {
#pragma unroll
    for (int k = 0; k < 17; ++k) x[k] = R(0.0);
    x[6] = R(1.0);
#pragma unroll
    for (int k = 13; k < 17; ++k) x[k] = C.hover_speed;
}

// nearest point of one env's query: per thread (BVH walk) or, in the
// warp-per-env kernels, warp-cooperative
template <bool WARP> __device__ __forceinline__ NearestResult nearest_q(const DevScene &S, int scene, const double *q) {
    if constexpr (WARP) {
        return nearest_point_warp(S, scene, q[0], q[1], q[2]);
    } else {
        const int p0 = __ldg(S.prim_offset + scene), p1 = __ldg(S.prim_offset + scene + 1);
        if (p1 - p0 <= NEAREST_SCAN_MAX) return nearest_point_scan(S, p0, p1, q[0], q[1], q[2]);
        return nearest_point(S, scene, q[0], q[1], q[2]);
    }
}

__device__ __forceinline__ xd norm3(xd a, xd b, xd c) { return r_sqrt(a * a + b * b + c * c); }

// base.py:141-146 _swarm_spawn_clear: candidate at least 2 r + 0.1 from every
// lower-index agent (their current positions); warp-parallel over j
template <class R>
__device__ bool swarm_spawn_clear(const EnvArgs<R> &A, long long i, const double *cand) {
    using S = typename storage_of<R>::type;
    const S *st = static_cast<const S *>(A.B.state);
    const xd min_sep = xd(2.0) * xd(A.T.collision_radius) + xd(0.1);
    bool close = false;
    for (long long j = threadIdx.x & 31; j < i; j += 32) {
        const xd d = norm3(xd((double)st[0 * A.B.ld + j]) - xd(cand[0]), xd((double)st[1 * A.B.ld + j]) - xd(cand[1]),
                           xd((double)st[2 * A.B.ld + j]) - xd(cand[2]));
        close |= d < min_sep;
    }
    return !__any_sync(0xffffffffu, close);
}

// base.py:114-147 for env i (shard-local index); returns false on SpawnFailure.
// WARP: all 32 lanes run it on the same env (same draws); `lead` writes.
// SWARM (warp only): also clear of the lower-index agents.
template <class R, bool WARP, bool SWARM = false>
__device__ bool spawn(const EnvArgs<R> &A, long long i, R *x, bool lead) {
    const qb_task &T = A.T;
    const qb_env_buffers &B = A.B;
    const long long gi = B.index_offset + i;
    const int rc = B.reset_count[i];
    const int scene = T.scene_perm[(int)((gi + rc) % T.n_scene_perm)];
    QB_CHECK(scene >= 0 && scene < A.S.n_scenes, "spawn scene index");
    Pcg64 r = pcg_load(B.rng + 4 * i);
    if (WARP) __syncwarp();  // every lane has read the old values
    if (lead) {
        B.agent_scene[i] = scene;
        B.reset_count[i] = rc + 1;
    }
    double pos[3] = {0.0, 0.0, 0.0};
    bool found = false;
    for (int k = 0; k < 1000; ++k) {
        sample_dist(T.spawn[0], r, pos);
        NearestResult nr = nearest_q<WARP>(A.S, scene, pos);
        if (__dsqrt_rn(nr.d2) < T.min_spawn_clearance) continue;
        if constexpr (SWARM) {
            if (!swarm_spawn_clear(A, i, pos)) continue;
        }
        found = true;
        break;
    }
    if (!found && lead) atomicAdd(B.error_count, 1);
    double vel[3], rpy[3], ang[3], q[4];
    sample_dist(T.spawn[1], r, vel);
    sample_dist(T.spawn[2], r, rpy);
    sample_dist(T.spawn[3], r, ang);
    quat_from_rpy(rpy, q);
    for (int k = 0; k < 3; ++k) {
        x[k] = from_dbl<R>(pos[k]);
        x[3 + k] = from_dbl<R>(vel[k]);
        x[10 + k] = from_dbl<R>(ang[k]);
    }
    for (int k = 0; k < 4; ++k) {
        x[6 + k] = from_dbl<R>(q[k]);
        x[13 + k] = A.C.hover_speed;
    }
    if (lead) {
        B.step_count[i] = 0;
        pcg_store(B.rng + 4 * i, r);
    }
    if (WARP) __syncwarp();  // the lead's writes are visible to the lanes that read them next
    return found;
}

struct Proximity {
    double dist, px, py, pz;
    bool collision, oob;
};

// base.py:214-224 in exact double
template <class R, bool WARP> __device__ __forceinline__ Proximity proximity(const EnvArgs<R> &A, int scene, const R *x) {
    double p[3] = {r_dbl(x[0]), r_dbl(x[1]), r_dbl(x[2])};
    NearestResult nr = nearest_q<WARP>(A.S, scene, p);
    Proximity out;
    out.dist = __dsqrt_rn(nr.d2);
    out.px = nr.px;
    out.py = nr.py;
    out.pz = nr.pz;
    out.collision = out.dist < A.T.collision_radius;
    const double *b = A.S.bounds + 6 * scene;
    bool inside = true;
    for (int k = 0; k < 3; ++k) {
        double lo = __dsub_rn(b[k], A.T.bounds_margin), hi = __dadd_rn(b[3 + k], A.T.bounds_margin);
        inside &= (p[k] >= lo) && (p[k] <= hi);
    }
    out.oob = !inside;
    return out;
}

// tasks.py:45-56 (navigation), 97-111 (landing); free: zero reward, no success
__device__ __forceinline__ void task_eval(const qb_task &T, const double *pp, const double *p, const double *v, double nd,
                                          bool collision, bool &success, double &reward) {
    success = false;
    reward = 0.0;
    if (T.task == QB_TASK_NAVIGATION) {
        xd dc = norm3(xd(p[0]) - xd(T.target[0]), xd(p[1]) - xd(T.target[1]), xd(p[2]) - xd(T.target[2]));
        xd dp = norm3(xd(pp[0]) - xd(T.target[0]), xd(pp[1]) - xd(T.target[1]), xd(pp[2]) - xd(T.target[2]));
        success = dc < xd(T.success_radius);
        xd speed2 = xd(v[0]) * xd(v[0]) + xd(v[1]) * xd(v[1]) + xd(v[2]) * xd(v[2]);
        xd prox = np_clip(xd(1.0) - xd(nd) / xd(T.safe_distance), xd(0.0), xd(1.0));
        reward = (xd(T.w_progress) * (dp - dc) - xd(T.w_speed) * speed2 - xd(T.w_obstacle) * prox).v;
    } else if (T.task == QB_TASK_LANDING) {
        xd h = np_max(xd(p[2]) - xd(T.pad_top) - xd(T.collision_radius), xd(0.0));
        xd speed2 = xd(v[0]) * xd(v[0]) + xd(v[1]) * xd(v[1]) + xd(v[2]) * xd(v[2]);
        xd speed = r_sqrt(speed2);
        xd ox = r_abs(xd(p[0]) - xd(T.pad_center[0])), oy = r_abs(xd(p[1]) - xd(T.pad_center[1]));
        bool centered = (ox <= xd(T.pad_half)) && (oy <= xd(T.pad_half));
        success = (h < xd(T.success_height)) && (speed < xd(T.success_speed)) && centered;
        reward = (xd(-T.w_height) * h + xd(T.w_speed_landing) * r_exp(-speed2) -
                  xd(T.w_collision) * xd(collision ? 1.0 : 0.0))
                     .v;
    }
}

template <class R> __device__ __forceinline__ void load_state(const EnvArgs<R> &A, long long i, R *x) {
    using S = typename storage_of<R>::type;
    const S *st = static_cast<const S *>(A.B.state);
#pragma unroll
    for (int k = 0; k < 17; ++k) x[k] = R(st[k * A.B.ld + i]);
}

template <class R> __device__ __forceinline__ void store_planes(void *dst, long long ld, long long i, const R *x) {
    using S = typename storage_of<R>::type;
    S *st = static_cast<S *>(dst);
#pragma unroll
    for (int k = 0; k < 17; ++k) st[k * ld + i] = to_store(x[k]);
}

template <class R>
__device__ __forceinline__ void write_post(const EnvArgs<R> &A, long long i, const Proximity &pr) {
    const qb_env_buffers &B = A.B;
    B.nearest_dist[i] = pr.dist;
    B.nearest_pt[3 * i] = pr.px;
    B.nearest_pt[3 * i + 1] = pr.py;
    B.nearest_pt[3 * i + 2] = pr.pz;
    B.collision[i] = pr.collision;
    B.out_of_bounds[i] = pr.oob;
}

// env index of this thread: one env per thread, or one per warp (WARP: every
// lane computes the env redundantly, lane 0 stores; used for small batches,
// where the warp-cooperative nearest-point query removes the dependent BVH
// walk from the step's critical path)
template <bool WARP> __device__ __forceinline__ long long env_index(bool &lead) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    lead = !WARP || (threadIdx.x & 31) == 0;
    return WARP ? (t >> 5) : t;
}

// mode 0: reset, mode 1: proximity refresh only
template <class R, bool WARP> __global__ void __launch_bounds__(128) k_env_reset(EnvArgs<R> A, uint64_t seed, int mode) {
    bool lead;
    const long long i = env_index<WARP>(lead);
    const qb_env_buffers &B = A.B;
    if (i >= B.n) return;
    R x[17];
    if (mode == 0 || mode == 3) {
        if (lead) {
            pcg_store(B.rng + 4 * i, pcg64_from_seed(seed + (uint64_t)(B.index_offset + i)));
            B.reset_count[i] = 0;
        }
        if (WARP) __syncwarp();
        hover_state(A.C, x);
        if (mode == 0) spawn<R, WARP>(A, i, x, lead);
        if (lead) {
            store_planes(B.state, B.ld, i, x);
            if (B.prev_state) store_planes(B.prev_state, B.ld, i, x);
            B.step_count[i] = 0;
            B.needs_respawn[i] = 0;
            B.terminated[i] = 0;
            B.truncated[i] = 0;
            B.success[i] = 0;
            B.nonfinite[i] = 0;
            B.reward[i] = 0.0f;
        }
    } else {
        load_state(A, i, x);
    }
    if (mode == 3) return;  // swarm reset: spawns and proximity follow
    QB_CHECK(B.agent_scene[i] >= 0 && B.agent_scene[i] < A.S.n_scenes, "env step scene index");
    const Proximity pr = proximity<R, WARP>(A, B.agent_scene[i], x);
    if (lead) write_post(A, i, pr);
}

// Swarm mode (one swarm = all envs of the buffers).  Spawns are sequential
// in agent order (base.py:101-102, 169-172): agent i must clear the agents
// j < i at their current positions, so one warp walks the agents, each spawn
// warp-parallel (nearest point over the scene, clearance over j < i).
template <class R> __global__ void __launch_bounds__(32) k_swarm_spawn(EnvArgs<R> A, int all) {
    const qb_env_buffers &B = A.B;
    const bool lead = threadIdx.x == 0;
    for (long long i = 0; i < B.n; ++i) {
        if (!all && !(A.T.auto_reset && B.needs_respawn[i])) continue;
        R x[17];
        hover_state(A.C, x);
        spawn<R, true, true>(A, i, x, lead);
        if (lead) {
            store_planes(B.state, B.ld, i, x);
            if (all && B.prev_state) store_planes(B.prev_state, B.ld, i, x);
            B.needs_respawn[i] = 0;
        }
        __syncwarp();
    }
}

// base.py:225-232 pairwise collision (d < 2 r), then -- after a step -- the
// task hooks and termination flags on the final collision flags; gap
// crossing (tasks.py:131-165) adds the nearest-agent penalty.
template <class R> __global__ void __launch_bounds__(128) k_swarm_post(EnvArgs<R> A, int after_step) {
    using S = typename storage_of<R>::type;
    const qb_env_buffers &B = A.B;
    const qb_task &T = A.T;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    const S *st = static_cast<const S *>(B.state);
    const double p[3] = {(double)st[i], (double)st[B.ld + i], (double)st[2 * B.ld + i]};
    const xd two_r = xd(2.0) * xd(T.collision_radius);
    bool hit = false;
    double dmin = infinity_d();
    for (long long j = 0; j < B.n; ++j) {
        if (j == i) continue;
        const xd d = norm3(xd(p[0]) - xd((double)st[j]), xd(p[1]) - xd((double)st[B.ld + j]),
                           xd(p[2]) - xd((double)st[2 * B.ld + j]));
        hit |= d < two_r;
        dmin = fmin(dmin, d.v);
    }
    const bool collision = B.collision[i] || hit;
    B.collision[i] = collision;
    if (!after_step) return;
    const S *ps = static_cast<const S *>(B.prev_state);
    const double pp[3] = {(double)ps[i], (double)ps[B.ld + i], (double)ps[2 * B.ld + i]};
    const double v[3] = {(double)st[3 * B.ld + i], (double)st[4 * B.ld + i], (double)st[5 * B.ld + i]};
    bool success;
    double reward;
    if (T.task == QB_TASK_GAP_CROSSING) {
        const double *tg = T.targets + 3 * i;
        const xd dc = norm3(xd(p[0]) - xd(tg[0]), xd(p[1]) - xd(tg[1]), xd(p[2]) - xd(tg[2]));
        const xd dp = norm3(xd(pp[0]) - xd(tg[0]), xd(pp[1]) - xd(tg[1]), xd(pp[2]) - xd(tg[2]));
        success = dc < xd(T.success_radius);
        const xd prox = np_clip(xd(1.0) - xd(B.nearest_dist[i]) / xd(T.safe_distance), xd(0.0), xd(1.0));
        xd rw = xd(T.w_progress) * (dp - dc) - xd(T.w_obstacle) * prox;
        if (B.n > 1) rw = rw - xd(T.w_agent) * py_max(xd(0.0), xd(1.0) - xd(dmin) / xd(T.safe_distance));
        reward = rw.v;
    } else {
        task_eval(T, pp, p, v, B.nearest_dist[i], collision, success, reward);
    }
    const bool terminated = success || collision || B.out_of_bounds[i] || B.nonfinite[i];
    const bool truncated = !terminated && B.step_count[i] >= T.episode_max_steps;
    B.success[i] = success;
    B.reward[i] = (float)reward;
    B.terminated[i] = terminated;
    B.truncated[i] = truncated;
    B.needs_respawn[i] = terminated || truncated;
}

// base.py:245-277, 306-309: other agents as render spheres and swarm states
template <class R>
__global__ void k_swarm_views(EnvArgs<R> A, typename storage_of<R>::type *spheres, int32_t *ids,
                              typename storage_of<R>::type *obs) {
    using S = typename storage_of<R>::type;
    const qb_env_buffers &B = A.B;
    const long long m = B.n - 1;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (m <= 0 || idx >= B.n * m) return;
    const long long i = idx / m, k = idx % m, j = k < i ? k : k + 1;
    const S *st = static_cast<const S *>(B.state);
    if (spheres) {
        for (int c = 0; c < 3; ++c) spheres[idx * 4 + c] = st[c * B.ld + j];
        spheres[idx * 4 + 3] = (S)A.T.collision_radius;
    }
    if (ids) ids[idx] = 60000 + (int32_t)(B.index_offset + j);  // DRONE_ID0 + j (base.py:23)
    if (obs)
        for (int c = 0; c < 13; ++c) obs[idx * 13 + c] = st[c * B.ld + j];
}

// SUB = 2: the default two substeps unrolled at compile time (FP32 batch path).
// PHASE 0: the fused step.  PHASE 1: auto-reset + controller + dynamics only
// (state, step count, non-finite flag and the pre-step state in prev_state);
// PHASE 2: proximity, task and flags on that state -- launched on a second
// stream, concurrently with the observation render, which reads only the state.
template <class R, int KIND, bool WARP, int SUB, int PHASE = 0>
__global__ void __launch_bounds__(128, QB_ENV_MINB) k_env_step(EnvArgs<R> A) {
    using S = typename storage_of<R>::type;
    bool lead;
    const long long i = env_index<WARP>(lead);
    const qb_env_buffers &B = A.B;
    const qb_task &T = A.T;
    if (i >= B.n) return;
    if (PHASE == 2) {
        R x[17];
        load_state(A, i, x);
        const S *ps = static_cast<const S *>(B.prev_state);
        const double pp[3] = {(double)ps[i], (double)ps[B.ld + i], (double)ps[2 * B.ld + i]};
        const bool ok = !B.nonfinite[i];
        const int steps = B.step_count[i];
        Proximity pr = proximity<R, WARP>(A, B.agent_scene[i], x);
        double p[3] = {r_dbl(x[0]), r_dbl(x[1]), r_dbl(x[2])};
        double v[3] = {r_dbl(x[3]), r_dbl(x[4]), r_dbl(x[5])};
        bool success;
        double reward;
        task_eval(T, pp, p, v, pr.dist, pr.collision, success, reward);
        const bool terminated = success || pr.collision || pr.oob || !ok;
        const bool truncated = !terminated && steps >= T.episode_max_steps;
        if (!lead) return;
        write_post(A, i, pr);
        B.success[i] = success;
        B.reward[i] = (float)reward;
        B.terminated[i] = terminated;
        B.truncated[i] = truncated;
        B.needs_respawn[i] = terminated || truncated;
        return;
    }
    // every per-env input is requested before the first store (one memory
    // round trip instead of four dependent ones at 20 warps/SM); a respawn
    // rewrites step count and scene, re-read on that (rare) path
    R x[17];
    load_state(A, i, x);
    const bool respawn = T.auto_reset && B.needs_respawn[i] && !T.swarm;
    R a[4], cmd[4];
    const S *act = static_cast<const S *>(B.action) + 4 * i;
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = R(act[k]);
    int steps = B.step_count[i] + 1;
    int scene = B.agent_scene[i];
    if (respawn) {
        spawn<R, WARP>(A, i, x, lead);
        steps = 1;
        scene = B.agent_scene[i];
    }
    R prev[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) prev[k] = x[k];
    if (B.prev_state && lead) store_planes(B.prev_state, B.ld, i, x);

    command_to_speeds<R, KIND>(A.C, x, a, cmd);
    const bool ok = dyn_step<R, SUB>(A.C, x, cmd) && !(r_isnan(a[0]) || r_isnan(a[1]) || r_isnan(a[2]) || r_isnan(a[3]));
    if (!ok) {
#pragma unroll
        for (int k = 0; k < 17; ++k) x[k] = prev[k];
    }
    if (PHASE == 1) {
        if (!lead) return;
        store_planes(B.state, B.ld, i, x);
        B.step_count[i] = steps;
        B.nonfinite[i] = !ok;
        return;
    }
    Proximity pr = proximity<R, WARP>(A, scene, x);

    double pp[3] = {r_dbl(prev[0]), r_dbl(prev[1]), r_dbl(prev[2])};
    double p[3] = {r_dbl(x[0]), r_dbl(x[1]), r_dbl(x[2])};
    double v[3] = {r_dbl(x[3]), r_dbl(x[4]), r_dbl(x[5])};
    bool success;
    double reward;
    task_eval(T, pp, p, v, pr.dist, pr.collision, success, reward);
    const bool terminated = success || pr.collision || pr.oob || !ok;
    const bool truncated = !terminated && steps >= T.episode_max_steps;
    if (!lead) return;

    store_planes(B.state, B.ld, i, x);
    B.step_count[i] = steps;
    B.nonfinite[i] = !ok;
    write_post(A, i, pr);
    B.success[i] = success;
    B.reward[i] = (float)reward;
    B.terminated[i] = terminated;
    B.truncated[i] = truncated;
    B.needs_respawn[i] = terminated || truncated;
}

__global__ void k_rng_seed(uint64_t seed, long long n, uint64_t *out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pcg_store(out + 4 * i, pcg64_from_seed(seed + (uint64_t)i));
}

__global__ void k_rng_doubles(long long n, uint64_t *rng, int k, double *out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Pcg64 r = pcg_load(rng + 4 * i);
    for (int j = 0; j < k; ++j) out[i * k + j] = pcg64_next_double(r);
    pcg_store(rng + 4 * i, r);
}

template <class R, int K, int PH = 0>
void launch_env_step(const EnvArgs<R> &A, bool warp, bool sub2, dim3 g, int BS, cudaStream_t st) {
    if constexpr (std::is_same<R, float>::value) {
        if (warp)
            sub2 ? k_env_step<R, K, true, 2, PH><<<g, BS, 0, st>>>(A) : k_env_step<R, K, true, 0, PH><<<g, BS, 0, st>>>(A);
        else
            sub2 ? k_env_step<R, K, false, 2, PH><<<g, BS, 0, st>>>(A) : k_env_step<R, K, false, 0, PH><<<g, BS, 0, st>>>(A);
    } else {
        warp ? k_env_step<R, K, true, 0, PH><<<g, BS, 0, st>>>(A) : k_env_step<R, K, false, 0, PH><<<g, BS, 0, st>>>(A);
    }
}

template <class R>
int dispatch_env(int mode, const qb_params *p, int kind, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
                 uint64_t seed, cudaStream_t st) {
    EnvArgs<R> A;
    A.C = make_consts<R>(*p);
    A.T = *task;
    A.B = *b;
    A.S = s->dev;
    const int BS = 128;
    // small batches: one warp per env (warp-cooperative nearest point) while
    // that still fits one wave of the machine
    const bool warp = b->n * 32 <= (long long)qb::sm_count() * 2048;
    dim3 g(qb::env_grid(warp ? b->n * 32 : b->n, BS));
    const bool swarm = task->swarm != 0;
    const dim3 gp(qb::env_grid(b->n, BS));
    auto reset_kernel = [&](int m) {
        if (warp)
            k_env_reset<R, true><<<g, BS, 0, st>>>(A, seed, m);
        else
            k_env_reset<R, false><<<g, BS, 0, st>>>(A, seed, m);
    };
    if (mode == 0 || mode == 2) {
        if (swarm && mode == 0) {  // init streams / flags, then spawn in agent order
            reset_kernel(3);
            k_swarm_spawn<R><<<1, 32, 0, st>>>(A, 1);
        }
        reset_kernel(mode == 0 && !swarm ? 0 : 1);
        if (swarm) k_swarm_post<R><<<gp, BS, 0, st>>>(A, 0);
        return qb::check_launch("env_reset");
    }
    if (mode == 4) {  // phase 2 of a split step (no command kind involved)
        if (warp)
            k_env_step<R, QB_CMD_ROTOR, true, 0, 2><<<g, BS, 0, st>>>(A);
        else
            k_env_step<R, QB_CMD_ROTOR, false, 0, 2><<<g, BS, 0, st>>>(A);
        return qb::check_launch("env_step_post");
    }
    if (swarm && task->auto_reset) k_swarm_spawn<R><<<1, 32, 0, st>>>(A, 0);
    const bool sub2 = std::is_same<R, float>::value && A.C.substeps == 2;
#define QB_ENV(K) (mode == 3 ? launch_env_step<R, K, 1>(A, warp, sub2, g, BS, st) : launch_env_step<R, K, 0>(A, warp, sub2, g, BS, st))
    switch (kind) {
        case QB_CMD_SRT: QB_ENV(QB_CMD_SRT); break;
        case QB_CMD_CTBR: QB_ENV(QB_CMD_CTBR); break;
        case QB_CMD_PS: QB_ENV(QB_CMD_PS); break;
        case QB_CMD_LV: QB_ENV(QB_CMD_LV); break;
        case QB_CMD_ROTOR: QB_ENV(QB_CMD_ROTOR); break;
        default: qb::set_error("unknown command kind %d", kind); return QB_EINVAL;
    }
#undef QB_ENV
    if (swarm) k_swarm_post<R><<<gp, BS, 0, st>>>(A, 1);
    return qb::check_launch("env_step");
}

template <class R> int dispatch_views(const qb_task *task, const qb_env_buffers *b, void *spheres, int32_t *ids, void *obs,
                                      cudaStream_t st) {
    using S = typename storage_of<R>::type;
    EnvArgs<R> A;
    A.T = *task;
    A.B = *b;
    const long long m = b->n - 1;
    if (m <= 0) return QB_OK;
    k_swarm_views<R><<<qb::env_grid(b->n * m, 128), 128, 0, st>>>(A, static_cast<S *>(spheres), ids,
                                                                 static_cast<S *>(obs));
    return qb::check_launch("env_swarm_views");
}

}  // namespace

namespace qb {
// mode 0 reset, 1 step, 2 refresh, 3 / 4 the two phases of a split step
int launch_swarm_views(const qb_task *task, const qb_env_buffers *b, void *spheres, int32_t *ids, void *obs,
                       cudaStream_t st) {
    if (b->n == 0) return QB_OK;
    if (b->dtype == QB_F32) return dispatch_views<float>(task, b, spheres, ids, obs, st);
    return dispatch_views<xd>(task, b, spheres, ids, obs, st);
}

int launch_env(int mode, const qb_params *p, int kind, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
               uint64_t seed, cudaStream_t st) {
    if (b->n == 0) return QB_OK;
    if (b->dtype == QB_F32) return dispatch_env<float>(mode, p, kind, task, s, b, seed, st);
    return dispatch_env<xd>(mode, p, kind, task, s, b, seed, st);
}

int launch_rng_seed(uint64_t seed, long long n, uint64_t *out, cudaStream_t st) {
    if (n == 0) return QB_OK;
    k_rng_seed<<<env_grid(n, 128), 128, 0, st>>>(seed, n, out);
    return check_launch("rng_seed");
}

int launch_rng_doubles(long long n, uint64_t *rng, int k, double *out, cudaStream_t st) {
    if (n == 0) return QB_OK;
    k_rng_doubles<<<env_grid(n, 128), 128, 0, st>>>(n, rng, k, out);
    return check_launch("rng_doubles");
}
}  // namespace qb
