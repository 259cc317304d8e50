/*
 * quadb200.h -- C-ABI of libquadb200.so, the sm_100a hot path of the
 * VisFly/quadsim batched simulator.
 *
 * The reference (/root/reference/pkg/src/quadsim) has no FFI of its own: its
 * hot path is entered through Python functions plus one flat-array numba
 * kernel.  Each entry point below replaces one of those call sites; the
 * citation names the reference interface it stands in for.  The Python
 * package paper_2407_14783_b200 binds these with ctypes (INTEGRATION.md shows
 * the binding a maintainer of the reference would add).
 *
 * Conventions
 *   - plain pointers + sizes; all per-step buffers are caller-owned DEVICE
 *     memory, passed with the cudaStream_t (as void*) to enqueue on;
 *   - the library allocates only scene handles (qb_scene_create/destroy) and
 *     never allocates, frees or synchronises inside a per-step call (the one
 *     exception: qb_env_step_io, the host-buffer bindings step, may
 *     synchronise its stream when asked to);
 *   - states are field-major planes: plane k (0..16, dynamics.py:3-8 order
 *     p v q omega rotor) of env i lives at state[k*ld + i];
 *   - every call returns 0 (QB_OK) or a QB_E* status; qb_last_error() gives a
 *     thread-local message.  Per-env failures (non-finite state, spawn
 *     failure) are written to caller buffers, never raised mid-stream;
 *   - dtype: QB_F32 (production) or QB_F64 (exact-double validation build,
 *     bit-identical to the reference wherever the reference evaluates only
 *     + - * / sqrt).
 */
#ifndef QUADB200_H
#define QUADB200_H

#include <stdint.h>

#include "qb_params.h"

#ifdef __cplusplus
extern "C" {
#endif

enum qb_status { QB_OK = 0, QB_EINVAL = 1, QB_ECUDA = 2, QB_ENOMEM = 3, QB_EEMPTY = 4 };
enum qb_dtype { QB_F32 = 0, QB_F64 = 1 };
enum qb_task_kind { QB_TASK_FREE = 0, QB_TASK_NAVIGATION = 1, QB_TASK_LANDING = 2, QB_TASK_GAP_CROSSING = 3 };
enum qb_dist_kind { QB_DIST_FIXED = 0, QB_DIST_UNIFORM = 1, QB_DIST_NORMAL = 2 };

const char *qb_last_error(void);
int qb_version(void);
int qb_device_sm_count(int32_t *out); /* SMs of the current device */

/* ---------------------------------------------------------------- dynamics */

/* control.command_to_rotor_speeds (control.py:242-252) followed by
 * dynamics.step (dynamics.py:231-253) for n envs.  action: (n,4) row-major in
 * the Command.as_array() layout of cmd_kind (qb_cmd_kind; QB_CMD_ROTOR =
 * desired rotor speeds as in gradients.step_jacobian).  rotor_cmd_out (n,4)
 * and nonfinite (n) may be NULL.  tape: when non-NULL the post-step state is
 * also written to tape (same plane layout, stride ld). */
int qb_dynamics_step(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, void *state,
                     const void *action, void *rotor_cmd_out, uint8_t *nonfinite, void *stream);

/* control.command_to_rotor_speeds alone (control.py:242-252): out (n,4). */
int qb_command_to_rotor_speeds(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld,
                               const void *state, const void *action, void *out, void *stream);

/* Controller stages (control.py:101-139): QB_STAGE_MIXER maps in (n,4)
 * [collective force, torque_b] to out (n,4) per-rotor thrusts and flags (n)
 * "saturated" (torque scaled down or collective clamped; may be NULL);
 * QB_STAGE_LV_TO_CTBR / QB_STAGE_PS_TO_CTBR map an LV / PS command (n,4) at
 * the state planes to out (n,4) [collective accel, body rates]. */
enum qb_control_stage { QB_STAGE_MIXER = 0, QB_STAGE_LV_TO_CTBR = 1, QB_STAGE_PS_TO_CTBR = 2 };
int qb_control_stage(const qb_params *p, int32_t stage, int32_t dtype, int64_t n, int64_t ld, const void *state,
                     const void *in, void *out, uint8_t *flags, void *stream);

/* Horizon rollout (gradients.rollout, gradients.py:200-215, batched and
 * tape-only): states_tape is (T+1) blocks of 17 planes (block stride 17*ld);
 * block 0 must hold the initial state.  actions (T, n, 4). */
int qb_rollout_forward(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, int32_t T,
                       void *states_tape, const void *actions, uint8_t *nonfinite, void *stream);

/* Reverse accumulation (gradients.rollout_grad, gradients.py:218-237),
 * matrix-free: per step lambda <- J^T lambda + g[t], grad_a[t] = Ja^T lambda,
 * with J, Ja the exact step Jacobians of step_jacobian (gradients.py:145-197)
 * never formed.  states_tape as written by qb_rollout_forward; g_traj (T+1)
 * blocks of 17 planes (dL/dstate, block stride 17*ld); grad_actions (T,n,4);
 * grad_init 17 planes.  Differentiable action kinds: QB_CMD_ROTOR (the
 * reference's), QB_CMD_CTBR and QB_CMD_SRT (through the controller + mixer;
 * beyond the reference, finite-difference pinned).  boundary (n, nullable):
 * 1 where a clamp sat exactly on a bound (StepJacobian.saturation_boundary).
 * action_grad_sum (T*4 doubles, nullable, accumulated): sum over envs of
 * grad_actions -- the shared-parameter gradient a multi-GPU run all-reduces. */
int qb_rollout_backward(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, int32_t T,
                        const void *states_tape, const void *actions, const void *g_traj, void *grad_actions,
                        void *grad_init, uint8_t *boundary, double *action_grad_sum, void *stream);

/* One-step VJP (the per-step factor of rollout_grad): given state (pre-step
 * planes), action (n,4) and lam_next (17 planes, dL/dnext_state), writes
 * lam_prev (17 planes, J^T lam) and grad_action (n,4, Ja^T lam). */
int qb_dynamics_vjp(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, const void *state,
                    const void *action, const void *lam_next, void *lam_prev, void *grad_action, uint8_t *boundary,
                    void *stream);

/* ------------------------------------------------------------------ scenes */

typedef struct qb_scene qb_scene;

/* Flattened primitive tables of S scenes concatenated (shapes.py:139-212
 * SceneArrays rows; type 0 sphere [c,r], 1 box [c,h,R(9)], 2 triangle
 * [a,b,c]); prim_offsets has S+1 entries.  Builds one binned-SAH BVH per
 * scene on the host and uploads float + double copies to the current
 * device (replaces Scene.arrays / build_bvh, shapes.py:197-212,
 * bvh.py:16-70). */
int qb_scene_create(int32_t n_scenes, const int64_t *prim_offsets, const int64_t *prim_type, const double *prim_data,
                    const int64_t *prim_oid, const double *prim_lo, const double *prim_hi, qb_scene **out);
int qb_scene_destroy(qb_scene *s);

/* The same scene set built on the device (replaces the host
 * flatten + build_bvh of shapes.py:197-212 / bvh.py:16-70 for scenes that
 * change per episode): prim_offsets is HOST (S+1 entries), every primitive
 * array is DEVICE memory on the current device.  The BVH is a linear BVH
 * (Morton order, Karras hierarchy, leaves of <= 4 primitives); renders and
 * queries equal those of a qb_scene_create handle bit for bit (results are
 * traversal-order independent), traversal cost differs.  Stream-ordered;
 * returns after the build has finished. */
int qb_scene_create_device(int32_t n_scenes, const int64_t *prim_offsets, const int64_t *prim_type,
                           const double *prim_data, const int64_t *prim_oid, const double *prim_lo,
                           const double *prim_hi, qb_scene **out, void *stream);

/* bvh.build_bvh (bvh.py:16-70) with this library's binned-SAH split, in the
 * reference's flat layout: node_count > 0 marks a leaf over
 * prim_order[first : first + count], 0 an internal node whose children are
 * first and first + 1; at most 4 primitives per leaf.  Host-only (no GPU).
 * Pass node_lo == NULL to get the node count in *n_nodes first. */
int qb_bvh_build(int64_t n, const double *prim_lo, const double *prim_hi, int64_t *n_nodes, double *node_lo,
                 double *node_hi, int64_t *node_first, int64_t *node_count, int64_t *prim_order);
/* stats: [n_nodes, n_prims, max_depth, n_scenes] */
int qb_scene_stats(const qb_scene *s, int64_t *out4);
/* raw bounds of scene k: lo.xyz hi.xyz (Scene.bounds, shapes.py:214-217) */
int qb_scene_bounds(const qb_scene *s, int32_t k, double *out6);

/* queries.nearest_point (queries.py:28-38 / kernels.py:120-182), exact
 * double, batched: q (n,3) f64 device; pt (n,3), d (n) distance, oid (n). */
int qb_nearest_point(const qb_scene *s, const int32_t *env_scene, int64_t n, const double *q, double *pt, double *dist,
                     int32_t *oid, double *dist2, void *stream); /* dist2: the squared distance (kernels.py returns it), may be NULL */

/* queries.raycast (queries.py:56-71 / kernels.py:389-399), batched; t=-1 on
 * miss.  o, d (n,3) in dtype; t (n) in dtype. */
int qb_raycast(const qb_scene *s, int32_t dtype, const int32_t *env_scene, int64_t n, const void *o, const void *d,
               double tmin, double tmax, void *t, int32_t *oid, void *stream);

/* ------------------------------------------------------------------ camera */

typedef struct qb_camera {
    int32_t width, height;
    double tan_half_h, tan_half_v, max_range; /* CameraModel, sensing.py:32-63 */
    double rotation[9];                       /* camera -> body, row-major */
    double translation[3];                    /* camera origin in body */
    int32_t mode;  /* FP32 kernel: 0 auto, 1 BVH packet traversal, 2 frustum-culling (scenes <= 256 prims) */
    int32_t pad_;
} qb_camera;

/* sensing.render_frames (sensing.py:77-100) -> kernels.render_batch
 * (kernels.py:402-451) for n envs whose poses are read from the state
 * planes.  depth (n,H,W) in dtype, seg (n,H,W) int32 (either may be NULL).
 * env_scene (n) selects the scene of each env (NULL = scene 0).  When
 * centroid_id > 0, centroid (n,2) receives the (col,row) pixel centroid of
 * that id or (-1,-1) (tasks._id_centroid, tasks.py:121-128).  extra (n,K,4)
 * spheres (x, y, z, r) in dtype + extra_ids (n,K): swarm agents
 * (kernels.py:438-445), DEVICE. */
int qb_render(const qb_scene *s, const qb_camera *cam, int32_t dtype, int64_t n, int64_t ld, const void *state,
              const int32_t *env_scene, void *depth, int32_t *seg, int32_t centroid_id, float *centroid,
              const void *extra, const int32_t *extra_ids, int32_t n_extra, void *stream);

/* Same renderer from explicit camera poses (render_batch's own inputs):
 * origins (n,3), rotations (n,3,3) camera->world, in dtype. */
int qb_render_poses(const qb_scene *s, const qb_camera *cam, int32_t dtype, int64_t n, const void *origins,
                    const void *rotations, const int32_t *env_scene, void *depth, int32_t *seg, const void *extra,
                    const int32_t *extra_ids, int32_t n_extra, void *stream);

/* --------------------------------------------------------------------- env */

typedef struct qb_dist {
    int32_t kind; /* qb_dist_kind (config.py:20-46) */
    int32_t pad_;
    double a[3]; /* fixed: value; uniform: low; normal: mean */
    double b[3]; /* uniform: high; normal: sigma */
} qb_dist;

typedef struct qb_task {
    int32_t task; /* qb_task_kind */
    int32_t auto_reset;
    int32_t episode_max_steps;
    int32_t n_scene_perm; /* entries of scene_perm (= number of scenes) */
    const int32_t *scene_perm; /* DEVICE (base.py:97-100) */
    double collision_radius, min_spawn_clearance, bounds_margin;
    qb_dist spawn[4]; /* position, velocity, orientation (rpy), angvel (config.py:57-61) */
    /* navigation (tasks.py:34-62) */
    double target[3];
    double success_radius, w_progress, w_speed, w_obstacle, safe_distance;
    /* landing (tasks.py:78-118) */
    double pad_center[2];
    double pad_half, success_height, success_speed, w_height, w_speed_landing, w_collision, pad_top;
    /* swarm mode (base.py:114-147, 214-232; one swarm = all n envs of the
     * buffers, one scene): spawns clear of lower-index agents by
     * 2 r + 0.1, pairwise collision at 2 r.  Gap crossing (tasks.py:131-174)
     * reuses success_radius / w_progress / w_obstacle / safe_distance. */
    int32_t swarm;
    int32_t pad2_;
    const double *targets; /* DEVICE (n,3) per-agent targets (gap crossing) */
    double w_agent;
} qb_task;

typedef struct qb_env_buffers {
    int64_t n, ld, index_offset; /* envs in this shard, plane stride, global index of env 0 */
    int32_t dtype, pad_;
    void *state;       /* 17 planes */
    void *prev_state;  /* 17 planes or NULL */
    const void *action; /* (n,4) */
    int32_t *step_count, *agent_scene, *reset_count;
    uint8_t *needs_respawn, *terminated, *truncated, *success, *collision, *out_of_bounds, *nonfinite;
    float *reward;
    double *nearest_dist; /* (n) */
    double *nearest_pt;   /* (n,3) */
    uint64_t *rng;        /* (n,4): pcg64 state hi/lo, inc hi/lo */
    int32_t *error_count; /* [1] spawn failures (SpawnFailure) */
} qb_env_buffers;

/* QuadEnvBase.reset(seed) (base.py:93-112) for a shard: per-env generators
 * default_rng(seed + index_offset + i), spawn sampling with clearance
 * rejection, proximity refresh. */
int qb_env_reset(const qb_params *p, const qb_task *task, const qb_scene *s, const qb_env_buffers *b, uint64_t seed,
                 void *stream);

/* QuadEnvBase.step (base.py:156-210) minus observation rendering, fused in
 * one kernel: lazy auto-reset of last step's finished envs, controller,
 * dynamics, non-finite freeze, proximity/collision/out-of-bounds, task
 * success + reward, terminated/truncated. */
int qb_env_step(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
                void *stream);

/* The same step in two launches (base.py:156-210): phase 1 = auto-reset,
 * controller, dynamics (writes state, step count, non-finite flag and the
 * pre-step state to prev_state, which must be non-NULL); phase 2 = proximity,
 * task success + reward, terminated/truncated on that state.  Phase 2 reads
 * nothing the observation render writes and the render reads nothing phase 2
 * writes, so a caller may run them on two streams after phase 1.  Results
 * equal qb_env_step's.  Not for swarm tasks. */
int qb_env_step_phase(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                      const qb_env_buffers *b, int32_t phase, void *stream);

/* Swarm views for the observation (base.py:245-277, 306-309): for every
 * agent i, the other agents j != i (ascending) as render spheres
 * (x, y, z, collision_radius) in dtype (n, n-1, 4) with ids DRONE_ID0 + j
 * (n, n-1), and their 13-component states (n, n-1, 13) in dtype.  Any output
 * may be NULL. */
int qb_env_swarm_views(const qb_task *task, const qb_env_buffers *b, void *spheres, int32_t *sphere_ids,
                       void *swarm_obs, void *stream);

/* Proximity refresh alone (base.py:214-224) on the current state. */
int qb_env_refresh(const qb_task *task, const qb_scene *s, const qb_env_buffers *b, void *stream);

/* ---------------------------------------------------------- observations */

/* Sensor noise models (sensing.py:163-235 NoiseSpec / apply_noise). */
enum qb_noise_kind {
    QB_NOISE_NORMAL = 0,     /* + sigma * N(0,1) */
    QB_NOISE_POISSON = 1,    /* Poisson(max(v,0) * scaling) / scaling */
    QB_NOISE_SALTPEPPER = 2, /* p: corrupt to the image min / max */
    QB_NOISE_SPECKLE = 3,    /* * (1 + sigma * N(0,1)) */
    QB_NOISE_REDWOOD = 4     /* disparity-domain N(0, sigma_disparity) + quantization (depth only) */
};
enum qb_sensor_kind { QB_SENSOR_DEPTH = 0, QB_SENSOR_SEGMENTATION = 1, QB_SENSOR_IMU = 2 };
#define QB_MAX_NOISE 4
#define QB_MAX_SENSORS 8

typedef struct qb_noise {
    int32_t kind; /* qb_noise_kind */
    int32_t pad_;
    double sigma, p, scaling, sigma_disparity, quantization;
} qb_noise;

typedef struct qb_sensor_obs {
    int32_t kind;    /* qb_sensor_kind */
    int32_t n_noise; /* noise models applied in order, <= QB_MAX_NOISE */
    qb_noise noise[QB_MAX_NOISE];
    int32_t width, height; /* camera sensors */
    const void *src; /* DEVICE rendered frames: depth (dtype) or segmentation (int32), (n,H,W); NULL for IMU */
    void *out;       /* DEVICE observation in dtype: (n,H,W), or (n,6) IMU [specific force_b, angvel_b] */
} qb_sensor_obs;

/* The sensor part of QuadEnvBase.get_observation (base.py:287-305) for a
 * shard: for every env, in sensor order, the ideal IMU reading
 * (sensing.py:124-147) and each sensor's noise chain, drawing from the env's
 * generator exactly as numpy's Generator does (standard_normal ziggurat,
 * poisson, random).  Sensors without noise (other than IMU) need no call. */
int qb_env_observe(const qb_params *p, const qb_env_buffers *b, int32_t n_sensors, const qb_sensor_obs *sensors,
                   void *stream);

/* ------------------------------------------------- flat-array host bindings */

/* The SPEC's "bindings" module (reset(handle, seed) /
 * step(handle, actions N x 4) -> (FlatObservation, rewards, terminated,
 * truncated, info), flat arrays across the boundary, freshly owned results):
 * one call runs a whole env step from HOST actions to HOST results.  It is
 * the one entry point that takes host buffers and may synchronise. */

/* One camera render of the step: DEVICE outputs (either may be NULL). */
typedef struct qb_io_view {
    qb_camera cam;
    void *depth;        /* (n,H,W) dtype */
    int32_t *seg;       /* (n,H,W) int32 object ids */
    void *seg_small;    /* optional (n,H,W) narrowed copy of seg for the host: uint8 or uint16 by
                           seg_small_bytes (lossless when every id < 256 / 65536) */
    int32_t centroid_id;
    int32_t seg_small_bytes; /* 1 (also 0) = uint8, 2 = uint16 */
    float *centroid;    /* (n,2) when centroid_id > 0 */
} qb_io_view;

/* One byte copy: a DEVICE -> DEVICE gather (packs) or DEVICE -> HOST copy (copies). */
typedef struct qb_io_copy {
    const void *src;
    void *dst;
    int64_t bytes;
} qb_io_copy;

#define QB_IO_MAX_PACKS 8

typedef struct qb_step_io {
    int32_t step;             /* 1: step the env with host_action first; 0: observe only (after reset) */
    int32_t sync;             /* 1: return after the copies completed (stream synchronised) */
    const void *host_action;  /* (n,4) dtype, HOST: pinned memory is read in place by the step kernel,
                                 pageable memory is first copied into b->action (DEVICE) */
    void *state_rows;         /* (n,13) dtype state observation rows (base.py:234-243), or NULL; DEVICE or
                                 pinned HOST memory (written through its device mapping) */
    int32_t n_views, n_copies;
    const qb_io_view *views;
    const qb_io_copy *copies; /* DEVICE -> HOST, in order */
    int32_t n_sensors, n_packs;
    const qb_sensor_obs *sensors; /* noise / IMU pass (qb_env_observe) after the renders, or NULL */
    const qb_io_copy *packs;  /* <= QB_IO_MAX_PACKS small gathers done by the same kernel as the
                                 state rows, from DEVICE to DEVICE or to pinned HOST memory (then
                                 the small results reach the host without any copy operation) */
} qb_step_io;

/* QuadEnvBase.step (base.py:156-210) + get_observation (:287-310) from host
 * actions to host results: H2D of the actions, the fused env step
 * (qb_env_step), every view's render, the sensor pass, one pack kernel (state
 * rows + gathers), the narrowed segmentation copies, then the D2H copies.  Not
 * for swarm tasks.  Batches of >= 4,096 envs without a sensor pass render in
 * up to 16 camera slices (>= 2,048 cameras each) alternating over two
 * streams; a copy that reads one whole per-camera output of a view
 * (depth, seg, seg_small) is issued per slice on a side stream as soon as the
 * slice is rendered, so the PCIe read-back overlaps the remaining renders
 * (the caller's stream waits for it; results are identical). */
int qb_env_step_io(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                   const qb_env_buffers *b, const qb_step_io *io, void *stream);

/* The same step captured once into a CUDA graph for repeated launches with
 * the same buffers (small batches are launch-latency-bound): every pointer of
 * p / task / b / io is fixed at capture; io->host_action must be PINNED host
 * memory (read in place; its contents change between launches, its address
 * may not); io->sync is ignored (the launch's `sync` decides). */
typedef struct qb_step_graph qb_step_graph;
int qb_env_step_graph_create(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                             const qb_env_buffers *b, const qb_step_io *io, qb_step_graph **out);
int qb_env_step_graph_launch(qb_step_graph *g, int32_t sync, void *stream);
int qb_env_step_graph_destroy(qb_step_graph *g);

/* numpy.random.default_rng(seed + i) seeding for i in [0,n): out (n,4). */
int qb_rng_seed(uint64_t seed, int64_t n, uint64_t *out, void *stream);
/* n draws of next_double from each stream (testing hook): out (n, k). */
int qb_rng_doubles(int64_t n, uint64_t *rng, int32_t k, double *out, void *stream);
/* k standard normals (numpy ziggurat) from each stream: out (n, k). */
int qb_rng_normals(int64_t n, uint64_t *rng, int32_t k, double *out, void *stream);
/* k Poisson draws per stream with means lam (n, k) (DEVICE): out (n, k) int64. */
int qb_rng_poissons(int64_t n, uint64_t *rng, int32_t k, const double *lam, int64_t *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* QUADB200_H */
