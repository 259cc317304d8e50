// qb_internal.h -- shared host-side plumbing of libquadb200.so (not public).
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/quadb200.h"
#include "qb_geometry.cuh"

namespace qb {

void set_error(const char *fmt, ...);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// grid for a one-env-per-thread kernel: enough blocks for n, at least a
// couple of waves, never beyond what n needs
inline int env_grid(long long n, int block) {
    long long g = (n + block - 1) / block;
    return (int)(g < 1 ? 1 : (g > 2147483647LL ? 2147483647LL : g));
}

int check_launch(const char *what);

int sm_count();

}  // namespace qb

#define QB_REQUIRE(cond, ...)          \
    do {                               \
        if (!(cond)) {                 \
            qb::set_error(__VA_ARGS__); \
            return QB_EINVAL;          \
        }                              \
    } while (0)

// scene handle (opaque in the public header)
struct qb_scene {
    int device;
    DevScene dev;
    long long n_nodes, n_prims;
    int max_depth;
    std::string err;
    void *allocs[32];
    int max_scene_prims;  // largest scene of the set (selects the culling renderer)
    int n_allocs;
    double *host_bounds;  // [S][6]
};

// kernel launchers implemented in the per-kernel translation units
namespace qb {
int scene_create_device(int n_scenes, const int64_t *prim_offsets, const int64_t *prim_type, const double *prim_data,
                        const int64_t *prim_oid, const double *prim_lo, const double *prim_hi, qb_scene **out,
                        cudaStream_t st);
int launch_dynamics_step(const qb_params *p, int kind, int dtype, long long n, long long ld, void *state,
                         const void *action, void *rotor_out, uint8_t *nonfinite, int T, const void *actions_seq,
                         cudaStream_t st);
int launch_control_stage(const qb_params *p, int stage, int dtype, long long n, long long ld, const void *state,
                         const void *in, void *out, uint8_t *flags, cudaStream_t st);
int launch_command(const qb_params *p, int kind, int dtype, long long n, long long ld, const void *state,
                   const void *action, void *out, cudaStream_t st);
int launch_vjp(const qb_params *p, int kind, int dtype, long long n, long long ld, int T, const void *states_tape,
               const void *actions, const void *g_traj, void *grad_actions, void *grad_init, uint8_t *boundary,
               double *action_grad_sum, cudaStream_t st);
int launch_render(const qb_scene *s, const qb_camera *cam, int dtype, long long n, long long ld, const void *state,
                  const void *origins, const void *rotations, const int32_t *env_scene, void *depth, int32_t *seg,
                  int32_t centroid_id, float *centroid, const void *extra, const int32_t *extra_ids, int n_extra,
                  cudaStream_t st);
int launch_nearest(const qb_scene *s, const int32_t *env_scene, long long n, const double *q, double *pt, double *dist,
                   int32_t *oid, double *dist2, cudaStream_t st);
int launch_raycast(const qb_scene *s, int dtype, const int32_t *env_scene, long long n, const void *o, const void *d,
                   double tmin, double tmax, void *t, int32_t *oid, cudaStream_t st);
int launch_env(int mode, const qb_params *p, int kind, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
               uint64_t seed, cudaStream_t st);
int launch_swarm_views(const qb_task *task, const qb_env_buffers *b, void *spheres, int32_t *ids, void *obs,
                       cudaStream_t st);
int launch_rng_seed(uint64_t seed, long long n, uint64_t *out, cudaStream_t st);
int launch_rng_doubles(long long n, uint64_t *rng, int k, double *out, cudaStream_t st);
int launch_rng_normals(long long n, uint64_t *rng, int k, double *out, cudaStream_t st);
int launch_rng_poissons(long long n, uint64_t *rng, int k, const double *lam, int64_t *out, cudaStream_t st);
int launch_observe(const qb_params *p, const qb_env_buffers *b, int n_sensors, const qb_sensor_obs *sensors,
                   cudaStream_t st);
int launch_io_pack(int dtype, long long n, long long ld, const void *planes, void *rows, int n_packs,
                   const qb_io_copy *packs, cudaStream_t st);
int launch_narrow(long long count, const int32_t *seg, void *out, int bytes, cudaStream_t st);
}  // namespace qb
