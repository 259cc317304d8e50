// qb_abi.cu -- extern "C" surface of libquadb200.so (include/quadb200.h):
// argument validation, thread-local error strings, scene construction
// (host binned-SAH BVH + float/double device copies) and the launch calls.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "qb_internal.h"
#include "qb_scene_pack.cuh"

namespace {
thread_local char g_err[512] = "";
}

namespace qb {

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return QB_ECUDA;
    }
    return QB_OK;
}

int sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

// ------------------------------------------------------------------ BVH
#ifndef QB_BVH_LEAF
#define QB_BVH_LEAF 4  // max primitives per leaf
#endif
#ifndef QB_BVH_BINS
#define QB_BVH_BINS 16  // SAH bins per axis
#endif
// Binned-SAH binary BVH over primitive AABBs.  Children of an internal node
// are adjacent (left = a, right = a + 1) and leaf primitives are contiguous,
// like the reference layout (bvh.py:1-8), but the split is the SAH-optimal
// bin boundary instead of the centroid median: fewer node visits per ray.
struct BNode {
    double lo[3], hi[3];
    int a, b;  // leaf: first, count (>0); internal: left child, -axis (<=0)
};

static double half_area(const double *lo, const double *hi) {
    double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    return dx * dy + dy * dz + dz * dx;
}

static int build_bvh(int n, const double *plo, const double *phi, std::vector<BNode> &nodes, std::vector<int> &order,
                     int &max_depth) {
    const int LEAF = QB_BVH_LEAF, BINS = QB_BVH_BINS, DEPTH_CAP = 56;
    order.resize(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::vector<double> cen(3 * (size_t)n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) cen[3 * i + k] = 0.5 * (plo[3 * i + k] + phi[3 * i + k]);
    nodes.clear();
    nodes.push_back(BNode{});
    struct Item {
        int node, begin, end, depth;
    };
    std::vector<Item> stack{{0, 0, n, 1}};
    max_depth = 1;
    while (!stack.empty()) {
        Item it = stack.back();
        stack.pop_back();
        max_depth = std::max(max_depth, it.depth);
        BNode &nd = nodes[it.node];
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int k = 0; k < 3; ++k) {
            nd.lo[k] = INFINITY;
            nd.hi[k] = -INFINITY;
        }
        for (int i = it.begin; i < it.end; ++i) {
            int p = order[i];
            for (int k = 0; k < 3; ++k) {
                nd.lo[k] = std::min(nd.lo[k], plo[3 * p + k]);
                nd.hi[k] = std::max(nd.hi[k], phi[3 * p + k]);
                clo[k] = std::min(clo[k], cen[3 * p + k]);
                chi[k] = std::max(chi[k], cen[3 * p + k]);
            }
        }
        int count = it.end - it.begin;
        if (count <= LEAF) {
            nd.a = it.begin;
            nd.b = count;
            continue;
        }
        // binned SAH over the three axes
        int best_axis = -1, best_bin = -1;
        double best_cost = INFINITY;
        if (it.depth < DEPTH_CAP) {
            for (int ax = 0; ax < 3; ++ax) {
                double ext = chi[ax] - clo[ax];
                if (!(ext > 0.0)) continue;
                double blo[BINS][3], bhi[BINS][3];
                int bcnt[BINS] = {0};
                for (int b = 0; b < BINS; ++b)
                    for (int k = 0; k < 3; ++k) {
                        blo[b][k] = INFINITY;
                        bhi[b][k] = -INFINITY;
                    }
                double scale = BINS / ext;
                for (int i = it.begin; i < it.end; ++i) {
                    int p = order[i];
                    int b = std::min(BINS - 1, (int)((cen[3 * p + ax] - clo[ax]) * scale));
                    ++bcnt[b];
                    for (int k = 0; k < 3; ++k) {
                        blo[b][k] = std::min(blo[b][k], plo[3 * p + k]);
                        bhi[b][k] = std::max(bhi[b][k], phi[3 * p + k]);
                    }
                }
                // suffix areas
                double rarea[BINS];
                int rcnt[BINS];
                double alo[3] = {INFINITY, INFINITY, INFINITY}, ahi[3] = {-INFINITY, -INFINITY, -INFINITY};
                int c = 0;
                for (int b = BINS - 1; b > 0; --b) {
                    for (int k = 0; k < 3; ++k) {
                        alo[k] = std::min(alo[k], blo[b][k]);
                        ahi[k] = std::max(ahi[k], bhi[b][k]);
                    }
                    c += bcnt[b];
                    rcnt[b] = c;
                    rarea[b] = c ? half_area(alo, ahi) : 0.0;
                }
                for (int k = 0; k < 3; ++k) {
                    alo[k] = INFINITY;
                    ahi[k] = -INFINITY;
                }
                c = 0;
                for (int b = 0; b < BINS - 1; ++b) {  // split between bin b and b+1
                    for (int k = 0; k < 3; ++k) {
                        alo[k] = std::min(alo[k], blo[b][k]);
                        ahi[k] = std::max(ahi[k], bhi[b][k]);
                    }
                    c += bcnt[b];
                    if (c == 0 || rcnt[b + 1] == 0) continue;
                    double cost = half_area(alo, ahi) * c + rarea[b + 1] * rcnt[b + 1];
                    if (cost < best_cost) {
                        best_cost = cost;
                        best_axis = ax;
                        best_bin = b;
                    }
                }
            }
        }
        int mid;
        int axis;
        if (best_axis >= 0) {
            axis = best_axis;
            double scale = BINS / (chi[axis] - clo[axis]);
            double c0 = clo[axis];
            auto pivot = std::partition(order.begin() + it.begin, order.begin() + it.end, [&](int p) {
                return std::min(BINS - 1, (int)((cen[3 * p + axis] - c0) * scale)) <= best_bin;
            });
            mid = (int)(pivot - order.begin());
        } else {  // degenerate centroids (or depth cap): median split on the widest axis
            axis = 0;
            double ext = -1.0;
            for (int k = 0; k < 3; ++k)
                if (chi[k] - clo[k] > ext) {
                    ext = chi[k] - clo[k];
                    axis = k;
                }
            mid = it.begin + count / 2;
            std::nth_element(order.begin() + it.begin, order.begin() + mid, order.begin() + it.end,
                             [&](int x, int y) { return cen[3 * x + axis] < cen[3 * y + axis]; });
        }
        if (mid <= it.begin || mid >= it.end) mid = it.begin + count / 2;
        int left = (int)nodes.size();
        nodes.push_back(BNode{});
        nodes.push_back(BNode{});
        nodes[it.node].a = left;  // (re-index: push_back may have moved nd)
        nodes[it.node].b = -axis;
        stack.push_back({left + 1, mid, it.end, it.depth + 1});
        stack.push_back({left, it.begin, mid, it.depth + 1});
    }
    return max_depth <= 62 ? 0 : -1;
}

using qbpack::cull_record;
using qbpack::f_down;
using qbpack::f_up;
using qbpack::i2f;
using qbpack::pack_prim;

template <class T> static T *dev_upload(qb_scene *s, const std::vector<T> &v) {
    void *p = nullptr;
    size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    s->allocs[s->n_allocs++] = p;
    if (!v.empty() && cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return static_cast<T *>(p);
}

}  // namespace qb

extern "C" {

const char *qb_last_error(void) { return g_err; }

int qb_version(void) { return 1; }

int qb_device_sm_count(int32_t *out) {
    QB_REQUIRE(out, "out is NULL");
    *out = qb::sm_count();
    return QB_OK;
}

int qb_dynamics_step(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, void *state,
                     const void *action, void *rotor_cmd_out, uint8_t *nonfinite, void *stream) {
    QB_REQUIRE(p && state && action, "qb_dynamics_step: NULL argument");
    QB_REQUIRE(n >= 0 && ld >= n, "qb_dynamics_step: bad n=%lld ld=%lld", (long long)n, (long long)ld);
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    return qb::launch_dynamics_step(p, cmd_kind, dtype, n, ld, state, action, rotor_cmd_out, nonfinite, 0, nullptr,
                                    qb::as_stream(stream));
}

int qb_command_to_rotor_speeds(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld,
                               const void *state, const void *action, void *out, void *stream) {
    QB_REQUIRE(p && state && action && out, "qb_command_to_rotor_speeds: NULL argument");
    QB_REQUIRE(n >= 0 && ld >= n, "bad n/ld");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    return qb::launch_command(p, cmd_kind, dtype, n, ld, state, action, out, qb::as_stream(stream));
}

int qb_rollout_forward(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, int32_t T,
                       void *states_tape, const void *actions, uint8_t *nonfinite, void *stream) {
    QB_REQUIRE(p && states_tape && actions, "qb_rollout_forward: NULL argument");
    QB_REQUIRE(n >= 0 && ld >= n && T >= 1, "bad n/ld/T");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    return qb::launch_dynamics_step(p, cmd_kind, dtype, n, ld, states_tape, nullptr, nullptr, nonfinite, T, actions,
                                    qb::as_stream(stream));
}

int qb_rollout_backward(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, int32_t T,
                        const void *states_tape, const void *actions, const void *g_traj, void *grad_actions,
                        void *grad_init, uint8_t *boundary, double *action_grad_sum, void *stream) {
    QB_REQUIRE(p && states_tape && actions && g_traj && grad_actions && grad_init, "qb_rollout_backward: NULL argument");
    QB_REQUIRE(n >= 0 && ld >= n && T >= 1, "bad n/ld/T");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    QB_REQUIRE(cmd_kind == QB_CMD_ROTOR || cmd_kind == QB_CMD_CTBR || cmd_kind == QB_CMD_SRT,
               "command kind %d is not differentiable (rotor, ctbr, srt are)", cmd_kind);
    return qb::launch_vjp(p, cmd_kind, dtype, n, ld, T, states_tape, actions, g_traj, grad_actions, grad_init, boundary,
                          action_grad_sum, qb::as_stream(stream));
}

int qb_dynamics_vjp(const qb_params *p, int32_t cmd_kind, int32_t dtype, int64_t n, int64_t ld, const void *state,
                    const void *action, const void *lam_next, void *lam_prev, void *grad_action, uint8_t *boundary,
                    void *stream) {
    QB_REQUIRE(p && state && action && lam_next && lam_prev && grad_action, "qb_dynamics_vjp: NULL argument");
    QB_REQUIRE(n >= 0 && ld >= n, "bad n/ld");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    QB_REQUIRE(cmd_kind == QB_CMD_ROTOR || cmd_kind == QB_CMD_CTBR || cmd_kind == QB_CMD_SRT,
               "command kind %d is not differentiable (rotor, ctbr, srt are)", cmd_kind);
    // T = -1: one step; g_traj = lam_next, grad_init = lam_prev
    return qb::launch_vjp(p, cmd_kind, dtype, n, ld, -1, state, action, lam_next, grad_action, lam_prev, boundary, nullptr,
                          qb::as_stream(stream));
}

int qb_scene_create(int32_t n_scenes, const int64_t *prim_offsets, const int64_t *prim_type, const double *prim_data,
                    const int64_t *prim_oid, const double *prim_lo, const double *prim_hi, qb_scene **out) {
    QB_REQUIRE(out && prim_offsets && n_scenes >= 1, "qb_scene_create: bad arguments");
    *out = nullptr;
    for (int s = 0; s < n_scenes; ++s)
        if (prim_offsets[s + 1] <= prim_offsets[s]) {
            qb::set_error("scene %d has no primitives", s);
            return QB_EEMPTY;
        }
    const long long P = prim_offsets[n_scenes];
    QB_REQUIRE(prim_type && prim_data && prim_oid && prim_lo && prim_hi, "qb_scene_create: NULL prim arrays");
    QB_REQUIRE(P < (1LL << 30), "too many primitives");
    for (long long i = 0; i < P; ++i) QB_REQUIRE(prim_type[i] >= 0 && prim_type[i] <= 2, "bad prim type at %lld", i);

    std::vector<int> roots(n_scenes);
    std::vector<double> bounds(6 * (size_t)n_scenes);
    std::vector<float4> nodef;
    std::vector<double> noded;
    std::vector<int2> nodei;
    std::vector<float4> primf(4 * (size_t)P);
    std::vector<double> primd(16 * (size_t)P);
    std::vector<int2> meta(P);
    std::vector<float4> primc(4 * (size_t)P);
    std::vector<int> prim_offset(n_scenes + 1);
    for (int s = 0; s <= n_scenes; ++s) prim_offset[s] = (int)prim_offsets[s];
    int max_depth = 0;
    for (int s = 0; s < n_scenes; ++s) {
        const long long off = prim_offsets[s], cnt = prim_offsets[s + 1] - off;
        std::vector<qb::BNode> nodes;
        std::vector<int> order;
        int depth = 0;
        if (qb::build_bvh((int)cnt, prim_lo + 3 * off, prim_hi + 3 * off, nodes, order, depth) != 0) {
            qb::set_error("BVH of scene %d too deep (%d)", s, depth);
            return QB_EINVAL;
        }
        max_depth = std::max(max_depth, depth);
        const int node_off = (int)nodei.size();
        roots[s] = node_off;
        for (int k = 0; k < 3; ++k) {
            double lo = INFINITY, hi = -INFINITY;
            for (long long i = off; i < off + cnt; ++i) {
                lo = std::min(lo, prim_lo[3 * i + k]);
                hi = std::max(hi, prim_hi[3 * i + k]);
            }
            bounds[6 * s + k] = lo;
            bounds[6 * s + 3 + k] = hi;
        }
        for (const qb::BNode &nd : nodes) {
            int a = nd.b > 0 ? (int)(nd.a + off) : nd.a + node_off;
            nodef.push_back(make_float4(qb::f_down(nd.lo[0]), qb::f_down(nd.lo[1]), qb::f_down(nd.lo[2]), qb::i2f(a)));
            nodef.push_back(make_float4(qb::f_up(nd.hi[0]), qb::f_up(nd.hi[1]), qb::f_up(nd.hi[2]), qb::i2f(nd.b)));
            for (int k = 0; k < 3; ++k) noded.push_back(nd.lo[k]);
            for (int k = 0; k < 3; ++k) noded.push_back(nd.hi[k]);
            nodei.push_back(make_int2(a, nd.b));
        }
        for (long long j = 0; j < cnt; ++j) {
            long long src = off + order[j], dst = off + j;
            qb::pack_prim((int)prim_type[src], prim_data + 16 * src, &primf[4 * dst]);
            qb::cull_record((int)prim_type[src], prim_data + 16 * src, &primc[4 * dst]);
            std::memcpy(&primd[16 * dst], prim_data + 16 * src, 16 * sizeof(double));
            QB_REQUIRE(prim_oid[src] > 0 && prim_oid[src] < (1LL << 31), "object ids must be positive int32");
            meta[dst] = make_int2((int)prim_type[src], (int)prim_oid[src]);
        }
    }
    qb_scene *sc = new qb_scene();
    sc->n_allocs = 0;
    cudaGetDevice(&sc->device);
    sc->n_nodes = (long long)nodei.size();
    sc->n_prims = P;
    sc->max_depth = max_depth;
    sc->max_scene_prims = 0;
    for (int s = 0; s < n_scenes; ++s)
        sc->max_scene_prims = std::max(sc->max_scene_prims, (int)(prim_offsets[s + 1] - prim_offsets[s]));
    sc->host_bounds = new double[6 * n_scenes];
    std::memcpy(sc->host_bounds, bounds.data(), sizeof(double) * 6 * n_scenes);
    DevScene &d = sc->dev;
    d.n_scenes = n_scenes;
    d.n_prims = (int)P;
    d.root = qb::dev_upload(sc, roots);
    d.bounds = qb::dev_upload(sc, bounds);
    d.nodef = qb::dev_upload(sc, nodef);
    d.noded = qb::dev_upload(sc, noded);
    d.nodei = qb::dev_upload(sc, nodei);
    d.primf = qb::dev_upload(sc, primf);
    d.primd = qb::dev_upload(sc, primd);
    d.meta = qb::dev_upload(sc, meta);
    d.prim_offset = qb::dev_upload(sc, prim_offset);
    d.primc = qb::dev_upload(sc, primc);
    d.tri_only = std::all_of(meta.begin(), meta.end(), [](const int2 &m) { return m.x == QB_TRIANGLE; });
    if (!d.root || !d.bounds || !d.nodef || !d.noded || !d.nodei || !d.primf || !d.primd || !d.meta || !d.prim_offset ||
        !d.primc) {
        qb::set_error("scene upload failed: %s", cudaGetErrorString(cudaGetLastError()));
        qb_scene_destroy(sc);
        return QB_ENOMEM;
    }
    *out = sc;
    return QB_OK;
}

int qb_scene_create_device(int32_t n_scenes, const int64_t *prim_offsets, const int64_t *prim_type,
                           const double *prim_data, const int64_t *prim_oid, const double *prim_lo,
                           const double *prim_hi, qb_scene **out, void *stream) {
    QB_REQUIRE(out && prim_offsets && n_scenes >= 1, "qb_scene_create_device: bad arguments");
    *out = nullptr;
    QB_REQUIRE(prim_offsets[0] == 0, "qb_scene_create_device: prim_offsets[0] must be 0");
    for (int s = 0; s < n_scenes; ++s)
        if (prim_offsets[s + 1] <= prim_offsets[s]) {
            qb::set_error("scene %d has no primitives", s);
            return QB_EEMPTY;
        }
    QB_REQUIRE(prim_offsets[n_scenes] < (1LL << 30), "too many primitives");
    QB_REQUIRE(prim_type && prim_data && prim_oid && prim_lo && prim_hi, "qb_scene_create_device: NULL prim arrays");
    return qb::scene_create_device(n_scenes, prim_offsets, prim_type, prim_data, prim_oid, prim_lo, prim_hi, out,
                                   qb::as_stream(stream));
}

int qb_bvh_build(int64_t n, const double *prim_lo, const double *prim_hi, int64_t *n_nodes, double *node_lo,
                 double *node_hi, int64_t *node_first, int64_t *node_count, int64_t *prim_order) {
    QB_REQUIRE(n > 0 && n < (1LL << 30) && prim_lo && prim_hi && n_nodes, "qb_bvh_build: bad arguments");
    std::vector<qb::BNode> nodes;
    std::vector<int> order;
    int depth = 0;
    if (qb::build_bvh((int)n, prim_lo, prim_hi, nodes, order, depth) != 0) {
        qb::set_error("qb_bvh_build: tree too deep (%d)", depth);
        return QB_EINVAL;
    }
    if (!node_lo) {
        *n_nodes = (int64_t)nodes.size();
        return QB_OK;
    }
    QB_REQUIRE(*n_nodes == (int64_t)nodes.size() && node_hi && node_first && node_count && prim_order,
               "qb_bvh_build: output arrays sized for %lld nodes", (long long)nodes.size());
    for (size_t i = 0; i < nodes.size(); ++i) {
        for (int k = 0; k < 3; ++k) {
            node_lo[3 * i + k] = nodes[i].lo[k];
            node_hi[3 * i + k] = nodes[i].hi[k];
        }
        node_first[i] = nodes[i].a;
        node_count[i] = nodes[i].b > 0 ? nodes[i].b : 0;
    }
    for (int64_t i = 0; i < n; ++i) prim_order[i] = order[i];
    return QB_OK;
}

int qb_control_stage(const qb_params *p, int32_t stage, int32_t dtype, int64_t n, int64_t ld, const void *state,
                     const void *in, void *out, uint8_t *flags, void *stream) {
    QB_REQUIRE(p && in && out && n >= 0, "qb_control_stage: bad arguments");
    QB_REQUIRE(stage >= QB_STAGE_MIXER && stage <= QB_STAGE_PS_TO_CTBR, "qb_control_stage: unknown stage %d", stage);
    QB_REQUIRE(stage == QB_STAGE_MIXER || (state && ld >= n), "qb_control_stage: state planes needed");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    return qb::launch_control_stage(p, stage, dtype, n, ld, state, in, out, flags, qb::as_stream(stream));
}

int qb_scene_destroy(qb_scene *s) {
    if (!s) return QB_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    for (int i = 0; i < s->n_allocs; ++i) cudaFree(s->allocs[i]);
    cudaSetDevice(prev);
    delete[] s->host_bounds;
    delete s;
    return QB_OK;
}

int qb_scene_stats(const qb_scene *s, int64_t *out4) {
    QB_REQUIRE(s && out4, "NULL argument");
    out4[0] = s->n_nodes;
    out4[1] = s->n_prims;
    out4[2] = s->max_depth;
    out4[3] = s->dev.n_scenes;
    return QB_OK;
}

int qb_scene_bounds(const qb_scene *s, int32_t k, double *out6) {
    QB_REQUIRE(s && out6 && k >= 0 && k < s->dev.n_scenes, "bad arguments");
    std::memcpy(out6, s->host_bounds + 6 * k, 6 * sizeof(double));
    return QB_OK;
}

int qb_nearest_point(const qb_scene *s, const int32_t *env_scene, int64_t n, const double *q, double *pt, double *dist,
                     int32_t *oid, double *dist2, void *stream) {
    QB_REQUIRE(s && q && n >= 0, "qb_nearest_point: bad arguments");
    return qb::launch_nearest(s, env_scene, n, q, pt, dist, oid, dist2, qb::as_stream(stream));
}

int qb_raycast(const qb_scene *s, int32_t dtype, const int32_t *env_scene, int64_t n, const void *o, const void *d,
               double tmin, double tmax, void *t, int32_t *oid, void *stream) {
    QB_REQUIRE(s && o && d && t && n >= 0, "qb_raycast: bad arguments");
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    return qb::launch_raycast(s, dtype, env_scene, n, o, d, tmin, tmax, t, oid, qb::as_stream(stream));
}

static int check_cam(const qb_camera *cam) {
    QB_REQUIRE(cam && cam->width >= 1 && cam->height >= 1, "camera resolution must be >= 1");
    QB_REQUIRE(cam->max_range > 0, "max_range must be > 0");
    return QB_OK;
}

int qb_render(const qb_scene *s, const qb_camera *cam, int32_t dtype, int64_t n, int64_t ld, const void *state,
              const int32_t *env_scene, void *depth, int32_t *seg, int32_t centroid_id, float *centroid,
              const void *extra, const int32_t *extra_ids, int32_t n_extra, void *stream) {
    QB_REQUIRE(s && state && n >= 0 && ld >= n, "qb_render: bad arguments");
    int rc = check_cam(cam);
    if (rc) return rc;
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    QB_REQUIRE(centroid_id <= 0 || centroid, "centroid buffer missing");
    QB_REQUIRE(n_extra == 0 || (extra && extra_ids), "extra spheres missing");
    return qb::launch_render(s, cam, dtype, n, ld, state, nullptr, nullptr, env_scene, depth, seg, centroid_id, centroid,
                             extra, extra_ids, n_extra, qb::as_stream(stream));
}

int qb_render_poses(const qb_scene *s, const qb_camera *cam, int32_t dtype, int64_t n, const void *origins,
                    const void *rotations, const int32_t *env_scene, void *depth, int32_t *seg, const void *extra,
                    const int32_t *extra_ids, int32_t n_extra, void *stream) {
    QB_REQUIRE(s && origins && rotations && n >= 0, "qb_render_poses: bad arguments");
    int rc = check_cam(cam);
    if (rc) return rc;
    QB_REQUIRE(dtype == QB_F32 || dtype == QB_F64, "bad dtype %d", dtype);
    QB_REQUIRE(n_extra == 0 || (extra && extra_ids), "extra spheres missing");
    return qb::launch_render(s, cam, dtype, n, n, nullptr, origins, rotations, env_scene, depth, seg, 0, nullptr, extra,
                             extra_ids, n_extra, qb::as_stream(stream));
}

static int check_env(const qb_task *task, const qb_scene *s, const qb_env_buffers *b) {
    QB_REQUIRE(task && s && b, "env: NULL argument");
    QB_REQUIRE(b->n >= 0 && b->ld >= b->n, "env: bad n/ld");
    QB_REQUIRE(b->dtype == QB_F32 || b->dtype == QB_F64, "env: bad dtype");
    QB_REQUIRE(b->state && b->step_count && b->agent_scene && b->reset_count && b->needs_respawn && b->terminated &&
                   b->truncated && b->success && b->collision && b->out_of_bounds && b->nonfinite && b->reward &&
                   b->nearest_dist && b->nearest_pt && b->rng && b->error_count,
               "env: a required buffer is NULL");
    QB_REQUIRE(task->scene_perm && task->n_scene_perm >= 1, "env: scene_perm missing");
    QB_REQUIRE(task->task >= 0 && task->task <= 3, "env: unknown task %d", task->task);
    QB_REQUIRE(task->task != QB_TASK_GAP_CROSSING || (task->swarm && task->targets),
               "env: gap crossing needs swarm mode and targets");
    QB_REQUIRE(!task->swarm || (b->prev_state && task->n_scene_perm == 1),
               "env: swarm mode needs prev_state tracking and exactly one scene");
    return QB_OK;
}

int qb_env_reset(const qb_params *p, const qb_task *task, const qb_scene *s, const qb_env_buffers *b, uint64_t seed,
                 void *stream) {
    QB_REQUIRE(p, "env: NULL params");
    int rc = check_env(task, s, b);
    if (rc) return rc;
    return qb::launch_env(0, p, 0, task, s, b, seed, qb::as_stream(stream));
}

int qb_env_step(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
                void *stream) {
    QB_REQUIRE(p, "env: NULL params");
    int rc = check_env(task, s, b);
    if (rc) return rc;
    QB_REQUIRE(b->action, "env: NULL action");
    return qb::launch_env(1, p, cmd_kind, task, s, b, 0, qb::as_stream(stream));
}

int qb_env_step_phase(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                      const qb_env_buffers *b, int32_t phase, void *stream) {
    QB_REQUIRE(p, "env: NULL params");
    QB_REQUIRE(phase == 1 || phase == 2, "env: phase must be 1 or 2");
    QB_REQUIRE(b && b->prev_state, "env: a split step needs prev_state");
    int rc = check_env(task, s, b);
    if (rc) return rc;
    QB_REQUIRE(!task->swarm, "env: swarm steps are not split");
    if (phase == 1) QB_REQUIRE(b->action, "env: NULL action");
    return qb::launch_env(phase == 1 ? 3 : 4, p, cmd_kind, task, s, b, 0, qb::as_stream(stream));
}

int qb_env_refresh(const qb_task *task, const qb_scene *s, const qb_env_buffers *b, void *stream) {
    int rc = check_env(task, s, b);
    if (rc) return rc;
    qb_params dummy;
    std::memset(&dummy, 0, sizeof(dummy));
    dummy.substeps = 1;
    dummy.mass = 1.0;
    for (int k = 0; k < 3; ++k) dummy.inertia[k] = 1.0;
    dummy.thrust_coeffs[0] = 1.0;
    return qb::launch_env(2, &dummy, 0, task, s, b, 0, qb::as_stream(stream));
}

int qb_env_swarm_views(const qb_task *task, const qb_env_buffers *b, void *spheres, int32_t *sphere_ids,
                       void *swarm_obs, void *stream) {
    QB_REQUIRE(task && b && b->state, "qb_env_swarm_views: NULL argument");
    QB_REQUIRE(b->dtype == QB_F32 || b->dtype == QB_F64, "qb_env_swarm_views: bad dtype %d", b->dtype);
    return qb::launch_swarm_views(task, b, spheres, sphere_ids, swarm_obs, qb::as_stream(stream));
}

int qb_env_observe(const qb_params *p, const qb_env_buffers *b, int32_t n_sensors, const qb_sensor_obs *sensors,
                   void *stream) {
    QB_REQUIRE(p && b && (sensors || n_sensors == 0), "qb_env_observe: NULL argument");
    QB_REQUIRE(b->n >= 0 && b->ld >= b->n && b->state && b->rng, "qb_env_observe: bad env buffers");
    QB_REQUIRE(b->dtype == QB_F32 || b->dtype == QB_F64, "qb_env_observe: bad dtype %d", b->dtype);
    return qb::launch_observe(p, b, n_sensors, sensors, qb::as_stream(stream));
}

static int check_step_io(const qb_params *p, const qb_task *task, const qb_scene *s, const qb_env_buffers *b,
                         const qb_step_io *io) {
    QB_REQUIRE(p && io, "qb_env_step_io: NULL argument");
    int rc = check_env(task, s, b);
    if (rc) return rc;
    QB_REQUIRE(!task->swarm, "qb_env_step_io: swarm tasks are not supported by the flat bindings");
    QB_REQUIRE(io->n_views >= 0 && (io->views || io->n_views == 0), "qb_env_step_io: bad views");
    QB_REQUIRE(io->n_copies >= 0 && (io->copies || io->n_copies == 0), "qb_env_step_io: bad copies");
    QB_REQUIRE(io->n_sensors >= 0 && (io->sensors || io->n_sensors == 0), "qb_env_step_io: bad sensors");
    for (int v = 0; v < io->n_views; ++v) {
        rc = check_cam(&io->views[v].cam);
        if (rc) return rc;
        QB_REQUIRE(io->views[v].centroid_id <= 0 || io->views[v].centroid, "qb_env_step_io: centroid buffer missing");
        QB_REQUIRE(!io->views[v].seg_small || io->views[v].seg, "qb_env_step_io: seg_small needs seg");
        QB_REQUIRE(io->views[v].seg_small_bytes >= 0 && io->views[v].seg_small_bytes <= 2,
                   "qb_env_step_io: seg_small_bytes must be 1 or 2");
    }
    for (int c = 0; c < io->n_copies; ++c)
        QB_REQUIRE(io->copies[c].bytes >= 0 && (io->copies[c].bytes == 0 || (io->copies[c].src && io->copies[c].dst)),
                   "qb_env_step_io: bad copy %d", c);
    QB_REQUIRE(io->n_packs >= 0 && io->n_packs <= QB_IO_MAX_PACKS && (io->packs || io->n_packs == 0),
               "qb_env_step_io: bad packs (max %d)", QB_IO_MAX_PACKS);
    for (int c = 0; c < io->n_packs; ++c)
        QB_REQUIRE(io->packs[c].bytes >= 0 && (io->packs[c].bytes == 0 || (io->packs[c].src && io->packs[c].dst)),
                   "qb_env_step_io: bad pack %d", c);
    QB_REQUIRE(!io->step || (io->host_action && b->action),
               "qb_env_step_io: host_action and the device action buffer are required");
    return QB_OK;
}

// Large batches overlap the frames' read-back with the renders: the cameras
// are rendered in io_slices() slices on the caller's stream and each slice's
// D2H copies run on a side stream as soon as the slice is done, so PCIe (the
// bound for a host-side consumer: ~56 GB/s against the ~500 GB/s of frames
// the renderer produces) starts after the first slice instead of after the
// whole batch.  Slices alternate between the caller's stream and a second
// render stream so one slice's last wave (its slowest cameras) runs beside
// the next slice's first.  Frames are per camera, so a slice's output is
// bit-identical.
namespace {
constexpr int IO_CHUNKS_MAX = 32;
#ifndef QB_IO_RSTREAMS
#define QB_IO_RSTREAMS 2
#endif
constexpr int IO_RSTREAMS = QB_IO_RSTREAMS;  // render streams, the caller's included
constexpr long long IO_CHUNK_MIN = 2048;  // cameras per slice at least
constexpr int IO_MAX_DEV = 64;
struct IoSide {
    cudaStream_t st = nullptr;   // the D2H copies
    cudaStream_t rs[IO_RSTREAMS - 1] = {};  // renders of slices j % IO_RSTREAMS != 0 (a slice's tail overlaps the next slices' start)
    cudaEvent_t ev[IO_CHUNKS_MAX] = {}, ev_step = nullptr, ev_rs[IO_RSTREAMS - 1] = {}, ev_done = nullptr;
};
// slices per step at most: 16 (QB_IO_SLICES overrides for experiments; 1 = no overlap)
int io_slices() {
    static const int v = [] {
        const char *e = std::getenv("QB_IO_SLICES");
        const int k = e ? std::atoi(e) : 16;
        return k < 1 ? 1 : (k > IO_CHUNKS_MAX ? IO_CHUNKS_MAX : k);
    }();
    return v;
}
std::mutex g_io_mu;  // guards g_io_side and orders the event reuse of concurrent callers
IoSide g_io_side[IO_MAX_DEV];

int small_bytes(const qb_io_view &vw) { return vw.seg_small_bytes == 2 ? 2 : 1; }

// bytes per camera of copy cp when it reads one whole per-camera output of a view, else 0
long long per_camera_bytes(const qb_io_copy &cp, const qb_step_io *io, long long n, size_t es) {
    for (int v = 0; v < io->n_views; ++v) {
        const qb_io_view &vw = io->views[v];
        const long long hw = (long long)vw.cam.width * vw.cam.height;
        const long long cands[3][2] = {{(long long)(uintptr_t)vw.depth, hw * (long long)es},
                                       {(long long)(uintptr_t)vw.seg_small, hw * small_bytes(vw)},
                                       {(long long)(uintptr_t)vw.seg, hw * 4}};
        for (auto &c : cands)
            if (c[0] && (long long)(uintptr_t)cp.src == c[0] && cp.bytes == n * c[1]) return c[1];
    }
    return 0;
}
}  // namespace

static int io_fail(const char *what, cudaError_t e) {
    qb::set_error("qb_env_step_io: %s: %s", what, cudaGetErrorString(e));
    return QB_ECUDA;
}

// renders (+ uint8 narrowing) of cameras [c0, c1) of every view
static int io_render_slice(const qb_scene *s, const qb_env_buffers *b, const qb_step_io *io, long long c0, long long c1,
                           cudaStream_t st) {
    const size_t es = b->dtype == QB_F32 ? 4 : 8;
    for (int v = 0; v < io->n_views; ++v) {
        const qb_io_view &vw = io->views[v];
        const long long hw = (long long)vw.cam.width * vw.cam.height;
        int rc = qb::launch_render(
            s, &vw.cam, b->dtype, c1 - c0, b->ld, static_cast<const char *>(b->state) + c0 * es, nullptr, nullptr,
            b->agent_scene ? b->agent_scene + c0 : nullptr, vw.depth ? static_cast<char *>(vw.depth) + c0 * hw * es : nullptr,
            vw.seg ? vw.seg + c0 * hw : nullptr, vw.centroid_id, vw.centroid ? vw.centroid + 2 * c0 : nullptr, nullptr,
            nullptr, 0, st);
        if (rc) return rc;
        if (vw.seg_small) {
            rc = qb::launch_narrow((c1 - c0) * hw, vw.seg + c0 * hw,
                                   static_cast<char *>(vw.seg_small) + c0 * hw * small_bytes(vw), small_bytes(vw), st);
            if (rc) return rc;
        }
    }
    return QB_OK;
}

// the step's work, enqueued on st (no synchronisation)
static int step_io_enqueue(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                           const qb_env_buffers *b, const qb_step_io *io, cudaStream_t st) {
    int rc = QB_OK;
    const size_t es = b->dtype == QB_F32 ? 4 : 8;
    if (io->step) {
        // pinned (page-locked) host actions are read by the step kernel itself
        // through their device mapping (one 16 B load per env over PCIe) instead
        // of a separate H2D copy; pageable ones are copied into b->action
        qb_env_buffers bb = *b;
        cudaPointerAttributes attr;
        if (cudaPointerGetAttributes(&attr, io->host_action) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
            attr.devicePointer) {
            bb.action = attr.devicePointer;
        } else {
            cudaGetLastError();  // (an unregistered pointer is not an error here)
            cudaError_t e = cudaMemcpyAsync(const_cast<void *>(b->action), io->host_action, (size_t)b->n * 4 * es,
                                            cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) {
                qb::set_error("qb_env_step_io: action copy: %s", cudaGetErrorString(e));
                return QB_ECUDA;
            }
        }
        rc = qb::launch_env(1, p, cmd_kind, task, s, &bb, 0, st);
        if (rc) return rc;
    }
    // the pipelined read-back (above): no sensor pass (it reads the whole
    // frames), not under stream capture (the graph path is for small batches)
    const int nsl = (int)std::min<long long>(io_slices(), b->n / IO_CHUNK_MIN);
    bool slices = nsl > 1 && io->n_views > 0 && io->n_sensors == 0;
    if (slices) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) slices = false;
        cudaGetLastError();
    }
    bool any_sliced = false;
    for (int c = 0; slices && c < io->n_copies; ++c) any_sliced |= per_camera_bytes(io->copies[c], io, b->n, es) > 0;
    if (slices && any_sliced) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess || dev < 0 || dev >= IO_MAX_DEV) return io_fail("device", e);
        std::lock_guard<std::mutex> lk(g_io_mu);
        IoSide &sd = g_io_side[dev];
        if (!sd.st) {
            e = cudaStreamCreateWithFlags(&sd.st, cudaStreamNonBlocking);
            for (int k = 0; e == cudaSuccess && k < IO_RSTREAMS - 1; ++k) {
                e = cudaStreamCreateWithFlags(&sd.rs[k], cudaStreamNonBlocking);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sd.ev_rs[k], cudaEventDisableTiming);
            }
            for (int k = 0; e == cudaSuccess && k < IO_CHUNKS_MAX; ++k)
                e = cudaEventCreateWithFlags(&sd.ev[k], cudaEventDisableTiming);
            for (cudaEvent_t *x : {&sd.ev_step, &sd.ev_done})
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(x, cudaEventDisableTiming);
            if (e != cudaSuccess) return io_fail("side streams", e);
        }
        // the second render stream starts after the env step
        if ((e = cudaEventRecord(sd.ev_step, st)) != cudaSuccess) return io_fail("step event", e);
        for (int k = 0; k < IO_RSTREAMS - 1; ++k)
            if ((e = cudaStreamWaitEvent(sd.rs[k], sd.ev_step, 0)) != cudaSuccess) return io_fail("step event", e);
        for (int j = 0; j < nsl; ++j) {
            const long long c0 = b->n * j / nsl, c1 = b->n * (j + 1) / nsl;
            cudaStream_t r = j % IO_RSTREAMS ? sd.rs[j % IO_RSTREAMS - 1] : st;
            rc = io_render_slice(s, b, io, c0, c1, r);
            if (rc) return rc;
            if ((e = cudaEventRecord(sd.ev[j], r)) != cudaSuccess || (e = cudaStreamWaitEvent(sd.st, sd.ev[j], 0)) != cudaSuccess)
                return io_fail("slice event", e);
            for (int c = 0; c < io->n_copies; ++c) {
                const qb_io_copy &cp = io->copies[c];
                const long long pc = per_camera_bytes(cp, io, b->n, es);
                if (!pc) continue;
                e = cudaMemcpyAsync(static_cast<char *>(cp.dst) + c0 * pc, static_cast<const char *>(cp.src) + c0 * pc,
                                    (size_t)((c1 - c0) * pc), cudaMemcpyDeviceToHost, sd.st);
                if (e != cudaSuccess) return io_fail("result copy", e);
            }
        }
        // every render done before the packs and the other copies (they may read a
        // view's outputs, e.g. the landing centroids), then the side copies
        for (int k = 0; k < IO_RSTREAMS - 1; ++k)
            if ((e = cudaEventRecord(sd.ev_rs[k], sd.rs[k])) != cudaSuccess ||
                (e = cudaStreamWaitEvent(st, sd.ev_rs[k], 0)) != cudaSuccess)
                return io_fail("join", e);
        if (io->state_rows || io->n_packs) {
            rc = qb::launch_io_pack(b->dtype, b->n, b->ld, b->state, io->state_rows, io->n_packs, io->packs, st);
            if (rc) return rc;
        }
        for (int c = 0; c < io->n_copies; ++c) {
            const qb_io_copy &cp = io->copies[c];
            if (!cp.bytes || per_camera_bytes(cp, io, b->n, es)) continue;
            e = cudaMemcpyAsync(cp.dst, cp.src, (size_t)cp.bytes, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return io_fail("result copy", e);
        }
        if ((e = cudaEventRecord(sd.ev_done, sd.st)) != cudaSuccess || (e = cudaStreamWaitEvent(st, sd.ev_done, 0)) != cudaSuccess)
            return io_fail("join", e);
        return QB_OK;
    }
    for (int v = 0; v < io->n_views; ++v) {
        const qb_io_view &vw = io->views[v];
        rc = qb::launch_render(s, &vw.cam, b->dtype, b->n, b->ld, b->state, nullptr, nullptr, b->agent_scene, vw.depth,
                               vw.seg, vw.centroid_id, vw.centroid, nullptr, nullptr, 0, st);
        if (rc) return rc;
    }
    if (io->n_sensors) {
        rc = qb::launch_observe(p, b, io->n_sensors, io->sensors, st);
        if (rc) return rc;
    }
    if (io->state_rows || io->n_packs) {
        rc = qb::launch_io_pack(b->dtype, b->n, b->ld, b->state, io->state_rows, io->n_packs, io->packs, st);
        if (rc) return rc;
    }
    for (int v = 0; v < io->n_views; ++v) {
        const qb_io_view &vw = io->views[v];
        if (!vw.seg_small) continue;
        rc = qb::launch_narrow((long long)b->n * vw.cam.width * vw.cam.height, vw.seg, vw.seg_small, small_bytes(vw), st);
        if (rc) return rc;
    }
    for (int c = 0; c < io->n_copies; ++c) {
        const qb_io_copy &cp = io->copies[c];
        if (!cp.bytes) continue;
        cudaError_t e = cudaMemcpyAsync(cp.dst, cp.src, (size_t)cp.bytes, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) {
            qb::set_error("qb_env_step_io: result copy %d: %s", c, cudaGetErrorString(e));
            return QB_ECUDA;
        }
    }
    return QB_OK;
}

int qb_env_step_io(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                   const qb_env_buffers *b, const qb_step_io *io, void *stream) {
    int rc = check_step_io(p, task, s, b, io);
    if (rc) return rc;
    cudaStream_t st = qb::as_stream(stream);
    rc = step_io_enqueue(p, cmd_kind, task, s, b, io, st);
    if (rc) return rc;
    if (io->sync) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            qb::set_error("qb_env_step_io: %s", cudaGetErrorString(e));
            return QB_ECUDA;
        }
    }
    return QB_OK;
}

struct qb_step_graph {
    cudaGraphExec_t exec;
};

int qb_env_step_graph_create(const qb_params *p, int32_t cmd_kind, const qb_task *task, const qb_scene *s,
                             const qb_env_buffers *b, const qb_step_io *io, qb_step_graph **out) {
    QB_REQUIRE(out, "qb_env_step_graph_create: NULL out");
    *out = nullptr;
    int rc = check_step_io(p, task, s, b, io);
    if (rc) return rc;
    if (io->step) {  // the graph reads the actions in place: a fixed pinned staging buffer
        cudaPointerAttributes attr;
        const bool pinned = cudaPointerGetAttributes(&attr, io->host_action) == cudaSuccess &&
                            attr.type == cudaMemoryTypeHost && attr.devicePointer;
        cudaGetLastError();
        QB_REQUIRE(pinned, "qb_env_step_graph_create: host_action must be pinned host memory");
    }
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
        qb::set_error("qb_env_step_graph_create: %s", cudaGetErrorString(cudaGetLastError()));
        return QB_ECUDA;
    }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
        rc = step_io_enqueue(p, cmd_kind, task, s, b, io, cs);
        e = cudaStreamEndCapture(cs, &g);
        if (rc == QB_OK && e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
    }
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    if (rc) return rc;
    if (e != cudaSuccess) {
        qb::set_error("qb_env_step_graph_create: %s", cudaGetErrorString(e));
        return QB_ECUDA;
    }
    *out = new qb_step_graph{exec};
    return QB_OK;
}

int qb_env_step_graph_launch(qb_step_graph *g, int32_t sync, void *stream) {
    QB_REQUIRE(g, "qb_env_step_graph_launch: NULL graph");
    cudaStream_t st = qb::as_stream(stream);
    cudaError_t e = cudaGraphLaunch(g->exec, st);
    if (e == cudaSuccess && sync) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        qb::set_error("qb_env_step_graph_launch: %s", cudaGetErrorString(e));
        return QB_ECUDA;
    }
    return QB_OK;
}

int qb_env_step_graph_destroy(qb_step_graph *g) {
    if (!g) return QB_OK;
    cudaGraphExecDestroy(g->exec);
    delete g;
    return QB_OK;
}

int qb_rng_seed(uint64_t seed, int64_t n, uint64_t *out, void *stream) {
    QB_REQUIRE(out && n >= 0, "qb_rng_seed: bad arguments");
    return qb::launch_rng_seed(seed, n, out, qb::as_stream(stream));
}

int qb_rng_doubles(int64_t n, uint64_t *rng, int32_t k, double *out, void *stream) {
    QB_REQUIRE(rng && out && n >= 0 && k >= 0, "qb_rng_doubles: bad arguments");
    return qb::launch_rng_doubles(n, rng, k, out, qb::as_stream(stream));
}

int qb_rng_normals(int64_t n, uint64_t *rng, int32_t k, double *out, void *stream) {
    QB_REQUIRE(rng && out && n >= 0 && k >= 0, "qb_rng_normals: bad arguments");
    return qb::launch_rng_normals(n, rng, k, out, qb::as_stream(stream));
}

int qb_rng_poissons(int64_t n, uint64_t *rng, int32_t k, const double *lam, int64_t *out, void *stream) {
    QB_REQUIRE(rng && lam && out && n >= 0 && k >= 0, "qb_rng_poissons: bad arguments");
    return qb::launch_rng_poissons(n, rng, k, lam, out, qb::as_stream(stream));
}

}  // extern "C"
