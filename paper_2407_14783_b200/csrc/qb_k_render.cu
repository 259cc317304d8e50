// qb_k_render.cu -- K2: batched pinhole depth + segmentation ray caster
// (sensing.render_frames -> kernels.render_batch, kernels.py:402-451), plus
// the batched nearest-point / raycast queries (kernels.py:120-182, 389-399).
//
// FP32 production kernels (one warp renders one camera, tile by tile; a tile
// is an 8x4 block of pixels, so the warp's 32 rays are coherent):
//   k_render_cull  scenes of <= 256 primitives: two-level frustum culling
//                  (camera, then tile) and warp-uniform ray tests of the few
//                  survivors -- see the comment above the kernel;
//   k_render_f     any scene: the BVH is walked as a PACKET: the traversal stack and the node sequence are
// warp-uniform, every lane slab-tests the node against its own ray and the
// warp descends while any lane still needs the node (__any_sync).  Node and
// primitive records are warp-broadcast loads through the read-only path, so
// a small scene lives in L1 and a large one in L2.  Depth (z-depth = t*cz)
// and the object id come from the same ray and are written together.  The
// landing task's pad centroid (tasks.py:121-128) is a warp reduction in the
// epilogue.  No tensor cores: nothing here is a contraction.
//
// FP64 validation kernel: one thread per pixel, the reference's exact
// operation order (qb_real.cuh xd), bit-identical to render_batch except
// where traversal-order-dependent pruning could matter at the last ulp.
#include <algorithm>

#include "qb_dynamics.cuh"
#include "qb_geometry.cuh"
#include <mutex>
#include <type_traits>

#include "qb_checks.cuh"
#include "qb_internal.h"

// BVH packet kernel: one camera per warp, QB_RF_BLOCK/32 warps per block and
// one block per QB_RF_BLOCK/32 cameras, so the hardware block scheduler
// balances the very uneven per-camera traversal cost; QB_RF_MINB caps registers
#ifndef QB_RF_BLOCK
#define QB_RF_BLOCK 64
#endif
#ifndef QB_RF_MINB
#define QB_RF_MINB 24
#endif

#ifdef QB_RF_STATS
__device__ unsigned long long g_rf_stats[4];  // tiles, node visits, prim tests, active lanes
extern "C" int qb_debug_render_stats(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_rf_stats, sizeof(g_rf_stats));
}
#endif
#ifdef QB_CULL_STATS
// culling renderer (scripts/cull_stats.py): cameras, candidates, tiles, survivors by record type
// (sphere, AABB, OBB, generic)
__device__ unsigned long long g_cull_stats[8];
extern "C" int qb_debug_cull_stats(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_cull_stats, sizeof(g_cull_stats));
}
#endif

// dynamic camera scheduling of the culling renderer's large launches: one
// claim counter per CUDA stream (slot chosen on the host per stream, zeroed
// in stream order before each launch), so launches on one stream are
// serialised on their counter and launches on different streams never share
// one (up to QB_CULL_SLOTS streams; beyond that slots are shared round-robin)
#ifndef QB_CULL_SLOTS
#define QB_CULL_SLOTS 256
#endif
__device__ unsigned int g_cull_next[QB_CULL_SLOTS];
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr float CULL_EPS = 1e-3f;  // conservative culling margin (m)
#ifndef QB_TPL_MAX
#define QB_TPL_MAX 64
#endif
constexpr int TPL_MAX = QB_TPL_MAX;  // tile-plane table entries (64x64 frames use 32)
constexpr int TILE_W = 8, TILE_H = 4;

struct CamF {
    int W, H;
    float th, tv, max_range;
    float rot[9];
    float trans[3];
};

struct CamD {
    int W, H;
    double th, tv, max_range;
    double rot[9];
    double trans[3];
};

// camera pose from the body pose (sensing.py:66-74): origin = p + R(q) t,
// R_cam->world = to_matrix(q) @ R_cam->body
template <class R>
__device__ __forceinline__ void camera_pose(const R *p, const R *q, const R *crot, const R *ctr, R *o, R *Rw) {
    R m[3][3];
    q_matrix(q, m);
    R ox, oy, oz;
    q_rot<R, 1>(q, ctr[0], ctr[1], ctr[2], ox, oy, oz);
    o[0] = p[0] + ox;
    o[1] = p[1] + oy;
    o[2] = p[2] + oz;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) Rw[3 * i + k] = m[i][0] * crot[k] + m[i][1] * crot[3 + k] + m[i][2] * crot[6 + k];
}

// conservative AABB vs half-space n.x + off >= 0 (n unit): the box's most
// positive corner along n
QB_D bool box_in_plane(const float4 &lo, const float4 &hi, float nx, float ny, float nz, float off) {
    const float px = nx >= 0.0f ? hi.x : lo.x, py = ny >= 0.0f ? hi.y : lo.y, pz = nz >= 0.0f ? hi.z : lo.z;
    return nx * px + ny * py + nz * pz + off >= -CULL_EPS;
}

// world half-space of a camera-space plane through the camera origin with
// normal (a, b, c) (not unit): inside iff n_w . (X - o) >= 0
QB_D void world_plane(const float *Rs, const float *o, float a, float b, float c, float &nx, float &ny, float &nz,
                      float &off) {
    const float inv = rsqrtf(a * a + b * b + c * c);
    a *= inv; b *= inv; c *= inv;
    nx = Rs[0] * a + Rs[1] * b + Rs[2] * c;
    ny = Rs[3] * a + Rs[4] * b + Rs[5] * c;
    nz = Rs[6] * a + Rs[7] * b + Rs[8] * c;
    off = -(nx * o[0] + ny * o[1] + nz * o[2]);
}

// K2 BVH packet renderer (large scenes).  One warp renders one camera:
//  1. camera frontier: lane-parallel breadth-first descent of the scene BVH,
//     keeping nodes whose box meets the camera frustum (4 image planes, near,
//     far), level by level while the frontier still fits in 32 entries
//     (one per lane) -- this replaces the top ~10 levels of every tile's walk;
//  2. per 8x4-pixel tile (one ray per lane): the frontier is culled against
//     the tile's 4 side planes (one entry per lane), each survivor is
//     slab-tested by all rays and pushed far-to-near with its warp-minimum
//     entry distance;
//  3. warp-uniform depth-first traversal from that stack: the current node is
//     carried as its (a, b) record taken from the parent's child fetch (one
//     dependent load per visit: the two adjacent child boxes), both children
//     are slab-tested by every lane, the nearer (lane majority) is visited and
//     the other pushed with its warp-minimum entry (REDUX.MIN on the float
//     bits; entries are >= 0); a pop is skipped unless some lane's hit still
//     lies beyond that entry.  Culling is conservative and the result (nearest
//     t, ties to the lowest id) is traversal-order independent.
#ifdef QB_RF_DEBUG
// debug trace of one (camera, pixel) through k_render_f (scripts/ builds only)
__device__ int g_dbg_target[3] = {-1, -1, -1};
__device__ int g_dbg_n = 0;
__device__ float4 g_dbg_log[8192];
#define QB_DBG(on, kind, a, b, c)                                                       \
    do {                                                                                \
        if (on) {                                                                       \
            int k_ = atomicAdd(&g_dbg_n, 1);                                            \
            if (k_ < 8192) g_dbg_log[k_] = make_float4((float)(kind), (float)(a), (float)(b), (float)(c)); \
        }                                                                               \
    } while (0)
#else
#define QB_DBG(on, kind, a, b, c) do {} while (0)
#endif

// EXACT: 64x64 frame, depth + segmentation, no swarm spheres; CENT: inline
// pad centroid; S1: split == 1 -- compile-time switches of the common
// launches (config 5: EXACT + CENT + S1), as in the culling renderer
template <bool FROM_STATE, bool EXACT = false, bool CENT = false, bool S1 = false, bool SEGP = true>
__global__ void __launch_bounds__(QB_RF_BLOCK, QB_RF_MINB) k_render_f(DevScene S, CamF cam, long long n, long long ld, const float *state,
                                                     const float *origins, const float *rotations, const int32_t *env_scene,
                                                     float *depth, int32_t *seg, int centroid_id, float *centroid,
                                                     const float *extra, const int32_t *extra_ids, int n_extra, int split) {
    constexpr int WPB = QB_RF_BLOCK / 32, STK = 96;  // stack: <= 32 frontier entries + one per tree level (<= 62)
    __shared__ int2 stk_s[WPB][STK];  // (node record packed as a * 8 + (b + 2), entry distance bits)
    __shared__ int fr_s[WPB][32];     // camera frontier (node indices)
    __shared__ float rw_s[WPB][9];    // camera rotation (kept out of registers)
    int2 *stk = stk_s[threadIdx.x >> 5];
    int *fr = fr_s[threadIdx.x >> 5];
    float *Rs = rw_s[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned lanes_below = (1u << lane) - 1u;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int W = EXACT ? 64 : cam.W, H = EXACT ? 64 : cam.H;
    if (S1) split = 1;
    const int tiles_x = (W + TILE_W - 1) / TILE_W, tiles_y = (H + TILE_H - 1) / TILE_H;
    const float tmin = 1e-9f;
    const float sx = 2.0f / W, sy = 2.0f / H;
    constexpr unsigned INF_BITS = 0x7f800000u;

    // small batches: `split` warps share one camera (each builds the camera
    // frontier and takes every split-th tile)
    for (long long wi = warp; wi < n * split; wi += nwarps) {
        const long long c = S1 ? wi : wi / split;
        const int part = S1 ? 0 : (int)(wi % split);
        float o[3];
        {
            float Rw[9];
            if (FROM_STATE) {
                float p[3] = {state[0 * ld + c], state[1 * ld + c], state[2 * ld + c]};
                float q[4] = {state[6 * ld + c], state[7 * ld + c], state[8 * ld + c], state[9 * ld + c]};
                camera_pose<float>(p, q, cam.rot, cam.trans, o, Rw);
            } else {
#pragma unroll
                for (int k = 0; k < 3; ++k) o[k] = origins[3 * c + k];
#pragma unroll
                for (int k = 0; k < 9; ++k) Rw[k] = rotations[9 * c + k];
            }
            __syncwarp();
            if (lane < 9) Rs[lane] = Rw[lane];  // (all lanes hold the same pose)
            __syncwarp();
        }
        const int scene = env_scene ? env_scene[c] : 0;
        int cnt = 0, sum_col = 0, sum_row = 0;

        // ---- 1. camera frontier
        int nf = 1;
        if (lane == 0) fr[0] = S.root[scene];
        __syncwarp();
        {
            const float xa = (0.5f * sx - 1.0f) * cam.th, xb = ((W - 0.5f) * sx - 1.0f) * cam.th;
            const float ya = (0.5f * sy - 1.0f) * cam.tv, yb = ((H - 0.5f) * sy - 1.0f) * cam.tv;
            float pn[6][3], po[6];
            world_plane(Rs, o, 1.0f, 0.0f, -xa, pn[0][0], pn[0][1], pn[0][2], po[0]);
            world_plane(Rs, o, -1.0f, 0.0f, xb, pn[1][0], pn[1][1], pn[1][2], po[1]);
            world_plane(Rs, o, 0.0f, 1.0f, -ya, pn[2][0], pn[2][1], pn[2][2], po[2]);
            world_plane(Rs, o, 0.0f, -1.0f, yb, pn[3][0], pn[3][1], pn[3][2], po[3]);
            world_plane(Rs, o, 0.0f, 0.0f, 1.0f, pn[4][0], pn[4][1], pn[4][2], po[4]);  // in front
            pn[5][0] = -pn[4][0]; pn[5][1] = -pn[4][1]; pn[5][2] = -pn[4][2];
            po[5] = -po[4] + cam.max_range;                                              // z-depth <= max range
            auto in_frustum = [&](const float4 &lo, const float4 &hi) {
                bool in = true;
#pragma unroll
                for (int k = 0; k < 6; ++k) in &= box_in_plane(lo, hi, pn[k][0], pn[k][1], pn[k][2], po[k]);
                return in;
            };
            for (int level = 0; level < 64; ++level) {
                const bool have = lane < nf;
                const int node = have ? fr[lane] : 0;
                const float4 lo = __ldg(S.nodef + 2 * node), hi = __ldg(S.nodef + 2 * node + 1);
                const int a = __float_as_int(lo.w), b = __float_as_int(hi.w);
                const bool inner = have && b <= 0;
                if (!__any_sync(FULL, inner)) break;
                bool kl = false, kr = false;
                if (inner) {
                    kl = in_frustum(__ldg(S.nodef + 2 * a), __ldg(S.nodef + 2 * a + 1));
                    kr = in_frustum(__ldg(S.nodef + 2 * a + 2), __ldg(S.nodef + 2 * a + 3));
                }
                const int nout = inner ? (int)kl + (int)kr : (have ? 1 : 0);
                const unsigned b0 = __ballot_sync(FULL, nout & 1), b1 = __ballot_sync(FULL, nout & 2);
                const int total = __popc(b0) + 2 * __popc(b1);
                if (total > 32) break;
                const int pos = __popc(b0 & lanes_below) + 2 * __popc(b1 & lanes_below);
                __syncwarp();
                if (inner) {
                    int q = pos;
                    if (kl) fr[q++] = a;
                    if (kr) fr[q] = a + 1;
                } else if (have) {
                    fr[pos] = node;
                }
                __syncwarp();
                nf = total;
                if (nf == 0) break;
            }
        }

        for (int tile = part; tile < tiles_x * tiles_y; tile += split) {
            const int j0 = (tile % tiles_x) * TILE_W, i0 = (tile / tiles_x) * TILE_H;
            const int j = j0 + (lane & 7);
            const int i = i0 + (lane >> 3);
            const bool valid = EXACT || ((j < W) && (i < H));
#ifdef QB_RF_DEBUG
            const bool dbg = c == g_dbg_target[0] && i == g_dbg_target[1] && j == g_dbg_target[2];
#else
            constexpr bool dbg = false;
#endif
            const float y = ((i + 0.5f) * sy - 1.0f) * cam.tv;
            const float x = ((j + 0.5f) * sx - 1.0f) * cam.th;
            const float n2 = x * x + y * y + 1.0f;
            float dx, dy, dz, tmax;
            {
                const float cz = rsqrtf(n2);
                const float cx = x * cz, cy = y * cz;
                dx = Rs[0] * cx + Rs[1] * cy + Rs[2] * cz;
                dy = Rs[3] * cx + Rs[4] * cy + Rs[5] * cz;
                dz = Rs[6] * cx + Rs[7] * cy + Rs[8] * cz;
                tmax = cam.max_range * (n2 * cz);  // max_range / cos(angle to the axis)
            }
            const float ix = rcp_approx(dx), iy = rcp_approx(dy), iz = rcp_approx(dz);
            const float oix = o[0] * ix, oiy = o[1] * iy, oiz = o[2] * iz;
            // the triangle test's shear axis: the dominant axis of a ray near the
            // tile centre, warp-uniform (a tile spans ~11 deg, so |d[kz]| >= 0.38)
            const int kz = __shfl_sync(FULL, dominant_axis(dx, dy, dz), 12);
            const Shear sh = ray_shear(kz, dx, dy, dz);  // per ray, once per tile (not per triangle test)

            // lanes outside the image carry best = -1: they never want a box
            float best = valid ? tmax : -1.0f;
            int bp = -1;  // nearest primitive so far; its object id is read once, after the traversal
            bool hit = false;
#ifdef QB_RF_STATS
            unsigned st_visit = 0, st_prim = 0, st_active = __popc(__ballot_sync(FULL, valid));
#endif

            // ---- 2. frontier entries meeting the tile's frustum, far-to-near on the stack
            int sp = 0;
            {
                const int jb = min(j0 + TILE_W, W) - 1, ib = min(i0 + TILE_H, H) - 1;
                const float xa = ((j0 + 0.5f) * sx - 1.0f) * cam.th, xb = ((jb + 0.5f) * sx - 1.0f) * cam.th;
                const float ya = ((i0 + 0.5f) * sy - 1.0f) * cam.tv, yb = ((ib + 0.5f) * sy - 1.0f) * cam.tv;
                bool in = false;
                if (lane < nf) {
                    const int node = fr[lane];
                    const float4 lo = __ldg(S.nodef + 2 * node), hi = __ldg(S.nodef + 2 * node + 1);
                    float nx, ny, nz, of;
                    world_plane(Rs, o, 1.0f, 0.0f, -xa, nx, ny, nz, of);
                    in = box_in_plane(lo, hi, nx, ny, nz, of);
                    world_plane(Rs, o, -1.0f, 0.0f, xb, nx, ny, nz, of);
                    in &= box_in_plane(lo, hi, nx, ny, nz, of);
                    world_plane(Rs, o, 0.0f, 1.0f, -ya, nx, ny, nz, of);
                    in &= box_in_plane(lo, hi, nx, ny, nz, of);
                    world_plane(Rs, o, 0.0f, -1.0f, yb, nx, ny, nz, of);
                    in &= box_in_plane(lo, hi, nx, ny, nz, of);
                }
                // survivors' entry distances (all rays), kept one per lane
                unsigned my_e = INF_BITS;
                int my_rec = 0, ns = 0;
#ifdef QB_RF_DEBUG
                for (int q = 0; q < nf; ++q) {
                    const int inq = __shfl_sync(FULL, (int)in, q);
                    QB_DBG(dbg, 1, fr[q], inq, nf);
                }
#endif
                for (unsigned m = __ballot_sync(FULL, in); m; m &= m - 1) {
                    const int node = fr[__ffs(m) - 1];
                    const float4 lo = __ldg(S.nodef + 2 * node), hi = __ldg(S.nodef + 2 * node + 1);
                    const float e = slab_enter_fma(lo, hi, oix, oiy, oiz, ix, iy, iz, best);
                    QB_DBG(dbg, 2, node, e, best);
                    const unsigned em = __reduce_min_sync(FULL, e <= best ? __float_as_uint(e) : INF_BITS);
                    if (em != INF_BITS) {
                        if (lane == ns) {
                            my_e = em;
                            my_rec = __float_as_int(lo.w) * 8 + (__float_as_int(hi.w) + 2);
                        }
                        ++ns;
                    }
                }
                // rank: farthest first (bottom of the stack), ties by lane
                int rank = 0;
                for (int q = 0; q < ns; ++q) {
                    const unsigned eq = __shfl_sync(FULL, my_e, q);
                    rank += (eq > my_e) || (eq == my_e && q < lane);
                }
                __syncwarp();
                QB_CHECK(lane >= ns || rank < STK, "k_render_f frontier stack");
                if (lane < ns) stk[rank] = make_int2(my_rec, (int)my_e);
                sp = ns;
                __syncwarp();
            }

            // ---- 3. depth-first traversal; (ca, cb): leaf {first, count > 0} or
            // internal {left child, -axis <= 0}; ca < 0: pop
            int ca = -1, cb = 0;
            while (true) {
                if (ca < 0) {
                    while (sp > 0) {
                        const int2 e = stk[--sp];
                        QB_DBG(dbg, 3, e.x >> 3, __uint_as_float((unsigned)e.y), best);
                        if (__any_sync(FULL, __uint_as_float((unsigned)e.y) <= best)) {
                            ca = e.x >> 3;
                            cb = (e.x & 7) - 2;
                            break;
                        }
                    }
                    __syncwarp();
                    if (ca < 0) break;
                }
#ifdef QB_RF_STATS
                ++st_visit;
#endif
                if (cb > 0) {
#ifdef QB_RF_STATS
                    st_prim += cb;
#endif
                    // tests return t <= best; ties (rare) go to the lower object id
                    auto take = [&](float t, int p) {
                        if (t > 0.0f && (t < best || !hit || __ldg(&S.meta[p].y) < __ldg(&S.meta[bp].y))) {
                            best = t;
                            bp = p;
                            hit = true;
                        }
                    };
                    if (S.tri_only) {
                        // meshes: no type load or dispatch, and the tile's shear axis is
                        // resolved once per leaf instead of per triangle
                        auto leaf = [&](auto kzc) {
                            constexpr int KZ = decltype(kzc)::value;
                            for (int p = ca; p < ca + cb; ++p) {
                                const float4 *pr = S.primf + 4 * p;
                                take(ray_triangle_wt<KZ>(__ldg(pr), __ldg(pr + 1), __ldg(pr + 2), o[0], o[1], o[2], sh, tmin,
                                                         best),
                                     p);
                            }
                        };
                        if (kz == 2)
                            leaf(std::integral_constant<int, 2>{});
                        else if (kz == 1)
                            leaf(std::integral_constant<int, 1>{});
                        else
                            leaf(std::integral_constant<int, 0>{});
                    } else {
                        for (int p = ca; p < ca + cb; ++p) {
                            // record and type loads issued together
                            const float4 *pr = S.primf + 4 * p;
                            const float4 ra = __ldg(pr), rb = __ldg(pr + 1), rc = __ldg(pr + 2);
                            const int ty = __ldg(&S.meta[p].x);
                            float t;
                            if (ty == QB_TRIANGLE)
                                t = ray_triangle_v(kz, ra, rb, rc, o[0], o[1], o[2], sh, tmin, best);
                            else if (ty == QB_BOX)
                                t = ray_box_v(ra, rb, rc, __ldg(pr + 3), o[0], o[1], o[2], dx, dy, dz, tmin, best);
                            else
                                t = ray_sphere_v(ra, rb.x, o[0], o[1], o[2], dx, dy, dz, tmin, best);
                            QB_DBG(dbg, 5, p, t, best);
                            take(t, p);
                        }
                    }
                    ca = -1;
                    continue;
                }
                const float4 llo = __ldg(S.nodef + 2 * ca), lhi = __ldg(S.nodef + 2 * ca + 1);
                const float4 rlo = __ldg(S.nodef + 2 * ca + 2), rhi = __ldg(S.nodef + 2 * ca + 3);
                const float el = slab_enter_fma(llo, lhi, oix, oiy, oiz, ix, iy, iz, best);
                const float er = slab_enter_fma(rlo, rhi, oix, oiy, oiz, ix, iy, iz, best);
                QB_DBG(dbg, 4, ca, el, er);
                const bool wl = el <= best, wr = er <= best;
                const bool hl = __any_sync(FULL, wl);
                const bool hr = __any_sync(FULL, wr);
                if (hl && hr) {
                    const bool left_first = __popc(__ballot_sync(FULL, el <= er)) >= 16;
                    const float4 nlo = left_first ? llo : rlo, nhi = left_first ? lhi : rhi;
                    const float4 flo = left_first ? rlo : llo, fhi = left_first ? rhi : lhi;
                    const float ef = left_first ? er : el;
                    const bool wf = left_first ? wr : wl;
                    const unsigned em = __reduce_min_sync(FULL, wf ? __float_as_uint(ef) : INF_BITS);
                    // every lane stores the (warp-uniform) entry: each lane's later pop
                    // then reads its own store.  A lane-0-only store is a cross-lane
                    // shared-memory dependency with no __syncwarp before the pop: the
                    // compiler may sink the store below the other lanes' loads, which then
                    // pop a stale entry and skip a subtree (seen as one C5 pixel reading a
                    // surface 0.6 m behind the one it should hit)
                    QB_CHECK(sp < STK, "k_render_f traversal stack");
                    stk[sp] = make_int2(__float_as_int(flo.w) * 8 + (__float_as_int(fhi.w) + 2), (int)em);
                    ++sp;
                    ca = __float_as_int(nlo.w);
                    cb = __float_as_int(nhi.w);
                } else if (hl || hr) {
                    ca = __float_as_int(hl ? llo.w : rlo.w);
                    cb = __float_as_int(hl ? lhi.w : rhi.w);
                } else {
                    ca = -1;
                }
            }
#ifdef QB_RF_STATS
            if (lane == 0) {
                atomicAdd(&g_rf_stats[0], 1ull);
                atomicAdd(&g_rf_stats[1], (unsigned long long)st_visit);
                atomicAdd(&g_rf_stats[2], (unsigned long long)st_prim);
                atomicAdd(&g_rf_stats[3], (unsigned long long)st_active);
            }
#endif
            float t = hit ? best : -1.0f;
            int oid = hit ? __ldg(&S.meta[bp].y) : -1;
            if (!EXACT && n_extra > 0) {  // swarm agents as spheres (kernels.py:438-445)
                for (int k = 0; k < n_extra; ++k) {
                    const float4 sph = *reinterpret_cast<const float4 *>(extra + (c * n_extra + k) * 4);
                    float ts = ray_sphere_v(sph, sph.w * sph.w, o[0], o[1], o[2], dx, dy, dz, tmin, tmax);
                    if (ts > 0.0f && (t < 0.0f || ts < t)) {
                        t = ts;
                        oid = extra_ids[c * n_extra + k];
                    }
                }
            }
            const int out_id = t > 0.0f ? oid : 0;
            if (valid) {
                const long long off = (c * H + i) * (long long)W + j;
                if (EXACT || depth) depth[off] = t > 0.0f ? t * rsqrtf(n2) : cam.max_range;
                if (EXACT ? SEGP : seg != nullptr) seg[off] = out_id;
                if ((EXACT ? CENT : centroid_id > 0) && out_id == centroid_id) {
                    cnt += 1;
                    sum_col += j;
                    sum_row += i;
                }
            }
        }
        if ((EXACT ? CENT : centroid_id > 0) && split == 1) {  // (split: the k_centroid pass)
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                cnt += __shfl_xor_sync(FULL, cnt, s);
                sum_col += __shfl_xor_sync(FULL, sum_col, s);
                sum_row += __shfl_xor_sync(FULL, sum_row, s);
            }
            if (lane == 0) {
                centroid[2 * c] = cnt ? (float)((double)sum_col / (double)cnt) : -1.0f;
                centroid[2 * c + 1] = cnt ? (float)((double)sum_row / (double)cnt) : -1.0f;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Culling renderer for small scenes (<= CULL_MAX primitives per scene, e.g.
// the 69-primitive navigation room).  One warp renders one camera:
//  1. camera culling: lane-parallel over the scene's primitives, 6 plane /
//     support-function tests (image frustum, near, far) -> candidate list;
//  2. per candidate (lane-parallel) a CAMERA-SPECIFIC record in shared
//     memory: its culling bounds in camera space and its ray-test constants
//     for this camera origin (sphere: o - c; box: slab numerators +-h - R^T(o-c);
//     oriented box: also R's columns), so a pixel's primitive test is just
//     the direction-dependent part (AABB ~15, OBB ~30, sphere ~18 instr);
//  3. per 8x4 tile: cull the records against the tile's 4 side planes in
//     camera space (lane-parallel), then ray-test the survivors
//     warp-uniformly with shared approximate reciprocals of the direction.
// Culling is conservative (support functions of spheres / OBBs / triangle
// bounding spheres, 1 mm margin); the per-pixel result -- nearest t, ties to
// the lowest id -- does not depend on test order, so ids equal the BVH
// kernel's and depths agree to FP32 rounding.
constexpr int CULL_MAX = 256;   // primitives per scene
#ifndef QB_CULL_MINB
#define QB_CULL_MINB 6  // 6 blocks at 80 registers without spills (rotation in shared memory); 6 with spills was 19% slower
#endif
#ifndef QB_CREC
#define QB_CREC 56
#endif
#ifndef QB_CULL_WARPS
#define QB_CULL_WARPS 4
#endif
constexpr int CULL_WARPS = QB_CULL_WARPS;  // warps (cameras) per block
constexpr int XMAX = 32;  // swarm spheres kept per camera after frustum culling (more: every sphere per ray)
constexpr int CREC = QB_CREC;   // precomputed records per camera (nav room: mean 21, max 58); more use the generic path (56 keeps 6 blocks/SM in shared memory)
// record word rec[k][1].w: a type flag in the top bits over the object id
// (flag bits, not an enum: an if-chain on distinct bits stays a chain of
// predicate tests, where an enum compare chain compiles to a jump table --
// a constant-bank load and an indirect branch per survivor); a record
// without a flag (triangles, ids >= 2^29) holds its primitive index in
// rec[k][1].x and takes the generic test
constexpr unsigned REC_AABB = 1u << 31, REC_OBB = 1u << 30, REC_SPHERE = 1u << 29, REC_ID = REC_SPHERE - 1u;

struct Plane {
    float x, y, z, off;
};

__device__ __forceinline__ Plane world_plane(const float *Rw, float cx, float cy, float cz, float off) {
    const float inv = rsqrtf(cx * cx + cy * cy + cz * cz);
    cx *= inv; cy *= inv; cz *= inv;
    return {Rw[0] * cx + Rw[1] * cy + Rw[2] * cz, Rw[3] * cx + Rw[4] * cy + Rw[5] * cz, Rw[6] * cx + Rw[7] * cy + Rw[8] * cz,
            off};
}

// keep unless the primitive's support along the plane normal is fully outside
__device__ __forceinline__ bool keep(const Plane &P, float rx, float ry, float rz, float4 c, float4 a0, float4 a1, float4 a2) {
    const float d = P.x * rx + P.y * ry + P.z * rz + P.off;
    const float s = c.w + fabsf(P.x * a0.x + P.y * a0.y + P.z * a0.z) + fabsf(P.x * a1.x + P.y * a1.y + P.z * a1.z) +
                    fabsf(P.x * a2.x + P.y * a2.y + P.z * a2.z);
    return d + s >= -CULL_EPS;
}


// slab intersection from precomputed numerators (kernels.py:203-246 semantics:
// entry clamped at tmin, exit returned when the origin is inside)
__device__ __forceinline__ float slab_hit(float nlx, float nly, float nlz, float nhx, float nhy, float nhz, float ix, float iy,
                                          float iz, float tmin, float tmax) {
    const float tax = nlx * ix, tbx = nhx * ix, tay = nly * iy, tby = nhy * iy, taz = nlz * iz, tbz = nhz * iz;
    const float t0 = fmaxf(fmaxf(fminf(tax, tbx), fminf(tay, tby)), fmaxf(fminf(taz, tbz), tmin));
    const float t1 = fminf(fminf(fmaxf(tax, tbx), fmaxf(tay, tby)), fminf(fmaxf(taz, tbz), tmax));
    if (t0 > t1) return -1.0f;
    // (t0 <= t1 <= tmax here: only the tmin tests remain)
    return t0 > tmin ? t0 : (t1 > tmin ? t1 : -1.0f);
}

// CENT: a pad centroid is reduced inline (landing, split == 1): a compile-time
// switch, so the common render carries no per-pixel centroid test.
// EXACT: a 64x64 frame with both outputs (the spec's camera, configs 2-5):
// compile-time sizes, no per-pixel bounds / null tests, the tile-plane table.
// S1: split == 1 (large batches: one warp per camera, cameras grid-strided).
// EXTRA: swarm spheres present (separate instance: no swarm shared memory or
// registers in the common case)
template <bool FROM_STATE, bool EXTRA, bool CENT, bool EXACT, bool S1, bool SEGP = true>
__global__ void __launch_bounds__(CULL_WARPS * 32, QB_CULL_MINB)
    k_render_cull(DevScene S, CamF cam, long long n, long long ld, const float *state, const float *origins,
                  const float *rotations, const int32_t *env_scene, float *depth, int32_t *seg, int centroid_id,
                  float *centroid, const float *extra, const int32_t *extra_ids, int n_extra, int split,
                  unsigned int *claim) {
    __shared__ int cand_s[CULL_WARPS][CULL_MAX];
    constexpr int XM = EXTRA ? XMAX : 1;
    __shared__ float rws_s[CULL_WARPS][9];               // camera rotation for the tile loop (out of registers)
    __shared__ float4 xcs_s[CULL_WARPS][XM];             // swarm spheres in the frustum: camera-space centre, r
    __shared__ int xk_s[CULL_WARPS][XM];                 // ... and their index k (ascending)
    __shared__ float4 rec_s[CULL_WARPS][CREC][4];      // shading records (warp-broadcast reads)
    __shared__ float cul_s[CULL_WARPS][13][CREC];      // culling bounds, SoA (conflict-free lane-parallel reads)
    __shared__ float4 tpl_s[TPL_MAX][2];               // per-tile camera-space planes (xl xr yt yb) (iL iR iT iB)
    const int wib = threadIdx.x >> 5;
    int *cand = cand_s[wib];
    float4 (*rec)[4] = rec_s[wib];
    float (*cul)[CREC] = cul_s[wib];
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    // EXACT: the 64x64 frame of the spec's camera, sizes known at compile time
    const int W = EXACT ? 64 : cam.W, H = EXACT ? 64 : cam.H;
    const int tiles_x = (W + TILE_W - 1) / TILE_W;
    const float tmin = 1e-9f;
    // pixel-centre image-plane coordinates: x(j) = ((j + 0.5) * 2/W - 1) * th
    const float sx = 2.0f / W, sy = 2.0f / H;
    constexpr int TH2 = 2 * TILE_H;
    const int tiles_y2 = (H + TH2 - 1) / TH2, n_tiles = tiles_y2 * tiles_x;
    // the tile planes depend on the tile only: one table per block
    const bool tpl = EXACT || n_tiles <= TPL_MAX;
    if (tpl) {
        for (int tl = threadIdx.x; tl < n_tiles; tl += blockDim.x) {
            const int i0 = (tl / tiles_x) * TH2, j0 = (tl % tiles_x) * TILE_W;
            const int j1 = min(j0 + TILE_W - 1, W - 1), i1 = min(i0 + TH2 - 1, H - 1);
            const float xl = ((j0 + 0.5f) * sx - 1.0f) * cam.th, xr = ((j1 + 0.5f) * sx - 1.0f) * cam.th;
            const float yt = ((i0 + 0.5f) * sy - 1.0f) * cam.tv, yb = ((i1 + 0.5f) * sy - 1.0f) * cam.tv;
            tpl_s[tl][0] = make_float4(xl, xr, yt, yb);
            tpl_s[tl][1] = make_float4(rsqrtf(1.f + xl * xl), rsqrtf(1.f + xr * xr), rsqrtf(1.f + yt * yt),
                                       rsqrtf(1.f + yb * yb));
        }
    }
    __syncthreads();

    // small batches: `split` warps share one camera, each taking every split-th tile
    if (S1) split = 1;
    // large batches (S1): after its first camera a warp claims the next
    // unclaimed one from the launch's counter -- per-camera costs vary (a wall
    // at 1 m vs a cluttered room), and static striding left SMs idle at the end
    for (long long wi = warp; wi < n * split;) {
        const long long c = S1 ? wi : wi / split;
        const int part = S1 ? 0 : (int)(wi % split);
        float o[3], Rw[9];
        if (FROM_STATE) {
            float p[3] = {state[0 * ld + c], state[1 * ld + c], state[2 * ld + c]};
            float q[4] = {state[6 * ld + c], state[7 * ld + c], state[8 * ld + c], state[9 * ld + c]};
            camera_pose<float>(p, q, cam.rot, cam.trans, o, Rw);
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) o[k] = origins[3 * c + k];
#pragma unroll
            for (int k = 0; k < 9; ++k) Rw[k] = rotations[9 * c + k];
        }
        const int scene = env_scene ? env_scene[c] : 0;
        QB_CHECK(scene >= 0 && scene < S.n_scenes, "k_render_cull scene index");
        const int p0 = S.prim_offset[scene], p1 = S.prim_offset[scene + 1];
        QB_CHECK(p1 - p0 <= CULL_MAX, "k_render_cull scene size");

        // ---- 1. camera frustum culling (image frustum, near z >= 0, far z <= max_range)
        int ncand = 0;  // warp-uniform
        {
            const Plane cp[6] = {world_plane(Rw, 1.f, 0.f, cam.th, 0.f), world_plane(Rw, -1.f, 0.f, cam.th, 0.f),
                                 world_plane(Rw, 0.f, 1.f, cam.tv, 0.f), world_plane(Rw, 0.f, -1.f, cam.tv, 0.f),
                                 world_plane(Rw, 0.f, 0.f, 1.f, 0.f), world_plane(Rw, 0.f, 0.f, -1.f, cam.max_range)};
            int &nc = ncand;
            for (int b = p0; b < p1; b += 32) {
                const int p = b + lane;
                bool k = false;
                if (p < p1) {
                    const float4 *cr = S.primc + 4 * p;
                    const float4 c0 = __ldg(cr), a0 = __ldg(cr + 1), a1 = __ldg(cr + 2), a2 = __ldg(cr + 3);
                    const float rx = c0.x - o[0], ry = c0.y - o[1], rz = c0.z - o[2];
                    k = true;
#pragma unroll
                    for (int q = 0; q < 6; ++q) k = k && keep(cp[q], rx, ry, rz, c0, a0, a1, a2);
                }
                const unsigned m = __ballot_sync(FULL, k);
                QB_CHECK(!k || nc + __popc(m & lt_mask) < CULL_MAX, "k_render_cull candidate list");
                if (k) cand[nc + __popc(m & lt_mask)] = p;
                nc += __popc(m);
            }
            __syncwarp();
            // ---- 2. camera-specific records
            for (int k = lane; k < min(nc, CREC); k += 32) {
                const int p = cand[k];
                const float4 *cr = S.primc + 4 * p;
                const float4 c0 = __ldg(cr), a0 = __ldg(cr + 1), a1 = __ldg(cr + 2), a2 = __ldg(cr + 3);
                const int2 mt = __ldg(S.meta + p);
                const float rx = c0.x - o[0], ry = c0.y - o[1], rz = c0.z - o[2];
                // camera-space culling bounds: v' = Rw^T v
                auto cs = [&](float x, float y, float z) {
                    return make_float3(Rw[0] * x + Rw[3] * y + Rw[6] * z, Rw[1] * x + Rw[4] * y + Rw[7] * z,
                                       Rw[2] * x + Rw[5] * y + Rw[8] * z);
                };
                const float3 cc = cs(rx, ry, rz), A0 = cs(a0.x, a0.y, a0.z), A1 = cs(a1.x, a1.y, a1.z),
                             A2 = cs(a2.x, a2.y, a2.z);
                unsigned type = 0;  // generic
                float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0, s2 = s0, s3 = s0;
                const float4 *pr = S.primf + 4 * p;
                if (mt.x == QB_SPHERE) {
                    const float4 pa = __ldg(pr), pb = __ldg(pr + 1);
                    type = REC_SPHERE;
                    s0 = make_float4(o[0] - pa.x, o[1] - pa.y, o[2] - pa.z, pb.x);  // m = o - c, r^2
                } else if (mt.x == QB_BOX) {
                    const float4 pa = __ldg(pr), pb = __ldg(pr + 1), pc = __ldg(pr + 2), pe = __ldg(pr + 3);
                    // R rows: (pb.z pb.w pc.x) (pc.y pc.z pc.w) (pe.x pe.y pe.z); local = R^T (o - c)
                    const float mx = o[0] - pa.x, my = o[1] - pa.y, mz = o[2] - pa.z;
                    const float lx = pb.z * mx + pc.y * my + pe.x * mz;
                    const float ly = pb.w * mx + pc.z * my + pe.y * mz;
                    const float lz = pc.x * mx + pc.w * my + pe.z * mz;
                    const float hx = pa.w, hy = pb.x, hz = pb.y;
                    s0 = make_float4(-hx - lx, -hy - ly, -hz - lz, hx - lx);
                    s1 = make_float4(hy - ly, hz - lz, 0.f, 0.f);
                    const bool ident = pb.z == 1.f && pb.w == 0.f && pc.x == 0.f && pc.y == 0.f && pc.z == 1.f &&
                                       pc.w == 0.f && pe.x == 0.f && pe.y == 0.f && pe.z == 1.f;
                    type = ident ? REC_AABB : REC_OBB;
                    s2 = make_float4(pb.z, pc.y, pe.x, pb.w);  // columns of R: local d = (col0.d, col1.d, col2.d)
                    s3 = make_float4(pc.z, pe.y, pc.x, pc.w);
                    s1.z = pe.z;
                }
                if ((unsigned)mt.y > REC_ID) type = 0;  // (the id does not fit the word: generic)
                s1.w = __uint_as_float(type ? type | (unsigned)mt.y : 0u);
                if (!type) s1.x = __int_as_float(p);
                rec[k][0] = s0;
                rec[k][1] = s1;
                rec[k][2] = s2;
                rec[k][3] = s3;
                const float cv[13] = {c0.w, cc.x, cc.y, cc.z, A0.x, A0.y, A0.z, A1.x, A1.y, A1.z, A2.x, A2.y, A2.z};
#pragma unroll
                for (int q = 0; q < 13; ++q) cul[q][k] = cv[q];
            }
            __syncwarp();
        }

        // swarm agents as spheres (kernels.py:438-445): keep the ones in the
        // camera frustum, in ascending k (ties go to the lowest k), with their
        // camera-space centres for the per-tile test
        int nx = 0;             // warp-uniform
        bool x_all = false;     // too many in view: test every sphere per ray
        if (EXTRA && n_extra > 0) {
            const Plane cp[6] = {world_plane(Rw, 1.f, 0.f, cam.th, 0.f), world_plane(Rw, -1.f, 0.f, cam.th, 0.f),
                                 world_plane(Rw, 0.f, 1.f, cam.tv, 0.f), world_plane(Rw, 0.f, -1.f, cam.tv, 0.f),
                                 world_plane(Rw, 0.f, 0.f, 1.f, 0.f), world_plane(Rw, 0.f, 0.f, -1.f, cam.max_range)};
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int b = 0; b < n_extra && !x_all; b += 32) {
                const int k = b + lane;
                bool in = false;
                float4 sph = z4;
                if (k < n_extra) {
                    sph = *reinterpret_cast<const float4 *>(extra + (c * n_extra + k) * 4);
                    const float rx = sph.x - o[0], ry = sph.y - o[1], rz = sph.z - o[2];
                    in = true;
#pragma unroll
                    for (int q = 0; q < 6; ++q) in = in && keep(cp[q], rx, ry, rz, sph, z4, z4, z4);
                    if (in) {  // camera space: v' = Rw^T v
                        sph = make_float4(Rw[0] * rx + Rw[3] * ry + Rw[6] * rz, Rw[1] * rx + Rw[4] * ry + Rw[7] * rz,
                                          Rw[2] * rx + Rw[5] * ry + Rw[8] * rz, sph.w);
                    }
                }
                const unsigned m = __ballot_sync(FULL, in);
                if (nx + __popc(m) > XM) {
                    x_all = true;
                } else {
                    if (in) {
                        const int pos = nx + __popc(m & lt_mask);
                        QB_CHECK(pos < XM, "k_render_cull swarm list");
                        xcs_s[wib][pos] = sph;
                        xk_s[wib][pos] = k;
                    }
                    nx += __popc(m);
                }
            }
            __syncwarp();
        }

#ifdef QB_CULL_STATS
        if (lane == 0 && part == 0) {
            atomicAdd(&g_cull_stats[0], 1ull);
            atomicAdd(&g_cull_stats[1], (unsigned long long)ncand);
        }
#endif
        // EXACT (64x64 = 8 x 8 tiles): the tile culling below evaluates, per tile, the
        // record's support against the tile's 4 border-pixel planes; every tile of a
        // column shares its L / R planes and every tile of a row its T / B planes, so
        // the same tests are run once per camera for the 8 columns and 8 rows (32
        // planes) and kept as two 8-bit masks per record -- a tile's test becomes two
        // bit lookups, with bit-identical decisions
        static_assert(CREC <= 64, "the EXACT tile masks live in two registers per lane");
        unsigned tm0 = 0, tm1 = 0;  // EXACT: the tile masks of records lane and lane + 32, in registers
        // (only when one warp renders all 64 tiles of the camera: a warp that takes
        // a few tiles of a split camera is better off testing its tiles directly)
        if (EXACT && S1) {
            const int nrec = min(ncand, CREC);
            for (int b = 0; b < nrec; b += 32) {
                const int k = b + lane;
                if (k < nrec) {
                    const float rr = cul[0][k], ccx = cul[1][k], ccy = cul[2][k], ccz = cul[3][k];
                    const float a0x = cul[4][k], a0y = cul[5][k], a0z = cul[6][k];
                    const float a1x = cul[7][k], a1y = cul[8][k], a1z = cul[9][k];
                    const float a2x = cul[10][k], a2y = cul[11][k], a2z = cul[12][k];
                    unsigned msk = 0;
#pragma unroll 1
                    for (int q = 0; q < 8; ++q) {  // column q: tiles tl = q + 8 r share xl, xr (tpl_s[q])
                        const float4 pa = tpl_s[q][0], pb = tpl_s[q][1];
                        const float xl = pa.x, xr = pa.y, iL = pb.x, iR = pb.y;
                        const float dL = (ccx - xl * ccz) * iL,
                                    sL = (fabsf(a0x - xl * a0z) + fabsf(a1x - xl * a1z) + fabsf(a2x - xl * a2z)) * iL;
                        const float dR = (xr * ccz - ccx) * iR,
                                    sR = (fabsf(xr * a0z - a0x) + fabsf(xr * a1z - a1x) + fabsf(xr * a2z - a2x)) * iR;
                        if ((dL + sL + rr >= -CULL_EPS) && (dR + sR + rr >= -CULL_EPS)) msk |= 1u << q;
                    }
#pragma unroll 1
                    for (int q = 0; q < 8; ++q) {  // row q: tiles tl = 8 q + c share yt, yb (tpl_s[8 q])
                        const float4 pa = tpl_s[8 * q][0], pb = tpl_s[8 * q][1];
                        const float yt = pa.z, yb = pa.w, iT = pb.z, iB = pb.w;
                        const float dT = (ccy - yt * ccz) * iT,
                                    sT = (fabsf(a0y - yt * a0z) + fabsf(a1y - yt * a1z) + fabsf(a2y - yt * a2z)) * iT;
                        const float dB = (yb * ccz - ccy) * iB,
                                    sB = (fabsf(yb * a0z - a0y) + fabsf(yb * a1z - a1y) + fabsf(yb * a2z - a2y)) * iB;
                        if ((dT + sT + rr >= -CULL_EPS) && (dB + sB + rr >= -CULL_EPS)) msk |= 1u << (8 + q);
                    }
                    if (b == 0) tm0 = msk; else tm1 = msk;
                }
            }
            // records beyond the budget (no culling data): every tile; none past ncand
            if (lane >= nrec && lane < ncand) tm0 = 0xffffu;
            if (lane + 32 >= nrec && lane + 32 < ncand) tm1 = 0xffffu;
        }
        int cnt = 0, sum_col = 0, sum_row = 0;
        __syncwarp();
        if (lane < 9) rws_s[wib][lane] = Rw[lane];  // (every lane holds the same pose)
        __syncwarp();
        // per-camera output planes (32-bit offsets inside one frame)
        float *depth_c = depth ? depth + c * (long long)H * W : nullptr;
        int32_t *seg_c = seg ? seg + c * (long long)H * W : nullptr;
        // an 8x8 tile per warp iteration, two pixels per lane (rows r and r+4):
        // the tile's culling and loop overhead is shared by 64 rays and each
        // candidate test runs two independent rays (ILP)
        int tx = part % tiles_x, ty = part / tiles_x;
        for (int tl = part; tl < n_tiles; tl += split) {
            const int i0 = ty * TH2, j0 = tx * TILE_W;
            const int j = j0 + (lane & 7);
            int ii[2] = {i0 + (lane >> 3), i0 + TILE_H + (lane >> 3)};
            // tile planes in CAMERA space through the pixel-centre rays of its border pixels
            float xl, xr, yt, yb, iL, iR, iT, iB;
            if (tpl) {
                const float4 pa = tpl_s[tl][0], pb = tpl_s[tl][1];
                xl = pa.x; xr = pa.y; yt = pa.z; yb = pa.w;
                iL = pb.x; iR = pb.y; iT = pb.z; iB = pb.w;
            } else {
                const int j1 = min(j0 + TILE_W - 1, W - 1), i1 = min(i0 + TH2 - 1, H - 1);
                xl = ((j0 + 0.5f) * sx - 1.0f) * cam.th; xr = ((j1 + 0.5f) * sx - 1.0f) * cam.th;
                yt = ((i0 + 0.5f) * sy - 1.0f) * cam.tv; yb = ((i1 + 0.5f) * sy - 1.0f) * cam.tv;
                iL = rsqrtf(1.f + xl * xl); iR = rsqrtf(1.f + xr * xr);
                iT = rsqrtf(1.f + yt * yt); iB = rsqrtf(1.f + yb * yb);
            }
#ifdef QB_CULL_STATS
            if (lane == 0) atomicAdd(&g_cull_stats[2], 1ull);
#endif
            if (S1) {  // consecutive tiles
                if (++tx == tiles_x) {
                    tx = 0;
                    ++ty;
                }
            } else {
                tx += split;
                while (tx >= tiles_x) {
                    tx -= tiles_x;
                    ++ty;
                }
            }
            const float x = ((j + 0.5f) * sx - 1.0f) * cam.th;
            // d = cz (x R0 + y R1 + R2) with R0..R2 the rotation's columns; the column
            // part x R0 + R2 is shared by the lane's two rays
            const float *Rs = rws_s[wib];
            const float ax = fmaf(x, Rs[0], Rs[2]), ay = fmaf(x, Rs[3], Rs[5]), az = fmaf(x, Rs[6], Rs[8]);
            float dx[2], dy[2], dz[2], ix[2], iy[2], iz[2], czv[2], tmx[2];
            // nearest hit so far as one key, (t bits) << 32 | object id: for t > 0 the
            // float bits order like t, so one unsigned min is "nearer, ties to the lower
            // id"; a miss (-1.0f) never wins; id INT_MAX: no hit yet
            unsigned long long bk[2];
            auto best_of = [&](int u) { return __uint_as_float((unsigned)(bk[u] >> 32)); };
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float y = ((ii[u] + 0.5f) * sy - 1.0f) * cam.tv;
                const float n2 = x * x + y * y + 1.0f;
                const float cz = rsqrtf(n2);
                dx[u] = cz * fmaf(y, Rs[1], ax);
                dy[u] = cz * fmaf(y, Rs[4], ay);
                dz[u] = cz * fmaf(y, Rs[7], az);
                ix[u] = rcp_approx(dx[u]);
                iy[u] = rcp_approx(dy[u]);
                iz[u] = rcp_approx(dz[u]);
                czv[u] = cz;
                tmx[u] = cam.max_range * (n2 * cz);  // max_range / cos(angle to the axis)
                bk[u] = ((unsigned long long)__float_as_uint(tmx[u]) << 32) | 0x7fffffffull;
            }
            for (int b = 0; b < ncand; b += 32) {
                const int k = b + lane;
                bool kp = false;
                if (EXACT && S1) {
                    const unsigned msk = b == 0 ? tm0 : (b == 32 ? tm1 : (k < ncand ? 0xffffu : 0u));
                    kp = ((msk >> (tl & 7)) & (msk >> (8 + (tl >> 3))) & 1u) != 0;
                } else if (k < ncand) {
                    if (k < CREC) {
                        // support = r + sum_k |n . A'_k|; L/R normals (+-1, 0, z), T/B (0, +-1, z)
                        const float rr = cul[0][k], ccx = cul[1][k], ccy = cul[2][k], ccz = cul[3][k];
                        const float a0x = cul[4][k], a0y = cul[5][k], a0z = cul[6][k];
                        const float a1x = cul[7][k], a1y = cul[8][k], a1z = cul[9][k];
                        const float a2x = cul[10][k], a2y = cul[11][k], a2z = cul[12][k];
                        const float dL = (ccx - xl * ccz) * iL,
                                    sL = (fabsf(a0x - xl * a0z) + fabsf(a1x - xl * a1z) + fabsf(a2x - xl * a2z)) * iL;
                        const float dR = (xr * ccz - ccx) * iR,
                                    sR = (fabsf(xr * a0z - a0x) + fabsf(xr * a1z - a1x) + fabsf(xr * a2z - a2x)) * iR;
                        const float dT = (ccy - yt * ccz) * iT,
                                    sT = (fabsf(a0y - yt * a0z) + fabsf(a1y - yt * a1z) + fabsf(a2y - yt * a2z)) * iT;
                        const float dB = (yb * ccz - ccy) * iB,
                                    sB = (fabsf(yb * a0z - a0y) + fabsf(yb * a1z - a1y) + fabsf(yb * a2z - a2y)) * iB;
                        kp = (dL + sL + rr >= -CULL_EPS) && (dR + sR + rr >= -CULL_EPS) && (dT + sT + rr >= -CULL_EPS) &&
                             (dB + sB + rr >= -CULL_EPS);
                    } else {
                        kp = true;  // beyond the record budget: no tile culling, generic test
                    }
                }
                unsigned m = __ballot_sync(FULL, kp);
                while (m) {
                    const int bit = __ffs(m) - 1;
                    m &= m - 1;
                    const int k2 = b + bit;
                    float t[2] = {-1.0f, -1.0f};
                    int oid;
#ifdef QB_CULL_STATS
                    if (lane == 0) {
                        const unsigned tw = k2 < CREC ? __float_as_uint(rec[k2][1].w) : 0u;
                        atomicAdd(&g_cull_stats[3 + ((tw & REC_SPHERE) ? 0 : (tw & REC_AABB) ? 1 : (tw & REC_OBB) ? 2 : 3)], 1ull);
                    }
#endif
                    int p = -1;  // generic: the primitive's own test
                    if (k2 < CREC) {
                        // both words at once: the flag (s1.w) selects the test, no dependent load
                        const float4 s0 = rec[k2][0], s1 = rec[k2][1];
                        const unsigned tw = __float_as_uint(s1.w);
                        oid = (int)(tw & REC_ID);
                        if (tw & REC_AABB) {
#pragma unroll
                            for (int u = 0; u < 2; ++u)
                                t[u] = slab_hit(s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, ix[u], iy[u], iz[u], tmin, best_of(u));
                        } else if (tw & REC_OBB) {
                            const float4 s2 = rec[k2][2], s3 = rec[k2][3];
                            // local direction = R^T d: columns (s2.x s2.y s2.z) (s2.w s3.x s3.y) (s3.z s3.w s1.z)
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const float lx = s2.x * dx[u] + s2.y * dy[u] + s2.z * dz[u];
                                const float ly = s2.w * dx[u] + s3.x * dy[u] + s3.y * dz[u];
                                const float lz = s3.z * dx[u] + s3.w * dy[u] + s1.z * dz[u];
                                t[u] = slab_hit(s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, rcp_approx(lx), rcp_approx(ly),
                                                rcp_approx(lz), tmin, best_of(u));
                            }
                        } else if (tw & REC_SPHERE) {
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const float bb = s0.x * dx[u] + s0.y * dy[u] + s0.z * dz[u];
                                const float fx = s0.x - bb * dx[u], fy = s0.y - bb * dy[u], fz = s0.z - bb * dz[u];
                                const float disc = s0.w - (fx * fx + fy * fy + fz * fz);
                                if (disc >= 0.0f) {
                                    const float sq = sqrtf(disc);
                                    const float ta = -bb - sq, tb = -bb + sq;
                                    // (a root beyond the nearest hit loses the key min below)
                                    t[u] = ta > tmin ? ta : (tb > tmin ? tb : -1.0f);
                                }
                            }
                        } else {
                            p = __float_as_int(s1.x);
                        }
                    } else {
                        p = cand[k2];
                    }
                    if (p >= 0) {  // triangles, records beyond the budget, ids too large for the word
                        // triangle shear axis of the tile, warp-uniform (see k_render_f); taken
                        // here, where every lane is (this branch depends on the survivor only)
                        const int kz = __shfl_sync(FULL, dominant_axis(dx[0], dy[0], dz[0]), 12);
                        const int2 mt = __ldg(S.meta + p);
                        oid = mt.y;
                        const float4 *pr = S.primf + 4 * p;
#pragma unroll
                        for (int u = 0; u < 2; ++u)
                            t[u] = mt.x == QB_SPHERE ? ray_sphere_f(pr, o[0], o[1], o[2], dx[u], dy[u], dz[u], tmin, best_of(u))
                                   : mt.x == QB_BOX  ? ray_box_f(pr, o[0], o[1], o[2], dx[u], dy[u], dz[u], tmin, best_of(u))
                                                     : ray_triangle_call(kz, pr, o[0], o[1], o[2], dx[u], dy[u], dz[u], tmin, best_of(u));
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        // tests return t <= best; ties go to the lowest object id
                        bk[u] = min(bk[u], ((unsigned long long)__float_as_uint(t[u]) << 32) | (unsigned)oid);
                }
            }
            float tt[2];
            int to[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const bool hit = (unsigned)bk[u] != 0x7fffffffu;
                tt[u] = hit ? best_of(u) : -1.0f;
                to[u] = hit ? (int)(unsigned)bk[u] : -1;
            }
            // swarm agents as spheres after the scene (kernels.py:438-445): a
            // sphere replaces the scene hit only when strictly nearer
            auto sphere_test = [&](int k) {
                const float4 sph = *reinterpret_cast<const float4 *>(extra + (c * n_extra + k) * 4);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float ts = ray_sphere_v(sph, sph.w * sph.w, o[0], o[1], o[2], dx[u], dy[u], dz[u], tmin, tmx[u]);
                    if (ts > 0.0f && (tt[u] < 0.0f || ts < tt[u])) {
                        tt[u] = ts;
                        to[u] = extra_ids[c * n_extra + k];
                    }
                }
            };
            if (!EXTRA) {
            } else if (x_all) {
                for (int k = 0; k < n_extra; ++k) sphere_test(k);
            } else if (nx > 0) {  // tile-cull the frustum survivors (sphere support = r), ascending k
                const float4 sp = xcs_s[wib][lane < nx ? lane : 0];
                const bool tin = lane < nx && (sp.x - xl * sp.z) * iL + sp.w >= -CULL_EPS &&
                                 (xr * sp.z - sp.x) * iR + sp.w >= -CULL_EPS && (sp.y - yt * sp.z) * iT + sp.w >= -CULL_EPS &&
                                 (yb * sp.z - sp.y) * iB + sp.w >= -CULL_EPS;
                for (unsigned m = __ballot_sync(FULL, tin); m; m &= m - 1) sphere_test(xk_s[wib][__ffs(m) - 1]);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = ii[u];
                const float t = tt[u];
                const int oid = to[u];
                const int out_id = t > 0.0f ? oid : 0;
                if (EXACT || (j < W && i < H)) {
                    const int off = i * W + j;
                    if (EXACT || depth_c) depth_c[off] = t > 0.0f ? t * czv[u] : cam.max_range;
                    if (EXACT ? SEGP : seg_c != nullptr) seg_c[off] = out_id;
                    if (CENT && out_id == centroid_id) {
                        cnt += 1;
                        sum_col += j;
                        sum_row += i;
                    }
                }
            }
        }
        if (CENT && split == 1) {
#pragma unroll
            for (int s2 = 16; s2 > 0; s2 >>= 1) {
                cnt += __shfl_xor_sync(FULL, cnt, s2);
                sum_col += __shfl_xor_sync(FULL, sum_col, s2);
                sum_row += __shfl_xor_sync(FULL, sum_row, s2);
            }
            if (lane == 0) {
                centroid[2 * c] = cnt ? (float)((double)sum_col / (double)cnt) : -1.0f;
                centroid[2 * c + 1] = cnt ? (float)((double)sum_row / (double)cnt) : -1.0f;
            }
        }
        __syncwarp();
        if (S1 && claim) {
            long long nx = 0;
            if (lane == 0) nx = (long long)atomicAdd(claim, 1u) + nwarps;
            wi = __shfl_sync(FULL, nx, 0);
        } else {
            wi += nwarps;
        }
    }
}

// exact-double validation renderer: one thread per pixel, reference order
template <bool FROM_STATE>
__global__ void __launch_bounds__(128) k_render_x(DevScene S, CamD cam, long long n, long long ld, const double *state,
                                                  const double *origins, const double *rotations,
                                                  const int32_t *env_scene, double *depth, int32_t *seg,
                                                  int centroid_id, float *centroid, const double *extra,
                                                  const int32_t *extra_ids, int n_extra) {
    const long long pix = (long long)cam.W * cam.H;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n * pix) return;
    const long long c = gid / pix;
    const int i = (int)((gid % pix) / cam.W), j = (int)(gid % cam.W);
    xd o[3], Rw[9];
    if (FROM_STATE) {
        xd p[3] = {xd(state[0 * ld + c]), xd(state[1 * ld + c]), xd(state[2 * ld + c])};
        xd q[4] = {xd(state[6 * ld + c]), xd(state[7 * ld + c]), xd(state[8 * ld + c]), xd(state[9 * ld + c])};
        xd cr[9], ct[3];
        for (int k = 0; k < 9; ++k) cr[k] = xd(cam.rot[k]);
        for (int k = 0; k < 3; ++k) ct[k] = xd(cam.trans[k]);
        camera_pose<xd>(p, q, cr, ct, o, Rw);
    } else {
        for (int k = 0; k < 3; ++k) o[k] = xd(origins[3 * c + k]);
        for (int k = 0; k < 9; ++k) Rw[k] = xd(rotations[9 * c + k]);
    }
    // kernels.py:423-437
    xd y = (xd(2.0) * (xd((double)i) + xd(0.5)) / xd((double)cam.H) - xd(1.0)) * xd(cam.tv);
    xd x = (xd(2.0) * (xd((double)j) + xd(0.5)) / xd((double)cam.W) - xd(1.0)) * xd(cam.th);
    xd norm = r_sqrt(x * x + y * y + xd(1.0));
    xd cz = xd(1.0) / norm;
    xd cx = x * cz, cy = y * cz;
    xd dx = Rw[0] * cx + Rw[1] * cy + Rw[2] * cz;
    xd dy = Rw[3] * cx + Rw[4] * cy + Rw[5] * cz;
    xd dz = Rw[6] * cx + Rw[7] * cy + Rw[8] * cz;
    xd tmax = xd(cam.max_range) / cz;
    int oid;
    double t = raycast_x(S, env_scene ? env_scene[c] : 0, o[0].v, o[1].v, o[2].v, dx.v, dy.v, dz.v, 1e-9, tmax.v, oid);
    for (int k = 0; k < n_extra; ++k) {  // swarm agents as spheres (kernels.py:438-445)
        const double *sp = extra + (c * n_extra + k) * 4;
        const xd ts = ray_sphere_ref<xd>(xd(sp[0]), xd(sp[1]), xd(sp[2]), xd(sp[3]), o[0], o[1], o[2], dx, dy, dz,
                                         xd(1e-9), tmax);
        if (ts.v > 0.0 && (t < 0.0 || ts.v < t)) {
            t = ts.v;
            oid = extra_ids[c * n_extra + k];
        }
    }
    const long long off = c * pix + (long long)i * cam.W + j;
    if (depth) depth[off] = t > 0.0 ? (xd(t) * cz).v : cam.max_range;
    if (seg) seg[off] = t > 0.0 ? oid : 0;
    (void)centroid_id;
    (void)centroid;
}

// centroid pass for the validation renderer (reads back its own seg)
__global__ void k_centroid(long long n, int W, int H, const int32_t *seg, int id, float *centroid) {
    long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    long long cnt = 0, sc = 0, sr = 0;
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j)
            if (seg[(c * H + i) * (long long)W + j] == id) {
                ++cnt;
                sc += j;
                sr += i;
            }
    centroid[2 * c] = cnt ? (float)((double)sc / (double)cnt) : -1.0f;
    centroid[2 * c + 1] = cnt ? (float)((double)sr / (double)cnt) : -1.0f;
}

__global__ void k_nearest(DevScene S, const int32_t *env_scene, long long n, const double *q, double *pt, double *dist,
                          int32_t *oid, double *dist2) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    NearestResult r = nearest_point(S, env_scene ? env_scene[i] : 0, q[3 * i], q[3 * i + 1], q[3 * i + 2]);
    if (pt) {
        pt[3 * i] = r.px;
        pt[3 * i + 1] = r.py;
        pt[3 * i + 2] = r.pz;
    }
    if (dist) dist[i] = __dsqrt_rn(r.d2);
    if (dist2) dist2[i] = r.d2;
    if (oid) oid[i] = r.oid;
}

template <class S_>
__global__ void k_raycast(DevScene S, const int32_t *env_scene, long long n, const S_ *o, const S_ *d, double tmin,
                          double tmax, S_ *t, int32_t *oid) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int id;
    int sc = env_scene ? env_scene[i] : 0;
    if constexpr (sizeof(S_) == 4) {
        t[i] = raycast_f(S, sc, o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], (float)tmin,
                         (float)tmax, id);
    } else {
        t[i] = raycast_x(S, sc, o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], tmin, tmax, id);
    }
    if (oid) oid[i] = id;
}

}  // namespace

namespace {
struct CullLaunch {
    const qb_scene *s;
    CamF c;
    long long n, ld;
    const float *state, *origins, *rotations;
    const int32_t *env_scene;
    float *depth;
    int32_t *seg;
    int centroid_id;
    float *centroid;
    const float *extra;
    const int32_t *extra_ids;
    int n_extra, split, blocks, B;
    cudaStream_t st;
    bool exact;
};

// the claim counter of a stream (host side: a small stream -> slot table)
unsigned int *claim_counter(cudaStream_t st) {
    static std::mutex mu;
    static cudaStream_t keys[QB_CULL_SLOTS];
    static int used = 0;
    int slot = -1;
    {
        std::lock_guard<std::mutex> lock(mu);
        for (int i = 0; i < used; ++i)
            if (keys[i] == st) slot = i;
        if (slot < 0) {
            if (used == QB_CULL_SLOTS) return nullptr;  // (static striding: a shared counter would race)
            slot = used++;
            keys[slot] = st;
        }
    }
    // the array's address on the current device, looked up once per device (also
    // keeps the lookup out of stream captures after the first launch)
    static void *base_of[64] = {nullptr};
    int dev = 0;
    cudaGetDevice(&dev);
    void *base = dev < 64 ? base_of[dev] : nullptr;
    if (!base) {
        if (cudaGetSymbolAddress(&base, g_cull_next) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;  // (static striding)
        }
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 64) base_of[dev] = base;
    }
    return static_cast<unsigned int *>(base) + slot;
}

template <bool FS, bool EX, bool CE, bool EXACT, bool S1, bool SEGP> void cull_kernel(const CullLaunch &L) {
    unsigned int *claim = nullptr;
    if (S1) {
        // not inside a stream capture: a graph replays on any stream, possibly
        // beside a direct launch that uses the same stream's counter
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(L.st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone)
            claim = claim_counter(L.st);
        cudaGetLastError();
        if (claim && cudaMemsetAsync(claim, 0, sizeof(unsigned int), L.st) != cudaSuccess) {
            cudaGetLastError();
            claim = nullptr;
        }
    }
    k_render_cull<FS, EX, CE, EXACT, S1, SEGP><<<L.blocks, L.B, 0, L.st>>>(
        L.s->dev, L.c, L.n, L.ld, FS ? L.state : nullptr, FS ? nullptr : L.origins, FS ? nullptr : L.rotations,
        L.env_scene, L.depth, L.seg, FS ? L.centroid_id : 0, FS ? L.centroid : nullptr, L.extra, L.extra_ids, L.n_extra,
        L.split, claim);
}

// compile-time variants: 64x64 frames (EXACT) with / without segmentation, split == 1
template <bool FS, bool EX, bool CE> void launch_cull(const CullLaunch &L) {
    if (L.exact && L.split == 1) {
        if (L.seg) cull_kernel<FS, EX, CE, true, true, true>(L);
        else cull_kernel<FS, EX, false, true, true, false>(L);
    } else if (L.exact) {
        if (L.seg) cull_kernel<FS, EX, CE, true, false, true>(L);
        else cull_kernel<FS, EX, false, true, false, false>(L);
    } else {
        cull_kernel<FS, EX, CE, false, false, true>(L);
    }
}
}  // namespace

namespace qb {

int launch_render(const qb_scene *s, const qb_camera *cam, int dtype, long long n, long long ld, const void *state,
                  const void *origins, const void *rotations, const int32_t *env_scene, void *depth, int32_t *seg,
                  int32_t centroid_id, float *centroid, const void *extra, const int32_t *extra_ids, int n_extra,
                  cudaStream_t st) {
    if (n == 0) return QB_OK;
    if (dtype == QB_F32) {
        CamF c;
        c.W = cam->width;
        c.H = cam->height;
        c.th = (float)cam->tan_half_h;
        c.tv = (float)cam->tan_half_v;
        c.max_range = (float)cam->max_range;
        for (int k = 0; k < 9; ++k) c.rot[k] = (float)cam->rotation[k];
        for (int k = 0; k < 3; ++k) c.trans[k] = (float)cam->translation[k];
        const int mode = cam->mode != 0 ? cam->mode : (s->max_scene_prims <= CULL_MAX ? 2 : 1);
        if (mode == 2) {
            if (s->max_scene_prims > CULL_MAX) {
                set_error("culling renderer supports scenes of <= %d primitives", CULL_MAX);
                return QB_EINVAL;
            }
            const int B = CULL_WARPS * 32;
            // fill the machine: ~24 resident warps per SM; small batches split a
            // camera's tiles across warps (the per-camera culling is repeated)
            const long long want = (long long)sm_count() * 24;
            const int tiles = ((c.H + 2 * TILE_H - 1) / (2 * TILE_H)) * ((c.W + TILE_W - 1) / TILE_W);
            int split = (int)std::min<long long>(tiles / 2 > 0 ? tiles / 2 : 1, std::max<long long>(1, want / std::max(n, 1LL)));
            if (split < 1) split = 1;
            if (split > 1 && !seg && centroid_id > 0) split = 1;  // centroid pass reads seg
            long long blocks = (n * split + CULL_WARPS - 1) / CULL_WARPS;
            long long max_blocks = (long long)sm_count() * 16;
            if (blocks > max_blocks) blocks = max_blocks;
            const bool cent = state && centroid_id > 0 && split == 1;  // inline centroid (else the k_centroid pass)
            const bool exact = depth && c.W == 64 && c.H == 64;
            const CullLaunch L{s, c, n, ld, (const float *)state, (const float *)origins, (const float *)rotations,
                               env_scene, (float *)depth, seg, centroid_id, centroid, (const float *)extra, extra_ids,
                               n_extra, split, (int)blocks, B, st, exact};
            if (state) {
                if (n_extra > 0) {
                    if (cent) launch_cull<true, true, true>(L); else launch_cull<true, true, false>(L);
                } else {
                    if (cent) launch_cull<true, false, true>(L); else launch_cull<true, false, false>(L);
                }
            } else {
                if (n_extra > 0) launch_cull<false, true, false>(L); else launch_cull<false, false, false>(L);
            }
            int rc = check_launch("render_cull_f32");
            if (rc || split == 1 || centroid_id <= 0) return rc;
            k_centroid<<<env_grid(n, 128), 128, 0, st>>>(n, c.W, c.H, seg, centroid_id, centroid);
            return check_launch("centroid");
        }
        const int B = QB_RF_BLOCK;
        // small batches split a camera's tiles over warps (one warp renders a
        // 64x64 frame in ~1 ms: 128 tiles in sequence) up to ~48 warps per SM
#ifndef QB_RF_WANT
#define QB_RF_WANT 48
#endif
#ifndef QB_RF_TPW
#define QB_RF_TPW 2
#endif
        const long long want = (long long)sm_count() * QB_RF_WANT;
        const int tiles = ((c.W + TILE_W - 1) / TILE_W) * ((c.H + TILE_H - 1) / TILE_H);
        int split = (int)std::min<long long>(std::max(tiles / QB_RF_TPW, 1), std::max<long long>(1, want / std::max(n, 1LL)));
        if (split > 1 && !seg && centroid_id > 0) split = 1;  // the centroid pass reads seg
        long long blocks = (n * split * 32 + B - 1) / B;
        if (blocks > 0x7fffffffLL) blocks = 0x7fffffffLL;  // grid-stride loop covers the rest
        const bool exact = state && depth && n_extra == 0 && c.W == 64 && c.H == 64;
        if (exact) {
#define QB_RF_X(CE, S1_, SG)                                                                                          \
    k_render_f<true, true, CE, S1_, SG><<<(int)blocks, B, 0, st>>>(s->dev, c, n, ld, (const float *)state, nullptr,     \
                                                                    nullptr, env_scene, (float *)depth, seg,          \
                                                                    centroid_id, centroid, nullptr, nullptr, 0, split)
            const bool ce = centroid_id > 0 && seg;
            if (!seg) {
                if (split == 1) QB_RF_X(false, true, false); else QB_RF_X(false, false, false);
            } else if (split == 1) {
                if (ce) QB_RF_X(true, true, true); else QB_RF_X(false, true, true);
            } else {
                if (ce) QB_RF_X(true, false, true); else QB_RF_X(false, false, true);
            }
#undef QB_RF_X
        } else if (state)
            k_render_f<true><<<(int)blocks, B, 0, st>>>(s->dev, c, n, ld, (const float *)state, nullptr, nullptr, env_scene,
                                                        (float *)depth, seg, centroid_id, centroid, (const float *)extra,
                                                        extra_ids, n_extra, split);
        else
            k_render_f<false><<<(int)blocks, B, 0, st>>>(s->dev, c, n, ld, nullptr, (const float *)origins,
                                                         (const float *)rotations, env_scene, (float *)depth, seg, 0, nullptr,
                                                         (const float *)extra, extra_ids, n_extra, split);
        int rc = check_launch("render_f32");
        if (rc || split == 1 || centroid_id <= 0 || !state) return rc;
        k_centroid<<<env_grid(n, 128), 128, 0, st>>>(n, c.W, c.H, seg, centroid_id, centroid);
        return check_launch("centroid");
    }
    CamD c;
    c.W = cam->width;
    c.H = cam->height;
    c.th = cam->tan_half_h;
    c.tv = cam->tan_half_v;
    c.max_range = cam->max_range;
    for (int k = 0; k < 9; ++k) c.rot[k] = cam->rotation[k];
    for (int k = 0; k < 3; ++k) c.trans[k] = cam->translation[k];
    long long total = n * (long long)c.W * c.H;
    const int B = 128;
    int blocks = (int)((total + B - 1) / B);
    if (state)
        k_render_x<true><<<blocks, B, 0, st>>>(s->dev, c, n, ld, (const double *)state, nullptr, nullptr, env_scene,
                                              (double *)depth, seg, centroid_id, centroid, (const double *)extra,
                                              extra_ids, n_extra);
    else
        k_render_x<false><<<blocks, B, 0, st>>>(s->dev, c, n, ld, nullptr, (const double *)origins,
                                               (const double *)rotations, env_scene, (double *)depth, seg, 0, nullptr,
                                               (const double *)extra, extra_ids, n_extra);
    int rc = check_launch("render_f64");
    if (rc) return rc;
    if (centroid_id > 0) {
        if (!seg) {
            set_error("centroid needs a seg buffer in the FP64 renderer");
            return QB_EINVAL;
        }
        k_centroid<<<env_grid(n, 128), 128, 0, st>>>(n, c.W, c.H, seg, centroid_id, centroid);
        return check_launch("centroid");
    }
    return QB_OK;
}

int launch_nearest(const qb_scene *s, const int32_t *env_scene, long long n, const double *q, double *pt, double *dist,
                   int32_t *oid, double *dist2, cudaStream_t st) {
    if (n == 0) return QB_OK;
    k_nearest<<<env_grid(n, 128), 128, 0, st>>>(s->dev, env_scene, n, q, pt, dist, oid, dist2);
    return check_launch("nearest_point");
}

int launch_raycast(const qb_scene *s, int dtype, const int32_t *env_scene, long long n, const void *o, const void *d,
                   double tmin, double tmax, void *t, int32_t *oid, cudaStream_t st) {
    if (n == 0) return QB_OK;
    if (dtype == QB_F32)
        k_raycast<float><<<env_grid(n, 128), 128, 0, st>>>(s->dev, env_scene, n, (const float *)o, (const float *)d, tmin,
                                                           tmax, (float *)t, oid);
    else
        k_raycast<double><<<env_grid(n, 128), 128, 0, st>>>(s->dev, env_scene, n, (const double *)o, (const double *)d,
                                                            tmin, tmax, (double *)t, oid);
    return check_launch("raycast");
}

}  // namespace qb

#ifdef QB_RF_DEBUG
extern "C" int qb_dbg_set(int cam, int i, int j) {
    int t[3] = {cam, i, j}, z = 0;
    cudaMemcpyToSymbol(g_dbg_target, t, sizeof(t));
    cudaMemcpyToSymbol(g_dbg_n, &z, sizeof(z));
    return 0;
}
extern "C" int qb_dbg_get(float4 *out, int *n) {
    cudaMemcpyFromSymbol(n, g_dbg_n, sizeof(int));
    cudaMemcpyFromSymbol(out, g_dbg_log, sizeof(float4) * 8192);
    return 0;
}
#endif
