// qb_geometry.cuh -- device scene layout + primitive queries (K2/K3 inner
// loops), templated on the scalar policy.
//
// Reference map (geometry/kernels.py):
//   closest_on_sphere / box / triangle   :18-109
//   aabb_dist2, nearest_point_query      :112-182
//   ray_sphere / ray_box / ray_triangle  :185-285
//   ray_aabb_enter, raycast_core         :288-386
//
// Result semantics are traversal-order independent (nearest t, ties to the
// lowest object id; nearest d^2, ties to the lowest id), so the BVH here is
// our own binned-SAH tree (qb_bvh.cpp), not the reference's median split.
#pragma once
#include "qb_real.cuh"

enum { QB_SPHERE = 0, QB_BOX = 1, QB_TRIANGLE = 2 };

// One scene set = S scenes, each with its own BVH root, all arrays
// concatenated.  Leaf primitives are stored contiguously in BVH order.
struct DevScene {
    int n_scenes;
    int n_prims;
    const int *root;        // [S]
    const double *bounds;   // [S][6] raw primitive bounds lo.xyz hi.xyz (shapes.py:214-217)
    const float4 *nodef;    // [M][2] (lo.xyz, a) (hi.xyz, b) -- float, bounds rounded outward
    const double *noded;    // [M][6] lo.xyz hi.xyz (exact double)
    const int2 *nodei;      // [M] (a, b): b>0 leaf {first=a,count=b}; b<=0 internal {left=a, axis=-b}
    const float4 *primf;    // [P][4] float prim records (see qb_abi.cu pack_prim)
    const double *primd;    // [P][16] reference prim_data rows
    const int2 *meta;       // [P] (type, object id)
    const int *prim_offset; // [S+1] first primitive of each scene (BVH order)
    const float4 *primc;    // [P][4] culling bounds: (centre, r) (A0, 0) (A1, 0) (A2, 0);
                            // support along unit n = r + sum_k |n . A_k| (A_k = box half-axes)
    int tri_only;           // every primitive is a triangle (meshes: no per-primitive type dispatch)
};

#ifdef __CUDACC__

// ------------------------------------------------------------- closest point
template <class R> struct V3 {
    R x, y, z;
};

// kernels.py:18-26
template <class R> QB_D V3<R> closest_on_sphere(R cx, R cy, R cz, R r, R qx, R qy, R qz) {
    R dx = qx - cx, dy = qy - cy, dz = qz - cz;
    R n = r_sqrt(dx * dx + dy * dy + dz * dz);
    if (n < R(1e-300)) return {cx + r, cy, cz};
    R s = r / n;
    return {cx + dx * s, cy + dy * s, cz + dz * s};
}

// kernels.py:29-58
template <class R> QB_D V3<R> closest_on_box(const R *d, R qx, R qy, R qz) {
    R cx = d[0], cy = d[1], cz = d[2], hx = d[3], hy = d[4], hz = d[5];
    R dx = qx - cx, dy = qy - cy, dz = qz - cz;
    R lx = d[6] * dx + d[9] * dy + d[12] * dz;
    R ly = d[7] * dx + d[10] * dy + d[13] * dz;
    R lz = d[8] * dx + d[11] * dy + d[14] * dz;
    R px = py_min(py_max(lx, -hx), hx), py = py_min(py_max(ly, -hy), hy), pz = py_min(py_max(lz, -hz), hz);
    if (px == lx && py == ly && pz == lz) {  // interior: nearest face
        R gx = hx - r_abs(lx), gy = hy - r_abs(ly), gz = hz - r_abs(lz);
        if (gx <= gy && gx <= gz)
            px = lx >= R(0.0) ? hx : -hx;
        else if (gy <= gz)
            py = ly >= R(0.0) ? hy : -hy;
        else
            pz = lz >= R(0.0) ? hz : -hz;
    }
    return {d[6] * px + d[7] * py + d[8] * pz + cx, d[9] * px + d[10] * py + d[11] * pz + cy,
            d[12] * px + d[13] * py + d[14] * pz + cz};
}

// kernels.py:61-99 (Ericson 5.1.5)
template <class R> QB_D V3<R> closest_on_triangle(const R *d, R px, R py, R pz) {
    R ax = d[0], ay = d[1], az = d[2], bx = d[3], by = d[4], bz = d[5], cx = d[6], cy = d[7], cz = d[8];
    R abx = bx - ax, aby = by - ay, abz = bz - az;
    R acx = cx - ax, acy = cy - ay, acz = cz - az;
    R apx = px - ax, apy = py - ay, apz = pz - az;
    R d1 = abx * apx + aby * apy + abz * apz;
    R d2 = acx * apx + acy * apy + acz * apz;
    if (d1 <= R(0.0) && d2 <= R(0.0)) return {ax, ay, az};
    R bpx = px - bx, bpy = py - by, bpz = pz - bz;
    R d3 = abx * bpx + aby * bpy + abz * bpz;
    R d4 = acx * bpx + acy * bpy + acz * bpz;
    if (d3 >= R(0.0) && d4 <= d3) return {bx, by, bz};
    R vc = d1 * d4 - d3 * d2;
    if (vc <= R(0.0) && d1 >= R(0.0) && d3 <= R(0.0)) {
        R v = d1 / (d1 - d3);
        return {ax + v * abx, ay + v * aby, az + v * abz};
    }
    R cpx = px - cx, cpy = py - cy, cpz = pz - cz;
    R d5 = abx * cpx + aby * cpy + abz * cpz;
    R d6 = acx * cpx + acy * cpy + acz * cpz;
    if (d6 >= R(0.0) && d5 <= d6) return {cx, cy, cz};
    R vb = d5 * d2 - d1 * d6;
    if (vb <= R(0.0) && d2 >= R(0.0) && d6 <= R(0.0)) {
        R w = d2 / (d2 - d6);
        return {ax + w * acx, ay + w * acy, az + w * acz};
    }
    R va = d3 * d6 - d5 * d4;
    if (va <= R(0.0) && (d4 - d3) >= R(0.0) && (d5 - d6) >= R(0.0)) {
        R w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return {bx + w * (cx - bx), by + w * (cy - by), bz + w * (cz - bz)};
    }
    R denom = R(1.0) / (va + vb + vc);
    R v = vb * denom, w = vc * denom;
    return {ax + abx * v + acx * w, ay + aby * v + acy * w, az + abz * v + acz * w};
}

// kernels.py:112-117
template <class R> QB_D R aabb_dist2(const double *b, R qx, R qy, R qz) {
    R dx = py_max(py_max(R(b[0]) - qx, R(0.0)), qx - R(b[3]));
    R dy = py_max(py_max(R(b[1]) - qy, R(0.0)), qy - R(b[4]));
    R dz = py_max(py_max(R(b[2]) - qz, R(0.0)), qz - R(b[5]));
    return dx * dx + dy * dy + dz * dz;
}

struct NearestResult {
    double px, py, pz, d2;
    int oid;
};

// kernels.py:120-182 in exact double over the double BVH of one scene.
// Result is the global minimum of d^2 (ties -> lowest id) like the reference.
QB_D NearestResult nearest_point(const DevScene &S, int scene, double qx_, double qy_, double qz_) {
    xd qx(qx_), qy(qy_), qz(qz_);
    int stack[64];
    int top = 0;
    stack[top++] = S.root[scene];
    xd best(infinity_d());
    int best_id = -1;
    xd bx(0.0), by(0.0), bz(0.0);
    while (top > 0) {
        int node = stack[--top];
        xd d2 = aabb_dist2<xd>(S.noded + 6 * node, qx, qy, qz);
        if (d2 > best) continue;
        int2 ni = S.nodei[node];
        if (ni.y > 0) {
            for (int p = ni.x; p < ni.x + ni.y; ++p) {
                int2 m = S.meta[p];
                const double *dd = S.primd + 16 * p;
                xd d[15];
#pragma unroll
                for (int k = 0; k < 15; ++k) d[k] = xd(dd[k]);
                V3<xd> c;
                if (m.x == QB_SPHERE)
                    c = closest_on_sphere<xd>(d[0], d[1], d[2], d[3], qx, qy, qz);
                else if (m.x == QB_BOX)
                    c = closest_on_box<xd>(d, qx, qy, qz);
                else
                    c = closest_on_triangle<xd>(d, qx, qy, qz);
                xd ex = qx - c.x, ey = qy - c.y, ez = qz - c.z;
                xd pd2 = ex * ex + ey * ey + ez * ez;
                if (pd2 < best || (pd2 == best && m.y < best_id)) {
                    best = pd2;
                    best_id = m.y;
                    bx = c.x; by = c.y; bz = c.z;
                }
            }
        } else {
            int l = ni.x, r = l + 1;
            xd dl = aabb_dist2<xd>(S.noded + 6 * l, qx, qy, qz);
            xd dr = aabb_dist2<xd>(S.noded + 6 * r, qx, qy, qz);
            if (dl <= dr) {
                if (dr <= best) stack[top++] = r;
                if (dl <= best) stack[top++] = l;
            } else {
                if (dl <= best) stack[top++] = l;
                if (dr <= best) stack[top++] = r;
            }
        }
    }
    return {bx.v, by.v, bz.v, best.v, best_id};
}

// Per-thread nearest point for tiny scenes (<= NEAREST_SCAN_MAX primitives,
// e.g. the 6-box garage): a straight scan in primitive order with the same
// (d2, lowest id, first primitive) result as the BVH walk, without its
// local-memory stack and node tests.
//
// Boxes whose rotation is exactly the identity (flagged by the packer) take
// closest_on_box with its products by 1 and by +0 written out: 1*a == a and
// 0*b == copysign(0, b) for finite b, so every sum sees the same operands and
// the result has the same bits (signed zeros included) without the 18
// rotation products and 9 loads; non-finite queries take the general form.
constexpr int NEAREST_SCAN_MAX = 16;
QB_D V3<xd> closest_on_aabb(const double *dd, xd qx, xd qy, xd qz) {
    const xd cx(__ldg(dd)), cy(__ldg(dd + 1)), cz(__ldg(dd + 2)), hx(__ldg(dd + 3)), hy(__ldg(dd + 4)), hz(__ldg(dd + 5));
    const xd dx = qx - cx, dy = qy - cy, dz = qz - cz;
    auto z = [](xd b) { return xd(copysign(0.0, b.v)); };  // +0 * b
    // lx = d6*dx + d9*dy + d12*dz with (d6, d9, d12) = (1, 0, 0), etc.
    const xd lx = (dx + z(dy)) + z(dz), ly = (z(dx) + dy) + z(dz), lz = (z(dx) + z(dy)) + dz;
    xd px = py_min(py_max(lx, -hx), hx), py = py_min(py_max(ly, -hy), hy), pz = py_min(py_max(lz, -hz), hz);
    if (px == lx && py == ly && pz == lz) {  // interior: nearest face
        const xd gx = hx - r_abs(lx), gy = hy - r_abs(ly), gz = hz - r_abs(lz);
        if (gx <= gy && gx <= gz)
            px = lx >= xd(0.0) ? hx : -hx;
        else if (gy <= gz)
            py = ly >= xd(0.0) ? hy : -hy;
        else
            pz = lz >= xd(0.0) ? hz : -hz;
    }
    // (d6*px + d7*py + d8*pz) + cx with (d6, d7, d8) = (1, 0, 0), etc.
    return {((px + z(py)) + z(pz)) + cx, ((z(px) + py) + z(pz)) + cy, ((z(px) + z(py)) + pz) + cz};
}

QB_D NearestResult nearest_point_scan(const DevScene &S, int p0, int p1, double qx_, double qy_, double qz_) {
    xd qx(qx_), qy(qy_), qz(qz_);
    const bool finite_q = isfinite(qx_) && isfinite(qy_) && isfinite(qz_);
    double best = infinity_d();
    int best_id = -1;
    double bx = 0.0, by = 0.0, bz = 0.0;
    for (int p = p0; p < p1; ++p) {
        const int2 m = __ldg(S.meta + p);
        const double *dd = S.primd + 16 * p;
        V3<xd> c;
        if (m.x == QB_BOX && finite_q && __ldg(&S.primf[4 * p + 3].w) != 0.0f) {
            c = closest_on_aabb(dd, qx, qy, qz);
        } else {
            xd d[15];
#pragma unroll
            for (int k = 0; k < 15; ++k) d[k] = xd(__ldg(dd + k));
            if (m.x == QB_SPHERE)
                c = closest_on_sphere<xd>(d[0], d[1], d[2], d[3], qx, qy, qz);
            else if (m.x == QB_BOX)
                c = closest_on_box<xd>(d, qx, qy, qz);
            else
                c = closest_on_triangle<xd>(d, qx, qy, qz);
        }
        xd ex = qx - c.x, ey = qy - c.y, ez = qz - c.z;
        const double pd2 = (ex * ex + ey * ey + ez * ez).v;
        if (pd2 < best || (pd2 == best && m.y < best_id)) {
            best = pd2;
            best_id = m.y;
            bx = c.x.v; by = c.y.v; bz = c.z.v;
        }
    }
    return {bx, by, bz, best, best_id};
}

// Warp-cooperative nearest point for small scenes (<= NEAREST_BRUTE_MAX
// primitives): the 32 lanes split the scene's primitives, each keeps its best
// (d2, object id, primitive) and a shuffle argmin picks the winner -- the same
// (d2, lowest id) result as the BVH walk above (which prunes only strictly
// farther boxes), at the latency of a few primitive tests instead of a
// dependent traversal.  All 32 lanes must call it with the same query; larger
// scenes fall back to the BVH walk in every lane.
constexpr int NEAREST_BRUTE_MAX = 1024;
QB_D NearestResult nearest_point_warp(const DevScene &S, int scene, double qx_, double qy_, double qz_) {
    const int p0 = S.prim_offset[scene], p1 = S.prim_offset[scene + 1];
    if (p1 - p0 > NEAREST_BRUTE_MAX) return nearest_point(S, scene, qx_, qy_, qz_);
    const unsigned FULLM = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    xd qx(qx_), qy(qy_), qz(qz_);
    double best = infinity_d();
    int best_id = 0x7fffffff, best_p = 0x7fffffff;
    double bx = 0.0, by = 0.0, bz = 0.0;
    for (int p = p0 + lane; p < p1; p += 32) {
        const int2 m = S.meta[p];
        const double *dd = S.primd + 16 * p;
        xd d[15];
#pragma unroll
        for (int k = 0; k < 15; ++k) d[k] = xd(dd[k]);
        V3<xd> c;
        if (m.x == QB_SPHERE)
            c = closest_on_sphere<xd>(d[0], d[1], d[2], d[3], qx, qy, qz);
        else if (m.x == QB_BOX)
            c = closest_on_box<xd>(d, qx, qy, qz);
        else
            c = closest_on_triangle<xd>(d, qx, qy, qz);
        xd ex = qx - c.x, ey = qy - c.y, ez = qz - c.z;
        const double pd2 = (ex * ex + ey * ey + ez * ez).v;
        if (pd2 < best || (pd2 == best && m.y < best_id)) {  // p ascends per lane
            best = pd2;
            best_id = m.y;
            best_p = p;
            bx = c.x.v; by = c.y.v; bz = c.z.v;
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const double od = __shfl_xor_sync(FULLM, best, s);
        const int oi = __shfl_xor_sync(FULLM, best_id, s), op = __shfl_xor_sync(FULLM, best_p, s);
        if (od < best || (od == best && (oi < best_id || (oi == best_id && op < best_p)))) {
            best = od;
            best_id = oi;
            best_p = op;
        }
    }
    const int owner = best_p == 0x7fffffff ? 0 : (best_p - p0) & 31;
    bx = __shfl_sync(FULLM, bx, owner);
    by = __shfl_sync(FULLM, by, owner);
    bz = __shfl_sync(FULLM, bz, owner);
    if (best_id == 0x7fffffff) return {0.0, 0.0, 0.0, best, -1};
    return {bx, by, bz, best, best_id};
}

// ---------------------------------------------------------------- ray tests
// Reference formulas (exact policy): kernels.py:185-275

template <class R>
QB_D R ray_sphere_ref(R cx, R cy, R cz, R r, R ox, R oy, R oz, R dx, R dy, R dz, R tmin, R tmax) {
    R mx = ox - cx, my = oy - cy, mz = oz - cz;
    R b = mx * dx + my * dy + mz * dz;
    R c = mx * mx + my * my + mz * mz - r * r;
    R disc = b * b - c;
    if (disc < R(0.0)) return R(-1.0);
    R s = r_sqrt(disc);
    R t = -b - s;
    if (t > tmin && t <= tmax) return t;
    t = -b + s;
    if (t > tmin && t <= tmax) return t;
    return R(-1.0);
}

template <class R> QB_D R ray_box_ref(const R *d, R ox, R oy, R oz, R dx, R dy, R dz, R tmin, R tmax) {
    R mx = ox - d[0], my = oy - d[1], mz = oz - d[2];
    R lo[3] = {d[6] * mx + d[9] * my + d[12] * mz, d[7] * mx + d[10] * my + d[13] * mz, d[8] * mx + d[11] * my + d[14] * mz};
    R ld[3] = {d[6] * dx + d[9] * dy + d[12] * dz, d[7] * dx + d[10] * dy + d[13] * dz, d[8] * dx + d[11] * dy + d[14] * dz};
    R t0 = tmin, t1 = tmax;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        R o = lo[a], dd = ld[a], h = d[3 + a];
        if (r_abs(dd) < R(1e-300)) {
            if (o < -h || o > h) return R(-1.0);
        } else {
            R inv = R(1.0) / dd;
            R ta = (-h - o) * inv, tb = (h - o) * inv;
            if (ta > tb) {
                R t = ta; ta = tb; tb = t;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
            if (t0 > t1) return R(-1.0);
        }
    }
    if (t0 > tmin && t0 <= tmax) return t0;
    if (t1 > tmin && t1 <= tmax) return t1;
    return R(-1.0);
}

template <class R> QB_D R ray_triangle_ref(const R *d, R ox, R oy, R oz, R dx, R dy, R dz, R tmin, R tmax) {
    R ax = d[0], ay = d[1], az = d[2];
    R e1x = d[3] - ax, e1y = d[4] - ay, e1z = d[5] - az;
    R e2x = d[6] - ax, e2y = d[7] - ay, e2z = d[8] - az;
    R px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
    R det = e1x * px + e1y * py + e1z * pz;
    if (r_abs(det) < R(1e-300)) return R(-1.0);
    R inv = R(1.0) / det;
    R tx = ox - ax, ty = oy - ay, tz = oz - az;
    R u = (tx * px + ty * py + tz * pz) * inv;
    if (u < R(0.0) || u > R(1.0)) return R(-1.0);
    R qx = ty * e1z - tz * e1y, qy = tz * e1x - tx * e1z, qz = tx * e1y - ty * e1x;
    R v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < R(0.0) || u + v > R(1.0)) return R(-1.0);
    R t = (e2x * qx + e2y * qy + e2z * qz) * inv;
    if (t > tmin && t <= tmax) return t;
    return R(-1.0);
}

// ---- FP32 production versions on the packed float records ---------------
// float record layouts (qb_scene_pack.cuh pack_prim):
//   sphere   : [cx cy cz r] [r*r 0 0 0] ...
//   box      : [cx cy cz hx] [hy hz r00 r01] [r02 r10 r11 r12] [r20 r21 r22 0]
//   triangle : [ax ay az bx] [by bz cx cy] [cz 0 0 0]  (vertices)

// 1/x from MUFU.RCP (~1 ulp): ray-setup reciprocals for slab tests against
// outward-rounded boxes, no IEEE-division slow path (no call, no stack frame)
QB_D float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// sphere (centre a.xyz, r^2 = r2) from registers: swarm agents in the epilogue
QB_D float ray_sphere_v(float4 a, float r2, float ox, float oy, float oz, float dx, float dy, float dz, float tmin,
                        float tmax) {
    float mx = ox - a.x, my = oy - a.y, mz = oz - a.z;
    float bb = mx * dx + my * dy + mz * dz;
    float fx = mx - bb * dx, fy = my - bb * dy, fz = mz - bb * dz;
    float disc = r2 - (fx * fx + fy * fy + fz * fz);
    if (disc < 0.0f) return -1.0f;
    float s = sqrtf(disc);
    float t = -bb - s;
    if (t > tmin && t <= tmax) return t;
    t = -bb + s;
    if (t > tmin && t <= tmax) return t;
    return -1.0f;
}

QB_D float ray_sphere_f(const float4 *p, float ox, float oy, float oz, float dx, float dy, float dz, float tmin, float tmax) {
    float4 a = __ldg(p), b = __ldg(p + 1);
    float mx = ox - a.x, my = oy - a.y, mz = oz - a.z;
    float bb = mx * dx + my * dy + mz * dz;
    // robust discriminant r^2 - |m - b d|^2 (no cancellation of |m|^2 - b^2)
    float fx = mx - bb * dx, fy = my - bb * dy, fz = mz - bb * dz;
    float disc = b.x - (fx * fx + fy * fy + fz * fz);
    if (disc < 0.0f) return -1.0f;
    float s = sqrtf(disc);
    float t = -bb - s;
    if (t > tmin && t <= tmax) return t;
    t = -bb + s;
    if (t > tmin && t <= tmax) return t;
    return -1.0f;
}

QB_D float ray_box_v(float4 a, float4 b, float4 c, float4 e, float ox, float oy, float oz, float dx, float dy, float dz,
                     float tmin, float tmax) {
    float mx = ox - a.x, my = oy - a.y, mz = oz - a.z;
    // R = [[b.z b.w c.x] [c.y c.z c.w] [e.x e.y e.z]] (local -> world); local = R^T m
    float lox = b.z * mx + c.y * my + e.x * mz;
    float loy = b.w * mx + c.z * my + e.y * mz;
    float loz = c.x * mx + c.w * my + e.z * mz;
    float ldx = b.z * dx + c.y * dy + e.x * dz;
    float ldy = b.w * dx + c.z * dy + e.y * dz;
    float ldz = c.x * dx + c.w * dy + e.z * dz;
    float hx = a.w, hy = b.x, hz = b.y;
    float ix = rcp_approx(ldx), iy = rcp_approx(ldy), iz = rcp_approx(ldz);
    // slabs; a zero direction gives +-inf (or NaN at the slab plane, which
    // fminf/fmaxf ignore -- the reference's `o outside -> miss` is the inf case)
    float tax = (-hx - lox) * ix, tbx = (hx - lox) * ix;
    float tay = (-hy - loy) * iy, tby = (hy - loy) * iy;
    float taz = (-hz - loz) * iz, tbz = (hz - loz) * iz;
    float t0 = fmaxf(fmaxf(fminf(tax, tbx), fminf(tay, tby)), fmaxf(fminf(taz, tbz), tmin));
    float t1 = fminf(fminf(fmaxf(tax, tbx), fmaxf(tay, tby)), fminf(fmaxf(taz, tbz), tmax));
    if (t0 > t1) return -1.0f;
    if (t0 > tmin && t0 <= tmax) return t0;
    if (t1 > tmin && t1 <= tmax) return t1;
    return -1.0f;
}

QB_D float ray_box_f(const float4 *p, float ox, float oy, float oz, float dx, float dy, float dz, float tmin, float tmax) {
    return ray_box_v(__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3), ox, oy, oz, dx, dy, dz, tmin, tmax);
}

// Watertight ray-triangle test (Woop, Benthin & Wald, JCGT 2013), two-sided
// like the reference's Moeller-Trumbore (kernels.py:249-275).  The record
// holds the three vertices as floats rounded from the reference's doubles,
// so triangles sharing an edge hold bit-identical copies of its end points.
// Each vertex is moved into a per-ray sheared frame (the ray becomes the KZ
// axis) by a deterministic function of that vertex alone, and the 2D edge
// functions are products rounded separately and then subtracted (no FMA
// contraction): swapping an edge's end points negates its value exactly.  A
// ray crossing a shared edge therefore lands inside exactly one of the two
// triangles (both when it hits the edge exactly) -- no cracks.  Moeller-
// Trumbore on float (a, e1, e2) records is not watertight: the two triangles
// round the shared edge differently and a ray can pass between them (found
// by the C5 parity test on the indoor hall: 1 pixel in 2.6e5 read a surface
// 0.6 m behind).
//
// KZ: any axis along which the ray direction is not small (callers pick the
// dominant axis of the ray or of its tile); kx, ky the other two, cyclic.
struct Shear {
    float sx, sy, sz;
};

// per-ray shear constants: sz = 1 / d[kz] (any deterministic per-ray value
// keeps the test watertight), sx = d[kx] sz, sy = d[ky] sz
QB_D Shear ray_shear(int kz, float dx, float dy, float dz) {
    const float dk = kz == 0 ? dx : (kz == 1 ? dy : dz);
    const float ax = kz == 0 ? dy : (kz == 1 ? dz : dx), ay = kz == 0 ? dz : (kz == 1 ? dx : dy);
    const float sz = rcp_approx(dk);
    return {ax * sz, ay * sz, sz};
}

template <int KZ>
QB_D float ray_triangle_wt(float4 r0, float4 r1, float4 r2, float ox, float oy, float oz, Shear sh, float tmin,
                           float tmax) {
    constexpr int KX = (KZ + 1) % 3, KY = (KZ + 2) % 3;
    const float sx = sh.sx, sy = sh.sy, sz = sh.sz;
    const float A[3] = {r0.x - ox, r0.y - oy, r0.z - oz};
    const float B[3] = {r0.w - ox, r1.x - oy, r1.y - oz};
    const float C[3] = {r1.z - ox, r1.w - oy, r2.x - oz};
    const float ax = fmaf(-sx, A[KZ], A[KX]), ay = fmaf(-sy, A[KZ], A[KY]);
    const float bx = fmaf(-sx, B[KZ], B[KX]), by = fmaf(-sy, B[KZ], B[KY]);
    const float cx = fmaf(-sx, C[KZ], C[KX]), cy = fmaf(-sy, C[KZ], C[KY]);
    const float U = __fsub_rn(__fmul_rn(cx, by), __fmul_rn(cy, bx));
    const float V = __fsub_rn(__fmul_rn(ax, cy), __fmul_rn(ay, cx));
    const float W = __fsub_rn(__fmul_rn(bx, ay), __fmul_rn(by, ax));
    if ((U < 0.0f || V < 0.0f || W < 0.0f) && (U > 0.0f || V > 0.0f || W > 0.0f)) return -1.0f;
    const float det = U + V + W;
    if (det == 0.0f) return -1.0f;
    // hit distance in ray-parameter units: z' = sz * P[KZ]
    const float T = fmaf(U, A[KZ], fmaf(V, B[KZ], W * C[KZ]));
    const float t = __fdividef(T * sz, det);
    if (t > tmin && t <= tmax) return t;
    return -1.0f;
}

// dominant axis of a direction (ties to the lower axis)
QB_D int dominant_axis(float dx, float dy, float dz) {
    const float x = fabsf(dx), y = fabsf(dy), z = fabsf(dz);
    return (x >= y && x >= z) ? 0 : (y >= z ? 1 : 2);
}

// triangle record passed by value (callers issue the record loads together
// with the primitive's metadata load); kz: the ray's (or its tile's, warp-
// uniform) dominant axis
QB_D float ray_triangle_v(int kz, float4 a, float4 b, float4 c, float ox, float oy, float oz, Shear sh, float tmin,
                          float tmax) {
    if (kz == 2) return ray_triangle_wt<2>(a, b, c, ox, oy, oz, sh, tmin, tmax);
    if (kz == 1) return ray_triangle_wt<1>(a, b, c, ox, oy, oz, sh, tmin, tmax);
    return ray_triangle_wt<0>(a, b, c, ox, oy, oz, sh, tmin, tmax);
}

QB_D float ray_triangle_v(int kz, float4 a, float4 b, float4 c, float ox, float oy, float oz, float dx, float dy, float dz,
                          float tmin, float tmax) {
    return ray_triangle_v(kz, a, b, c, ox, oy, oz, ray_shear(kz, dx, dy, dz), tmin, tmax);
}

QB_D float ray_triangle_f(int kz, const float4 *p, float ox, float oy, float oz, float dx, float dy, float dz, float tmin,
                          float tmax) {
    return ray_triangle_v(kz, __ldg(p), __ldg(p + 1), __ldg(p + 2), ox, oy, oz, dx, dy, dz, tmin, tmax);
}

// out-of-line copy for kernels where triangles are the rare case (the
// culling renderer's analytic rooms): keeps the three shear variants out of
// the caller's register allocation
static __device__ __noinline__ float ray_triangle_call(int kz, const float4 *p, float ox, float oy, float oz, float dx,
                                                       float dy, float dz, float tmin, float tmax) {
    return ray_triangle_f(kz, p, ox, oy, oz, dx, dy, dz, tmin, tmax);
}

// FP32 slab entry (kernels.py:288-319 semantics: entry clamped at 0, INF = miss)
QB_D float slab_enter_f(const float4 lo, const float4 hi, float ox, float oy, float oz, float ix, float iy, float iz,
                        float tmax) {
    float tax = (lo.x - ox) * ix, tbx = (hi.x - ox) * ix;
    float tay = (lo.y - oy) * iy, tby = (hi.y - oy) * iy;
    float taz = (lo.z - oz) * iz, tbz = (hi.z - oz) * iz;
    float t0 = fmaxf(fmaxf(fminf(tax, tbx), fminf(tay, tby)), fmaxf(fminf(taz, tbz), 0.0f));
    float t1 = fminf(fminf(fmaxf(tax, tbx), fmaxf(tay, tby)), fminf(fmaxf(taz, tbz), tmax));
    return t0 <= t1 ? t0 : infinity_f();
}

// same test with the ray folded into FMAs: (b - o) * i == fma(b, i, -o*i),
// oi = o * i precomputed per ray (node bounds are inflated outward, so the
// ~1-ulp difference cannot drop a primitive the box contains)
QB_D float slab_enter_fma(const float4 lo, const float4 hi, float oix, float oiy, float oiz, float ix, float iy, float iz,
                          float tmax) {
    float tax = fmaf(lo.x, ix, -oix), tbx = fmaf(hi.x, ix, -oix);
    float tay = fmaf(lo.y, iy, -oiy), tby = fmaf(hi.y, iy, -oiy);
    float taz = fmaf(lo.z, iz, -oiz), tbz = fmaf(hi.z, iz, -oiz);
    float t0 = fmaxf(fmaxf(fminf(tax, tbx), fminf(tay, tby)), fmaxf(fminf(taz, tbz), 0.0f));
    float t1 = fminf(fminf(fmaxf(tax, tbx), fmaxf(tay, tby)), fminf(fmaxf(taz, tbz), tmax));
    return t0 <= t1 ? t0 : infinity_f();
}

// exact-double slab entry, reference order
QB_D xd slab_enter_x(const double *b, xd ox, xd oy, xd oz, xd ix, xd iy, xd iz, xd tmax) {
    xd t0(0.0), t1 = tmax, ta, tb;
    xd o[3] = {ox, oy, oz}, iv[3] = {ix, iy, iz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ta = (xd(b[a]) - o[a]) * iv[a];
        tb = (xd(b[3 + a]) - o[a]) * iv[a];
        if (ta > tb) {
            xd t = ta; ta = tb; tb = t;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
    }
    if (t0 > t1) return xd(infinity_d());
    return t0;
}

QB_D xd inv_dir_x(xd d) {
    if (r_abs(d) > xd(1e-300)) return xd(1.0) / d;
    return d >= xd(0.0) ? xd(infinity_d()) : xd(-infinity_d());
}

// kernels.py:322-386 for one ray, exact double (validation / public raycast).
// Returns t (or -1) and the hit id.
QB_D double raycast_x(const DevScene &S, int scene, double ox_, double oy_, double oz_, double dx_, double dy_, double dz_,
                      double tmin_, double tmax_, int &id_out) {
    xd ox(ox_), oy(oy_), oz(oz_), dx(dx_), dy(dy_), dz(dz_), tmin(tmin_);
    xd ix = inv_dir_x(dx), iy = inv_dir_x(dy), iz = inv_dir_x(dz);
    int stack[64];
    int top = 0;
    stack[top++] = S.root[scene];
    xd best_t(tmax_);
    int best_id = -1;
    bool hit = false;
    while (top > 0) {
        int node = stack[--top];
        xd enter = slab_enter_x(S.noded + 6 * node, ox, oy, oz, ix, iy, iz, best_t);
        if (enter > best_t) continue;
        int2 ni = S.nodei[node];
        if (ni.y > 0) {
            for (int p = ni.x; p < ni.x + ni.y; ++p) {
                int2 m = S.meta[p];
                const double *dd = S.primd + 16 * p;
                xd d[15];
#pragma unroll
                for (int k = 0; k < 15; ++k) d[k] = xd(dd[k]);
                xd t;
                if (m.x == QB_SPHERE)
                    t = ray_sphere_ref<xd>(d[0], d[1], d[2], d[3], ox, oy, oz, dx, dy, dz, tmin, best_t);
                else if (m.x == QB_BOX)
                    t = ray_box_ref<xd>(d, ox, oy, oz, dx, dy, dz, tmin, best_t);
                else
                    t = ray_triangle_ref<xd>(d, ox, oy, oz, dx, dy, dz, tmin, best_t);
                if (t > xd(0.0)) {
                    if (t < best_t || !hit || (t == best_t && m.y < best_id)) {
                        best_t = t;
                        best_id = m.y;
                        hit = true;
                    }
                }
            }
        } else {
            int l = ni.x, r = l + 1;
            xd el = slab_enter_x(S.noded + 6 * l, ox, oy, oz, ix, iy, iz, best_t);
            xd er = slab_enter_x(S.noded + 6 * r, ox, oy, oz, ix, iy, iz, best_t);
            if (el <= er) {
                if (er <= best_t) stack[top++] = r;
                if (el <= best_t) stack[top++] = l;
            } else {
                if (el <= best_t) stack[top++] = l;
                if (er <= best_t) stack[top++] = r;
            }
        }
    }
    id_out = hit ? best_id : -1;
    return hit ? best_t.v : -1.0;
}

// FP32 single-ray traversal (public raycast in the production precision)
QB_D float raycast_f(const DevScene &S, int scene, float ox, float oy, float oz, float dx, float dy, float dz, float tmin,
                     float tmax, int &id_out) {
    float ix = 1.0f / dx, iy = 1.0f / dy, iz = 1.0f / dz;
    const int kz = dominant_axis(dx, dy, dz);
    int stack[64];
    int top = 0;
    stack[top++] = S.root[scene];
    float best_t = tmax;
    int best_id = -1;
    bool hit = false;
    while (top > 0) {
        int node = stack[--top];
        float4 lo = __ldg(S.nodef + 2 * node), hi = __ldg(S.nodef + 2 * node + 1);
        if (slab_enter_f(lo, hi, ox, oy, oz, ix, iy, iz, best_t) > best_t) continue;
        int a = __float_as_int(lo.w), b = __float_as_int(hi.w);
        if (b > 0) {
            for (int p = a; p < a + b; ++p) {
                int2 m = __ldg(S.meta + p);
                const float4 *pr = S.primf + 4 * p;
                float t = m.x == QB_SPHERE ? ray_sphere_f(pr, ox, oy, oz, dx, dy, dz, tmin, best_t)
                          : m.x == QB_BOX  ? ray_box_f(pr, ox, oy, oz, dx, dy, dz, tmin, best_t)
                                           : ray_triangle_f(kz, pr, ox, oy, oz, dx, dy, dz, tmin, best_t);
                if (t > 0.0f && (t < best_t || !hit || (t == best_t && m.y < best_id))) {
                    best_t = t;
                    best_id = m.y;
                    hit = true;
                }
            }
        } else {
            stack[top++] = a + 1;
            stack[top++] = a;
        }
    }
    id_out = hit ? best_id : -1;
    return hit ? best_t : -1.0f;
}

#endif  // __CUDACC__
