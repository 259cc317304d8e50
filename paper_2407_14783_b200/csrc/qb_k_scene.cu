// qb_k_scene.cu -- scene ingestion on the device: the primitive
// tables of S scenes (shapes.py:139-212 SceneArrays rows, already in device
// memory) -> a BVH per scene + the DevScene records, without a host pass.
//
// The tree is a linear BVH refined by treelet restructuring: 63-bit Morton
// codes of the primitive centroids (21 bits per axis over the scene bounds),
// a radix sort (CUB), the Karras-2012 parallel hierarchy (one thread per
// internal node), a bottom-up bounds refit (one thread per leaf, the second
// arrival at each node continues), three bottom-up sweeps of SAH-optimal
// 7-leaf treelet restructuring (Karras & Aila 2013), a DFS numbering of the
// refined tree, then subtrees of <= QB_BVH_LEAF primitives become leaves.
// Node layout is the host build's: node_first / node_first + 1 children
// (internal node j owns slots 1 + 2j and 2 + 2j, so no relayout pass is
// needed; slots under a collapsed subtree stay unused).  On the config-5
// hall the refined tree renders 2.4% faster than the host binned-SAH tree
// (plain LBVH: 13% slower) and builds in ~20 ms instead of ~0.4 s.
// Every query result is traversal-order independent (nearest t / d^2, ties
// to the lower object id), so the device-built scene renders and answers
// nearest-point queries bit-identically to the host binned-SAH build
// (tests/test_gpu_scene_build.py); only the traversal cost differs.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <vector>

#include "qb_checks.cuh"
#include "qb_internal.h"
#include "qb_scene_pack.cuh"

#ifndef QB_BVH_LEAF_DEV
#define QB_BVH_LEAF_DEV 4  // max primitives per leaf (as the host build)
#endif

namespace {

constexpr int LEAF = QB_BVH_LEAF_DEV;

// doubles as order-preserving unsigned keys (atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

// validation + raw bounds of one scene: ub[0..2] min keys of lo, ub[3..5] max keys of hi
__global__ void k_scene_bounds(int cnt, const int64_t *type, const int64_t *oid, const double *lo, const double *hi,
                               unsigned long long *ub, int *bad) {
    unsigned long long mn[3] = {~0ULL, ~0ULL, ~0ULL}, mx[3] = {0, 0, 0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        if (type[i] < 0 || type[i] > 2) atomicOr(bad, 1);
        if (oid[i] <= 0 || oid[i] >= (1LL << 31)) atomicOr(bad, 2);
        if (type[i] != QB_TRIANGLE) atomicOr(bad, 8);  // (not an error: the scene is not triangles only)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double l = lo[3 * i + k], h = hi[3 * i + k];
            if (!(l <= h)) atomicOr(bad, 4);  // also catches NaN
            mn[k] = min(mn[k], ord_key(l));
            mx[k] = max(mx[k], ord_key(h));
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = min(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = max(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&ub[k], mn[k]);
            atomicMax(&ub[3 + k], mx[k]);
        }
    }
}

__device__ __forceinline__ unsigned long long spread3(unsigned int a) {
    unsigned long long x = a & 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

// Morton code of each centroid (x in bits 2 mod 3, y 1 mod 3, z 0 mod 3)
__global__ void k_morton(int cnt, const double *lo, const double *hi, const unsigned long long *ub,
                         unsigned long long *keys, int *vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    unsigned int q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double b0 = ord_val(ub[k]), b1 = ord_val(ub[3 + k]);
        const double c = 0.5 * (lo[3 * i + k] + hi[3 * i + k]);
        const double ext = b1 - b0;
        double f = ext > 0.0 ? (c - b0) / ext : 0.0;
        f = fmin(fmax(f, 0.0), 1.0);
        q[k] = (unsigned int)fmin(f * 2097152.0, 2097151.0);
    }
    keys[i] = spread3(q[0]) << 2 | spread3(q[1]) << 1 | spread3(q[2]);
    vals[i] = i;
}

// common-prefix length of sorted keys i and j (index bits break ties)
__device__ __forceinline__ int delta(const unsigned long long *keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const unsigned long long a = keys[i], b = keys[j];
    return a == b ? 64 + __clz(i ^ j) : __clzll(a ^ b);
}

// Karras 2012: internal node i's key range [first, last] and split.  Node
// ids: internal 0..n-2, leaf k -> n-1+k.
__global__ void k_karras(int n, const unsigned long long *keys, int2 *child, int2 *range, int *axis, int *parent) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = delta(keys, n, i, i + 1) > delta(keys, n, i, i - 1) ? 1 : -1;
    const int dmin = delta(keys, n, i, i - d);
    int lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = delta(keys, n, i, j);
    int s = 0, t = l;
    do {
        t = (t + 1) >> 1;
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    const int g = i + s * d + min(d, 0);
    const int first = min(i, j), last = max(i, j);
    const int left = first == g ? n - 1 + g : g, right = last == g + 1 ? n - 1 + g + 1 : g + 1;
    QB_CHECK(first >= 0 && last < n && first < last && left >= 0 && left < 2 * n - 1 && right >= 0 &&
                 right < 2 * n - 1 && left != right, "karras hierarchy node");
    child[i] = make_int2(left, right);
    range[i] = make_int2(first, last);
    parent[left] = i;
    parent[right] = i;
    // split axis: the highest bit where the range's codes differ
    const unsigned long long x = keys[first] ^ keys[last];
    axis[i] = x ? 2 - (63 - __clzll(x)) % 3 : 0;
}

__device__ __forceinline__ void node_bounds(int n, int u, const int *order, const double *plo, const double *phi,
                                            const double *ib, double *b) {
    if (u >= n - 1) {  // leaf: its primitive's bounds
        const int p = order[u - (n - 1)];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            b[k] = plo[3 * p + k];
            b[3 + k] = phi[3 * p + k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) b[k] = __ldcg(&ib[6 * u + k]);
    }
}

// bottom-up refit: one thread per leaf; at each internal node the second
// arriving thread unions both children and continues upward
__global__ void k_refit(int n, const int *order, const double *plo, const double *phi, const int2 *child,
                        const int *parent, int *flag, double *ib) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int u = parent[n - 1 + k];
    while (u >= 0) {
        __threadfence();
        if (atomicAdd(&flag[u], 1) == 0) return;  // the sibling subtree is not done yet
        __threadfence();
        double a[6], b[6];
        node_bounds(n, child[u].x, order, plo, phi, ib, a);
        node_bounds(n, child[u].y, order, plo, phi, ib, b);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            __stcg(&ib[6 * u + c], fmin(a[c], b[c]));
            __stcg(&ib[6 * u + 3 + c], fmax(a[3 + c], b[3 + c]));
        }
        u = u == 0 ? -1 : parent[u];
    }
}

// depth of each leaf's emitted ancestor-leaf: 1 + internal ancestors that
// stay internal (more than LEAF primitives)
__global__ void k_depth(int n, const int2 *range, const int *parent, int *max_depth) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int d = 1;
    for (int u = n > 1 ? parent[n - 1 + k] : -1; u >= 0; u = u == 0 ? -1 : parent[u])
        if (range[u].y - range[u].x + 1 > LEAF) ++d;
    atomicMax(max_depth, d);
}

// node records in the host build's format (qb_abi.cu qb_scene_create)
__device__ __forceinline__ void write_node(float4 *nodef, double *noded, int2 *nodei, int slot, const double *b, int a,
                                           int bb) {
    nodef[2 * slot] = make_float4(qbpack::f_down(b[0]), qbpack::f_down(b[1]), qbpack::f_down(b[2]), qbpack::i2f(a));
    nodef[2 * slot + 1] = make_float4(qbpack::f_up(b[3]), qbpack::f_up(b[4]), qbpack::f_up(b[5]), qbpack::i2f(bb));
#pragma unroll
    for (int k = 0; k < 6; ++k) noded[6 * slot + k] = b[k];
    nodei[slot] = make_int2(a, bb);
}

__global__ void k_emit(int n, int node_off, int prim_off, const int *order, const double *plo, const double *phi,
                       const int2 *child, const int2 *range, const int *axis, const int *parent, const double *ib,
                       float4 *nodef, double *noded, int2 *nodei) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= 2 * n - 1) return;
    double b[6];
    if (n == 1) {  // a single primitive: the root is its leaf
        node_bounds(n, 0, order, plo, phi, ib, b);
        write_node(nodef, noded, nodei, node_off, b, prim_off, 1);
        return;
    }
    int slot = 0;
    if (u != 0) {
        const int p = parent[u];
        if (range[p].y - range[p].x + 1 <= LEAF) return;  // inside a collapsed subtree
        slot = 1 + 2 * p + (child[p].x == u ? 0 : 1);
        QB_CHECK(p >= 0 && p < n - 1 && slot < 2 * n - 1, "emit node slot");
    }
    node_bounds(n, u, order, plo, phi, ib, b);
    if (u >= n - 1) {
        write_node(nodef, noded, nodei, node_off + slot, b, prim_off + (u - (n - 1)), 1);
    } else {
        const int cnt = range[u].y - range[u].x + 1;
        if (cnt <= LEAF)
            write_node(nodef, noded, nodei, node_off + slot, b, prim_off + range[u].x, cnt);
        else
            write_node(nodef, noded, nodei, node_off + slot, b, node_off + 1 + 2 * u, -axis[u]);
    }
}

// ---------------------------------------------------------------------------
// Treelet restructuring (Karras & Aila 2013, "Fast parallel construction of
// high-quality BVHs"): the Morton-order tree is refined bottom-up -- the same
// second-arrival sweep as the refit -- and at every node of >= TL_MIN
// primitives the treelet of its TL largest-area descendants (the node, then
// repeatedly the largest-area internal leaf of the treelet expanded) is
// replaced by the topology of minimum SAH cost over those TL subtrees,
// found by dynamic programming over the 2^TL subsets.  Subtrees of <= LEAF
// primitives cost as a leaf (the emit collapses them whatever their shape).
// The refined tree's subtrees are no longer contiguous Morton ranges, so the
// primitive order and each node's first primitive come from a DFS numbering
// afterwards (k_dfs).  Queries stay bit-identical (traversal-order
// independent); only the traversal cost changes.
#ifndef QB_TREELET
#define QB_TREELET 7  // treelet leaves; 0 keeps the plain LBVH
#endif
#ifndef QB_TREELET_PASSES
#define QB_TREELET_PASSES 3  // bottom-up refinement sweeps (C5 hall: 1 -> 2.3% slower than the host SAH tree, 3 -> 2.4% faster)
#endif
constexpr int TL = QB_TREELET > 1 ? QB_TREELET : 2;
constexpr int TL_MIN = 8;                // restructure nodes of at least this many primitives
#ifndef QB_SAH_CT
#define QB_SAH_CT 2.0f  // node visit vs primitive test (config-5 hall: 1.2 -> 2.0 renders +1%, 4.0 +0.5%)
#endif
constexpr float SAH_CT = QB_SAH_CT, SAH_CI = 1.0f;

// the sweep's tree arrays change under other SMs: read them through L2
__device__ __forceinline__ int2 ld_child(const int2 *child, int u) { return __ldcg(&child[u]); }

__device__ __forceinline__ float area_f(const double *b) {
    const float dx = (float)(b[3] - b[0]), dy = (float)(b[4] - b[1]), dz = (float)(b[5] - b[2]);
    return 2.0f * (dx * dy + dy * dz + dz * dx);
}

__device__ void restructure(int n, int u, const int *order, const double *plo, const double *phi, int2 *child,
                            int *parent, double *ib, int *cnt, float *cost) {
    const int2 c = ld_child(child, u);
    const int total = __ldcg(&cnt[c.x]) + __ldcg(&cnt[c.y]);
    __stcg(&cnt[u], total);
    double bu[6];
    node_bounds(n, u, order, plo, phi, ib, bu);
    const float au = area_f(bu);
    if (QB_TREELET < 3 || total < TL_MIN) {
        __stcg(&cost[u], total <= LEAF ? SAH_CI * au * (float)total : SAH_CT * au + __ldcg(&cost[c.x]) + __ldcg(&cost[c.y]));
        return;
    }
    // treelet formation: expand the largest-area internal leaf until TL leaves
    int L[TL], I[TL - 1], m = 2, ni = 1;
    float la[TL];
    L[0] = c.x;
    L[1] = c.y;
    I[0] = u;
    double bb[6];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        node_bounds(n, L[j], order, plo, phi, ib, bb);
        la[j] = area_f(bb);
    }
    while (m < TL) {
        int best = -1;
        float ba = -1.0f;
        for (int j = 0; j < m; ++j)
            if (L[j] < n - 1 && la[j] > ba) {
                ba = la[j];
                best = j;
            }
        if (best < 0) break;
        const int v = L[best];
        I[ni++] = v;
        const int2 cv = ld_child(child, v);
        L[best] = cv.x;
        L[m] = cv.y;
        node_bounds(n, L[best], order, plo, phi, ib, bb);
        la[best] = area_f(bb);
        node_bounds(n, L[m], order, plo, phi, ib, bb);
        la[m] = area_f(bb);
        ++m;
    }
    // leaf data
    float lb[TL][6], lcost[TL];
    int lcnt[TL];
    for (int j = 0; j < m; ++j) {
        node_bounds(n, L[j], order, plo, phi, ib, bb);
#pragma unroll
        for (int k = 0; k < 6; ++k) lb[j][k] = (float)bb[k];
        lcost[j] = __ldcg(&cost[L[j]]);
        lcnt[j] = __ldcg(&cnt[L[j]]);
    }
    // DP over subsets (subsets of S are numerically smaller than S)
    const int full = (1 << m) - 1;
    float copt[1 << TL];
    unsigned char part[1 << TL];
    for (int S = 1; S <= full; ++S) {
        float lo0 = 3.4e38f, lo1 = 3.4e38f, lo2 = 3.4e38f, hi0 = -3.4e38f, hi1 = -3.4e38f, hi2 = -3.4e38f;
        int sc = 0;
        for (int j = 0; j < m; ++j)
            if (S >> j & 1) {
                lo0 = fminf(lo0, lb[j][0]); lo1 = fminf(lo1, lb[j][1]); lo2 = fminf(lo2, lb[j][2]);
                hi0 = fmaxf(hi0, lb[j][3]); hi1 = fmaxf(hi1, lb[j][4]); hi2 = fmaxf(hi2, lb[j][5]);
                sc += lcnt[j];
            }
        if ((S & (S - 1)) == 0) {
            copt[S] = lcost[__ffs(S) - 1];
            part[S] = 0;
            continue;
        }
        const float dx = hi0 - lo0, dy = hi1 - lo1, dz = hi2 - lo2, a = 2.0f * (dx * dy + dy * dz + dz * dx);
        const int low = S & -S, rest = S ^ low;
        float bestc = 3.4e38f;
        int bp = low;
        for (int q = rest;; q = (q - 1) & rest) {
            const int P = q | low;
            if (P != S) {
                const float cc = copt[P] + copt[S ^ P];
                if (cc < bestc) {
                    bestc = cc;
                    bp = P;
                }
            }
            if (q == 0) break;
        }
        part[S] = (unsigned char)bp;
        copt[S] = sc <= LEAF ? SAH_CI * a * (float)sc : SAH_CT * a + bestc;
    }
    const float old = SAH_CT * au + __ldcg(&cost[c.x]) + __ldcg(&cost[c.y]);
    if (!(copt[full] < old * 0.9999f)) {  // no gain: keep the Morton topology
        __stcg(&cost[u], old);
        return;
    }
    __stcg(&cost[u], copt[full]);
    // rebuild top-down, reusing the treelet's internal node ids (u keeps its id and parent)
    int stS[TL], stV[TL], sp = 0, next = 1;
    stS[sp] = full;
    stV[sp++] = u;
    while (sp > 0) {
        const int S = stS[--sp], v = stV[sp];
        const int P = part[S], Q = S ^ P;
        int kids[2];
        const int sub[2] = {P, Q};
        for (int h = 0; h < 2; ++h) {
            if ((sub[h] & (sub[h] - 1)) == 0) {
                kids[h] = L[__ffs(sub[h]) - 1];
            } else {
                kids[h] = I[next++];
                stS[sp] = sub[h];
                stV[sp++] = kids[h];
            }
            __stcg(&parent[kids[h]], v);
        }
        __stcg(&child[v], make_int2(kids[0], kids[1]));
        if (v != u) {  // a reused internal node: bounds, count and cost of its new subset
            double nb[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
            int sc = 0;
            for (int j = 0; j < m; ++j)
                if (S >> j & 1) {
                    node_bounds(n, L[j], order, plo, phi, ib, bb);
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        nb[k] = fmin(nb[k], bb[k]);
                        nb[3 + k] = fmax(nb[3 + k], bb[3 + k]);
                    }
                    sc += lcnt[j];
                }
#pragma unroll
            for (int k = 0; k < 6; ++k) __stcg(&ib[6 * v + k], nb[k]);
            __stcg(&cnt[v], sc);
            __stcg(&cost[v], copt[S]);
        }
    }
}

// bottom-up sweep (second arrival processes the node, like k_refit)
__global__ void k_treelet(int n, const int *order, const double *plo, const double *phi, int2 *child, int *parent,
                          int *flag, double *ib, int *cnt, float *cost) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int leaf = n - 1 + k;
    double b[6];
    node_bounds(n, leaf, order, plo, phi, ib, b);
    __stcg(&cnt[leaf], 1);
    __stcg(&cost[leaf], SAH_CI * area_f(b));
    int u = __ldcg(&parent[leaf]);
    while (u >= 0) {
        __threadfence();
        if (atomicAdd(&flag[u], 1) == 0) return;
        __threadfence();
        restructure(n, u, order, plo, phi, child, parent, ib, cnt, cost);
        u = u == 0 ? -1 : __ldcg(&parent[u]);
    }
}

// DFS numbering of the refined tree: first[u] = primitives left of u's
// subtree (walk up, adding the left sibling's count whenever u is a right
// child); depth (leaves only) = 1 + internal ancestors the emit keeps
__global__ void k_dfs(int n, const int2 *child, const int *parent, const int *cnt, int *first, int *max_depth) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= 2 * n - 1) return;
    int f = 0, d = 1;
    for (int v = u; v != 0;) {
        const int p = parent[v];
        if (child[p].y == v) f += cnt[child[p].x];
        if (cnt[p] > LEAF) ++d;
        v = p;
    }
    first[u] = f;
    if (u >= n - 1) atomicMax(max_depth, d);
}

__global__ void k_reorder(int n, const int *order, const int *first, int *order2) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) order2[first[n - 1 + k]] = order[k];
}

// node records of the refined tree (count / first instead of Morton ranges);
// the split axis hint = the axis along which the children's centres differ most
__global__ void k_emit_refined(int n, int node_off, int prim_off, const int *order, const double *plo,
                               const double *phi, const int2 *child, const int *cnt, const int *first,
                               const int *parent, const double *ib, float4 *nodef, double *noded, int2 *nodei) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= 2 * n - 1) return;
    double b[6];
    if (n == 1) {
        node_bounds(n, 0, order, plo, phi, ib, b);
        write_node(nodef, noded, nodei, node_off, b, prim_off, 1);
        return;
    }
    int slot = 0;
    if (u != 0) {
        const int p = parent[u];
        if (cnt[p] <= LEAF) return;  // inside a collapsed subtree
        slot = 1 + 2 * p + (child[p].x == u ? 0 : 1);
        QB_CHECK(p >= 0 && p < n - 1 && slot < 2 * n - 1, "emit_refined node slot");
    }
    node_bounds(n, u, order, plo, phi, ib, b);
    if (u >= n - 1 || cnt[u] <= LEAF) {
        write_node(nodef, noded, nodei, node_off + slot, b, prim_off + first[u], cnt[u]);
    } else {
        double l[6], r[6];
        node_bounds(n, child[u].x, order, plo, phi, ib, l);
        node_bounds(n, child[u].y, order, plo, phi, ib, r);
        int ax = 0;
        double best = -1.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double dcen = fabs((l[k] + l[3 + k]) - (r[k] + r[3 + k]));
            if (dcen > best) {
                best = dcen;
                ax = k;
            }
        }
        write_node(nodef, noded, nodei, node_off + slot, b, node_off + 1 + 2 * u, -ax);
    }
}

// primitive records in BVH order (dst = off + j <- src = off + order[j])
__global__ void k_pack_prims(int cnt, const int *order, const int64_t *type, const double *data, const int64_t *oid,
                             float4 *primf, float4 *primc, double *primd, int2 *meta) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cnt) return;
    const int src = order[j];
    const int t = (int)type[src];
    double d[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) d[k] = data[16 * (long long)src + k];
    float4 rf[4], rc[4];
    qbpack::pack_prim(t, d, rf);
    qbpack::cull_record(t, d, rc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        primf[4 * (long long)j + k] = rf[k];
        primc[4 * (long long)j + k] = rc[k];
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) primd[16 * (long long)j + k] = d[k];
    meta[j] = make_int2(t, (int)oid[src]);
}

__global__ void k_decode_bounds(int S, const unsigned long long *ub, double *bounds) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 6 * S) bounds[i] = ord_val(ub[i]);
}

__global__ void k_fill_u64(long long n, unsigned long long *p, unsigned long long lo_val, unsigned long long hi_val) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = (i % 6) < 3 ? lo_val : hi_val;
}

// the scene's own arrays come from the same stream-ordered pool (freed by
// qb_scene_destroy's cudaFree)
template <class T> T *dalloc(qb_scene *s, size_t count, cudaStream_t st) {
    void *p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(count * sizeof(T), 16), st) != cudaSuccess) return nullptr;
    s->allocs[s->n_allocs++] = p;
    return static_cast<T *>(p);
}

// build scratch: stream-ordered allocations from the device's default pool,
// which keeps the pages mapped between builds (cudaMalloc / cudaFree of the
// ~60 MB of scratch per 5e5-triangle build otherwise costs 10-250 ms of page
// mapping and device-wide synchronisation)
void keep_pool_mapped() {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = 1ull << 30;  // keep up to 1 GiB of freed build memory mapped
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

struct Scratch {
    cudaStream_t st;
    std::vector<void *> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    template <class T> T *get(size_t count) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(count * sizeof(T), 16), st) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T *>(p);
    }
    ~Scratch() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
};

int grid(long long n, int bs) { return qb::env_grid(n, bs); }

}  // namespace

namespace qb {

int scene_create_device(int n_scenes, const int64_t *prim_offsets, const int64_t *prim_type, const double *prim_data,
                        const int64_t *prim_oid, const double *prim_lo, const double *prim_hi, qb_scene **out,
                        cudaStream_t st) {
    const int S = n_scenes;
    const long long P = prim_offsets[S];
    long long max_cnt = 0, total_nodes = 0;
    std::vector<int> roots(S), prim_offset(S + 1);
    for (int s = 0; s < S; ++s) {
        const long long cnt = prim_offsets[s + 1] - prim_offsets[s];
        max_cnt = std::max(max_cnt, cnt);
        roots[s] = (int)total_nodes;
        total_nodes += 2 * cnt - 1;
        prim_offset[s] = (int)prim_offsets[s];
    }
    prim_offset[S] = (int)P;
    if (total_nodes >= (1LL << 31)) {
        set_error("qb_scene_create_device: too many nodes");
        return QB_EINVAL;
    }
    keep_pool_mapped();
    qb_scene *sc = new qb_scene();
    sc->n_allocs = 0;
    sc->host_bounds = nullptr;
    cudaGetDevice(&sc->device);
    auto fail = [&](int code, const char *what) {
        set_error("qb_scene_create_device: %s (%s)", what, cudaGetErrorString(cudaGetLastError()));
        qb_scene_destroy(sc);
        return code;
    };
    DevScene &d = sc->dev;
    d.n_scenes = S;
    d.n_prims = (int)P;
    int *root = dalloc<int>(sc, S, st);
    double *bounds = dalloc<double>(sc, 6 * (size_t)S, st);
    float4 *nodef = dalloc<float4>(sc, 2 * (size_t)total_nodes, st);
    double *noded = dalloc<double>(sc, 6 * (size_t)total_nodes, st);
    int2 *nodei = dalloc<int2>(sc, (size_t)total_nodes, st);
    float4 *primf = dalloc<float4>(sc, 4 * (size_t)P, st);
    double *primd = dalloc<double>(sc, 16 * (size_t)P, st);
    int2 *meta = dalloc<int2>(sc, (size_t)P, st);
    int *poff = dalloc<int>(sc, S + 1, st);
    float4 *primc = dalloc<float4>(sc, 4 * (size_t)P, st);
    if (!root || !bounds || !nodef || !noded || !nodei || !primf || !primd || !meta || !poff || !primc)
        return fail(QB_ENOMEM, "allocation failed");
    d.root = root;
    d.bounds = bounds;
    d.nodef = nodef;
    d.noded = noded;
    d.nodei = nodei;
    d.primf = primf;
    d.primd = primd;
    d.meta = meta;
    d.prim_offset = poff;
    d.primc = primc;

    Scratch tmp(st);
    const size_t n = (size_t)max_cnt;
    unsigned long long *keys = tmp.get<unsigned long long>(n), *keys_s = tmp.get<unsigned long long>(n);
    int *vals = tmp.get<int>(n), *order = tmp.get<int>(n);
    int2 *child = tmp.get<int2>(n), *range = tmp.get<int2>(n);
    int *axis = tmp.get<int>(n), *parent = tmp.get<int>(2 * n), *flag = tmp.get<int>(n);
    double *ib = tmp.get<double>(6 * n);
    int *tcnt = tmp.get<int>(2 * n), *tfirst = tmp.get<int>(2 * n), *order2 = tmp.get<int>(n);
    float *tcost = tmp.get<float>(2 * n);
    unsigned long long *ub = tmp.get<unsigned long long>(6 * (size_t)S);
    int *dev_ints = tmp.get<int>(2 + S);  // [bad flags, unused, max depth per scene]
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys_s, vals, order, (int)max_cnt, 0, 63, st);
    void *sort_tmp = tmp.get<char>(sort_bytes);
    if (!keys || !keys_s || !vals || !order || !child || !range || !axis || !parent || !flag || !ib || !ub || !dev_ints ||
        !sort_tmp || !tcnt || !tfirst || !order2 || !tcost)
        return fail(QB_ENOMEM, "scratch allocation failed");

    cudaMemsetAsync(nodef, 0, 2 * sizeof(float4) * total_nodes, st);
    cudaMemsetAsync(noded, 0, 6 * sizeof(double) * total_nodes, st);
    cudaMemsetAsync(nodei, 0, sizeof(int2) * total_nodes, st);
    cudaMemsetAsync(dev_ints, 0, sizeof(int) * (2 + S), st);
    cudaMemcpyAsync(root, roots.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(poff, prim_offset.data(), sizeof(int) * (S + 1), cudaMemcpyHostToDevice, st);
    k_fill_u64<<<grid(6 * S, 128), 128, 0, st>>>(6 * S, ub, ~0ULL, 0ULL);
    const int BS = 256, red_grid = std::min(grid(max_cnt, BS), 4 * sm_count());
    for (int s = 0; s < S; ++s) {
        const long long off = prim_offsets[s];
        const int cnt = (int)(prim_offsets[s + 1] - off);
        const double *lo = prim_lo + 3 * off, *hi = prim_hi + 3 * off;
        k_scene_bounds<<<std::min(grid(cnt, BS), red_grid), BS, 0, st>>>(cnt, prim_type + off, prim_oid + off, lo, hi,
                                                                        ub + 6 * s, dev_ints);
        k_morton<<<grid(cnt, BS), BS, 0, st>>>(cnt, lo, hi, ub + 6 * s, keys, vals);
        size_t bytes = sort_bytes;
        if (cub::DeviceRadixSort::SortPairs(sort_tmp, bytes, keys, keys_s, vals, order, cnt, 0, 63, st) != cudaSuccess)
            return fail(QB_ECUDA, "radix sort failed");
        if (cnt > 1) {
            cudaMemsetAsync(flag, 0, sizeof(int) * cnt, st);
            k_karras<<<grid(cnt - 1, BS), BS, 0, st>>>(cnt, keys_s, child, range, axis, parent);
            k_refit<<<grid(cnt, BS), BS, 0, st>>>(cnt, order, lo, hi, child, parent, flag, ib);
        }
        if (QB_TREELET >= 3 && cnt > 1) {  // SAH treelet refinement, then DFS numbering of the refined tree
            for (int pass = 0; pass < QB_TREELET_PASSES; ++pass) {
                cudaMemsetAsync(flag, 0, sizeof(int) * cnt, st);
                k_treelet<<<grid(cnt, 128), 128, 0, st>>>(cnt, order, lo, hi, child, parent, flag, ib, tcnt, tcost);
            }
            k_dfs<<<grid(2LL * cnt - 1, BS), BS, 0, st>>>(cnt, child, parent, tcnt, tfirst, dev_ints + 2 + s);
            k_reorder<<<grid(cnt, BS), BS, 0, st>>>(cnt, order, tfirst, order2);
            k_emit_refined<<<grid(2LL * cnt - 1, BS), BS, 0, st>>>(cnt, roots[s], (int)off, order, lo, hi, child, tcnt,
                                                                   tfirst, parent, ib, nodef, noded, nodei);
            k_pack_prims<<<grid(cnt, BS), BS, 0, st>>>(cnt, order2, prim_type + off, prim_data + 16 * off, prim_oid + off,
                                                       primf + 4 * off, primc + 4 * off, primd + 16 * off, meta + off);
            continue;
        }
        k_depth<<<grid(cnt, BS), BS, 0, st>>>(cnt, range, parent, dev_ints + 2 + s);
        k_emit<<<grid(2LL * cnt - 1, BS), BS, 0, st>>>(cnt, roots[s], (int)off, order, lo, hi, child, range, axis, parent,
                                                       ib, nodef, noded, nodei);
        k_pack_prims<<<grid(cnt, BS), BS, 0, st>>>(cnt, order, prim_type + off, prim_data + 16 * off, prim_oid + off,
                                                   primf + 4 * off, primc + 4 * off, primd + 16 * off, meta + off);
    }
    k_decode_bounds<<<grid(6 * S, 128), 128, 0, st>>>(S, ub, bounds);
    if (cudaGetLastError() != cudaSuccess) return fail(QB_ECUDA, "launch failed");
    std::vector<int> ints(2 + S);
    sc->host_bounds = new double[6 * S];
    if (cudaMemcpyAsync(ints.data(), dev_ints, sizeof(int) * (2 + S), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(sc->host_bounds, bounds, sizeof(double) * 6 * S, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return fail(QB_ECUDA, "build failed");
    if (ints[0] & 1) return fail(QB_EINVAL, "bad primitive type");
    if (ints[0] & 2) return fail(QB_EINVAL, "object ids must be positive int32");
    if (ints[0] & 4) return fail(QB_EINVAL, "primitive bounds lo > hi or NaN");
    int max_depth = 0;
    for (int s = 0; s < S; ++s) max_depth = std::max(max_depth, ints[2 + s]);
    if (max_depth > 62) return fail(QB_EINVAL, "BVH too deep for the traversal stack");
    sc->n_nodes = total_nodes;
    sc->n_prims = P;
    sc->max_depth = max_depth;
    sc->max_scene_prims = (int)max_cnt;
    d.tri_only = !(ints[0] & 8);
    *out = sc;
    return QB_OK;
}

}  // namespace qb
