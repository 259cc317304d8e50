"""bvh.build_bvh drop-in (bvh.py:16-70): the library's binned-SAH BVH
(csrc/qb_abi.cu, host C++) returned in the reference's flat layout.

node_count[i] > 0 marks a leaf owning prim_order[node_first[i] :
node_first[i] + node_count[i]]; node_count[i] == 0 an internal node whose
children are node_first[i] and node_first[i] + 1; at most LEAF_SIZE
primitives per leaf.  The split is the SAH-optimal bin boundary rather than
the centroid median, so the tree differs from the reference's; traversal
results (nearest t / distance, ties to the lowest object id) do not.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _native as nat

LEAF_SIZE = 4


def build_bvh(prim_lo, prim_hi):
    lo = np.ascontiguousarray(prim_lo, dtype=np.float64)
    hi = np.ascontiguousarray(prim_hi, dtype=np.float64)
    n = len(lo)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    count = np.zeros(1, np.int64)
    lib = nat.load(require_cuda=False)
    nat.check(lib.qb_bvh_build(n, P(lo), P(hi), P(count), None, None, None, None, None), "qb_bvh_build")
    m = int(count[0])
    node_lo, node_hi = np.empty((m, 3)), np.empty((m, 3))
    node_first, node_count, order = np.empty(m, np.int64), np.empty(m, np.int64), np.empty(n, np.int64)
    nat.check(lib.qb_bvh_build(n, P(lo), P(hi), P(count), P(node_lo), P(node_hi), P(node_first), P(node_count), P(order)),
              "qb_bvh_build")
    return node_lo, node_hi, node_first, node_count, order
