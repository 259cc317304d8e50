"""A set of scenes resident on one CUDA device (qb_scene handle).

One handle holds S scenes, each with its own BVH, so envs spread over
several scenes are stepped and rendered by a single launch (the reference
loops over scene groups, env/base.py:262-276).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _native as nat
from ..errors import EmptyScene


class DeviceScenes:
    def __init__(self, scenes, device=None):
        import torch

        nat.require_cuda()
        self.scenes = list(scenes)
        if not self.scenes:
            raise EmptyScene("no scenes")
        self.device = torch.device("cuda", 0) if device is None else torch.device(device)
        tables = [s.arrays for s in self.scenes]
        counts = [len(t) for t in tables]
        if min(counts) == 0:
            raise EmptyScene("scene has no objects")
        offsets = np.zeros(len(tables) + 1, np.int64)
        offsets[1:] = np.cumsum(counts)
        cat = lambda name, dt: np.ascontiguousarray(np.concatenate([getattr(t, name) for t in tables]), dtype=dt)  # noqa: E731
        ptype, pdata, poid = cat("prim_type", np.int64), cat("prim_data", np.float64), cat("prim_object_id", np.int64)
        plo, phi = cat("prim_aabb_lo", np.float64), cat("prim_aabb_hi", np.float64)
        handle = ctypes.c_void_p()
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        with torch.cuda.device(self.device):
            nat.check(nat.lib().qb_scene_create(len(tables), P(offsets), P(ptype), P(pdata), P(poid), P(plo), P(phi),
                                                ctypes.byref(handle)), "qb_scene_create")
        self.handle = handle
        self._lib = nat.lib()
        stats = np.zeros(4, np.int64)
        nat.check(self._lib.qb_scene_stats(handle, P(stats)), "qb_scene_stats")
        self.n_nodes, self.n_prims, self.max_depth, self.n_scenes = (int(x) for x in stats)
        b = np.zeros((len(tables), 6))
        for k in range(len(tables)):
            nat.check(self._lib.qb_scene_bounds(handle, k, P(b[k])), "qb_scene_bounds")
        self.bounds = b  # raw primitive bounds per scene (shapes.py:214-217)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.qb_scene_destroy(h)
            except Exception:
                pass
            self.handle = None

    def __repr__(self):
        return f"DeviceScenes({self.n_scenes} scenes, {self.n_prims} prims, {self.n_nodes} nodes, depth {self.max_depth})"
