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


def flatten_on_device(scene, device):
    """shapes.py:139-212 (Scene -> SceneArrays rows) with the triangle meshes
    expanded on the device: one upload of all vertices and index triples,
    vertices[triangles] -> (T,16) rows and per-row AABBs scattered into the
    host flatten's row order, no host pass per triangle.  Spheres and boxes
    (a handful per scene) take the host rows.  Returns device tensors
    (type, data, oid, lo, hi)."""
    import torch

    from .shapes import PRIM_DATA_WIDTH, TRIANGLE, TriMesh, _rows

    objs = scene.objects
    if not objs:
        raise EmptyScene("scene has no objects")
    is_mesh = [isinstance(o.shape, TriMesh) for o in objs]
    counts = np.array([len(o.shape.triangles) if m else 1 for o, m in zip(objs, is_mesh)], np.int64)
    starts = np.concatenate([[0], np.cumsum(counts)])
    P = int(starts[-1])
    f64 = dict(dtype=torch.float64, device=device)
    data = torch.zeros((P, PRIM_DATA_WIDTH), **f64)
    lo, hi = torch.empty((P, 3), **f64), torch.empty((P, 3), **f64)
    kinds = np.zeros(len(objs), np.int64)
    meshes = [k for k, m in enumerate(is_mesh) if m]
    if meshes:
        voff = np.concatenate([[0], np.cumsum([len(objs[k].shape.vertices) for k in meshes])])
        v = torch.as_tensor(np.concatenate([objs[k].shape.vertices for k in meshes]), **f64)
        t = torch.as_tensor(np.concatenate([objs[k].shape.triangles + voff[j] for j, k in enumerate(meshes)]),
                            dtype=torch.int64, device=device)
        tri = v[t]  # (T,3,3)
        mc = torch.as_tensor(counts[meshes], device=device)
        first = torch.as_tensor(starts[meshes], device=device) - torch.as_tensor(np.concatenate([[0], np.cumsum(counts[meshes])[:-1]]), device=device)
        dst = torch.arange(len(t), device=device) + torch.repeat_interleave(first, mc)
        data[dst, :9] = tri.reshape(-1, 9)
        lo[dst], hi[dst] = tri.amin(dim=1), tri.amax(dim=1)
        kinds[meshes] = TRIANGLE
    others = [k for k, m in enumerate(is_mesh) if not m]
    if others:
        rows = [_rows(objs[k]) for k in others]
        kinds[others] = [r[0] for r in rows]
        dst = torch.as_tensor(starts[others], device=device)
        data[dst] = torch.as_tensor(np.concatenate([r[1] for r in rows]), **f64)
        lo[dst] = torch.as_tensor(np.concatenate([r[2] for r in rows]), **f64)
        hi[dst] = torch.as_tensor(np.concatenate([r[3] for r in rows]), **f64)
    cnt = torch.as_tensor(counts, device=device)
    ptype = torch.repeat_interleave(torch.as_tensor(kinds, device=device), cnt)
    poid = torch.repeat_interleave(torch.as_tensor([o.id for o in objs], dtype=torch.int64, device=device), cnt)
    return ptype, data, poid, lo, hi


class DeviceScenes:
    """S scenes on one device.  build="host": the host flatten + binned-SAH
    BVH (qb_scene_create, the default: the better tree for static scenes);
    build="device": flatten + linear BVH on the GPU (qb_scene_create_device,
    SURVEY F3) for scenes that change per episode -- same renders and query
    results bit for bit."""

    def __init__(self, scenes, device=None, build="host"):
        import torch

        nat.require_cuda()
        self.scenes = list(scenes)
        if not self.scenes:
            raise EmptyScene("no scenes")
        if build not in ("host", "device"):
            raise ValueError(f"build must be 'host' or 'device', got {build!r}")
        self.build = build
        self.device = torch.device("cuda", 0) if device is None else torch.device(device)
        handle = ctypes.c_void_p()
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        if build == "device":
            with torch.cuda.device(self.device):
                parts = [flatten_on_device(s, self.device) for s in self.scenes]
                offsets = np.zeros(len(parts) + 1, np.int64)
                offsets[1:] = np.cumsum([len(p[0]) for p in parts])
                ptype, pdata, poid, plo, phi = (torch.cat([p[k] for p in parts]).contiguous() for k in range(5))
                nat.check(nat.lib().qb_scene_create_device(
                    len(parts), P(offsets), ptype.data_ptr(), pdata.data_ptr(), poid.data_ptr(), plo.data_ptr(),
                    phi.data_ptr(), ctypes.byref(handle), nat.stream_of()), "qb_scene_create_device")
        else:
            tables = [s.arrays for s in self.scenes]
            counts = [len(t) for t in tables]
            if min(counts) == 0:
                raise EmptyScene("scene has no objects")
            offsets = np.zeros(len(tables) + 1, np.int64)
            offsets[1:] = np.cumsum(counts)
            cat = lambda name, dt: np.ascontiguousarray(np.concatenate([getattr(t, name) for t in tables]), dtype=dt)  # noqa: E731
            ptype, pdata, poid = cat("prim_type", np.int64), cat("prim_data", np.float64), cat("prim_object_id", np.int64)
            plo, phi = cat("prim_aabb_lo", np.float64), cat("prim_aabb_hi", np.float64)
            with torch.cuda.device(self.device):
                nat.check(nat.lib().qb_scene_create(len(tables), P(offsets), P(ptype), P(pdata), P(poid), P(plo), P(phi),
                                                    ctypes.byref(handle)), "qb_scene_create")
        self.handle = handle
        self._lib = nat.lib()
        stats = np.zeros(4, np.int64)
        nat.check(self._lib.qb_scene_stats(handle, P(stats)), "qb_scene_stats")
        self.n_nodes, self.n_prims, self.max_depth, self.n_scenes = (int(x) for x in stats)
        b = np.zeros((len(self.scenes), 6))
        for k in range(len(self.scenes)):
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
