"""Spatial queries over a Scene, executed by the sm_100a library.

Same signatures and semantics as the reference (geometry/queries.py:28-80):
`nearest_point` is the global closest surface point with ties to the lowest
object id (exact double, bit-identical to kernels.py:120-182), `raycast`
the nearest hit with t in (0, max_range].  The batched forms take / return
CUDA tensors and are what the env kernels use internally.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .. import _native as nat
from .shapes import Scene


@dataclass(frozen=True)
class ProximityResult:
    point: np.ndarray
    distance: float
    object_id: int


@dataclass(frozen=True)
class RayHit:
    t: float
    object_id: int


def nearest_points(scene_or_dev, queries, env_scene=None):
    """Batched nearest point: queries (N,3) -> (point (N,3) f64, distance (N,) f64, id (N,) int32) on device."""
    import torch

    dev = scene_or_dev.device() if isinstance(scene_or_dev, Scene) else scene_or_dev
    q = torch.as_tensor(queries, dtype=torch.float64, device=dev.device).reshape(-1, 3).contiguous()
    n = q.shape[0]
    pt = torch.empty((n, 3), dtype=torch.float64, device=q.device)
    d = torch.empty(n, dtype=torch.float64, device=q.device)
    oid = torch.empty(n, dtype=torch.int32, device=q.device)
    with torch.cuda.device(q.device):
        nat.check(nat.lib().qb_nearest_point(dev.handle, nat.ptr(env_scene), n, nat.ptr(q), nat.ptr(pt), nat.ptr(d),
                                             nat.ptr(oid), None, nat.stream_of()), "qb_nearest_point")
    return pt, d, oid


def raycasts(scene_or_dev, origins, directions, max_range: float, tmin: float = 0.0, dtype=None, env_scene=None):
    """Batched raycast: (N,3) origins / unit directions -> (t (N,), id (N,)); t = -1 on miss."""
    import torch

    dev = scene_or_dev.device() if isinstance(scene_or_dev, Scene) else scene_or_dev
    dtype = dtype or torch.float32
    o = torch.as_tensor(origins, dtype=dtype, device=dev.device).reshape(-1, 3).contiguous()
    d = torch.as_tensor(directions, dtype=dtype, device=dev.device).reshape(-1, 3).contiguous()
    n = o.shape[0]
    t = torch.empty(n, dtype=dtype, device=o.device)
    oid = torch.empty(n, dtype=torch.int32, device=o.device)
    code = nat.QB_F32 if dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(o.device):
        nat.check(nat.lib().qb_raycast(dev.handle, code, nat.ptr(env_scene), n, nat.ptr(o), nat.ptr(d), float(tmin),
                                       float(max_range), nat.ptr(t), nat.ptr(oid), nat.stream_of()), "qb_raycast")
    return t, oid


def nearest_point(scene: Scene, query) -> ProximityResult:
    pt, d, oid = nearest_points(scene, np.asarray(query, dtype=float).reshape(1, 3))
    return ProximityResult(pt[0].cpu().numpy(), float(d[0]), int(oid[0]))


def nearest_distances(scene: Scene, positions) -> np.ndarray:
    _, d, _ = nearest_points(scene, np.atleast_2d(np.asarray(positions, dtype=float)))
    return d.cpu().numpy()


def raycast(scene: Scene, origin, direction, max_range: float) -> Optional[RayHit]:
    import torch

    d = np.asarray(direction, dtype=float).reshape(3)
    n = np.linalg.norm(d)
    if abs(n - 1.0) > 1e-9:
        raise ValueError(f"direction must be unit length, |d| = {n}")
    t, oid = raycasts(scene, np.asarray(origin, float).reshape(1, 3), d.reshape(1, 3), max_range, dtype=torch.float64)
    if float(t[0]) < 0.0:
        return None
    return RayHit(float(t[0]), int(oid[0]))


def collision_check(scene: Scene, position, radius: float) -> bool:
    if radius <= 0:
        raise ValueError("radius must be > 0")
    return nearest_point(scene, position).distance < radius
