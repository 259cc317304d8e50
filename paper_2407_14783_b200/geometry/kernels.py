"""geometry.kernels drop-in (kernels.py:120-182, 389-451): the reference's
flat-array entry points, served by the device kernels.

The BVH arrays the reference threads through every call are accepted and
ignored: the primitive table (prim_type, prim_data, prim_oid) is uploaded
once (cached by the array's identity) with the library's own BVH, and the
results -- nearest point / squared distance / object id, first hit t / id,
z-depth + id images -- do not depend on the tree.  Every entry point runs the
exact-double ("xd") kernels, so the outputs equal the reference's bit for
bit; the FP32 production renderer is what the environment path uses.
"""

from __future__ import annotations

import numpy as np

from .. import _native as nat

INF = np.inf
_SCENES = {}


class _Table:
    def __init__(self, t):
        self.arrays = t


def prim_aabbs(prim_type, prim_data):
    """Per-primitive AABBs from the reference's 16-double rows (shapes.py _rows)."""
    from .shapes import BOX, SPHERE

    t, d = np.asarray(prim_type), np.asarray(prim_data, dtype=np.float64)
    lo, hi = np.empty((len(t), 3)), np.empty((len(t), 3))
    s = t == SPHERE
    lo[s], hi[s] = d[s, :3] - d[s, 3:4], d[s, :3] + d[s, 3:4]
    b = t == BOX
    if b.any():
        reach = np.einsum("nij,nj->ni", np.abs(d[b, 6:15].reshape(-1, 3, 3)), d[b, 3:6])
        lo[b], hi[b] = d[b, :3] - reach, d[b, :3] + reach
    tri = ~(s | b)
    if tri.any():
        v = d[tri, :9].reshape(-1, 3, 3)
        lo[tri], hi[tri] = v.min(axis=1), v.max(axis=1)
    return lo, hi


def _device_scene(prim_type, prim_data, prim_oid):
    import torch

    from .device import DeviceScenes
    from .shapes import PrimTable

    dev = torch.cuda.current_device()
    key = (id(prim_data), prim_data.__array_interface__["data"][0], prim_data.shape, dev)
    hit = _SCENES.get(key)
    if hit is None:
        lo, hi = prim_aabbs(prim_type, prim_data)
        table = PrimTable(np.ascontiguousarray(prim_type, np.int64), np.ascontiguousarray(prim_data, np.float64),
                          np.ascontiguousarray(prim_oid, np.int64), lo, hi)
        hit = (DeviceScenes([_Table(table)], device=torch.device("cuda", dev)), prim_data)  # keep the key alive
        _SCENES[key] = hit
    return hit[0]


def nearest_point_query(node_lo, node_hi, node_first, node_count, prim_order, prim_type, prim_data, prim_oid, qx, qy, qz):
    """Returns (point x, y, z, distance^2, object id) (kernels.py:120-182)."""
    import torch

    dev = _device_scene(prim_type, prim_data, prim_oid)
    q = torch.tensor([[qx, qy, qz]], dtype=torch.float64, device=dev.device)
    pt = torch.empty((1, 3), dtype=torch.float64, device=dev.device)
    d2 = torch.empty(1, dtype=torch.float64, device=dev.device)
    oid = torch.empty(1, dtype=torch.int32, device=dev.device)
    with torch.cuda.device(dev.device):
        nat.check(nat.lib().qb_nearest_point(dev.handle, None, 1, nat.ptr(q), nat.ptr(pt), None, nat.ptr(oid), nat.ptr(d2),
                                             nat.stream_of()), "qb_nearest_point")
    p = pt.cpu().numpy()[0]
    return float(p[0]), float(p[1]), float(p[2]), float(d2.item()), np.int64(oid.item())


def raycast_query(node_lo, node_hi, node_first, node_count, prim_order, prim_type, prim_data, prim_oid,
                  ox, oy, oz, dx, dy, dz, tmin, tmax):
    """Returns (t, object id); t < 0 means no hit within (tmin, tmax] (kernels.py:389-399)."""
    import torch

    dev = _device_scene(prim_type, prim_data, prim_oid)
    o = torch.tensor([[ox, oy, oz]], dtype=torch.float64, device=dev.device)
    d = torch.tensor([[dx, dy, dz]], dtype=torch.float64, device=dev.device)
    t = torch.empty(1, dtype=torch.float64, device=dev.device)
    oid = torch.empty(1, dtype=torch.int32, device=dev.device)
    with torch.cuda.device(dev.device):
        nat.check(nat.lib().qb_raycast(dev.handle, nat.QB_F64, None, 1, nat.ptr(o), nat.ptr(d), float(tmin), float(tmax),
                                       nat.ptr(t), nat.ptr(oid), nat.stream_of()), "qb_raycast")
    tv = float(t.item())
    return (tv, np.int64(oid.item())) if tv > 0.0 else (-1.0, np.int64(-1))


def render_batch(node_lo, node_hi, node_first, node_count, prim_order, prim_type, prim_data, prim_oid,
                 origins, rotations, width, height, tan_half_h, tan_half_v, max_range, extra_spheres, extra_ids,
                 out_depth, out_id):
    """Pinhole z-depth + object-id render for a batch of camera poses
    (kernels.py:402-451); fills out_depth (A,H,W) and out_id (A,H,W) in place.
    origins (A,3), rotations (A,3,3) camera->world, extra_spheres (A,K,4)
    per-view spheres with extra_ids (A,K) (swarm agents)."""
    import torch

    dev = _device_scene(prim_type, prim_data, prim_oid)
    n = len(origins)
    cam = nat.QbCamera()
    cam.width, cam.height = int(width), int(height)
    cam.tan_half_h, cam.tan_half_v, cam.max_range = float(tan_half_h), float(tan_half_v), float(max_range)
    cam.rotation[:] = np.eye(3).reshape(9).tolist()  # poses are given camera->world
    td = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float64), device=dev.device)  # noqa: E731
    o, r = td(origins), td(np.asarray(rotations).reshape(n, 9))
    k = int(np.asarray(extra_spheres).shape[1]) if extra_spheres is not None and np.asarray(extra_spheres).ndim == 3 else 0
    ex = td(extra_spheres) if k else None
    ids = torch.as_tensor(np.asarray(extra_ids, np.int32), device=dev.device) if k else None
    depth = torch.empty((n, int(height), int(width)), dtype=torch.float64, device=dev.device)
    seg = torch.empty((n, int(height), int(width)), dtype=torch.int32, device=dev.device)
    with torch.cuda.device(dev.device):
        nat.check(nat.lib().qb_render_poses(dev.handle, cam, nat.QB_F64, n, nat.ptr(o), nat.ptr(r), None, nat.ptr(depth),
                                            nat.ptr(seg), nat.ptr(ex), nat.ptr(ids), k, nat.stream_of()),
                  "qb_render_poses")
    out_depth[...] = depth.cpu().numpy()
    out_id[...] = seg.cpu().numpy()
