"""Depth / segmentation cameras (reference sensing.py:20-114) on the K2 kernel.

Camera frame: +x right, +y down, +z forward; `rotation` is camera->body,
`translation` the camera origin in the body frame.  Depth is z-depth
(t * cz); pixels with no hit read exactly max_range and id 0; depth and ids
come from the same rays.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

FORWARD = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
DOWNWARD = np.array([[0.0, -1.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 0.0, -1.0]])


@dataclass(frozen=True)
class CameraModel:
    width: int = 64
    height: int = 64
    vertical_fov: float = math.pi / 2
    rotation: np.ndarray = field(default_factory=lambda: FORWARD.copy())
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    max_range: float = 10.0
    depth_convention: str = "zdepth"

    def __post_init__(self):
        object.__setattr__(self, "rotation", np.asarray(self.rotation, dtype=float).reshape(3, 3))
        object.__setattr__(self, "translation", np.asarray(self.translation, dtype=float).reshape(3))
        if self.width < 1 or self.height < 1:
            raise ValueError("camera resolution must be >= 1")
        if not (0.0 < self.vertical_fov < math.pi):
            raise ValueError("vertical_fov must be in (0, pi)")
        if self.depth_convention != "zdepth":
            raise ValueError("only the zdepth convention is implemented")

    @property
    def tan_half_v(self) -> float:
        return math.tan(self.vertical_fov / 2.0)

    @property
    def tan_half_h(self) -> float:
        return self.tan_half_v * self.width / self.height

    @property
    def focal_px(self) -> float:
        return (self.height / 2.0) / self.tan_half_v

    def native(self, mode: int = 0):
        """qb_camera; mode 0 auto, 1 BVH packet kernel, 2 frustum-culling kernel."""
        c = nat.QbCamera()
        c.mode = int(mode)
        c.width, c.height = int(self.width), int(self.height)
        c.tan_half_h, c.tan_half_v, c.max_range = self.tan_half_h, self.tan_half_v, float(self.max_range)
        c.rotation[:] = self.rotation.reshape(9).tolist()
        c.translation[:] = self.translation.tolist()
        return c


def _rotate(q, v):
    w = q[..., 0]
    ux, uy, uz = q[..., 1], q[..., 2], q[..., 3]
    vx, vy, vz = v[..., 0], v[..., 1], v[..., 2]
    tx, ty, tz = uy * vz - uz * vy, uz * vx - ux * vz, ux * vy - uy * vx
    sx, sy, sz = uy * tz - uz * ty, uz * tx - ux * tz, ux * ty - uy * tx
    return np.stack([vx + 2.0 * (w * tx + sx), vy + 2.0 * (w * ty + sy), vz + 2.0 * (w * tz + sz)], axis=-1)


def _matrix(q):
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([
        np.stack([1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)], -1),
        np.stack([2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)], -1),
        np.stack([2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)], -1),
    ], -2)


def camera_pose_world(body_position, body_orientation, camera: CameraModel):
    """World camera origins (n,3) and camera->world rotations (n,3,3) (sensing.py:66-74)."""
    pos = np.atleast_2d(np.asarray(body_position, dtype=float))
    quat = np.atleast_2d(np.asarray(body_orientation, dtype=float))
    origins = pos + _rotate(quat, np.broadcast_to(camera.translation, pos.shape))
    rot = np.einsum("nij,jk->nik", _matrix(quat), camera.rotation)
    return origins, np.ascontiguousarray(rot)


def render_frames(scene, body_position, body_orientation, camera: CameraModel, extra_spheres=None, extra_ids=None,
                  dtype=None, env_scene=None):
    """Depth + id images for a batch of body poses (sensing.py:77-100).

    numpy poses -> numpy (depth float, ids int64) like the reference; CUDA
    tensor poses -> CUDA tensors (depth float32/64, ids int32).  dtype
    float64 selects the exact-double validation renderer.
    """
    import torch

    host = not isinstance(body_position, torch.Tensor)
    dev = scene.device() if hasattr(scene, "objects") else scene
    if host:
        origins, rots = camera_pose_world(body_position, body_orientation, camera)
    else:
        origins, rots = camera_pose_world(body_position.detach().double().cpu().numpy(),
                                          body_orientation.detach().double().cpu().numpy(), camera)
    dtype = dtype or torch.float32
    n = origins.shape[0]
    o = torch.as_tensor(origins, dtype=dtype, device=dev.device).contiguous()
    r = torch.as_tensor(rots, dtype=dtype, device=dev.device).contiguous()
    depth = torch.empty((n, camera.height, camera.width), dtype=dtype, device=dev.device)
    seg = torch.empty((n, camera.height, camera.width), dtype=torch.int32, device=dev.device)
    code = nat.QB_F32 if dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(dev.device):
        if extra_spheres is not None and np.asarray(extra_spheres).size:
            # swarm spheres need per-view poses inside the kernel: go through the state path
            return _render_with_extra(dev, o, r, camera, extra_spheres, extra_ids, host, dtype)
        nat.check(nat.lib().qb_render_poses(dev.handle, camera.native(), code, n, nat.ptr(o), nat.ptr(r), nat.ptr(env_scene),
                                            nat.ptr(depth), nat.ptr(seg), nat.stream_of()), "qb_render_poses")
    if host:
        return depth.double().cpu().numpy(), seg.long().cpu().numpy()
    return depth, seg


def _render_with_extra(dev, o, r, camera, extra, extra_ids, host, dtype):
    raise NotImplementedError("extra spheres through render_frames: use the env swarm path (F2)")


def render_depth(scene, body_position, body_orientation, camera: CameraModel):
    single = np.asarray(body_position).ndim == 1
    d, _ = render_frames(scene, body_position, body_orientation, camera)
    return d[0] if single else d


def render_segmentation(scene, body_position, body_orientation, camera: CameraModel):
    single = np.asarray(body_position).ndim == 1
    _, s = render_frames(scene, body_position, body_orientation, camera)
    return s[0] if single else s


def render_state(dev_scenes, camera: CameraModel, planes, env_scene=None, depth=None, seg=None, centroid_id: int = 0,
                 centroid=None, extra=None, extra_ids=None, mode: int = 0):
    """K2 straight from the (17,N) state planes (the env observation path).

    mode: 0 auto (frustum-culling kernel for scenes <= 256 primitives, BVH
    packet kernel otherwise), 1 force BVH, 2 force culling."""
    import torch

    n = planes.shape[1]
    code = nat.QB_F32 if planes.dtype == torch.float32 else nat.QB_F64
    k = 0 if extra is None else extra.shape[1]
    nat.check(nat.lib().qb_render(dev_scenes.handle, camera.native(mode), code, n, planes.stride(0), nat.ptr(planes),
                                  nat.ptr(env_scene), nat.ptr(depth), nat.ptr(seg), int(centroid_id), nat.ptr(centroid),
                                  nat.ptr(extra), nat.ptr(extra_ids), k, nat.stream_of()), "qb_render")
    return depth, seg
