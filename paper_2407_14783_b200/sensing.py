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
from . import quatmath

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


_rotate = quatmath.rotate
_matrix = quatmath.to_matrix


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
    ex = ex_ids = None
    k = 0
    if extra_spheres is not None and (extra_spheres.numel() if isinstance(extra_spheres, torch.Tensor)
                                      else np.asarray(extra_spheres).size):
        # per-view spheres [x y z r] + their ids (kernels.py:438-445: swarm agents, ids 60000 + j)
        ex = torch.as_tensor(extra_spheres, dtype=dtype, device=dev.device).reshape(n, -1, 4).contiguous()
        k = ex.shape[1]
        if extra_ids is None:
            raise ValueError("extra_spheres needs extra_ids")
        ex_ids = torch.as_tensor(extra_ids, device=dev.device).to(torch.int32).reshape(n, k).contiguous()
    with torch.cuda.device(dev.device):
        nat.check(nat.lib().qb_render_poses(dev.handle, camera.native(), code, n, nat.ptr(o), nat.ptr(r), nat.ptr(env_scene),
                                            nat.ptr(depth), nat.ptr(seg), nat.ptr(ex), nat.ptr(ex_ids), k,
                                            nat.stream_of()),
                  "qb_render_poses")
    if host:
        return depth.double().cpu().numpy(), seg.long().cpu().numpy()
    return depth, seg


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


# ---------------------------------------------------------------------------
# IMU (sensing.py:121-147)


@dataclass
class ImuReading:
    specific_force_b: object  # (N, 3) accelerometer, gravity excluded
    angvel_b: object  # (N, 3) gyro


def body_wrench(state, params):
    """Thrust + drag wrench at the current state (sensing.py:131-147), on the
    state's device: thrusts k2 w^2 + k1 w + k0, drag -c v_B |v_B| with
    v_B = R(q)^T v, force_z += t0 + t1 + t2 + t3, torque = sum_i t_i g_i."""
    import torch

    from .dynamics import Wrench

    planes = state.planes.double()
    k2, k1, k0 = params.thrust_coeffs
    w = planes[13:17]
    thr = k2 * w ** 2 + k1 * w + k0
    q, v = planes[6:10], planes[3:6]
    ux, uy, uz = -q[1], -q[2], -q[3]
    tx, ty, tz = uy * v[2] - uz * v[1], uz * v[0] - ux * v[2], ux * v[1] - uy * v[0]
    sx, sy, sz = uy * tz - uz * ty, uz * tx - ux * tz, ux * ty - uy * tx
    vb = torch.stack([v[0] + 2.0 * (q[0] * tx + sx), v[1] + 2.0 * (q[0] * ty + sy), v[2] + 2.0 * (q[0] * tz + sz)])
    c = torch.as_tensor(0.5 * params.air_density * np.asarray(params.drag_coeffs) * params.cross_area,
                        dtype=torch.float64, device=planes.device)[:, None]
    force = -c * vb * vb.abs()
    force[2] += thr[0] + thr[1] + thr[2] + thr[3]
    g = torch.as_tensor(np.asarray(params.torque_arms), dtype=torch.float64, device=planes.device)
    torque = torch.stack([thr[0] * g[0, a] + thr[1] * g[1, a] + thr[2] * g[2, a] + thr[3] * g[3, a] for a in range(3)])
    return Wrench(force.T, torque.T)


def imu_read(state, wrench, params) -> ImuReading:
    """Ideal IMU: specific force (f+d)/m in the body frame, gyro = body rates."""
    return ImuReading(wrench.force_b / params.mass, state.planes[10:13].T.double().clone())


# ---------------------------------------------------------------------------
# Noise models (sensing.py:150-235).  apply_noise runs on the device with the
# numpy Generator's own PCG64 state (read, advanced on the GPU, written back),
# drawing exactly what numpy would: ziggurat standard normals, PTRS/mult
# Poisson, next_double uniforms (csrc/qb_rng.cuh, qb_k_observe.cu).

DEPTH_KINDS = {"normal", "poisson", "saltpepper", "speckle", "redwood"}
IMAGE_KINDS = {"normal", "poisson", "saltpepper", "speckle"}
IMU_KINDS = {"normal"}
_SENSOR_KINDS = {"depth": DEPTH_KINDS, "rgb": IMAGE_KINDS, "segmentation": IMAGE_KINDS, "imu": IMU_KINDS}


@dataclass(frozen=True)
class NoiseSpec:
    """One noise model attachment (sensing.py:165-192).

    normal sigma (additive Gaussian), poisson scaling, saltpepper p,
    speckle sigma (multiplicative), redwood sigma_disparity + quantization
    (disparity domain, depth only)."""

    kind: str
    sigma: float = 0.0
    p: float = 0.0
    scaling: float = 1.0
    sigma_disparity: float = 0.0
    quantization: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "kind", self.kind.lower())
        if self.kind not in DEPTH_KINDS:
            raise ValueError(f"unknown noise kind {self.kind!r}")
        if min(self.sigma, self.p, self.scaling, self.sigma_disparity, self.quantization) < 0:
            raise ValueError("noise parameters must be nonnegative")
        if not 0.0 <= self.p <= 1.0:
            raise ValueError("saltpepper p must be in [0, 1]")

    def native(self):
        n = nat.QbNoise()
        n.kind = nat.NOISE_KINDS[self.kind]
        n.sigma, n.p, n.scaling = self.sigma, self.p, self.scaling
        n.sigma_disparity, n.quantization = self.sigma_disparity, self.quantization
        return n


def check_noise(spec: NoiseSpec, sensor: str):
    """The validity table of sensing.py:198-205."""
    from .errors import InvalidNoiseForSensor

    sensor = sensor.lower()
    if sensor not in _SENSOR_KINDS:
        raise InvalidNoiseForSensor(f"unknown sensor type {sensor!r}")
    if spec.kind not in _SENSOR_KINDS[sensor]:
        raise InvalidNoiseForSensor(f"noise {spec.kind!r} is not defined for {sensor!r} data")


def sensor_obs(kind: str, noise, out, src=None, width: int = 1, height: int = 1):
    """A qb_sensor_obs record (observation pass of one sensor)."""
    so = nat.QbSensorObs()
    so.kind = nat.SENSOR_KINDS["segmentation" if kind == "rgb" else kind]
    if len(noise) > nat.QB_MAX_NOISE:
        raise ValueError(f"at most {nat.QB_MAX_NOISE} noise models per sensor")
    so.n_noise = len(noise)
    for m, spec in enumerate(noise):
        so.noise[m] = spec.native()
    so.width, so.height = int(width), int(height)
    so.src = nat.ptr(src)
    so.out = nat.ptr(out)
    return so


def _pcg_words(bitgen):
    st = bitgen.state
    if st.get("bit_generator") != "PCG64":
        raise TypeError("apply_noise needs a numpy Generator on a PCG64 bit generator")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return [s >> 64, s & m, inc >> 64, inc & m]


def apply_noise(data, spec: NoiseSpec, rng, sensor: str = "depth"):
    """sensing.py:195-235 on the GPU, deterministic under (and advancing) the
    numpy Generator's state: same draws, same values as the reference.
    numpy in -> numpy float64 out; CUDA tensor in -> CUDA float64 tensor out."""
    import torch

    check_noise(spec, sensor)
    host = not isinstance(data, torch.Tensor)
    x = torch.as_tensor(np.asarray(data, dtype=float) if host else data, dtype=torch.float64)
    x = x.to(device=torch.device("cuda", torch.cuda.current_device()) if host else x.device).contiguous()
    out = torch.empty_like(x)
    words = _pcg_words(rng.bit_generator)
    rng_buf = torch.tensor([[w - (1 << 64) if w >= (1 << 63) else w for w in words]], dtype=torch.int64, device=x.device)
    planes = torch.zeros((17, 1), dtype=torch.float64, device=x.device)
    b = nat.QbEnvBuffers()
    b.n, b.ld, b.index_offset, b.dtype = 1, 1, 0, nat.QB_F64
    b.state, b.rng = planes.data_ptr(), rng_buf.data_ptr()
    # values are already float: run the chain as a float-image pass over size x 1
    so = sensor_obs("depth", (spec,), out, src=x, width=max(x.numel(), 1), height=1)
    if x.numel():
        from .params import native_params

        with torch.cuda.device(x.device):
            nat.check(nat.lib().qb_env_observe(native_params(), b, 1, ctypes_pointer(so), nat.stream_of()),
                      "qb_env_observe")
        w = [int(v) & ((1 << 64) - 1) for v in rng_buf[0].tolist()]
        st = rng.bit_generator.state
        st["state"]["state"] = (w[0] << 64) | w[1]
        rng.bit_generator.state = st
    return out.cpu().numpy() if host else out


def ctypes_pointer(obj):
    import ctypes

    return ctypes.cast(ctypes.pointer(obj), ctypes.c_void_p)


# ---------------------------------------------------------------------------
# 16-bit PGM export (sensing.py:238-274): millimeter depth, raw object ids.
# Host file I/O on observations copied back from the device.

PGM_MAXVAL = 65535


def _host(image):
    import torch

    return image.detach().cpu().numpy() if isinstance(image, torch.Tensor) else np.asarray(image)


def write_pgm16(path, image):
    """Binary 16-bit PGM (big-endian samples, PNM spec)."""
    image = _host(image)
    if image.ndim != 2:
        raise ValueError("expected a 2-D image")
    data = np.clip(np.round(image), 0, PGM_MAXVAL).astype(">u2")
    with open(path, "wb") as fh:
        fh.write(f"P5\n{image.shape[1]} {image.shape[0]}\n{PGM_MAXVAL}\n".encode())
        fh.write(data.tobytes())


def read_pgm16(path) -> np.ndarray:
    with open(path, "rb") as fh:
        magic = fh.readline().strip()
        if magic != b"P5":
            raise ValueError(f"not a binary PGM file: {magic!r}")
        width, height = (int(v) for v in fh.readline().split())
        maxval = int(fh.readline())
        data = np.frombuffer(fh.read(), dtype=">u2" if maxval > 255 else "u1", count=width * height)
    return data.reshape(height, width).astype(np.int64)


def export_depth_mm(path, depth_m):
    """Depth frame in millimeters, quantized to 16 bit."""
    write_pgm16(path, _host(depth_m).astype(np.float64) * 1000.0)


def export_segmentation(path, ids):
    write_pgm16(path, ids)
