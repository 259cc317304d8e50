"""ctypes binding of libquadb200.so (include/quadb200.h).

The library is loaded lazily on first use and there is no fallback: if it is
missing, or no CUDA device is present, every entry point raises.  Structs
here mirror include/qb_params.h and include/quadb200.h field for field
(tests/test_native_abi.py checks sizes and exported symbols).
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QB_LIB_PATH") or os.path.join(_HERE, "libquadb200.so")  # override: A/B builds in scripts/

QB_F32, QB_F64 = 0, 1
CMD = {"srt": 0, "ctbr": 1, "ps": 2, "lv": 3, "rotor": 4}
TASKS = {"free": 0, "navigation": 1, "landing": 2, "gap_crossing": 3}
DISTS = {"fixed": 0, "uniform": 1, "normal": 2}

c_double3 = ctypes.c_double * 3


class QbParams(ctypes.Structure):
    _fields_ = [
        ("mass", ctypes.c_double),
        ("inertia", c_double3),
        ("gravity", c_double3),
        ("torque_arms", c_double3 * 4),
        ("thrust_coeffs", c_double3),
        ("drag_c", c_double3),
        ("rotor_lo", ctypes.c_double),
        ("rotor_hi", ctypes.c_double),
        ("alloc_inv", (ctypes.c_double * 4) * 4),
        ("thrust_lo", ctypes.c_double),
        ("thrust_hi", ctypes.c_double),
        ("hover_speed", ctypes.c_double),
        ("physics_dt", ctypes.c_double),
        ("half_dt", ctypes.c_double),
        ("sixth_dt", ctypes.c_double),
        ("lag_alpha", ctypes.c_double),
        ("substeps", ctypes.c_int32),
        ("integrator", ctypes.c_int32),
        ("rate_p", c_double3),
        ("attitude_p", c_double3),
        ("vel_p", c_double3),
        ("vel_d", c_double3),
        ("pos_p", c_double3),
        ("pos_d", c_double3),
        ("max_speed", ctypes.c_double),
        ("max_tilt_accel", ctypes.c_double),
    ]


class QbCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("tan_half_h", ctypes.c_double),
        ("tan_half_v", ctypes.c_double),
        ("max_range", ctypes.c_double),
        ("rotation", ctypes.c_double * 9),
        ("translation", c_double3),
        ("mode", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
    ]


class QbDist(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad_", ctypes.c_int32), ("a", c_double3), ("b", c_double3)]


class QbTask(ctypes.Structure):
    _fields_ = [
        ("task", ctypes.c_int32),
        ("auto_reset", ctypes.c_int32),
        ("episode_max_steps", ctypes.c_int32),
        ("n_scene_perm", ctypes.c_int32),
        ("scene_perm", ctypes.c_void_p),
        ("collision_radius", ctypes.c_double),
        ("min_spawn_clearance", ctypes.c_double),
        ("bounds_margin", ctypes.c_double),
        ("spawn", QbDist * 4),
        ("target", c_double3),
        ("success_radius", ctypes.c_double),
        ("w_progress", ctypes.c_double),
        ("w_speed", ctypes.c_double),
        ("w_obstacle", ctypes.c_double),
        ("safe_distance", ctypes.c_double),
        ("pad_center", ctypes.c_double * 2),
        ("pad_half", ctypes.c_double),
        ("success_height", ctypes.c_double),
        ("success_speed", ctypes.c_double),
        ("w_height", ctypes.c_double),
        ("w_speed_landing", ctypes.c_double),
        ("w_collision", ctypes.c_double),
        ("pad_top", ctypes.c_double),
        ("swarm", ctypes.c_int32),
        ("pad2_", ctypes.c_int32),
        ("targets", ctypes.c_void_p),
        ("w_agent", ctypes.c_double),
    ]


_P = ctypes.c_void_p


class QbEnvBuffers(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("index_offset", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("state", _P),
        ("prev_state", _P),
        ("action", _P),
        ("step_count", _P),
        ("agent_scene", _P),
        ("reset_count", _P),
        ("needs_respawn", _P),
        ("terminated", _P),
        ("truncated", _P),
        ("success", _P),
        ("collision", _P),
        ("out_of_bounds", _P),
        ("nonfinite", _P),
        ("reward", _P),
        ("nearest_dist", _P),
        ("nearest_pt", _P),
        ("rng", _P),
        ("error_count", _P),
    ]


QB_MAX_NOISE, QB_MAX_SENSORS = 4, 8
NOISE_KINDS = {"normal": 0, "poisson": 1, "saltpepper": 2, "speckle": 3, "redwood": 4}
SENSOR_KINDS = {"depth": 0, "segmentation": 1, "imu": 2}


class QbNoise(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("sigma", ctypes.c_double),
        ("p", ctypes.c_double),
        ("scaling", ctypes.c_double),
        ("sigma_disparity", ctypes.c_double),
        ("quantization", ctypes.c_double),
    ]


class QbSensorObs(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n_noise", ctypes.c_int32),
        ("noise", QbNoise * QB_MAX_NOISE),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("src", _P),
        ("out", _P),
    ]


class QbIoView(ctypes.Structure):
    _fields_ = [
        ("cam", QbCamera),
        ("depth", _P),
        ("seg", _P),
        ("seg_small", _P),
        ("centroid_id", ctypes.c_int32),
        ("seg_small_bytes", ctypes.c_int32),
        ("centroid", _P),
    ]


class QbIoCopy(ctypes.Structure):
    _fields_ = [("src", _P), ("dst", _P), ("bytes", ctypes.c_int64)]


class QbStepIo(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_int32),
        ("sync", ctypes.c_int32),
        ("host_action", _P),
        ("state_rows", _P),
        ("n_views", ctypes.c_int32),
        ("n_copies", ctypes.c_int32),
        ("views", _P),
        ("copies", _P),
        ("n_sensors", ctypes.c_int32),
        ("n_packs", ctypes.c_int32),
        ("sensors", _P),
        ("packs", _P),
    ]


# exported symbol -> (argtypes, restype)
_I64, _I32, _U64, _D = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
_PP = ctypes.POINTER
SIGNATURES = {
    "qb_last_error": ([], ctypes.c_char_p),
    "qb_version": ([], ctypes.c_int),
    "qb_device_sm_count": ([_PP(_I32)], ctypes.c_int),
    "qb_dynamics_step": ([_PP(QbParams), _I32, _I32, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_command_to_rotor_speeds": ([_PP(QbParams), _I32, _I32, _I64, _I64, _P, _P, _P, _P], ctypes.c_int),
    "qb_rollout_forward": ([_PP(QbParams), _I32, _I32, _I64, _I64, _I32, _P, _P, _P, _P], ctypes.c_int),
    "qb_rollout_backward": ([_PP(QbParams), _I32, _I32, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_dynamics_vjp": ([_PP(QbParams), _I32, _I32, _I64, _I64, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_scene_create": ([_I32, _P, _P, _P, _P, _P, _P, _PP(_P)], ctypes.c_int),
    "qb_scene_destroy": ([_P], ctypes.c_int),
    "qb_scene_create_device": ([_I32, _P, _P, _P, _P, _P, _P, _PP(_P), _P], ctypes.c_int),
    "qb_control_stage": ([_PP(QbParams), _I32, _I32, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_bvh_build": ([_I64, _P, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_scene_stats": ([_P, _P], ctypes.c_int),
    "qb_scene_bounds": ([_P, _I32, _P], ctypes.c_int),
    "qb_nearest_point": ([_P, _P, _I64, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "qb_raycast": ([_P, _I32, _P, _I64, _P, _P, _D, _D, _P, _P, _P], ctypes.c_int),
    "qb_render": ([_P, _PP(QbCamera), _I32, _I64, _I64, _P, _P, _P, _P, _I32, _P, _P, _P, _I32, _P], ctypes.c_int),
    "qb_render_poses": ([_P, _PP(QbCamera), _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _I32, _P], ctypes.c_int),
    "qb_env_reset": ([_PP(QbParams), _PP(QbTask), _P, _PP(QbEnvBuffers), _U64, _P], ctypes.c_int),
    "qb_env_step": ([_PP(QbParams), _I32, _PP(QbTask), _P, _PP(QbEnvBuffers), _P], ctypes.c_int),
    "qb_env_refresh": ([_PP(QbTask), _P, _PP(QbEnvBuffers), _P], ctypes.c_int),
    "qb_env_step_phase": ([_PP(QbParams), _I32, _PP(QbTask), _P, _PP(QbEnvBuffers), _I32, _P], ctypes.c_int),
    "qb_env_swarm_views": ([_PP(QbTask), _PP(QbEnvBuffers), _P, _P, _P, _P], ctypes.c_int),
    "qb_rng_seed": ([_U64, _I64, _P, _P], ctypes.c_int),
    "qb_rng_doubles": ([_I64, _P, _I32, _P, _P], ctypes.c_int),
    "qb_rng_normals": ([_I64, _P, _I32, _P, _P], ctypes.c_int),
    "qb_rng_poissons": ([_I64, _P, _I32, _P, _P, _P], ctypes.c_int),
    "qb_env_observe": ([_PP(QbParams), _PP(QbEnvBuffers), _I32, _P, _P], ctypes.c_int),
    "qb_env_step_io": ([_PP(QbParams), _I32, _PP(QbTask), _P, _PP(QbEnvBuffers), _PP(QbStepIo), _P], ctypes.c_int),
    "qb_env_step_graph_create": ([_PP(QbParams), _I32, _PP(QbTask), _P, _PP(QbEnvBuffers), _PP(QbStepIo), _PP(_P)],
                                 ctypes.c_int),
    "qb_env_step_graph_launch": ([_P, _I32, _P], ctypes.c_int),
    "qb_env_step_graph_destroy": ([_P], ctypes.c_int),
}

_lib = None


def load(require_cuda: bool = True):
    """Load libquadb200.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: build it with `python -m paper_2407_14783_b200.build` "
                          "(this package has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib():
    if _lib is None:
        load()
    return _lib


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().qb_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'libquadb200'} failed (status {rc}): {msg}")


def ptr(t) -> ctypes.c_void_p:
    """Device/host address of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_of(device=None) -> ctypes.c_void_p:
    """The current CUDA stream (of `device`, default the current device) as a
    raw handle -- through torch's C accessor, not a Stream object (the object
    path resolves the device index in Python: ~10 us per call)."""
    import torch

    idx = torch._C._cuda_getDevice() if device is None else torch.cuda._utils._get_device_index(device, optional=True)
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


def require_cuda(t=None):
    import torch

    if not torch.cuda.is_available():
        raise NativeError("paper_2407_14783_b200 runs on CUDA devices only (no CPU fallback); no GPU is visible")
    if t is not None and not t.is_cuda:
        raise NativeError("expected a CUDA tensor")
