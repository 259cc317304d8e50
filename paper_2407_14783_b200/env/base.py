"""Gym-shaped batched environment on the GPU (reference env/base.py).

`QuadEnvBase` keeps the reference surface -- `reset(seed) -> observations`,
`step(action) -> StepResult(observations, reward, terminated, truncated,
info)`, the task hooks, `state` / `prev_state` / `nearest_dist` /
`nearest_pt` / flags -- but a step is two kernel launches on the current
stream, with no host synchronisation:

  1. qb_env_step   (K1+K3 fused: auto-reset, controller, dynamics, proximity,
                    task reward / success, terminated / truncated)
  2. qb_render     (K2, once per distinct camera: depth + segmentation from the
                    same rays, landing pad centroid in the epilogue)

Small camera batches (<= 9472 agents, the warp-per-env range) split step 1
into qb_env_step_phase 1 (auto-reset, controller, dynamics) and phase 2
(proximity, reward, flags) on a side stream that runs under the render and
joins before step() returns (`split_step`; results bit-equal to the fused
launch).

Observations and flags are device tensors.  `observations[i]` / `info[i]`
materialise the reference's per-agent dicts on demand (a host copy), so code
written against the reference keeps working; batched consumers index by key
(`observations["depth"]`) and never leave the GPU.  Like the reference's
fresh per-step arrays, a StepResult does not change when the env steps on:
reward / flags / info are a one-copy snapshot of the step's output block and
the state observation a snapshot of the planes; rendered frames are
double-buffered (valid through the next step, StaleObservations after that
unless materialised or cloned).

Sharding: an env built with `shard=(rank, world)` owns the contiguous global
index range [rank*N/world, (rank+1)*N/world).  Streams are keyed by the
global index, so env i evolves identically for any world size.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass

import os

import numpy as np

from .. import _native as nat
from ..control import COMMAND_TYPES
from ..dynamics import QuadState
from ..errors import ActionShapeMismatch, ConfigError, NotReset, SpawnFailure
from ..geometry.device import DeviceScenes
from ..params import ControllerGains, QuadParams, SimConfig, native_params
from ..sensing import render_state
from ..sharding import shard_range

DRONE_ID0 = 60000


class StaleObservations(RuntimeError):
    """Observations indexed after the env overwrote their buffers."""


class Observations(Sequence):
    """Batched observation dict that also indexes like the reference list.

    obs["depth"] -> (N,H,W) CUDA tensor; obs[i] -> {"state": (13,), ...} numpy
    dict for agent i (reference layout, float64, segmentation cast to float).

    The reference returns fresh arrays every step (base.py:287-310).  Here the
    state is a per-step snapshot and the rendered images live in one of two
    buffer sets the env alternates between, so the observations of step k stay
    valid through step k+1 (the usual act-then-step loop) without copying
    2 GB of frames per step at config 3.  Step k+2 overwrites them: indexing
    an Observations that old raises StaleObservations -- except obs[i] once it
    was materialised (obs[i] / as_reference() copy everything to the host on
    first use) -- and `clone()` gives a device copy that never goes stale.
    """

    def __init__(self, data: dict, n: int, seg_keys=(), env=None, gen: int = 0):
        self._data = data
        self._n = n
        self._seg_keys = set(seg_keys)
        self._host = None
        self._env = env
        self._gen = gen

    def _check_fresh(self):
        if self._env is not None and self._env._obs_gen - self._gen >= 2:
            raise StaleObservations(f"observations of step {self._gen} were overwritten by step {self._env._obs_gen}: "
                                    f"index or clone() them before stepping twice (the env double-buffers its frames)")

    def keys(self):
        return self._data.keys()

    def items(self):
        self._check_fresh()
        return self._data.items()

    def __contains__(self, key):
        return key in self._data if isinstance(key, str) else super().__contains__(key)

    def __len__(self):
        return self._n

    def clone(self) -> "Observations":
        """A device copy that the env never overwrites."""
        self._check_fresh()
        return Observations({k: v.clone() for k, v in self._data.items()}, self._n, self._seg_keys)

    def _materialize(self):
        if self._host is None:
            self._check_fresh()
            self._host = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in self._data.items()}
        return self._host

    def __getitem__(self, key):
        if isinstance(key, str):  # the device tensor itself: valid through the next step only
            self._check_fresh()
            return self._data[key]
        if isinstance(key, slice):
            return [self[i] for i in range(*key.indices(self._n))]
        h = self._materialize()
        i = int(key)
        if not -self._n <= i < self._n:
            raise IndexError(i)
        return {k: v[i] for k, v in h.items()}

    def as_reference(self) -> list:
        """The reference's list of per-agent dicts (base.py:287-310)."""
        return [self[i] for i in range(self._n)]


class Info(Sequence):
    """Per-agent info dicts (base.py:195-207), materialised lazily from the
    step's own snapshot (later steps never change them)."""

    _KEYS = ("success", "collision", "out_of_bounds", "nonfinite", "nearest_distance", "scene", "step")

    def __init__(self, data, n: int):
        self._data = data  # a dict, or a callable building it on first use (per-step views are not free)
        self._n = n
        self._host = None

    @property
    def data(self) -> dict:
        if callable(self._data):
            self._data = self._data()
        return self._data

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, str):
            return self.data[i]
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(self._n))]
        if self._host is None:
            self._host = {k: self.data[k].detach().cpu().numpy() for k in self._KEYS}
        h = self._host
        i = int(i)
        if not -self._n <= i < self._n:
            raise IndexError(i)
        return {
            "success": bool(h["success"][i]), "collision": bool(h["collision"][i]),
            "out_of_bounds": bool(h["out_of_bounds"][i]), "nonfinite": bool(h["nonfinite"][i]),
            "nearest_distance": float(h["nearest_distance"][i]), "scene": int(h["scene"][i]), "step": int(h["step"][i]),
        }


class _Snapshot:
    """Holder of the typed views of one step's output snapshot."""


@dataclass
class StepResult:
    """base.py:37-43.  reward / terminated / truncated / info are this step's
    own device tensors (a snapshot: later steps do not change them);
    as_reference() converts to the reference's numpy / list-of-dict form."""

    observations: Observations
    reward: object
    terminated: object
    truncated: object
    info: Info

    def as_reference(self):
        cpu = lambda t: t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)  # noqa: E731
        return StepResult(self.observations.as_reference(), cpu(self.reward).astype(np.float64),
                          cpu(self.terminated).astype(bool), cpu(self.truncated).astype(bool),
                          [self.info[i] for i in range(len(self.info))])


def _dist(d, spec):
    d.kind = nat.DISTS[spec.kind]
    if spec.kind == "fixed":
        d.a[:] = spec.value.tolist()
    elif spec.kind == "uniform":
        d.a[:], d.b[:] = spec.low.tolist(), spec.high.tolist()
    else:
        d.a[:], d.b[:] = spec.mean.tolist(), spec.sigma.tolist()


class QuadEnvBase:
    """Batched quadrotor environment; tasks override the three hooks."""

    TASK = "free"

    def __init__(self, config, params: QuadParams = None, sim: SimConfig = None, gains: ControllerGains = None,
                 device=None, dtype=None, shard=(0, 1), track_prev_state: bool = True, scene_build: str = "host"):
        import torch

        nat.require_cuda()
        self.swarm = config.mode == "swarm"
        if self.swarm and shard[1] != 1:
            raise ConfigError("swarm mode runs one swarm per env (all agents interact): replicate envs across ranks "
                              "instead of sharding one")
        if self.swarm and not track_prev_state:
            raise ConfigError("swarm mode needs prev_state tracking")
        self.config = config
        self.params = params if params is not None else QuadParams()
        self.sim = sim if sim is not None else SimConfig()
        self.gains = gains if gains is not None else ControllerGains()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._dev_idx = self.device.index
        self.dtype = dtype or torch.float32
        rank, world = shard
        total = config.num_agents
        lo, hi = shard_range(rank, world, total)
        self.global_num_agents = total
        self.index_offset = lo
        self.num_agents = hi - lo
        self.scenes = [spec.materialize() for spec in config.scenes]
        self.sensor_cameras = [(s, None if s.kind == "imu" else s.camera()) for s in config.sensors]
        with torch.cuda.device(self.device):
            self.dev_scenes = DeviceScenes(self.scenes, device=self.device, build=scene_build)
        self._P = native_params(self.params, self.sim, self.gains)
        self._kind = nat.CMD[config.command_type]
        self._alloc(track_prev_state)
        self._task = self._pack_task()
        self._reset_done = False
        self._custom_hooks = self._has_custom_hooks()
        # small batches with a camera: step in two launches so the proximity /
        # reward phase runs on a side stream under the observation render
        # (qb_env_step_phase; both read only the post-dynamics state)
        self.split_step = (not self.swarm and self._prev is not None and any(c is not None for _, c in self.sensor_cameras)
                           and self.num_agents * 32 <= torch.cuda.get_device_properties(self.device).multi_processor_count * 2048)
        if os.environ.get("QB_SPLIT_STEP") == "0":  # A/B switch
            self.split_step = False
        self._post_stream = None

    # ------------------------------------------------------------------ setup
    def _cur_stream(self):
        """The device's current torch Stream, re-fetched only when the raw
        current stream changed (torch.cuda.current_stream() costs ~10 us)."""
        import torch

        raw = torch._C._cuda_getCurrentRawStream(self._dev_idx)
        if raw != getattr(self, "_stream_raw", None):
            self._stream_obj = torch.cuda.current_stream(self.device)
            self._stream_raw = raw
        return self._stream_obj

    def _devctx(self):
        """torch.cuda.device(self.device) unless it is already current (the
        context manager costs several microseconds per step)."""
        import contextlib

        import torch

        if torch._C._cuda_getDevice() == self._dev_idx:
            return contextlib.nullcontext()
        return torch.cuda.device(self.device)

    def _has_custom_hooks(self) -> bool:
        # a user subclass overriding the Lst-1 hooks gets them called after
        # the fused kernel (flags are then recombined on the device)
        return (type(self).get_reward is not QuadEnvBase.get_reward
                or type(self).get_success is not QuadEnvBase.get_success)

    def _alloc(self, track_prev):
        import torch

        n, dev, dt = self.num_agents, self.device, self.dtype
        z = lambda *shape, dtype=torch.uint8: torch.zeros(shape, dtype=dtype, device=dev)  # noqa: E731
        self._planes = torch.zeros((17, n), dtype=dt, device=dev)
        self._prev = torch.zeros((17, n), dtype=dt, device=dev) if track_prev else None
        self._action = torch.zeros((n, 4), dtype=dt, device=dev)
        # host actions go through two pinned staging buffers; a buffer is only
        # refilled once the device has consumed its previous copy (event), so
        # a host loop may run ahead of the GPU without corrupting actions
        self._action_host = [torch.zeros((n, 4), dtype=dt, pin_memory=True) for _ in range(2)]
        self._action_host_np = [b.numpy() for b in self._action_host]  # (host-side writes without torch ops)
        self._action_host_ev = [None, None]
        self._action_host_i = 0
        # per-step outputs in ONE allocation: a StepResult snapshots them with one copy
        self._outblk = z(self._outblk_bytes(n))
        self._outblk_lay = self._outblk_layout(n)[0]
        self._out_views(self._outblk, self)
        self._reset_counts = z(n, dtype=torch.int32)
        self._rng = z(n, 4, dtype=torch.int64)
        self._errors = z(1, dtype=torch.int32)
        self._scene_perm = z(len(self.scenes), dtype=torch.int32)
        # observation buffers: one render per distinct camera, two buffer sets
        # (step k renders into set k % 2: the previous step's frames stay valid)
        self._cams, self._sensor_slot = {}, {}
        for spec, cam in self.sensor_cameras:
            if cam is None:
                continue
            key = (cam.width, cam.height, cam.vertical_fov, tuple(cam.rotation.ravel()), tuple(cam.translation), cam.max_range)
            if key not in self._cams:
                self._cams[key] = {"camera": cam, "depth": None, "seg": None, "centroid": None, "names": []}
            slot = self._cams[key]
            self._sensor_slot[spec.name] = slot
            if spec.kind == "depth" and slot["depth"] is None:
                slot["depth_pair"] = [torch.zeros((n, cam.height, cam.width), dtype=dt, device=dev) for _ in range(2)]
            if spec.kind == "segmentation" and slot["seg"] is None:
                slot["seg_pair"] = [torch.zeros((n, cam.height, cam.width), dtype=torch.int32, device=dev) for _ in range(2)]
            for k in ("depth", "seg"):
                if slot.get(k + "_pair"):
                    slot[k] = slot[k + "_pair"][0]
            if not spec.noise:
                slot["names"].append((spec.name, spec.kind))
        for slot in self._cams.values():
            if self._centroid_id(slot):
                slot["centroid_pair"] = [torch.zeros((n, 2), dtype=torch.float32, device=dev) for _ in range(2)]
                slot["centroid"] = slot["centroid_pair"][0]
        # the observation pass (qb_env_observe): IMU readings and noisy camera
        # sensors, in config order -- the order their draws leave each env's
        # generator (base.py:287-305)
        self._obs_sensors, self._noise_error = [], None
        from ..sensing import check_noise, sensor_obs

        for spec, cam in self.sensor_cameras:
            try:
                for nz in spec.noise:
                    check_noise(nz, spec.kind)
            except Exception as e:  # the reference raises on the first observation
                self._noise_error = self._noise_error or e
            outs, recs = [], []
            for i in range(2):
                if spec.kind == "imu":
                    out = torch.zeros((n, 6), dtype=dt, device=dev)
                    rec = sensor_obs("imu", spec.noise, out)
                elif spec.noise:
                    slot = self._sensor_slot[spec.name]
                    out = torch.zeros((n, cam.height, cam.width), dtype=dt, device=dev)
                    src = slot["depth_pair"][i] if spec.kind == "depth" else slot["seg_pair"][i]
                    rec = sensor_obs(spec.kind, spec.noise, out, src=src, width=cam.width, height=cam.height)
                else:
                    break
                outs.append(out)
                recs.append(rec)
            if outs:
                self._obs_sensors.append({"name": spec.name, "kind": spec.kind, "out": outs[0], "outs": outs,
                                          "recs": recs})
        if self._obs_sensors:
            self._obs_arrays = [(nat.QbSensorObs * len(self._obs_sensors))(*[o["recs"][i] for o in self._obs_sensors])
                                for i in range(2)]
            self._obs_array = self._obs_arrays[0]
        # swarm mode: the other agents as render spheres + the swarm observation
        self._swarm_spheres = self._swarm_ids = self._swarm_obs = None
        if self.swarm and n > 1:
            self._swarm_spheres = torch.zeros((n, n - 1, 4), dtype=dt, device=dev)
            self._swarm_ids = torch.zeros((n, n - 1), dtype=torch.int32, device=dev)
            self._swarm_obs_pair = [torch.zeros((n, n - 1, 13), dtype=dt, device=dev) for _ in range(2)]
            self._swarm_obs = self._swarm_obs_pair[0]
        self._obs_i, self._obs_gen = 0, 0
        bufs = nat.QbEnvBuffers()
        bufs.n, bufs.ld, bufs.index_offset = n, n, self.index_offset
        bufs.dtype = nat.QB_F32 if dt == torch.float32 else nat.QB_F64
        for field, t in (("state", self._planes), ("prev_state", self._prev), ("action", self._action),
                         ("step_count", self.step_counts), ("agent_scene", self.agent_scene), ("reset_count", self._reset_counts),
                         ("needs_respawn", self._needs_respawn), ("terminated", self._terminated),
                         ("truncated", self._truncated), ("success", self._success), ("collision", self._collision),
                         ("out_of_bounds", self._oob), ("nonfinite", self._nonfinite), ("reward", self._reward),
                         ("nearest_dist", self.nearest_dist), ("nearest_pt", self.nearest_pt), ("rng", self._rng),
                         ("error_count", self._errors)):
            setattr(bufs, field, None if t is None else t.data_ptr())
        self._bufs = bufs

    # per-step output block: flags (7 x n u8) | reward f32 | step i32 | scene i32 | nearest dist f64 | point f64 x 3
    @staticmethod
    def _outblk_layout(n):
        r8 = lambda x: (x + 7) // 8 * 8  # noqa: E731
        off, lay = 0, {}
        for name, nbytes in (("flags", 7 * n), ("reward", 4 * n), ("step", 4 * n), ("scene", 4 * n),
                             ("dist", 8 * n), ("pt", 24 * n)):
            lay[name] = (off, off + nbytes)
            off = r8(off + nbytes)
        return lay, off

    @classmethod
    def _outblk_bytes(cls, n):
        return max(cls._outblk_layout(n)[1], 8)

    def _out_views(self, blk, into):
        """Typed views of a per-step output block (the env's own, or a snapshot)."""
        import torch

        n = self.num_agents
        lay, _ = self._outblk_layout(n)
        v = lambda k, dt: blk[lay[k][0]:lay[k][1]].view(dt)  # noqa: E731
        flags = v("flags", torch.uint8).view(7, n)
        (into._needs_respawn, into._terminated, into._truncated, into._success, into._collision, into._oob,
         into._nonfinite) = flags.unbind(0)
        into._flags = flags
        into._reward = v("reward", torch.float32)
        into.step_counts = v("step", torch.int32)
        into.agent_scene = v("scene", torch.int32)
        into.nearest_dist = v("dist", torch.float64)
        into.nearest_pt = v("pt", torch.float64).view(n, 3)
        return into

    def _flip_observation_buffers(self):
        """Step k renders into buffer set k % 2 (see Observations)."""
        self._obs_i ^= 1
        i = self._obs_i
        for slot in self._cams.values():
            for k in ("depth", "seg", "centroid"):
                if slot.get(k + "_pair"):
                    slot[k] = slot[k + "_pair"][i]
        for o in self._obs_sensors:
            o["out"] = o["outs"][i]
        if self._obs_sensors:
            self._obs_array = self._obs_arrays[i]
        if self._swarm_obs is not None:
            self._swarm_obs = self._swarm_obs_pair[i]
        self._obs_gen += 1

    def _pack_task(self):
        c = self.config
        t = nat.QbTask()
        t.task = nat.TASKS[self.TASK]
        t.auto_reset = int(bool(c.auto_reset))
        t.episode_max_steps = int(c.episode_max_steps)
        t.n_scene_perm = len(self.scenes)
        t.scene_perm = self._scene_perm.data_ptr()
        t.collision_radius, t.min_spawn_clearance, t.bounds_margin = c.collision_radius, c.min_spawn_clearance, c.bounds_margin
        t.swarm = int(self.swarm)
        r = c.randomization
        for k, spec in enumerate((r.position, r.velocity, r.orientation, r.angvel)):
            _dist(t.spawn[k], spec)
        self._task_fields(t)
        return t

    def _task_fields(self, t):
        """Task subclasses fill their qb_task section."""

    # ------------------------------------------------------------------ hooks
    def get_reward(self):
        return self._reward

    def get_success(self):
        return self._success.bool()

    def _extra_observations(self, obs: dict):
        """Task subclasses add their observation keys (e.g. target)."""

    # ------------------------------------------------------------------ state views
    @property
    def state(self) -> QuadState:
        return QuadState(self._planes)

    @property
    def prev_state(self) -> QuadState:
        if self._prev is None:
            raise AttributeError("prev_state tracking disabled (track_prev_state=False)")
        return QuadState(self._prev)

    collision = property(lambda s: s._collision.bool())
    out_of_bounds = property(lambda s: s._oob.bool())
    nonfinite = property(lambda s: s._nonfinite.bool())

    # ------------------------------------------------------------------ reset / step
    def reset(self, seed: int = 0) -> Observations:
        """Fresh initial states for every agent; deterministic per seed (base.py:93-112)."""
        self._reset_state(seed)
        return self.get_observation()

    def _reset_state(self, seed: int):
        """reset() without the observation: scene permutation, spawns, proximity."""
        import torch

        s = len(self.scenes)
        perm = np.random.default_rng(int(seed)).permutation(s) if self.config.scene_sampling == "shuffled" else np.arange(s)
        with torch.cuda.device(self.device):
            self._scene_perm.copy_(torch.as_tensor(perm, dtype=torch.int32))
            self._errors.zero_()
            nat.check(nat.lib().qb_env_reset(self._P, self._task, self.dev_scenes.handle, self._bufs, int(seed) & (2**64 - 1),
                                             nat.stream_of()), "qb_env_reset")
            nfail = int(self._errors.item())  # reset is allowed to synchronise
        if nfail:
            raise SpawnFailure(f"{nfail} agents: no spawn with clearance >= {self.config.min_spawn_clearance} in 1000 attempts")
        self._reset_done = True
        self._pending_errors = None

    def _stage_action(self, action):
        import torch

        expected = COMMAND_TYPES[self.config.command_type]
        if not isinstance(action, expected):
            raise ActionShapeMismatch(f"expected {expected.__name__} commands (config command_type="
                                      f"{self.config.command_type!r}), got {type(action).__name__}")
        arr = action.as_array()
        if arr.shape[0] != self.num_agents:
            raise ActionShapeMismatch(f"action batch {arr.shape[0]} != num_agents {self.num_agents}")
        if isinstance(arr, torch.Tensor) and arr.is_cuda:
            if arr.dtype == self.dtype and arr.is_contiguous() and arr.device == self.device:
                return arr
            self._action.copy_(arr)
            return self._action
        k = self._action_host_i
        self._action_host_i ^= 1
        if self._action_host_ev[k] is not None:
            self._action_host_ev[k].synchronize()
        buf = self._action_host[k]
        np.copyto(self._action_host_np[k], np.asarray(arr), casting="unsafe")
        self._action.copy_(buf, non_blocking=True)
        ev = self._action_host_ev[k] or torch.cuda.Event()
        ev.record(self._cur_stream())
        self._action_host_ev[k] = ev
        return self._action

    def step(self, action) -> StepResult:
        """One control step for every agent (base.py:156-210), asynchronous."""
        import torch

        if not self._reset_done:
            raise NotReset("call reset() before step()")
        if self._noise_error is not None:  # before any launch (the reference raises on the first observation)
            raise self._noise_error
        self._check_async_errors()
        a = self._stage_action(action)
        self._bufs.action = a.data_ptr()
        with self._devctx():
            if self.split_step:
                join = self._launch_split_dynamics()
                try:
                    self._record_async_errors()
                    obs = self.get_observation()
                finally:  # phase 2 always rejoins the main stream
                    join()
            else:
                nat.check(nat.lib().qb_env_step(self._P, self._kind, self._task, self.dev_scenes.handle, self._bufs,
                                                nat.stream_of()), "qb_env_step")
                self._record_async_errors()
                obs = self.get_observation()
        if self._custom_hooks:
            success = torch.as_tensor(self.get_success(), device=self.device).bool()
            reward = torch.as_tensor(self.get_reward(), device=self.device)
            terminated = success | self.collision | self.out_of_bounds | self.nonfinite
            truncated = ~terminated & (self.step_counts >= self.config.episode_max_steps)
            self._needs_respawn.copy_((terminated | truncated).to(torch.uint8))
        # this step's outputs, snapshotted with one device copy: the reference
        # returns fresh arrays per step (base.py:186-210); the Info views are
        # built on first use
        blk = self._outblk.clone()
        n = self.num_agents
        lay = self._outblk_lay
        flags = blk[lay["flags"][0]:lay["flags"][1]].view(7, n).view(torch.bool)
        if not self._custom_hooks:
            success, reward = flags[3], blk[lay["reward"][0]:lay["reward"][1]].view(torch.float32)
            terminated, truncated = flags[1], flags[2]

        def info_views(blk=blk, flags=flags, success=success):
            snap = self._out_views(blk, _Snapshot())
            return {"success": success, "collision": flags[4], "out_of_bounds": flags[5], "nonfinite": flags[6],
                    "nearest_distance": snap.nearest_dist, "scene": snap.agent_scene, "step": snap.step_counts}

        return StepResult(obs, reward, terminated, truncated, Info(info_views, n))

    def _record_async_errors(self):
        import torch

        if getattr(self, "_err_host", None) is None:
            self._err_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._err_event = torch.cuda.Event()
        self._err_host.copy_(self._errors, non_blocking=True)
        self._err_event.record(self._cur_stream())
        self._pending_errors = True

    def _check_async_errors(self):
        if getattr(self, "_pending_errors", None) and self._err_event.query() and int(self._err_host[0]) > 0:
            n = int(self._err_host[0])
            self._errors.zero_()
            raise SpawnFailure(f"{n} respawns found no spawn with clearance >= {self.config.min_spawn_clearance}")

    def _render_and_observe(self):
        """Launch the observation kernels into the next buffer set: K2 once per
        distinct camera, then the sensor pass (IMU + noise chains) if any
        sensor needs it."""
        self._flip_observation_buffers()
        self._render()
        self._observe()

    def _render(self):
        if self._swarm_obs is not None:  # other agents as spheres + swarm states (base.py:245-277, 306-309)
            nat.check(nat.lib().qb_env_swarm_views(self._task, self._bufs, nat.ptr(self._swarm_spheres),
                                                   nat.ptr(self._swarm_ids), nat.ptr(self._swarm_obs), nat.stream_of()),
                      "qb_env_swarm_views")
        for slot in self._cams.values():
            cid = self._centroid_id(slot)
            render_state(self.dev_scenes, slot["camera"], self._planes, env_scene=self.agent_scene, depth=slot["depth"],
                         seg=slot["seg"], centroid_id=cid, centroid=slot["centroid"] if cid else None,
                         extra=self._swarm_spheres, extra_ids=self._swarm_ids)

    def _observe(self):
        if self._obs_sensors:
            import ctypes

            nat.check(nat.lib().qb_env_observe(self._P, self._bufs, len(self._obs_sensors),
                                               ctypes.cast(self._obs_array, ctypes.c_void_p), nat.stream_of()),
                      "qb_env_observe")

    def get_observation(self) -> Observations:
        """Render every camera once, run the sensor pass and assemble the
        batched observation dict."""
        if self._noise_error is not None:
            raise self._noise_error
        self._render_and_observe()
        obs = {"state": self._planes[0:13].clone().T}  # a snapshot: rows 0..12 of the planes are contiguous
        seg_keys = []
        for spec, cam in self.sensor_cameras:
            noisy = next((o for o in self._obs_sensors if o["name"] == spec.name), None)
            if noisy is not None:
                obs[spec.name] = noisy["out"]
                continue
            slot = self._sensor_slot[spec.name]
            obs[spec.name] = slot["depth"] if spec.kind == "depth" else slot["seg"]
            if spec.kind == "segmentation":
                seg_keys.append(spec.name)
        if self._swarm_obs is not None:
            obs["swarm"] = self._swarm_obs
        self._extra_observations(obs)
        return Observations(obs, self.num_agents, seg_keys, env=self, gen=self._obs_gen)

    def _centroid_id(self, slot) -> int:
        return 0

    def state_vector(self, i: int) -> np.ndarray:
        return self._planes[0:13, i].double().cpu().numpy()

    # ------------------------------------------------------------------ graph capture
    def make_step_graph(self, actions):
        """Capture env steps (K1+K3 and K2) into one CUDA graph.

        `actions`: a device tensor (N,4) -- one step per replay -- or (K,N,4):
        K consecutive steps, step k reading actions[k].  Returns a callable that
        replays the graph; refill `actions` in place between replays.  For
        latency-bound small batches (configs 1/2, N=100) this removes the
        per-step host launch overhead.

        Capture needs warm-up launches (2 K real steps with whatever `actions`
        holds); the env's state, flags, counters and RNG streams are saved
        before them and restored after, so making the graph does not advance
        the env.  Each replay surfaces respawn failures of the previous one
        (SpawnFailure), as step() does."""
        import torch

        if not self._reset_done:
            raise NotReset("call reset() before make_step_graph()")
        seq = actions if actions.dim() == 3 else actions.unsqueeze(0)
        if seq.shape[1:] != (self.num_agents, 4) or not seq.is_cuda or seq.dtype != self.dtype:
            raise ActionShapeMismatch(f"graph actions must be a ({self.num_agents},4) or (K,{self.num_agents},4) "
                                      f"{self.dtype} CUDA tensor")
        keep = [t for t in (self._planes, self._prev, self._outblk, self._rng, self._reset_counts, self._errors)
                if t is not None]
        saved = [t.clone() for t in keep]
        stream = torch.cuda.Stream(device=self.device)
        stream.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for _ in range(2):  # warm-up on the capture stream
                for k in range(seq.shape[0]):
                    self._bufs.action = seq[k].data_ptr()
                    self._launch_step()
            torch.cuda.current_stream().synchronize()
            with torch.cuda.graph(g, stream=stream):
                for k in range(seq.shape[0]):
                    self._bufs.action = seq[k].data_ptr()
                    self._launch_step()
            for t, v in zip(keep, saved):  # undo the warm-up
                t.copy_(v)
        torch.cuda.current_stream(self.device).wait_stream(stream)
        # replays write the observation buffer sets in the captured order, so
        # after every replay the last captured step's set is the current one
        self._graph_keepalive = seq
        k_steps = seq.shape[0]

        def replay():
            self._check_async_errors()
            g.replay()
            self._obs_gen += k_steps
            self._record_async_errors()

        return replay

    def _launch_split_dynamics(self):
        """Phase 1 on the current stream, phase 2 forked onto the post stream;
        returns the join to call after the observation launches."""
        import torch

        lib, main = nat.lib(), torch.cuda.current_stream()
        if self._post_stream is None:
            self._post_stream = torch.cuda.Stream()
        nat.check(lib.qb_env_step_phase(self._P, self._kind, self._task, self.dev_scenes.handle, self._bufs, 1,
                                        nat.stream_of()), "qb_env_step_phase")
        self._post_stream.wait_stream(main)
        with torch.cuda.stream(self._post_stream):
            nat.check(lib.qb_env_step_phase(self._P, self._kind, self._task, self.dev_scenes.handle, self._bufs, 2,
                                            nat.stream_of()), "qb_env_step_phase")
        return lambda: main.wait_stream(self._post_stream)

    def _launch_step(self):
        if self.split_step:
            join = self._launch_split_dynamics()
            self._render_and_observe()
            join()
            return
        nat.check(nat.lib().qb_env_step(self._P, self._kind, self._task, self.dev_scenes.handle, self._bufs,
                                        nat.stream_of()), "qb_env_step")
        self._render_and_observe()
