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
(`observations["depth"]`) and never leave the GPU.

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


class Observations(Sequence):
    """Batched observation dict that also indexes like the reference list.

    obs["depth"] -> (N,H,W) CUDA tensor; obs[i] -> {"state": (13,), ...} numpy
    dict for agent i (reference layout, float64, segmentation cast to float).
    The tensors are the env's persistent device buffers: the next step
    overwrites them (clone, or index obs[i] before stepping, to keep them).
    """

    def __init__(self, data: dict, n: int, seg_keys=()):
        self._data = data
        self._n = n
        self._seg_keys = set(seg_keys)
        self._host = None

    def keys(self):
        return self._data.keys()

    def items(self):
        return self._data.items()

    def __contains__(self, key):
        return key in self._data if isinstance(key, str) else super().__contains__(key)

    def __len__(self):
        return self._n

    def _materialize(self):
        if self._host is None:
            self._host = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in self._data.items()}
        return self._host

    def __getitem__(self, key):
        if isinstance(key, str):
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
    """Per-agent info dicts (base.py:195-207), materialised lazily."""

    _KEYS = ("success", "collision", "out_of_bounds", "nonfinite", "nearest_distance", "scene", "step")

    def __init__(self, data: dict, n: int):
        self.data = data
        self._n = n
        self._host = None

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, str):
            return self.data[i]
        if self._host is None:
            self._host = {k: self.data[k].detach().cpu().numpy() for k in self._KEYS}
        h = self._host
        i = int(i)
        return {
            "success": bool(h["success"][i]), "collision": bool(h["collision"][i]),
            "out_of_bounds": bool(h["out_of_bounds"][i]), "nonfinite": bool(h["nonfinite"][i]),
            "nearest_distance": float(h["nearest_distance"][i]), "scene": int(h["scene"][i]), "step": int(h["step"][i]),
        }


@dataclass
class StepResult:
    observations: Observations
    reward: object
    terminated: object
    truncated: object
    info: Info


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
        self._action_host_ev = [None, None]
        self._action_host_i = 0
        self.step_counts = z(n, dtype=torch.int32)
        self.agent_scene = z(n, dtype=torch.int32)
        self._reset_counts = z(n, dtype=torch.int32)
        self._flags = z(7, n)
        (self._needs_respawn, self._terminated, self._truncated, self._success, self._collision, self._oob,
         self._nonfinite) = self._flags.unbind(0)
        self._reward = z(n, dtype=torch.float32)
        self.nearest_dist = z(n, dtype=torch.float64)
        self.nearest_pt = z(n, 3, dtype=torch.float64)
        self._rng = z(n, 4, dtype=torch.int64)
        self._errors = z(1, dtype=torch.int32)
        self._scene_perm = z(len(self.scenes), dtype=torch.int32)
        # observation buffers: one render per distinct camera
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
                slot["depth"] = torch.zeros((n, cam.height, cam.width), dtype=dt, device=dev)
            if spec.kind == "segmentation" and slot["seg"] is None:
                slot["seg"] = torch.zeros((n, cam.height, cam.width), dtype=torch.int32, device=dev)
            spec_slot = slot
            if not spec.noise:
                spec_slot["names"].append((spec.name, spec.kind))
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
            if spec.kind == "imu":
                out = torch.zeros((n, 6), dtype=dt, device=dev)
                rec = sensor_obs("imu", spec.noise, out)
            elif spec.noise:
                slot = self._sensor_slot[spec.name]
                out = torch.zeros((n, cam.height, cam.width), dtype=dt, device=dev)
                src = slot["depth"] if spec.kind == "depth" else slot["seg"]
                rec = sensor_obs(spec.kind, spec.noise, out, src=src, width=cam.width, height=cam.height)
            else:
                continue
            self._obs_sensors.append({"name": spec.name, "kind": spec.kind, "out": out, "rec": rec})
        if self._obs_sensors:
            arr = (nat.QbSensorObs * len(self._obs_sensors))(*[o["rec"] for o in self._obs_sensors])
            self._obs_array = arr
        # swarm mode: the other agents as render spheres + the swarm observation
        self._swarm_spheres = self._swarm_ids = self._swarm_obs = None
        if self.swarm and n > 1:
            self._swarm_spheres = torch.zeros((n, n - 1, 4), dtype=dt, device=dev)
            self._swarm_ids = torch.zeros((n, n - 1), dtype=torch.int32, device=dev)
            self._swarm_obs = torch.zeros((n, n - 1, 13), dtype=dt, device=dev)
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
        return self.get_observation()

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
        buf.copy_(torch.as_tensor(np.asarray(arr), dtype=self.dtype))
        self._action.copy_(buf, non_blocking=True)
        ev = self._action_host_ev[k] or torch.cuda.Event()
        ev.record()
        self._action_host_ev[k] = ev
        return self._action

    def step(self, action) -> StepResult:
        """One control step for every agent (base.py:156-210), asynchronous."""
        import torch

        if not self._reset_done:
            raise NotReset("call reset() before step()")
        self._check_async_errors()
        a = self._stage_action(action)
        self._bufs.action = a.data_ptr()
        with torch.cuda.device(self.device):
            if self.split_step:
                join = self._launch_split_dynamics()
                self._record_async_errors()
                obs = self.get_observation()
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
        else:
            success, reward = self._success.bool(), self._reward
            terminated, truncated = self._terminated.bool(), self._truncated.bool()
        info = Info({"success": success, "collision": self.collision, "out_of_bounds": self.out_of_bounds,
                     "nonfinite": self.nonfinite, "nearest_distance": self.nearest_dist, "scene": self.agent_scene,
                     "step": self.step_counts}, self.num_agents)
        return StepResult(obs, reward, terminated, truncated, info)

    def _record_async_errors(self):
        import torch

        if getattr(self, "_err_host", None) is None:
            self._err_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._err_event = torch.cuda.Event()
        self._err_host.copy_(self._errors, non_blocking=True)
        self._err_event.record()
        self._pending_errors = True

    def _check_async_errors(self):
        if getattr(self, "_pending_errors", None) and self._err_event.query() and int(self._err_host[0]) > 0:
            n = int(self._err_host[0])
            self._errors.zero_()
            raise SpawnFailure(f"{n} respawns found no spawn with clearance >= {self.config.min_spawn_clearance}")

    def _render_and_observe(self):
        """Launch the observation kernels: K2 once per distinct camera, then
        the sensor pass (IMU + noise chains) if any sensor needs it."""
        self._render()
        self._observe()

    def _render(self):
        if self._swarm_obs is not None:  # other agents as spheres + swarm states (base.py:245-277, 306-309)
            nat.check(nat.lib().qb_env_swarm_views(self._task, self._bufs, nat.ptr(self._swarm_spheres),
                                                   nat.ptr(self._swarm_ids), nat.ptr(self._swarm_obs), nat.stream_of()),
                      "qb_env_swarm_views")
        for slot in self._cams.values():
            cid = self._centroid_id(slot)
            if cid and slot["centroid"] is None:
                import torch

                slot["centroid"] = torch.zeros((self.num_agents, 2), dtype=torch.float32, device=self.device)
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
        obs = {"state": self._planes[0:13].T}
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
        return Observations(obs, self.num_agents, seg_keys)

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
        per-step host launch overhead."""
        import torch

        seq = actions if actions.dim() == 3 else actions.unsqueeze(0)
        if seq.shape[1:] != (self.num_agents, 4) or not seq.is_cuda or seq.dtype != self.dtype:
            raise ActionShapeMismatch(f"graph actions must be a ({self.num_agents},4) or (K,{self.num_agents},4) "
                                      f"{self.dtype} CUDA tensor")
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
        torch.cuda.current_stream(self.device).wait_stream(stream)
        self._graph_keepalive = seq
        return g.replay

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
