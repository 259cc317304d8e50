"""Flat-array bindings (the reference's "bindings" module).

The reference specifies -- but never built -- a thin adapter that exposes
reset/step to external RL frameworks through a flat-array foreign-call
boundary:

    make_env(config) -> handle
    reset(handle, seed) -> FlatObservation
    step(handle, actions: N x 4 array) -> (FlatObservation, rewards, terminated, truncated, info)

Here a handle owns one batched GPU env (`env.make_env`) and a step is ONE
native call, `qb_env_step_io` (include/quadb200.h): the host actions are
copied to the device, the fused env step and every camera render run, the
state rows / narrowed (uint8 or uint16) segmentation are packed on the device, and the results are
copied back into host arrays before the call returns.  No torch op runs per
step, so the host cost of a step is one ctypes call (about 10-20 us at
100 envs) instead of the batched Python env's tensor bookkeeping.

Semantics (SPEC.md "bindings"):
  * actions: (N, 4) in the config's command layout (`Command.as_array()`):
    CTBR / SRT on the wire, LV / PS by config-selected conversion;
  * every step returns freshly owned numpy arrays (no views of stale
    buffers), unless the caller passes `out=` buffers (`handle.outputs()`,
    pinned host memory, reused step after step -- the zero-copy path);
  * float width: state / depth / rewards are float32 (the reference's are
    float64), segmentation is uint8 / uint16 when every object id of the
    scenes fits in one / two bytes and int32 otherwise (lossless; "documented
    float-width conversion");
  * a handle is single-owner: a call while another call on the same handle
    is running raises; calls after close() raise.

Swarm configs are not exposed (their observation is N x (N-1) x 13 and the
reference's bindings would not ship it either).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import ActionShapeMismatch, ConfigError, NotReset, SpawnFailure


GRAPH_MAX_AGENTS = 4096  # batches up to this size replay a reused-buffer step as a CUDA graph


class HandleClosed(RuntimeError):
    """A call on a handle after close()."""


class HandleBusy(RuntimeError):
    """Concurrent calls on one single-owner handle (SPEC.md: rejected)."""


@dataclass
class FlatObservation:
    """Contiguous arrays per observation key plus a layout descriptor
    ({key: (shape, dtype)}) that round-trips."""

    arrays: dict
    layout: dict

    def __getitem__(self, key):
        return self.arrays[key]

    def keys(self):
        return self.arrays.keys()


class FlatEnv:
    """One bindings handle.  Use the module functions or the methods."""

    def __init__(self, config, params=None, sim=None, gains=None, device=None, shard=(0, 1), scene_build="host"):
        import torch

        from .env import EnvConfig, load_env_file, make_env

        if not isinstance(config, EnvConfig):  # a config file path (SPEC: make_env(config path))
            config, p2, s2, g2 = load_env_file(config)
            params, sim, gains = params or p2, sim or s2, gains or g2
        if config.mode == "swarm":
            raise ConfigError("the flat bindings do not expose swarm mode")
        self._lock = threading.Lock()
        self._closed = False
        self.env = make_env(config, params, sim, gains, device=device, shard=shard, scene_build=scene_build)
        if self.env._custom_hooks:
            raise ConfigError("the flat bindings run the fused task hooks only")
        env, n = self.env, self.env.num_agents
        self.num_agents = n
        self._dev = env.device
        dt_np = np.float32 if env.dtype == torch.float32 else np.float64
        self._dt_np = dt_np
        max_id = max((int(s.arrays.prim_object_id.max()) if s.arrays.prim_object_id.size else 0) for s in env.scenes)
        min_id = min((int(s.arrays.prim_object_id.min()) if s.arrays.prim_object_id.size else 0) for s in env.scenes)
        # lossless narrowing of the segmentation ids for the read-back (the bytes PCIe carries)
        self.seg_dtype = (np.int32 if min_id < 0 or max_id >= 65536 else np.uint8 if max_id < 256 else np.uint16)
        # the small per-step results travel as ONE device block and ONE D2H copy:
        # [state rows (n,13) | output block (flags, reward, counters, nearest point) | spawn-failure count]
        es = 4 if dt_np == np.float32 else 8
        r16 = lambda x: (x + 15) // 16 * 16  # noqa: E731
        lay, _ = env._outblk_layout(n)
        self._outblk_layout, self._outblk_nbytes = lay, env._outblk_bytes(n)
        self._off_outblk = r16(n * 13 * es)
        self._off_err = self._off_outblk + r16(self._outblk_nbytes)
        self._small_nbytes = self._off_err + 16
        with torch.cuda.device(self._dev):
            self._small = torch.zeros(self._small_nbytes, dtype=torch.uint8, device=self._dev)
            self._rows = self._small[:n * 13 * es].view(env.dtype).view(n, 13)
            # every call synchronises its stream, so the env's own (current) stream is used
            self._stream = torch.cuda.current_stream(self._dev)
        # one qb_io_view per distinct camera (renders into the env's buffer set 0)
        views = []
        with torch.cuda.device(self._dev):
            for slot in env._cams.values():
                v = nat.QbIoView()
                v.cam = slot["camera"].native(0)
                depth = slot.get("depth_pair", [None])[0]
                seg = slot.get("seg_pair", [None])[0]
                v.depth = nat.ptr(depth)
                v.seg = nat.ptr(seg)
                cid = env._centroid_id(slot)
                v.centroid_id = int(cid)
                v.centroid = nat.ptr(slot["centroid_pair"][0]) if cid else None
                seg_host = None
                if seg is not None and self.seg_dtype != np.int32:
                    w = np.dtype(self.seg_dtype).itemsize
                    seg_host = torch.zeros(seg.shape, dtype=torch.uint8 if w == 1 else torch.int16, device=self._dev)
                    v.seg_small, v.seg_small_bytes = nat.ptr(seg_host), w
                slot["_io"] = {"depth": depth, "seg": seg_host if seg_host is not None else seg,
                               "centroid": slot["centroid_pair"][0] if cid else None}
                views.append(v)
        self._views = (nat.QbIoView * max(1, len(views)))(*views)
        self._n_views = len(views)
        # sensor pass (noise chains, IMU) into buffer set 0
        self._n_sensors = len(env._obs_sensors)
        self._sensors = env._obs_arrays[0] if env._obs_sensors else None
        # observation keys in the reference's order (base.py:287-310)
        src = []  # images: (key, device tensor, shape, numpy dtype), one D2H copy each
        for spec, cam in env.sensor_cameras:
            noisy = next((o for o in env._obs_sensors if o["name"] == spec.name), None)
            if noisy is not None:
                t = noisy["outs"][0]
                src.append((spec.name, t, tuple(t.shape), dt_np))
                continue
            slot = env._sensor_slot[spec.name]["_io"]
            if spec.kind == "depth":
                src.append((spec.name, slot["depth"], tuple(slot["depth"].shape), dt_np))
            else:
                t = slot["seg"]
                src.append((spec.name, t, tuple(t.shape), self.seg_dtype))
        self._target_const = None
        if hasattr(env, "_target_obs"):  # navigation / gap: a constant per-agent target
            self._target_const = env._target_obs.detach().cpu().numpy().astype(dt_np)
        else:
            for slot in env._cams.values():
                if slot["_io"]["centroid"] is not None:  # landing: the pad centroid of this step
                    src.append(("target", slot["_io"]["centroid"], (n, 2), np.float32))
        self._src = src
        self.layout = {"state": ((n, 13), np.dtype(dt_np).str)}
        self.layout.update({k: (shape, np.dtype(dt).str) for k, _, shape, dt in src})
        if self._target_const is not None:
            self.layout["target"] = (self._target_const.shape, self._target_const.dtype.str)
        self._io = nat.QbStepIo()
        self._io.sync = 1
        self._io.state_rows = nat.ptr(self._rows)
        self._io.n_views = self._n_views
        self._io.views = ctypes.cast(self._views, ctypes.c_void_p)
        self._io.n_sensors = self._n_sensors
        self._io.sensors = ctypes.cast(self._sensors, ctypes.c_void_p) if self._sensors is not None else None
        base = self._small.data_ptr()
        self._packs = (nat.QbIoCopy * 2)()
        self._packs[0].src, self._packs[0].dst, self._packs[0].bytes = (env._outblk.data_ptr(), base + self._off_outblk,
                                                                       self._outblk_nbytes)
        self._packs[1].src, self._packs[1].dst, self._packs[1].bytes = env._errors.data_ptr(), base + self._off_err, 4
        self._io.n_packs = 2
        self._io.packs = ctypes.cast(self._packs, ctypes.c_void_p)
        self._copies = (nat.QbIoCopy * (len(src) + 1))()
        self._copies[0].src, self._copies[0].bytes = base, self._small_nbytes
        self._io.n_copies = len(src) + 1
        self._io.copies = ctypes.cast(self._copies, ctypes.c_void_p)
        self._reset_done = False
        self._cache = None  # (out dict, its error-count view, the step result built on it)
        self._graph = None  # CUDA graph of the cached step (small batches)
        self._lib = nat.lib()
        self._stream_ptr = ctypes.c_void_p(self._stream.cuda_stream)
        self._step_fn = self._lib.qb_env_step_io
        self._args = (env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs)
        self._io_ref = ctypes.byref(self._io)

    # ------------------------------------------------------------------ step graph
    def _make_graph(self):
        import torch

        self._stage = torch.zeros((self.num_agents, 4), dtype=_torch_dtype(self._dt_np), pin_memory=True).numpy()
        self._io.step = 1
        self._io.host_action = self._stage.ctypes.data
        g = ctypes.c_void_p()
        nat.check(self._lib.qb_env_step_graph_create(*self._args, self._io_ref, ctypes.byref(g)), "qb_env_step_graph_create")
        self._graph = g

    def _drop_graph(self):
        if getattr(self, "_graph", None) is not None:
            self._lib.qb_env_step_graph_destroy(self._graph)
            self._graph = None

    def __del__(self):
        try:
            self._drop_graph()
        except Exception:
            pass

    # ------------------------------------------------------------------ buffers
    def outputs(self, pinned: bool = True) -> dict:
        """A host buffer set for `out=` (pinned: the D2H copies run at full
        PCIe speed and no per-step allocation happens).  Arrays written by a
        step stay valid until the caller passes the same set again."""
        import torch

        out = {k: torch.empty(shape, dtype=_torch_dtype(dt), pin_memory=pinned).numpy().view(dt)
               for k, _, shape, dt in self._src}
        small = torch.empty(self._small_nbytes + 16, dtype=torch.uint8, pin_memory=pinned)
        off = (-small.data_ptr()) % 16  # 16-byte aligned: the pack kernel writes it with vector stores
        out["_small"] = small.numpy()[off:off + self._small_nbytes]
        out["_pinned"] = pinned  # pinned: the small results are written straight into it by the pack kernel
        return out

    # ------------------------------------------------------------------ calls
    def _enter(self):
        if self._closed:
            raise HandleClosed("handle is closed")
        if not self._lock.acquire(blocking=False):
            raise HandleBusy("concurrent call on a single-owner handle")

    def close(self):
        self._enter()
        try:
            self._drop_graph()
            self._closed = True
            self.env = None
        finally:
            self._lock.release()

    def reset(self, seed: int = 0, out: dict | None = None) -> FlatObservation:
        import torch

        self._enter()
        try:
            with torch.cuda.device(self._dev):
                self.env._reset_state(seed)  # spawns only: the observation (and its noise draws) comes from _run
                self._reset_done = True
                return self._run(step=False, actions=None, out=out)[0]
        finally:
            self._lock.release()

    def step(self, actions, out: dict | None = None):
        self._enter()
        try:
            if not self._reset_done:
                raise NotReset("call reset() before step()")
            a = actions.as_array() if hasattr(actions, "as_array") else actions
            a = np.asarray(a)
            if a.shape != (self.num_agents, 4):
                raise ActionShapeMismatch(f"actions must be ({self.num_agents}, 4), got {a.shape}")
            if a.dtype != self._dt_np or not a.flags.c_contiguous:
                a = np.ascontiguousarray(a, dtype=self._dt_np)
            return self._run(step=True, actions=a, out=out)
        finally:
            self._lock.release()

    def _run(self, step, actions, out):
        env = self.env
        cached = self._cache
        if step and out is not None and cached is not None and cached[0] is out:
            # the caller's buffer set of the previous step again: every pointer in the
            # io block and every returned view is unchanged -- one native call; small
            # batches (launch-latency-bound) replay the step as a CUDA graph that reads
            # its actions from a fixed pinned staging buffer
            if self.num_agents <= GRAPH_MAX_AGENTS:
                if self._graph is None:
                    self._make_graph()
                np.copyto(self._stage, actions)
                nat.check(self._lib.qb_env_step_graph_launch(self._graph, 1, self._stream_ptr), "qb_env_step_graph_launch")
            else:
                self._io.host_action = actions.ctypes.data
                nat.check(self._step_fn(*self._args, self._io_ref, self._stream_ptr), "qb_env_step_io")
            if cached[1][0] > 0:
                nfail = int(cached[1][0])
                env._errors.zero_()
                raise SpawnFailure(f"{nfail} respawns found no spawn with clearance >= {env.config.min_spawn_clearance}")
            return cached[2]
        self._drop_graph()
        self._cache = None
        if out is None:  # freshly owned arrays every call (pageable host memory)
            out = {k: np.empty(shape, dtype=dt) for k, _, shape, dt in self._src}
            out["_small"] = np.empty(self._small_nbytes, dtype=np.uint8)
        small = out["_small"]
        cp, io = self._copies, self._io
        for i, (k, t, shape, dt) in enumerate(self._src, 1):
            cp[i].src, cp[i].dst, cp[i].bytes = t.data_ptr(), out[k].ctypes.data, out[k].nbytes
        if out.get("_pinned"):  # zero-copy: rows + flags/reward + error count written into host memory by the pack kernel
            host = small.ctypes.data
            io.state_rows = host
            self._packs[0].dst, self._packs[1].dst = host + self._off_outblk, host + self._off_err
            io.copies = ctypes.addressof(cp) + ctypes.sizeof(nat.QbIoCopy)  # skip copy 0
            io.n_copies = len(self._src)
        else:  # packed in device memory, one D2H copy
            base = self._small.data_ptr()
            io.state_rows = base
            self._packs[0].dst, self._packs[1].dst = base + self._off_outblk, base + self._off_err
            cp[0].dst = small.ctypes.data
            io.copies = ctypes.addressof(cp)
            io.n_copies = len(self._src) + 1
        self._io.step = 1 if step else 0
        self._io.host_action = actions.ctypes.data if step else None
        if step:
            env._bufs.action = env._action.data_ptr()
        nat.check(self._step_fn(*self._args, self._io_ref, self._stream_ptr), "qb_env_step_io")
        n, lay, o = self.num_agents, self._outblk_layout, self._off_outblk
        v = lambda key, dt: small[o + lay[key][0]:o + lay[key][1]].view(dt)  # noqa: E731
        if step:
            nfail = int(small[self._off_err:self._off_err + 4].view(np.int32)[0])
            if nfail > 0:
                env._errors.zero_()
                raise SpawnFailure(f"{nfail} respawns found no spawn with clearance >= {env.config.min_spawn_clearance}")
        arrays = {"state": small[:n * 13 * self._rows.element_size()].view(self._dt_np).reshape(n, 13)}
        arrays.update({k: out[k] for k, _, _, _ in self._src})
        if self._target_const is not None:
            arrays["target"] = self._target_const.copy()
        obs = FlatObservation(arrays, self.layout)
        if not step:
            return obs, None
        flags = v("flags", np.bool_).reshape(7, n)
        info = {"success": flags[3], "collision": flags[4], "out_of_bounds": flags[5], "nonfinite": flags[6],
                "nearest_distance": v("dist", np.float64), "scene": v("scene", np.int32), "step": v("step", np.int32)}
        result = (obs, v("reward", np.float32), flags[1], flags[2], info)
        if "_pinned" in out:  # a caller-owned set (outputs()): reused calls take the fast path
            self._cache = (out, small[self._off_err:self._off_err + 4].view(np.int32), result)
        return result


def _torch_dtype(dt):
    import torch

    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8,
            np.dtype(np.uint16): torch.int16, np.dtype(np.int32): torch.int32}[np.dtype(dt)]  # (uint16: same bytes)


# ---------------------------------------------------------------- module API (SPEC.md names)


def make_env(config, params=None, sim=None, gains=None, device=None, shard=(0, 1), scene_build="host") -> FlatEnv:
    """config: an EnvConfig or the path of an env config file (load_env_file).
    shard=(rank, world): this handle owns the rank's contiguous slice of the
    config's agents (multi-GPU, one handle per GPU); scene_build "device"
    builds large meshes on the GPU (as env.make_env)."""
    return FlatEnv(config, params, sim, gains, device, shard, scene_build)


def reset(handle: FlatEnv, seed: int = 0, out=None) -> FlatObservation:
    return handle.reset(seed, out=out)


def step(handle: FlatEnv, actions, out=None):
    return handle.step(actions, out=out)


def close(handle: FlatEnv) -> None:
    handle.close()
