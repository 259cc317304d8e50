"""ORACLE restatement of the reference env step (TEST INFRASTRUCTURE ONLY).

Follows env/base.py:93-232 (reset, _spawn_agent, step, _refresh_proximity)
and env/tasks.py:19-128 (free / navigation / landing hooks) for parallel
mode, with the heavy kernels in oracle/quadsim_oracle.c.  Per-agent numpy
generators (default_rng(seed + i), base.py:95) are used exactly as the
reference uses them, so spawns are bit-identical.

Configs are duck-typed: anything with the reference EnvConfig fields works
(the reference's own dataclasses or paper_2407_14783_b200.env.config).
Scenes are passed in already flattened (OracleScene), one per config scene.
"""

from __future__ import annotations

import math

import numpy as np

from . import (DOWNWARD, FORWARD, CMD_KINDS, OracleScene, camera_pose_world, command_to_rotor_speeds, dynamics_step,
               pack_params)

PAD_ID = 9  # generate.py:15
DRONE_ID0 = 60000  # base.py:34
PAD_TOP = 0.02  # generate.py:91


def _quat_from_rpy(rpy):
    """base.py:313-319 via quatmath.from_axis_angle / multiply."""

    def aa(axis, angle):
        axis = np.asarray(axis, dtype=float)
        axis = axis / np.linalg.norm(axis)
        half = 0.5 * angle
        return np.concatenate([[np.cos(half)], np.sin(half) * axis])

    def mul(q, p):
        qw, qx, qy, qz = q
        pw, px, py, pz = p
        return np.array([qw * pw - qx * px - qy * py - qz * pz, qw * px + qx * pw + qy * pz - qz * py,
                         qw * py - qx * pz + qy * pw + qz * px, qw * pz + qx * py - qy * px + qz * pw])

    roll, pitch, yaw = rpy
    return mul(aa([0, 0, 1.0], yaw), mul(aa([0, 1.0, 0], pitch), aa([1.0, 0, 0], roll)))


def _sample(dist, rng):
    """config.py:41-46 DistSpec.sample."""
    if dist.kind == "fixed":
        return np.asarray(dist.value, float).copy()
    if dist.kind == "uniform":
        return rng.uniform(np.asarray(dist.low, float), np.asarray(dist.high, float))
    return np.asarray(dist.mean, float) + np.asarray(dist.sigma, float) * rng.standard_normal(3)


def apply_noise(data, spec, rng, sensor="depth"):
    """sensing.py:195-235 (validity table checked by the caller)."""
    values = np.asarray(data, dtype=float)
    if spec.kind == "normal":
        return values.copy() if spec.sigma == 0.0 else values + spec.sigma * rng.standard_normal(values.shape)
    if spec.kind == "poisson":
        return rng.poisson(np.maximum(values, 0.0) * spec.scaling).astype(float) / spec.scaling
    if spec.kind == "saltpepper":
        out = values.copy()
        if spec.p == 0.0:
            return out
        corrupt = rng.random(values.shape) < spec.p
        salt = rng.random(values.shape) < 0.5
        lo, hi = values.min(), values.max()
        out[corrupt & salt] = hi
        out[corrupt & ~salt] = lo
        return out
    if spec.kind == "speckle":
        return values.copy() if spec.sigma == 0.0 else values * (1.0 + spec.sigma * rng.standard_normal(values.shape))
    disparity = 1.0 / np.maximum(values, 1e-6)  # redwood
    if spec.sigma_disparity > 0.0:
        disparity = disparity + spec.sigma_disparity * rng.standard_normal(values.shape)
    if spec.quantization > 0.0:
        disparity = np.round(disparity / spec.quantization) * spec.quantization
    disparity = np.maximum(disparity, 1.0 / (values.max() + 1.0) if values.size else 1e-6)
    return 1.0 / disparity


def imu_readings(state, P):
    """sensing.py:124-147: [(thrust + drag)_B / m, body rates] per agent."""
    w = state[:, 13:17]
    k2, k1, k0 = P.thrust_coeffs[0], P.thrust_coeffs[1], P.thrust_coeffs[2]
    thr = k2 * w ** 2 + k1 * w + k0
    q, v = state[:, 6:10], state[:, 3:6]
    ux, uy, uz = -q[:, 1], -q[:, 2], -q[:, 3]
    tx, ty, tz = uy * v[:, 2] - uz * v[:, 1], uz * v[:, 0] - ux * v[:, 2], ux * v[:, 1] - uy * v[:, 0]
    sx, sy, sz = uy * tz - uz * ty, uz * tx - ux * tz, ux * ty - uy * tx
    vb = np.stack([v[:, 0] + 2.0 * (q[:, 0] * tx + sx), v[:, 1] + 2.0 * (q[:, 0] * ty + sy),
                   v[:, 2] + 2.0 * (q[:, 0] * tz + sz)], axis=1)
    c = np.array([P.drag_c[0], P.drag_c[1], P.drag_c[2]])
    force = -c * vb * np.abs(vb)
    force[:, 2] += thr[:, 0] + thr[:, 1] + thr[:, 2] + thr[:, 3]
    return np.concatenate([force / P.mass, state[:, 10:13]], axis=1)


class OracleEnv:
    def __init__(self, config, scenes, params, sim, gains):
        self.config = config
        self.scenes = list(scenes)
        self.P = pack_params(params, sim, gains)
        self.n = config.num_agents
        self.task = config.task
        tp = dict(config.task_params)
        if self.task == "navigation":  # tasks.py:34-43
            self.target = np.asarray(tp.get("target", [4.2, 0.0, 2.0]), float).reshape(3)
            self.success_radius = float(tp.get("success_radius", 0.5))
            self.w_progress = float(tp.get("w_progress", 10.0))
            self.w_speed = float(tp.get("w_speed", 0.02))
            self.w_obstacle = float(tp.get("w_obstacle", 0.5))
            self.safe_distance = float(tp.get("safe_distance", 1.0))
        elif self.task == "landing":  # tasks.py:78-95
            spec = config.scenes[0]
            self.pad_center = np.asarray(tp.get("pad_center", spec.pad_center), float).reshape(2)
            self.pad_half = float(spec.pad_size) / 2.0
            self.success_height = float(tp.get("success_height", 0.1))
            self.success_speed = float(tp.get("success_speed", 0.1))
            self.w_height = float(tp.get("w_height", 0.1))
            self.w_speed = float(tp.get("w_speed", 0.5))
            self.w_collision = float(tp.get("w_collision", 1.0))
            self.seg_sensor = [s.name for s in config.sensors if s.kind == "segmentation"][-1]
        elif self.task == "gap_crossing":  # tasks.py:134-149
            default = [[3.5, -1.5 + 1.5 * i, 1.5] for i in range(config.num_agents)]
            self.targets = np.asarray(tp.get("targets", default), float).reshape(config.num_agents, 3)
            self.success_radius = float(tp.get("success_radius", 0.5))
            self.w_progress = float(tp.get("w_progress", 10.0))
            self.w_obstacle = float(tp.get("w_obstacle", 0.5))
            self.w_agent = float(tp.get("w_agent", 0.5))
            self.safe_distance = float(tp.get("safe_distance", 0.8))
        elif self.task != "free":
            raise NotImplementedError(self.task)
        self.swarm = config.mode == "swarm"
        self.bounds = [(sc.bounds_lo - config.bounds_margin, sc.bounds_hi + config.bounds_margin) for sc in self.scenes]
        self.state = np.zeros((self.n, 17))
        self.agent_scene = np.zeros(self.n, int)
        self.step_counts = np.zeros(self.n, int)
        self.needs_respawn = np.zeros(self.n, bool)
        self.nearest_dist = np.full(self.n, np.inf)
        self.nearest_pt = np.zeros((self.n, 3))
        self.collision = np.zeros(self.n, bool)
        self.oob = np.zeros(self.n, bool)
        self.nonfinite = np.zeros(self.n, bool)
        self.seg_cache = {}

    # ----------------------------------------------------------------- reset
    def reset(self, seed=0):
        """base.py:93-112."""
        self.rngs = [np.random.default_rng(int(seed) + i) for i in range(self.n)]
        ns = len(self.scenes)
        if self.config.scene_sampling == "shuffled":
            self.scene_perm = np.random.default_rng(int(seed)).permutation(ns)
        else:
            self.scene_perm = np.arange(ns)
        self.reset_counts = np.zeros(self.n, int)
        self.state[:] = 0.0
        self.state[:, 6] = 1.0
        self.state[:, 13:17] = self.P.hover_speed
        for i in range(self.n):
            self._spawn(i)
        self.prev_state = self.state.copy()
        self.step_counts[:] = 0
        self.needs_respawn[:] = False
        self.collision[:] = False
        self.oob[:] = False
        self.nonfinite[:] = False
        self._refresh_proximity()
        return self.observe()

    def _spawn(self, i):
        """base.py:114-147."""
        self.agent_scene[i] = 0 if self.swarm else self.scene_perm[(i + self.reset_counts[i]) % len(self.scenes)]
        self.reset_counts[i] += 1
        rng = self.rngs[i]
        rand = self.config.randomization
        scene = self.scenes[self.agent_scene[i]]
        pos = None
        for _ in range(1000):
            cand = _sample(rand.position, rng)
            _, d, _ = scene.nearest_point(cand[None])
            if d[0] < self.config.min_spawn_clearance:
                continue
            if self.swarm:  # base.py:141-146 _swarm_spawn_clear
                min_sep = 2.0 * self.config.collision_radius + 0.1
                if any(np.linalg.norm(self.state[j, 0:3] - cand) < min_sep for j in range(i)):
                    continue
            pos = cand
            break
        if pos is None:
            raise RuntimeError(f"SpawnFailure agent {i}")
        vel = _sample(rand.velocity, rng)
        quat = _quat_from_rpy(_sample(rand.orientation, rng))
        ang = _sample(rand.angvel, rng)
        self.state[i, 0:3] = pos
        self.state[i, 3:6] = vel
        self.state[i, 6:10] = quat
        self.state[i, 10:13] = ang
        self.state[i, 13:17] = self.P.hover_speed
        self.step_counts[i] = 0

    # ------------------------------------------------------------------ step
    def step(self, action):
        """base.py:156-210 (parallel mode). `action` is the (N,4) as_array()."""
        action = np.asarray(action, float).reshape(self.n, 4)
        if self.config.auto_reset and self.needs_respawn.any():
            for i in np.nonzero(self.needs_respawn)[0]:
                self._spawn(int(i))
            self.needs_respawn[:] = False
        self.prev_state = self.state.copy()
        cmds = command_to_rotor_speeds(self.P, self.config.command_type, self.state, action)
        nxt, bad = dynamics_step(self.P, self.state, cmds)
        nxt[bad] = self.prev_state[bad]
        self.state = nxt
        self.nonfinite = bad
        self.step_counts += 1
        self._refresh_proximity()
        success = self.get_success()
        reward = self.get_reward()
        obs = self.observe()
        terminated = success | self.collision | self.oob | self.nonfinite
        truncated = ~terminated & (self.step_counts >= self.config.episode_max_steps)
        self.needs_respawn = terminated | truncated
        return obs, reward, terminated, truncated, success

    def _refresh_proximity(self):
        """base.py:214-224."""
        for s in range(len(self.scenes)):
            m = self.agent_scene == s
            if not m.any():
                continue
            pt, d, _ = self.scenes[s].nearest_point(self.state[m, 0:3])
            self.nearest_pt[m] = pt
            self.nearest_dist[m] = d
            lo, hi = self.bounds[s]
            p = self.state[m, 0:3]
            self.oob[m] = ~(np.all(p >= lo, axis=1) & np.all(p <= hi, axis=1))
        self.collision = self.nearest_dist < self.config.collision_radius
        if self.swarm and self.n > 1:  # base.py:225-232
            pos = self.state[:, 0:3]
            for i in range(self.n):
                for j in range(i + 1, self.n):
                    if np.linalg.norm(pos[i] - pos[j]) < 2.0 * self.config.collision_radius:
                        self.collision[i] = True
                        self.collision[j] = True

    # ----------------------------------------------------------------- tasks
    def _dist(self, x):
        d = x[:, 0:3] - self.target[None, :]
        return np.sqrt(d[:, 0] ** 2 + d[:, 1] ** 2 + d[:, 2] ** 2)

    def _height(self):
        return np.maximum(self.state[:, 2] - PAD_TOP - self.config.collision_radius, 0.0)

    def _gap_dist(self, x):  # tasks.py:151-153
        d = x[:, 0:3] - self.targets
        return np.sqrt(d[:, 0] ** 2 + d[:, 1] ** 2 + d[:, 2] ** 2)

    def get_success(self):
        if self.task == "gap_crossing":  # tasks.py:155-156
            return self._gap_dist(self.state) < self.success_radius
        if self.task == "navigation":  # tasks.py:49-50
            return self._dist(self.state) < self.success_radius
        if self.task == "landing":  # tasks.py:101-106
            speed = np.linalg.norm(self.state[:, 3:6], axis=1)
            off = np.abs(self.state[:, 0:2] - self.pad_center[None, :])
            centered = (off[:, 0] <= self.pad_half) & (off[:, 1] <= self.pad_half)
            return (self._height() < self.success_height) & (speed < self.success_speed) & centered
        return np.zeros(self.n, bool)

    def get_reward(self):
        if self.task == "gap_crossing":  # tasks.py:158-169
            progress = self._gap_dist(self.prev_state) - self._gap_dist(self.state)
            proximity = np.clip(1.0 - self.nearest_dist / self.safe_distance, 0.0, 1.0)
            reward = self.w_progress * progress - self.w_obstacle * proximity
            if self.n > 1:
                pos = self.state[:, 0:3]
                for i in range(self.n):
                    dmin = min(np.linalg.norm(pos[i] - pos[j]) for j in range(self.n) if j != i)
                    reward[i] -= self.w_agent * max(0.0, 1.0 - dmin / self.safe_distance)
            return reward
        if self.task == "navigation":  # tasks.py:52-56
            progress = self._dist(self.prev_state) - self._dist(self.state)
            speed2 = (self.state[:, 3:6] ** 2).sum(axis=1)
            prox = np.clip(1.0 - self.nearest_dist / self.safe_distance, 0.0, 1.0)
            return self.w_progress * progress - self.w_speed * speed2 - self.w_obstacle * prox
        if self.task == "landing":  # tasks.py:108-111
            speed2 = (self.state[:, 3:6] ** 2).sum(axis=1)
            return -self.w_height * self._height() + self.w_speed * np.exp(-speed2) - self.w_collision * self.collision
        return np.zeros(self.n)

    # ----------------------------------------------------------- observation
    def render(self, sensor):
        """base.py:256-277 for one camera sensor."""
        H, W = sensor.height, sensor.width
        rot = FORWARD if sensor.orientation == "forward" else DOWNWARD
        depth = np.empty((self.n, H, W))
        seg = np.empty((self.n, H, W), np.int64)
        tv = math.tan(sensor.vertical_fov / 2.0)
        th = tv * W / H
        for s in np.unique(self.agent_scene):
            m = np.nonzero(self.agent_scene == s)[0]
            o, r = camera_pose_world(self.state[m, 0:3], self.state[m, 6:10], rot, sensor.translation)
            extra = ids = None
            if self.swarm and self.n > 1:  # base.py:245-255, 268-272
                extra = np.empty((len(m), self.n - 1, 4))
                ids = np.empty((len(m), self.n - 1), np.int64)
                for k, a in enumerate(m):
                    others = [j for j in range(self.n) if j != a]
                    extra[k, :, 0:3] = self.state[others, 0:3]
                    extra[k, :, 3] = self.config.collision_radius
                    ids[k] = DRONE_ID0 + np.array(others)
            d, i = self.scenes[s].render(o, r, W, H, th, tv, sensor.max_range, extra, ids)
            depth[m] = d
            seg[m] = i
        return depth, seg

    def observe(self):
        """base.py:287-310 + tasks.py:58-62, 113-118 (batched form)."""
        obs = {"state": self.state[:, 0:13].copy()}
        for sensor in self.config.sensors:
            if sensor.kind == "imu":  # base.py:290-296
                reading = imu_readings(self.state, self.P)
                for i in range(self.n):
                    for nz in sensor.noise:
                        reading[i] = apply_noise(reading[i], nz, self.rngs[i], "imu")
                obs[sensor.name] = reading
                continue
            depth, seg = self.render(sensor)
            img = depth if sensor.kind == "depth" else seg.astype(float)
            if sensor.noise:  # base.py:298-303, per agent on its own generator
                img = img.copy()
                for i in range(self.n):
                    for nz in sensor.noise:
                        img[i] = apply_noise(img[i], nz, self.rngs[i], sensor.kind)
            obs[sensor.name] = img
            self.seg_cache[sensor.name] = seg
        if self.swarm and self.n > 1:  # base.py:306-309
            obs["swarm"] = np.stack([self.state[[j for j in range(self.n) if j != i], 0:13] for i in range(self.n)])
        if self.task == "navigation":
            obs["target"] = np.broadcast_to(self.target, (self.n, 3)).copy()
        elif self.task == "gap_crossing":  # tasks.py:171-174
            obs["target"] = self.targets.copy()
        elif self.task == "landing":  # tasks.py:121-128
            seg = self.seg_cache[self.seg_sensor]
            tgt = np.full((self.n, 2), -1.0)
            for i in range(self.n):
                rows, cols = np.nonzero(seg[i] == PAD_ID)
                if len(rows):
                    tgt[i] = [cols.mean(), rows.mean()]
            obs["target"] = tgt
        return obs
