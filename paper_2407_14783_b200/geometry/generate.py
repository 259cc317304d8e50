"""Procedural scenes (inputs of the BASELINE configs).

The cluttered / garage / landing / gap / floor layouts reproduce the
reference generators (geometry/generate.py:21-116) draw for draw -- same
numpy Generator calls in the same order -- so `navigation_config(scene_seed=0)`
yields the reference's 69-primitive room exactly (pinned by
tests/test_geometry_host.py against tests/golden/geometry.npz).

`indoor_mesh_scene` is new: the ~5e5-triangle indoor scene of config 5
(Habitat datasets are unavailable offline), fully tessellated so it exercises
the triangle path of the renderer.
"""

from __future__ import annotations

import math

import numpy as np

from .. import quatmath
from .shapes import AABB, Box, Scene, SceneObject, Sphere, TriMesh

WALL_THICKNESS = 0.2
FLOOR_ID = 1
PAD_ID = 9
PAD_TOP = 0.02
WALL_IDS = (2, 3, 4, 5, 6)
OBSTACLE_ID0 = 7


def _axis_angle_matrix(axis, angle) -> np.ndarray:
    """to_matrix(from_axis_angle(axis, angle)) (quatmath.py:75-113)."""
    return quatmath.to_matrix(quatmath.from_axis_angle(axis, angle))


def room_shell(volume: AABB, thickness: float = WALL_THICKNESS, ceiling: bool = True):
    """Floor (id 1), ceiling (2), four walls (3-6); inner faces touch `volume`."""
    lo, hi = volume.lo, volume.hi
    mid = 0.5 * (lo + hi)
    sx, sy, sz = hi - lo
    t = thickness
    slab = lambda oid, c, h: SceneObject(oid, Box(c, h))  # noqa: E731
    objs = [
        slab(FLOOR_ID, [mid[0], mid[1], lo[2] - t / 2], [sx / 2 + t, sy / 2 + t, t / 2]),
        slab(3, [lo[0] - t / 2, mid[1], mid[2]], [t / 2, sy / 2 + t, sz / 2 + t]),
        slab(4, [hi[0] + t / 2, mid[1], mid[2]], [t / 2, sy / 2 + t, sz / 2 + t]),
        slab(5, [mid[0], lo[1] - t / 2, mid[2]], [sx / 2 + t, t / 2, sz / 2 + t]),
        slab(6, [mid[0], hi[1] + t / 2, mid[2]], [sx / 2 + t, t / 2, sz / 2 + t]),
    ]
    if ceiling:
        objs.insert(1, slab(2, [mid[0], mid[1], hi[2] + t / 2], [sx / 2 + t, sy / 2 + t, t / 2]))
    return objs


def generate_cluttered_scene(seed: int, volume: AABB, density: float, size_range=(0.1, 0.3), walls: bool = True) -> Scene:
    """Poisson(density * V) random spheres / oriented boxes in a room."""
    if density < 0:
        raise ValueError("density must be >= 0")
    rng = np.random.default_rng(seed)
    n = int(rng.poisson(density * volume.volume))
    objs = room_shell(volume) if walls else []
    lo_s, hi_s = size_range
    for k in range(n):
        c = rng.uniform(volume.lo, volume.hi)
        if rng.random() < 0.5:
            shape = Sphere(c, float(rng.uniform(lo_s, hi_s)))
        else:
            half = rng.uniform(lo_s, hi_s, size=3)
            axis = rng.normal(size=3)
            angle = rng.uniform(0.0, 2.0 * np.pi)
            shape = Box(c, half, _axis_angle_matrix(axis, angle))
        objs.append(SceneObject(OBSTACLE_ID0 + k, shape))
    return Scene(objs)


def _default_hall():
    return AABB([-6.0, -6.0, 0.0], [6.0, 6.0, 4.0])


def garage_scene(volume: AABB = None) -> Scene:
    return Scene(room_shell(volume or _default_hall()))


def landing_scene(pad_center=(0.0, 0.0), pad_size: float = 0.5, volume: AABB = None) -> Scene:
    px, py = pad_center
    pad = SceneObject(PAD_ID, Box([px, py, 0.01], [pad_size / 2, pad_size / 2, 0.01]))
    return Scene(room_shell(volume or _default_hall()) + [pad])


def gap_scene(gap_width: float = 1.0, wall_x: float = 0.0, volume: AABB = None) -> Scene:
    volume = volume or _default_hall()
    objs = room_shell(volume)
    lo, hi = volume.lo, volume.hi
    cz, hz, t = 0.5 * (lo[2] + hi[2]), 0.5 * (hi[2] - lo[2]), 0.1
    g = gap_width / 2
    if lo[1] < -g:
        objs.append(SceneObject(OBSTACLE_ID0, Box([wall_x, 0.5 * (lo[1] - g), cz], [t, 0.5 * (-g - lo[1]), hz])))
    if hi[1] > g:
        objs.append(SceneObject(OBSTACLE_ID0 + 1, Box([wall_x, 0.5 * (g + hi[1]), cz], [t, 0.5 * (hi[1] - g), hz])))
    return Scene(objs)


def floor_scene(z: float = 0.0, half_size: float = 500.0) -> Scene:
    return Scene([SceneObject(FLOOR_ID, Box([0.0, 0.0, z - 0.05], [half_size, half_size, 0.05]))])


# ---------------------------------------------------------------------------
# config-5 indoor mesh scene


def _grid_quad(origin, u, v, nu, nv):
    """Tessellated parallelogram origin + s*u + t*v, s,t in [0,1]: 2*nu*nv tris."""
    s = np.linspace(0.0, 1.0, nu + 1)
    t = np.linspace(0.0, 1.0, nv + 1)
    S, T = np.meshgrid(s, t, indexing="ij")
    verts = origin[None, None] + S[..., None] * u[None, None] + T[..., None] * v[None, None]
    verts = verts.reshape(-1, 3)
    idx = np.arange((nu + 1) * (nv + 1)).reshape(nu + 1, nv + 1)
    a, b, c, d = idx[:-1, :-1].ravel(), idx[1:, :-1].ravel(), idx[1:, 1:].ravel(), idx[:-1, 1:].ravel()
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)])
    return verts, tris


def _box_mesh(center, half, rot, n):
    """Closed box, each face an n x n grid."""
    c, h = np.asarray(center, float), np.asarray(half, float)
    vs, ts, base = [], [], 0
    for ax in range(3):
        for sgn in (-1.0, 1.0):
            u_ax, v_ax = [(1, 2), (2, 0), (0, 1)][ax]
            o = np.zeros(3)
            o[ax] = sgn * h[ax]
            o[u_ax], o[v_ax] = -h[u_ax], -h[v_ax]
            u = np.zeros(3)
            v = np.zeros(3)
            u[u_ax], v[v_ax] = 2 * h[u_ax], 2 * h[v_ax]
            if sgn < 0:
                u, v = v, u
                o[u_ax], o[v_ax] = -h[u_ax], -h[v_ax]
            vv, tt = _grid_quad(o, u, v, n, n)
            vs.append(vv)
            ts.append(tt + base)
            base += len(vv)
    verts = np.concatenate(vs) @ np.asarray(rot, float).T + c
    return verts, np.concatenate(ts)


def _cylinder_mesh(center, radius, height, segments, rings):
    ang = np.linspace(0.0, 2.0 * np.pi, segments, endpoint=False)
    z = np.linspace(0.0, height, rings + 1)
    ring = np.stack([radius * np.cos(ang), radius * np.sin(ang)], 1)
    verts = np.concatenate([np.column_stack([ring, np.full(segments, zz)]) for zz in z])
    tris = []
    for r in range(rings):
        a = r * segments + np.arange(segments)
        b = r * segments + (np.arange(segments) + 1) % segments
        tris.append(np.stack([a, b, b + segments], 1))
        tris.append(np.stack([a, b + segments, a + segments], 1))
    top = len(verts)
    verts = np.concatenate([verts, [[0.0, 0.0, height]]])
    a = rings * segments + np.arange(segments)
    b = rings * segments + (np.arange(segments) + 1) % segments
    tris.append(np.stack([a, b, np.full(segments, top)], 1))
    return verts + np.asarray(center, float), np.concatenate(tris)


def cluttered_mesh_scene(seed: int, volume: AABB, density: float, size_range=(0.1, 0.3), segments: int = 16) -> Scene:
    """BASELINE config 2's "procedural box/cylinder mesh scene" (SURVEY 8-D C2
    variant b): generate_cluttered_scene's room and obstacles, same Generator
    draws and object ids, every object tessellated into a TriMesh -- boxes
    (walls included) as 12 triangles, each sphere as the closed cylinder
    circumscribing it (radius r, height 2r, `segments`-gon)."""
    base = generate_cluttered_scene(seed, volume, density, size_range)
    objs = []
    for o in base.objects:
        s = o.shape
        if isinstance(s, Box):
            v, t = _box_mesh(s.center, s.half_extents, s.rotation, 1)
        else:
            r = s.radius
            v, t = _cylinder_mesh(s.center - np.array([0.0, 0.0, r]), r, 2.0 * r, segments, 1)
            bottom = len(v)  # close the bottom (the top cap is in _cylinder_mesh)
            v = np.concatenate([v, (s.center - np.array([0.0, 0.0, r]))[None]])
            a = np.arange(segments)
            t = np.concatenate([t, np.stack([(a + 1) % segments, a, np.full(segments, bottom)], 1)])
        objs.append(SceneObject(o.id, TriMesh(v, t)))
    return Scene(objs)


def indoor_mesh_scene(seed: int = 0, target_triangles: int = 500_000, size=(30.0, 30.0, 6.0)) -> Scene:
    """Procedural indoor hall of ~target_triangles triangles (config 5).

    Tessellated floor / ceiling / walls, columns (cylinders), furniture
    (rotated boxes) and a landing pad (id PAD_ID) at the hall centre; every
    object is a TriMesh.  Deterministic for a given seed.
    """
    rng = np.random.default_rng(seed)
    sx, sy, sz = size
    objs = []
    oid = 1
    # shell: floor, ceiling, 4 walls as dense grids (~20% of the budget)
    shell_tris = int(0.2 * target_triangles)
    g = max(4, int(math.sqrt(shell_tris / 12)))
    lo = np.array([-sx / 2, -sy / 2, 0.0])
    faces = [
        (lo, np.array([sx, 0, 0]), np.array([0, sy, 0])),
        (lo + [0, 0, sz], np.array([0, sy, 0]), np.array([sx, 0, 0])),
        (lo, np.array([0, 0, sz]), np.array([0, sy, 0])),
        (lo + [sx, 0, 0], np.array([0, sy, 0]), np.array([0, 0, sz])),
        (lo, np.array([sx, 0, 0]), np.array([0, 0, sz])),
        (lo + [0, sy, 0], np.array([0, 0, sz]), np.array([sx, 0, 0])),
    ]
    for o, u, v in faces:
        verts, tris = _grid_quad(o.astype(float), u.astype(float), v.astype(float), g, g)
        objs.append(SceneObject(oid, TriMesh(verts, tris)))
        oid += 1
        if oid == PAD_ID:
            oid += 1
    pv, pt = _box_mesh([0.0, 0.0, 0.01], [0.25, 0.25, 0.01], np.eye(3), 2)
    objs.append(SceneObject(PAD_ID, TriMesh(pv, pt)))
    budget = target_triangles - sum(len(ob.shape.triangles) for ob in objs)
    # columns and furniture share the rest
    while budget > 0:
        if rng.random() < 0.35:
            segs, rings = 48, int(rng.integers(8, 24))
            r = float(rng.uniform(0.15, 0.45))
            c = [rng.uniform(-sx / 2 + 1, sx / 2 - 1), rng.uniform(-sy / 2 + 1, sy / 2 - 1), 0.0]
            if abs(c[0]) < 2.0 and abs(c[1]) < 2.0:
                continue
            verts, tris = _cylinder_mesh(c, r, sz, segs, rings)
        else:
            n = int(rng.integers(3, 9))
            half = rng.uniform([0.2, 0.2, 0.2], [1.2, 1.2, 0.9])
            c = [rng.uniform(-sx / 2 + 1, sx / 2 - 1), rng.uniform(-sy / 2 + 1, sy / 2 - 1), rng.uniform(half[2], sz - half[2])]
            if abs(c[0]) < 2.0 and abs(c[1]) < 2.0:
                continue
            verts, tris = _box_mesh(c, half, _axis_angle_matrix([0, 0, 1.0], rng.uniform(0, 2 * np.pi)), n)
        tris = tris[: max(1, budget)] if len(tris) > budget else tris
        objs.append(SceneObject(oid, TriMesh(verts, tris)))
        oid += 1
        if oid == PAD_ID:
            oid += 1
        budget -= len(tris)
    return Scene(objs)
