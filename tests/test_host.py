"""CPU-only tests of the host side: generators, constant folding, configs,
and the C-ABI library surface (loads and exports every declared symbol; no
compute calls without a GPU)."""

import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden
from paper_2407_14783_b200 import _native as nat
from paper_2407_14783_b200.errors import ConfigError
from paper_2407_14783_b200.geometry import (AABB, Box, Scene, SceneObject, Sphere, TriMesh, gap_scene, garage_scene,
                                            generate_cluttered_scene, indoor_mesh_scene, landing_scene)
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig, native_params


@pytest.mark.parametrize("name,make", [
    ("nav", lambda: generate_cluttered_scene(0, AABB([-5, -5, 0], [5, 5, 4]), 0.15)),
    ("landing", landing_scene), ("garage", garage_scene), ("gap", lambda: gap_scene(1.0)),
    ("garage10", lambda: garage_scene(AABB([-5, -5, 0], [5, 5, 4]))),
])
def test_scene_generators_reproduce_reference(ggeo, name, make):
    t = make().arrays
    for ours, key in ((t.prim_type, "prim_type"), (t.prim_data, "prim_data"), (t.prim_object_id, "prim_oid"),
                      (t.prim_aabb_lo, "prim_lo"), (t.prim_aabb_hi, "prim_hi")):
        assert np.array_equal(ours, ggeo[f"{name}_{key}"]), key
    b = make().bounds
    assert np.array_equal(np.stack([b.lo, b.hi]), ggeo[f"{name}_bounds"])


def test_trimesh_flatten_matches_reference(ggeo):
    # the golden "tess" scene is TriMesh-only; re-flatten its triangles through our Scene
    tri = ggeo["tess_prim_data"][:, :9].reshape(-1, 3, 3)
    oid = ggeo["tess_prim_oid"]
    objs = []
    for o in np.unique(oid):
        t = tri[oid == o]
        objs.append(SceneObject(int(o), TriMesh(t.reshape(-1, 3), np.arange(3 * len(t)).reshape(-1, 3))))
    a = Scene(objs).arrays
    assert np.array_equal(a.prim_data, ggeo["tess_prim_data"])
    assert np.array_equal(a.prim_aabb_lo, ggeo["tess_prim_lo"]) and np.array_equal(a.prim_aabb_hi, ggeo["tess_prim_hi"])


def test_indoor_mesh_scene_size():
    s = indoor_mesh_scene(seed=0, target_triangles=60_000)
    n = len(s.arrays)
    assert 55_000 <= n <= 60_000
    assert 9 in {o.id for o in s.objects}  # landing pad id (generate.py PAD_ID)


@pytest.mark.parametrize("sim", [SimConfig(), SimConfig(integrator="euler", substeps=4), SimConfig(control_dt=0.01, substeps=3)])
def test_native_params_equal_oracle_folding(sim):
    ours = native_params(QuadParams(), sim, ControllerGains())
    ref = oracle.pack_params(QuadParams(), sim, ControllerGains())
    assert bytes(ours) == bytes(ref)


def test_hover_speed_matches_reference(gdyn):
    assert QuadParams().hover_speed == float(gdyn["hover_speed"])


def test_config_validation():
    from paper_2407_14783_b200.env import DistSpec, EnvConfig, SceneSpec, SensorSpec, env_config_from_table

    with pytest.raises(ConfigError):
        EnvConfig(num_agents=0)
    with pytest.raises(ConfigError):
        EnvConfig(mode="swarm", scenes=(SceneSpec(), SceneSpec()))
    with pytest.raises(ConfigError):
        DistSpec("uniform", low=[1, 1, 1], high=[0, 0, 0])
    with pytest.raises(ConfigError):
        SensorSpec(kind="lidar")
    with pytest.raises(ConfigError):
        env_config_from_table({"num_agents": 2, "bogus": 1})
    with pytest.raises(ConfigError):
        QuadParams(mass=-1.0)
    cfg = env_config_from_table({"num_agents": 3, "task": "navigation", "command_type": "lv",
                                 "scenes": [{"kind": "cluttered", "seed": 2}],
                                 "randomization": {"position": {"kind": "uniform", "low": [0, 0, 1], "high": [1, 1, 2]}},
                                 "sensors": [{"kind": "depth", "width": 32, "height": 16}]})
    assert cfg.num_agents == 3 and cfg.sensors[0].camera().width == 32


def _header_functions():
    text = open(os.path.join(ROOT, "include", "quadb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    path = nat.LIB_PATH
    assert os.path.exists(path), "build libquadb200.so first (python -m paper_2407_14783_b200.build)"
    lib = ctypes.CDLL(path)  # loading needs no GPU
    declared = _header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/quadb200.h but not exported"
        assert name in nat.SIGNATURES, f"{name} has no ctypes signature"
    assert set(nat.SIGNATURES) == set(declared)
    lib.qb_last_error.restype = ctypes.c_char_p
    assert lib.qb_version() == 1


def test_ctypes_struct_layouts_match_c():
    src = os.path.join(ROOT, "include")
    prog = ("#include <stdio.h>\n#include <stddef.h>\n#include \"quadb200.h\"\n"
            "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(qb_params), sizeof(qb_task),"
            " sizeof(qb_env_buffers), sizeof(qb_camera), sizeof(qb_dist), offsetof(qb_params, substeps),"
            " offsetof(qb_task, target), sizeof(qb_noise), sizeof(qb_sensor_obs), offsetof(qb_sensor_obs, src));"
            " printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(qb_io_view), offsetof(qb_io_view, centroid), sizeof(qb_io_copy),"
            " sizeof(qb_step_io), offsetof(qb_step_io, sensors));}\n")
    exe = "/tmp/qb_layout"
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    r = subprocess.run([cc, "-x", "c", "-I", src, "-o", exe, "-"], input=prog, text=True, capture_output=True)
    assert r.returncode == 0, r.stderr
    got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(nat.QbParams), ctypes.sizeof(nat.QbTask), ctypes.sizeof(nat.QbEnvBuffers),
            ctypes.sizeof(nat.QbCamera), ctypes.sizeof(nat.QbDist), nat.QbParams.substeps.offset, nat.QbTask.target.offset,
            ctypes.sizeof(nat.QbNoise), ctypes.sizeof(nat.QbSensorObs), nat.QbSensorObs.src.offset,
            ctypes.sizeof(nat.QbIoView), nat.QbIoView.centroid.offset, ctypes.sizeof(nat.QbIoCopy),
            ctypes.sizeof(nat.QbStepIo), nat.QbStepIo.sensors.offset]
    assert got == want


def test_product_has_no_cpu_fallback(monkeypatch):
    """The package must fail loudly (not silently fall back) without CUDA."""
    import torch

    from paper_2407_14783_b200.errors import NativeError

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    from paper_2407_14783_b200.env import make_env, navigation_config

    with pytest.raises(NativeError):
        make_env(navigation_config(num_agents=2))


def test_oracle_is_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2407_14783_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", src, flags=re.M), f


def test_pgm_export_matches_reference_bytes(tmp_path):
    """sensing.py:238-274: byte-identical 16-bit PGM files (golden from the reference)."""
    from conftest import golden
    from paper_2407_14783_b200 import sensing

    g = golden("pgm")
    sensing.export_depth_mm(tmp_path / "a.pgm", g["depth"])
    sensing.export_segmentation(tmp_path / "b.pgm", g["ids"])
    assert np.array_equal(np.frombuffer((tmp_path / "a.pgm").read_bytes(), np.uint8), g["depth_pgm"])
    assert np.array_equal(np.frombuffer((tmp_path / "b.pgm").read_bytes(), np.uint8), g["ids_pgm"])
    back = sensing.read_pgm16(tmp_path / "b.pgm")
    assert np.array_equal(back, np.clip(g["ids"], 0, 65535))


def test_build_bvh_dropin_layout():
    """bvh.build_bvh drop-in: the reference's flat layout, every primitive in
    exactly one leaf of <= LEAF_SIZE, boxes nested, children adjacent."""
    from conftest import golden
    from paper_2407_14783_b200.geometry.bvh import LEAF_SIZE, build_bvh

    g = golden("geometry")
    lo, hi = g["tess_prim_lo"], g["tess_prim_hi"]
    node_lo, node_hi, first, count, order = build_bvh(lo, hi)
    assert sorted(order.tolist()) == list(range(len(lo)))
    seen = np.zeros(len(lo), int)
    stack = [0]
    while stack:
        i = stack.pop()
        if count[i] > 0:
            assert count[i] <= LEAF_SIZE
            for p in order[first[i]:first[i] + count[i]]:
                seen[p] += 1
                assert np.all(lo[p] >= node_lo[i]) and np.all(hi[p] <= node_hi[i])
        else:
            for c in (first[i], first[i] + 1):
                assert np.all(node_lo[c] >= node_lo[i]) and np.all(node_hi[c] <= node_hi[i])
                stack.append(c)
    assert np.all(seen == 1)


def test_episode_log_bytes_match_reference(tmp_path):
    from conftest import golden
    from paper_2407_14783_b200.env.logs import EpisodeLogWriter, read_episode_log

    g = golden("logs")
    path = tmp_path / "ep.jsonl"
    with EpisodeLogWriter(path) as w:
        w.append_step(7, g["states"], g["actions"], g["rewards"],
                      {"collision": np.array([False, True, False]), "success": np.zeros(3, bool)})
    assert np.array_equal(np.frombuffer(path.read_bytes(), np.uint8), g["log"])
    assert read_episode_log(path)[1]["flags"] == {"collision": True, "success": False}


def test_abi_argument_validation_without_gpu():
    """Host-side validation of the newer entry points returns a status and a
    message before touching the device (no GPU needed)."""
    import ctypes

    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.params import native_params

    lib = nat.load(require_cuda=False)
    lib.qb_last_error.restype = ctypes.c_char_p
    P = native_params()
    # IMU sensors take Gaussian noise only (sensing.py:150-160 validity table)
    so = nat.QbSensorObs()
    so.kind, so.n_noise = nat.SENSOR_KINDS["imu"], 1
    so.noise[0].kind = nat.NOISE_KINDS["poisson"]
    so.out = 1
    state = (ctypes.c_float * 17)()
    rng = (ctypes.c_uint64 * 4)()
    b = nat.QbEnvBuffers()
    b.n, b.ld, b.dtype = 1, 1, nat.QB_F32
    b.state, b.rng = ctypes.addressof(state), ctypes.addressof(rng)
    rc = lib.qb_env_observe(P, b, 1, ctypes.cast(ctypes.pointer(so), ctypes.c_void_p), None)
    assert rc != 0 and b"not defined" in lib.qb_last_error()
    # Redwood is depth-only
    so.kind, so.noise[0].kind, so.src, so.width, so.height = nat.SENSOR_KINDS["segmentation"], nat.NOISE_KINDS["redwood"], 1, 4, 4
    assert lib.qb_env_observe(P, b, 1, ctypes.cast(ctypes.pointer(so), ctypes.c_void_p), None) != 0
    # unknown controller stage / missing state planes
    buf = (ctypes.c_float * 8)()
    assert lib.qb_control_stage(P, 7, nat.QB_F32, 1, 1, None, ctypes.addressof(buf), ctypes.addressof(buf), None, None) != 0
    assert lib.qb_control_stage(P, 1, nat.QB_F32, 1, 1, None, ctypes.addressof(buf), ctypes.addressof(buf), None, None) != 0
    assert b"state planes" in lib.qb_last_error()
    # split env step: phase 1 or 2 only, and the pre-step state buffer is required
    assert lib.qb_env_step_phase(P, 0, None, None, b, 3, None) != 0 and b"phase" in lib.qb_last_error()
    assert lib.qb_env_step_phase(P, 0, None, None, b, 1, None) != 0 and b"prev_state" in lib.qb_last_error()
    # empty primitive set
    cnt = ctypes.c_int64(0)
    assert lib.qb_bvh_build(0, None, None, ctypes.byref(cnt), None, None, None, None, None) != 0


def test_cluttered_mesh_scene_tessellates_the_nav_room():
    """Config 2's mesh room: the analytic navigation scene's objects (same
    Generator draws, same ids), boxes as 12 triangles, spheres as closed
    16-gon cylinders (64 triangles) circumscribing them."""
    import numpy as np

    from paper_2407_14783_b200.env import SceneSpec
    from paper_2407_14783_b200.geometry import Box, TriMesh

    kw = dict(seed=0, volume_lo=[-5, -5, 0], volume_hi=[5, 5, 4])
    ana = SceneSpec(kind="cluttered", **kw).materialize()
    mesh = SceneSpec(kind="cluttered_mesh", **kw).materialize()
    assert [o.id for o in ana.objects] == [o.id for o in mesh.objects]
    for a, m in zip(ana.objects, mesh.objects):
        assert isinstance(m.shape, TriMesh)
        v = m.shape.vertices
        if isinstance(a.shape, Box):
            assert len(m.shape.triangles) == 12
            loc = (v - a.shape.center) @ a.shape.rotation  # local coordinates: the box corners
            assert np.allclose(np.abs(loc), a.shape.half_extents)
        else:
            assert len(m.shape.triangles) == 64
            c, r = a.shape.center, a.shape.radius
            rad = np.linalg.norm(v[:, :2] - c[:2], axis=1)
            assert np.allclose(rad[rad > 1e-9], r) and (rad <= 1e-9).sum() == 2  # 32 ring vertices + 2 cap centres
            assert np.isclose(v[:, 2].min(), c[2] - r) and np.isclose(v[:, 2].max(), c[2] + r)
    t = mesh.arrays
    assert (t.prim_type == 2).all() and len(t) == 2076


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference's algorithm on the host cores,
    the driver's reference arm) prints one JSON line with the contract keys, on
    the same metric / unit / workload as our arm; runs without a GPU."""
    import json

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    import bench

    assert line["metric"] == bench.METRIC and line["config"]["workload"] == bench.WORKLOADS["c1"]
