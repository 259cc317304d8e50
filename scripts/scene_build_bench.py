"""F3 measurement: the config-5 hall (5e5 triangles) built on the host (binned
SAH) and on the device (flatten + LBVH), build times and the FP32 BVH render
rate of 32768 down cameras with each tree (frames stay on the device)."""
import time

import numpy as np
import torch

from paper_2407_14783_b200.geometry import indoor_mesh_scene
from paper_2407_14783_b200.geometry.device import DeviceScenes
from paper_2407_14783_b200.sensing import DOWNWARD, CameraModel, render_state

sc = indoor_mesh_scene(0)
sc.arrays
DeviceScenes([sc], build="device")  # warm-up (CUB, allocator)
torch.cuda.synchronize()
res = {}
for build in ("host", "device"):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ds = DeviceScenes([sc], build=build)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    res[build] = (ds, min(ts))
n = 32768
rng = np.random.default_rng(0)
pl = torch.zeros((17, n), device="cuda")
pl[0:3] = torch.as_tensor(rng.uniform([-12, -12, 1.0], [12, 12, 4.5], (n, 3)).T, dtype=torch.float32)
pl[6] = 1.0
cam = CameraModel(rotation=DOWNWARD)
d = torch.empty((n, 64, 64), device="cuda")
s = torch.empty((n, 64, 64), dtype=torch.int32, device="cuda")
out = {}
for build, (ds, bt) in res.items():
    render_state(ds, cam, pl, depth=d, seg=s, mode=1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        render_state(ds, cam, pl, depth=d, seg=s, mode=1)
    ev[1].record()
    torch.cuda.synchronize()
    fps = 5 * n / ev[0].elapsed_time(ev[1]) * 1e3
    out[build] = (d.clone(), s.clone())
    print(f"{build:6s} build {bt * 1e3:8.1f} ms  nodes {ds.n_nodes:8d} depth {ds.max_depth:3d}  render {fps:.4g} frames/s")
# the device build alone (flatten excluded): qb_scene_create_device
import ctypes
from paper_2407_14783_b200 import _native as nat
from paper_2407_14783_b200.geometry.device import flatten_on_device
t0 = time.perf_counter()
parts = flatten_on_device(sc, torch.device("cuda"))
torch.cuda.synchronize()
t1 = time.perf_counter()
offs = np.array([0, len(parts[0])], np.int64)
h = ctypes.c_void_p()
nat.check(nat.lib().qb_scene_create_device(1, offs.ctypes.data_as(ctypes.c_void_p), *[p.data_ptr() for p in parts],
                                           ctypes.byref(h), nat.stream_of()))
t2 = time.perf_counter()
nat.lib().qb_scene_destroy(h)
print(f"device flatten {1e3 * (t1 - t0):.1f} ms, qb_scene_create_device {1e3 * (t2 - t1):.1f} ms")
print("renders equal:", torch.equal(out["host"][0], out["device"][0]) and torch.equal(out["host"][1], out["device"][1]))
