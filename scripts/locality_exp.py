"""Does camera locality per SM matter for the BVH renderer?  Same cameras,
(a) spread over the hall in random order, (b) sorted by cell, (c) all inside
one small patch."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2407_14783_b200._native as nat
from paper_2407_14783_b200.geometry import indoor_mesh_scene
from paper_2407_14783_b200.sensing import CameraModel, DOWNWARD

scene = indoor_mesh_scene(0)
dev = scene.device()
cam = CameraModel(rotation=DOWNWARD)
n = 131072
rng = np.random.default_rng(0)
def run(org, label):
    rot = np.tile(DOWNWARD.reshape(1, 9), (n, 1))
    o = torch.as_tensor(org, dtype=torch.float32, device="cuda").contiguous()
    r = torch.as_tensor(rot, dtype=torch.float32, device="cuda").contiguous()
    d = torch.empty((n, 64, 64), device="cuda"); s = torch.empty((n, 64, 64), dtype=torch.int32, device="cuda")
    def go():
        nat.check(nat.lib().qb_render_poses(dev.handle, cam.native(1), nat.QB_F32, n, nat.ptr(o), nat.ptr(r), None,
                                           nat.ptr(d), nat.ptr(s), None, None, 0, nat.stream_of()))
    go(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); go(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"{label:10s} {np.median(ts):8.2f} ms  {n / np.median(ts) * 1e3:.3e} frames/s  mean depth {float(d.mean()):.3f}")

full = np.stack([rng.uniform(-12, 12, n), rng.uniform(-12, 12, n), rng.uniform(1.0, 4.5, n)], 1)
run(full, "random")
cell = (np.floor((full[:, 0] + 12) / 0.5) * 100 + np.floor((full[:, 1] + 12) / 0.5)).astype(int)
run(full[np.argsort(cell, kind="stable")], "sorted")
patch = np.stack([rng.uniform(4, 6, n), rng.uniform(4, 6, n), rng.uniform(1.0, 4.5, n)], 1)
run(patch, "patch2m")
