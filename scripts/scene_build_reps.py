"""qb_scene_create_device on the config-5 hall, repeated: wall time per build."""
import ctypes
import time

import numpy as np
import torch

from paper_2407_14783_b200 import _native as nat
from paper_2407_14783_b200.geometry import indoor_mesh_scene
from paper_2407_14783_b200.geometry.device import flatten_on_device

sc = indoor_mesh_scene(0)
parts = flatten_on_device(sc, torch.device("cuda"))
torch.cuda.synchronize()
offs = np.array([0, len(parts[0])], np.int64)
for r in range(8):
    h = ctypes.c_void_p()
    t0 = time.perf_counter()
    nat.check(nat.lib().qb_scene_create_device(1, offs.ctypes.data_as(ctypes.c_void_p), *[p.data_ptr() for p in parts],
                                               ctypes.byref(h), nat.stream_of()))
    t1 = time.perf_counter()
    nat.lib().qb_scene_destroy(h)
    t2 = time.perf_counter()
    print(f"rep {r}: create {1e3 * (t1 - t0):.1f} ms, destroy {1e3 * (t2 - t1):.1f} ms")
