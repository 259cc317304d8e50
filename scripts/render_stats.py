"""Node-visit statistics of the FP32 BVH packet renderer (build with -D QB_RF_STATS -D QB_RF_WIDE=0)."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch

import paper_2407_14783_b200._native as nat
from paper_2407_14783_b200.control import LV
from paper_2407_14783_b200.env import DistSpec, EnvConfig, InitRandomization, SceneSpec, SensorSpec, make_env

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = EnvConfig(num_agents=n, task="landing", command_type="lv", episode_max_steps=512,
                scenes=(SceneSpec(kind="indoor", seed=0),),
                randomization=InitRandomization(position=DistSpec("uniform", low=[-12, -12, 1.0], high=[12, 12, 4.5])),
                min_spawn_clearance=0.3,
                sensors=(SensorSpec(kind="depth", name="depth", orientation="down"),
                         SensorSpec(kind="segmentation", name="vision", orientation="down")))
env = make_env(cfg)
env.reset(seed=0)
lib = nat.lib()
buf = (ctypes.c_ulonglong * 4)()
lib.qb_debug_render_stats(buf)
base = list(buf)
act = torch.zeros((n, 4), device="cuda")
r = env.step(LV(act[:, :3], act[:, 3]))
torch.cuda.synchronize()
lib.qb_debug_render_stats(buf)
d = [b - a for a, b in zip(base, buf)]
tiles = d[0]
print(f"tiles {tiles}  visits/tile {d[1] / tiles:.1f}  prims/tile {d[2] / tiles:.1f}  active lanes {d[3] / tiles:.1f}")
dep = r.observations["depth"]
print("depth mean", float(dep.mean()), "min", float(dep.min()), "max", float(dep.max()))
