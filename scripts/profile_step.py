"""Short nav workload for ncu: a few env steps (K1+K3 fused + K2 render)."""
import sys
sys.path.insert(0, ".")
import argparse
import torch
from paper_2407_14783_b200.env import make_env, navigation_config
from paper_2407_14783_b200.control import LV

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=16384)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
env = make_env(navigation_config(0, a.envs, with_segmentation=True))
env.reset(seed=0)
act = torch.zeros((a.envs, 4), device="cuda")
act[:, 0] = 1.0
for _ in range(a.steps):
    env.step(LV(act[:, :3], act[:, 3]))
torch.cuda.synchronize()
print("ok")
