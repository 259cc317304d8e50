"""Host-to-host step latency of the flat bindings (qb_env_step_io) vs env.step, config 1 / 2a sizes."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2407_14783_b200 import bindings
from paper_2407_14783_b200.env import EnvConfig, navigation_config

for name, cfg in (("c1", EnvConfig(num_agents=100, command_type="ctbr", episode_max_steps=1000)),
                  ("c2a", navigation_config(0, 100))):
    h = bindings.make_env(cfg)
    out = h.outputs()
    bindings.reset(h, 0, out=out)
    a = torch.zeros((100, 4), pin_memory=True).numpy()
    a[:, 0] = 9.81 if name == "c1" else 0.5
    for _ in range(50):
        bindings.step(h, a, out=out)
    for fresh in (False, True):
        t = time.perf_counter()
        K = 2000
        for _ in range(K):
            bindings.step(h, a, out=None if fresh else out)
        dt = (time.perf_counter() - t) / K
        print(f"{name} bindings fresh={fresh}: {dt*1e6:.1f} us/step, {100/dt:.3g} env-steps/s")
