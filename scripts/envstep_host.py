"""Host cost of the batched Python env.step at config 1 (100 envs): numpy actions, device results."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_14783_b200.control import CTBR
from paper_2407_14783_b200.env import EnvConfig, make_env

env = make_env(EnvConfig(num_agents=100, command_type="ctbr", episode_max_steps=1000))
env.reset(seed=0)
rng = np.random.default_rng(0)
a = [CTBR(np.full(100, 9.81), rng.normal(scale=0.3, size=(100, 3))) for _ in range(8)]
for k in range(50):
    env.step(a[k % 8])
torch.cuda.synchronize()
K = 2000
t = time.perf_counter()
for k in range(K):
    r = env.step(a[k % 8])
torch.cuda.synchronize()
print(f"env.step numpy CTBR, 100 envs: {(time.perf_counter() - t) / K * 1e6:.1f} us/step")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for k in range(500):
    r = env.step(a[k % 8])
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
