"""Time the fused K1+K3 env step (qb_env_step) at 4M envs, free flight in the
garage (the bench's roofline_env_step workload): ms per launch, GB/s at 272
algorithmic B/env-step."""
import torch

import paper_2407_14783_b200._native as nat
from paper_2407_14783_b200.env import EnvConfig, make_env

n = 1 << 22
env = make_env(EnvConfig(num_agents=n, command_type="ctbr", episode_max_steps=10**6))
env.reset(seed=0)
act = torch.zeros((n, 4), device="cuda")
act[:, 0] = 9.81
act[:, 1:] = torch.randn((n, 3), device="cuda") * 0.3
env._bufs.action = act.data_ptr()


def launch():
    nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))


for _ in range(3):
    launch()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize()
ev[0].record()
for _ in range(20):
    launch()
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 20
print(f"env_step 4M: {ms:.4f} ms/launch, {272 * n / ms / 1e6:.0f} GB/s")
