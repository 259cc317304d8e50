"""Small deterministic workloads for ncu captures (one mode per process)."""
import sys
sys.path.insert(0, ".")
import argparse
import torch

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["nav", "indoor", "dyn", "bptt", "hover", "noise", "envbig"])
ap.add_argument("--envs", type=int, default=16384)
a = ap.parse_args()
if a.mode in ("nav", "indoor"):
    from paper_2407_14783_b200.control import LV
    from paper_2407_14783_b200.env import DistSpec, EnvConfig, InitRandomization, SceneSpec, SensorSpec, make_env, navigation_config
    if a.mode == "nav":
        cfg = navigation_config(0, a.envs, with_segmentation=True)
    else:
        cfg = EnvConfig(num_agents=a.envs, task="landing", command_type="lv", scenes=(SceneSpec(kind="indoor", seed=0),),
                        randomization=InitRandomization(position=DistSpec("uniform", low=[-12, -12, 1.0], high=[12, 12, 4.5])),
                        sensors=(SensorSpec(kind="depth", name="depth", orientation="down"),
                                 SensorSpec(kind="segmentation", name="vision", orientation="down")))
    env = make_env(cfg)
    env.reset(seed=0)
    act = torch.zeros((a.envs, 4), device="cuda")
    act[:, 0] = 1.0
    for _ in range(3):
        env.step(LV(act[:, :3], act[:, 3]))
elif a.mode == "noise":  # config 3 + the c3n sensor noise chains
    import bench
    from paper_2407_14783_b200.control import LV

    env, _ = bench.env_workload("c3n", 0, 1, a.envs)
    env.reset(seed=0)
    act = torch.zeros((a.envs, 4), device="cuda")
    act[:, 0] = 1.0
    for _ in range(3):
        env.step(LV(act[:, :3], act[:, 3]))
elif a.mode == "envbig":  # the bench's K1+K3 roofline workload (free flight, garage)
    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.env import EnvConfig, make_env

    env = make_env(EnvConfig(num_agents=a.envs, command_type="ctbr", episode_max_steps=10**6))
    env.reset(seed=0)
    act = torch.zeros((a.envs, 4), device="cuda")
    act[:, 0] = 9.81
    env._bufs.action = act.data_ptr()
    for _ in range(3):
        nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
elif a.mode == "hover":  # config 1: 100 envs, CTBR, default scene, no sensors
    from paper_2407_14783_b200.control import CTBR
    from paper_2407_14783_b200.env import EnvConfig, make_env
    env = make_env(EnvConfig(num_agents=a.envs, command_type="ctbr", episode_max_steps=1000))
    env.reset(seed=0)
    act = torch.zeros((a.envs, 4), device="cuda")
    act[:, 0] = 9.81
    for _ in range(3):
        env.step(CTBR(act[:, 0], act[:, 1:]))
elif a.mode == "dyn":
    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.params import native_params
    n = a.envs
    P = native_params()
    pl = torch.zeros((17, n), device="cuda"); pl[6] = 1.0; pl[13:17] = 900.0
    act = torch.zeros((n, 4), device="cuda"); act[:, 0] = 9.81
    for _ in range(3):
        nat.check(nat.lib().qb_dynamics_step(P, nat.CMD["ctbr"], nat.QB_F32, n, n, nat.ptr(pl), nat.ptr(act), None, None, nat.stream_of()))
else:
    from paper_2407_14783_b200 import gradients as G
    from paper_2407_14783_b200.params import native_params
    n, T = a.envs, 64
    P = native_params()
    init = torch.zeros((17, n), device="cuda"); init[6] = 1.0; init[13:17] = 900.0
    acts = 900.0 + torch.randn((T, n, 4), device="cuda") * 20
    for _ in range(2):
        tape, _ = G.rollout_planes(P, "rotor", init, acts)
        g = torch.zeros_like(tape); g[-1, 0:3] = 1.0
        G.backward_planes(P, "rotor", tape, acts, g)
torch.cuda.synchronize()
print("ok", a.mode)
