"""Bench-state parity diagnosis: config 3 after ~1.5k steps (the state bench.py's parity leg sees)."""
import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2407_14783_b200._native as nat
from oracle.parity import env_step_parity, oracle_scenes
from paper_2407_14783_b200.control import LV
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1460
env, cfg = bench.env_workload("c3", 0, 1, 65536)
env.reset(seed=0)
a = bench.make_actions("c3", 65536, 8, 0)
for i in range(steps):
    env._bufs.action = a[i % 8].data_ptr()
    nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
torch.cuda.synchronize()
n = env.num_agents
rng = np.random.default_rng(99)
for rep in range(3):
    act = np.concatenate([rng.normal(scale=1.5, size=(n, 3)) + [1.0, 0, 0], rng.uniform(-np.pi, np.pi, (n, 1))], 1)
    res = env.step(LV(act[:, :3], act[:, 3]))
    torch.cuda.synchronize()
    sample = np.sort(rng.choice(n, size=2048, replace=False))
    r = env_step_parity(env, cfg, res.observations, act, oracle_scenes(cfg), (QuadParams(), SimConfig(), ControllerGains()), sample)
    print(json.dumps(r["render"]))
    st = env._planes.T.double().cpu().numpy()
    for d in r.get("non_grazing_detail", [])[:16]:
        c = d["camera"]
        d["speed"] = float(np.linalg.norm(st[c, 3:6])); d["omega"] = float(np.linalg.norm(st[c, 10:13]))
        d["steps"] = int(env.step_counts[c]); d["qnorm"] = float(np.linalg.norm(st[c, 6:10]))
        print(json.dumps(d))

# --- which stage disagrees: cull (mode 2) / BVH (mode 1) FP32 kernels, FP64 kernel, oracle, oracle on normalised q
from paper_2407_14783_b200.sensing import render_state
from oracle import camera_pose_world
det = r.get("non_grazing_detail", [])
cams = sorted({d["camera"] for d in det})
if cams:
    idx = torch.as_tensor(cams, device="cuda")
    pl = env._planes[:, idx].contiguous()
    cam = cfg.sensors[0].camera()
    k = len(cams)
    outs = {}
    for mode in (1, 2):
        d = torch.zeros((k, 64, 64), device="cuda"); s = torch.zeros((k, 64, 64), dtype=torch.int32, device="cuda")
        render_state(env.dev_scenes, cam, pl, depth=d, seg=s, mode=mode)
        outs[f"f32_mode{mode}"] = d.double().cpu().numpy()
    pl64 = pl.double().contiguous()
    d = torch.zeros((k, 64, 64), dtype=torch.float64, device="cuda"); s = torch.zeros((k, 64, 64), dtype=torch.int32, device="cuda")
    render_state(env.dev_scenes, cam, pl64, depth=d, seg=s)
    outs["f64_kernel"] = d.cpu().numpy()
    stk = pl64.T.cpu().numpy()
    sc = oracle_scenes(cfg)[0]
    o_, r_ = camera_pose_world(stk[:, 0:3], stk[:, 6:10], cam.rotation, cam.translation)
    outs["oracle"] = sc.render(o_, r_, 64, 64, cam.tan_half_h, cam.tan_half_v, cam.max_range)[0]
    qn = stk[:, 6:10] / np.linalg.norm(stk[:, 6:10], axis=1, keepdims=True)
    o2, r2 = camera_pose_world(stk[:, 0:3], qn, cam.rotation, cam.translation)
    outs["oracle_qnorm"] = sc.render(o2, r2, 64, 64, cam.tan_half_h, cam.tan_half_v, cam.max_range)[0]
    for dd in det[:10]:
        c = cams.index(dd["camera"]); i, j = dd["pixel"]
        print({kk: round(float(v[c, i, j]), 7) for kk, v in outs.items()}, "id", dd["ref_id"])
    sc_arr = cfg.scenes[0].materialize().arrays
    ids = sorted({dd["ref_id"] for dd in det})
    print("prim types of failing ids:", {i: int(sc_arr.prim_type[np.nonzero(sc_arr.prim_object_id == i)[0][0]]) for i in ids})
