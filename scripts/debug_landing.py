import dataclasses, sys
sys.path[:0] = [".", "tests"]
import numpy as np, torch
import oracle
from conftest import golden, scene_from_golden
from paper_2407_14783_b200 import _native as nat
from paper_2407_14783_b200.control import command_from_array
from paper_2407_14783_b200.env import landing_config, make_env
from paper_2407_14783_b200.sensing import render_state

g = golden("env_landing")
cfg = dataclasses.replace(landing_config(8), episode_max_steps=250)
env = make_env(cfg)
env.reset(seed=1)
osc = scene_from_golden(golden("geometry"), "landing")
for t in range(16):
    pre = g["full_state"][t - 1] if t > 0 else g["reset_full_state"]
    done_prev = (g["terminated"][t - 1] | g["truncated"][t - 1]) if t > 0 else np.zeros(8, bool)
    env._planes.copy_(torch.as_tensor(pre.T, dtype=torch.float32))
    env._needs_respawn.copy_(torch.as_tensor(done_prev.astype(np.uint8)))
    res = env.step(command_from_array("lv", g["actions"][t]))
seg_env = res.observations["vision"].cpu().numpy().copy()
st = env._planes.T.double().cpu().numpy()
print("agent_scene", env.agent_scene.cpu().numpy(), "steps", env.step_counts.cpu().numpy())
cam = cfg.sensors[0].camera()
o, r = oracle.camera_pose_world(st[:, 0:3], st[:, 6:10], cam.rotation, cam.translation)
d0, i0 = osc.render(o, r, 64, 64, cam.tan_half_h, cam.tan_half_v, cam.max_range)
for a in range(8):
    bad = seg_env[a] != i0[a]
    print("agent", a, "mismatch", int(bad.sum()), "pos", st[a, :3], "q", st[a, 6:10])
    if bad.any():
        ij = np.argwhere(bad)
        print("   pixels", ij[:12].tolist(), "gpu ids", seg_env[a][bad][:12], "ref", i0[a][bad][:12])
# re-render now (same state) through the state path, batch and single
seg = torch.empty((8, 64, 64), dtype=torch.int32, device="cuda")
cen = torch.empty((8, 2), device="cuda")
render_state(env.dev_scenes, cam, env._planes, env_scene=env.agent_scene, seg=seg, centroid_id=9, centroid=cen)
s2 = seg.cpu().numpy()
print("re-render batch mismatches vs env obs", int((s2 != seg_env).sum()), "vs oracle", int((s2 != i0).sum()))
render_state(env.dev_scenes, cam, env._planes, env_scene=env.agent_scene, seg=seg)
print("re-render no-centroid mismatches vs oracle", int((seg.cpu().numpy() != i0).sum()))
pl = env._planes.clone()
np.save("gpurun_out/landing_planes.npy", pl.cpu().numpy())
one = pl[:, 2:3].contiguous()
seg1 = torch.empty((1, 64, 64), dtype=torch.int32, device="cuda")
render_state(env.dev_scenes, cam, one, seg=seg1)
print("single exact-state render mismatches", int((seg1.cpu().numpy()[0] != i0[2]).sum()))
# planes with agent 2 in slot 0 of 8 (others copies)
eight = pl[:, [2] * 8].contiguous()
seg8 = torch.empty((8, 64, 64), dtype=torch.int32, device="cuda")
render_state(env.dev_scenes, cam, eight, seg=seg8)
print("8 copies mismatches per slot", [int((seg8.cpu().numpy()[k] != i0[2]).sum()) for k in range(8)])
from paper_2407_14783_b200.geometry.queries import raycasts
x = st[2]
o2, r2 = oracle.camera_pose_world(x[None, 0:3], x[None, 6:10], cam.rotation, cam.translation)
dirs, ijs = [], [(62, 62), (63, 60), (10, 10)]
for (i, j) in ijs:
    yy = (2 * (i + 0.5) / 64 - 1); xx = (2 * (j + 0.5) / 64 - 1)
    nn = np.sqrt(xx * xx + yy * yy + 1)
    dirs.append(r2[0] @ np.array([xx / nn, yy / nn, 1 / nn]))
t32, id32 = raycasts(env.dev_scenes, np.repeat(o2, 3, 0), np.array(dirs), 10 * np.sqrt(3), tmin=1e-9)
print("per-thread raycast_f", t32.cpu().numpy(), id32.cpu().numpy())
