"""Survivor statistics of the culling renderer at config 3 (build with -D QB_CULL_STATS):
candidates per camera after frustum culling, survivors per 8x8 tile by record type."""
import ctypes, sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2407_14783_b200._native as nat

env, cfg = bench.env_workload("c3", 0, 1, 65536)
env.reset(seed=0)
a = bench.make_actions("c3", 65536, 8, 0)
for i in range(200):
    env._bufs.action = a[i % 8].data_ptr()
    nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
lib = nat.lib()
buf = (ctypes.c_ulonglong * 8)()
lib.qb_debug_cull_stats(buf)
base = list(buf)
env._render()
torch.cuda.synchronize()
lib.qb_debug_cull_stats(buf)
d = [b - a for a, b in zip(base, buf)]
cams, cand, tiles = d[0], d[1], d[2]
print(f"cameras {cams}, candidates/camera {cand / cams:.2f}, tiles {tiles} ({tiles / cams:.1f}/camera)")
print("survivors per tile: sphere %.2f AABB %.2f OBB %.2f generic %.2f total %.2f" % (
    d[3] / tiles, d[4] / tiles, d[5] / tiles, d[6] / tiles, sum(d[3:7]) / tiles))
