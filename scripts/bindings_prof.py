"""Where the host-to-host bindings step spends its time (config 1, 100 envs)."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2407_14783_b200 import bindings, _native as nat
from paper_2407_14783_b200.env import EnvConfig

def tm(f, K=3000):
    for _ in range(100): f()
    t = time.perf_counter()
    for _ in range(K): f()
    return (time.perf_counter() - t) / K * 1e6

lib = nat.lib()
print("ctypes qb_version: %.2f us" % tm(lambda: lib.qb_version()))
h = bindings.make_env(EnvConfig(num_agents=100, command_type="ctbr", episode_max_steps=1000))
out = h.outputs()
bindings.reset(h, 0, out=out)
a = torch.zeros((100, 4), pin_memory=True).numpy(); a[:, 0] = 9.81
print("full step: %.2f us" % tm(lambda: bindings.step(h, a, out=out)))
print("observe only (pack + D2H + sync): %.2f us" % tm(lambda: h._run(False, None, out)))
io = h._io
args = h._args
def raw():
    io.step = 1; io.host_action = a.ctypes.data
    lib.qb_env_step_io(*args, h._io_ref, h._stream_ptr)
print("raw ctypes step_io: %.2f us" % tm(raw))
io.n_copies = 0
print("raw, no D2H: %.2f us" % tm(raw))
io.n_packs = 0; io.state_rows = None
print("raw, no pack/D2H: %.2f us" % tm(raw))
io.sync = 0
def raw_nosync():
    raw(); torch.cuda.synchronize()
print("raw, no pack/D2H, torch sync: %.2f us" % tm(raw_nosync))
env = h.env
s = torch.cuda.current_stream()
def kern():
    lib.qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, h._stream_ptr)
print("qb_env_step launch only: %.2f us" % tm(lambda: (kern(), torch.cuda.synchronize())))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [kern() for _ in range(1000)]; e1.record(); torch.cuda.synchronize()
print("qb_env_step back-to-back GPU: %.2f us" % (e0.elapsed_time(e1)))
