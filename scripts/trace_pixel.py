"""Trace one (camera, pixel) through k_render_f: needs the QB_RF_DEBUG build
(scripts/build_dbg.sh) and a saved body state (scripts/_dbg/c5px.npz, 17 floats);
writes the event log (kind, a, b, c) to gpurun_out/dbg_trace.npy."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2407_14783_b200._native as nat
nat.LIB_PATH = "/root/repo/scripts/_dbg/libquadb200_dbg.so"
from paper_2407_14783_b200.env import SceneSpec
from paper_2407_14783_b200.geometry.device import DeviceScenes
from paper_2407_14783_b200.sensing import CameraModel, DOWNWARD, render_state
d = np.load("scripts/_dbg/c5px.npz")
sc = SceneSpec(kind="indoor", seed=0).materialize()
ds = DeviceScenes([sc], device="cuda")
cam = CameraModel(rotation=DOWNWARD)
lib = nat.lib()
lib.qb_dbg_set(0, 20, 18)
pl = torch.as_tensor(d["state"][:, None], device="cuda").contiguous()
dep = torch.empty((1, 64, 64), device="cuda"); seg = torch.empty((1, 64, 64), dtype=torch.int32, device="cuda")
render_state(ds, cam, pl, depth=dep, seg=seg)
torch.cuda.synchronize()
buf = np.zeros((8192, 4), np.float32); n = ctypes.c_int(0)
lib.qb_dbg_get(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n))
print("depth", dep[0, 20, 18].item(), "events", n.value)
np.save("gpurun_out/dbg_trace.npy", buf[:n.value])
print("trace says best after target:", "see npy")
