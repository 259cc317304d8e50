"""Time the split adjoint at config 4 (rotor, ctbr) with the library in QB_LIB_PATH."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2407_14783_b200 import gradients as G
from paper_2407_14783_b200.params import native_params
P = native_params()
n, T = 16384, 64
init = torch.zeros((17, n), device="cuda"); init[6] = 1.0; init[13:17] = 900.0
for kind in ("rotor", "ctbr"):
    acts = 900.0 + torch.randn((T, n, 4), device="cuda") * 20 if kind == "rotor" else \
        torch.cat([torch.full((T, n, 1), 9.81, device="cuda"), torch.randn((T, n, 3), device="cuda") * 0.3], 2)
    tape, _ = G.rollout_planes(P, kind, init, acts)
    g = torch.zeros_like(tape); g[-1, 0:3] = 1.0
    for _ in range(3):
        G.backward_planes(P, kind, tape, acts, g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        G.backward_planes(P, kind, tape, acts, g)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1] if len(sys.argv) > 1 else "", kind, "%.4f ms" % (e0.elapsed_time(e1) / 20), flush=True)
