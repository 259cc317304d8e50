"""K1 adjoint timing at config 4 (16384 envs x H=64) and the 8-GPU strong-scaling shard (2048 envs):
split two-warp kernel vs the one-thread-per-env kernel (QB_ADJOINT_FUSED=1)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_14783_b200 import gradients as G
from paper_2407_14783_b200.params import native_params

P = native_params()
for n in (16384, 2048, 131072):
    T = 64
    init = torch.zeros((17, n), device="cuda"); init[6] = 1.0; init[13:17] = 900.0
    init[0:3] = (torch.rand((3, n), device="cuda") - 0.5) * 0.2
    for kind in ("rotor", "ctbr"):
        acts = 900.0 + torch.randn((T, n, 4), device="cuda") * 20 if kind == "rotor" else \
            torch.cat([torch.full((T, n, 1), 9.81, device="cuda"), torch.randn((T, n, 3), device="cuda") * 0.3], 2)
        tape, _ = G.rollout_planes(P, kind, init, acts)
        g = torch.zeros_like(tape); g[-1, 0:3] = 1.0
        res = {}
        for mode in ("split", "fused"):
            os.environ["QB_ADJOINT_FUSED"] = "1" if mode == "fused" else "0"
            for _ in range(3):
                G.backward_planes(P, kind, tape, acts, g)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                G.backward_planes(P, kind, tape, acts, g)
            e1.record(); torch.cuda.synchronize()
            res[mode] = e0.elapsed_time(e1) / 20
        e0.record()
        for _ in range(20):
            G.rollout_planes(P, kind, init, acts)
        e1.record(); torch.cuda.synchronize()
        print(f"n={n} {kind}: bwd split {res['split']:.4f} ms, fused {res['fused']:.4f} ms ({res['fused']/res['split']:.2f}x); "
              f"fwd {e0.elapsed_time(e1)/20:.4f} ms", flush=True)
