"""Time K1 (qb_dynamics_step, CTBR, RK4 x2) at 16.7M envs with an L2 flush
between launches: ms per launch and HBM fraction at 152 B/env-step."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.run_dynamics_roofline(bench.peaks()[0])
print(json.dumps({k: r.get(k) for k in ("ms", "frac", "achieved", "env_steps_per_sec")}))
