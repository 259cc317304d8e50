"""bindings.step host-to-host time of a workload (bench.run_e2e) under the
current QB_IO_SLICES (run once per setting: the library reads it once)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = bench.workload_config(kind, bench.ENVS[kind])
r = bench.run_e2e(cfg, 0, 1, kind)
print(f"{kind} slices={os.environ.get('QB_IO_SLICES', '16')} e2e {r['value']:.4g} env-steps/s "
      f"{r['ms_per_step']:.2f} ms/step d2h {r['d2h_bytes_per_step'] / 1e9:.2f} GB")
