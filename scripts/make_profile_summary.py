"""Condense the round's ncu captures (gpurun_out/<round>_*.ncu-rep, QB_ROUND=r1|r2) into profiles/.

profiles/ncu_summary.json  per-kernel figures bench.py quotes (DRAM bytes per
                           unit -> roofline "traffic"), one entry per kernel
profiles/<round>_ncu_raw_summary.json  the raw metric rows (scripts/ncu_summary.py)
"""
import json
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_summary import read  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
DEST = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles")  # (on the GPU box: gpurun_out/prof)
RND = os.environ.get("QB_ROUND", "r1")
ROUND_TEXT = {"r1": "round 1", "r2": "round 2"}.get(RND, RND)
CAPTURES = {  # report -> (kernel key, units in the captured launch, unit)
    f"{RND}_render_cull": ("k_render_cull", 16384, "camera (64x64, depth+seg), 69-prim nav room"),
    f"{RND}_render_bvh": ("k_render_f", 32768, "camera (64x64, down depth+seg), 5e5-tri hall"),
    f"{RND}_env_step": ("k_env_step", 65536, "env"),
    f"{RND}_dyn_step": ("k_dyn_step", 4194304, "env"),
    f"{RND}_bptt": (None, 16384 * 64, "env-step"),
    f"{RND}_observe": ("k_env_observe", 16384, "env (C3n sensor pass: depth N -> Redwood, seg salt-and-pepper, IMU)"),
    f"{RND}_env_big": ("k_env_step_4m", 4194304, "env (K1+K3 fused step, free flight, garage)"),
}


def num(v):
    return float(str(v).split()[0])


def scale(v):
    unit = str(v).split()[1] if len(str(v).split()) > 1 else ""
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1.0)


summary, raw = {}, {}
for rep, (key, units, unit) in CAPTURES.items():
    path = os.path.join(OUT, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    rows = read(path)
    raw[rep] = rows
    for r in rows:
        k = key or ("k_rollout_fwd" if "rollout_fwd" in r["kernel"] else "k_rollout_bwd")
        dram = num(r["dram__bytes_read.sum"]) * scale(r["dram__bytes_read.sum"]) + \
            num(r["dram__bytes_write.sum"]) * scale(r["dram__bytes_write.sum"])
        summary[k] = {
            "units": units, "unit": unit,
            "dram_bytes_per_unit": dram / units,
            "time_ms": num(r["gpu__time_duration.sum"]) * scale(r["gpu__time_duration.sum"]),
            "issue_active_pct": num(r["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            "warps_active_pct": num(r["sm__warps_active.avg.pct_of_peak_sustained_active"]),
            "dram_throughput_pct": num(r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
            "fma_pipe_pct": num(r["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]),
            "l1_hit_pct": num(r["l1tex__t_sector_hit_rate.pct"]),
            "l2_hit_pct": num(r["lts__t_sector_hit_rate.pct"]),
            "registers": num(r["launch__registers_per_thread"]),
            "warp_instructions_per_unit": num(r["smsp__inst_executed.sum"]) / units,
            "source": f"{rep}.ncu-rep (ncu --set full --clock-control none, {ROUND_TEXT})",
        }
os.makedirs(DEST, exist_ok=True)
with open(os.path.join(DEST, "ncu_summary.json"), "w") as f:
    json.dump(summary, f, indent=1)
with open(os.path.join(DEST, f"{RND}_ncu_raw_summary.json"), "w") as f:
    json.dump(raw, f, indent=1)
if os.path.exists(os.path.join(OUT, f"{RND}_launches.csv")):
    shutil.copy(os.path.join(OUT, f"{RND}_launches.csv"), os.path.join(DEST, f"{RND}_launch_list.csv"))
# per-line source tables of the two renderers (for reading back without the .ncu-rep)
for rep in (f"{RND}_render_cull", f"{RND}_render_bvh", f"{RND}_observe", f"{RND}_env_big", f"{RND}_bptt"):
    path = os.path.join(OUT, rep + ".ncu-rep")
    if os.path.exists(path):
        import subprocess

        out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                             capture_output=True, text=True).stdout
        with open(os.path.join(DEST, rep + "_source.csv"), "w") as f:
            f.write(out)
print(json.dumps({k: {kk: v[kk] for kk in ("time_ms", "dram_bytes_per_unit", "issue_active_pct", "warps_active_pct",
                                            "warp_instructions_per_unit")} for k, v in summary.items()}, indent=1))
