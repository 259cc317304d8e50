# ncu capture of the K2 culling renderer: raw metrics + source-line table
mkdir -p gpurun_out
M=${1:-8}
python -m paper_2407_14783_b200.build  > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python scripts/profile_kernels.py nav --envs 100 > gpurun_out/p_envs0.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 2 -c 1 -o gpurun_out/envs \
  python scripts/profile_kernels.py nav --envs 100 > gpurun_out/p_envs.log 2>&1; echo ncu=$?
ncu -i gpurun_out/envs.ncu-rep --page raw --csv > gpurun_out/envs_raw.csv 2>/dev/null
ncu -i gpurun_out/envs.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/envs_src.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/envs_src.csv 60 > gpurun_out/envs_lines.txt
rm -f gpurun_out/envs.ncu-rep gpurun_out/envs_src.csv
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/envs_raw.csv')))
h, v = rows[0], rows[2]
want = ['gpu__time_duration.sum', 'sm__inst_executed_pipe_fp64', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'pipe_fp64', 'pipe_alu', 'pipe_fma', 'pipe_xu', 'stall']
for k, x in zip(h, v):
    if any(w in k for w in want) and 'pct' in k or k in want[:8]:
        print(k, x)
PY
