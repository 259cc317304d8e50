# ncu capture (source lines) of one kernel of a profile_kernels.py workload:
#   bash scripts/gpu_prof_one.sh <regex> <mode> <envs> <name>
mkdir -p gpurun_out/prof
python scripts/profile_kernels.py $2 --envs $3 > gpurun_out/po_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -o gpurun_out/$4 \
    python scripts/profile_kernels.py $2 --envs $3 > gpurun_out/po.log 2>&1; echo prof=$?
ncu -i gpurun_out/$4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/$4_source.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/prof/$4_source.csv 60 > gpurun_out/prof/$4_hot_lines.txt
ncu -i gpurun_out/$4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread > gpurun_out/prof/$4_raw.csv 2>/dev/null
rm -f gpurun_out/$4.ncu-rep gpurun_out/prof/$4_source.csv
