# ncu capture of the K1 adjoint at config 4 (source-level stall reasons)
mkdir -p gpurun_out/prof
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/pa.log 2>&1 && \
  $NCU -k regex:k_rollout_bwd -s 1 -c 1 -o gpurun_out/adj python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/pa2.log 2>&1; echo adj=$?
ncu -i gpurun_out/adj.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/adj_source.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/prof/adj_source.csv 45 > gpurun_out/prof/adj_hot_lines.txt
ncu -i gpurun_out/adj.ncu-rep --page details --csv > gpurun_out/prof/adj_details.csv 2>/dev/null
rm -f gpurun_out/adj.ncu-rep gpurun_out/prof/adj_source.csv
