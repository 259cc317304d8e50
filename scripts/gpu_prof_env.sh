mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py hover --envs 100 > gpurun_out/p_hover.log 2>&1 && \
  $NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/r1_env_hover python scripts/profile_kernels.py hover --envs 100 > gpurun_out/p7.log 2>&1; echo hover=$?
