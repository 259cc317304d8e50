mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p_eb.log 2>&1 && \
  $NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/r1_env_big python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p9.log 2>&1; echo envbig=$?
