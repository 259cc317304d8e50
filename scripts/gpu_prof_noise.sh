mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p_noise.log 2>&1 && \
  $NCU -k regex:k_env_observe -s 1 -c 1 -o gpurun_out/r1_observe python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p8.log 2>&1; echo observe=$?
