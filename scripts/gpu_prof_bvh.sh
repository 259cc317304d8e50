mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p_plain2.log 2>&1 && \
  $NCU -k regex:k_render_f -s 1 -c 1 -o gpurun_out/r1_render_bvh python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p3.log 2>&1; echo bvh=$?
