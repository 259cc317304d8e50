mkdir -p gpurun_out
python scripts/profile_kernels.py indoor --envs 16384 > gpurun_out/p_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_render_f -s 1 -c 1 -o gpurun_out/r1b_render_bvh python scripts/profile_kernels.py indoor --envs 16384 > gpurun_out/p3.log 2>&1; echo bvh=$?
