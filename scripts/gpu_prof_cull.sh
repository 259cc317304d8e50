mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p_plain.log 2>&1 && \
  $NCU -k regex:k_render_cull -s 1 -c 1 -o gpurun_out/r1_render_cull python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p1.log 2>&1; echo cull=$?
