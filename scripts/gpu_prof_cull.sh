mkdir -p gpurun_out
python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p_plain.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:k_render_cull -s 1 -c 1 -o gpurun_out/r1b_render_cull python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p1.log 2>&1; echo cull=$?
