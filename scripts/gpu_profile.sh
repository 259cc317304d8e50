# ncu captures of every hot kernel (one GPU, one process at a time) + the bench launch list
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p_plain.log 2>&1 && \
  $NCU -k regex:k_render_cull -s 1 -c 1 -o gpurun_out/r1_render_cull python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p1.log 2>&1; echo cull=$?
$NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/r1_env_step python scripts/profile_kernels.py nav --envs 65536 > gpurun_out/p2.log 2>&1; echo envstep=$?
python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p_plain2.log 2>&1 && \
  $NCU -k regex:k_render_f -s 1 -c 1 -o gpurun_out/r1_render_bvh python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p3.log 2>&1; echo bvh=$?
$NCU -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/r1_dyn_step python scripts/profile_kernels.py dyn --envs 4194304 > gpurun_out/p4.log 2>&1; echo dyn=$?
python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/p_plain5.log 2>&1 && \
  $NCU -k regex:k_rollout -s 2 -c 2 -o gpurun_out/r1_bptt python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/p5.log 2>&1; echo bptt=$?
python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p_noise.log 2>&1 && \
  $NCU -k regex:k_env_observe -s 1 -c 1 -o gpurun_out/r1_observe python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p8.log 2>&1; echo observe=$?
python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p_eb.log 2>&1 && \
  $NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/r1_env_big python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p9.log 2>&1; echo envbig=$?
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p6.log 2>&1; echo launches=$?
# condense on the box (the .ncu-rep files exceed what gpurun copies back)
python scripts/make_profile_summary.py gpurun_out/prof > gpurun_out/prof_summary.log 2>&1; echo summary=$?
rm -f gpurun_out/r1_bptt.ncu-rep gpurun_out/r1_env_step.ncu-rep gpurun_out/r1_dyn_step.ncu-rep gpurun_out/r1_env_big.ncu-rep gpurun_out/r1_observe.ncu-rep
du -sh gpurun_out
