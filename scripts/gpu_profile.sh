# ncu captures of every hot kernel (one GPU, one process at a time) + the bench launch list.
# QB_ROUND (default r2) names the captures; condensed on the box into gpurun_out/prof (-> profiles/).
mkdir -p gpurun_out
R=${QB_ROUND:-r2}
export QB_ROUND=$R
NCU="ncu --set full --clock-control none --import-source on"
python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p_plain.log 2>&1 && \
  $NCU -k regex:k_render_cull -s 1 -c 1 -o gpurun_out/${R}_render_cull python scripts/profile_kernels.py nav --envs 16384 > gpurun_out/p1.log 2>&1; echo cull=$?
$NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/${R}_env_step python scripts/profile_kernels.py nav --envs 65536 > gpurun_out/p2.log 2>&1; echo envstep=$?
python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p_plain2.log 2>&1 && \
  $NCU -k regex:k_render_f -s 1 -c 1 -o gpurun_out/${R}_render_bvh python scripts/profile_kernels.py indoor --envs 32768 > gpurun_out/p3.log 2>&1; echo bvh=$?
$NCU -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/${R}_dyn_step python scripts/profile_kernels.py dyn --envs 4194304 > gpurun_out/p4.log 2>&1; echo dyn=$?
python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/p_plain5.log 2>&1 && \
  $NCU -k regex:k_rollout -s 2 -c 2 -o gpurun_out/${R}_bptt python scripts/profile_kernels.py bptt --envs 16384 > gpurun_out/p5.log 2>&1; echo bptt=$?
python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p_noise.log 2>&1 && \
  $NCU -k regex:k_env_observe -s 1 -c 1 -o gpurun_out/${R}_observe python scripts/profile_kernels.py noise --envs 16384 > gpurun_out/p8.log 2>&1; echo observe=$?
python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p_eb.log 2>&1 && \
  $NCU -k regex:k_env_step -s 1 -c 1 -o gpurun_out/${R}_env_big python scripts/profile_kernels.py envbig --envs 4194304 > gpurun_out/p9.log 2>&1; echo envbig=$?
# launch list of the default bench command (config 3 line only: the sub-records / sustained leg would
# put thousands of launches under ncu)
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/b_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/p6.log 2>&1; echo launches=$?
# condense on the box (the .ncu-rep files exceed what gpurun copies back)
python scripts/make_profile_summary.py gpurun_out/prof > gpurun_out/prof_summary.log 2>&1; echo summary=$?
for k in render_cull render_bvh observe env_big bptt; do
  [ -f gpurun_out/prof/${R}_${k}_source.csv ] && python scripts/ncu_lines.py gpurun_out/prof/${R}_${k}_source.csv 60 > gpurun_out/prof/${R}_${k}_hot_lines.txt
done
rm -f gpurun_out/${R}_bptt.ncu-rep gpurun_out/${R}_env_step.ncu-rep gpurun_out/${R}_dyn_step.ncu-rep gpurun_out/${R}_env_big.ncu-rep gpurun_out/${R}_observe.ncu-rep
du -sh gpurun_out
