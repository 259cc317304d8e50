mkdir -p gpurun_out
python scripts/profile_step.py --envs 16384 --steps 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python scripts/profile_step.py --envs 16384 --steps 3 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 -o gpurun_out/prof_render_r1 python scripts/profile_step.py --envs 16384 --steps 3 > gpurun_out/ncu_render.log 2>&1; echo render=$?
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 1 -c 1 -o gpurun_out/prof_envstep_r1 python scripts/profile_step.py --envs 16384 --steps 3 > gpurun_out/ncu_env.log 2>&1; echo env=$?
