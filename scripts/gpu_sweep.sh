# tuning sweep: BVH kernel block/regs (c5), K1 register cap (roofline_dynamics)
mkdir -p gpurun_out
for cfg in "128 8" "128 6" "64 12" "64 16" "256 4"; do
  set -- $cfg
  python -m paper_2407_14783_b200.build -D QB_RF_BLOCK=$1 -D QB_RF_MINB=$2 > /dev/null 2>&1
  timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw_c5_$1_$2.log 2>&1; echo c5_$1_$2=$?
done
for m in 8 6 5 4; do
  python -m paper_2407_14783_b200.build -D QB_DYN_MINB=$m > /dev/null 2>&1
  timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw_k1_$m.log 2>&1; echo k1_$m=$?
done
