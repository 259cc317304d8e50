# A/B of two prebuilt libraries (paper_2407_14783_b200/_ab/{base,new}.so) on the small-batch workloads
mkdir -p gpurun_out
for v in base new base new; do
  cp paper_2407_14783_b200/_ab/$v.so paper_2407_14783_b200/libquadb200.so
  for w in ${WL:-c2 c2a}; do
    timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_${v}_$w.log 2>&1
    echo "$v $w $(tail -1 gpurun_out/ab_${v}_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])")"
  done
done
cp paper_2407_14783_b200/_ab/new.so paper_2407_14783_b200/libquadb200.so
