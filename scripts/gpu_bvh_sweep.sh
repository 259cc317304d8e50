# host SAH tree quality sweep for config 5: bins per axis x max leaf size
mkdir -p gpurun_out
for cfg in "16 4" "32 4" "64 4" "16 2" "16 8" "32 2"; do
set -- $cfg
python -m paper_2407_14783_b200.build -D QB_BVH_BINS=$1 -D QB_BVH_LEAF=$2 > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
echo "bins $1 leaf $2: $(PYTHONPATH=. timeout 300 python scripts/scene_build_bench.py 2>&1 | grep '^host')"
done
