#!/bin/bash
# quick A/B variant: recompile ONE translation unit with extra -D flags and link it with the
# production objects of the other units -> scripts/_dbg/<name>.so (select with QB_LIB_PATH)
# usage: bash scripts/quick_variant.sh <name> <unit.cu> -DFLAG ...
set -e
cd "$(dirname "$0")/.."
name=$1; unit=$2; shift 2
mkdir -p scripts/_dbg/q_$name
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -O2 -Iinclude \
    -Ipaper_2407_14783_b200/csrc -ccbin /usr/bin/g++ "$@" -c paper_2407_14783_b200/csrc/$unit -o scripts/_dbg/q_$name/${unit%.cu}.o
objs=""
for o in paper_2407_14783_b200/_build/*.o; do
  b=$(basename $o)
  if [ "$b" = "${unit%.cu}.o" ]; then objs="$objs scripts/_dbg/q_$name/$b"; else objs="$objs $o"; fi
done
$NV $ARCH -ccbin /usr/bin/g++ -shared -cudart static -o scripts/_dbg/$name.so $objs
echo scripts/_dbg/$name.so
