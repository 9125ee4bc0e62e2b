#!/bin/bash
# A/B of compile-time variants (one GPU call): for each define set, build
# libmg with MG_NVCC_DEFINES and run a timing command; the default build is
# restored at the end.
# usage: bash tools/define_ab.sh TAG "CMD" "DEFS_A" "DEFS_B" ...
TAG=$1; CMD=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
i=0
for v in "$@"; do
  MG_NVCC_DEFINES="$v" python -m paper_2104_13755_b200.build > $O/build_$i.log 2>&1
  echo "== $i [$v]" >> $O/ab.txt
  MG_NVCC_DEFINES="$v" bash -c "$CMD" >> $O/ab.txt 2>&1
  i=$((i+1))
done
python -m paper_2104_13755_b200.build > $O/build_default.log 2>&1
