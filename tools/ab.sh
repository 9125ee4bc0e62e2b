#!/bin/bash
# A/B bench of env variants, interleaved and repeated (one GPU call).
# usage: bash tools/ab.sh TAG CONFIG REPEATS "ENV_A" "ENV_B" ...
TAG=$1; CFG=$2; REP=$3; shift 3
O=gpurun_out/$TAG
mkdir -p $O
for r in $(seq 1 $REP); do
  i=0
  for v in "$@"; do
    env $v timeout 600 python bench.py --config $CFG --steps 8 --warmup 3 --no-cpu-baseline > $O/ab_c${CFG}_${i}_$r.json 2> /dev/null
    echo "$i $r $v" >> $O/ab_c${CFG}_index.txt
    i=$((i+1))
  done
done
