#!/bin/bash
# Launch-mode sweep: bench lines for env-var variants of libmg (one GPU call).
# usage: bash tools/sweep.sh TAG CONFIG "ENV1" "ENV2" ...
TAG=$1; CFG=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
i=0
for v in "$@"; do
  env $v timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > $O/sweep_c${CFG}_$i.json 2> $O/sweep_c${CFG}_$i.err
  echo "$i $v" >> $O/sweep_c${CFG}_index.txt
  i=$((i+1))
done
