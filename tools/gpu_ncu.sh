#!/bin/bash
# One gpurun call: plain run of the ncu target, then one `ncu --set full`
# capture of the kernels matching REGEX.
# usage: bash tools/gpu_ncu.sh TAG REGEX COUNT [CONFIG] [CYCLES]
TAG=$1; RX=$2; CNT=${3:-3}; CFG=${4:-4}; CYC=${5:-1}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ncu_target.py --config $CFG --cycles $CYC > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c $CNT \
  -o $O/prof python tools/ncu_target.py --config $CFG --cycles $CYC > $O/ncu.log 2>&1
echo "rc=$?" >> $O/ncu.log
