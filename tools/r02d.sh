#!/bin/bash
# Galerkin phase-1 vector loads A/B + coarsest-factor shuffle variant A/B +
# 32x32 factor micro-benchmarks (one gpurun call)
O=gpurun_out/r02d
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/chol32 tools/chol32_bench.cu > $O/chol32_build.log 2>&1 && /tmp/chol32 > $O/chol32.txt 2>&1
bash tools/define_ab.sh r02d_chol "python tools/chol_trace.py 5 2>&1 | grep -E 'panel  5|total'; timeout 600 python -m pytest tests -m gpu -q -x -k 'assembly_galerkin' 2>&1 | tail -1" "-DMG_CHOL_TRACE" "-DMG_CHOL_TRACE -DMG_CHOL_SHFL=1"
bash tools/define_ab.sh r02d "timeout 900 python -m pytest tests -m gpu -q -x -k 'assembly_galerkin or full_size_parity' 2>&1 | tail -1; for c in 4 3 5; do python tools/galerkin_time.py \$c; done" "-DMG_GALT_VEC=1" "-DMG_GALT_VEC=0" "-DMG_GALT_VEC=1"
echo done > $O/DONE
