#!/bin/bash
# A/B: one-tile GS kernel also at 2 lanes per row (C4 level 1) now that the tiles are balanced;
# GPU tests on the candidate build.
O=gpurun_out/r02l
mkdir -p $O
bash tools/define_ab.sh r02l "bash tools/gs_time.sh 4; bash tools/gs_time.sh 4" "-DMG_ONE_TILE_MIN_LPR=4" "-DMG_ONE_TILE_MIN_LPR=2"
MG_NVCC_DEFINES="-DMG_ONE_TILE_MIN_LPR=2" python -m paper_2104_13755_b200.build > $O/build_c.log 2>&1
MG_NVCC_DEFINES="-DMG_ONE_TILE_MIN_LPR=2" timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_minlpr2.log 2>&1; echo "rc=$?" >> $O/pytest_minlpr2.log
python -m paper_2104_13755_b200.build > $O/build_default2.log 2>&1
