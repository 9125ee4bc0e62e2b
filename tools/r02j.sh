#!/bin/bash
# A/B: balanced tiles on the lanes-per-row levels (MG_LPR_BALANCE), + GPU tests of the default
O=gpurun_out/r02j
mkdir -p $O
bash tools/define_ab.sh r02j "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5" "-DMG_LPR_BALANCE=1" "-DMG_LPR_BALANCE=0"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
