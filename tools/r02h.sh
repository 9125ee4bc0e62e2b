#!/bin/bash
# One gpurun call: GPU tests, A/B of the 64-entry prefetch of the wide
# lanes-per-row groups (MG_LPR_PREFETCH64), GS trace.
O=gpurun_out/r02h
mkdir -p $O
python -m paper_2104_13755_b200.build > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/define_ab.sh r02h "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5; bash tools/gs_time.sh 2" "-DMG_LPR_PREFETCH64=1" "-DMG_LPR_PREFETCH64=0"
MG_NVCC_DEFINES="-DMG_GS_TRACE" python -m paper_2104_13755_b200.build > $O/build_trace.log 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE" timeout 600 python tools/gs_trace.py 4 > $O/trace_c4.txt 2>&1
python -m paper_2104_13755_b200.build > $O/build_default2.log 2>&1
