#!/bin/bash
# One gpurun call: full GPU tests of the mixed-width lanes-per-row tiles, A/B
# against the uniform widths and with the next-pass L2 prefetch, GS trace.
O=gpurun_out/r02g
mkdir -p $O
python -m paper_2104_13755_b200.build > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/define_ab.sh r02g "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5" "-DMG_MIXED_LPR=1" "-DMG_MIXED_LPR=0" "-DMG_MIXED_LPR=1 -DMG_NEXT_PREFETCH=1"
MG_NVCC_DEFINES="-DMG_GS_TRACE" python -m paper_2104_13755_b200.build > $O/build_trace.log 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE" timeout 600 python tools/gs_trace.py 4 > $O/trace_c4_mixed.txt 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE" timeout 600 python tools/gs_trace.py 3 > $O/trace_c3_mixed.txt 2>&1
python -m paper_2104_13755_b200.build > $O/build_default2.log 2>&1
