#!/bin/bash
# One gpurun call: tests of the changed kernels, A/B of the cotan rows per
# group, GS pass timeline (trace build) on C4 and C3.
O=gpurun_out/r02f
mkdir -p $O
python -m paper_2104_13755_b200.build > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "cotan_long_rows or full_size_parity or assembly_galerkin or solve_parity or launch_modes or dirichlet or bilaplacian or mcf_loop" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
MG_NVCC_DEFINES="-DMG_GS_TRACE -DMG_ONE_TILE_MIN_LPR=2" python -m paper_2104_13755_b200.build > $O/build_trace.log 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE -DMG_ONE_TILE_MIN_LPR=2" timeout 600 python tools/gs_trace.py 4 > $O/trace_c4_onetile.txt 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE -DMG_ONE_TILE=0" python -m paper_2104_13755_b200.build > $O/build_trace2.log 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE -DMG_ONE_TILE=0" timeout 600 python tools/gs_trace.py 4 > $O/trace_c4_pipe.txt 2>&1
MG_NVCC_DEFINES="-DMG_GS_TRACE -DMG_ONE_TILE=0" timeout 600 python tools/gs_trace.py 3 > $O/trace_c3_pipe.txt 2>&1
bash tools/define_ab.sh r02f "bash tools/gs_time.sh 4; bash tools/gs_time.sh 5; bash tools/gs_time.sh 3" "-DMG_COT_R=2" "-DMG_COT_R=1" "-DMG_COT_R=4"
