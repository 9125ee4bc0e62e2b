#!/bin/bash
# One gpurun call: quick GPU tests of the changed kernels, then A/B of the
# one-tile GS kernel (MG_ONE_TILE) on C4 / C3 / C5 / C2.
O=gpurun_out/r02e
mkdir -p $O
python -m paper_2104_13755_b200.build > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "cotan_long_rows or full_size_parity or assembly_galerkin or solve_parity or launch_modes or dirichlet or bilaplacian or columns_are_independent" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/define_ab.sh r02e "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5; bash tools/gs_time.sh 2" "-DMG_ONE_TILE=1" "-DMG_ONE_TILE=0" "-DMG_GS_PER_SM=2"
