#!/bin/bash
# A/B: CTA size of the small-level GS passes (k_lpr_sweep, 16/32 lanes per row): 256 / 128 / 64 threads;
# default build also carries the full-tile whole-level passes on the lanes-per-row levels
O=gpurun_out/r02k
mkdir -p $O
bash tools/define_ab.sh r02k "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5" "-DMG_LPR_GS_BLOCK=256" "-DMG_LPR_GS_BLOCK=128" "-DMG_LPR_GS_BLOCK=64"
