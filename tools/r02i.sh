#!/bin/bash
# A/B: entries per row prefetched by the wide lanes-per-row groups (64 / 128)
bash tools/define_ab.sh r02i "bash tools/gs_time.sh 4; bash tools/gs_time.sh 3; bash tools/gs_time.sh 5" "-DMG_LPR_WIDE_ENTRIES=64" "-DMG_LPR_WIDE_ENTRIES=128"
