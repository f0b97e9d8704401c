#!/bin/bash
# DP shapes per image width (tools/prof_dp_phases.py, forward cycles per row) — tools only
# usage: tools/sweep_phases.sh "W H" "v1 v2 ..."
for wh in $1; do :; done
IFS=';' read -ra SIZES <<< "${1:-7680 4320;3840 2160;2160 3072;1920 1080}"
for wh in "${SIZES[@]}"; do
  set -- $wh
  for v in ${VARIANTS:-"" 1 4 6 11 12 17 18}; do
    CARVE_DP_VARIANT=$v timeout 120 python tools/prof_dp_phases.py $1 $2 2>&1 | grep -v "^ phase2 first" | tr '\n' ' '; echo
  done
done
