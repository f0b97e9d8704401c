#!/bin/bash
# DP shapes per image width (tools/prof_dp_phases.py, forward cycles per row) — tools only
for wh in "7680 4320" "3840 2160" "2160 3072" "1920 1080"; do
  set -- $wh
  for v in "" 1 3 6 10 11 12 13 17 18; do
    CARVE_DP_VARIANT=$v timeout 120 python tools/prof_dp_phases.py $1 $2 2>&1 | grep -v "^ phase2 first" | tr '\n' ' '; echo
  done
done
