for v in 7 12 0 13 2 14 1 15; do CARVE_DP_VARIANT=$v CARVE_DP_MAX_NCL=16 timeout 60 python tools/prof_dp_phases.py 1920 1080; done
