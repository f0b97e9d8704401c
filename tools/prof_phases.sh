for w in 32 64 128 512 1920; do CARVE_DP_VARIANT=12 timeout 60 python tools/prof_dp_phases.py $w 1080; done
