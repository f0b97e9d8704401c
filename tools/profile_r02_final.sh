#!/bin/bash
# Round-2 final-build ncu captures (run from the repo root under gpurun; reports stay in /tmp on the box,
# summaries land in gpurun_out/r02f/): one --set full launch each of the hot kernels per configuration.
set -u
O=gpurun_out/r02f; R=/tmp/r02f
mkdir -p $O $R
cap() {  # name kernel-regex skip command...
  local n=$1 k=$2 s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o $R/full_$n "$@" > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py $R/full_$n.ncu-rep > $O/summary_$n.txt 2>&1
}
cap c2_k_dp2 k_dp2 200 python tools/one_carve.py
cap c2_k_compact_bulk k_compact_bulk 100 python tools/one_carve.py
cap c3_k_energy k_energy 2 python tools/one_carve.py 3840 2160 3072 1728
cap c3_k_dp2 k_dp2 1300 python tools/one_carve.py 3840 2160 3072 1728
cap c4_k_energy k_energy 1 python tools/one_carve.py 7680 4320 7168 4320
cap c4_k_compact_bulk k_compact_bulk 20 python tools/one_carve.py 7680 4320 7168 4320
export CARVE_DEVICE_SPLIT_MIN=100000
cap c5_k_dp2 k_dp2 20 python tools/sweep_batch.py --child 1024
cap c5_k_compact_bulk k_compact_bulk 20 python tools/sweep_batch.py --child 1024
python tools/ncu_traffic.py $R > $O/traffic.json 2> $O/traffic.err
for f in $R/full_*.ncu-rep; do n=$(basename $f .ncu-rep); python tools/ncu_opmix.py $f > $O/opmix_$n.txt 2>&1; done
ls -la $O
