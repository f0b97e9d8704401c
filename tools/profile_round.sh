#!/bin/bash
# GPU-box profiling recipe for the round's committed evidence (run from the repo root under gpurun):
#   1. the default bench line (no profiler), 2. the ncu launch list of the same bench command,
#   3. one `ncu --set full` capture per hot kernel (DP, removal, K1) on the C2 workload.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
B="python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launches.log 2>&1
for k in k_dp2 k_compact_warp k_energy_rows; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/full_$k $B > gpurun_out/ncu_full_$k.log 2>&1 || true
done
ls -la gpurun_out
