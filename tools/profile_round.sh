#!/bin/bash
# GPU-box profiling recipe for the round's committed evidence (run from the repo root under gpurun):
#   1. the default bench line (no profiler), 2. the ncu launch list of the same bench command (C2 part)
#      and of the C5 batch bench, 3. one `ncu --set full` capture per hot kernel: DP, removal and K1 on
#      the C2 workload, the fused batch DP and the batch removal on C5 (1024 images).
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
B="python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_c5.log 2>&1 || true
for k in k_dp2 k_compact_bulk k_energy_rows; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/full_$k $B > gpurun_out/ncu_full_$k.log 2>&1 || true
done
for k in k_dp2 k_compact_bulk; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/full_batch_$k \
      python tools/sweep_batch.py --child 1024 > gpurun_out/ncu_full_batch_$k.log 2>&1 || true
done
ls -la gpurun_out
