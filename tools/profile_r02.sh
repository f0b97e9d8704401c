#!/bin/bash
# Round-2 GPU-box profiling recipe (run from the repo root under gpurun; outputs in gpurun_out/r02/):
#  1. bench lines: the default line (C2 + C3 + C5 + per-rank shares, with CPU baselines), and C4;
#  2. ncu launch lists (gpu__time_duration.sum, --clock-control none) of the C2 bench command and
#     of one C5 batch carve;
#  3. one `ncu --set full` capture per HBM-bound kernel at C3 and C4 (K1 k_energy_rows, K4
#     k_compact_bulk) and the DP at C2 -> DRAM bytes per launch (tools/ncu_traffic.py).
set -u
O=gpurun_out/r02
mkdir -p $O
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --config c4 --steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
B="python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file $O/launches_c2.csv $B > $O/ncu_launches_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c5.csv \
    python tools/sweep_batch.py --child 1024 > $O/ncu_launches_c5.log 2>&1
for cfg in "c3 3840 2160 3072 1728" "c4 7680 4320 7168 4320"; do
  set -- $cfg
  ncu --set full --clock-control none --import-source on -k regex:k_energy_rows -s 2 -c 1 -o $O/full_$1_k_energy_rows \
      python tools/one_carve.py $2 $3 $4 $5 > $O/ncu_full_$1_k1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_compact_bulk -s 20 -c 1 -o $O/full_$1_k_compact_bulk \
      python tools/one_carve.py $2 $3 $4 $5 > $O/ncu_full_$1_k4.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_dp2 -s 200 -c 1 -o $O/full_c2_k_dp2 \
    python tools/one_carve.py > $O/ncu_full_c2_dp.log 2>&1
python tools/ncu_traffic.py $O > $O/traffic.json 2> $O/traffic.err
ls -la $O
