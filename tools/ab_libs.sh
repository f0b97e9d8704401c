#!/bin/bash
# A/B of experimental libraries (tools only): tools/ab_libs.sh name1 name2 ... (build/exp/NAME/libcarve_cuda.so)
# per library: the C5-shaped batch at 1024 and 128 images (one launch per seam) and the C2 bench line
export CARVE_DEVICE_SPLIT_MIN=100000
for rep in 1 2; do
for n in "$@"; do
  export CARVE_LIB=build/exp/$n/libcarve_cuda.so
  for b in 1024 128; do
    echo "$n $(python tools/sweep_batch.py --child $b)"
  done
  echo "$n c2 $(python bench.py --no-batch --no-cpu-baseline --steps 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d.get("c3",{}).get("value"))')"
done
done
