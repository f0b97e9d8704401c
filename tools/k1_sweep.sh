#!/bin/bash
# K1 launch shapes at C2/C3/C4 (bench kernel events) — tools only
for c in c2 c3 c4; do
  for v in 2 4 5 6; do
    CARVE_K1V=$v timeout 200 python bench.py --config $c --steps 2 --no-cpu-baseline > /tmp/k1_$c_$v.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('/tmp/k1_$c_$v.json')); k=d['kernels']['k_energy_full']; print('$c k1v=$v', round(k['avg_us'],2), 'us', round(k['gbs']/6536.4,4), d['verified_vs_golden'])"
  done
done
