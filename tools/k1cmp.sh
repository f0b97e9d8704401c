for k in ${KS:-1 0}; do for c in c4 c3; do CARVE_K1=$k timeout 400 python bench.py --config $c --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/k1_${k}_$c.json; python -c "
import json; d=json.load(open('gpurun_out/k1_${k}_$c.json')); v=d['kernels']['k_energy_full']; print('K1=$k $c', round(v['avg_us'],1), 'us', round(v['gbs']), 'GB/s', d['ms_per_step'])"; done; done
