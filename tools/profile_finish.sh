#!/bin/bash
# Run on the GPU box after tools/profile_round.sh: distil the ncu reports into the text/JSON
# summaries committed under profiles/ and drop the large reports gpurun cannot bring back
# (its copy-back limit is 64 MiB).
cd gpurun_out
(for f in full_k_dp2 full_k_compact_bulk full_k_energy_rows full_batch_k_dp2 full_batch_k_compact_bulk; do
   [ -f $f.ncu-rep ] || continue
   echo "### $f.ncu-rep"; python ../tools/ncu_summary.py $f.ncu-rep 2>&1 | head -30
   python ../tools/ncu_hot.py $f.ncu-rep 0 2>&1 | head -1
 done) > ncu_full_summary.txt
python ../tools/dp_ncu_metrics.py full_k_dp2.ncu-rep > dp_ncu_metrics.json 2>/dev/null || true
python ../tools/dp_ncu_metrics.py full_batch_k_dp2.ncu-rep 2>/dev/null | sed 's/C2 bench, one DP launch/C5 batch of 1024 images, 21st DP launch/' > batch_dp_ncu_metrics.json || true
python - <<'PY'
import csv, io, json, subprocess, os
def dram(rep):
    if not os.path.exists(rep): return None
    out = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    r = list(csv.reader(io.StringIO(out))); h=r[0]; u=r[1]; v=r[2]
    m = {k:(val,unit) for k,val,unit in zip(h,v,u)}
    sc = {'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
    return int(sum(float(m[k][0].replace(',',''))*sc[m[k][1]] for k in ('dram__bytes_read.sum','dram__bytes_write.sum')))
t = {"source": "ncu --set full --clock-control none, one launch each (tools/profile_round.sh + tools/profile_finish.sh; profiles/r01_ncu_full_summary.txt), cold cache: C2 = 5th launch of each kernel of `python bench.py --steps 2 --warmup 3 --no-batch --no-cpu-baseline`; C5 = 21st launch of `python tools/sweep_batch.py --child 1024`",
     "bytes_per_launch": {"c2": {"k_dp_seam": dram('full_k_dp2.ncu-rep'), "k_compact": dram('full_k_compact_bulk.ncu-rep'), "k_energy_full": dram('full_k_energy_rows.ncu-rep')},
                          "c5": {"k_dp_seam": dram('full_batch_k_dp2.ncu-rep'), "k_compact": dram('full_batch_k_compact_bulk.ncu-rep')}},
     "workload": {"c2": "C2 1920x1080, W ~1916 at the captured launch", "c5": "C5 1024 images 1024x768, W = 1004 at the captured launch"}}
json.dump(t, open('traffic.json','w'), indent=1)
PY
(python ../tools/launch_summary.py launches_c2.csv; echo; echo "C5 (python bench.py --config c5 --steps 1 --warmup 3, first 400 launches):"; python ../tools/launch_summary.py launches_c5.csv) > launches_summary.txt 2>&1
du -sh *.ncu-rep; rm -f *.ncu-rep
ls -la
