"""Distil the DP kernel's ncu --set full capture into the figures the north star asks for
(per-row latency, shared-memory bandwidth fraction, time stalled on
barriers). Usage: python tools/dp_ncu_metrics.py full_k_dp2.ncu-rep > profiles/r01_dp_ncu_metrics.json"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, v = raw[0], raw[2]
m = dict(zip(h, v))
f = lambda k: float(str(m.get(k, "nan")).replace(",", ""))
nsm_active = int(f("launch__grid_size"))  # one CTA per SM (cluster kernel, 1 block/SM)
nsm = int(f("device__attribute_multiprocessor_count"))
smem_all = f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed") / 100
# stall reasons from the raw page (smsp__pcsamp_warps_issue_stalled_*)
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in h
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
total = sum(st.values()) or 1.0
share = {k: round(x / total, 4) for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x / total >= 0.005}
out = {
    "source": rep.split("/")[-1] + " (ncu --set full --clock-control none, C2 bench, one DP launch)",
    "duration_us": f("gpu__time_duration.sum") / 1e3 if f("gpu__time_duration.sum") > 1e3 else f("gpu__time_duration.sum"),
    "active_sms": nsm_active, "sms": nsm,
    "smem_wavefronts_frac_of_peak_all_sms": smem_all,
    "smem_wavefronts_frac_of_peak_active_sms": smem_all * nsm / max(nsm_active, 1),
    "smem_bank_reads_max_sm_frac": f("l1tex__data_bank_reads.max.pct_of_peak_sustained_elapsed") / 100,
    "stall_share": share,
    "barrier_stall_share": round((st.get("barrier", 0) + st.get("membar", 0)) / total, 4),
    "note": "halo waits are mbarrier try_wait spins (long_scoreboard on the wait loop), cluster barriers are 'barrier'",
}
print(json.dumps(out, indent=1))
