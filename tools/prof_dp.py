"""GPU-side timing probe (not a bench): per-kernel event times of one carve
under different conditions, to separate clock effects from kernel cost."""
import json, subprocess, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_21207_b200 as cv

W, H, TW = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1920, 1080, 1728))]
img = cv.make_test_image(W, H)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty((H, TW, 3), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def one(profile=False, do_flush=False):
    if do_flush: flush.zero_()
    if profile: cv.set_kernel_events(True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); cv.carve_device(d_in.data_ptr(), W, H, TW, H, d_out.data_ptr(), None, s.cuda_stream); b.record(s)
    torch.cuda.synchronize()
    st = cv.kernel_event_stats() if profile else None
    if profile: cv.set_kernel_events(False)
    return a.elapsed_time(b), st
for _ in range(3): one()
res = {}
for name, kw in [("plain", {}), ("flush", {"do_flush": True}), ("prof", {"profile": True}), ("prof_flush", {"profile": True, "do_flush": True})]:
    ts = []; st = None
    for _ in range(3):
        t, st = one(**kw); ts.append(t)
    res[name] = {"ms": ts, "dp_avg_us": (1e3 * st["k_dp_seam"]["ms_total"] / st["k_dp_seam"]["launches"]) if st else None,
                 "compact_avg_us": (1e3 * st["k_compact"]["ms_total"] / st["k_compact"]["launches"]) if st else None}
print(json.dumps(res, indent=1))
