"""GPU sweep (not a bench): DP variants for the batched C5 path (n images per launch)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch, numpy as np
    import paper_2410_21207_b200 as cv
    n = int(sys.argv[2]); W, H, TW = 1024, 768, 896
    imgs = np.stack([cv.make_test_image(W, H, k) for k in range(n)])
    d_in = torch.from_numpy(imgs).cuda(); d_out = torch.empty((n, H, TW, 3), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    run = lambda: cv.carve_batch_device(d_in.data_ptr(), n, W, H, TW, H, d_out.data_ptr(), s.cuda_stream)
    run(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); run(); b.record(s); torch.cuda.synchronize()
    cv.set_kernel_events(True); run(); torch.cuda.synchronize(); st = cv.kernel_event_stats(); cv.set_kernel_events(False)
    print(json.dumps({"variant": os.environ.get("CARVE_DP_VARIANT"), "n": n, "ms": a.elapsed_time(b),
                      "img_per_s": n / (a.elapsed_time(b) / 1e3),
                      "dp_ms_per_seam": st["k_dp_seam"]["ms_total"] / st["k_dp_seam"]["launches"],
                      "compact_ms_per_seam": st["k_compact"]["ms_total"] / st["k_compact"]["launches"]}))
    sys.exit(0)
n = sys.argv[1] if len(sys.argv) > 1 else "256"
for v in os.environ.get("VARIANTS", "5,6,0,3").split(","):
    env = dict(os.environ, CARVE_DP_VARIANT=v, CARVE_DP_MAX_NCL="16")
    r = subprocess.run([sys.executable, __file__, "--child", n], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or ("FAIL v%s: %s" % (v, r.stderr.strip()[-300:])), flush=True)
