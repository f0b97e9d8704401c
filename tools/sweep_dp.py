"""GPU sweep (not a bench): DP kernel variant x config -> avg DP launch time,
per-row ns, carve correctness vs golden. Usage: python tools/sweep_dp.py [c1 c2 ...]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = {"c1": (512, 512, 448, 512), "c2": (1920, 1080, 1728, 1080), "c3": (3840, 2160, 3072, 1728),
       "c4": (7680, 4320, 7168, 4320), "c5": (1024, 768, 896, 768)}
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch, numpy as np
    import paper_2410_21207_b200 as cv, oracle
    name = sys.argv[2]
    W, H, TW, TH = CFG[name]
    gold = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))["configs"]
    img = cv.make_test_image(W, H)
    d_in = torch.from_numpy(img).cuda(); d_out = torch.empty((TH, TW, 3), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    run = lambda: cv.carve_device(d_in.data_ptr(), W, H, TW, TH, d_out.data_ptr(), None, s.cuda_stream)
    run(); torch.cuda.synchronize()
    ok = (f"{oracle.fnv1a64(d_out.cpu().numpy()):016x}" == gold[name.upper()]["output"]) if "output" in gold.get(name.upper(), {}) else None
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); run(); b.record(s); torch.cuda.synchronize()
    cv.set_kernel_events(True); run(); torch.cuda.synchronize(); st = cv.kernel_event_stats(); cv.set_kernel_events(False)
    dp = st.get("k_dp_seam"); cp = st.get("k_compact")
    print(json.dumps({"cfg": name, "variant": os.environ.get("CARVE_DP_VARIANT"), "ok": ok, "carve_ms": a.elapsed_time(b),
                      "dp_us": 1e3 * dp["ms_total"] / dp["launches"], "ns_per_row": 1e6 * dp["ms_total"] / dp["launches"] / H,
                      "compact_us": 1e3 * cp["ms_total"] / cp["launches"]}))
    sys.exit(0)
names = sys.argv[1:] or ["c2"]
variants = os.environ.get("VARIANTS", "0,1,2,3,4,5,6,7,8").split(",")
for name in names:
    for v in variants:
        env = dict(os.environ, CARVE_DP_VARIANT=v, CARVE_DP_MAX_NCL="16")
        r = subprocess.run([sys.executable, __file__, "--child", name], env=env, capture_output=True, text=True, timeout=600)
        print(r.stdout.strip() or ("FAIL v%s %s: %s" % (v, name, r.stderr.strip()[-300:])), flush=True)
