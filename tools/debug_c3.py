import sys, os, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, paper_2410_21207_b200 as cv, oracle
    w, h, tw, th = map(int, sys.argv[2:6])
    img = cv.make_test_image(w, h)
    try:
        out = cv.carve(img, tw, th)
        ok = "?"
        if (w - tw) + (h - th) <= 12 and w * h <= 4e6:
            ok = np.array_equal(out, oracle.port().carve(img, tw, th))
        print("OK", w, h, tw, th, ok)
    except Exception as ex:
        print("ERR", w, h, tw, th, ex)
    sys.exit(0)
cases = [(3840, 2160, 3830, 2160), (3840, 2160, 3840, 2150), (2160, 3072, 2150, 3072), (1000, 3000, 990, 3000),
         (2160, 1000, 2150, 1000), (1000, 2000, 995, 2000), (500, 2000, 495, 2000), (300, 1100, 295, 1100),
         (300, 1025, 295, 1025), (300, 1024, 295, 1024), (300, 1023, 295, 1023)]
for v in sys.argv[1].split(","):
    for c in cases:
        env = dict(os.environ, CARVE_DP_VARIANT=v, CARVE_DP_MAX_NCL="16")
        r = subprocess.run([sys.executable, __file__, "--child", *map(str, c)], env=env, capture_output=True, text=True, timeout=300)
        print("v" + v, (r.stdout.strip() or r.stderr.strip()[-200:]), flush=True)
