import sys, os, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import numpy as np, paper_2410_21207_b200 as cv
    w, h, tw, th = map(int, sys.argv[2:6])
    img = cv.make_test_image(w, h)
    try:
        cv.carve(img, tw, th); print("OK", tw, th)
    except Exception as ex:
        print("ERR", tw, th, ex)
    sys.exit(0)
def run(*c):
    r = subprocess.run([sys.executable, __file__, "--child", *map(str, c)], capture_output=True, text=True, timeout=300)
    out = r.stdout.strip() or r.stderr.strip()[-300:]
    print(out, flush=True)
    return out.startswith("OK")
# width phase bisection
lo, hi = 3072, 3840   # hi ok (no seams)
if run(3840, 2160, 3072, 2160):
    print("width phase fine")
    lo2, hi2 = 1728, 2160
    while hi2 - lo2 > 1:
        mid = (lo2 + hi2) // 2
        if run(3840, 2160, 3072, mid): hi2 = mid
        else: lo2 = mid
    print("height phase first failing target", lo2)
else:
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if run(3840, 2160, mid, 2160): hi = mid
        else: lo = mid
    print("width phase first failing target", lo)
