import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle, paper_2410_21207_b200 as cv
P = oracle.port()
rng = np.random.default_rng(1)
for (w, h) in [(3, 3), (9, 6), (33, 5), (130, 20), (1921, 7)]:
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    s = [int(rng.integers(0, w))]
    for _ in range(h - 1):
        s.append(int(np.clip(s[-1] + rng.integers(-1, 2), 0, w - 1)))
    a = cv.remove_seam(img, s); b = P.remove_seam(img, s)
    bad = np.argwhere((a != b).any(-1))
    print("remove", w, h, "seam", s[:8], "bad", len(bad), bad[:5].tolist())
img = cv.make_test_image(96, 64)
e = cv.energy_e1_rgb(img); print("energy eq", np.array_equal(e, P.energy_e1_rgb(img)))
sg = cv.dp_seam(e).seam; sp = P.dp_seam(e)[0]; print("seam eq", np.array_equal(sg, sp))
for tw, th in [(95, 64), (90, 64), (80, 64), (96, 63), (96, 56), (80, 56)]:
    o, ss, _ = cv.carve(img, tw, th, seams=True); po, ps = P.carve(img, tw, th, seams=True)
    flat = np.concatenate(ss) if ss else np.zeros(0, np.int32)
    first = next((k for k in range(len(ss)) if not np.array_equal(ss[k], ps[sum(len(x) for x in ss[:k]):][:len(ss[k])])), None)
    print("carve", tw, th, "pix eq", np.array_equal(o, po), "seams eq", np.array_equal(flat, ps), "first bad seam", first)
