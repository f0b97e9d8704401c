"""Quick single-image carve checks against the oracle (tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, paper_2410_21207_b200 as cv
port = oracle.port()
for (w, h, tw, th) in [(40, 30, 36, 30), (10, 8, 10, 5), (200, 120, 180, 100), (1920, 1080, 1910, 1080), (3, 3, 1, 1)]:
    img = port.make_test_image(w, h)
    want, ws = port.carve(img, tw, th, seams=True)
    got, gs, _ = cv.carve(img, tw, th, seams=True)
    flat = np.concatenate(gs) if gs else np.zeros(0, np.int32)
    print((w, h, tw, th), "ok" if np.array_equal(got, want) and np.array_equal(flat, ws) else "MISMATCH", flush=True)
