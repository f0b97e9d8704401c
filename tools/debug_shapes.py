import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2410_21207_b200 as cv
shapes = [(w, h) for h in range(1, 7) for w in range(1, 14)]
start = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for idx in range(start, len(shapes)):
    w, h = shapes[idx]
    e = (np.arange(w * h, dtype=np.float64).reshape(h, w) * 7) % 5
    try:
        cv.dp_seam(e)
    except Exception as ex:
        print("FAIL", idx, w, h, ex, flush=True)
        sys.exit(idx + 1)
print("ALLOK", flush=True)
