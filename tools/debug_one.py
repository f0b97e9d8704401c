import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2410_21207_b200 as cv
z = np.load("tests/golden/corpus.npz")
e = z["e13"].astype(np.float64)
print(e.shape)
try:
    r = cv.dp_seam(e); print("ok", r.seam)
except Exception as ex:
    print("ERR", ex)
