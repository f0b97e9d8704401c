import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2410_21207_b200 as cv
print(cv.library_path())
z = np.load("tests/golden/corpus.npz")
bad = 0
for k in range(int(z["n"])):
    e = z[f"e{k}"].astype(np.float64)
    try:
        r = cv.dp_seam(e)
    except Exception as ex:
        print(k, e.shape, "ERR", ex); break
    if not (np.array_equal(r.seam, z[f"s{k}"]) and np.array_equal(r.table.b, z[f"b{k}"].astype(np.int32)) and np.array_equal(r.table.m, z[f"m{k}"].astype(np.float64))):
        bad += 1
        if bad < 5: print(k, e.shape, "MISMATCH seam", np.array_equal(r.seam, z[f"s{k}"]), "b", np.array_equal(r.table.b, z[f"b{k}"].astype(np.int32)), "m", np.array_equal(r.table.m, z[f"m{k}"].astype(np.float64)))
print("bad", bad)
