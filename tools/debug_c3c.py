import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2410_21207_b200 as cv, oracle
P = oracle.port()
img = cv.make_test_image(3840, 2160)
mid = cv.carve(img, 3072, 1917)          # works
t = np.ascontiguousarray(mid.transpose(1, 0, 2))   # the transposed phase's image: width 1917, height 3072
e = P.energy_e1_rgb(t)
print("e range", e.min(), e.max(), np.isfinite(e).all(), flush=True)
s_ref, m_ref, b_ref = P.dp_seam(e)
print("ref seam ends", s_ref[:3], s_ref[-3:], "min", s_ref.min(), "max", s_ref.max(), flush=True)
try:
    seam = cv.find_seam(e, cv.SolverKind.Dynamic)
    print("gpu find_seam eq", np.array_equal(seam, s_ref), flush=True)
except Exception as ex:
    print("find_seam ERR", ex, flush=True); sys.exit(0)
r = cv.dp_seam(e)
print("tables eq", np.array_equal(r.table.m, m_ref), np.array_equal(r.table.b, b_ref))
