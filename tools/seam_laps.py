"""Per-seam device laps of one carve (tools only): python tools/seam_laps.py W H TW TH
(energy / solve / remove from the %globaltimer stamps, carve_cuda_seam_timing)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_21207_b200 as cv  # noqa: E402

W, H, TW, TH = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (1920, 1080, 1728, 1080)
img = cv.make_test_image(W, H)
for _ in range(3):
    out, seams, tim = cv.carve(img, TW, TH, seams=True, timings=True)
e = np.array([t.energy_s for t in tim]) * 1e6
s = np.array([t.solve_s for t in tim]) * 1e6
r = np.array([t.remove_s for t in tim]) * 1e6
print(f"{W}x{H}->{TW}x{TH}: {len(tim)} seams; energy mean {e.mean():.2f} us, solve mean {s.mean():.2f} "
      f"(min {s.min():.2f} max {s.max():.2f}), remove mean {r.mean():.2f} (min {r.min():.2f} max {r.max():.2f})")
