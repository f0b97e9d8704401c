"""Per-warp phase breakdown of one DP launch (clock64 counters, MODE 2 kernel)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2410_21207_b200 as cv, oracle
W, H = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1920, 1080)
e = oracle.port().energy_e1_rgb(oracle.port().make_test_image(W, H))
lib = cv.library()
f = lib.carve_cuda_dp_profile
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
buf = np.zeros(8 * 512, np.int64); nw = C.c_int()
for rep in range(2):
    st = f(e.ctypes.data, W, H, buf.ctypes.data, buf.size, C.addressof(nw))
    assert st == 0, lib.carve_cuda_last_error()
G = nw.value; a = buf[: 8 * G].reshape(G, 8)
print(f"variant={os.environ.get('CARVE_DP_VARIANT')} W={W} H={H} warps={G}")
print(" fwd cycles/row   mean %.1f  min %.1f  max %.1f" % ((a[:, 0] / H).mean(), (a[:, 0] / H).min(), (a[:, 0] / H).max()))
print(" wait cycles/row  mean %.1f  min %.1f  max %.1f" % ((a[:, 1] / H).mean(), (a[:, 1] / H).min(), (a[:, 1] / H).max()))
print(" argmin+p1 cycles mean %.0f, phase2 cycles mean %.0f max %.0f" % (a[:, 2].mean(), a[:, 3].mean(), a[:, 3].max()))
w = a[:, 5] > 0
if w.any():
    print(" phase2 first block: start->data %.0f, rows %.0f, walk %.0f cycles (mean over %d warps)" %
          (a[w, 5].mean(), a[w, 6].mean(), a[w, 7].mean(), int(w.sum())))
