import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2410_21207_b200 as cv
img = cv.make_test_image(1920, 1080)
pin = torch.from_numpy(img).pin_memory().numpy()
for k in range(8):
    t = time.perf_counter(); out = cv.carve(pin, 1728, 1080); print(k, round((time.perf_counter() - t) * 1e3, 2), 'ms')
outp = torch.empty((1080, 1728, 3), dtype=torch.uint8).pin_memory().numpy()
for k in range(4):
    t = time.perf_counter(); outp[...] = cv.carve(pin, 1728, 1080); print('copy', k, round((time.perf_counter() - t) * 1e3, 2), 'ms')
