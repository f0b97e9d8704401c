"""Profiling driver (tools only): one C2-sized device-resident carve after a warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_21207_b200 as cv
W, H, TW, TH = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (1920, 1080, 1728, 1080)
img = torch.from_numpy(cv.make_test_image(W, H)).cuda()
out = torch.empty((TH, TW, 3), dtype=torch.uint8, device="cuda")
for _ in range(2):
    cv.carve_device(img.data_ptr(), W, H, TW, TH, out.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
