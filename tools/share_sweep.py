"""GPU sweep (not a bench): C5 throughput of one GPU's share of the 1024-image
batch at world sizes 1/2/4/8 (1024/G images), device-resident and end to end
through carve_batch from pinned host buffers. Environment overrides (e.g.
CARVE_DP_VARIANT, CARVE_PIPE_CHUNK) pass through to the library.

    python tools/share_sweep.py [n ...]          # default 1024 512 256 128
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_21207_b200 as cv  # noqa: E402

W, H, TW = 1024, 768, 896


def main():
    grid = "--grid" in sys.argv
    ns = [int(x) for x in sys.argv[1:] if not x.startswith("--")] or [1024, 512, 256, 128]
    nmax = max(ns)
    pin_in = torch.empty((nmax, H, W, 3), dtype=torch.uint8, pin_memory=True)
    for k in range(nmax):
        pin_in[k].numpy()[...] = cv.make_test_image(W, H, k)
    pin_out = torch.empty((nmax, H, TW, 3), dtype=torch.uint8, pin_memory=True)
    d_in = pin_in.cuda()
    d_out = torch.empty((nmax, H, TW, 3), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    combos = [{}]
    if grid:  # host pipelines x chunk sizes, device split counts (env read per call)
        combos = [{"CARVE_PIPELINES": str(p), "CARVE_PIPE_CHUNK": str(c), "CARVE_DEVICE_SPLIT": str(p),
                   "CARVE_DEVICE_SPLIT_MIN": "16"} for p in (1, 2, 3, 4) for c in (32, 64, 128, 256)]
    for n in ns:
      for env in combos:
        if env.get("CARVE_PIPE_CHUNK") and int(env["CARVE_PIPE_CHUNK"]) > n:
            continue
        for k in ("CARVE_PIPELINES", "CARVE_PIPE_CHUNK", "CARVE_DEVICE_SPLIT", "CARVE_DEVICE_SPLIT_MIN"):
            os.environ.pop(k, None)
        os.environ.update(env)
        def dev():
            cv.carve_batch_device(d_in.data_ptr(), n, W, H, TW, H, d_out.data_ptr(), s.cuda_stream)
        for _ in range(2):
            dev()
        torch.cuda.synchronize()
        reps = 3
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            dev()
        b.record(s)
        torch.cuda.synchronize()
        dev_ips = n * reps / (a.elapsed_time(b) / 1e3)
        ins = [pin_in[k].numpy() for k in range(n)]
        outs = [pin_out[k].numpy() for k in range(n)]
        cv.carve_batch(ins, TW, H, devices=[0], out=outs)
        t = time.perf_counter()
        for _ in range(reps):
            cv.carve_batch(ins, TW, H, devices=[0], out=outs)
        e2e_ips = n * reps / (time.perf_counter() - t)
        print(json.dumps({"n": n, "dev_img_s": round(dev_ips, 1), "e2e_img_s": round(e2e_ips, 1),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("CARVE_")}}), flush=True)


if __name__ == "__main__":
    main()
