#!/usr/bin/env python
"""Benchmark of the B200 seam-carving engine (BASELINE.json metric:
"seams removed/sec (1080p, 4K) and images/sec batched at 1/2/4/8 B200 vs CPU").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5] [--impl ours|reference]

A step is one carve of the configuration's synthetic input(s) (make_test_image,
bench.hpp:67-94). Default config C2: 1920x1080 -> 1728x1080 (192 vertical
seams) per GPU; under torchrun each rank carves its own image (weak scaling,
no collective on the data path) and `value` is the total
seams/s over all ranks, timed as the max over ranks. C5 (--config c5) shards a
batch of 1024 1024x768 images by image across ranks (strong scaling, images/s).

`value`: inputs resident in HBM, one carve enqueued through the device entry
point, CUDA events on the launching stream, L2 flushed between steps.
`e2e`: the public host API (paper_2410_21207_b200.carve / carve_batch) from
pinned host buffers, host<->device copies inside the timed region.
`--impl reference`: the reference's CPU implementation (oracle/_ref, the
reference compiled unmodified) on this host, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (W, H, target_w, target_h, images, description)
    "c1": (512, 512, 448, 512, 1, "C1 512x512 -> 448x512 (64 vertical seams)"),
    "c2": (1920, 1080, 1728, 1080, 1, "C2 1920x1080 -> 1728x1080 (192 vertical seams)"),
    "c3": (3840, 2160, 3072, 1728, 1, "C3 3840x2160 -> 3072x1728 (768 vertical + 432 transposed horizontal seams)"),
    "c4": (7680, 4320, 7168, 4320, 1, "C4 7680x4320 -> 7168x4320 (512 vertical seams)"),
    "c5": (1024, 768, 896, 768, 1024, "C5 batch of 1024 1024x768 -> 896x768 (128 seams each)"),
}

HBM_FALLBACK_GBS = 6650.0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous per-rank share of n independent images (no data exchange)."""
    return n * rank // world, n * (rank + 1) // world


class Clocks:
    """nvidia-smi clock/throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"carve_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
            sm = [float(r[0]) for r in rows]
            mx = max(float(r[1]) for r in rows)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].strip() == "Active"})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}
        except Exception as e:  # no nvidia-smi
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)[:80]}


# ------------------------------------------------------------------------------------
def run_reference(args, cfg_name):
    """--impl reference: the reference CPU path (oracle/_ref) on this host, rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    W, H, TW, TH, N, desc = CONFIGS[cfg_name]
    ref = oracle.reference() if oracle.have_reference() else None
    kind = "reference" if ref else "port"
    nproc = os.cpu_count() or 1
    seams_per_img = (W - TW) + (H - TH)
    if cfg_name == "c5":
        sample = max(nproc, 16)  # images per step (bounded sample of the batch)
        imgs = [oracle.port().make_test_image(W, H, k) for k in range(sample)]

        def step():
            if ref:
                ref.carve_batch(imgs, TW, nproc)
            else:
                for x in imgs:
                    oracle.port().carve(x, TW)
        unit_per_step, unit = sample, "images/s"
        used_cores = nproc
        sample_desc = f"{sample} of the 1024 images per step, {nproc} threads x reference dp carve_to_width"
        solver_desc = "dp x nproc threads (one image per thread)"
    else:
        img = oracle.port().make_test_image(W, H)
        # bounded sample: seams per step chosen so one step is a few seconds
        budget = {"c1": seams_per_img, "c2": seams_per_img, "c3": 24, "c4": 8}[cfg_name]
        tw = max(TW, W - budget) if budget <= W - TW else TW
        th = H if budget <= W - TW else TH

        def run(solver, workers):
            t = time.perf_counter()
            if ref:
                ref.carve(img, tw, th, solver=solver, workers=workers)
            else:
                oracle.port().carve(img, tw, th)
            return time.perf_counter() - t
        t_dp = run(0, 1)
        t_par = run(1, nproc) if ref else float("inf")
        solver, workers = (0, 1) if t_dp <= t_par else (1, nproc)
        used_cores = workers
        solver_desc = f"{'dp' if solver == 0 else f'pardp({nproc} workers)'} (faster of dp {t_dp:.2f}s / pardp {t_par:.2f}s)"

        def step():
            run(solver, workers)
        unit_per_step, unit = (W - tw) + (H - th), "seams/s"
        sample_desc = f"{unit_per_step} seams of {desc} per step"
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = unit_per_step * args.steps / total
    line = {
        "impl": "reference", "metric": "images removed-seam batches/sec" if cfg_name == "c5" else "seams removed/sec",
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "none (CPU)",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_test_image, bench.hpp:67-94)",
        "config": {"workload": desc, "solver": solver_desc},
        "cpu_baseline": {"value": value, "unit": unit, "cores": used_cores, "kind": kind, "sample": sample_desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if cfg_name == "c5":
        line["metric"] = "images/sec"
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg_name):
    """Rank 0, N=1 only: the reference CPU path on a bounded sample (~10-30 s)."""
    import oracle

    W, H, TW, TH, N, desc = CONFIGS[cfg_name]
    nproc = os.cpu_count() or 1
    ref = oracle.reference() if oracle.have_reference() else None
    kind = "reference" if ref else "port"
    if cfg_name == "c5":
        imgs = [oracle.port().make_test_image(W, H, k) for k in range(nproc)]
        t = time.perf_counter()
        if ref:
            ref.carve_batch(imgs, TW, nproc)
        else:
            for x in imgs:
                oracle.port().carve(x, TW)
        dt = time.perf_counter() - t
        return {"value": len(imgs) / dt, "unit": "images/s", "cores": nproc if ref else 1, "kind": kind,
                "sample": f"{len(imgs)} images, one reference dp carve_to_width per host thread"}
    img = oracle.port().make_test_image(W, H)
    n = {"c1": W - TW, "c2": W - TW, "c3": 16, "c4": 6}[cfg_name]
    res = {}
    for solver, workers in ((0, 1), (1, nproc)):
        if not ref and solver == 1:
            continue
        t = time.perf_counter()
        if ref:
            ref.carve(img, W - n, H, solver=solver, workers=workers)
        else:
            oracle.port().carve(img, W - n)
        res[(solver, workers)] = n / (time.perf_counter() - t)
    best = max(res, key=res.get)
    names = {(0, 1): "dp 1 thread", (1, nproc): f"pardp {nproc} workers"}
    return {"value": res[best], "unit": "seams/s", "cores": best[1], "kind": kind,
            "sample": f"{n} vertical seams of {desc}; faster of " +
                      ", ".join(f"{names[k]} {v:.2f} seams/s" for k, v in res.items())}


# ------------------------------------------------------------------------------------
class Ranks:
    """torchrun plumbing: one process per GPU, NCCL only for the barrier and the
    max-over-ranks timing reduce (the data path has no collective)."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=f"cuda:{self.local}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def measure(cfg_name, args, rk, distinct_max=None):
    """One configuration: device-resident timed region (CUDA events, L2 flushed),
    per-kernel attribution pass, e2e through the public host API."""
    import torch

    import oracle  # checker only (golden hash of the benchmarked output)
    import paper_2410_21207_b200 as cv

    rank, world, local = rk.rank, rk.world, rk.local
    W, H, TW, TH, N, desc = CONFIGS[cfg_name]
    batch = N > 1
    lo, hi = shard(N, world, rank) if batch else (0, 1)
    n_local = hi - lo
    seams_per_img = (W - TW) + (H - TH)
    n_distinct = min(n_local, distinct_max or n_local)

    # synthetic inputs (host, outside timing), pinned host buffers for e2e
    pin_in = torch.empty((n_local, H, W, 3), dtype=torch.uint8, pin_memory=True)
    for k in range(n_local):
        if k < n_distinct:
            pin_in[k].numpy()[...] = cv.make_test_image(W, H, (lo + k) if batch else rank)
        else:
            pin_in[k].copy_(pin_in[k % n_distinct])
    pin_out = torch.empty((n_local, TH, TW, 3), dtype=torch.uint8, pin_memory=True)
    d_in = pin_in.to(f"cuda:{local}")
    d_out = torch.empty((n_local, TH, TW, 3), dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def enqueue():
        if batch:
            cv.carve_batch_device(d_in.data_ptr(), n_local, W, H, TW, TH, d_out.data_ptr(), sptr)
        else:
            cv.carve_device(d_in.data_ptr(), W, H, TW, TH, d_out.data_ptr(), None, sptr)

    for _ in range(args.warmup):
        enqueue()
    torch.cuda.synchronize()

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"]
    out0 = d_out[0].cpu().numpy()
    gkey, verified = cfg_name.upper(), None
    if not batch and "output" in gold.get(gkey, {}) and rank == 0:
        verified = f"{oracle.fnv1a64(out0):016x}" == gold[gkey]["output"]
    elif batch and str(lo) in gold.get("C5", {}).get("samples", {}):
        verified = f"{oracle.fnv1a64(out0):016x}" == gold["C5"]["samples"][str(lo)]["output"]

    # ---- device-resident timed region -------------------------------------------------
    cv.reset_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        rk.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()  # evict L2 between steps (outside the events)
            evs[k][0].record(stream)
            enqueue()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        rk.barrier()
    launches = cv.launch_count()
    dev_ms = rk.max(sum(a.elapsed_time(b) for a, b in evs))
    units_total = N if batch else seams_per_img * world
    value = units_total * args.steps / (dev_ms / 1e3)

    # ---- kernel attribution pass (same workload, per-kernel CUDA events) ------------
    kern = kernel_profile(cv, enqueue, stream, W, H, TW, TH, n_local)

    # ---- end-to-end through the public host API (pinned host buffers) ---------------
    in_views = [pin_in[k].numpy() for k in range(n_local)]
    out_views = [pin_out[k].numpy() for k in range(n_local)]

    def api_step():
        if batch:
            cv.carve_batch(in_views, TW, TH, devices=[local], out=out_views)
        else:
            cv.carve(in_views[0], TW, TH, out=out_views[0])

    for _ in range(args.warmup):  # same W untimed warm-up steps as the device-resident region
        api_step()
    rk.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        api_step()
    e2e_s = rk.max(time.perf_counter() - t0)
    unit = "images/s" if batch else "seams/s"
    e2e = {"value": units_total * args.steps / e2e_s, "unit": unit,
           "h2d_bytes_per_step": W * H * 3 * n_local, "d2h_bytes_per_step": TW * TH * 3 * n_local,
           "api": "paper_2410_21207_b200.carve_batch" if batch else "paper_2410_21207_b200.carve"}
    del d_in, d_out, flush
    torch.cuda.empty_cache()
    return {"value": value, "unit": unit, "ms_per_step": dev_ms / args.steps, "e2e": e2e, "kernels": kern,
            "gpu_launches": launches, "verified_vs_golden": verified, "clocks": clk.summary(), "batch": batch,
            "desc": desc, "n_local": n_local, "n_distinct": n_distinct}


def measured_traffic(kernel, cfg_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu
    --set full capture (profiles/r01_traffic.json), for the workload it was taken on."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r01_traffic.json")))
        return t["bytes_per_launch"].get(cfg_name, {}).get(kernel)
    except Exception:
        return None


# DP rows per launch (the DP is a row-serial chain: its real bound is latency per row)
DP_ROWS = {"c1": 512, "c2": 1080, "c3": (768 * 2160 + 432 * 3072) / 1200, "c4": 4320, "c5": 768}
# one warp's dependent row step (2 shuffles + 2 compare/selects + DADD), measured on B200 by
# tools/microbench.cu (profiles/r01_microbench_latency.txt)
CHAIN_CYCLES_PER_ROW = 59.0


def roofline_of(kern, cfg_name="c2", sm_mhz=None):
    peak, peak_src = peaks()
    dom = max(kern, key=lambda k: kern[k]["ms_total"]) if kern else None
    if not dom:
        return None
    kd = kern[dom]
    r = {"kernel": dom, "bound": "hbm", "achieved": kd["gbs"], "peak": peak, "unit": "GB/s",
         "frac": kd["gbs"] / peak, "traffic": measured_traffic(dom, cfg_name), "peak_source": peak_src,
         "bytes_per_launch": kd["bytes_per_launch"], "avg_launch_us": kd["avg_us"], "share_of_step": kd["share"],
         # HBM fraction of every timed kernel (algorithmic bytes / event time / peak). The removal's
         # algorithmic bytes follow SURVEY.md §8d (a full-row copy: read W, write W-1); the in-place
         # kernels move only the part right of the seam, so that fraction can exceed 1 — the
         # DRAM-measured fraction (ncu bytes per launch / event time) is in dram_frac_by_kernel
         "hbm_frac_by_kernel": {k: round(v["gbs"] / peak, 4) for k, v in kern.items()},
         "dram_frac_by_kernel": {k: round(measured_traffic(k, cfg_name) / (v["avg_us"] * 1e3) / peak, 4)
                                 for k, v in kern.items() if measured_traffic(k, cfg_name)}}
    if dom == "k_dp_seam" and cfg_name in DP_ROWS and cfg_name != "c5":
        ns_row = kd["avg_us"] * 1e3 / DP_ROWS[cfg_name]
        floor = CHAIN_CYCLES_PER_ROW / ((sm_mhz or 1965.0) / 1e3)
        r["latency"] = {"note": "the DP is latency-bound (row-serial chain), not HBM-bound",
                        "ns_per_row": ns_row, "chain_floor_ns_per_row": floor, "frac_of_chain_floor": floor / ns_row}
        try:  # shared-memory fraction and barrier stalls of the committed C2 ncu capture
            nm = json.load(open(os.path.join(ROOT, "profiles", "r01_dp_ncu_metrics.json")))
            if cfg_name == "c2":
                r["latency"].update(smem_frac_active_sms=nm["smem_wavefronts_frac_of_peak_active_sms"],
                                    barrier_stall_share=nm["barrier_stall_share"],
                                    halo_wait_stall_share=nm["stall_share"].get("long_scoreboard"),
                                    ncu_source="profiles/r01_dp_ncu_metrics.json")
        except Exception:
            pass
    return r


def run_ours(args, cfg_name):
    import torch

    import paper_2410_21207_b200 as cv

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device")
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    cv.set_device(local)
    rk = Ranks()
    m = measure(cfg_name, args, rk)
    batch = m["batch"]
    line = {
        "metric": "images/sec" if batch else "seams removed/sec",
        "value": m["value"], "unit": m["unit"], "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong" if batch else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_test_image, bench.hpp:67-94)",
        "config": {"workload": m["desc"] + ("" if batch else " per GPU"), "images_per_gpu": m["n_local"],
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"image-sharded x{world}, no collective"},
        "e2e": m["e2e"], "gpu_launches": m["gpu_launches"], "roofline": roofline_of(m["kernels"], cfg_name, (m["clocks"] or {}).get("sm_mhz")),
        "kernels": m["kernels"], "verified_vs_golden": m["verified_vs_golden"], "clocks": m["clocks"],
    }
    if not batch and not args.no_batch:
        # the metric's second half: images/s batched, 1024 x (1024x768 -> 896x768), sharded by image
        b = measure("c5", argparse.Namespace(steps=max(2, min(args.steps, 3)), warmup=3), rk, distinct_max=128)
        line["batch"] = {"metric": "images/sec", "value": b["value"], "unit": b["unit"], "workload": b["desc"],
                         "ms_per_step": b["ms_per_step"], "scaling": "strong", "e2e": b["e2e"],
                         "images_per_gpu": b["n_local"],
                         "data": f"{b['n_distinct']} distinct make_test_image variants per GPU, tiled to "
                                 f"{b['n_local']} images", "verified_vs_golden": b["verified_vs_golden"],
                         "roofline": roofline_of(b["kernels"], "c5", (b["clocks"] or {}).get("sm_mhz")), "kernels": b["kernels"],
                         "gpu_launches": b["gpu_launches"], "clocks": b["clocks"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg_name)
        if "batch" in line:
            line["batch"]["cpu_baseline"] = cpu_baseline("c5")
    if rank == 0:
        print(json.dumps(line), flush=True)
    rk.close()


def kernel_profile(cv, enqueue, stream, W, H, TW, TH, n_local):
    """One extra carve with per-kernel CUDA events (library profiling mode):
    average launch duration, share of the step and algorithmic GB/s per kernel
    (algorithmic bytes per SURVEY.md §8d)."""
    try:
        cv.set_kernel_events(True)
    except AttributeError:
        return {}
    try:
        enqueue()
        import torch
        torch.cuda.synchronize()
        stats = cv.kernel_event_stats()
    finally:
        cv.set_kernel_events(False)
    total = sum(s["ms_total"] for s in stats.values()) or 1.0
    for k, s in stats.items():
        s["share"] = s["ms_total"] / total
        s["avg_us"] = 1e3 * s["ms_total"] / max(1, s["launches"])
        s["bytes_per_launch"] = s["bytes_total"] / max(1, s["launches"])
        s["gbs"] = s["bytes_total"] / (s["ms_total"] * 1e-3) / 1e9 if s["ms_total"] else 0.0
    return stats


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="skip the C5 batch object in the default line")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, args.config)
    else:
        run_ours(args, args.config)


if __name__ == "__main__":
    main()
