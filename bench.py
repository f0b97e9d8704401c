#!/usr/bin/env python
"""Benchmark of the B200 seam-carving engine (BASELINE.json metric:
"seams removed/sec (1080p, 4K) and images/sec batched at 1/2/4/8 B200 vs CPU").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference] [--emulate-world G]

A step is one carve of the configuration's synthetic input(s) (make_test_image,
bench.hpp:67-94). The default line is C2 (1920x1080 -> 1728x1080, 192 vertical
seams) per GPU; under torchrun each rank carves its own image (weak scaling, no
collective on the data path) and `value` is the total seams/s
over all ranks, timed as the max over ranks. The default line also carries the
metric's other halves as objects: `c3` (4K: 3840x2160 -> 3072x1728, 768
vertical + 432 transposed horizontal seams), `batch` (C5: 1024 distinct
1024x768 images -> 896x768, sharded by image over the ranks) and
`batch.shares` — the per-rank share of the 1024-image batch at 2/4/8 GPUs
(512/256/128 images) timed on this one GPU, device-resident and end to end,
with the projected efficiency of an image-sharded G-GPU run (no data crosses
GPUs, so a rank's time is its share's time).

`value`: inputs resident in HBM, one carve enqueued through the device entry
point, CUDA events on the launching stream, L2 flushed (256 MiB write) between
steps. `e2e`: the public host API (paper_2410_21207_b200.carve / carve_batch)
from pinned host buffers, host<->device copies inside the timed region.
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
from concurrent.futures import ThreadPoolExecutor

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
SHARES = (2, 4, 8)  # world sizes whose per-rank C5 share is timed on one GPU

HBM_FALLBACK_GBS = 6650.0
L2_NOTE = "GPU arm: L2 flushed (256 MiB write) between timed steps; CPU arm: n/a"


def config_of(cfg_name: str) -> dict:
    """The `config` dict both arms print (byte-identical for the same workload)."""
    W, H, TW, TH, N, desc = CONFIGS[cfg_name]
    unit = "images sharded by image over the ranks" if N > 1 else "one image per rank"
    return {"workload": f"{desc}; {unit}", "l2": L2_NOTE}


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


def make_images(cv, W, H, variants, out=None):
    """make_test_image variants (host, outside timing), generated on host threads."""
    arrs = out if out is not None else [np.empty((H, W, 3), np.uint8) for _ in variants]

    def gen(k):
        arrs[k][...] = cv.make_test_image(W, H, variants[k])
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(gen, range(len(variants))))
    return arrs


class Clocks:
    """nvidia-smi clock/throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"carve_clocks_{os.getpid()}_{index}.csv")

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
        "impl": "reference", "metric": "images/sec" if cfg_name == "c5" else "seams removed/sec",
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "none (CPU)",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_test_image, bench.hpp:67-94)",
        "config": config_of(cfg_name), "setup": {"solver": solver_desc, "host_threads": used_cores},
        "cpu_baseline": {"value": value, "unit": unit, "cores": used_cores, "kind": kind, "sample": sample_desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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


class Inputs:
    """One configuration's synthetic inputs: pinned host copies (e2e) and device
    copies (device-resident timing) of this rank's images, plus outputs."""

    def __init__(self, cv, cfg_name, rank, world, local):
        import torch

        W, H, TW, TH, N, desc = CONFIGS[cfg_name]
        self.batch = N > 1
        self.lo, self.hi = shard(N, world, rank) if self.batch else (0, 1)
        n = self.hi - self.lo
        self.pin_in = torch.empty((n, H, W, 3), dtype=torch.uint8, pin_memory=True)
        views = [self.pin_in[k].numpy() for k in range(n)]
        # every image distinct: batch image k is make_test_image variant k (the
        # golden C5 samples use the same rule); single images: variant = rank
        make_images(cv, W, H, [self.lo + k for k in range(n)] if self.batch else [rank], views)
        self.pin_out = torch.empty((n, TH, TW, 3), dtype=torch.uint8, pin_memory=True)
        self.d_in = self.pin_in.to(f"cuda:{local}")
        self.d_out = torch.empty((n, TH, TW, 3), dtype=torch.uint8, device=f"cuda:{local}")
        self.in_views = views
        self.out_views = [self.pin_out[k].numpy() for k in range(n)]
        self.n = n


def measure(cfg_name, args, rk, inputs=None, n_share=None, profile=True):
    """One configuration: device-resident timed region (CUDA events, L2 flushed),
    per-kernel attribution pass, e2e through the public host API. `n_share`
    (batches): time only the first n_share images of this rank's inputs."""
    import torch

    import oracle  # checker only (golden hash of the benchmarked output)
    import paper_2410_21207_b200 as cv

    rank, world, local = rk.rank, rk.world, rk.local
    W, H, TW, TH, N, desc = CONFIGS[cfg_name]
    inp = inputs or Inputs(cv, cfg_name, rank, world, local)
    batch = inp.batch
    n_local = n_share or inp.n
    seams_per_img = (W - TW) + (H - TH)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    d_seams = None if batch else torch.empty(max(1, (W - TW) * H + (H - TH) * TW), dtype=torch.int32,
                                             device=f"cuda:{local}")

    def enqueue(seams=False):
        if batch:
            cv.carve_batch_device(inp.d_in.data_ptr(), n_local, W, H, TW, TH, inp.d_out.data_ptr(), sptr)
        else:
            cv.carve_device(inp.d_in.data_ptr(), W, H, TW, TH, inp.d_out.data_ptr(),
                            d_seams.data_ptr() if seams else None, sptr)

    for _ in range(args.warmup):
        enqueue()
    torch.cuda.synchronize()

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"]
    verified = None
    if not batch and "output" in gold.get(cfg_name.upper(), {}) and rank == 0:
        verified = f"{oracle.fnv1a64(inp.d_out[0].cpu().numpy()):016x}" == gold[cfg_name.upper()]["output"]
    elif batch:
        samples = {int(k) - inp.lo: v["output"] for k, v in gold.get("C5", {}).get("samples", {}).items()
                   if 0 <= int(k) - inp.lo < n_local}
        if samples:
            verified = all(f"{oracle.fnv1a64(inp.d_out[k].cpu().numpy()):016x}" == h for k, h in samples.items())

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
    units_total = (n_local * world) if batch else seams_per_img * world
    value = units_total * args.steps / (dev_ms / 1e3)

    # ---- kernel attribution pass (same workload, per-kernel CUDA events) ------------
    kern = {}
    if profile:
        kern = kernel_profile(cv, lambda: enqueue(seams=True), W, H, TW, TH, n_local, flush)
        if not batch:
            moved = inplace_removal_bytes(d_seams.cpu().numpy(), W, H, TW, TH)
            k = kern.get("k_compact")
            if k:
                # the in-place removal moves only the part of a row right of the seam:
                # bytes it must read + write (RGBX 4 B + FP64 energy 8 B per element),
                # plus the library's count for each phase's last (transposing) launch
                k["moved_bytes_per_launch"] = moved["bytes"] / k["launches"]
                k["moved_gbs"] = moved["bytes"] / (k["ms_total"] * 1e-3) / 1e9

    # ---- end-to-end through the public host API (pinned host buffers) ---------------
    ins, outs = inp.in_views[:n_local], inp.out_views[:n_local]

    def api_step():
        if batch:
            cv.carve_batch(ins, TW, TH, devices=[local], out=outs)
        else:
            cv.carve(ins[0], TW, TH, out=outs[0])

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
    del flush
    return {"value": value, "unit": unit, "ms_per_step": dev_ms / args.steps, "e2e": e2e, "kernels": kern,
            "gpu_launches": launches, "verified_vs_golden": verified, "clocks": clk.summary(), "batch": batch,
            "desc": desc, "n_local": n_local}


def inplace_removal_bytes(seams, W, H, TW, TH):
    """Bytes the in-place removal (k_compact_bulk, single images) must move for the
    recorded seams: per row, the aligned part right of the seam is read (TMA, from
    floor4(s) rounded to 4 elements) and written back shifted (Wn - floor4(s)),
    RGBX 4 B + FP64 energy 8 B per element. Each phase's last removal is the
    transposing kernel: 4 B read + 3 B written per pixel (library count)."""
    total, off = 0.0, 0
    for (w0, h, k) in ((W, H, W - TW), (H, TW, H - TH)):
        for t in range(k):
            s = seams[off:off + h].astype(np.int64)
            off += h
            w = w0 - t
            if t + 1 == k:
                total += 3.0 * h * (2.0 * w - 1)
                continue
            a = s & ~3
            total += 12.0 * float((((w - a + 3) & ~3) + (w - 1 - a)).sum())
    return {"bytes": total}


def kernel_profile(cv, enqueue, W, H, TW, TH, n_local, flush=None):
    """One extra carve with per-kernel CUDA events (library profiling mode):
    average launch duration, share of the step and algorithmic GB/s per kernel
    (algorithmic bytes per SURVEY.md §8d). Like a timed step it starts
    from a flushed L2 (the flush buffer is then read back, so its dirty lines are written
    out before the carve instead of during its first kernels), and the GPU is held in a
    sleep kernel while the host enqueues the carve, so no event pair measures host
    submission latency (the first launches of an idle GPU otherwise do)."""
    import torch

    if flush is not None:
        flush.zero_()
        flush.sum(dtype=torch.int64)
    cv.set_kernel_events(True)
    try:
        torch.cuda._sleep(50_000_000)  # ~25 ms at 2 GHz: covers the enqueue of every launch
        enqueue()
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


def measured_traffic(kernel, cfg_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu
    --set full captures (profiles/r02_traffic.json, else r01), for the workload
    they were taken on."""
    for f in ("r02_traffic.json", "r01_traffic.json"):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", f)))
            v = t["bytes_per_launch"].get(cfg_name, {}).get(kernel)
            if v:
                return v
        except Exception:
            pass
    return None


def measured_inst(kernel, cfg_name):
    """Warp instructions per launch (ncu smsp__inst_executed.sum) from the committed capture
    (profiles/r02_traffic.json `inst_per_launch`), for the workload it was taken on."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
        return t.get("inst_per_launch", {}).get(cfg_name, {}).get(kernel)
    except Exception:
        return None


# DP rows per launch (the DP is a row-serial chain: its real bound is latency per row)
DP_ROWS = {"c1": 512, "c2": 1080, "c3": (768 * 2160 + 432 * 3072) / 1200, "c4": 4320, "c5": 768}
# one warp's dependent row step (2 shuffles + 2 compare/selects + DADD), measured on B200 by
# tools/microbench.cu (profiles/r01_microbench_latency.txt)
CHAIN_CYCLES_PER_ROW = 59.0


def roofline_of(kern, cfg_name="c2", sm_mhz=None):
    """The dominant kernel's bound. Single images: the DP (K2+K3) is a row-serial
    latency chain, reported as ns per row against the measured chain floor; the
    HBM-bound kernels (K1 energy, K4 removal) are reported against the measured
    HBM peak in `hbm_kernels` — algorithmic bytes / event time, and ncu DRAM
    bytes / event time where a capture exists (profiles/r0*_traffic.json)."""
    peak, peak_src = peaks()
    dom = max(kern, key=lambda k: kern[k]["ms_total"]) if kern else None
    if not dom:
        return None
    kd = kern[dom]
    hbm = {}
    for k, v in kern.items():
        e = {"algorithmic_gbs": round(v["gbs"], 1), "frac": round(v["gbs"] / peak, 4),
             "avg_launch_us": round(v["avg_us"], 3), "bytes_per_launch": v["bytes_per_launch"]}
        if "moved_gbs" in v:
            e["moved_gbs"] = round(v["moved_gbs"], 1)
            e["moved_frac"] = round(v["moved_gbs"] / peak, 4)
        t = measured_traffic(k, cfg_name)
        if t:
            e["dram_bytes_per_launch"] = t
            e["dram_frac"] = round(t / (v["avg_us"] * 1e3) / peak, 4)
        hbm[k] = e
    r = {"kernel": dom, "traffic": measured_traffic(dom, cfg_name), "bytes_per_launch": kd["bytes_per_launch"],
         "avg_launch_us": kd["avg_us"], "share_of_step": kd["share"], "peak_source": peak_src,
         "hbm_kernels": hbm}
    if dom == "k_dp_seam" and cfg_name != "c5":
        ns_row = kd["avg_us"] * 1e3 / DP_ROWS[cfg_name]
        floor = CHAIN_CYCLES_PER_ROW / ((sm_mhz or 1965.0) / 1e3)
        r.update(bound="latency", achieved=ns_row, peak=floor, unit="ns/row (lower is better)",
                 frac=floor / ns_row, frac_of_chain_floor=floor / ns_row,
                 note="row-serial DP chain; peak = measured 59-cycle chain floor at the sampled SM clock; "
                      "its HBM view: " + f"{kd['gbs']:.0f} GB/s = {kd['gbs'] / peak:.3f} of {peak:.0f} GB/s")
        for f in ("r02_dp_ncu_metrics.json", "r01_dp_ncu_metrics.json"):
            try:  # shared-memory fraction and barrier stalls of the committed C2 ncu capture
                nm = json.load(open(os.path.join(ROOT, "profiles", f)))
            except Exception:
                continue
            if cfg_name == "c2":
                r.update(smem_frac_active_sms=nm["smem_wavefronts_frac_of_peak_active_sms"],
                         barrier_stall_share=nm["barrier_stall_share"],
                         halo_wait_stall_share=nm["stall_share"].get("long_scoreboard"),
                         ncu_source="profiles/" + f)
            break
    elif dom == "k_dp_seam" and measured_inst(dom, cfg_name):
        # the batch DP is issue-bound (ncu: FP64 and XU pipes below half busy, issue slots
        # ~70 % busy): instruction issue rate against one warp-instruction per scheduler per
        # cycle, 4 schedulers per SM, at the sampled SM clock
        inst = measured_inst(dom, cfg_name)
        try:
            import torch
            nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        except Exception:
            nsm = 148
        achieved = inst / (kd["avg_us"] * 1e-6) / 1e9
        ipeak = nsm * 4 * (sm_mhz or 1965.0) / 1e3
        r.update(bound="issue", achieved=achieved, peak=ipeak, unit="G warp-instructions/s", frac=achieved / ipeak,
                 inst_per_launch=inst, hbm_frac=kd["gbs"] / peak,
                 note=f"issue-bound fused DP: {inst:.4g} warp instructions per launch (ncu, profiles/r02_traffic.json) "
                      f"over the live launch time; peak = {nsm} SMs x 4 schedulers x SM clock; its HBM view: "
                      f"{kd['gbs']:.0f} GB/s = {kd['gbs'] / peak:.3f} of {peak:.0f} GB/s")
    else:
        r.update(bound="hbm", achieved=kd["gbs"], peak=peak, unit="GB/s", frac=kd["gbs"] / peak)
    return r


def batch_object(cv, args, rk, local):
    """C5 (1024 distinct images, sharded by image over the ranks) plus, at N=1,
    the per-rank share of a 2/4/8-GPU run timed on this GPU."""
    inp = Inputs(cv, "c5", rk.rank, rk.world, local)
    nargs = argparse.Namespace(steps=max(2, min(args.steps, 3)), warmup=3)
    b = measure("c5", nargs, rk, inputs=inp)
    obj = {"metric": "images/sec", "value": b["value"], "unit": b["unit"], "config": config_of("c5"),
           "ms_per_step": b["ms_per_step"], "scaling": "strong", "e2e": b["e2e"], "images_per_gpu": b["n_local"],
           "data": f"{inp.n} distinct make_test_image variants (variant = image index) per GPU",
           "verified_vs_golden": b["verified_vs_golden"],
           "roofline": roofline_of(b["kernels"], "c5", (b["clocks"] or {}).get("sm_mhz")), "kernels": b["kernels"],
           "gpu_launches": b["gpu_launches"], "clocks": b["clocks"]}
    if rk.world == 1 and not args.no_shares:
        shares = {}
        for G in SHARES:
            n = inp.n // G
            s = measure("c5", nargs, rk, inputs=inp, n_share=n, profile=False)
            shares[str(G)] = {
                "images": n, "device_img_s": s["value"], "e2e_img_s": s["e2e"]["value"],
                "projected_job_img_s_e2e": G * s["e2e"]["value"], "projected_job_img_s_device": G * s["value"],
                "projected_efficiency_e2e": s["e2e"]["value"] / b["e2e"]["value"],
                "projected_efficiency_device": s["value"] / b["value"], "clocks": s["clocks"],
                "verified_vs_golden": s["verified_vs_golden"]}
        obj["shares"] = {
            "note": "one rank's share of the 1024-image batch at G GPUs, timed on this one GPU (device-resident "
                    "and e2e from pinned host buffers through carve_batch); ranks share nothing, so a G-GPU run's "
                    "time is its slowest share's time; projected efficiency = share rate / 1024-image rate",
            **shares}
    return obj


def run_ours(args, cfg_name, default_line):
    import torch

    import paper_2410_21207_b200 as cv

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device")
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    cv.set_device(local)
    rk = Ranks()
    if cfg_name == "c5" and args.emulate_world:
        # one rank's share of a G-GPU run, on this GPU
        inp = Inputs(cv, "c5", 0, args.emulate_world, local)
        m = measure("c5", args, rk, inputs=inp)
    else:
        m = measure(cfg_name, args, rk)
    batch = m["batch"]
    line = {
        "metric": "images/sec" if batch else "seams removed/sec",
        "value": m["value"], "unit": m["unit"], "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong" if batch else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_test_image, bench.hpp:67-94)",
        "config": config_of(cfg_name),
        "setup": {"images_per_gpu": m["n_local"], "parallelism": f"image-sharded x{world}, no collective",
                  "emulated_world": args.emulate_world or None},
        "e2e": m["e2e"], "gpu_launches": m["gpu_launches"],
        "roofline": roofline_of(m["kernels"], cfg_name, (m["clocks"] or {}).get("sm_mhz")),
        "kernels": m["kernels"], "verified_vs_golden": m["verified_vs_golden"], "clocks": m["clocks"],
    }
    if default_line:
        # the metric's other halves: 4K seams/s and the C5 batch (+ per-rank shares)
        c3 = measure("c3", argparse.Namespace(steps=max(2, min(args.steps, 3)), warmup=3), rk)
        line["c3"] = {"metric": "seams removed/sec", "value": c3["value"], "unit": c3["unit"],
                      "config": config_of("c3"), "ms_per_step": c3["ms_per_step"], "e2e": c3["e2e"],
                      "verified_vs_golden": c3["verified_vs_golden"],
                      "roofline": roofline_of(c3["kernels"], "c3", (c3["clocks"] or {}).get("sm_mhz")),
                      "kernels": c3["kernels"], "gpu_launches": c3["gpu_launches"], "clocks": c3["clocks"]}
        line["batch"] = batch_object(cv, args, rk, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg_name)
        if "c3" in line:
            line["c3"]["cpu_baseline"] = cpu_baseline("c3")
        if "batch" in line:
            line["batch"]["cpu_baseline"] = cpu_baseline("c5")
    if rank == 0:
        print(json.dumps(line), flush=True)
    rk.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="--config c5: time one rank's share (1024/G images) of a G-GPU run on this GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="default line: skip the C3 and C5 objects")
    ap.add_argument("--no-shares", action="store_true", help="default line: skip the per-rank share timings")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    cfg = args.config or "c2"
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg, default_line=args.config is None and not args.no_batch)


if __name__ == "__main__":
    main()
