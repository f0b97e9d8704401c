"""Regenerate the golden vectors in tests/golden/ from the REFERENCE ITSELF.

The reference ships no golden files, so every fixture
here is produced by /root/reference/proj/include compiled unmodified through
oracle/ref_shim.cpp (oracle/_ref/libcarve_ref.so). Run in the build
container (the reference tree does not exist on the GPU box):

    make -C oracle && python tests/golden/make_golden.py [--full]

--full also carves C3 (3840x2160 -> 3072x1728) and C4 (7680x4320 -> 7168x4320)
with the reference `dp` path, which takes ~15 CPU-minutes.

Outputs:
  golden.json    hashes (FNV-1a-64) of final pixels per config, of seam lists,
                 of the C1 initial energy bits and of the C1 seam-0 cost table
  corpus.npz     tie-heavy DP corpus: maps (integer-valued), reference seams,
                 predecessor tables and cost tables
  small.npz      small images with their reference energies and carve outputs
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, W, H, target_w, target_h) — BASELINE.json configs, SURVEY.md §8d
CONFIGS = {
    "C1": (512, 512, 448, 512),
    "C2": (1920, 1080, 1728, 1080),
    "C3": (3840, 2160, 3072, 1728),
    "C4": (7680, 4320, 7168, 4320),
}
C5 = (1024, 768, 896)
C5_SAMPLE = [0, 1, 2, 3, 255, 511, 767, 1023]


def h64(a: np.ndarray) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def corpus(ref) -> dict:
    """Tie-heavy DP corpus: integer-valued maps like
    tests/oracles.hpp:120-129, constant maps, steps, and the narrow shapes of
    test_solvers.cpp:302-308."""
    rng = np.random.default_rng(0xACCE55)
    maps = []
    for _ in range(1000):  # acceptance.cpp:95-101 shape range (<= 12x12)
        w, h = rng.integers(1, 13, 2)
        maps.append(np.floor(rng.uniform(0, 100, (h, w))))
    for (w, h) in [(1, 7), (2, 5), (300, 1), (3, 3), (257, 63), (200, 200), (130, 40), (64, 64), (7, 30), (1, 1)]:
        maps.append(np.floor(rng.uniform(0, 100, (h, w))))
    for (w, h) in [(6, 4), (33, 17), (1, 9), (65, 3)]:
        maps.append(np.zeros((h, w)))  # all ties
    step = np.zeros((5, 8))
    step[:, 4:] = 255.0
    maps.append(step)
    maps.append(np.floor(rng.uniform(0, 3, (40, 97))))  # dense ties
    out = {"n": np.array(len(maps))}
    for k, m in enumerate(maps):
        seam, mt, bt = ref.dp_seam(m)
        seam_p, mt_p, bt_p = ref.dp_seam(m, solver=1, workers=4)
        assert (seam == seam_p).all() and (mt == mt_p).all() and (bt == bt_p).all()
        out[f"e{k}"] = m.astype(np.uint16)
        out[f"s{k}"] = seam
        out[f"b{k}"] = bt.astype(np.int16)
        out[f"m{k}"] = mt.astype(np.uint32)  # integer sums: exact
        assert (out[f"m{k}"].astype(np.float64) == mt).all()
    return out


def small_images(ref) -> dict:
    rng = np.random.default_rng(7)
    out = {}
    shapes = [(1, 1, 1, 1), (2, 1, 1, 1), (3, 5, 2, 3), (9, 6, 5, 6), (10, 8, 10, 5), (24, 16, 10, 16),
              (37, 23, 20, 15), (64, 48, 40, 30), (97, 33, 50, 33), (128, 96, 64, 96), (5, 40, 3, 20)]
    k = 0
    for (w, h, tw, th) in shapes:
        for kind in ("random", "fixture"):
            if kind == "random":
                img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
            else:
                img = ref.make_test_image(w, h)
            carved, seams = ref.carve(img, tw, th, solver=1, workers=4, seams=True)
            carved_dp = ref.carve(img, tw, th, solver=0)
            assert (carved == carved_dp).all()
            out[f"img{k}"] = img
            out[f"e{k}"] = ref.energy_e1_rgb(img)
            out[f"out{k}"] = carved
            out[f"seams{k}"] = seams
            out[f"tgt{k}"] = np.array([tw, th], np.int32)
            k += 1
    out["n"] = np.array(k)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true", help="also carve C3/C4 with the reference (slow)")
    args = ap.parse_args()
    ref = oracle.reference()
    port = oracle.port()
    gold = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference compiled in place)",
            "hash": "FNV-1a-64 over the raw bytes (offset 0xcbf29ce484222325, prime 0x100000001b3)",
            "configs": {}}
    path = os.path.join(HERE, "golden.json")
    if os.path.exists(path):
        gold["configs"] = json.load(open(path)).get("configs", {})

    names = ["C1", "C2"] + (["C3", "C4"] if args.full else [])
    for name in names:
        w, h, tw, th = CONFIGS[name]
        img = ref.make_test_image(w, h)
        assert (img == port.make_test_image(w, h)).all()
        t = time.time()
        out, seams = ref.carve(img, tw, th, solver=0, seams=True)
        dt = time.time() - t
        rec = {"W": w, "H": h, "target_w": tw, "target_h": th, "input": h64(img), "output": h64(out),
               "seams": h64(seams), "ref_dp_seconds": round(dt, 3)}
        if name == "C1":
            e = ref.energy_e1_rgb(img)
            seam, m, b = ref.dp_seam(e)
            rec.update(energy0=h64(e), table0_m=h64(m), table0_b=h64(b), seam0=h64(seam))
        gold["configs"][name] = rec
        print(name, rec, flush=True)
        json.dump(gold, open(path, "w"), indent=1)

    w, h, tw = C5
    c5 = {}
    for k in C5_SAMPLE:
        img = port.make_test_image(w, h, k)
        out = ref.carve(img, tw, h, solver=0)
        c5[str(k)] = {"input": h64(img), "output": h64(out)}
    gold["configs"]["C5"] = {"W": w, "H": h, "target_w": tw, "target_h": h, "variant_rule":
                             "variant k xors k into the make_test_image seed (k=0: reference fixture)",
                             "samples": c5}
    json.dump(gold, open(path, "w"), indent=1)

    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **corpus(ref))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small_images(ref))
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
