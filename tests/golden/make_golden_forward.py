"""Golden vectors for the forward-energy DP and CarveConfig::recompute=false
(SURVEY.md §8f row 4), generated from the REFERENCE ITSELF (oracle/_ref, the
reference headers compiled unmodified). Run in the build container:

    make -C oracle && python tests/golden/make_golden_forward.py

Outputs:
  forward.npz   luma maps with forward_costs (energy.hpp:196-216) and
                dp_seam_forward tables/seams (solvers.hpp:294-326); arbitrary
                cost planes with their dp_seam_forward tables/seams; small images
                carved with forward=true, with recompute=false and with both
                (run_resize order)
  golden.json   configs["C1_FORWARD"], ["C1_NORECOMPUTE"], ["C1_FORWARD_NORECOMPUTE"]:
                FNV-1a-64 of the 512x512 -> 448x512 carve output and seams
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def h64(a: np.ndarray) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def main() -> None:
    ref = oracle.reference()
    rng = np.random.default_rng(0xF0)
    out = {}
    maps = []
    for _ in range(300):  # tie-heavy integer lumas and real-valued lumas, <= 12x12
        w, h = (int(v) for v in rng.integers(1, 13, 2))
        maps.append(np.floor(rng.uniform(0, 6, (h, w))))
    for (w, h) in [(1, 1), (1, 9), (9, 1), (2, 5), (64, 64), (257, 63), (130, 40), (300, 7), (4000, 5)]:
        maps.append(rng.uniform(0, 255, (h, w)))
    maps.append(np.full((3, 4), 55.0))
    maps.append(np.array([0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0], float).reshape(4, 4))
    for k, g in enumerate(maps):
        out[f"g{k}"] = g
        out[f"cl{k}"], out[f"cu{k}"], out[f"cr{k}"] = ref.forward_costs(g)
        out[f"seam{k}"], out[f"m{k}"], out[f"b{k}"] = ref.dp_seam_forward(g)
    out["nmaps"] = np.array(len(maps))
    shapes = [(1, 1, 1, 1), (2, 1, 1, 1), (3, 5, 2, 3), (9, 6, 5, 6), (10, 8, 10, 5), (24, 16, 10, 16),
              (37, 23, 20, 15), (64, 48, 40, 30), (97, 33, 50, 33), (128, 96, 64, 96), (5, 40, 3, 20)]
    k = 0
    for (w, h, tw, th) in shapes:
        for kind in ("random", "fixture"):
            img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8) if kind == "random" else ref.make_test_image(w, h)
            out[f"img{k}"] = img
            out[f"tgt{k}"] = np.array([tw, th], np.int32)
            out[f"fwd{k}"], out[f"fwdseams{k}"] = ref.carve_cfg(img, tw, th, forward=True, seams=True)
            out[f"norec{k}"], out[f"norecseams{k}"] = ref.carve_cfg(img, tw, th, recompute=False, seams=True)
            k += 1
    out["nimgs"] = np.array(k)
    # round 2: dp_seam_forward with arbitrary caller costs (gray supplies only the
    # dimensions, solvers.hpp:294-326) and forward + recompute=false carves, whose
    # cost planes are carved by drop_columns (carver.hpp:175-184)
    rng2 = np.random.default_rng(0xF1)
    ncm = 0
    cost_shapes = [tuple(int(v) for v in rng2.integers(1, 13, 2)) for _ in range(120)]
    cost_shapes += [(1, 1), (1, 9), (9, 1), (300, 40), (2000, 9), (64, 700), (130, 33)]
    for j, (w, h) in enumerate(cost_shapes):
        if j % 3 == 0:  # integer costs: many ties
            cs = [np.floor(rng2.uniform(0, 4, (h, w))) for _ in range(3)]
        elif j % 3 == 1:  # signed real costs
            cs = [rng2.uniform(-50, 50, (h, w)) for _ in range(3)]
        else:  # costs of some other luma (not this image's forward_costs)
            cs = list(ref.forward_costs(rng2.uniform(0, 255, (h, w))))
        for key, c in zip(("fcl", "fcu", "fcr"), cs):
            out[f"{key}{ncm}"] = c
        out[f"fseam{ncm}"], out[f"fm{ncm}"], out[f"fb{ncm}"] = ref.dp_seam_forward_costs(*cs)
        ncm += 1
    out["ncostmaps"] = np.array(ncm)
    for j in range(k):
        img, (tw, th) = out[f"img{j}"], (int(v) for v in out[f"tgt{j}"])
        out[f"fnr{j}"], out[f"fnrseams{j}"] = ref.carve_cfg(img, tw, th, forward=True, recompute=False, seams=True)
    np.savez_compressed(os.path.join(HERE, "forward.npz"), **out)

    path = os.path.join(HERE, "golden.json")
    gold = json.load(open(path))
    img = ref.make_test_image(512, 512)
    for name, fwd, rec in (("C1_FORWARD", True, True), ("C1_NORECOMPUTE", False, False),
                           ("C1_FORWARD_NORECOMPUTE", True, False)):
        o, s = ref.carve_cfg(img, 448, 512, forward=fwd, recompute=rec, seams=True)
        gold["configs"][name] = {"W": 512, "H": 512, "target_w": 448, "target_h": 512, "forward": fwd,
                                 "recompute": rec, "input": h64(img), "output": h64(o), "seams": h64(s)}
    json.dump(gold, open(path, "w"), indent=1)
    print("wrote forward.npz:", len(maps), "maps,", k, "images;", gold["configs"]["C1_FORWARD"])


if __name__ == "__main__":
    main()
