"""Golden vectors for seam recording and enlargement,
generated from the REFERENCE ITSELF (oracle/_ref, the reference headers
compiled unmodified). Run in the build container:

    make -C oracle && python tests/golden/make_golden_enlarge.py

Outputs:
  enlarge.npz   small images with record_seams (carver.hpp:226-262), run_enlarge
                (cli.hpp:262-277 -> enlarge_to_width, carver.hpp:266-285) and
                insert_seam (carver.hpp:137-140) results
  golden.json   configs["ENLARGE"]: FNV-1a-64 of a 512x384 -> 640x480 enlargement
                (output pixels and recorded seams) and of a 512x512 record_seams(64)
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


def random_seam(rng, w: int, h: int) -> np.ndarray:
    s = [int(rng.integers(0, w))]
    for _ in range(1, h):
        s.append(int(np.clip(s[-1] + rng.integers(-1, 2), 0, w - 1)))
    return np.array(s, np.int32)


def main() -> None:
    ref = oracle.reference()
    rng = np.random.default_rng(11)
    out = {}
    # (w, h, record count, enlarge target w, enlarge target h)
    shapes = [(1, 1, 0, 1, 1), (2, 1, 1, 3, 1), (1, 3, 0, 1, 5), (5, 5, 4, 9, 5), (6, 4, 3, 11, 4), (15, 9, 6, 20, 12),
              (24, 16, 10, 30, 20), (37, 23, 20, 50, 30), (64, 48, 40, 100, 60), (97, 33, 50, 120, 40),
              (3, 40, 2, 5, 70), (128, 96, 64, 200, 150)]
    k = 0
    for (w, h, cnt, tw, th) in shapes:
        for kind in ("random", "fixture"):
            img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8) if kind == "random" else ref.make_test_image(w, h)
            out[f"img{k}"] = img
            out[f"rec{k}"] = ref.record_seams(img, cnt)
            enl, seams = ref.enlarge(img, tw, th, seams=True)
            out[f"enl{k}"] = enl
            out[f"enlseams{k}"] = seams
            out[f"tgt{k}"] = np.array([cnt, tw, th], np.int32)
            seam = random_seam(rng, w, h)
            out[f"iseam{k}"] = seam
            out[f"ins{k}"] = ref.insert_seam(img, seam)
            k += 1
    out["n"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "enlarge.npz"), **out)

    path = os.path.join(HERE, "golden.json")
    gold = json.load(open(path))
    img = ref.make_test_image(512, 384)
    enl, seams = ref.enlarge(img, 640, 480, seams=True)
    img2 = ref.make_test_image(512, 512)
    rec = ref.record_seams(img2, 64)
    gold["configs"]["ENLARGE"] = {"W": 512, "H": 384, "target_w": 640, "target_h": 480, "input": h64(img),
                                  "output": h64(enl), "seams": h64(seams),
                                  "record": {"W": 512, "H": 512, "count": 64, "seams": h64(rec)}}
    json.dump(gold, open(path, "w"), indent=1)
    print("wrote enlarge.npz with", k, "cases;", gold["configs"]["ENLARGE"])


if __name__ == "__main__":
    main()
