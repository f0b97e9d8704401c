"""Golden vectors for object removal, generated from the
REFERENCE ITSELF (oracle/_ref, the reference headers compiled unmodified):

    make -C oracle && python tests/golden/make_golden_masks.py

Outputs:
  masks.npz     apply_mask (energy.hpp:220-241), mask_from_image (:244-253) and
                remove_object (carver.hpp:287-340; restore on/off, forward on/off,
                vertical and transposed orientations) on small images
  golden.json   configs["REMOVE_OBJECT"]: FNV-1a-64 of a 256x192 removal
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
    rng = np.random.default_rng(0x3A5C)
    out = {}
    k = 0
    for t in range(60):
        h, w = (int(v) for v in rng.integers(2, 16, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8) if t % 2 else ref.make_test_image(w, h)
        mask = np.zeros((h, w), np.uint8)
        top, left = int(rng.integers(0, h)), int(rng.integers(0, w))
        mh, mw = int(rng.integers(1, max(2, (h - top) // 2 + 1))), int(rng.integers(1, max(2, (w - left) // 2 + 1)))
        mask[top:top + mh, left:left + mw] = 1 + (t % 3)  # nonzero flags of any value mark
        if t % 9 == 0:
            mask[rng.integers(0, h, 3), rng.integers(0, w, 3)] = 1  # scattered cells
        fwd, restore = bool(t % 4 == 1), bool(t % 2 == 0)
        try:
            res, seams, n = ref.remove_object(img, mask, fwd, restore)
        except oracle.OracleError as ex:
            res, seams, n = np.zeros((0, 0, 3), np.uint8), np.zeros(0, np.int32), -ex.status
        e = rng.uniform(0, 100, (h, w))
        out[f"img{k}"], out[f"mask{k}"], out[f"e{k}"] = img, mask, e
        out[f"flags{k}"] = np.array([int(fwd), int(restore)], np.int32)
        out[f"res{k}"], out[f"n{k}"] = res, np.array(n, np.int32)
        out[f"seams{k}"] = seams[: max(n, 0) * max(h, w)]
        out[f"biased{k}"] = ref.apply_mask(e, mask)
        out[f"mfi{k}"] = ref.mask_from_image(img)
        k += 1
    out["n"] = np.array(k)
    # round 2: detail::remove_object_vertical (carver.hpp:289-321) on masks of any
    # shape, wider than tall and empty included (no orientation choice, no empty check)
    rng2 = np.random.default_rng(0x3A5D)
    nv = 0
    for t in range(24):
        h, w = (int(v) for v in rng2.integers(3, 18, 2))
        img = rng2.integers(0, 256, (h, w, 3), dtype=np.uint8) if t % 2 else ref.make_test_image(w, h)
        mask = np.zeros((h, w), np.uint8)
        if t % 8:
            top, left = int(rng2.integers(0, h)), int(rng2.integers(0, w))
            mask[top:top + int(rng2.integers(1, 3)), left:left + int(rng2.integers(1, w - left + 1))] = 1  # wide
        restore = bool(t % 3)
        try:
            res, seams, n = ref.remove_object_vertical(img, mask, restore)
        except oracle.OracleError as ex:
            res, seams, n = np.zeros((0, 0, 3), np.uint8), np.zeros(0, np.int32), -ex.status
        out[f"vimg{nv}"], out[f"vmask{nv}"], out[f"vrestore{nv}"] = img, mask, np.array(int(restore), np.int32)
        out[f"vres{nv}"], out[f"vseams{nv}"], out[f"vn{nv}"] = res, seams, np.array(n, np.int32)
        nv += 1
    out["nvert"] = np.array(nv)
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **out)

    path = os.path.join(HERE, "golden.json")
    gold = json.load(open(path))
    img = ref.make_test_image(256, 192)
    mask = np.zeros((192, 256), np.uint8)
    mask[60:140, 100:130] = 1
    res, seams, n = ref.remove_object(img, mask, False, True)
    res2, seams2, n2 = ref.remove_object(img, mask, False, False)
    gold["configs"]["REMOVE_OBJECT"] = {"W": 256, "H": 192, "mask_rect": [60, 140, 100, 130], "input": h64(img),
                                        "restored": h64(res), "unrestored": h64(res2), "seam_count": n,
                                        "seams": h64(seams[: n * 192])}
    json.dump(gold, open(path, "w"), indent=1)
    print("wrote masks.npz with", k, "cases;", gold["configs"]["REMOVE_OBJECT"])


if __name__ == "__main__":
    main()
