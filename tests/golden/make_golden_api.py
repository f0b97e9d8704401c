"""Golden vectors for the remove_seam overloads on scalar planes
(remove_seam(LumaGrid / EnergyMap / RemovalMask) = detail::drop_columns,
carver.hpp:57-112), generated from the REFERENCE ITSELF (oracle/_ref, the
reference headers compiled unmodified). Run in the build container:

    make -C oracle && python tests/golden/make_golden_api.py

Output: api.npz — for each case k: the plane (float64 luma/energy or uint8
mask), the seam (connected or not: the reference does not validate these
overloads), and the reference's result.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    ref = oracle.reference()
    rng = np.random.default_rng(0xA91)
    out = {}
    shapes = [(1, 1), (2, 1), (1, 5), (3, 3), (17, 4), (64, 64), (257, 63), (1000, 3), (5, 300)]
    shapes += [tuple(int(v) for v in rng.integers(1, 40, 2)) for _ in range(40)]
    k = 0
    for (w, h) in shapes:
        for kind in ("luma", "energy", "mask"):
            if kind == "mask":
                plane = (rng.random((h, w)) < 0.3).astype(np.uint8)
            else:
                plane = rng.uniform(0, 510, (h, w))
            if k % 2:  # a connected seam
                s = np.empty(h, np.int32)
                s[0] = rng.integers(0, w)
                for i in range(1, h):
                    s[i] = np.clip(s[i - 1] + rng.integers(-1, 2), 0, w - 1)
            else:  # arbitrary per-row columns
                s = rng.integers(0, w, h).astype(np.int32)
            out[f"plane{k}"] = plane
            out[f"seam{k}"] = s
            out[f"kind{k}"] = np.array(kind)
            out[f"want{k}"] = ref.remove_seam_plane(plane, s, kind)
            k += 1
    out["n"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)
    print("wrote api.npz:", k, "cases")


if __name__ == "__main__":
    main()
