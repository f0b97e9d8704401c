"""Object removal on the GPU: apply_mask, mask_from_image
and the device-resident remove_object loop against the reference-generated
fixtures (tests/golden/make_golden_masks.py) and the CPU oracle.

Mirrors test_carver.cpp:278-345 (remove_object), test_energy.cpp:202-275
(apply_mask, mask ingestion), acceptance.cpp:259-284.
"""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2410_21207_b200 as cv

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def h64(a):
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def _seam_len(mask):
    ys, xs = np.nonzero(mask)
    h, w = mask.shape
    return h if xs.max() - xs.min() <= ys.max() - ys.min() else w


def test_masks_golden():
    z = np.load(os.path.join(GOLD, "masks.npz"))
    for k in range(int(z["n"])):
        img, mask = z[f"img{k}"], z[f"mask{k}"]
        assert np.array_equal(bits(cv.apply_mask(z[f"e{k}"], mask)), bits(z[f"biased{k}"])), k
        assert np.array_equal(cv.mask_from_image(img), z[f"mfi{k}"]), k
        fwd, restore = (int(v) for v in z[f"flags{k}"])
        n = int(z[f"n{k}"])
        cfg = cv.CarveConfig(forward=bool(fwd))
        if n < 0:
            with pytest.raises(cv.CarveError) as ei:
                cv.remove_object(img, mask, cfg, bool(restore))
            assert int(ei.value.code) == -n, k  # Errc values are the C status codes (1 + ordinal)
            continue
        res, rep = cv.remove_object(img, mask, cfg, bool(restore))
        assert rep.seam_count == n and np.array_equal(res, z[f"res{k}"]), k
        L = n * _seam_len(mask)
        flat = np.concatenate(rep.seams) if rep.seams else np.zeros(0, np.int32)
        assert np.array_equal(flat, z[f"seams{k}"][:L]), k


def test_remove_object_golden_config():
    c = json.load(open(os.path.join(GOLD, "golden.json")))["configs"]["REMOVE_OBJECT"]
    img = cv.make_test_image(c["W"], c["H"])
    t, b, l, r = c["mask_rect"]
    mask = np.zeros((c["H"], c["W"]), np.uint8)
    mask[t:b, l:r] = 1
    res, rep = cv.remove_object(img, mask)
    assert h64(res) == c["restored"] and rep.seam_count == c["seam_count"]
    assert h64(np.concatenate(rep.seams)) == c["seams"]
    res2, _ = cv.remove_object(img, mask, restore=False)
    assert h64(res2) == c["unrestored"]


@pytest.mark.parametrize("w,h", [(40, 30), (30, 40), (130, 70), (300, 20)])
def test_remove_object_vs_oracle(w, h):
    port = oracle.port()
    rng = np.random.default_rng(w * h)
    img = port.make_test_image(w, h)
    for _ in range(3):
        mask = np.zeros((h, w), np.uint8)
        t, l = int(rng.integers(0, h - 4)), int(rng.integers(0, w - 4))
        mask[t:t + int(rng.integers(1, 5)), l:l + int(rng.integers(1, 5))] = 1
        for restore in (False, True):
            want, seams, n = port.remove_object(img, mask, False, restore)
            got, rep = cv.remove_object(img, mask, restore=restore)
            assert np.array_equal(got, want) and rep.seam_count == n
            L = n * _seam_len(mask)
            assert np.array_equal(np.concatenate(rep.seams), seams[:L])


def test_remove_object_reference_cases():
    # test_carver.cpp:279-287: full-column mask carved in one seam and restored
    cols = [50, 120, 60, 70, 80]
    g = np.repeat(np.array(cols, np.uint8)[None, :, None], 5, axis=0).repeat(3, axis=2)
    mask = np.zeros((5, 5), np.uint8)
    mask[:, 1] = 1
    out, rep = cv.remove_object(g, mask)
    assert rep.seam_count == 1 and rep.seams[0].tolist() == [1, 1, 1, 1, 1] and out.shape == (5, 5, 3)
    # :288-307 orientation by bounding box
    g = cv.make_test_image(7, 9)
    mask = np.zeros((9, 7), np.uint8)
    mask[2:6, 3:5] = 1
    out, rep = cv.remove_object(g, mask, restore=False)
    assert all(len(s) == 9 for s in rep.seams) and out.shape == (9, 7 - rep.seam_count, 3)
    g = cv.make_test_image(9, 7)
    mask = np.zeros((7, 9), np.uint8)
    mask[3:5, 2:6] = 1
    out, rep = cv.remove_object(g, mask, restore=False)
    assert all(len(s) == 9 for s in rep.seams) and out.shape == (7 - rep.seam_count, 9, 3)
    # :335-344 errors
    with pytest.raises(cv.CarveError) as ei:
        cv.remove_object(np.zeros((4, 4, 3), np.uint8), np.zeros((4, 4), np.uint8))
    assert ei.value.code == cv.Errc.empty_mask
    with pytest.raises(cv.CarveError) as ei:
        cv.remove_object(np.zeros((4, 4, 3), np.uint8), np.ones((4, 3), np.uint8))
    assert ei.value.code == cv.Errc.dimension_mismatch
    # test_energy.cpp:203-223 apply_mask
    e = np.random.default_rng(17).uniform(0, 10, (5, 5))
    assert np.array_equal(cv.apply_mask(e, np.zeros((5, 5), np.uint8)), e)
    assert (cv.apply_mask(np.ones((3, 3)), np.ones((3, 3), np.uint8)) == -4000.0).all()
    # test_energy.cpp:266-275 mask ingestion
    img = np.zeros((3, 4, 3), np.uint8)
    img[1, 2] = 255
    img[2, 1] = 200
    m = cv.mask_from_image(img)
    assert m.sum() == 2 and m[1, 2] and m[2, 1]
    assert cv.mask_bounds(m) == (1, 1, 2, 2)


def test_remove_object_vertical_golden():
    """detail::remove_object_vertical (carver.hpp:289-321) against the reference:
    the column loop whatever the mask's shape, an empty mask carves nothing."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "masks.npz"))
    for k in range(int(z["nvert"])):
        img, mask, restore = z[f"vimg{k}"], z[f"vmask{k}"], bool(z[f"vrestore{k}"])
        n = int(z[f"vn{k}"])
        if n < 0:
            with pytest.raises(cv.CarveError) as ei:
                cv.remove_object_vertical(img, mask, restore=restore)
            assert ei.value.code == -n, k
            continue
        out, rep = cv.remove_object_vertical(img, mask, restore=restore)
        assert rep.seam_count == n, k
        assert np.array_equal(out, z[f"vres{k}"]), k
        flat = np.concatenate(rep.seams) if rep.seams else np.zeros(0, np.int32)
        assert np.array_equal(flat, z[f"vseams{k}"][: flat.size]), k


def test_remove_object_report_timings():
    """The report's per-seam laps (carver.hpp:299-309) come from device timestamps:
    energy (mask statistics + biased map), solve (DP), remove (removal + fix-up)."""
    img = cv.make_test_image(96, 64)
    mask = np.zeros((64, 96), np.uint8)
    mask[10:50, 40:47] = 1
    out, rep = cv.remove_object(img, mask, restore=False)
    assert rep.seam_count >= 7 and len(rep.per_seam) == rep.seam_count
    for t in rep.per_seam:
        assert t.energy_s > 0 and t.solve_s > 0 and t.remove_s > 0
    assert rep.total_s >= sum(t.energy_s + t.solve_s + t.remove_s for t in rep.per_seam)
