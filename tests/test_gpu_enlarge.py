"""Parity of seam recording and enlargement on the GPU
against the reference-generated fixtures (tests/golden/make_golden_enlarge.py)
and the CPU oracle. Bar: identical recorded columns and identical pixels.

Mirrors the reference's own pins: test_carver.cpp:75-105 (insert_seam),
:213-254 (enlarge_to_width), :256-276 (record_seams), acceptance.cpp:250-257
(enlarge by k then carve by k restores the dimensions), test_cli.cpp:185-188.
"""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2410_21207_b200 as cv

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def h64(a):
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def test_enlarge_fixtures():
    z = np.load(os.path.join(GOLD, "enlarge.npz"))
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        cnt, tw, th = (int(v) for v in z[f"tgt{k}"])
        seams, rep = cv.record_seams(img, cnt)
        got = np.stack(seams) if seams else np.zeros((0, img.shape[0]), np.int32)
        assert np.array_equal(got, z[f"rec{k}"]), k
        assert rep.seam_count == cnt and len(rep.per_seam) == cnt
        out, s = cv.enlarge(img, tw, th, seams=True)
        assert np.array_equal(out, z[f"enl{k}"]), k
        assert np.array_equal(s, z[f"enlseams{k}"][: s.size]), k
        assert np.array_equal(cv.insert_seam(img, z[f"iseam{k}"]), z[f"ins{k}"]), k


def test_enlarge_golden_config():
    c = json.load(open(os.path.join(GOLD, "golden.json")))["configs"]["ENLARGE"]
    img = cv.make_test_image(c["W"], c["H"])
    assert h64(img) == c["input"]
    out, seams = cv.enlarge(img, c["target_w"], c["target_h"], seams=True)
    assert h64(out) == c["output"] and h64(seams) == c["seams"]
    r = c["record"]
    rec, _ = cv.record_seams(cv.make_test_image(r["W"], r["H"]), r["count"])
    assert h64(np.stack(rec)) == r["seams"]


@pytest.mark.parametrize("w,h", [(2, 2), (7, 3), (33, 17), (130, 40), (300, 65), (1000, 9)])
def test_enlarge_random_vs_oracle(port, w, h):
    rng = np.random.default_rng(w * 31 + h)
    for img in (rng.integers(0, 256, (h, w, 3), dtype=np.uint8), port.make_test_image(w, h)):
        for cnt in sorted({0, 1, w // 3, w - 1}):
            seams, _ = cv.record_seams(img, cnt)
            got = np.stack(seams) if seams else np.zeros((0, h), np.int32)
            assert np.array_equal(got, port.record_seams(img, cnt))
        tw, th = w + max(1, w // 2) if w > 1 else 1, h + (h // 2)
        assert np.array_equal(cv.enlarge(img, tw, th), port.enlarge(img, tw, th))
        assert np.array_equal(cv.enlarge(img, 2 * w - 1, h), port.enlarge(img, 2 * w - 1, h))


def test_insert_seam_cases():
    # test_carver.cpp:76-92
    g = np.array([[[9, 8, 7]]], np.uint8)
    out = cv.insert_seam(g, [0])
    assert out.shape == (1, 2, 3) and (out == [9, 8, 7]).all()
    g = np.array([[[0, 0, 0], [100, 100, 100]]], np.uint8)
    assert cv.insert_seam(g, [0]).tolist() == [[[0, 0, 0], [50, 50, 50], [100, 100, 100]]]
    # test_carver.cpp:93-104: insert then remove at the inserted position restores the grid
    rng = np.random.default_rng(2)
    for _ in range(20):
        h, w = (int(v) for v in rng.integers(1, 10, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        s = [int(rng.integers(0, w))]
        for _ in range(1, h):
            s.append(int(np.clip(s[-1] + rng.integers(-1, 2), 0, w - 1)))
        wider = cv.insert_seam(img, s)
        assert np.array_equal(cv.remove_seam(wider, [c + 1 for c in s]), img)
    with pytest.raises(cv.CarveError) as ei:
        cv.insert_seam(np.zeros((2, 3, 3), np.uint8), [0, 2])
    assert ei.value.code == cv.Errc.invalid_seam


def test_enlarge_to_width_cases():
    # test_carver.cpp:214-231
    rng = np.random.default_rng(7)
    g = rng.integers(0, 256, (5, 5, 3), dtype=np.uint8)
    out, rep = cv.enlarge_to_width(g, 5)
    assert np.array_equal(out, g) and rep.seam_count == 0
    g = np.array([[[10, 20, 30], [30, 40, 50]]], np.uint8)
    out, rep = cv.enlarge_to_width(g, 3)
    assert rep.seam_count == 1 and rep.seams[0].tolist() == [0]
    assert out.tolist() == [[[10, 20, 30], [20, 30, 40], [30, 40, 50]]]
    # :233-245 / acceptance.cpp:250-257: enlarge by k then carve by k restores the dimensions
    rng = np.random.default_rng(8)
    for _ in range(8):
        h, w = (int(v) for v in rng.integers(3, 15, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        k = int(rng.integers(1, w))
        wider, _ = cv.enlarge_to_width(img, w + k)
        assert wider.shape == (h, w + k, 3)
        back, _ = cv.carve_to_width(wider, w)
        assert back.shape == img.shape
    # :247-253 target bounds
    g = cv.make_test_image(6, 4)
    for tw, code in [(5, cv.Errc.invalid_target), (12, cv.Errc.target_too_large)]:
        with pytest.raises(cv.CarveError) as ei:
            cv.enlarge_to_width(g, tw)
        assert ei.value.code == code
    assert cv.enlarge_to_width(g, 11)[0].shape == (4, 11, 3)


def test_record_seams_cases():
    # test_carver.cpp:257-270: recorded original coordinates are distinct per row
    g = cv.make_test_image(15, 9)
    seams, rep = cv.record_seams(g, 6)
    assert len(seams) == 6 and rep.seam_count == 6 and len(rep.per_seam) == 6
    cols = np.stack(seams)
    for i in range(9):
        c = np.sort(cols[:, i])
        assert (np.diff(c) > 0).all() and c[0] >= 0 and c[-1] < 15
    # :271-275
    with pytest.raises(cv.CarveError) as ei:
        cv.record_seams(np.zeros((4, 4, 3), np.uint8), 4)
    assert ei.value.code == cv.Errc.invalid_target
