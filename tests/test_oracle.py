"""CPU suite: pins the oracle (oracle/carve_oracle.c) before it is trusted.

1. against the reference itself compiled from /root/reference (oracle/_ref),
   when that build is present;
2. against the committed golden vectors (tests/golden/, generated from the
   reference by tests/golden/make_golden.py) — always.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def port():
    return oracle.port()


@pytest.fixture(scope="module")
def gold():
    return json.load(open(os.path.join(GOLD, "golden.json")))


need_ref = pytest.mark.skipif(not oracle.have_reference(), reason="oracle/_ref not built (no /root/reference)")


def test_fixture_generator_matches_golden(port, gold):
    for name in ("C1", "C2", "C3", "C4"):
        c = gold["configs"].get(name)
        if c is None:
            continue
        img = port.make_test_image(c["W"], c["H"])
        assert f"{oracle.fnv1a64(img):016x}" == c["input"], name
    for k, rec in gold["configs"]["C5"]["samples"].items():
        img = port.make_test_image(gold["configs"]["C5"]["W"], gold["configs"]["C5"]["H"], int(k))
        assert f"{oracle.fnv1a64(img):016x}" == rec["input"], k


def test_c1_energy_and_table_golden(port, gold):
    c = gold["configs"]["C1"]
    img = port.make_test_image(512, 512)
    e = port.energy_e1_rgb(img)
    assert f"{oracle.fnv1a64(e):016x}" == c["energy0"]
    seam, m, b = port.dp_seam(e)
    assert f"{oracle.fnv1a64(m):016x}" == c["table0_m"]
    assert f"{oracle.fnv1a64(b):016x}" == c["table0_b"]
    assert f"{oracle.fnv1a64(seam):016x}" == c["seam0"]


def test_c1_full_carve_golden(port, gold):
    c = gold["configs"]["C1"]
    out, seams = port.carve(port.make_test_image(512, 512), 448, seams=True)
    assert f"{oracle.fnv1a64(out):016x}" == c["output"]
    assert f"{oracle.fnv1a64(seams):016x}" == c["seams"]


def test_corpus_golden(port):
    z = np.load(os.path.join(GOLD, "corpus.npz"))
    for k in range(int(z["n"])):
        e = z[f"e{k}"].astype(np.float64)
        seam, m, b = port.dp_seam(e)
        assert np.array_equal(seam, z[f"s{k}"]), k
        assert np.array_equal(b, z[f"b{k}"].astype(np.int32)), k
        assert np.array_equal(m, z[f"m{k}"].astype(np.float64)), k


def test_small_images_golden(port):
    z = np.load(os.path.join(GOLD, "small.npz"))
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        tw, th = (int(v) for v in z[f"tgt{k}"])
        assert np.array_equal(bits(port.energy_e1_rgb(img)), bits(z[f"e{k}"])), k
        out, seams = port.carve(img, tw, th, seams=True)
        assert np.array_equal(out, z[f"out{k}"]), k
        assert np.array_equal(seams, z[f"seams{k}"][: seams.size]), k


def test_port_reference_cases(port):
    # test_solvers.cpp:152-174, test_energy.cpp:33-64, test_carver.cpp:34-73
    seam, m, _ = port.dp_seam(np.array([[1, 2, 3], [4, 1, 6], [7, 8, 1]], np.float64))
    assert m.tolist() == [[1, 2, 3], [5, 2, 8], [9, 10, 3]] and seam.tolist() == [0, 1, 2]
    assert port.dp_seam(np.array([[8.0, 2, 6, 2]]))[0].tolist() == [1]
    assert port.energy_e1_luma(np.array([[0.0, 100.0, 0.0]])).tolist() == [[100.0, 0.0, 100.0]]
    assert port.validate_seam([0, 2], 3, 2) == 6  # invalid_seam
    with pytest.raises(oracle.OracleError):
        port.remove_seam(np.zeros((2, 1, 3), np.uint8), [0, 0])


@need_ref
def test_port_vs_reference_random(port):
    ref = oracle.reference()
    rng = np.random.default_rng(11)
    for _ in range(40):
        w, h = (int(x) for x in rng.integers(1, 40, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        assert np.array_equal(bits(port.to_grayscale(img)), bits(ref.to_grayscale(img)))
        assert np.array_equal(bits(port.energy_e1_rgb(img)), bits(ref.energy_e1_rgb(img)))
        assert np.array_equal(port.transpose(img), ref.transpose(img))
        e = ref.energy_e1_rgb(img)
        s1, m1, b1 = port.dp_seam(e)
        s2, m2, b2 = ref.dp_seam(e)
        assert np.array_equal(s1, s2) and np.array_equal(bits(m1), bits(m2)) and np.array_equal(b1, b2)
        tw, th = int(rng.integers(1, w + 1)), int(rng.integers(1, h + 1))
        o1, q1 = port.carve(img, tw, th, seams=True)
        o2, q2 = ref.carve(img, tw, th, seams=True)
        assert np.array_equal(o1, o2) and np.array_equal(q1, q2)


@need_ref
def test_port_vs_reference_fixture(port):
    ref = oracle.reference()
    for (w, h) in [(1, 1), (2, 3), (640, 360), (1920, 1080)]:
        assert np.array_equal(port.make_test_image(w, h), ref.make_test_image(w, h))


@need_ref
def test_reference_pardp_equals_dp():
    ref = oracle.reference()
    img = ref.make_test_image(300, 200)
    e = ref.energy_e1_rgb(img)
    a = ref.dp_seam(e, 0)
    b = ref.dp_seam(e, 1, 4)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


# -- seam recording and enlargement ---------------------------
def test_enlarge_golden(port):
    """The C restatement of record_seams / enlarge_to_width (replay with shifts) /
    insert_seam against the reference-generated fixtures (make_golden_enlarge.py)."""
    z = np.load(os.path.join(GOLD, "enlarge.npz"))
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        cnt, tw, th = (int(v) for v in z[f"tgt{k}"])
        assert np.array_equal(port.record_seams(img, cnt), z[f"rec{k}"]), k
        out, seams = port.enlarge(img, tw, th, seams=True)
        assert np.array_equal(out, z[f"enl{k}"]), k
        assert np.array_equal(seams, z[f"enlseams{k}"][: seams.size]), k
        assert np.array_equal(port.insert_seam(img, z[f"iseam{k}"]), z[f"ins{k}"]), k


def test_enlarge_golden_config(port, gold):
    c = gold["configs"]["ENLARGE"]
    img = port.make_test_image(c["W"], c["H"])
    assert f"{oracle.fnv1a64(img):016x}" == c["input"]
    out, seams = port.enlarge(img, c["target_w"], c["target_h"], seams=True)
    assert f"{oracle.fnv1a64(out):016x}" == c["output"]
    assert f"{oracle.fnv1a64(seams):016x}" == c["seams"]
    r = c["record"]
    rec = port.record_seams(port.make_test_image(r["W"], r["H"]), r["count"])
    assert f"{oracle.fnv1a64(rec):016x}" == r["seams"]


def test_enlarge_errors(port):
    # test_carver.cpp:247-253, :271-275
    g = port.make_test_image(6, 4)
    for (tw, th, st) in [(5, 4, 1 + 9), (12, 4, 1 + 10), (6, 3, 1 + 9), (6, 8, 1 + 10)]:
        with pytest.raises(oracle.OracleError) as ei:
            port.enlarge(g, tw, th)
        assert ei.value.status == st
    assert port.enlarge(g, 11, 4).shape == (4, 11, 3)
    with pytest.raises(oracle.OracleError) as ei:
        port.record_seams(np.zeros((4, 4, 3), np.uint8), 4)
    assert ei.value.status == 1 + 9


@need_ref
def test_enlarge_port_vs_reference_random(port):
    ref = oracle.reference()
    rng = np.random.default_rng(21)
    for _ in range(40):
        h, w = (int(v) for v in rng.integers(1, 16, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        cnt = int(rng.integers(0, w))
        assert np.array_equal(port.record_seams(img, cnt), ref.record_seams(img, cnt))
        tw, th = w + int(rng.integers(0, w)), h + int(rng.integers(0, h))
        a, sa = port.enlarge(img, tw, th, seams=True)
        b, sb = ref.enlarge(img, tw, th, seams=True)
        assert np.array_equal(a, b) and np.array_equal(sa, sb)


# -- forward energy and recompute=false ---------------------------
def fbits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_forward_golden(port):
    """The C restatement of forward_costs / dp_seam_forward / the forward and
    recompute=false carve loops against the reference-generated fixtures."""
    z = np.load(os.path.join(GOLD, "forward.npz"))
    for k in range(int(z["nmaps"])):
        g = z[f"g{k}"]
        for got, key in zip(port.forward_costs(g), ("cl", "cu", "cr")):
            assert np.array_equal(fbits(got), fbits(z[f"{key}{k}"])), (k, key)
        seam, m, b = port.dp_seam_forward(g)
        assert np.array_equal(seam, z[f"seam{k}"]) and np.array_equal(b, z[f"b{k}"]), k
        assert np.array_equal(fbits(m), fbits(z[f"m{k}"])), k
    for k in range(int(z["nimgs"])):
        img = z[f"img{k}"]
        tw, th = (int(v) for v in z[f"tgt{k}"])
        o, s = port.carve_cfg(img, tw, th, forward=True, seams=True)
        assert np.array_equal(o, z[f"fwd{k}"]) and np.array_equal(s, z[f"fwdseams{k}"][: s.size]), k
        o, s = port.carve_cfg(img, tw, th, recompute=False, seams=True)
        assert np.array_equal(o, z[f"norec{k}"]) and np.array_equal(s, z[f"norecseams{k}"][: s.size]), k


def test_forward_reference_cases(port):
    # test_solvers.cpp:222-249: constant image -> leftmost seam; diagonal edge
    assert port.dp_seam_forward(np.full((3, 4), 55.0))[0].tolist() == [0, 0, 0]
    g = np.array([0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0], float).reshape(4, 4)
    assert port.dp_seam_forward(g)[0].tolist() == [2, 3, 3, 3]
    # test_energy.cpp:178-190: hand-evaluated 2x3 costs
    cl, cu, cr = port.forward_costs(np.array([[10, 50, 20], [80, 40, 90]], float))
    assert cu.tolist() == [[40, 10, 30], [40, 10, 50]]
    assert cl.tolist() == [[40, 50, 60], [110, 40, 70]]
    assert cr.tolist() == [[80, 40, 30], [70, 50, 120]]


@need_ref
def test_forward_port_vs_reference_random(port):
    ref = oracle.reference()
    rng = np.random.default_rng(44)
    for t in range(30):
        h, w = (int(v) for v in rng.integers(1, 20, 2))
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8) if t % 2 else port.make_test_image(w, h)
        tw, th = int(rng.integers(1, w + 1)), int(rng.integers(1, h + 1))
        for fwd, rec in ((True, True), (False, False)):
            a, sa = port.carve_cfg(img, tw, th, fwd, rec, seams=True)
            b, sb = ref.carve_cfg(img, tw, th, fwd, rec, seams=True)
            assert np.array_equal(a, b) and np.array_equal(sa, sb)


# -- object removal ------------------------------------------------
def _seam_len(mask):
    ys, xs = np.nonzero(mask)
    h, w = mask.shape
    return h if xs.max() - xs.min() <= ys.max() - ys.min() else w


def test_masks_golden(port):
    z = np.load(os.path.join(GOLD, "masks.npz"))
    for k in range(int(z["n"])):
        img, mask = z[f"img{k}"], z[f"mask{k}"]
        assert np.array_equal(fbits(port.apply_mask(z[f"e{k}"], mask)), fbits(z[f"biased{k}"])), k
        assert np.array_equal(port.mask_from_image(img), z[f"mfi{k}"]), k
        fwd, restore = (int(v) for v in z[f"flags{k}"])
        n = int(z[f"n{k}"])
        if n < 0:
            with pytest.raises(oracle.OracleError) as ei:
                port.remove_object(img, mask, fwd, restore)
            assert ei.value.status == -n, k
            continue
        res, seams, got_n = port.remove_object(img, mask, fwd, restore)
        L = n * _seam_len(mask)
        assert got_n == n and np.array_equal(res, z[f"res{k}"]), k
        assert np.array_equal(seams[:L], z[f"seams{k}"][:L]), k


def test_remove_seam_planes_port_golden(port):
    """The C restatement of detail::drop_columns against the reference's api.npz."""
    z = np.load(os.path.join(GOLD, "api.npz"))
    for k in range(int(z["n"])):
        got = port.remove_seam_plane(z[f"plane{k}"], z[f"seam{k}"])
        assert np.array_equal(got.view(np.uint8), z[f"want{k}"].view(np.uint8)), k


def test_forward_costs_norecompute_port_golden(port):
    """The C restatement of dp_seam_forward(gray, costs) with arbitrary costs and
    of the forward + recompute=false loop against the reference's forward.npz."""
    z = np.load(os.path.join(GOLD, "forward.npz"))
    for k in range(int(z["ncostmaps"])):
        s, m, b = port.dp_seam_forward_costs(z[f"fcl{k}"], z[f"fcu{k}"], z[f"fcr{k}"])
        assert np.array_equal(s, z[f"fseam{k}"]) and np.array_equal(b, z[f"fb{k}"]), k
        assert np.array_equal(m.view(np.uint64), z[f"fm{k}"].view(np.uint64)), k
    for k in range(int(z["nimgs"])):
        tw, th = (int(v) for v in z[f"tgt{k}"])
        out, seams = port.carve_cfg(z[f"img{k}"], tw, th, forward=True, recompute=False, seams=True)
        assert np.array_equal(out, z[f"fnr{k}"]) and np.array_equal(seams, z[f"fnrseams{k}"][: seams.size]), k
