"""Forward energy and CarveConfig::recompute=false on the GPU (SURVEY.md §8f
row 4) against the reference-generated fixtures (tests/golden/make_golden_forward.py)
and the CPU oracle. Bar: FP64-bit-identical transition costs and cost tables,
identical seams and carved pixels.

Mirrors test_energy.cpp:169-200 (forward_costs), test_solvers.cpp:221-275
(dp_seam_forward), test_carver.cpp:160-188 (forward / recompute configs).
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


@pytest.fixture(scope="module")
def z():
    return np.load(os.path.join(GOLD, "forward.npz"))


def test_forward_costs_and_tables_golden(z):
    for k in range(int(z["nmaps"])):
        g = z[f"g{k}"]
        for got, key in zip(cv.forward_costs(g), ("cl", "cu", "cr")):
            assert np.array_equal(bits(got), bits(z[f"{key}{k}"])), (k, key)
        r = cv.dp_seam_forward(g)
        assert np.array_equal(r.seam, z[f"seam{k}"]), k
        assert np.array_equal(r.table.b, z[f"b{k}"]), k
        assert np.array_equal(bits(r.table.m), bits(z[f"m{k}"])), k


def test_forward_and_norecompute_carves_golden(z):
    for k in range(int(z["nimgs"])):
        img = z[f"img{k}"]
        tw, th = (int(v) for v in z[f"tgt{k}"])
        for key, kw in (("fwd", dict(forward=True)), ("norec", dict(recompute=False))):
            out, seams, _ = cv.carve(img, tw, th, seams=True, **kw)
            assert np.array_equal(out, z[f"{key}{k}"]), (k, key)
            flat = np.concatenate(seams) if seams else np.zeros(0, np.int32)
            assert np.array_equal(flat, z[f"{key}seams{k}"][: flat.size]), (k, key)


@pytest.mark.parametrize("name", ["C1_FORWARD", "C1_NORECOMPUTE", "C1_FORWARD_NORECOMPUTE"])
def test_c1_config_golden(name):
    c = json.load(open(os.path.join(GOLD, "golden.json")))["configs"][name]
    img = cv.make_test_image(c["W"], c["H"])
    out, seams, _ = cv.carve(img, c["target_w"], c["target_h"], seams=True, forward=c["forward"],
                             recompute=c["recompute"])
    assert h64(out) == c["output"] and h64(np.concatenate(seams)) == c["seams"]


@pytest.mark.parametrize("w,h", [(2, 2), (33, 17), (130, 40), (300, 65), (1100, 21), (4097, 12)])
def test_forward_random_vs_oracle(w, h):
    port = oracle.port()
    rng = np.random.default_rng(w + 7 * h)
    for img in (rng.integers(0, 256, (h, w, 3), dtype=np.uint8), port.make_test_image(w, h)):
        tw, th = max(1, w - max(1, w // 8)), max(1, h - h // 4)
        want, ws = port.carve_cfg(img, tw, th, forward=True, seams=True)
        got, gs, _ = cv.carve(img, tw, th, seams=True, forward=True)
        assert np.array_equal(got, want)
        assert np.array_equal(np.concatenate(gs), ws)
        g = rng.uniform(0, 255, (h, w))
        r = cv.dp_seam_forward(g)
        s, m, b = port.dp_seam_forward(g)
        assert np.array_equal(r.seam, s) and np.array_equal(r.table.b, b) and np.array_equal(bits(r.table.m), bits(m))


def test_forward_api_contract():
    # test_solvers.cpp:222-249, :262-275
    assert cv.dp_seam_forward(np.full((3, 4), 55.0)).seam.tolist() == [0, 0, 0]
    g = np.array([0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0, 200, 200, 200, 0, 0], float).reshape(4, 4)
    assert cv.dp_seam_forward(g, cv.forward_costs(g)).seam.tolist() == [2, 3, 3, 3]
    with pytest.raises(cv.CarveError) as ei:
        cv.dp_seam_forward(np.zeros((2, 3)), cv.forward_costs(np.zeros((2, 2))))
    assert ei.value.code == cv.Errc.dimension_mismatch
    # test_energy.cpp:170-190
    cl, cu, cr = cv.forward_costs(np.full((3, 4), 90.0))
    assert not cl.any() and not cu.any() and not cr.any()
    cl, cu, cr = cv.forward_costs(np.array([[10, 50, 20], [80, 40, 90]], float))
    assert cu.tolist() == [[40, 10, 30], [40, 10, 50]] and cl.tolist() == [[40, 50, 60], [110, 40, 70]]
    assert cr.tolist() == [[80, 40, 30], [70, 50, 120]]
    # test_carver.cpp:160-188
    img = cv.make_test_image(14, 10)
    for solver in (cv.SolverKind.Dynamic, cv.SolverKind.ParallelDynamic):
        out, rep = cv.carve_to_width(img, 9, cv.CarveConfig(solver=solver, forward=True))
        assert out.shape == (10, 9, 3)
        for t, s in enumerate(rep.seams):
            assert cv.validate_seam(s, 14 - t, 10) is None
    with pytest.raises(cv.CarveError) as ei:
        cv.carve_to_width(np.zeros((4, 4, 3), np.uint8), 2, cv.CarveConfig(solver=cv.SolverKind.Greedy, forward=True))
    assert ei.value.code == cv.Errc.usage_error
    out, rep = cv.carve_to_width(cv.make_test_image(16, 12), 8, cv.CarveConfig(recompute=False))
    assert out.shape == (12, 8, 3) and rep.seam_count == 8
    out, rep = cv.carve_to_width(img, 9, cv.CarveConfig(forward=True, recompute=False))
    assert out.shape == (10, 9, 3) and rep.seam_count == 5
    # non-finite caller costs: the engine fails loudly instead of guessing the
    # reference's best = +inf semantics
    g = np.zeros((3, 4))
    cl, cu, cr = cv.forward_costs(g)
    cu[1, 2] = np.inf
    with pytest.raises(cv.CarveError) as ei:
        cv.dp_seam_forward(g, (cl, cu, cr))
    assert ei.value.code == cv.Errc.usage_error


def test_forward_arbitrary_costs_golden(z):
    """dp_seam_forward(gray, costs) with caller costs that are not
    forward_costs(gray): integer (tie-heavy), signed real, another image's costs."""
    for k in range(int(z["ncostmaps"])):
        cs = (z[f"fcl{k}"], z[f"fcu{k}"], z[f"fcr{k}"])
        g = np.zeros_like(cs[0])
        r = cv.dp_seam_forward(g, cs)
        assert np.array_equal(r.seam, z[f"fseam{k}"]), k
        assert np.array_equal(r.table.b, z[f"fb{k}"]), k
        assert np.array_equal(bits(r.table.m), bits(z[f"fm{k}"])), k


def test_forward_norecompute_carves_golden(z):
    """forward + recompute=false: the phase's forward costs are computed once and
    carved alongside the image (carver.hpp:175-184)."""
    for k in range(int(z["nimgs"])):
        img = z[f"img{k}"]
        tw, th = (int(v) for v in z[f"tgt{k}"])
        out, seams, _ = cv.carve(img, tw, th, seams=True, forward=True, recompute=False)
        assert np.array_equal(out, z[f"fnr{k}"]), k
        flat = np.concatenate(seams) if seams else np.zeros(0, np.int32)
        assert np.array_equal(flat, z[f"fnrseams{k}"][: flat.size]), k


@pytest.mark.parametrize("w,h", [(33, 17), (300, 65), (1100, 21), (2500, 40)])
def test_forward_norecompute_random_vs_oracle(w, h):
    port = oracle.port()
    rng = np.random.default_rng(3 * w + h)
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    tw, th = w - max(1, w // 10), h - max(1, h // 5)
    want, ws = port.carve_cfg(img, tw, th, forward=True, recompute=False, seams=True)
    got, gs, _ = cv.carve(img, tw, th, seams=True, forward=True, recompute=False)
    assert np.array_equal(got, want)
    assert np.array_equal(np.concatenate(gs), ws)
    cs = [rng.uniform(-9, 99, (h, w)) for _ in range(3)]
    r = cv.dp_seam_forward(np.zeros((h, w)), cs)
    s, m, b = port.dp_seam_forward_costs(*cs)
    assert np.array_equal(r.seam, s) and np.array_equal(r.table.b, b) and np.array_equal(bits(r.table.m), bits(m))
