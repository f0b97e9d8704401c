"""Parity of the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden vectors. Bar: bit-exact everywhere — FP64 bits of
energies and cost tables, seam column indices, carved pixels.

Mirrors the reference's own pins: test_solvers.cpp:152-326,
test_energy.cpp:33-64, test_carver.cpp:34-210, acceptance.cpp:108-122,212-218.
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


@pytest.fixture(scope="module")
def port():
    return oracle.port()


@pytest.fixture(scope="module")
def gold():
    return json.load(open(os.path.join(GOLD, "golden.json")))


# -- K1 energy --------------------------------------------------------------------
@pytest.mark.parametrize("w,h", [(1, 1), (1, 7), (7, 1), (2, 2), (3, 5), (63, 17), (64, 16), (65, 17),
                                 (130, 33), (512, 512), (1920, 1080)])
def test_energy_rgb_bitexact(port, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    for img in (rng.integers(0, 256, (h, w, 3), dtype=np.uint8), port.make_test_image(w, h)):
        assert np.array_equal(bits(cv.energy_e1_rgb(img)), bits(port.energy_e1_rgb(img)))
        assert np.array_equal(bits(cv.to_grayscale(img)), bits(port.to_grayscale(img)))


@pytest.mark.parametrize("k1v", ["0", "1", "2", "3", "4", "5", "6", "-1"])
def test_energy_every_k1_shape_bitexact(port, monkeypatch, k1v):
    """Each K1 launch shape (CARVE_K1V: 2 or 3 CTAs/SM, prefetch depth, run
    length; -1 = the size-based default, which switches shape at 4 Mpx)."""
    monkeypatch.setenv("CARVE_K1V", k1v)
    for w, h in [(130, 33), (1920, 1080), (2500, 1700)]:
        img = port.make_test_image(w, h)
        assert np.array_equal(bits(cv.energy_e1_rgb(img)), bits(port.energy_e1_rgb(img)))


def test_energy_luma_reference_cases():
    # test_energy.cpp:33-64
    assert (cv.energy_e1(np.full((4, 6), 123.0)) == 0).all()
    e = cv.energy_e1(np.array([[0.0, 100.0, 0.0]]))
    assert e.tolist() == [[100.0, 0.0, 100.0]]
    g = np.zeros((5, 8))
    g[:, 4:] = 255.0
    e = cv.energy_e1(g)
    exp = np.zeros((5, 8))
    exp[:, 3:5] = 255.0
    assert np.array_equal(e, exp)


def test_energy_luma_random(port):
    rng = np.random.default_rng(3)
    for (w, h) in [(1, 1), (9, 4), (100, 37)]:
        g = rng.uniform(0, 255, (h, w))
        assert np.array_equal(bits(cv.energy_e1(g)), bits(port.energy_e1_luma(g)))


def test_energy_golden_c1(port, gold):
    img = cv.make_test_image(512, 512)
    assert f"{oracle.fnv1a64(img):016x}" == gold["configs"]["C1"]["input"]
    assert f"{oracle.fnv1a64(cv.energy_e1_rgb(img)):016x}" == gold["configs"]["C1"]["energy0"]


# -- K2/K3 DP ---------------------------------------------------------------------
def test_dp_corpus_tables_bitexact():
    z = np.load(os.path.join(GOLD, "corpus.npz"))
    for k in range(int(z["n"])):
        e = z[f"e{k}"].astype(np.float64)
        r = cv.dp_seam(e)
        assert np.array_equal(r.seam, z[f"s{k}"]), k
        assert np.array_equal(r.table.b, z[f"b{k}"].astype(np.int32)), k
        assert np.array_equal(r.table.m, z[f"m{k}"].astype(np.float64)), k


def test_dp_worked_example():
    # test_solvers.cpp:156-174
    m = np.array([[1, 2, 3], [4, 1, 6], [7, 8, 1]], np.float64)
    r = cv.dp_seam(m)
    assert r.table.m.tolist() == [[1, 2, 3], [5, 2, 8], [9, 10, 3]]
    assert r.seam.tolist() == [0, 1, 2]
    assert cv.dp_seam(np.array([[8.0, 2, 6, 2]])).seam.tolist() == [1]  # :152-155


@pytest.mark.parametrize("w,h", [(1, 1), (1, 300), (2, 5), (300, 1), (31, 9), (33, 70), (257, 63), (1024, 768),
                                 (1025, 40), (2048, 50), (2049, 65), (4097, 40), (7680, 70), (8192, 33)])
def test_dp_random_real_energies(port, w, h):
    """Real-valued (non-integer) FP64 energies from the fixture: bit-exact m, b, seam."""
    img = port.make_test_image(w, h)
    e = port.energy_e1_rgb(img)
    seam, m, b = port.dp_seam(e)
    r = cv.dp_seam(e)
    assert np.array_equal(r.seam, seam)
    assert np.array_equal(bits(r.table.m), bits(m))
    assert np.array_equal(r.table.b, b)
    assert np.array_equal(cv.find_seam(e, cv.SolverKind.Dynamic), seam)


def test_dp_ties_everywhere(port):
    for (w, h) in [(1, 5), (6, 4), (64, 64), (1000, 300), (3000, 97)]:
        e = np.zeros((h, w))
        r = cv.dp_seam(e)
        assert (r.seam == 0).all()
        rng = np.random.default_rng(w)
        e = np.floor(rng.uniform(0, 2, (h, w)))
        seam, m, b = port.dp_seam(e)
        r = cv.dp_seam(e)
        assert np.array_equal(r.seam, seam) and np.array_equal(r.table.b, b) and np.array_equal(r.table.m, m)


def test_dp_1080_fixture_matches(port):
    # acceptance.cpp:212-218 (criterion 7's parity half)
    img = port.make_test_image(1080, 1080)
    e = port.energy_e1_rgb(img)
    seam, m, b = port.dp_seam(e)
    r = cv.parallel_dp_seam(e, 4)
    assert np.array_equal(r.seam, seam) and np.array_equal(bits(r.table.m), bits(m)) and np.array_equal(r.table.b, b)


# -- K4 removal, transpose ----------------------------------------------------------
def test_remove_seam_cases(port):
    g = np.zeros((1, 2, 3), np.uint8)
    g[0, 0] = 1
    g[0, 1] = 2
    assert cv.remove_seam(g, [0]).tolist() == [[[2, 2, 2]]]  # test_carver.cpp:35-42
    rng = np.random.default_rng(1)
    for (w, h) in [(3, 3), (9, 6), (33, 5), (130, 20), (1921, 7)]:
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        s = [int(rng.integers(0, w))]
        for _ in range(h - 1):
            s.append(int(np.clip(s[-1] + rng.integers(-1, 2), 0, w - 1)))
        assert np.array_equal(cv.remove_seam(img, s), port.remove_seam(img, s))


def test_remove_seam_errors():
    with pytest.raises(cv.CarveError) as ei:
        cv.remove_seam(np.zeros((2, 1, 3), np.uint8), [0, 0])
    assert ei.value.code == cv.Errc.width_too_small
    with pytest.raises(cv.CarveError) as ei:
        cv.remove_seam(np.zeros((2, 3, 3), np.uint8), [0, 2])
    assert ei.value.code == cv.Errc.invalid_seam


def test_transpose(port):
    rng = np.random.default_rng(2)
    for (w, h) in [(1, 1), (3, 2), (5, 4), (33, 65), (100, 7)]:
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        t = cv.transpose(img)
        assert np.array_equal(t, port.transpose(img))
        assert np.array_equal(cv.transpose(t), img)


# -- whole pipeline -------------------------------------------------------------------
def test_carve_small_golden(dp_mode):
    z = np.load(os.path.join(GOLD, "small.npz"))
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        tw, th = (int(v) for v in z[f"tgt{k}"])
        out, seams, _ = cv.carve(img, tw, th, seams=True)
        assert np.array_equal(out, z[f"out{k}"]), k
        flat = np.concatenate(seams) if seams else np.zeros(0, np.int32)
        ref = z[f"seams{k}"][: flat.size]
        assert np.array_equal(flat, ref), k
        assert np.array_equal(bits(cv.energy_e1_rgb(img)), bits(z[f"e{k}"])), k


@pytest.fixture(params=["plane", "fused"])
def dp_mode(request, monkeypatch):
    """Run a test under both DP modes: the incremental energy plane (single-image
    default) and the fused RGBX-recompute mode (batch default), CARVE_FUSED."""
    monkeypatch.setenv("CARVE_FUSED", "1" if request.param == "fused" else "0")
    return request.param


@pytest.mark.parametrize("w,h,tw,th", [(64, 48, 40, 48), (100, 80, 60, 50), (37, 120, 30, 100), (200, 3, 150, 3),
                                       (5, 200, 5, 100), (260, 140, 129, 70), (2, 2, 1, 1), (3, 1, 1, 1),
                                       (1, 9, 1, 4)])
def test_carve_vs_port(port, dp_mode, w, h, tw, th):
    rng = np.random.default_rng(w + h)
    for img in (port.make_test_image(w, h), rng.integers(0, 256, (h, w, 3), dtype=np.uint8),
                np.full((h, w, 3), 77, np.uint8)):
        out, s_ref = port.carve(img, tw, th, seams=True)
        got, seams, tim = cv.carve(img, tw, th, seams=True, timings=True)
        assert np.array_equal(got, out)
        flat = np.concatenate(seams) if seams else np.zeros(0, np.int32)
        assert np.array_equal(flat, s_ref)
        assert len(tim) == len(seams)


def test_carve_reference_api_contract():
    # test_carver.cpp:117-142, 160-168, 202-210
    g = np.zeros((4, 4, 3), np.uint8)
    for j, v in enumerate([10, 50, 10, 90]):
        g[:, j] = v
    out, rep = cv.carve_to_width(g, 3)
    assert rep.seam_count == 1 and rep.seams[0].tolist() == [1, 1, 1, 1]
    assert np.array_equal(out, g[:, [0, 2, 3]])
    img = cv.make_test_image(24, 16)
    out, rep = cv.carve_to_width(img, 10)
    assert out.shape == (16, 10, 3) and rep.seam_count == 14 and len(rep.per_seam) == 14
    for t, s in enumerate(rep.seams):
        cv.validate_seam(s, 24 - t, 16)
    assert rep.total_s >= sum(x.energy_s + x.solve_s + x.remove_s for x in rep.per_seam)
    out, rep = cv.carve_to_width(img, 24)
    assert np.array_equal(out, img) and rep.seam_count == 0
    for bad in (0, 25):
        with pytest.raises(cv.CarveError) as ei:
            cv.carve_to_width(img, bad)
        assert ei.value.code == cv.Errc.invalid_target
    rng = np.random.default_rng(6)
    g = rng.integers(0, 256, (8, 10, 3), dtype=np.uint8)
    direct = cv.carve_to_height(g, 5)[0]
    sandwich = cv.transpose(cv.carve_to_width(cv.transpose(g), 5)[0])
    assert np.array_equal(direct, sandwich)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_golden(gold, dp_mode, name):
    c = gold["configs"][name]
    img = cv.make_test_image(c["W"], c["H"])
    assert f"{oracle.fnv1a64(img):016x}" == c["input"]
    out, seams, _ = cv.carve(img, c["target_w"], c["target_h"], seams=True)
    assert f"{oracle.fnv1a64(out):016x}" == c["output"]
    assert f"{oracle.fnv1a64(np.concatenate(seams)):016x}" == c["seams"]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_config_golden_full(gold, dp_mode, name):
    c = gold["configs"].get(name)
    if c is None:
        pytest.skip(f"{name} golden not generated")
    img = cv.make_test_image(c["W"], c["H"])
    assert f"{oracle.fnv1a64(img):016x}" == c["input"]
    out, seams, _ = cv.carve(img, c["target_w"], c["target_h"], seams=True)
    assert f"{oracle.fnv1a64(out):016x}" == c["output"]
    assert f"{oracle.fnv1a64(np.concatenate(seams)):016x}" == c["seams"]


def test_batch_golden_sample(gold, dp_mode):
    c = gold["configs"]["C5"]
    ks = [int(k) for k in c["samples"]]
    imgs = [cv.make_test_image(c["W"], c["H"], k) for k in ks]
    outs = cv.carve_batch(imgs, c["target_w"], c["target_h"])
    for k, img, out in zip(ks, imgs, outs):
        assert f"{oracle.fnv1a64(img):016x}" == c["samples"][str(k)]["input"]
        assert f"{oracle.fnv1a64(out):016x}" == c["samples"][str(k)]["output"], k


def test_native_kernels_launched():
    cv.reset_launch_count()
    cv.carve(cv.make_test_image(64, 32), 60)
    # unpack + energy + pad fill + 4 x dp + 3 in-place removals + the last removal fused with the pack
    assert cv.launch_count() == 11


def test_batch_pipelined_chunks_match_oracle(port):
    # >= 2 x 256 images per device takes the copy/compute pipeline (double-buffered
    # chunks on separate copy streams); every image must equal its single carve
    n, w, h, tw, th = 600, 40, 24, 33, 20
    imgs = [port.make_test_image(w, h, k % 37) for k in range(n)]
    outs = cv.carve_batch(imgs, tw, th)
    want = {k: port.carve(imgs[k], tw, th) for k in range(37)}
    for k in range(n):
        assert np.array_equal(outs[k], want[k % 37]), k


def test_batch_unaligned_image_strides(port):
    # 37x23 packed images are 2553 bytes apart and 30x19 outputs 1710 bytes apart:
    # most images start off a 4-byte boundary, which takes the byte-wise side of
    # the 4-pixel RGB<->RGBX conversion, and 4-pixel groups straddle plane rows
    n, w, h, tw, th = 21, 37, 23, 30, 19
    imgs = [port.make_test_image(w, h, k) for k in range(n)]
    outs = cv.carve_batch(imgs, tw, th)
    for k in range(n):
        assert np.array_equal(outs[k], port.carve(imgs[k], tw, th)), k


def test_batch_two_pipelines_match_oracle(port):
    # >= 4 x 256 images per device: two concurrent copy/compute pipelines (their own
    # long-lived contexts and streams) share the device; halves split on a chunk
    # boundary (768 + 332 images here, the second with a ragged last chunk)
    n, w, h, tw, th = 1100, 36, 20, 30, 17
    imgs = [port.make_test_image(w, h, k % 41) for k in range(n)]
    want = {k: port.carve(imgs[k], tw, th) for k in range(41)}
    for _ in range(2):  # the second call reuses the pipeline contexts
        outs = cv.carve_batch(imgs, tw, th)
        for k in range(n):
            assert np.array_equal(outs[k], want[k % 41]), k


@pytest.mark.parametrize("variant", range(17))
def test_every_dp_variant_bitexact(port, monkeypatch, variant):
    """Each DP shape of the variant table (forced with CARVE_DP_VARIANT; the
    default order only reaches some of them at a given width): cost tables and
    seams of a real-valued map, a plane-mode carve and a fused batch carve."""
    monkeypatch.setenv("CARVE_DP_VARIANT", str(variant))
    img = port.make_test_image(500, 77)
    e = port.energy_e1_rgb(img)
    seam, m, b = port.dp_seam(e)
    r = cv.dp_seam(e)
    assert np.array_equal(r.seam, seam)
    assert np.array_equal(bits(r.table.m), bits(m))
    assert np.array_equal(r.table.b, b)
    monkeypatch.setenv("CARVE_DP_GATHER", "0")  # phase 1 over DSMEM (the tall/wide-image path)
    r = cv.dp_seam(e)
    assert np.array_equal(r.seam, seam)
    tall = port.energy_e1_rgb(port.make_test_image(300, 700))
    assert np.array_equal(cv.dp_seam(tall).seam, port.dp_seam(tall)[0])
    monkeypatch.delenv("CARVE_DP_GATHER")
    want = port.carve(img, 480, 70)
    monkeypatch.setenv("CARVE_FUSED", "0")
    assert np.array_equal(cv.carve(img, 480, 70), want)
    monkeypatch.setenv("CARVE_FUSED", "1")
    imgs = [img, port.make_test_image(500, 77, 3)]
    outs = cv.carve_batch(imgs, 480, 70)
    assert np.array_equal(outs[0], want)
    assert np.array_equal(outs[1], port.carve(imgs[1], 480, 70))


@pytest.mark.parametrize("variant", ["0", "8", "12"])
def test_phase1_handoff_carves_match_oracle(port, monkeypatch, variant):
    """Phase 1 with the label table left distributed (CARVE_DP_GATHER=0): the backtrack
    token moves between the cluster's CTAs whenever the seam crosses a 128- or 160-column
    CTA boundary. Whole carves (100 seams, both orientations) against the oracle."""
    monkeypatch.setenv("CARVE_DP_GATHER", "0")
    monkeypatch.setenv("CARVE_DP_VARIANT", variant)
    for k, (w, h, tw, th) in enumerate([(700, 300, 600, 300), (640, 200, 600, 140)]):
        img = port.make_test_image(w, h, k + 5)
        assert np.array_equal(cv.carve(img, tw, th), port.carve(img, tw, th))


def _right_heavy_image(w, h):
    # grey ramp flattening towards the right edge: the last column has the least energy,
    # so seams run down column W-1 (the removal's "nothing moves" case, incl. W-1 = 0 mod 4)
    j = np.arange(w, dtype=np.float64)
    v = np.clip(np.round(255.0 - 0.25 * (w - 1 - j) ** 2), 0, 255).astype(np.uint8)
    return np.repeat(np.repeat(v[None, :, None], h, axis=0), 3, axis=2).copy()


@pytest.mark.parametrize("w", [33, 34, 35, 36, 37, 65])
def test_fused_removal_last_column_seams(port, monkeypatch, w):
    """Seams in the last column keep the RGBX replica column right (the fused DP and the
    forward costs read it); W=33 removes column W-1 with W-1 = 0 mod 4 on the first seam."""
    monkeypatch.setenv("CARVE_FUSED", "1")
    img = _right_heavy_image(w, 12)
    tw = w - 6
    want, want_seams = port.carve(img, tw, 12, seams=True)
    if w == 33:
        assert (want_seams.reshape(-1, 12) == np.arange(w - 1, tw - 1, -1)[:, None]).all()
    outs = cv.carve_batch([img, img[::-1].copy()], tw, 12)
    assert np.array_equal(outs[0], want)
    assert np.array_equal(outs[1], port.carve(img[::-1].copy(), tw, 12))
    out, seams, _ = cv.carve(img, tw, 12, seams=True, forward=True)
    fout, fseams = port.carve_cfg(img, tw, 12, forward=True, seams=True)
    assert np.array_equal(out, fout)
    assert np.array_equal(np.concatenate(seams), fseams)


@pytest.mark.parametrize("split", ["1", "2", "3"])
def test_batch_device_resident_split_matches_oracle(port, monkeypatch, split):
    """carve_batch_device (the bench's device-resident path) on device buffers, with
    the batch split into concurrent sub-batches (CARVE_DEVICE_SPLIT) forked from and
    joined back into the caller's stream."""
    import torch
    monkeypatch.setenv("CARVE_DEVICE_SPLIT", split)
    n, w, h, tw, th = 780, 45, 26, 37, 21  # >= 256 images per sub-batch: 3 sub-batches at most
    imgs = [port.make_test_image(w, h, k % 23) for k in range(n)]
    d_in = torch.from_numpy(np.stack(imgs)).cuda()
    d_out = torch.empty((n, th, tw, 3), dtype=torch.uint8, device="cuda")
    d_out.fill_(7)
    st = torch.cuda.current_stream()
    cv.carve_batch_device(d_in.data_ptr(), n, w, h, tw, th, d_out.data_ptr(), st.cuda_stream)
    st.synchronize()
    outs = d_out.cpu().numpy()
    want = {k: port.carve(imgs[k], tw, th) for k in range(23)}
    for k in range(n):
        assert np.array_equal(outs[k], want[k % 23]), k


def test_remove_seam_planes_golden(golden_dir):
    """remove_seam(LumaGrid / EnergyMap / RemovalMask) = detail::drop_columns
    (carver.hpp:57-112) against the reference-generated api.npz: FP64 bits and
    mask bytes, connected and arbitrary per-row columns."""
    z = np.load(os.path.join(golden_dir, "api.npz"))
    for k in range(int(z["n"])):
        got = cv.remove_seam(z[f"plane{k}"], z[f"seam{k}"])
        want = z[f"want{k}"]
        assert got.dtype == want.dtype and got.shape == want.shape, k
        if want.dtype == np.float64:
            assert np.array_equal(bits(got), bits(want)), k
        else:
            assert np.array_equal(got, want), k


def test_remove_seam_planes_errors():
    for plane in (np.zeros((3, 4)), np.zeros((3, 4), np.uint8)):
        for bad in ([0, 1], [0, 4, 1], [-1, 0, 0]):
            with pytest.raises(cv.CarveError) as ei:
                cv.remove_seam(plane, bad)
            assert ei.value.code == cv.Errc.invalid_seam
    # width 1 -> width 0 (the reference's drop_columns yields an empty grid)
    assert cv.remove_seam(np.ones((5, 1)), [0] * 5).shape == (5, 0)


def test_carve_report_timings_are_device_laps(monkeypatch):
    """SeamTiming (carver.hpp:23-27) from device timestamps: a phase's first seam's
    energy is the K1 map, later seams' the DP prologue's 2-column fix-up; solve is
    the DP, remove the removal kernel. Fused batches compute energy inside the DP."""
    img = cv.make_test_image(300, 200)
    out, seams, tim = cv.carve(img, 280, 190, seams=True, timings=True)
    assert len(tim) == 30
    for t in tim:
        assert t.energy_s > 0 and t.solve_s > 0 and t.remove_s > 0
    _, rep = cv.carve_to_width(img, 290, cv.CarveConfig(forward=True))
    assert all(t.energy_s == 0 and t.solve_s > 0 and t.remove_s > 0 for t in rep.per_seam)
    _, rep = cv.enlarge_to_width(img, 310)
    assert len(rep.per_seam) == 10 and all(t.solve_s > 0 for t in rep.per_seam)


@pytest.mark.parametrize("w,h,tw,th", [(13000, 40, 12995, 37), (18000, 20, 17996, 20), (64, 40000, 60, 40000),
                                       (300, 9000, 296, 9000)])
def test_size_envelope_matches_oracle(port, w, h, tw, th):
    """Beyond the on-chip limits of round 1: widths above 12288 (the 1536-column
    CTA shape), rows wider than a removal slot (the warp-per-row removal), label
    tables larger than shared memory (kept in global memory)."""
    img = port.make_test_image(w, h)
    want, ws = port.carve(img, tw, th, seams=True)
    got, gs, _ = cv.carve(img, tw, th, seams=True)
    assert np.array_equal(got, want)
    assert np.array_equal(np.concatenate(gs), ws)


def test_global_label_table_forced(port, monkeypatch):
    """The global-memory label table (CARVE_DP_GLABELS=1) on ordinary sizes: tables,
    seams and carves identical."""
    monkeypatch.setenv("CARVE_DP_GLABELS", "1")
    e = port.energy_e1_rgb(port.make_test_image(700, 300))
    seam, m, b = port.dp_seam(e)
    r = cv.dp_seam(e)
    assert np.array_equal(r.seam, seam) and np.array_equal(r.table.b, b)
    img = port.make_test_image(260, 140)
    assert np.array_equal(cv.carve(img, 240, 120), port.carve(img, 240, 120))
    imgs = [port.make_test_image(90, 60, k) for k in range(3)]
    for o, x in zip(cv.carve_batch(imgs, 80, 55), imgs):
        assert np.array_equal(o, port.carve(x, 80, 55))
