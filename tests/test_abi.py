"""CPU suite: the C-ABI library loads, exports every symbol include/carve_cuda.h
declares, and its host-side logic (argument validation, error codes, the
fixture generator) behaves like the reference — no kernel launches here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2410_21207_b200 as cv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "carve_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(carve_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(cv.library_path())
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", cv.library_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_make_test_image_matches_oracle():
    for (w, h, k) in [(1, 1, 0), (24, 16, 0), (512, 512, 0), (1024, 768, 3), (77, 5, 1023)]:
        assert np.array_equal(cv.make_test_image(w, h, k), oracle.port().make_test_image(w, h, k))


def test_host_validation_codes():
    assert cv.library().carve_cuda_validate_seam(None, 0, 3, 0) == 0
    cv.validate_seam([0, 1, 2], 3, 3)
    for bad, w, h in [([0, 2], 3, 2), ([0, 3], 3, 2), ([0], 3, 2), ([-1, 0], 3, 2)]:
        with pytest.raises(cv.CarveError) as ei:
            cv.validate_seam(bad, w, h)
        assert ei.value.code == cv.Errc.invalid_seam
    img = np.zeros((4, 4, 3), np.uint8)
    for tw in (0, 5):
        with pytest.raises(cv.CarveError) as ei:
            cv.carve_to_width(img, tw)
        assert ei.value.code == cv.Errc.invalid_target
    for th in (0, 5):
        with pytest.raises(cv.CarveError) as ei:
            cv.carve_to_height(img, th)
        assert ei.value.code == cv.Errc.invalid_target


def test_unsupported_paths_fail_loudly():
    img = np.zeros((4, 4, 3), np.uint8)
    with pytest.raises(cv.CarveError) as ei:
        cv.carve_to_width(img, 3, cv.CarveConfig(solver=cv.SolverKind.Greedy))
    assert ei.value.code == cv.Errc.usage_error
    with pytest.raises(cv.CarveError) as ei:
        cv.carve_to_width(img, 3, cv.CarveConfig(solver=cv.SolverKind.Greedy, forward=True))
    assert ei.value.code == cv.Errc.usage_error
    with pytest.raises(cv.CarveError) as ei:
        cv.compute_energy(np.zeros((3, 3)), cv.EnergyFn.hog)
    assert ei.value.code == cv.Errc.usage_error


@pytest.mark.skipif(cv.device_count() > 0, reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(cv.CarveError) as ei:
        cv.carve(np.zeros((4, 4, 3), np.uint8), 3)
    assert ei.value.code == cv.Errc.device_failure
    with pytest.raises(cv.CarveError) as ei:
        cv.dp_seam(np.zeros((3, 3)))
    assert ei.value.code == cv.Errc.device_failure


def test_missing_library_raises(tmp_path, monkeypatch):
    import importlib

    mod = importlib.reload(cv)
    monkeypatch.setattr(mod, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(mod, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mod.library()
    importlib.reload(cv)


def test_batch_plan_host_logic(monkeypatch):
    """carve_batch's pipeline shape (SURVEY.md §8e work queue): chunks never
    exceed the per-device share, and the env overrides are read per call."""
    for n, ndev in [(1, 1), (6, 2), (128, 1), (256, 1), (1024, 1), (1024, 8), (1025, 4), (5000, 3)]:
        p, ch = cv.batch_plan(n, 1024, 768, 896, 768, ndev)
        share = -(-n // ndev)
        assert 1 <= ch <= share and 1 <= p <= 4
        assert p <= -(-share // ch)
    # the measured default shape (profiles/r02_share_grid_b.txt): 4 pipelines, quarter-share
    # chunks up to 128 images, at least 16
    assert [cv.batch_plan(n, 1024, 768, 896, 768, nd) for n, nd in [(1024, 1), (256, 1), (128, 1), (1024, 8)]] == \
        [(4, 128), (4, 64), (4, 32), (4, 32)]
    assert cv.batch_plan(20, 1024, 768, 896, 768, 1) == (2, 16)
    monkeypatch.setenv("CARVE_PIPE_CHUNK", "16")
    monkeypatch.setenv("CARVE_PIPELINES", "3")
    assert cv.batch_plan(1025, 64, 48, 56, 48, 2) == (3, 16)
    assert cv.batch_plan(20, 64, 48, 56, 48, 2) == (1, 10)
    for bad in [(0, 8, 8, 8, 8, 1), (4, 8, 8, 9, 8, 1), (4, 8, 8, 8, 8, 0)]:
        with pytest.raises(cv.CarveError):
            cv.batch_plan(*bad)
