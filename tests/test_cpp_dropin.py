"""The C++ drop-in surface: include/carve/*.hpp (through tools/carve_parity.cpp)
and the `carve resize` CLI (tools/carve_main.cpp), mirroring the reference's
CLI tests (tests/test_cli.cpp) and acceptance criterion 9 (acceptance.cpp:288-301)."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CARVE = os.path.join(ROOT, "build", "carve")
PARITY = os.path.join(ROOT, "build", "carve_parity")


@pytest.fixture(scope="module", autouse=True)
def tools_built():
    if not (os.path.exists(CARVE) and os.path.exists(PARITY)):
        subprocess.run(["make", "-s", "-C", ROOT, "tools"], check=True)


def write_ppm(path, img):
    h, w, _ = img.shape
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(np.ascontiguousarray(img).tobytes())


def read_ppm(path):
    data = open(path, "rb").read()
    parts = data.split(maxsplit=4)
    assert parts[0] == b"P6"
    w, h = int(parts[1]), int(parts[2])
    return np.frombuffer(parts[4][: w * h * 3], np.uint8).reshape(h, w, 3)


def run(*args, env=None):
    return subprocess.run([CARVE, *args], capture_output=True, text=True, env=env)


# ---- host-only behaviour (no GPU needed) ---------------------------------------------
def test_cli_usage_errors_exit_1(tmp_path):
    assert run().returncode == 1
    assert run("resize", "--input", "a.ppm").returncode == 1  # missing --output
    assert run("resize", "--input", "a", "--output", "b", "--scale", "0").returncode == 1
    assert run("resize", "--input", "a", "--output", "b", "--scale", "0.5", "--width", "3").returncode == 1
    assert run("enlarge", "--input", "a").returncode == 1  # missing --output
    assert run("seams", "--input", "a", "--output", "b").returncode == 1  # --count is required
    assert run("seams", "--input", "a", "--output", "b", "--count", "0").returncode == 1
    assert run("remove-object", "--input", "a", "--output", "b").returncode == 1
    r = run("resize", "--input", "a", "--output", "b", "--solver", "quantum")
    assert r.returncode == 1 and "carve:" in r.stderr


def test_cli_energy_usage_errors_exit_1(tmp_path):
    # cli.hpp:184-187, 288-291: --energy required, output must be .png, e1 only on the B200 path
    p = tmp_path / "a.ppm"
    write_ppm(p, np.zeros((4, 4, 3), np.uint8))
    assert run("energy", "--input", str(p), "--output", str(tmp_path / "o.png")).returncode == 1
    assert run("energy", "--input", str(p), "--output", str(tmp_path / "o.ppm"), "--energy", "e1").returncode == 1
    assert run("energy", "--input", str(p), "--output", str(tmp_path / "o.png"), "--energy", "x").returncode == 1
    assert run("energy", "--input", str(p), "--output", str(tmp_path / "o.png"), "--energy", "e1",
               "--scale", "0.5").returncode == 1


def read_png_gray(path):
    import struct
    import zlib
    data = open(path, "rb").read()
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat, w, h = 8, b"", None, None
    while pos < len(data):
        n, kind = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + n]
        if kind == b"IHDR":
            w, h, depth, ctype = struct.unpack(">IIBB", body[:10])
            assert depth == 8 and ctype == 0
        elif kind == b"IDAT":
            idat += body
        pos += 12 + n
    raw = zlib.decompress(idat)
    out, prev = np.zeros((h, w), np.uint8), np.zeros(w, np.int32)
    for i in range(h):
        f, row = raw[i * (w + 1)], np.frombuffer(raw[i * (w + 1) + 1:(i + 1) * (w + 1)], np.uint8).astype(np.int32)
        cur = np.zeros(w, np.int32)
        for j in range(w):
            a = cur[j - 1] if j else 0
            b, c = prev[j], (prev[j - 1] if j else 0)
            pred = {0: 0, 1: a, 2: b, 3: (a + b) // 2}.get(f)
            if f == 4:
                pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                pred = a if pa <= pb and pa <= pc else (b if pb <= pc else c)
            cur[j] = (row[j] + pred) & 255
        out[i], prev = cur, cur
    return out


@pytest.mark.gpu
def test_cli_energy_matches_oracle(tmp_path):
    """`carve energy` (cli.hpp:288-299): normalize_to_gray(e1) as an 8-bit gray PNG."""
    img = oracle.port().make_test_image(67, 41)
    src = tmp_path / "in.ppm"
    write_ppm(src, img)
    r = run("energy", "--input", str(src), "--output", str(tmp_path / "e.png"), "--energy", "e1")
    assert r.returncode == 0, r.stderr
    e = oracle.port().energy_e1_rgb(img)
    lo, hi = e.min(), e.max()
    want = np.floor((e - lo) / (hi - lo) * 255.0 + 0.5).astype(np.uint8)  # std::lround, non-negative
    assert np.array_equal(read_png_gray(tmp_path / "e.png"), want)
    r = run("energy", "--input", str(src), "--output", str(tmp_path / "h.png"), "--energy", "hog")
    assert r.returncode == 1 and "not supported" in r.stderr


def test_cli_runtime_errors_exit_2(tmp_path):
    r = run("resize", "--input", str(tmp_path / "missing.ppm"), "--output", str(tmp_path / "o.ppm"), "--scale", "0.5")
    assert r.returncode == 2 and "no such file" in r.stderr
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(b"P3\n1 1\n255\n0 0 0\n")
    assert run("resize", "--input", str(bad), "--output", str(tmp_path / "o.ppm"), "--scale", "0.5").returncode == 2


def test_cli_bad_workers_env(tmp_path):
    p = tmp_path / "a.ppm"
    write_ppm(p, np.zeros((4, 4, 3), np.uint8))
    env = dict(os.environ, CARVE_WORKERS="-3")
    assert run("resize", "--input", str(p), "--output", str(tmp_path / "o.ppm"), "--scale", "0.5", env=env).returncode == 1


# ---- through the GPU ----------------------------------------------------------------------
@pytest.mark.gpu
def test_cpp_headers_selftest():
    r = subprocess.run([PARITY, "selftest"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_cpp_headers_golden(name):
    c = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"][name]
    r = subprocess.run([PARITY, "hash", str(c["W"]), str(c["H"]), str(c["target_w"]), str(c["target_h"])],
                       capture_output=True, text=True, check=True)
    assert r.stdout.split() == [c["input"], c["output"], c["seams"]]


@pytest.mark.gpu
def test_cli_resize_matches_oracle_and_is_worker_invariant(tmp_path):
    # acceptance criterion 9: byte-identical output for CARVE_WORKERS=1 and =8
    img = oracle.port().make_test_image(180, 180)
    src = tmp_path / "in.ppm"
    write_ppm(src, img)
    outs = []
    for workers in ("1", "8"):
        dst = tmp_path / f"out{workers}.ppm"
        env = dict(os.environ, CARVE_WORKERS=workers)
        r = run("resize", "--input", str(src), "--output", str(dst), "--scale", "0.5", "--height", "150",
                "--solver", "pardp", env=env)
        assert r.returncode == 0, r.stderr
        outs.append(dst.read_bytes())
    assert outs[0] == outs[1]
    want = oracle.port().carve(img, 90, 150)
    assert np.array_equal(read_ppm(tmp_path / "out1.ppm"), want)


@pytest.mark.gpu
def test_cli_enlarge_and_seams_match_oracle(tmp_path):
    # cli.hpp:262-277 (enlarge) and :301-309 (seams); test_cli.cpp:185-188
    port = oracle.port()
    img = port.make_test_image(40, 30)
    src = tmp_path / "in.ppm"
    write_ppm(src, img)
    r = run("enlarge", "--input", str(src), "--output", str(tmp_path / "e.ppm"), "--width", "55", "--height", "41")
    assert r.returncode == 0, r.stderr
    assert np.array_equal(read_ppm(tmp_path / "e.ppm"), port.enlarge(img, 55, 41))
    r = run("enlarge", "--input", str(src), "--output", str(tmp_path / "e2.ppm"), "--scale", "1.25")
    assert r.returncode == 0, r.stderr
    assert np.array_equal(read_ppm(tmp_path / "e2.ppm"), port.enlarge(img, 50, 30))
    r = run("enlarge", "--input", str(src), "--output", str(tmp_path / "e3.ppm"), "--width", "80")
    assert r.returncode == 2 and "2*width-1" in r.stderr  # target_too_large is a runtime error
    r = run("seams", "--input", str(src), "--output", str(tmp_path / "s.ppm"), "--count", "5")
    assert r.returncode == 0, r.stderr
    want = img.copy()
    for seam in port.record_seams(img, 5):
        want[np.arange(30), seam] = (255, 0, 0)
    assert np.array_equal(read_ppm(tmp_path / "s.ppm"), want)


@pytest.mark.gpu
def test_cli_remove_object_matches_oracle(tmp_path):
    # cli.hpp:279-287: mask_from_image of --mask, remove_object, optional --no-restore
    port = oracle.port()
    img = port.make_test_image(48, 36)
    mimg = np.zeros((36, 48, 3), np.uint8)
    mimg[10:20, 20:26] = 255
    write_ppm(tmp_path / "in.ppm", img)
    write_ppm(tmp_path / "m.ppm", mimg)
    mask = port.mask_from_image(mimg)
    for extra, restore in (([], True), (["--no-restore"], False)):
        out = tmp_path / f"o{int(restore)}.ppm"
        r = run("remove-object", "--input", str(tmp_path / "in.ppm"), "--mask", str(tmp_path / "m.ppm"),
                "--output", str(out), *extra)
        assert r.returncode == 0, r.stderr
        assert np.array_equal(read_ppm(out), port.remove_object(img, mask, False, restore)[0])


@pytest.mark.gpu
def test_cli_resize_png_in_png_out(tmp_path):
    # raster.hpp:128-146 load_image / save_image with PNG on both ends
    img = oracle.port().make_test_image(64, 48)
    ppm = tmp_path / "in.ppm"
    write_ppm(ppm, img)
    subprocess.run([PARITY, "convert", str(ppm), str(tmp_path / "in.png")], check=True)
    r = run("resize", "--input", str(tmp_path / "in.png"), "--output", str(tmp_path / "out.png"), "--width", "50",
            "--height", "40")
    assert r.returncode == 0, r.stderr
    subprocess.run([PARITY, "convert", str(tmp_path / "out.png"), str(tmp_path / "out.ppm")], check=True)
    assert np.array_equal(read_ppm(tmp_path / "out.ppm"), oracle.port().carve(img, 50, 40))
