"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the CPU checkers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product
(``paper_2410_21207_b200``) never imports it and has no CPU fallback.

Two checkers, same numpy-level API:

* ``port()``      — ``build/liboracle.so``, the C restatement in
  ``carve_oracle.c`` (each function cites the reference file:line it follows).
* ``reference()`` — ``_ref/libcarve_ref.so``, the reference headers under
  ``/root/reference/proj/include`` compiled unmodified through ``ref_shim.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcarve_ref.so")

_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_f8p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i4p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def build() -> None:
    """Compile the checkers (the reference leg only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Checker:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.path = path

    def _fn(self, name, *argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = list(argtypes)
        f.restype = restype
        return f

    def _check(self, st: int) -> None:
        if st:
            raise OracleError(st, self.last_error())

    def last_error(self) -> str:
        return ""

    # -- shared numpy API ------------------------------------------------
    def to_grayscale(self, img: np.ndarray) -> np.ndarray:
        h, w, _ = img.shape
        out = np.empty((h, w), np.float64)
        self._check(self._fn("to_grayscale", _u8p, C.c_int, C.c_int, _f8p)(np.ascontiguousarray(img), w, h, out))
        return out

    def energy_e1_luma(self, luma: np.ndarray) -> np.ndarray:
        h, w = luma.shape
        out = np.empty((h, w), np.float64)
        self._check(self._fn("energy_e1_luma", _f8p, C.c_int, C.c_int, _f8p)(np.ascontiguousarray(luma, np.float64), w, h, out))
        return out

    def energy_e1_rgb(self, img: np.ndarray) -> np.ndarray:
        h, w, _ = img.shape
        out = np.empty((h, w), np.float64)
        self._check(self._fn("energy_e1_rgb", _u8p, C.c_int, C.c_int, _f8p)(np.ascontiguousarray(img), w, h, out))
        return out

    def transpose(self, img: np.ndarray) -> np.ndarray:
        h, w, _ = img.shape
        out = np.empty((w, h, 3), np.uint8)
        self._check(self._fn("transpose", _u8p, C.c_int, C.c_int, _u8p)(np.ascontiguousarray(img), w, h, out))
        return out


    def forward_costs(self, luma: np.ndarray):
        """energy.hpp:196-216 -> (left, up, right)"""
        h, w = luma.shape
        outs = [np.empty((h, w), np.float64) for _ in range(3)]
        self._check(self._fn("forward_costs", _f8p, C.c_int, C.c_int, _f8p, _f8p, _f8p)(
            np.ascontiguousarray(luma, np.float64), w, h, *outs))
        return tuple(outs)

    def dp_seam_forward(self, luma: np.ndarray):
        """solvers.hpp:294-326 with forward_costs(luma) -> (seam, m, b)"""
        h, w = luma.shape
        m = np.empty((h, w), np.float64)
        b = np.empty((h, w), np.int32)
        seam = np.empty(h, np.int32)
        self._check(self._fn("dp_seam_forward", _f8p, C.c_int, C.c_int, _f8p, _i4p, _i4p)(
            np.ascontiguousarray(luma, np.float64), w, h, m, b, seam))
        return seam, m, b

    def dp_seam_forward_costs(self, cl: np.ndarray, cu: np.ndarray, cr: np.ndarray):
        """solvers.hpp:294-326 with arbitrary costs -> (seam, m, b)"""
        h, w = cl.shape
        m = np.empty((h, w), np.float64)
        b = np.empty((h, w), np.int32)
        seam = np.empty(h, np.int32)
        self._check(self._fn("dp_seam_forward_costs", _f8p, _f8p, _f8p, C.c_int, C.c_int, _f8p, _i4p, _i4p)(
            *(np.ascontiguousarray(x, np.float64) for x in (cl, cu, cr)), w, h, m, b, seam))
        return seam, m, b

    def carve_cfg(self, img: np.ndarray, target_w: int, target_h: int | None = None, forward: bool = False,
                  recompute: bool = True, seams: bool = False):
        """run_resize with CarveConfig::forward / ::recompute"""
        h, w, _ = img.shape
        th = h if target_h is None else target_h
        out = np.empty((th, target_w, 3), np.uint8)
        n = (w - target_w) * h + (h - th) * target_w
        s = np.empty(max(n, 1), np.int32)
        f = self._fn("carve_cfg", _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p)
        self._check(f(np.ascontiguousarray(img), w, h, target_w, th, int(forward), int(recompute), out, s.ctypes.data))
        return (out, s[:n]) if seams else out

    def apply_mask(self, e: np.ndarray, mask: np.ndarray) -> np.ndarray:
        """energy.hpp:220-241"""
        h, w = e.shape
        out = np.empty((h, w), np.float64)
        self._check(self._fn("apply_mask", _f8p, C.c_int, C.c_int, _u8p, _f8p)(
            np.ascontiguousarray(e, np.float64), w, h, np.ascontiguousarray(mask, np.uint8), out))
        return out

    def mask_from_image(self, img: np.ndarray) -> np.ndarray:
        """energy.hpp:244-253"""
        h, w, _ = img.shape
        out = np.empty((h, w), np.uint8)
        self._check(self._fn("mask_from_image", _u8p, C.c_int, C.c_int, _u8p)(np.ascontiguousarray(img), w, h, out))
        return out

    def remove_object(self, img: np.ndarray, mask: np.ndarray, forward: bool = False, restore: bool = True):
        """carver.hpp:327-340 -> (result, seams list)"""
        h, w, _ = img.shape
        out = np.empty(w * h * 3, np.uint8)
        dims = np.zeros(2, np.int32)
        seams = np.zeros(max(w * h, 1), np.int32)
        n = np.zeros(1, np.int32)
        f = self._fn("remove_object", _u8p, C.c_int, C.c_int, _u8p, C.c_int, C.c_int, _u8p, _i4p, _i4p, _i4p)
        self._check(f(np.ascontiguousarray(img), w, h, np.ascontiguousarray(mask, np.uint8), int(forward),
                      int(restore), out, dims, seams, n))
        ow, oh = int(dims[0]), int(dims[1])
        res = out[: ow * oh * 3].reshape(oh, ow, 3).copy()
        return res, seams, int(n[0])

    def insert_seam(self, img: np.ndarray, seam) -> np.ndarray:
        """carver.hpp:137-140"""
        h, w, _ = img.shape
        s = np.ascontiguousarray(seam, np.int32)
        out = np.empty((h, w + 1, 3), np.uint8)
        self._check(self._fn("insert_seam", _u8p, C.c_int, C.c_int, _i4p, C.c_int, _u8p)(
            np.ascontiguousarray(img), w, h, s, len(s), out))
        return out

    def record_seams(self, img: np.ndarray, count: int) -> np.ndarray:
        """carver.hpp:226-262: (count, h) original-coordinate columns."""
        h, w, _ = img.shape
        out = np.empty((max(count, 0), h), np.int32)
        self._check(self._fn("record_seams", _u8p, C.c_int, C.c_int, C.c_int, C.c_void_p)(
            np.ascontiguousarray(img), w, h, count, out.ctypes.data))
        return out

    def enlarge(self, img: np.ndarray, target_w: int, target_h: int | None = None, seams: bool = False):
        """run_enlarge (cli.hpp:262-277): enlarge_to_width on the width, then on the transpose."""
        h, w, _ = img.shape
        th = h if target_h is None else target_h
        out = np.empty((th, target_w, 3), np.uint8)
        n = max(target_w - w, 0) * h + max(th - h, 0) * target_w
        s = np.empty(max(n, 1), np.int32)
        f = self._fn("enlarge", _u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p)
        self._check(f(np.ascontiguousarray(img), w, h, target_w, th, out, s.ctypes.data))
        return (out, s[:n]) if seams else out


class Port(_Checker):
    """The C restatement (carve_oracle.c)."""

    prefix = "or_"

    def remove_seam_plane(self, plane: np.ndarray, seam) -> np.ndarray:
        """carver.hpp:57-67, 84-112: a float64 (LumaGrid/EnergyMap) or uint8 (RemovalMask) plane."""
        a = np.ascontiguousarray(plane)
        h, w = a.shape
        s = np.ascontiguousarray(seam, np.int32)
        out = np.empty((h, max(w - 1, 0)), a.dtype)
        f = self._fn("drop_columns", C.c_void_p, C.c_int, C.c_int, _i4p, C.c_int, C.c_int, C.c_void_p)
        self._check(f(a.ctypes.data, w, h, s, len(s), a.dtype.itemsize, out.ctypes.data))
        return out

    def make_test_image(self, w: int, h: int, variant: int = 0) -> np.ndarray:
        out = np.empty((h, w, 3), np.uint8)
        self._check(self._fn("make_test_image", C.c_int, C.c_int, C.c_uint32, _u8p)(w, h, variant, out))
        return out

    def dp_seam(self, e: np.ndarray, table: bool = True):
        h, w = e.shape
        m = np.empty((h, w), np.float64) if table else None
        b = np.empty((h, w), np.int32) if table else None
        seam = np.empty(h, np.int32)
        f = self._fn("dp_seam", _f8p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, _i4p)
        self._check(f(np.ascontiguousarray(e, np.float64), w, h,
                      m.ctypes.data if table else None, b.ctypes.data if table else None, seam))
        return seam, m, b

    def validate_seam(self, seam, w: int, h: int) -> int:
        s = np.ascontiguousarray(seam, np.int32)
        return self._fn("validate_seam", _i4p, C.c_int, C.c_int, C.c_int)(s, len(s), w, h)

    def remove_seam(self, img: np.ndarray, seam) -> np.ndarray:
        h, w, _ = img.shape
        s = np.ascontiguousarray(seam, np.int32)
        out = np.empty((h, max(w - 1, 0), 3), np.uint8)
        self._check(self._fn("remove_seam", _u8p, C.c_int, C.c_int, _i4p, C.c_int, C.c_void_p)(
            np.ascontiguousarray(img), w, h, s, len(s), out.ctypes.data))
        return out

    def carve(self, img: np.ndarray, target_w: int, target_h: int | None = None, seams: bool = False):
        h, w, _ = img.shape
        th = h if target_h is None else target_h
        out = np.empty((th, target_w, 3), np.uint8)
        n_seam_ints = (w - target_w) * h + (h - th) * target_w
        s = np.empty(max(n_seam_ints, 1), np.int32) if seams else None
        f = self._fn("carve", _u8p, C.c_int, C.c_int, C.c_int, C.c_int, _u8p, C.c_void_p)
        self._check(f(np.ascontiguousarray(img), w, h, target_w, th, out, s.ctypes.data if seams else None))
        return (out, s[:n_seam_ints]) if seams else out

    def fnv1a64(self, buf: np.ndarray) -> int:
        b = np.ascontiguousarray(buf).view(np.uint8).ravel()
        return int(self._fn("fnv1a64", _u8p, C.c_size_t, restype=C.c_uint64)(b, b.size))


class Reference(_Checker):
    """The unmodified reference, compiled from /root/reference (ref_shim.cpp)."""

    prefix = "ref_"

    def remove_seam_plane(self, plane: np.ndarray, seam, kind: str = "energy") -> np.ndarray:
        """remove_seam(LumaGrid) (kind "luma"), (EnergyMap) ("energy") or (RemovalMask) (uint8 plane)."""
        a = np.ascontiguousarray(plane)
        h, w = a.shape
        s = np.ascontiguousarray(seam, np.int32)
        out = np.empty((h, max(w - 1, 0)), a.dtype)
        if a.dtype == np.uint8:
            f = self._fn("remove_seam_u8", _u8p, C.c_int, C.c_int, _i4p, C.c_int, C.c_void_p)
            self._check(f(a, w, h, s, len(s), out.ctypes.data))
        else:
            f = self._fn("remove_seam_f64", _f8p, C.c_int, C.c_int, _i4p, C.c_int, C.c_int, C.c_void_p)
            self._check(f(a, w, h, s, len(s), 0 if kind == "luma" else 1, out.ctypes.data))
        return out

    def remove_object_vertical(self, img: np.ndarray, mask: np.ndarray, restore: bool = True):
        """carver.hpp:289-321 detail::remove_object_vertical -> (result, seams, count)"""
        h, w, _ = img.shape
        out = np.empty(w * h * 3, np.uint8)
        dims = np.zeros(2, np.int32)
        seams = np.zeros(max(w * h, 1), np.int32)
        n = np.zeros(1, np.int32)
        f = self._fn("remove_object_vertical", _u8p, C.c_int, C.c_int, _u8p, C.c_int, _u8p, _i4p, _i4p, _i4p)
        self._check(f(np.ascontiguousarray(img), w, h, np.ascontiguousarray(mask, np.uint8), int(restore), out, dims,
                      seams, n))
        ow, oh = int(dims[0]), int(dims[1])
        return out[: ow * oh * 3].reshape(oh, ow, 3).copy(), seams[: int(n[0]) * h], int(n[0])

    def bench_record(self, img: np.ndarray, full: bool, scale: float = 1.0, forward: bool = False, reps: int = 1):
        """BenchRecord fields of time_full_carve / time_single_seam (bench.hpp:140-201)."""
        h, w, _ = img.shape
        out = np.zeros(5, np.int32)
        sc = np.zeros(1, np.float64)
        f = self._fn("bench_record", _u8p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _i4p, _f8p)
        self._check(f(np.ascontiguousarray(img), w, h, int(full), scale, int(forward), reps, out, sc))
        return {"solver": int(out[0]), "n": int(out[1]), "phase": int(out[2]),
                "scale": float(sc[0]) if out[3] else None, "repetitions": int(out[4])}

    def last_error(self) -> str:
        return self._fn("last_error", restype=C.c_char_p)().decode()

    def hardware_concurrency(self) -> int:
        return int(self._fn("hardware_concurrency", restype=C.c_uint)())

    def make_test_image(self, w: int, h: int) -> np.ndarray:
        out = np.empty((h, w, 3), np.uint8)
        self._check(self._fn("make_test_image", C.c_int, C.c_int, _u8p)(w, h, out))
        return out

    def dp_seam(self, e: np.ndarray, solver: int = 0, workers: int = 0):
        h, w = e.shape
        m = np.empty((h, w), np.float64)
        b = np.empty((h, w), np.int32)
        seam = np.empty(h, np.int32)
        f = self._fn("dp_seam", _f8p, C.c_int, C.c_int, C.c_int, C.c_uint, _f8p, _i4p, _i4p)
        self._check(f(np.ascontiguousarray(e, np.float64), w, h, solver, workers, m, b, seam))
        return seam, m, b

    def validate_seam(self, seam, w: int, h: int) -> int:
        s = np.ascontiguousarray(seam, np.int32)
        return self._fn("validate_seam", _i4p, C.c_int, C.c_int, C.c_int)(s, len(s), w, h)

    def remove_seam(self, img: np.ndarray, seam) -> np.ndarray:
        h, w, _ = img.shape
        s = np.ascontiguousarray(seam, np.int32)
        out = np.empty((h, max(w - 1, 0), 3), np.uint8)
        self._check(self._fn("remove_seam", _u8p, C.c_int, C.c_int, _i4p, C.c_int, C.c_void_p)(
            np.ascontiguousarray(img), w, h, s, len(s), out.ctypes.data))
        return out

    def carve(self, img: np.ndarray, target_w: int, target_h: int | None = None, solver: int = 0,
              workers: int = 0, seams: bool = False):
        h, w, _ = img.shape
        th = h if target_h is None else target_h
        out = np.empty((th, target_w, 3), np.uint8)
        n_seam_ints = (w - target_w) * h + (h - th) * target_w
        s = np.empty(max(n_seam_ints, 1), np.int32) if seams else None
        times = np.zeros(2, np.float64)
        f = self._fn("carve", _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint, _u8p, C.c_void_p, _f8p)
        self._check(f(np.ascontiguousarray(img), w, h, target_w, th, solver, workers, out,
                      s.ctypes.data if seams else None, times))
        return (out, s[:n_seam_ints]) if seams else out

    def carve_batch(self, imgs: list[np.ndarray], target_w: int, threads: int, solver: int = 0,
                    workers: int = 1) -> list[np.ndarray]:
        n = len(imgs)
        h, w, _ = imgs[0].shape
        ins = [np.ascontiguousarray(x) for x in imgs]
        outs = [np.empty((h, target_w, 3), np.uint8) for _ in range(n)]
        in_ptrs = (C.c_void_p * n)(*[x.ctypes.data for x in ins])
        out_ptrs = (C.c_void_p * n)(*[x.ctypes.data for x in outs])
        f = self._fn("carve_batch", C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint, C.c_uint, C.c_void_p)
        self._check(f(in_ptrs, n, w, h, target_w, solver, workers, threads, out_ptrs))
        return outs


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port(PORT_SO)
    return _port


def reference() -> Reference:
    global _ref
    if _ref is None:
        _ref = Reference(REF_SO)
    return _ref


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def fnv1a64(buf: np.ndarray) -> int:
    """FNV-1a-64 (offset 0xcbf29ce484222325, prime 0x100000001b3), SURVEY.md §8c."""
    return port().fnv1a64(buf)
