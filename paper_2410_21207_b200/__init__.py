"""B200-native seam carving (arXiv 2410.21207 DP path) — Python host mirror.

Every function here mirrors a reference entry point in
/root/reference/proj/include/carve/ (same name, argument meaning and error
behaviour) and runs on the GPU through the C ABI of ``libcarve_cuda.so``
(``include/carve_cuda.h``). There is no CPU fallback: if the library is
missing, importing a compute function raises; if no sm_100 device is present,
calls raise ``CarveError`` with code ``Errc.device_failure``.

Images are numpy ``uint8`` arrays of shape (H, W, 3) — the row-major packed
``PixelGrid`` (raster.hpp:28-42). Luma/energy maps are (H, W) float64 arrays
(``LumaGrid``/``EnergyMap``, raster.hpp:45-59, energy.hpp:16-23).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Errc", "CarveError", "SolverKind", "EnergyFn", "CarveConfig", "SolverOptions", "SeamTiming",
    "CarveReport", "CostTable", "SeamResult", "make_test_image", "to_grayscale", "energy_e1", "compute_energy",
    "energy_e1_rgb", "dp_seam", "parallel_dp_seam", "find_seam", "validate_seam", "remove_seam", "transpose",
    "carve_to_width", "carve_to_height", "carve", "carve_batch", "carve_device", "carve_batch_device",
    "insert_seam", "record_seams", "enlarge_to_width", "enlarge", "forward_costs", "dp_seam_forward",
    "apply_mask", "mask_from_image", "mask_bounds", "remove_object",
    "library", "library_path", "device_count", "launch_count", "reset_launch_count",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CARVE_LIB") or os.path.join(HERE, "libcarve_cuda.so")


class Errc(enum.IntEnum):
    """error.hpp:8-26 (ordinal + 1 as returned by the C ABI), plus device failure."""
    file_not_found = 1
    unsupported_format = 2
    corrupt_image = 3
    io_failure = 4
    dimension_mismatch = 5
    invalid_seam = 6
    image_too_large = 7
    empty_image = 8
    width_too_small = 9
    invalid_target = 10
    target_too_large = 11
    empty_mask = 12
    insufficient_data = 13
    size_exceeds_source = 14
    solver_cap_violated = 15
    empty_input = 16
    usage_error = 17
    device_failure = 100


class CarveError(RuntimeError):
    """carve::Error (error.hpp:28-35): carries the Errc code."""

    def __init__(self, code: int, what: str):
        super().__init__(what)
        try:
            self.code = Errc(code)
        except ValueError:
            self.code = Errc.device_failure


class SolverKind(enum.Enum):  # solvers.hpp:21
    BruteForce = "bruteforce"
    Greedy = "greedy"
    Dynamic = "dp"
    ParallelDynamic = "pardp"


class EnergyFn(enum.Enum):  # energy.hpp:52
    e1 = "e1"
    e2 = "e2"
    hog = "hog"
    entropy = "entropy"


@dataclass
class SolverOptions:  # solvers.hpp:64-67
    brute_cap: int = 16
    workers: int = 0  # accepted for drop-in compatibility; never changes output


@dataclass
class CarveConfig:  # carver.hpp:15-21
    solver: SolverKind = SolverKind.ParallelDynamic
    energy_fn: EnergyFn = EnergyFn.e1
    forward: bool = False
    recompute: bool = True
    solver_opts: SolverOptions = field(default_factory=SolverOptions)


@dataclass
class SeamTiming:  # carver.hpp:23-27
    energy_s: float = 0.0
    solve_s: float = 0.0
    remove_s: float = 0.0


@dataclass
class CarveReport:  # carver.hpp:29-34
    seam_count: int = 0
    per_seam: list = field(default_factory=list)
    seams: list = field(default_factory=list)
    total_s: float = 0.0


@dataclass
class CostTable:  # solvers.hpp:42-55
    width: int
    height: int
    m: np.ndarray  # (H, W) float64 accumulated minimum costs
    b: np.ndarray  # (H, W) int32 predecessor columns

    def cost(self, row: int, col: int) -> float:
        return float(self.m[row, col])

    def back(self, row: int, col: int) -> int:
        return int(self.b[row, col])

    def __eq__(self, other) -> bool:  # operator== compares m and b exactly (:54)
        return (isinstance(other, CostTable) and self.width == other.width and self.height == other.height
                and np.array_equal(self.m.view(np.uint64), other.m.view(np.uint64))
                and np.array_equal(self.b, other.b))


@dataclass
class SeamResult:  # solvers.hpp:57-60
    seam: np.ndarray
    table: CostTable


class _Timing(C.Structure):
    _fields_ = [("energy_s", C.c_double), ("solve_s", C.c_double), ("remove_s", C.c_double)]


_lib = None
_u8p = C.POINTER(C.c_uint8)


def library_path() -> str:
    return LIB_PATH


def library() -> C.CDLL:
    """Load libcarve_cuda.so (in-tree build). Raises if it was not built —
    there is deliberately no fallback implementation."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                               "the B200 engine has no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        vp, i = C.c_void_p, C.c_int
        sigs = {
            "carve_cuda_last_error": ([], C.c_char_p),
            "carve_cuda_version": ([], C.c_char_p),
            "carve_cuda_device_count": ([], i),
            "carve_cuda_set_device": ([i], i),
            "carve_cuda_launch_count": ([], C.c_uint64),
            "carve_cuda_reset_launch_count": ([], None),
            "carve_cuda_to_grayscale": ([vp, i, i, vp], i),
            "carve_cuda_energy_e1_rgb": ([vp, i, i, vp], i),
            "carve_cuda_energy_e1_luma": ([vp, i, i, vp], i),
            "carve_cuda_transpose_rgb": ([vp, i, i, vp], i),
            "carve_cuda_dp_seam": ([vp, i, i, vp, vp, vp], i),
            "carve_cuda_validate_seam": ([vp, i, i, i], i),
            "carve_cuda_remove_seam_rgb": ([vp, i, i, vp, i, vp], i),
            "carve_cuda_insert_seam_rgb": ([vp, i, i, vp, i, vp], i),
            "carve_cuda_record_seams": ([vp, i, i, i, vp, vp, vp], i),
            "carve_cuda_enlarge": ([vp, i, i, i, i, vp, vp, vp], i),
            "carve_cuda_enlarge_timed": ([vp, i, i, i, i, vp, vp, vp, vp], i),
            "carve_cuda_carve": ([vp, i, i, i, i, vp, vp, vp], i),
            "carve_cuda_carve_cfg": ([vp, i, i, i, i, vp, vp, vp, vp], i),
            "carve_cuda_forward_costs": ([vp, i, i, vp, vp, vp], i),
            "carve_cuda_mask_from_rgb": ([vp, i, i, vp], i),
            "carve_cuda_apply_mask": ([vp, i, i, vp, vp], i),
            "carve_cuda_remove_object": ([vp, i, i, vp, vp, i, vp, vp, vp, vp, vp], i),
            "carve_cuda_remove_object_ex": ([vp, i, i, vp, vp, i, i, vp, vp, vp, vp, vp, vp], i),
            "carve_cuda_dp_seam_forward": ([vp, i, i, vp, vp, vp], i),
            "carve_cuda_dp_seam_forward_costs": ([vp, vp, vp, i, i, vp, vp, vp], i),
            "carve_cuda_remove_seam_f64": ([vp, i, i, vp, i, vp], i),
            "carve_cuda_remove_seam_u8": ([vp, i, i, vp, i, vp], i),
            "carve_cuda_carve_batch": ([vp, i, i, i, i, i, vp, vp, i], i),
            "carve_cuda_batch_plan": ([i, i, i, i, i, i, vp, vp], i),
            "carve_cuda_carve_device": ([vp, i, i, i, i, vp, vp, vp], i),
            "carve_cuda_carve_batch_device": ([vp, i, i, i, i, i, vp, vp], i),
            "carve_make_test_image": ([i, i, C.c_uint32, vp], i),
            "carve_cuda_set_kernel_events": ([i], i),
            "carve_cuda_kernel_event_stats": ([i, vp, vp, vp], i),
        }
        for name, (args, res) in sigs.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
    return _lib


def _check(status: int) -> None:
    if status:
        msg = library().carve_cuda_last_error().decode()
        raise CarveError(status, msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _img(img: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 3 or a.shape[2] != 3:
        raise CarveError(Errc.dimension_mismatch, "image must have shape (H, W, 3)")
    return a


def device_count() -> int:
    return int(library().carve_cuda_device_count())


def set_device(device: int) -> None:
    _check(library().carve_cuda_set_device(device))


def launch_count() -> int:
    """Kernels this library launched on the calling thread since the last reset."""
    return int(library().carve_cuda_launch_count())


def reset_launch_count() -> None:
    library().carve_cuda_reset_launch_count()


KERNEL_KINDS = {0: "k_energy_full", 1: "k_dp_seam", 2: "k_compact", 3: "k_unpack", 4: "k_pack", 5: "k_transpose"}


def set_kernel_events(on: bool) -> None:
    """Bracket every kernel the carve driver launches with CUDA events (bench attribution)."""
    _check(library().carve_cuda_set_kernel_events(1 if on else 0))


def kernel_event_stats() -> dict:
    """Per kernel: total event ms, launches, algorithmic bytes."""
    out = {}
    for kind, name in KERNEL_KINDS.items():
        ms, n, by = C.c_double(), C.c_uint64(), C.c_double()
        _check(library().carve_cuda_kernel_event_stats(kind, C.addressof(ms), C.addressof(n), C.addressof(by)))
        if n.value:
            out[name] = {"ms_total": ms.value, "launches": int(n.value), "bytes_total": by.value}
    return out


def _unsupported(what: str):
    raise CarveError(Errc.usage_error, f"{what} is not supported by the B200 engine")


# -- bench fixture (bench.hpp:67-94) -------------------------------------------
def make_test_image(width: int, height: int, variant: int = 0) -> np.ndarray:
    out = np.empty((max(height, 0), max(width, 0), 3), np.uint8)
    _check(library().carve_make_test_image(width, height, variant, _ptr(out)))
    return out


# -- raster / energy -------------------------------------------------------------
def to_grayscale(img: np.ndarray) -> np.ndarray:
    """raster.hpp:61-71"""
    a = _img(img)
    h, w, _ = a.shape
    out = np.empty((h, w), np.float64)
    _check(library().carve_cuda_to_grayscale(_ptr(a), w, h, _ptr(out)))
    return out


def energy_e1(gray: np.ndarray) -> np.ndarray:
    """energy.hpp:89-98 on a LumaGrid (any float64 plane)."""
    g = np.ascontiguousarray(gray, dtype=np.float64)
    h, w = g.shape
    out = np.empty((h, w), np.float64)
    _check(library().carve_cuda_energy_e1_luma(_ptr(g), w, h, _ptr(out)))
    return out


def energy_e1_rgb(img: np.ndarray) -> np.ndarray:
    """energy_e1(to_grayscale(img)) fused on the device (carver.hpp:161-162)."""
    a = _img(img)
    h, w, _ = a.shape
    out = np.empty((h, w), np.float64)
    _check(library().carve_cuda_energy_e1_rgb(_ptr(a), w, h, _ptr(out)))
    return out


def compute_energy(gray: np.ndarray, fn: EnergyFn = EnergyFn.e1) -> np.ndarray:
    """energy.hpp:186-194; only e1 is on the B200 path."""
    if EnergyFn(fn) is not EnergyFn.e1:
        _unsupported(f"energy function {EnergyFn(fn).value}")
    return energy_e1(gray)


def transpose(img: np.ndarray) -> np.ndarray:
    """raster.hpp:73-79"""
    a = _img(img)
    h, w, _ = a.shape
    out = np.empty((w, h, 3), np.uint8)
    _check(library().carve_cuda_transpose_rgb(_ptr(a), w, h, _ptr(out)))
    return out


# -- solvers ------------------------------------------------------------------------
def dp_seam(energy: np.ndarray) -> SeamResult:
    """solvers.hpp:263-289 — seam plus the full cost table."""
    e = np.ascontiguousarray(energy, dtype=np.float64)
    if e.ndim != 2 or e.size == 0:
        raise CarveError(Errc.empty_image, "image is empty")
    h, w = e.shape
    m = np.empty((h, w), np.float64)
    b = np.empty((h, w), np.int32)
    seam = np.empty(h, np.int32)
    _check(library().carve_cuda_dp_seam(_ptr(e), w, h, _ptr(m), _ptr(b), _ptr(seam)))
    return SeamResult(seam, CostTable(w, h, m, b))


def parallel_dp_seam(energy: np.ndarray, workers: int = 0) -> SeamResult:
    """solvers.hpp:331-347 — same table as dp_seam for every worker count."""
    return dp_seam(energy)


def find_seam(energy: np.ndarray, kind: SolverKind = SolverKind.ParallelDynamic,
              opts: SolverOptions | None = None) -> np.ndarray:
    """solvers.hpp:350-358"""
    kind = SolverKind(kind)
    if kind not in (SolverKind.Dynamic, SolverKind.ParallelDynamic):
        _unsupported(f"solver {kind.value}")
    e = np.ascontiguousarray(energy, dtype=np.float64)
    if e.ndim != 2 or e.size == 0:
        raise CarveError(Errc.empty_image, "image is empty")
    h, w = e.shape
    seam = np.empty(h, np.int32)
    _check(library().carve_cuda_dp_seam(_ptr(e), w, h, None, None, _ptr(seam)))
    return seam


def validate_seam(seam, width: int, height: int) -> None:
    """solvers.hpp:69-78"""
    s = np.ascontiguousarray(seam, dtype=np.int32)
    _check(library().carve_cuda_validate_seam(_ptr(s), len(s), width, height))


# -- pipelines --------------------------------------------------------------------
def remove_seam(img: np.ndarray, seam) -> np.ndarray:
    """remove_seam overloads (carver.hpp:71-112), dispatched on the array like the
    reference's on the type: (H, W, 3) uint8 PixelGrid (validated seam, W >= 2);
    (H, W) float64 LumaGrid / EnergyMap and (H, W) uint8 RemovalMask =
    detail::drop_columns (carver.hpp:57-67), no connectivity requirement."""
    arr = np.asarray(img)
    if arr.ndim == 2:
        s = np.ascontiguousarray(seam, dtype=np.int32)
        h, w = arr.shape
        if arr.dtype == np.uint8:
            a = np.ascontiguousarray(arr)
            out = np.empty((h, max(w - 1, 0)), np.uint8)
            _check(library().carve_cuda_remove_seam_u8(_ptr(a), w, h, _ptr(s), len(s), _ptr(out)))
        else:
            a = np.ascontiguousarray(arr, dtype=np.float64)
            out = np.empty((h, max(w - 1, 0)), np.float64)
            _check(library().carve_cuda_remove_seam_f64(_ptr(a), w, h, _ptr(s), len(s), _ptr(out)))
        return out
    a = _img(img)
    h, w, _ = a.shape
    s = np.ascontiguousarray(seam, dtype=np.int32)
    out = np.empty((h, max(w - 1, 0), 3), np.uint8)
    _check(library().carve_cuda_remove_seam_rgb(_ptr(a), w, h, _ptr(s), len(s), _ptr(out)))
    return out


def _check_config(cfg: CarveConfig | None) -> None:
    if cfg is None:
        return
    if cfg.forward and SolverKind(cfg.solver) not in (SolverKind.Dynamic, SolverKind.ParallelDynamic):
        raise CarveError(Errc.usage_error, "forward energy requires the dp or pardp solver")  # carver.hpp:51-54
    if SolverKind(cfg.solver) not in (SolverKind.Dynamic, SolverKind.ParallelDynamic):
        _unsupported(f"solver {SolverKind(cfg.solver).value}")
    if not cfg.forward and EnergyFn(cfg.energy_fn) is not EnergyFn.e1:
        _unsupported(f"energy function {EnergyFn(cfg.energy_fn).value}")


class _Config(C.Structure):  # carve_cuda_config
    _fields_ = [("forward", C.c_int), ("recompute", C.c_int)]


def _abi_config(cfg: CarveConfig | None = None, forward: bool = False, recompute: bool = True):
    if cfg is not None:
        forward, recompute = cfg.forward, cfg.recompute
    return _Config(int(bool(forward)), int(bool(recompute)))


def carve(img: np.ndarray, target_width: int, target_height: int | None = None, *, seams: bool = False,
          timings: bool = False, out: np.ndarray | None = None, forward: bool = False, recompute: bool = True):
    """run_resize semantics (cli.hpp:249-256): carve_to_width then carve_to_height.
    Returns the carved image, plus (seams, timings) lists when requested. `out`
    (optional, C-contiguous uint8 target_height x target_width x 3, e.g. pinned
    memory) receives the image instead of a fresh array."""
    a = _img(img)
    h, w, _ = a.shape
    th = h if target_height is None else int(target_height)
    tw = int(target_width)
    if tw < 1 or tw > w:
        raise CarveError(Errc.invalid_target, "target width must be in [1, width]")
    if th < 1 or th > h:
        raise CarveError(Errc.invalid_target, "target height must be in [1, height]")
    if out is None:
        out = np.empty((th, tw, 3), np.uint8)
    elif out.shape != (th, tw, 3) or out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise CarveError(Errc.usage_error, "out must be a C-contiguous uint8 array of shape (th, tw, 3)")
    n_ints = (w - tw) * h + (h - th) * tw
    nseams = (w - tw) + (h - th)
    s = np.empty(max(n_ints, 1), np.int32)
    t = (_Timing * max(nseams, 1))()
    if forward or not recompute:  # CarveConfig::forward / ::recompute (carver.hpp:15-24)
        cfg = _abi_config(forward=forward, recompute=recompute)
        _check(library().carve_cuda_carve_cfg(_ptr(a), w, h, tw, th, C.byref(cfg), _ptr(out),
                                              _ptr(s) if seams else None, C.cast(t, C.c_void_p) if timings else None))
    else:
        _check(library().carve_cuda_carve(_ptr(a), w, h, tw, th, _ptr(out), _ptr(s) if seams else None,
                                          C.cast(t, C.c_void_p) if timings else None))
    if not (seams or timings):
        return out
    seam_list = []
    if seams:
        off = 0
        for _ in range(w - tw):
            seam_list.append(s[off:off + h].copy())
            off += h
        for _ in range(h - th):
            seam_list.append(s[off:off + tw].copy())
            off += tw
    tim = [SeamTiming(t[k].energy_s, t[k].solve_s, t[k].remove_s) for k in range(nseams)] if timings else []
    return out, seam_list, tim


def _report(seams, tims, total_s) -> CarveReport:
    return CarveReport(seam_count=len(seams), per_seam=tims, seams=seams, total_s=total_s)


def carve_to_width(img: np.ndarray, target_width: int, cfg: CarveConfig | None = None):
    """carver.hpp:191-214 — returns (carved, CarveReport)."""
    import time
    a = _img(img)
    h, w, _ = a.shape
    if target_width < 1 or target_width > w:
        raise CarveError(Errc.invalid_target, "target width must be in [1, width]")
    _check_config(cfg)
    t0 = time.perf_counter()
    c = cfg or CarveConfig()
    out, seams, tims = carve(a, target_width, h, seams=True, timings=True, forward=c.forward, recompute=c.recompute)
    return out, _report(seams, tims, time.perf_counter() - t0)


def forward_costs(luma: np.ndarray):
    """energy.hpp:196-216 -> (cost_left, cost_up, cost_right), on the device."""
    g = np.ascontiguousarray(luma, dtype=np.float64)
    h, w = g.shape
    outs = [np.empty((h, w), np.float64) for _ in range(3)]
    _check(library().carve_cuda_forward_costs(_ptr(g), w, h, *[_ptr(o) for o in outs]))
    return tuple(outs)


def dp_seam_forward(luma: np.ndarray, costs=None) -> SeamResult:
    """solvers.hpp:294-326 forward-energy DP on the device. costs = (left, up,
    right) planes, any finite values (the reference's gray only supplies the
    dimensions); None = forward_costs(luma), derived on the device."""
    g = np.ascontiguousarray(luma, dtype=np.float64)
    if g.ndim != 2 or g.size == 0:
        raise CarveError(Errc.empty_image, "image is empty")
    h, w = g.shape
    m = np.empty((h, w), np.float64)
    b = np.empty((h, w), np.int32)
    seam = np.empty(h, np.int32)
    if costs is not None:
        if len(costs) != 3 or any(np.shape(c) != (h, w) for c in costs):
            raise CarveError(Errc.dimension_mismatch, "forward costs do not match image dimensions")
        cl, cu, cr = (np.ascontiguousarray(c, dtype=np.float64) for c in costs)
        _check(library().carve_cuda_dp_seam_forward_costs(_ptr(cl), _ptr(cu), _ptr(cr), w, h, _ptr(m), _ptr(b),
                                                          _ptr(seam)))
    else:
        _check(library().carve_cuda_dp_seam_forward(_ptr(g), w, h, _ptr(m), _ptr(b), _ptr(seam)))
    return SeamResult(seam, CostTable(w, h, m, b))


def mask_from_image(img: np.ndarray) -> np.ndarray:
    """energy.hpp:244-253 — uint8 flags (luma >= 128), on the device."""
    a = _img(img)
    h, w, _ = a.shape
    out = np.empty((h, w), np.uint8)
    _check(library().carve_cuda_mask_from_rgb(_ptr(a), w, h, _ptr(out)))
    return out


def apply_mask(energy: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """energy.hpp:220-241 — masked cells -> -1000*(h*m + 1), on the device."""
    e = np.ascontiguousarray(energy, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    if e.shape != m.shape:
        raise CarveError(Errc.dimension_mismatch, "mask dimensions do not match energy map")
    h, w = e.shape
    out = np.empty((h, w), np.float64)
    _check(library().carve_cuda_apply_mask(_ptr(e), w, h, _ptr(m), _ptr(out)))
    return out


def mask_bounds(mask: np.ndarray):
    """energy.hpp:266-283 — (top, left, bottom, right), inclusive; bottom < top when empty."""
    ys, xs = np.nonzero(np.asarray(mask))
    if ys.size == 0:
        h, w = np.shape(mask)
        return (h, w, -1, -1)
    return (int(ys.min()), int(xs.min()), int(ys.max()), int(xs.max()))


def _remove_object(img, mask, cfg, restore, orientation):
    import time
    a = _img(img)
    h, w, _ = a.shape
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    if m.shape != (h, w):
        raise CarveError(Errc.dimension_mismatch, "mask dimensions do not match image")
    t0 = time.perf_counter()
    buf = np.empty(max(w * h * 3, 1), np.uint8)
    flat = np.empty(max(w * h, 1), np.int32)
    tim = (_Timing * max(w, h, 1))()
    ow, oh, ns = C.c_int(), C.c_int(), C.c_int()
    c = _abi_config(cfg)
    _check(library().carve_cuda_remove_object_ex(_ptr(a), w, h, _ptr(m), C.byref(c), int(bool(restore)), orientation,
                                                 _ptr(buf), C.byref(ow), C.byref(oh), _ptr(flat), C.byref(ns),
                                                 C.cast(tim, C.c_void_p)))
    out = buf[: ow.value * oh.value * 3].reshape(oh.value, ow.value, 3).copy()
    top, left, bottom, right = mask_bounds(m)
    n = h if (orientation == 1 or right - left <= bottom - top) else w
    seams = [flat[t * n:(t + 1) * n].copy() for t in range(ns.value)]
    per = [SeamTiming(tim[t].energy_s, tim[t].solve_s, tim[t].remove_s) for t in range(ns.value)]
    return out, _report(seams, per, time.perf_counter() - t0)


def remove_object(img: np.ndarray, mask: np.ndarray, cfg: CarveConfig | None = None, restore: bool = True):
    """carver.hpp:327-340 — returns (result, CarveReport). The removal loop and
    the restoring enlargement run on the device; per-seam timings from device
    timestamps."""
    _check_config(cfg)
    return _remove_object(img, mask, cfg, restore, 0)


def remove_object_vertical(img: np.ndarray, mask: np.ndarray, cfg: CarveConfig | None = None,
                           restore: bool = True):
    """detail::remove_object_vertical (carver.hpp:289-321): the loop along columns
    whatever the mask's shape; an empty mask carves nothing."""
    return _remove_object(img, mask, cfg, restore, 1)


def insert_seam(img: np.ndarray, seam) -> np.ndarray:
    """carver.hpp:137-140 — one pixel per row right of the seam, the rounded
    mean of its neighbours (duplicating at the right border)."""
    a = _img(img)
    h, w, _ = a.shape
    s = np.ascontiguousarray(seam, dtype=np.int32)
    out = np.empty((h, w + 1, 3), np.uint8)
    _check(library().carve_cuda_insert_seam_rgb(_ptr(a), w, h, _ptr(s), len(s), _ptr(out)))
    return out


def record_seams(img: np.ndarray, count: int, cfg: CarveConfig | None = None):
    """carver.hpp:226-262 — the removal loop on a scratch copy; returns
    (seams in original-image coordinates, CarveReport)."""
    import time
    a = _img(img)
    h, w, _ = a.shape
    _check_config(cfg)
    count = int(count)
    t0 = time.perf_counter()
    s = np.empty((max(count, 0), h), np.int32)
    t = (_Timing * max(count, 1))()
    c = _abi_config(cfg)
    _check(library().carve_cuda_record_seams(_ptr(a), w, h, count, C.byref(c), _ptr(s) if count > 0 else None,
                                             C.cast(t, C.c_void_p)))
    seams = [s[k].copy() for k in range(count)]
    tims = [SeamTiming(t[k].energy_s, t[k].solve_s, t[k].remove_s) for k in range(count)]
    return seams, _report(seams, tims, time.perf_counter() - t0)


def enlarge(img: np.ndarray, target_width: int, target_height: int | None = None, *, seams: bool = False,
            cfg: CarveConfig | None = None, timings: bool = False):
    """run_enlarge (cli.hpp:262-277): enlarge_to_width on the width, then on the
    transpose for the height. Returns the image (plus the recorded seams of both
    phases, concatenated, when `seams`; plus their per-seam SeamTimings when
    `timings`)."""
    a = _img(img)
    h, w, _ = a.shape
    th = h if target_height is None else int(target_height)
    tw = int(target_width)
    n = max(tw - w, 0) * h + max(th - h, 0) * tw
    out = np.empty((max(th, 0), max(tw, 0), 3), np.uint8)
    s = np.empty(max(n, 1), np.int32)
    nt = max(tw - w, 0) + max(th - h, 0)
    t = (_Timing * max(nt, 1))()
    c = _abi_config(cfg)
    _check(library().carve_cuda_enlarge_timed(_ptr(a), w, h, tw, th, C.byref(c), _ptr(out), _ptr(s),
                                              C.cast(t, C.c_void_p) if timings else None))
    res = [out]
    if seams:
        res.append(s[:n])
    if timings:
        res.append([SeamTiming(t[k].energy_s, t[k].solve_s, t[k].remove_s) for k in range(nt)])
    return res[0] if len(res) == 1 else tuple(res)


def enlarge_to_width(img: np.ndarray, target_width: int, cfg: CarveConfig | None = None):
    """carver.hpp:266-285 — returns (enlarged, CarveReport with the recorded seams)."""
    import time
    a = _img(img)
    h, w, _ = a.shape
    _check_config(cfg)
    t0 = time.perf_counter()
    out, flat, tims = enlarge(a, target_width, h, seams=True, cfg=cfg, timings=True)
    k = int(target_width) - w
    seams = [flat[t * h:(t + 1) * h].copy() for t in range(k)]
    return out, _report(seams, tims[:k], time.perf_counter() - t0)


def carve_to_height(img: np.ndarray, target_height: int, cfg: CarveConfig | None = None):
    """carver.hpp:216-222 — transpose ∘ carve_to_width ∘ transpose, on the device."""
    import time
    a = _img(img)
    h, w, _ = a.shape
    if target_height < 1 or target_height > h:
        raise CarveError(Errc.invalid_target, "target height must be in [1, height]")
    _check_config(cfg)
    t0 = time.perf_counter()
    c = cfg or CarveConfig()
    out, seams, tims = carve(a, w, target_height, seams=True, timings=True, forward=c.forward, recompute=c.recompute)
    return out, _report(seams, tims, time.perf_counter() - t0)


def carve_batch(imgs, target_width: int, target_height: int | None = None, devices=None, out=None) -> list:
    """Batch of same-size images, sharded by image across devices.
    `out` (optional): preallocated C-contiguous (th, tw, 3) uint8 arrays to fill."""
    arrs = [_img(x) for x in imgs]
    if not arrs:
        raise CarveError(Errc.empty_input, "empty batch")
    h, w, _ = arrs[0].shape
    if any(x.shape != arrs[0].shape for x in arrs):
        raise CarveError(Errc.dimension_mismatch, "batch images must share one size")
    th = h if target_height is None else int(target_height)
    if out is None:
        outs = [np.empty((th, target_width, 3), np.uint8) for _ in arrs]
    else:
        outs = list(out)
        if len(outs) != len(arrs) or any(o.shape != (th, target_width, 3) or o.dtype != np.uint8
                                         or not o.flags.c_contiguous for o in outs):
            raise CarveError(Errc.dimension_mismatch, "out arrays must be C-contiguous (th, tw, 3) uint8")
    n = len(arrs)
    ins = (C.c_void_p * n)(*[_ptr(x) for x in arrs])
    ous = (C.c_void_p * n)(*[_ptr(x) for x in outs])
    if devices is None:
        devs, nd = None, 0
    else:
        devs = (C.c_int * len(devices))(*devices)
        nd = len(devices)
    _check(library().carve_cuda_carve_batch(C.cast(ins, C.c_void_p), n, w, h, target_width, th,
                                            C.cast(ous, C.c_void_p), C.cast(devs, C.c_void_p) if devs else None, nd))
    return outs


def batch_plan(n: int, width: int, height: int, target_width: int, target_height: int, ndev: int = 1):
    """(pipelines per device, images per chunk) that carve_batch uses (host logic only)."""
    p, ch = C.c_int(), C.c_int()
    _check(library().carve_cuda_batch_plan(n, width, height, target_width, target_height, ndev, C.addressof(p),
                                           C.addressof(ch)))
    return p.value, ch.value


def carve_device(d_in: int, width: int, height: int, target_width: int, target_height: int, d_out: int,
                 d_seams: int | None = None, stream: int | None = None) -> None:
    """Enqueue a carve of a device-resident packed image (no host sync)."""
    _check(library().carve_cuda_carve_device(d_in, width, height, target_width, target_height, d_out, d_seams,
                                             stream))


def carve_batch_device(d_in: int, n: int, width: int, height: int, target_width: int, target_height: int,
                       d_out: int, stream: int | None = None) -> None:
    """Enqueue a carve of n contiguous device-resident packed images (no host sync)."""
    _check(library().carve_cuda_carve_batch_device(d_in, n, width, height, target_width, target_height, d_out,
                                                   stream))
