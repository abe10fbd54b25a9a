"""ctypes binding of the C ABI in include/blfls/blfls.h (libblfls.so).

There is no CPU fallback: if the shared object is missing or no sm_100 device
is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# BLFLS_LIBRARY: an A/B experiments build (build.py --experiments -> _lib_exp/)
LIB_PATH = Path(os.environ.get("BLFLS_LIBRARY") or Path(__file__).resolve().parent / "_lib" / "libblfls.so")

BLFLS_OK = 0
BLFLS_EINVAL = 1
BLFLS_ENONFINITE = 2
BLFLS_ECUDA = 3
BLFLS_ENOMEM = 4
BLFLS_EUNSUPPORTED = 5

DEVICE_PTRS = 0
HOST_PTRS = 1
CHECK_FINITE = 2
SYNC = 4
NO_GRAPH = 8
TIME_STAGES = 16
ASYNC = 32
BACKEND_BRUTE = 0
BACKEND_GRID = 1
BACKEND_DT = 2

# every symbol include/blfls/blfls.h declares
EXPORTS = (
    "blfls_plan_create", "blfls_plan_destroy", "blfls_run", "blfls_sync", "blfls_filter_gradients",
    "blfls_filter_gradients_rows", "blfls_solve", "blfls_rfft2", "blfls_irfft2",
    "blfls_generate", "blfls_last_stats", "blfls_stage_times", "blfls_debug_ranges", "blfls_mufu_peak", "blfls_last_error",
    "blfls_version", "blfls_abi_version", "blfls_gaussian_blur", "blfls_blf_brute",
    "blfls_forward_gradients", "blfls_filter_gradients_rows_peers", "blfls_multi_create",
    "blfls_multi_run", "blfls_multi_destroy", "blfls_host_alloc", "blfls_host_free",
)

MULTI_BATCH = 0
MULTI_BAND = 1


class BlflsError(RuntimeError):
    """Base error of the CUDA path."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class InvalidArgument(BlflsError, ValueError):
    """std::invalid_argument of the reference (shape / parameter / non-finite)."""


class CudaError(BlflsError):
    pass


class Unsupported(BlflsError, NotImplementedError):
    pass


class Params(C.Structure):
    _fields_ = [
        ("height", C.c_int), ("width", C.c_int), ("channels", C.c_int),
        ("guide_channels", C.c_int), ("radius", C.c_int), ("sigma_s", C.c_double),
        ("sigma_r", C.c_double), ("lambda_", C.c_double), ("max_batch", C.c_int),
        ("device", C.c_int), ("pad", C.c_int), ("backend", C.c_int),
        ("dt_iterations", C.c_int),
    ]


class Stats(C.Structure):
    _fields_ = [("radius", C.c_int), ("blf_launches", C.c_longlong),
                ("kernel_launches", C.c_longlong), ("exps", C.c_double)]


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: the CUDA extension is not built "
                    "(run paper_1812_07122_b200.build.build()); there is no CPU fallback")
            L = C.CDLL(str(LIB_PATH))
            vp, fp, ip = C.c_void_p, C.c_void_p, C.c_int
            L.blfls_plan_create.argtypes = [C.POINTER(Params), C.POINTER(vp)]
            L.blfls_plan_destroy.argtypes = [vp]
            L.blfls_run.argtypes = [vp, fp, fp, ip, ip, fp, vp, C.c_uint]
            L.blfls_sync.argtypes = [vp]
            L.blfls_filter_gradients.argtypes = [vp, fp, fp, ip, fp, fp, vp, C.c_uint]
            L.blfls_filter_gradients_rows.argtypes = [vp, fp, fp, ip, ip, fp, fp, vp, C.c_uint]
            L.blfls_solve.argtypes = [vp, fp, fp, fp, ip, fp, vp, C.c_uint]
            L.blfls_rfft2.argtypes = [vp, fp, ip, fp, vp, C.c_uint]
            L.blfls_irfft2.argtypes = [vp, fp, ip, fp, vp, C.c_uint]
            L.blfls_generate.argtypes = [ip, ip, ip, C.POINTER(C.c_uint64), ip, C.c_double,
                                         C.c_double, fp, vp, ip]
            L.blfls_last_stats.argtypes = [vp, C.POINTER(Stats)]
            L.blfls_stage_times.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
            L.blfls_debug_ranges.argtypes = [vp, C.POINTER(C.c_float)]
            L.blfls_mufu_peak.argtypes = [ip, C.POINTER(C.c_double), C.POINTER(C.c_double)]
            L.blfls_gaussian_blur.argtypes = [fp, ip, ip, ip, C.c_double, fp, ip, vp, C.c_uint]
            L.blfls_filter_gradients_rows_peers.argtypes = [vp, fp, fp, ip, ip, C.POINTER(C.c_void_p),
                                                            C.POINTER(C.c_void_p), ip, vp, C.c_uint]
            L.blfls_forward_gradients.argtypes = [fp, ip, ip, ip, fp, fp, ip, vp, C.c_uint]
            L.blfls_blf_brute.argtypes = [fp, ip, fp, ip, ip, ip, ip, ip, C.c_double, C.c_double, fp,
                                          ip, vp, C.c_uint]
            L.blfls_multi_create.argtypes = [C.POINTER(Params), C.POINTER(C.c_int), ip, ip, C.POINTER(vp)]
            L.blfls_multi_run.argtypes = [vp, fp, fp, ip, ip, fp, C.c_uint]
            L.blfls_multi_destroy.argtypes = [vp]
            L.blfls_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
            L.blfls_host_free.argtypes = [vp]
            L.blfls_last_error.restype = C.c_char_p
            L.blfls_version.restype = C.c_char_p
            for name in EXPORTS:
                if name not in ("blfls_last_error", "blfls_version", "blfls_abi_version"):
                    getattr(L, name).restype = C.c_int
            _lib = L
    return _lib


def check(status: int) -> None:
    if status == BLFLS_OK:
        return
    msg = lib().blfls_last_error().decode(errors="replace")
    if status in (BLFLS_EINVAL, BLFLS_ENONFINITE):
        raise InvalidArgument(status, msg)
    if status == BLFLS_EUNSUPPORTED:
        raise Unsupported(status, msg)
    raise CudaError(status, msg)


class Plan:
    """Owns a blfls_plan_t (one per host thread / stream, like the C ABI says)."""

    def __init__(self, height, width, channels, guide_channels, radius, sigma_s, sigma_r, lam,
                 max_batch=1, device=0, pad=0, backend=0, dt_iterations=0):
        self.params = Params(int(height), int(width), int(channels), int(guide_channels),
                             int(radius), float(sigma_s), float(sigma_r), float(lam),
                             int(max_batch), int(device), int(pad), int(backend),
                             int(dt_iterations))
        h = C.c_void_p()
        check(lib().blfls_plan_create(C.byref(self.params), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.blfls_plan_destroy(h)
            self.handle = None

    def sync(self) -> None:
        """Wait for all calls on this plan (reports deferred non-finite input)."""
        check(lib().blfls_sync(self.handle))

    def stage_times(self):
        """(ms sums, launch counts) per stage: minmax, blf, r2c, col, c2r."""
        ms = (C.c_double * 5)()
        n = (C.c_longlong * 5)()
        check(lib().blfls_stage_times(self.handle, ms, n))
        return list(ms), list(n)

    def debug_ranges(self):
        """[[slot0 (lo, hi) per image], [slot1 ...]] as floats."""
        n = 4 * self.params.max_batch
        buf = (C.c_float * n)()
        check(lib().blfls_debug_ranges(self.handle, buf))
        v = list(buf)
        mb = self.params.max_batch
        return [[(v[2 * i], v[2 * i + 1]) for i in range(mb)],
                [(v[2 * mb + 2 * i], v[2 * mb + 2 * i + 1]) for i in range(mb)]]

    def stats(self) -> Stats:
        s = Stats()
        check(lib().blfls_last_stats(self.handle, C.byref(s)))
        return s


class MultiPlan:
    """blfls_multi_* (one process, several device entries; a device may
    repeat): MULTI_BATCH shards the batch, MULTI_BAND splits one image into
    row bands with NVLink peer stores.  Host float32 buffers."""

    def __init__(self, params: Params, devices, mode=MULTI_BATCH):
        self.params = params
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(lib().blfls_multi_create(C.byref(params), devs, len(devices), int(mode), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.blfls_multi_destroy(h)
            self.handle = None

    def run(self, img, guide, batch, iters, out, check_finite=True):
        """img / guide / out: C-contiguous float32 numpy arrays (host)."""
        ptr = lambda a: None if a is None else a.ctypes.data
        check(lib().blfls_multi_run(self.handle, ptr(img), ptr(guide), int(batch), int(iters), ptr(out),
                                    HOST_PTRS | (CHECK_FINITE if check_finite else 0)))


def mufu_peak(device: int = 0):
    """Measured MUFU.EX2 rate (ex2/s) and SM clock (Hz) of `device`."""
    rate, clk = C.c_double(), C.c_double()
    check(lib().blfls_mufu_peak(int(device), C.byref(rate), C.byref(clk)))
    return rate.value, clk.value
