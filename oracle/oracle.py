"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.

Two libraries:

* ``oracle/liboracle.so``      -- the C restatement (oracle/blfls_oracle.c).
* ``oracle/_ref/libepls_ref.so`` -- the reference's own translation units
  compiled unmodified from /root/reference/proj (oracle/Makefile) plus shims.
  Built only where /root/reference exists; the built file travels to the GPU
  box with the repo snapshot.

Arrays are float64 planar C x H x W (the reference PlanarImage layout,
/root/reference/proj/include/epls/image.hpp:9-41).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libepls_ref.so"
REF_SRC = Path("/root/reference/proj")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


class OracleError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} returned status {status}")
        self.status = status


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and oracle/_ref when the reference tree is present)."""
    targets = ["all"]
    if ref is None:
        ref = REF_SRC.is_dir()
    if ref:
        targets.append("ref")
    cmd = ["make", "-s", "-C", str(HERE)]
    if subprocess.run([*cmd, f"-j{os.cpu_count() or 4}", *targets]).returncode != 0:
        # a parallel make can lose a compiler to memory pressure; finish serially
        subprocess.run([*cmd, "-j1", *targets], check=True)


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        build(ref=path == REF_SO)
    return C.CDLL(str(path))


_lib: C.CDLL | None = None
_ref: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load(ORACLE_SO)
        _lib.orc_uniform_at.restype = C.c_double
        _lib.orc_uniform_at.argtypes = [C.c_uint64, C.c_uint64]
        _lib.orc_splitmix64_at.restype = C.c_uint64
        _lib.orc_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        _lib.orc_diff_gain_sq.restype = C.c_double
        _lib.orc_nc_box_radius.restype = C.c_double
        _lib.orc_nc_box_radius.argtypes = [C.c_double, C.c_int, C.c_int]
        _lib.orc_gen_plane.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _fp]
        for name in ("orc_blf_ls", "orc_blf_ls_timed", "orc_blf_ls_pad", "orc_smooth_brute", "orc_blf_brute_r",
                     "orc_lsgrad_solve_fft", "orc_dense_solve"):
            getattr(_lib, name).restype = C.c_int
    return _lib


def ref_available() -> bool:
    return REF_SO.exists() or REF_SRC.is_dir()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        _ref = _load(REF_SO)
        _ref.ref_max_abs_gradient.restype = C.c_double
        _ref.ref_nc_box_radius.restype = C.c_double
        _ref.ref_nc_box_radius.argtypes = [C.c_double, C.c_int, C.c_int]
        _ref.ref_random_image.argtypes = [C.c_int, C.c_int, C.c_int, C.c_ulonglong, C.c_double,
                                          C.c_double, _dp]
        _ref.ref_natural_scene.argtypes = [C.c_int, C.c_int, C.c_int, C.c_ulonglong, _dp]
    return _ref


def _d(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _shape3(a: np.ndarray):
    if a.ndim == 2:
        return 1, a.shape[0], a.shape[1]
    return a.shape


def _check(fn: str, st: int):
    if st != 0:
        raise OracleError(fn, st)


# ---------------------------------------------------------------- oracle --

def blf_ls(img, guide=None, *, lam, sigma_s, sigma_r, iters, radius, timed=False, pad=0):
    """North-star cascade (orc_blf_ls): f <- smooth_brute(f) `iters` times
    (with the reference's reflect padding when pad > 0)."""
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    gc = 0 if gd is None else _shape3(gd)[0]
    if pad:
        assert not timed
        st = lib().orc_blf_ls_pad(_d(g), c, h, w, _d(gd), gc, int(radius), C.c_double(sigma_s),
                                  C.c_double(sigma_r), C.c_double(lam), int(iters), int(pad), _d(out))
        _check("orc_blf_ls_pad", st)
        return out
    if timed:
        tb, ts = C.c_double(), C.c_double()
        st = lib().orc_blf_ls_timed(_d(g), c, h, w, _d(gd), gc, int(radius), C.c_double(sigma_s),
                                    C.c_double(sigma_r), C.c_double(lam), int(iters), _d(out),
                                    C.byref(tb), C.byref(ts))
        _check("orc_blf_ls_timed", st)
        return out, tb.value, ts.value
    st = lib().orc_blf_ls(_d(g), c, h, w, _d(gd), gc, int(radius), C.c_double(sigma_s),
                          C.c_double(sigma_r), C.c_double(lam), int(iters), _d(out))
    _check("orc_blf_ls", st)
    return out


def smooth_brute(img, guide=None, *, lam, sigma_s, sigma_r, radius, pad=0):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    st = lib().orc_smooth_brute(_d(g), c, h, w, _d(gd), int(radius), C.c_double(sigma_s),
                                C.c_double(sigma_r), C.c_double(lam), int(pad), _d(out))
    _check("orc_smooth_brute", st)
    return out


def blf_brute_r(src, guide, *, sigma_s, sigma_r, radius=-1):
    s = _f64(src)
    gd = _f64(guide)
    cs, h, w = _shape3(s)
    cg = _shape3(gd)[0]
    out = np.empty((cs, h, w))
    st = lib().orc_blf_brute_r(_d(s), cs, _d(gd), cg, h, w, int(radius), C.c_double(sigma_s),
                               C.c_double(sigma_r), _d(out))
    _check("orc_blf_brute_r", st)
    return out


def forward_gradients(img):
    g = _f64(img)
    c, h, w = _shape3(g)
    gx = np.empty((c, h, w))
    gy = np.empty((c, h, w))
    lib().orc_forward_gradients(_d(g), c, h, w, _d(gx), _d(gy))
    return gx, gy


def normalize_to_unit(img):
    g = _f64(img)
    out = np.empty_like(g)
    lo, hi = C.c_double(), C.c_double()
    st = lib().orc_normalize_to_unit(_d(g), C.c_size_t(g.size), _d(out), C.byref(lo), C.byref(hi))
    _check("orc_normalize_to_unit", st)
    return out, lo.value, hi.value


def lsgrad_solve_fft(g, tx, ty, *, lam, pad=0):
    g = _f64(g)
    c, h, w = _shape3(g)
    u = np.empty((c, h, w))
    st = lib().orc_lsgrad_solve_fft(_d(g), _d(None if tx is None else _f64(tx)),
                                    _d(None if ty is None else _f64(ty)), c, h, w,
                                    C.c_double(lam), int(pad), _d(u))
    _check("orc_lsgrad_solve_fft", st)
    return u


def dense_solve(g, tx, ty, *, lam):
    g = _f64(g)
    c, h, w = _shape3(g)
    u = np.empty((c, h, w))
    st = lib().orc_dense_solve(_d(g), _d(None if tx is None else _f64(tx)),
                               _d(None if ty is None else _f64(ty)), c, h, w, C.c_double(lam), _d(u))
    _check("orc_dense_solve", st)
    return u


def rfft2(x):
    x = _f64(x)
    h, w = x.shape
    spec = np.empty((h, w // 2 + 1), dtype=np.complex128)
    lib().orc_rfft2(_d(x), h, w, spec.ctypes.data_as(_dp))
    return spec


def irfft2(spec, w):
    s = np.ascontiguousarray(spec, dtype=np.complex128).copy()
    h = s.shape[0]
    out = np.empty((h, w))
    lib().orc_irfft2(s.ctypes.data_as(_dp), h, w, _d(out))
    return out


def fft1d(x, sign=-1):
    x = np.ascontiguousarray(x, dtype=np.complex128)
    out = np.empty_like(x)
    lib().orc_fft1d(len(x), x.ctypes.data_as(_dp), out.ctypes.data_as(_dp), int(sign))
    return out


def naive_dft2(img):
    g = _f64(img)
    h, w = g.shape
    spec = np.empty((h, w), dtype=np.complex128)
    lib().orc_naive_dft2(_d(g), h, w, spec.ctypes.data_as(_dp))
    return spec


def nc_box_radius(sigma_s, it, total) -> float:
    return lib().orc_nc_box_radius(sigma_s, it, total)


def nc_filter(src, guide, *, sigma_s, sigma_r, iters=3):
    """orc_nc_filter (domain_transform.cpp:138-156)."""
    s_ = _f64(src)
    gd = _f64(guide)
    cs, h, w = _shape3(s_)
    out = np.empty((cs, h, w))
    _check("orc_nc_filter", lib().orc_nc_filter(_d(s_), cs, _d(gd), _shape3(gd)[0], h, w,
                                                C.c_double(sigma_s), C.c_double(sigma_r), int(iters),
                                                _d(out)))
    return out


def smooth_nc(img, guide=None, *, lam, sigma_s, sigma_r, dt_iters=3, pad=0):
    """One smooth() call with SmootherKind::NC_LS (pipelines.cpp:57-94)."""
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    _check("orc_smooth_nc", lib().orc_smooth_nc(_d(g), c, h, w, _d(gd), C.c_double(sigma_s),
                                                C.c_double(sigma_r), int(dt_iters), C.c_double(lam),
                                                int(pad), _d(out)))
    return out


def nc_ls(img, guide=None, *, lam, sigma_s, sigma_r, dt_iters=3, iters=1, pad=0):
    """NC-LS cascade: `iters` smooth_nc calls, guide fixed (1-channel guide replicated)."""
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    gc = 0 if gd is None else _shape3(gd)[0]
    _check("orc_nc_ls", lib().orc_nc_ls(_d(g), c, h, w, _d(gd), gc, C.c_double(sigma_s),
                                        C.c_double(sigma_r), int(dt_iters), C.c_double(lam),
                                        int(iters), int(pad), _d(out)))
    return out


def gaussian_blur(img, sigma):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    _check("orc_gaussian_blur", lib().orc_gaussian_blur(_d(g), c, h, w, C.c_double(sigma), _d(out)))
    return out


def rolling_nc_ls(img, *, lam, sigma_s, sigma_r, dt_iters=3, pad=0, n=3, init_sigma=2.5):
    """pipelines.cpp:96-117."""
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    _check("orc_rolling_nc_ls",
           lib().orc_rolling_nc_ls(_d(g), c, h, w, C.c_double(sigma_s), C.c_double(sigma_r),
                                   int(dt_iters), C.c_double(lam), int(pad), int(n),
                                   C.c_double(init_sigma), _d(out)))
    return out


def gen_plane(seed, h, w, *, n_sites, noise_sigma=0.03, p_sp=0.0) -> np.ndarray:
    out = np.empty((h, w), dtype=np.float32)
    lib().orc_gen_plane(C.c_uint64(seed), h, w, n_sites, C.c_double(noise_sigma), C.c_double(p_sp),
                        out.ctypes.data_as(_fp))
    return out


def uniform_at(seed, j) -> float:
    return lib().orc_uniform_at(seed, j)


def num_threads() -> int:
    return lib().orc_num_threads()


# ------------------------------------------------------------- reference --

def ref_blf_brute(src, guide, *, sigma_s, sigma_r, serial=False):
    s = _f64(src)
    gd = _f64(guide)
    cs, h, w = _shape3(s)
    cg = _shape3(gd)[0]
    out = np.empty((cs, h, w))
    fn = ref().ref_serial_blf_brute if serial else ref().ref_blf_brute
    st = fn(_d(s), cs, _d(gd), cg, h, w, C.c_double(sigma_s), C.c_double(sigma_r), _d(out))
    _check("ref_blf_brute", st)
    return out


def ref_forward_gradients(img):
    g = _f64(img)
    c, h, w = _shape3(g)
    gx = np.empty((c, h, w))
    gy = np.empty((c, h, w))
    _check("ref_forward_gradients", ref().ref_forward_gradients(_d(g), c, h, w, _d(gx), _d(gy)))
    return gx, gy


def ref_normalize_to_unit(img):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    lo, hi = C.c_double(), C.c_double()
    _check("ref_normalize_to_unit",
           ref().ref_normalize_to_unit(_d(g), c, h, w, _d(out), C.byref(lo), C.byref(hi)))
    return out, lo.value, hi.value


def ref_lsgrad_solve_fft(g, tx, ty, *, lam, pad=0):
    g = _f64(g)
    c, h, w = _shape3(g)
    u = np.empty((c, h, w))
    _check("ref_lsgrad_solve_fft",
           ref().ref_lsgrad_solve_fft(_d(g), _d(_f64(tx)), _d(_f64(ty)), c, h, w, C.c_double(lam),
                                      int(pad), _d(u)))
    return u


def ref_ls_solve_fft(g, *, lam, pad=0):
    g = _f64(g)
    c, h, w = _shape3(g)
    u = np.empty((c, h, w))
    _check("ref_ls_solve_fft", ref().ref_ls_solve_fft(_d(g), c, h, w, C.c_double(lam), int(pad), _d(u)))
    return u


def ref_dense_solve(g, tx=None, ty=None, *, lam):
    g = _f64(g)
    c, h, w = _shape3(g)
    u = np.empty((c, h, w))
    _check("ref_dense_solve",
           ref().ref_dense_solve(_d(g), _d(None if tx is None else _f64(tx)),
                                 _d(None if ty is None else _f64(ty)), c, h, w, C.c_double(lam), _d(u)))
    return u


def ref_smooth_brute(img, guide=None, *, lam, sigma_s, sigma_r, radius, pad=0):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    _check("ref_smooth_brute",
           ref().ref_smooth_brute(_d(g), c, h, w, _d(gd), int(radius), C.c_double(sigma_s),
                                  C.c_double(sigma_r), C.c_double(lam), int(pad), _d(out)))
    return out


def ref_smooth_grid(img, guide=None, *, lam, sigma_s, sigma_r, pad=0):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    _check("ref_smooth_grid",
           ref().ref_smooth_grid(_d(g), c, h, w, _d(gd), C.c_double(sigma_s), C.c_double(sigma_r),
                                 C.c_double(lam), int(pad), _d(out)))
    return out


def ref_blf_ls(img, guide=None, *, lam, sigma_s, sigma_r, iters, radius, timed=False, pad=0):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    gc = 0 if gd is None else _shape3(gd)[0]
    tb, ts = C.c_double(), C.c_double()
    _check("ref_blf_ls",
           ref().ref_blf_ls_pad(_d(g), c, h, w, _d(gd), gc, int(radius), C.c_double(sigma_s),
                                C.c_double(sigma_r), C.c_double(lam), int(iters), int(pad), _d(out),
                                C.byref(tb), C.byref(ts)))
    if timed:
        return out, tb.value, ts.value
    return out


def ref_nc_box_radius(sigma_s, it, total) -> float:
    return ref().ref_nc_box_radius(sigma_s, it, total)


def ref_nc_filter(src, guide, *, sigma_s, sigma_r, iters=3, serial=False):
    s_ = _f64(src)
    gd = _f64(guide)
    cs, h, w = _shape3(s_)
    out = np.empty((cs, h, w))
    fn = "ref_serial_nc_filter" if serial else "ref_nc_filter"
    _check(fn, getattr(ref(), fn)(_d(s_), cs, _d(gd), _shape3(gd)[0], h, w, C.c_double(sigma_s),
                                  C.c_double(sigma_r), int(iters), _d(out)))
    return out


def ref_smooth_nc(img, guide=None, *, lam, sigma_s, sigma_r, dt_iters=3, pad=0):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    gd = None if guide is None else _f64(guide)
    _check("ref_smooth_nc", ref().ref_smooth_nc(_d(g), c, h, w, _d(gd), C.c_double(sigma_s),
                                                C.c_double(sigma_r), int(dt_iters), C.c_double(lam),
                                                int(pad), _d(out)))
    return out


def ref_rolling_nc_ls(img, *, lam, sigma_s, sigma_r, dt_iters=3, pad=0, n=3, init_sigma=2.5):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    _check("ref_rolling_nc_ls",
           ref().ref_rolling_nc_ls(_d(g), c, h, w, C.c_double(sigma_s), C.c_double(sigma_r),
                                   int(dt_iters), C.c_double(lam), int(pad), int(n),
                                   C.c_double(init_sigma), _d(out)))
    return out


def ref_random_image(w, h, c, seed, lo=0.0, hi=1.0):
    out = np.empty((c, h, w))
    _check("ref_random_image", ref().ref_random_image(w, h, c, seed, lo, hi, _d(out)))
    return out


def ref_natural_scene(w, h, c, seed=7):
    out = np.empty((c, h, w))
    _check("ref_natural_scene", ref().ref_natural_scene(w, h, c, seed, _d(out)))
    return out


def ref_gaussian_blur(img, sigma):
    g = _f64(img)
    c, h, w = _shape3(g)
    out = np.empty((c, h, w))
    _check("ref_gaussian_blur", ref().ref_gaussian_blur(_d(g), c, h, w, C.c_double(sigma), _d(out)))
    return out
