"""Host-side mirror of the reference's BLF-LS entry points over the C ABI.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj, namespace ``epls``):

=========================  ==================================================
this module                reference
=========================  ==================================================
``SmootherSpec``           ``SmootherSpec`` (include/epls/pipelines.hpp:16-23)
``RangeSpatialParams``     ``RangeSpatialParams`` (bilateral.hpp:10-13)
``SolveParams``            ``SolveParams`` (solver.hpp:12-15)
``smooth(g, spec)``        ``smooth`` (pipelines.cpp:57-94), BLF_LS, NC_LS and LS
``DtParams``               ``DtParams`` (domain_transform.hpp:7-11)
``RollingParams``          ``RollingParams`` (pipelines.hpp:25-28)
``nc_ls``                  NC_LS cascade: ``iters`` smooth() calls (nc_filter)
``rolling_nc_ls``          ``rolling_nc_ls`` (pipelines.cpp:96-117)
``texture_removal``        ``texture_removal`` (applications.cpp:66-70)
``clipart_cleanup``        ``clipart_cleanup`` (applications.cpp:72-76)
``gaussian_blur``          ``gaussian_blur`` (image.cpp:114-158)
``blf_brute``              ``blf_brute`` (bilateral.cpp:28-77), standalone filter
``forward_gradients``      ``forward_gradients`` (image.cpp:72-95)
``flash_no_flash``         ``flash_no_flash`` (applications.cpp:58-64)
``blf_ls``                 the north-star cascade: ``iters`` smooth() calls
``filter_gradients``       ``filter_gradients`` (pipelines.cpp:33-53)
``lsgrad_solve_fft``       ``lsgrad_solve_fft`` (solver.cpp:88-124)
``ls_solve_fft``           ``ls_solve_fft`` (solver.cpp:67-86)
``rfft2`` / ``irfft2``     ``detail::rfft2`` / ``irfft2`` (fft2d.hpp:11,14)
=========================  ==================================================

Differences, all deliberate and documented in DESIGN.md: the bilateral stage
is the brute-force filter (the north star) where the reference's smooth()
runs the bilateral grid (``backend="grid"`` runs the grid too); the window
radius is explicit (``radius``; ``None`` means the reference's
ceil(3 sigma_s)); images cross the API as fp32 (the filters evaluate the
gradients in double, the FFT solve in fp32).

Images are numpy arrays (host memory; copied through the C ABI with
``BLFLS_HOST_PTRS``) or CUDA torch tensors (device memory, current stream).
Shapes: (H, W), (C, H, W) or (B, C, H, W), C in {1, 3}.
``std::invalid_argument`` of the reference surfaces as ``InvalidArgument``
(a ``ValueError``).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _capi
from ._capi import (ASYNC, CHECK_FINITE, DEVICE_PTRS, HOST_PTRS, NO_GRAPH, SYNC, CudaError,
                    InvalidArgument, Plan, Unsupported, check, lib)

__all__ = [
    "SmootherKind", "RangeSpatialParams", "SolveParams", "SmootherSpec", "smooth",
    "flash_no_flash", "blf_ls", "nc_ls", "rolling_nc_ls", "texture_removal", "clipart_cleanup",
    "gaussian_blur", "blf_brute", "forward_gradients", "DtParams", "RollingParams", "filter_gradients", "lsgrad_solve_fft", "ls_solve_fft",
    "rfft2", "irfft2", "generate", "get_plan", "sync_plans", "InvalidArgument", "CudaError",
    "Unsupported",
]


class SmootherKind(enum.Enum):
    LS = 0
    WLS = 1
    BLF_LS = 2
    NC_LS = 3


@dataclass
class RangeSpatialParams:
    sigma_s: float = 8.0
    sigma_r: float = 0.1


@dataclass
class SolveParams:
    lam: float = 1024.0
    pad: int = 16


@dataclass
class DtParams:
    sigma_s: float = 8.0
    sigma_r: float = 0.1
    iterations: int = 3


@dataclass
class RollingParams:
    n: int = 3
    init_sigma: float = 2.5


@dataclass
class SmootherSpec:
    kind: SmootherKind = SmootherKind.BLF_LS
    blf: RangeSpatialParams = field(default_factory=lambda: RangeSpatialParams(12.0, 0.04))
    solve: SolveParams = field(default_factory=SolveParams)
    guidance: Any = None          # non-owning guide image of the same shape (or 1 channel)
    radius: int | None = None     # BLF window radius; None = ceil(3 sigma_s) (bilateral.cpp:37)
    backend: str = "brute"        # "brute" (north star) or "grid" (the reference smooth()'s blf_grid)
    dt: DtParams = field(default_factory=lambda: DtParams(12.0, 0.05, 3))  # NC_LS filter


# ----------------------------------------------------------------- plans --

_tls = threading.local()


_BACKENDS = {"brute": _capi.BACKEND_BRUTE, "grid": _capi.BACKEND_GRID, "dt": _capi.BACKEND_DT}


def _backend(name) -> int:
    if name not in _BACKENDS:
        raise InvalidArgument(_capi.BLFLS_EINVAL, f"unknown backend {name!r} (brute | grid | dt)")
    return _BACKENDS[name]


def get_plan(h, w, c, gc, radius, sigma_s, sigma_r, lam, batch, device, pad=0,
             backend="brute", dt_iterations=0) -> Plan:
    """Per-thread plan cache (plans are not thread-safe, blfls.h)."""
    cache = getattr(_tls, "plans", None)
    if cache is None:
        cache = _tls.plans = {}
    be = _backend(backend)
    key = (h, w, c, gc, radius, float(sigma_s), float(sigma_r), float(lam), device, int(pad), be,
           int(dt_iterations))
    p = cache.get(key)
    if p is None or p.params.max_batch < batch:
        p = Plan(h, w, c, gc, radius, sigma_s, sigma_r, lam, max_batch=max(batch, 1), device=device,
                 pad=pad, backend=be, dt_iterations=dt_iterations)
        cache[key] = p
    return p


def _radius(radius, sigma_s):
    if radius is None:
        return int(math.ceil(3.0 * sigma_s))
    return int(radius)


class _Img:
    """Normalises an input image to a contiguous fp32 buffer + pointer."""

    def __init__(self, x, name="image"):
        self.torch = False
        self.orig_dtype = None
        try:
            import torch  # noqa: F401
            is_tensor = isinstance(x, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_tensor = False
        if is_tensor:
            import torch
            if not x.is_cuda:
                x = x.detach().cpu().numpy()
            else:
                self.torch = True
                self.orig_dtype = x.dtype
                self.t = x.detach().to(torch.float32).contiguous()
                self.shape = tuple(self.t.shape)
                self.device = self.t.device.index
                self.ptr = self.t.data_ptr()
        if not self.torch:
            a = np.asarray(x)
            if a.dtype.kind not in "fiu":
                raise InvalidArgument(_capi.BLFLS_EINVAL, f"{name}: numeric array required")
            self.orig_dtype = a.dtype if a.dtype.kind == "f" else np.dtype(np.float64)
            self.a = np.ascontiguousarray(a, dtype=np.float32)
            self.shape = self.a.shape
            self.device = None
            self.ptr = self.a.ctypes.data
        if len(self.shape) == 2:
            self.b, self.c, (self.h, self.w) = 1, 1, self.shape
        elif len(self.shape) == 3:
            self.b, (self.c, self.h, self.w) = 1, self.shape
        elif len(self.shape) == 4:
            self.b, self.c, self.h, self.w = self.shape
        else:
            raise InvalidArgument(_capi.BLFLS_EINVAL, f"{name}: expected (H,W), (C,H,W) or (B,C,H,W)")
        if self.c not in (1, 3):
            raise InvalidArgument(_capi.BLFLS_EINVAL, "PlanarImage: channels must be 1 or 3")

    def empty_like(self, shape=None):
        shape = self.shape if shape is None else shape
        if self.torch:
            import torch
            return torch.empty(shape, dtype=torch.float32, device=self.t.device)
        return np.empty(shape, dtype=np.float32)

    def finish(self, out):
        if self.torch:
            return out if self.orig_dtype == out.dtype else out.to(self.orig_dtype)
        return out.astype(self.orig_dtype, copy=False)


def _ptr(x):
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream_and_flags(img: _Img):
    if img.torch:
        import torch
        return C.c_void_p(torch.cuda.current_stream(img.t.device).cuda_stream), DEVICE_PTRS
    return C.c_void_p(0), HOST_PTRS


def _device(img: _Img, guide: _Img | None) -> int:
    if img.torch:
        if guide is not None and (not guide.torch or guide.device != img.device):
            raise InvalidArgument(_capi.BLFLS_EINVAL, "guide must live on the image's device")
        return img.device
    if guide is not None and guide.torch:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "guide must be host memory like the image")
    return 0


# ------------------------------------------------------------ entry points --

def blf_ls(image, guide=None, *, lam: float, sigma_s: float, sigma_r: float, iters: int = 1,
           radius: int | None = None, check_finite: bool = True, use_graph: bool = True,
           out=None, extra_flags: int = 0, wait: bool = True, pad: int = 0,
           backend: str = "brute", dt_iterations: int = 0):
    """BLF-LS: ``iters`` cascaded smooth() passes with the brute-force (joint) BLF.

    ``guide`` (optional) has 1 channel or the image's channel count and is held
    fixed over the iterations.  ``pad`` reflect-pads every smooth() input before
    the gradients and the solve and crops the result (SolveParams::pad,
    pipelines.cpp:76-92; the reference default is 16, the BASELINE configs
    use 0 = periodic).  ``backend="grid"`` filters the gradients with the
    bilateral grid the reference's smooth() runs (bilateral.cpp:112-207)
    instead of the brute-force window.  Returns the smoothed image in the input's type
    (written into ``out`` when given: an fp32 array/tensor of the image's shape
    in the same memory space, e.g. pinned host memory).

    ``wait=False`` with host memory (``out`` required, input already fp32
    contiguous) returns immediately: H2D, compute and D2H are queued on the
    plan's copy/compute streams so consecutive calls overlap; call
    ``get_plan(...).sync()`` (or ``sync_plans()``) before reading ``out``.
    With CUDA tensors the work is ordered on the current stream as always and
    only the non-finite check's verdict is deferred to that sync.
    """
    img = _Img(image)
    gd = None if guide is None else _Img(guide, "guide")
    if gd is not None:
        if (gd.h, gd.w) != (img.h, img.w) or gd.b != img.b or gd.c not in (1, img.c):
            raise InvalidArgument(_capi.BLFLS_EINVAL,
                                  "smooth: guidance image shape does not match input")
    r = _radius(radius, sigma_s) if backend == "brute" else 0
    dev = _device(img, gd)
    if int(pad) < 0:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "solver: pad must be >= 0")
    plan = get_plan(img.h, img.w, img.c, 0 if gd is None else gd.c, r, sigma_s, sigma_r, lam,
                    img.b, dev, pad=int(pad), backend=backend, dt_iterations=dt_iterations)
    if out is None:
        out = img.empty_like()
        finish = True
    else:
        if isinstance(out, np.ndarray):
            if img.torch or out.dtype != np.float32 or out.shape != tuple(img.shape) \
                    or not out.flags.c_contiguous:
                raise InvalidArgument(_capi.BLFLS_EINVAL, "out: fp32 host array of the image shape")
        else:
            import torch
            if out.dtype != torch.float32 or tuple(out.shape) != tuple(img.shape) \
                    or not out.is_contiguous() or out.is_cuda != img.torch:
                raise InvalidArgument(_capi.BLFLS_EINVAL, "out: fp32 tensor of the image shape")
            if not out.is_cuda:
                out = out.numpy()
        finish = False
    stream, flags = _stream_and_flags(img)
    if check_finite:
        flags |= CHECK_FINITE
    if not use_graph:
        flags |= NO_GRAPH
    flags |= int(extra_flags)
    if not wait and img.torch:
        # device tensors: ordered on the current stream as usual; only the
        # non-finite verdict is deferred to get_plan(...).sync() / sync_plans()
        flags |= ASYNC
    elif not wait:
        if img.torch or finish:
            raise InvalidArgument(_capi.BLFLS_EINVAL, "wait=False needs host memory and `out`")
        src = image.numpy() if hasattr(image, "numpy") and not isinstance(image, np.ndarray) else image
        if not (isinstance(src, np.ndarray) and src.dtype == np.float32 and src.flags.c_contiguous):
            raise InvalidArgument(_capi.BLFLS_EINVAL,
                                  "wait=False needs a contiguous fp32 input that outlives the call")
        flags |= ASYNC
    check(lib().blfls_run(plan.handle, img.ptr, None if gd is None else gd.ptr, img.b, int(iters),
                          _ptr(out), stream, flags))
    return img.finish(out) if finish else out


def sync_plans() -> None:
    """Wait for every plan of this thread (after ``blf_ls(..., wait=False)``)."""
    for p in getattr(_tls, "plans", {}).values():
        p.sync()


def nc_ls(image, guide=None, *, lam: float, sigma_s: float, sigma_r: float,
          dt_iterations: int = 3, iters: int = 1, pad: int = 0, **kw):
    """NC-LS: ``iters`` cascaded smooth() passes with SmootherKind::NC_LS, i.e.
    the gradients filtered by nc_filter (domain_transform.cpp:138-156) with
    DtParams{sigma_s, sigma_r, dt_iterations}; otherwise as ``blf_ls``."""
    if int(dt_iterations) < 1:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "nc_filter: iterations must be >= 1")
    return blf_ls(image, guide, lam=lam, sigma_s=sigma_s, sigma_r=sigma_r, iters=iters, pad=pad,
                  backend="dt", dt_iterations=int(dt_iterations), **kw)


def gaussian_blur(img, sigma: float):
    """``gaussian_blur`` (image.cpp:114-158) on the GPU: radius ceil(3 sigma),
    clamped borders, double accumulation; fp32 in and out."""
    im = _Img(img)
    out = im.empty_like()
    stream, flags = _stream_and_flags(im)
    dev = im.device if im.torch else 0
    check(lib().blfls_gaussian_blur(im.ptr, im.b * im.c, im.h, im.w, float(sigma), _ptr(out), dev,
                                    stream, flags))
    return im.finish(out)


def forward_gradients(img):
    """``forward_gradients`` (image.cpp:72-95): circular forward differences
    per channel; returns (gx, gy) in the input's type."""
    im = _Img(img)
    gx, gy = im.empty_like(), im.empty_like()
    stream, flags = _stream_and_flags(im)
    dev = im.device if im.torch else 0
    check(lib().blfls_forward_gradients(im.ptr, im.b * im.c, im.h, im.w, _ptr(gx), _ptr(gy), dev,
                                        stream, flags))
    return im.finish(gx), im.finish(gy)


def blf_brute(src, guide=None, params: RangeSpatialParams = None, *, radius: int | None = None):
    """``blf_brute`` (bilateral.cpp:28-77): the brute-force (joint) bilateral
    filter of arbitrary planes.  ``guide`` has 1 channel or ``src``'s count
    (None: ``src`` guides itself); the range distance is the Euclidean norm
    over the guide channels; ``radius`` None is the reference's ceil(3 sigma_s)."""
    params = params or RangeSpatialParams()
    img = _Img(src)
    gd = None if guide is None else _Img(guide, "guide")
    if gd is not None and ((gd.h, gd.w) != (img.h, img.w) or gd.b != img.b):
        raise InvalidArgument(_capi.BLFLS_EINVAL, "bilateral: src and guide dimensions differ")
    dev = _device(img, gd)
    out = img.empty_like()
    stream, flags = _stream_and_flags(img)
    check(lib().blfls_blf_brute(img.ptr, img.c, None if gd is None else gd.ptr,
                                img.c if gd is None else gd.c, img.h, img.w, img.b,
                                -1 if radius is None else int(radius), float(params.sigma_s),
                                float(params.sigma_r), _ptr(out), dev, stream,
                                flags | CHECK_FINITE))
    return img.finish(out)


def rolling_nc_ls(g, dt: DtParams, sp: SolveParams, rp: RollingParams):
    """``rolling_nc_ls`` (pipelines.cpp:96-117): NC_LS smoothing of the original
    input guided first by a Gaussian-blurred copy, then by the previous
    round's output."""
    if rp.n < 1:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "rolling_nc_ls: n must be >= 1")
    if not rp.init_sigma > 0.0:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "rolling_nc_ls: init_sigma must be positive")
    guide = gaussian_blur(g, rp.init_sigma)
    u = None
    for _ in range(rp.n):
        u = nc_ls(g, guide, lam=sp.lam, sigma_s=dt.sigma_s, sigma_r=dt.sigma_r,
                  dt_iterations=dt.iterations, pad=sp.pad)
        guide = u
    return u


def texture_removal(g, dt: DtParams, rp: RollingParams, sp: SolveParams):
    """applications.cpp:66-70."""
    return rolling_nc_ls(g, dt, sp, rp)


def clipart_cleanup(g, dt: DtParams, rp: RollingParams, sp: SolveParams):
    """applications.cpp:72-76."""
    return rolling_nc_ls(g, dt, sp, rp)


def smooth(g, spec: SmootherSpec):
    """``epls::smooth`` (pipelines.cpp:57-94) for kinds BLF_LS (brute-force BLF,
    or the grid with ``backend="grid"``), NC_LS and LS, including the
    reference's reflect padding ``spec.solve.pad`` (default 16)."""
    if spec.kind == SmootherKind.BLF_LS:
        return blf_ls(g, spec.guidance, lam=spec.solve.lam, sigma_s=spec.blf.sigma_s,
                      sigma_r=spec.blf.sigma_r, iters=1, radius=spec.radius, pad=spec.solve.pad,
                      backend=spec.backend)
    if spec.kind == SmootherKind.NC_LS:
        return nc_ls(g, spec.guidance, lam=spec.solve.lam, sigma_s=spec.dt.sigma_s,
                     sigma_r=spec.dt.sigma_r, dt_iterations=spec.dt.iterations,
                     pad=spec.solve.pad)
    if spec.kind == SmootherKind.LS:
        # affine-equivariant, so normalise/denormalise (pipelines.cpp:64,68) is the identity
        return ls_solve_fft(g, spec.solve)
    raise Unsupported(_capi.BLFLS_EUNSUPPORTED, f"smooth: {spec.kind} is out of scope")


def flash_no_flash(noflash, flash, spec: SmootherSpec):
    """``flash_no_flash`` (applications.cpp:58-64): joint smoothing guided by `flash`."""
    a, b = _Img(noflash), _Img(flash, "guide")
    if a.shape != b.shape:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "flash_no_flash: image shapes differ")
    s = SmootherSpec(spec.kind, spec.blf, spec.solve, flash, spec.radius, spec.backend, spec.dt)
    return smooth(noflash, s)


def filter_gradients(image, guide=None, *, sigma_s: float, sigma_r: float,
                     radius: int | None = None, backend: str = "brute", dt_iterations: int = 0):
    """Gradient targets of one smooth() call (pipelines.cpp:33-53: brute-force BLF,
    ``backend="grid"`` blf_grid, ``backend="dt"`` nc_filter with
    ``dt_iterations``), in the reference's normalised units.  Returns (tx, ty)."""
    img = _Img(image)
    gd = None if guide is None else _Img(guide, "guide")
    r = _radius(radius, sigma_s) if backend == "brute" else 0
    dev = _device(img, gd)
    plan = get_plan(img.h, img.w, img.c, 0 if gd is None else gd.c, r, sigma_s, sigma_r, 0.0,
                    img.b, dev, backend=backend, dt_iterations=dt_iterations)
    tx, ty = img.empty_like(), img.empty_like()
    stream, flags = _stream_and_flags(img)
    check(lib().blfls_filter_gradients(plan.handle, img.ptr, None if gd is None else gd.ptr, img.b,
                                       _ptr(tx), _ptr(ty), stream, flags | CHECK_FINITE))
    return img.finish(tx), img.finish(ty)


def lsgrad_solve_fft(g, target, params: SolveParams):
    """``lsgrad_solve_fft`` (solver.cpp:88-124); target = (tx, ty) or None; the image
    and targets are reflect-padded by ``params.pad`` and the result cropped."""
    if params.pad < 0:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "solver: pad must be >= 0")
    if not (params.lam >= 0.0) or not math.isfinite(params.lam):
        raise InvalidArgument(_capi.BLFLS_EINVAL, "solver: lambda must be finite and >= 0")
    img = _Img(g)
    txp = typ = None
    if target is not None:
        tx, ty = _Img(target[0], "target"), _Img(target[1], "target")
        if tx.shape != img.shape or ty.shape != img.shape:
            raise InvalidArgument(_capi.BLFLS_EINVAL,
                                  "lsgrad_solve_fft: target shape does not match image")
        txp, typ = tx.ptr, ty.ptr
    plan = get_plan(img.h, img.w, img.c, 0, 1, 1.0, 1.0, params.lam, img.b,
                    _device(img, None), pad=int(params.pad))
    out = img.empty_like()
    stream, flags = _stream_and_flags(img)
    check(lib().blfls_solve(plan.handle, img.ptr, txp, typ, img.b, _ptr(out), stream,
                            flags | CHECK_FINITE))
    return img.finish(out)


def ls_solve_fft(g, params: SolveParams):
    """``ls_solve_fft`` (solver.cpp:67-86)."""
    return lsgrad_solve_fft(g, None, params)


def rfft2(x):
    """``detail::rfft2`` of each plane: complex64 (…, H, W//2+1)."""
    img = _Img(x)
    plan = get_plan(img.h, img.w, img.c, 0, 1, 1.0, 1.0, 0.0, img.b, _device(img, None))
    shape = tuple(img.shape[:-1]) + (img.w // 2 + 1,)
    if img.torch:
        import torch
        out = torch.empty(shape, dtype=torch.complex64, device=img.t.device)
    else:
        out = np.empty(shape, dtype=np.complex64)
    stream, flags = _stream_and_flags(img)
    check(lib().blfls_rfft2(plan.handle, img.ptr, img.b, _ptr(out), stream, flags))
    return out


def irfft2(spec, width: int):
    """``detail::irfft2`` (with the 1/(H W) scaling) back to (…, H, width)."""
    is_t = False
    try:
        import torch
        is_t = isinstance(spec, torch.Tensor) and spec.is_cuda
    except ImportError:  # pragma: no cover
        pass
    if is_t:
        s = spec.to(torch.complex64).contiguous()
    else:
        s = np.ascontiguousarray(spec, dtype=np.complex64)
    shape = tuple(s.shape[:-1]) + (int(width),)
    if len(shape) == 2:
        b, c, h = 1, 1, shape[0]
    elif len(shape) == 3:
        b, (c, h) = 1, shape[:2]
    else:
        b, c, h = shape[:3]
    if s.shape[-1] != width // 2 + 1:
        raise InvalidArgument(_capi.BLFLS_EINVAL, "irfft2: spectrum width does not match")
    dev = s.device.index if is_t else 0
    plan = get_plan(h, width, c, 0, 1, 1.0, 1.0, 0.0, b, dev)
    if is_t:
        out = torch.empty(shape, dtype=torch.float32, device=s.device)
        stream, flags = C.c_void_p(torch.cuda.current_stream(s.device).cuda_stream), DEVICE_PTRS
    else:
        out = np.empty(shape, dtype=np.float32)
        stream, flags = C.c_void_p(0), HOST_PTRS
    check(lib().blfls_irfft2(plan.handle, _ptr(s), b, _ptr(out), stream, flags))
    return out


def generate(height: int, width: int, seeds, *, n_sites: int, noise_sigma: float = 0.03,
             p_salt_pepper: float = 0.0, device: int = 0):
    """BASELINE synthetic planes on the GPU: torch.float32 (len(seeds), H, W)."""
    import torch
    seeds = [int(s) for s in seeds]
    out = torch.empty((len(seeds), height, width), dtype=torch.float32, device=f"cuda:{device}")
    arr = (C.c_uint64 * len(seeds))(*seeds)
    stream = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    check(lib().blfls_generate(int(height), int(width), len(seeds), arr, int(n_sites),
                               float(noise_sigma), float(p_salt_pepper), out.data_ptr(), stream,
                               int(device)))
    return out
