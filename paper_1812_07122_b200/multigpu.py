"""Multi-GPU drivers: one process per GPU, torch.distributed for the plumbing.

Two decompositions:

* **batch** (config 5): the images of a batch are independent units; each
  rank smooths its shard (contiguous block of the batch) with no data-path
  collective.  `gather=True` all-gathers the results.
* **band** (config 4, one huge image): each rank filters the gradients of a
  row band ``[y0, y1)`` of the full image (blfls_filter_gradients_rows: the
  BLF window reads the full image, clips at the global top/bottom, and gy
  wraps at y = H-1), the bands are all-gathered (NCCL over NVLink), and every
  rank runs the (cheap) full-image FFT solve redundantly, so each rank holds
  the whole next iterate and the next iteration needs no halo exchange.  The
  per-image min/max of the normalisation is computed locally on the full
  image (identical on every rank).

The band driver is written against two callables so its host logic
(partition, padding, gather order, iteration) is tested on CPU with the
`gloo` backend (tests/test_multigpu.py); the GPU binding below plugs in the
C-ABI entry points.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Callable, Sequence

__all__ = ["band_rows", "band_blf_ls", "batch_shard", "batch_blf_ls", "gpu_band_ops"]


def _all_gather(out, inp, group):
    """out[r] = inp of rank r.  NCCL: one all_gather_into_tensor (NVLink /
    NVSwitch); other backends (gloo, CPU tests): the list form."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), inp, group=group)


def band_rows(height: int, world: int) -> list[tuple[int, int]]:
    """Row bands of (almost) equal height; every band is non-empty when
    height >= world.  Band b = rows [y0, y1)."""
    if world < 1 or height < world:
        raise ValueError("band_rows: need 1 <= world <= height")
    per = math.ceil(height / world)
    out = []
    for b in range(world):
        y0 = min(b * per, height)
        y1 = min(y0 + per, height)
        out.append((y0, y1))
    if any(y1 <= y0 for y0, y1 in out):
        # fall back to the balanced split (e.g. height=5, world=4)
        base, extra = divmod(height, world)
        out, y = [], 0
        for b in range(world):
            h = base + (1 if b < extra else 0)
            out.append((y, y + h))
            y += h
    return out


def batch_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [i0, i1) of a batch for `rank` (balanced)."""
    base, extra = divmod(batch, world)
    i0 = rank * base + min(rank, extra)
    return i0, i0 + base + (1 if rank < extra else 0)


def band_blf_ls(f0, guide, iters: int, *, filter_rows: Callable = None, solve: Callable,
                group=None, xp=None, peers=None):
    """Band-decomposed BLF-LS cascade.

    f0: the full image (C, H, W) on this rank (every rank holds it).
    filter_rows(f, guide, y0, y1) -> (tx_band, ty_band) of shape (C, y1-y0, W)
        targets of the band in RAW units (blfls_filter_gradients_rows); the
        bands are then all-gathered (NCCL over NVLink / NVSwitch, gloo on CPU).
    peers: the fused exchange instead (blfls_filter_gradients_rows_peers): an
        object with .filter(f, guide, y0, y1) that stores the band's targets
        straight into every rank's full-height buffers, .barrier() (all ranks'
        stores visible / all ranks done reading) and .targets() -> (tx, ty)
        of this rank; no separate collective.
    solve(f, tx, ty) -> next full image (blfls_solve).
    Returns the final full image (identical on every rank).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    C_, H, W = f0.shape
    bands = band_rows(H, world)
    hb = max(y1 - y0 for y0, y1 in bands)
    f = f0
    for _ in range(iters):
        y0, y1 = bands[rank]
        if peers is not None:
            peers.barrier()  # every rank finished reading the previous targets
            peers.filter(f, guide, y0, y1)
            peers.barrier()  # every band's targets landed in every rank's buffers
            tx, ty = peers.targets()
            f = solve(f, tx, ty)
            continue
        tx_b, ty_b = filter_rows(f, guide, y0, y1)
        # pad to the common band height so all ranks contribute equal chunks
        pad = torch.zeros((2, C_, hb, W), dtype=f.dtype, device=f.device)
        pad[0, :, : y1 - y0] = tx_b
        pad[1, :, : y1 - y0] = ty_b
        if world > 1:
            gathered = torch.empty((world, 2, C_, hb, W), dtype=f.dtype, device=f.device)
            _all_gather(gathered, pad.contiguous(), group)
        else:
            gathered = pad[None]
        tx = torch.cat([gathered[b, 0, :, : y1b - y0b] for b, (y0b, y1b) in enumerate(bands)], dim=1)
        ty = torch.cat([gathered[b, 1, :, : y1b - y0b] for b, (y0b, y1b) in enumerate(bands)], dim=1)
        f = solve(f, tx.contiguous(), ty.contiguous())
    return f


class GpuBandPeers:
    """Fused band exchange on CUDA: tx / ty live in symmetric memory
    (torch.distributed._symmetric_memory: every rank maps every peer's
    buffer over NVLink), blfls_filter_gradients_rows_peers stores each band's
    targets into all of them from the filter kernel's epilogue, and the
    symmetric-memory device barrier orders the stores against the solve."""

    def __init__(self, plan, channels, height, width, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        from . import _capi
        self.plan, self.lib, self._capi = plan, _capi.lib(), _capi
        self.device = device
        group = group or dist.group.WORLD
        n = channels * height * width
        self.buf = symm.empty((2, channels, height, width), dtype=torch.float32, device=device)
        self.hdl = symm.rendezvous(self.buf, group)
        ptrs = list(self.hdl.buffer_ptrs)
        self.np = len(ptrs)
        self.txp = (C.c_void_p * self.np)(*[p for p in ptrs])
        self.typ = (C.c_void_p * self.np)(*[p + 4 * n for p in ptrs])

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def filter(self, f, guide, y0, y1):
        self._capi.check(self.lib.blfls_filter_gradients_rows_peers(
            self.plan.handle, f.data_ptr(), None if guide is None else guide.data_ptr(), y0, y1,
            self.txp, self.typ, self.np, self._stream(), self._capi.DEVICE_PTRS))

    def barrier(self):
        self.hdl.barrier(channel=0)

    def targets(self):
        return self.buf[0], self.buf[1]


def batch_blf_ls(images, guides, *, lam, sigma_s, sigma_r, iters, radius, group=None,
                 gather=False, **kw):
    """Batch-sharded BLF-LS: rank r smooths images[i0:i1] of the full batch
    (every rank passes the same full batch, or only needs its shard).  Extra
    keywords go to ``blf_ls`` (``pad``, ``backend="grid"|"dt"``,
    ``dt_iterations``): images are independent under every gradient filter."""
    import torch
    import torch.distributed as dist

    from .blfls import blf_ls
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    i0, i1 = batch_shard(images.shape[0], world, rank)
    out = blf_ls(images[i0:i1], None if guides is None else guides[i0:i1], lam=lam,
                 sigma_s=sigma_s, sigma_r=sigma_r, iters=iters, radius=radius, **kw)
    if not gather or world == 1:
        return out, (i0, i1)
    per = math.ceil(images.shape[0] / world)
    buf = torch.zeros((per,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    buf[: out.shape[0]] = out
    allb = torch.empty((world, per) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    _all_gather(allb, buf, group)
    parts = [allb[r, : batch_shard(images.shape[0], world, r)[1] - batch_shard(images.shape[0], world, r)[0]]
             for r in range(world)]
    return torch.cat(parts, dim=0), (0, images.shape[0])


def gpu_band_ops(height, width, channels, guide_channels, *, lam, sigma_s, sigma_r, radius,
                 device, fused=False, group=None):
    """(filter_rows, solve) bound to the C ABI on CUDA `device` for band_blf_ls;
    fused=True returns (GpuBandPeers, solve) for the fused peer-store exchange
    and raises when symmetric memory is unavailable (use fused=False for the
    NCCL all-gather exchange)."""
    import torch

    from . import _capi
    from .blfls import get_plan
    plan = get_plan(height, width, channels, guide_channels, radius, sigma_s, sigma_r, lam, 1,
                    device)
    L = _capi.lib()

    def stream():
        return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)

    def filter_rows(f, guide, y0, y1):
        tx = torch.empty((channels, y1 - y0, width), dtype=torch.float32, device=f.device)
        ty = torch.empty_like(tx)
        _capi.check(L.blfls_filter_gradients_rows(plan.handle, f.data_ptr(),
                                                  None if guide is None else guide.data_ptr(),
                                                  y0, y1, tx.data_ptr(), ty.data_ptr(), stream(),
                                                  _capi.DEVICE_PTRS))
        return tx, ty

    def solve(f, tx, ty):
        u = torch.empty_like(f)
        _capi.check(L.blfls_solve(plan.handle, f.data_ptr(), tx.data_ptr(), ty.data_ptr(), 1,
                                  u.data_ptr(), stream(), _capi.DEVICE_PTRS))
        return u

    if fused:
        # no silent fallback: a failed symmetric-memory rendezvous raises; the
        # caller picks the all-gather exchange explicitly (fused=False)
        return GpuBandPeers(plan, channels, height, width, device, group), solve
    return filter_rows, solve
