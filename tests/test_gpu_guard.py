"""Out-of-bounds checks without compute-sanitizer (closed on the GPU pool):
every device input and output of the C-ABI entry points lives inside a
larger buffer whose guard regions (1 MiB before and after) hold NaN.  A
kernel that reads outside its input pulls NaN into a finite result; one that
writes outside its output overwrites a guard.  Both are checked on the
paths that use atomics (bilateral grid splat), peer stores (fused band
exchange), ordered-integer min/max epilogues and the multi-GPU entry."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 1 << 18  # floats (1 MiB) on each side


class Guarded:
    def __init__(self, shape, fill=None):
        import torch
        n = int(np.prod(shape))
        self.buf = torch.full((n + 2 * GUARD,), float("nan"), device="cuda")
        self.t = self.buf[GUARD:GUARD + n].view(*shape)
        if fill is not None:
            self.t.copy_(torch.as_tensor(fill, device="cuda"))

    def guards_intact(self):
        import torch
        torch.cuda.synchronize()
        return bool(torch.isnan(self.buf[:GUARD]).all()) and bool(torch.isnan(self.buf[-GUARD:]).all())


def _img(oracle, c, h, w, seed):
    return np.stack([oracle.gen_plane(seed * 10 + k, h, w, n_sites=12) for k in range(c)]).astype(np.float32)


@pytest.mark.parametrize("backend,guide,r,sr", [("brute", 0, 7, 0.1), ("brute", 1, 7, 0.1), ("brute", 1, 7, 0.05),
                                                ("brute", 0, 5, 0.05), ("brute", 3, 5, 0.1), ("brute", 0, 15, 0.08),
                                                ("grid", 0, 0, 0.1), ("grid", 1, 0, 0.1), ("dt", 0, 0, 0.1)])
def test_blf_ls_stays_in_bounds(gpu, oracle, backend, guide, r, sr):
    import torch
    b, c, h, w = 2, 3, 72, 136
    x = Guarded((b, c, h, w), np.stack([_img(oracle, c, h, w, 3 + i) for i in range(b)]))
    g = None
    if guide:
        g = Guarded((b, guide, h, w), np.stack([_img(oracle, guide, h, w, 9 + i) for i in range(b)]))
    out = Guarded((b, c, h, w))
    kw = dict(lam=1000.0, sigma_s=3.0 if backend != "brute" else float(r), sigma_r=sr, iters=2,
              backend=backend)
    if backend == "brute":
        kw["radius"] = r
    gpu.blf_ls(x.t, None if g is None else g.t, out=out.t, **kw)
    torch.cuda.synchronize()
    assert out.guards_intact() and x.guards_intact()
    assert bool(torch.isfinite(out.t).all())


def test_stage_entry_points_stay_in_bounds(gpu, oracle):
    import torch
    c, h, w = 3, 64, 96
    x = Guarded((c, h, w), _img(oracle, c, h, w, 21))
    g = Guarded((1, h, w), _img(oracle, 1, h, w, 22))
    tx, ty = gpu.filter_gradients(x.t, g.t, sigma_s=7.0, sigma_r=0.1, radius=7)
    assert bool(torch.isfinite(tx).all()) and bool(torch.isfinite(ty).all())
    gtx = Guarded((c, h, w), tx)
    gty = Guarded((c, h, w), ty)
    u = gpu.lsgrad_solve_fft(x.t, (gtx.t, gty.t), gpu.SolveParams(1000.0, 0))
    assert bool(torch.isfinite(u).all())
    for t in (x, g, gtx, gty):
        assert t.guards_intact()


@pytest.mark.parametrize("nb", [2, 3])
def test_peer_store_epilogue_stays_in_bounds(gpu, oracle, nb):
    """blfls_filter_gradients_rows_peers: every band stores into nb full-height
    destination buffers (the fused band exchange), none outside them."""
    import ctypes as C

    import torch

    from paper_1812_07122_b200 import _capi
    from paper_1812_07122_b200.blfls import get_plan
    from paper_1812_07122_b200.multigpu import band_rows
    c, h, w = 1, 96, 128
    x = Guarded((c, h, w), _img(oracle, c, h, w, 31))
    plan = get_plan(h, w, c, 0, 15, 12.0, 0.08, 2000.0, 1, 0)
    dst = [(Guarded((c, h, w)), Guarded((c, h, w))) for _ in range(nb)]
    txp = (C.c_void_p * nb)(*[d[0].t.data_ptr() for d in dst])
    typ = (C.c_void_p * nb)(*[d[1].t.data_ptr() for d in dst])
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for y0, y1 in band_rows(h, nb):
        _capi.check(_capi.lib().blfls_filter_gradients_rows_peers(plan.handle, x.t.data_ptr(), None, y0, y1,
                                                                  txp, typ, nb, st, _capi.DEVICE_PTRS))
    torch.cuda.synchronize()
    for a, b_ in dst:
        assert a.guards_intact() and b_.guards_intact()
        assert bool(torch.isfinite(a.t).all()) and bool(torch.isfinite(b_.t).all())
        assert torch.equal(a.t, dst[0][0].t) and torch.equal(b_.t, dst[0][1].t)
