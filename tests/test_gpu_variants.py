"""Kernel-variant coverage on the GPU without environment knobs (the
production library ignores BLFLS_* variables; only a -DBLFLS_EXPERIMENTS
build reads them).  Every variant the default library selects at run time
is reached through inputs that make the library choose it:

- the column pass (k_col_tri.cu since r02; r01 switched between a pipelined
  and a plain column FFT on the spectrum size): the same images solved in a
  small batch and inside a larger batch must give the same bits.
- the exponent forms of the packed filters: factorised (XF) when
  2 range_coef^2 <= 60, i.e. sigma_r >= 0.07753, the difference form below
  (k_blf_j3.cu launch_j3, k_blf_p2.cu launch_p2).  Both sides of the switch
  are compared with the oracle, on images whose gradients reach +-range
  (binary stripes: the largest exponent argument 2 coef^2 the XF bound
  allows) and on the synthetic generator's images.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_OUT = 1e-4
TOL_TARGET = 2e-5
LOG2E = 1.4426950408889634
# sigma_r at which 2 range_coef^2 = 60, range_coef = sqrt(log2 e / (8 sigma_r^2))
SIGMA_R_SWITCH = math.sqrt(LOG2E / (8.0 * 30.0))


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def test_switch_constant():
    assert 0.0775 < SIGMA_R_SWITCH < 0.0776


def test_pipelined_and_plain_column_pass_agree(gpu, oracle):
    """1024-point columns: 2 RGB images alone and among 4 (r01: 6 planes x 4.3 MB
    of spectrum ran the pipelined column FFT, 12 planes the plain one; the
    tridiagonal column pass of r02 is one kernel, still batch-invariant)."""
    h = w = 1024
    imgs = np.stack([np.stack([oracle.gen_plane(600 + 10 * i + c, h, w, n_sites=12) for c in range(3)])
                     for i in range(4)]).astype(np.float32)
    kw = dict(lam=1000.0, sigma_s=3.0, sigma_r=0.1, iters=2, radius=3)
    small = gpu.blf_ls(imgs[:2], **kw)
    large = gpu.blf_ls(imgs, **kw)
    assert np.array_equal(small, large[:2])
    # and the plain solve stage against the oracle on one plane
    rng = np.random.default_rng(3)
    g = rng.random((1, 1024, 64)).astype(np.float32)
    tx, ty = rng.uniform(-0.2, 0.2, (2, 1, 1024, 64)).astype(np.float32)
    u = gpu.lsgrad_solve_fft(g, (tx, ty), gpu.SolveParams(1000.0, 0))
    assert maxabs(u, oracle.lsgrad_solve_fft(g, tx, ty, lam=1000.0)) <= 5e-5


def _stripes(h, w, period, phase=0):
    y, x = np.mgrid[0:h, 0:w]
    return (((x + y // 3 + phase) // period) % 2).astype(np.float64)


def _oracle_targets(oracle, img, guide, sigma_s, sigma_r, radius):
    """filter_gradients (pipelines.cpp:33-53) with brute force: per channel and
    axis, blf_brute on the (v+1)/2-remapped gradients, guided by the guide's
    gradient of the same axis (its only channel for a gray guide)."""
    gn, _, _ = oracle.normalize_to_unit(img)
    gx, gy = oracle.forward_gradients(gn)
    if guide is None:
        hx, hy = gx, gy
    else:
        hn, _, _ = oracle.normalize_to_unit(guide)
        hx, hy = oracle.forward_gradients(hn)
    out = []
    for src, gd in ((gx, hx), (gy, hy)):
        t = []
        for c in range(img.shape[0]):
            k = c if gd.shape[0] > 1 else 0
            t.append(2.0 * oracle.blf_brute_r((src[c:c + 1] + 1) / 2, (gd[k:k + 1] + 1) / 2,
                                              sigma_s=sigma_s, sigma_r=sigma_r, radius=radius)[0] - 1.0)
        out.append(np.stack(t))
    return out


@pytest.mark.parametrize("side", ["difference", "factorised"])
@pytest.mark.parametrize("kind", ["self", "joint_gray"])
@pytest.mark.parametrize("pattern", ["stripes", "generator"])
def test_exponent_form_switch_vs_oracle(gpu, oracle, side, kind, pattern):
    sr = SIGMA_R_SWITCH * (0.995 if side == "difference" else 1.005)
    h, w, r = 48, 80, 7
    if pattern == "stripes":
        # binary stripes: every gradient is 0 or +-(hi - lo)
        img = np.stack([_stripes(h, w, 2 + c, c) for c in range(3)])
        guide = _stripes(h, w, 3, 1)[None]
    else:
        img = np.stack([oracle.gen_plane(70 + c, h, w, n_sites=12) for c in range(3)]).astype(np.float64)
        guide = oracle.gen_plane(90, h, w, n_sites=12)[None].astype(np.float64)
    if kind == "self":
        guide = None
    img32 = img.astype(np.float32)
    g32 = None if guide is None else guide.astype(np.float32)
    tx, ty = gpu.filter_gradients(img32, g32, sigma_s=7.0, sigma_r=sr, radius=r)
    rx, ry = _oracle_targets(oracle, img32.astype(np.float64),
                             None if guide is None else g32.astype(np.float64), 7.0, sr, r)
    assert maxabs(tx, rx) <= TOL_TARGET
    assert maxabs(ty, ry) <= TOL_TARGET
    out = gpu.blf_ls(img32, g32, lam=1000.0, sigma_s=7.0, sigma_r=sr, iters=2, radius=r)
    ref = oracle.blf_ls(img32.astype(np.float64), None if guide is None else g32.astype(np.float64),
                        lam=1000.0, sigma_s=7.0, sigma_r=sr, iters=2, radius=r)
    assert maxabs(out, ref) <= TOL_OUT


def test_tma_row_c2r_matches_plain(gpu, oracle):
    """The row c2r streams its spectrum rows through TMA bulk copies
    (k2_row_c2r_tma) when a launch's spectra exceed 64 MB: 10 planes of
    2048^2 (166 MB of spectra) -> the TMA pass; the same planes two at a
    time (33 MB) -> k2_row_c2r.  Bit-identical images (and hence the fused
    min/max)."""
    import torch
    h = w = 2048
    rng = np.random.default_rng(11)
    g = torch.from_numpy(rng.random((10, 1, h, w), dtype=np.float32)).cuda()
    tx = (torch.rand_like(g) - 0.5) * 0.1
    ty = (torch.rand_like(g) - 0.5) * 0.1
    big = gpu.lsgrad_solve_fft(g, (tx, ty), gpu.SolveParams(1000.0, 0))
    for i in range(0, 10, 2):
        small = gpu.lsgrad_solve_fft(g[i:i + 2].contiguous(), (tx[i:i + 2].contiguous(), ty[i:i + 2].contiguous()),
                                     gpu.SolveParams(1000.0, 0))
        assert torch.equal(small, big[i:i + 2]), i
    ref = oracle.lsgrad_solve_fft(g[3].cpu().numpy(), tx[3].cpu().numpy(), ty[3].cpu().numpy(), lam=1000.0)
    assert maxabs(big[3].cpu().numpy(), ref) <= 5e-5
