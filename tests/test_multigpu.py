"""Multi-GPU host logic on CPU: world_size 2 over gloo (127.0.0.1).

The band driver (paper_1812_07122_b200.multigpu.band_blf_ls) is run with
the CPU oracle standing in for the two device stages; its result must equal
the single-process oracle cascade.  The batch sharding is checked the same way.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1812_07122_b200.multigpu import band_blf_ls, band_rows, batch_shard  # noqa: E402

PRM = dict(lam=800.0, sigma_s=3.0, sigma_r=0.1, radius=4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_ops():
    from oracle import oracle as O

    def filter_rows(f, guide, y0, y1):
        g = f.double().numpy()
        gn, lo, hi = O.normalize_to_unit(g)
        rng = hi - lo
        if guide is not None:
            gd = guide.double().numpy()
            gdn, _, _ = O.normalize_to_unit(gd)
            gx_g, gy_g = O.forward_gradients(np.repeat(gdn, g.shape[0], axis=0) if gdn.shape[0] == 1 else gdn)
        gx, gy = O.forward_gradients(gn)
        if guide is None:
            gx_g, gy_g = gx, gy
        out = []
        for src, gd in ((gx, gx_g), (gy, gy_g)):
            t = np.stack([2.0 * O.blf_brute_r((src[c:c + 1] + 1) / 2, (gd[c:c + 1] + 1) / 2,
                                              sigma_s=PRM["sigma_s"], sigma_r=PRM["sigma_r"],
                                              radius=PRM["radius"])[0] - 1.0
                          for c in range(g.shape[0])])
            out.append(torch.from_numpy(t[:, y0:y1] * rng))
        return out[0], out[1]

    def solve(f, tx, ty):
        u = O.lsgrad_solve_fft(f.double().numpy(), tx.double().numpy(), ty.double().numpy(),
                               lam=PRM["lam"])
        return torch.from_numpy(u)

    return filter_rows, solve


def _band_worker(rank, world, port, img, guide, iters, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fr, so = oracle_ops()
        out = band_blf_ls(torch.from_numpy(img), None if guide is None else torch.from_numpy(guide),
                          iters, filter_rows=fr, solve=so)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, fn, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_band_rows_partition():
    for h in (5, 16, 17, 1080, 4096):
        for w in (1, 2, 3, 4, 8):
            if h < w:
                continue
            b = band_rows(h, w)
            assert b[0][0] == 0 and b[-1][1] == h
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert all(y1 > y0 for y0, y1 in b)
    with pytest.raises(ValueError):
        band_rows(3, 4)


def test_batch_shard_partition():
    for n in (1, 7, 64):
        for w in (1, 2, 3, 8):
            sh = [batch_shard(n, w, r) for r in range(w)]
            assert sh[0][0] == 0 and sh[-1][1] == n
            assert all(sh[i][1] == sh[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("h,w,c,guided", [(24, 20, 1, False), (23, 16, 3, True)])
def test_band_driver_world2_matches_cascade(oracle, h, w, c, guided):
    rng = np.random.default_rng(h * w)
    img = rng.random((c, h, w))
    guide = rng.random((1, h, w)) if guided else None
    res = _run(2, _band_worker, img, guide, 2)
    ref = oracle.blf_ls(img, guide, iters=2, **PRM)
    for r in (0, 1):
        assert np.abs(res[r] - ref).max() < 1e-10
    assert np.array_equal(res[0], res[1])


def _batch_worker(rank, world, port, imgs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        i0, i1 = batch_shard(imgs.shape[0], world, rank)
        mine = np.stack([O.blf_ls(imgs[i], iters=1, **PRM) for i in range(i0, i1)])
        per = -(-imgs.shape[0] // world)
        buf = torch.zeros((per,) + mine.shape[1:], dtype=torch.float64)
        buf[: mine.shape[0]] = torch.from_numpy(mine)
        allb = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(allb, buf)
        parts = [allb[r][: batch_shard(imgs.shape[0], world, r)[1] - batch_shard(imgs.shape[0], world, r)[0]]
                 for r in range(world)]
        q.put((rank, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def test_batch_sharding_world2(oracle):
    rng = np.random.default_rng(5)
    imgs = rng.random((3, 1, 16, 20))
    res = _run(2, _batch_worker, imgs)
    for i in range(3):
        ref = oracle.blf_ls(imgs[i], iters=1, **PRM)
        assert np.abs(res[0][i] - ref).max() == 0.0


def _batch_api_worker(rank, world, port, imgs, q):
    """Runs the real multigpu.batch_blf_ls host path (shard, all_gather over
    gloo, reassembly); the per-shard device call is replaced by the oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1812_07122_b200 import blfls
        from paper_1812_07122_b200.multigpu import batch_blf_ls

        def fake_blf_ls(images, guides, *, lam, sigma_s, sigma_r, iters, radius, backend="brute",
                        dt_iterations=0, pad=0):
            assert backend == "dt" and dt_iterations == 2 and guides is None
            outs = [O.nc_ls(images[i].numpy(), lam=lam, sigma_s=sigma_s, sigma_r=sigma_r,
                            dt_iters=dt_iterations, iters=iters, pad=pad)
                    for i in range(images.shape[0])]
            return torch.from_numpy(np.stack(outs))

        blfls.blf_ls = fake_blf_ls
        out, span = batch_blf_ls(torch.from_numpy(imgs), None, lam=500.0, sigma_s=3.0, sigma_r=0.1,
                                 iters=1, radius=0, gather=True, backend="dt", dt_iterations=2, pad=2)
        assert span == (0, imgs.shape[0])
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_batch_blf_ls_api_world2_dt_backend(oracle):
    rng = np.random.default_rng(9)
    imgs = rng.random((3, 1, 18, 22))
    res = _run(2, _batch_api_worker, imgs)
    for r in range(2):
        for i in range(3):
            ref = oracle.nc_ls(imgs[i], lam=500.0, sigma_s=3.0, sigma_r=0.1, dt_iters=2, pad=2)
            assert np.abs(res[r][i] - ref).max() == 0.0


class _SharedPeers:
    """CPU stand-in for GpuBandPeers: every rank's full-height targets live in
    shared-memory tensors all processes map (like NVLink peer buffers); the
    filter writes its band into all of them, dist.barrier is the device
    barrier."""

    def __init__(self, bufs, rank):
        self.bufs, self.rank = bufs, rank

    def filter(self, f, guide, y0, y1):
        fr, _ = oracle_ops()
        tx_b, ty_b = fr(f, guide, y0, y1)
        for b in self.bufs:
            b[0, :, y0:y1] = tx_b
            b[1, :, y0:y1] = ty_b

    def barrier(self):
        dist.barrier()

    def targets(self):
        b = self.bufs[self.rank]
        return b[0].clone(), b[1].clone()


def _band_peer_worker(rank, world, port, img, bufs, iters, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, so = oracle_ops()
        out = band_blf_ls(torch.from_numpy(img), None, iters, solve=so,
                          peers=_SharedPeers(bufs, rank))
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


def test_band_driver_peer_exchange_world2(oracle):
    """The fused-exchange band driver (peer stores + barriers, no collective)
    equals the single-process cascade on every rank."""
    rng = np.random.default_rng(11)
    img = rng.random((1, 24, 20))
    bufs = [torch.zeros((2, 1, 24, 20), dtype=torch.float64).share_memory_() for _ in range(2)]
    res = _run(2, _band_peer_worker, img, bufs, 2)
    ref = oracle.blf_ls(img, iters=2, **PRM)
    for r in range(2):
        assert np.abs(res[r] - ref).max() <= 1e-12
