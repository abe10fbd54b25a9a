"""Accuracy of the solve's column pass (run once per library: default = tridiagonal,
BLFLS_LIBRARY=..._lib_exp/libblfls.so BLFLS_COL_TRI=0 = column FFT pair):
max-abs error of lsgrad_solve_fft against a float64 numpy solve, and the
self-vs-self-guided difference of tests/test_gpu_parity.py."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1812_07122_b200 as P  # noqa: E402


def ref_solve(g, tx, ty, lam):
    h, w = g.shape[-2:]
    div = (np.roll(tx, 1, -1) - tx) + (np.roll(ty, 1, -2) - ty)
    u = np.arange(h)[:, None]
    v = np.arange(w // 2 + 1)[None, :]
    den = 1 + lam * (4 * np.sin(np.pi * u / h) ** 2 + 4 * np.sin(np.pi * v / w) ** 2)
    return np.fft.irfft2(np.fft.rfft2(g + lam * div) / den, s=(h, w))


print("library", os.environ.get("BLFLS_LIBRARY", "default"), "COL_TRI", os.environ.get("BLFLS_COL_TRI", "1"))
rng = np.random.default_rng(5)
for (h, w, lam) in [(512, 512, 1000.0), (1024, 1024, 1000.0), (1080, 1920, 500.0), (2048, 2048, 1000.0),
                    (4096, 4096, 2000.0), (1024, 1024, 1.0e5)]:
    g = np.cumsum(rng.standard_normal((1, h, w)), 1)
    g = ((g - g.min()) / (g.max() - g.min())).astype(np.float32)
    tx, ty = (rng.uniform(-0.05, 0.05, (2, 1, h, w))).astype(np.float32)
    u = P.lsgrad_solve_fft(g, (tx, ty), P.SolveParams(lam, 0))
    ref = ref_solve(g.astype(np.float64), tx.astype(np.float64), ty.astype(np.float64), lam)
    print(f"solve {h}x{w} lambda {lam:g}: max-abs {np.abs(u - ref).max():.3e}")
from oracle import oracle as O  # noqa: E402  (test infrastructure: the generator only)

g = np.stack([O.gen_plane(4 * 10 + k, 32, 40, n_sites=12, p_sp=0.0) for k in range(3)])
a = P.blf_ls(g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, iters=1, radius=4)
b = P.blf_ls(g, g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, iters=1, radius=4)
print(f"self vs guided-by-self (32x40x3, lambda 1024): max-abs {np.abs(np.asarray(a) - np.asarray(b)).max():.3e}")
