"""Measured GPU-vs-oracle errors of the NC-LS / rolling paths (for the test
tolerances): python tools/nc_errors.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1812_07122_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def img(c, h, w, seed):
    return np.stack([O.gen_plane(seed * 10 + k, h, w, n_sites=12) for k in range(c)])


for (c, h, w, ss, sr, pad) in [(3, 64, 80, 8.0, 0.02, 16), (1, 128, 128, 12.0, 0.05, 0),
                               (3, 96, 96, 4.0, 0.1, 16)]:
    g = img(c, h, w, h + w)
    a = P.nc_ls(g, lam=1024.0, sigma_s=ss, sigma_r=sr, pad=pad)
    b = O.nc_ls(g.astype(np.float64), lam=1024.0, sigma_s=ss, sigma_r=sr, pad=pad)
    print(f"nc_ls {c}x{h}x{w} ss={ss} sr={sr} pad={pad}: max {np.abs(a - b).max():.3e} "
          f"mean {np.abs(a - b).mean():.3e}")
    for n, s0 in ((3, 2.5), (2, 0.75)):
        a = P.rolling_nc_ls(g, P.DtParams(ss, sr, 3), P.SolveParams(1024.0, pad), P.RollingParams(n, s0))
        b = O.rolling_nc_ls(g.astype(np.float64), lam=1024.0, sigma_s=ss, sigma_r=sr, pad=pad, n=n,
                            init_sigma=s0)
        d = np.abs(a - b)
        print(f"  rolling n={n} s0={s0}: max {d.max():.3e} mean {d.mean():.3e} "
              f"frac>1e-4 {(d > 1e-4).mean():.2e}")
