"""Max-abs error of the GPU path against the CPU oracle at every BASELINE
configuration at full size (c5: images 0 and 63 of the 64-image batch), per
iteration count; writes one line per config (profiles/r01_parity_errors.txt)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1812_07122_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

for name in ["c1", "c2", "c3", "c4", "c5"]:
    cfg = P.CONFIGS[name]
    n = cfg.batch
    planes = [s for i in range(n) for s in cfg.seeds(i)]
    img = P.generate(cfg.height, cfg.width, planes, n_sites=cfg.n_sites,
                     p_salt_pepper=cfg.p_salt_pepper).view(n, cfg.channels, cfg.height, cfg.width)
    guide = None
    if cfg.guide:
        guide = P.generate(cfg.height, cfg.width, [cfg.guide_seed(i) for i in range(n)],
                           n_sites=cfg.n_sites).view(n, 1, cfg.height, cfg.width)
    out = P.blf_ls(img, guide, lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, iters=cfg.iters,
                   radius=cfg.radius)
    torch.cuda.synchronize()
    for i in sorted({0, n - 1}):
        t0 = time.time()
        ref = O.blf_ls(img[i].cpu().numpy().astype(np.float64),
                       None if guide is None else guide[i].cpu().numpy().astype(np.float64),
                       lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, iters=cfg.iters,
                       radius=cfg.radius)
        err = np.abs(out[i].cpu().numpy().astype(np.float64) - ref)
        print(f"{name} image {i}/{n}: {cfg.channels}x{cfg.height}x{cfg.width} r={cfg.radius} iters={cfg.iters} "
              f"max-abs {err.max():.3e} mean-abs {err.mean():.3e} (gate 1e-4; oracle {time.time() - t0:.1f} s)",
              flush=True)
