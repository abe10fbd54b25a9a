"""Run one BASELINE config through blf_ls (for ncu captures): --config c5 --images 4 --reps 2."""
import argparse
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1812_07122_b200 as P
from paper_1812_07122_b200.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--images", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
n = a.images or cfg.batch
seeds = [s for i in range(n) for s in cfg.seeds(i)]
img = P.generate(cfg.height, cfg.width, seeds, n_sites=cfg.n_sites,
                 p_salt_pepper=cfg.p_salt_pepper).view(n, cfg.channels, cfg.height, cfg.width)
guide = None
if cfg.guide:
    guide = P.generate(cfg.height, cfg.width, [cfg.guide_seed(i) for i in range(n)],
                       n_sites=cfg.n_sites).view(n, 1, cfg.height, cfg.width)
for _ in range(a.reps):
    out = P.blf_ls(img, guide, lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r,
                   iters=cfg.iters, radius=cfg.radius, check_finite=False, use_graph=False)
torch.cuda.synchronize()
print("ok", tuple(out.shape), float(out.mean()))
