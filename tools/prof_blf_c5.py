"""One c5-shaped filter_gradients call (4 images of 2048^2 RGB, gray guide,
r = 7, sigma_r = 0.1) twice: the target of an ncu capture of the BLF kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1812_07122_b200 as P  # noqa: E402
from paper_1812_07122_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["c5"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
img = P.generate(cfg.height, cfg.width, [s for i in range(n) for s in cfg.seeds(i)],
                 n_sites=cfg.n_sites).view(n, 3, cfg.height, cfg.width)
guide = P.generate(cfg.height, cfg.width, [cfg.guide_seed(i) for i in range(n)],
                   n_sites=cfg.n_sites).view(n, 1, cfg.height, cfg.width)
for _ in range(2):
    P.filter_gradients(img, guide, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, radius=cfg.radius)
torch.cuda.synchronize()
print("ok")
