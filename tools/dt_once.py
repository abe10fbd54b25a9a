"""One NC-LS (DT backend) smooth at a BASELINE config (for ncu launch lists):
python tools/dt_once.py [config] [images]."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1812_07122_b200 as P  # noqa: E402
from paper_1812_07122_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
img = torch.rand(n, cfg.channels, cfg.height, cfg.width, device="cuda")
guide = torch.rand(n, 1, cfg.height, cfg.width, device="cuda") if cfg.guide else None
kw = {"use_graph": False} if os.environ.get("DT_NOGRAPH") else {}
for _ in range(2):
    P.nc_ls(img, guide, lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, **kw)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    P.nc_ls(img, guide, lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, **kw)
b.record()
torch.cuda.synchronize()
print(f"{a.elapsed_time(b) / 5:.3f} ms per smooth ({n} images)")
