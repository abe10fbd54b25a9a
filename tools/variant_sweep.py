"""Time the BLF stage of a config under kernel-variant env settings.
usage: variant_sweep.py CONFIG IMAGES 'ENV=V,ENV2=V' 'ENV=V' ..."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1812_07122_b200 as P
from paper_1812_07122_b200 import _capi, blfls
from paper_1812_07122_b200.configs import CONFIGS

cfg = CONFIGS[sys.argv[1]]
n = int(sys.argv[2]) or cfg.batch
seeds = [s for i in range(n) for s in cfg.seeds(i)]
img = P.generate(cfg.height, cfg.width, seeds, n_sites=cfg.n_sites,
                 p_salt_pepper=cfg.p_salt_pepper).view(n, cfg.channels, cfg.height, cfg.width)
guide = None
if cfg.guide:
    guide = P.generate(cfg.height, cfg.width, [cfg.guide_seed(i) for i in range(n)],
                       n_sites=cfg.n_sites).view(n, 1, cfg.height, cfg.width)
base = None
for spec in sys.argv[3:]:
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k in list(os.environ):
        if k.startswith("BLFLS_"):
            del os.environ[k]
    os.environ.update(env)
    blfls._tls.plans = {}
    kw = dict(lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, iters=cfg.iters,
              radius=cfg.radius, check_finite=False)
    out = P.blf_ls(img, guide, **kw)
    for _ in range(2):
        P.blf_ls(img, guide, **kw)
    plan = P.get_plan(cfg.height, cfg.width, cfg.channels, 1 if cfg.guide else 0, cfg.radius,
                      cfg.sigma_s, cfg.sigma_r, cfg.lam, n, 0)
    plan.stage_times()
    for _ in range(3):
        P.blf_ls(img, guide, extra_flags=_capi.TIME_STAGES, **kw)
    torch.cuda.synchronize()
    ms, cnt = plan.stage_times()
    st = plan.stats()
    blf = ms[1] / cnt[1]
    rate = st.exps / st.blf_launches / (blf * 1e-3) / 1e9
    if base is None:
        base = out
    drift = (out - base).abs().max().item()
    print(f"{cfg.name} [{spec:32s}] blf {blf:8.3f} ms {rate:7.0f} Gexp/s ({rate/4624:.3f} of MUFU) "
          f"solve {sum(ms[2:5])/cnt[2]:.3f} ms/iter drift {drift:.2e}", flush=True)
