"""Sweep the SFU-offload period of k_grad_blf: BLF launch time and output drift."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1812_07122_b200 as P
from paper_1812_07122_b200 import _capi, blfls
from paper_1812_07122_b200.configs import CONFIGS, Config

cases = [CONFIGS["c2"], CONFIGS["c3"],
         Config("c4s", 4, 2048, 2048, 1, 1, 15, 12.0, 0.08, 2000.0, 2, n_sites=64),
         Config("c5s", 5, 2048, 2048, 3, 4, 7, 7.0, 0.1, 1000.0, 3, guide=True)]
for cfg in cases:
    n = cfg.batch
    seeds = [s for i in range(n) for s in cfg.seeds(i)]
    img = P.generate(cfg.height, cfg.width, seeds, n_sites=cfg.n_sites,
                     p_salt_pepper=cfg.p_salt_pepper).view(n, cfg.channels, cfg.height, cfg.width)
    guide = None
    if cfg.guide:
        guide = P.generate(cfg.height, cfg.width, [cfg.guide_seed(i) for i in range(n)],
                           n_sites=cfg.n_sites).view(n, 1, cfg.height, cfg.width)
    base = None
    for period in (0, 4, 5, 6, 8, 12, -1):
        os.environ["BLFLS_POLY_PERIOD"] = str(period)
        blfls._tls.plans = {}
        kw = dict(lam=cfg.lam, sigma_s=cfg.sigma_s, sigma_r=cfg.sigma_r, iters=cfg.iters,
                  radius=cfg.radius, check_finite=False)
        out = P.blf_ls(img, guide, **kw)
        for _ in range(3):
            P.blf_ls(img, guide, **kw)
        plan = P.get_plan(cfg.height, cfg.width, cfg.channels, 1 if cfg.guide else 0, cfg.radius,
                          cfg.sigma_s, cfg.sigma_r, cfg.lam, n, 0)
        plan.stage_times()
        for _ in range(5):
            P.blf_ls(img, guide, extra_flags=_capi.TIME_STAGES, **kw)
        torch.cuda.synchronize()
        ms, cnt = plan.stage_times()
        st = plan.stats()
        blf = ms[1] / cnt[1]
        rate = st.exps / st.blf_launches / (blf * 1e-3) / 1e9
        if base is None:
            base = out
        drift = (out - base).abs().max().item()
        print(f"{cfg.name} period={period:3d} blf {blf:.3f} ms  {rate:7.0f} Gexp/s  drift {drift:.2e}",
              flush=True)
print("mufu peak", _capi.mufu_peak(0))
