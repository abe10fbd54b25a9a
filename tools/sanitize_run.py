"""Exercise every kernel path on small inputs (for compute-sanitizer:
memcheck and racecheck, one tool per run; logs under profiles/)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1812_07122_b200 as P
from paper_1812_07122_b200.multigpu import band_rows, gpu_band_ops

rng = np.random.default_rng(0)
def img(c, h, w):
    return rng.random((c, h, w)).astype(np.float32)

kw = dict(lam=500.0, sigma_s=2.0, sigma_r=0.1)
P.blf_ls(img(1, 64, 64), iters=2, radius=5, **kw)                       # CT? no: RT sizes
P.blf_ls(img(3, 48, 80), iters=2, radius=7, **kw)
P.blf_ls(img(3, 40, 64), img(1, 40, 64), iters=2, radius=7, **kw)      # shared gray guide
P.blf_ls(img(3, 40, 64), img(3, 40, 64), iters=2, radius=5, **kw)      # per-channel guide
P.blf_ls(img(1, 45, 37), iters=2, radius=3, pad=3, **kw)                # padded, prime 43
P.blf_ls(img(1, 33, 35), iters=2, radius=9, **kw)                       # odd W, generic radius
P.blf_ls(img(1, 512, 512), iters=1, radius=5, **kw)                     # CT engine sizes
P.blf_ls(img(3, 128, 2048 // 8 * 8), iters=1, radius=3, **kw)
x = img(1, 30, 18)
P.irfft2(P.rfft2(x), 18)
P.lsgrad_solve_fft(x, (img(1, 30, 18), img(1, 30, 18)), P.SolveParams(10.0, 2))
P.filter_gradients(img(3, 40, 56), sigma_s=2.0, sigma_r=0.1, radius=4)
t = torch.from_numpy(img(1, 96, 128)).cuda()
fr, so = gpu_band_ops(96, 128, 1, 0, lam=500.0, sigma_s=2.0, sigma_r=0.1, radius=5, device=0)
for y0, y1 in band_rows(96, 3):
    fr(t, None, y0, y1)
P.generate(64, 64, [1, 2], n_sites=12, p_salt_pepper=0.05)
outs = [np.empty((3, 48, 64), np.float32) for _ in range(3)]
for o in outs:
    P.blf_ls(img(3, 48, 64), out=o, wait=False, iters=1, radius=5, **kw)
P.sync_plans()
# the other gradient filters and the padded host-pointer solve
P.blf_ls(img(3, 48, 64), iters=1, backend="grid", **kw)
P.blf_ls(img(3, 48, 64), img(1, 48, 64), iters=1, backend="grid", pad=4, **kw)
P.nc_ls(img(3, 40, 56), dt_iterations=2, **kw)
P.lsgrad_solve_fft(img(3, 30, 40), (img(3, 30, 40), img(3, 30, 40)), P.SolveParams(10.0, 16))
# the shared-guide and self-guided packed kernels at the c5 / c2 radius, both exponent forms
P.blf_ls(img(3, 64, 128), img(1, 64, 128), iters=1, radius=7, lam=1000.0, sigma_s=7.0, sigma_r=0.1)
P.blf_ls(img(3, 64, 128), img(1, 64, 128), iters=1, radius=7, lam=1000.0, sigma_s=7.0, sigma_r=0.05)
P.blf_ls(img(3, 64, 128), iters=1, radius=7, lam=1000.0, sigma_s=7.0, sigma_r=0.1)
# the single-process multi-GPU entry (two entries on device 0): batch and band
from paper_1812_07122_b200 import _capi
prm = _capi.Params(40, 64, 3, 1, 7, 7.0, 0.1, 1000.0, 3, 0, 0, 0, 0)
m = _capi.MultiPlan(prm, [0, 0], _capi.MULTI_BATCH)
m.run(img(9, 40, 64).reshape(3, 3, 40, 64), img(3, 40, 64).reshape(3, 1, 40, 64), 3, 2,
      np.empty((3, 3, 40, 64), np.float32))
prm = _capi.Params(96, 128, 1, 0, 15, 12.0, 0.08, 2000.0, 1, 0, 0, 0, 0)
m = _capi.MultiPlan(prm, [0, 0, 0], _capi.MULTI_BAND)
m.run(img(1, 96, 128), None, 1, 2, np.empty((1, 96, 128), np.float32))
torch.cuda.synchronize()
print("sanitize run ok")
