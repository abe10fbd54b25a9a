"""Diagnostic: per-iteration GPU vs oracle error for a multi-iteration case."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1812_07122_b200 as P
from oracle import oracle as O

def run(c, h, w, r, ss, sr, lam, iters, seed):
    img = np.stack([O.gen_plane(seed * 10 + k, h, w, n_sites=12) for k in range(c)])
    f_o = img.astype(np.float64)
    f_g = img.copy()
    print(f"case c={c} {h}x{w} r={r} ss={ss} sr={sr} lam={lam}")
    for k in range(iters):
        f_o1 = O.blf_ls(f_o, lam=lam, sigma_s=ss, sigma_r=sr, iters=1, radius=r)
        f_g1 = P.blf_ls(f_g, lam=lam, sigma_s=ss, sigma_r=sr, iters=1, radius=r)
        # same input to both: isolates the per-iteration error
        g_from_o = P.blf_ls(f_o.astype(np.float32), lam=lam, sigma_s=ss, sigma_r=sr, iters=1, radius=r)
        tx, ty = P.filter_gradients(f_o.astype(np.float32), sigma_s=ss, sigma_r=sr, radius=r)
        gn, lo, hi = O.normalize_to_unit(f_o)
        gx, gy = O.forward_gradients(gn)
        rx = 2 * O.blf_brute_r((gx + 1) / 2, (gx + 1) / 2, sigma_s=ss, sigma_r=sr, radius=r) - 1
        print(f" it{k}: range [{f_o.min():.4f},{f_o.max():.4f}] chain err {np.abs(f_g1-f_o1).max():.2e} "
              f"same-input err {np.abs(g_from_o-f_o1).max():.2e} tx err {np.abs(tx-rx).max():.2e} "
              f"|tx| {np.abs(rx).max():.3f}")
        f_o, f_g = f_o1, f_g1
    full = P.blf_ls(img, lam=lam, sigma_s=ss, sigma_r=sr, iters=iters, radius=r)
    print(f" fused {iters} iters err {np.abs(full - f_o).max():.2e}")

run(1, 60, 50, 15, 12.0, 0.08, 2000.0, 2, 1 + 60 + 7)
run(1, 32, 40, 3, 2.0, 0.1, 1000.0, 2, 9)
run(3, 48, 80, 7, 7.0, 0.1, 1000.0, 3, 7 + 3 + 48)

def ranges(c, h, w, r, ss, sr, lam, iters, seed, graph=True):
    img = np.stack([O.gen_plane(seed * 10 + k, h, w, n_sites=12) for k in range(c)])
    out = P.blf_ls(img, lam=lam, sigma_s=ss, sigma_r=sr, iters=iters, radius=r, use_graph=graph)
    plan = P.get_plan(h, w, c, 0, r, ss, sr, lam, 1, 0)
    one = P.blf_ls(img, lam=lam, sigma_s=ss, sigma_r=sr, iters=1, radius=r)
    print(f" graph={graph} ranges {plan.debug_ranges()} true range after it0 [{one.min():.6f},{one.max():.6f}]")

ranges(1, 32, 40, 3, 2.0, 0.1, 1000.0, 2, 9)
ranges(1, 32, 40, 3, 2.0, 0.1, 1000.0, 2, 9, graph=False)
ranges(3, 48, 80, 7, 7.0, 0.1, 1000.0, 2, 58)
