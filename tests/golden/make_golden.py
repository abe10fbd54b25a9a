"""Regenerate tests/golden/*.npz from the REFERENCE translation units.

Run here (needs /root/reference for oracle/_ref):  python tests/golden/make_golden.py
Each file holds the fp32 input (and guide) and the double-precision output of
the reference pipeline pieces (oracle/ref_shim/ref_capi.cpp:ref_blf_ls), plus
one iteration's filter_gradients targets.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE))

from cases import CASES, GRID_CASES, NC_CASES  # noqa: E402
from oracle import oracle as O  # noqa: E402


def scene(kind, w, h, c, seed):
    if kind == "natural":
        return O.ref_natural_scene(w, h, c, seed)
    if kind == "random":
        return O.ref_random_image(w, h, c, seed)
    if kind == "constant":
        return np.full((c, h, w), 0.55)
    raise ValueError(kind)


def main():
    for cs in CASES:
        img = scene(cs["scene"], cs["w"], cs["h"], cs["c"], cs["seed"]).astype(np.float32)
        guide = None
        if cs["guide"] is not None:
            kind, seed, gc = cs["guide"]
            guide = scene(kind, cs["w"], cs["h"], gc, seed).astype(np.float32)
        out = O.ref_blf_ls(img.astype(np.float64), None if guide is None else guide.astype(np.float64),
                           lam=cs["lam"], sigma_s=cs["sigma_s"], sigma_r=cs["sigma_r"],
                           iters=cs["iters"], radius=cs["radius"], pad=cs.get("pad", 0))
        arrays = dict(img=img, out=out)
        if guide is not None:
            arrays["guide"] = guide
        np.savez_compressed(HERE / f"{cs['name']}.npz", **arrays)
        print(cs["name"], out.shape, float(np.abs(out - img).max()))
    for cs in GRID_CASES:
        img = scene(cs["scene"], cs["w"], cs["h"], cs["c"], cs["seed"]).astype(np.float32)
        guide = None
        if cs["guide"] is not None:
            kind, seed, gc = cs["guide"]
            guide = scene(kind, cs["w"], cs["h"], gc, seed).astype(np.float32)
        f = img.astype(np.float64)
        for _ in range(cs["iters"]):
            f = O.ref_smooth_grid(f, None if guide is None else guide.astype(np.float64),
                                  lam=cs["lam"], sigma_s=cs["sigma_s"], sigma_r=cs["sigma_r"],
                                  pad=cs["pad"])
        arrays = dict(img=img, out=f)
        if guide is not None:
            arrays["guide"] = guide
        np.savez_compressed(HERE / f"{cs['name']}.npz", **arrays)
        print(cs["name"], f.shape, float(np.abs(f - img).max()))
    for cs in NC_CASES:
        img = scene(cs["scene"], cs["w"], cs["h"], cs["c"], cs["seed"]).astype(np.float32)
        arrays = {"img": img}
        if cs.get("rolling"):
            out = O.ref_rolling_nc_ls(img.astype(np.float64), lam=cs["lam"], sigma_s=cs["sigma_s"],
                                      sigma_r=cs["sigma_r"], dt_iters=cs["dt_iters"], pad=cs["pad"],
                                      n=cs["n"], init_sigma=cs["init_sigma"])
        else:
            guide = None
            if cs["guide"] is not None:
                kind, seed, gc = cs["guide"]
                guide = scene(kind, cs["w"], cs["h"], gc, seed).astype(np.float32)
                arrays["guide"] = guide
            out = O.ref_smooth_nc(img.astype(np.float64),
                                  None if guide is None else guide.astype(np.float64),
                                  lam=cs["lam"], sigma_s=cs["sigma_s"], sigma_r=cs["sigma_r"],
                                  dt_iters=cs["dt_iters"], pad=cs["pad"])
        arrays["out"] = out
        np.savez_compressed(HERE / f"{cs['name']}.npz", **arrays)
        print(cs["name"], out.shape, float(np.abs(out - img).max()))


if __name__ == "__main__":
    main()
