"""Kernel-variant equivalence on the GPU: a default kernel and the variant an
environment knob selects must produce bit-identical targets (the knobs are
read once per process, so each side runs in its own subprocess).

- BLFLS_J3P=1 / 2: the persistent cp.async-prefetching shared-gray-guide
  filter (k_blf_j3p, copies before / spread over the filter loop) against
  the one-CTA-per-tile k_blf_j3 (both in the difference form,
  BLFLS_J3_XF=0).
- the factorised-exponent shared-guide (k_blf_j3) and self-guided (k_blf_p2)
  kernels (default where they apply) against the difference form: equal to
  fp32 round-off (not bit-identical).
- BLFLS_COL_PIPE=1: the pipelined column pass (k2_col_pipe: persistent,
  double-buffered cp.async strips) against k2_col, through full BLF-LS runs
  at every column length with a high-radix geometry.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1812_07122_b200 as P
from oracle import oracle as O
out = {{}}
for (b, h, w, r) in {shapes!r}:
    img = np.stack([np.stack([O.gen_plane(900 + 10 * i + c, h, w, n_sites=12) for c in range(3)])
                    for i in range(b)])
    guide = np.stack([O.gen_plane(1900 + i, h, w, n_sites=12)[None] for i in range(b)])
    if b == 1:
        img, guide = img[0], guide[0]
    tx, ty = P.filter_gradients(img, guide, sigma_s=7.0, sigma_r=0.1, radius=r)
    out[f"tx_{{b}}_{{h}}_{{w}}_{{r}}"] = np.asarray(tx)
    out[f"ty_{{b}}_{{h}}_{{w}}_{{r}}"] = np.asarray(ty)
np.savez({path!r}, **out)
"""

# W % 4 == 0 runs the persistent kernel (ragged last tile columns / rows,
# images smaller than a tile, batches); other widths fall back to k_blf_j3
SHAPES = [(1, 40, 64, 7), (2, 50, 132, 7), (2, 16, 16, 5), (1, 70, 300, 5), (5, 64, 200, 7),
          (1, 64, 64, 15), (1, 37, 68, 3), (3, 37, 129, 7), (1, 33, 47, 15)]


_SOLVE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1812_07122_b200 as P
from oracle import oracle as O
out = {{}}
for (b, c, h, w) in {shapes!r}:
    img = np.stack([np.stack([O.gen_plane(700 + 10 * i + k, h, w, n_sites=12) for k in range(c)])
                    for i in range(b)])
    if b == 1:
        img = img[0]
    u = P.blf_ls(img, lam=1000.0, sigma_s=3.0, sigma_r=0.1, iters=2, radius=3)
    out[f"u_{{b}}_{{c}}_{{h}}_{{w}}"] = np.asarray(u)
np.savez({path!r}, **out)
"""

# column lengths of the high-radix column geometries (k_solve2.cu), odd and
# even half-spectrum widths, several planes
SOLVE_SHAPES = [(1, 1, 512, 64), (2, 3, 512, 70), (1, 3, 1024, 96), (1, 1, 1080, 48), (1, 3, 2048, 40),
                (3, 1, 2048, 32), (1, 1, 4096, 18)]


def _run(tmp_path, name, env, script=_SCRIPT, shapes=SHAPES):
    path = str(tmp_path / f"{name}.npz")
    code = script.format(root=str(ROOT), shapes=shapes, path=path)
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", code], check=True, env=e, cwd=str(ROOT), timeout=600)
    return np.load(path)


@pytest.mark.parametrize("variant", ["1", "2"])
def test_shared_guide_persistent_matches_per_tile(tmp_path, variant):
    a = _run(tmp_path, "persistent", {"BLFLS_J3P": variant, "BLFLS_J3_XF": "0"})
    b = _run(tmp_path, "per_tile", {"BLFLS_J3P": "0", "BLFLS_J3_XF": "0"})
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def test_pipelined_column_pass_matches_k2_col(tmp_path):
    a = _run(tmp_path, "pipe", {"BLFLS_COL_PIPE": "1"}, _SOLVE_SCRIPT, SOLVE_SHAPES)
    b = _run(tmp_path, "plain", {"BLFLS_COL_PIPE": "0"}, _SOLVE_SCRIPT, SOLVE_SHAPES)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def test_shared_guide_factorised_exponent_close_to_difference_form(tmp_path):
    a = _run(tmp_path, "xf", {"BLFLS_J3_XF": "1"})
    b = _run(tmp_path, "diff", {"BLFLS_J3_XF": "0"})
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        # targets in raw gradient units of [0,1]-range images: the factorised
        # exponent rounds 2ab (|2ab| <= 36 at sigma_r = 0.1) instead of (a - b)^2
        assert np.max(np.abs(a[k].astype(np.float64) - b[k])) <= 2e-5, k


_SELF_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1812_07122_b200 as P
from oracle import oracle as O
out = {{}}
for (b, c, h, w, r, sr) in {shapes!r}:
    img = np.stack([np.stack([O.gen_plane(400 + 10 * i + k, h, w, n_sites=12) for k in range(c)])
                    for i in range(b)])
    if b == 1:
        img = img[0]
    tx, ty = P.filter_gradients(img, sigma_s=float(r), sigma_r=sr, radius=r)
    out[f"tx_{{b}}_{{c}}_{{h}}_{{w}}_{{r}}_{{sr}}"] = np.asarray(tx)
    out[f"ty_{{b}}_{{c}}_{{h}}_{{w}}_{{r}}_{{sr}}"] = np.asarray(ty)
np.savez({path!r}, **out)
"""

# self-guided radii of the packed kernel, sigma_r where the factorised form applies
SELF_SHAPES = [(1, 3, 40, 64, 7, 0.1), (2, 1, 70, 130, 15, 0.08), (1, 3, 33, 47, 5, 0.2),
               (1, 1, 96, 128, 7, 0.3)]


def test_self_guided_factorised_exponent_close_to_difference_form(tmp_path):
    a = _run(tmp_path, "xf", {"BLFLS_P2_XF": "1"}, _SELF_SCRIPT, SELF_SHAPES)
    b = _run(tmp_path, "diff", {"BLFLS_P2_XF": "0"}, _SELF_SCRIPT, SELF_SHAPES)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.max(np.abs(a[k].astype(np.float64) - b[k])) <= 2e-5, k
