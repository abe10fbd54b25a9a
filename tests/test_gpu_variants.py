"""Kernel-variant equivalence on the GPU: a default kernel and the variant an
environment knob selects must produce bit-identical targets (the knobs are
read once per process, so each side runs in its own subprocess).

- BLFLS_J3P=1 / 2: the persistent cp.async-prefetching shared-gray-guide
  filter (k_blf_j3p, copies before / spread over the filter loop) against
  the default one-CTA-per-tile k_blf_j3.
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


def _run(tmp_path, name, env):
    path = str(tmp_path / f"{name}.npz")
    code = _SCRIPT.format(root=str(ROOT), shapes=SHAPES, path=path)
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", code], check=True, env=e, cwd=str(ROOT), timeout=600)
    return np.load(path)


@pytest.mark.parametrize("variant", ["1", "2"])
def test_shared_guide_persistent_matches_per_tile(tmp_path, variant):
    a = _run(tmp_path, "persistent", {"BLFLS_J3P": variant})
    b = _run(tmp_path, "per_tile", {"BLFLS_J3P": "0"})
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
