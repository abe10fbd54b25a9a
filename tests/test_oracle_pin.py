"""Pin the CPU oracle (oracle/blfls_oracle.c) before trusting it.

1. Against the reference translation units compiled unmodified (oracle/_ref)
   on the reference's own seeded inputs -- bit-exact or round-off level.
2. Against the reference's known-answer tests for this path, restated
   (test_bilateral.cpp, test_solver.cpp, test_image.cpp, test_pipelines.cpp,
   acceptance_main.cpp c1/c2/c8).
3. Against the committed golden vectors (tests/golden/, generated from the
   reference by tests/golden/make_golden.py), which also works where
   /root/reference is absent.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
from cases import CASES  # noqa: E402


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


# ----------------------------------------------------------- vs reference --

def test_splitmix_matches_reference_random_image(ref):
    # testimage.cpp:11-23,114-120: draw j of the sequential stream
    img = ref.ref_random_image(7, 5, 3, 31, -1.0, 3.0)
    flat = img.reshape(-1)
    ours = np.array([-1.0 + 4.0 * ref.uniform_at(31, j) for j in range(flat.size)])
    assert maxabs(flat, ours) == 0.0


@pytest.mark.parametrize("sigma_s,sigma_r,shape,seed", [
    (2.0, 0.1, (1, 18, 24), 5), (1.0, 0.05, (1, 31, 40), 8), (2.0, 0.1, (3, 6, 7), 9),
])
def test_blf_brute_bitexact_vs_reference(ref, sigma_s, sigma_r, shape, seed):
    c, h, w = shape
    g = ref.ref_random_image(w, h, c, seed)
    a = ref.ref_blf_brute(g, g, sigma_s=sigma_s, sigma_r=sigma_r)
    b = ref.blf_brute_r(g, g, sigma_s=sigma_s, sigma_r=sigma_r, radius=-1)
    assert maxabs(a, b) == 0.0
    # serial::blf_brute (serial.cpp:44-77), two exps per tap
    s = ref.ref_blf_brute(g, g, sigma_s=sigma_s, sigma_r=sigma_r, serial=True)
    assert maxabs(s, b) < 1e-12


def test_blf_joint_guide_bitexact_vs_reference(ref):
    src = ref.ref_natural_scene(20, 16, 3, 4)
    gd = ref.ref_natural_scene(20, 16, 1, 7)
    a = ref.ref_blf_brute(src, gd, sigma_s=1.5, sigma_r=0.08)
    b = ref.blf_brute_r(src, gd, sigma_s=1.5, sigma_r=0.08)
    assert maxabs(a, b) == 0.0


def test_forward_gradients_and_normalize_vs_reference(ref):
    g = ref.ref_random_image(13, 9, 3, 71, -3.0, 17.0)
    gx, gy = ref.ref_forward_gradients(g)
    ox, oy = ref.forward_gradients(g)
    assert maxabs(gx, ox) == 0.0 and maxabs(gy, oy) == 0.0
    n1, lo1, hi1 = ref.ref_normalize_to_unit(g)
    n2, lo2, hi2 = ref.normalize_to_unit(g)
    assert (lo1, hi1) == (lo2, hi2) and maxabs(n1, n2) == 0.0


@pytest.mark.parametrize("h,w,lam,pad", [(16, 16, 7.0, 0), (30, 18, 1000.0, 0), (15, 10, 3.0, 0),
                                         (13, 9, 50.0, 4)])
def test_lsgrad_vs_reference(ref, h, w, lam, pad):
    g = ref.ref_random_image(w, h, 1, 13)
    tx = ref.ref_random_image(w, h, 1, 14, -1.0, 1.0)
    ty = ref.ref_random_image(w, h, 1, 15, -1.0, 1.0)
    a = ref.ref_lsgrad_solve_fft(g, tx, ty, lam=lam, pad=pad)
    b = ref.lsgrad_solve_fft(g, tx, ty, lam=lam, pad=pad)
    assert maxabs(a, b) < 1e-13


@pytest.mark.parametrize("radius", [6, 4])
def test_smooth_brute_vs_reference(ref, radius):
    # radius 6 == ceil(3*2.0): the reference's unmodified blf_brute runs inside
    g = ref.ref_natural_scene(40, 32, 3, 4)
    a = ref.ref_smooth_brute(g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, radius=radius)
    b = ref.smooth_brute(g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, radius=radius)
    assert maxabs(a, b) < 1e-13


def test_cascade_and_joint_vs_reference(ref):
    g = ref.ref_natural_scene(24, 20, 3, 8)
    gd = ref.ref_natural_scene(24, 20, 1, 9)
    for guide in (None, gd):
        a = ref.ref_blf_ls(g, guide, lam=500.0, sigma_s=1.0, sigma_r=0.1, iters=3, radius=3)
        b = ref.blf_ls(g, guide, lam=500.0, sigma_s=1.0, sigma_r=0.1, iters=3, radius=3)
        assert maxabs(a, b) < 1e-13


def test_grid_pipeline_runs(ref):
    # the reference's shipped smooth() (bilateral grid) links and runs here
    g = ref.ref_natural_scene(32, 32, 1, 3)
    u = ref.ref_smooth_grid(g, lam=100.0, sigma_s=4.0, sigma_r=0.1, pad=0)
    assert np.isfinite(u).all() and maxabs(u, g) < 0.5


# ------------------------------------------------------- reference KATs --

def test_fft_convention_naive_dft(oracle):
    # test_solver.cpp:25-42,81-89: forward exp(-i), half spectrum
    rng = np.random.default_rng(31)
    for h, w in [(4, 4), (6, 8), (5, 9), (13, 7)]:
        x = rng.random((h, w))
        full = oracle.naive_dft2(x)
        half = oracle.rfft2(x)
        assert maxabs(half, full[:, : w // 2 + 1]) < 1e-12
        assert maxabs(oracle.irfft2(half, w), x) < 1e-13


def test_fft_vs_numpy_mixed_radix(oracle):
    rng = np.random.default_rng(1)
    for h, w in [(60, 48), (135, 240), (27, 50), (14, 11)]:
        x = rng.random((h, w))
        assert maxabs(oracle.rfft2(x), np.fft.rfft2(x)) < 1e-10


def test_otf_convolution_theorem(oracle):
    # test_solver.cpp:81-89: F(Dx^T-kernel conv) = ox * F
    rng = np.random.default_rng(4)
    x = rng.random((4, 4))
    conv = np.roll(x, 1, axis=1) - x
    v = np.arange(4)
    ox = np.exp(-2j * np.pi * v / 4) - 1.0
    assert maxabs(oracle.naive_dft2(conv), oracle.naive_dft2(x) * ox[None, :]) < 1e-12


def test_lsgrad_fixed_point(oracle):
    # test_solver.cpp:120-127 / acceptance c2: lsgrad(g, grad g) = g
    rng = np.random.default_rng(55)
    for lam in (32.0, 1024.0):
        g = rng.random((1, 32, 32))
        gx, gy = oracle.forward_gradients(g)
        assert maxabs(oracle.lsgrad_solve_fft(g, gx, gy, lam=lam), g) < 1e-10


def test_lsgrad_vs_dense_sweep(oracle):
    # test_solver.cpp:136-161 / acceptance c1
    rng = np.random.default_rng(1000)
    for i in range(10):
        g = rng.random((1, 8, 8))
        tx, ty = rng.uniform(-1, 1, (2, 1, 8, 8))
        lam = 0.5 + 7.3 * i
        assert maxabs(oracle.lsgrad_solve_fft(g, tx, ty, lam=lam),
                      oracle.dense_solve(g, tx, ty, lam=lam)) < 1e-8
        assert maxabs(oracle.lsgrad_solve_fft(g, None, None, lam=lam),
                      oracle.dense_solve(g, None, None, lam=lam)) < 1e-8


def test_lambda_zero_identity_and_constants(oracle):
    # test_solver.cpp:101-112
    rng = np.random.default_rng(71)
    g = rng.random((3, 9, 13))
    assert maxabs(oracle.lsgrad_solve_fft(g, None, None, lam=0.0), g) < 1e-12
    c = np.full((1, 10, 12), 0.63)
    assert maxabs(oracle.lsgrad_solve_fft(c, None, None, lam=512.0), c) < 1e-10


def test_blf_properties(oracle):
    # test_bilateral.cpp:49-55 constant fixed point, 101-107 convex hull, 109-116 mirror
    rng = np.random.default_rng(4)
    src = np.full((1, 13, 17), 0.37)
    gd = rng.random((1, 13, 17))
    assert maxabs(oracle.blf_brute_r(src, gd, sigma_s=3.0, sigma_r=0.1), src) < 1e-12
    img = rng.random((1, 20, 20))
    out = oracle.blf_brute_r(img, img, sigma_s=2.5, sigma_r=0.15)
    assert out.min() >= img.min() - 1e-12 and out.max() <= img.max() + 1e-12
    a = oracle.blf_brute_r(img, img, sigma_s=2.0, sigma_r=0.1, radius=4)[:, :, ::-1]
    b = oracle.blf_brute_r(img[:, :, ::-1].copy(), img[:, :, ::-1].copy(), sigma_s=2.0, sigma_r=0.1,
                           radius=4)
    assert maxabs(a, b) < 1e-13


def test_blf_validation(oracle):
    a = np.full((1, 8, 8), 0.5)
    with pytest.raises(oracle.OracleError):
        oracle.blf_brute_r(a, a, sigma_s=0.0, sigma_r=0.1)
    with pytest.raises(oracle.OracleError):
        oracle.blf_brute_r(a, a, sigma_s=2.0, sigma_r=-0.1)
    bad = a.copy()
    bad[0, 3, 3] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.blf_ls(bad, lam=1.0, sigma_s=1.0, sigma_r=0.1, iters=1, radius=2)


def test_pipeline_properties(oracle):
    # test_pipelines.cpp:33-38 constants, 40-47 identity, 58-69 fidelity monotone in lambda
    c = np.full((3, 30, 40), 0.55)
    assert maxabs(oracle.blf_ls(c, lam=1024.0, sigma_s=2.0, sigma_r=0.05, iters=2, radius=4), c) < 1e-6
    rng = np.random.default_rng(3)
    g = rng.random((1, 40, 48))
    u = oracle.blf_ls(g, lam=1e-9, sigma_s=2.0, sigma_r=1e6, iters=1, radius=4)
    assert maxabs(u, g) < 1e-4
    prev = -1.0
    for lam in (32.0, 128.0, 512.0, 1024.0):
        d = float(np.mean((oracle.blf_ls(g, lam=lam, sigma_s=2.0, sigma_r=0.05, iters=1, radius=4)
                           - g) ** 2))
        assert d >= prev - 1e-15
        prev = d


def test_guidance_equal_input_matches_self(oracle):
    # test_pipelines.cpp:49-56 (exact equality in the reference)
    rng = np.random.default_rng(4)
    g = rng.random((3, 32, 40))
    a = oracle.blf_ls(g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, iters=1, radius=4)
    b = oracle.blf_ls(g, g, lam=1024.0, sigma_s=2.0, sigma_r=0.05, iters=1, radius=4)
    assert maxabs(a, b) == 0.0


# -------------------------------------------------------- golden vectors --

@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_golden(oracle, case):
    d = np.load(HERE / "golden" / f"{case['name']}.npz")
    img = d["img"].astype(np.float64)
    guide = d["guide"].astype(np.float64) if "guide" in d else None
    out = oracle.blf_ls(img, guide, lam=case["lam"], sigma_s=case["sigma_s"],
                        sigma_r=case["sigma_r"], iters=case["iters"], radius=case["radius"],
                        pad=case.get("pad", 0))
    assert maxabs(out, d["out"]) < 1e-12


@pytest.mark.parametrize("pad", [1, 5, 16])
def test_padded_cascade_vs_reference(ref, pad):
    # pipelines.cpp:76-92 (reflect_pad -> gradients -> filter -> solve -> crop)
    g = ref.ref_natural_scene(30, 22, 3, 14)
    gd = ref.ref_natural_scene(30, 22, 1, 15)
    for guide in (None, gd):
        a = ref.ref_blf_ls(g, guide, lam=700.0, sigma_s=1.5, sigma_r=0.1, iters=2, radius=3, pad=pad)
        b = ref.blf_ls(g, guide, lam=700.0, sigma_s=1.5, sigma_r=0.1, iters=2, radius=3, pad=pad)
        assert maxabs(a, b) < 1e-13


# ------------------------------------------------------------- generator --

def test_generator_deterministic_and_ranged(oracle):
    a = oracle.gen_plane(2000, 64, 96, n_sites=12)
    b = oracle.gen_plane(2000, 64, 96, n_sites=12)
    assert (a == b).all()
    assert a.min() >= 0.0 and a.max() <= 1.0
    c = oracle.gen_plane(2001, 64, 96, n_sites=12)
    assert not (a == c).all()
    base = oracle.gen_plane(3000, 128, 128, n_sites=12)
    sp = oracle.gen_plane(3000, 128, 128, n_sites=12, p_sp=0.05)
    changed = sp != base
    frac0 = float(np.mean(changed & (sp == 0.0)))
    frac1 = float(np.mean(changed & (sp == 1.0)))
    assert changed.sum() == ((sp == 0.0) & changed).sum() + ((sp == 1.0) & changed).sum()
    assert 0.015 < frac0 < 0.035 and 0.015 < frac1 < 0.035


def test_generator_matches_spec(oracle):
    # draw layout: sites at 3s..3s+2, pixel i at 3K + 3i + {0,1,2}
    seed, h, w, k = 77, 9, 11, 3
    img = oracle.gen_plane(seed, h, w, n_sites=k, noise_sigma=0.03)
    sites = [(oracle.uniform_at(seed, 3 * s) * w, oracle.uniform_at(seed, 3 * s + 1) * h,
              oracle.uniform_at(seed, 3 * s + 2)) for s in range(k)]
    for y in range(h):
        for x in range(w):
            d = [(x - sx) ** 2 + (y - sy) ** 2 for sx, sy, _ in sites]
            best = int(np.argmin(d))
            i = y * w + x
            u1 = oracle.uniform_at(seed, 3 * k + 3 * i)
            u2 = oracle.uniform_at(seed, 3 * k + 3 * i + 1)
            v = sites[best][2] + 0.2 * ((x / (w - 1) + y / (h - 1)) / 2 - 0.5)
            v += 0.03 * math.sqrt(-2 * math.log(1 - u1)) * math.cos(2 * math.pi * u2)
            v = min(max(v, 0.0), 1.0)
            assert img[y, x] == np.float32(v)
