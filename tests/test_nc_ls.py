"""NC-LS: the domain-transform gradient filter
nc_filter (domain_transform.cpp), SmootherKind::NC_LS smooth()
(pipelines.cpp:48), gaussian_blur (image.cpp:114-158) and rolling_nc_ls
(pipelines.cpp:96-117).

CPU part: the oracle restatement is pinned bit-for-bit against the reference
translation units (oracle/_ref) and the committed golden vectors.  GPU part:
the sm_100a path through the C ABI against the oracle.  The DT filter keeps
the reference's sequential recurrences in double, so its targets equal the
reference's up to the final fp32 rounding (TOL_DT_TARGET); the full smooth
adds the fp32 FFT solve (TOL_OUT, as BLF-LS).  Rolling guidance feeds fp32
outputs back as guides, where the reference keeps double: a guide difference
of ~1e-7 can move a window bound by one sample, so rolling is held to
TOL_ROLL (max) and TOL_ROLL_MEAN (mean)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
from cases import NC_CASES  # noqa: E402

TOL_DT_TARGET = 1e-6
TOL_OUT = 1e-4
TOL_ROLL = 5e-3
TOL_ROLL_MEAN = 5e-5


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def _img(oracle, c, h, w, seed, sites=12):
    return np.stack([oracle.gen_plane(seed * 10 + k, h, w, n_sites=sites) for k in range(c)])


# ------------------------------------------------------------- CPU pins --

def test_oracle_nc_filter_matches_reference(ref):
    rng = np.random.default_rng(3)
    for (c, cg, h, w, ss, sr, it) in [(3, 3, 24, 31, 3.0, 0.1, 3), (1, 1, 17, 40, 8.0, 0.02, 2),
                                      (3, 1, 33, 20, 5.0, 0.5, 1), (1, 1, 1, 8, 2.0, 0.5, 1)]:
        src = rng.random((c, h, w))
        guide = rng.random((cg, h, w))
        a = ref.nc_filter(src, guide, sigma_s=ss, sigma_r=sr, iters=it)
        assert np.array_equal(a, ref.ref_nc_filter(src, guide, sigma_s=ss, sigma_r=sr, iters=it))
        # the sliding-window kernel equals the reference's scalar one (test_domain_transform.cpp:51-70)
        s = ref.ref_nc_filter(src, guide, sigma_s=ss, sigma_r=sr, iters=it, serial=True)
        assert maxabs(a, s) < 1e-10
    for it in (1, 2, 3, 5):
        for k in range(1, it + 1):
            assert ref.nc_box_radius(12.0, k, it) == ref.ref_nc_box_radius(12.0, k, it)


def test_oracle_smooth_nc_and_rolling_match_reference(ref):
    img = ref.ref_natural_scene(40, 32, 3, 5)
    gd = ref.ref_natural_scene(40, 32, 3, 9)
    for pad in (0, 5):
        a = ref.smooth_nc(img, lam=800.0, sigma_s=6.0, sigma_r=0.05, pad=pad)
        assert np.array_equal(a, ref.ref_smooth_nc(img, lam=800.0, sigma_s=6.0, sigma_r=0.05, pad=pad))
    a = ref.smooth_nc(img, gd, lam=800.0, sigma_s=6.0, sigma_r=0.05, dt_iters=2)
    assert np.array_equal(a, ref.ref_smooth_nc(img, gd, lam=800.0, sigma_s=6.0, sigma_r=0.05,
                                               dt_iters=2))
    assert np.array_equal(ref.gaussian_blur(img, 2.5), ref.ref_gaussian_blur(img, 2.5))
    a = ref.rolling_nc_ls(img, lam=1024.0, sigma_s=8.0, sigma_r=0.02, pad=16, n=2)
    assert np.array_equal(a, ref.ref_rolling_nc_ls(img, lam=1024.0, sigma_s=8.0, sigma_r=0.02,
                                                   pad=16, n=2))


@pytest.mark.parametrize("case", NC_CASES, ids=[c["name"] for c in NC_CASES])
def test_oracle_nc_golden(oracle, case):
    d = np.load(HERE / "golden" / f"{case['name']}.npz")
    if case.get("rolling"):
        out = oracle.rolling_nc_ls(d["img"], lam=case["lam"], sigma_s=case["sigma_s"],
                                   sigma_r=case["sigma_r"], dt_iters=case["dt_iters"],
                                   pad=case["pad"], n=case["n"], init_sigma=case["init_sigma"])
    else:
        guide = d["guide"] if "guide" in d else None
        out = oracle.smooth_nc(d["img"], guide, lam=case["lam"], sigma_s=case["sigma_s"],
                               sigma_r=case["sigma_r"], dt_iters=case["dt_iters"], pad=case["pad"])
    assert maxabs(out, d["out"]) <= 1e-12


def test_oracle_dt_properties(oracle):
    """test_domain_transform.cpp:23-44: constants are fixed points; an
    infinite-contrast guide step blocks all mixing."""
    src = np.full((3, 11, 15), 0.3)
    guide = np.full((3, 11, 15), 0.8)
    assert maxabs(oracle.nc_filter(src, guide, sigma_s=4.0, sigma_r=0.1, iters=3), src) < 1e-12
    vals = np.array([0.1, 0.5, 0.3, 0.9, 0.2, 0.6, 0.4, 0.8])
    out = oracle.nc_filter(vals[None, None], (np.arange(8) >= 4).astype(float)[None, None],
                           sigma_s=2.0, sigma_r=1e-4, iters=1)[0, 0]
    assert np.allclose(out[:4], vals[:4].mean(), rtol=1e-12)
    assert np.allclose(out[4:], vals[4:].mean(), rtol=1e-12)


# ------------------------------------------------------------------ GPU --

@pytest.mark.gpu
@pytest.mark.parametrize("c,h,w,ss,sr,it,guide", [
    (3, 40, 56, 6.0, 0.05, 3, None),
    (1, 64, 48, 12.0, 0.05, 3, None),
    (3, 37, 29, 3.0, 0.2, 1, "rgb"),
    (3, 48, 64, 8.0, 0.02, 2, "gray"),
    (1, 2, 96, 4.0, 0.1, 3, None),
    (1, 96, 2, 4.0, 0.1, 3, None),
    (3, 150, 140, 20.0, 0.01, 4, None),   # multiple 128-row scan blocks, ragged tiles
])
def test_dt_targets_exact(gpu, oracle, c, h, w, ss, sr, it, guide):
    """filter_gradients(backend="dt") = 2 nc_filter(src01, guide01) - 1 of the
    oracle (pipelines.cpp:33-53), exact in double, then rounded to fp32."""
    img = _img(oracle, c, h, w, 7 + h)
    gd = None
    if guide == "rgb":
        gd = _img(oracle, 3, h, w, 99)
    elif guide == "gray":
        gd = _img(oracle, 1, h, w, 98)
    tx, ty = gpu.filter_gradients(img, gd, sigma_s=ss, sigma_r=sr, backend="dt", dt_iterations=it)
    gn, _, _ = oracle.normalize_to_unit(img.astype(np.float64))
    gx, gy = oracle.forward_gradients(gn)
    if gd is None:
        ggx, ggy = gx, gy
    else:
        gdn, _, _ = oracle.normalize_to_unit(gd.astype(np.float64))
        ggx, ggy = oracle.forward_gradients(gdn)
    for t, sgr, ggr in ((tx, gx, ggx), (ty, gy, ggy)):
        ref = np.stack([
            2.0 * oracle.nc_filter((sgr[k:k + 1] + 1.0) * 0.5,
                                   (ggr[k if ggr.shape[0] > 1 else 0:][:1] + 1.0) * 0.5,
                                   sigma_s=ss, sigma_r=sr, iters=it)[0] - 1.0 for k in range(c)])
        assert maxabs(t, ref) <= TOL_DT_TARGET


@pytest.mark.gpu
@pytest.mark.parametrize("case", NC_CASES, ids=[c["name"] for c in NC_CASES])
def test_nc_golden_vectors(gpu, case):
    d = np.load(HERE / "golden" / f"{case['name']}.npz")
    if case.get("rolling"):
        out = gpu.rolling_nc_ls(d["img"], gpu.DtParams(case["sigma_s"], case["sigma_r"],
                                                       case["dt_iters"]),
                                gpu.SolveParams(case["lam"], case["pad"]),
                                gpu.RollingParams(case["n"], case["init_sigma"]))
        assert maxabs(out, d["out"]) <= TOL_ROLL
        assert float(np.mean(np.abs(out - d["out"]))) <= TOL_ROLL_MEAN
        return
    guide = d["guide"] if "guide" in d else None
    spec = gpu.SmootherSpec(kind=gpu.SmootherKind.NC_LS,
                            dt=gpu.DtParams(case["sigma_s"], case["sigma_r"], case["dt_iters"]),
                            solve=gpu.SolveParams(case["lam"], case["pad"]), guidance=guide)
    assert maxabs(gpu.smooth(d["img"], spec), d["out"]) <= TOL_OUT


@pytest.mark.gpu
def test_nc_ls_vs_oracle(gpu, oracle):
    for (c, h, w, ss, sr, it, iters, pad, gc) in [(3, 72, 96, 8.0, 0.05, 3, 1, 0, 0),
                                                 (1, 100, 60, 12.0, 0.05, 3, 2, 16, 0),
                                                 (3, 64, 64, 6.0, 0.1, 2, 3, 0, 1),
                                                 (3, 50, 70, 4.0, 0.03, 3, 1, 7, 3)]:
        img = _img(oracle, c, h, w, 31 + h)
        gd = None if gc == 0 else _img(oracle, gc, h, w, 77)
        out = gpu.nc_ls(img, gd, lam=900.0, sigma_s=ss, sigma_r=sr, dt_iterations=it, iters=iters,
                        pad=pad)
        ref = oracle.nc_ls(img.astype(np.float64), None if gd is None else gd.astype(np.float64),
                           lam=900.0, sigma_s=ss, sigma_r=sr, dt_iters=it, iters=iters, pad=pad)
        assert maxabs(out, ref) <= TOL_OUT


@pytest.mark.gpu
def test_nc_ls_batch_and_device_tensors(gpu, oracle):
    import torch
    imgs = np.stack([_img(oracle, 3, 48, 40, 50 + b) for b in range(3)]).astype(np.float32)
    out = gpu.nc_ls(torch.from_numpy(imgs).cuda(), lam=700.0, sigma_s=5.0, sigma_r=0.05).cpu().numpy()
    for b in range(3):
        ref = oracle.nc_ls(imgs[b].astype(np.float64), lam=700.0, sigma_s=5.0, sigma_r=0.05)
        assert maxabs(out[b], ref) <= TOL_OUT


@pytest.mark.gpu
def test_nc_ls_properties(gpu, oracle):
    """test_pipelines.cpp:34-38 (constants are fixed points) and
    test_domain_transform.cpp:86-91 (repeated runs are deterministic)."""
    const = np.full((3, 30, 40), 0.55, np.float32)
    spec = gpu.SmootherSpec(kind=gpu.SmootherKind.NC_LS, dt=gpu.DtParams(6.0, 0.05, 3))
    assert maxabs(gpu.smooth(const, spec), const) < 1e-6
    img = _img(oracle, 3, 24, 32, 12)
    spec = gpu.SmootherSpec(kind=gpu.SmootherKind.NC_LS, dt=gpu.DtParams(8.0, 0.02, 3))
    a, b = gpu.smooth(img, spec), gpu.smooth(img, spec)
    assert a.tobytes() == b.tobytes()
    with pytest.raises(gpu.InvalidArgument):
        gpu.nc_ls(img, lam=1.0, sigma_s=2.0, sigma_r=0.1, dt_iterations=0)
    with pytest.raises(gpu.InvalidArgument):
        gpu.nc_ls(img, lam=1.0, sigma_s=0.0, sigma_r=0.1)


@pytest.mark.gpu
def test_gaussian_blur_vs_oracle(gpu, oracle):
    import torch
    img = _img(oracle, 3, 37, 53, 4)
    for sigma in (0.75, 2.5, 6.0):
        ref = oracle.gaussian_blur(img.astype(np.float64), sigma)
        assert maxabs(gpu.gaussian_blur(img, sigma), ref) <= 1e-6
        t = gpu.gaussian_blur(torch.from_numpy(img).cuda(), sigma).cpu().numpy()
        assert maxabs(t, ref) <= 1e-6
    with pytest.raises(gpu.InvalidArgument):
        gpu.gaussian_blur(img, 0.0)


@pytest.mark.gpu
def test_rolling_nc_ls(gpu, oracle):
    img = _img(oracle, 3, 64, 80, 21)
    dt, sp = gpu.DtParams(8.0, 0.02, 3), gpu.SolveParams(1024.0, 16)
    for rp in (gpu.RollingParams(3, 2.5), gpu.RollingParams(2, 0.75)):
        out = gpu.rolling_nc_ls(img, dt, sp, rp)
        ref = oracle.rolling_nc_ls(img.astype(np.float64), lam=1024.0, sigma_s=8.0, sigma_r=0.02,
                                   pad=16, n=rp.n, init_sigma=rp.init_sigma)
        assert maxabs(out, ref) <= TOL_ROLL
        assert float(np.mean(np.abs(out - ref))) <= TOL_ROLL_MEAN
    # test_pipelines.cpp:98-111: a no-op initial blur equals joint smoothing by the input
    g = _img(oracle, 1, 32, 32, 11)
    rolled = gpu.rolling_nc_ls(g, gpu.DtParams(4.0, 0.05, 3), gpu.SolveParams(1024.0, 8),
                               gpu.RollingParams(1, 1e-3))
    joint = gpu.smooth(g, gpu.SmootherSpec(kind=gpu.SmootherKind.NC_LS,
                                           dt=gpu.DtParams(4.0, 0.05, 3),
                                           solve=gpu.SolveParams(1024.0, 8), guidance=g))
    assert maxabs(rolled, joint) < 1e-4
    # test_pipelines.cpp:113-118: rolling keeps constants
    cst = np.full((1, 24, 24), 0.8, np.float32)
    for n in (1, 2, 3):
        assert maxabs(gpu.rolling_nc_ls(cst, gpu.DtParams(8.0, 0.02, 3), gpu.SolveParams(),
                                        gpu.RollingParams(n, 2.5)), cst) < 1e-6
    with pytest.raises(gpu.InvalidArgument):
        gpu.rolling_nc_ls(cst, dt, sp, gpu.RollingParams(0, 2.5))


@pytest.mark.gpu
def test_dt_batch_rgb_guide_odd_pad(gpu, oracle):
    """Batched NC-LS with a per-channel RGB guide (mode 1), odd sizes and
    reflect padding: every image of the batch matches its own oracle run."""
    imgs = np.stack([_img(oracle, 3, 37, 53, 300 + b) for b in range(2)]).astype(np.float32)
    gds = np.stack([_img(oracle, 3, 37, 53, 400 + b) for b in range(2)]).astype(np.float32)
    out = gpu.nc_ls(imgs, gds, lam=600.0, sigma_s=5.0, sigma_r=0.05, dt_iterations=2, iters=2, pad=5)
    for b in range(2):
        ref = oracle.nc_ls(imgs[b].astype(np.float64), gds[b].astype(np.float64), lam=600.0,
                           sigma_s=5.0, sigma_r=0.05, dt_iters=2, iters=2, pad=5)
        assert maxabs(out[b], ref) <= TOL_OUT


@pytest.mark.gpu
def test_dt_gray_guide_shared_by_rgb(gpu, oracle):
    """One grayscale guide for an RGB image: replicated per channel exactly as
    the oracle's cascade does (the reference requires equal channel counts)."""
    img = _img(oracle, 3, 48, 40, 310)
    gd = _img(oracle, 1, 48, 40, 311)
    out = gpu.nc_ls(img, gd, lam=800.0, sigma_s=6.0, sigma_r=0.04)
    ref = oracle.nc_ls(img.astype(np.float64), gd.astype(np.float64), lam=800.0, sigma_s=6.0,
                       sigma_r=0.04)
    assert maxabs(out, ref) <= TOL_OUT
