"""Golden-vector cases (shared by make_golden.py and the tests).

Inputs come from the reference's own seeded test-image generators
(testimage.cpp: natural_scene, random_image) rounded to fp32, because the GPU
path consumes fp32.  Outputs are the reference pipeline pieces run in double
(oracle/_ref): smooth() with the unmodified brute-force blf_brute whenever
radius == ceil(3 sigma_s), iterated `iters` times with the guide fixed.
"""
CASES = [
    # name, (w, h, c), scene, seed, guide, (sigma_s, sigma_r, lambda, iters, radius)
    dict(name="gray_40x32_self", w=40, h=32, c=1, scene="natural", seed=3, guide=None,
         sigma_s=2.0, sigma_r=0.05, lam=200.0, iters=1, radius=6),
    dict(name="gray_40x32_r3_it2", w=40, h=32, c=1, scene="natural", seed=9, guide=None,
         sigma_s=2.0, sigma_r=0.1, lam=1000.0, iters=2, radius=3),
    dict(name="rgb_24x20_self_it3", w=24, h=20, c=3, scene="natural", seed=8, guide=None,
         sigma_s=1.5, sigma_r=0.1, lam=500.0, iters=3, radius=5),
    dict(name="rgb_30x18_joint_rgb", w=30, h=18, c=3, scene="natural", seed=4, guide=("natural", 5, 3),
         sigma_s=1.0, sigma_r=0.08, lam=300.0, iters=2, radius=3),
    dict(name="rgb_32x24_joint_gray", w=32, h=24, c=3, scene="natural", seed=6, guide=("natural", 11, 1),
         sigma_s=1.0, sigma_r=0.1, lam=1000.0, iters=3, radius=3),
    dict(name="gray_15x13_odd", w=15, h=13, c=1, scene="random", seed=21, guide=None,
         sigma_s=1.0, sigma_r=0.15, lam=7.0, iters=1, radius=3),
    dict(name="gray_36x20_constant", w=36, h=20, c=1, scene="constant", seed=0, guide=None,
         sigma_s=2.0, sigma_r=0.05, lam=1000.0, iters=2, radius=6),
    dict(name="gray_48x40_wide_range", w=48, h=40, c=1, scene="natural", seed=3, guide=None,
         sigma_s=2.0, sigma_r=1e6, lam=1e-9, iters=1, radius=6),
    # reflect padding (SolveParams::pad, the reference default is 16); the
    # padded grids carry prime factors 43 and 17 (direct-DFT FFT stages)
    dict(name="gray_37x45_pad3", w=37, h=45, c=1, scene="natural", seed=12, guide=None,
         sigma_s=1.0, sigma_r=0.1, lam=300.0, iters=2, radius=3, pad=3),
    dict(name="rgb_34x30_pad16_default", w=34, h=30, c=3, scene="natural", seed=13, guide=None,
         sigma_s=1.0, sigma_r=0.04, lam=1024.0, iters=1, radius=3, pad=16),
    dict(name="rgb_32x24_joint_gray_pad4", w=32, h=24, c=3, scene="natural", seed=6,
         guide=("natural", 11, 1), sigma_s=1.0, sigma_r=0.1, lam=1000.0, iters=2, radius=3, pad=4),
]

# The reference's own smooth() (bilateral grid, pipelines.cpp:47) cascaded
# `iters` times with the guide fixed: the GPU grid backend's parity targets.
GRID_CASES = [
    dict(name="grid_gray_64x48_self", w=64, h=48, c=1, scene="natural", seed=21, guide=None,
         sigma_s=4.0, sigma_r=0.1, lam=500.0, iters=1, pad=0),
    dict(name="grid_rgb_48x40_self_pad16", w=48, h=40, c=3, scene="natural", seed=22, guide=None,
         sigma_s=12.0, sigma_r=0.04, lam=1024.0, iters=1, pad=16),
    dict(name="grid_rgb_56x40_joint_it2", w=56, h=40, c=3, scene="natural", seed=23,
         guide=("natural", 24, 3), sigma_s=6.0, sigma_r=0.05, lam=800.0, iters=2, pad=0),
]

# The reference's smooth() with SmootherKind::NC_LS (nc_filter,
# pipelines.cpp:48) and rolling_nc_ls (pipelines.cpp:96-117): the GPU
# domain-transform backend's parity targets.  guide = None (self) or a
# same-channel guide image like the reference requires.
NC_CASES = [
    dict(name="nc_gray_48x40_self", w=48, h=40, c=1, scene="natural", seed=31, guide=None,
         sigma_s=6.0, sigma_r=0.05, dt_iters=3, lam=800.0, pad=0),
    dict(name="nc_rgb_40x32_self_pad16", w=40, h=32, c=3, scene="natural", seed=32, guide=None,
         sigma_s=12.0, sigma_r=0.05, dt_iters=3, lam=1024.0, pad=16),
    dict(name="nc_rgb_36x28_joint_it2", w=36, h=28, c=3, scene="natural", seed=33,
         guide=("natural", 34, 3), sigma_s=4.0, sigma_r=0.1, dt_iters=2, lam=600.0, pad=3),
    dict(name="nc_gray_33x25_random", w=33, h=25, c=1, scene="random", seed=35, guide=None,
         sigma_s=3.0, sigma_r=0.2, dt_iters=1, lam=50.0, pad=0),
    dict(name="rolling_rgb_40x32_texture", w=40, h=32, c=3, scene="natural", seed=36, guide=None,
         sigma_s=8.0, sigma_r=0.02, dt_iters=3, lam=1024.0, pad=16, rolling=True, n=3,
         init_sigma=2.5),
    dict(name="rolling_gray_32x32_clipart", w=32, h=32, c=1, scene="natural", seed=37, guide=None,
         sigma_s=6.0, sigma_r=0.02, dt_iters=3, lam=1024.0, pad=16, rolling=True, n=2,
         init_sigma=0.75),
]
