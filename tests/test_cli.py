"""The epls-style CLI (tools/blfls_cli.cpp): exit codes like the reference
(tests/test_cli.cpp:74-85 of the reference), PFM/PNM I/O conventions, and on a
GPU the pixel-exact lambda-0 round trip (test_cli.cpp:45-59) and run-to-run
byte-identical output (test_cli.cpp:87-99)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def cli():
    from paper_1812_07122_b200 import build
    build.build()
    return str(build.CLI)


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300)


def write_pfm(path, img):
    """img: (C, H, W) float; PFM little endian, rows bottom-up."""
    c, h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P{'F' if c == 3 else 'f'}\n{w} {h}\n-1.0\n".encode())
        f.write(np.ascontiguousarray(img.transpose(1, 2, 0)[::-1]).astype("<f4").tobytes())


def read_pfm(path):
    data = Path(path).read_bytes()
    parts = data.split(b"\n", 3)
    c = 3 if parts[0] == b"PF" else 1
    w, h = map(int, parts[1].split())
    scale = float(parts[2])
    arr = np.frombuffer(parts[3], dtype="<f4" if scale < 0 else ">f4").reshape(h, w, c)
    return arr[::-1].transpose(2, 0, 1).astype(np.float64)


def write_pgm(path, img8):
    h, w = img8.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode())
        f.write(img8.astype(np.uint8).tobytes())


def test_usage_errors_exit_2(cli, tmp_path):
    assert run(cli).returncode == 2
    assert run(cli, "frobnicate", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "smooth").returncode == 2
    assert run(cli, "smooth", "--method", "bogus", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "smooth", "--sigma-s", "-1", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "smooth", "--pad", "-1", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "joint", "in.pfm", "out.pfm").returncode == 2  # --guide required
    assert run(cli, "smooth", "--method", "nc-ls", "--iterations", "0", "in.pfm", "o.pfm").returncode == 2
    assert run(cli, "texture", "--n", "0", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "clipart", "--init-sigma", "-1", "in.pfm", "out.pfm").returncode == 2
    assert run(cli, "texture", "--method", "ls", "in.pfm", "out.pfm").returncode == 2  # no --method


def test_unreadable_input_exits_1(cli, tmp_path):
    assert run(cli, "smooth", "/nonexistent/input.pfm", tmp_path / "o.pfm").returncode == 1
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P7\n1 1\n")
    assert run(cli, "smooth", bad, tmp_path / "o.pfm").returncode == 1
    assert run(cli, "smooth", tmp_path / "x.png", tmp_path / "o.pfm").returncode == 1


@pytest.mark.gpu
def test_ls_lambda0_pgm_round_trip_pixel_exact(gpu, cli, tmp_path):
    rng = np.random.default_rng(81)
    img8 = rng.integers(0, 256, (32, 40))
    write_pgm(tmp_path / "in.pgm", img8)
    r = run(cli, "smooth", "--method", "ls", "--lambda", "0", tmp_path / "in.pgm", tmp_path / "out.pgm")
    assert r.returncode == 0, r.stderr
    data = (tmp_path / "out.pgm").read_bytes()
    out = np.frombuffer(data[-32 * 40:], dtype=np.uint8).reshape(32, 40)
    assert np.array_equal(out, img8)


@pytest.mark.gpu
def test_blf_ls_pfm_matches_api_and_is_deterministic(gpu, cli, oracle, tmp_path):
    img = np.stack([oracle.gen_plane(900 + c, 48, 64, n_sites=12) for c in range(3)])
    write_pfm(tmp_path / "in.pfm", img)
    args = ["--sigma-s", "3", "--sigma-r", "0.1", "--lambda", "500", "--radius", "5", "--iters", "2",
            "--pad", "0"]
    for k in (1, 2):
        r = run(cli, "smooth", *args, tmp_path / "in.pfm", tmp_path / f"o{k}.pfm")
        assert r.returncode == 0, r.stderr
    assert (tmp_path / "o1.pfm").read_bytes() == (tmp_path / "o2.pfm").read_bytes()
    out = read_pfm(tmp_path / "o1.pfm")
    api = gpu.blf_ls(img, lam=500.0, sigma_s=3.0, sigma_r=0.1, iters=2, radius=5)
    assert np.abs(out - api).max() == 0.0
    ref = oracle.blf_ls(img.astype(np.float64), lam=500.0, sigma_s=3.0, sigma_r=0.1, iters=2, radius=5)
    assert np.abs(out - ref).max() <= 1e-4


@pytest.mark.gpu
def test_joint_subcommand(gpu, cli, oracle, tmp_path):
    img = np.stack([oracle.gen_plane(910 + c, 40, 48, n_sites=12) for c in range(3)])
    guide = oracle.gen_plane(999, 40, 48, n_sites=12)[None]
    write_pfm(tmp_path / "in.pfm", img)
    write_pfm(tmp_path / "g.pfm", np.repeat(guide, 3, axis=0))
    r = run(cli, "joint", "--guide", tmp_path / "g.pfm", "--sigma-r", "0.1", "--sigma-s", "3",
            "--radius", "4", "--lambda", "800", "--pad", "0", tmp_path / "in.pfm", tmp_path / "o.pfm")
    assert r.returncode == 0, r.stderr
    out = read_pfm(tmp_path / "o.pfm")
    ref = oracle.blf_ls(img.astype(np.float64), guide.astype(np.float64), lam=800.0, sigma_s=3.0,
                        sigma_r=0.1, iters=1, radius=4)
    assert np.abs(out - ref).max() <= 1e-4


@pytest.mark.gpu
def test_reference_default_padding(gpu, cli, oracle, tmp_path):
    """`smooth` with no --pad uses the reference default 16 (epls_main.cpp:34)."""
    img = np.stack([oracle.gen_plane(950 + c, 30, 34, n_sites=12) for c in range(3)])
    write_pfm(tmp_path / "in.pfm", img)
    r = run(cli, "smooth", "--sigma-s", "1", "--sigma-r", "0.1", "--radius", "3", "--lambda", "600",
            tmp_path / "in.pfm", tmp_path / "o.pfm")
    assert r.returncode == 0, r.stderr
    ref = oracle.blf_ls(img.astype(np.float64), lam=600.0, sigma_s=1.0, sigma_r=0.1, iters=1,
                        radius=3, pad=16)
    assert np.abs(read_pfm(tmp_path / "o.pfm") - ref).max() <= 1e-4


@pytest.mark.gpu
def test_grid_backend_reproduces_reference_cli_defaults(gpu, cli, oracle, tmp_path):
    """`blfls smooth --blf grid in out` = `epls smooth in out` (method blf-ls,
    sigma 12 / 0.04, lambda 1024, pad 16: the reference CLI's defaults)."""
    if not oracle.REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    img = np.stack([oracle.gen_plane(970 + c, 40, 48, n_sites=12) for c in range(3)])
    write_pfm(tmp_path / "in.pfm", img)
    r = run(cli, "smooth", "--blf", "grid", tmp_path / "in.pfm", tmp_path / "o.pfm")
    assert r.returncode == 0, r.stderr
    ref = oracle.ref_smooth_grid(img.astype(np.float64), lam=1024.0, sigma_s=12.0, sigma_r=0.04,
                                 pad=16)
    assert np.abs(read_pfm(tmp_path / "o.pfm") - ref).max() <= 1e-4


@pytest.mark.gpu
def test_nc_ls_method(gpu, cli, oracle, tmp_path):
    """`smooth --method nc-ls` = smooth() with SmootherKind::NC_LS (make_spec,
    epls_main.cpp:48-63): DtParams{sigma_s, sigma_r, --iterations}."""
    img = np.stack([oracle.gen_plane(930 + c, 44, 52, n_sites=12) for c in range(3)])
    write_pfm(tmp_path / "in.pfm", img)
    r = run(cli, "smooth", "--method", "nc-ls", "--sigma-s", "6", "--sigma-r", "0.05",
            "--iterations", "2", "--lambda", "700", tmp_path / "in.pfm", tmp_path / "o.pfm")
    assert r.returncode == 0, r.stderr
    ref = oracle.smooth_nc(img.astype(np.float64), lam=700.0, sigma_s=6.0, sigma_r=0.05, dt_iters=2,
                           pad=16)
    assert np.abs(read_pfm(tmp_path / "o.pfm") - ref).max() <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("cmd,ss,sr,n,s0", [("texture", 8.0, 0.02, 3, 2.5),
                                            ("clipart", 6.0, 0.02, 2, 0.75)])
def test_rolling_subcommands_use_reference_defaults(gpu, cli, oracle, tmp_path, cmd, ss, sr, n, s0):
    """`texture` / `clipart` with no flags = texture_removal / clipart_cleanup
    with the reference CLI's preparse defaults (epls_main.cpp:181-192)."""
    img = np.stack([oracle.gen_plane(960 + c, 40, 48, n_sites=12) for c in range(3)])
    write_pfm(tmp_path / "in.pfm", img)
    r = run(cli, cmd, tmp_path / "in.pfm", tmp_path / "o.pfm")
    assert r.returncode == 0, r.stderr
    ref = oracle.rolling_nc_ls(img.astype(np.float64), lam=1024.0, sigma_s=ss, sigma_r=sr,
                               dt_iters=3, pad=16, n=n, init_sigma=s0)
    d = np.abs(read_pfm(tmp_path / "o.pfm") - ref)
    assert d.max() <= 5e-3 and d.mean() <= 5e-5


def test_raster_codec_round_trips(cli, tmp_path):
    """`blfls convert` (no device): PFM in both byte orders with header
    comments, 8- and 16-bit PGM / PPM, PFM -> PPM quantisation."""
    rng = np.random.default_rng(5)
    img = rng.random((3, 7, 9)).astype(np.float32)
    # big-endian PFM with a comment and CRLF-free tokens split over lines
    c, h, w = img.shape
    be = tmp_path / "be.pfm"
    with open(be, "wb") as f:
        f.write(f"PF\n# made by a test\n{w}\n{h}\n1.0\n".encode())
        f.write(np.ascontiguousarray(img.transpose(1, 2, 0)[::-1]).astype(">f4").tobytes())
    assert run(cli, "convert", be, tmp_path / "le.pfm").returncode == 0
    np.testing.assert_array_equal(read_pfm(tmp_path / "le.pfm"), img.astype(np.float64))
    # 16-bit PGM in, PFM out: value / maxval
    g16 = rng.integers(0, 1001, (5, 6))
    with open(tmp_path / "g16.pgm", "wb") as f:
        f.write(b"P5 6 5 1000\n" + g16.astype(">u2").tobytes())
    assert run(cli, "convert", tmp_path / "g16.pgm", tmp_path / "g16.pfm").returncode == 0
    np.testing.assert_allclose(read_pfm(tmp_path / "g16.pfm")[0], g16 / 1000.0, rtol=0, atol=1e-7)
    # PFM -> 8-bit PPM: clamp to [0, 1], round to nearest
    v = np.array([[[-0.2, 0.0, 0.5 / 255, 0.4, 1.0, 1.7]]] * 3, np.float32)
    write_pfm(tmp_path / "v.pfm", v)
    assert run(cli, "convert", tmp_path / "v.pfm", tmp_path / "v.ppm").returncode == 0
    data = (tmp_path / "v.ppm").read_bytes()
    assert data.startswith(b"P6\n6 1\n255\n")
    px = np.frombuffer(data[len(b"P6\n6 1\n255\n"):], np.uint8).reshape(1, 6, 3)[..., 0]
    assert px.tolist() == [[0, 0, 1, 102, 255, 255]]
    # truncated payload and bad magic are I/O errors (exit 1)
    (tmp_path / "t.pgm").write_bytes(b"P5\n4 4\n255\n" + bytes(10))
    assert run(cli, "convert", tmp_path / "t.pgm", tmp_path / "o.pgm").returncode == 1
    (tmp_path / "m.pgm").write_bytes(b"P2\n1 1\n255\n0\n")
    assert run(cli, "convert", tmp_path / "m.pgm", tmp_path / "o.pgm").returncode == 1
