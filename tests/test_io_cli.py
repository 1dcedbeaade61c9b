"""Netpbm I/O and CLI front end (host side; the GPU runs are marked gpu).

Mirrors the reference's test_io.py / test_cli.py checks
(/root/reference/pkg/tests/test_io.py, test_cli.py) for the formats and the
CLI surface this package implements."""
import numpy as np
import pytest

import oracle
from paper_2505_22938_b200 import ShapeSpec, make_kernel, read_image, write_image
from paper_2505_22938_b200.cli import BENCH_CSV_HEADER, main, parse_shape


@pytest.mark.parametrize("dtype,shape", [
    (np.uint8, (13, 17)), (np.uint8, (13, 17, 3)), (np.uint16, (9, 5)),
    (np.uint16, (9, 5, 3)), (np.float32, (11, 7)), (np.float32, (11, 7, 3))])
def test_round_trip(tmp_path, rng, dtype, shape):
    if dtype == np.float32:
        img, ext = rng.standard_normal(shape).astype(np.float32), "pfm"
    else:
        img = rng.integers(0, np.iinfo(dtype).max + 1, shape).astype(dtype)
        ext = "ppm" if len(shape) == 3 else "pgm"
    p1, p2 = tmp_path / f"a.{ext}", tmp_path / f"b.{ext}"
    write_image(p1, img)
    again = read_image(p1)
    assert again.dtype == img.dtype and np.array_equal(again, img)
    write_image(p2, again)
    assert p1.read_bytes() == p2.read_bytes()


def test_pinned_read_matches(tmp_path, rng):
    img = rng.integers(0, 65536, (33, 21, 3)).astype(np.uint16)
    write_image(tmp_path / "x.ppm", img)
    import torch
    got = read_image(tmp_path / "x.ppm", pinned=torch.cuda.is_available())
    assert np.array_equal(got, img)


def test_pgm16_big_endian_and_pfm_layout(tmp_path):
    write_image(tmp_path / "x.pgm", np.array([[0x0102]], np.uint16))
    assert (tmp_path / "x.pgm").read_bytes().endswith(b"\x01\x02")
    write_image(tmp_path / "x.pfm", np.array([[1.0, 2.0], [3.0, 4.0]], np.float32))
    data = (tmp_path / "x.pfm").read_bytes()
    assert data.startswith(b"Pf\n2 2\n-1.0\n")
    assert np.frombuffer(data[-16:], "<f4").tolist() == [3.0, 4.0, 1.0, 2.0]
    # big-endian PFM (positive scale) reads too
    be = b"Pf\n2 1\n1.0\n" + np.array([5.0, 6.0], ">f4").tobytes()
    (tmp_path / "b.pfm").write_bytes(be)
    assert read_image(tmp_path / "b.pfm").tolist() == [[5.0, 6.0]]


def test_header_comments_and_bad_files(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# a comment\n2 1\n# another\n255\n\x07\x09")
    assert read_image(p).tolist() == [[7, 9]]
    p.write_bytes(b"P4\n1 1\n255\n\x00")
    with pytest.raises(ValueError, match="magic"):
        read_image(p)
    p.write_bytes(b"P5\n1 1\n100\n\x00")
    with pytest.raises(ValueError, match="maxval"):
        read_image(p)
    p.write_bytes(b"P5\n4 4\n255\n\x00")
    with pytest.raises(ValueError, match="truncated"):
        read_image(p)
    with pytest.raises(ValueError, match="dtype"):
        write_image(tmp_path / "x.pgm", np.zeros((3, 3), np.int64))


def test_parse_shape():
    assert parse_shape("circle", 5) == ShapeSpec("circle", 5)
    assert parse_shape("square", 3) == ShapeSpec("square", 3)
    assert parse_shape("poly:6", 4) == ShapeSpec("regular_polygon", 4, sides=6)
    assert parse_shape("poly:8:22.5", 4) == ShapeSpec("regular_polygon", 4, sides=8,
                                                      rotation_deg=22.5)
    with pytest.raises(ValueError):
        parse_shape("blob", 4)


@pytest.fixture
def gray_pgm(tmp_path, rng):
    img = rng.integers(0, 256, (72, 64)).astype(np.uint8)
    path = tmp_path / "in.pgm"
    write_image(path, img)
    return path, img


def test_usage_error_exits_2(gray_pgm, tmp_path):
    path, _ = gray_pgm
    for argv in (["filter", str(path), str(tmp_path / "o.pgm"), "--radius"],
                 ["filter", str(path), str(tmp_path / "o.pgm"), "--radius", "3",
                  "--engine", "warp"]):
        with pytest.raises(SystemExit) as exc:
            main(argv)
        assert exc.value.code == 2


def test_processing_error_exits_1(tmp_path, gray_pgm, capsys):
    # validation errors are raised by the host prologue, before any device work
    path, _ = gray_pgm
    assert main(["filter", str(tmp_path / "missing.pgm"), str(tmp_path / "o.pgm"),
                 "--radius", "3"]) == 1
    assert main(["filter", str(path), str(tmp_path / "o.pgm"), "--radius", "300"]) == 1
    assert main(["filter", str(path), str(tmp_path / "o.pgm"), "--radius", "3",
                 "--percentile", "150"]) == 1
    assert "error" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_filter_matches_oracle(tmp_path, gray_pgm):
    path, img = gray_pgm
    out = tmp_path / "out.pgm"
    assert main(["filter", str(path), str(out), "--radius", "0"]) == 0
    assert np.array_equal(read_image(out), img)
    for extra, pct in ((["--percentile", "30"], 0.3), (["--shape", "poly:6"], 0.5)):
        assert main(["filter", str(path), str(out), "--radius", "6", *extra]) == 0
        shape = ShapeSpec("regular_polygon", 6, sides=6) if "poly:6" in extra else \
            ShapeSpec("circle", 6)
        assert np.array_equal(read_image(out), oracle.fast_filter(img, shape, pct))
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    for dest in (a, b):
        assert main(["filter", str(path), str(dest), "--radius", "7", "--engine", "fast"]) == 0
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_cli_percentile_zero_and_map(tmp_path, gray_pgm, rng):
    path, img = gray_pgm
    out = tmp_path / "out.pgm"
    assert main(["filter", str(path), str(out), "--radius", "5", "--percentile", "0"]) == 0
    k = make_kernel(ShapeSpec("circle", 5))
    padded = np.pad(img, 5, mode="edge")
    got = read_image(out)
    y, x = 30, 20
    assert got[y, x] == min(padded[y + 5 + dy, x + 5 + dx] for dx, dy in zip(k.off_dx, k.off_dy))
    pmap = rng.integers(0, 101, img.shape).astype(np.uint8)
    write_image(tmp_path / "p.pgm", pmap)
    assert main(["filter", str(path), str(out), "--radius", "4", "--percentile-map",
                 str(tmp_path / "p.pgm")]) == 0
    want = oracle.fast_filter(img, ShapeSpec("circle", 4), pmap.astype(np.float64) / 100.0)
    assert np.array_equal(read_image(out), want)


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path, rng, capsys):
    img = rng.integers(0, 256, (128, 128)).astype(np.uint8)
    write_image(tmp_path / "in.pgm", img)
    assert main(["bench", str(tmp_path / "in.pgm"), "--radii", "2,4", "--repeats", "1",
                 "--engine", "fast"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == BENCH_CSV_HEADER and len(lines) == 3
    for line, radius in zip(lines[1:], (2, 4)):
        f = line.split(",")
        assert int(f[0]) == radius and f[1] == "fast" and f[2] == "uint8"
        mp, ms, mps = float(f[3]), float(f[4]), float(f[5])
        assert mp == pytest.approx(128 * 128 / 1e6, abs=5e-4)
        assert ms > 0 and mps == pytest.approx(mp / (ms / 1e3), rel=0.05)
