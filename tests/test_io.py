"""Input/output formats (io.hpp): PGM P5 8/16-bit round trips,
clamping + half-away-from-zero rounding on export, header comments, matrix and
PSF text formats with the reference's renormalisation rule and errors."""
import numpy as np
import pytest

from paper_1211_0393_b200 import io


def test_pgm_round_trip_8_and_16_bit(tmp_path):
    rng = np.random.default_rng(0)
    for maxval in (255, 4095, 65535):
        px = rng.integers(0, maxval + 1, size=(7, 11)).astype(np.float64)
        p = str(tmp_path / f"a{maxval}.pgm")
        io.write_pgm(p, px, maxval)
        got, mv = io.read_pgm(p)
        assert mv == maxval and got.shape == (7, 11) and np.array_equal(got, px)


def test_pgm_export_clamps_and_rounds_half_away(tmp_path):
    p = str(tmp_path / "r.pgm")
    io.write_pgm(p, np.array([[-3.0, 0.5, 1.5, 2.5, 254.6, 300.0]]), 255)
    got, _ = io.read_pgm(p)
    assert got.tolist() == [[0, 1, 2, 3, 255, 255]]


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# comment\n2 1\n255\n\x01\x02")
    got, _ = io.read_pgm(str(p))
    assert got.tolist() == [[1.0, 2.0]]
    (tmp_path / "t.pgm").write_bytes(b"P5\n2 2\n255\n\x01")
    with pytest.raises(io.IOError_, match="truncated"):
        io.read_pgm(str(tmp_path / "t.pgm"))
    (tmp_path / "p2.pgm").write_bytes(b"P2\n1 1\n255\n1")
    with pytest.raises(io.IOError_, match="P5"):
        io.read_pgm(str(tmp_path / "p2.pgm"))
    with pytest.raises(ValueError):
        io.write_pgm(str(tmp_path / "x.pgm"), np.zeros((1, 1)), 70000)


def test_matrix_and_psf_text(tmp_path):
    m = np.random.default_rng(1).uniform(size=(3, 4))
    io.write_matrix_text(str(tmp_path / "m.txt"), m)
    assert np.array_equal(io.read_matrix_text(str(tmp_path / "m.txt")), m)
    taps = np.random.default_rng(2).uniform(size=(3, 5))
    taps /= taps.sum()
    io.write_psf(str(tmp_path / "k.txt"), taps)
    assert np.array_equal(io.read_psf(str(tmp_path / "k.txt")), taps)
    # sub-1% deviation is renormalised, larger fails (io.hpp:123-135)
    io.write_psf(str(tmp_path / "k2.txt"), taps * 1.005)
    assert abs(io.read_psf(str(tmp_path / "k2.txt")).sum() - 1.0) < 1e-15
    io.write_psf(str(tmp_path / "k3.txt"), taps * 1.05)
    with pytest.raises(io.IOError_, match="1%"):
        io.read_psf(str(tmp_path / "k3.txt"))
    # PGM masks are divided by their mass
    io.write_pgm(str(tmp_path / "k.pgm"), np.array([[0, 1, 0], [1, 4, 1], [0, 1, 0]], float), 255)
    k = io.read_psf(str(tmp_path / "k.pgm"))
    assert abs(k.sum() - 1.0) < 1e-15 and k[1, 1] == 0.5
