"""Input/output formats of the path's callers (io.hpp).

Binary PGM (P5, maxval <= 65535, big-endian 16-bit samples above 255), the
plain-text matrix format ("rows cols" header, %.17g values) and the PSF text
format ("q1 q2" header then the (2q1+1) x (2q2+1) taps), with the reference's
validation and mask renormalisation rules.  Host-side (these files feed the
GPU path; nothing here runs per iteration).
"""
from __future__ import annotations

import numpy as np

MASS_TOL = 1e-12  # Psf::kMassTol (psf.hpp)


class IOError_(RuntimeError):
    """io_fail: std::runtime_error carrying 'path: why' (io.hpp:20-23)."""


def _fail(path: str, why: str):
    raise IOError_(f"{path}: {why}")


def _tokens(buf: bytes, pos: int, count: int):
    """PNM header tokens, skipping whitespace and '#' comments (io.hpp:25-41)."""
    out = []
    n = len(buf)
    while len(out) < count:
        while pos < n and buf[pos:pos + 1].isspace():
            pos += 1
        if pos < n and buf[pos:pos + 1] == b"#":
            while pos < n and buf[pos:pos + 1] not in (b"\n", b"\r"):
                pos += 1
            continue
        start = pos
        while pos < n and not buf[pos:pos + 1].isspace() and buf[pos:pos + 1] != b"#":
            pos += 1
        if start == pos:
            break
        out.append(buf[start:pos].decode("ascii", "replace"))
    return out, pos


def read_pgm(path: str):
    """Returns (pixels float64 [rows, cols], maxval) (io.hpp:46-67)."""
    try:
        buf = open(path, "rb").read()
    except OSError:
        _fail(path, "cannot open")
    toks, pos = _tokens(buf, 0, 4)
    if len(toks) < 1 or toks[0] != "P5":
        _fail(path, "not a binary PGM (P5)")
    try:
        w, h, maxval = (int(t) for t in toks[1:4])
    except ValueError:
        _fail(path, "bad header")
    if w <= 0 or h <= 0:
        _fail(path, "bad dimensions")
    if maxval <= 0 or maxval > 65535:
        _fail(path, "unsupported maxval")
    pos += 1  # single whitespace after maxval
    wide = maxval > 255
    need = w * h * (2 if wide else 1)
    data = buf[pos:pos + need]
    if len(data) < need:
        _fail(path, "truncated pixel data")
    px = np.frombuffer(data, dtype=">u2" if wide else np.uint8).reshape(h, w).astype(np.float64)
    return px, maxval


def write_pgm(path: str, px, maxval: int = 255):
    """Clamps to [0, maxval] and rounds to nearest on export (io.hpp:69-90)."""
    if not (0 < maxval <= 65535):
        raise ValueError("write_pgm: unsupported maxval")
    px = np.asarray(px, dtype=np.float64)
    v = np.clip(np.round(px), 0.0, float(maxval))  # std::round: half away from zero
    v = np.where(np.abs(px - np.trunc(px)) == 0.5, np.clip(np.trunc(px) + np.sign(px), 0, maxval), v)
    wide = maxval > 255
    body = v.astype(">u2" if wide else np.uint8).tobytes()
    try:
        with open(path, "wb") as fh:
            fh.write(b"P5\n%d %d\n%d\n" % (px.shape[1], px.shape[0], maxval))
            fh.write(body)
    except OSError:
        _fail(path, "cannot open for writing")


def write_matrix_text(path: str, m):
    m = np.asarray(m, dtype=np.float64)
    with open(path, "w") as fh:
        fh.write("%d %d\n" % m.shape)
        for row in m:
            fh.write(" ".join("%.17g" % v for v in row) + "\n")


def read_matrix_text(path: str):
    try:
        toks = open(path).read().split()
    except OSError:
        _fail(path, "cannot open")
    try:
        rows, cols = int(toks[0]), int(toks[1])
    except (IndexError, ValueError):
        _fail(path, "bad matrix header")
    if rows <= 0 or cols <= 0:
        _fail(path, "bad matrix header")
    vals = toks[2:2 + rows * cols]
    if len(vals) < rows * cols:
        _fail(path, "truncated matrix data")
    return np.array([float(v) for v in vals]).reshape(rows, cols)


def _renormalize_mask(taps, path: str):
    """Tiny deviations pass, sub-1% deviations are renormalised, worse fails
    (io.hpp:123-135)."""
    s = float(taps.sum())
    if s <= 0.0:
        _fail(path, "mask has nonpositive total mass")
    dev = abs(s - 1.0)
    if dev <= MASS_TOL:
        return taps
    if dev < 0.01:
        return taps / s
    _fail(path, "mask mass deviates from 1 by more than 1%")


def read_psf(path: str):
    """PSF text ("q1 q2" + taps) or a PGM mask divided by its mass (io.hpp:137-162)."""
    try:
        head = open(path, "rb").read(2)
    except OSError:
        _fail(path, "cannot open")
    if head == b"P5":
        px, _ = read_pgm(path)
        if px.shape[0] % 2 != 1 or px.shape[1] % 2 != 1:
            raise ValueError("read_psf: PGM mask must have odd dimensions")
        s = float(px.sum())
        if s <= 0.0:
            _fail(path, "PGM mask has zero mass")
        return px / s
    toks = open(path).read().split()
    try:
        q1, q2 = int(toks[0]), int(toks[1])
    except (IndexError, ValueError):
        _fail(path, "bad PSF header")
    if q1 < 0 or q2 < 0:
        _fail(path, "bad PSF header")
    n = (2 * q1 + 1) * (2 * q2 + 1)
    vals = toks[2:2 + n]
    if len(vals) < n:
        _fail(path, "truncated PSF data")
    taps = np.array([float(v) for v in vals]).reshape(2 * q1 + 1, 2 * q2 + 1)
    return _renormalize_mask(taps, path)


def write_psf(path: str, taps):
    taps = np.asarray(taps, dtype=np.float64)
    with open(path, "w") as fh:
        fh.write("%d %d\n" % ((taps.shape[0] - 1) // 2, (taps.shape[1] - 1) // 2))
        for row in taps:
            fh.write(" ".join("%.17g" % v for v in row) + "\n")
