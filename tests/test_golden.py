"""Oracle (CPU) and GPU path against the committed scipy-generated golden
fixtures at the BASELINE DST-I lengths (tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_scipy.npz"))
LENGTHS = [254, 510, 1022, 2046, 8190]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m", LENGTHS)
def test_oracle_dst_and_ar_at_config_lengths(oracle, m):
    x = np.random.default_rng(m).uniform(-1, 1, m)
    assert rel(oracle.sine1_forward(x), G[f"dst1_{m}"]) <= 1e-14
    x2 = np.random.default_rng(m + 1).uniform(-1, 1, m + 2)
    assert rel(oracle.ar_inverse(x2), G[f"arinv_{m + 2}"]) <= 1e-14
    assert rel(oracle.ar_forward(x2), G[f"arfwd_{m + 2}"]) <= 1e-14


def test_oracle_tensor_apply_golden(oracle):
    X = np.random.default_rng(256).uniform(-1, 1, (256, 256))
    assert rel(oracle.tensor_apply(oracle.KIND_ARINV, X), G["tensor_arinv_256"]) <= 1e-14
    assert rel(oracle.tensor_apply(oracle.KIND_AR, X), G["tensor_arfwd_256"]) <= 1e-14
    assert rel(oracle.tensor_apply(oracle.KIND_SINEI, X), G["tensor_sine1_256"]) <= 1e-14


@pytest.mark.gpu
def test_gpu_tensor_apply_golden(dbx):
    X = np.random.default_rng(256).uniform(-1, 1, (256, 256))
    assert rel(dbx.tensor_apply(dbx.TransformKind.AntiReflectiveInverse, X), G["tensor_arinv_256"]) <= 1e-13
    assert rel(dbx.tensor_apply(dbx.TransformKind.AntiReflective, X), G["tensor_arfwd_256"]) <= 1e-13
    assert rel(dbx.tensor_apply(dbx.TransformKind.SineI, X), G["tensor_sine1_256"]) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("m", LENGTHS)
def test_gpu_ar_lines_golden(dbx, m):
    """A 3-row image whose middle row is the golden input: the row pass of
    tensor_apply applies T~_n along it; the 3-point column transform mixes the
    rows, so compare against the same separable composition built from goldens."""
    n = m + 2
    x2 = np.random.default_rng(m + 1).uniform(-1, 1, n)
    X = np.zeros((3, n))
    X[1] = x2
    got = dbx.tensor_apply(dbx.TransformKind.AntiReflectiveInverse, X)
    # column transform T~_3 applied to e_1 (middle row): T~_3 e_1 = (0, Q_1 * 1, 0) = (0, 1, 0)
    assert rel(got[1], G[f"arinv_{n}"]) <= 1e-13
    # rows 0 and 2 are zero up to rounding: the packed DST shares one complex
    # DFT between two lines, so a zero line sees ~1e-16 crosstalk of its partner
    scale = np.abs(got[1]).max()
    assert np.abs(got[0]).max() <= 1e-14 * scale and np.abs(got[2]).max() <= 1e-14 * scale
