"""Generates tests/golden/*.npz with scipy.fft (pocketfft), an implementation
independent of both the oracle's FFT and FFTW.  scipy's dst(type=1) has FFTW's
RODFT00 convention y_k = 2 sum_j x_j sin(pi (j+1)(k+1)/(m+1)) (the reference's
sine1_forward scales it by 0.5*sqrt(2/(m+1)), transforms.hpp:114-121).

Inputs are regenerated from numpy seeds in the tests, so only outputs are stored.
Run: python tests/golden/make_golden.py
"""
import os

import numpy as np
import scipy.fft as sf

HERE = os.path.dirname(os.path.abspath(__file__))
LENGTHS = [254, 510, 1022, 2046, 8190]  # interior DST-I lengths of the BASELINE configs


def sine1(v):
    m = v.shape[-1]
    return sf.dst(v, type=1, axis=-1) * 0.5 * np.sqrt(2.0 / (m + 1))


def ar_params(m):
    p = 1.0 - np.arange(1, m - 1) / (m - 1)
    return p, np.sqrt(1.0 + p @ p)


def ar_inverse(v):  # transforms.hpp:163-173, along the last axis
    m = v.shape[-1]
    p, a = ar_params(m)
    inner = v[..., 1:-1] - v[..., :1] * p - v[..., -1:] * p[::-1]
    out = np.empty_like(v)
    out[..., 0] = a * v[..., 0]
    out[..., -1] = a * v[..., -1]
    out[..., 1:-1] = sine1(inner)
    return out


def ar_forward(v):  # transforms.hpp:148-160
    m = v.shape[-1]
    p, a = ar_params(m)
    out = np.empty_like(v)
    out[..., 0] = v[..., 0] / a
    out[..., -1] = v[..., -1] / a
    out[..., 1:-1] = sine1(v[..., 1:-1]) + (v[..., :1] / a) * p + (v[..., -1:] / a) * p[::-1]
    return out


def tensor(fn, x):  # columns then rows (transforms.hpp:179-192)
    return fn(fn(x.T).T)


def main():
    out = {}
    for m in LENGTHS:
        x = np.random.default_rng(m).uniform(-1, 1, m)
        out[f"dst1_{m}"] = sine1(x)
        x2 = np.random.default_rng(m + 1).uniform(-1, 1, m + 2)
        out[f"arinv_{m + 2}"] = ar_inverse(x2)
        out[f"arfwd_{m + 2}"] = ar_forward(x2)
    X = np.random.default_rng(256).uniform(-1, 1, (256, 256))
    out["tensor_arinv_256"] = tensor(ar_inverse, X)
    out["tensor_arfwd_256"] = tensor(ar_forward, X)
    out["tensor_sine1_256"] = tensor(sine1, X)
    np.savez_compressed(os.path.join(HERE, "golden_scipy.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
