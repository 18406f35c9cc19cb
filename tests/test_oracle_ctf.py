"""Pins for oracle O6-O7 (CTF on the DFT grid, DFT, CTF application, Parseval).

Pinned against SPEC worked values (golden file), numpy.fft (library DFT),
a direct O(D^4) circular convolution, and mathematical identities.
"""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
CTF_GOLD = {e["cite"]: e for e in GOLD["ctf"]}


def astig(du=15000.0, dv=14300.0, ang=0.3, kV=300.0, cs=2.7, a=0.1, ph=0.0, bf=0.0):
    return np.array([du, dv, ang, kV, cs, a, ph, bf])


def test_wavelength_300kV(orc):
    ex = CTF_GOLD["S:241"]
    assert abs(orc.wavelength_A(ex["kV"]) - ex["lambda"]) < ex["tol"]
    # textbook values: 200 kV -> 0.02508 A, 100 kV -> 0.03701 A
    assert abs(orc.wavelength_A(200.0) - 0.02508) < 1e-5
    assert abs(orc.wavelength_A(100.0) - 0.03701) < 1e-5


def test_ctf_special_cases(orc):
    D, px = 16, 1.5
    C = orc.ctf(np.array([0, 0, 0.4, 300, 0, 1.0, 0, 0]), D, px)
    assert np.all(C == CTF_GOLD["S:239"]["value"])
    C = orc.ctf(np.array([12000, 11000, 0.4, 300, 2.7, 0.0, 0, 0]), D, px)
    assert C[0, 0] == CTF_GOLD["S:240"]["value"]
    C = orc.ctf(astig(a=0.07), D, px)
    assert abs(C[0, 0] + 0.07) < 1e-15      # C(0) = -alpha cos(phase)


def test_ctf_bounded_by_envelope(orc):
    D, px = 32, 1.2
    p = astig(bf=80.0)
    C = orc.ctf(p, D, px)
    k = np.fft.fftfreq(D, d=px)
    s2 = k[None, :] ** 2 + k[:, None] ** 2
    env = np.exp(-80.0 * s2 / 4.0)
    # Nyquist-averaged bins are bounded by the largest alias envelope (same |f|)
    assert np.all(np.abs(C) <= env * (1 + 1e-12) + 1e-15)


def test_ctf_hermitian_even_exact(orc):
    """Reading L12: C(k) = C(-k mod D) bitwise for astigmatic CTFs."""
    for D in (16, 32, 34):
        C = orc.ctf(astig(), D, 1.31)
        Cn = C[(-np.arange(D)) % D][:, (-np.arange(D)) % D]
        assert np.array_equal(C, Cn)


def test_ctf_only_nyquist_changed(orc):
    """Off the Nyquist row/column C equals the raw CTF at the unique alias."""
    D, px = 16, 1.31
    p = astig()
    C = orc.ctf(p, D, px)
    f = np.fft.fftfreq(D, d=px)
    for ky in range(D):
        for kx in range(D):
            if ky == D // 2 or kx == D // 2:
                continue
            assert C[ky, kx] == orc.ctf_raw(p, f[kx], f[ky])
    # the corner bin averages 4 aliases
    n = 1.0 / (2 * px)
    corner = np.mean([orc.ctf_raw(p, a, b) for a in (n, -n) for b in (n, -n)])
    assert abs(C[D // 2, D // 2] - corner) < 1e-15


def test_dft_matches_numpy(orc):
    rng = np.random.default_rng(0)
    for D in (8, 16, 18):
        x = rng.standard_normal((D, D))
        F = orc.dft2(x)
        assert np.abs(F - np.fft.fft2(x)).max() < 1e-12 * np.abs(F).max()
        y = orc.dft2(F.real, F.imag, inverse=True)
        assert np.abs(y.real - x).max() < 1e-13 and np.abs(y.imag).max() < 1e-13


def test_apply_ctf_identities(orc):
    rng = np.random.default_rng(1)
    D = 16
    x = rng.standard_normal((D, D))
    out, r = orc.apply_ctf(np.ones((D, D)), x)
    assert np.abs(out - x).max() < 1e-13
    out, r = orc.apply_ctf(-np.ones((D, D)), x)
    assert np.abs(out + x).max() < 1e-13


def test_apply_ctf_real_and_equals_circular_convolution(orc):
    """output equals direct O(D^4) circular convolution with the real PSF;
    with the Hermitian fix the imaginary residue vanishes (reading L12)."""
    rng = np.random.default_rng(2)
    D, px = 16, 1.31
    C = orc.ctf(astig(ang=0.9), D, px)
    psf = np.fft.ifft2(C)
    assert np.abs(psf.imag).max() < 1e-15
    psf = psf.real
    x = rng.standard_normal((D, D))
    out, r = orc.apply_ctf(C, x)
    assert r < 1e-12
    direct = np.zeros((D, D))
    for v in range(D):
        for u in range(D):
            acc = 0.0
            for vp in range(D):
                for up in range(D):
                    acc += x[vp, up] * psf[(v - vp) % D, (u - up) % D]
            direct[v, u] = acc
    assert np.abs(direct - out).max() < 1e-12 * np.abs(out).max()
    # delta image -> the PSF
    delta = np.zeros((D, D)); delta[3, 5] = 1.0
    o2, _ = orc.apply_ctf(C, delta)
    assert np.abs(o2 - np.roll(np.roll(psf, 3, 0), 5, 1)).max() < 1e-14


def test_unsymmetrised_ctf_would_be_complex(orc):
    """Why L12 is needed: the raw CTF on an even grid is not Hermitian for
    astigmatism angles outside {0, pi/2}."""
    D, px = 16, 1.31
    p = astig(ang=0.3)
    f = np.fft.fftfreq(D, d=px)  # Nyquist bin only as -1/(2px)
    Craw = np.array([[orc.ctf_raw(p, f[kx], f[ky]) for kx in range(D)] for ky in range(D)])
    x = np.random.default_rng(3).standard_normal((D, D))
    _, r = orc.apply_ctf(Craw, x)
    assert r > 1e-3
    _, r2 = orc.apply_ctf(orc.ctf(p, D, px), x)
    assert r2 < 1e-12


def test_ctf_composition_and_linearity(orc):
    rng = np.random.default_rng(4)
    D, px = 16, 1.31
    C1, C2 = orc.ctf(astig(), D, px), orc.ctf(astig(du=21000, dv=20000, ang=1.2), D, px)
    x, y = rng.standard_normal((2, D, D))
    a, _ = orc.apply_ctf(C2, orc.apply_ctf(C1, x)[0])
    b, _ = orc.apply_ctf(C1 * C2, x)
    assert np.abs(a - b).max() < 1e-13
    l1, _ = orc.apply_ctf(C1, 2.0 * x - 3.0 * y)
    l2 = 2.0 * orc.apply_ctf(C1, x)[0] - 3.0 * orc.apply_ctf(C1, y)[0]
    assert np.abs(l1 - l2).max() < 1e-12
