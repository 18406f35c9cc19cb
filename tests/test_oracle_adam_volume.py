"""Pins for oracle O11 (Adam) and O12 (density query / volume).

Adam is pinned to torch.optim.Adam (fp64, CPU; the PyTorch form adopted by
reading L15) and to the first-step closed form; the volume to SPEC worked
values, the Gaussian mass closed form and the masking tail bound.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
LR = np.array([0.03, 5e-3, 1e-3, 5e-2])  # (mean, log_scale, quat, density)


def rand_state(rng, N):
    p = rng.standard_normal((3, N, 4))
    p[1, :, 3] = 0.0
    p[2] /= np.linalg.norm(p[2], axis=1, keepdims=True)
    return p


def test_adam_first_step_closed_form(orc):
    rng = np.random.default_rng(0)
    N = 9
    p0 = rand_state(rng, N)
    g = rng.standard_normal((3, N, 4))
    p1, m, v = orc.adam(p0, g, np.zeros_like(p0), np.zeros_like(p0), 1, LR)
    lr = np.empty_like(p0)
    lr[0, :, :3], lr[0, :, 3], lr[1], lr[2] = LR[0], LR[3], LR[1], LR[2]
    expect = p0 - lr * g / (np.abs(g) + 1e-8)
    expect[1, :, 3] = p0[1, :, 3]                    # pad lane never updated
    assert np.abs(p1[:2] - expect[:2]).max() < 1e-15
    q = expect[2] / np.linalg.norm(expect[2], axis=1, keepdims=True)
    assert np.abs(p1[2] - q).max() < 1e-15
    assert np.abs(np.linalg.norm(p1[2], axis=1) - 1).max() < 1e-15


def test_adam_zero_gradient_unchanged(orc):
    rng = np.random.default_rng(1)
    p0 = rand_state(rng, 5)
    z = np.zeros_like(p0)
    p1, m, v = orc.adam(p0, z, z, z, 1, LR)
    assert np.array_equal(p1[:2], p0[:2])
    assert np.abs(p1[2] - p0[2]).max() < 1e-15


def test_adam_matches_torch(orc):
    """Several steps vs torch.optim.Adam (fp64) on the non-quaternion classes."""
    rng = np.random.default_rng(2)
    N = 7
    p = rand_state(rng, N)
    m = np.zeros_like(p); v = np.zeros_like(p)
    tp = [torch.tensor(p[0, :, :3].copy(), requires_grad=True), torch.tensor(p[0, :, 3].copy(), requires_grad=True),
          torch.tensor(p[1, :, :3].copy(), requires_grad=True)]
    opt = torch.optim.Adam([{"params": [tp[0]], "lr": LR[0]}, {"params": [tp[1]], "lr": LR[3]},
                            {"params": [tp[2]], "lr": LR[1]}], betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 6):
        g = rng.standard_normal((3, N, 4))
        p, m, v = orc.adam(p, g, m, v, t, LR)
        tp[0].grad = torch.tensor(g[0, :, :3]); tp[1].grad = torch.tensor(g[0, :, 3]); tp[2].grad = torch.tensor(g[1, :, :3])
        opt.step()
    assert np.abs(p[0, :, :3] - tp[0].detach().numpy()).max() < 1e-13
    assert np.abs(p[0, :, 3] - tp[1].detach().numpy()).max() < 1e-13
    assert np.abs(p[1, :, :3] - tp[2].detach().numpy()).max() < 1e-13


def one(mu, s, q, rho):
    return (np.array([[*mu, rho]], float), np.array([[*s, 0.0]], float), np.array([q], float))


def test_volume_spec_values(orc):
    Dv, vs = 16, 1.0
    vol = orc.volume(one([0, 0, 0], [0, 0, 0], [1, 0, 0, 0], 1.0), Dv, vs)
    ex = {e["cite"]: e for e in GOLD["query_density"]}
    assert vol[8, 8, 8] == ex["S:66"]["value"]                   # voxel (8,8,8) centre = origin
    assert abs(vol[8, 8, 9] - ex["S:67"]["value"]) < 1e-15       # 1 A along x
    assert np.all(orc.volume(one([0, 0, 0], [0, 0, 0], [1, 0, 0, 0], 0.0), Dv, vs) == 0.0)


def test_volume_mass(orc):
    rng = np.random.default_rng(3)
    Dv, vs = 40, 1.0
    for _ in range(3):
        s = np.log(rng.uniform(1.5, 2.3, 3))
        q, rho = rng.standard_normal(4), rng.uniform(0.5, 2)
        vol = orc.volume(one(rng.uniform(-1.5, 1.5, 3), s, q, rho), Dv, vs, masked=False)
        expect = rho * (2 * math.pi) ** 1.5 * math.exp(s.sum())
        assert abs(vol.sum() * vs ** 3 - expect) < 1e-8 * expect


def test_volume_masked_tail_and_additivity(orc):
    rng = np.random.default_rng(4)
    Dv, vs, N = 20, 1.2, 6
    params = (np.c_[rng.uniform(-6, 6, (N, 3)), rng.uniform(0.5, 1.5, N)],
              np.c_[np.log(rng.uniform(0.9, 1.8, (N, 3))), np.zeros(N)], rng.standard_normal((N, 4)))
    full = orc.volume(params, Dv, vs, masked=False)
    msk = orc.volume(params, Dv, vs, masked=True)
    # outside the k=3 box Q >= 9, so each culled kernel contributes <= rho e^{-4.5}
    assert np.abs(full - msk).max() <= math.exp(-4.5) * params[0][:, 3].sum()
    assert np.all(msk <= full + 1e-15)
    a = orc.volume(tuple(p[:3] for p in params), Dv, vs)
    b = orc.volume(tuple(p[3:] for p in params), Dv, vs)
    assert np.abs(a + b - msk).max() < 1e-14 * np.abs(msk).max()


def test_volume_box_is_tightest_ellipsoid_box(orc):
    """O12 pin (both sides of the box): a single Gaussian's masked volume is non-zero exactly on
    the integer voxel box of its k = 3 ellipsoid {d : d^T Sigma^-1 d <= 9}.  The ellipsoid's
    axis extents come from an independent parametric sampling of its surface (scipy rotation,
    numpy Cholesky): mu + 3 L u over unit vectors u.  A box that is too small (voxels of the
    ellipsoid box missing) or too large (extra voxels) both fail."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(12)
    Dv, vs, k = 24, 1.1, 3.0
    # unit vectors on a fine sphere grid: the sampled extreme is within ~1e-6 of the true one
    th, ph = np.meshgrid(np.linspace(0, np.pi, 801), np.linspace(0, 2 * np.pi, 1601), indexing="ij")
    U = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)]).reshape(3, -1)
    checked = 0
    for _ in range(12):
        mu = rng.uniform(-4, 4, 3)
        s = np.log(rng.uniform(0.5, 2.2, 3))
        q = rng.standard_normal(4)
        R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
        S = R @ np.diag(np.exp(2 * s)) @ R.T
        pts = mu[:, None] + k * np.linalg.cholesky(S) @ U
        lo = pts.min(1) / vs + Dv // 2
        hi = pts.max(1) / vs + Dv // 2
        if np.any(np.abs(lo - np.round(lo)) < 1e-4) or np.any(np.abs(hi - np.round(hi)) < 1e-4):
            continue   # a bound this close to an integer cannot be decided by sampling
        elo = np.clip(np.ceil(lo), 0, Dv).astype(int)
        ehi = np.clip(np.floor(hi), -1, Dv - 1).astype(int)
        vol = orc.volume(one(mu, s, q, 1.0), Dv, vs, masked=True)   # [c][b][a], x = a fastest
        nz = np.nonzero(vol)
        got_lo = [nz[2].min(), nz[1].min(), nz[0].min()]
        got_hi = [nz[2].max(), nz[1].max(), nz[0].max()]
        assert got_lo == list(elo) and got_hi == list(ehi), (got_lo, got_hi, elo, ehi)
        # and the support is the full box (no holes: exp(-Q/2) > 0 in fp64 for Q <= ~1400)
        assert len(nz[0]) == np.prod(ehi - elo + 1)
        checked += 1
    assert checked >= 8
