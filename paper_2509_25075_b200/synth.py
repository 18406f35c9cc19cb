"""Seeded synthetic workloads shaped like the paper's EMPIAR / CryoBench inputs.

This module holds none of the method's arithmetic (no projection, CTF, loss or
gradient): it only draws seeded inputs, generated in fp64 and rounded to fp32
once (reading L20), which both the CUDA path and the oracle consume.  The
recipe is DESIGN.md §4.

Configs (BASELINE.json ``configs``; N = number of Gaussians, the paper's M):
  T  tiny            N=512     D=32   px=4.0  (CPU oracle runs in seconds)
  S  small protein   N=10k     D=128  px=3.0
  R  EMPIAR-10028    N=50k     D=256  px=1.31 (Nyquist 2.62 A)
  P  EMPIAR-10180    N=100k    D=256  px=1.31
  X  stress          N=500k    D=384  px=1.0
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    N: int          # Gaussians
    D: int          # image edge (even)
    px: float       # Angstrom / pixel
    particles: int  # nominal dataset size (defines an epoch only)

    @property
    def ball_radius(self) -> float:
        """Phantom ball radius in Angstrom: 0.3 * D * px (60% of the box)."""
        return 0.3 * self.D * self.px

    @property
    def sigma0(self) -> float:
        """Phantom scale in Angstrom: 0.5 x Poisson mean nearest-neighbour
        distance 0.554 (V_ball/N)^(1/3) (SPEC init rule S:98)."""
        vball = 4.0 / 3.0 * np.pi * self.ball_radius ** 3
        return 0.5 * 0.554 * (vball / self.N) ** (1.0 / 3.0)


CONFIGS = {
    "T": Workload("T", 512, 32, 4.0, 64),
    "S": Workload("S", 10_000, 128, 3.0, 50_000),
    "R": Workload("R", 50_000, 256, 1.31, 105_000),
    "P": Workload("P", 100_000, 256, 1.31, 130_000),
    "X": Workload("X", 500_000, 384, 1.0, 1_000_000),
    # desk-scale round trip (SPEC acceptance 3): M = 2000 model Gaussians, d = 64,
    # 1.5 A pixels, n = 2000 particles; ground truth = a 200-Gaussian phantom ("A_gt")
    "A": Workload("A", 2_000, 64, 1.5, 2_000),
    "A_gt": Workload("A_gt", 200, 64, 1.5, 2_000),
}


def seed_for(*parts) -> int:
    """seed = hash(config, purpose, ...) as a stable 63-bit integer."""
    h = hashlib.sha256("/".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0
    return q


def morton_order(xyz: np.ndarray, bits: int = 10) -> np.ndarray:
    """Permutation sorting points by the Morton (Z-order) code of their position
    (a memory-layout choice: spatially close Gaussians get close ids)."""
    lo, hi = xyz.min(0), xyz.max(0)
    g = ((xyz - lo) / np.maximum(hi - lo, 1e-12) * ((1 << bits) - 1)).astype(np.uint64)
    code = np.zeros(len(xyz), np.uint64)
    for b in range(bits):
        for ax in range(3):
            code |= ((g[:, ax] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + ax)
    return np.argsort(code, kind="stable")


def phantom(w: Workload, seed: int, morton: bool = True):
    """Ground-truth 'protein': centres uniform in a ball of radius 0.3 D px,
    s = ln sigma0 + U(-0.3, 0.3), q uniform on S^3, rho ~ U(0.5, 1.5).
    Returns (mean_rho[N,4], log_scale[N,4], quat[N,4]) float64."""
    rng = np.random.default_rng(seed)
    N = w.N
    d = rng.standard_normal((N, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = w.ball_radius * rng.random(N) ** (1.0 / 3.0)
    mu = d * r[:, None]
    s = np.log(w.sigma0) + rng.uniform(-0.3, 0.3, (N, 3))
    q = _unit_quats(rng, N)
    rho = rng.uniform(0.5, 1.5, N)
    if morton:
        perm = morton_order(mu)
        mu, s, q, rho = mu[perm], s[perm], q[perm], rho[perm]
    mean_rho = np.concatenate([mu, rho[:, None]], 1)
    log_scale = np.concatenate([s, np.zeros((N, 1))], 1)
    return mean_rho, log_scale, q


def steady_model(w: Workload, seed: int, morton: bool = True):
    """Headline model state: the phantom perturbed by mu += N(0, (0.3 sigma0)^2),
    s += N(0, 0.1^2), rho *= U(0.8, 1.2)."""
    mr, ls, q = phantom(w, seed_for(w.name, "phantom", seed), morton)
    rng = np.random.default_rng(seed_for(w.name, "model", seed))
    mr = mr.copy(); ls = ls.copy()
    mr[:, :3] += rng.normal(0.0, 0.3 * w.sigma0, (w.N, 3))
    ls[:, :3] += rng.normal(0.0, 0.1, (w.N, 3))
    mr[:, 3] *= rng.uniform(0.8, 1.2, w.N)
    return mr, ls, q


def init_model(w: Workload, seed: int, morton: bool = True):
    """SPEC random_init: centres uniform in the cube of half-width the
    ball radius, isotropic sigma = 0.5 x mean NN distance, q uniform, rho = 0.1."""
    rng = np.random.default_rng(seed_for(w.name, "init", seed))
    e = w.ball_radius
    mu = rng.uniform(-e, e, (w.N, 3))
    sig = 0.5 * 0.554 * ((2 * e) ** 3 / w.N) ** (1.0 / 3.0)
    q = _unit_quats(rng, w.N)
    if morton:
        perm = morton_order(mu)
        mu, q = mu[perm], q[perm]
    mr = np.concatenate([mu, np.full((w.N, 1), 0.1)], 1)
    ls = np.concatenate([np.full((w.N, 3), np.log(sig)), np.zeros((w.N, 1))], 1)
    return mr, ls, q


def random_rotations(rng, n):
    """Haar-uniform rotation matrices from the QR decomposition of Gaussian
    matrices (sign-fixed, det +1).  Row-major [n,3,3]."""
    a = rng.standard_normal((n, 3, 3))
    qm, rm = np.linalg.qr(a)
    sgn = np.sign(np.einsum("nii->ni", rm))
    sgn[sgn == 0] = 1.0
    qm = qm * sgn[:, None, :]
    det = np.linalg.det(qm)
    qm[det < 0, :, 0] *= -1.0
    return qm


def particles(w: Workload, B: int, seed: int):
    """Per-particle inputs: rot[B,9] (uniform rotation), shift[B,2] (U(-2,2) px,
    in Angstrom), ctf[B,8] (du, dv A; astig rad; kV; Cs mm; amp contrast; phase; B)."""
    rng = np.random.default_rng(seed_for(w.name, "pose", seed))
    rot = random_rotations(rng, B).reshape(B, 9)
    shift = rng.uniform(-2.0, 2.0, (B, 2)) * w.px
    rc = np.random.default_rng(seed_for(w.name, "ctf", seed))
    mean_df = rc.uniform(10_000.0, 25_000.0, B)
    ddf = rc.uniform(0.0, 1_000.0, B)
    ctf = np.stack([mean_df + 0.5 * ddf, mean_df - 0.5 * ddf, rc.uniform(0.0, np.pi, B),
                    np.full(B, 300.0), np.full(B, 2.7), np.full(B, 0.1), np.zeros(B), np.zeros(B)], 1)
    return rot, shift, ctf


def noise_images(w: Workload, B: int, seed: int, scale: float = 1.0):
    rng = np.random.default_rng(seed_for(w.name, "noise", seed))
    return rng.standard_normal((B, w.D, w.D)) * scale


def f32(*arrays):
    """Round fp64 arrays to fp32 once (both consumers read these bytes)."""
    out = tuple(np.ascontiguousarray(np.asarray(a, dtype=np.float32)) for a in arrays)
    return out if len(out) > 1 else out[0]
