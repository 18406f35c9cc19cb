"""Pins for oracle O7-O10 (loss, image gradient, per-(i,j) backward, finalize).

Pinned by central finite differences of the oracle's own loss with the masks
frozen at the base point ("differentiate what you compute"), the
Parseval identity against numpy.fft, the rho-rescale identity, the
zero-residual / zero-CTF special cases and exact locality.
"""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

CLASSES = {"mu": [0, 1, 2], "rho": [3], "s": [4, 5, 6], "q": [8, 9, 10, 11]}


def tiny_case(seed, N=8, B=2, D=16, px=1.0, obs_scale=1.0):
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-0.25 * D * px, 0.25 * D * px, (N, 3))
    s = np.log(rng.uniform(0.8, 1.6, (N, 3)) * px)
    q = rng.standard_normal((N, 4))
    rho = rng.uniform(0.5, 1.5, N)
    params = [np.c_[mu, rho], np.c_[s, np.zeros(N)], q]
    rot = np.stack([Rotation.random(random_state=seed * 10 + i).as_matrix().reshape(9) for i in range(B)])
    shift = rng.uniform(-1.5, 1.5, (B, 2))
    ctf = np.stack([[rng.uniform(9000, 16000), rng.uniform(8000, 15000), rng.uniform(0, np.pi),
                     300.0, 2.7, 0.1, 0.0, rng.uniform(0, 20)] for _ in range(B)])
    obs = rng.standard_normal((B, D, D)) * obs_scale
    return params, rot, shift, ctf, obs, D, px


def flat_to_params(params, j, c, delta):
    p = [a.copy() for a in params]
    arr, comp = (0, c) if c < 4 else ((1, c - 4) if c < 8 else (2, c - 8))
    p[arr][j, comp] += delta
    return p


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gradient_vs_central_fd(orc, seed):
    params, rot, shift, ctf, obs, D, px = tiny_case(seed)
    aabb, vis, _ = orc.splats(params, rot, shift, D, px)
    frozen = (aabb, vis)
    base = orc.loss_grad(params, rot, shift, ctf, obs, D, px, frozen=frozen)
    g = base["grad"]
    N = g.shape[0]
    fd = np.zeros_like(g)
    for j in range(N):
        for c in [0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 11]:
            h = 1e-5 if c < 3 else 1e-6
            lp = orc.loss_grad(flat_to_params(params, j, c, h), rot, shift, ctf, obs, D, px, frozen=frozen)["total"]
            lm = orc.loss_grad(flat_to_params(params, j, c, -h), rot, shift, ctf, obs, D, px, frozen=frozen)["total"]
            fd[j, c] = (lp - lm) / (2 * h)
    for name, cols in CLASSES.items():
        err = np.abs(fd[:, cols] - g[:, cols]).max() / np.abs(g[:, cols]).max()
        assert err < 1e-6, (name, err)
    # quaternion gradient is tangent to the sphere
    qh = params[2] / np.linalg.norm(params[2], axis=1, keepdims=True)
    radial = np.abs((g[:, 8:12] * qh).sum(1)).max() / np.abs(g[:, 8:12]).max()
    assert radial < 1e-12


def test_parseval_loss_and_pred_real(orc):
    params, rot, shift, ctf, obs, D, px = tiny_case(4, D=18)
    out = orc.loss_grad(params, rot, shift, ctf, obs, D, px, want=("proj", "pred"))
    for i in range(rot.shape[0]):
        C = orc.ctf(ctf[i], D, px)
        R = C * np.fft.fft2(out["proj"][i]) - np.fft.fft2(obs[i])
        parseval = (np.abs(R) ** 2).sum() / D ** 2
        assert abs(parseval - out["loss"][i]) < 1e-12 * out["loss"][i]
        assert abs(((out["pred"][i] - obs[i]) ** 2).sum() - out["loss"][i]) < 1e-12 * out["loss"][i]
        ref = np.fft.ifft2(C * np.fft.fft2(out["proj"][i]))
        assert np.abs(ref.imag).max() < 1e-12 * np.abs(ref.real).max()
        assert np.abs(ref.real - out["pred"][i]).max() < 1e-12 * np.abs(ref.real).max()


def test_rho_rescale_identity(orc):
    """dL/dc at c=1 for rho -> c rho equals sum_j rho_j dL/drho_j = 2(<P,P> - <P,O>)."""
    params, rot, shift, ctf, obs, D, px = tiny_case(5)
    out = orc.loss_grad(params, rot, shift, ctf, obs, D, px, want=("pred",))
    lhs = (params[0][:, 3] * out["grad"][:, 3]).sum()
    P = out["pred"]
    rhs = 2.0 * ((P * P).sum() - (P * obs).sum())
    assert abs(lhs - rhs) < 1e-12 * abs(rhs)


def test_zero_residual_and_zero_ctf(orc):
    params, rot, shift, ctf, obs, D, px = tiny_case(6)
    out = orc.loss_grad(params, rot, shift, ctf, obs, D, px, want=("pred",))
    at_min = orc.loss_grad(params, rot, shift, ctf, out["pred"], D, px)
    assert np.all(at_min["loss"] == 0.0) and np.all(at_min["grad"] == 0.0)
    zero_ctf = ctf.copy()
    zero_ctf[:, 0:2] = 0.0; zero_ctf[:, 4] = 0.0; zero_ctf[:, 5] = 0.0; zero_ctf[:, 6] = 0.0
    z = orc.loss_grad(params, rot, shift, zero_ctf, obs, D, px)
    assert np.allclose(z["loss"], (obs ** 2).sum((1, 2)), rtol=1e-14)
    assert np.all(z["grad"] == 0.0)


def test_culled_gaussian_has_exact_zero_row(orc):
    """a Gaussian culled from every tile (off-frame) gets an exactly zero row."""
    params, rot, shift, ctf, obs, D, px = tiny_case(7)
    params[0][2, :3] = [1e4, -1e4, 3e3]
    params[0][5, 3] = 0.0    # rho = 0 -> |amp| = 0 <= tau -> culled
    out = orc.loss_grad(params, rot, shift, ctf, obs, D, px)
    assert np.all(out["grad"][2] == 0.0) and np.all(out["grad"][5] == 0.0)
    assert np.abs(out["grad"][0]).max() > 0


def test_batch_gradient_is_sum_over_particles(orc):
    """The batch loss is a sum over particles (reading L14), so the DP all-reduce
    of per-shard gradients equals the full-batch gradient."""
    params, rot, shift, ctf, obs, D, px = tiny_case(8, B=4)
    full = orc.loss_grad(params, rot, shift, ctf, obs, D, px)
    a = orc.loss_grad(params, rot[:1], shift[:1], ctf[:1], obs[:1], D, px)
    b = orc.loss_grad(params, rot[1:], shift[1:], ctf[1:], obs[1:], D, px)
    assert np.abs(a["grad"] + b["grad"] - full["grad"]).max() < 1e-12 * np.abs(full["grad"]).max()
    assert abs(a["total"] + b["total"] - full["total"]) < 1e-12 * full["total"]


@pytest.mark.parametrize("pixmask", [2, 4, 6])
def test_pixel_mask_variants_gradient_vs_fd(orc, pixmask):
    """SURVEY §8(f1) variants (exact ellipse Q <= k^2, per-pixel tau of Eq. 8): the oracle
    gradient restricted to the kept pixels equals central finite differences of its own loss
    (a step of 1e-6 moves no pixel across a mask boundary in these cases)."""
    params, rot, shift, ctf, obs, D, px = tiny_case(4)
    aabb, vis, _ = orc.splats(params, rot, shift, D, px)
    tau = 0.05
    frozen = (aabb, vis)
    base = orc.loss_grad(params, rot, shift, ctf, obs, D, px, tau=tau, frozen=frozen, pixmask=pixmask)
    plain = orc.loss_grad(params, rot, shift, ctf, obs, D, px, tau=tau, frozen=frozen)
    assert abs(base["total"] - plain["total"]) > 1e-9 * plain["total"]   # the mask changes the result
    g = base["grad"]
    fd = np.zeros_like(g)
    for j in range(g.shape[0]):
        for c in [0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 11]:
            h = 1e-5 if c < 3 else 1e-6
            lp = orc.loss_grad(flat_to_params(params, j, c, h), rot, shift, ctf, obs, D, px, tau=tau,
                               frozen=frozen, pixmask=pixmask)["total"]
            lm = orc.loss_grad(flat_to_params(params, j, c, -h), rot, shift, ctf, obs, D, px, tau=tau,
                               frozen=frozen, pixmask=pixmask)["total"]
            fd[j, c] = (lp - lm) / (2 * h)
    for name, cols in CLASSES.items():
        err = np.abs(fd[:, cols] - g[:, cols]).max() / np.abs(g[:, cols]).max()
        assert err < 1e-6, (name, err)
