"""Training loop around the GEM step.

* ``fit``: epochs x ceil(n / batch) Adam steps over seeded, shuffled minibatches (SPEC train,
  S:358-361); every arithmetic step of a training step runs in libgem.so through
  ``gem.Trainer``; the per-epoch mean loss is read once per epoch.
* ``save_checkpoint`` / ``load_checkpoint``: parameters, Adam moments and the Adam step count
  in a small versioned binary format; save -> load -> save is byte-identical and, since the GPU
  step is bitwise deterministic, resuming reproduces the uninterrupted run bit for bit.
* ``split_halves``: the gold-standard half split.
* ``fsc`` / ``resolution`` / ``gsfsc``: Fourier shell correlation of two half-map volumes and
  the 0.143 criterion (Eq. 9).  An evaluation metric, not part of the training step:
  computed on the host with numpy.
* ``simulate`` / ``train_halves``: the synthetic round trip (SPEC acceptance 3) -- images
  of a ground-truth Gaussian set through libgem's forward + CTF plus noise, then two independent
  half-set reconstructions whose volumes (gem_render_volume) give the GSFSC.
"""
from __future__ import annotations

import os
import struct

import numpy as np

MAGIC = b"GEMCKPT1"
VERSION = 1
_HDR = struct.Struct("<8sIIqqq")   # magic, version, flags, N, adam_t, epoch


class CheckpointError(ValueError):
    """Malformed checkpoint: bad magic, unsupported version or truncated payload."""


def epoch_batches(n: int, batch: int, seed: int, epoch: int):
    """Particle index batches of one epoch: a seeded permutation cut into ceil(n / batch) batches."""
    perm = np.random.default_rng((seed, epoch)).permutation(n)
    return [perm[k:k + batch] for k in range(0, n, batch)]


def fit(trainer, data: dict, epochs: int, batch: int, seed: int = 0, start_epoch: int = 0,
        checkpoint: str | None = None, checkpoint_every: int = 0):
    """Train ``trainer`` (gem.Trainer) on ``data`` = {'rot' [n,9], 'shift' [n,2], 'ctf' [n,8],
    'obs' [n,D,D]} device tensors.  Returns the per-epoch mean loss (sum over pixels per particle,
    averaged over the epoch's particles)."""
    import torch
    n = data["rot"].shape[0]
    dev = data["rot"].device
    history = []
    for ep in range(start_epoch, epochs):
        tot = torch.zeros((), dtype=torch.float64, device=dev)
        for idx in epoch_batches(n, batch, seed, ep):
            sel = torch.as_tensor(idx, device=dev)
            loss = trainer.train_step(*(data[k].index_select(0, sel).contiguous()
                                        for k in ("rot", "shift", "ctf", "obs")))
            tot += loss[-1]
        history.append(float(tot) / n)
        if not np.isfinite(history[-1]):
            raise FloatingPointError(f"non-finite loss in epoch {ep}")
        trainer.step_ctx.stats(check=True)   # raises if any step's tile lists overflowed (sticky flag)
        if checkpoint and checkpoint_every and (ep + 1) % checkpoint_every == 0:
            save_checkpoint(checkpoint, trainer.params.t, trainer.m.t, trainer.v.t, trainer.t, ep + 1)
    return history


def save_checkpoint(path: str, params, m, v, adam_t: int, epoch: int, flags: int = 0):
    """Write params, Adam m and v ([3, N, 4] float32 tensors or arrays) atomically."""
    arrs = [np.ascontiguousarray(_np(a), dtype=np.float32) for a in (params, m, v)]
    N = arrs[0].shape[1]
    for a in arrs:
        if a.shape != (3, N, 4):
            raise CheckpointError(f"expected [3, N, 4] arrays, got {a.shape}")
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(_HDR.pack(MAGIC, VERSION, flags, N, int(adam_t), int(epoch)))
        for a in arrs:
            f.write(a.tobytes())
    os.replace(tmp, path)


def load_checkpoint(path: str):
    """Returns (params, m, v, adam_t, epoch, flags); arrays are float32 [3, N, 4]."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HDR.size:
        raise CheckpointError("truncated header")
    magic, version, flags, N, adam_t, epoch = _HDR.unpack_from(raw)
    if magic != MAGIC:
        raise CheckpointError("not a GEM checkpoint (bad magic)")
    if version != VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    need = _HDR.size + 3 * 3 * N * 4 * 4
    if len(raw) != need:
        raise CheckpointError(f"truncated payload: {len(raw)} of {need} bytes")
    body = np.frombuffer(raw, dtype=np.float32, offset=_HDR.size).reshape(3, 3, N, 4)
    return body[0].copy(), body[1].copy(), body[2].copy(), adam_t, epoch, flags


def restore(trainer, path: str) -> int:
    """Load a checkpoint into a gem.Trainer (parameters, moments, Adam step); returns the epoch."""
    import torch
    p, m, v, t, epoch, _ = load_checkpoint(path)
    for dst, src in ((trainer.params.t, p), (trainer.m.t, m), (trainer.v.t, v)):
        dst.copy_(torch.from_numpy(src))
    trainer.t = t
    return epoch


def split_halves(n: int, seed: int):
    """Seeded random half split: even positions of a permutation -> half A, odd -> half B."""
    perm = np.random.default_rng(seed).permutation(n)
    return np.sort(perm[0::2]), np.sort(perm[1::2])


def fsc(vol_a, vol_b):
    """Fourier shell correlation of two cubic volumes (Eq. 9): shells of integer radius
    |k| in [s, s+1), s = 0 .. D/2.  Returns the FSC per shell."""
    a, b = (np.asarray(x, dtype=np.float64) for x in (vol_a, vol_b))
    if a.shape != b.shape or a.ndim != 3 or len(set(a.shape)) != 1:
        raise ValueError("fsc needs two cubic volumes of the same shape")
    D = a.shape[0]
    Fa, Fb = np.fft.fftn(a), np.fft.fftn(b)
    k = np.fft.fftfreq(D) * D
    r = np.sqrt(k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2)
    shell = np.floor(r).astype(np.int64)
    ns = D // 2 + 1
    m = shell < ns
    num = np.bincount(shell[m], (Fa * np.conj(Fb)).real[m], ns)
    da = np.bincount(shell[m], (np.abs(Fa) ** 2)[m], ns)
    db = np.bincount(shell[m], (np.abs(Fb) ** 2)[m], ns)
    den = np.sqrt(da * db)
    return np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0)


def resolution(curve, D: int, voxel_size: float, threshold: float = 0.143) -> float:
    """Resolution (Angstrom) where the FSC first drops below ``threshold`` (Fig. 4 caption,
    P:335-347): walking shells s >= 1 from low to high frequency, the crossing between shell s-1
    (>= threshold) and shell s (< threshold) is linearly interpolated to the shell coordinate
    s* = s-1 + (c[s-1] - threshold) / (c[s-1] - c[s]) and reported as D * voxel_size / s*
    (shell s has frequency s / (D voxel_size)).  No crossing -> 2 * voxel_size (Nyquist); a curve
    already below threshold at shell 1 reports D * voxel_size (the box)."""
    c = np.asarray(curve, dtype=np.float64)
    for s in range(1, len(c)):
        if c[s] < threshold:
            if s == 1 and c[0] < threshold:
                return float(D * voxel_size)
            lo = c[s - 1]
            frac = (lo - threshold) / (lo - c[s]) if lo > c[s] else 0.0
            sstar = (s - 1) + min(max(frac, 0.0), 1.0)
            return float(D * voxel_size / max(sstar, 1.0))
    return 2.0 * voxel_size


def gsfsc(vol_a, vol_b, voxel_size: float, threshold: float = 0.143):
    """Gold-standard FSC of two half-map volumes: (curve, resolution at ``threshold``)."""
    c = fsc(vol_a, vol_b)
    return c, resolution(c, np.asarray(vol_a).shape[0], voxel_size, threshold)


def simulate(phantom, data: dict, D: int, pixel_size: float, snr: float, seed: int, batch: int = 64):
    """Observed images of a ground-truth Gaussian set ``phantom`` (gem.SoA) for the poses/CTFs in
    ``data`` (rot, shift, ctf device tensors): the GEM forward through the CTF (wide cull, k = 5)
    plus white noise with per-image variance var(clean) / snr.  Fills data['obs']."""
    import torch
    from . import gem
    n = data["rot"].shape[0]
    dev = data["rot"].device
    gen = gem.GemStep(gem.GemConfig(D=D, pixel_size=pixel_size, n_gauss=phantom.N, max_batch=batch,
                                    cull_k=5.0), dev)
    obs = torch.empty(n, D, D, device=dev)
    zeros = torch.zeros(batch, D, D, device=dev)
    g = torch.Generator(device=dev).manual_seed(seed)
    for s0 in range(0, n, batch):
        sl = slice(s0, min(n, s0 + batch))
        b = sl.stop - sl.start
        gen.forward(phantom, data["rot"][sl], data["shift"][sl], data["ctf"][sl], zeros[:b], pred=obs[sl])
        clean = obs[sl]
        sd = clean.std(dim=(1, 2), keepdim=True) / snr ** 0.5
        obs[sl] = clean + sd * torch.randn(clean.shape, device=dev, generator=g)
    torch.cuda.current_stream(dev).synchronize()
    gen.close()
    data["obs"] = obs
    return data


def train_halves(make_trainer, data: dict, epochs: int, batch: int, seed: int):
    """Gold-standard training: split the particles in two seeded halves
    and train an independent model on each (derived seeds).  ``make_trainer(h)`` returns a fresh
    gem.Trainer for half h in {0, 1}; its initial state should come from a seed derived from h
    too, so the halves share nothing (a shared random init correlates the halves' high
    frequencies and inflates the GSFSC).  Returns (trainer_a, trainer_b, history_a, history_b)."""
    import torch
    n = data["rot"].shape[0]
    out = []
    for h, idx in enumerate(split_halves(n, seed)):
        sel = torch.as_tensor(idx, device=data["rot"].device)
        half = {k: v.index_select(0, sel) for k, v in data.items()}
        tr = make_trainer(h)
        out.append((tr, fit(tr, half, epochs, batch, seed=seed * 2 + 1 + h)))
    return out[0][0], out[1][0], out[0][1], out[1][1]


def roundtrip(n: int = 2000, epochs: int = 30, batch: int = 64, snr: float = 0.5, seed: int = 0,
              ablations=("full", "no_rotation", "isotropic_scale", "both"), lr_scale: float = 1.0,
              device=None):
    """SPEC acceptance 3/4 on config A: simulate ``n`` images of the 200-Gaussian
    ground truth (A_gt) at d = 64, 1.5 A, ``snr``; for each ablation train two independent
    half-set models of 2000 Gaussians from SPEC random_init (one init seed per half) for
    ``epochs``; render both half volumes (gem_render_volume, d^3 at the pixel size) and report
    the GSFSC resolution at 0.143 and FSC(mean of halves, ground truth) at 0.5, in Angstrom."""
    import time
    import torch
    from . import gem, synth
    dev = device or torch.device("cuda", 0)
    w, wg = synth.CONFIGS["A"], synth.CONFIGS["A_gt"]
    px = float(np.float32(w.px))
    gt = gem.SoA.from_arrays(*synth.f32(*synth.phantom(wg, synth.seed_for("A_gt", "phantom", seed))),
                             device=dev)
    rot, shift, ctf = synth.f32(*synth.particles(w, n, seed))
    data = {k: torch.from_numpy(a).to(dev) for k, a in (("rot", rot), ("shift", shift), ("ctf", ctf))}
    simulate(gt, data, w.D, px, snr, seed=1000 + seed)
    vctx = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=1), dev)
    gctx = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=px, n_gauss=wg.N, max_batch=1), dev)
    vol_gt = gctx.render_volume(gt, w.D, px).cpu().numpy()
    out = {}
    for abl in ablations:
        def make(h):
            cfg = gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=batch, ablation=abl,
                                lr_mean=1e-3 * w.ball_radius * lr_scale)
            P0 = synth.f32(*synth.init_model(w, 2 * seed + h))
            return gem.Trainer(cfg, gem.SoA.from_arrays(*P0, device=dev), dev)
        t0 = time.time()
        a, b, ha, hb = train_halves(make, data, epochs, batch, seed)
        torch.cuda.synchronize(dev)
        dt = time.time() - t0
        va = vctx.render_volume(a.params, w.D, px).cpu().numpy()
        vb = vctx.render_volume(b.params, w.D, px).cpu().numpy()
        curve, res = gsfsc(va, vb, px)
        out[abl] = {"gsfsc_A": res, "fsc_gt_0.5_A": resolution(fsc(0.5 * (va + vb), vol_gt), w.D, px, 0.5),
                    "loss_first": [ha[0], hb[0]], "loss_last": [ha[-1], hb[-1]], "train_s": dt,
                    "steps": 2 * epochs * -(-(n // 2) // batch), "gsfsc_curve": [float(x) for x in curve]}
        a.step_ctx.close(); b.step_ctx.close()
    vctx.close(); gctx.close()
    return out


def _np(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(a)
