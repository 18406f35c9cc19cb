"""Training loop around the GEM step.

* ``fit``: epochs x ceil(n / batch) Adam steps over seeded, shuffled minibatches (SPEC train,
  S:358-361); every arithmetic step of a training step runs in libgem.so through
  ``gem.Trainer``; the per-epoch mean loss is read once per epoch.
* ``save_checkpoint`` / ``load_checkpoint``: parameters, Adam moments and the Adam step count
  in a small versioned binary format; save -> load -> save is byte-identical and, since the GPU
  step is bitwise deterministic, resuming reproduces the uninterrupted run bit for bit.
* ``split_halves``: the gold-standard half split.
* ``fsc`` / ``resolution``: Fourier shell correlation of two half-map volumes and the 0.143
  criterion (Eq. 9).  An evaluation metric, not part of the training step: computed on
  the host with numpy.
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
    """Resolution (Angstrom) at the first shell s >= 1 where the FSC falls below ``threshold``:
    D * voxel_size / s; returns 2 * voxel_size (Nyquist) if it never does."""
    for s in range(1, len(curve)):
        if curve[s] < threshold:
            return D * voxel_size / s
    return 2.0 * voxel_size


def _np(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(a)
