"""Training-loop plumbing: half split, FSC metric, checkpoint format (CPU);
seeded determinism and bit-exact resume of the GPU training loop (GPU)."""
import math
import os

import numpy as np
import pytest

from paper_2509_25075_b200 import synth
from paper_2509_25075_b200 import train as T


def test_split_halves_partition():
    a, b = T.split_halves(101, seed=3)
    assert abs(len(a) - len(b)) <= 1
    assert len(np.intersect1d(a, b)) == 0
    assert np.array_equal(np.union1d(a, b), np.arange(101))
    a2, b2 = T.split_halves(101, seed=3)
    assert np.array_equal(a, a2) and np.array_equal(b, b2)


def test_epoch_batches_cover_each_particle_once():
    bs = T.epoch_batches(37, 8, seed=1, epoch=2)
    assert len(bs) == math.ceil(37 / 8)
    assert np.array_equal(np.sort(np.concatenate(bs)), np.arange(37))
    assert not np.array_equal(np.concatenate(bs), np.concatenate(T.epoch_batches(37, 8, seed=1, epoch=3)))


def test_fsc_identical_independent_and_scaled():
    rng = np.random.default_rng(0)
    v = rng.standard_normal((24, 24, 24))
    assert np.allclose(T.fsc(v, v), 1.0)
    assert np.allclose(T.fsc(v, 3.5 * v), 1.0)          # FSC is scale invariant
    assert np.allclose(T.fsc(v, -v)[1:], -1.0)
    w = rng.standard_normal((24, 24, 24))
    assert np.abs(T.fsc(v, w)[2:]).max() < 0.35         # independent noise: no correlation
    # a shared low-pass signal plus independent noise: FSC high at low shells, low at high shells
    k = np.fft.fftfreq(24) * 24
    r = np.sqrt(k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2)
    sig = np.fft.ifftn(np.fft.fftn(rng.standard_normal((24, 24, 24))) * (r < 4)).real * 30
    c = T.fsc(sig + v, sig + w)
    assert c[1] > 0.9 and c[10] < 0.3
    res = T.resolution(c, 24, 2.0)
    assert 24 * 2.0 / 10 <= res <= 24 * 2.0 / 3


def test_checkpoint_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(1)
    p, m, v = (rng.standard_normal((3, 17, 4)).astype(np.float32) for _ in range(3))
    f1, f2 = str(tmp_path / "a.ckpt"), str(tmp_path / "b.ckpt")
    T.save_checkpoint(f1, p, m, v, adam_t=42, epoch=7)
    p2, m2, v2, t, ep, _ = T.load_checkpoint(f1)
    assert np.array_equal(p, p2) and np.array_equal(m, m2) and np.array_equal(v, v2) and (t, ep) == (42, 7)
    T.save_checkpoint(f2, p2, m2, v2, adam_t=t, epoch=ep)
    assert open(f1, "rb").read() == open(f2, "rb").read()   # save -> load -> save is byte-identical
    raw = bytearray(open(f1, "rb").read())
    raw[0:8] = b"XXXXXXXX"
    open(f2, "wb").write(bytes(raw))
    with pytest.raises(T.CheckpointError):
        T.load_checkpoint(f2)
    open(f2, "wb").write(open(f1, "rb").read()[:-5])
    with pytest.raises(T.CheckpointError):
        T.load_checkpoint(f2)


@pytest.mark.gpu
def test_fit_deterministic_and_resume_bitwise(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_25075_b200 import gem
    w = synth.CONFIGS["T"]
    dev = torch.device("cuda", 0)
    n, B = 24, 8
    rot, shift, ctf = synth.f32(*synth.particles(w, n, 5))
    obs = synth.f32(synth.noise_images(w, n, 5, scale=1.0))
    data = {k: torch.from_numpy(a).to(dev) for k, a in (("rot", rot), ("shift", shift), ("ctf", ctf), ("obs", obs))}
    P0 = synth.f32(*synth.init_model(w, 0))
    px = float(np.float32(w.px))

    def trainer():
        cfg = gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B)
        return gem.Trainer(cfg, gem.SoA.from_arrays(*P0, device=dev), dev)

    a = trainer()
    ha = T.fit(a, data, epochs=3, batch=B, seed=9)
    b = trainer()
    hb = T.fit(b, data, epochs=3, batch=B, seed=9)
    assert ha == hb and np.array_equal(a.params.t.cpu().numpy(), b.params.t.cpu().numpy())
    assert ha[-1] < ha[0]   # the loss goes down on this toy
    ck = str(tmp_path / "r.ckpt")
    c = trainer()
    T.fit(c, data, epochs=1, batch=B, seed=9, checkpoint=ck, checkpoint_every=1)
    d = trainer()
    ep = T.restore(d, ck)
    T.fit(d, data, epochs=3, batch=B, seed=9, start_epoch=ep)
    assert np.array_equal(d.params.t.cpu().numpy(), a.params.t.cpu().numpy())
    assert np.array_equal(d.m.t.cpu().numpy(), a.m.t.cpu().numpy())
