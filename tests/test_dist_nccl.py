"""Data-parallel step over NCCL on real GPUs: two ranks, one GPU each,
each rendering its own particle shard through libgem; the one all-reduce (gradient + appended
loss, gem.Trainer) must give every rank the single-process full-batch gradient and loss, and
the replicated Adam step must leave the parameters bit-identical (replicas_identical).
Needs >= 2 visible GPUs (skipped otherwise: the round's GPU box has one)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2509_25075_b200 import synth
    w = synth.CONFIGS["T"]
    mr, ls, q = synth.f32(*synth.steady_model(w, 0))
    rot, shift, ctf = synth.f32(*synth.particles(w, 8, 5))
    obs = synth.f32(synth.noise_images(w, 8, 5, scale=2.0))
    return w, (mr, ls, q), rot, shift, ctf, obs


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_2509_25075_b200 import gem
    w, params, rot, shift, ctf, obs = _case()
    idx = gem.shard_indices(8, world, rank, batch=4, step=0, seed=3)
    cfg = gem.GemConfig(D=w.D, pixel_size=float(np.float32(w.px)), n_gauss=w.N, max_batch=4)
    tr = gem.Trainer(cfg, gem.SoA.from_arrays(*params, dev), dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a[idx])).to(dev)
    tr.train_step(t(rot), t(shift), t(ctf), t(obs))
    torch.cuda.synchronize()
    same = gem.replicas_identical([tr.params.t, tr.m.t, tr.v.t])
    np.save(os.path.join(outdir, f"g{rank}.npy"), tr.grad.t.cpu().numpy())
    np.save(os.path.join(outdir, f"l{rank}.npy"), tr.global_loss.cpu().numpy())
    np.save(os.path.join(outdir, f"idx{rank}.npy"), idx)
    np.save(os.path.join(outdir, f"h{rank}.npy"), np.array([same]))
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_nccl_two_ranks_equal_full_batch(tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_2509_25075_b200 import gem
    w, params, rot, shift, ctf, obs = _case()
    idx = np.concatenate([np.load(tmp_path / f"idx{r}.npy") for r in range(world)])
    assert len(set(idx.tolist())) == 8
    dev = torch.device("cuda", 0)
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=float(np.float32(w.px)), n_gauss=w.N, max_batch=8), dev)
    P = gem.SoA.from_arrays(*params, dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a[idx])).to(dev)
    loss = st.forward(P, t(rot), t(shift), t(ctf), t(obs))
    g = gem.SoA.zeros(w.N, dev)
    st.backward(P, g)
    ref = g.t.cpu().numpy().astype(np.float64)
    g0, g1 = np.load(tmp_path / "g0.npy"), np.load(tmp_path / "g1.npy")
    assert np.array_equal(g0, g1)                               # identical reduced bytes on every rank
    for arr in range(3):                                        # per SoA array (mu|rho, s, q)
        assert np.abs(g0[arr] - ref[arr]).max() <= 1e-5 * np.abs(ref[arr]).max()
    l0 = float(np.load(tmp_path / "l0.npy")[0])
    assert abs(l0 - float(loss[-1])) <= 1e-5 * float(loss[-1])   # loss summed alongside the gradient
    assert np.load(tmp_path / "h0.npy")[0] and np.load(tmp_path / "h1.npy")[0]
