"""Data-parallel host logic on CPU (gloo, world_size 2): particle sharding,
the one all-reduce of the [3, N, 4] gradient buffer, and replicated Adam.

The per-rank backward is the oracle here (no GPU); the code under test is
paper_2509_25075_b200.gem.allreduce_grad / shard_indices — the same functions
bench.py and Trainer use with NCCL on GPUs.  The loss is a sum over particles
(reading L14), so the all-reduced shard gradients must equal the full-batch
gradient.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2509_25075_b200 import synth
    w = synth.Workload("Tdp", 96, 16, 2.0, 8)
    mr, ls, q = synth.f32(*synth.steady_model(w, 0))
    rot, shift, ctf = synth.f32(*synth.particles(w, 8, 0))
    obs = synth.f32(synth.noise_images(w, 8, 0, scale=3.0))
    return w, (mr, ls, q), rot, shift, ctf, obs


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2509_25075_b200 import gem
    w, params, rot, shift, ctf, obs = _case()
    idx = gem.shard_indices(8, world, rank, batch=4, step=0, seed=3)
    out = oracle.loss_grad(params, rot[idx], shift[idx], ctf[idx], obs[idx], w.D, float(np.float32(w.px)))
    # gem.Trainer's single payload: the [3, N, 4] gradient, then the rank's total loss, then pad
    N = params[0].shape[0]
    flat = torch.zeros(12 * N + 4, dtype=torch.float32)
    flat[: 12 * N] = torch.from_numpy(oracle.grad_to_soa(out["grad"]).astype(np.float32)).reshape(-1)
    flat[12 * N] = float(out["total"])
    gem.allreduce_flat(flat)
    g = gem.SoA(flat[: 12 * N].view(3, N, 4))
    np.save(os.path.join(outdir, f"loss{rank}.npy"), flat[12 * N:].numpy())
    p = np.stack(params).astype(np.float64)
    p1, _, _ = oracle.adam(p, g.t.numpy().astype(np.float64), np.zeros_like(p), np.zeros_like(p), 1,
                           [1e-3, 5e-3, 1e-3, 5e-2])
    same = gem.replicas_identical([torch.from_numpy(p1.astype(np.float32)), g.t])
    # a perturbed replica must be detected
    p2 = p1.astype(np.float32).copy()
    if rank == 1:
        p2.flat[7] = np.nextafter(p2.flat[7], np.float32(np.inf))
    diff = gem.replicas_identical([torch.from_numpy(p2)])
    np.save(os.path.join(outdir, f"g{rank}.npy"), g.t.numpy())
    np.save(os.path.join(outdir, f"idx{rank}.npy"), idx)
    np.save(os.path.join(outdir, f"h{rank}.npy"), np.array([same, diff]))
    dist.destroy_process_group()


def test_shard_indices_disjoint_and_deterministic():
    from paper_2509_25075_b200 import gem
    a = [gem.shard_indices(100, 4, r, batch=10, step=3, seed=1) for r in range(4)]
    b = [gem.shard_indices(100, 4, r, batch=10, step=3, seed=1) for r in range(4)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    allidx = np.concatenate(a)
    assert len(set(allidx.tolist())) == 40
    for r in range(4):
        assert np.all((a[r] >= 25 * r) & (a[r] < 25 * (r + 1)))


@pytest.mark.timeout(300)
def test_gloo_allreduce_equals_full_batch(tmp_path, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w, params, rot, shift, ctf, obs = _case()
    idx = np.concatenate([np.load(tmp_path / f"idx{r}.npy") for r in range(world)])
    assert len(set(idx.tolist())) == 8
    full = orc.loss_grad(params, rot[idx], shift[idx], ctf[idx], obs[idx], w.D, float(np.float32(w.px)))
    ref = orc.grad_to_soa(full["grad"])
    g0, g1 = np.load(tmp_path / "g0.npy"), np.load(tmp_path / "g1.npy")
    assert np.array_equal(g0, g1)                    # every rank holds identical reduced bytes
    assert np.abs(g0 - ref).max() <= 1e-6 * np.abs(ref).max()
    l0 = np.load(tmp_path / "loss0.npy")
    assert abs(l0[0] - full["total"]) <= 1e-6 * full["total"] and np.all(l0[1:] == 0)   # loss summed alongside
    h0 = np.load(tmp_path / "h0.npy")
    assert h0[0] and not h0[1]                        # replicated Adam stays bit-identical; a 1-ulp drift is caught
