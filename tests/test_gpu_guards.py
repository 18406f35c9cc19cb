"""Out-of-bounds write checks (a substitute for compute-sanitizer memcheck, which is closed on
this pool; profiles/r2/peaks.json): canary bytes after the library's workspace and after every
caller-owned output must be untouched by a training step, a volume query and the list export,
across the launch variants (8x8 / 16x16 tiles, fused waves, z-sort, per-pixel masks, ragged D
and N, B below max_batch)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_25075_b200 import synth  # noqa: E402

CANARY = 12345.678


def _guarded(n, dev, extra=64):
    t = torch.full((n + extra,), CANARY, dtype=torch.float32, device=dev)
    return t, t[:n]


@pytest.mark.parametrize("kw,D,N,B,maxb", [
    (dict(tile=8), 32, 512, 5, 6), (dict(tile=16), 40, 1500, 3, 3), (dict(tile=8, fused=True, wave=2), 36, 700, 5, 5),
    (dict(tile=8, zsort=True), 32, 512, 4, 4), (dict(tile=8, pixel_mask="ellipse+tau", tau=1e-3, exact_tiles=True), 32, 512, 3, 3),
])
def test_no_writes_past_workspace_or_outputs(kw, D, N, B, maxb):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_25075_b200 import gem
    dev = torch.device("cuda", 0)
    w = synth.Workload("G", N, D, 4.0, 64)
    mr, ls, q = synth.f32(*synth.steady_model(w, 0))
    rot, shift, ctf = synth.f32(*synth.particles(w, B, 0))
    obs = synth.f32(synth.noise_images(w, B, 0, scale=float(np.abs(mr[:, 3]).mean() * math.sqrt(2 * math.pi) * w.sigma0)))
    st = gem.GemStep(gem.GemConfig(D=D, pixel_size=4.0, n_gauss=N, max_batch=maxb, **kw), dev, guard_bytes=1 << 16)
    P = gem.SoA.from_arrays(mr, ls, q, dev)
    t = lambda a: torch.from_numpy(a).to(dev)
    pf, proj = _guarded(B * D * D, dev)
    qf, pred = _guarded(B * D * D, dev)
    gfull = torch.full((3 * N * 4 + 64,), CANARY, dtype=torch.float32, device=dev)
    grad = gem.SoA(gfull[: 3 * N * 4].view(3, N, 4))
    lf = torch.full((B + 1 + 16,), CANARY, dtype=torch.float64, device=dev)
    st.forward(P, t(rot), t(shift), t(ctf), t(obs), loss=lf[: B + 1], proj=proj.view(B, D, D), pred=pred.view(B, D, D))
    st.backward(P, grad)
    m, v = gem.SoA.zeros(N, dev), gem.SoA.zeros(N, dev)
    st.step(P, grad, m, v, 1)
    vf, vol = _guarded(D ** 3, dev)
    st.render_volume(P, D, 4.0, out=vol.view(D, D, D))
    st.export_lists(B - 1)
    torch.cuda.synchronize()
    assert st.stats(check=False)["status"] == 0
    assert st.guard_intact()
    for full, n in ((pf, B * D * D), (qf, B * D * D), (gfull, 3 * N * 4), (vf, D ** 3)):
        assert bool((full[n:] == CANARY).all())
    assert bool((lf[B + 1:] == CANARY).all())
    assert torch.isfinite(proj).all() and torch.isfinite(grad.t).all() and torch.isfinite(vol).all()
