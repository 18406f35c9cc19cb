"""One small GEM training step (config T, B = 6, 8x8 and 16x16 tiles, fused waves, z-sort, the
per-pixel masks) plus a volume query, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_step.py"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import gem, synth  # noqa: E402

w = synth.CONFIGS["T"]
B = 6
dev = torch.device("cuda", 0)
mr, ls, q = synth.f32(*synth.steady_model(w, 0))
rot, shift, ctf = synth.f32(*synth.particles(w, B, 0))
obs = synth.f32(synth.noise_images(w, B, 0, scale=float(np.abs(mr[:, 3]).mean() * math.sqrt(2 * math.pi) * w.sigma0)))
t = lambda a: torch.from_numpy(a).to(dev)
px = float(np.float32(w.px))
variants = [dict(tile=8), dict(tile=16), dict(tile=8, fused=True, wave=4), dict(tile=8, zsort=True),
            dict(tile=8, pixel_mask="ellipse+tau", tau=1e-3, exact_tiles=True)]
for kw in variants:
    cfg = gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B, **kw)
    tr = gem.Trainer(cfg, gem.SoA.from_arrays(mr, ls, q, dev), dev)
    for _ in range(2):
        tr.train_step(t(rot), t(shift), t(ctf), t(obs))
    torch.cuda.synchronize()
    s = tr.step_ctx.stats()
    v = tr.step_ctx.render_volume(tr.params, 32, px)
    torch.cuda.synchronize()
    print(kw, "ok", s["entries"], float(v.sum()))
print("sanitize step done")
