"""Table 1's memory metric: peak device memory of one GEM
training step vs (N Gaussians, D, batch B).  For each configuration: the libgem workspace
(gem_workspace_bytes: every buffer of the step, cuFFT work area included), the training state
(params, grad, Adam m and v: 4 x 48 N bytes), the batch inputs, and the measured peak of the
torch allocator plus the device-wide used-memory growth (catches cuFFT plan internals) over one
train step.  No buffer of the step scales with D^3.  Writes one JSON document."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import binding as b, gem, synth  # noqa: E402

GRID = [(10_000, 128, 8), (10_000, 128, 128), (50_000, 128, 8), (50_000, 256, 8), (50_000, 256, 128),
        (100_000, 256, 128), (100_000, 512, 8), (500_000, 384, 32)]


def measure(N, D, B, dev):
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    base = torch.cuda.memory_allocated(dev)
    w = synth.Workload("M", N, D, 256 * 1.31 / D, B)
    px = float(np.float32(w.px))
    cfg = gem.GemConfig(D=D, pixel_size=px, n_gauss=N, max_batch=B)
    ws = b.lib().gem_workspace_bytes(ctypes.byref(cfg.c()))
    params = gem.SoA.from_arrays(*synth.f32(*synth.steady_model(w, 0)), device=dev)
    rot, shift, ctf = (torch.from_numpy(a).to(dev) for a in synth.f32(*synth.particles(w, B, 0)))
    obs = torch.randn(B, D, D, device=dev)
    tr = gem.Trainer(cfg, params, dev)
    tr.train_step(rot, shift, ctf, obs)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info(dev)
    peak = torch.cuda.max_memory_allocated(dev) - base
    r = {"N": N, "D": D, "B": B, "workspace_gb": ws / 1e9, "state_gb": 4 * 48 * N / 1e9,
         "inputs_gb": B * (9 + 2 + 8 + D * D) * 4 / 1e9, "torch_peak_gb": peak / 1e9,
         "device_used_gb": (free0 - free1) / 1e9, "d3_volume_gb_if_dense": D ** 3 * 4 / 1e9}
    tr.step_ctx.close()
    del tr, params, rot, shift, ctf, obs
    return r


def main():
    dev = torch.device("cuda", 0)
    rows = [measure(N, D, B, dev) for N, D, B in GRID]
    for r in rows:
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    out = sys.argv[1] if len(sys.argv) > 1 else None
    if out:
        with open(out, "w") as f:
            json.dump({"rows": rows, "note": "peak device memory of one training step (Table 1 metric, "
                       "P:270-279); paper context: GEM 1.54 GB on EMPIAR-10028 on an RTX A6000 (P:279)"}, f, indent=1)


if __name__ == "__main__":
    main()
