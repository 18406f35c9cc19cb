"""Does a concurrent host->device copy slow the device-resident step?  Steps of config R (random
observations; timing only) alone, then with a background stream copying 67 MB pinned buffers in a
loop; and the copy bandwidth alone vs during the steps."""
import os, sys, threading
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import gem, synth  # noqa: E402

dev = torch.device("cuda", 0)
w = synth.CONFIGS["R"]
B = 256
px = float(np.float32(w.px))
mr, ls, q = synth.f32(*synth.steady_model(w, 0))
tr = gem.Trainer(gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B, lr_mean=1e-3 * w.ball_radius),
                 gem.SoA.from_arrays(mr, ls, q, dev), dev)
rot, sh, ctf = (torch.from_numpy(a).to(dev) for a in synth.f32(*synth.particles(w, B, 5)))
obs = torch.randn(B, w.D, w.D, device=dev)
s = tr.step_ctx.stream
for _ in range(3):
    tr.train_step(rot, sh, ctf, obs)
torch.cuda.synchronize()

def steps(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        tr.train_step(rot, sh, ctf, obs)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

print("step alone: %.3f ms" % steps(20))
src = torch.empty(B * w.D * w.D, dtype=torch.float32, pin_memory=True)
dst = torch.empty(B * w.D * w.D, dtype=torch.float32, device=dev)
cs = torch.cuda.Stream(dev)
with torch.cuda.stream(cs):
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(cs)
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    c1.record(cs)
torch.cuda.synchronize()
print("copy alone: %.3f ms per 67 MB" % (c0.elapsed_time(c1) / 10))
with torch.cuda.stream(cs):
    c0.record(cs)
    for _ in range(30):
        dst.copy_(src, non_blocking=True)
    c1.record(cs)
t = steps(20)
torch.cuda.synchronize()
print("step with a concurrent copy loop: %.3f ms; copy during it: %.3f ms per 67 MB" % (t, c0.elapsed_time(c1) / 30))

# host-mode steps through the C ABI (GEM_MEM_HOST): GPU time and host enqueue time per step
import time
hsrc = [a.cpu().pin_memory() for a in (rot, sh, ctf, obs)]
hloss = torch.empty(B + 1, dtype=torch.float64, pin_memory=True)
for _ in range(3):
    tr.train_step(*hsrc, host=True, loss=hloss)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
t0 = time.perf_counter()
for _ in range(20):
    tr.train_step(*hsrc, host=True, loss=hloss)
t1 = time.perf_counter()
e1.record(s)
torch.cuda.synchronize()
print("host mode: %.3f ms per step on the GPU, %.3f ms per step to enqueue on the host" %
      (e0.elapsed_time(e1) / 20, (t1 - t0) * 1e3 / 20))
t0 = time.perf_counter()
for _ in range(20):
    tr.train_step(rot, sh, ctf, obs)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("device mode: %.3f ms per step to enqueue on the host" % ((t1 - t0) * 1e3 / 20))

# per-phase device time (events on the launching streams) of device-mode vs host-mode steps
g = tr.step_ctx
def phases(host):
    g.profile(True)
    for _ in range(20):
        if host:
            tr.train_step(*hsrc, host=True, loss=hloss)
        else:
            tr.train_step(rot, sh, ctf, obs)
    torch.cuda.synchronize()
    g.profile(False)
    return {k: v[1] / v[0] for k, v in g.profile_read().items()}
dv, hv = phases(False), phases(True)
print("phase            device-mode  host-mode  (ms per launch)")
for k in dv:
    print("%-16s %10.4f %10.4f" % (k, dv[k], hv.get(k, float("nan"))))
