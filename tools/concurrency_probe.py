"""Would two half-batch pipelines on two streams beat one full batch?  Two libgem contexts (B = 128
each, separate workspaces and parameter copies), forward + backward + Adam per step: sequential on
one stream vs concurrent on two streams; and one B = 256 context for reference."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import gem, synth  # noqa: E402

dev = torch.device("cuda", 0)
w = synth.CONFIGS["R"]
px = float(np.float32(w.px))
mr, ls, q = synth.f32(*synth.steady_model(w, 0))
rot, sh, ctf = (torch.from_numpy(a).to(dev) for a in synth.f32(*synth.particles(w, 256, 5)))
obs = torch.randn(256, w.D, w.D, device=dev)

def trainer(B, stream):
    cfg = gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B, lr_mean=1e-3 * w.ball_radius)
    tr = gem.Trainer(cfg, gem.SoA.from_arrays(mr, ls, q, dev), dev)
    tr.step_ctx.stream = stream
    return tr

def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

s0 = torch.cuda.current_stream(dev)
full = trainer(256, s0)
print("B=256 one context: %.3f ms per 256 particles" % timeit(lambda: full.train_step(rot, sh, ctf, obs)))
sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ta, tb = trainer(128, s0), trainer(128, s0)
def seq():
    ta.train_step(rot[:128], sh[:128], ctf[:128], obs[:128])
    tb.train_step(rot[128:], sh[128:], ctf[128:], obs[128:])
print("2 x B=128 sequential: %.3f ms per 256 particles" % timeit(seq))
ta.step_ctx.stream, tb.step_ctx.stream = sa, sb
def conc():
    ev = torch.cuda.Event()
    ev.record(s0)
    sa.wait_event(ev); sb.wait_event(ev)
    with torch.cuda.stream(sa):
        ta.train_step(rot[:128], sh[:128], ctf[:128], obs[:128])
    with torch.cuda.stream(sb):
        tb.train_step(rot[128:], sh[128:], ctf[128:], obs[128:])
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa); eb.record(sb)
    s0.wait_event(ea); s0.wait_event(eb)
print("2 x B=128 concurrent (two streams): %.3f ms per 256 particles" % timeit(conc))

def stag(split):
    # stream b starts once stream a has finished `split` (its splat..loss, i.e. its forward):
    # b's forward overlaps a's backward
    ev = torch.cuda.Event()
    ev.record(s0)
    sa.wait_event(ev); sb.wait_event(ev)
    ga, gb = ta.step_ctx, tb.step_ctx
    with torch.cuda.stream(sa):
        la = ga.forward(ta.params, rot[:128], sh[:128], ctf[:128], obs[:128])
        mid = torch.cuda.Event(); mid.record(sa)
        ga.backward(ta.params, ta.grad)
        ta.t += 1; ga.step(ta.params, ta.grad, ta.m, ta.v, ta.t)
    with torch.cuda.stream(sb):
        if split:
            sb.wait_event(mid)
        lb = gb.forward(tb.params, rot[128:], sh[128:], ctf[128:], obs[128:])
        gb.backward(tb.params, tb.grad)
        tb.t += 1; gb.step(tb.params, tb.grad, tb.m, tb.v, tb.t)
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa); eb.record(sb)
    s0.wait_event(ea); s0.wait_event(eb)
print("2 x B=128 two streams, raw calls: %.3f ms per 256 particles" % timeit(lambda: stag(False)))
print("2 x B=128 two streams, b's forward after a's: %.3f ms per 256 particles" % timeit(lambda: stag(True)))

def lanes():
    # the library-internal two-lane step this probe models: both halves' forward + backward on two
    # streams, then one Adam (the gradient merge, ~3 us, is left out)
    ev = torch.cuda.Event()
    ev.record(s0)
    sa.wait_event(ev); sb.wait_event(ev)
    ga, gb = ta.step_ctx, tb.step_ctx
    with torch.cuda.stream(sa):
        ga.forward(ta.params, rot[:128], sh[:128], ctf[:128], obs[:128])
        ga.backward(ta.params, ta.grad)
    with torch.cuda.stream(sb):
        gb.forward(tb.params, rot[128:], sh[128:], ctf[128:], obs[128:])
        gb.backward(tb.params, tb.grad)
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa); eb.record(sb)
    s0.wait_event(ea); s0.wait_event(eb)
    ta.t += 1
    ga.stream = s0
    ga.step(ta.params, ta.grad, ta.m, ta.v, ta.t)
    ga.stream = sa
print("two lanes + one Adam: %.3f ms per 256 particles" % timeit(lanes))
print("B=256 one context (again): %.3f ms per 256 particles" % timeit(lambda: full.train_step(rot, sh, ctf, obs)))
