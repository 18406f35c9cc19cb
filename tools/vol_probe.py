"""Volume query timing probe: config R model (trained-state proxy: the steady model), Dv = 256."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25075_b200 import gem, synth  # noqa: E402
w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "R"]
dev = torch.device("cuda", 0)
mr, ls, q = synth.f32(*synth.steady_model(w, 0))
st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=float(np.float32(w.px)), n_gauss=w.N, max_batch=8), dev)
P = gem.SoA.from_arrays(mr, ls, q, dev)
out = torch.empty((w.D,) * 3, device=dev)
for _ in range(3):
    st.render_volume(P, w.D, float(np.float32(w.px)), out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st.stream)
for _ in range(10):
    st.render_volume(P, w.D, float(np.float32(w.px)), out=out)
e1.record(st.stream)
torch.cuda.synchronize()
print("ms per call (incl. host sync):", e0.elapsed_time(e1) / 10)
