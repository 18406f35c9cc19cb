"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same
seeded fp32 inputs.  Bars (BASELINE.json north star; DESIGN.md §3 L19/L22):
  * cull lists and AABBs bit-exact (ties: oracle bound within 1e-9 px of an integer);
  * images / predictions / volume: per-image max-norm relative error <= 1e-5;
  * loss: relative error <= 1e-5;
  * gradients: per-class (mu, rho, s, q) max-norm relative error <= 1e-4;
  * Adam given an identical gradient input: <= 1e-6.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_25075_b200 import synth  # noqa: E402

CLASSES = {"mu": [0, 1, 2], "rho": [3], "s": [4, 5, 6], "q": [8, 9, 10, 11]}
IMG_TOL, GRAD_TOL, LOSS_TOL = 1e-5, 1e-4, 1e-5


@pytest.fixture(scope="module")
def gem():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_25075_b200 import gem as g
    return g


def make_case(wname="T", B=4, seed=0, N=None, D=None, state="steady", morton=True):
    w = synth.CONFIGS[wname]
    if N is not None or D is not None:
        w = synth.Workload(w.name + "x", N or w.N, D or w.D, w.px, w.particles)
    model = synth.steady_model if state == "steady" else synth.init_model
    mr, ls, q = model(w, seed, morton)
    rot, shift, ctf = synth.particles(w, B, seed)
    mr, ls, q, rot, shift, ctf = synth.f32(mr, ls, q, rot, shift, ctf)
    # observed images: noise at the scale of a typical pixel (the residual is O(signal))
    amp_scale = float(np.mean(np.abs(mr[:, 3])) * math.sqrt(2 * math.pi) * w.sigma0)
    obs = synth.f32(synth.noise_images(w, B, seed, scale=amp_scale))
    return dict(w=w, params=(mr, ls, q), rot=rot, shift=shift, ctf=ctf, obs=obs, px=float(np.float32(w.px)))


def run_gpu(gem, case, tile=8, want_lists=False, cap=0, host=False, fused=False, wave=0, zsort=False,
            want_pred=True):
    w = case["w"]
    B = case["rot"].shape[0]
    cfg = gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=B, tile=tile, list_capacity=cap,
                        fused=fused, wave=wave, zsort=zsort)
    st = gem.GemStep(cfg)
    dev = st.device
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    if host:
        mk = lambda a: torch.from_numpy(a).pin_memory()
    else:
        mk = lambda a: torch.from_numpy(a).to(dev)
    rot, shift, ctf, obs = (mk(case[k]) for k in ("rot", "shift", "ctf", "obs"))
    proj = torch.empty(B, w.D, w.D, device=dev)
    pred = torch.empty(B, w.D, w.D, device=dev) if want_pred else None
    loss = st.forward(P, rot, shift, ctf, obs, proj=proj, pred=pred, host=host)
    grad = gem.SoA.zeros(w.N, dev)
    st.backward(P, grad)
    torch.cuda.synchronize()
    out = dict(st=st, P=P, loss=loss.cpu().numpy().copy(), proj=proj.cpu().numpy(),
               pred=pred.cpu().numpy() if want_pred else None,
               grad=grad.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy(), grad_soa=grad)
    if want_lists:
        first = 0 if not fused else B - ((B - 1) % wave + 1)   # only the last wave is resident when fused
        out["lists"] = [st.export_lists(i) for i in range(first, B)]
        out["lists_first"] = first
    out["stats"] = st.stats(check=False)
    return out


def oracle_out(orc, case, want=("proj", "pred")):
    w = case["w"]
    return orc.loss_grad(case["params"], case["rot"], case["shift"], case["ctf"], case["obs"], w.D, case["px"],
                         want=want)


def maxnorm_rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def assert_lists_exact(orc, case, lists, tile, first=0, tau=0.0):
    w = case["w"]
    aabb, vis, sp = orc.splats(case["params"], case["rot"], case["shift"], w.D, case["px"], tau=tau)
    tile_off, base, ids = orc.lists(aabb, vis, w.D, tile)
    ties = 0
    for ii, (g_off, g_ids, g_box) in enumerate(lists):
        i = first + ii
        g_vis = (g_box[:, 0] <= g_box[:, 1]) & (g_box[:, 2] <= g_box[:, 3])
        bad = np.nonzero((g_vis != vis[i].astype(bool)) |
                         (vis[i].astype(bool) & np.any(g_box != aabb[i], axis=1)))[0]
        for j in bad:  # reading L22: allowed only if the oracle bound is within 1e-9 px of an integer
            mx, my, A, C = sp[i, j, 0], sp[i, j, 1], sp[i, j, 8], sp[i, j, 9]
            rx, ry = 3.0 * math.sqrt(A), 3.0 * math.sqrt(C)
            bounds = [(mx - rx) / case["px"] + w.D // 2, (mx + rx) / case["px"] + w.D // 2,
                      (my - ry) / case["px"] + w.D // 2, (my + ry) / case["px"] + w.D // 2]
            assert min(abs(b - round(b)) for b in bounds) < 1e-9, (i, j, g_box[j], aabb[i, j])
            ties += 1
        if ties == 0:
            o_ids = ids[base[i]: base[i] + tile_off[i, -1]]
            assert np.array_equal(g_off, tile_off[i]), i
            # O4: every tile's list in ascending Gaussian id, element by element
            assert np.array_equal(g_ids, o_ids), i
    return ties


# --------------------------------------------------------------------------- tests
@pytest.mark.parametrize("tile,fused", [(16, False), (8, False), (16, True), (8, True)])
def test_T_lists_images_loss_grads(gem, orc, tile, fused):
    case = make_case("T", B=6, seed=1)
    g = run_gpu(gem, case, tile=tile, want_lists=True, fused=fused, wave=4 if fused else 0)   # waves of 4 + 2
    assert g["stats"]["status"] == 0, g["stats"]
    assert_lists_exact(orc, case, g["lists"], tile, g["lists_first"])
    o = oracle_out(orc, case)
    for i in range(case["rot"].shape[0]):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
        assert maxnorm_rel(g["pred"][i], o["pred"][i]) < IMG_TOL
    assert np.all(np.abs(g["loss"][:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    assert abs(g["loss"][-1] - o["total"]) < LOSS_TOL * o["total"]
    for name, cols in CLASSES.items():
        err = maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols])
        assert err < GRAD_TOL, (name, err)
    assert np.all(g["grad"][:, 7] == 0.0)


@pytest.mark.parametrize("tile,D", [(16, 40), (8, 40), (8, 36)])
def test_ragged_shapes_and_culled_rows(gem, orc, tile, D):
    """D not a multiple of the tile (partial edge tiles, a 5 x 5 tile grid), N not a multiple of
    the 4096-Gaussian chunk, B=3; Gaussians pushed off-frame get exactly-zero gradient rows."""
    case = make_case("T", B=3, seed=2, N=1500, D=D)
    mr = case["params"][0].copy()
    mr[5, :3] = [1e4, 1e4, 0]
    mr[1400, :3] = [-5e3, 2e3, 1e3]
    mr[77, 3] = 0.0   # rho = 0 -> |amp| = 0 <= tau: culled
    case["params"] = (mr, case["params"][1], case["params"][2])
    g = run_gpu(gem, case, tile=tile, want_lists=True)
    assert_lists_exact(orc, case, g["lists"], tile)
    o = oracle_out(orc, case)
    for i in range(3):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name
    for j in (5, 1400, 77):
        assert np.all(g["grad"][j] == 0.0)


def test_init_state_and_unsorted_ids(gem, orc):
    """SPEC random_init model state (3.6x more pairs) with Gaussian ids in random order."""
    case = make_case("T", B=4, seed=3, state="init", morton=False)
    g = run_gpu(gem, case, want_lists=True)
    assert_lists_exact(orc, case, g["lists"], 8)
    o = oracle_out(orc, case)
    for i in range(4):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
    for name, cols in CLASSES.items():
        if name == "q":
            continue
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name
    # init-state Gaussians are isotropic, so dL/dq is identically zero (rotation does
    # not change Sigma): the GPU's q-gradient must be fp32 noise next to the s-gradient.
    assert np.abs(o["grad"][:, 8:12]).max() < 1e-12 * np.abs(o["grad"][:, 4:7]).max()
    assert np.abs(g["grad"][:, 8:12]).max() < GRAD_TOL * np.abs(o["grad"][:, 4:7]).max()


def test_S_config_two_particles(gem, orc):
    case = make_case("S", B=2, seed=4)
    g = run_gpu(gem, case, want_lists=True, fused=True, wave=1)
    assert_lists_exact(orc, case, g["lists"], 8, g["lists_first"])
    o = oracle_out(orc, case)
    for i in range(2):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
        assert maxnorm_rel(g["pred"][i], o["pred"][i]) < IMG_TOL
    assert np.all(np.abs(g["loss"][:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name


def test_step_bitwise_deterministic_and_linear_in_rho(gem):
    case = make_case("T", B=4, seed=5)
    a = run_gpu(gem, case)
    b = run_gpu(gem, case)
    assert np.array_equal(a["proj"], b["proj"])
    assert np.array_equal(a["loss"], b["loss"])
    assert np.array_equal(a["grad"], b["grad"])
    mr = case["params"][0].copy()
    mr[:, 3] *= 2.0
    c = run_gpu(gem, dict(case, params=(mr, case["params"][1], case["params"][2])))
    assert np.array_equal(c["proj"], 2.0 * a["proj"])


def test_host_memory_batch_matches_device(gem):
    case = make_case("T", B=4, seed=6)
    a = run_gpu(gem, case)
    h = run_gpu(gem, case, host=True)
    assert np.array_equal(a["proj"], h["proj"]) and np.array_equal(a["loss"], h["loss"])
    # the backward writes one slot per (particle, Gaussian) and reduces them in a fixed order:
    # no atomics, so the gradient is bitwise reproducible too
    assert np.array_equal(a["grad"], h["grad"])
    # fused waves of 2 (and a ragged last wave of 1): each wave's images copied and awaited apart
    case5 = make_case("T", B=5, seed=6)
    af = run_gpu(gem, case5, fused=True, wave=2)
    hf = run_gpu(gem, case5, fused=True, wave=2, host=True)
    assert np.array_equal(af["proj"], hf["proj"]) and np.array_equal(af["loss"], hf["loss"])
    assert np.array_equal(af["grad"], hf["grad"])


def test_host_memory_back_to_back_steps(gem):
    """GEM_MEM_HOST steps enqueued back to back with no host synchronisation: call k + 1's inputs
    are copied into the other half of the double-buffered staging while call k runs.  Each
    step's loss and gradient (into its own gradient buffer) are bitwise those of the same batch
    run alone from device memory, so no copy overwrote staging still in use (the rotations the
    backward reads, the images the side stream transforms)."""
    case = make_case("T", B=4, seed=6)
    w = case["w"]
    dev = torch.device("cuda", 0)
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=4))
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    rng = np.random.default_rng(3)
    batches = []
    for k, nb in enumerate((4, 3, 4, 2, 4)):   # varying batch sizes share the staging halves
        perm = rng.permutation(4)[:nb]
        batches.append([np.ascontiguousarray(case[n][perm]) for n in ("rot", "shift", "ctf", "obs")])
    hosts = [[torch.from_numpy(a).pin_memory() for a in bt] for bt in batches]
    losses = [torch.empty(bt[0].shape[0] + 1, dtype=torch.float64, pin_memory=True) for bt in batches]
    grads = [gem.SoA.zeros(w.N, dev) for _ in batches]
    for k, bt in enumerate(hosts):
        st.forward(P, *bt, loss=losses[k], host=True)
        st.backward(P, grads[k])
    torch.cuda.synchronize()
    for k, bt in enumerate(batches):
        ref_loss = st.forward(P, *(torch.from_numpy(a).to(dev) for a in bt))
        ref = gem.SoA.zeros(w.N, dev)
        st.backward(P, ref)
        torch.cuda.synchronize()
        assert np.array_equal(losses[k].numpy(), ref_loss.cpu().numpy()), k
        assert torch.equal(grads[k].t, ref.t), k


def test_adam_step_identical_gradient_input(gem, orc):
    case = make_case("T", B=2, seed=7)
    g = run_gpu(gem, case)
    st, P, grad = g["st"], g["P"], g["grad_soa"]
    dev = P.t.device
    p0 = P.t.cpu().numpy().astype(np.float64)
    m = gem.SoA.zeros(P.N, dev); v = gem.SoA.zeros(P.N, dev)
    cfg = st.cfg
    lr = np.array([cfg.lr_mean, cfg.lr_log_scale, cfg.lr_quat, cfg.lr_density], np.float32).astype(np.float64)
    gnp = grad.t.cpu().numpy().astype(np.float64)
    mo = np.zeros_like(p0); vo = np.zeros_like(p0); po = p0
    for t in (1, 2, 3):
        st.step(P, grad, m, v, t)
        po, mo, vo = orc.adam(po, gnp, mo, vo, t, lr, cfg.beta1, float(np.float32(cfg.beta2)), float(np.float32(cfg.eps)))
    torch.cuda.synchronize()
    pg = P.t.cpu().numpy().astype(np.float64)
    assert np.abs(pg - po).max() <= 1e-6 * np.abs(po).max()
    assert np.array_equal(pg[1, :, 3], p0[1, :, 3])                        # pad lane untouched
    assert np.abs(np.linalg.norm(pg[2], axis=1) - 1).max() < 1e-6


def test_render_volume(gem, orc):
    case = make_case("T", B=1, seed=8)
    g = run_gpu(gem, case)
    w = case["w"]
    Dv, vs = 32, float(np.float32(w.px))
    vol = g["st"].render_volume(g["P"], Dv, vs).cpu().numpy()
    ref = orc.volume(case["params"], Dv, vs, masked=True)
    assert maxnorm_rel(vol, ref) < IMG_TOL
    # Dv not a multiple of the 8^3 brick
    vol2 = g["st"].render_volume(g["P"], 27, vs).cpu().numpy()
    ref2 = orc.volume(case["params"], 27, vs, masked=True)
    assert maxnorm_rel(vol2, ref2) < IMG_TOL


@pytest.mark.parametrize("stretch", [False, True])
def test_render_volume_bricks(gem, orc, stretch):
    """Volume query over many 8^3 bricks (Dv = 48 and a ragged 45): boxes spanning several
    bricks, the z-column recurrence and, with needle-like Gaussians (one axis x e^1.5, one
    x e^-1), its direct-evaluation path."""
    case = make_case("T", B=1, seed=31, N=1500, D=48)
    mr, ls, q = case["params"]
    if stretch:
        ls = ls.copy()
        ls[:, 0] += 1.5
        ls[:, 1] -= 1.0
    w = case["w"]
    vs = float(np.float32(w.px))
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=vs, n_gauss=w.N, max_batch=1))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    for Dv in (48, 45):
        vol = st.render_volume(P, Dv, vs).cpu().numpy()
        ref = orc.volume((mr, ls, q), Dv, vs, masked=True)
        assert maxnorm_rel(vol, ref) < IMG_TOL, Dv


def test_render_volume_full_grid(gem, orc):
    """Row a11 at the bench's grid: Dv = D = 256 of config R (32^3 bricks, the headline model's
    Gaussian sizes), on a seeded 1200-Gaussian subset of the steady model so the fp64 oracle
    finishes in seconds; the whole 256^3 volume is compared."""
    w = synth.CONFIGS["R"]
    mr, ls, q = synth.f32(*synth.steady_model(w, 0))
    sel = np.sort(np.random.default_rng(5).choice(w.N, 1200, replace=False))
    mr, ls, q = mr[sel], ls[sel], q[sel]
    vs = float(np.float32(w.px))
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=vs, n_gauss=len(sel), max_batch=1))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    vol = st.render_volume(P, w.D, vs).cpu().numpy()
    ref = orc.volume((mr, ls, q), w.D, vs, masked=True)
    assert maxnorm_rel(vol, ref) < IMG_TOL


def test_render_volume_wide_gaussians(gem, orc):
    """Gaussians whose voxel boxes span up to 5^3 bricks: the count pass takes a slot for the
    first 8 bricks of each, the rest go through the second counter and the fill's atomic cursor
    (volume.cu k_vol_prep / k_vol_fill); against the oracle, and bitwise reproducible."""
    case = make_case("T", B=1, seed=73, N=60, D=32)
    mr, ls, q = case["params"]
    ls = ls.copy()
    ls[:, :3] = np.log(np.float32(6.0)) + 0.2 * np.random.default_rng(2).standard_normal((60, 3)).astype(np.float32)
    vs = 2.0   # sigma ~ 3 voxels: boxes ~ 18 voxels, 3-4 bricks per axis
    st = gem.GemStep(gem.GemConfig(D=32, pixel_size=vs, n_gauss=60, max_batch=1))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    a = st.render_volume(P, 64, vs).cpu().numpy()
    b = st.render_volume(P, 64, vs).cpu().numpy()
    assert np.array_equal(a, b)
    ref = orc.volume((mr, ls, q), 64, vs, masked=True)
    assert maxnorm_rel(a, ref) < IMG_TOL


def test_render_volume_large_grid(gem, orc):
    """Dv = 416 (> 2^17 bricks): the general multi-block scan, every brick's slot taken by the
    fill's atomic (no pre-taken slots), against the oracle."""
    case = make_case("T", B=1, seed=71, N=80, D=32)
    mr, ls, q = case["params"]
    mr = mr.copy()
    mr[:, :3] *= 6.0   # spread over the large grid
    vs = 2.0
    st = gem.GemStep(gem.GemConfig(D=32, pixel_size=vs, n_gauss=80, max_batch=1))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    vol = st.render_volume(P, 416, vs).cpu().numpy()
    ref = orc.volume((mr, ls, q), 416, vs, masked=True)
    assert np.abs(ref).max() > 0
    assert maxnorm_rel(vol, ref) < IMG_TOL


def test_empty_lists_all_offframe(gem):
    case = make_case("T", B=2, seed=9)
    mr = case["params"][0].copy()
    mr[:, :3] += 1e5
    g = run_gpu(gem, dict(case, params=(mr, case["params"][1], case["params"][2])), want_lists=True)
    assert np.all(g["proj"] == 0.0) and np.all(g["grad"] == 0.0)
    assert all(l[0][-1] == 0 for l in g["lists"])
    assert np.allclose(g["loss"][:-1], (case["obs"].astype(np.float64) ** 2).sum((1, 2)), rtol=1e-5)


def test_errors_and_capacity(gem):
    from paper_2509_25075_b200 import binding as b
    case = make_case("T", B=2, seed=10)
    w = case["w"]
    with pytest.raises(b.GemError) as e:
        gem.GemStep(gem.GemConfig(D=31, pixel_size=1.0, n_gauss=10, max_batch=1))
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=1, list_capacity=10))
    dev = st.device
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    grad = gem.SoA.zeros(w.N, dev)
    with pytest.raises(b.GemError) as e:
        st.backward(P, grad)
    assert e.value.status == b.GEM_E_STATE
    t = lambda a: torch.from_numpy(a).to(dev)
    with pytest.raises(b.GemError) as e:
        st.forward(P, t(case["rot"]), t(case["shift"]), t(case["ctf"]), t(case["obs"]))
    assert e.value.status == b.GEM_E_SHAPE
    st.forward(P, t(case["rot"][:1]), t(case["shift"][:1]), t(case["ctf"][:1]), t(case["obs"][:1]))
    s = st.stats(check=False)
    assert s["status"] == b.GEM_E_CAPACITY and s["overflow"] == 1 and s["entries"] > 10
    # the overflow flag is sticky across forwards until gem_stats reads it: an overflowing
    # forward followed by one that fits (all Gaussians off-frame) still reports it once
    st.forward(P, t(case["rot"][:1]), t(case["shift"][:1]), t(case["ctf"][:1]), t(case["obs"][:1]))
    mr_off = case["params"][0].copy()
    mr_off[:, :3] += 1e5
    P_off = gem.SoA.from_arrays(mr_off, case["params"][1], case["params"][2], device=dev)
    st.forward(P_off, t(case["rot"][:1]), t(case["shift"][:1]), t(case["ctf"][:1]), t(case["obs"][:1]))
    s = st.stats(check=False)
    assert s["entries"] == 0 and s["overflow"] == 1 and s["status"] == b.GEM_E_CAPACITY
    s = st.stats(check=False)
    assert s["overflow"] == 0 and s["status"] == b.GEM_OK


def test_workspace_has_no_cubic_term(gem):
    """S:193 / S:639: workspace grows with B*N and B*D^2, never D^3."""
    from paper_2509_25075_b200 import binding as b
    import ctypes
    L = b.lib()
    def ws(D, N=10000, B=8):
        c = gem.GemConfig(D=D, pixel_size=1.0, n_gauss=N, max_batch=B).c()
        return L.gem_workspace_bytes(ctypes.byref(c))
    r = ws(256) / ws(128)
    assert r < 4.6, r    # quadratic at most (plus lists); D^3 would give 8
    # SPEC acceptance 6: at M = 50 000 and d = 128 -> 256 the step's whole device footprint
    # (workspace + params/grad/m/v + batch inputs) grows by <= 1.3x; a dense d^3 path grows 8x
    def total(D, N=50000, B=8):
        return ws(D, N, B) + 4 * 48 * N + B * (19 + D * D) * 4
    r2 = total(256) / total(128)
    assert r2 <= 1.3, r2


def test_host_pipeline_matches_device_steps(gem):
    """gem.HostPipeline (pinned host batches, double-buffered side-stream copies) must give the
    same parameters, bit for bit, as the same training steps on device-resident inputs."""
    case = make_case("T", B=3, seed=11)
    w = case["w"]
    B = 3
    dev = torch.device("cuda", 0)
    cfg = gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=B)
    batches_np = []
    for k in range(4):
        rot, shift, ctf = synth.f32(*synth.particles(w, B, 100 + k))
        obs = case["obs"] * np.float32(1.0 + 0.1 * k)
        batches_np.append((rot, shift, ctf, obs))
    P0 = gem.SoA.from_arrays(*case["params"], device=dev)
    tr_a = gem.Trainer(cfg, gem.SoA(P0.t.clone()), dev)
    for b in batches_np:
        tr_a.train_step(*(torch.from_numpy(x).to(dev) for x in b))
    tr_b = gem.Trainer(cfg, gem.SoA(P0.t.clone()), dev)
    pipe = gem.HostPipeline(tr_b, B, w.D)
    lh = pipe.run([[torch.from_numpy(x).pin_memory() for x in b] for b in batches_np])
    torch.cuda.synchronize()
    assert np.array_equal(tr_a.params.t.cpu().numpy(), tr_b.params.t.cpu().numpy())
    assert np.isfinite(lh.numpy()).all() and lh[-1] > 0


@pytest.mark.parametrize("D", [64, 48])
def test_forward_without_outputs(gem, orc, D):
    """The training/bench path: no projection or prediction requested, so the render writes the
    workspace's projection buffer, which the column kernel then reuses for the packed gradient
    rows (row path, D = 64) or the C2R output (2D path, D = 48).  Loss and gradients equal those
    of the run that returns the images (bitwise on the row path; the 2D cuFFT plans may pick
    another kernel for another input alignment, so there to rounding) and the oracle's."""
    case = make_case("T", B=3, seed=33, N=900, D=D)
    w = case["w"]
    st = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=3, list_capacity=1 << 18))
    dev = st.device
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    t = lambda a: torch.from_numpy(a).to(dev)
    args = [t(case[k]) for k in ("rot", "shift", "ctf", "obs")]
    loss_a = st.forward(P, *args).cpu().numpy().copy()
    grad_a = gem.SoA.zeros(w.N, dev)
    st.backward(P, grad_a)
    proj = torch.empty(3, w.D, w.D, device=dev)
    pred = torch.empty(3, w.D, w.D, device=dev)
    loss_b = st.forward(P, *args, proj=proj, pred=pred).cpu().numpy().copy()
    grad_b = gem.SoA.zeros(w.N, dev)
    st.backward(P, grad_b)
    torch.cuda.synchronize()
    assert st.stats(check=False)["status"] == 0
    if D == 64:
        assert np.array_equal(loss_a, loss_b)
        assert torch.equal(grad_a.t, grad_b.t)
    else:
        assert np.allclose(loss_a, loss_b, rtol=1e-6, atol=0)
        gb = grad_b.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
        g_a = grad_a.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
        for name, cols in CLASSES.items():
            assert maxnorm_rel(g_a[:, cols], gb[:, cols]) < 1e-5, name
    o = oracle_out(orc, case, want=())
    assert np.all(np.abs(loss_a[:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    ga = grad_a.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
    for name, cols in CLASSES.items():
        assert maxnorm_rel(ga[:, cols], o["grad"][:, cols]) < GRAD_TOL, name


@pytest.mark.parametrize("want_pred", [True, False])
def test_R_config_full_size(gem, orc, want_pred):
    """BASELINE config R at full size (N = 50,000, D = 256, px = 1.31 A) in the bench's launch
    configuration (default 8x8 tiles, non-fused), one particle: bit-exact lists and the whole
    projection, prediction, loss and every gradient class against the un-culled fp64 oracle
    (~3e9 Gaussian-pixel terms per pass on the host cores); with and without predicted images
    (the bench's call has none)."""
    case = make_case("R", B=1, seed=12)
    g = run_gpu(gem, case, tile=8, want_lists=True, want_pred=want_pred)
    assert g["stats"]["status"] == 0, g["stats"]
    assert_lists_exact(orc, case, g["lists"], 8)
    o = oracle_out(orc, case)
    assert maxnorm_rel(g["proj"][0], o["proj"][0]) < IMG_TOL
    if want_pred:
        assert maxnorm_rel(g["pred"][0], o["pred"][0]) < IMG_TOL
    assert abs(g["loss"][-1] - o["total"]) < LOSS_TOL * o["total"]
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name


def test_R_config_bench_batch_sampled(gem, orc):
    """The bench's exact launch configuration (config R, B = 256 particles per step, 8x8 tiles):
    lists, projection and per-particle loss of three sampled particles against the oracle, and a
    property for the summed gradient that holds at any size: the batch gradient equals the sum
    of the gradients of its four 64-particle quarters."""
    B = 256
    case = make_case("R", B=B, seed=13)
    g = run_gpu(gem, case, tile=8, want_pred=False)
    assert g["stats"]["status"] == 0, g["stats"]
    st = g["st"]
    for i in (0, 127, 255):
        sub = dict(case, rot=case["rot"][i:i + 1], shift=case["shift"][i:i + 1], ctf=case["ctf"][i:i + 1],
                   obs=case["obs"][i:i + 1])
        assert_lists_exact(orc, sub, [st.export_lists(i)], 8)
        o = oracle_out(orc, sub, want=("proj",))
        assert maxnorm_rel(g["proj"][i], o["proj"][0]) < IMG_TOL
        assert abs(g["loss"][i] - o["total"]) < LOSS_TOL * o["total"]
    parts = []
    for q in range(4):
        sl = slice(64 * q, 64 * q + 64)
        sub = dict(case, rot=case["rot"][sl], shift=case["shift"][sl], ctf=case["ctf"][sl], obs=case["obs"][sl])
        parts.append(run_gpu(gem, sub, tile=8, want_pred=False)["grad"].astype(np.float64))
    tot = sum(parts)
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], tot[:, cols]) < 1e-5, name


@pytest.mark.parametrize("ablation", ["no_rotation", "isotropic_scale", "both"])
def test_ablation_flags(gem, orc, ablation):
    """Table 5 ablations: no_rotation keeps q = (1,0,0,0) with an exactly zero
    quaternion gradient; isotropic_scale leaves the three log-scales of every Gaussian equal after
    every step.  The other gradient classes are the unablated ones (oracle)."""
    case = make_case("T", B=3, seed=14)
    w = case["w"]
    dev = torch.device("cuda", 0)
    mr, ls, q = (a.copy() for a in case["params"])
    if ablation in ("no_rotation", "both"):
        q[:] = [1.0, 0.0, 0.0, 0.0]
    if ablation in ("isotropic_scale", "both"):
        ls[:, :3] = ls[:, :3].mean(axis=1, keepdims=True)
    case = dict(case, params=(mr, ls, q))
    cfg = gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=3, ablation=ablation)
    tr = gem.Trainer(cfg, gem.SoA.from_arrays(mr, ls, q, dev), dev)
    t = lambda a: torch.from_numpy(a).to(dev)
    tr.step_ctx.forward(tr.params, t(case["rot"]), t(case["shift"]), t(case["ctf"]), t(case["obs"]))
    tr.step_ctx.backward(tr.params, tr.grad)
    g = tr.grad.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
    o = oracle_out(orc, case, want=())
    for name, cols in CLASSES.items():
        if name == "q" and ablation in ("no_rotation", "both"):
            assert np.all(g[:, 8:12] == 0.0)
        elif name == "q":   # isotropic Gaussians: dL/dq is identically zero, fp32 noise on the GPU
            assert np.abs(g[:, 8:12]).max() < GRAD_TOL * np.abs(o["grad"][:, 4:7]).max()
        else:
            assert maxnorm_rel(g[:, cols], o["grad"][:, cols]) < GRAD_TOL, name
    for k in range(3):
        tr.train_step(t(case["rot"]), t(case["shift"]), t(case["ctf"]), t(case["obs"]))
        p = tr.params.t.cpu().numpy()
        if ablation in ("no_rotation", "both"):
            assert np.all(p[2] == np.array([1, 0, 0, 0], np.float32))
        if ablation in ("isotropic_scale", "both"):
            assert np.all(p[1][:, 0] == p[1][:, 1]) and np.all(p[1][:, 1] == p[1][:, 2])
        assert np.isfinite(p).all()


def assert_zsorted_lists_exact(orc, case, lists, tile):
    """f1: with GEM_FLAG_ZSORT every exported tile list equals the oracle's O4z list
    element by element -- the (depth, id) order is a bit-exact function of the inputs."""
    w = case["w"]
    aabb, vis, sp = orc.splats(case["params"], case["rot"], case["shift"], w.D, case["px"])
    tile_off, base, ids = orc.lists(aabb, vis, w.D, tile)
    zs = orc.zsort_lists(tile_off, base, ids, sp)
    n = 0
    for i, (g_off, g_ids, _) in enumerate(lists):
        assert np.array_equal(g_off, tile_off[i]), i
        assert np.array_equal(g_ids, zs[base[i]: base[i] + tile_off[i, -1]]), i
        n += len(g_ids)
    return n


@pytest.mark.parametrize("wname,B,tile", [("T", 4, 8), ("T", 3, 16), ("S", 2, 8)])
def test_zsort_lists_exact_and_parity(gem, orc, wname, B, tile):
    case = make_case(wname, B=B, seed=21)
    g = run_gpu(gem, case, tile=tile, want_lists=True, zsort=True)
    assert assert_zsorted_lists_exact(orc, case, g["lists"], tile) > 0
    o = oracle_out(orc, case)
    for i in range(B):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL, i
    assert np.all(np.abs(g["loss"][:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name
    # deterministic: a second run gives the same lists and bytes
    g2 = run_gpu(gem, case, tile=tile, want_lists=True, zsort=True)
    assert np.array_equal(g["proj"], g2["proj"]) and np.array_equal(g["grad"], g2["grad"])
    assert all(np.array_equal(a[1], b[1]) for a, b in zip(g["lists"], g2["lists"]))


def test_zsort_long_segments_merge_path(gem, orc):
    """Tile lists longer than the 4096-entry shared-memory sort take the run + merge path."""
    rng = np.random.default_rng(3)
    N, D, B = 9000, 32, 2
    w = synth.Workload("Z", N, D, 1.0, B)
    mu = np.concatenate([rng.uniform(-2.0, 2.0, (N, 2)), rng.uniform(-20.0, 20.0, (N, 1))], 1)
    mr = np.concatenate([mu, rng.uniform(0.5, 1.5, (N, 1))], 1)
    ls = np.concatenate([np.log(rng.uniform(1.5, 2.5, (N, 3))), np.zeros((N, 1))], 1)
    q = rng.standard_normal((N, 4)); q /= np.linalg.norm(q, axis=1, keepdims=True)
    rot, shift, ctf = synth.particles(w, B, 4)
    mr, ls, q, rot, shift, ctf = synth.f32(mr, ls, q, rot, np.zeros((B, 2)), ctf)
    case = dict(w=w, params=(mr, ls, q), rot=rot, shift=shift, ctf=ctf,
                obs=synth.f32(synth.noise_images(w, B, 4, scale=5.0)), px=1.0)
    g = run_gpu(gem, case, tile=8, want_lists=True, zsort=True)
    lens = [np.diff(off).max() for off, _, _ in g["lists"]]
    assert max(lens) > 4096, lens
    assert assert_zsorted_lists_exact(orc, case, g["lists"], 8) > 0
    o = oracle_out(orc, case, want=("proj",))
    for i in range(B):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL, i


PIXMASK = {"ellipse": 2, "tau": 4, "ellipse+tau": 6}


def mask_ties(orc, case, pixmask, tau, k=3.0, band=1e-4):
    """(i, j, pixel) triples whose mask decision is within `band` of the boundary in Q."""
    w = case["w"]
    aabb, vis, sp = orc.splats(case["params"], case["rot"], case["shift"], w.D, case["px"], k=k, tau=tau)
    n = 0
    half = w.D // 2
    for i in range(aabb.shape[0]):
        for j in np.nonzero(vis[i])[0]:
            u0, u1, v0, v1 = aabb[i, j]
            u, v = np.meshgrid(np.arange(u0, u1 + 1), np.arange(v0, v1 + 1))
            dx = (u - half) * case["px"] - sp[i, j, 0]
            dy = (v - half) * case["px"] - sp[i, j, 1]
            Q = sp[i, j, 3] * dx * dx + 2 * sp[i, j, 4] * dx * dy + sp[i, j, 5] * dy * dy
            t = []
            if pixmask & 2:
                t.append(k * k)
            if pixmask & 4:
                t.append(2.0 * math.log(abs(sp[i, j, 6]) / tau))
            n += sum(int(np.sum(np.abs(Q - tt) < band)) for tt in t)
    return n


@pytest.mark.parametrize("variant,exact", [("ellipse", False), ("tau", False), ("ellipse+tau", False),
                                           ("ellipse", True), ("ellipse+tau", True)])
def test_pixel_mask_variants(gem, orc, variant, exact):
    """f1: per-pixel selection (exact k-sigma ellipse, per-pixel tau of Eq. 8) on the GPU against
    the oracle (masks applied in forward and backward).  Cases are chosen with no pixel within
    1e-4 (in Q) of a mask boundary, where fp32 and fp64 could decide differently (the GPU's
    value carries <= ~32 ulp of recurrence rounding, ~1e-5 in Q)."""
    pm = PIXMASK[variant]
    tau = 0.5 if pm & 4 else 0.0
    for seed in range(40, 60):
        case = make_case("T", B=3, seed=seed)
        if mask_ties(orc, case, pm, tau) == 0:
            break
    else:
        pytest.fail("no tie-free case")
    w = case["w"]
    cfg = gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=3, tau=tau, pixel_mask=variant,
                        exact_tiles=exact)
    st = gem.GemStep(cfg)
    dev = st.device
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    t = lambda a: torch.from_numpy(a).to(dev)
    proj = torch.empty(3, w.D, w.D, device=dev)
    loss = st.forward(P, t(case["rot"]), t(case["shift"]), t(case["ctf"]), t(case["obs"]), proj=proj)
    grad = gem.SoA.zeros(w.N, dev)
    st.backward(P, grad)
    torch.cuda.synchronize()
    g = grad.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
    o = orc.loss_grad(case["params"], case["rot"], case["shift"], case["ctf"], case["obs"], w.D, case["px"],
                      tau=tau, want=("proj",), pixmask=pm)
    plain = orc.loss_grad(case["params"], case["rot"], case["shift"], case["ctf"], case["obs"], w.D, case["px"],
                          tau=tau, want=("proj",))
    assert np.abs(o["proj"] - plain["proj"]).max() > 1e-3 * np.abs(plain["proj"]).max()   # the mask bites
    pr = proj.cpu().numpy()
    for i in range(3):
        assert maxnorm_rel(pr[i], o["proj"][i]) < IMG_TOL, i
    lo = loss.cpu().numpy()
    assert np.all(np.abs(lo[:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g[:, cols], o["grad"][:, cols]) < GRAD_TOL, name
    if not exact:
        assert_lists_exact(orc, case, [st.export_lists(i) for i in range(3)], 8, tau=tau)   # AABB lists
        return
    # exact ellipse-tile intersection: the lists hold exactly the tiles with a kept pixel (O4m)
    off, base, ids = orc.lists_pixmask(case["params"], case["rot"], case["shift"], w.D, case["px"], 8, pm, tau=tau)
    pruned = 0
    for i in range(3):
        g_off, g_ids, _ = st.export_lists(i)
        assert np.array_equal(g_off, off[i]), i
        o_ids = ids[base[i]: base[i] + off[i, -1]]
        for t in range(len(g_off) - 1):
            assert np.array_equal(np.sort(g_ids[g_off[t]:g_off[t + 1]]), o_ids[off[i, t]:off[i, t + 1]]), (i, t)
        aabb, vis, _ = orc.splats(case["params"], case["rot"][i:i + 1], case["shift"][i:i + 1], w.D, case["px"],
                                  tau=tau)
        pruned += orc.lists(aabb, vis, w.D, 8)[0][0, -1] - g_off[-1]
    assert pruned > 0   # AABB-corner tiles without a kept pixel are gone


def test_X_config_sampled(gem, orc):
    """Config X (500 000 Gaussians, D = 384: 48 x 48 tiles, a non-power-of-two tile grid):
    particle 0's lists are bit-exact, 256 sampled pixels of two particles match the oracle's
    per-pixel projection, and the batch gradient equals the sum of its halves' gradients."""
    B = 4
    case = make_case("X", B=B, seed=17)
    w = case["w"]
    g = run_gpu(gem, case, tile=8)
    assert g["stats"]["status"] == 0, g["stats"]
    sub0 = dict(case, rot=case["rot"][:1], shift=case["shift"][:1], ctf=case["ctf"][:1], obs=case["obs"][:1])
    assert_lists_exact(orc, sub0, [g["st"].export_lists(0)], 8)
    rng = np.random.default_rng(5)
    pix = rng.integers(w.D // 4, 3 * w.D // 4, (256, 2)).astype(np.int32)   # mostly inside the object
    for i in (0, 3):
        ref = orc.project_pixels(case["params"], case["rot"][i], case["shift"][i], w.D, case["px"], pix)
        got = g["proj"][i][pix[:, 1], pix[:, 0]]
        full_max = np.abs(g["proj"][i]).max()
        assert np.abs(got - ref).max() < IMG_TOL * full_max, i
    assert np.all(np.isfinite(g["loss"]))
    parts = []
    for h in range(2):
        sl = slice(2 * h, 2 * h + 2)
        sub = dict(case, rot=case["rot"][sl], shift=case["shift"][sl], ctf=case["ctf"][sl], obs=case["obs"][sl])
        parts.append(run_gpu(gem, sub, tile=8, want_pred=False)["grad"].astype(np.float64))
    tot = parts[0] + parts[1]
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], tot[:, cols]) < 1e-5, name


@pytest.mark.parametrize("tile", [8, 16])
def test_negative_densities(gem, orc, tile):
    """Training can drive densities negative; those Gaussians take the recurrence (fast) path
    with a negative amplitude and must match the oracle like positive ones."""
    case = make_case("T", B=3, seed=23)
    mr = case["params"][0].copy()
    rng = np.random.default_rng(2)
    neg = rng.random(mr.shape[0]) < 0.3
    mr[neg, 3] *= -1.0
    case["params"] = (mr, case["params"][1], case["params"][2])
    g = run_gpu(gem, case, tile=tile, want_lists=True)
    assert_lists_exact(orc, case, g["lists"], tile)
    o = oracle_out(orc, case)
    for i in range(3):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name


@pytest.mark.parametrize("D", [64, 128, 256, 48])
def test_spectral_paths(gem, orc, D):
    """The row-column spectral path (D = 64 / 128 / 256: cuFFT 1D rows + k_ctf_colspec<8, 8> /
    <16, 8> / <16, 16>, whose packed gradient rows Z = A + iB take the in-lane (S = 2) and the
    cross-lane (S = 1) pairing) and the 2D fallback (D = 48: 2D cuFFT + k_ctf_loss +
    k_dldi_pack) against the oracle: images, prediction, loss and gradients."""
    case = make_case("T", B=3, seed=29, N=800, D=D)
    g = run_gpu(gem, case, cap=1 << 18)   # the default list capacity is sized for N, not for D
    assert g["stats"]["overflow"] == 0
    o = oracle_out(orc, case)
    for i in range(3):
        assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL
        assert maxnorm_rel(g["pred"][i], o["pred"][i]) < IMG_TOL
    assert np.all(np.abs(g["loss"][:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    for name, cols in CLASSES.items():
        assert maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols]) < GRAD_TOL, name


def test_P_config_sampled(gem, orc):
    """Config P (100 000 Gaussians, D = 256: 25 binning chunks): particle 0's lists are
    bit-exact and 256 sampled pixels of both particles match the oracle's per-pixel projection."""
    B = 2
    case = make_case("P", B=B, seed=31)
    w = case["w"]
    g = run_gpu(gem, case, tile=8)
    assert g["stats"]["status"] == 0, g["stats"]
    sub0 = dict(case, rot=case["rot"][:1], shift=case["shift"][:1], ctf=case["ctf"][:1], obs=case["obs"][:1])
    assert_lists_exact(orc, sub0, [g["st"].export_lists(0)], 8)
    rng = np.random.default_rng(6)
    pix = rng.integers(w.D // 4, 3 * w.D // 4, (256, 2)).astype(np.int32)
    for i in range(B):
        ref = orc.project_pixels(case["params"], case["rot"][i], case["shift"][i], w.D, case["px"], pix)
        got = g["proj"][i][pix[:, 1], pix[:, 0]]
        assert np.abs(got - ref).max() < IMG_TOL * np.abs(g["proj"][i]).max(), i
    assert np.all(np.isfinite(g["loss"])) and np.all(np.isfinite(g["grad"]))


def test_flag_combination_zsort_ellipse_no_rotation(gem, orc):
    """Flags compose: z-sorted AABB lists (f1), the exact-ellipse pixel mask (f1) and the
    No Rotation ablation (f3) together, against the oracle's O4z lists, masked images, loss and
    gradients (q = identity, its gradient exactly zero)."""
    for seed in range(60, 80):
        case = make_case("T", B=3, seed=seed)
        mr, ls, q = (a.copy() for a in case["params"])
        q[:] = [1.0, 0.0, 0.0, 0.0]
        case = dict(case, params=(mr, ls, q))
        if mask_ties(orc, case, 2, 0.0) == 0:
            break
    else:
        pytest.fail("no tie-free case")
    w = case["w"]
    dev = torch.device("cuda", 0)
    cfg = gem.GemConfig(D=w.D, pixel_size=case["px"], n_gauss=w.N, max_batch=3, zsort=True, pixel_mask="ellipse",
                        ablation="no_rotation")
    st = gem.GemStep(cfg, dev)
    P = gem.SoA.from_arrays(*case["params"], device=dev)
    t = lambda a: torch.from_numpy(a).to(dev)
    proj = torch.empty(3, w.D, w.D, device=dev)
    loss = st.forward(P, t(case["rot"]), t(case["shift"]), t(case["ctf"]), t(case["obs"]), proj=proj)
    grad = gem.SoA.zeros(w.N, dev)
    st.backward(P, grad)
    torch.cuda.synchronize()
    assert assert_zsorted_lists_exact(orc, case, [st.export_lists(i) for i in range(3)], 8) > 0
    o = orc.loss_grad(case["params"], case["rot"], case["shift"], case["ctf"], case["obs"], w.D, case["px"],
                      want=("proj",), pixmask=2)
    pr = proj.cpu().numpy()
    for i in range(3):
        assert maxnorm_rel(pr[i], o["proj"][i]) < IMG_TOL, i
    lo = loss.cpu().numpy()
    assert np.all(np.abs(lo[:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    g = grad.t.permute(1, 0, 2).reshape(w.N, 12).cpu().numpy()
    assert np.all(g[:, 8:12] == 0.0)
    for name, cols in CLASSES.items():
        if name != "q":
            assert maxnorm_rel(g[:, cols], o["grad"][:, cols]) < GRAD_TOL, name


# ------------------------------------------------------------ round 2: parity gaps
def assert_step_matches_oracle(orc, case, g, img=True):
    o = oracle_out(orc, case, want=("proj", "pred") if img else ())
    B = case["rot"].shape[0]
    if img:
        for i in range(B):
            assert maxnorm_rel(g["proj"][i], o["proj"][i]) < IMG_TOL, i
            assert maxnorm_rel(g["pred"][i], o["pred"][i]) < IMG_TOL, i
    assert np.all(np.abs(g["loss"][:-1] - o["loss"]) < LOSS_TOL * o["loss"])
    assert abs(g["loss"][-1] - o["total"]) < LOSS_TOL * o["total"]
    for name, cols in CLASSES.items():
        err = maxnorm_rel(g["grad"][:, cols], o["grad"][:, cols])
        assert err < GRAD_TOL, (name, err)
    return o


@pytest.mark.parametrize("B", [9, 20, 33])
@pytest.mark.parametrize("tile,fused", [(8, False), (16, False), (8, True), (16, True)])
def test_multichunk_backward_vs_oracle(gem, orc, B, tile, fused):
    """The backward sums each Gaussian's partials over chunks of 8 particles (render.cu kBwdP)
    and the reduction adds the chunks in order (optim.cu k_reduce_finalize).  B = 9, 20, 33 give
    2, 3 and 5 chunks with a partial last chunk (1, 4 and 1 particles); fused mode renders in
    waves of 7 (its own chunking per wave).  Gradients per class against the oracle, images and
    losses too."""
    case = make_case("T", B=B, seed=40 + B)
    g = run_gpu(gem, case, tile=tile, fused=fused, wave=7 if fused else 0)
    assert g["stats"]["status"] == 0, g["stats"]
    assert_step_matches_oracle(orc, case, g)


@pytest.mark.parametrize("tile", [8, 16])
@pytest.mark.parametrize("major,minor", [(1.6, -0.5), (2.2, -0.4)])
def test_needle_gaussians_direct_paths(gem, orc, tile, major, minor):
    """Needle-shaped Gaussians (one axis x e^major, one x e^minor: aspect ratios ~6-20, minor
    sigma ~0.3-0.45 px): their boxes span many tiles and the recurrence factors at far box
    corners leave the normal range, so the forward (render.cu k_render_fwd_le / k_render_fwd)
    and the backward (k_render_bwd) take their direct exp-per-pixel paths for those entries;
    the rest of the model takes the recurrence.  Images, loss and gradients against the oracle."""
    case = make_case("T", B=4, seed=51, N=400)
    mr, ls, q = (a.copy() for a in case["params"])
    sel = np.arange(0, 400, 3)
    ls[sel, 0] += major
    ls[sel, 1] += minor
    case["params"] = (mr, ls, q)
    # the direct paths are taken: some box has a first-column corner with log2 e < -100
    # (Q > 100 / (log2(e) / 2) = 138.6), the forward's and backward's threshold
    w = case["w"]
    aabb, vis, sp = orc.splats(case["params"], case["rot"], case["shift"], w.D, case["px"])
    x = lambda u: (u - w.D // 2) * case["px"]
    Q = lambda s_, u, v: s_[3] * (x(u) - s_[0]) ** 2 + 2 * s_[4] * (x(u) - s_[0]) * (x(v) - s_[1]) + s_[5] * (x(v) - s_[1]) ** 2
    n_direct = sum(1 for i in range(4) for j in sel if vis[i, j] and
                   max(Q(sp[i, j], aabb[i, j, 0], aabb[i, j, 2]), Q(sp[i, j], aabb[i, j, 0], aabb[i, j, 3])) > 138.7)
    assert n_direct > 20, n_direct
    g = run_gpu(gem, case, tile=tile, want_lists=True)
    assert g["stats"]["status"] == 0, g["stats"]
    assert_lists_exact(orc, case, g["lists"], tile)
    assert_step_matches_oracle(orc, case, g)


def test_degenerate_gaussians_skipped_zero_rows_counted(gem, orc):
    """Reading L18: a Gaussian with q = 0, a non-finite density, a non-finite
    centre or an overflowing log-scale (exp(2 s) = inf in fp64) is skipped in every pair, gets an
    exactly-zero gradient row and is counted; the step stays finite and every other row equals
    the oracle's."""
    case = make_case("T", B=3, seed=52)
    mr, ls, q = (a.copy() for a in case["params"])
    q[3] = 0.0
    mr[10, 3] = np.nan
    mr[11, 0] = np.inf
    ls[12, 1] = 400.0
    ls[13, 2] = np.nan
    q[14, 2] = np.inf
    case["params"] = (mr, ls, q)
    bad = [3, 10, 11, 12, 13, 14]
    g = run_gpu(gem, case, want_lists=True)
    st = g["stats"]
    assert st["status"] == 0 and st["degenerate"] == len(bad) and st["nonfinite"] == 0, st
    for j in bad:
        assert np.all(g["grad"][j] == 0.0), j
    assert np.isfinite(g["grad"]).all() and np.isfinite(g["loss"]).all()
    for lst in g["lists"]:
        assert not np.isin(lst[1], bad).any()
    o = assert_step_matches_oracle(orc, case, g)
    for j in bad:
        assert np.all(o["grad"][j] == 0.0), j


def test_nonfinite_loss_is_reported(gem):
    """a non-finite loss must abort training.  A NaN in an observed image makes the
    loss non-finite; gem_stats reports GEM_E_NONFINITE (and the Python wrapper raises)."""
    from paper_2509_25075_b200 import binding as b
    case = make_case("T", B=2, seed=53)
    case["obs"] = case["obs"].copy()
    case["obs"][1, 5, 7] = np.nan
    g = run_gpu(gem, case)
    assert g["stats"]["status"] == b.GEM_E_NONFINITE and g["stats"]["nonfinite"] == 1
    assert not np.isfinite(g["loss"][1]) and np.isfinite(g["loss"][0])
    with pytest.raises(b.GemError) as e:
        g["st"].stats()
    assert e.value.status == b.GEM_E_NONFINITE


@pytest.mark.parametrize("D,tile", [(848, 8), (1696, 16)])
def test_boxes_exact_at_large_D(gem, orc, D, tile):
    """at large D one fp32 ulp of a pixel coordinate approaches the splat's exactness
    margin; the margin now scales with |bound| (prep_bin.cu k_splat_count).  Gaussians spread over
    the whole frame (|coordinates| up to ~D/2 px), one particle, the largest D each tile size
    supports (the splat's shared tile histograms bound the tile grid; a larger D is rejected):
    every AABB and list equals the oracle's (reading L22)."""
    from paper_2509_25075_b200 import binding as b
    with pytest.raises(b.GemError) as e:
        gem.GemStep(gem.GemConfig(D=2 * D, pixel_size=0.5, n_gauss=10, max_batch=1, tile=tile))
    assert e.value.status == b.GEM_E_INVALID
    rng = np.random.default_rng(D)
    N, px = 4000, 0.5
    w = synth.Workload("big", N, D, px, 1)
    mu = rng.uniform(-0.48, 0.48, (N, 3)) * D * px
    ls = np.c_[np.log(rng.uniform(0.4, 6.0, (N, 3)) * px), np.zeros(N)]
    q = rng.standard_normal((N, 4))
    mr = np.c_[mu, rng.uniform(0.5, 1.5, N)]
    rot, shift, ctf = synth.particles(w, 1, 7)
    mr, ls, q, rot, shift, ctf = synth.f32(mr, ls, q, rot, shift, ctf)
    obs = np.zeros((1, D, D), np.float32)
    case = dict(w=w, params=(mr, ls, q), rot=rot, shift=shift, ctf=ctf, obs=obs, px=float(np.float32(px)))
    st = gem.GemStep(gem.GemConfig(D=D, pixel_size=case["px"], n_gauss=N, max_batch=1, tile=tile))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    t = lambda a: torch.from_numpy(a).to(st.device)
    st.forward(P, t(rot), t(shift), t(ctf), t(obs))
    torch.cuda.synchronize()
    assert st.stats(check=False)["status"] == 0
    ties = assert_lists_exact(orc, case, [st.export_lists(0)], tile)
    assert ties == 0


def test_render_volume_bitwise_reproducible(gem, orc):
    """Row a11: brick lists are filled with atomics, but every brick sorts its list by Gaussian id
    before accumulating (volume.cu k_vol_render), so repeated queries are bitwise identical; a
    brick whose list exceeds the in-shared-memory sort (> 1024 entries: a dense cluster of wide
    Gaussians) takes the global-memory ranking path, against the oracle too."""
    case = make_case("T", B=1, seed=61, N=3000, D=32)
    mr, ls, q = case["params"]
    st = gem.GemStep(gem.GemConfig(D=32, pixel_size=4.0, n_gauss=3000, max_batch=1))
    P = gem.SoA.from_arrays(mr, ls, q, device=st.device)
    a = st.render_volume(P, 40, 4.0).cpu().numpy()
    b = st.render_volume(P, 40, 4.0).cpu().numpy()
    assert np.array_equal(a, b)
    # 1500 wide Gaussians around the centre: >1024 entries in the central bricks
    mr2, ls2 = mr.copy(), ls.copy()
    mr2[:1500, :3] *= 0.05
    ls2[:1500, :3] += 1.0
    P2 = gem.SoA.from_arrays(mr2, ls2, q, device=st.device)
    c = st.render_volume(P2, 40, 4.0).cpu().numpy()
    d = st.render_volume(P2, 40, 4.0).cpu().numpy()
    assert np.array_equal(c, d)
    ref = orc.volume((mr2, ls2, q), 40, 4.0, masked=True)
    assert maxnorm_rel(c, ref) < IMG_TOL
