"""Python API over libgem.so: one GEM training step on one GPU, and its
data-parallel wrapper (one process per GPU, NCCL all-reduce of the gradient).

PyTorch is used only for device memory, streams and process groups; every
arithmetic step of the path runs in libgem.so's kernels (binding.py does
argument marshalling only).
"""
from __future__ import annotations

import ctypes
import dataclasses

import torch

from . import binding as _b


@dataclasses.dataclass
class GemConfig:
    D: int
    pixel_size: float
    n_gauss: int
    max_batch: int
    cull_k: float = 3.0
    tau: float = 0.0
    tile: int = 8
    list_capacity: int = 0
    lr_mean: float = 1e-3
    lr_log_scale: float = 5e-3
    lr_quat: float = 1e-3
    lr_density: float = 5e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    fused: bool = False   # L2-resident wave pipeline (GEM_FLAG_FUSED)
    wave: int = 0         # particles per wave (0 = auto)
    ablation: str = "full"   # Table 5: full | no_rotation | isotropic_scale | both
    zsort: bool = False      # P:227 z-sorted per-tile lists (GEM_FLAG_ZSORT)
    pixel_mask: str = "aabb"  # Eq. 8 per-pixel selection: aabb | ellipse | tau | ellipse+tau
    exact_tiles: bool = False  # with a pixel mask: lists hold only tiles with a kept pixel

    def c(self) -> _b.GemConfigC:
        return _b.GemConfigC(self.D, self.pixel_size, self.n_gauss, self.max_batch, self.cull_k, self.tau, self.tile,
                             self.list_capacity, self.lr_mean, self.lr_log_scale, self.lr_quat, self.lr_density,
                             self.beta1, self.beta2, self.eps, self.flags(), self.wave)

    def flags(self) -> int:
        if self.ablation not in ("full", "no_rotation", "isotropic_scale", "both"):
            raise ValueError(f"unknown ablation {self.ablation!r}")
        f = _b.GEM_FLAG_FUSED if self.fused else 0
        if self.zsort:
            f |= _b.GEM_FLAG_ZSORT
        if self.pixel_mask not in ("aabb", "ellipse", "tau", "ellipse+tau"):
            raise ValueError(f"unknown pixel_mask {self.pixel_mask!r}")
        if "ellipse" in self.pixel_mask:
            f |= _b.GEM_FLAG_ELLIPSE
        if "tau" in self.pixel_mask:
            f |= _b.GEM_FLAG_PIXEL_TAU
        if self.exact_tiles:
            f |= _b.GEM_FLAG_EXACT_TILES
        if self.ablation in ("no_rotation", "both"):
            f |= _b.GEM_FLAG_NO_ROTATION
        if self.ablation in ("isotropic_scale", "both"):
            f |= _b.GEM_FLAG_ISOTROPIC
        return f


class SoA:
    """Gaussian parameter store a0: one contiguous float32 tensor [3, N, 4]
    = (mean_rho, log_scale, quat) so a gradient is one buffer (one all-reduce)."""

    def __init__(self, t: torch.Tensor):
        assert t.dtype == torch.float32 and t.dim() == 3 and t.shape[0] == 3 and t.shape[2] == 4
        assert t.is_contiguous() and t.data_ptr() % 16 == 0
        self.t = t

    @classmethod
    def zeros(cls, N, device):
        return cls(torch.zeros(3, N, 4, dtype=torch.float32, device=device))

    @classmethod
    def from_arrays(cls, mean_rho, log_scale, quat, device):
        t = torch.stack([torch.as_tensor(a, dtype=torch.float32) for a in (mean_rho, log_scale, quat)])
        return cls(t.to(device).contiguous())

    @property
    def N(self):
        return self.t.shape[1]

    def c(self) -> _b.GemSoaC:
        base, step = self.t.data_ptr(), self.t.stride(0) * 4
        return _b.GemSoaC(base, base + step, base + 2 * step)


def _ptr(t):
    return None if t is None else t.data_ptr()


class GemStep:
    """Owns one libgem context, its workspace (a torch uint8 tensor) and stream."""

    def __init__(self, cfg: GemConfig, device=None, stream: torch.cuda.Stream | None = None, guard_bytes: int = 0):
        """guard_bytes > 0 (tests): that many canary bytes (0xA5) follow the workspace; see
        guard_intact()."""
        self.cfg = cfg
        self.device = torch.device(device or "cuda")
        self.lib = _b.lib()
        self.stream = stream or torch.cuda.current_stream(self.device)
        c = cfg.c()
        nbytes = self.lib.gem_workspace_bytes(ctypes.byref(c))
        if nbytes == 0:
            raise _b.GemError(_b.GEM_E_INVALID, "gem_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256 + guard_bytes, dtype=torch.uint8, device=self.device)
        off = (-self.workspace.data_ptr()) % 256
        self._ws_ptr = self.workspace.data_ptr() + off
        self._ws_bytes = nbytes
        self._guard = self.workspace[off + nbytes: off + nbytes + guard_bytes] if guard_bytes else None
        if self._guard is not None:
            self._guard.fill_(0xA5)
        h = ctypes.c_void_p()
        _b.check(self.lib.gem_init(ctypes.byref(c), self._ws_ptr, nbytes, self.stream.cuda_stream, ctypes.byref(h)),
                 "gem_init")
        self.ctx = h
        self.launches = 0

    def guard_intact(self) -> bool:
        """True if no kernel wrote past the end of the workspace (the canary bytes are intact)."""
        torch.cuda.synchronize(self.device)
        return self._guard is None or bool((self._guard == 0xA5).all())

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.gem_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- calls
    def forward(self, params: SoA, rot, shift, ctf, observed, loss=None, proj=None, pred=None, host=False):
        """gem_forward.  Device tensors (or pinned host tensors with host=True).
        Returns the loss tensor [B+1] (float64; per particle then total)."""
        B = rot.shape[0]
        if loss is None:
            loss = torch.empty(B + 1, dtype=torch.float64, device="cpu" if host else self.device,
                               pin_memory=host)
        bt = _b.GemBatchC(B, _b.GEM_MEM_HOST if host else _b.GEM_MEM_DEVICE, rot.data_ptr(), shift.data_ptr(),
                          ctf.data_ptr(), observed.data_ptr())
        sp = params.c()
        _b.check(self.lib.gem_forward(self.ctx, ctypes.byref(sp), ctypes.byref(bt), loss.data_ptr(), _ptr(proj),
                                      _ptr(pred), self.stream.cuda_stream), "gem_forward")
        self.launches += self.lib.gem_last_launch_count(self.ctx)
        return loss

    def backward(self, params: SoA, grad: SoA):
        sp, sg = params.c(), grad.c()
        _b.check(self.lib.gem_backward(self.ctx, ctypes.byref(sp), ctypes.byref(sg), self.stream.cuda_stream),
                 "gem_backward")
        self.launches += self.lib.gem_last_launch_count(self.ctx)

    def step(self, params: SoA, grad: SoA, m: SoA, v: SoA, t: int):
        sp, sg, sm, sv = params.c(), grad.c(), m.c(), v.c()
        _b.check(self.lib.gem_step(self.ctx, ctypes.byref(sp), ctypes.byref(sg), ctypes.byref(sm), ctypes.byref(sv),
                                   int(t), self.stream.cuda_stream), "gem_step")
        self.launches += self.lib.gem_last_launch_count(self.ctx)

    def render_volume(self, params: SoA, Dv: int, voxel_size: float, out=None):
        if out is None:
            out = torch.empty((Dv, Dv, Dv), dtype=torch.float32, device=self.device)
        nbytes = self.lib.gem_volume_scratch_bytes(self.ctx, Dv, voxel_size)
        gb = 4096 if self._guard is not None else 0
        scratch = torch.empty(nbytes + 256 + gb, dtype=torch.uint8, device=self.device)
        off = (-scratch.data_ptr()) % 256
        ptr = scratch.data_ptr() + off
        if gb:
            scratch[off + nbytes: off + nbytes + gb].fill_(0xA5)
        sp = params.c()
        _b.check(self.lib.gem_render_volume(self.ctx, ctypes.byref(sp), Dv, voxel_size, out.data_ptr(), ptr, nbytes,
                                            self.stream.cuda_stream), "gem_render_volume")
        self.launches += self.lib.gem_last_launch_count(self.ctx)
        if gb and not bool((scratch[off + nbytes: off + nbytes + gb] == 0xA5).all()):
            raise RuntimeError("gem_render_volume wrote past its scratch buffer")
        return out

    def export_lists(self, particle: int):
        import numpy as np
        nt = -(-self.cfg.D // self.cfg.tile)
        NT = nt * nt
        tile_off = np.zeros(NT + 1, np.int32)
        aabb = np.zeros((self.cfg.n_gauss, 4), np.int32)
        _b.check(self.lib.gem_export_lists(self.ctx, particle, tile_off.ctypes.data, None, 0, aabb.ctypes.data),
                 "gem_export_lists")
        ids = np.zeros(max(int(tile_off[-1]), 1), np.int32)
        _b.check(self.lib.gem_export_lists(self.ctx, particle, None, ids.ctypes.data, ids.size, None),
                 "gem_export_lists")
        return tile_off, ids[: tile_off[-1]], aabb

    def profile(self, enable: bool):
        _b.check(self.lib.gem_profile_enable(self.ctx, int(enable)), "gem_profile_enable")

    def profile_read(self):
        """{kernel: (launches, total_ms)} recorded with CUDA events on the launching stream."""
        buf = (_b.GemKernelTimeC * 32)()
        n = self.lib.gem_profile_read(self.ctx, buf, 32)
        if n < 0:
            raise _b.GemError(_b.GEM_E_CUDA, "gem_profile_read")
        return {buf[k].name.decode(): (buf[k].launches, buf[k].total_ms) for k in range(min(n, 32))}

    def stats(self, check=True):
        st = _b.GemStatsC()
        s = self.lib.gem_stats(self.ctx, ctypes.byref(st))
        if check:
            _b.check(s, "gem_stats")
        return {k: getattr(st, k) for k, _ in _b.GemStatsC._fields_} | {"status": s}


class Trainer:
    """One data-parallel GEM training step per call:
    gem_forward -> gem_backward -> all_reduce(grad, SUM) over NCCL -> gem_step.
    Parameters and Adam moments are replicated; particles are sharded."""

    def __init__(self, cfg: GemConfig, params: SoA, device=None, group=None):
        self.step_ctx = GemStep(cfg, device)
        self.params = params
        N = params.N
        dev = params.t.device
        # one contiguous fp32 buffer: the [3, N, 4] gradient, then the rank's total loss (and 3
        # pad words, keeping 16-byte alignment): SURVEY §8(a) a9's single all-reduce payload
        self.flat = torch.zeros(12 * N + 4, dtype=torch.float32, device=dev)
        self.grad = SoA(self.flat[: 12 * N].view(3, N, 4))
        self.m = SoA.zeros(N, dev)
        self.v = SoA.zeros(N, dev)
        self.t = 0
        self.group = group
        # with more than one rank: the loss summed over ranks after each step (fp32), all-reduced
        # with the gradient; one rank has its total in train_step's returned loss[-1]
        self.global_loss = self.flat[12 * N: 12 * N + 1]

    def train_step(self, rot, shift, ctf, observed, host=False, loss=None):
        g = self.step_ctx
        loss = g.forward(self.params, rot, shift, ctf, observed, loss=loss, host=host)
        g.backward(self.params, self.grad)
        if _world(self.group) > 1:
            with torch.cuda.stream(g.stream) if self.flat.is_cuda else _nullctx():
                self.global_loss.copy_(loss[-1:], non_blocking=True)   # the rank's total, appended
                allreduce_flat(self.flat, self.group)                  # gradient + loss: one collective
        self.t += 1
        g.step(self.params, self.grad, self.m, self.v, self.t)
        return loss


class HostPipeline:
    """End-to-end training from pinned host batches through the public API: the inputs of step
    k+1 are copied host->device on a side stream into the other half of a double buffer while
    step k runs, and every step's loss is read back to pinned host memory.  Every input byte of
    every step still crosses PCIe inside the caller's timed region; only the overlap is new."""

    def __init__(self, trainer: "Trainer", B: int, D: int):
        dev = trainer.params.t.device
        self.tr = trainer
        self.compute = trainer.step_ctx.stream
        self.copy = torch.cuda.Stream(dev)
        mk = lambda *shape: torch.empty(*shape, dtype=torch.float32, device=dev)
        self.bufs = [(mk(B, 9), mk(B, 2), mk(B, 8), mk(B, D, D)) for _ in range(2)]
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self.used = [False, False]
        self.loss_host = torch.empty(B + 1, dtype=torch.float64, pin_memory=True)

    def _load(self, slot, batch):
        with torch.cuda.stream(self.copy):
            if self.used[slot]:
                self.copy.wait_event(self.free[slot])   # step k-1 finished reading this buffer
            for dst, src in zip(self.bufs[slot], batch):
                dst.copy_(src, non_blocking=True)
            self.ready[slot].record(self.copy)

    def run(self, batches):
        """batches: sequence of pinned host (rot [B,9], shift [B,2], ctf [B,8], observed [B,D,D]).
        Returns the pinned host loss of the last step (valid after a stream sync)."""
        n = len(batches)
        self._load(0, batches[0])
        for k in range(n):
            slot = k % 2
            if k + 1 < n:
                self._load(1 - slot, batches[k + 1])
            self.compute.wait_event(self.ready[slot])
            loss = self.tr.train_step(*self.bufs[slot])
            self.free[slot].record(self.compute)
            self.used[slot] = True
            with torch.cuda.stream(self.compute):
                self.loss_host.copy_(loss, non_blocking=True)
        return self.loss_host


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _world(group=None) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def allreduce_flat(flat: "torch.Tensor", group=None):
    """Sum a contiguous fp32 buffer (gradient + appended loss) over the data-parallel ranks."""
    import torch.distributed as dist
    if _world(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def allreduce_grad(grad: SoA, group=None):
    """Sum the [3, N, 4] gradient over the data-parallel ranks (one collective;
    NCCL over NVLink on GPUs, gloo on CPU tests).  No-op without a process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad.t, op=dist.ReduceOp.SUM, group=group)
    return grad


def replicas_identical(tensors, group=None) -> bool:
    """the replicated parameters / Adam moments must stay bit-identical across the
    data-parallel ranks.  A 64-bit checksum of the raw bytes of `tensors` (a diagnostic outside
    the training step) is all-gathered and compared; True without a process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return True
    h = torch.zeros(1, dtype=torch.int64, device=tensors[0].device)
    for t in tensors:
        w = t.detach().contiguous().view(torch.int32).reshape(-1).to(torch.int64)
        idx = torch.arange(1, w.numel() + 1, device=w.device, dtype=torch.int64)
        h += (w * idx).sum()                 # position-weighted: permutations change the sum
    hs = [torch.zeros_like(h) for _ in range(dist.get_world_size(group))]
    dist.all_gather(hs, h, group=group)
    return all(bool((x == hs[0]).all()) for x in hs)


def shard_indices(n_particles: int, world: int, rank: int, batch: int, step: int, seed: int = 0):
    """Particle ids rank `rank` processes at `step`: a contiguous disjoint shard
    per rank, drawn with a per-epoch seeded permutation."""
    import numpy as np
    per = n_particles // world
    lo = rank * per
    per_epoch = max(per // batch, 1)
    epoch, k = divmod(step, per_epoch)
    perm = np.random.default_rng((seed, rank, epoch)).permutation(per)
    idx = perm[(k * batch) % per: (k * batch) % per + batch]
    if idx.size < batch:
        idx = np.concatenate([idx, perm[: batch - idx.size]])
    return lo + idx
