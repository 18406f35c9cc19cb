#!/usr/bin/env python
"""bench.py — throughput of one GEM training step on B200 (particle images/s).

A "step" is one pass of the whole hot path over one
batch of B particles per GPU: Gaussian prep, splat + cull/bin, per-tile lists,
projection, cuFFT + fused CTF/loss, backward scatter, finalize, NCCL all-reduce
of the N x 12 gradient (N>1) and the fused Adam update.  Workload: config R of
BASELINE.json (EMPIAR-10028-shaped: N = 50,000 Gaussians, D = 256, px 1.31 A),
synthetic seeded inputs, weak scaling (B per GPU fixed).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  Multi-GPU: launched by torch.distributed.run,
one rank per GPU, NCCL; the timed region is bracketed by barrier + sync and the
elapsed time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2509_25075_b200 import synth  # noqa: E402

METRIC = "particle images/sec per train step (fwd+bwd) at D=256"
SNR = 0.1
# algorithmic work per useful (Gaussian, pixel) pair of the direct method (DESIGN.md
# §5): FP32 lane-ops (an FMA counts once) -- the roofline's unit -- and FLOPs (an FMA counts twice)
LANEOPS_FWD_PAIR = 9
LANEOPS_BWD_PAIR = 22
FLOP_FWD_PAIR = 12
FLOP_BWD_PAIR = 25


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["gem", "reference"], default="gem")
    ap.add_argument("--config", default="R", choices=sorted(synth.CONFIGS))
    ap.add_argument("--batch", type=int, default=256, help="particles per GPU per step")
    ap.add_argument("--tile", type=int, default=8)
    ap.add_argument("--state", default="steady", choices=["steady", "init"])
    ap.add_argument("--ring", type=int, default=1024, help="distinct device-resident particles per GPU")
    ap.add_argument("--fused", action="store_true", help="L2-resident wave pipeline (GEM_FLAG_FUSED)")
    ap.add_argument("--wave", type=int, default=0, help="particles per wave (0 = auto)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: this many particles per step in total, split over the GPUs")
    ap.add_argument("--zsort", action="store_true", help="P:227 z-sorted tile lists (GEM_FLAG_ZSORT)")
    ap.add_argument("--no-volume", action="store_true", help="skip the gem_render_volume timing (row a11)")
    ap.add_argument("--pixel-mask", default="aabb", choices=["aabb", "ellipse", "tau", "ellipse+tau"],
                    help="Eq. 8 per-pixel selection variant (GEM_FLAG_ELLIPSE / GEM_FLAG_PIXEL_TAU)")
    ap.add_argument("--tau", type=float, default=0.0)
    ap.add_argument("--exact-tiles", action="store_true", help="with --pixel-mask: lists of tiles with a kept pixel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="skip the second, per-kernel profiled pass (no breakdown, no roofline)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# BASELINE.json's configs: what each synthetic workload is shaped like
SHAPES = {"T": "tiny synthetic", "S": "CryoBench-like small protein", "R": "EMPIAR-10028-shaped ribosome",
          "P": "EMPIAR-10180-shaped spliceosome", "X": "large-scale stress", "A": "desk-scale round trip"}


def measured_traffic(kernel, workload, batch, tile, variant):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json); None unless this run has the captured configuration."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p))
        cap = t["config"]
        if (workload, batch, tile, variant) != (cap["workload"], cap["batch"], cap["tile"], cap["variant"]):
            return None
        return t[kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def fp32_peak_tflops(sm_mhz):
    """148 SMs x 128 FP32 lanes x 2 FLOP/FMA x clock (B200_PROFILING.md unit counts)."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def fp32_peak_tlaneops(sm_mhz):
    """148 SMs x 128 FP32 lanes x clock: FP32 lane-operations per second (T/s)."""
    return 148 * 128 * sm_mhz * 1e6 / 1e12


def cpu_info():
    """CPU model, sockets and threads of the host (lscpu), for the cpu_baseline record."""
    info = {}
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["cpu_model"] = v
            elif k == "Socket(s)":
                info["sockets"] = int(v) if v.isdigit() else v
            elif k == "CPU(s)":
                info["host_threads"] = int(v) if v.isdigit() else v
            elif k == "Thread(s) per core":
                info["threads_per_core"] = int(v) if v.isdigit() else v
    except Exception:
        pass
    return info


class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu_index = int(gpu_index)
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu_index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while True:
            mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((time.perf_counter(), mhz, r))
            self._ready.set()
            if self._stop.wait(0.002):
                break

    def __enter__(self):
        self._ready = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            self._ready.wait(timeout=5)   # sampling runs before the timed region starts
        except Exception:
            self.t = None
        return self

    def mark(self, which):
        """Host time of the timed region's start / end (samples outside it are dropped)."""
        setattr(self, which, time.perf_counter())

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=2)

    def summary(self):
        t0, t1 = getattr(self, "start", None), getattr(self, "end", None)
        inside = [x for x in self.samples if t0 is None or t1 is None or t0 <= x[0] <= t1]
        if not inside and self.samples:   # region shorter than the sampling period: nearest sample
            mid = 0.5 * (t0 + t1) if t0 is not None and t1 is not None else self.samples[-1][0]
            inside = [min(self.samples, key=lambda x: abs(x[0] - mid))]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, _, r in inside for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(m for _, m, _ in inside), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(inside)}


# --------------------------------------------------------------- CPU oracle
def oracle_step_sample(w, n_particles, seed=7):
    """One oracle training step (forward, backward, Adam) on n particles of workload w.
    Returns seconds.  TEST/BASELINE infrastructure: the oracle as it stands."""
    import oracle
    mr, ls, q = synth.steady_model(w, 0)
    rot, shift, ctf = synth.particles(w, n_particles, seed)
    obs = synth.noise_images(w, n_particles, seed)
    mr, ls, q, rot, shift, ctf, obs = synth.f32(mr, ls, q, rot, shift, ctf, obs)
    px = float(np.float32(w.px))
    t0 = time.perf_counter()
    out = oracle.loss_grad((mr, ls, q), rot, shift, ctf, obs, w.D, px)
    p = np.stack([mr, ls, q]).astype(np.float64)
    z = np.zeros_like(p)
    oracle.adam(p, oracle.grad_to_soa(out["grad"]), z, z, 1, [1e-3, 5e-3, 1e-3, 5e-2])
    return time.perf_counter() - t0


def cpu_cores():
    env = os.environ.get("OMP_NUM_THREADS")
    return int(env) if env else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def cpu_baseline(w, budget_s=15.0):
    import oracle
    oracle.lib()
    t1 = oracle_step_sample(w, 1)
    n = int(max(1, min(16, budget_s // max(t1, 1e-3))))
    t = oracle_step_sample(w, n) if n > 1 else t1
    return {"value": n / t, "unit": "particles/s", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"{n} particle(s) of workload {w.name} (N={w.N}, D={w.D}): full fp64 forward "
                      f"(masked sum over every Gaussian x pixel), DFT CTF/loss, backward, Adam; {t:.1f} s",
            **cpu_info()}


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle as it stands on the host cores, timed on a
    bounded sample per step (rank 0 only)."""
    if rank != 0:
        return 0
    if world > 1:
        # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 is the only rank that works here, so
        # it takes the host's cores (read by libgomp when the oracle library is first loaded)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                                            else os.cpu_count())
    w = synth.CONFIGS[args.config]
    t1 = oracle_step_sample(w, 1)
    budget = 150.0
    steps = args.steps
    warm = args.warmup
    per_step = 1
    if (steps + warm) * t1 > budget:
        steps = max(1, int(budget // t1) - warm)
    for _ in range(warm):
        oracle_step_sample(w, per_step, seed=11)
    tt = 0.0
    for k in range(steps):
        tt += oracle_step_sample(w, per_step, seed=100 + k)
    value = steps * per_step / tt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * tt / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.name}: N={w.N} Gaussians, D={w.D}, px={w.px} A", "batch_per_step": per_step,
                       "requested_steps": args.steps},
            "cpu_baseline": {"value": value, "unit": "particles/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": f"{per_step} particle per step x {steps} steps", **cpu_info()},
            "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2509_25075_b200 import gem

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator set-up lines (ranks, transports: NVLink / NVLS) on stderr for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        if rank == 0:
            print(f"[bench] NCCL process group: world={world} backend={dist.get_backend()} "
                  f"nccl={torch.cuda.nccl.version()}", file=sys.stderr, flush=True)

    w = synth.CONFIGS[args.config]
    # weak scaling (default): B particles per GPU; strong scaling: a fixed global batch split
    B = args.batch if not args.global_batch else max(1, args.global_batch // world)
    ring = max(args.ring // B, 1) * B
    px = float(np.float32(w.px))
    model = synth.steady_model if args.state == "steady" else synth.init_model
    mr, ls, q = synth.f32(*model(w, 0))
    params = gem.SoA.from_arrays(mr, ls, q, dev)
    phantom = gem.SoA.from_arrays(*synth.f32(*synth.phantom(w, synth.seed_for(w.name, "phantom", 0))), dev)
    cfg = gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B, tile=args.tile,
                        lr_mean=1e-3 * w.ball_radius, fused=args.fused, wave=args.wave, zsort=args.zsort,
                        pixel_mask=args.pixel_mask, tau=args.tau, exact_tiles=args.exact_tiles)

    # device-resident ring of distinct synthetic particles (per-rank seeds)
    rot_np, sh_np, ctf_np = synth.f32(*synth.particles(w, ring, 1000 + rank))
    rot, shift, ctf = (torch.from_numpy(a).to(dev) for a in (rot_np, sh_np, ctf_np))
    obs = torch.empty(ring, w.D, w.D, device=dev)
    gen = gem.GemStep(gem.GemConfig(D=w.D, pixel_size=px, n_gauss=w.N, max_batch=B, tile=args.tile, cull_k=5.0), dev)
    zeros = torch.zeros(B, w.D, w.D, device=dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    for s0 in range(0, ring, B):
        sl = slice(s0, s0 + B)
        gen.forward(phantom, rot[sl], shift[sl], ctf[sl], zeros, pred=obs[sl])
        clean = obs[sl]
        sd = clean.std(dim=(1, 2), keepdim=True) / SNR ** 0.5
        obs[sl] = clean + sd * torch.randn(clean.shape, device=dev, generator=g)
    del gen
    torch.cuda.synchronize()

    tr = gem.Trainer(cfg, params, dev)
    sc = tr.step_ctx

    def step(k, host=False, src=None):
        s0 = (k * B) % ring
        sl = slice(s0, s0 + B)
        if host:
            return tr.train_step(src[0][sl], src[1][sl], src[2][sl], src[3][sl], host=True, loss=src[4])
        return tr.train_step(rot[sl], shift[sl], ctf[sl], obs[sl])

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    gpu_id = int(vis.split(",")[local]) if vis and vis.split(",")[local].isdigit() else local
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = sc.launches
    with ClockSampler(gpu_id) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk.mark("start")
        ev0.record(stream)
        for k in range(args.steps):
            step(args.warmup + k)
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark("end")
        if world > 1:
            dist.barrier()
    launches = sc.launches - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-kernel times: a second pass over the same K steps with a CUDA event pair around every
    # launch group on the launching stream (the events add ~4 us of gap per pair, so they are
    # kept out of the timed region above)
    kern = {}
    if not args.no_kernel_events:
        sc.profile(True)
        for k in range(args.steps):
            step(args.warmup + k)
        torch.cuda.synchronize()
        sc.profile(False)
        kern = sc.profile_read()
    st = sc.stats(check=False)
    value = world * B * args.steps / (ms / 1e3)

    # ---- e2e: the same steps from pinned HOST inputs through the C ABI's own host path
    # (gem_batch.memory = GEM_MEM_HOST: every call copies its poses, CTFs and observed images
    # host->device on libgem's copy stream into double-buffered staging -- so call k + 1's copy
    # runs behind call k's kernels -- and writes the loss to pinned host memory).  Also
    # reported: gem.HostPipeline, which double-buffers the next step's copy from Python, and the
    # PCIe bound: the same bytes through one pinned host->device copy, measured here.
    e2e = None
    if not args.no_e2e:
        hsrc = [a.cpu().pin_memory() for a in (rot, shift, ctf, obs)]
        hloss = torch.empty(B + 1, dtype=torch.float64, pin_memory=True)
        hsrc.append(hloss)

        def timed(fn):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            if world > 1:
                tt = torch.tensor([t], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
            return t

        # the PCIe roofline of the e2e path: one step's input bytes as one pinned H2D copy
        hb = torch.empty(B * (9 + 2 + 8 + w.D * w.D), dtype=torch.float32, pin_memory=True)
        db = torch.empty_like(hb, device=dev)
        for _ in range(3):
            db.copy_(hb, non_blocking=True)
        h2d_ms = timed(lambda: [db.copy_(hb, non_blocking=True) for _ in range(10)]) / 10
        h2d_gbs = hb.numel() * 4 / (h2d_ms * 1e-3) / 1e9
        del hb, db
        for k in range(2):
            step(k, host=True, src=hsrc)

        def abi_steps():
            for k in range(args.steps):
                step(args.warmup + k, host=True, src=hsrc)
        ems = timed(abi_steps)
        _ = float(hloss[-1])  # the last step's loss, read on the host
        pipe = gem.HostPipeline(tr, B, w.D)
        batch = lambda k: [a[((k * B) % ring):((k * B) % ring) + B] for a in hsrc[:4]]
        pipe.run([batch(k) for k in range(2)])
        holder = {}
        pms = timed(lambda: holder.setdefault("lh", pipe.run([batch(args.warmup + k) for k in range(args.steps)])))
        _ = float(holder["lh"][-1])
        e2e = {"value": world * B * args.steps / (ems / 1e3), "unit": "particles/s",
               "h2d_bytes_per_step": B * (9 + 2 + 8 + w.D * w.D) * 4, "d2h_bytes_per_step": (B + 1) * 8,
               "path": "C ABI gem_forward with gem_batch.memory = GEM_MEM_HOST (pinned host poses, CTFs, "
                       "images copied inside every call on libgem's copy stream, double-buffered across calls) "
                       "+ gem_backward + all-reduce + gem_step",
               "pcie": {"bound": "h2d", "h2d_gbs_measured": h2d_gbs,
                        "achieved_gbs": B * (9 + 2 + 8 + w.D * w.D) * 4 * args.steps / (ems * 1e-3) / 1e9,
                        "frac": (B * (9 + 2 + 8 + w.D * w.D) * 4 * args.steps / (ems * 1e-3) / 1e9) / h2d_gbs,
                        "ceiling_particles_per_s": world * h2d_gbs * 1e9 / (4 * (9 + 2 + 8 + w.D * w.D)),
                        "note": "one step's input bytes as a single pinned host->device copy, timed here; the "
                                "e2e value cannot exceed ceiling_particles_per_s with fp32 images"},
               "host_pipeline": {"value": world * B * args.steps / (pms / 1e3), "unit": "particles/s",
                                 "path": "gem.HostPipeline: the next step's inputs copied on a Python side "
                                         "stream, double-buffered behind the current step"}}

    # Table 1's memory metric: what the training step holds on the device.  The
    # synthetic data ring is a dataset stand-in and is reported apart.
    memory = {"workspace_gb": sc._ws_bytes / 1e9, "train_state_gb": 4 * 48 * w.N / 1e9,
              "step_total_gb": (sc._ws_bytes + 4 * 48 * w.N + B * (19 + w.D * w.D) * 4) / 1e9,
              "torch_peak_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
              "data_ring_gb": ring * (19 + w.D * w.D) * 4 / 1e9,
              "d3_buffers": 0, "paper_gem_peak_gb_10028": 1.54}

    # replicated parameters and moments stay bit-identical (checked after timing)
    replicas = gem.replicas_identical([tr.params.t, tr.m.t, tr.v.t]) if world > 1 else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks, peak_src = measured_peaks()
    clocks = clk.summary()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    total_kernel_ms = sum(v[1] for v in kern.values())
    kernels = {k: {"ms_per_step": v[1] / max(args.steps, 1), "launch_groups": v[0],
                   "share": v[1] / total_kernel_ms if total_kernel_ms else None} for k, v in kern.items()}
    pairs = int(st["pairs"])
    variant = (f"{args.state}|fused={args.fused}|zsort={args.zsort}|mask={args.pixel_mask}"
               f"|exact={args.exact_tiles}")
    dominant = max(kern, key=lambda k: kern[k][1]) if kern else None
    roof = None
    if dominant in ("render_fwd", "render_bwd"):
        per_pair = LANEOPS_FWD_PAIR if dominant == "render_fwd" else LANEOPS_BWD_PAIR
        flop_pair = FLOP_FWD_PAIR if dominant == "render_fwd" else FLOP_BWD_PAIR
        avg_s = kern[dominant][1] / kern[dominant][0] / 1e3          # per launch (one wave)
        sec = kern[dominant][1] / 1e3
        achieved = per_pair * pairs * args.steps / sec / 1e12
        peak = fp32_peak_tlaneops(sm_max)
        roof = {"bound": "alu", "kernel": dominant, "achieved": achieved, "peak": peak,
                "unit": "T FP32 lane-ops/s", "frac": achieved / peak,
                "traffic": measured_traffic(dominant, args.config, B, args.tile, variant),
                "work_per_launch": f"{per_pair} FP32 lane-ops (SURVEY 8(d), an FMA counted once) x {pairs} useful "
                                   f"(Gaussian, pixel) pairs per step, {kern[dominant][0] // max(args.steps, 1)} "
                                   "launch(es) per step",
                "avg_launch_ms": avg_s * 1e3,
                "peak_source": f"148 SMs x 128 FP32 lanes x {sm_max:.0f} MHz ({peak_src} sm_max_mhz)",
                "flop_fma2": {"achieved_tflops": flop_pair * pairs * args.steps / sec / 1e12,
                              "peak_tflops": fp32_peak_tflops(sm_max),
                              "frac": flop_pair * pairs * args.steps / sec / 1e12 / fp32_peak_tflops(sm_max),
                              "note": f"{flop_pair} FLOP per pair with an FMA = 2 FLOP"}}
        other = "render_bwd" if dominant == "render_fwd" else "render_fwd"
        if other in kern:
            op = LANEOPS_BWD_PAIR if other == "render_bwd" else LANEOPS_FWD_PAIR
            osec = kern[other][1] / 1e3
            roof["other_render_kernel"] = {"kernel": other, "ms_per_step": kern[other][1] / max(args.steps, 1),
                                           "frac": op * pairs * args.steps / osec / 1e12 / peak}
    elif dominant is not None:
        roof = {"bound": "hbm", "kernel": dominant, "achieved": None, "peak": float(peaks.get("hbm_gbs", 6650.0)),
                "unit": "GB/s", "frac": None, "traffic": None}

    # SURVEY §8(d) step-level roofline: T_roof = FP32 lane-ops of the method (31 per useful pair:
    # forward 9 + backward 22, an FMA counted once) at the FP32 peak + the cuFFT/CTF chain's
    # implementation-minimum HBM bytes (5 D^2 4 + 6 D (D/2+1) 8 per particle) at the HBM peak
    lane_ops = 31.0 * pairs
    chain_bytes = B * (5.0 * w.D * w.D * 4 + 6.0 * w.D * (w.D // 2 + 1) * 8)
    t_fp32 = lane_ops / (148 * 128 * sm_max * 1e6)
    t_hbm = chain_bytes / (float(peaks.get("hbm_gbs", 6537.6)) * 1e9)
    t_roof = t_fp32 + t_hbm
    step_roof = {"t_roof_ms": t_roof * 1e3, "t_step_ms": ms / args.steps, "frac": t_roof / (ms / args.steps / 1e3),
                 "model": "31 FP32 lane-ops per useful pair at 148 SM x 128 lanes x f_max + cuFFT/CTF chain "
                          "bytes at the measured HBM copy bandwidth (SURVEY 8(d))"}

    # §8(a) row a11: the volume query gem_render_volume at Dv = D on the trained model, timed
    # outside the step (CUDA events on the library's stream, 2 warm-up + 5 timed calls); its
    # algorithmic traffic is the 4 Dv^3 bytes of the volume written once
    vol = None
    if not args.no_volume:
        Dv = w.D
        vout = torch.empty((Dv, Dv, Dv), dtype=torch.float32, device=dev)
        for _ in range(2):
            sc.render_volume(tr.params, Dv, px, out=vout)
        vs = sc.stream
        ve0, ve1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        l0 = sc.launches
        sc.profile(True)
        ve0.record(vs)
        for _ in range(5):
            sc.render_volume(tr.params, Dv, px, out=vout)
        ve1.record(vs)
        torch.cuda.synchronize()
        sc.profile(False)
        vdev = sc.profile_read().get("volume", (0, 0.0))
        vms = vdev[1] / max(vdev[0], 1)   # device time per call (event pair around its launches)
        hbm = float(peaks.get("hbm_gbs", 6537.6))
        vol = {"Dv": Dv, "voxel_A": px, "ms": vms, "ms_per_call_with_host_sync": ve0.elapsed_time(ve1) / 5,
               "achieved_gbs": 4.0 * Dv ** 3 / (vms * 1e-3) / 1e9, "peak_gbs": hbm,
               "frac": 4.0 * Dv ** 3 / (vms * 1e-3) / 1e9 / hbm, "bound": "latency (the per-sub-brick record chain) + XU; frac is against the HBM floor of the 4 Dv^3 B write",
               "gpu_launches_per_call": (sc.launches - l0) / 5,
               "includes": "brick count, scan, brick-list fill, staging (sorted brick-local records, empty bricks zeroed) and the sub-brick render; the call's overflow "
                           "check (a 24 B D2H + stream sync) only in ms_per_call_with_host_sync"}
        del vout

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(w)
        except Exception as e:  # oracle build failure must not kill the bench line
            cpu = {"value": None, "unit": "particles/s", "cores": cpu_cores(), "kind": "oracle", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{w.name}: {SHAPES.get(w.name, 'synthetic')}, N={w.N} Gaussians, D={w.D}, px={w.px} A",
                   "model_state": args.state, "batch_per_gpu": B, "global_batch": B * world, "tile": args.tile,
                   "fused_waves": args.fused, "wave": int(st["wave"]), "zsort": args.zsort, "pixel_mask": args.pixel_mask, "tau": args.tau,
                   "exact_tiles": args.exact_tiles,
                   "ring_particles_per_gpu": ring, "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2: per-step working set (splat records "
                         f"{B * w.N * 32 / 1e6:.0f} MB + images) and a {ring}-particle ring "
                         f"({ring * w.D * w.D * 4 / 1e6:.0f} MB) exceed the 126 MB L2",
                   "useful_pairs_per_step": pairs, "list_entries_per_step": int(st["entries"]),
                   "list_capacity": int(st["capacity"]), "list_overflow": int(st["overflow"]),
                   "nonfinite": int(st["nonfinite"]), "degenerate_gaussians": int(st["degenerate"])},
        "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks,
        "memory": memory, "replicas_identical": replicas, "volume": vol,
        "kernels": kernels,
        "kernel_times": "CUDA event pair around each launch group, second pass over the same K steps",
    }
    print(json.dumps(line), flush=True)
    if st["overflow"] or st["nonfinite"]:
        # truncated tile lists (list capacity exceeded) or a non-finite loss: the step's outputs
        # are invalid (include/gem.h), so the run fails instead of reporting a number
        print(f"[bench] invalid run: list_overflow={st['overflow']} nonfinite={st['nonfinite']}", file=sys.stderr)
        return 3
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
