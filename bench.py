#!/usr/bin/env python
"""ParaStep denoise latency on B200 — the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

One "step" = one complete denoise (T reverse steps) of one synthetic latent
with the named predictor; at N GPUs it is ParaStep with degree N over NCCL
(N = 1: the sequential sampler, degree 1). ``value`` = mean denoise latency
(ms, device time from CUDA events, max over ranks), inputs resident in HBM;
L2 is flushed (a 512 MiB write) between timed iterations. ``e2e`` = the same
run through the public sampler API with x_T copied in from pinned host
memory and the full Trajectory (T x-records, T eps-records, x0) copied back
and materialised as numpy — the drop-in's user-visible latency.

Default workload (BASELINE.json configs[1]): small random-init DiT
(DiT-S/2-shaped, spec "dit_s2"), latent 4x32x32, 50 deterministic steps
("DDIM" -> the reference's sigma_mode="zero"), fp32 path (3xTF32 tcgen05
GEMMs), warm-up 5 for degree > 1.

``--impl reference`` times the reference's own CPU sampler (pkg/src/parastep,
installed in baseline/_ref; else the oracle port) driving the oracle DiT
through its import seam, on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1] (and configs[0]'s workload on the GPU)
    "small_dit_fp32": dict(spec="dit_s2", precision="fp32", T=50, sigma="zero", warmup=5,
                           baseline_config=1),
    # configs[2]
    "dit_xl2_bf16": dict(spec="dit_xl2", precision="bf16", T=50, sigma="zero", warmup=5,
                         baseline_config=2),
    # configs[3]: CogVideoX-2b-shaped 3D-attention DiT, latent 13x60x90x16, 17,550 tokens;
    # warm-up 13 is the paper's CogVideoX setting (R/PAPER.md:253)
    "cogvideox_bf16": dict(spec="cogvideox_2b", precision="bf16", T=50, sigma="zero", warmup=13,
                           baseline_config=3, max_batch=4),
    # configs[4]: AudioLDM2-large-shaped U-Net, mel latent 8x256x16, 200 steps;
    # warm-up 1 is the paper's AudioLDM2 setting (R/PAPER.md:253)
    "audioldm2_unet_bf16": dict(spec="audioldm2_large", family="unet", precision="bf16", T=200,
                                sigma="zero", warmup=1, baseline_config=4),
    # the reference's own MLP at data_dim 4096 (C1-ref), fp64
    "c1ref_mlp": dict(spec=None, precision="fp64", T=50, sigma="zero", warmup=5,
                      baseline_config=0),
}

L2_FLUSH_BYTES = 512 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ helpers
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


def build_predictor(cfg, max_batch):
    if cfg["spec"] is None:
        from paper_2505_14741_b200.predictor import TrainConfig, init_weights

        return init_weights(TrainConfig(data_dim=4096, hidden=(64, 64), embed_dim=16, seed=7))
    if cfg.get("family") == "unet":
        from paper_2505_14741_b200.unet import UNetWeights

        return UNetWeights(cfg["spec"], seed=0, max_batch=max_batch)
    from paper_2505_14741_b200.dit import DiTWeights

    return DiTWeights(cfg["spec"], seed=0, precision=cfg["precision"], max_batch=max_batch)


def run_cfg(cfg, n, degree, strategy=None):
    from paper_2505_14741_b200.engines import RunConfig

    if strategy is None:
        strategy = "sequential" if (degree == 1 and not USE_NCCL) else "parastep"
    return RunConfig(steps=cfg["T"], warmup=cfg["warmup"] if degree > 1 else 0,
                     strategy=strategy, degree=degree, seed=0, data_dim=n)


# ------------------------------------------------------------------ CPU reference
class _StopSample(Exception):
    pass


def reference_module():
    """The reference package: baseline/_ref (pip --target install) if present."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "parastep")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import parastep.engines as RE
        import parastep.protocol.worker as RW
        from parastep import commodel, schedule

        return "reference", RE, RW, schedule, commodel
    return "port", None, None, None, None


def cpu_predictor(cfg):
    from oracle import core
    from oracle.dit import DiT

    if cfg["spec"] is None:
        return core.MLP.init(4096, hidden=(64, 64), embed_dim=16, seed=7)
    if cfg.get("family") == "unet":
        from oracle.unet import UNet
        from paper_2505_14741_b200.unet_spec import UNET_SPECS

        return UNet(UNET_SPECS[cfg["spec"]], seed=0)
    from paper_2505_14741_b200.spec import SPECS

    return DiT(SPECS[cfg["spec"]], seed=0)


def cpu_reference_run(cfg, max_forwards=None, degree=1):
    """Run the reference's sampler on host cores (oracle predictor injected
    through its import seam, engines.py:40): sequential, or its ParaStep
    (Algorithm 1 emulation, engines.py:232-277) at degree > 1. Returns
    (elapsed_s, forwards_done, x0 or None, kind)."""
    import numpy as np

    kind, RE, RW, RS, _ = reference_module()
    pred = cpu_predictor(cfg)
    count = [0]

    def fwd(w, x, t, T):
        if max_forwards is not None and count[0] >= max_forwards:
            raise _StopSample()
        count[0] += 1
        return pred(np.asarray(x, dtype=np.float64), t, T)

    n = pred.data_dim
    if kind == "reference":
        class Shim:
            data_dim = n
            ballast = 1

        RE.forward = fwd
        RE.forward_batch = lambda w, xs, ts, T: [fwd(w, x, t, T) for x, t in zip(xs, ts)]
        RW.forward = fwd
        sched = RS.make_default_schedule(cfg["T"], cfg["sigma"])
        if degree > 1:
            rcfg = RE.RunConfig(steps=cfg["T"], warmup=cfg["warmup"], strategy="parastep",
                                degree=degree, seed=0, data_dim=n)
        else:
            rcfg = RE.RunConfig(steps=cfg["T"], seed=0, data_dim=n)
        t0 = time.perf_counter()
        try:
            x0 = RE.run_strategy(Shim(), sched, rcfg).x0
        except _StopSample:
            x0 = None
        return time.perf_counter() - t0, count[0], x0, kind
    from oracle import core, engines as oeng

    t0 = time.perf_counter()
    try:
        x0 = oeng.sequential(lambda x, t, T: fwd(None, x, t, T), core.Sched(cfg["T"], cfg["sigma"]),
                             n, 0)["x0"]
    except _StopSample:
        x0 = None
    return time.perf_counter() - t0, count[0], x0, kind


def call_count(T, warmup, p):
    """Busiest-device predictor calls: warmup + ceil((T-warmup)/p) (commodel.py:60-68)."""
    return warmup + -(-(T - warmup) // p)


def reference_loop_run(cfg, degree):
    """One complete run of the reference's own loop on host cores, the oracle
    predictor injected through its import seam (engines.py:40,
    protocol/worker.py:45): degree 1 -> run_strategy(sequential)
    (engines.py:196-205); degree p > 1 -> run_loopback (worker.py:244-285),
    p worker threads exchanging over the reference's in-process transport.
    Returns (seconds, per-rank timings or None, kind)."""
    import numpy as np

    kind, RE, RW, RS, _ = reference_module()
    pred = cpu_predictor(cfg)
    n = pred.data_dim

    def fwd(w, x, t, T):
        return pred(np.asarray(x, dtype=np.float64), t, T)

    if kind != "reference":  # the oracle port (baseline/_ref absent): sequential only
        from oracle import core, engines as oeng

        t0 = time.perf_counter()
        oeng.sequential(lambda x, t, T: fwd(None, x, t, T), core.Sched(cfg["T"], cfg["sigma"]),
                        n, 0)
        return time.perf_counter() - t0, None, kind

    class Shim:
        data_dim = n
        ballast = 1

    RE.forward = fwd
    RE.forward_batch = lambda w, xs, ts, T: [fwd(w, x, t, T) for x, t in zip(xs, ts)]
    RW.forward = fwd
    sched = RS.make_default_schedule(cfg["T"], cfg["sigma"])
    if degree == 1:
        rcfg = RE.RunConfig(steps=cfg["T"], seed=0, data_dim=n)
        t0 = time.perf_counter()
        RE.run_strategy(Shim(), sched, rcfg)
        return time.perf_counter() - t0, None, kind
    rcfg = RE.RunConfig(steps=cfg["T"], warmup=cfg["warmup"], strategy="parastep",
                        degree=degree, seed=0, data_dim=n)
    from threadpoolctl import threadpool_limits

    # p concurrent workers share the host cores: cores/p BLAS threads each (the
    # reference's bench pins its workers, bench.py:233-236)
    per = max(1, len(os.sched_getaffinity(0)) // degree)
    with threadpool_limits(limits=per):
        t0 = time.perf_counter()
        res = RW.run_loopback(Shim(), sched, rcfg)
        el = time.perf_counter() - t0
    tims = [{"forward_s": t.forward_s, "comm_s": t.comm_s, "recv_wait_s": t.recv_wait_s}
            for t in res.timings]
    return res.loop_latency_s or el, tims, kind


# configs whose full reference run fits a bench step (~5 s per DiT-S/2 denoise
# on 16 host cores); the larger ones time a sample of forwards and extrapolate
REF_FULL_RUN = ("small_dit_fp32", "c1ref_mlp")


def reference_arm(args, cfg, world, rank):
    if rank != 0:
        return
    ncores = len(os.sched_getaffinity(0))
    T, w = cfg["T"], cfg["warmup"] if world > 1 else 0
    calls = call_count(T, w, world)
    full = args.config in REF_FULL_RUN and args.ref_sample == 0
    times, tims = [], None
    kind = "port"
    for i in range(args.warmup + args.steps):
        if full:
            el, tims, kind = reference_loop_run(cfg, world)
            ms = el * 1e3
        else:
            sample = max(1, min(T, args.ref_sample or 3))
            el, done, _, kind = cpu_reference_run(cfg, max_forwards=sample)
            ms = el / done * calls * 1e3
        if i >= args.warmup:
            times.append(ms)
    val = statistics.mean(times)
    if full:
        what = ("run_strategy(sequential)" if world == 1 else
                f"run_loopback(parastep, degree {world}, warm-up {w}): {world} worker threads, "
                f"{max(1, ncores // world)} BLAS threads each")
        sample = (f"one complete {T}-step denoise per bench step through the reference's "
                  f"{what}; oracle DiT predictor (numpy f64) via the import seam")
    else:
        sample = (f"first {max(1, min(T, args.ref_sample or 3))} of {T} sampler steps of the "
                  f"reference's sequential loop per bench step, extrapolated x{calls} predictor "
                  f"calls (busiest device at degree {world}, commodel.call_count_per_device)")
    out = {
        "impl": "reference",
        "metric": f"denoise latency ({T} steps, degree {world})",
        "value": val, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": val, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded reference RNG)",
        "config": config_block(args, cfg, world),
        "cpu_baseline": {"value": val, "unit": "ms", "cores": ncores, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": val, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "samples_ms": times,
    }
    if tims:
        out["per_worker"] = tims
    print(json.dumps(out), flush=True)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def config_block(args, cfg, world):
    from paper_2505_14741_b200.spec import SPECS

    b = {"workload": args.config, "baseline_config_index": cfg["baseline_config"],
         "steps_T": cfg["T"], "sampler": f"DDPM posterior-mean, sigma_mode={cfg['sigma']} "
                                          "(the reference's deterministic 'DDIM' mode)",
         "degree": world, "warmup_steps": cfg["warmup"] if world > 1 else 0,
         "precision": cfg["precision"], "l2": "flushed (512 MiB write) between timed runs",
         "parallelism": f"parastep-d{world}" if world > 1 else "sequential (degree 1)"}
    if cfg.get("family") == "unet":
        from paper_2505_14741_b200.unet_spec import UNET_SPECS

        s = UNET_SPECS[cfg["spec"]]
        b.update({"predictor": cfg["spec"], "latent": f"{s.in_channels}x{s.height}x{s.width}",
                  "channels": list(s.channels), "attention_levels": list(s.attn),
                  "resblocks_per_level": s.layers, "transformer_depth": s.depth})
    elif cfg["spec"]:
        s = SPECS[cfg["spec"]]
        b.update({"predictor": cfg["spec"], "latent": f"{s.channels}x{s.height}x{s.width}"
                  if s.frames == 1 else f"{s.frames}x{s.height}x{s.width}x{s.channels}",
                  "hidden": s.hidden, "depth": s.depth, "heads": s.heads, "tokens": s.tokens,
                  "text_tokens": s.text_tokens, "rope": s.rope})
    else:
        b.update({"predictor": "reference MLP 4112-64-64-4096", "latent": "4x32x32"})
    return b


# ------------------------------------------------------------------ GPU arm
USE_NCCL = False  # set in main(): world > 1, or --force-nccl (1-rank NCCL path check)


EXCHANGE = {"want": "peer", "used": None}  # --exchange; what the NCCL-group runs used
SHARED_GPU = {"on": False}  # PS_BENCH_SHARED_GPU=1: N ranks on one GPU (code-path test)


def make_sampler(w, sched, rcfg, world, record=False, external_init=False):
    if world == 1 and not (USE_NCCL and rcfg.strategy == "parastep"):
        from paper_2505_14741_b200.engines import DeviceSampler

        return DeviceSampler(w, sched, rcfg, record=record, external_init=external_init)
    from paper_2505_14741_b200.protocol import NcclSampler

    if EXCHANGE["want"] == "peer":
        try:
            s = NcclSampler(w, sched, rcfg, record=record, external_init=external_init,
                            exchange="peer")
            EXCHANGE["used"] = "peer"
            return s
        except Exception as exc:  # IPC / P2P unavailable: the NCCL all-gather path
            log(f"peer exchange unavailable ({exc}); using the NCCL all-gather")
    EXCHANGE["used"] = "nccl"
    return NcclSampler(w, sched, rcfg, record=record, external_init=external_init)


def launches_of(s):
    return s.ops.launches if hasattr(s, "ops") else s.launches


def time_runs(sampler, K, W, flush, torch, dist, world, seed0=0):
    for i in range(W):
        sampler.run(seed0 + i, graph=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = []
    for i in range(K):
        flush.zero_()  # untimed: evict L2 between timed runs
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        sampler.run(seed0 + i, graph=True)
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    if world > 1:
        t = torch.tensor(ms, device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.tolist()
        dist.barrier()
    return ms


def gemm_roofline(w, cfg, torch, bf16_peak):
    """Dominant GEMM: of the block's four tcgen05 GEMMs (qkv, proj, fc1, fc2;
    one launch each per block) the one with the longest launch - the
    largest share of the step (profiles/r2_launches_*_by_grid.txt) - timed
    with CUDA events around back-to-back launches on the current stream."""
    if cfg["spec"] is None or cfg.get("family") == "unet":
        return None
    names = ("qkv", "proj", "fc1", "fc2")
    iters = 50
    times = {}
    for which in range(4):
        w.bench_gemm(which, 1, 3)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        w.bench_gemm(which, 1, iters)
        b.record()
        torch.cuda.synchronize()
        times[which] = a.elapsed_time(b) / iters * 1e-3
    which = max(times, key=times.get)
    M, N, K = w.gemm_shape(which, 1)
    t = times[which]
    flops = 2.0 * M * N * K
    if cfg["precision"] == "bf16":
        peak, note = bf16_peak, "measured bf16 dense (burst)"
    else:
        peak = bf16_peak / 2 / 3
        note = ("3xTF32: measured bf16 dense x 1/2 (tf32 rate) / 3 passes = fp32-accurate "
                "tensor peak")
    achieved = flops / t / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{cfg['spec']}_{cfg['precision']}_{names[which]}")
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": f"gemm_tc {names[which]} M={M} N={N} K={K} ({cfg['precision']})",
            "launch_us": t * 1e6, "peak_note": note,
            "block_gemm_launch_us": {names[i]: times[i] * 1e6 for i in range(4)}}


def attn_roofline(w, cfg, bf16_peak):
    """The tcgen05 attention kernel on one lane's full head set (device time of
    back-to-back launches, CUDA events inside ps_attn_probe)."""
    if cfg["spec"] is None or cfg.get("family") == "unet" or cfg["precision"] != "bf16":
        return None
    from paper_2505_14741_b200 import _lib

    s = w.spec
    L, H, D = s.seq_len, s.heads, s.hidden
    iters = 3 if L > 8192 else 50
    lib = _lib.load()
    lib.ps_attn_probe(1, L, H, D, 2, 1)
    us = lib.ps_attn_probe(1, L, H, D, 2, iters)
    flops = 4.0 * L * L * (D // H) * H
    achieved = flops / (us * 1e-6) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{cfg['spec']}_{cfg['precision']}_attn")
    return {"bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
            "frac": achieved / bf16_peak, "traffic": traffic,
            "kernel": f"fmha_tc L={L} heads={H} head_dim={D // H} (bf16)", "launch_us": us,
            "peak_note": "measured bf16 dense (burst); MUFU ex2 bounds head_dim 64 at ~1/2 of it"}


def dominant_is_attention(w, cfg):
    """Per-forward FLOPs: attention 4 L^2 D vs the block GEMMs 2 L (4 D^2 + 2 D F)."""
    if cfg["spec"] is None or cfg.get("family") == "unet":
        return False
    s = w.spec
    L, D = s.seq_len, s.hidden
    return 4.0 * L * L * D > 2.0 * L * (4 * D * D + 2 * D * s.mlp_hidden)


def sched_roofline(torch, hbm_peak):
    """The fused apply kernel on an HBM-sized vector (8 apply steps, fp32)."""
    from paper_2505_14741_b200 import _lib
    from paper_2505_14741_b200.schedule import make_default_schedule, step_coeffs

    lib = _lib.load()
    n = 1 << 26
    c = 8
    x = torch.randn(n, device="cuda")
    eps = torch.randn((c, n), device="cuda")
    seed = torch.zeros(1, dtype=torch.int64, device="cuda")
    sch = make_default_schedule(50, "zero")
    steps = _lib.step_array([step_coeffs(sch, t) for t in range(20, 20 - c, -1)])
    E = _lib.ptr_array([_lib.ptr(eps) + k * n * 4 for k in range(c)])
    R = _lib.ptr_array([0] * c)

    def go():
        _lib.check(lib.ps_sched_cycle(_lib.ptr(x), _lib.ptr(x), n, _lib.PS_F32, _lib.ptr(seed), c,
                                      steps, E, R, 0, 0, _lib.step_array([]), _lib.ptr_array([]),
                                      _lib.ptr_array([]), _lib.stream_ptr()), "cycle")

    go()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    iters = 10
    a.record()
    for _ in range(iters):
        go()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / iters * 1e-3
    bytes_ = (c + 2) * n * 4
    gbs = bytes_ / t / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": gbs / hbm_peak, "kernel": f"sched_cycle apply c={c} fp32 n=2^26 (zero mode)",
            "launch_us": t * 1e6}


# configs whose whole CPU reference denoise fits a bench run (~5 s DiT-S/2,
# ~50 s DiT-XL/2 on 16 host cores); the U-Net (~10 min) is sampled
CPU_FULL = ("small_dit_fp32", "c1ref_mlp", "dit_xl2_bf16")
# reference-sampler fixtures (tests/golden/make_golden_large.py) for the
# configs whose CPU trajectory does not fit a bench run
FIXTURES = {"dit_xl2_bf16": "dit_xl2_traj.npz", "audioldm2_unet_bf16": "unet_traj.npz",
            "cogvideox_bf16": "cogvideox_fwd.npz"}


def cpu_leg(args, cfg, w, sched, n, torch):
    """cpu_baseline: the reference's sequential sampler on the host cores,
    driving the oracle predictor (one complete denoise where CPU_FULL, else
    the first forwards extrapolated); the CogVideoX-shaped config times ONE
    full-shape oracle forward (~117 TFLOP, minutes) and extrapolates by the
    T calls. Returns (cpu dict, rel-MAE of our x0 vs the live CPU x0 or None)."""
    import numpy as np

    ncores = len(os.sched_getaffinity(0))
    if cfg["spec"] == "cogvideox_2b":
        # one full-shape forward is ~1 h of f64 numpy on 8 cores (the fixture's
        # run): time ONE block at the full sequence (17,776 rows) plus the
        # embeddings, and extrapolate by depth and the T calls
        import dataclasses

        from oracle.dit import DiT
        from paper_2505_14741_b200.spec import SPECS

        full = SPECS[cfg["spec"]]
        pred = DiT(dataclasses.replace(full, depth=1), seed=0)
        x = np.random.default_rng(0).standard_normal(pred.data_dim)
        t0 = time.perf_counter()
        pred(x, 37, cfg["T"])
        el = time.perf_counter() - t0
        return ({"value": el * full.depth * cfg["T"] * 1e3, "unit": "ms", "cores": ncores,
                 "kind": "port", "cpu_model": cpu_model(),
                 "sample": f"one block of the oracle predictor at the full 17,776-row sequence "
                           f"(numpy f64, {el:.0f} s incl. embeddings), extrapolated "
                           f"x{full.depth} blocks x{cfg['T']} calls; sampler steps omitted"},
                None)
    full = args.config in CPU_FULL
    el, done, x0_ref, kind = cpu_reference_run(
        cfg, max_forwards=None if full else (args.ref_sample or 3))
    cpu = {"value": el / done * cfg["T"] * 1e3, "unit": "ms", "cores": ncores, "kind": kind,
           "cpu_model": cpu_model(),
           "sample": (f"one full {cfg['T']}-step sequential denoise (seed 0)" if full else
                      f"first {done} of {cfg['T']} steps, extrapolated x{cfg['T']}")}
    rel = None
    if x0_ref is not None:
        seq = make_sampler(w, sched, run_cfg(cfg, n, 1), 1, record=False)
        seq.run(0)
        torch.cuda.synchronize()
        from paper_2505_14741_b200.numerics import rel_mae

        rel = rel_mae(x0_ref, seq.x0_device.double().cpu().numpy())
    return cpu, rel


def fixture_rel(args, cfg, w, sampler, world, rank, torch, extra):
    """rel-MAE (Eq. 7) of our seed-0 result against the reference sampler's
    fixture for this config: x0 of the same strategy and degree, or (the
    CogVideoX-shaped config, whose CPU trajectory takes hours) one forward's
    eps at t = 37 on the reference's x_T. None if no fixture applies."""
    import numpy as np

    name = FIXTURES.get(args.config)
    if name is None:
        return None
    path = os.path.join(ROOT, "tests", "golden", name)
    if not os.path.exists(path):
        return None
    g = np.load(path)
    from paper_2505_14741_b200.numerics import rel_mae

    if "eps" in g.files:  # per-forward fixture
        if rank != 0:
            return None
        from paper_2505_14741_b200 import predictor as P
        from paper_2505_14741_b200.engines import RunConfig, initial_state

        x = initial_state(RunConfig(steps=int(g["T"]), seed=int(g["seed"]), data_dim=w.data_dim))
        eps = P.forward(w, x, int(g["t"]), int(g["T"]))
        extra["rel_mae_source"] = (f"one full-shape forward (t={int(g['t'])}) vs the oracle "
                                   f"predictor's eps on the reference's x_T (tests/golden/{name}); "
                                   "a CPU 50-step trajectory at this shape takes hours")
        return rel_mae(g["eps"].astype(np.float64), eps)
    tag = "seq" if world == 1 else f"ps{world}"
    if f"{tag}_x0" not in g.files:
        return None
    sampler.run(0, graph=True)
    torch.cuda.synchronize()
    x0 = (sampler.x0_device if hasattr(sampler, "x0_device") else sampler.ops.x)
    x0 = x0.double().cpu().numpy()
    extra["rel_mae_source"] = (f"x0 (seed 0) vs the reference sampler's {tag} trajectory "
                               f"(tests/golden/{name})")
    if f"{tag}_vs_seq_rel_mae" in g.files:
        extra["reference_parastep_vs_sequential_rel_mae"] = float(g[f"{tag}_vs_seq_rel_mae"])
    return rel_mae(g[f"{tag}_x0"], x0) if rank == 0 else None


def multi_gpu_report(w, sched, cfg, n, world, rank, value, flush, torch, dist):
    """N > 1: the reference bench's comparison row (bench.py:216-255) on this
    box: the sequential (degree-1) latency on rank 0's GPU, the speed-up, the
    call-count bound T / (w + ceil((T-w)/d)) and the Amdahl bound
    (commodel.py:51-68), and every rank's device-clock split of one run into
    forward / exchange wait / apply (worker.py:65-85, RankTimings) plus the
    measured exchange ledger."""
    from paper_2505_14741_b200.protocol import NcclSampler

    T, wu = cfg["T"], cfg["warmup"]
    rep = {}
    # per-rank phase split: one eager run with device-clock stamps
    ts = NcclSampler(w, sched, run_cfg(cfg, n, world), record=False,
                     exchange=EXCHANGE["used"] or "nccl", timed=True)
    for _ in range(2):
        dist.barrier()
        ts.run(0)
        res = ts.result()
    census = ts.traffic_census()
    rep["per_rank"] = [{"rank": r, "loop_ms": t.loop_s * 1e3, "forward_ms": t.forward_s * 1e3,
                        "exchange_wait_ms": t.exchange_wait_s * 1e3, "apply_ms": t.apply_s * 1e3}
                       for r, t in enumerate(res.timings)]
    rep["per_rank_note"] = ("one eager (not graph-replayed) run with %globaltimer stamps between "
                            "phases; loop_ms includes host launch gaps the timed graph runs omit")
    rep["exchange_ledger"] = {"rounds": census["rounds"], "sent_bytes": census["sent"],
                              "received_bytes": census["received"],
                              "verified": census["ok"]}
    if hasattr(ts.ops, "px") and ts.ops.px is not None:
        dist.barrier()
        ts.ops.px.close()
    dist.barrier()
    seq = None
    if rank == 0:
        from paper_2505_14741_b200.engines import DeviceSampler, RunConfig

        scfg = RunConfig(steps=T, warmup=0, strategy="sequential", degree=1, seed=0, data_dim=n)
        ss = DeviceSampler(w, sched, scfg)
        ss.run(0, graph=True)
        seq = statistics.mean(time_runs(ss, 3, 2, flush, torch, dist, 1))
    dist.barrier()
    calls = call_count(T, wu, world)
    m = wu / T
    rep.update({
        "sequential_ms": seq,
        "speedup_vs_sequential": (seq / value) if seq else None,
        "call_count_per_device": calls,
        "speedup_bound_callcount": T / calls,
        "speedup_bound_amdahl": 1.0 / (m + (1.0 - m) / world),
    })
    return rep


def our_arm(args, cfg, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_14741_b200.schedule import make_default_schedule

    torch.cuda.set_device(local)
    hbm_peak, bf16_peak, peak_src = measured_peaks()
    w = build_predictor(cfg, max_batch=cfg.get("max_batch", 8))
    n = w.data_dim
    sched = make_default_schedule(cfg["T"], cfg["sigma"])
    rcfg = run_cfg(cfg, n, world)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    sampler = make_sampler(w, sched, rcfg, world)
    clocks = ClockSampler(local)
    sampler.run(0, graph=True)  # capture
    torch.cuda.synchronize()
    with clocks:
        ms = time_runs(sampler, args.steps, args.warmup, flush, torch, dist, world)
    launches = launches_of(sampler)
    value = statistics.mean(ms)

    # e2e through the public API: host x_T in (pinned), full Trajectory out
    es = 8 if w.state_dtype_code == 0 else 4
    x_host = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(
        torch.float64 if es == 8 else torch.float32).pin_memory()
    e2s = make_sampler(w, sched, rcfg, world, record=True, external_init=True)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2s.run(i, graph=True, x_init=x_host)
        if hasattr(e2s, "trajectory"):
            tr = e2s.trajectory()
            assert tr.steps == cfg["T"]
        else:
            res = e2s.result()  # rank 0: full Trajectory; others: x0
            assert res.x0.shape[0] == n
        dt = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            e2e_ms.append(dt)
    if world > 1:
        t = torch.tensor(e2e_ms, device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.tolist()
    e2e = statistics.mean(e2e_ms)
    d2h = ((2 * cfg["T"] + 1) * n * es) if rank == 0 else n * es

    roof = gemm_roofline(w, cfg, torch, bf16_peak) if rank == 0 else None
    roof_attn = attn_roofline(w, cfg, bf16_peak) if rank == 0 else None
    if roof_attn is not None and dominant_is_attention(w, cfg):
        roof, roof_attn = roof_attn, roof  # the attention kernel dominates the step
    roof_sched = sched_roofline(torch, hbm_peak) if rank == 0 else None

    extra = {}
    cpu = None
    rel = None
    if rank == 0 and world == 1:
        # single-GPU BatchStep (lanes batched into one forward): the paper's s=2/4/8
        for d in [d for d in args.batchstep if d <= cfg.get("max_batch", 8)]:
            bs = make_sampler(w, sched, run_cfg(cfg, n, d, "batchstep"), 1)
            bs.run(0, graph=True)
            bms = time_runs(bs, max(2, args.steps // 2), 1, flush, torch, dist, 1)
            extra[f"batchstep_d{d}_ms"] = statistics.mean(bms)
            extra[f"batchstep_d{d}_speedup"] = value / statistics.mean(bms)
            extra[f"batchstep_d{d}_bound_callcount"] = cfg["T"] / call_count(cfg["T"],
                                                                            cfg["warmup"], d)
        if not args.no_cpu_baseline:
            cpu, rel = cpu_leg(args, cfg, w, sched, n, torch)
    if rel is None and world > 1 and args.config in CPU_FULL and not args.no_cpu_baseline:
        # degree-d parity: the reference's own ParaStep (Algorithm 1) on rank 0's
        # host cores vs this run's x0 (seed 0, identical on every rank)
        sampler.run(0, graph=True)
        torch.cuda.synchronize()
        if rank == 0 and reference_module()[0] == "reference":
            from paper_2505_14741_b200.numerics import rel_mae

            _, _, x0_ref, _ = cpu_reference_run(cfg, degree=world)
            rel = rel_mae(x0_ref, sampler.ops.x.double().cpu().numpy())
            extra["rel_mae_source"] = (f"x0 (seed 0) vs the reference's ParaStep emulation at "
                                       f"degree {world} on host cores (run live)")
        dist.barrier()
    if rel is None:
        rel = fixture_rel(args, cfg, w, sampler, world, rank, torch, extra)
    if world > 1:
        extra.update(multi_gpu_report(w, sched, cfg, n, world, rank, value, flush, torch, dist))
    if rank != 0:
        return
    out = {
        "metric": f"denoise latency ({cfg['T']} steps, degree {world})",
        "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": {"fp32": "f32", "bf16": "bf16", "fp64": "f64"}[cfg["precision"]],
        "data": "synthetic: seeded reference-RNG latent, random-init weights (Xavier, ref. "
                "convention)",
        "config": config_block(args, cfg, world),
        "clocks": clocks.summary(),
        "e2e": {"value": e2e, "unit": "ms", "h2d_bytes_per_step": n * es,
                "d2h_bytes_per_step": d2h,
                "api": "DeviceSampler.sample path: x_T from pinned host, Trajectory to numpy"},
        "gpu_launches": launches * args.steps,
        "launches_per_denoise": launches,
        "roofline": roof,
        "roofline_sched": roof_sched,
        "roofline_other": roof_attn,
        "peaks_source": peak_src,
        "cpu_baseline": cpu,
        "rel_mae_vs_reference": rel,
        "samples_ms": ms,
    }
    out.update(extra)
    if SHARED_GPU["on"]:
        out["shared_gpu_test"] = ("all ranks on cuda:0 (PS_BENCH_SHARED_GPU=1): exercises the "
                                  "multi-rank code path; not a multi-GPU measurement")
    if USE_NCCL:
        out["config"]["exchange"] = {
            "peer": "peer memory: CUDA-IPC-mapped lane eps read over NVLink by the fused "
                    "apply kernel, release/acquire flags (csrc/peer.cu)",
            "nccl": "NCCL all_gather_into_tensor"}.get(EXCHANGE["used"], EXCHANGE["used"])
    print(json.dumps(out), flush=True)


def free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """``--gpus N > 1`` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run ourselves; the rank-0 JSON line passes through."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"error: --gpus {args.gpus} needs {args.gpus} CUDA devices, {have} visible")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log("spawning: " + " ".join(cmd))
    return subprocess.call(cmd, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="small_dit_fp32", choices=sorted(CONFIGS))
    ap.add_argument("--batchstep", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="reference arm: 0 = one complete run per bench step where it fits "
                         "(DiT-S/2, C1-ref MLP); else sampler steps timed and extrapolated")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=("peer", "nccl"), default="peer",
                    help="multi-GPU eps exchange: CUDA-IPC peer memory read by the fused apply "
                         "kernel (default), or the NCCL all-gather")
    ap.add_argument("--force-nccl", action="store_true",
                    help="run the NCCL rank loop even at one rank (path check under torchrun)")
    args = ap.parse_args()
    under_torchrun = "WORLD_SIZE" in os.environ
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        # the CPU arm runs on rank 0 only; without torchrun it runs in this
        # process at degree --gpus
        world, rank, local = dist_setup()
        if not under_torchrun:
            world = args.gpus
        reference_arm(args, cfg, world, rank)
        return 0
    if args.gpus > 1 and not under_torchrun:
        return spawn_ranks(args)
    world, rank, local = dist_setup()
    if world != args.gpus:
        log(f"error: --gpus {args.gpus} but WORLD_SIZE {world}")
        return 2
    global USE_NCCL
    USE_NCCL = world > 1 or args.force_nccl
    EXCHANGE["want"] = args.exchange
    if USE_NCCL:
        import torch
        import torch.distributed as dist

        if world > torch.cuda.device_count():
            if os.environ.get("PS_BENCH_SHARED_GPU") != "1":
                log(f"error: {world} ranks but {torch.cuda.device_count()} CUDA devices: "
                    "one rank per GPU is required")
                return 2
            # code-path test only (tests/test_gpu_bench_multi.py): every rank on
            # cuda:0, gloo bootstrap, peer exchange; the timings are not a
            # multi-GPU measurement and the line says so
            SHARED_GPU["on"] = True
            EXCHANGE["want"] = "peer"
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        our_arm(args, cfg, world, rank, local)
    finally:
        if USE_NCCL:
            import torch.distributed as dist

            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
