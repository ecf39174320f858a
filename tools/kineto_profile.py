"""Per-kernel device time inside the real (CUDA-graph, PDL) denoise, via the
CUPTI activity trace torch.profiler records (no serialisation, unlike ncu).

    python tools/kineto_profile.py --config small_dit_fp32 [--steps 10] [--graph]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2505_14741_b200.schedule import make_default_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="small_dit_fp32")
ap.add_argument("--degree", type=int, default=1)
ap.add_argument("--strategy", default=None)
ap.add_argument("--steps", type=int, default=None)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--trace", default=None)
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
if a.steps:
    cfg["T"] = a.steps
    cfg["warmup"] = min(cfg["warmup"], a.steps - 1)
w = bench.build_predictor(cfg, max_batch=8)
sched = make_default_schedule(cfg["T"], cfg["sigma"])
rc = bench.run_cfg(cfg, w.data_dim, a.degree, a.strategy)
s = bench.make_sampler(w, sched, rc, 1)
s.run(0, graph=a.graph)
s.run(0, graph=a.graph)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.run(1, graph=a.graph)
    torch.cuda.synchronize()
if a.trace:
    prof.export_chrome_trace(a.trace)
tot, cnt = collections.defaultdict(float), collections.Counter()
first, last = None, None
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    name = ev.name.split("(")[0][:60]
    tot[name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    cnt[name] += 1
T = sum(tot.values())
print(f"config {a.config} T={cfg['T']} graph={a.graph}: kernel time sum {T/1e3:.3f} ms")
print(f"{'kernel':60s} {'n':>6s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{k:60s} {cnt[k]:6d} {v:10.1f} {100*v/T:5.1f}% {v/cnt[k]:8.2f}")
