"""One eager denoise (no CUDA graph) for ncu launch lists / captures.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_denoise.py --config small_dit_fp32
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_14741_b200.schedule import make_default_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="small_dit_fp32")
ap.add_argument("--degree", type=int, default=1)
ap.add_argument("--strategy", default=None)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--steps", type=int, default=None, help="override T (fewer forwards under ncu)")
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
if a.steps:
    cfg["T"] = a.steps
    cfg["warmup"] = min(cfg["warmup"], a.steps - 1)
w = bench.build_predictor(cfg, max_batch=8)
sched = make_default_schedule(cfg["T"], cfg["sigma"])
rc = bench.run_cfg(cfg, w.data_dim, a.degree, a.strategy)
s = bench.make_sampler(w, sched, rc, 1)
for i in range(a.runs):
    s.run(i)
torch.cuda.synchronize()
print("launches per denoise:", s.launches)
