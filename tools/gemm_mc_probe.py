"""tcgen05 GEMM time (us, back-to-back launches) with the A tile multicast
across 4 / 2 / 1 N-tile CTAs of a cluster.

    python tools/gemm_mc_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
shapes = [(256, 384, 384), (256, 1152, 384), (256, 1536, 384), (256, 384, 1536),
          (256, 1152, 1152), (256, 3456, 1152), (256, 4608, 1152), (256, 1152, 4608),
          (2048, 4608, 1152), (2048, 1152, 4608), (4096, 128, 1152), (1024, 256, 2304),
          (17550, 7680, 1920), (17550, 1920, 7680)]
print(f"{'M':>6} {'N':>5} {'K':>5} prec   mc4    mc2    mc1  TF/s(best)")
for M, N, K in shapes:
    for prec in (1, 0):
        if M > 4096 and prec == 0:
            continue
        it = 5 if M > 4096 else 30
        r = [lib.ps_gemm_probe(M, N, K, prec, d, it) for d in (512, 256, 0)]
        tf = 2 * M * N * K / (min(r) * 1e-6) / 1e12
        print(f"{M:6d} {N:5d} {K:5d} {'bf16' if prec else 'tf3x'} " +
              " ".join(f"{v:6.1f}" for v in r) + f"  {tf:7.1f}", flush=True)
