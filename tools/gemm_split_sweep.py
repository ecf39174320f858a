"""Split-K policy sweep: GEMM time (us) at the DiT/U-Net small-M shapes for
minimum K-blocks per split 4 / 2 / 1 (ps_gemm_tune).

    python tools/gemm_split_sweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
shapes = [(256, 16, 384), (256, 384, 384), (256, 1152, 384), (256, 1536, 384), (256, 384, 1536),
          (256, 1152, 1152), (256, 3456, 1152), (256, 4608, 1152), (256, 1152, 4608),
          (4096, 128, 1152), (1024, 256, 2304), (256, 384, 3456), (64, 640, 5760)]
mins = (4, 2, 1)
print(f"{'M':>5} {'N':>5} {'K':>5} prec " + " ".join(f"kb>={m:<3d}" for m in mins))
for M, N, K in shapes:
    for prec in (1, 0):
        r = []
        for m in mins:
            lib.ps_gemm_tune(m)
            r.append(lib.ps_gemm_probe(M, N, K, prec, 0, 30))
        lib.ps_gemm_tune(4)
        print(f"{M:5d} {N:5d} {K:5d} {'bf16' if prec else 'tf3x'} " +
              " ".join(f"{v:7.1f}" for v in r), flush=True)
