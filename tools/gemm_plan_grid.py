"""Calibration grid: GEMM time (us) for every (BN, split-K) at the small-M
shapes, next to the planner's own choice.

    python tools/gemm_plan_grid.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
shapes = [(0, 256, 1152, 384), (0, 256, 384, 384), (0, 256, 1536, 384), (0, 256, 384, 1536),
          (0, 256, 16, 384), (1, 256, 3456, 1152), (1, 256, 1152, 1152), (1, 256, 4608, 1152),
          (1, 256, 1152, 4608), (1, 4096, 128, 1152), (1, 1024, 256, 2304), (1, 4096, 256, 1152),
          (1, 1024, 768, 256)]
combos = [(bn, s) for bn in (32, 64, 128) for s in (1, 2, 4, 8)]
print("prec M N K auto | " + " ".join(f"{bn}/{s}" for bn, s in combos))
for prec, M, N, K in shapes:
    lib.ps_gemm_force(0, 0)
    auto = lib.ps_gemm_probe(M, N, K, prec, 0, 20)
    r = []
    for bn, s in combos:
        tiles = ((M + 127) // 128) * ((N + bn - 1) // bn)
        nk = (K + (63 if prec else 31)) // (64 if prec else 32)
        if tiles * s > (148 if s <= 2 else 128) or nk < s or (prec == 0 and bn == 128 and s == 1 and False):
            r.append("   -  ")
            continue
        lib.ps_gemm_force(bn, s)
        r.append(f"{lib.ps_gemm_probe(M, N, K, prec, 0, 20):6.1f}")
    lib.ps_gemm_force(0, 0)
    print(f"{'bf16' if prec else 'tf3x'} {M} {N} {K} {auto:6.1f} | " + " ".join(r), flush=True)
