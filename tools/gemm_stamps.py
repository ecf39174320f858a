"""Per-phase timeline (us, clock64 / SM clock) of one tcgen05 GEMM CTA.

    python tools/gemm_stamps.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
MHZ = 1965.0
PH = ["prologue", "pdl_wait", "->tma0", "->stage0", "->stageN", "->accum", "epilogue", "exit",
      "sk:part", "sk:sync1", "sk:reduce"]
shapes = [(256, 16, 384), (256, 384, 384), (256, 1152, 384), (256, 1536, 384), (256, 384, 1536),
          (256, 1152, 1152), (256, 4608, 1152), (256, 1152, 4608), (4096, 128, 1152),
          (1024, 256, 2304)]
print(f"{'M':>5} {'N':>5} {'K':>5} prec {'us':>6} " + " ".join(f"{p:>8s}" for p in PH))
for M, N, K in shapes:
    for prec in (1, 0):
        us = lib.ps_gemm_probe(M, N, K, prec, 16, 3)
        st = (C.c_longlong * 12)()
        lib.ps_gemm_stamps(st)
        d = [(st[i + 1] - st[i]) / MHZ for i in range(8)]
        # split-K epilogue: accum -> partials written -> sync -> reduced
        d += [(st[9] - st[6]) / MHZ, (st[10] - st[9]) / MHZ, (st[11] - st[10]) / MHZ] \
            if st[9] > st[6] else [0.0, 0.0, 0.0]
        print(f"{M:5d} {N:5d} {K:5d} {'bf16' if prec else 'tf3x'} {us:6.1f} " +
              " ".join(f"{v:8.2f}" for v in d), flush=True)
