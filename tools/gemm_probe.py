"""Pipeline-isolation probe of the tcgen05 GEMM (ps_gemm_probe).

columns: full kernel | no MMA | no TMA | neither | neither + no stores |
empty kernel (same launch config) | full without cluster split-K."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
shapes = [(256, 4608, 1152), (256, 1152, 1152), (256, 1152, 4608), (256, 3456, 1152),
          (256, 1536, 384), (256, 384, 384), (256, 384, 1536), (256, 1152, 384),
          (2048, 4608, 1152), (8192, 8192, 8192)]
dbgs = (0, 1, 2, 3, 7, 8, 32, 64)
print(f"{'M':>6} {'N':>6} {'K':>6} prec   full  noMMA  noTMA   none nostor  empty nosplit incta"
      "  TF/s(full)")
for M, N, K in shapes:
    for prec in (1, 0):
        if M * N * K > 8192 ** 3 // 2 and prec == 0:
            continue
        r = [lib.ps_gemm_probe(M, N, K, prec, d, 20) for d in dbgs]
        tf = 2 * M * N * K / (r[0] * 1e-6) / 1e12
        print(f"{M:6d} {N:6d} {K:6d} {'bf16' if prec else 'tf3x'} " +
              " ".join(f"{v:6.1f}" for v in r) + f"  {tf:7.1f}")
