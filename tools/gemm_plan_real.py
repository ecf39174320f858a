"""Block-GEMM time (us, back-to-back launches with CUDA events, real weights
and epilogue-free store) of the DiT-S/2 fp32 layers for forced (BN, split-K)
plans vs the planner's own choice.

    python tools/gemm_plan_real.py [spec] [precision]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_14741_b200 import _lib  # noqa: E402
from paper_2505_14741_b200.dit import DiTWeights  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "dit_s2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
lib = _lib.load(require_gpu=True)
names = ("qkv", "proj", "fc1", "fc2")


def times(w):
    out = []
    for which in range(4):
        w.bench_gemm(which, 1, 5)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        w.bench_gemm(which, 1, 100)
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 10.0)
    return out


print("plan      " + "  ".join(f"{n:>6s}" for n in names))
lib.ps_gemm_force(0, 0)
w = DiTWeights(spec, seed=0, precision=prec, max_batch=1)
print("auto      " + "  ".join(f"{t:6.2f}" for t in times(w)), flush=True)
del w
for bn in (32, 64, 128):
    for s in (1, 2, 4, 8):
        lib.ps_gemm_force(bn, s)
        try:
            w = DiTWeights(spec, seed=0, precision=prec, max_batch=1)
            print(f"{bn:3d}/{s:<5d} " + "  ".join(f"{t:6.2f}" for t in times(w)), flush=True)
            del w
        except Exception as exc:  # plan not launchable at this shape
            print(f"{bn:3d}/{s:<5d} - ({str(exc)[:60]})", flush=True)
lib.ps_gemm_force(0, 0)
