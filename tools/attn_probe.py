"""Attention kernel timing (device us of back-to-back launches, zero operands).

    python tools/attn_probe.py            # CogVideoX-shaped and DiT-shaped heads
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
SHAPES = [("cogvideox_2b", 1, 17550, 30, 1920), ("dit_s2 bf16 L=256", 1, 256, 6, 384),
          ("dit_xl2 L=256 dh=72", 1, 256, 16, 1152), ("dit_xl2 x8 lanes", 8, 256, 16, 1152),
          ("L=4096 H=16", 1, 4096, 16, 1024), ("L=8192 H=8", 2, 8192, 8, 512)]
print(f"{'shape':24s} {'impl':>4s} {'us':>10s} {'TFLOP/s':>8s}")
for name, B, L, H, D in SHAPES:
    flops = 4.0 * B * L * L * D
    for impl in (1, 3, 4):  # mma.sync, tcgen05 with 1 / 2 query tiles per CTA
        iters = 3 if L > 10000 else 20
        us = lib.ps_attn_probe(B, L, H, D, impl, iters)
        tf = flops / (us * 1e-6) / 1e12 if us > 0 else float("nan")
        print(f"{name:24s} {impl:4d} {us:10.1f} {tf:8.1f}", flush=True)
