"""fp32-path attention at the DiT-S/2 shape: mma.sync key-split (impl 5) vs
tcgen05 3xTF32 (impl 6), mean device us of back-to-back launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
for L, H, D in ((256, 6, 384), (1728, 2, 64), (16, 2, 64)):
    for impl in (5, 6):
        lib.ps_attn_probe(1, L, H, D, impl, 3)
        us = lib.ps_attn_probe(1, L, H, D, impl, 200)
        print(f"L={L} H={H} D={D} impl={impl}: {us:.2f} us", flush=True)
