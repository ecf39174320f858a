"""fp32-path (3xTF32 mma.sync) short-sequence attention timing vs key-split
warps (PS_ATTN_KS_WARPS), plus accuracy against torch fp64.

    PS_ATTN_KS_WARPS=8 python tools/attn_fp32_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
kw = os.environ.get("PS_ATTN_KS_WARPS", "default")
for name, B, L, H, D in [("dit_s2 fp32", 1, 256, 6, 384), ("dit_s2 x8", 8, 256, 6, 384),
                         ("dit_xl2 fp32", 1, 256, 16, 1152)]:
    us = lib.ps_attn_probe(B, L, H, D, 5, 50)
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn((B * L, 3 * D), device="cuda", generator=g)
    out = torch.zeros((B * L, D), device="cuda")
    _lib.check(lib.ps_attn_test(_lib.ptr(qkv), _lib.ptr(out), B, L, H, D, 5, _lib.stream_ptr()), "t")
    dh = D // H
    x = qkv.double().view(B, L, 3, H, dh)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    ref = torch.softmax(q @ k.transpose(-1, -2) / dh ** 0.5, -1) @ v
    ref = ref.permute(0, 2, 1, 3).reshape(B * L, D)
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    print(f"kw={kw:8s} {name:14s} {us:7.2f} us  max rel err {err:.2e}", flush=True)
