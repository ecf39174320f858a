"""Launch one instance of a named hot kernel for an `ncu --set full` capture.

    ncu --set full -k regex:fmha -c 1 -o out python tools/ncu_targets.py fmha_cogvideox
targets: fmha_cogvideox, fmha_xl, fmha_f32_s2, sched, gemm_s2_fc1, gemm_s2_fc2, gemm_xl_fc1,
gemm_xl_fc2, gemm_cog_fc1, unet
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_14741_b200 import _lib  # noqa: E402

lib = _lib.load(require_gpu=True)
t = sys.argv[1]
if t == "fmha_cogvideox":
    lib.ps_attn_probe(1, 17550, 30, 1920, 2, 1)
elif t == "fmha_f32_s2":  # fp32-path tcgen05 attention at the DiT-S/2 head set
    lib.ps_attn_probe(1, 256, 6, 384, 6, 1)
elif t == "fmha_xl":
    lib.ps_attn_probe(1, 256, 16, 1152, 2, 1)
elif t == "sched":
    import bench

    bench.sched_roofline(torch, 6550.7)
elif t == "gemm_s2_fc1":
    lib.ps_gemm_probe(256, 1536, 384, 0, 0, 1)
elif t == "gemm_s2_fc2":
    lib.ps_gemm_probe(256, 384, 1536, 0, 0, 1)
elif t == "gemm_xl_fc2":
    lib.ps_gemm_probe(256, 1152, 4608, 1, 0, 1)
elif t == "gemm_xl_fc1":
    lib.ps_gemm_probe(256, 4608, 1152, 1, 0, 1)
elif t == "gemm_cog_fc1":
    lib.ps_gemm_probe(17550, 7680, 1920, 1, 0, 1)
elif t == "unet":
    import bench
    from paper_2505_14741_b200.schedule import make_default_schedule

    cfg = dict(bench.CONFIGS["audioldm2_unet_bf16"], T=2, warmup=1)
    w = bench.build_predictor(cfg, max_batch=1)
    s = bench.make_sampler(w, make_default_schedule(2, "zero"), bench.run_cfg(cfg, w.data_dim, 1), 1)
    s.run(0)
torch.cuda.synchronize()
