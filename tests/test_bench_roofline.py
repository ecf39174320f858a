"""bench.py reports the roofline of the step's dominant kernel: the attention
kernel where attention FLOPs exceed the block GEMMs' (CogVideoX-shaped), the
fc1 GEMM otherwise (DiT-S/2, DiT-XL/2). CPU-only: shape arithmetic."""
import os
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2505_14741_b200.spec import SPECS  # noqa: E402


def _dominant(spec_name, family=None):
    cfg = {"spec": spec_name}
    if family:
        cfg["family"] = family
    w = SimpleNamespace(spec=SPECS[spec_name]) if spec_name in SPECS else None
    return bench.dominant_is_attention(w, cfg)


def test_attention_dominates_cogvideox_shape():
    assert _dominant("cogvideox_2b")


def test_gemm_dominates_dit_shapes():
    assert not _dominant("dit_s2")
    assert not _dominant("dit_xl2")


def test_no_attention_roofline_without_spec_or_for_unet():
    assert not bench.dominant_is_attention(None, {"spec": None})
    assert not bench.dominant_is_attention(None, {"spec": "audioldm2_large", "family": "unet"})
