"""Architecture tables for the DiT-shaped noise predictors (no compute here).

The reference predictor is a 2-D toy MLP (pkg/src/parastep/predictor.py:133-150);
BASELINE.json's configs name DiT-shaped predictors the reference never
defines. This file pins them once, shared by the CUDA product path
(``dit.py``) and the CPU oracle (``oracle/dit.py``), so both build the same
network from the same seed:

* conditioning is the timestep only (the reference omits the conditioning
  signal c, R/SPEC.md:8); the frequency embedding uses the reference's own
  ``time_embed`` convention (predictor.py:44-65) at width ``freq_dim``;
* weights use the reference's Xavier-uniform init convention
  (predictor.py:202-215): layer i draws fan_in*fan_out uniforms from stream
  (WEIGHT_INIT<<32)|i, W = (2u-1)*sqrt(6/(fan_in+fan_out)) reshaped
  (fan_in, fan_out) row-major, zero bias. ``layer_table`` fixes the order i.
  (No adaLN-Zero: zero-init gates would make every block the identity.)

Block (DiT, adaLN modulation from SiLU(c)):
    mod = SiLU(c) @ W_ada + b_ada -> shift1, scale1, gate1, shift2, scale2, gate2
    x += gate1 * (attn(LN(x) * (1 + scale1) + shift1) @ W_o + b_o)
    x += gate2 * (gelu_tanh((LN(x) * (1 + scale2) + shift2) @ W_1 + b_1) @ W_2 + b_2)
LN has no affine parameters, eps 1e-6. Final layer: adaLN shift/scale, LN,
linear to patch*patch*C. Patch vectors are ordered (c, ph, pw); tokens are
ordered (f, hp, wp) row-major.

Fixed sin-cos position embedding added after the patch projection:
    e1(d, pos)[k]       = sin(pos * w_k),  e1(d, pos)[d/2 + k] = cos(pos * w_k),
    w_k = 10000^(-k/(d/2)),  k < d/2
    F == 1:  [e1(D/2, hp), e1(D/2, wp)]
    F  > 1:  [e1(D/4, f), e1(3D/8, hp), e1(3D/8, wp)]

Text tokens and RoPE (the CogVideoX-shaped spec; ``text_tokens`` > 0 and
``rope``), following CogVideoX's transformer block structure:
    * the sequence is [text_tokens text rows | video tokens]; the text rows
      start from a fixed synthetic conditioning state drawn once per weight
      seed, txt = normal(seed, stream (7<<32)|0)[text_tokens * D] row-major
      (standing in for the T5 encoder output after CogVideoX's text
      projection), and run through every block with the video rows;
    * expert adaLN: b{i}.ada projects to 12D = [video shift1, scale1, gate1,
      shift2, scale2, gate2 | the same six for the text rows]; each row uses
      its own class's six vectors;
    * attention runs over all text + video rows; q and k of the video rows
      get 3D rotary embeddings (CogVideoX-5b's, interleaved pairs): head dims
      split into t / h / w bands of dh/4, 3dh/8, 3dh/8; pair i of band a with
      width d_a rotates by angle pos_a * 10000^(-2k/d_a) (k = i - band start):
          q'[2i]   = q[2i] cos - q[2i+1] sin,   q'[2i+1] = q[2i+1] cos + q[2i] sin;
      with RoPE there is no additive position embedding;
    * the final adaLN + linear run on the video rows only.

Latent layouts (the RNG counter is the flat index in this order, so the
layout must equal the flatten order the reference's 1-D vector uses):
    "CHW"  — C x H x W (F = 1), e.g. 4x32x32
    "FHWC" — F x H x W x C, channels-last, e.g. 13x60x90x16
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class DiTSpec:
    name: str
    channels: int
    frames: int
    height: int
    width: int
    layout: str  # "CHW" or "FHWC"
    patch: int
    hidden: int
    depth: int
    heads: int
    mlp_ratio: int = 4
    freq_dim: int = 256
    text_tokens: int = 0
    rope: bool = False

    @property
    def data_dim(self) -> int:
        return self.channels * self.frames * self.height * self.width

    @property
    def grid_h(self) -> int:
        return self.height // self.patch

    @property
    def grid_w(self) -> int:
        return self.width // self.patch

    @property
    def tokens(self) -> int:
        return self.frames * self.grid_h * self.grid_w

    @property
    def seq_len(self) -> int:
        """Rows per sample through the blocks: text tokens + video tokens."""
        return self.text_tokens + self.tokens

    @property
    def ada_width(self) -> int:
        """adaLN outputs per block: 6D, or 12D with text rows (expert adaLN)."""
        return (12 if self.text_tokens else 6) * self.hidden

    @property
    def patch_dim(self) -> int:
        return self.channels * self.patch * self.patch

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def mlp_hidden(self) -> int:
        return self.hidden * self.mlp_ratio

    def validate(self) -> None:
        if self.layout not in ("CHW", "FHWC"):
            raise ValueError(f"unknown latent layout {self.layout!r}")
        if self.layout == "CHW" and self.frames != 1:
            raise ValueError("CHW layout has a single frame")
        if self.height % self.patch or self.width % self.patch:
            raise ValueError("latent size must be a multiple of the patch")
        if self.hidden % self.heads:
            raise ValueError("hidden must divide into heads")
        if self.hidden % 4 or self.freq_dim % 2:
            raise ValueError("hidden must be a multiple of 4, freq_dim even")
        if self.rope and self.head_dim % 8:
            raise ValueError("RoPE needs head_dim % 8 == 0 (t/h/w bands of dh/4, 3dh/8)")

    def flops_per_forward(self) -> int:
        """2 x MACs of all GEMMs + attention (QK^T and PV), one sample."""
        L, D, Lv = self.seq_len, self.hidden, self.tokens
        per_block = L * D * (3 * D + D + 2 * self.mlp_hidden)
        gemm = Lv * self.patch_dim * D + self.depth * per_block + L * D * self.patch_dim
        attn = self.depth * 2 * L * L * D
        return 2 * (gemm + attn)


def layer_table(s: DiTSpec) -> list[tuple[str, int, int]]:
    """(name, fan_in, fan_out) in init-stream order."""
    D = s.hidden
    out = [("patch", s.patch_dim, D), ("temb1", s.freq_dim, D), ("temb2", D, D)]
    for i in range(s.depth):
        out += [
            (f"b{i}.ada", D, s.ada_width),
            (f"b{i}.qkv", D, 3 * D),
            (f"b{i}.proj", D, D),
            (f"b{i}.fc1", D, s.mlp_hidden),
            (f"b{i}.fc2", s.mlp_hidden, D),
        ]
    out += [("final.ada", D, 2 * D), ("final.out", D, s.patch_dim)]
    return out


SPECS = {
    # test-sized
    "dit_tiny": DiTSpec("dit_tiny", 4, 1, 8, 8, "CHW", 2, 64, 2, 2, freq_dim=32),
    "dit_tiny_video": DiTSpec("dit_tiny_video", 4, 3, 8, 12, "FHWC", 2, 96, 2, 3, freq_dim=32),
    # long sequence (1728 tokens): exercises the long-L attention kernel
    "dit_long_video": DiTSpec("dit_long_video", 4, 3, 48, 48, "FHWC", 2, 64, 1, 2, freq_dim=32),
    # BASELINE.json configs[0..1]: "small random-init DiT", latent 4x32x32
    "dit_s2": DiTSpec("dit_s2", 4, 1, 32, 32, "CHW", 2, 384, 12, 6),
    # configs[2]: DiT-XL/2-shaped
    "dit_xl2": DiTSpec("dit_xl2", 4, 1, 32, 32, "CHW", 2, 1152, 28, 16),
    # test-sized text + RoPE variant (the CogVideoX-shaped block structure)
    "dit_tiny_text": DiTSpec("dit_tiny_text", 4, 3, 8, 12, "FHWC", 2, 128, 2, 2, freq_dim=32,
                             text_tokens=10, rope=True),
    # configs[3]: CogVideoX-2b-shaped, latent 13x60x90x16 (channels-last):
    # 30 layers, hidden 1920, 30 heads of 64, 226 text tokens (CogVideoX's
    # max_text_seq_length) + 17,550 video tokens, expert adaLN, 3D RoPE
    "cogvideox_2b": DiTSpec("cogvideox_2b", 16, 13, 60, 90, "FHWC", 2, 1920, 30, 30,
                            text_tokens=226, rope=True),
}
