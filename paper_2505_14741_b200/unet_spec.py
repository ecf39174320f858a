"""Architecture and execution plan of the U-Net-shaped noise predictor
(BASELINE.json configs[4]: "AudioLDM2-large-shaped U-Net, mel latent 8x256x16").
No compute here: the CUDA executor (csrc/unet.cu) runs ``plan()``'s op list
and the CPU oracle (oracle/unet.py) interprets the same spec independently.

The reference predictor is an MLP (pkg/src/parastep/predictor.py:133-150)
and has no U-Net, so the network is pinned here, after the public
AudioLDM2 / diffusers UNet2DConditionModel layout, conditioned on the
timestep only (the reference omits the conditioning signal c, R/SPEC.md:8 —
so the cross-attention layers are absent, as in the DiT specs):

    emb    = SiLU(temb2(SiLU(temb1(time_embed(t, freq_dim)))))   (time_embed:
             the reference's interleaved sin/cos of absolute t, predictor.py:44-65)
    h      = conv_in(x)                      3x3, in_ch -> C0
    down l = 0..n-1:  layers x [ResBlock(C_l) (+ Transformer if attn[l])], then
                      (l < n-1) Downsample = 3x3 conv stride 2, pad 1
             every output above (and conv_in's) is pushed as a skip
    mid    = ResBlock, Transformer, ResBlock at C_{n-1}
    up   l = n-1..0:  (layers+1) x [ResBlock(concat(h, skip.pop()) -> C_l)
                      (+ Transformer if attn[l])], then (l > 0) Upsample =
                      nearest 2x + 3x3 conv
    eps    = conv_out(SiLU(GN(h)))           3x3, C0 -> in_ch

    ResBlock(x: Cin -> Cout):
        h   = conv3x3(SiLU(GN(x))) + temb_r(emb)          (emb already SiLU'd)
        h   = conv3x3(SiLU(GN(h)))
        out = (Cin == Cout ? x : conv1x1(x)) + h
    Transformer(h: C channels, tokens = H*W row-major):
        x   = proj_in(GN(h))                               (GroupNorm, no SiLU)
        depth x:  x += proj(attn(qkv(LN(x))));  x += fc2(gelu_tanh(fc1(LN(x))))
        out = h + proj_out(x)

GroupNorm: ``groups`` groups, eps 1e-5, no affine; Transformer's GN eps 1e-6;
LN: no affine, eps 1e-6; attention heads of ``head_dim`` 64 (the tcgen05
attention's width); MLP ratio 4; GELU tanh form. 3x3 convs pad 1; conv
weights are (fan_in = 9*Cin ordered (ky, kx, cin), fan_out = Cout), 1x1 and
linears (fan_in, fan_out), all drawn with the reference's Xavier-uniform
stream convention (predictor.py:202-215) in ``layer_table`` order, zero bias.
Latent layout: C x H x W (the reference's flat-vector order; the RNG counter
is the flat index), activations channels-last H x W x C on device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

# op kinds / operand producers (must match csrc/unet.cu)
OP_CONV, OP_LINEAR, OP_ATTN = 0, 1, 2
PRE_NONE, PRE_CONVERT, PRE_GN, PRE_GN_SILU, PRE_LN = 0, 1, 2, 3, 4
RS_NONE, RS_DOWN, RS_UP = 0, 1, 2
BUF_LATENT, BUF_EPS = -2, -3  # the forward's x input / eps output (CHW)


@dataclass(frozen=True)
class UNetSpec:
    name: str
    in_channels: int
    height: int
    width: int
    channels: tuple
    attn: tuple
    layers: int = 2
    depth: int = 1  # transformer layers per attention block
    head_dim: int = 64
    groups: int = 32
    mlp_ratio: int = 4

    @property
    def data_dim(self) -> int:
        return self.in_channels * self.height * self.width

    @property
    def freq_dim(self) -> int:
        return self.channels[0]

    @property
    def temb_dim(self) -> int:
        return 4 * self.channels[0]

    def validate(self) -> None:
        n = len(self.channels)
        if len(self.attn) != n:
            raise ValueError("attn flags must match the levels")
        if self.height % (1 << (n - 1)) or self.width % (1 << (n - 1)):
            raise ValueError("latent size must halve n-1 times")
        for c in self.channels:
            if c % self.groups or c % 8:
                raise ValueError("channels must be multiples of groups and of 8")
        for c, a in zip(self.channels, self.attn):
            if a and c % self.head_dim:
                raise ValueError("attention channels must be a multiple of head_dim")
        if self.in_channels % 8:
            raise ValueError("in_channels must be a multiple of 8 (tensor-core K)")


@dataclass
class Op:
    kind: int
    layer: int = -1          # index into layer_table (weights), -1 none
    pre: int = PRE_NONE      # A-operand producer
    in1: int = -1            # buffer ids (BUF_LATENT for conv_in)
    in2: int = -1            # concatenated second input (skip), -1 none
    c1: int = 0
    c2: int = 0
    h: int = 0               # input spatial size
    w: int = 0
    taps: int = 1            # 9 = 3x3 conv, 1 = 1x1 / linear
    resample: int = RS_NONE
    cout: int = 0
    temb_layer: int = -1     # this ResBlock's time projection layer
    temb_off: int = -1       # its column offset in the concatenated time table
    resid: int = -1          # buffer added in the epilogue
    out: int = -1            # output buffer id (BUF_EPS for conv_out)
    out_bf16: int = 0        # output written as bf16 (a later op's A operand)
    out2: int = -1           # bf16 shadow of an fp32 output (a later op's A operand), -1 none
    act: int = 0             # 1 = GELU-tanh epilogue
    heads: int = 0           # OP_ATTN
    eps: float = 1e-5        # GN / LN epsilon of the producer
    name: str = ""

    @property
    def out_hw(self) -> tuple[int, int]:
        if self.resample == RS_DOWN:
            return self.h // 2, self.w // 2
        if self.resample == RS_UP:
            return self.h * 2, self.w * 2
        return self.h, self.w


@dataclass
class Plan:
    spec: UNetSpec
    layers: list = field(default_factory=list)    # (name, fan_in, fan_out)
    ops: list = field(default_factory=list)
    bufs: list = field(default_factory=list)      # (elements per sample, is_bf16)
    temb_cols: int = 0                            # sum of the ResBlocks' Cout

    def buf(self, elems: int, bf16: bool = False) -> int:
        self.bufs.append((elems, bf16))
        return len(self.bufs) - 1

    def layer(self, name: str, fi: int, fo: int) -> int:
        self.layers.append((name, fi, fo))
        return len(self.layers) - 1

    def flops_per_forward(self) -> int:
        """2 x MACs of all convolutions / linears + attention (QK^T, PV), one sample."""
        f = 0
        for op in self.ops:
            if op.kind == OP_ATTN:
                L = op.h * op.w
                f += 2 * 2 * L * L * op.c1
            else:
                ho, wo = op.out_hw
                f += 2 * ho * wo * op.taps * (op.c1 + op.c2) * op.cout
        s = self.spec
        f += 2 * (s.freq_dim * s.temb_dim + s.temb_dim * s.temb_dim + s.temb_dim * self.temb_cols)
        return f


def plan(s: UNetSpec) -> Plan:
    """The op list in execution order; layer_table order == creation order."""
    s.validate()
    p = Plan(s)
    T = s.temb_dim
    p.layer("temb1", s.freq_dim, T)
    p.layer("temb2", T, T)
    H, W = s.height, s.width

    def resblock(name, x, cin, x2, cin2, cout, h, w):
        ctot = cin + cin2
        hw = h * w
        t = p.buf(hw * cout)
        toff = p.temb_cols
        p.temb_cols += cout
        l1 = p.layer(f"{name}.conv1", 9 * ctot, cout)
        lt = p.layer(f"{name}.temb", T, cout)
        p.ops.append(Op(OP_CONV, l1, PRE_GN_SILU, x, x2, cin, cin2, h, w, 9, RS_NONE, cout,
                        temb_layer=lt, temb_off=toff, out=t, name=f"{name}.conv1"))
        l2 = p.layer(f"{name}.conv2", 9 * cout, cout)
        o = p.buf(hw * cout)
        if ctot != cout:
            ls = p.layer(f"{name}.skip", ctot, cout)
            p.ops.append(Op(OP_LINEAR, ls, PRE_CONVERT, x, x2, cin, cin2, h, w, 1, RS_NONE, cout,
                            out=o, name=f"{name}.skip"))
            resid = o
        else:
            assert x2 == -1, "a concatenated input always changes the width"
            resid = x
        p.ops.append(Op(OP_CONV, l2, PRE_GN_SILU, t, -1, cout, 0, h, w, 9, RS_NONE, cout,
                        resid=resid, out=o, name=f"{name}.conv2"))
        return o

    def transformer(name, hbuf, c, h, w):
        hw = h * w
        x = p.buf(hw * c)
        lp = p.layer(f"{name}.proj_in", c, c)
        p.ops.append(Op(OP_LINEAR, lp, PRE_GN, hbuf, -1, c, 0, h, w, 1, RS_NONE, c, out=x,
                        eps=1e-6, name=f"{name}.proj_in"))
        qkv = p.buf(hw * 3 * c, bf16=True)
        ob = p.buf(hw * c, bf16=True)
        hid = p.buf(hw * s.mlp_ratio * c, bf16=True)
        xb = p.buf(hw * c, bf16=True)  # bf16 shadow of x after the last block: proj_out's A
        for d in range(s.depth):
            nd = f"{name}.t{d}"
            lq = p.layer(f"{nd}.qkv", c, 3 * c)
            lo = p.layer(f"{nd}.proj", c, c)
            l1 = p.layer(f"{nd}.fc1", c, s.mlp_ratio * c)
            l2 = p.layer(f"{nd}.fc2", s.mlp_ratio * c, c)
            p.ops.append(Op(OP_LINEAR, lq, PRE_LN, x, -1, c, 0, h, w, 1, RS_NONE, 3 * c, out=qkv,
                            out_bf16=1, eps=1e-6, name=f"{nd}.qkv"))
            p.ops.append(Op(OP_ATTN, -1, PRE_NONE, qkv, -1, c, 0, h, w, out=ob,
                            heads=c // s.head_dim, name=f"{nd}.attn"))
            p.ops.append(Op(OP_LINEAR, lo, PRE_NONE, ob, -1, c, 0, h, w, 1, RS_NONE, c, resid=x,
                            out=x, name=f"{nd}.proj"))
            p.ops.append(Op(OP_LINEAR, l1, PRE_LN, x, -1, c, 0, h, w, 1, RS_NONE,
                            s.mlp_ratio * c, out=hid, out_bf16=1, act=1, eps=1e-6,
                            name=f"{nd}.fc1"))
            p.ops.append(Op(OP_LINEAR, l2, PRE_NONE, hid, -1, s.mlp_ratio * c, 0, h, w, 1,
                            RS_NONE, c, resid=x, out=x, out2=xb if d == s.depth - 1 else -1,
                            name=f"{nd}.fc2"))
        o = p.buf(hw * c)
        lo = p.layer(f"{name}.proj_out", c, c)
        # A = the bf16 shadow the last fc2 epilogue wrote (same RN rounding as a
        # convert gather, one launch fewer)
        p.ops.append(Op(OP_LINEAR, lo, PRE_NONE, xb, -1, c, 0, h, w, 1, RS_NONE, c, resid=hbuf,
                        out=o, name=f"{name}.proj_out"))
        return o

    n = len(s.channels)
    c0 = s.channels[0]
    h0 = p.buf(H * W * c0)
    l = p.layer("conv_in", 9 * s.in_channels, c0)
    p.ops.append(Op(OP_CONV, l, PRE_CONVERT, BUF_LATENT, -1, s.in_channels, 0, H, W, 9, RS_NONE,
                    c0, out=h0, name="conv_in"))
    skips = [(h0, c0)]
    cur, cc, h, w = h0, c0, H, W
    for lv in range(n):
        co = s.channels[lv]
        for r in range(s.layers):
            cur = resblock(f"down{lv}.res{r}", cur, cc, -1, 0, co, h, w)
            cc = co
            if s.attn[lv]:
                cur = transformer(f"down{lv}.attn{r}", cur, cc, h, w)
            skips.append((cur, cc))
        if lv < n - 1:
            d = p.buf((h // 2) * (w // 2) * cc)
            ld = p.layer(f"down{lv}.downsample", 9 * cc, cc)
            p.ops.append(Op(OP_CONV, ld, PRE_CONVERT, cur, -1, cc, 0, h, w, 9, RS_DOWN, cc,
                            out=d, name=f"down{lv}.downsample"))
            cur, h, w = d, h // 2, w // 2
            skips.append((cur, cc))
    cur = resblock("mid.res0", cur, cc, -1, 0, cc, h, w)
    cur = transformer("mid.attn", cur, cc, h, w)
    cur = resblock("mid.res1", cur, cc, -1, 0, cc, h, w)
    for lv in reversed(range(n)):
        co = s.channels[lv]
        for r in range(s.layers + 1):
            sk, skc = skips.pop()
            cur = resblock(f"up{lv}.res{r}", cur, cc, sk, skc, co, h, w)
            cc = co
            if s.attn[lv]:
                cur = transformer(f"up{lv}.attn{r}", cur, cc, h, w)
        if lv > 0:
            u = p.buf(4 * h * w * cc)
            lu = p.layer(f"up{lv}.upsample", 9 * cc, cc)
            p.ops.append(Op(OP_CONV, lu, PRE_CONVERT, cur, -1, cc, 0, h, w, 9, RS_UP, cc, out=u,
                            name=f"up{lv}.upsample"))
            cur, h, w = u, 2 * h, 2 * w
    assert not skips
    l = p.layer("conv_out", 9 * cc, s.in_channels)
    p.ops.append(Op(OP_CONV, l, PRE_GN_SILU, cur, -1, cc, 0, h, w, 9, RS_NONE, s.in_channels,
                    out=BUF_EPS, name="conv_out"))
    return p


def layer_table(s: UNetSpec) -> list[tuple[str, int, int]]:
    return plan(s).layers


UNET_SPECS = {
    # test-sized: 2 levels, attention at level 1 (16 tokens), 2-channel groups
    "unet_tiny": UNetSpec("unet_tiny", 8, 16, 8, (32, 64), (False, True), layers=1,
                          groups=8),
    "unet_small": UNetSpec("unet_small", 8, 32, 16, (64, 128), (False, True), layers=2,
                           groups=16),
    # BASELINE.json configs[4]: AudioLDM2-large-shaped (public config widths
    # 128/256/384/640, 2 ResBlocks per level, attention below level 0, 2
    # transformer layers per attention block), mel latent 8 x 256 x 16
    "audioldm2_large": UNetSpec("audioldm2_large", 8, 256, 16, (128, 256, 384, 640),
                                (False, True, True, True), layers=2, depth=2),
}
