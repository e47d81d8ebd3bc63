"""The consistency-distilled UNet Phi (kind ``"unet"``) on tcgen05/TMEM kernels.

No reference implementation exists: the reference package
ships analytic stand-ins only.  This module defines the build's network --
an EDM2-style magnitude-preserving UNet with the
sCM/consistency preconditioning -- and runs it as a sequence of NHWC bf16
implicit-GEMM convolutions (``ig_conv_tc``: TMA -> SMEM -> tcgen05.mma ->
TMEM -> fused epilogue).  ``oracle/unet_ref.py`` is the fp32 CPU restatement
the parity tests compare against (same weights, rounded to bf16).

Phi at outer step s (1-based, T = steps) for one window:
    sigma      = config.sigma_for(s, T)
    x_noisy    = sigma * x                       if s == T   (x = unit seed noise)
               = x + sigma * z_s(X, Y)           otherwise   (consistency renoise,
                                                  z_s = noise stream 301 + s)
    F          = net(c_in(sigma) * x_noisy, conditioning, c_noise(sigma))
    Phi        = c_skip(sigma) * x_noisy + c_out(sigma) * F
Everything per pixel is a pure function of the window and absolute
coordinates, so overlapping windows stay seed-consistent.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from ._native import ConvParams, call, lib, check
from .grid import Region
from .noise import STREAM_RENOISE

MP_SILU_GAIN = 1.0 / 0.596   # EDM2 mp_silu: silu(x) / 0.596
RES_T = 1.0 / 3.0            # mp_sum blend of the residual branch (EDM2 uses 0.3;
#                              1/3 makes ra/rb = 2 exactly, see UNetDevice.forward)
RES_RA = (1 - RES_T) / math.sqrt((1 - RES_T) ** 2 + RES_T ** 2)
RES_RB = RES_T / math.sqrt((1 - RES_T) ** 2 + RES_T ** 2)
# identity-skip blocks: IG_IDENT_RES=1 adds the residual in the c2 epilogue instead
# of as a K chunk of 2 * I in the same accumulator; measured slower (r02,
# tools/ab_layers.sh: enc0.0.c2 779 -> 707 TFLOP/s), so the K chunk stays
IDENT_RES = os.environ.get("IG_IDENT_RES", "0") == "1"
RES_Q = 2.0                  # ra / rb
ATTN_T = 0.3                 # EDM2 attn_balance: x = mp_sum(x, attn(x), t=0.3)
Q_SCALE = 0.125 * math.log2(math.e)   # softmax 1/sqrt(64) in log2 units, carried by q
ATTN_RA = (1 - ATTN_T) / math.sqrt((1 - ATTN_T) ** 2 + ATTN_T ** 2)
ATTN_RB = ATTN_T / math.sqrt((1 - ATTN_T) ** 2 + ATTN_T ** 2)
FUSED_STEM = True            # input gather fused into the stem GEMM (ig_unet_stem)
FUSED_UP = True              # 2x upsample folded into the consumer convs' TMA loads
FUSED_OUT = True             # output conv + preconditioning in one kernel (ig_unet_out_head)
FUSED_GUTTER = True          # narrow levels (w <= 64) in the gutter layout (1-D tap shifts)
# encoder 2x2 pool written by the producing conv's epilogue (bit-exact, tested).
# The epilogue's global stores are its limiter: with 16-byte stores (every warp
# store touching 32 lines for half a sector each) the fused pool measured slower
# (r01: enc0.0.c2 479 -> 847 us); with whole-sector 32-byte stores (r02)
# enc0.0.c2 + pool 512 -> 467 us and enc1.0.c2 + pool 312 -> 293 us, forward
# 7.69 -> 7.59 ms per 64 windows (median of 4 alternated runs).  IG_FUSED_POOL:
# 0 off, 2 only into standard-layout levels.
FUSED_POOL = int(os.environ.get("IG_FUSED_POOL", "1"))
FUSED_QKV = True             # attention q / k / v projections as one ig_conv_qkv launch


@dataclass(frozen=True)
class UNetConfig:
    """Architecture + preconditioning of the Phi network (build-defined)."""

    data_channels: int = 1          # C of the sampler
    cond_channels: int = 0          # conditioning planes (features) concatenated
    base: int = 64
    mults: tuple[int, ...] = (1, 2, 2, 4)
    blocks: int = 1                 # residual blocks per encoder level (decoder: +1)
    sigmas: tuple[float, ...] = (80.0, 1.0)   # sigma of the T, T-1, ... outer steps
    sigma_data: float = 0.5
    weight_seed: int = 0
    emb_dim: int = 64               # Fourier features of c_noise
    cin_pad: int = 64               # input planes padded to one 64-channel K block
    attn_levels: tuple[int, ...] = (3,)   # EDM2 self-attention after the blocks of these
    #                                       levels (heads of 64 channels; 32^2 at 256 px)

    def sigma_for(self, outer_step: int, steps: int) -> float:
        k = steps - outer_step
        return self.sigmas[min(k, len(self.sigmas) - 1)]

    def in_planes(self) -> int:
        # x, conditioning planes, conditioning mask, constant ones
        extra = (self.cond_channels + 1) if self.cond_channels else 0
        return self.data_channels + extra + 1

    def channels(self) -> list[int]:
        return [self.base * m for m in self.mults]


def precond(cfg: UNetConfig, sigma: float):
    sd = cfg.sigma_data
    c_skip = sd * sd / (sigma * sigma + sd * sd)
    c_out = sigma * sd / math.sqrt(sigma * sigma + sd * sd)
    c_in = 1.0 / math.sqrt(sigma * sigma + sd * sd)
    c_noise = math.log(sigma) / 4.0
    return c_skip, c_out, c_in, c_noise


# ---------------------------------------------------------------------------
# layer program (shared with the CPU oracle)

@dataclass
class ConvSpec:
    name: str
    cin: int          # total input channels (sum of sources)
    cout: int
    taps: int         # 9 (3x3) or 1 (1x1)
    cout_pad: int = 0
    modulated: bool = False   # per-step per-channel (1 + emb) scale


@dataclass
class Program:
    """Static layer list of the network (names -> conv specs) and the op
    sequence the forward executes."""

    convs: dict = field(default_factory=dict)
    ops: list = field(default_factory=list)


def build_program(cfg: UNetConfig) -> Program:
    prog = Program()
    ch = cfg.channels()
    L = len(ch)

    def conv(name, cin, cout, taps, modulated=False, cout_pad=0):
        prog.convs[name] = ConvSpec(name, cin, cout, taps, cout_pad or cout, modulated)

    attn = []      # (block name, channels): registered after every other conv so the
    #                adding attention leaves the other layers' weight draws unchanged
    # encoder; the stem 3x3 conv over in_planes() planes runs tap-packed as a
    # 1x1 GEMM over 9 * in_planes <= cin_pad channels (see ig_unet_gather_input)
    conv("stem", cfg.cin_pad, ch[0], 1)
    prog.ops.append(("stem",))
    skips = [ch[0]]
    cur = ch[0]
    for lv in range(L):
        for b in range(cfg.blocks):
            nm = f"enc{lv}.{b}"
            conv(nm + ".c1", cur, ch[lv], 9, modulated=True)
            conv(nm + ".c2", ch[lv], ch[lv], 9)
            if cur != ch[lv]:
                conv(nm + ".skip", cur, ch[lv], 1)
            prog.ops.append(("enc", nm, cur != ch[lv]))
            cur = ch[lv]
            if lv in cfg.attn_levels:
                prog.ops.append(("attn", nm, lv))
                attn.append((nm, cur))
            skips.append(cur)
        if lv < L - 1:
            prog.ops.append(("down",))
            skips.append(cur)
    # decoder
    for lv in reversed(range(L)):
        for b in range(cfg.blocks + 1):
            nm = f"dec{lv}.{b}"
            sk = skips.pop()
            conv(nm + ".c1", cur + sk, ch[lv], 9, modulated=True)
            conv(nm + ".c2", ch[lv], ch[lv], 9)
            conv(nm + ".skip", cur + sk, ch[lv], 1)
            prog.ops.append(("dec", nm))
            cur = ch[lv]
            if lv in cfg.attn_levels:
                prog.ops.append(("attn", nm, lv))
                attn.append((nm, cur))
        if lv > 0:
            prog.ops.append(("up",))
    conv("out", cur, cfg.data_channels, 9, cout_pad=16)
    prog.ops.append(("out",))
    for nm, c in attn:
        conv(nm + ".qkv", c, 3 * c, 1)      # rows [q (c) | k (c) | v (c)], heads of 64
        conv(nm + ".proj", c, c, 1)
    assert not skips
    return prog


def conv_flops(cfg: UNetConfig, h: int, w: int, padded: bool = False,
               stem_head: bool = True) -> float:
    """Algorithmic FLOPs of one window (real input/output channels unless
    `padded`): sum over convs of 2 * H * W * Cin * Cout * taps, plus the
    attention contractions.  ``stem_head=False`` leaves out the input stem and
    the output head (the fused stem / head kernels, timed apart from the
    tensor-core convolutions)."""
    prog = build_program(cfg)
    res = {}
    # resolution of each conv: walk the ops
    r = (h, w)
    lv_res = []
    for lv in range(len(cfg.mults)):
        lv_res.append((h >> lv, w >> lv))
    total = 0.0
    for name, cs in prog.convs.items():
        if name in ("stem", "out") and not stem_head:
            continue
        if name in ("stem", "out"):
            hh, ww = h, w
        else:
            lv = int(name[3:].split(".")[0])
            hh, ww = lv_res[lv]
        cout = cs.cout_pad if padded else cs.cout
        if name == "stem" and not padded:
            total += 2.0 * hh * ww * cfg.in_planes() * cout * 9    # the real 3x3 conv
        else:
            total += 2.0 * hh * ww * cs.cin * cout * cs.taps
    # attention: q k^T and p v (4 N^2 C per layer; q/k/v/proj are 1x1 convs above)
    for op in prog.ops:
        if op[0] == "attn":
            hh, ww = lv_res[op[2]]
            tokens = hh * ww
            total += 4.0 * tokens * tokens * cfg.channels()[op[2]]
    return total


def make_weights(cfg: UNetConfig) -> dict:
    """Deterministic magnitude-preserving init (torch.manual_seed(weight_seed)).

    Raw weights ~ N(0, 1); the effective weight of output row co is
    w_raw[co] / rms(w_raw[co]) / sqrt(fan_in) (EDM2 MPConv forced
    normalisation).  Returned as float32 CPU tensors [cout][taps][cin]
    (K-major), zero-padded to cout_pad rows, plus the per-step embedding
    projections.  Stem weights on padding input planes are zero.
    """
    prog = build_program(cfg)
    g = torch.Generator().manual_seed(cfg.weight_seed)
    out = {}
    for name, cs in prog.convs.items():
        stem = name == "stem"
        cin_real = cfg.in_planes() if stem else cs.cin
        taps = 9 if stem else cs.taps
        wr = torch.randn(cs.cout, taps, cin_real, generator=g, dtype=torch.float32)
        rms = wr.pow(2).mean(dim=(1, 2), keepdim=True).sqrt()
        fan_in = taps * cin_real
        weff = wr / (rms + 1e-4) / math.sqrt(fan_in)
        if stem:
            out["stem.3x3"] = weff                       # [cout][9][P] (oracle form)
            full = torch.zeros(cs.cout_pad, 1, cs.cin, dtype=torch.float32)
            full[:cs.cout, 0, :9 * cin_real] = weff.reshape(cs.cout, 9 * cin_real)
        else:
            full = torch.zeros(cs.cout_pad, cs.taps, cs.cin, dtype=torch.float32)
            full[:cs.cout, :, :cin_real] = weff
        out[name] = full
        if cs.modulated:
            out[name + ".emb"] = torch.randn(cs.cout, cfg.emb_dim, generator=g) / math.sqrt(
                cfg.emb_dim)
    out["fourier.freq"] = torch.randn(cfg.emb_dim // 2, generator=g)
    out["fourier.phase"] = torch.rand(cfg.emb_dim // 2, generator=g)
    out["out.gain"] = torch.tensor(1.0)
    return out


def round_bf16(w: torch.Tensor) -> torch.Tensor:
    return w.to(torch.bfloat16).to(torch.float32)


def modulation(cfg: UNetConfig, weights: dict, name: str, sigma: float) -> torch.Tensor:
    """Per-channel (1 + emb) scale of a modulated conv at noise level sigma
    (float32, CPU): emb = W_emb @ mp_silu(fourier(c_noise))."""
    c_noise = math.log(sigma) / 4.0
    f = weights["fourier.freq"]
    ph = weights["fourier.phase"]
    arg = 2.0 * math.pi * (f * c_noise + ph)
    feat = torch.cat([torch.cos(arg), torch.sin(arg)]) * math.sqrt(2.0)
    feat = torch.nn.functional.silu(feat) * MP_SILU_GAIN
    emb = weights[name + ".emb"] @ feat
    return (1.0 + emb).to(torch.float32)


# ---------------------------------------------------------------------------
# device model

class UNetDevice:
    """Weights resident in HBM (bf16, K-major) and the forward pass."""

    def __init__(self, cfg: UNetConfig):
        self.cfg = cfg
        self.prog = build_program(cfg)
        self.host = make_weights(cfg)
        d = dev.device()
        self.w = {}
        for name, cs in self.prog.convs.items():
            self.w[name] = self.host[name].reshape(cs.cout_pad, -1).to(torch.bfloat16).to(d)
        self.ones = {}
        self.zeros = {}
        self._mod_cache = {}

    def _vec1(self, n):
        if n not in self.ones:
            self.ones[n] = torch.ones(n, dtype=torch.float32, device=dev.device())
            self.zeros[n] = torch.zeros(n, dtype=torch.float32, device=dev.device())
        return self.ones[n], self.zeros[n]

    def _scale(self, name, sigma):
        key = (name, sigma)
        if key not in self._mod_cache:
            self._mod_cache[key] = modulation(self.cfg, self.host, name, sigma).to(dev.device())
        return self._mod_cache[key]

    def _skip_weights(self, name, cin, cout):
        """q * W_skip (bf16) for the fused skip GEMM of block `name`; the
        identity when the block keeps its channel count.  q = ra / rb = 2
        (RES_T = 1/3), so the scaling is exact in bf16."""
        key = name + ".wskip"
        if key not in self.w:
            q = RES_Q
            if name + ".skip" in self.prog.convs:
                wsk = self.w[name + ".skip"].float() * q
            else:
                wsk = torch.eye(cout, cin, device=dev.device()) * q
            self.w[key] = wsk.to(torch.bfloat16).contiguous()
        return self.w[key]

    def _rb(self, n):
        key = ("rb", n)
        if key not in self._mod_cache:
            self._mod_cache[key] = torch.full((n,), RES_RB, dtype=torch.float32,
                                              device=dev.device())
        return self._mod_cache[key]

    # -- primitive launches -------------------------------------------------
    def conv(self, name, a, b, sigma, out0=True, out1=True, skip=None, wskip=None,
             scale=None, up2=False, up_in=0, gutter=0, pool=None, res=None):
        """gutter bit 0: activations in the gutter layout (n, h, w+2, c); bit 1:
        the up_in low-res sources are."""
        cs = self.prog.convs[name]
        n, h, w, ca = a.shape
        if up_in & 1:                 # a is the low-res tensor, read 2x upsampled
            h, w = 2 * h, 2 * (w - 2 if gutter & 2 else w)
        elif gutter & 1:
            w = w - 2
        cb = 0 if b is None else b.shape[3]
        assert ca + cb == cs.cin, (name, ca, cb, cs.cin)
        if scale is None and cs.modulated:
            scale = self._scale(name, sigma)      # None: identity
        oh, ow = (2 * h, 2 * w) if up2 else (h, w + 2 if gutter & 1 else w)
        o0 = torch.empty((n, oh, ow, cs.cout_pad), dtype=torch.bfloat16, device=a.device) \
            if out0 else None
        o1 = torch.empty((n, oh, ow, cs.cout_pad), dtype=torch.bfloat16, device=a.device) \
            if out1 else None
        sa = skip[0] if skip else None
        sb = skip[1] if skip and len(skip) > 1 else None
        # res: (tensor, ra, rb) -> the epilogue's mp_sum ra * res + rb * acc
        rp, ra_, rb_ = (None, 0.0, 1.0) if res is None else res
        p = ConvParams(n, h, w, ca, cb, cs.cout_pad, cs.taps, a.data_ptr(), dev.ptr(b),
                       self.w[name].data_ptr(), dev.ptr(scale), None, dev.ptr(rp), float(ra_),
                       float(rb_), MP_SILU_GAIN, dev.ptr(o0), dev.ptr(o1),
                       0 if sa is None else sa.shape[3], 0 if sb is None else sb.shape[3],
                       dev.ptr(sa), dev.ptr(sb), dev.ptr(wskip), int(up2), int(up_in),
                       int(gutter), dev.ptr(pool[0] if pool else None),
                       dev.ptr(pool[1] if pool else None))
        conv_launch(p)
        return o0, o1

    def forward(self, x_in: torch.Tensor, sigma: float) -> torch.Tensor:
        """x_in: (n, H, W, cin_pad) bf16 -> F (n, H, W, 16) bf16.

        Residual blocks: x' = rb * (conv2(h) + q * skip(x)) = ra*skip + rb*conv2
        (mp_sum).  The skip branch (1x1 conv, or identity) is accumulated into
        conv2's TMEM accumulator as extra K blocks (no separate launch, no
        residual read), and the epilogue scales by rb."""
        x, xa = self.conv("stem", x_in, None, sigma)
        return self.forward_after_stem(x, xa, sigma)

    def attention(self, nm: str, x: torch.Tensor):
        """EDM2 self-attention block on x (standard NHWC layout):
        x' = mp_sum(x, proj(attn(norm(q), norm(k), norm(v))), t=0.3), returns
        (x', mp_silu(x')).  q/k/v and proj are 1x1 convs on the tensor cores,
        the projection's epilogue applies the mp_sum and the activation."""
        n, h, w, c = x.shape
        hw = h * w
        wq = self.w[nm + ".qkv"]                         # [3c][1][c] bf16
        q, k, v = (torch.empty_like(x) for _ in range(3))
        # the conv epilogues normalise each 64-channel head (q also carries the
        # softmax scale 1/8 * log2 e), so the attention kernel reads them as is
        if FUSED_QKV and c == 256:                      # one launch, 3x the work items
            p = ConvParams(n, h, w, c, 0, c, 1, x.data_ptr(), None, wq.data_ptr(), None, None,
                           None, 0.0, 1.0, 1.0, q.data_ptr(), None)
            p.head_norm, p.head_scale = 1, Q_SCALE
            conv_launch(p, qkv=(k, v))
        else:
            for j, dst in enumerate((q, k, v)):
                p = ConvParams(n, h, w, c, 0, c, 1, x.data_ptr(), None,
                               wq.data_ptr() + j * c * c * 2, None, None, None, 0.0, 1.0, 1.0,
                               dst.data_ptr(), None)
                p.head_norm = 2 if j == 2 else 1      # v in f16 (the PV MMA's operand)
                p.head_scale = Q_SCALE if j == 0 else 1.0
                conv_launch(p)
        y = torch.empty_like(x)
        st = dev.stream_ptr()
        attn_launch(lambda: call("ig_attention", q.data_ptr(), k.data_ptr(), v.data_ptr(), n,
                                 hw, c, y.data_ptr(), st))
        xo, xa = torch.empty_like(x), torch.empty_like(x)
        p = ConvParams(n, h, w, c, 0, c, 1, y.data_ptr(), None, self.w[nm + ".proj"].data_ptr(),
                       None, None, x.data_ptr(), float(ATTN_RA), float(ATTN_RB), MP_SILU_GAIN,
                       xo.data_ptr(), xa.data_ptr())
        conv_launch(p)
        return xo, xa

    @staticmethod
    def _fusable_pool(h1: torch.Tensor, gut: bool, cout: int) -> bool:
        """The c2 conv producing (x, xa) can also write their 2x2 pool: the
        2-D CTA-pair kernel runs it (mirror of ig_conv_tc's dispatch)."""
        n, h, w, _ = h1.shape
        return bool(FUSED_POOL and not gut and w % 128 == 0 and h % 2 == 0
                    and cout in (64, 128) and (n * (w // 128) * (h // 2)) % 2 == 0)

    def _gutter(self, lv: int, w: int) -> bool:
        """Level lv (width w) keeps its activations in the gutter layout: narrow
        levels below the stem whose convs the CTA-pair kernel covers."""
        return bool(FUSED_GUTTER and lv >= 1 and w <= 64 and lv not in self.cfg.attn_levels
                    and self.cfg.channels()[lv] in (64, 128, 256))

    def forward_after_stem(self, x: torch.Tensor, xa: torch.Tensor, sigma: float, head=None):
        """The network after the stem: (x, mp_silu(x)) -> F.

        head = (x_noisy, c_skip, c_out, phi): when the fused output head
        applies, Phi = c_skip * x_noisy + c_out * F is written into phi and
        None is returned (F is never materialised)."""
        skips = [(x, xa)]
        ops = self.prog.ops
        pool = None     # fused-pool outputs of the last encoder block
        up = 0          # (x, xa) are low-res and the next block reads them upsampled
        lv, w = 0, x.shape[2]       # level and logical width of (x, xa)
        gut = self._gutter(lv, w)   # (x, xa) in the gutter layout
        for k in range(1, len(ops)):
            op = ops[k]
            nxt = ops[k + 1][0] if k + 1 < len(ops) else None
            # a block output feeding an attention block is only read as x (the
            # attention returns a new (x, mp_silu(x))); the output layer only
            # reads mp_silu(x): those tensors are not written at all
            want0, want1 = nxt != "out", nxt != "attn"
            if op[0] == "enc":
                nm = op[1]
                g = int(gut)
                _, h1 = self.conv(nm + ".c1", xa, None, sigma, out0=False, gutter=g)
                c2 = self.prog.convs[nm + ".c2"]
                wsk = self._skip_weights(nm, x.shape[3], c2.cout)
                pool = None
                if k + 1 < len(ops) and ops[k + 1][0] == "down" and \
                        self._fusable_pool(h1, gut, c2.cout_pad) and \
                        (FUSED_POOL != 2 or not self._gutter(lv + 1, w // 2)):
                    # the 2x2 pool of this block's output, written by its epilogue
                    ng = self._gutter(lv + 1, w // 2)
                    n_, h_ = h1.shape[0], h1.shape[1]
                    shp = (n_, h_ // 2, w // 2 + (2 if ng else 0), c2.cout_pad)
                    pool = (torch.empty(shp, dtype=torch.bfloat16, device=h1.device),
                            torch.empty(shp, dtype=torch.bfloat16, device=h1.device))
                    g |= 4 * int(ng)
                if IDENT_RES and pool is None and nm + ".skip" not in self.prog.convs:
                    # identity skip: the residual read in the epilogue, ra * x + rb * c2(h),
                    # instead of a K chunk of 2 * I -- a lone skip chunk per tile held a
                    # halo slot for only 16 MMAs (the next tile's box then arrived late)
                    x, xa = self.conv(nm + ".c2", h1, None, sigma, gutter=g,
                                      res=(x, RES_RA, RES_RB), out0=want0, out1=want1)
                else:
                    x, xa = self.conv(nm + ".c2", h1, None, sigma, skip=(x,), wskip=wsk,
                                      scale=self._rb(c2.cout_pad), gutter=g, pool=pool,
                                      out0=want0 or pool is not None, out1=want1)
                skips.append((x, xa))
            elif op[0] == "attn":
                x, xa = self.attention(op[1], x)
                if ops[k - 1][0] == "enc":
                    skips[-1] = (x, xa)      # the block output pushed as the skip
            elif op[0] == "down":
                ng = self._gutter(lv + 1, w // 2)
                if pool is not None:
                    x, xa = pool
                    pool = None
                else:
                    x, xa = pool_launch(x, w, int(gut) | (int(ng) << 1))
                lv, w, gut = lv + 1, w // 2, ng
                skips.append((x, xa))
            elif op[0] == "dec":
                nm = op[1]
                s, sa = skips.pop()
                if up:
                    # low-res (x, xa) of level lv+1, possibly in the gutter layout
                    g = 2 * int(up_gut)
                else:
                    g = int(gut)
                _, h1 = self.conv(nm + ".c1", xa, sa, sigma, out0=False, up_in=up, gutter=g)
                c2 = self.prog.convs[nm + ".c2"]
                wsk = self._skip_weights(nm, x.shape[3] + s.shape[3], c2.cout)
                # (ConvParams.up2 can write the 2x-upsampled outputs from the
                # epilogue directly, but its 4x scattered stores measured slower
                # (r01: 132 vs 121 ms/step) than the separate coalesced kernel)
                x, xa = self.conv(nm + ".c2", h1, None, sigma, skip=(x, s), wskip=wsk,
                                  scale=self._rb(c2.cout_pad), up_in=2 if up else 0, gutter=g,
                                  out0=want0, out1=want1)
                up = 0
            elif op[0] == "up":
                ng = self._gutter(lv - 1, 2 * w)
                if FUSED_UP and (2 * w) % 128 == 0 and not ng:
                    up, up_gut = 1, gut     # upsample inside the next convs' TMA loads
                else:
                    lay = int(gut) | (int(ng) << 1)
                    x, xa = upsample_launch(x, w, lay), upsample_launch(xa, w, lay)
                lv, w, gut = lv - 1, 2 * w, ng
            elif op[0] == "out":
                n, h, w, c = xa.shape
                C = self.cfg.data_channels
                if head is not None and FUSED_OUT and c == 64 and C <= 8 and w % 128 == 0 \
                        and h % 4 == 0:
                    x_noisy, c_skip, c_out, phi = head
                    call("ig_unet_out_head", xa.data_ptr(), n, h, w, c,
                         self.w["out"].data_ptr(), self.prog.convs["out"].cout_pad, C,
                         x_noisy.data_ptr(), float(c_skip), float(c_out), phi.data_ptr(),
                         dev.stream_ptr())
                    return None
                f, _ = self.conv("out", xa, None, sigma, out1=False)
                return f
        raise AssertionError("program without output layer")


_MODELS: dict = {}


def model_for(cfg: UNetConfig) -> UNetDevice:
    m = _MODELS.get(cfg)
    if m is None:
        m = _MODELS[cfg] = UNetDevice(cfg)
    return m


_WS = None


class _ConvTimer:
    """Optional CUDA-event bracketing of every ig_conv_tc launch (bench.py's
    roofline: per-launch device time on the launching stream).  Events come
    from a pool created up front: constructing two torch.cuda.Event objects per
    launch inside the timed region cost ~1% of the bench step on the host."""

    def __init__(self):
        self.on = False
        self.events = []
        self._pool = []
        self._next = 0

    def enable(self, stream=None, reserve=4096):
        while len(self._pool) < reserve:
            self._pool.append(torch.cuda.Event(enable_timing=True))
        self.on, self.events, self._next = True, [], 0

    def pair(self):
        if self._next + 2 > len(self._pool):
            self._pool.extend(torch.cuda.Event(enable_timing=True) for _ in range(256))
        a, b = self._pool[self._next], self._pool[self._next + 1]
        self._next += 2
        return a, b

    def disable(self):
        self.on, self.events, self._next = False, [], 0

    def collect(self):
        torch.cuda.synchronize()
        total = sum(a.elapsed_time(b) for a, b in self.events)
        return total, len(self.events)


TIMING = _ConvTimer()


def conv_launch(p: ConvParams, qkv=None):
    """ig_conv_tc(p); qkv = (k, v): ig_conv_qkv (p.out0 = q, weights [3c][c])."""
    global _WS
    nbytes = int(lib().ig_conv_workspace_bytes())
    if nbytes and (_WS is None or _WS.numel() < nbytes):
        _WS = torch.empty(nbytes, dtype=torch.uint8, device=dev.device())
    if TIMING.on:
        a, b = TIMING.pair()
        a.record()
    if qkv is not None:
        check(lib().ig_conv_qkv(p, qkv[0].data_ptr(), qkv[1].data_ptr(), dev.stream_ptr()),
              "ig_conv_qkv")
    else:
        check(lib().ig_conv_tc(p, dev.ptr(_WS) if nbytes else None, dev.stream_ptr()),
              "ig_conv_tc")
    if TIMING.on:
        b.record()
        TIMING.events.append((a, b))


def attn_launch(fn):
    """Attention kernels under the same per-launch event timer as the convs
    (bench.py's tensor-core roofline covers both)."""
    if TIMING.on:
        a, b = TIMING.pair()
        a.record()
    fn()
    if TIMING.on:
        b.record()
        TIMING.events.append((a, b))


def pool_launch(x: torch.Tensor, w: int | None = None, layout: int = 0):
    """2x2 mean pool -> (out, mp_silu(out)); w = logical width, layout bit 0 /
    bit 1: input / output in the gutter layout."""
    n, h, wx, c = x.shape
    w = wx if w is None else w
    ow = w // 2 + (2 if layout & 2 else 0)
    o = torch.empty((n, h // 2, ow, c), dtype=torch.bfloat16, device=x.device)
    oa = torch.empty_like(o)
    call("ig_avgpool2_bf16", x.data_ptr(), n, h, w, c, o.data_ptr(), oa.data_ptr(), layout,
         dev.stream_ptr())
    return o, oa


def upsample_launch(x: torch.Tensor, w: int | None = None, layout: int = 0):
    n, h, wx, c = x.shape
    w = wx if w is None else w
    ow = 2 * w + (2 if layout & 2 else 0)
    o = torch.empty((n, 2 * h, ow, c), dtype=torch.bfloat16, device=x.device)
    call("ig_upsample2_bf16", x.data_ptr(), n, h, w, c, o.data_ptr(), layout, dev.stream_ptr())
    return o


def unet_phi_batch(cfg: UNetConfig, src: torch.Tensor, src_region: Region | None,
                   wxy: torch.Tensor, win: int, outer_step: int, cond, seed: int,
                   steps: int | None = None) -> torch.Tensor:
    """Phi (n, C, win, win) float32 for a batch of windows (see module doc)."""
    steps = steps if steps is not None else len(cfg.sigmas)
    model = model_for(cfg)
    n = int(wxy.shape[0])
    C = cfg.data_channels
    sigma = cfg.sigma_for(outer_step, steps)
    c_skip, c_out, c_in, _ = precond(cfg, sigma)
    src32 = src if src.dtype == torch.float32 else src.to(torch.float32)
    batched = src_region is None
    sx0, sy0 = (0, 0) if batched else (src_region.x0, src_region.y0)
    if cond is not None and cfg.cond_channels:
        cp = cond.parent if cond.parent.dtype == torch.float32 else cond.parent.float()
        cargs = (cp.data_ptr(), cond.region.x0, cond.region.y0, cp.shape[-1], cp.shape[-2],
                 min(cp.shape[0], cfg.cond_channels), cond.scale,
                 -1 if cond.mask_channel is None else cond.mask_channel, cond.seed)
    else:
        cargs = (None, 0, 0, 0, 0, 0, 1, -1, 0)
    phi = torch.empty((n, C, win, win), dtype=torch.float32, device=src.device)
    # windows are processed in chunks so activation memory stays bounded
    # (~8 MB per window per live 64-channel tensor at 256^2); Phi of a window
    # does not depend on its chunk (the kernels are batch invariant)
    chunk = max(1, min(n, max_windows_per_forward(win)))
    for k0 in range(0, n, chunk):
        m = min(chunk, n - k0)
        x_noisy = torch.empty((m, C, win, win), dtype=torch.float32, device=src.device)
        sptr = src32[k0:k0 + m].data_ptr() if batched else src32.data_ptr()
        common = (sptr, int(batched), sx0, sy0, src32.shape[-1], src32.shape[-2], C,
                  wxy[k0:k0 + m].data_ptr(), m, *cargs[:-1], cargs[-1] & ((1 << 64) - 1),
                  seed & ((1 << 64) - 1), STREAM_RENOISE + outer_step, float(sigma), float(c_in),
                  int(outer_step == steps))
        if FUSED_STEM and model.prog.convs["stem"].cout_pad == 64:
            # gather + tap-packed stem GEMM in one kernel (input never hits HBM)
            x = torch.empty((m, win, win, 64), dtype=torch.bfloat16, device=src.device)
            xa = torch.empty_like(x)
            call("ig_unet_stem", *common, win, cfg.in_planes(), model.w["stem"].data_ptr(),
                 MP_SILU_GAIN, x.data_ptr(), xa.data_ptr(), x_noisy.data_ptr(),
                 dev.stream_ptr())
            f = model.forward_after_stem(x, xa, sigma,
                                         head=(x_noisy, c_skip, c_out, phi[k0:k0 + m]))
        else:
            x_in = torch.empty((m, win, win, cfg.cin_pad), dtype=torch.bfloat16,
                               device=src.device)
            call("ig_unet_gather_input", *common, x_in.data_ptr(), win, cfg.cin_pad,
                 cfg.in_planes(), x_noisy.data_ptr(), dev.stream_ptr())
            f = model.forward(x_in, sigma)
        if f is not None:
            call("ig_unet_output", f.data_ptr(), m, win, win, 16, x_noisy.data_ptr(), C,
                 float(c_skip), float(c_out), 0, phi[k0:k0 + m].data_ptr(), dev.stream_ptr())
    return phi


def max_windows_per_forward(win: int) -> int:
    """Windows per UNet forward: ~3 GB per 64-channel activation tensor
    (IG_UNET_CHUNK overrides, for A/B timing of the chunk size)."""
    env = os.environ.get("IG_UNET_CHUNK")
    if env:
        return max(1, int(env))
    return max(16, int(3.2e9 // (win * win * 64 * 2)))
