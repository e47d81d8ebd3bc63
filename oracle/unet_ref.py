"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

float32 torch-CPU restatement of the build-defined UNet Phi
(paper_2512_08309_b200/unet.py).  The reference package has no UNet
(SURVEY 8(a) a34), so this is the checker for the tcgen05 path: NCHW fp32
convolutions (torch.nn.functional.conv2d) with the SAME weights rounded to
bf16 (isolating activation precision), same preconditioning, same renoise.
Model *definition* (layer list, weight init, modulation) is imported from the
product module -- it is the specification, not the computation under test.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from paper_2512_08309_b200.unet import (ATTN_T, MP_SILU_GAIN, RES_T, build_program, make_weights,
                                        modulation, precond, round_bf16)

from . import port


def mp_silu(x):
    return F.silu(x) * MP_SILU_GAIN


class UNetRef:
    def __init__(self, cfg):
        self.cfg = cfg
        self.prog = build_program(cfg)
        self.host = make_weights(cfg)
        self.w = {}
        self.pad = {}
        for name, cs in self.prog.convs.items():
            if name == "stem":
                # the device runs the stem tap-packed; the oracle keeps the 3x3 form
                w = round_bf16(self.host["stem.3x3"])       # [cout][9][P]
                P = w.shape[2]
                full = torch.zeros(cs.cout_pad, 3, 3, cfg.cin_pad)
                full[:w.shape[0], :, :, :P] = w.reshape(w.shape[0], 3, 3, P)
                self.w[name] = full.permute(0, 3, 1, 2).contiguous()
                self.pad[name] = 1
                continue
            w = round_bf16(self.host[name])                  # [cout_pad][taps][cin]
            k = 3 if cs.taps == 9 else 1
            self.w[name] = w.reshape(cs.cout_pad, k, k, cs.cin).permute(0, 3, 1, 2).contiguous()
            self.pad[name] = k // 2

    def conv(self, name, x, sigma):
        cs = self.prog.convs[name]
        y = F.conv2d(x, self.w[name], padding=self.pad[name])
        if cs.modulated:
            y = y * modulation(self.cfg, self.host, name, sigma)[None, :, None, None]
        return y

    def attention(self, nm, x, sigma):
        """EDM2 self-attention block (fp32): heads of 64 channels, q/k/v unit-RMS
        normalised per token, softmax(q k^T / 8) v, 1x1 projection, mp_sum."""
        n, c, h, w = x.shape
        qkv = self.conv(nm + ".qkv", x, sigma).reshape(n, 3, c // 64, 64, h * w)

        def nrm(t):
            return t / (1e-4 + t.norm(dim=2, keepdim=True) / 8.0)

        q, k, v = nrm(qkv[:, 0]), nrm(qkv[:, 1]), nrm(qkv[:, 2])     # (n, heads, 64, hw)
        p = torch.einsum("nhdq,nhdk->nhqk", q, k / 8.0).softmax(dim=-1)
        y = torch.einsum("nhqk,nhdk->nhdq", p, v).reshape(n, c, h, w)
        y = self.conv(nm + ".proj", y, sigma)
        nrm_t = math.sqrt((1 - ATTN_T) ** 2 + ATTN_T ** 2)
        return ((1 - ATTN_T) * x + ATTN_T * y) / nrm_t

    @torch.no_grad()
    def forward(self, x_in, sigma):
        """x_in (n, cin_pad, H, W) fp32 -> F (n, cout_pad, H, W)."""
        nrm = math.sqrt((1 - RES_T) ** 2 + RES_T ** 2)
        ra, rb = (1 - RES_T) / nrm, RES_T / nrm
        x = self.conv("stem", x_in, sigma)
        skips = [x]
        prev = None
        for op in self.prog.ops[1:]:
            if op[0] == "enc":
                nm, has_skip = op[1], op[2]
                h = mp_silu(self.conv(nm + ".c1", mp_silu(x), sigma))
                res = self.conv(nm + ".skip", x, sigma) if has_skip else x
                x = ra * res + rb * self.conv(nm + ".c2", h, sigma)
                skips.append(x)
            elif op[0] == "attn":
                x = self.attention(op[1], x, sigma)
                if prev == "enc":
                    skips[-1] = x
            elif op[0] == "down":
                x = F.avg_pool2d(x, 2)
                skips.append(x)
            elif op[0] == "dec":
                nm = op[1]
                s = skips.pop()
                cat = torch.cat([x, s], dim=1)
                h = mp_silu(self.conv(nm + ".c1", mp_silu(cat), sigma))
                res = self.conv(nm + ".skip", cat, sigma)
                x = ra * res + rb * self.conv(nm + ".c2", h, sigma)
            elif op[0] == "up":
                x = F.interpolate(x, scale_factor=2, mode="nearest")
            elif op[0] == "out":
                return self.conv("out", mp_silu(x), sigma)
            prev = op[0]
        raise AssertionError


_CACHE = {}


def ref_model(cfg):
    if cfg not in _CACHE:
        _CACHE[cfg] = UNetRef(cfg)
    return _CACHE[cfg]


def unet_phi(cfg, steps, seed):
    """Phi callable for port.Stage: (x (C,H,W), y, outer_step, win_box) -> (C,H,W)."""
    model = ref_model(cfg)

    def phi(x, y, s, win):
        sigma = cfg.sigma_for(s, steps)
        c_skip, c_out, c_in, _ = precond(cfg, sigma)
        x = np.asarray(x, dtype=np.float32)
        C, H, W = x.shape
        if s == steps:
            xn = np.float32(sigma) * x
        else:
            z = port.noise(seed, 301 + s, win, C)
            xn = x + np.float32(sigma) * z
        planes = np.zeros((cfg.cin_pad, H, W), dtype=np.float32)
        planes[:C] = np.float32(c_in) * xn
        p = C
        if cfg.cond_channels:
            if y is not None:
                ch, m = y
                planes[p:p + cfg.cond_channels] = ch[:cfg.cond_channels]
                planes[p + cfg.cond_channels] = m
            p += cfg.cond_channels + 1
        planes[p] = 1.0
        f = model.forward(torch.from_numpy(planes)[None], sigma)[0, :C].numpy()
        return np.float32(c_skip) * xn + np.float32(c_out) * f

    return phi
