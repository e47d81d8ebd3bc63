"""Test helpers for the sharded (multi-rank) path: a CPU executor on the
oracle port, so the planner + halo-exchange protocol can run under gloo."""

import numpy as np
import torch

from oracle import port


class PortExecutor:
    """Window cache + canonical blend on the numpy oracle (CPU)."""

    def __init__(self, steps, H, s, spec, seed, eps=0.01):
        self.steps, self.H, self.s, self.spec, self.seed = steps, H, s, spec, seed
        self.W = port.tent(H, eps).astype(np.float32)
        self.cache = {t: {} for t in range(steps)}
        self.generated = 0

    def image(self, t, r):
        if t == self.steps:
            return port.noise(self.seed, 0, r, 1)
        A = np.zeros((1, r.h, r.w), dtype=np.float32)
        B = np.zeros((r.h, r.w), dtype=np.float32)
        for (i, j) in port.kappa(self.H, self.s, (0, 0), r):
            win = port.win_box(self.H, self.s, (0, 0), i, j)
            d = self.cache[t][(i, j)]
            ov = win.inter(r)
            ys, xs = slice(ov.y0 - r.y0, ov.y1 - r.y0), slice(ov.x0 - r.x0, ov.x1 - r.x0)
            wy, wx = slice(ov.y0 - win.y0, ov.y1 - win.y0), slice(ov.x0 - win.x0, ov.x1 - win.x0)
            A[:, ys, xs] += (self.W[None] * d)[:, wy, wx]
            B[ys, xs] += self.W[wy, wx]
        out = np.zeros_like(A)
        np.divide(A, B[None], out=out, where=B[None] > 0)
        return out

    def generate(self, t, idxs):
        out = {}
        for (i, j) in idxs:
            win = port.win_box(self.H, self.s, (0, 0), i, j)
            x = self.image(t + 1, win)
            d = port.phi_analytic(self.spec, x, None, t + 1).astype(np.float32)
            self.cache[t][(i, j)] = d
            self.generated += 1
            out[(i, j)] = torch.from_numpy(d)
        return out

    def inject(self, t, windows):
        for idx, data in windows.items():
            self.cache[t][idx] = data.numpy() if isinstance(data, torch.Tensor) else data

    def query(self, region):
        return self.image(0, port.Box(region.x0, region.y0, region.width, region.height))
