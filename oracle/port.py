"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Numpy restatement of the reference hot path, evaluated *densely*: every step
image is computed once over the nested union covers, windows are visited in
canonical (j, i) order and summed per pixel with the reference's float32 op
sequence.  Each function cites the reference lines it restates
(paths relative to /root/reference/pkg/src/infigrid/).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_U64 = (1 << 64) - 1
GAMMA = np.uint64(0x9E3779B97F4A7C15)

# ----------------------------------------------------------------------------
# geometry (grid.py:21-180)


class Box:
    """Half-open lattice rectangle (grid.py:21-84)."""

    __slots__ = ("x0", "y0", "w", "h")

    def __init__(self, x0, y0, w, h):
        self.x0, self.y0, self.w, self.h = int(x0), int(y0), int(w), int(h)

    @property
    def x1(self):
        return self.x0 + self.w

    @property
    def y1(self):
        return self.y0 + self.h

    def union(self, o):
        x0, y0 = min(self.x0, o.x0), min(self.y0, o.y0)
        return Box(x0, y0, max(self.x1, o.x1) - x0, max(self.y1, o.y1) - y0)

    def inter(self, o):
        x0, y0 = max(self.x0, o.x0), max(self.y0, o.y0)
        x1, y1 = min(self.x1, o.x1), min(self.y1, o.y1)
        return None if x1 <= x0 or y1 <= y0 else Box(x0, y0, x1 - x0, y1 - y0)

    def grow(self, m):
        return Box(self.x0 - m, self.y0 - m, self.w + 2 * m, self.h + 2 * m)

    def coarsen(self, f):
        """grid.py:76-84: floor start, ceil end."""
        if f == 1:
            return self
        x0, y0 = self.x0 // f, self.y0 // f
        return Box(x0, y0, -(-self.x1 // f) - x0, -(-self.y1 // f) - y0)

    def tup(self):
        return (self.x0, self.y0, self.w, self.h)


def win_box(H, s, off, i, j):
    """grid.py:106-111."""
    return Box(i * s + off[0], j * s + off[1], H, H)


def kappa(H, s, off, r: Box):
    """grid.py:114-130: windows meeting r, canonical (j, i) order."""
    def span(a0, n, o):
        return -((o + H - 1 - a0) // s), (a0 + n - 1 - o) // s
    ilo, ihi = span(r.x0, r.w, off[0])
    jlo, jhi = span(r.y0, r.h, off[1])
    return [(i, j) for j in range(jlo, jhi + 1) for i in range(ilo, ihi + 1)]


def cover(H, s, off, r: Box):
    """grid.py:139-145."""
    ks = kappa(H, s, off, r)
    out = win_box(H, s, off, *ks[0])
    for k in ks[1:]:
        out = out.union(win_box(H, s, off, *k))
    return out


def tent(H, eps):
    """grid.py:148-180: separable tent weights, float64."""
    if H == 1:
        p = np.ones(1)
    else:
        half = H // 2
        idx = np.arange(H)
        if H % 2:
            d = np.abs(idx - half) / half
        else:
            d = np.minimum(np.abs(idx - (half - 1)), np.abs(idx - half))
            d = d / max(half - 1, 1) if half > 1 else np.zeros(H)
        p = eps + (1.0 - eps) * (1.0 - d)
    p = p.astype(np.float64)
    return np.outer(p, p)


# ----------------------------------------------------------------------------
# noise (noise.py:39-86)

_clib = None


def _c():
    global _clib
    if _clib is None:
        path = os.path.join(_HERE, "liboracle_noise.so")
        if os.path.exists(path):
            L = ctypes.CDLL(path)
            L.oracle_noise_region.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
            L.oracle_noise_f64.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_uint32]
            L.oracle_noise_f64.restype = ctypes.c_double
            _clib = L
        else:
            _clib = False
    return _clib


def _fin(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def noise_np(seed, stream, r: Box, channels=1, ch0=0):
    """Pure numpy restatement (noise.py:49-64, :74-86)."""
    xs = np.arange(r.x0, r.x1, dtype=np.int64).astype(np.uint64)[None, :]
    ys = np.arange(r.y0, r.y1, dtype=np.int64).astype(np.uint64)[:, None]
    out = np.empty((channels, r.h, r.w), dtype=np.float32)
    with np.errstate(over="ignore"):
        h0 = _fin((np.uint64(seed & _U64) ^ np.uint64(stream & 0xFFFFFFFF)) + GAMMA)
        hx = _fin((h0 ^ xs) + GAMMA)
        hxy = _fin((hx ^ ys) + GAMMA)
        for c in range(channels):
            h = _fin((hxy ^ np.uint64((ch0 + c) & 0xFFFFFFFF)) + GAMMA)
            h2 = _fin(h + GAMMA)
            u1 = np.maximum((h >> np.uint64(32)).astype(np.float64) * 2.0 ** -32, 2.0 ** -32)
            u2 = (h2 >> np.uint64(32)).astype(np.float64) * 2.0 ** -32
            out[c] = (np.sqrt(-2.0 * np.log(u1)) * np.cos((2.0 * np.pi) * u2)).astype(np.float32)
    return out


def noise(seed, stream, r: Box, channels=1, ch0=0):
    """C restatement when built (faster), else numpy."""
    L = _c()
    if not L:
        return noise_np(seed, stream, r, channels, ch0)
    out = np.empty((channels, r.h, r.w), dtype=np.float32)
    L.oracle_noise_region(seed & _U64, stream & 0xFFFFFFFF, r.x0, r.y0, r.w, r.h, ch0, channels,
                          out.ctypes.data)
    return out


# ----------------------------------------------------------------------------
# transforms (transforms.py)

def box_mean(x, r):
    """transforms.py:29-51: rows then columns, clamp-to-edge, acc then / k."""
    if r == 0:
        return x.copy()
    k = 2 * r + 1
    cur = x
    for axis in (-2, -1):
        n = cur.shape[axis]
        acc = np.zeros_like(cur)
        for off in range(-r, r + 1):
            idx = np.clip(np.arange(n) + off, 0, n - 1)
            acc += np.take(cur, idx, axis=axis)
        cur = acc / cur.dtype.type(k)
    return cur


def pairwise(v, dtype):
    """numpy pairwise summation order (loops_utils.h.src) of a 1-D block."""
    n = len(v)
    if n < 8:
        s = dtype(-0.0)
        for a in v:
            s = dtype(s + a)
        return s
    if n <= 128:
        r = [dtype(a) for a in v[:8]]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] = dtype(r[j] + v[i + j])
            i += 8
        s = dtype(dtype(dtype(r[0] + r[1]) + dtype(r[2] + r[3]))
                  + dtype(dtype(r[4] + r[5]) + dtype(r[6] + r[7])))
        while i < n:
            s = dtype(s + v[i])
            i += 1
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return dtype(pairwise(v[:n2], dtype) + pairwise(v[n2:], dtype))


def block_mean(x, f):
    """transforms.py:61-67 (numpy .mean(axis=(-3,-1)) order)."""
    h, w = x.shape[-2:]
    lead = x.shape[:-2]
    v = x.reshape(lead + (h // f, f, w // f, f))
    if f >= 8:
        # vectorised pairwise over the last axis, rows summed sequentially
        out = np.zeros(lead + (h // f, w // f), dtype=x.dtype)
        for rr in range(f):
            row = v[..., rr, :, :]  # (..., h/f, w/f, f)
            out = out + _pairwise_last(row)
        return out / (f * f)
    out = np.zeros(lead + (h // f, w // f), dtype=x.dtype)
    for rr in range(f):
        s = np.full(lead + (h // f, w // f), -0.0, dtype=x.dtype)
        for cc in range(f):
            s = s + v[..., rr, :, cc]
        out = out + s
    return out / (f * f)


def _pairwise_last(a):
    """pairwise() vectorised over leading axes (n = a.shape[-1] in [8, 128])."""
    n = a.shape[-1]
    if n > 128:
        n2 = n // 2
        n2 -= n2 % 8
        return _pairwise_last(a[..., :n2]) + _pairwise_last(a[..., n2:])
    r = [a[..., j].copy() for j in range(8)]
    i = 8
    while i < n - n % 8:
        for j in range(8):
            r[j] = r[j] + a[..., i + j]
        i += 8
    s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        s = s + a[..., i]
        i += 1
    return s


def up(x, f):
    return np.repeat(np.repeat(x, f, axis=-2), f, axis=-1)


def laplacian_encode(x, f=8, blur=1):
    """transforms.py:89-95."""
    x64 = np.asarray(x).astype(np.float64)
    b = x64
    for _ in range(blur):
        b = box_mean(b, 1)
    low = block_mean(b, f)
    return low, x64 - up(low, f)


def laplacian_decode(low, high, f, dtype):
    """transforms.py:98-101."""
    return (up(low, f) + high).astype(dtype)


def laplacian_stabilize(low, high, f, blur=1):
    """transforms.py:104-114."""
    b = up(low, f) + high
    for _ in range(blur):
        b = box_mean(b, 1)
    return block_mean(b, f), high


def signed_sqrt(x):
    return np.sign(x) * np.sqrt(np.abs(x))


def signed_square(x):
    return np.sign(x) * x * x


# ----------------------------------------------------------------------------
# Phi (denoise.py:75-185)

def phi_analytic(spec, x, y, t):
    """denoise.py:89-113.  spec: dict with kind/radius/lambdas/inner_*;
    y: None or (target_channels, mask)."""
    kind = spec["kind"]
    if kind == "identity":
        return x.copy()

    def shrink(v, lam):
        if lam == 0.0:
            return v.copy()
        dt = v.dtype.type
        return dt(1.0 - lam) * v + dt(lam) * box_mean(v, spec["radius"])

    def cond(v, lam):
        b = shrink(v, lam)
        if y is None or y[1] is None:
            return b
        return b + y[1] * (y[0][0] - b)

    lams = spec.get("lambdas", [0.5]) or [0.5]
    lam_t = lams[min(t - 1, len(lams) - 1)] if lams else 0.5
    if kind == "shrink_smooth":
        return shrink(x, lam_t)
    if kind == "cond_affine":
        return cond(x, lam_t)
    k = spec["inner_steps"]
    out = x
    for st in range(k):
        frac = st / (k - 1) if k > 1 else 0.0
        lam = spec["lambda_start"] * (spec["lambda_end"] / spec["lambda_start"]) ** frac
        out = shrink(out, lam) if spec["inner_kind"] == "shrink_smooth" else cond(out, lam)
    return out


def conditioning(parent, preg: Box, scale, win: Box, seed, mask=None):
    """denoise.py:116-163 -> (channels, mask)."""
    need = win.coarsen(scale)
    cx, cy = need.x0 - preg.x0, need.y0 - preg.y0
    crop = parent[:, cy:cy + need.h, cx:cx + need.w]
    px, py = win.x0 - need.x0 * scale, win.y0 - need.y0 * scale
    ch = np.ascontiguousarray(up(crop, scale)[:, py:py + win.h, px:px + win.w])
    if mask is None:
        m = np.ones((win.h, win.w), dtype=ch.dtype)
    else:
        mc = mask[cy:cy + need.h, cx:cx + need.w]
        m = np.ascontiguousarray(up(mc, scale)[py:py + win.h, px:px + win.w]).astype(ch.dtype)
    if not np.all(m >= 1.0):
        fill = noise(seed, 101, win, ch.shape[0]).astype(ch.dtype)
        ch = np.where((m < 1.0)[None], fill, ch)
    return ch, m


def patch_features(e, p):
    """denoise.py:166-185: (mean, p5, ones)."""
    h, w = e.shape
    blk = e.reshape(h // p, p, w // p, p).transpose(0, 2, 1, 3).reshape(h // p, w // p, p * p)
    dt = e.dtype.type
    if p * p >= 8:
        s = dt(0) + _pairwise_last(blk)
    else:
        s = np.full((h // p, w // p), -0.0, dtype=e.dtype)
        for q in range(p * p):
            s = s + blk[..., q]
        s = dt(0) + s
    mean = s / dt(p * p)
    rank = max(math.ceil(0.05 * p * p), 1)
    p5 = np.sort(blk, axis=-1)[..., rank - 1]
    return np.stack([mean, p5, np.ones_like(mean)])


# ----------------------------------------------------------------------------
# base maps (pipeline.py:87-139)

def procedural(seed, cell, r: Box, channels, stream=7):
    gx0, gy0 = r.x0 // cell, r.y0 // cell
    gx1, gy1 = (r.x1 - 1) // cell + 1, (r.y1 - 1) // cell + 1
    lat = noise(seed, stream, Box(gx0, gy0, gx1 - gx0 + 1, gy1 - gy0 + 1), channels)
    fx = np.arange(r.x0, r.x1) / cell - gx0
    fy = np.arange(r.y0, r.y1) / cell - gy0
    ix, iy = np.floor(fx).astype(np.int64), np.floor(fy).astype(np.int64)
    tx, ty = (fx - ix)[None, None, :], (fy - iy)[None, :, None]
    g = lambda dy, dx: lat[:, iy[:, None] + dy, ix[None, :] + dx]  # noqa: E731
    top = g(0, 0) * (1 - tx) + g(0, 1) * tx
    bot = g(1, 0) * (1 - tx) + g(1, 1) * tx
    return (top * (1 - ty) + bot * ty).astype(np.float32)


def corrupt(vals, levels, seed, r: Box):
    out = vals.copy()
    for c, lv in enumerate(levels):
        if lv != 0.0:
            out[c] = out[c] + np.float32(lv) * noise(seed, 201 + c, r, 1)[0]
    return out


# ----------------------------------------------------------------------------
# dense sampler (sampler.py:119-168 + store.py:338-354, 428-436, 549-554)

class Stage:
    """One sampler: steps, per-step (H, s, offset), Phi, seed, channels, eps.

    phi: callable(x, y, outer_step, win_box) -> Phi (window), or an analytic
    spec dict.  base: callable(Box) -> (C, h, w) pure base field, or None for
    seed noise.  cond: None or (scale, mask_channel, margin, feature_fn) where
    feature_fn(Box) gives the conditioning tensor over a coarse region.
    """

    def __init__(self, steps, layouts, phi, seed, channels=1, eps=0.01, dtype=np.float32,
                 base=None, cond=None, weights=None):
        self.steps = steps
        self.layouts = layouts if isinstance(layouts, (list, tuple)) and \
            isinstance(layouts[0], (list, tuple)) else [layouts] * steps
        self.phi = phi
        self.seed = seed
        self.C = channels
        self.eps = eps
        self.dtype = dtype
        self.base = base
        self.cond = cond
        self.weights = weights

    def lay(self, t):
        H, s = self.layouts[t][0], self.layouts[t][1]
        off = tuple(self.layouts[t][2:4]) if len(self.layouts[t]) >= 4 else (0, 0)
        return H, s, off

    def covers(self, r: Box, t0=0):
        regs = {t0: r}
        for t in range(t0, self.steps):
            H, s, off = self.lay(t)
            regs[t + 1] = cover(H, s, off, regs[t])
        return regs

    def base_values(self, r: Box):
        if self.base is None:
            return noise(self.seed, 0, r, self.C).astype(self.dtype)
        return np.asarray(self.base(r), dtype=self.dtype)

    def cond_region(self, r: Box, t0=0):
        """Coarse region the conditioning dependency reads for a query."""
        scale, _mc, margin, _fn = self.cond
        regs = self.covers(r, t0)
        need = None
        for t in range(t0, self.steps):
            H, s, off = self.lay(t)
            for k in kappa(H, s, off, regs[t]):
                q = win_box(H, s, off, *k).coarsen(scale).grow(margin)
                need = q if need is None else need.union(q)
        return need

    def run(self, r: Box, t0=0, cond_slab=None):
        """Step-t0 image over r (dict of every step image for inspection)."""
        regs = self.covers(r, t0)
        J = self.base_values(regs[self.steps])
        images = {self.steps: (J, regs[self.steps])}
        if self.cond is not None and cond_slab is None:
            creg = self.cond_region(r, t0)
            cond_slab = (self.cond[3](creg), creg)
        for t in reversed(range(t0, self.steps)):
            H, s, off = self.lay(t)
            W = (tent(H, self.eps) if self.weights is None else self.weights[t]).astype(self.dtype)
            out_r, src_r = regs[t], regs[t + 1]
            A = np.zeros((self.C, out_r.h, out_r.w), dtype=self.dtype)
            B = np.zeros((out_r.h, out_r.w), dtype=self.dtype)
            for (i, j) in kappa(H, s, off, out_r):
                win = win_box(H, s, off, i, j)
                x = J[:, win.y0 - src_r.y0:win.y1 - src_r.y0, win.x0 - src_r.x0:win.x1 - src_r.x0]
                y = None
                if self.cond is not None:
                    scale, mch, _m, _fn = self.cond
                    slab, sreg = cond_slab
                    y = conditioning(slab, sreg, scale, win, self.seed,
                                     mask=None if mch is None else slab[mch])
                if callable(self.phi):
                    d = self.phi(x, y, t + 1, win)
                else:
                    d = phi_analytic(self.phi, np.ascontiguousarray(x), y, t + 1)
                d = np.asarray(d).astype(self.dtype)
                ov = win.inter(out_r)
                ys = slice(ov.y0 - out_r.y0, ov.y1 - out_r.y0)
                xs = slice(ov.x0 - out_r.x0, ov.x1 - out_r.x0)
                wy = slice(ov.y0 - win.y0, ov.y1 - win.y0)
                wx = slice(ov.x0 - win.x0, ov.x1 - win.x0)
                A[:, ys, xs] += (W[None] * d)[:, wy, wx]
                B[ys, xs] += W[wy, wx]
            Jn = np.zeros_like(A)
            np.divide(A, B[None], out=Jn, where=B[None] > 0)
            J = Jn
            images[t] = (J, out_r)
        return images[t0][0], images


# ----------------------------------------------------------------------------
# hierarchy (pipeline.py:181-246)

def pipeline_dense(stages, seed, user_map_fn, r: Box):
    """stages: list of dicts (steps, window, stride, phi(spec dict or callable),
    scale, channels, eps, corruption, patch, cond_margin).  user_map_fn(Box,
    channels) -> f32 map.  Returns the finest stage's J_0 over r."""

    def make(k):
        st = stages[k]
        base = None
        if k == 0 and user_map_fn is not None:
            levels = st.get("corruption") or (0.0,) * st.get("channels", 1)
            base = lambda b, _st=st, _lv=levels: corrupt(  # noqa: E731
                user_map_fn(b, _st.get("channels", 1)), _lv, seed, b)
        cond = None
        if k > 0:
            prev = stages[k - 1]
            p = prev.get("patch", 4)
            parent_stage = make(k - 1)

            def feat(creg, _ps=parent_stage, _p=p):
                fine = Box(creg.x0 * _p, creg.y0 * _p, creg.w * _p, creg.h * _p)
                out, _ = _ps.run(fine)
                return patch_features(out[0], _p)

            cond = (st.get("scale", 1) * p, 2, st.get("cond_margin", 1), feat)
        return Stage(st["steps"], (st["window"], st["stride"]), st["phi"], seed + k,
                     channels=st.get("channels", 1), eps=st.get("eps", 0.01), base=base,
                     cond=cond)

    out, _ = make(len(stages) - 1).run(r)
    return out
