"""Per-layer roofline table from an ncu launch list of tools/prof_step.py.

python tools/layer_table.py launches.csv [--windows 64]

Matches the launches of the LAST UNet forward to the layer program and prints,
per launch: time, algorithmic TFLOP/s, minimal HBM bytes (activations in/out,
residual), and the max(tensor, HBM) bound time using MEASURED_PEAKS.json.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.unet import UNetConfig, build_program  # noqa: E402


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
            out.append((d["Kernel Name"].split("(")[0], v))
    return out


def layer_ops(cfg, win):
    """Expected launch sequence of one forward: (kind, name, h, cin, cout, taps, outs, res[,
    rd]) -- rd, when given, is the input channels read per output pixel (a source read
    2x upsampled inside the TMA load counts a quarter of its channels)."""
    prog = build_program(cfg)
    ch = cfg.channels()
    fused = unet.FUSED_STEM
    seq = [] if fused else [("gather", "gather", win, 0, cfg.cin_pad, 0, 1, 0)]
    h = win
    c = ch[0]
    pooled = False
    up = False        # the next decoder block reads its low-res inputs upsampled in the TMA load
    for k, op in enumerate(prog.ops):
        nxt = prog.ops[k + 1][0] if k + 1 < len(prog.ops) else None
        c2_outs = 1 if nxt in ("attn", "out") else 2     # unet.forward_after_stem
        if op[0] == "stem":
            # fused: reads the f32 source plane(s), writes x_noisy (f32) + x/xa
            seq.append(("conv", "stem", h, cfg.cin_pad, ch[0], 1, 2, 0))
        elif op[0] == "enc":
            nm, has_skip = op[1], op[2]
            c1 = prog.convs[nm + ".c1"]
            seq.append(("conv", nm + ".c1", h, c1.cin, c1.cout, 9, 1, 0))
            c2 = prog.convs[nm + ".c2"]
            # the 2x2 pool written by the c2 epilogue (unet._fusable_pool): two more
            # outputs at a quarter of the pixels, no separate pool launch
            pooled = bool(unet.FUSED_POOL and nxt == "down" and h % 128 == 0
                          and c2.cout in (64, 128))
            # c2 with the fused skip GEMM: reads the block input (c1.cin) once more
            seq.append(("conv", nm + ".c2", h, c2.cin, c2.cout, 9, c2_outs + 0.5 * pooled,
                        c1.cin / c2.cout))
            c = c2.cout
        elif op[0] == "attn":
            nm = op[1]
            if unet.FUSED_QKV and c == 256:          # one ig_conv_qkv launch
                seq.append(("conv", nm + ".qkv", h, c, 3 * c, 1, 1, 0))
            else:
                for j in "qkv":
                    seq.append(("conv", f"{nm}.{j}", h, c, c, 1, 1, 0))
            seq.append(("attn", nm + ".attn", h, c, 0, 0, 0, 0))
            seq.append(("conv", nm + ".proj", h, c, c, 1, 2, 1))
        elif op[0] == "down":
            if not pooled:
                seq.append(("pool", "down", h, c, 0, 0, 0, 0))
            pooled = False
            h //= 2
        elif op[0] == "dec":
            nm = op[1]
            c1 = prog.convs[nm + ".c1"]
            sk = c1.cin - c                                  # skip-connection channels
            rd1 = (c / 4 if up else c) + sk                  # x (maybe low-res) + skip
            seq.append(("conv", nm + ".c1", h, c1.cin, c1.cout, 9, 1, 0, rd1))
            c2 = prog.convs[nm + ".c2"]
            seq.append(("conv", nm + ".c2", h, c2.cin, c2.cout, 9, c2_outs, c1.cin / c2.cout,
                        c2.cin + rd1))
            c = c2.cout
            up = False
        elif op[0] == "up":
            if not (unet.FUSED_UP and (2 * h) % 128 == 0):   # else folded into the TMA loads
                seq.append(("up", "up.x", h, c, 0, 0, 0, 0))
                seq.append(("up", "up.xa", h, c, 0, 0, 0, 0))
            else:
                up = True
            h *= 2
        elif op[0] == "out":
            if unet.FUSED_OUT and h % 4 == 0 and h % 128 == 0:
                # mma.sync head: real cout = data_channels; writes Phi (f32)
                seq.append(("conv", "out_head", h, ch[0], cfg.data_channels, 9, 0, 0))
            else:
                seq.append(("conv", "out", h, ch[0], 16, 9, 1, 0))
                seq.append(("output", "output", h, 0, 0, 0, 0, 0))
    return seq


def main():
    path = sys.argv[1]
    n = int(sys.argv[sys.argv.index("--windows") + 1]) if "--windows" in sys.argv else 64
    cfg = UNetConfig()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    tf, bw = peaks["bf16_tflops_sustained"] * 1e12, peaks["hbm_gbs"] * 1e9
    L = [x for x in launches(path) if not x[0].startswith("void at::")]
    seq = layer_ops(cfg, 256)
    last = L[-len(seq):]
    tot_t = tot_b = 0.0
    print(f"{'layer':14s} {'kernel':28s} {'us':>8s} {'TF/s':>7s} {'GB/s':>7s} {'bound_us':>8s} {'eff':>5s}")
    for (kind, name, h, cin, cout, taps, outs, res, *rd), (kname, us) in zip(seq, last):
        px = n * h * h
        fl = 2.0 * px * cin * cout * taps if kind == "conv" else 0.0
        if kind == "attn":             # q k^T + p v per window: 4 N^2 C
            fl = 4.0 * n * (h * h) ** 2 * cin
        if kind == "conv":
            by = px * 2 * ((rd[0] if rd else cin + cout * res) + cout * outs)
        elif kind in ("attn", "attn_prep"):
            by = px * 2 * cin * 4
        elif kind == "up":
            by = px * 2 * cin * 5            # read h^2 c, write (2h)^2 c
        elif kind == "pool":
            by = px * 2 * cin * 1.5          # read x, write pool(x) and its mp_silu
        else:
            by = 0.0
        bound = max(fl / tf, by / bw) * 1e6
        tot_t += us
        tot_b += bound
        print(f"{name:14s} {kname[-28:]:28s} {us:8.1f} {fl / us / 1e6:7.1f} {by / us / 1e3:7.0f} "
              f"{bound:8.1f} {bound / us if us else 0:5.2f}")
    print(f"total {tot_t:.1f} us, sum of per-layer bounds {tot_b:.1f} us ({tot_b / tot_t:.2f})")


if __name__ == "__main__":
    main()
