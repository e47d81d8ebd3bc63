"""profiles/r02/traffic.json (read by bench.py's roofline.traffic) from this
round's ncu --set full summaries of two tensor-core UNet launches, next to
each launch's algorithmic bytes (every input read once, every output written
once; 64 windows of 256^2, bf16).

python tools/traffic_json.py DIR > traffic.json   (DIR holds ncu_dec0c1_dyn_full.json,
                                                   ncu_dec1c2_full.json)
"""
import json
import os
import sys

W, B = 64, 2                      # windows per launch, bytes per bf16 element
PX0, PX1, PX2 = 256 * 256, 128 * 128, 64 * 64

LAUNCHES = [
    ("dec0c1_dyn", "dec0.0.c1", "conv_halo2_kernel<64, 2, 0, 1> (DYN)",
     W * (PX1 * 128 + PX0 * 64 + PX0 * 64) * B,
     "reads the 128-ch 128^2 decoder input once (upsampled inside the TMA load) and the "
     "64-ch 256^2 skip once, writes the 64-ch 256^2 h once"),
    ("dec1c2", "dec1.0.c2", "conv_halo2_kernel<128, 2, 0, 0>",
     W * (PX1 * 128 + PX2 * 128 + PX1 * 128 + 2 * PX1 * 128) * B,
     "reads h (128 ch) and the 256-ch block input of the fused 1x1 skip GEMM (half of it at "
     "64^2, upsampled in the TMA load) once, writes x and mp_silu(x) once"),
]


def entry(d, name, layer, kernel, alg, note):
    path = os.path.join(d, f"ncu_{name}_full.json")
    s = json.load(open(path))
    rd = s["dram_read"]["value"] * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}[s["dram_read"]["unit"]]
    wr = s["dram_write"]["value"] * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}[s["dram_write"]["unit"]]
    return {"layer": layer, "kernel": kernel, "windows": W, "algorithmic_bytes": alg,
            "algorithmic_note": note, "dram_read": int(rd), "dram_write": int(wr),
            "duration_us": s["duration"]["value"],
            "source": f"profiles/r02/ncu_{name}_full.json (ncu --set full, clock-control none)",
            "dram_bytes": int(rd + wr), "dram_over_algorithmic": round((rd + wr) / alg, 4),
            "per_launch": "one launch over 64 windows"}


d = sys.argv[1]
first, *rest = [entry(d, *spec) for spec in LAUNCHES]
first["other"] = rest
print(json.dumps(first, indent=1))
