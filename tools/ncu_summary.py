"""Summarise one kernel of an ncu --set full report as JSON (for profiles/).

python tools/ncu_summary.py report.ncu-rep [--kernel-index 0] [--label TEXT] > out.json

Keeps the numbers the DESIGN / bench roofline cite: duration, DRAM bytes and
throughput, tensor-pipe and issue utilisation, occupancy, the top warp-stall
reasons, and the SASS mnemonics that prove tcgen05 / TMA are in use.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active":
        "tensor_pipe_active_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_mem_active_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed":
        "tensor_active_realtime_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    idx = int(sys.argv[sys.argv.index("--kernel-index") + 1]) if "--kernel-index" in sys.argv else 0
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else ""
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2 + idx]
    out = {"report": rep.split("/")[-1], "label": label}
    stalls = []
    for k, u, v in zip(hdr, units, data):
        if k == "Kernel Name":
            out["kernel"] = v
        if k in KEYS:
            try:
                out[KEYS[k]] = {"value": float(v.replace(",", "")), "unit": u}
            except ValueError:
                out[KEYS[k]] = v
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    out["top_stalls"] = [{"reason": k, "share": round(s / tot, 3)}
                         for s, k in sorted(stalls, reverse=True)[:6]]
    sass = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    mn = {}
    for tag in ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTCBAR", "LDTM", "STTM", "HMMA",
                "MUFU.EX2", "SYNCS"):
        mn[tag] = sass.count(tag)
    out["sass_mnemonic_lines"] = mn
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
