"""Condense an ncu --set full report (one launch) into the figures the bench line and
DESIGN.md cite: duration, DRAM bytes, issue activity, occupancy, divergence.
Usage: python tools/ncu_summary.py <rep.ncu-rep> <out.json> [source-tag]"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
tag = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))


def num(k):
    v = m.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


dur_ns = num("gpu__time_duration.sum")
unit = dict(zip(hdr, units)).get("gpu__time_duration.sum", "")
dur_ns *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
u = dict(zip(hdr, units))


def to_bytes(v, k):
    s = u.get(k, "byte")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(s, 1)


summary = {
    "kernel": m.get("Kernel Name"),
    "source": tag,
    "duration_ns": dur_ns,
    "dram_bytes_read": to_bytes(rd, "dram__bytes_read.sum") if rd is not None else None,
    "dram_bytes_write": to_bytes(wr, "dram__bytes_write.sum") if wr is not None else None,
    "registers_per_thread": num("launch__registers_per_thread"),
    "grid": m.get("launch__grid_size"), "block": m.get("launch__block_size"),
    "issue_slots_busy_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "warp_cycles_per_issued": num("smsp__average_warps_issue_stalled_per_issue_active.ratio") or num(
        "smsp__average_warp_latency_per_inst_issued.ratio"),
    "inst_executed": num("smsp__inst_executed.sum"),
    "thread_inst_executed": num("sass__thread_inst_executed_true_per_opcode"),
    "achieved_warps_per_sm": num("sm__warps_active.avg.per_cycle_active"),
    "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
}
if summary["inst_executed"] and summary["thread_inst_executed"]:
    summary["active_threads_per_warp"] = summary["thread_inst_executed"] / summary["inst_executed"]
if summary["dram_bytes_read"] is not None and summary["dram_bytes_write"] is not None:
    summary["dram_bytes_per_launch"] = summary["dram_bytes_read"] + summary["dram_bytes_write"]
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
