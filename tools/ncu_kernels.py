"""Condense an ncu --set full report holding several pipeline kernels (one or more
launches each) into per-stage figures for bench.py's ``kernels`` list:
duration, DRAM bytes, issue activity, occupancy, lane efficiency, L2 atomics.

Usage: python tools/ncu_kernels.py <rep.ncu-rep> <out.json> [source-tag]

Stage labels match bench.py ``stage_profile``; a stage's figures are those of the
first launch of its kernel(s) after the report's start (the first sfg_apply_kernel
launch of a round is K2, later ones re-materialize deferred inputs for the tail)."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
tag = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
U = dict(zip(hdr, units))


def num(m, k):
    v = m.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def scaled(m, k):
    v = num(m, k)
    if v is None:
        return None
    s = U.get(k, "")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "nsecond": 1, "us": 1e3,
                "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(s, 1)


def figures(m):
    f = {"duration_ns": scaled(m, "gpu__time_duration.sum"),
         "dram_bytes_read": scaled(m, "dram__bytes_read.sum"), "dram_bytes_write": scaled(m, "dram__bytes_write.sum"),
         "registers_per_thread": num(m, "launch__registers_per_thread"),
         "grid": m.get("launch__grid_size"), "block": m.get("launch__block_size"),
         "issue_slots_busy_pct": num(m, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
         "inst_executed": num(m, "smsp__inst_executed.sum"),
         "thread_inst_executed": num(m, "sass__thread_inst_executed_true_per_opcode"),
         "achieved_warps_per_sm": num(m, "sm__warps_active.avg.per_cycle_active"),
         "dram_throughput_pct": num(m, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
         "l2_atom_sectors": num(m, "lts__t_sectors_srcunit_tex_op_atom.sum"),
         "l2_red_sectors": num(m, "lts__t_sectors_srcunit_tex_op_red.sum"),
         "l2_atom_requests": num(m, "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum"),
         "l2_red_requests": num(m, "lts__t_requests_srcunit_tex_op_red.sum")}
    if f["inst_executed"] and f["thread_inst_executed"]:
        f["active_threads_per_warp"] = f["thread_inst_executed"] / f["inst_executed"]
    if f["dram_bytes_read"] is not None and f["dram_bytes_write"] is not None:
        f["traffic"] = f["dram_bytes_read"] + f["dram_bytes_write"]
    return f


launches = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
fused = "unfused" not in sys.argv[4:]    # K2 built inside the bulk pass (the default engine)
BULK = "K2+K3 bulk sfg_jit_execute (payload build fused)" if fused else "K3 bulk sfg_jit_execute"
K4 = "K4 triage (stop/absorb/admit + scans)"
stages = {}
seen_apply = False
for m in launches:
    name = m.get("Kernel Name", "").split("(")[0]
    if name.startswith("sfg_plan_kernel") or name.startswith("sfg_mutate"):
        label = "K1 sfg_plan + sfg_mutate (+ scans)"
    elif name.startswith("sfg_apply"):
        label = "K2 sfg_apply" if not (seen_apply or fused) else None   # later launches: the tail's re-materialize
        seen_apply = True
    elif name == "sfg_jit_execute":
        label = BULK
    elif name == "sfg_jit_tail":
        label = "K3 tail sfg_apply + sfg_jit_tail"
    elif name in ("sfg_stop_kernel", "sfg_absorb_kernel", "sfg_admit_kernel"):
        label = K4
    elif name.startswith("sfg_seq_walk"):
        label = "seqgen walk (candidate successors)"
    elif name.startswith("sfg_seq_mutate"):
        label = "seqgen mutate (children from their start positions)"
    else:
        label = None
    if label is None:
        continue
    f = figures(m)
    f["ncu_kernel"] = name
    prev = stages.get(label)
    if prev is None:
        stages[label] = f
    elif (label.startswith("K1") or label == K4) and name not in prev["ncu_kernel"].split(" + "):
        # plan + mutate, stop + absorb + admit: sum the kernels of the stage
        for k in ("duration_ns", "dram_bytes_read", "dram_bytes_write", "traffic", "l2_atom_sectors",
                  "l2_red_sectors"):
            if prev.get(k) is not None and f.get(k) is not None:
                prev[k] += f[k]
        prev["ncu_kernel"] += " + " + name
out_d = {}
for label, f in stages.items():
    out_d[label] = {"traffic": f.get("traffic"), "traffic_source": f"ncu --set full --clock-control none ({tag})",
                    "ncu": f}
json.dump(out_d, open(out, "w"), indent=1)
print(json.dumps(out_d, indent=1))
