#!/usr/bin/env python
"""Benchmark: instrumented fuzz execs/s of the B200 fuzzing inner loop.

Metric (BASELINE.json): fuzz execs/sec, one exec = parent pick + type-aware
mutation + one COMPUTE phase (execute, sanitize, cover) + triage, i.e. the
reference's ``compute_runs`` unit (campaign.py:648-652, 748).

Workload: C2 of SURVEY.md §8(d) — the tiled matmul target with
stride/size-argument OOB bugs (paper_2603_05725_b200/workloads/matmul.man),
master_seed 11, batched rounds of R = 2^20 inputs.  One step = one round.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--round R] [--impl ours|reference]

--impl reference times the reference's own CPU loop on all host cores, same
metric and workload: the unmodified reference ``fuzz_loop`` (installed offline
into baseline/_ref, which travels with the repo) in one process per core, or,
when that is absent, the CPU port of the loop (oracle/, test infrastructure).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "instrumented fuzz execs/sec"
UNIT = "execs/s"
WORKLOAD = "C2 tiled matmul 8x8x8, grid 2 x block 4, stride/size OOB (workloads/matmul.man), seed 11"


# ---------------------------------------------------------------- CPU reference arm


def _cpu_worker(workload, seed, round_size, counter, stop):
    """One process of the CPU baseline: the oracle port of the reference loop on the
    bench workload (the GPU arm's batched contract and round size), running until
    ``stop`` is set; every finished input increments the shared ``counter``."""
    from oracle.loop import batched_loop
    from paper_2603_05725_b200.workloads import load

    def on_exec():
        with counter.get_lock():
            counter.value += 1
        return stop.is_set()

    while not stop.is_set():
        batched_loop(load(workload), master_seed=seed, iterations=1 << 40, round_size=round_size,
                     keep_records=False, on_exec=on_exec)


class CpuPool:
    """``procs`` persistent CPU campaigns (one per host core).  ``window(s)`` counts
    the inputs all of them finish in ``s`` seconds of wall time, so a sample is
    bounded by the clock, not by the length of any one input (budget-bound matmul
    inputs take seconds each in Python); INIT happens before the first window."""

    def __init__(self, workload: str, round_size: int, procs: int | None = None):
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        self.procs = procs or os.cpu_count() or 1
        self.counter = ctx.Value("q", 0)
        self.stop = ctx.Event()
        self.ps = [ctx.Process(target=_cpu_worker, args=(workload, 11 + i, round_size, self.counter, self.stop),
                               daemon=True) for i in range(self.procs)]
        for q in self.ps:
            q.start()

    def count(self) -> int:
        with self.counter.get_lock():
            return self.counter.value

    def window(self, seconds: float):
        c0, t0 = self.count(), time.perf_counter()
        time.sleep(seconds)
        c1, t1 = self.count(), time.perf_counter()
        return c1 - c0, t1 - t0

    def close(self):
        self.stop.set()
        for q in self.ps:
            q.join(timeout=2)
            if q.is_alive():
                q.terminate()


def cpu_rate(workload: str, seconds: float, round_size: int, warm: float = 3.0):
    """Aggregate execs/s of the CPU baseline over one ``seconds`` window (after
    ``warm`` seconds of start-up: imports, INIT, first inputs)."""
    pool = CpuPool(workload, round_size)
    try:
        pool.window(warm)
        execs, wall = pool.window(seconds)
    finally:
        pool.close()
    return execs / wall, execs, wall, pool.procs


REF_PATH = REPO / "baseline" / "_ref"


def reference_available() -> bool:
    return (REF_PATH / "simt_forge" / "campaign.py").exists()


def _ref_worker(workload, seed, seconds, q):
    """One process of the reference arm: the reference's own fuzz_loop (public API,
    amortized, one worker) on the bench workload until its wall-clock limit
    (campaign.py:733-735); reports (compute_runs, wall_seconds)."""
    sys.path.insert(0, str(REF_PATH))
    from simt_forge import campaign as rc
    m = rc.load_harness(REPO / "paper_2603_05725_b200" / "workloads" / f"{workload}.man")
    s = rc.fuzz_loop(m, rc.CampaignConfig(master_seed=seed, iterations=10 ** 12, max_wall_seconds=seconds))
    q.put((s.compute_runs, s.wall_seconds))


def ref_rate(workload: str, seconds: float, procs: int | None = None):
    """Aggregate execs/s of the unmodified reference fuzz_loop in ``procs`` processes
    (master seeds 11, 12, ...), each one campaign of ``seconds`` (INIT included, as
    in the reference's own execs_per_second, campaign.py:648-652)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    procs = procs or os.cpu_count() or 1
    q = ctx.Queue()
    ps = [ctx.Process(target=_ref_worker, args=(workload, 11 + i, seconds, q), daemon=True) for i in range(procs)]
    for p in ps:
        p.start()
    res = [q.get(timeout=seconds + 600) for _ in ps]
    for p in ps:
        p.join(timeout=5)
    execs = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return execs / wall, execs, wall, procs


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(a):
    if reference_available() and not a.ref_port:
        return run_reference_fuzz_loop(a)
    return run_reference_port(a)


def run_reference_fuzz_loop(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # each step: one wall-clock-bounded reference campaign per host core, sized so the
    # whole --steps K --warmup W run takes a few minutes (3-10 s per step)
    sec = a.ref_seconds if a.ref_seconds else min(10.0, max(3.0, 150.0 / (a.steps + a.warmup)))
    per_step, total = [], 0
    for s in range(a.warmup + a.steps):
        rate, execs, wall, procs = ref_rate(a.workload, sec)
        if s >= a.warmup:
            per_step.append(wall)
            total += execs
    value = total / sum(per_step)
    sample = (f"unmodified reference fuzz_loop (baseline/_ref, amortized, 1 worker) on {a.workload}, one "
              f"{sec:.1f} s campaign per process per step, {procs} processes, master seeds 11..{10 + procs}; "
              f"CPU {_cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * statistics.mean(per_step),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_reference_port(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step = []
    total_execs = 0
    # each step is one window of the persistent CPU campaigns, sized so the whole
    # --steps K --warmup W run takes ~2 minutes (1-10 s per step)
    sec = a.ref_seconds if a.ref_seconds else min(10.0, max(1.0, 120.0 / (a.steps + a.warmup)))
    pool = CpuPool(a.workload, a.round)
    try:
        pool.window(3.0)                       # start-up: imports, INIT
        for s in range(a.warmup + a.steps):
            execs, wall = pool.window(sec)
            if s >= a.warmup:
                per_step.append(wall)
                total_execs += execs
    finally:
        pool.close()
    procs = pool.procs
    value = total_execs / sum(per_step)
    sample = (f"oracle port of the reference loop (batched contract, rounds of {a.round}) in {procs} processes, "
              f"{sec:.2f}s windows per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * statistics.mean(per_step),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- GPU arm


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML during the timed region
    (in-process: no nvidia-smi subprocesses contending with the run)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 0.05):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        # NVML is initialized here, before the timed region: nvmlInit takes driver
        # locks for tens of ms and stalled kernel launches when it ran inside it
        self._nv = self._h = self._mx = None
        if os.environ.get("SFG_BENCH_NO_NVML"):    # diagnostics: no sampling at all
            return
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nv = nv
        except Exception:
            self._nv = None

    def _run(self):
        nv, h, mx = self._nv, self._h, self._mx
        if nv is None:
            return
        while not self._stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)
        # NVML left initialized in the process was seen to stall later kernel launches
        # (end-to-end runs after the timed region 20-35 % slower in 2 of 5 runs)
        if self._nv is not None and not os.environ.get("SFG_BENCH_NVML_KEEP"):
            try:
                self._nv.nvmlShutdown()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({k for _, _, r in self.rows for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML"}


def run_ours(a):
    import paper_2603_05725_b200  # noqa: F401  (sets CUDA_DEVICE_MAX_CONNECTIONS before the context exists)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU; SFG_DIST_BACKEND=gloo lets several ranks share a GPU (tests of
    # the multi-rank path on a one-GPU box: collectives staged through host memory)
    backend = os.environ.get("SFG_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        dist.init_process_group(backend)
    from paper_2603_05725_b200.engine import DeviceCampaign
    from paper_2603_05725_b200.workloads import load

    from paper_2603_05725_b200.shard import RoundComm

    m = load(a.workload)
    D = a.depth
    # one campaign, each global round sharded over the ranks (R inputs per GPU per
    # round, weak scaling); per-round merge over NCCL
    comm = RoundComm()
    # weak (default): R inputs per GPU per round; strong: R inputs per round in total
    # (each rank R / N), so every N runs the same campaign (equal campaign digests)
    R = a.round if a.scaling == "strong" else a.round * world
    dc = DeviceCampaign(m, master_seed=11, comm=comm)
    dc.timing = True

    def all_streams_done(ev):
        cur = torch.cuda.current_stream()
        for sl in dc.slots:
            if sl is not None:
                cur.wait_stream(sl.stream)
        ev.record(cur)

    clock = ClockSampler(local % torch.cuda.device_count())   # NVML initialized outside the timed region
    it = 1
    dc.run_rounds(it, it + a.warmup * R, R, depth=D)
    it += a.warmup * R
    dc.reserve(D, a.round)     # all in-flight rounds' buffers exist before the timed region
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = dc.launches
    dc.exec_events.clear()
    fin = []                    # host clock at each round's finalization (diagnostics)
    with clock as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        t0.record()
        results = dc.run_rounds(it, it + a.steps * R, R, depth=D,
                                on_round=lambda res: fin.append((time.perf_counter() - h0, res.n_admitted,
                                                                 getattr(res.slot, "sub_host", h0) - h0)))
        all_streams_done(t1)
        torch.cuda.synchronize()
    it += a.steps * R
    launches = dc.launches - launches0
    digest = campaign_digest(dc)          # findings / coverage / corpus after the timed rounds
    executed = sum(r.executed for r in results)
    # K3 per round: bulk pass (every input, long ones deferred) and the whole execute
    bulk_ms = [s.elapsed_time(b) for s, b, e in dc.exec_events if b is not None]
    k3_ms = [s.elapsed_time(e) for s, b, e in dc.exec_events]
    t_local = t0.elapsed_time(t1) / 1000.0
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = executed / t_max
    ms = [t_max * 1000 / a.steps]


    # ---- dominant kernel roofline.  K3's bulk pass (sfg_jit_execute) runs every input
    # of the round; its algorithmic off-chip bytes are the child payload read once plus
    # the verdict and edge-count rows written.  It is bound by the
    # issue latency of each simulated thread's dependent instruction chain, not by HBM:
    # the HBM fraction is reported as measured, the issue figures beside it.
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    bulk_s = statistics.mean(bulk_ms) / 1000.0
    bytes_exec = dc.algorithmic_exec_bytes()
    achieved = bytes_exec * a.round / bulk_s / 1e9
    retired = dc.retired_mean(results[-1].slot)
    collectives = comm.calls
    prof = {}
    # ncu figures of the same kernels (tools/ncu_kernels.py on the latest capture)
    nk = REPO / "profiles" / "r02_ncu_kernels.json"
    ncu_k = json.loads(nk.read_text()) if nk.exists() else {}
    bulk_n = next((v for k, v in ncu_k.items() if "bulk" in k), None)
    tail_n = next((v for k, v in ncu_k.items() if "tail" in k), None)
    if bulk_n:
        b = bulk_n["ncu"]
        prof = {"dram_bytes_per_launch": bulk_n.get("traffic"), "source": bulk_n.get("traffic_source"),
                "issue_slots_busy_pct": b.get("issue_slots_busy_pct"),
                "active_threads_per_warp": b.get("active_threads_per_warp"),
                "warp_cycles_per_issued": None}
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": prof.get("dram_bytes_per_launch"), "kernel": "sfg_jit_execute (K3 bulk pass)",
            "bytes_per_exec": bytes_exec, "launch_ms": statistics.mean(bulk_ms),
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs (of measured)" if peaks else "fallback 6.65 TB/s (of fallback)"),
            "traffic_source": prof.get("source"),
            "note": "latency-bound dependent integer/branch chains per simulated thread; see issue_roofline"}
    sm_mhz = clk.summary().get("sm_mhz") or 1965.0
    issue = {"sim_instr_per_s": retired * R / (t_max / a.steps), "sim_instr_per_exec": retired,
             "bulk_ms_per_launch": statistics.mean(bulk_ms), "k3_ms_per_round": statistics.mean(k3_ms),
             "k3_ms_per_round_max": max(k3_ms), "rounds_in_flight": D, "soft_cap": dc.soft_cap,
             "ncu_issue_slots_busy_pct": prof.get("issue_slots_busy_pct"),
             "ncu_warp_cycles_per_issued": prof.get("warp_cycles_per_issued"),
             "ncu_active_threads_per_warp": prof.get("active_threads_per_warp"),
             "lane_instr_peak_per_s": 148 * 4 * 32 * sm_mhz * 1e6}
    # the long-input pass (sfg_jit_tail): most of the serialized kernel time, few SMs
    # at a time; same issue/latency bound (ncu figures of one launch run alone)
    tprof = {}
    if tail_n:
        t_ = tail_n["ncu"]
        tprof = {"duration_ns": t_.get("duration_ns"), "issue_slots_busy_pct": t_.get("issue_slots_busy_pct"),
                 "achieved_warps_per_sm": t_.get("achieved_warps_per_sm"), "dram_bytes_per_launch": tail_n.get("traffic"),
                 "warp_cycles_per_issued": None}
    issue["tail_pass"] = {"kernel": "sfg_jit_tail", "ms_per_round_after_bulk": statistics.mean(
        e - b for e, b in zip(k3_ms, bulk_ms)) if bulk_ms else None,
        "ncu_duration_ms_alone": (tprof.get("duration_ns") or 0) / 1e6 or None,
        "ncu_issue_slots_busy_pct": tprof.get("issue_slots_busy_pct"),
        "ncu_warp_cycles_per_issued": tprof.get("warp_cycles_per_issued"),
        "ncu_achieved_warps_per_sm": tprof.get("achieved_warps_per_sm"),
        "ncu_dram_bytes_per_launch": tprof.get("dram_bytes_per_launch")}

    # ---- per-kernel rooflines from an isolated pass: a few more rounds one at a time
    # (depth 1, nothing overlapping), CUDA events at every stage boundary
    kernels = stage_profile(dc, it, R, a, peaks, torch) if world == 1 else None
    if kernels:
        dom = max(kernels, key=lambda k: k["ms_per_round"])
        roof = {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                "frac": dom["achieved_gbs"] / hbm_peak, "traffic": dom.get("traffic"), "kernel": dom["kernel"],
                "bytes_per_exec": dom["bytes_per_exec"], "launch_ms": dom["ms_per_round"],
                "share_of_round": dom["share"],
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (of measured)" if peaks else "fallback 6.65 TB/s"),
                "traffic_source": dom.get("traffic_source"),
                "timing": "isolated pass: rounds one at a time after the timed region, CUDA events on the round's "
                          "stream around the stage",
                "note": dom.get("note", "")}

    # ---- end to end through the public API with host buffers (the device-timed
    # campaign's buffers go back to the allocator first)
    if os.environ.get("SFG_BENCH_TIMELINE"):
        with open(os.environ["SFG_BENCH_TIMELINE"], "w") as f:
            for k, ((s_, b_, e_), (h, adm, sub)) in enumerate(zip(dc.exec_events, fin)):
                f.write(f"{k} exec_start {t0.elapsed_time(s_):.1f} bulk_end {t0.elapsed_time(b_):.1f} "
                        f"tail_end {t0.elapsed_time(e_):.1f} host_final {h * 1e3:.1f} admitted {adm} "
                        f"host_submit {sub * 1e3:.1f}\n")
    dc.close()
    dc.slots.clear()
    dc._aux = None
    del results                 # round results hold their slots: free them all
    import gc
    gc.collect()
    e2e = run_e2e(a, m, torch, R, world)
    if world == 1 and not a.no_sequential:
        e2e["sequential_discipline"] = run_e2e_sequential(a, m, torch)
    if world == 1:
        e2e["dedupe_inputs"] = run_e2e_dedupe(a, m, torch, R)
    if world == 1 and not a.no_cold:
        # the child process needs the device memory this process's caching allocator holds
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        e2e["cold"] = run_e2e_cold(a, R, cache=True)
        e2e["cold_no_jit_cache"] = run_e2e_cold(a, R, cache=False)

    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu:
            if reference_available() and not a.ref_port:
                rate, execs, wall, procs = ref_rate(a.workload, a.cpu_seconds)
                cpu = {"value": rate, "unit": UNIT, "cores": procs, "kind": "reference",
                       "sample": f"unmodified reference fuzz_loop (baseline/_ref) on {a.workload}, one {a.cpu_seconds}"
                                 f" s campaign per process, {procs} processes, {execs} execs; CPU {_cpu_model()}"}
            else:
                rate, execs, wall, procs = cpu_rate(a.workload, a.cpu_seconds, a.round)
                cpu = {"value": rate, "unit": UNIT, "cores": procs, "kind": "port",
                       "sample": f"oracle port of the reference loop on {a.workload} (batched contract, rounds of "
                                 f"{a.round}) in {procs} processes, one {a.cpu_seconds}s window after 3 s of "
                                 f"start-up, {execs} execs; CPU {_cpu_model()}"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": t_max * 1000 / a.steps, "higher_is_better": True,
                "scaling": a.scaling, "vs_baseline": None, "dtype": "i32/f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "round_size": R, "execs_per_step": R,
                           "rounds_in_flight": D, "engine": "jit" if dc.jit else "interpreter",
                           "l2": f"inputs larger than L2: {D} rounds in flight hold ~{D * R * 1900 >> 20} MiB of "
                                 "round buffers (126 MB L2)", "parallelism": f"shard{world}",
                           "merge": f"per-round {backend.upper()} MIN/SUM all-reduce + all-gather ({collectives} collectives)"
                           if world > 1 else "none (1 GPU)"},
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "roofline": roof,
                "kernels": kernels, "issue_roofline": issue, "cpu_baseline": cpu, "campaign_digest": digest}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(a, m, torch, R, world):
    """The same metric end to end through the public API a user calls:
    ``campaign.fuzz_loop(manifest, CampaignConfig)`` (drop-in for the reference's
    ``fuzz_loop``, campaign.py:683), wall-clocked around the call.  Its host<->device
    traffic is counted from the tensors the campaign copies: program tables, the
    post-INIT baseline image and the seed corpus up; every round's verdict scalars,
    dedupe-key counts and new findings / admissions down."""
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    import torch.distributed as dist
    # a campaign long enough that pipeline fill/drain (the first rounds run at a low
    # speculation depth, one slowest-round latency at either end, ~0.2 s on C2) does
    # not dominate: four times the timed steps, at least 96 rounds
    steps = max(4 * a.steps, 96)
    cfg = CampaignConfig(master_seed=11, iterations=steps * R, round_size=R, pipeline_depth=a.depth,
                         distributed=world > 1)
    # three whole campaigns, the median reported (a ~0.4 s campaign sees sporadic
    # host-side stalls: one run in several is up to 2x slower); all three listed
    runs = []
    for _ in range(3):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        s = fuzz_loop(m, cfg)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = torch.tensor([wall], dtype=torch.float64,
                         device="cuda" if os.environ.get("SFG_DIST_BACKEND", "nccl") == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        runs.append((float(t.item()), s))
    wall, s = sorted(runs, key=lambda r: r[0])[1]
    tr = s.device_transfer
    return {"value": s.compute_runs / wall, "unit": UNIT, "h2d_bytes_per_step": tr["h2d_bytes"] / steps,
            "d2h_bytes_per_step": tr["d2h_bytes"] / steps, "wall_s": wall, "execs": s.compute_runs, "rounds": steps,
            "campaigns": [r[1].compute_runs / r[0] for r in runs], "reported": "median of the 3 campaigns",
            "api": "campaign.fuzz_loop(manifest, CampaignConfig) -> CampaignSummary",
            "includes": "program build (JIT cache hit), INIT baseline, corpus upload, all rounds, result objects",
            "findings_unique": len(s.findings), "stop": s.stop_reason, "setup_s": tr.get("setup_s")}


def campaign_digest(dc) -> dict:
    """sha256 of the campaign state: findings.txt, coverage.rec and the corpus ids
    (equal across GPU counts with --scaling strong; tests/test_bench_parity.py pins
    the same state against the reference for the first rounds)."""
    import hashlib
    from paper_2603_05725_b200.coverage import build_report, report_to_rec
    findings = dc.findings.render_text()
    cov = report_to_rec(build_report(dc.coverage_map()))
    corpus = "\n".join(e[0].id for e in dc.host_entries)
    h = hashlib.sha256((findings + "\0" + cov + "\0" + corpus).encode()).hexdigest()
    return {"sha256": h, "findings_unique": len(dc.findings), "findings_total": dc.findings.total,
            "corpus": len(dc.host_entries), "rounds": dc.rounds}


# algorithmic off-chip bytes per exec of each stage: what the stage
# must read and write given its inputs and outputs, not what the layout moves
def _stage_bytes(dc):
    from paper_2603_05725_b200.lowering import CHILD, VAL, VERDICT
    seed = dc.host_entries[0][0]
    payload = sum(len(v.data) for v in seed.args if hasattr(v, "data"))
    scalars = 4 * sum(1 for v in seed.args if not hasattr(v, "data"))
    E = dc.E
    return {
        "K1 sfg_plan + sfg_mutate (+ scans)": (2 * dc.n_args * VAL.itemsize + CHILD.itemsize,
                                               "parent value descriptors read, child record + descriptors "
                                               "written (the stage's own layout: 64-B descriptors)"),
        "K2 sfg_apply": (2 * payload, "parent payload read + child work region written"),
        "sfg_order (3 kernels)": (8 + dc.n_args * VAL.itemsize, "descriptors read, bucket + position written"),
        "K3 bulk sfg_jit_execute": (payload + scalars + 64 + 4 * ((E + 31) // 32),
                                    "child payload read once + 64-B verdict + hit bitmap (SURVEY.md §8(d))"),
        "K2+K3 bulk sfg_jit_execute (payload build fused)": (
            payload + scalars + 64 + 4 * ((E + 31) // 32),
            "parent payload read once (the child's is built in the pass) + 64-B verdict + hit bitmap "
            "(SURVEY.md §8(d))"),
        "K3 tail sfg_apply + sfg_jit_tail": (payload + scalars + 64 + 4 * ((E + 31) // 32),
                                             "as the bulk pass, for the deferred inputs; per round input"),
        "K4 triage (stop/absorb/admit + scans)": (VERDICT.itemsize + 4 * E + 24,
                                                  "verdict + edge-count row read, admission / alloc words written"),
    }


def stage_profile(dc, it, R, a, peaks, torch):
    """Each stage's device time per round with nothing overlapping: ``a.profile_rounds``
    rounds run one at a time (depth 1) after the timed region."""
    bulk = "K2+K3 bulk sfg_jit_execute (payload build fused)" if dc.fuse_apply else "K3 bulk sfg_jit_execute"
    pairs = [("submit", "mutated", "K1 sfg_plan + sfg_mutate (+ scans)")] + \
        ([] if dc.fuse_apply else [("mutated", "applied", "K2 sfg_apply")]) + \
        [("applied", "ordered", "sfg_order (3 kernels)"), ("ordered", "bulk", bulk),
             ("bulk", "tail", "K3 tail sfg_apply + sfg_jit_tail"),
             ("triage_start", "triaged", "K4 triage (stop/absorb/admit + scans)")]
    dc.stage_marks = []
    dc.run_rounds(it, it + a.profile_rounds * R, R, depth=1)
    torch.cuda.synchronize()
    marks = {}
    for ri, name, ev in dc.stage_marks:
        marks.setdefault(ri, {})[name] = ev          # last mark of a stage wins (re-runs)
    dc.stage_marks = None
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    sizes = _stage_bytes(dc)
    ncu = {}
    nf = REPO / "profiles" / "r02_ncu_kernels.json"
    if nf.exists():
        ncu = json.loads(nf.read_text())
    out = []
    for s0, s1, label in pairs:
        ms = [m[s0].elapsed_time(m[s1]) for m in marks.values() if s0 in m and s1 in m]
        if not ms:
            continue
        t = statistics.mean(ms)
        bpe, what = sizes[label]
        gbs = bpe * R / (t / 1000.0) / 1e9 if t > 0 else 0.0
        k = {"kernel": label, "ms_per_round": t, "bytes_per_exec": bpe, "bytes_note": what,
             "achieved_gbs": gbs, "hbm_frac": gbs / hbm, "rounds": len(ms)}
        if "bulk" in label:
            k["note"] = ("issue / latency bound: each lane runs its input's simulated threads' dependent chains "
                         "(issue_roofline); DRAM traffic above the algorithmic bytes is the 64-B argument "
                         "descriptors read (9 x 64 B per input on C2) and the lane's allocator tables in local memory")
        n = ncu.get(label)
        if n:
            k.update(n)
        out.append(k)
    total = sum(k["ms_per_round"] for k in out)
    for k in out:
        k["share"] = k["ms_per_round"] / total if total else None
    return out


def run_e2e_dedupe(a, m, torch, R):
    """Informational, not the headline: the same campaign with the opt-in
    CampaignConfig(dedupe_inputs=True) -- children of a round with the same parent
    and the same set of ops run once and share the verdict (identical results, fewer
    executions than inputs)."""
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    steps = max(4 * a.steps, 96)
    cfg = CampaignConfig(master_seed=11, iterations=steps * R, round_size=R, pipeline_depth=a.depth,
                         dedupe_inputs=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = fuzz_loop(m, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"value": s.compute_runs / wall, "unit": UNIT, "wall_s": wall, "execs": s.compute_runs,
            "note": "opt-in dedupe_inputs=True: duplicate children share one execution (not the headline)",
            "api": "campaign.fuzz_loop(manifest, CampaignConfig(dedupe_inputs=True))"}


def run_e2e_sequential(a, m, torch):
    """fuzz_loop with discipline="sequential": the reference fuzz_loop's own stream
    discipline (one worker stream, live corpus), byte-identical output directories
    (tests/test_gpu_parity.py), on the same workload and round size: children
    generated in parallel from the worker stream (seqgen), rounds chained
    speculatively on the device and cut after each admission."""
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    iters = a.sequential_execs
    cfg = CampaignConfig(master_seed=11, iterations=iters, round_size=a.round, discipline="sequential")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = fuzz_loop(m, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"value": s.compute_runs / wall, "unit": UNIT, "wall_s": wall, "execs": s.compute_runs,
            "rounds": s.device_transfer["rounds"], "corpus_interesting": s.corpus.interesting,
            "api": "campaign.fuzz_loop(manifest, CampaignConfig(discipline='sequential'))"}


def run_e2e_cold(a, R, cache: bool):
    """fuzz_loop in a fresh process (CUDA context, program build, allocation of the
    round buffers all inside the measurement).  cache=False: an empty JIT cubin cache,
    so the NVRTC compile of the specialized kernels is included as well."""
    import tempfile
    env = dict(os.environ)
    tmp = None
    if not cache:
        tmp = tempfile.mkdtemp(prefix="sfg_jit_cold_")
        env["SFG_JIT_CACHE"] = tmp
    cmd = [sys.executable, str(REPO / "bench.py"), "--e2e-cold-child", "--round", str(R), "--depth", str(a.depth),
           "--workload", a.workload, "--steps", str(a.steps)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        return json.loads(line[-1]) if line else {"error": r.stderr[-400:]}
    except Exception as e:  # noqa: BLE001 - reported, not fatal to the bench line
        return {"error": str(e)}


def e2e_cold_child(a):
    t_proc = time.perf_counter()
    import torch
    import paper_2603_05725_b200  # noqa: F401
    from paper_2603_05725_b200 import _native
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    from paper_2603_05725_b200.workloads import load
    t0 = time.perf_counter()
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    t_ctx = time.perf_counter() - t0
    steps = max(2 * a.steps, 48)
    m = load(a.workload)
    s = fuzz_loop(m, CampaignConfig(master_seed=11, iterations=steps * a.round, round_size=a.round,
                                    pipeline_depth=a.depth))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(json.dumps({"value": s.compute_runs / wall, "unit": UNIT, "wall_s": wall, "execs": s.compute_runs,
                      "context_s": t_ctx, "setup_s": s.device_transfer.get("setup_s"),
                      "import_s": t0 - t_proc, **_native.jit_stats(),
                      "includes": "CUDA context, program build (NVRTC or on-disk cubin cache), INIT baseline, "
                                  "round-buffer allocation, all rounds, result objects (python/torch import excluded)"}))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=96)
    p.add_argument("--warmup", type=int, default=3)
    # one round = 2^20 inputs (BASELINE.json configs[1]: 1M execs on 1 B200): a round's
    # latency is its slowest input (~15 ms), so larger rounds amortize pipeline fill /
    # drain over more work (R = 2^18 / 2^19 / 2^20: 90 / 103 / 110 M execs/s, 20 steps)
    p.add_argument("--round", type=int, default=1 << 20)
    p.add_argument("--depth", type=int, default=24, help="rounds in flight (speculative pipelining); at most "
                   "~30 so that every round's stream has its own hardware queue (CUDA_DEVICE_MAX_CONNECTIONS=32)")
    p.add_argument("--workload", default="matmul")
    p.add_argument("--profile-rounds", type=int, default=4, help="rounds of the isolated per-kernel pass")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--ref-seconds", type=float, default=0.0,
                   help="seconds per process per reference step (default: 120 s / (steps + warmup), 1-10 s)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--ref-port", action="store_true", help="reference arm / CPU baseline: the oracle port even "
                   "when the reference is installed in baseline/_ref")
    p.add_argument("--no-cold", action="store_true", help="skip the cold-process end-to-end runs")
    p.add_argument("--no-sequential", action="store_true", help="skip the sequential-discipline e2e run")
    p.add_argument("--sequential-execs", type=int, default=1 << 25)
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: --round inputs per GPU per round; strong: --round inputs per round over all GPUs "
                        "(the same campaign at every N)")
    p.add_argument("--e2e-cold-child", action="store_true", help=argparse.SUPPRESS)
    a = p.parse_args()
    if a.e2e_cold_child:
        e2e_cold_child(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
