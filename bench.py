#!/usr/bin/env python3
"""Benchmark of the B200 REI hot path (BASELINE.json metric: candidate REs/sec and
time-to-minimal-RE on the hardest benchmark).

Default workload (BASELINE configs[4], the paper's hardest known-spec class):
Table 1 row 1 = the Section 5 specification, binary alphabet,
cost homomorphism (1,1,1,1,1); one *step* = one full ``rei_solve`` from level 1 to
the first level holding a precise CS (c* = 28), i.e. one pass of every
hot-path row (Q, S, concat, union, precision test, dedup, append, reconstruction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With N > 1 (``--gpus N`` spawns its ranks with torch.distributed.run, or runs under
torchrun) the ranks run ONE sharded search (every large level's work
lists are partitioned across ranks; the CSs new to a rank go to their hash owners by
NCCL all-to-all, the owners deduplicate, the uniques are all-gathered; small levels
run on every rank; "scaling": "strong"); ``--multi replicas`` runs N independent
searches instead ("scaling": "weak").  Time is the max over ranks.  At N = 1 the line
also carries a ``secondary`` measurement of BASELINE configs[1] (c2-t1-s0, the HBM
hash set).
``--impl reference`` times the CPU oracle (oracle/, the only reference this tier
has) on a bounded sample.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import specgen  # noqa: E402

# ------------------------------------------------------------------ workloads

WORKLOADS = {
    # name: (spec, max_cost, description)
    "table1-row1": (specgen.TABLE1_ROW1, 40,
                    "Table 1 row 1 / Section 5 spec (P:1345, P:1779-1782), costs (1,1,1,1,1), "
                    "solve to the minimal precise regex (c*=28, P:1798)"),
    "table1-row8": (specgen.TABLE1_ROW8, 400,
                    "Table 1 row 8 (P:1352): same spec, costs (10,10,10,1,10), solve to c*"),
    "c1-toy": (specgen.C1_TOY, 40, "BASELINE configs[0] paper-style toy"),
    "c2-t1-s0": (specgen.gen_type1("01", 6, 10, 10, 0), 40,
                 "BASELINE configs[1]: Type 1 (P:1239-1242) binary, le=6, p=n=10, SplitMix64 seed 0 "
                 "(|IC|=58, two-word CS, 64-bit-key hash set)"),
    "c2-t1-s3": (specgen.gen_type1("01", 6, 10, 10, 3), 40,
                 "BASELINE configs[1]: Type 1 binary, le=6, p=n=10, seed 3 (|IC|=55)"),
    "c3-planted-s1": (specgen.gen_planted("01", "(0+1)*1(0+1)(0+1)(0+1)", 10, 10, 6, 10, 1), 40,
                      "BASELINE configs[2]: planted binary target (DESIGN.md recipe), |IC|=115 (two-u64 CS, "
                      "indexed hash set), unit costs (c*=18)"),
    "c3-planted-s1-nu": (specgen.gen_planted("01", "(0+1)*1(0+1)(0+1)(0+1)", 10, 10, 6, 10, 1,
                                             costs=(20, 20, 20, 5, 30)), 800,
                         "BASELINE configs[2]: the same spec, non-uniform costs (20,20,20,5,30) (P:1356 style), "
                         "c*=325, 1.2e9 candidates"),
    "c4-planted-s0": (specgen.gen_planted("abcd", "(a+b+c)*d(a+c)(b+d)", 10, 10, 4, 8, 0), 40,
                      "BASELINE configs[3]: planted 4-symbol target, |IC|=148 (256-bit CS), unit costs (c*=16), "
                      "5e8 candidates"),
    "c3-big": (specgen.gen_planted("01", "(0+1)*0(0+1)(0+1)(0+1)(0+1)", 10, 10, 6, 10, 2, costs=(20, 20, 20, 5, 30)),
               800, "BASELINE configs[2] at throughput scale: planted binary target, |IC|=103 (128-bit CS), costs "
                    "(20,20,20,5,30) (P:1356 style), c*=375, 1.45e10 candidates, 1.7e9 cached CSs"),
    "c4-big": (specgen.gen_planted("abcd", "(a+b+c)*d(a+c)(b+d)", 10, 10, 6, 10, 1, costs=(20, 20, 20, 5, 30)),
               800, "BASELINE configs[3] at throughput scale: planted 4-symbol target, |IC|=188 (256-bit CS), costs "
                    "(20,20,20,5,30), c*=315, 1.26e10 candidates, 8e8 cached CSs"),
    "c2-t2-s4": (specgen.gen_type2("01", 6, 10, 10, 4), 40,
                 "BASELINE configs[1]: Type 2 (P:1244-1253) binary, le=6, p=n=10, seed 4 "
                 "(|IC|=48, c*=25, ~2.7e10 candidates, 1.5e9 cached CSs)"),
}
# Paper numbers for the same workload on its own hardware (context):
PAPER = {
    "table1-row1": {"reps": 26774099142, "gpu_s": 4.9512, "cpu_s": 5080.7850,
                    "hw": "Colab A100-SXM4-40GB (P:1147-1153)"},
    "table1-row8": {"reps": 23349552935, "gpu_s": 4.9096, "cpu_s": 4519.9456,
                    "hw": "Colab A100-SXM4-40GB (P:1147-1153)"},
}
ORACLE_SAMPLE_COST = {"table1-row1": 18, "table1-row8": 150, "c1-toy": 8, "c2-t1-s0": 16, "c2-t1-s3": 16,
                      "c2-t2-s4": 16, "c3-planted-s1": 13, "c3-planted-s1-nu": 245, "c4-planted-s0": 11,
                      "c3-big": 245, "c4-big": 230}
# cpu_baseline sample
REFERENCE_STEP_COST = {"table1-row1": 16, "table1-row8": 140, "c1-toy": 8, "c2-t1-s0": 14, "c2-t1-s3": 14,
                       "c2-t2-s4": 14, "c3-planted-s1": 12, "c3-planted-s1-nu": 230, "c4-planted-s0": 10,
                       "c3-big": 230, "c4-big": 215}
# --impl reference step

METRIC = "candidate REs/sec"
UNIT = "cand/s"

# Algorithmic integer lane-ops per candidate (SURVEY 8(d) model):
#   union  ~ 7*W32 + 12   (OR, precision test, hash/probe address, compare)
#   concat ~ union + S_in_active/32 + 2*W32 (bit-sliced fold + epsilon terms)
def ops_per_candidate(kind: str, w32: int, s_in: int) -> float:
    base = 7 * w32 + 12
    if kind == "concat":
        return base + (s_in / 2) / 32 + 2 * w32
    return base


THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"rei_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            if bits & 0x1:  # idle samples are not "under load"
                continue
            sm.append(s)
            mx.append(m)
            for b, name in THROTTLE_BITS.items():
                if bits & b:
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def reduce_over_ranks(total_ms, cands, device, world, sum_work=True):
    """Device time = max over ranks; work = sum over ranks (replicas) or rank 0's
    (sharded: every rank reports the same global candidate count)."""
    if world <= 1:
        return float(total_ms), float(cands)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(total_ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([float(cands)], dtype=torch.float64, device=device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM if sum_work else dist.ReduceOp.MAX)
    return float(t.item()), float(c.item())


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_int_peaks():
    """Integer-pipe and random-sector ceilings measured on B200 by
    scripts/microbench/peaks.cu (profiles/r02_peaks_microbench.jsonl)."""
    out = {"alu_lane_ops_per_clk_per_sm": 64.0, "issue_lane_ops_per_s": None, "alu_lane_ops_per_s": None,
           "random_reads_per_s": None, "source": "B300_MICROARCH fallback (ALU rt_SMSP = 2)"}
    path = os.path.join(ROOT, "profiles", "r02_peaks_microbench.jsonl")
    if not os.path.exists(path):
        return out
    rows = [json.loads(l) for l in open(path) if l.strip()]
    alu = [r["lane_ops_per_s"] for r in rows if r.get("test") == "int_pipe" and r.get("op") == "lop3"]
    mix = [r["lane_ops_per_s"] for r in rows if r.get("test") == "int_pipe" and r.get("op") == "lop3+imad"]
    rnd = [r["reads_per_s"] for r in rows if r.get("test") == "random_sector_read" and r.get("table_gib", 0) >= 16]
    out.update({
        "alu_lane_ops_per_s": max(alu) if alu else None,
        "issue_lane_ops_per_s": max(mix) if mix else None,
        "random_reads_per_s": max(rnd) if rnd else None,
        "source": "profiles/r02_peaks_microbench.jsonl (scripts/microbench/peaks.cu on one B200)",
    })
    return out


def host_cpu():
    """Host CPU model and usable core count (cpu_baseline context)."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001 -- context only
        pass
    return {"model": model, "nproc": os.cpu_count()}


def oracle_rate(spec, max_cost):
    import oracle
    t0 = time.perf_counter()
    r = oracle.Oracle.from_spec(spec).solve(max_cost)
    dt = time.perf_counter() - t0
    return r.cand_complete, dt, r


# ------------------------------------------------------------------ reference arm

def run_reference(args, rank):
    if rank != 0:
        return 0
    spec, _, desc = WORKLOADS[args.workload]
    mc = REFERENCE_STEP_COST[args.workload]
    for _ in range(args.warmup):
        oracle_rate(spec, mc)
    cands, secs = 0, 0.0
    for _ in range(args.steps):
        c, dt, _ = oracle_rate(spec, mc)
        cands += c
        secs += dt
    value = cands / secs
    sample = (f"oracle (single-threaded C++, oracle/rei_oracle.cpp) levels 1..{mc} of {args.workload} "
              f"per step ({cands // args.steps} candidates)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": {"workload": args.workload, "description": desc,
                                        "sample_max_cost": mc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm

def roofline_of(kstats, kresults, kstep_ms, ic_words, w32, world, kernel_pass, workload, mode="hash64"):
    """Dominant kernel's achieved rate vs its binding ceiling."""
    dom = max(("concat", "union", "unary", "transpose"), key=lambda k: kstats[k][1])
    dom_launches, dom_ms = kstats[dom]
    evaluated = 0
    for rr in kresults:
        for l in rr.levels:
            evaluated += {"concat": l.eval_c, "union": l.eval_u}.get(dom, l.cand_q + l.cand_s)
    s_in = sum(max(0, len(w) - 1) for w in ic_words)
    peaks, peaks_kind = load_peaks()
    ip = load_int_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    alu_peak = ip["alu_lane_ops_per_s"] or 64 * 148 * sm_mhz * 1e6
    issue_peak = ip["issue_lane_ops_per_s"] or 128 * 148 * sm_mhz * 1e6
    opc = ops_per_candidate(dom, w32, s_in)
    per_s = (evaluated / dom_launches) / (dom_ms / dom_launches / 1000.0) if dom_launches and dom_ms else 0.0
    achieved = per_s * opc
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(workload, {}).get(dom)
    traffic_note = ("DRAM bytes (read + write) of the longest launch of this kernel in one ncu --set full "
                    "capture (profiles/roofline_traffic.json)") if traffic else None
    roof = {
        "bound": "alu", "achieved": achieved / 1e12, "peak": alu_peak / 1e12, "unit": "Tops/s",
        "frac": achieved / alu_peak, "frac_issue": achieved / issue_peak, "traffic": traffic,
        "traffic_note": traffic_note,
        "kernel": f"k_{dom}<W32={w32}>", "ops_per_candidate": opc, "candidates_per_s": per_s,
        "launches": dom_launches, "avg_launch_ms": dom_ms / max(1, dom_launches),
        "share_of_step": dom_ms / sum(kstep_ms) if world == 1 and kstep_ms else None,
        "measured_in": kernel_pass,
        "peak_source": f"INT32 ALU pipe (LOP3/IADD3) measured: {alu_peak:.4g} lane-ops/s = 64/clk/SM "
                       f"({ip['source']}); frac_issue uses the measured ALU+FMA issue rate "
                       f"{issue_peak:.4g} lane-ops/s (128/clk/SM)",
    }
    if w32 >= 2:
        # |IC| > 32: the dedup set is an HBM hash table: one random 32-byte
        # sector per probed candidate (the 64-bit key slot), plus the cached entry on a
        # fingerprint match when keys are indexed (W32 >= 4).  Bound: the measured rate
        # of random 32-byte reads from a table >> L2 (scripts/microbench/peaks.cu);
        # the copy-bandwidth fraction is given beside it.
        # inline keys (hash64, 16/32-byte inline slots): the slot is the key -> one sector;
        # indexed keys: the 8-byte slot plus the arena CS on a fingerprint match
        sectors = 1 if mode in ("hash64", "inline") else 1 + (4 * w32 + 31) // 32
        bps = 32 * sectors
        rnd = ip["random_reads_per_s"] or 36.3e9
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
        achieved_b = per_s * bps
        roof.update({
            "bound": "hbm", "achieved": achieved_b / 1e9, "peak": rnd * 32 / 1e9, "unit": "GB/s",
            "frac": achieved_b / (rnd * 32), "frac_of_copy_bw": achieved_b / hbm_peak,
            "bytes_per_candidate": bps, "random_reads_per_s_peak": rnd,
            "peak_source": f"measured random 32-B reads from a >= 16 GiB table: {rnd:.4g}/s x 32 B "
                           f"({ip['source']}); copy bandwidth {hbm_peak / 1e9:.0f} GB/s ({peaks_kind})",
        })
    return roof


def measure(args, workload, rank, world, local_rank, stream, flush, sharded, steps, warmup, primary=True):
    """Timed solves of one workload (+ sequential kernel pass, e2e through the C ABI)."""
    import torch
    import torch.distributed as dist
    from paper_2305_18575_b200 import Solver, nccl_unique_id

    spec, max_cost, desc = WORKLOADS[workload]

    def nccl_kw():
        if not sharded:
            return {}
        # one sharded search over all ranks: rank 0's ncclUniqueId is
        # broadcast with torch.distributed; rei_init / rei_solve are then collective
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return dict(world_size=world, rank=rank, nccl_id=box[0])

    def barrier():
        if world > 1:
            dist.barrier()

    # no fallback: a failing multi-GPU init or solve raises (and the run fails)
    solver = Solver.from_spec(spec, device=local_rank, stream=stream, **nccl_kw())
    for _ in range(warmup):
        r = solver.solve(max_cost)
        assert r.status == "found", r.status
    torch.cuda.synchronize()
    # no per-kernel CUDA events in the timed region (they cost host time per launch); the
    # per-kernel times come from the events passes after it
    launches0 = solver.launch_count()
    # no Python garbage collection inside the timed regions (a full collection with torch
    # loaded pauses the host for tens of ms, and the solve's host-side level loop with it)
    gc.collect()
    gc.disable()
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, cands, results = [], 0, []
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.add_(1)  # write > L2 between timed steps
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = solver.solve(max_cost)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        cands += r.candidates
        results.append(r)
    clocks = sampler.stop()
    gc.enable()
    launches = solver.launch_count() - launches0
    # per-kernel event pass in the timed configuration (same context, same streams)
    solver.reset_kernel_stats()
    tresults, tstep_ms = [], []
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.add_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tresults.append(solver.solve(max_cost))
        e1.record(stream)
        e1.synchronize()
        tstep_ms.append(e0.elapsed_time(e1))
    kstats_timed = solver.kernel_stats()
    ic_words = solver.ic()
    mode = solver.dedup_mode()
    solver.close()  # the kernel pass and the e2e solves below run one context at a time
    dev = torch.device("cuda", local_rank)
    total_ms, all_cands = reduce_over_ranks(sum(step_ms), cands, dev, world, sum_work=not sharded)
    value = all_cands / (total_ms / 1000.0)
    w32 = results[0].cs_words

    # SURVEY 8(d) throughput: candidates of the complete levels / their device time
    comp_c = sum(l.cand for rr in results for l in rr.levels if l.complete == 1)
    comp_ms = sum(l.ms for rr in results for l in rr.levels if l.complete == 1)

    # ---- roofline of the dominant kernel (CUDA events on the launching stream).  In the
    # timed region a level's kernels overlap on concurrent streams, so one kernel's event
    # span includes SMs lent to another (the timed-region fraction is a lower bound); the
    # reported fraction comes from a sequential pass (REI_CONCURRENT=0, same workload,
    # L2 flushed) -- the launch order ncu serialises too.  Concat goes first there
    # (REI_UNION_FIRST=0): with union first on one stream, a union hit at c* makes the
    # concat launches of that level exit at once.
    roof_timed = roofline_of(kstats_timed, tresults, tstep_ms, ic_words, w32, world,
                             "timed configuration, per-kernel events pass", workload, mode)
    kresults, kstep_ms, kstats, kernel_pass = tresults, tstep_ms, kstats_timed, "timed configuration"
    if world == 1:
        prev = {k: os.environ.get(k) for k in ("REI_CONCURRENT", "REI_UNION_FIRST")}
        os.environ["REI_CONCURRENT"] = "0"
        os.environ["REI_UNION_FIRST"] = "0"
        try:
            ksolver = Solver.from_spec(spec, device=local_rank, stream=stream)
        finally:
            for k, v in prev.items():
                if v is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = v
        ksolver.solve(max_cost)
        torch.cuda.synchronize()
        ksolver.reset_kernel_stats()
        kresults, kstep_ms = [], []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.add_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            kresults.append(ksolver.solve(max_cost))
            e1.record(stream)
            e1.synchronize()
            kstep_ms.append(e0.elapsed_time(e1))
        kstats = ksolver.kernel_stats()
        ksolver.close()
        kernel_pass = f"sequential-stream pass (REI_CONCURRENT=0, REI_UNION_FIRST=0), {steps} steps, L2 flushed"
    roofline = roofline_of(kstats, kresults, kstep_ms, ic_words, w32, world, kernel_pass, workload, mode)
    roofline["frac_timed_region"] = roof_timed["frac"]
    roofline["kernel_timed_region"] = roof_timed["kernel"]

    # ---- end to end through the public API with host buffers (rei_init + rei_solve + result)
    e2e = None
    n_e2e = max(1, min(steps, 5))
    e2e_s, e2e_cands, h2d, d2h = 0.0, 0, 0, 0
    init_ms, solve_ms = [], []
    gc.collect()
    gc.disable()
    for rep in range(n_e2e + 1):  # rep 0: untimed warm-up (first context on the pool)
        with torch.cuda.stream(stream):
            flush.add_(1)
        torch.cuda.synchronize()
        kw = nccl_kw()
        barrier()
        t0 = time.perf_counter()
        s2 = Solver.from_spec(spec, device=local_rank, stream=stream, **kw)
        t_init = time.perf_counter()
        r2 = s2.solve(max_cost)
        _ = r2.regex  # result already copied to the host by rei_solve
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hb, db = s2.transfer_bytes()
        s2.close()
        if rep == 0:
            continue
        e2e_s += t1 - t0
        init_ms.append(1000 * (t_init - t0))
        solve_ms.append(1000 * (t1 - t_init))
        e2e_cands += r2.candidates
        h2d += hb
        d2h += db
    gc.enable()
    e2e_t, e2e_c = reduce_over_ranks(1000 * e2e_s, e2e_cands, dev, world, sum_work=not sharded)
    e2e = {"value": e2e_c / (e2e_t / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d // n_e2e,
           "d2h_bytes_per_step": d2h // n_e2e,
           "time_to_minimal_re_ms": e2e_t / n_e2e,
           "init_ms_median": statistics.median(init_ms), "solve_ms_median": statistics.median(solve_ms),
           "init_ms": [round(x, 3) for x in init_ms], "solve_ms": [round(x, 3) for x in solve_ms],
           "warmup_reps": 1,
           "note": "rei_init (host strings -> device precompute) + rei_solve + result, host wall clock"}
    r0 = results[-1]
    return {
        "value": value, "total_ms": total_ms, "cands": cands, "results": results, "step_ms": step_ms,
        "roofline": roofline, "e2e": e2e, "launches": launches, "clocks": clocks, "desc": desc,
        "max_cost": max_cost, "spec": spec,
        "complete_levels": {"value": comp_c / (comp_ms / 1000.0) if comp_ms else None, "unit": UNIT,
                            "candidates_per_step": comp_c / steps, "device_ms_per_step": comp_ms / steps,
                            "note": "SURVEY 8(d): candidates of complete levels / their device time "
                                    "(CUDA events per level)"},
        "config": {
            "workload": workload, "description": desc, "max_cost": max_cost,
            "n_ic": r0.n_ic, "cs_bits": 32 * r0.cs_words, "dedup": mode, "cstar": r0.cost, "regex": r0.regex,
            "candidates_per_step": cands / steps,
            "candidates_through_last_complete_level": r0.cand_complete,
            "time_to_minimal_re_ms": statistics.median(step_ms),
            "time_to_minimal_re_ms_all": [round(x, 3) for x in step_ms],
        },
    }


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2305_18575_b200 import build

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(device=dev)
    sharded = world > 1 and args.multi == "shard"
    # L2 flush buffer (> 126 MB L2), written between timed steps
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device=dev)
    m = measure(args, args.workload, rank, world, local_rank, stream, flush, sharded, args.steps, args.warmup)

    # ---- CPU oracle baseline (rank 0, N=1 only, bounded sample)
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mc = ORACLE_SAMPLE_COST[args.workload]
        c, dt, _ = oracle_rate(m["spec"], mc)
        hc = host_cpu()
        cpu_baseline = {"value": c / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
                        "host_cpu": hc["model"], "host_nproc": hc["nproc"],
                        "sample": f"oracle/rei_oracle.cpp levels 1..{mc} of {args.workload}: "
                                  f"{c} candidates in {dt:.1f} s on 1 host core ({hc['model']})"}

    # ---- secondary workload (N=1): BASELINE configs[1], the HBM hash set (the headline
    # C5 workload dedups in an L2-resident bitmap)
    secondary = None
    if world == 1 and args.secondary and args.secondary != args.workload:
        s = measure(args, args.secondary, rank, world, local_rank, stream, flush, False,
                    max(3, args.steps // 2), 3)
        secondary = {"workload": args.secondary, "metric": METRIC, "value": s["value"], "unit": UNIT,
                     "ms_per_step": s["total_ms"] / max(1, len(s["step_ms"])), "config": s["config"],
                     "roofline": s["roofline"], "e2e": s["e2e"], "complete_levels": s["complete_levels"],
                     "gpu_launches": s["launches"], "clocks": s["clocks"]}

    paper = PAPER.get(args.workload)
    vs = None
    if paper:
        vs = m["value"] / (paper["reps"] / paper["gpu_s"])
    cfg = dict(m["config"])
    cfg.update({
        "l2": f"{args.flush_mb} MiB buffer written between timed steps (L2 flush)",
        "parallelism": (f"shard{world} (level work lists partitioned; hash-owner NCCL all-to-all, "
                        "owner dedup, all-gather of the uniques)" if sharded else f"replicas{world}")
        if world > 1 else "single",
        "paper_context": paper,
        "vs_baseline_note": "value / paper's |REs| per GPU-second on A100 for this spec; the paper's "
                            "|REs| counting convention differs from reading A9 (DESIGN.md)" if paper else None,
    })
    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["total_ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": vs, "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "roofline": m["roofline"],
        "cpu_baseline": cpu_baseline,
        "e2e": m["e2e"],
        "complete_levels": m["complete_levels"],
        "gpu_launches": m["launches"],
        "clocks": m["clocks"],
        "secondary": secondary,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="table1-row1")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary", default="c2-t1-s0",
                    help="N=1: also measure this workload (BASELINE configs[1], HBM hash set); '' = off")
    ap.add_argument("--multi", choices=["shard", "replicas"], default="shard",
                    help="N > 1: one sharded search (default) or N independent replicas")
    args = ap.parse_args()
    if args.secondary in ("", "none", "off"):
        args.secondary = None
    elif args.secondary not in WORKLOADS:
        raise SystemExit(f"--secondary {args.secondary}: not a workload ({', '.join(sorted(WORKLOADS))})")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: become N ranks (one process per GPU)
        # under torch.distributed.run on this node
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
