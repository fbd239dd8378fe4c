"""Benchmark: converged fine-grid points/s on BASELINE config 2 (2049^2,
F = 1 + 0.5 sin(20 pi x) sin(20 pi y), centre source), the full method matrix
of BASELINE.json: fmm, fsm, and fmsm / hcm / fhcm at 8, 16, 32, 64-point cells.

One step = one solve of every method-config in the matrix (14 solves).  The
K timed steps are submitted together as one list schedule on the GPU
(eik_plan_run_batch: each solve's persistent kernel on its own SMs, one
stream each, a solve starting as soon as SMs free up -- the device
counterpart of the reference runner's --jobs pool), so a step's long
replays overlap the next step's solves.  `value` is the whole-job throughput
(grid points converged / device time of the K steps) with the speed fields
already resident in HBM; `e2e` is the same metric through the public API
(eik_solve_batch over the K steps' solves) with pinned host buffers (H2D of
F and tables, D2H of u inside the timed region).  `single_step_ms` is one
step alone; `methods` lists each solve's time inside the schedule and alone
on the whole GPU (`solo_ms`).  Prints one JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
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

import numpy as np

# one hardware work queue per stream for the concurrent solves; must be set
# before anything in the process creates the CUDA context
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CELL_SIZES = [8, 16, 32, 64]
METHODS = ["fmm", "fsm", "fmsm", "hcm", "fhcm"]


def matrix(cfg):
    rows = [("fmm", 0), ("fsm", 0)]
    for cs in CELL_SIZES:
        for meth in ("fmsm", "hcm", "fhcm"):
            rows.append((meth, cs))
    return rows


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def run_reference(args):
    """Reference arm: the unmodified reference (oracle/_ref, built from
    /root/reference) on the host cores, one method-config per thread (the
    reference's own --jobs model, experiment.cpp:284-310)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    from paper_1110_6220_b200 import configs
    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libeikref.so not built"}))
        return
    cfg = configs.config2()
    p = cfg.problem
    M = p.grid.size()
    rows = matrix(cfg)
    cores = os.cpu_count() or 1

    def one(row):
        meth, cs = row
        cx = p.grid.m // cs if cs else 0
        return O.ref_solve(p, meth, cx, cx).elapsed_ms

    times = []
    per = {}
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=min(cores, len(rows))) as ex:
            ms = list(ex.map(one, rows))
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            for r, t in zip(rows, ms):
                per.setdefault(f"{r[0]}" + (f"/{r[1]}" if r[1] else ""), []).append(t)
    step_s = statistics.mean(times)
    value = len(rows) * M / step_s
    out = {
        "impl": "reference", "metric": "converged fine-grid points/s", "value": value,
        "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config 2)",
        "config": {"workload": "c2_sinusoid_2049_method_matrix", "grid": 2049,
                   "methods": METHODS, "cell_sizes": CELL_SIZES},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": min(cores, len(rows)),
                         "kind": "reference",
                         "sample": f"the full {len(rows)}-solve C2 matrix per step, one solve per "
                                   f"thread (reference solves are single-threaded)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "per_solve_ms": {k: statistics.mean(v) for k, v in per.items()},
    }
    print(json.dumps(out))


def fsm_roof(methods, M, hbm, peak_kind):
    """Roofline line of the global-sweep kernel (FSM) inside the C2 step."""
    f = methods.get("fsm")
    if not f:
        return None
    ach = 24.0 * M * f["sweeps"] / (f["solo_ms"] / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "fsm_wavefront (C2, alone on the GPU)",
            "achieved": round(ach, 2), "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "algorithmic_bytes": 24.0 * M * f["sweeps"], "peak_kind": peak_kind,
            "note": "u + C (67 MB) stay in L2; the fp64 wavefront chain (m + n steps per "
                    "direction turn) bounds it, not HBM"}


def measure_fsm_c5(hbm, peak_kind):
    """FSM on BASELINE config 5 with the field resident: best of 2 device
    times, algorithmic bytes 24 B per node per sweep; DRAM
    traffic per launch from the committed ncu capture of the same solve."""
    import paper_1110_6220_b200 as E
    from paper_1110_6220_b200 import configs
    p5 = configs.config5().problem
    M5 = p5.grid.m * p5.grid.n
    plan = E.Plan(p5, "fsm")
    best = None
    for _ in range(2):
        o = plan.run()
        best = o if best is None or o.device_ms < best.device_ms else best
    plan.close()
    del p5
    traffic = None
    try:
        import csv
        with open(os.path.join(ROOT, "profiles", "r01_fsm_c5_v4_metrics.csv")) as f:
            rows = [r for r in csv.reader(x for x in f if not x.startswith("=="))]
        hdr = rows[0]
        vals = {r[hdr.index("Metric Name")]: float(r[hdr.index("Metric Value")]) for r in rows[1:]}
        traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except (OSError, ValueError, KeyError, IndexError):
        pass
    ms = best.device_ms
    nbytes = 24.0 * M5 * best.sweeps
    ach = nbytes / (ms / 1e3) / 1e9
    return {"workload": "c5_sinsum_32769_64_sources_fsm", "points": M5, "device_ms": round(ms, 3),
            "sweeps": best.sweeps, "points_per_s": M5 / (ms / 1e3),
            "roofline": {"bound": "hbm", "kernel": "fsm_wavefront", "achieved": round(ach, 2),
                         "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                         "algorithmic_bytes": nbytes, "peak_kind": peak_kind},
            "ref_cpu_estimate": "~1-1.3 h on one core (SURVEY 8(d)); not run"}


def cpu_baseline_single_core():
    """Single-core reference timing on a bounded sample: one solve of every
    method-config of the matrix except FSM, plus FSM (13 s) -- ~20 s."""
    from oracle import oracle as O
    from paper_1110_6220_b200 import configs
    if not O.have_ref():
        return None
    p = configs.config2().problem
    rows = matrix(None)
    tot = 0.0
    for meth, cs in rows:
        cx = p.grid.m // cs if cs else 0
        tot += O.ref_solve(p, meth, cx, cx).elapsed_ms
    return {"value": len(rows) * p.grid.size() / (tot / 1e3), "unit": "points/s", "cores": 1,
            "kind": "reference",
            "sample": f"one pass of the {len(rows)}-solve C2 matrix on 1 core "
                      f"({tot / 1e3:.1f} s, solver call only as experiment.cpp:204-213)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the config-5 FSM measurement (HBM-scale global sweep)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    rank, world, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    import paper_1110_6220_b200 as E
    from paper_1110_6220_b200 import configs
    E.set_device(local)  # the library's own CUDA runtime: select the rank's GPU there too

    # Weak scaling: every rank solves its own replica of the C2 matrix (the
    # method matrix does not shard; SURVEY.md §8e -- row strips are for C5).
    cfg = configs.config2()
    p = cfg.problem
    g = p.grid
    M = g.size()
    rows = matrix(cfg)
    # One plan set (the 14 solves of a step) per timed step: the K steps are
    # submitted together and run as one list schedule on the GPU
    # (eik_plan_run_batch), so a step's long replays overlap the next step's
    # solves.  Every plan keeps its own inputs and buffers resident.
    K = max(1, args.steps)
    tables, cells_of = {}, {}
    for meth, cs in rows:
        if cs and cs not in tables:
            cells_of[cs] = E.build_cells(g, g.m // cs, g.m // cs)
            tables[cs] = E.cell_tables(p, cells_of[cs])
    keys = [f"{meth}" + (f"/{cs}" if cs else "") for meth, cs in rows]
    sets = [[E.Plan(p, meth, cells_of.get(cs), tables.get(cs)) for meth, cs in rows]
            for _ in range(K)]
    plan_list = sets[0]
    all_plans = [pl for st in sets for pl in st]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush_l2():
        flush.zero_()
        torch.cuda.synchronize()

    # W warm-up steps (whole K-step schedules until at least W steps ran)
    for _ in range(max(1, -(-args.warmup // K))):
        E.run_batch(all_plans)
    flush_l2()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        outs, total_ms = E.run_batch(all_plans)
    torch.cuda.synchronize()
    launches = sum(o.kernel_launches for o in outs)
    per_all = {}
    for i, o in enumerate(outs):
        per_all.setdefault(keys[i % len(rows)], []).append((o.device_ms + o.host_ms, o))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    mean_ms = total_ms / K
    value = world * len(rows) * M / (mean_ms / 1e3)

    # one step alone (its 14 solves concurrently, nothing overlapping it) and
    # each solve alone on the whole GPU: latencies, outside the timed region
    flush_l2()
    _, single_step_ms = E.run_batch(plan_list)

    # each solve alone on the whole GPU (latency; outside the timed region)
    solo = {}
    for k, pl in zip(keys, plan_list):
        flush_l2()
        o = pl.run()
        solo[k] = o.device_ms + o.host_ms

    # per-method table with the reference's counters beside ours
    with open(os.path.join(ROOT, "tests", "golden", "big.json")) as f:
        gold = json.load(f)
    methods = {}
    hbm, peak_kind = peaks()
    best = None
    for k, lst in per_all.items():
        t = statistics.mean(x[0] for x in lst)
        o = lst[-1][1]
        meth = k.split("/")[0]
        cs = int(k.split("/")[1]) if "/" in k else 0
        ref = gold.get(f"c2/{k}", {})
        if meth in ("fsm", "fmm"):
            nbytes = 24.0 * M * o.sweeps  # 24 B per node per sweep
        else:
            nbytes = (24.0 * cs * cs + 32.0 * cs) * (o.heap_removals if meth != "fmsm"
                                                      else (g.m // cs) ** 2)
        ach = nbytes / (t / 1e3) / 1e9
        methods[k] = {"ms": round(t, 3), "solo_ms": round(solo[k], 3), "ctas": o.ctas,
                      "points_per_s": M / (t / 1e3), "sweeps": o.sweeps,
                      "ref_sweeps": ref.get("sweeps"), "heap_removals": o.heap_removals,
                      "ref_heap_removals": ref.get("heap_removals"),
                      "node_updates": o.node_updates, "ref_node_updates": ref.get("node_updates"),
                      "host_ms": round(o.host_ms, 3), "algorithmic_GBps": round(ach, 2),
                      "ref_cpu_ms": ref.get("ms")}
        if best is None or t > best[1]:
            best = (k, t, nbytes, ach)
    dom_k, dom_t, dom_bytes, dom_ach = best
    # DRAM bytes of the dominant launch from a committed `ncu --set full`
    # capture (profiles/r01_traffic.json), when it profiled this same solve
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            traffic = json.load(f).get(dom_k, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    roofline = {"bound": "hbm", "kernel": dom_k, "achieved": round(dom_ach, 2), "peak": hbm,
                "unit": "GB/s", "frac": dom_ach / hbm, "traffic": traffic,
                "algorithmic_bytes": dom_bytes, "peak_kind": peak_kind,
                "note": "the longest solve of the concurrent step (its kernel's duration inside "
                        "the step); latency-bound fp64 dependency chains; algorithmic bytes per "
                        "SURVEY §8(d)"}

    # e2e: public API (eik_solve_batch), pinned host buffers, H2D + solves +
    # D2H of every solve of the step inside the timed region
    pinned_F = torch.empty(M, dtype=torch.float64, pin_memory=True).numpy()
    pinned_F[:] = p.sampled_speed()
    p_pin = E.Problem(g, p.speed, p.exit_nodes, p.exit_cost, p.exit_points, p.exit_point_cost,
                      _F=pinned_F)
    pinned_u = [torch.empty(M, dtype=torch.float64, pin_memory=True).numpy()
                for _ in range(K * len(rows))]
    jobs = [(p_pin, meth, cells_of.get(cs), tables.get(cs)) for meth, cs in rows] * K
    h2d = d2h = 0
    for meth, cs in rows:
        h2d += 8 * M + 16 * len(p.exit_nodes)
        if cs:
            tb = tables[cs]
            h2d += 8 * sum(len(a) for a in (tb.probe_w, tb.probe_e, tb.probe_s, tb.probe_n, tb.center))
        d2h += 8 * M
    E.solve_batch(jobs, outs=pinned_u)  # warm-up (device buffer cache)
    flush_l2()
    t0 = time.perf_counter()
    E.solve_batch(jobs, outs=pinned_u)  # the K steps' solves, uploads and downloads
    e2e_s = (time.perf_counter() - t0) / K
    if world > 1:  # the slowest rank's end-to-end time, like the device timing
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # the global sweep at BASELINE config 5 (32769^2, 1.07e9 points, u + F ~17 GB):
    # the one configuration of the path where HBM, not the dependency chain
    # alone, is in reach; measured after the timed region, rank 0 at N = 1
    fsm_c5 = None
    if not args.no_c5 and rank == 0 and world == 1:
        fsm_c5 = measure_fsm_c5(hbm, peak_kind)

    cpu = None if args.no_cpu_baseline or rank != 0 else cpu_baseline_single_core()
    if rank == 0:
        out = {
            "metric": "converged fine-grid points/s", "value": value, "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE config 2)",
            "config": {"workload": "c2_sinusoid_2049_method_matrix", "grid": 2049,
                       "methods": METHODS, "cell_sizes": CELL_SIZES,
                       "parallelism": f"replicas x{world}",
                       "concurrency": f"{len(rows)} solves per step, each on its own SMs "
                                      "(eik_plan_run_batch list schedule)",
                       "steps_overlap": f"the {K} timed steps run as one list schedule "
                                        "(a step's long replays overlap the next step's "
                                        "solves); single_step_ms is one step alone",
                       "l2": f"inputs larger than L2 ({K * len(rows)} resident plans, "
                             "~0.2 GB each); one 256 MB flush before the timed region"},
            "e2e": {"value": world * len(rows) * M / e2e_s, "unit": "points/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "single_step_ms": single_step_ms,
            "roofline": roofline, "roofline_fsm_c2": fsm_roof(methods, M, hbm, peak_kind),
            "fsm_c5": fsm_c5, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary(), "methods": methods,
        }
        print(json.dumps(out))
    for plan in all_plans:
        plan.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
