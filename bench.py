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
METRIC = "converged fine-grid points/s"
# identical in both arms (the driver compares the arms' config objects)
CONFIG = {"workload": "c2_sinusoid_2049_method_matrix", "grid": 2049,
          "speed": "1 + 0.5 sin(20 pi x) sin(20 pi y), centre point source",
          "methods": METHODS, "cell_sizes": CELL_SIZES,
          "step": "one solve of each of the 14 method-configs (fmm, fsm, fmsm/hcm/fhcm x 8,16,32,64)",
          "l2": "inputs larger than L2 (resident plans ~0.2 GB each, K steps); one 256 MB flush "
                "before the timed region"}


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_lib():
    """The unmodified reference (oracle/_ref/libeikref.so, built from
    /root/reference by oracle/Makefile) through plain ctypes: the reference
    arm imports nothing from paper_1110_6220_b200 and maps none of its code."""
    import ctypes as C
    path = os.path.join(ROOT, "oracle", "_ref", "libeikref.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    lib.ref_bench_sinusoid.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.ref_bench_sinusoid.restype = C.c_int
    lib.ref_last_error.restype = C.c_char_p
    return lib


_REF_METHOD = {"fmm": 0, "fsm": 1, "lsm": 2, "hcm": 3, "fhcm": 4, "fmsm": 5}


def run_reference(args):
    """Reference arm: the unmodified reference on the box's host cores.  Every
    step is the full 14-solve C2 matrix, built by the reference itself (its
    SpeedSpec and build_problem, oracle/ref_shim.cpp ref_bench_sinusoid).  All
    W warm-up steps' solves, then all K timed steps' solves, go through ONE
    work queue on nproc threads (the reference's --jobs model,
    experiment.cpp:284-310, with no barrier between steps; longest solves
    first), so every core stays busy; value = 14 M K / wall time."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor
    rank, world, _ = dist_env()
    if rank != 0:
        return
    lib = _ref_lib()
    if lib is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libeikref.so not built"}))
        return
    m = CONFIG["grid"]
    M = m * m
    rows = matrix(None)
    cores = os.cpu_count() or 1

    def one(row):
        meth, cs = row
        ms, sm = C.c_double(), C.c_double()
        rc = lib.ref_bench_sinusoid(_REF_METHOD[meth], m, 0.5, 20, m // cs if cs else 0,
                                    C.byref(ms), C.byref(sm))
        if rc:
            raise RuntimeError(lib.ref_last_error().decode())
        return row, ms.value

    def run_all(jobs):
        with ThreadPoolExecutor(max_workers=cores) as ex:
            return list(ex.map(one, jobs))

    warm = run_all(rows * max(1, args.warmup))
    est = {}
    for row, ms in warm:
        est.setdefault(row, []).append(ms)
    order = sorted(rows, key=lambda r: -statistics.mean(est[r]))  # longest first
    t0 = time.perf_counter()
    res = run_all([r for r in order for _ in range(args.steps)])
    wall = time.perf_counter() - t0
    per = {}
    for (meth, cs), ms in res:
        per.setdefault(meth + (f"/{cs}" if cs else ""), []).append(ms)
    step_s = wall / args.steps
    value = len(rows) * M / step_s
    core_s = sum(ms for _, ms in res) / 1e3
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config 2)",
        "config": CONFIG,
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "reference",
                         "cpu_model": cpu_model(), "nproc": cores,
                         "sample": f"{args.steps} steps x {len(rows)} solves of the C2 matrix on "
                                   f"one {cores}-thread work queue (longest first, no per-step "
                                   f"barrier); {core_s:.1f} core-s in {wall:.1f} s wall "
                                   f"({core_s / wall / cores:.0%} of the cores busy)"},
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
                    "direction turn) bounds it, not HBM; clean super-blocks are passed "
                    "over unstreamed (DESIGN 4(1))"}


def _ncu_dram(path):
    """dram__bytes_read.sum + dram__bytes_write.sum from a committed ncu csv."""
    import csv
    try:
        with open(os.path.join(ROOT, "profiles", path)) as f:
            rows = [r for r in csv.reader(x for x in f if not x.startswith("=="))]
        hdr = rows[0]
        vals = {r[hdr.index("Metric Name")]: float(r[hdr.index("Metric Value")]) for r in rows[1:]}
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except (OSError, ValueError, KeyError, IndexError):
        return None


# Per-config lines (BASELINE configs 3, 4, 5): each solve alone on the GPU,
# best of 2 device times, inputs resident; FMSM's host Part I is included in
# its time.  The reference's counters and its solve time (one core of the
# machine that generated the goldens) are listed beside ours.
CONFIG_ROWS = {
    "c3": [("fsm", 0), ("fmm", 0), ("lsm", 0), ("fmsm", 16), ("hcm", 16), ("fhcm", 16),
           ("fmsm", 48), ("hcm", 48), ("fhcm", 48)],
    "c4": [("fsm", 0), ("fmm", 0), ("lsm", 0), ("fmsm", 16), ("hcm", 16), ("fhcm", 16),
           ("fmsm", 32), ("hcm", 32), ("fhcm", 32)],
    "c5": [("fsm", 0), ("fmsm", 32), ("fhcm", 32), ("hcm", 32)],
}


def measure_configs(hbm, peak_kind):
    import paper_1110_6220_b200 as E
    from paper_1110_6220_b200 import configs
    gold = {}
    for fn, pre in (("c34.json", ""), ("extra.json", None), ("c5_full.json", "")):
        try:
            with open(os.path.join(ROOT, "tests", "golden", fn)) as f:
                d = json.load(f)
        except OSError:
            continue
        if pre is None:
            for name, v in d.get("lsm", {}).items():
                gold[f"{name}/lsm"] = v
        else:
            for k, v in d.items():
                gold[k.replace("c5_full/", "c5/")] = v
    out = {}
    for name, rows in CONFIG_ROWS.items():
        cfg = {"c3": configs.config3, "c4": configs.config4, "c5": configs.config5}[name]()
        p = cfg.problem
        M = p.grid.size()
        for meth, cs in rows:
            key = f"{name}/{meth}" + (f"/{cs}" if cs else "")
            cells = E.build_cells(p.grid, p.grid.m // cs, p.grid.m // cs) if cs else None
            plan = E.Plan(p, meth, cells)
            best = None
            for _ in range(2):
                o = plan.run()
                if best is None or o.device_ms + o.host_ms < best.device_ms + best.host_ms:
                    best = o
            plan.close()
            t = best.device_ms + best.host_ms
            ref = gold.get(key, {})
            row = {"ms": round(t, 3), "device_ms": round(best.device_ms, 3),
                   "host_ms": round(best.host_ms, 3), "points_per_s": M / (t / 1e3),
                   "sweeps": best.sweeps, "node_updates": best.node_updates,
                   "heap_removals": best.heap_removals, "ref_sweeps": ref.get("sweeps"),
                   "ref_node_updates": ref.get("node_updates"),
                   "ref_heap_removals": ref.get("heap_removals"),
                   "ref_cpu_ms_golden_host": ref.get("ms")}
            if meth in ("fsm", "lsm"):
                nbytes = 24.0 * M * best.sweeps
                ach = nbytes / (best.device_ms / 1e3) / 1e9
                row["roofline"] = {"bound": "hbm", "achieved": round(ach, 2), "peak": hbm,
                                   "unit": "GB/s", "frac": ach / hbm, "algorithmic_bytes": nbytes,
                                   "peak_kind": peak_kind}
                if key == "c5/fsm":
                    row["roofline"]["traffic"] = (_ncu_dram("r02_fsm_c5_metrics.csv") or
                                                  _ncu_dram("r01_fsm_c5_v4_metrics.csv"))
                    row["roofline"]["note"] = (
                        "algorithmic = 24 B per node per sweep (SURVEY 8(d)); the measured DRAM "
                        "traffic is below it because super-blocks that cannot change are passed "
                        "over unstreamed (DESIGN 4(1)); the bound is the sweep's dependency chain")
            out[key] = row
        del p, cfg
    return out


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
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config lines (configs 3, 4, 5 at full size)")
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
    traffic, prof = None, {}
    for fn in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                prof = json.load(f).get(dom_k, {})
        except (OSError, ValueError):
            prof = {}
        if prof:
            traffic = prof.get("dram_bytes_per_launch")
            break
    roofline = {"bound": "hbm", "kernel": dom_k, "achieved": round(dom_ach, 2), "peak": hbm,
                "unit": "GB/s", "frac": dom_ach / hbm, "traffic": traffic,
                "algorithmic_bytes": dom_bytes, "peak_kind": peak_kind,
                # the in-cell regime's own bounds, from the committed
                # `ncu --set full` capture of this solve alone
                "fp64_pipe_frac": prof.get("fp64_pipe_pct_of_peak", 0) / 100 if prof else None,
                "issue_active_frac": prof.get("issue_active_pct", 0) / 100 if prof else None,
                "smem_wavefront_frac": (prof.get("smem_wavefronts_pct_of_peak", 0) / 100
                                        if prof else None),
                "note": "the longest solve of the concurrent step (its kernel's duration inside "
                        "the step); latency-bound fp64 dependency chains (one warp per cell, "
                        "a serial committer), so HBM, fp64 pipe and shared memory are all far "
                        "from their peaks; algorithmic bytes per SURVEY §8(d)"}

    # e2e: public API (eik_solve_batch), pinned host buffers, H2D + solves +
    # D2H of every solve of the step inside the timed region
    pinned_F = torch.empty(M, dtype=torch.float64, pin_memory=True).numpy()
    pinned_F[:] = p.sampled_speed()
    p_pin = E.Problem(g, p.speed, p.exit_nodes, p.exit_cost, p.exit_points, p.exit_point_cost,
                      _F=pinned_F)
    pinned_u = [torch.empty(M, dtype=torch.float64, pin_memory=True).numpy()
                for _ in range(K * len(rows))]
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
        t[...] = a
        return t
    tables_pin = {cs: E.CellTables(*[pinned(x) for x in (tb.probe_w, tb.probe_e, tb.probe_s,
                                                         tb.probe_n, tb.center)])
                  for cs, tb in tables.items()}
    jobs = [(p_pin, meth, cells_of.get(cs), tables_pin.get(cs)) for meth, cs in rows] * K
    h2d = d2h = 0
    for meth, cs in rows:
        h2d += 8 * M + 16 * len(p.exit_nodes)
        if cs:
            tb = tables[cs]
            h2d += 8 * sum(len(a) for a in (tb.probe_w, tb.probe_e, tb.probe_s, tb.probe_n, tb.center))
        d2h += 8 * M
    for _ in range(2):  # warm-up: device buffer cache, streams, lazily loaded kernels
        E.solve_batch(jobs, outs=pinned_u)
    flush_l2()
    t0 = time.perf_counter()
    E.solve_batch(jobs, outs=pinned_u)  # the K steps' solves, uploads and downloads
    e2e_s = (time.perf_counter() - t0) / K
    if world > 1:  # the slowest rank's end-to-end time, like the device timing
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # per-config lines (configs 3, 4 and 5 at full size), after the timed
    # region, rank 0 at N = 1
    per_config = None
    if not args.no_configs and rank == 0 and world == 1:
        for plan in all_plans:
            plan.close()
        all_plans = []
        per_config = measure_configs(hbm, peak_kind)

    # N > 1: config 5 (32769^2) sharded as row strips over the ranks
    # (distributed.fsm_solve_strips: NCCL edge-row exchange and change-flag
    # all-reduce, rounds stream-ordered); each rank samples and holds only its
    # strip, the field stays sharded; device time = max over ranks
    c5_sharded = None
    if world > 1 and not args.no_configs:
        from paper_1110_6220_b200.distributed import fsm_solve_strips, strip_bounds
        p5 = configs.config5().problem
        r5 = fsm_solve_strips(p5, gather="none")
        M5 = p5.grid.size()
        a5, b5 = strip_bounds(p5.grid.n, world, rank)
        c5_sharded = {"workload": "c5_sinsum_32769_fsm_row_strips", "ranks": world,
                      "rounds": r5.sweeps, "device_ms": round(r5.device_ms, 3),
                      "points_per_s": M5 / (r5.device_ms / 1e3),
                      "rows_per_rank": b5 - a5,
                      "bytes_per_rank_u_C_F": 24 * (b5 - a5 + 2) * p5.grid.m,
                      "note": "strip-Jacobi (SURVEY 8(e) option A): same fixed point, more "
                              "rounds than fsm_solve's 28 sweeps"}
        # FMSM/32 sharded by row strips of cells, by levels of the cell DAG
        # (distributed.fmsm_solve_strips: bit-exact fmsm_solve)
        from paper_1110_6220_b200.distributed import fmsm_solve_strips
        cfg5 = configs.config5()
        cs5 = cfg5.cells_for(32)
        cells5 = E.build_cells(p5.grid, cs5, cs5)
        f5 = fmsm_solve_strips(p5, cells5, gather="none")
        c5_sharded["fmsm32"] = {"levels": f5.levels, "device_ms": round(f5.device_ms, 3),
                                "points_per_s": M5 / (f5.device_ms / 1e3),
                                "sweeps": f5.sweeps, "node_updates": f5.node_updates,
                                "edge_rows_sent_by_rank0": f5.exchanges,
                                "note": "Part II by DAG levels over row strips of cells, edge "
                                        "rows exchanged after the levels that changed them; "
                                        "Part I on every rank's host, not in device_ms"}
        del p5

    cpu = None if args.no_cpu_baseline or rank != 0 else cpu_baseline_single_core()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE config 2)",
            "config": CONFIG,
            "schedule": {"parallelism": f"replicas x{world}",
                         "concurrency": f"{len(rows)} solves per step, each on its own SMs "
                                        "(eik_plan_run_batch list schedule)",
                         "steps_overlap": f"the {K} timed steps run as one list schedule "
                                          "(a step's long replays overlap the next step's "
                                          "solves); single_step_ms is one step alone"},
            "e2e": {"value": world * len(rows) * M / e2e_s, "unit": "points/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "single_step_ms": single_step_ms,
            "roofline": roofline, "roofline_fsm_c2": fsm_roof(methods, M, hbm, peak_kind),
            # the HBM-bound global sweep at its full size (config 5, 1.07e9 nodes)
            "roofline_fsm_c5": ((per_config or {}).get("c5/fsm") or {}).get("roofline"),
            "configs": per_config, "c5_sharded": c5_sharded, "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(), "methods": methods,
        }
        print(json.dumps(out))
    for plan in all_plans:
        plan.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
