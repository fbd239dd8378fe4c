"""Time eik_solve_batch (the bench's e2e call) on K steps of the C2 matrix.
Development aid: EIK_BATCH_TRACE=1 prints each job's timeline.
usage: python scripts/e2e_probe.py K"""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = configs.config2().problem
g = p.grid
M = g.size()
rows = [("fmm", 0), ("fsm", 0)] + [(m, cs) for cs in (8, 16, 32, 64) for m in ("fmsm", "hcm", "fhcm")]
tables, cells_of = {}, {}
for meth, cs in rows:
    if cs and cs not in tables:
        cells_of[cs] = E.build_cells(g, g.m // cs, g.m // cs)
        tables[cs] = E.cell_tables(p, cells_of[cs])
pinned_F = torch.empty(M, dtype=torch.float64, pin_memory=True).numpy()
pinned_F[:] = p.sampled_speed()
p_pin = E.Problem(g, p.speed, p.exit_nodes, p.exit_cost, p.exit_points, p.exit_point_cost,
                  _F=pinned_F)
outs = [torch.empty(M, dtype=torch.float64, pin_memory=True).numpy() for _ in range(K * len(rows))]
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
    t[...] = a
    return t


tables = {cs: E.CellTables(*[pinned(x) for x in (tb.probe_w, tb.probe_e, tb.probe_s, tb.probe_n,
                                                 tb.center)]) for cs, tb in tables.items()}
jobs = [(p_pin, meth, cells_of.get(cs), tables.get(cs)) for meth, cs in rows] * K
for rep in range(3):
    t0 = time.perf_counter()
    res, ms = E.solve_batch(jobs, outs=outs)
    dt = time.perf_counter() - t0
    print(f"K={K} rep {rep}: wall {dt * 1e3:.1f} ms ({dt * 1e3 / K:.1f} per step), device {ms:.1f} ms,"
          f" e2e {14 * M * K / dt / 1e6:.1f} M points/s", flush=True)
