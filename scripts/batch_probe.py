"""Concurrent method matrix (eik_plan_run_batch) against sequential solves on
C2: makespan, per-solve device times, bitwise equality.  Development aid."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

cfg = configs.config2()
p = cfg.problem
g = p.grid
rows = [("fmm", 0), ("fsm", 0)] + [(m, cs) for cs in (8, 16, 32, 64) for m in ("fmsm", "hcm", "fhcm")]
if len(sys.argv) > 1:
    rows = [r for r in rows if f"{r[0]}/{r[1]}" in sys.argv[1].split(",") or r[0] in sys.argv[1].split(",")]
tables, plans = {}, []
for meth, cs in rows:
    cells = E.build_cells(g, g.m // cs, g.m // cs) if cs else None
    if cells is not None and cs not in tables:
        tables[cs] = E.cell_tables(p, cells)
    plans.append(E.Plan(p, meth, cells, tables.get(cs)))
for pl, r in zip(plans, rows):
    print(r, "capacity", pl.capacity())
seq_u, seq_ms = [], 0.0
for pl, r in zip(plans, rows):
    u = np.empty(g.size())
    o = pl.run(u)
    seq_u.append(u)
    seq_ms += o.device_ms
    print("seq", r, round(o.device_ms, 2))
print("sequential sum ms", round(seq_ms, 1))
for rep in range(int(os.environ.get("REPS", "5"))):
    us = [np.empty(g.size()) for _ in plans]
    t0 = time.perf_counter()
    outs, ms = E.run_batch(plans, us)
    wall = (time.perf_counter() - t0) * 1e3
    same = all(np.array_equal(a.view(np.int64), b.view(np.int64)) for a, b in zip(us, seq_u))
    print("batch ms", round(ms, 1), "wall", round(wall, 1), "bitwise equal", same)
    print("  per-solve", {f"{r[0]}/{r[1]}": round(o.device_ms, 1) for r, o in zip(rows, outs)})
    print("  ctas", {f"{r[0]}/{r[1]}": o.ctas for r, o in zip(rows, outs)})
