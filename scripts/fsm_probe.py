"""Decompose FSM wavefront time into per-step latency and per-strip lag.

Runs the resident FSM on thin grids (n = 32*s rows, m columns) so that
time(sweep) ~ (m + 31) * t_step + (s - 1) * lag; prints the fit."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402

rows = []
for m, n in [(4096, 32), (16384, 32), (4096, 64), (4096, 128), (4096, 256), (4096, 512),
             (2049, 2049)]:
    g = E.Grid(m, n, 1.0 / 64, 0.0, 0.0)
    p = E.build_problem(g, E.speed_constant(), E.ExitSpec.node_set([(0, 0)]))
    plan = E.Plan(p, "fsm")
    ts = [plan.run().device_ms for _ in range(4)]
    o = plan.run()
    executed = o.sweeps + 2  # lookahead D=3 runs D-1 extra sweeps
    t = min(ts)
    per_sweep_us = t * 1e3 / executed
    rows.append((m, n, o.sweeps, t, per_sweep_us))
    print(f"m={m:6d} n={n:5d} sweeps={o.sweeps:3d} dev_ms={t:8.3f} us/sweep={per_sweep_us:9.2f} "
          f"ns/step(1strip)={per_sweep_us * 1e3 / (m + 31):7.1f}", flush=True)
    plan.close()
