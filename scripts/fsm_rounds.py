"""Sweep-by-sweep FSM (the sharded path's launches, one rank): time and result
against the single-launch solve.  usage: python scripts/fsm_rounds.py [c2|c3|c4|c5]
EIK_FSM_CONT=0: every launch evaluates every node (the behaviour before the
change bits were carried across launches)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402
from paper_1110_6220_b200.distributed import DeviceStripSweeper, strip_problem  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    p = configs.CONFIGS[name]().problem
    plan = E.Plan(p, "fsm")
    ref = np.empty(p.grid.m * p.grid.n) if name != "c5" else None
    o = plan.run(ref)
    plan.close()
    g = p.grid
    local = strip_problem(p, 0, g.n)
    sw = DeviceStripSweeper(local)
    inf_row = np.full(g.m, np.inf)
    sw.set_rows(0, 1, inf_row)
    sw.set_rows(local.grid.n - 1, 1, inf_row)
    t0 = time.time()
    k = 0
    while True:
        changed = sw.sweep(k)
        k += 1
        # a sharded run rewrites its ghost rows after every round
        sw.set_rows(0, 1, inf_row)
        sw.set_rows(local.grid.n - 1, 1, inf_row)
        if not changed:
            break
    dt = time.time() - t0
    same = None
    if ref is not None:
        out = np.empty(g.n * g.m)
        sw.get_rows(1, g.n, out)
        same = bool(np.array_equal(out.view(np.int64), ref.view(np.int64)))
    sw.close()
    print(f"{name}: single launch {o.device_ms:.1f} ms, {o.sweeps} sweeps | sweep by sweep "
          f"{k} launches in {dt * 1e3:.1f} ms wall | bitwise equal: {same}", flush=True)
