"""Quick device timing of resident solves (development aid, not the bench)."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2")
ap.add_argument("--methods", default="fsm")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
for cname in a.configs.split(","):
    cfg = configs.CONFIGS[cname]()
    p = cfg.problem
    M = p.grid.size()
    for method in a.methods.split(","):
        sizes = [None] if method in ("fsm", "fmm") else cfg.cell_sizes
        for cs in sizes:
            cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs)) if cs else None
            try:
                plan = E.Plan(p, method, cells)
            except NotImplementedError as e:
                print(cname, method, "not implemented:", e)
                continue
            ts = []
            for _ in range(a.reps):
                o = plan.run()
                ts.append(o.device_ms)
            t0 = time.time()
            o = plan.run()
            wall = (time.time() - t0) * 1e3
            best = min(ts)
            print(f"{cname} {method:5s} cs={cs} M={M} sweeps={o.sweeps} pops={o.heap_removals} "
                  f"dev_ms={best:.3f} (all {['%.3f' % t for t in ts]}) wall_ms={wall:.2f} "
                  f"Gpts/s={M / best / 1e6:.3f} launches={o.kernel_launches} spec(hit,wait,self)={o.spec}", flush=True)
            plan.close()
