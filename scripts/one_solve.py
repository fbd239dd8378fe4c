"""Run one resident solve (profiling target).  Development aid.
usage: python scripts/one_solve.py CONFIG METHOD [CELL_NODES] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1]]()
method = sys.argv[2]
cs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
p = cfg.problem
cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs)) if cs else None
plan = E.Plan(p, method, cells)
for _ in range(reps):
    o = plan.run()
print(method, cs, "device_ms", round(o.device_ms, 3), "pops", o.heap_removals, flush=True)
