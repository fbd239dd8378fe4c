import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
cfg = configs.config2(); p = cfg.problem
for cs in (8, 16, 32, 64):
    cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs))
    plan = E.Plan(p, "hcm", cells)
    for _ in range(3): o = plan.run()
    print("hcm", cs, "ms", round(o.device_ms, 2), "rounds", o.rounds, "pops", o.heap_removals, "sweeps", o.sweeps, flush=True)
    plan.close()
