"""FMSM fine pass at capped CTA counts (the batch gives FMSM 16 CTAs).
Development aid.  usage: python scripts/fmsm_caps.py [cell sizes...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

cfg = configs.config2()
p = cfg.problem
for cs in [int(x) for x in sys.argv[1:]] or [8, 16, 32, 64]:
    cells = E.build_cells(p.grid, p.grid.m // cs, p.grid.m // cs)
    plan = E.Plan(p, "fmsm", cells)
    for cap in (8, 16, 32, 64, 0):
        plan.set_ctas(cap)
        best = min(plan.run().device_ms for _ in range(3))
        print(f"fmsm/{cs} ctas {cap or 'all'}: {best:.2f} ms", flush=True)
