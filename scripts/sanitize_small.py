"""Every device path on small problems -- the target of the compute-sanitizer
runs (memcheck, synccheck) recorded under profiles/.  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

p = configs.config2(129).problem
g = p.grid
jobs = [("fsm", None), ("lsm", None), ("fmm", None)]
for c in (4, 8, 16):
    cells = E.build_cells(g, c, c)
    jobs += [("fmsm", cells), ("hcm", cells), ("hcm_exact", cells), ("fhcm", cells)]
big = E.build_cells(g, 1, 1)  # one 129-node cell: the band-split, in-place engines
jobs += [("hcm_exact", big), ("fhcm", big), ("fmsm", E.build_cells(g, 2, 2))]
for method, cells in jobs:
    o = E.solve(p, method, cells)
    assert np.isfinite(o.values).all(), method
    print(method, cells.cells_x if cells else 0, o.sweeps, o.heap_removals, flush=True)
outs, _ = E.solve_batch([(p, m, c, None) for m, c in jobs[:8]])
order = E.fmm_solve(p, E.FmmOptions(record_acceptance_order=True)).acceptance_order
m5 = E.solve_multi(configs.config5(129).problem, "fsm", [0, 0])
print("batch", len(outs), "order", order.size, "multi", m5.sweeps, "ok")
