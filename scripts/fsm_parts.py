"""Strip-Jacobi partitions on one device: time / sweeps / max |u - exact GS| per part size.
usage: python scripts/fsm_parts.py CONFIG METHOD PART_ROWS..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

name, method = sys.argv[1], sys.argv[2]
p = configs.CONFIGS[name]().problem
plan = E.Plan(p, method)
M = p.grid.m * p.grid.n
u = np.empty(M)
ref = None
for pr in [0] + [int(x) for x in sys.argv[3:]]:
    plan.set_partitions(pr)
    best = None
    for _ in range(2):
        o = plan.run(u_host=u)
        best = o if best is None or o.device_ms < best.device_ms else best
    if ref is None:
        ref = u.copy()
        d = 0.0
    else:
        d = float(np.max(np.abs(u - ref)))
    print(f"{name} {method} part_rows={pr} device_ms={best.device_ms:.3f} sweeps={best.sweeps} "
          f"max|du|={d:.3e}", flush=True)
