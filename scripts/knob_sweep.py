"""Solo device time of one method under EIK_* knob settings.  Development aid.
usage: python scripts/knob_sweep.py CONFIG METHOD CELL_NODES KNOB=v[,KNOB=v] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1]]()
method, cs = sys.argv[2], int(sys.argv[3])
p = cfg.problem
cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs)) if cs else None
for spec in sys.argv[4:]:
    env = dict(kv.split("=") for kv in spec.split(",")) if spec != "-" else {}
    for k, v in env.items():
        os.environ[k] = v
    E.lib.eik_debug_reload_knobs()
    plan = E.Plan(p, method, cells)
    best = None
    for _ in range(3):
        o = plan.run()
        best = o if best is None or o.device_ms < best.device_ms else best
    plan.close()
    for k in env:
        del os.environ[k]
    print(f"{sys.argv[1]} {method}/{cs} {spec}: {best.device_ms:.2f} ms pops {best.heap_removals} "
          f"ctas {best.ctas} spec {best.spec}", flush=True)
