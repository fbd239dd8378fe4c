"""HCM band scheduler: device time / pops / rounds vs the band-width scale.
Development aid.  usage: python scripts/band_sweep.py CONFIG CELL_NODES scale..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1110_6220_b200 as E  # noqa: E402
from paper_1110_6220_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1]]()
cs = int(sys.argv[2])
p = cfg.problem
cells = E.build_cells(p.grid, cfg.cells_for(cs), cfg.cells_for(cs))
for sc in sys.argv[3:]:
    os.environ["EIK_HCM_BAND"] = sc
    E.lib.eik_debug_reload_knobs()
    plan = E.Plan(p, "hcm", cells)
    best = None
    for _ in range(3):
        o = plan.run()
        best = o if best is None or o.device_ms < best.device_ms else best
    plan.close()
    print(f"{sys.argv[1]} hcm/{cs} band x{sc}: {best.device_ms:.2f} ms pops {best.heap_removals} "
          f"rounds {best.rounds} sweeps {best.sweeps} ctas {best.ctas}", flush=True)
