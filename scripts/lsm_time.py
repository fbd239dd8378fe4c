import sys, os
sys.path.insert(0, os.getcwd())
import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
for name in ("c2", "c3", "c4"):
    p = configs.CONFIGS[name]().problem
    plan = E.Plan(p, "lsm")
    best = min(plan.run().device_ms for _ in range(3))
    o = plan.run()
    print(name, "lsm ms", round(best, 2), "sweeps", o.sweeps, "updates", o.node_updates, flush=True)
    plan.close()
