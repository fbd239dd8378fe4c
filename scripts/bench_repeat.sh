# headline repeatability: N runs of the 20-step bench (value, e2e, FSM ms in the batch)
N=${1:-4}
for i in $(seq $N); do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), d['methods']['fsm']['ms'], d['methods']['fhcm/8']['ms'])"; done
