# list-schedule variants of the bench step, 3 runs each (value Mpts/s, ms/step, e2e)
run() { for i in 1 2 3; do env "$@" timeout 600 python bench.py --no-c5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e6,1), round(d['ms_per_step'],1), round(d['e2e']['value']/1e6,1))"; done; }
for v in ${VARIANTS:-"X=0"}; do run $v; done
