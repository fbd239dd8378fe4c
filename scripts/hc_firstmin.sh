# FHCM workers chasing their bucket's minimum (EIK_HC_FIRST_MIN rows of 32
# workers, pools up to EIK_HC_FIRST_MIN_POOL) at the batch's pools and solo
set -e
timeout 600 python -m pytest tests/test_gpu_cells.py -m gpu -x -q -k "fhcm or hcm" 2>&1 | tail -3
for fm in 0 2; do
  for cap in 6 11 24 148; do
    echo "first_min=$fm ctas=$cap"
    EIK_HC_FIRST_MIN=$fm EIK_HC_CTAS=$cap timeout 120 python scripts/one_solve.py c2 fhcm 8 3
  done
  for cs in 16 32; do EIK_HC_FIRST_MIN=$fm timeout 120 python scripts/one_solve.py c2 fhcm $cs 3; done
done
run() {
  env $1 timeout 300 python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 value', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), 'ms', round(d['ms_per_step'],1))"
}
for i in 1 2; do run EIK_HC_FIRST_MIN=0; run EIK_HC_FIRST_MIN=2; done
