# slice scale / FMSM CTA sweep at the driver's step count (20 timed steps)
run() {
  env $1 timeout 300 python bench.py --steps ${2:-20} --warmup 5 --no-configs --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 K=${2:-20} value', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), 'ms', round(d['ms_per_step'],1), 'fmsm8', d['methods']['fmsm/8'].get('solo_ms'), d['methods']['fmsm/8'].get('host_ms'))"
}
for s in 0.5 0.75 1.0; do run EIK_BATCH_SMS_SCALE=$s; done
run EIK_BATCH_SMS_SCALE=1.0 3
run EIK_BATCH_SMS_SCALE=2.0 3
run "EIK_BATCH_SMS_SCALE=1.0 EIK_BATCH_FMSM_CTAS=8"
run "EIK_BATCH_SMS_SCALE=0.75 EIK_BATCH_FMSM_CTAS=8"
