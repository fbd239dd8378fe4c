# Development aid: K-step bench against the heap-cell slice scale and the admission order.
for sc in 1.5 2.0 2.5; do for g in 0 1; do
  echo "scale $sc guess-order $g"
  if [ $g = 1 ]; then export EIK_BATCH_GUESS_ORDER=1; else unset EIK_BATCH_GUESS_ORDER; fi
  EIK_BATCH_SMS_SCALE=$sc python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['ms_per_step'],1), round(d['single_step_ms'],1), round(d['e2e']['value']/1e6,1))"
done; done
