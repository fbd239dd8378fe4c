# FSM wavefront A/B: EIK_FSM_RING=0 (4 strips per CTA, global mailboxes) vs the default
for v in ${VARS:-1 0}; do
  echo "=== RING=$v"
  EIK_FSM_RING=$v timeout 120 python scripts/fsm_trace.py gpurun_out 2>&1 | grep -E "==|k= 0|k= 1 " | cut -c1-400
  EIK_FSM_RING=$v timeout 300 python scripts/fsm_bench.py ${CFGS:-c2 c3} 2>&1
done
