# FSM wavefront: trace (per strip-sweep timing, polls, computed steps) and device
# times per config; EIK_FSM_NOSKIP=1 for the variant without clean-step skipping
for v in ${VARS:-0 1}; do
  echo "=== NOSKIP=$v"
  if [ "$v" = 1 ]; then export EIK_FSM_NOSKIP=1; else unset EIK_FSM_NOSKIP; fi
  timeout 120 python scripts/fsm_trace.py gpurun_out 2>&1 | grep -E "==|k= 0|k= 1 " | cut -c1-400
  timeout 300 python scripts/fsm_bench.py ${CFGS:-c2 c3} 2>&1
done
