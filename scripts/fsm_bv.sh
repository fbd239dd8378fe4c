for bv in 0 1 2; do echo "BV=$bv"; EIK_FSM_BV=$bv timeout 300 python scripts/fsm_bench.py c2 c3 c4 c5 2>&1; done
