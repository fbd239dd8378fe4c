for pf in 0 2 4 8 4,l2 8,l2 16,l2; do echo "PF=$pf"; EIK_FSM_PF=$pf timeout 300 python scripts/fsm_bench.py c5 c2 2>&1; done
