# warp-state breakdown of the FSM wavefront on config 5 (one launch)
set -e
python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/prof_c5_plain.log 2>&1
ncu --clock-control none -k regex:fsm_wavefront -c 1 --section WarpStateStats --section MemoryWorkloadAnalysis_Tables \
    --csv --page details --log-file gpurun_out/r01_fsm_c5_v5_warpstate.csv python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/prof_c5.log 2>&1
