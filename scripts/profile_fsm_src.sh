# ncu source-level capture (SASS stall sampling) of the FSM wavefront on C2,
# one launch alone on the GPU; run plain first
set -e
python scripts/one_solve.py c2 fsm 0 1 > gpurun_out/fsm_src_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fsm_wavefront -c 1 \
    -o gpurun_out/fsm_src -f python scripts/one_solve.py c2 fsm 0 1 > gpurun_out/fsm_src_ncu.log 2>&1
