# ncu evidence for the FSM wavefront (kernel 1): C2 full set, C5 HBM / pipe counters.
set -e
python scripts/one_solve.py c2 fsm 0 1 > gpurun_out/prof_fsm_c2_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fsm_wavefront -c 1 \
    -o gpurun_out/r01_fsm_c2_full -f python scripts/one_solve.py c2 fsm 0 1 > gpurun_out/prof_fsm_c2.log 2>&1
python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/prof_fsm_c5_plain.log 2>&1
ncu --clock-control none -k regex:fsm_wavefront -c 1 --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --log-file gpurun_out/r01_fsm_c5_metrics.csv python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/prof_fsm_c5.log 2>&1
