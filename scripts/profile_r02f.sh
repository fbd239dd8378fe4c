# round-2 captures after the FSM super-block skipping (one GPU; each command
# first run plain to exit 0):
#   1. ncu metrics of the FSM wavefront on config 5 (one launch): DRAM bytes,
#      duration, L2 bytes, fp64 pipe, warps active
#   2. ncu --set full of the FSM wavefront on config 2
#   3. the launch list of the bench step
set -e
python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/r02f_plain.log 2>&1
ncu --clock-control none -k regex:fsm_wavefront -c 1 --csv \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_bytes.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active \
    --log-file gpurun_out/r02f_fsm_c5_metrics.csv python scripts/one_solve.py c5 fsm 0 1 > gpurun_out/r02f_ncu1.log 2>&1
python scripts/one_solve.py c2 fsm 0 1 >> gpurun_out/r02f_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fsm_wavefront -c 1 \
    -o gpurun_out/r02f_fsm_c2_full -f python scripts/one_solve.py c2 fsm 0 1 > gpurun_out/r02f_ncu2.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/r02f_bench_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    --no-configs > gpurun_out/r02f_ncu3.log 2>&1
python scripts/one_solve.py c2 fhcm 8 1 >> gpurun_out/r02f_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:heapcell_spec -c 1 \
    -o gpurun_out/r02f_fhcm8_full -f python scripts/one_solve.py c2 fhcm 8 1 > gpurun_out/r02f_ncu4.log 2>&1
python scripts/fsm_trace.py gpurun_out c5 > /dev/null 2>&1
python scripts/fsm_trace_summary.py gpurun_out/trace_c5.txt > gpurun_out/r02f_fsm_c5_trace.txt
rm -f gpurun_out/trace_c5.txt
