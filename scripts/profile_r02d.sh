# round-2 captures after the record / TMA changes (second pass: heap-cell TMA tiles) (one GPU, each command
# first run plain to exit 0):
#   1. ncu --set full of the FHCM/8 replay (heapcell_spec) and the FMSM/8
#      dataflow (fmsm_dataflow), C2, each alone on the GPU
#   2. the launch list of the bench step (gpu__time_duration per launch)
set -e
python scripts/one_solve.py c2 fhcm 8 1 > gpurun_out/r02d_plain.log 2>&1
python scripts/one_solve.py c2 fmsm 8 1 >> gpurun_out/r02d_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:heapcell_spec -c 1 \
    -o gpurun_out/r02d_fhcm8_full -f python scripts/one_solve.py c2 fhcm 8 1 > gpurun_out/r02d_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fmsm_dataflow -c 1 \
    -o gpurun_out/r02d_fmsm8_full -f python scripts/one_solve.py c2 fmsm 8 1 > gpurun_out/r02d_ncu2.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/r02d_bench_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02d_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    --no-configs > gpurun_out/r02d_ncu3.log 2>&1
