# full ncu capture of the heap-cell replay (C2, HCM at 8-node cells, alone on the GPU)
set -e
python scripts/one_solve.py c2 hcm 8 1 > gpurun_out/prof_hcm8_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:heapcell_spec -c 1 \
    -o gpurun_out/r01_hcm8_v3_full -f python scripts/one_solve.py c2 hcm 8 1 > gpurun_out/prof_hcm8.log 2>&1
