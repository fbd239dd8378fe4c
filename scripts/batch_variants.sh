# Development aid: batch makespan under heap-cell launch variants.
echo "== default"; REPS=4 python scripts/batch_probe.py | grep "batch ms"
echo "== 8 warps, 1 CTA/SM"; EIK_HC_WARPS=8 EIK_HC_MIN_SMEM=120000 REPS=4 python scripts/batch_probe.py | grep "batch ms"
echo "== 4 warps, 1 CTA/SM"; EIK_HC_WARPS=4 EIK_HC_MIN_SMEM=120000 REPS=4 python scripts/batch_probe.py | grep "batch ms"
echo "== 8 warps, 1 CTA/SM solo"; for m in hcm fhcm; do for cs in 8 16 32 64; do EIK_HC_WARPS=8 EIK_HC_MIN_SMEM=120000 python scripts/one_solve.py c2 $m $cs 2; done; done
