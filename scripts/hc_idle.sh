# Development aid: heap-cell device time against the worker back-off.
for ns in 0 50 100 200 400; do for m in hcm fhcm; do for cs in 8 32; do
  echo "idle $ns"; EIK_HC_IDLE_NS=$ns timeout 120 python scripts/one_solve.py c2 $m $cs 2
done; done; done
