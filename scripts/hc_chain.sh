# Development aid: chain modes at small cells (device time, then the profile line).
for ch in 1 2; do for m in hcm fhcm; do for cs in 8 16; do
  echo "chain $ch"; EIK_HC_CHAIN=$ch timeout 120 python scripts/one_solve.py c2 $m $cs 2
  EIK_HC_CHAIN=$ch EIK_HC_PROFILE=1 timeout 120 python scripts/one_solve.py c2 $m $cs 1 2>&1 | grep "misses\|hits"
done; done; done
