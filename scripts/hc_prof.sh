set -x
for m in hcm fhcm; do for cs in 8 16 32 64; do
  timeout 120 python scripts/one_solve.py c2 $m $cs 2
  EIK_HC_PROFILE=1 timeout 120 python scripts/one_solve.py c2 $m $cs 1
  EIK_HC_PROFILE=1 EIK_HC_CTAS=1 timeout 120 python scripts/one_solve.py c2 $m $cs 1
done; done
