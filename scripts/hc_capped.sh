# heap-cell solves on the batch's slice sizes (EIK_HC_CTAS caps the grid)
for mc in "hcm 8 11" "fhcm 8 11" "hcm 64 8" "fhcm 64 8" "hcm 16 8" "hcm 32 6"; do
  set -- $mc
  EIK_HC_CTAS=$3 timeout 120 python scripts/one_solve.py c2 $1 $2 3
done
