for mc in "hcm 8" "fhcm 8" "hcm 64" "hcm 16"; do
  set -- $mc
  timeout 120 python scripts/one_solve.py c2 $1 $2 2
  EIK_HC_PROFILE=1 timeout 120 python scripts/one_solve.py c2 $1 $2 1
done
