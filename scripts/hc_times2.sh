for mc in "hcm 8" "fhcm 8" "hcm 16" "hcm 32" "hcm 64" "fhcm 64"; do
  set -- $mc
  timeout 120 python scripts/one_solve.py c2 $1 $2 3
done
