for cs in 8 16 32 64; do timeout 120 python scripts/one_solve.py c2 fhcm $cs 3; done
EIK_HC_PROFILE=1 timeout 120 python scripts/one_solve.py c2 fhcm 8 1
