for sf in 0 1; do echo "HCM SKIP_FROM=$sf"; for cs in 8 16 32 64; do EIK_HC_SKIP_FROM=$sf timeout 120 python scripts/one_solve.py c2 hcm $cs 3; done; done
for sf in 0 1 2 100; do echo "FHCM SKIP_FROM_FAST=$sf"; for cs in 8 16 32 64; do EIK_HC_SKIP_FROM_FAST=$sf timeout 120 python scripts/one_solve.py c2 fhcm $cs 3; done; done
