# adaptive band (x1..x64 of the base) across configs
for cs in 8 16 32 64; do timeout 100 python scripts/one_solve.py c2 hcm $cs 3; done
timeout 300 python scripts/one_solve.py c3 hcm 16 2
timeout 300 python scripts/one_solve.py c3 hcm 48 2
timeout 300 python scripts/one_solve.py c4 hcm 16 2
timeout 300 python scripts/one_solve.py c4 hcm 32 2
timeout 600 python scripts/one_solve.py c5 hcm 32 2
