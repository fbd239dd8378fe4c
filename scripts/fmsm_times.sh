for cs in 8 16 32 64; do timeout 120 python scripts/one_solve.py c2 fmsm $cs 3; done
bash scripts/hc_times2.sh
