# Development aid: device time of every heap-cell configuration of the bench.
for m in hcm fhcm; do for cs in 8 16 32 64; do
  timeout 120 python scripts/one_solve.py c2 $m $cs 2
done; done
