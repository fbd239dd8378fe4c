# Development aid: heap-cell device time against the number of worker CTAs.
for n in 5 10 19 37 75; do for m in hcm fhcm; do for cs in 8 16 32 64; do
  echo "ctas $n"; EIK_HC_CTAS=$n timeout 120 python scripts/one_solve.py c2 $m $cs 1
done; done; done
