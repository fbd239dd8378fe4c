# Development aid: HCM device time against the first sweep that uses the vote-skip engine.
for sf in 0 1 2 3; do for cs in 8 16 32 64; do
  echo "skip_from $sf"; EIK_HC_SKIP_FROM=$sf timeout 120 python scripts/one_solve.py c2 hcm $cs 2
done; done
