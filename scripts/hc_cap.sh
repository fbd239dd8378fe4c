# Development aid: heap-cell solo times against the committer's smem bucket
# capacity and worker warps per CTA.
for cap in 64 128; do for w in 2 4 8; do for m in hcm fhcm; do for cs in 8 16; do
  echo "cap $cap warps $w"; EIK_HC_HEAP_CAP=$cap EIK_HC_WARPS=$w timeout 120 python scripts/one_solve.py c2 $m $cs 2
done; done; done; done
