# adaptive band: narrowing threshold sweep (solo, and the 20-step batch)
for t in 128 256 512 1024; do
  echo "== shrink $t"
  for c in "c2 hcm 8" "c2 hcm 16" "c2 hcm 64" "c3 hcm 16" "c4 hcm 16" "c4 hcm 32"; do
    EIK_HCM_BAND_SHRINK=$t timeout 200 python scripts/one_solve.py $c 2
  done
  EIK_HCM_BAND_SHRINK=$t timeout 300 python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('batch value', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1))"
done
