# cell tiles by TMA vs loads (EIK_TILE_TMA): FHCM replay (cost tiles), HCM band (value + cost tiles)
for t in 0 1; do
  for cs in 8 16 32 64; do EIK_TILE_TMA=$t timeout 120 python scripts/one_solve.py c2 fhcm $cs 3; done
  for cs in 8 16 32 64; do EIK_TILE_TMA=$t timeout 120 python scripts/one_solve.py c2 hcm $cs 3; done
  EIK_TILE_TMA=$t timeout 300 python scripts/one_solve.py c4 hcm 16 2
done
