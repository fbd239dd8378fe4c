# Development aid: heap-cell device time against the SMs it holds (1 CTA per SM).
for n in 8 13 20 30 45; do for m in hcm fhcm; do for cs in 8 16 32 64; do
  echo "sms $n"; EIK_HC_CTAS=$n timeout 120 python scripts/one_solve.py c2 $m $cs 1
done; done; done
