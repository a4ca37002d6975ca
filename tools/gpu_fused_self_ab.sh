# fused-self (m = 1) vs plain HEMM timing, real and complex, with and without the fused tail
for cfg in "60000 3000 20 real" "42432 3000 20"; do
  TAG=plain python tools/hemm_timing.py $cfg
  TAG=fself FUSED_SELF=1 python tools/hemm_timing.py $cfg
  TAG=fself_notail CHASE_FUSED_NO_TAIL=1 FUSED_SELF=1 python tools/hemm_timing.py $cfg
done
