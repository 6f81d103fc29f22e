for cfg in "" "LS_CONV_N256=128" "LS_CONV_N256=128 LS_CONV_MT128=2" "LS_CONV_MT128=2"; do
  for r in 1 2; do echo "[$cfg] $(env $cfg python scripts/time_unet.py 2>&1 | tail -1)"; done
done
