for v in 3 1; do for r in 1 2; do echo "LS_CONV_PX2=$v $(LS_CONV_PX2=$v python scripts/time_unet.py | tail -1)"; done; done
